"""Wide parity sweep (one-off measurement, not a test): many more token rows than tests/test_gpu_baseline.py's
192 per rank, at the configurations with the thinnest FP32 margins. Prints worst err / bound per rank."""
import os, sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2506_04667_b200 as fd
from oracle import pyoracle as po
if len(sys.argv) > 1:
    fd.select_library(sys.argv[1])
T = os.cpu_count() or 8
only = sys.argv[2].split(",") if len(sys.argv) > 2 else None
for name, (S, H, D, E, P, nrows) in {"c3_p4": (8192, 2048, 2048, 32, 4, 3072), "c4_p1": (16384, 2048, 2048, 128, 1, 6144),
                                     "c2": (4096, 2048, 2048, 16, 1, 4096)}.items():
    if only and name not in only:
        continue
    for seed in (0, 1):
        cfg = fd.MoeConfig(tokens_per_device=S, embed_dim=H, ffn_dim=D, experts_total=E, devices=P, topk=2, seed=seed)
        model = fd.make_model(cfg); shards = fd.make_shards(cfg)
        res = fd.forward(cfg, shards, model, fd.ForwardOptions(exact_gate=os.environ.get("EXACT_GATE") == "1"))
        for d in range(P):
            want_route = po.gate(shards[d], model.wg, cfg.topk, fd.expert_capacity(cfg))
            rows = np.arange(min(nrows, S))
            t0 = time.time()
            want = po.ffn_rows(shards[d], model, cfg, want_route, rows, threads=T).astype(np.float64)
            got = res.outputs[d][rows].astype(np.float64)
            r = np.abs(got - want) / (1e-5 + 1e-4 * np.abs(want))
            k = np.unravel_index(np.argmax(r), r.shape)
            print(f"   worst element row {rows[k[0]]} col {k[1]}: want {want[k]:.6e} got {got[k]:.6e}")
            print(f"{name} seed {seed} rank {d}: rows {len(rows)} worst err/bound {r.max():.3f} over {(r > 1).sum()} "
                  f"p99.99 {np.quantile(r, 0.9999):.3f} ({time.time() - t0:.0f} s)", flush=True)
