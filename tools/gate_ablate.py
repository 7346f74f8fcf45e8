"""Gate-phase timing: exact vs certified (+ ablations via FDMOE_DEBUG bits 32/64)."""
import os, sys
import numpy as np
sys.path.insert(0, '.')
import torch
import paper_2506_04667_b200 as fd
fd.select_library(fd._build.DEV_LIB)   # ablation bits / chunk log: development build
S = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
E = int(sys.argv[2]) if len(sys.argv) > 2 else 128
cfg = fd.MoeConfig(tokens_per_device=S, embed_dim=2048, ffn_dim=2048, experts_total=E, devices=1, topk=2)
op = fd.Operator(cfg); op.set_weights(fd.make_model(cfg))
x = torch.from_numpy(fd.make_shards(cfg)[0]).cuda(); y = torch.empty_like(x)
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
for exact, dbg, name in [(True, 0, "exact"), (False, 0, "certified"), (False, 32, "cert no-norm"),
                         (False, 64, "cert no-flush"), (False, 96, "cert no-norm no-flush"),
                         (False, 96 + 128, "cert no-load"), (False, 96 + 256, "cert no-math"),
                         (False, 96 + 128 + 256, "cert no-load no-math"), (True, 128, "exact no-load")]:
    os.environ["FDMOE_DEBUG"] = str(dbg)
    o = fd.ForwardOptions(exact_gate=exact)
    for _ in range(3):
        op.forward_device([x.data_ptr()], [y.data_ptr()], [st.cuda_stream], opts=o)
    op.sync()
    t = op.trace(0) / 1e3
    g = t[:, 1] - t[:, 0]
    print(f"{name:24s} kernel {op.last_kernel_ms():.3f} ms  gate phase med {np.median(g):6.1f} min {g.min():6.1f} max {g.max():6.1f} us")
os.environ.pop("FDMOE_DEBUG")
