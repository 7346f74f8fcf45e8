"""Latency of the BASELINE.json configurations on one B200 (virtual ranks stand in for EP > 1):
c1 S=1024 H=1024 D=2048 E=8; c2 S=4096 H=D=2048 E=16; c3 S=8192 E=32 EP=2/4; c4 S=16384 E=128;
c5 S=2048/rank E=16/rank bf16 EP=1/2/4 (weak scaling). Prints one JSON line per config."""
import json, sys
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2506_04667_b200 as fd

CFGS = [
    ("c1", 1024, 1024, 2048, 8, 1, fd.Precision.fp32),
    ("c2", 4096, 2048, 2048, 16, 1, fd.Precision.fp32),
    ("c3-ep2(virtual)", 8192, 2048, 2048, 32, 2, fd.Precision.fp32),
    ("c3-ep4(virtual)", 8192, 2048, 2048, 32, 4, fd.Precision.fp32),
    ("c4", 16384, 2048, 2048, 128, 1, fd.Precision.fp32),
    ("c5-ep1", 2048, 2048, 2048, 16, 1, fd.Precision.bf16),
    ("c5-ep2(virtual)", 2048, 2048, 2048, 32, 2, fd.Precision.bf16),
    ("c5-ep4(virtual)", 2048, 2048, 2048, 64, 4, fd.Precision.bf16),
]
for name, S, H, D, E, P, prec in CFGS:
    cfg = fd.MoeConfig(tokens_per_device=S, embed_dim=H, ffn_dim=D, experts_total=E, devices=P, topk=2,
                       tile_rows=128, tile_cols=64, precision=prec)
    op = fd.Operator(cfg)
    op.set_weights(fd.make_model(cfg))
    xs = [torch.from_numpy(s).cuda() for s in fd.make_shards(cfg)]
    ys = [torch.empty_like(x) for x in xs]
    st = torch.cuda.Stream(); torch.cuda.set_stream(st)
    args = ([x.data_ptr() for x in xs], [y.data_ptr() for y in ys], [st.cuda_stream] * P)
    for _ in range(3):
        op.forward_device(*args)
    op.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    e0.record(st)
    for _ in range(n):
        op.forward_device(*args)
    e1.record(st)
    torch.cuda.synchronize()
    op.sync()
    ms = e0.elapsed_time(e1) / n
    print(json.dumps({"config": name, "tokens_per_rank": S, "H": H, "D": D, "E": E, "ranks": P,
                      "precision": "fp32" if prec == 0 else "bf16", "ms": round(ms, 4),
                      "tokens_per_s": round(S * P / (ms * 1e-3)),
                      "ctas_per_rank": op.info()["ctas_per_rank"]}), flush=True)
    op.close()
