"""Quick parity of a library build: python tools/dev/parity_quick.py LIB PREC -> max_rel_error vs the oracle."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2506_04667_b200 as fd
from oracle import pyoracle as po
fd.select_library(sys.argv[1])
prec = int(sys.argv[2])
for S, E, P in ((2048, 16, 1), (512, 16, 2)):
    cfg = fd.MoeConfig(tokens_per_device=S, embed_dim=512, ffn_dim=1024, experts_total=E, devices=P, topk=2,
                       precision=prec, seed=7)
    m = fd.make_model(cfg); sh = fd.make_shards(cfg)
    op = fd.Operator(cfg); op.set_weights(m)
    r = op.forward(sh)
    info = op.info()
    want = [po.dense_forward(sh[d], m, cfg, threads=16) for d in range(P)]
    print(S, E, P, "fused", info["fused_combine"], "max_rel_error", fd.max_rel_error(r.outputs, want))
    op.close()
