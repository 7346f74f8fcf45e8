import sys, numpy as np, ctypes as C
sys.path.insert(0, '.')
import torch
import paper_2506_04667_b200 as fd
cfg = fd.MoeConfig(tokens_per_device=1024, embed_dim=256, ffn_dim=256, experts_total=8, devices=1, topk=2)
op = fd.Operator(cfg); op.set_weights(fd.make_model(cfg))
r = op.forward(fd.make_shards(cfg))
info = op.info(); print(info)
buf = np.zeros((info["ctas_per_rank"], 8), np.uint64); n = C.c_int32()
fd._check(fd.lib().fdmoe_read_trace(op._h, 0, fd._ptr(buf), buf.size, C.byref(n)))
print(n.value); print(buf[:4]); print(buf[-2:])
