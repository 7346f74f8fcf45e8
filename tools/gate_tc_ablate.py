"""Tensor-core gate phase timing under ablations (development build): which stream bounds the logits."""
import os, sys
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2506_04667_b200 as fd
fd.select_library(fd._build.DEV_LIB)
cfg = fd.MoeConfig(tokens_per_device=16384, embed_dim=2048, ffn_dim=2048, experts_total=128, devices=1, topk=2,
                   tile_rows=128, tile_cols=64, precision=0)
op = fd.Operator(cfg); op.set_weights(fd.make_model(cfg))
x = torch.from_numpy(fd.make_shards(cfg)[0]).cuda(); y = torch.empty_like(x)
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
for name, d in (("base", 0), ("no Wg TMA", 512), ("no token TMA", 1024), ("no TMA", 1536), ("no epi fold", 2048),
                ("no TMA+fold", 3584), ("no convert", 1), ("no norm", 32), ("no cvt/norm/TMA/fold", 1 + 32 + 3584)):
    os.environ["FDMOE_DEBUG"] = str(d)
    tc = []
    for _ in range(5):
        op.forward_device([x.data_ptr()], [y.data_ptr()], [st.cuda_stream]); op.sync()
        t = op.trace(0) / 1e3
        tc.append(np.median(t[:, 28]))
    print(f"{name:14s} gate-tc-logits median {np.median(tc[1:]):7.1f} us   (load {np.median(t[:, 29]):7.1f}, route {np.median(t[:, 24]):7.1f})")
