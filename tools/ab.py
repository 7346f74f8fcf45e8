"""A/B timing of a library build: python tools/ab.py <lib.so> [prec] [S] [E] -> median layer-kernel ms at c4 shape."""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2506_04667_b200 as fd
fd.select_library(sys.argv[1])
prec = int(sys.argv[2]) if len(sys.argv) > 2 else 0
S = int(sys.argv[3]) if len(sys.argv) > 3 else 16384
E = int(sys.argv[4]) if len(sys.argv) > 4 else 128
cfg = fd.MoeConfig(tokens_per_device=S, embed_dim=2048, ffn_dim=2048, experts_total=E, devices=1, topk=2,
                   tile_rows=128, tile_cols=64, precision=prec)
op = fd.Operator(cfg); op.set_weights(fd.make_model(cfg))
x = torch.from_numpy(fd.make_shards(cfg)[0]).cuda(); y = torch.empty_like(x)
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
ms = []
for i in range(25):
    op.forward_device([x.data_ptr()], [y.data_ptr()], [st.cuda_stream]); op.sync()
    if i >= 5: ms.append(op.last_kernel_ms())
print(f"{sys.argv[1]} prec={prec} S={S} E={E}: median {np.median(ms):.4f} ms  min {np.min(ms):.4f}")
