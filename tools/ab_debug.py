"""A/B of FDMOE_DEBUG bit sets on the development library, interleaved in one process:
python tools/ab_debug.py PREC S E bits[,bits...] -> median layer-kernel ms per bit set."""
import os, sys
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2506_04667_b200 as fd
fd.select_library(fd._build.DEV_LIB)
prec, S, E = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
sets = [int(b) for b in sys.argv[4].split(",")]
Hd = int(sys.argv[5]) if len(sys.argv) > 5 else 2048
Dd = int(sys.argv[6]) if len(sys.argv) > 6 else 2048
cfg = fd.MoeConfig(tokens_per_device=S, embed_dim=Hd, ffn_dim=Dd, experts_total=E, devices=1, topk=2,
                   tile_rows=128, tile_cols=64, precision=prec)
op = fd.Operator(cfg); op.set_weights(fd.make_model(cfg))
x = torch.from_numpy(fd.make_shards(cfg)[0]).cuda(); y = torch.empty_like(x)
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
ms = {b: [] for b in sets}
for rnd in range(6):
    for b in sets:
        os.environ["FDMOE_DEBUG"] = str(b)
        for i in range(6):
            op.forward_device([x.data_ptr()], [y.data_ptr()], [st.cuda_stream]); op.sync()
            if i >= 2: ms[b].append(op.last_kernel_ms())
for b in sets:
    print(f"prec={prec} S={S} E={E} debug={b:5d}: median {np.median(ms[b]):.4f} ms  min {np.min(ms[b]):.4f}")
