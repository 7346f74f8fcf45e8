import os, sys, numpy as np
os.environ["FDMOE_CHUNKLOG"] = "1"
sys.path.insert(0, '.')
import torch
import paper_2506_04667_b200 as fd
fd.select_library(fd._build.DEV_LIB)   # ablation bits / chunk log: development build
cfg = fd.MoeConfig(tokens_per_device=16384, embed_dim=2048, ffn_dim=2048, experts_total=128, devices=1, topk=2,
                   tile_rows=128, tile_cols=64, precision=int(sys.argv[1]) if len(sys.argv) > 1 else 0)
op = fd.Operator(cfg); op.set_weights(fd.make_model(cfg))
x = torch.from_numpy(fd.make_shards(cfg)[0]).cuda(); y = torch.empty_like(x)
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
for _ in range(3):
    op.forward_device([x.data_ptr()], [y.data_ptr()], [st.cuda_stream])
op.sync()
lg = np.zeros((512, 4), np.uint64)
fd._check(fd.lib().fdmoe_read_chunklog(op._h, fd._ptr(lg)))
lg = lg.astype(np.int64)
d = np.diff(lg[:, 0])
print("chunk period (cycles): median", np.median(d[:200]), "mean", d[:200].mean())
print("periods 60..130:", list(d[60:130]))
