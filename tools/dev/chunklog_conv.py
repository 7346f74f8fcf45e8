"""FP32 FFN converter timeline, CTA 0 warp 0 (development build chunk log rows 320..383), per half-stage."""
import os, sys, numpy as np
os.environ["FDMOE_CHUNKLOG"] = "1"
sys.path.insert(0, '.')
import torch
import paper_2506_04667_b200 as fd
fd.select_library(fd._build.DEV_LIB)
cfg = fd.MoeConfig(tokens_per_device=16384, embed_dim=2048, ffn_dim=2048, experts_total=128, devices=1, topk=2,
                   tile_rows=128, tile_cols=64, precision=0)
op = fd.Operator(cfg); op.set_weights(fd.make_model(cfg))
x = torch.from_numpy(fd.make_shards(cfg)[0]).cuda(); y = torch.empty_like(x)
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
for _ in range(3):
    op.forward_device([x.data_ptr()], [y.data_ptr()], [st.cuda_stream])
op.sync()
lg = np.zeros((512, 4), np.uint64)
fd._check(fd.lib().fdmoe_read_chunklog(op._h, fd._ptr(lg)))
r = lg[320:384].astype(np.int64)
print("per half-stage (cycles): weight-stage wait, A-slot wait, convert+store+arrive, period")
per = np.diff(r[:, 3])
for i in range(8, 40):
    print(f"  {r[i,0]:6d} {r[i,1]:6d} {r[i,2]:6d} {per[i]:6d}")
print("mean", r[8:60, :3].mean(axis=0).round(0), "period", per[8:60].mean().round(0))
