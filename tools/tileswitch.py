"""CTA 0's MMA-warp stage timeline (FDMOE_CHUNKLOG): steady-state stage period vs tile-switch gaps."""
import os, sys
os.environ["FDMOE_CHUNKLOG"] = "1"
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2506_04667_b200 as fd
fd.select_library(fd._build.DEV_LIB)   # ablation bits / chunk log: development build
prec = int(sys.argv[1]) if len(sys.argv) > 1 else 0
cfg = fd.MoeConfig(tokens_per_device=16384, embed_dim=2048, ffn_dim=2048, experts_total=128, devices=1, topk=2,
                   tile_rows=128, tile_cols=64, precision=prec)
op = fd.Operator(cfg); op.set_weights(fd.make_model(cfg))
x = torch.from_numpy(fd.make_shards(cfg)[0]).cuda(); y = torch.empty_like(x)
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
for _ in range(3):
    op.forward_device([x.data_ptr()], [y.data_ptr()], [st.cuda_stream])
op.sync()
lg = np.zeros((512, 4), np.uint64)
fd._check(fd.lib().fdmoe_read_chunklog(op._h, fd._ptr(lg)))
lg = lg.astype(np.int64)[:256]
lg[:, 1] &= (1 << 62) - 1
end = lg[:, 0]
per = np.diff(end)
nk = 2048 // (64 if prec == 0 else 128)   # stages per tile (2-atom stages)
is_first = (np.arange(1, 256) % nk) == 0
print(f"stages/tile {nk}: steady period median {np.median(per[~is_first]):.0f} mean {per[~is_first].mean():.0f} cyc;"
      f" tile-switch period median {np.median(per[is_first]):.0f} (n={is_first.sum()})")
iss = lg[1:, 0] - lg[1:, 2]
print(f"issue->commit median {np.median(iss):.0f}; stage start gap (prev commit -> this issue) median "
      f"{np.median(lg[1:, 2] - lg[:-1, 0]):.0f}")
print("tile-switch periods:", list(per[is_first][:8]))
full = np.zeros((512, 4), np.uint64)
fd._check(fd.lib().fdmoe_read_chunklog(op._h, fd._ptr(full)))
ep = full.astype(np.int64)[256:]
ep = ep[ep[:, 1] > 0]
for ty in (0, 1):
    e = ep[ep[:, 0] == ty]
    if len(e):
        print(f"epilogue gemm{ty} tiles {len(e)}: loop {np.median(e[:, 1]):.0f} (tmem ld+wait {np.median(e[:, 2]):.0f}) signal {np.median(e[:, 3]):.0f} cyc")
