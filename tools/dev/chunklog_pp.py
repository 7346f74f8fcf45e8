"""FP32 two-issuer per-tile timeline of CTA 0 (development build chunk log): tile cycles, accumulator wait, and the
token / A / hand-off waits summed over the tile's half-stages, per issuer warp."""
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
for dbg in (0, 29):
    os.environ["FDMOE_DEBUG"] = str(dbg)
    for _ in range(3):
        op.forward_device([x.data_ptr()], [y.data_ptr()], [st.cuda_stream])
    op.sync()
    print("debug", dbg, "kernel ms", op.last_kernel_ms())
    lg = np.zeros((512, 4), np.uint64)
    fd._check(fd.lib().fdmoe_read_chunklog(op._h, fd._ptr(lg)))
    for par in (0, 1):
        r = lg[128 * par:128 * par + 128]
        n = int((r[:, 0] > 0).sum())
        print(f" issuer {par}: {n} tiles; type, tile kcyc, acc wait, token wait, A wait, hand-off wait (kcyc):")
        for t in range(n):
            a = int(r[t, 3]) & 0xffffffff; h = int(r[t, 3]) >> 32
            print(f"   {int(r[t,0]) & 255} {(int(r[t,0]) >> 8) / 1e3:7.1f} {int(r[t,1]) / 1e3:6.1f} {int(r[t,2]) / 1e3:6.1f} {a / 1e3:6.1f} {h / 1e3:6.1f}")
