"""Tensor-core gate, CTA 0, per stage and issuer warp (development build chunk log; the FFN's log is overwritten
later in the launch, so the FFN is disabled here by reading the log of the gate before it: FDMOE_DEBUG unused)."""
import os, sys, numpy as np
os.environ["FDMOE_CHUNKLOG"] = "1"
sys.path.insert(0, '.')
import torch
import paper_2506_04667_b200 as fd
fd.select_library(fd._build.DEV_LIB)
S = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
E = int(sys.argv[2]) if len(sys.argv) > 2 else 128
cfg = fd.MoeConfig(tokens_per_device=S, embed_dim=2048, ffn_dim=2048, experts_total=E, devices=1, topk=2,
                   tile_rows=128, tile_cols=64, precision=0)
op = fd.Operator(cfg); op.set_weights(fd.make_model(cfg))
x = torch.from_numpy(fd.make_shards(cfg)[0]).cuda(); y = torch.empty_like(x)
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
for _ in range(3):
    op.forward_device([x.data_ptr()], [y.data_ptr()], [st.cuda_stream])
op.sync()
lg = np.zeros((512, 4), np.uint64)
fd._check(fd.lib().fdmoe_read_chunklog(op._h, fd._ptr(lg)))
for par in (0, 1):
    r = lg[384 + 64 * par:384 + 64 * par + 34].astype(np.int64)
    print(f"issuer {par}: per stage (cycles) acc wait / token-plane wait / A wait / hand-off wait + issue")
    print("  mean", r[2:32].mean(axis=0).round(0), " first rows:", r[:6].tolist())
for par in (0, 1):
    r = lg[384 + 64 * par:384 + 64 * (par + 1)].astype(np.int64)
    nz = int((r.sum(axis=1) > 0).sum())
    print(f"issuer {par}: {nz} logged stages, {r.sum() / 1e3:.1f} kcycles in the logged iterations")
tr = op.trace(0).astype(np.float64)
print(f"CTA 0 gate roles: start {tr[0, 38] / 1e3:.1f} us, epilogue done {tr[0, 39] / 1e3:.1f} us")
