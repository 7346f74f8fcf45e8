"""FP32 MMA-warp half-stage timeline of CTA 0 (development build chunk log): afull wait, issue, commit, period."""
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
    lg = np.zeros((512, 4), np.uint64)
    fd._check(fd.lib().fdmoe_read_chunklog(op._h, fd._ptr(lg)))
    lg = lg[:256].astype(np.int64)
    lg = lg[lg[:, 0] > 0]
    w, iss, com = lg[:, 1] - lg[:, 0], lg[:, 2] - lg[:, 1], lg[:, 3] - lg[:, 2]
    per = np.diff(lg[:, 0])
    sl = slice(64, 250)   # past the first tiles (gate / start-up)
    print(f"debug={dbg}: half-stages {len(lg)}; period med {np.median(per[sl]):.0f} mean {per[sl].mean():.0f}; "
          f"afull wait med {np.median(w[sl]):.0f} mean {w[sl].mean():.0f}; issue(12 MMA) med {np.median(iss[sl]):.0f} "
          f"mean {iss[sl].mean():.0f}; commit med {np.median(com[sl]):.0f}")
    print("  periods 100..140:", list(per[100:140]))
    print("  issue   100..140:", list(iss[100:140]))
    print("  wait    100..140:", list(w[100:140]))
