"""Kernel time for a list of FDMOE_DEBUG values (one process, weights generated once)."""
import os, sys
if os.environ.get("CHUNK"): os.environ["FDMOE_CHUNKLOG"] = "1"
import numpy as np
sys.path.insert(0, '.')
import torch
import paper_2506_04667_b200 as fd
fd.select_library(fd._build.DEV_LIB)   # ablation bits / chunk log: development build
prec = int(sys.argv[1])
vals = [int(v) for v in sys.argv[2].split(",")]
cfg = fd.MoeConfig(tokens_per_device=16384, embed_dim=2048, ffn_dim=2048, experts_total=128, devices=1, topk=2,
                   tile_rows=128, tile_cols=64, precision=prec)
op = fd.Operator(cfg); op.set_weights(fd.make_model(cfg))
x = torch.from_numpy(fd.make_shards(cfg)[0]).cuda(); y = torch.empty_like(x)
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
for d in vals:
    os.environ["FDMOE_DEBUG"] = str(d)
    ms = []
    for _ in range(6):
        op.forward_device([x.data_ptr()], [y.data_ptr()], [st.cuda_stream]); op.sync(); ms.append(op.last_kernel_ms())
    t = op.trace(0)
    ffn = np.median(t[:, 4] - t[:, 3]) / 1e3
    lg = np.zeros((512, 4), np.uint64)
    fd._check(fd.lib().fdmoe_read_chunklog(op._h, fd._ptr(lg)))
    lg = lg.astype(np.int64)
    done_flag = (lg[1:250, 1] >> 62) & 1
    lg[:, 1] &= (1 << 62) - 1
    per = np.diff(lg[:256, 0])[:250]
    wait = np.median(lg[1:250, 2] - lg[1:250, 1]); iss = np.median(lg[1:250, 0] - lg[1:250, 2])
    gap = np.median(lg[1:250, 1] - lg[0:249, 0])
    cv = np.median(lg[260:500], axis=0)
    print(f"prec {prec} debug={d:8d} kernel {np.median(ms[2:]):.3f} ms  ffn {ffn:7.1f} us  stage cyc med {np.median(per):6.0f} mean {per.mean():6.0f} | wait {wait:5.0f} issue {iss:5.0f} commit->next {gap:4.0f} ready-already {done_flag.mean():.2f} wait|ready {np.median((lg[1:250, 2] - lg[1:250, 1])[done_flag == 1]) if done_flag.any() else -1:5.0f} || conv: wfull {cv[0]:5.0f} lds {cv[1]:5.0f} done-wait {cv[2]:5.0f} cvt+st {cv[3]:5.0f}", flush=True)
