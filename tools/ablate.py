"""FFN-phase ablations via FDMOE_DEBUG bits, one process (weights generated once)."""
import os, sys
import numpy as np
sys.path.insert(0, '.')
import torch
import paper_2506_04667_b200 as fd
fd.select_library(fd._build.DEV_LIB)   # ablation bits / chunk log: development build
S = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
E = int(sys.argv[2]) if len(sys.argv) > 2 else 128
prec = int(sys.argv[3]) if len(sys.argv) > 3 else 0
cfg = fd.MoeConfig(tokens_per_device=S, embed_dim=2048, ffn_dim=2048, experts_total=E, devices=1, topk=2,
                   tile_rows=128, tile_cols=64, precision=prec)
op = fd.Operator(cfg); op.set_weights(fd.make_model(cfg))
x = torch.from_numpy(fd.make_shards(cfg)[0]).cuda(); y = torch.empty_like(x)
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
names = {0: "baseline", 1: "no convert/STTM", 4: "no epilogue stores",
         8: "no token TMA", 16: "no weight TMA", 24: "no TMA at all", 5: "no conv + no epi", 29: "all off"}
for d, n in names.items():
    os.environ["FDMOE_DEBUG"] = str(d)
    for _ in range(3):
        op.forward_device([x.data_ptr()], [y.data_ptr()], [st.cuda_stream])
    op.sync()
    t = op.trace(0)
    ffn = np.median(t[:, 4] - t[:, 3]) / 1e3
    cyc = ffn * 1e3 * 1.965
    w = {k: np.mean(t[:, i]) / cyc * 100 for k, i in (("mma<-x", 8), ("mma<-a", 9), ("mma<-acc", 10), ("mma<-task", 16),
         ("conv<-w", 11), ("conv<-a", 12), ("prod fetch", 17), ("epi busy", 18))}
    print(f"debug={d:2d} {n:24s} kernel {op.last_kernel_ms():.3f} ms   ffn phase {ffn:7.1f} us  tiles/CTA {np.mean(t[:, 19]):.1f}  " +
          " ".join(f"{k} {v:4.1f}%" for k, v in w.items()))
os.environ.pop("FDMOE_DEBUG")
