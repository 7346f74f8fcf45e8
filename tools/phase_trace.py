"""Phase breakdown of one layer launch from the device trace (per-CTA %globaltimer stamps)."""
import os, sys, json, numpy as np
sys.path.insert(0, '.')
import torch
import paper_2506_04667_b200 as fd
# per-role wait accounting is compiled into the development build only; FDMOE_PHASE_LIB=<lib.so> traces another
# build (phase stamps only: the wait columns read 0)
fd.select_library(os.environ.get("FDMOE_PHASE_LIB", fd._build.DEV_LIB))
S, E = int(sys.argv[1]) if len(sys.argv) > 1 else 16384, int(sys.argv[2]) if len(sys.argv) > 2 else 128
prec = int(sys.argv[3]) if len(sys.argv) > 3 else 0
Hd = int(sys.argv[4]) if len(sys.argv) > 4 else 2048
Dd = int(sys.argv[5]) if len(sys.argv) > 5 else 2048
cfg = fd.MoeConfig(tokens_per_device=S, embed_dim=Hd, ffn_dim=Dd, experts_total=E, devices=1, topk=2,
                   tile_rows=128, tile_cols=64, precision=prec)
op = fd.Operator(cfg); op.set_weights(fd.make_model(cfg))
x = torch.from_numpy(fd.make_shards(cfg)[0]).cuda(); y = torch.empty_like(x)
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
for _ in range(4):
    op.forward_device([x.data_ptr()], [y.data_ptr()], [st.cuda_stream]); op.sync()
tr = op.trace(0).astype(np.float64)   # ns (phase columns) / raw counters (7..19)
t = tr / 1e3   # us
names = ["start", "gate", "barrier", "dispatch", "ffn", "combine", "end"]
print("kernel ms", op.last_kernel_ms())
for i, n in enumerate(names):
    print(f"{n:9s} min {t[:, i].min():9.1f}  med {np.median(t[:, i]):9.1f}  max {t[:, i].max():9.1f} us")
for i, n in ((38, "gate-roles0"), (39, "gate-epi-end"), (28, "gate-tc-logits"), (29, "gate-load"), (30, "gate-decide"), (31, "gate-exp"), (24, "gate-route"), (25, "gate-pairs"), (26, "gate-full"), (36, "full-chains"), (37, "full-routed"), (20, "prefix"), (21, "slots"), (22, "slot-barrier"), (23, "push")):
    print(f"{n:12s} min {t[:, i].min():9.1f}  med {np.median(t[:, i]):9.1f}  max {t[:, i].max():9.1f} us")
g = t[:, 1]
worst = int(np.argmax(g))
print(f"slowest gate CTA {worst}: logits {t[worst, 24]/1:.1f} pairs {t[worst, 25]:.1f} full {t[worst, 26]:.1f} us "
      f"(full-exact tokens {int(round(t[worst, 27] * 1e3))}); median CTA: logits {np.median(t[:, 24]):.1f} "
      f"pairs {np.median(t[:, 25]):.1f} full {np.median(t[:, 26]):.1f}")
print("ffn tiles per CTA: min", int(tr[:, 7].min()), "max", int(tr[:, 7].max()), "sum", int(tr[:, 7].sum()))
raw = tr
for a, b, ca, cb, n in ((0, 3, 32, 33, "start..FFN"), (3, 4, 33, 34, "FFN"), (0, 6, 32, 35, "launch")):
    mhz = (raw[:, cb] - raw[:, ca]) / np.maximum(raw[:, b] - raw[:, a], 1) * 1e3
    print(f"effective SM clock {n:11s}: median {np.median(mhz):7.1f} MHz (min {mhz.min():.1f}, max {mhz.max():.1f})")
ffn_cyc = (t[:, 4] - t[:, 3]).mean() * 1e3 * 1.965   # ns -> cycles at max clock (approx)
for i, n in enumerate(["mma<-tokens", "mma<-weights", "mma<-acc", "conv<-wTMA", "conv<-tmemA", "prod<-wslot", "prod<-xslot", "epi<-acc"]):
    print(f"wait {n:14s} mean {tr[:, 8 + i].mean() / 1e3:9.1f} kcyc  ({100 * tr[:, 8 + i].mean() / ffn_cyc:5.1f}% of FFN phase)")
# distributed full-exact pass: the CTAs that finish it last (owner routing / late chains)
nfull = np.round(tr[:, 27]).astype(int)
print("full-exact tokens listed per CTA (nonzero):", {int(c): int(n) for c, n in enumerate(nfull) if n})
for c in np.argsort(-t[:, 37])[:4]:
    print(f"CTA {c:3d}: gate {t[c, 1]:.1f} full-chains {t[c, 36]:.1f} full-routed {t[c, 37]:.1f} "
          f"prefix {t[c, 20]:.1f} us")
