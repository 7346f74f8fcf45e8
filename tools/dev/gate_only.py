import os, sys, numpy as np
sys.path.insert(0, '.')
import torch
import paper_2506_04667_b200 as fd
fd.select_library(fd._build.DEV_LIB)
S, E, prec = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
cfg = fd.MoeConfig(tokens_per_device=S, embed_dim=2048, ffn_dim=2048, experts_total=E, devices=1, topk=2,
                   tile_rows=128, tile_cols=64, precision=prec)
op = fd.Operator(cfg); op.set_weights(fd.make_model(cfg))
x = torch.from_numpy(fd.make_shards(cfg)[0]).cuda(); y = torch.empty_like(x)
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
for _ in range(3):
    op.forward_device([x.data_ptr()], [y.data_ptr()], [st.cuda_stream]); op.sync()
os.environ["FDMOE_DEBUG"] = "65536"
for _ in range(3):
    try:
        op.forward_device([x.data_ptr()], [y.data_ptr()], [st.cuda_stream]); op.sync()
    except Exception as ex:
        print("host:", str(ex)[:100])
t = op.trace(0).astype(np.float64) / 1e3
act = t[:, 23] > 0
print("kernel ms", op.last_kernel_ms(), "CTAs with gate tiles", int(act.sum()))
for i, n in ((38, "roles start"), (20, "mma par0 loop end"), (21, "mma par1 loop end"), (22, "epi folds done"), (23, "epi rows written"), (39, "epi done"), (28, "gate tc barrier")):
    v = t[act, i]
    print(f"{n:18s} min {v.min():7.1f} med {np.median(v):7.1f} max {v.max():7.1f} us")
