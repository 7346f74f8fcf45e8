"""Run the layer kernel N times at a given shape (driver for ncu captures)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2506_04667_b200 as fd
S = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
E = int(sys.argv[2]) if len(sys.argv) > 2 else 128
prec = int(sys.argv[3]) if len(sys.argv) > 3 else 0
n = int(sys.argv[4]) if len(sys.argv) > 4 else 4
cfg = fd.MoeConfig(tokens_per_device=S, embed_dim=2048, ffn_dim=2048, experts_total=E, devices=1, topk=2,
                   tile_rows=128, tile_cols=64, precision=prec)
op = fd.Operator(cfg); op.set_weights(fd.make_model(cfg))
x = torch.from_numpy(fd.make_shards(cfg)[0]).cuda(); y = torch.empty_like(x)
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
for _ in range(n):
    op.forward_device([x.data_ptr()], [y.data_ptr()], [st.cuda_stream])
op.sync()
print("last kernel ms", op.last_kernel_ms())
