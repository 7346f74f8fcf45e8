"""FFN pipeline-skeleton rates (cycles per tcgen05.mma, M=128 K=8 tf32, 148 SMs): which part of the FP32
MMA warp's protocol costs tensor throughput (debug_pipe_kernel modes, fdmoe_kernel.cu). Interleaved rounds."""
import sys, ctypes as C
import numpy as np
sys.path.insert(0, '.')
import paper_2506_04667_b200 as fd
names = {0: "one acc, A ring at 384 (the kernel's)", 1: "corr/main accumulators, A at 384 (the kernel's)",
         112: "var7: FFN order, one acc, A at 384", 128: "var8: FFN order, one acc, A at 256",
         176: "var11: corr/main, A at 256, corr at 384", 144: "var9: A at 128, D at 256",
         3: "corr/main + A-ring handshake", 15: "corr/main + A-ring + st + token ring"}
res = {m: [] for m in names}
ref, ffn2, ffn3 = [], [], []
for rnd in range(4):
    for w, lst in ((2, ffn2), (3, ffn3)):
        v = C.c_double()
        fd.dev_check(fd.dev_lib().fdmoe_debug_mma_rate(0, 1 | (w << 4) | (148 << 8), 128, 48001, C.byref(v)))
        lst.append(v.value)
    for m in names:
        v = C.c_double()
        fd.dev_check(fd.dev_lib().fdmoe_debug_mma_rate(16 + m, 1, 128, 4000, C.byref(v)))
        res[m].append(v.value)
    v = C.c_double()
    fd.dev_check(fd.dev_lib().fdmoe_debug_mma_rate(0, 1 | (1 << 4) | (148 << 8), 128, 40001, C.byref(v)))
    ref.append(v.value)
for m, n in names.items():
    print(f"mode={m:3d} {n:48s}: min {min(res[m]):6.1f} med {np.median(res[m]):6.1f}  {['%.1f' % x for x in res[m]]}")
print("mma_rate reference (N=128 walk):", ['%.1f' % x for x in ref])
print("mma_rate harness, FFN 12-pattern, A at 256:", ['%.1f' % x for x in ffn2])
print("mma_rate harness, FFN 12-pattern, A at 384:", ['%.1f' % x for x in ffn3])
