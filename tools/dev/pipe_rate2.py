"""Harness effects on the free-running FFN issue pattern (debug_pipe_kernel mode 112 = var7)."""
import sys, ctypes as C
sys.path.insert(0, '.')
import paper_2506_04667_b200 as fd
for m, n in ((112, "warp 11, 384 thr, garbage A"), (112 | 1024, "warp 11, 384 thr, valid A"),
             (112 | 256, "warp 0, 384 thr, garbage A"), (112 | 256 | 1024, "warp 0, 384 thr, valid A"),
             (112 | 256 | 512, "warp 0, 128 thr, garbage A"), (112 | 256 | 512 | 1024, "warp 0, 128 thr, valid A"),
             (1 | 1024, "corr/main, warp 11, valid A"), (3 | 1024, "corr/main + handshake, valid A"),
             (15 | 1024, "full skeleton, valid A")):
    v = C.c_double()
    fd.dev_check(fd.dev_lib().fdmoe_debug_mma_rate(16 + m, 1, 128, 4000, C.byref(v)))
    print(f"mode={m:5d} {n:36s}: {v.value:6.1f} cyc/mma")
