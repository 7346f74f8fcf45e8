"""tcgen05 tf32 MMA rate (A from TMEM, N=128, 148 SMs) while 8 other warps generate converter-like noise."""
import sys, ctypes as C
sys.path.insert(0, '.')
import paper_2506_04667_b200 as fd
for mode, name in ((0, "quiet"), (1, "try_wait spinning"), (2, "LDS.128 streams"), (3, "tcgen05.st streams"), (4, "LDS + st")):
    v = C.c_double()
    fd.dev_check(fd.dev_lib().fdmoe_debug_mma_rate(0, 1 | (1 << 4) | (148 << 8) | (mode << 16), 128, 40001, C.byref(v)))
    print(f"tf32 TS N=128 148 SMs, noise {name:20s}: {v.value:7.1f} cyc/mma")
