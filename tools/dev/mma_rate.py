import sys, ctypes as C
sys.path.insert(0, '.')
import paper_2506_04667_b200 as fd
for spin in (0, 1):
    for N in (128, 256):
        v = C.c_double()
        fd.dev_check(fd.dev_lib().fdmoe_debug_mma_rate(0, 1 | (1 << 4) | (148 << 8) | (spin << 16), N, 40001, C.byref(v)))
        print(f"148 SMs tf32 TS N={N:3d} {'+ 8 warps spinning on try_wait' if spin else 'quiet                          '}: {v.value:7.1f} cyc/mma")
