"""tcgen05.mma tf32 (M=128, N=128, K=8, A from TMEM) rate vs operand reuse and loop structure, 148 SMs."""
import sys, ctypes as C
sys.path.insert(0, '.')
import paper_2506_04667_b200 as fd
for w in (1, 2, 4, 7):
    v = C.c_double()
    fd.dev_check(fd.dev_lib().fdmoe_debug_mma_rate(0, 1 | (w << 4) | (148 << 8), 128, 48001, C.byref(v)))
    print(f"mma_rate walk {w}: {v.value:6.1f} cyc/mma")
for m in (112, 240, 112 | 2048):
    v = C.c_double()
    fd.dev_check(fd.dev_lib().fdmoe_debug_mma_rate(16 + m, 1, 128, 4000, C.byref(v)))
    print(f"pipe mode {m}: {v.value:6.1f} cyc/mma")
