import sys, numpy as np, subprocess, threading, time
sys.path.insert(0, '.')
import paper_2506_04667_b200 as fd
for v, name in ((12, "product-major, 1 SM, short"), (12 | 16, "product-major, 1 SM, 100x longer"), (12 | 16 | 32, "product-major, 148 SMs, 100x longer"), (4 | 16 | 32, "k-step-major, 148 SMs, long")):
    o = np.zeros(4, np.uint64)
    t0 = time.time()
    fd.dev_check(fd.dev_lib().fdmoe_debug_latency(2000 + v, fd._ptr(o)))
    print(f"{name:40s}: {int(o[1]):6d} cyc per chunk (12 MMAs, tensor work 768)  wall {time.time()-t0:.3f}s")
