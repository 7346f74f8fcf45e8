import sys, numpy as np
sys.path.insert(0, '.')
import paper_2506_04667_b200 as fd
for n in (1, 4, 12, 24, 48):
    o = np.zeros(4, np.uint64)
    fd.dev_check(fd.dev_lib().fdmoe_debug_latency(n, fd._ptr(o)))
    print(f"n={n:3d} MMAs: issue {int(o[0]):6d} cyc, issue->commit observed {int(o[1]):6d} cyc "
          f"(work {64*n}), 8x st.x16+wait {int(o[2])} cyc, mbar wake(2000 delay) {int(o[3])} cyc")
for v, name in ((0, "12 MMAs/chunk only"), (1, "+ tcgen05.fence::after_thread_sync"), (2, "+ tcgen05.commit"), (3, "+ fence + commit"), (4, "+ mbarrier try_wait (complete)"), (7, "fence + commit + try_wait")):
    o = np.zeros(4, np.uint64)
    fd.dev_check(fd.dev_lib().fdmoe_debug_latency(1000 + v, fd._ptr(o)))
    print(f"{name:40s}: {int(o[1]):6d} cyc per 12-MMA chunk (tensor work 768)")
