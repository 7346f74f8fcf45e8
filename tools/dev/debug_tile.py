import sys, numpy as np
sys.path.insert(0, '.')
import paper_2506_04667_b200 as fd
for K in (64, 256, 512, 1024, 2048):
    rng = np.random.default_rng(K)
    A = rng.standard_normal((128, K)).astype(np.float32); B = rng.standard_normal((256, K)).astype(np.float32)
    D = np.empty((128, 256), np.float32)
    fd.dev_check(fd.dev_lib().fdmoe_debug_gemm(0, K, fd._ptr(A), fd._ptr(B), fd._ptr(D)))
    want = A.astype(np.float64) @ B.astype(np.float64).T
    f32 = (A @ B.T)  # numpy fp32 (pairwise/blocked sum)
    seq = np.zeros((128,256), np.float32)
    for k in range(K): seq = (seq + (A[:, k:k+1] * B[:, k][None, :]).astype(np.float32)).astype(np.float32)
    n = np.abs(want).max()
    print(K, "tc3xtf32 %.2e" % (np.abs(D-want).max()/n), "seqfp32 %.2e" % (np.abs(seq-want).max()/n), "np %.2e" % (np.abs(f32-want).max()/n))
