"""Characterise tcgen05 kind::tf32 FP32 accumulation: signed error of one 128x128 tile (3xTF32 through
the layer's machinery) against the exact float64 product, for random-sign and all-positive data."""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_2506_04667_b200 as fd

for kind in ("normal", "positive"):
    for K in (256, 512, 1024, 2048, 4096):
        rng = np.random.default_rng(K)
        W = rng.standard_normal((128, K)).astype(np.float32)
        X = rng.standard_normal((128, K)).astype(np.float32)
        if kind == "positive":
            W, X = np.abs(W), np.abs(X)
        D = np.empty((128, 128), np.float32)
        fd._check(fd.lib().fdmoe_debug_gemm(0, K, fd._ptr(W), fd._ptr(X), fd._ptr(D)))
        exact = W.astype(np.float64) @ X.astype(np.float64).T
        # sequential FP32 (reference order) for comparison, on 8 rows
        seq = np.zeros((8, 128), np.float32)
        for k in range(K):
            seq = (seq + (W[:8, k:k + 1] * X[None, :, k])).astype(np.float32)
        scale = np.sqrt(np.mean(exact ** 2))
        e = (D - exact) / scale
        es = (seq - exact[:8]) / scale
        print(f"{kind:8s} K={K:5d}  tc: mean {e.mean():+.2e} rms {np.sqrt((e**2).mean()):.2e} max {np.abs(e).max():.2e}"
              f" | seq fp32: mean {es.mean():+.2e} rms {np.sqrt((es**2).mean()):.2e} max {np.abs(es).max():.2e}")
