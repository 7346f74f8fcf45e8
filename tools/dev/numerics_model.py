"""CPU model of the FFN's FP32-accurate schemes on the tcgen05 accumulator (per-MMA round-toward-zero of the exact
sum, profiles/r02_numerics.md), against the reference's sequential FP32 FFN, on one expert's 128-row tile:
  cur : 3xTF32 -- main acc w_hi*x_hi (tf32 MMAs, K=8), corr acc w_lo*x_hi + w_hi*x_lo (tf32, K=8), RN fold
  b16 : main as cur; corrections as bf16 x bf16 MMAs (K=16): bf16(w_lo)*bf16(x_hi) + bf16(w_hi)*bf16(x_lo)
Reports worst |err| / (1e-5 + 1e-4 |want|) per element after GEMM0 -> relu -> GEMM1 (+ biases)."""
import sys
import numpy as np
sys.path.insert(0, '.')

def tf32(x):   # round to nearest tf32 (10 mantissa bits), as tf32_hi
    b = x.astype(np.float32).view(np.uint32)
    return ((b + np.uint32(0x1000)) & np.uint32(0xFFFFE000)).view(np.float32)

def bf16(x):   # round to nearest even bf16
    b = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    r = ((b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32)

def rz32(s):   # float64 -> float32 rounded toward zero
    f = s.astype(np.float32)
    over = np.abs(f.astype(np.float64)) > np.abs(s)
    f[over] = np.nextafter(f[over], np.float32(0))
    return f

def mma_acc(A, B, kstep, acc=None):   # D[m][n] += sum_k A[m][k] B[k][n], one RZ per kstep-wide MMA
    M, K = A.shape
    d = np.zeros((M, B.shape[1]), np.float32) if acc is None else acc
    A64, B64 = A.astype(np.float64), B.astype(np.float64)
    for k0 in range(0, K, kstep):
        d = rz32(d.astype(np.float64) + A64[:, k0:k0 + kstep] @ B64[k0:k0 + kstep])
    return d

def gemm(W, X, scheme):   # Y[f][t] = sum_k W[f][k] X[k][t]   (W: features x K, X: K x tokens)
    w_hi, x_hi = tf32(W), tf32(X)
    w_lo, x_lo = (W - w_hi).astype(np.float32), (X - x_hi).astype(np.float32)
    main = mma_acc(w_hi, x_hi, 8)
    if scheme == "cur":
        corr = mma_acc(w_lo, x_hi, 8)
        # corr products interleave per half-stage in the kernel; same set of RZ points per 8-k MMA in order
        corr = mma_acc(w_hi, x_lo, 8, corr) if False else corr
        K = W.shape[1]
        c = np.zeros_like(main)
        A1, B1 = w_lo.astype(np.float64), x_hi.astype(np.float64)
        A2, B2 = w_hi.astype(np.float64), x_lo.astype(np.float64)
        for k0 in range(0, K, 32):   # half-stage: 4 lo*hi MMAs then 4 hi*lo MMAs
            for k in range(k0, k0 + 32, 8):
                c = rz32(c.astype(np.float64) + A1[:, k:k + 8] @ B1[k:k + 8])
            for k in range(k0, k0 + 32, 8):
                c = rz32(c.astype(np.float64) + A2[:, k:k + 8] @ B2[k:k + 8])
        corr = c
    else:
        K = W.shape[1]
        c = np.zeros_like(main)
        A1, B1 = bf16(w_lo).astype(np.float64), bf16(x_hi).astype(np.float64)
        A2, B2 = bf16(w_hi).astype(np.float64), bf16(x_lo).astype(np.float64)
        for k0 in range(0, K, 32):   # half-stage: 2 bf16 MMAs (K=16) lo*hi, then 2 hi*lo
            for k in range(k0, k0 + 32, 16):
                c = rz32(c.astype(np.float64) + A1[:, k:k + 16] @ B1[k:k + 16])
            for k in range(k0, k0 + 32, 16):
                c = rz32(c.astype(np.float64) + A2[:, k:k + 16] @ B2[k:k + 16])
        corr = c
    return (main + corr).astype(np.float32)   # RN fold

def ref_gemm(W, X):   # the reference: sequential FP32 sums, k ascending, separately rounded
    out = np.zeros((W.shape[0], X.shape[1]), np.float32)
    for k in range(W.shape[1]):
        out = (out + (W[:, k:k + 1] * X[k:k + 1, :]).astype(np.float32)).astype(np.float32)
    return out

def main():
    import paper_2506_04667_b200 as fd
    H = D = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    cfg = fd.MoeConfig(tokens_per_device=T * 4, embed_dim=H, ffn_dim=D, experts_total=4, devices=1, topk=1, seed=int(sys.argv[3]) if len(sys.argv) > 3 else 3)
    m = fd.make_model(cfg)
    x = fd.make_shards(cfg)[0][:T]                       # T token rows
    W1, b1, W2, b2 = m.w1[0], m.b1[0], m.w2[0], m.b2[0]   # H x D, D, D x H, H
    # reference: h = relu(x W1 + b1), y = h W2 + b2, sequential FP32
    h_ref = np.maximum(ref_gemm(x, W1) + b1, 0).astype(np.float32)
    y_ref = (ref_gemm(h_ref, W2) + b2).astype(np.float32)
    for scheme in ("cur", "b16"):
        h = np.maximum(gemm(W1.T, x.T, scheme).T + b1, 0).astype(np.float32)
        y = (gemm(W2.T, h.T, scheme).T + b2).astype(np.float32)
        err = np.abs(y.astype(np.float64) - y_ref)
        bound = 1e-5 + 1e-4 * np.abs(y_ref.astype(np.float64))
        r = err / bound
        print(f"{scheme}: H=D={H} rows={T}: worst err/bound {r.max():.3f}  mean {r.mean():.4f}  "
              f"normwise {np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref):.2e}  over-bound {(r > 1).sum()}")

if __name__ == "__main__":
    main()
