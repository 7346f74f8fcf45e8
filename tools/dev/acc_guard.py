"""Internal precision of one tcgen05 kind::tf32 MMA (K = 8 products + accumulator), through the layer's
tile machinery (debug GEMM): sums whose exact value needs bits below the accumulator's ulp show whether
products are truncated on alignment (guard bits) and how the final rounding goes. X = 1, so
D[f] = sum_k W[f][k]; first MMA k = 0..7 (accumulator 0), second k = 8..15 (accumulator = first sum)."""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_2506_04667_b200 as fd

K = 64
W = np.zeros((128, K), np.float32)
X = np.ones((128, K), np.float32)
cases = []
def case(name, vals, expect_exact):
    f = len(cases)
    for k, v in vals:
        W[f, k] = v
    cases.append((name, f, expect_exact))
t = lambda e: np.float32(2.0 ** e)
case("1 + 7*2^-25 (one MMA)", [(0, 1.0)] + [(k, t(-25)) for k in range(1, 8)], 1 + 7 * 2.0 ** -25)
case("1 | + 8*2^-25 (acc + MMA)", [(0, 1.0)] + [(k, t(-25)) for k in range(8, 16)], 1 + 8 * 2.0 ** -25)
case("1 | + 8*2^-26 (acc + MMA)", [(0, 1.0)] + [(k, t(-26)) for k in range(8, 16)], 1 + 8 * 2.0 ** -26)
case("1 | + 8*2^-27 (acc + MMA)", [(0, 1.0)] + [(k, t(-27)) for k in range(8, 16)], 1 + 8 * 2.0 ** -27)
case("1 + 7*2^-26 (one MMA)", [(0, 1.0)] + [(k, t(-26)) for k in range(1, 8)], 1 + 7 * 2.0 ** -26)
case("1 - 7*2^-25 (one MMA)", [(0, 1.0)] + [(k, -t(-25)) for k in range(1, 8)], 1 - 7 * 2.0 ** -25)
case("1 | - 8*2^-26 (acc + MMA)", [(0, 1.0)] + [(k, -t(-26)) for k in range(8, 16)], 1 - 8 * 2.0 ** -26)
case("-1 | - 8*2^-25 (acc + MMA)", [(0, -1.0)] + [(k, -t(-25)) for k in range(8, 16)], -1 - 8 * 2.0 ** -25)
case("1 + 2^-24 (one MMA)", [(0, 1.0), (1, t(-24))], 1 + 2.0 ** -24)
case("1 + 3*2^-24 (one MMA)", [(0, 1.0), (1, t(-24)), (2, t(-23))], 1 + 3 * 2.0 ** -24)
case("2^-30*8 then +1 (small acc, big MMA)", [(k, t(-30)) for k in range(0, 8)] + [(8, 1.0)], 1 + 8 * 2.0 ** -30)
D = np.empty((128, 128), np.float32)
fd._check(fd.lib().fdmoe_debug_gemm(0, K, fd._ptr(W), fd._ptr(X), fd._ptr(D)))
for name, f, ex in cases:
    got = float(D[f, 0])
    rn = float(np.float32(ex))
    print(f"{name:34s} exact {ex:.10f}  got {got:.10f}  (got-exact)/2^-24 = {(got - ex) / 2.0 ** -24:+.2f}  "
          f"RN would be {rn:.10f}")
