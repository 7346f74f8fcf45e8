/*
 * moe_oracle.h — CPU ORACLE for the FlashDMoE MoE-layer forward (TEST INFRASTRUCTURE ONLY).
 *
 * This is a plain-C restatement of the reference's dense oracle and fused gate
 * (/root/reference/proj/include/moefabric/{config,gate,oracle,tiled_blas,layout}.hpp).
 * It exists to CHECK the CUDA product path; only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it. The product library never links it.
 *
 * Parity pinning:
 *   - bit-identical to the reference's own forward()/dense_moe_forward()/gate_forward()
 *     compiled from /root/reference by oracle/Makefile into oracle/_ref/ (tests/test_oracle_pin.py);
 *   - against the reference unit tests' known answers (tests/test_oracle_kat.py);
 *   - orc_expf_restated() matches glibc expf on every float in [-110, 0] (tests/test_expf_pin.py).
 *
 * Build: gcc -O3 -ffp-contract=off (no -march): the reference's FP32 rounding sequence
 * (separate mul and add, ascending k) must not be contracted into FMAs.
 */
#ifndef MOE_ORACLE_H
#define MOE_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_RELU = 0, ORC_GELU = 1, ORC_IDENTITY = 2 };

/* config.hpp:94-101 — C = max(1, ceil(cf*S/E - 1e-9)) in long double. */
int64_t orc_expert_capacity(int64_t tokens, int64_t experts, double cf);
/* config.hpp:104-106 */
int64_t orc_padded_capacity(int64_t capacity, int64_t tile_rows);
/* layout.hpp:106-113 */
uint64_t orc_size_L(int64_t tokens, int64_t embed, int64_t experts, int64_t tile_rows);

/* tiled_blas.hpp:58-67 / oracle.hpp:31-38 */
float orc_activation(int act, float x);

/* glibc expf restated (table algorithm, FMA variant) — used to pin the GPU softmax. */
float orc_expf_restated(float x);
/* libm expf, exported so tests compare through one ABI. */
float orc_expf_libm(float x);
void orc_expf_libm_batch(const float* x, float* y, int64_t n);
/* Exhaustive sweep of all floats with bit patterns in [lo_bits, hi_bits] (sign included):
   returns the number of mismatches between orc_expf_restated and libm expf. */
uint64_t orc_expf_sweep(uint32_t lo_bits, uint32_t hi_bits);

/*
 * gate.hpp:57-106 (gate_forward_with_capacity). A: S x H, Wg: H x E (row-major FP32).
 * Outputs: g_phi S x E; tbl_tok/tbl_w E x max(cap,1) (token -1 = empty);
 * slot_counts[E]; dropped[2*S*k] as (token, expert) pairs in emission order; *n_dropped.
 * picks_e/picks_w (nullable) S x k: per token the k picks in pick order with their weights;
 * picks_slot (nullable) S x k: slot index or -1 when capacity-dropped.
 */
void orc_gate(const float* A, const float* Wg, int64_t S, int64_t H, int64_t E, int64_t k,
              int64_t cap, float* g_phi, int64_t* tbl_tok, float* tbl_w, int64_t* slot_counts,
              int64_t* dropped, int64_t* n_dropped, int32_t* picks_e, float* picks_w,
              int32_t* picks_slot);

/*
 * oracle.hpp:44-111 (dense_moe_forward_with_capacity) for one device shard.
 * W1: E x H x D, B1: E x D, W2: E x D x H, B2: E x H (per global expert, row-major).
 * out: S x H (overwritten). threads > 1 parallelises the per-token FFN after the
 * (sequential) routing pass; every output element is computed by the identical
 * instruction sequence, so results do not depend on the thread count.
 */
void orc_dense_forward(const float* A, const float* Wg, const float* W1, const float* B1,
                       const float* W2, const float* B2, int64_t S, int64_t H, int64_t D,
                       int64_t E, int64_t k, int64_t cap, int act, float* out, int threads);

/* oracle.hpp:97-107 for the token ids rows[0..n_rows) only, given orc_gate's picks
 * (picks_slot -1 = dropped). out: n_rows x H; row r equals orc_dense_forward's row rows[r]. */
void orc_ffn_rows(const float* A, const float* W1, const float* B1, const float* W2, const float* B2,
                  int64_t H, int64_t D, int64_t k, int act, const int32_t* picks_e,
                  const int32_t* picks_slot, const float* picks_w, const int64_t* rows, int64_t n_rows,
                  float* out, int threads);

/* oracle.hpp:18-28 */
void orc_naive_matmul(const float* a, const float* b, int64_t m, int64_t k, int64_t n, float* c);

#ifdef __cplusplus
}
#endif
#endif
