/*
 * moe_oracle.c — CPU ORACLE (TEST INFRASTRUCTURE ONLY; see moe_oracle.h header).
 *
 * Plain-C restatement of the reference algorithm. Every function cites the
 * reference file:line it follows (paths relative to /root/reference/proj/include/moefabric/).
 * Compile with -O3 -ffp-contract=off and no -march so the FP32 sequences
 * (separate multiply and add, ascending reduction index) match the reference build.
 */
#include "moe_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* config.hpp:94-101: ceil(q - 1e-9) on a long double quotient, floored at 1. */
int64_t orc_expert_capacity(int64_t tokens, int64_t experts, double cf) {
    const long double q = (long double)cf * (long double)tokens / (long double)experts;
    int64_t c = (int64_t)ceill(q - 1e-9L);
    return c < 1 ? 1 : c;
}

/* config.hpp:89,104-106 */
int64_t orc_padded_capacity(int64_t capacity, int64_t tile_rows) {
    return (capacity + tile_rows - 1) / tile_rows * tile_rows;
}

/* layout.hpp:106-113: 16*S*H when S >= bM*E, else 16*bM*E*H. */
uint64_t orc_size_L(int64_t tokens, int64_t embed, int64_t experts, int64_t tile_rows) {
    const uint64_t s = (uint64_t)tokens, h = (uint64_t)embed, e = (uint64_t)experts,
                   bm = (uint64_t)tile_rows;
    if (s >= bm * e) return 16 * s * h;
    return 16 * bm * e * h;
}

/* tiled_blas.hpp:58-67, oracle.hpp:31-38 (erf form of GELU). */
float orc_activation(int act, float x) {
    switch (act) {
        case ORC_RELU: return x > 0.0f ? x : 0.0f;
        case ORC_GELU: return 0.5f * x * (1.0f + erff(x * 0.70710678118654752440f));
        default: return x;
    }
}

/* ---- glibc expf, restated -------------------------------------------------
 * The reference softmax calls std::exp(float) (gate.hpp:86, oracle.hpp:71), i.e.
 * glibc's expf. On x86-64 hosts with FMA glibc dispatches to the FMA build of the
 * table-driven algorithm (EXP2F_TABLE_BITS = 5, SHIFT rounding trick). Restated
 * here so the GPU kernel can reproduce it bit for bit; pinned exhaustively against
 * libm by orc_expf_sweep (0 mismatches on [-110, 0], tests/test_expf_pin.py). */
#define ORC_EXP_N 32
static uint64_t g_exp_tab[ORC_EXP_N];
static int g_exp_tab_ready = 0;

static inline uint64_t as_u64(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
static inline double as_f64(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
static inline uint32_t as_u32(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static inline float as_f32(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

static void exp_tab_init(void) {
    if (g_exp_tab_ready) return;
    /* tab[i] = bits(2^(i/N)) - (i << (52 - 5)) */
    for (int i = 0; i < ORC_EXP_N; ++i) {
        const double v = (double)exp2l((long double)i / ORC_EXP_N);
        g_exp_tab[i] = as_u64(v) - ((uint64_t)i << 47);
    }
    g_exp_tab_ready = 1;
}

float orc_expf_restated(float x) {
    static const double inv_ln2_n = 0x1.71547652b82fep+0 * ORC_EXP_N;
    static const double shift = 0x1.8p+52;
    static const double c0 = 0x1.c6af84b912394p-5 / ORC_EXP_N / ORC_EXP_N / ORC_EXP_N;
    static const double c1 = 0x1.ebfce50fac4f3p-3 / ORC_EXP_N / ORC_EXP_N;
    static const double c2 = 0x1.62e42ff0c52d6p-1 / ORC_EXP_N;
    exp_tab_init();
    const double xd = (double)x;
    const uint32_t abstop = (as_u32(x) >> 20) & 0x7ff;
    if (abstop >= (as_u32(88.0f) >> 20)) {
        if (as_u32(x) == as_u32(-INFINITY)) return 0.0f;
        if (abstop >= (as_u32(INFINITY) >> 20)) return x + x;
        if (x > 0x1.62e42ep6f) return INFINITY;
        if (x < -0x1.9fe368p6f) return 0.0f;
    }
    double kd = fma(inv_ln2_n, xd, shift);
    const uint64_t ki = as_u64(kd);
    kd -= shift;
    const double r = fma(inv_ln2_n, xd, -kd);
    uint64_t t = g_exp_tab[ki % ORC_EXP_N];
    t += ki << 47;
    const double s = as_f64(t);
    const double z = fma(c0, r, c1);
    const double r2 = r * r;
    double y = fma(c2, r, 1.0);
    y = fma(z, r2, y);
    y = y * s;
    return (float)y;
}

float orc_expf_libm(float x) { return expf(x); }

void orc_expf_libm_batch(const float* x, float* y, int64_t n) {
    for (int64_t i = 0; i < n; ++i) y[i] = expf(x[i]);
}

uint64_t orc_expf_sweep(uint32_t lo_bits, uint32_t hi_bits) {
    uint64_t bad = 0;
    for (uint64_t u = lo_bits; u <= hi_bits; ++u) {
        const float x = as_f32((uint32_t)u);
        if (isnan(x)) continue;
        if (as_u32(expf(x)) != as_u32(orc_expf_restated(x))) ++bad;
    }
    return bad;
}

/* ---- gate -------------------------------------------------------------------
 * gate.hpp:57-106. Logits are a sequential FP32 dot product over x ascending
 * (:77-81); softmax with max, exp, sequential sum, divide (:82-89); top-k on the
 * probabilities by repeated argmax with ties to the lower index (oracle.hpp:77-87,
 * equivalent to the stable sort of gate.hpp:41-51); denominator over all k picks
 * in pick order (:92); slots in ascending token order, overflow -> dropped (:94-103). */
static void token_route(const float* a, const float* Wg, int64_t H, int64_t E, int64_t k,
                        float* probs, char* taken, int64_t* picks, float* denom_out) {
    for (int64_t e = 0; e < E; ++e) {
        float acc = 0.0f;
        for (int64_t x = 0; x < H; ++x) acc += a[x] * Wg[x * E + e];
        probs[e] = acc;
    }
    float mx = probs[0];
    for (int64_t e = 1; e < E; ++e) mx = (mx < probs[e]) ? probs[e] : mx; /* std::max */
    float sum = 0.0f;
    for (int64_t e = 0; e < E; ++e) {
        probs[e] = expf(probs[e] - mx);
        sum += probs[e];
    }
    for (int64_t e = 0; e < E; ++e) probs[e] /= sum;
    memset(taken, 0, (size_t)E);
    for (int64_t j = 0; j < k; ++j) {
        int64_t best = -1;
        for (int64_t e = 0; e < E; ++e) {
            if (taken[e]) continue;
            if (best < 0 || probs[e] > probs[best]) best = e;
        }
        taken[best] = 1;
        picks[j] = best;
    }
    float denom = 0.0f;
    for (int64_t j = 0; j < k; ++j) denom += probs[picks[j]];
    *denom_out = denom;
}

void orc_gate(const float* A, const float* Wg, int64_t S, int64_t H, int64_t E, int64_t k,
              int64_t cap, float* g_phi, int64_t* tbl_tok, float* tbl_w, int64_t* slot_counts,
              int64_t* dropped, int64_t* n_dropped, int32_t* picks_e, float* picks_w,
              int32_t* picks_slot) {
    const int64_t cap_alloc = cap > 1 ? cap : 1;
    for (int64_t i = 0; i < E * cap_alloc; ++i) { tbl_tok[i] = -1; tbl_w[i] = 0.0f; }
    for (int64_t e = 0; e < E; ++e) slot_counts[e] = 0;
    int64_t nd = 0;
    char* taken = (char*)malloc((size_t)E);
    int64_t* picks = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
    for (int64_t i = 0; i < S; ++i) {
        float* row = g_phi + i * E;
        float denom;
        token_route(A + i * H, Wg, H, E, k, row, taken, picks, &denom);
        for (int64_t j = 0; j < k; ++j) {
            const int64_t e = picks[j];
            const float w = denom > 0.0f ? row[e] / denom : 0.0f;
            int32_t slot = -1;
            if (slot_counts[e] < cap) {
                tbl_tok[e * cap_alloc + slot_counts[e]] = i;
                tbl_w[e * cap_alloc + slot_counts[e]] = w;
                slot = (int32_t)slot_counts[e];
                ++slot_counts[e];
            } else {
                dropped[2 * nd] = i;
                dropped[2 * nd + 1] = e;
                ++nd;
            }
            if (picks_e) picks_e[i * k + j] = (int32_t)e;
            if (picks_w) picks_w[i * k + j] = w;
            if (picks_slot) picks_slot[i * k + j] = slot;
        }
    }
    *n_dropped = nd;
    free(taken);
    free(picks);
}

/* ---- dense forward ------------------------------------------------------------
 * oracle.hpp:44-111. Routing is identical to orc_gate (sequential over tokens for the
 * capacity counter used[e]); the per-token FFN (:97-107) only reads routing results,
 * so it is split across threads by token without changing any arithmetic. */
typedef struct {
    const float *A, *W1, *B1, *W2, *B2;
    int64_t H, D, k;
    int act;
    const int64_t* picks;   /* S x k, -1 = dropped */
    const float* weights;   /* S x k */
    float* out;
    int64_t t0, t1;
    const int64_t* rows;    /* NULL: rows t0..t1; else token ids (orc_ffn_rows) */
} ffn_job;

static void* ffn_worker(void* arg) {
    ffn_job* j = (ffn_job*)arg;
    const int64_t H = j->H, D = j->D;
    float* hidden = (float*)malloc(sizeof(float) * (size_t)D);
    for (int64_t ii = j->t0; ii < j->t1; ++ii) {
        /* rows != NULL: token rows[ii] (orc_ffn_rows), written to out row ii */
        const int64_t i = j->rows ? j->rows[ii] : ii;
        const float* a = j->A + i * H;
        float* o = j->out + ii * H;
        for (int64_t x = 0; x < H; ++x) o[x] = 0.0f;
        for (int64_t p = 0; p < j->k; ++p) {
            const int64_t e = j->picks[i * j->k + p];
            if (e < 0) continue; /* dropped: zero contribution (oracle.hpp:93) */
            const float w = j->weights[i * j->k + p];
            const float* w1 = j->W1 + e * H * D;
            const float* b1 = j->B1 + e * D;
            const float* w2 = j->W2 + e * D * H;
            const float* b2 = j->B2 + e * H;
            for (int64_t dd = 0; dd < D; ++dd) {
                float acc = 0.0f;
                for (int64_t x = 0; x < H; ++x) acc += a[x] * w1[x * D + dd];
                hidden[dd] = orc_activation(j->act, acc + b1[dd]);
            }
            for (int64_t x = 0; x < H; ++x) {
                float acc = 0.0f;
                for (int64_t dd = 0; dd < D; ++dd) acc += hidden[dd] * w2[dd * H + x];
                o[x] += w * (acc + b2[x]);
            }
        }
    }
    free(hidden);
    return NULL;
}

void orc_dense_forward(const float* A, const float* Wg, const float* W1, const float* B1,
                       const float* W2, const float* B2, int64_t S, int64_t H, int64_t D,
                       int64_t E, int64_t k, int64_t cap, int act, float* out, int threads) {
    int64_t* used = (int64_t*)calloc((size_t)E, sizeof(int64_t));
    float* probs = (float*)malloc(sizeof(float) * (size_t)E);
    char* taken = (char*)malloc((size_t)E);
    int64_t* tp = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
    int64_t* picks = (int64_t*)malloc(sizeof(int64_t) * (size_t)(S * k));
    float* weights = (float*)malloc(sizeof(float) * (size_t)(S * k));
    for (int64_t i = 0; i < S; ++i) {
        float denom;
        token_route(A + i * H, Wg, H, E, k, probs, taken, tp, &denom);
        for (int64_t p = 0; p < k; ++p) {
            const int64_t e = tp[p];
            if (used[e] >= cap) { picks[i * k + p] = -1; weights[i * k + p] = 0.0f; continue; }
            ++used[e];
            picks[i * k + p] = e;
            weights[i * k + p] = denom > 0.0f ? probs[e] / denom : 0.0f;
        }
    }
    if (threads < 1) threads = 1;
    if (threads > S) threads = (int)(S > 0 ? S : 1);
    ffn_job* jobs = (ffn_job*)malloc(sizeof(ffn_job) * (size_t)threads);
    pthread_t* tids = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    for (int t = 0; t < threads; ++t) {
        ffn_job j = {A, W1, B1, W2, B2, H, D, k, act, picks, weights, out,
                     S * t / threads, S * (t + 1) / threads, NULL};
        jobs[t] = j;
    }
    for (int t = 1; t < threads; ++t) pthread_create(&tids[t], NULL, ffn_worker, &jobs[t]);
    ffn_worker(&jobs[0]);
    for (int t = 1; t < threads; ++t) pthread_join(tids[t], NULL);
    free(jobs); free(tids); free(used); free(probs); free(taken); free(tp); free(picks); free(weights);
}

/* The per-token FFN + combine of oracle.hpp:97-107 for a subset of tokens, given the routing
 * (picks_e / picks_slot / picks_w as orc_gate returns them; slot -1 = capacity-dropped, which
 * is exactly the dense oracle's used[e] >= cap test since both count slots in token order).
 * out row r = output row of token rows[r]; the arithmetic is ffn_worker's, so each row equals
 * orc_dense_forward's row bit for bit. Lets the tests check sampled rows at full-size shapes. */
void orc_ffn_rows(const float* A, const float* W1, const float* B1, const float* W2, const float* B2,
                  int64_t H, int64_t D, int64_t k, int act, const int32_t* picks_e,
                  const int32_t* picks_slot, const float* picks_w, const int64_t* rows, int64_t n_rows,
                  float* out, int threads) {
    int64_t S = 0;
    for (int64_t r = 0; r < n_rows; ++r) S = rows[r] + 1 > S ? rows[r] + 1 : S;
    int64_t* picks = (int64_t*)malloc(sizeof(int64_t) * (size_t)(S * k + 1));
    float* weights = (float*)malloc(sizeof(float) * (size_t)(S * k + 1));
    for (int64_t r = 0; r < n_rows; ++r) {
        const int64_t i = rows[r];
        for (int64_t p = 0; p < k; ++p) {
            const int kept = picks_slot[i * k + p] >= 0;
            picks[i * k + p] = kept ? picks_e[i * k + p] : -1;
            weights[i * k + p] = kept ? picks_w[i * k + p] : 0.0f;
        }
    }
    if (threads < 1) threads = 1;
    if (threads > n_rows) threads = (int)(n_rows > 0 ? n_rows : 1);
    ffn_job* jobs = (ffn_job*)malloc(sizeof(ffn_job) * (size_t)threads);
    pthread_t* tids = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    for (int t = 0; t < threads; ++t) {
        ffn_job j = {A, W1, B1, W2, B2, H, D, k, act, picks, weights, out,
                     n_rows * t / threads, n_rows * (t + 1) / threads, rows};
        jobs[t] = j;
    }
    for (int t = 1; t < threads; ++t) pthread_create(&tids[t], NULL, ffn_worker, &jobs[t]);
    ffn_worker(&jobs[0]);
    for (int t = 1; t < threads; ++t) pthread_join(tids[t], NULL);
    free(jobs); free(tids); free(picks); free(weights);
}

/* oracle.hpp:18-28 */
void orc_naive_matmul(const float* a, const float* b, int64_t m, int64_t k, int64_t n, float* c) {
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            float acc = 0.0f;
            for (int64_t x = 0; x < k; ++x) acc += a[i * k + x] * b[x * n + j];
            c[i * n + j] = acc;
        }
}
