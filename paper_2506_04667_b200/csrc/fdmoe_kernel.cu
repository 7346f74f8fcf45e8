// fdmoe_kernel.cu — the FlashDMoE MoE-layer forward as ONE persistent sm_100a kernel
// per GPU. Phases inside the single launch:
//
//   1. exact gate        logits (sequential FP32, as gate.hpp:77-81), softmax with a
//                        bit-exact restatement of glibc expf (gate.hpp:82-89), top-k on
//                        probabilities with lower-index tie-break (gate.hpp:41-51, 91),
//                        combine weights over all k picks (gate.hpp:92-95)
//      -- rank-local grid barrier (slot assignment needs every token's picks) --
//   2. slots + dispatch  capacity slots in ascending token order (gate.hpp:94-103) via
//                        per-CTA prefix counts; each kept row is pushed with 16-byte
//                        stores straight into the owning rank's receive buffer (peer
//                        memory over NVLink, or local), tf32 hi/lo-split or bf16; the
//                        last CTA to finish a packet publishes a release.sys signal
//                        carrying the row count (zero-row packets signal too,
//                        runtime.hpp:328-331)
//   3. expert FFN        tile queue (one atomic head per rank): warp 10 waits for the
//                        packet signals / GEMM0 row-tile counters, then TMA-streams
//                        operands into a smem ring; warps 0-3 split the weights into
//                        tf32 hi/lo TMEM operands; warp 11 issues tcgen05.mma into
//                        double-buffered TMEM accumulators; warps 4-7 drain TMEM:
//                        GEMM0 epilogue = +b1, activation, split -> C1 scratch;
//                        GEMM1 epilogue = +b2, rows stored directly into the ORIGIN
//                        rank's combine buffer + per-tile release.sys signal
//                        (runtime.hpp:652-699, pgas.hpp:99-113)
//   4. combine           per token, O = sum over kept picks in pick order of w * y
//                        (oracle.hpp:102-107, tiled_blas.hpp:125-135)
#include <cuda_bf16.h>
#include <cstdint>

#include "fdmoe_device.cuh"

namespace fdmoe {

// ---------------------------------------------------------------- glibc expf
// Table-driven expf of glibc (EXP2F_TABLE_BITS = 5), FMA build — restated in
// oracle/moe_oracle.c:orc_expf_restated and pinned against libm on every float in
// [-110, 0]. Explicit __fma_rn/__dmul_rn/__dadd_rn so nvcc cannot re-associate.
__device__ __constant__ unsigned long long c_exp_tab[32] = {
    0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull,
    0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull,
    0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull,
    0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull,
    0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull,
    0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull,
    0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull,
    0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull,
};

// `tab` = the 32-entry table staged in shared memory (c_exp_tab copied by the kernel prologue): the
// per-lane indices diverge, and divergent __constant__ loads serialise up to 32-way.
__device__ __forceinline__ float expf_glibc(float x, const unsigned long long* __restrict__ tab) {
    const double inv_ln2_n = 0x1.71547652b82fep+0 * 32.0;
    const double shift = 0x1.8p+52;
    const double c0 = 0x1.c6af84b912394p-5 / 32.0 / 32.0 / 32.0;
    const double c1 = 0x1.ebfce50fac4f3p-3 / 32.0 / 32.0;
    const double c2 = 0x1.62e42ff0c52d6p-1 / 32.0;
    const uint32_t ux = __float_as_uint(x);
    const uint32_t abstop = (ux >> 20) & 0x7ff;
    if (abstop >= (0x42b00000u >> 20)) {                    // |x| >= 88 or NaN
        if (ux == 0xff800000u) return 0.0f;                 // -inf
        if (abstop >= (0x7f800000u >> 20)) return x + x;    // inf / nan
        if (x > 0x1.62e42ep6f) return __int_as_float(0x7f800000);
        if (x < -0x1.9fe368p6f) return 0.0f;
    }
    const double xd = (double)x;
    double kd = __fma_rn(inv_ln2_n, xd, shift);
    const unsigned long long ki = (unsigned long long)__double_as_longlong(kd);
    kd = __dsub_rn(kd, shift);
    const double r = __fma_rn(inv_ln2_n, xd, -kd);
    unsigned long long t = tab[ki & 31ull];
    t += ki << 47;
    const double s = __longlong_as_double((long long)t);
    const double z = __fma_rn(c0, r, c1);
    const double r2 = __dmul_rn(r, r);
    double y = __fma_rn(c2, r, 1.0);
    y = __fma_rn(z, r2, y);
    y = __dmul_rn(y, s);
    return __double2float_rn(y);
}

// tiled_blas.hpp:58-67 (erf form of GELU)
__device__ __forceinline__ float activation(int act, float x) {
    if (act == 0) return x > 0.0f ? x : 0.0f;
    if (act == 1) return 0.5f * x * (1.0f + erff(x * 0.70710678118654752440f));
    return x;
}

// tf32 "hi" part rounded to nearest (ties away), so |lo| <= 2^-11 |x| and x - hi is exact in FP32.
__device__ __forceinline__ float tf32_hi(float x) {
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
// Two floats as a bf16x2 word (round to nearest even): the low half holds the even-k element.
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
    __nv_bfloat162 p = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&p);
}
// FFN FP32-accurate operand format (round 2, "tf32 main + bf16 corrections"): x = x_hi + x_lo with x_hi = tf32(x)
// (round to nearest) and x_lo exact. The main products w_hi*x_hi run as kind::tf32 MMAs (exact products); the two
// correction products w_lo*x_hi + w_hi*x_lo, 2^-11 smaller, run as kind::f16 bf16 x bf16 MMAs on bf16(w_lo),
// bf16(x_hi), bf16(w_hi), bf16(x_lo): one K=16 MMA does the work of two K=8 tf32 ones, so a 32-k half-stage is
// 4 tf32 + 4 bf16 MMAs (512 tensor cycles) instead of 12 tf32 (768). Each bf16 product is within 2^-20 |w||x| of
// the exact correction product (bf16 keeps 8 of the operand's bits), below the tf32 main accumulator's per-MMA
// truncation (profiles/r02_numerics.md, tools/dev/numerics_model.py). Planes per 32-k atom (128 bytes per row):
//   plane 0: x_hi as tf32 (FP32 words)
//   plane 1: bf16(x_hi[k0..31]) (64 bytes) | bf16(x_lo[k0..31]) (64 bytes)
// and the TMEM weight half-stage: cols [0,32) w_hi tf32, [32,48) bf16x2(w_lo), [48,64) bf16x2(w_hi).
// The tensor-core gate keeps all-tf32 corrections (its certificate, k1_tc, is derived for them).
constexpr bool kCorrBf16 = true;
// FFN FP32 main accumulation split over K into the two TMEM main buffers (gemm_mma_fp32_pp / gemm_epilogue)
#ifdef FDMOE_NO_SPLITK
constexpr bool kSplitK = false;
#else
constexpr bool kSplitK = true;
#endif

// ---------------------------------------------------------------- error / watchdog
__device__ __noinline__ void raise_error(const LaunchParams& P, const RankCtx& R, uint32_t code, uint32_t where,
                                         uint32_t a, uint32_t b) {
    if (atomicCAS(R.err, 0u, code) == 0u) {
        R.err[1] = where;
        R.err[2] = a;
        R.err[3] = b;
    }
    atomicExch(P.abort_flag, 1u);
    __threadfence_system();
}

// Spin until *flag carries this epoch; returns the low 32 bits (count) or -1 on abort/timeout.
__device__ __forceinline__ int64_t wait_epoch_flag(const LaunchParams& P, const RankCtx& R,
                                                   const unsigned long long* flag, uint32_t where) {
    uint64_t v = ld_acquire_sys(flag);
    if ((uint32_t)(v >> 32) == P.epoch) return (int64_t)(uint32_t)v;
    const uint64_t t0 = globaltimer();
    uint32_t n = 0;
    while (true) {
        v = ld_acquire_sys(flag);
        if ((uint32_t)(v >> 32) == P.epoch) return (int64_t)(uint32_t)v;
        if ((++n & 255u) == 0) {
            if (ld_volatile_u32(P.abort_flag)) return -1;
            if (globaltimer() - t0 > P.budget_ns) {
                raise_error(P, R, kErrTimeout, where, (uint32_t)(v >> 32), (uint32_t)v);
                return -1;
            }
        }
    }
}

__device__ __forceinline__ bool wait_counter(const LaunchParams& P, const RankCtx& R, const uint32_t* ctr,
                                             uint32_t target, uint32_t where) {
    if (ld_acquire_gpu_u32(ctr) >= target) return true;
    const uint64_t t0 = globaltimer();
    uint32_t n = 0;
    while (ld_acquire_gpu_u32(ctr) < target) {
        if ((++n & 255u) == 0) {
            if (ld_volatile_u32(P.abort_flag)) return false;
            if (globaltimer() - t0 > P.budget_ns) {
                raise_error(P, R, kErrTimeout, where, target, ld_volatile_u32(ctr));
                return false;
            }
        }
    }
    return true;
}

__device__ __forceinline__ bool wait_counter_eq(const LaunchParams& P, const RankCtx& R, const uint32_t* ctr,
                                                uint32_t target, uint32_t where) {
    if (ld_acquire_gpu_u32(ctr) == target) return true;
    const uint64_t t0 = globaltimer();
    uint32_t n = 0;
    while (ld_acquire_gpu_u32(ctr) != target) {
        if ((++n & 255u) == 0) {
            if (ld_volatile_u32(P.abort_flag)) return false;
            if (globaltimer() - t0 > P.budget_ns) {
                raise_error(P, R, kErrTimeout, where, target, ld_volatile_u32(ctr));
                return false;
            }
        }
    }
    return true;
}

// Rank-local grid barrier over the co-resident CTAs of one rank (cooperative launch).
// The counter is monotonic across launches; `gen` is this barrier's global index.
__device__ bool rank_barrier(const LaunchParams& P, const RankCtx& R, unsigned long long gen) {
    __shared__ int s_ok;
    __syncthreads();
    if (threadIdx.x == 0) {
        s_ok = 1;
        __threadfence();
        atomicAdd(R.bar, 1ull);
        const unsigned long long target = (gen + 1ull) * (unsigned long long)P.ctas_per_rank;
        const uint64_t t0 = globaltimer();
        uint32_t n = 0;
        while (ld_acquire_gpu_u64(R.bar) < target) {
            if ((++n & 255u) == 0) {
                if (ld_volatile_u32(P.abort_flag)) { s_ok = 0; break; }
                if (globaltimer() - t0 > P.budget_ns) {
                    raise_error(P, R, kErrTimeout, 100, (uint32_t)target, 0);
                    s_ok = 0;
                    break;
                }
            }
        }
    }
    __syncthreads();
    return s_ok != 0;
}

// Device event log (fdmoe_read_events; the reference's TraceBuffer::emit, trace.hpp:79-96).
__device__ __forceinline__ void emit_event(const LaunchParams& P, const RankCtx& R, int kind, int cta, int type,
                                           uint64_t t0, uint64_t t1, int src, int expert, int rb, int cb, int peer,
                                           long long value) {
    if (!P.trace_events) return;
    const uint32_t i = atomicAdd(R.ev_ctr, 1u);
    if (i >= R.ev_cap) return;
    DevEvent e;
    e.t0 = t0; e.t1 = t1; e.kind = kind; e.cta = cta; e.type = type; e.src = src; e.expert = expert;
    e.rb = rb; e.cb = cb; e.peer = peer; e.value = value;
    R.ev[i] = e;
}

// Group barrier over every CTA of every rank (ScheduleMode::sequential's SpinBarrier,
// runtime.hpp:175-198, 885-908): rank-local barrier, then CTA 0 of each rank publishes an
// epoch-tagged arrival into every peer's gbar[id][rank] (st.release.sys over NVLink) and waits
// for all P arrivals in its own heap; a second rank-local barrier releases the rank's CTAs.
// Arrival words carry the epoch; `>=` tolerates a peer that has already moved to the next launch.
__device__ bool group_barrier(const LaunchParams& P, const RankCtx& R, unsigned long long gen, int id, int cta) {
    if (!rank_barrier(P, R, gen)) return false;
    __shared__ int s_gok;
    if (threadIdx.x == 0) {
        s_gok = 1;
        const uint64_t t0 = globaltimer();
        if (cta == 0) {
            emit_event(P, R, kEvBarrierEnter, cta, 0, t0, 0, -1, -1, -1, -1, -1, id);
            __threadfence_system();
            for (int q = 0; q < P.P; ++q) {
                unsigned long long* f =
                    reinterpret_cast<unsigned long long*>(R.peer_heap[q] + R.hl.gbar) + (size_t)id * P.P + R.rank;
                st_release_sys(f, ((uint64_t)P.epoch << 32) | 1u);
            }
            const unsigned long long* mine =
                reinterpret_cast<const unsigned long long*>(R.peer_heap[R.rank] + R.hl.gbar) + (size_t)id * P.P;
            uint32_t n = 0;
            for (int q = 0; q < P.P && s_gok; ++q) {
                while ((uint32_t)(ld_acquire_sys(mine + q) >> 32) < P.epoch) {
                    if ((++n & 255u) == 0) {
                        if (ld_volatile_u32(P.abort_flag)) { s_gok = 0; break; }
                        if (globaltimer() - t0 > P.budget_ns) {
                            raise_error(P, R, kErrTimeout, 110 + id, (uint32_t)q, 0);
                            s_gok = 0;
                            break;
                        }
                    }
                }
            }
            emit_event(P, R, kEvBarrierExit, cta, 0, globaltimer(), 0, -1, -1, -1, -1, -1, id);
        }
    }
    __syncthreads();
    const bool ok = s_gok != 0;
    if (!rank_barrier(P, R, gen + 1)) return false;
    return ok;
}

// ================================================================ phase 1: gate
// Each CTA owns a contiguous, balanced token range (its gate blocks [b0, b1)), processed in
// sub-tiles of <= gate_sub(Ep) tokens (120 at E <= 128); K streams through a 3-stage cp.async ring
//   sA[stage][sub][36]  token rows (32 K values + 4 pad floats: conflict-free LDS.128)
//   sW[stage][32][Ep]   Wg rows
// and every thread owns a 5-token x 8-expert tile of logits (one pass, all 384 threads busy).
//
// Two ways to get the reference's routing (gate.hpp:57-106):
//  * exact (ForwardOptions::exact_gate): logits as the reference computes them — FP32 sequential
//    dot products over x ascending, multiply and add rounded separately (gate.hpp:77-81 built
//    -ffp-contract=off) — then max / glibc expf / sequential sum / divide / top-k: G_phi, weights
//    and picks bit-identical.
//  * certified (default): one FFMA per MAC, and a rigorous per-token bound on |z~_e - z_ref_e|:
//    both chains are sequential sums, whose error is <= u * sum_i |partial_i| (Higham, Accuracy and
//    Stability, eq. 4.3). Partials inside a 32-term chunk are bounded by the chunk-start partial plus
//    the chunk's |products|, so with Sab = sum over chunk ends of |z~ partial| (one FADD per chunk)
//        beta_e = u' * (64 * Sab + k1 * |a| |w_e|),   k1 = 66 + 2H gamma_{H+1}
//    (u' = 2^-24 * 1.001; the k1 term covers product rounding and the chains' mutual distance).
//    Typical beta ~ 3e-4 for unit-scale logits at H = 2048 — 40x tighter than gamma_H |a||w|.
//    Per token: with intervals [z~ - beta, z~ + beta], experts whose upper bound is below the k-th
//    largest lower bound (less a margin covering expf/divide rounding) are provably not picked. If
//    exactly k candidates remain and their order is separated, the reference's picks, order, slots
//    and drops are proven identical. Otherwise the candidates (<= 8) get their EXACT reference
//    logits (a separately-rounded chain per (token, expert) pair, staged through smem), and the
//    picks are decided on exact values when their gaps exceed the rounding of expf/divide; tokens
//    with ties or near-ties fall back to the full exact path. G_phi and combine weights of
//    non-full-exact tokens derive from z~ (relative error ~1e-6: tolerance, not bits).
constexpr int kGateTT = 5;                  // tokens per thread tile
constexpr int kGateTE = 8;                  // experts per thread tile
constexpr int kGateSubMax = 120;
constexpr int kGateStages = 3;
constexpr int kGateApitch = kGateKC + 4;
constexpr int kGateMaxCand = 8;             // candidate experts per token for the pair pass
constexpr int kGatePairCap = 256;           // (token, expert) pairs per sub-tile
constexpr int kGatePairBatch = 16;          // pairs per smem-staged batch (one thread each)
constexpr int kGatePairX = 256;             // x-chunk of the pair pass
constexpr int kGatePairPitch = 2 * kGatePairX + 4;
__host__ __device__ constexpr int gate_sub(int Ep) {
    return kGateTT * (kThreads / (Ep / kGateTE)) < kGateSubMax ? kGateTT * (kThreads / (Ep / kGateTE)) : kGateSubMax;
}
__host__ __device__ constexpr int gate_region_floats(int Ep) {
    return gate_sub(Ep) * Ep + kGateStages * gate_sub(Ep) * kGateApitch + kGateStages * kGateKC * Ep;
}
constexpr int gate_region_max() {
    int m = 0;
    for (int Ep = 8; Ep <= kMaxExperts; Ep += 8) m = gate_region_floats(Ep) > m ? gate_region_floats(Ep) : m;
    return m;
}
constexpr int kGateRegionFloats = gate_region_max();
static_assert(kGateSubMax * 129 + 2 * kGatePairBatch * kGatePairPitch <= kGateRegionFloats, "pair buffer fits");
constexpr int kGateSmemBytes = ((kGateRegionFloats * 4 + 15) & ~15) + kMaxExperts * 4 /*sCnt*/ + kGateSubMax * (4 + 8 + 4 + 4 + 4) +
                               kGatePairCap * 12 + 16;
static_assert(kGateTok <= 32, "slot assignment maps one gate block onto one warp");

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(valid ? 16 : 0)
                 : "memory");
}
// same, with an L2 cache-policy hint (the gate's token rows are read again by the row push ~100 us later)
__device__ __forceinline__ void cp_async16_hint(void* dst, const void* src, uint64_t policy) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "l"(policy)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void gate_token_range(const LaunchParams& P, int cta, int& tokA, int& tokB, int& b0,
                                                 int& b1) {
    const int nblk = (P.S + kGateTok - 1) / kGateTok;
    b0 = (int)((long long)nblk * cta / P.ctas_per_rank);
    b1 = (int)((long long)nblk * (cta + 1) / P.ctas_per_rank);
    tokA = b0 * kGateTok;
    tokB = min(P.S, b1 * kGateTok);
}

struct GateSmem {
    float* sL;       // [sub][Ep] logits -> exps
    float* sA;       // [stages][sub][36]
    float* sW;       // [stages][32][Ep]
    float* sPair;    // [2][16][kGatePairPitch] pair-pass staging (aliases sA/sW, never sL)
    int* sCnt;       // [Ep] CTA-level pick counts
    float* sSab;     // [sub] max over experts of sum |chunk-end partial|
    double* sNa;     // [sub] |a|^2
    int* sTP0;       // [sub] first pair of token t
    int* sTNC;       // [sub] candidate count of token t (0: routed or full-exact)
    int* sFull;      // [sub] tokens for the full exact pass
    int* sPT;        // [cap] pair token
    int* sPE;        // [cap] pair expert
    float* sPZ;      // [cap] pair exact logit
    const unsigned long long* tab;   // glibc expf table (shared memory)
    int sub;
};

// Expert column of a thread's float4 group j (j % 4 == 0): group q = j / 4 of thread eg covers
// experts q * Ep / (TE / 4) + 4 eg + [0, 4) — a warp's float4 loads are contiguous (no bank conflicts).
__device__ __forceinline__ int gate_col(int eg, int j, int Ep, int TE) { return (j >> 2) * (Ep / (TE >> 2)) + 4 * eg; }

// two independent round-to-nearest FMAs in one FFMA2: (d0, d1) += a * (b0, b1)
__device__ __forceinline__ void ffma2_bcast(float& d0, float& d1, float a, float b0, float b1) {
    unsigned long long d, b;
    asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(d0), "f"(d1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(b) : "f"(b0), "f"(b1));
    asm("{\n\t.reg .b64 aa;\n\tmov.b64 aa, {%2, %2};\n\tfma.rn.f32x2 %0, aa, %1, %0;\n\t}" : "+l"(d) : "l"(b), "f"(a));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(d));
}

// Logits of `ts` tokens (token t = rows ? rows[t] : tok0 + t) into sL[t][e]. Thread tile TT x TE.
// FAST: fma chain + chunk-end |partial| sums into sSab + |a|^2 into sNa; else the reference chain.
template <bool FAST, int TT, int TE>
__device__ void gate_logits(const LaunchParams& P, const RankCtx& R, const float* __restrict__ A, int tok0,
                            const int* rows, int ts, const GateSmem& g) {
    const int E = P.E, H = P.H;
    const int Ep = (E + 7) & ~7;
    const int tid = threadIdx.x;
    const bool w_vec = (E & 3) == 0;
    const int n_eg = Ep / TE;
    const int n_tg = (ts + TT - 1) / TT;
    const int n_items = n_tg * n_eg;
    const int nk = H / kGateKC;   // envelope: H % 32 == 0
    const uint64_t pol_a = FD_DBG(kDbgEvictNormal) ? l2_policy_evict_normal() : l2_policy_evict_last();   // token rows: keep for the dispatch push
    for (int base = 0; base < n_items; base += kThreads) {   // item rounds (re-stream K per round)
        auto load_stage = [&](int st, int kb) {
            if (FD_DBG(kDbgGateNoLoad)) { cp_async_commit(); return; }
            float* a = g.sA + st * g.sub * kGateApitch;
            float* w = g.sW + st * kGateKC * Ep;
            const int k0 = kb * kGateKC;
            for (int i = tid; i < ts * 8; i += kThreads) {
                const int t = i >> 3, c = i & 7;
                const int tok = rows ? rows[t] : tok0 + t;
                cp_async16_hint(a + t * kGateApitch + c * 4, A + (size_t)tok * H + k0 + c * 4, pol_a);
            }
            if (w_vec) {
                const int cpr = Ep >> 2;
                for (int i = tid; i < kGateKC * cpr; i += kThreads) {
                    const int kk = i / cpr, c = i - kk * cpr;
                    const bool ok = c * 4 < E;
                    cp_async16(w + kk * Ep + c * 4, R.wg + (size_t)(k0 + kk) * E + (ok ? c * 4 : 0), ok);
                }
            } else {
                for (int i = tid; i < kGateKC * Ep; i += kThreads) {
                    const int kk = i / Ep, e = i % Ep;
                    w[kk * Ep + e] = e < E ? R.wg[(size_t)(k0 + kk) * E + e] : 0.0f;
                }
            }
            cp_async_commit();
        };
        float acc[TT][TE], sab[TT];   // sab: sum over chunk ends of max_j |partial| (bounds every j's sum)
#pragma unroll
        for (int i = 0; i < TT; ++i) {
            sab[i] = 0.0f;
#pragma unroll
            for (int j = 0; j < TE; ++j) acc[i][j] = 0.0f;
        }
        double ss = 0.0;
        const int item = base + tid;
        const int tg = item / n_eg, eg = item % n_eg;
        const bool active = item < n_items;

        __syncthreads();   // previous users of sA/sW/sL are done
        for (int st = 0; st < kGateStages - 1; ++st)
            if (st < nk) load_stage(st, st); else cp_async_commit();
        for (int kb = 0; kb < nk; ++kb) {
            const int st = kb % kGateStages;
            cp_async_wait<kGateStages - 2>();   // chunk kb landed (kb + 1 may still be in flight)
            __syncthreads();                     // ... for every thread, and everyone is past chunk kb - 1,
            // so its slot takes chunk kb + 2 now: one barrier per chunk instead of two
            if (kb + kGateStages - 1 < nk) load_stage((kb + kGateStages - 1) % kGateStages, kb + kGateStages - 1);
            else cp_async_commit();
            const float* a = g.sA + st * g.sub * kGateApitch;
            const float* w = g.sW + st * kGateKC * Ep;
            if (FAST && tid < ts && !(FD_DBG(kDbgGateNoNorm))) {   // |a|^2: 32-term float chunks, double sum
                const float* ar = a + tid * kGateApitch;
                float cs = 0.0f;
#pragma unroll
                for (int kk = 0; kk < kGateKC; ++kk) cs = __fmaf_rn(ar[kk], ar[kk], cs);
                ss += (double)cs;
            }
            if (active && !(FD_DBG(kDbgGateNoMath))) {
                const float* ar = a + (TT * tg) * kGateApitch;
#pragma unroll 8
                for (int kk = 0; kk < kGateKC; ++kk) {
                    float av[TT], wv[TE];
#pragma unroll
                    for (int i = 0; i < TT; ++i) av[i] = ar[i * kGateApitch + kk];
#pragma unroll
                    for (int j = 0; j < TE; j += 4) {   // float4 groups spread Ep/(TE/4) apart: conflict-free
                        const float4 w4 = *reinterpret_cast<const float4*>(w + kk * Ep + gate_col(eg, j, Ep, TE));
                        wv[j] = w4.x; wv[j + 1] = w4.y; wv[j + 2] = w4.z; wv[j + 3] = w4.w;
                    }
#pragma unroll
                    for (int i = 0; i < TT; ++i)
#pragma unroll
                        for (int j = 0; j < TE; j += 2) {
                            if (FAST) {
                                ffma2_bcast(acc[i][j], acc[i][j + 1], av[i], wv[j], wv[j + 1]);
                            } else {
                                acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(av[i], wv[j]));
                                acc[i][j + 1] = __fadd_rn(acc[i][j + 1], __fmul_rn(av[i], wv[j + 1]));
                            }
                        }
                }
                if (FAST) {
#pragma unroll
                    for (int i = 0; i < TT; ++i) {
                        float m = 0.0f;
#pragma unroll
                        for (int j = 0; j < TE; ++j) m = fmaxf(m, fabsf(acc[i][j]));
                        sab[i] += m;
                    }
                }
            }
        }
        cp_async_wait<0>();
        if (active) {
#pragma unroll
            for (int i = 0; i < TT; ++i) {
                if (TT * tg + i >= ts) continue;
#pragma unroll
                for (int j = 0; j < TE; ++j) g.sL[(TT * tg + i) * Ep + gate_col(eg, j & ~3, Ep, TE) + (j & 3)] = acc[i][j];
                // non-negative floats order like their bit patterns; rounding of the running sum
                // is covered by u' (1.001 u)
                if (FAST) atomicMax(reinterpret_cast<int*>(g.sSab) + TT * tg + i, __float_as_int(sab[i]));
            }
        }
        if (FAST && tid < ts) g.sNa[tid] = ss;
    }
    __syncthreads();
}

// warp argmax with lower-index tie-break
__device__ __forceinline__ void warp_argmax(float& v, int& i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, i, o);
        if (ov > v || (ov == v && oi < i)) { v = ov; i = oi; }
    }
}

// Routing outputs of one token from (approximate) logits in `row` with max `mx` and picks pe[0..K)
// (one warp): G_phi and weights derive from row; expert ids are already decided.
__device__ __forceinline__ void write_routing_from_row(const LaunchParams& P, const RankCtx& R, float* row, float mx,
                                                       int tok, const int (&pe)[8], int* sCnt,
                                                       const unsigned long long* g_tab) {
    const int E = P.E, K = P.k, lane = threadIdx.x & 31;
    float part = 0.0f;
    for (int e = lane; e < E; e += 32) {
        const float x = expf_glibc(__fsub_rn(row[e], mx), g_tab);
        row[e] = x;
        part += x;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    const float inv = 1.0f / part;
    __syncwarp();
    for (int e = lane; e < E; e += 32) R.g_phi[(size_t)tok * E + e] = row[e] * inv;
    if (lane == 0) {
        float denom = 0.0f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (j >= K) break;
            denom += row[pe[j]] * inv;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (j >= K) break;
            R.pick_e[(size_t)tok * K + j] = pe[j];
            R.pick_w[(size_t)tok * K + j] = denom > 0.0f ? row[pe[j]] * inv / denom : 0.0f;
            atomicAdd(&sCnt[pe[j]], 1);
        }
    }
    __syncwarp();
}

// Exact routing of one token from its exact logits in `row` (one warp): gate.hpp:82-103.
__device__ void route_exact(const LaunchParams& P, const RankCtx& R, float* row, int tok, int* sCnt,
                            const unsigned long long* tab) {
    const int E = P.E, K = P.k, lane = threadIdx.x & 31;
    // max is exact and order-free (x - max only feeds expf; +-0 ties give equal results)
    float mx = row[0];
    for (int e = lane; e < E; e += 32) mx = fmaxf(mx, row[e]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    for (int e = lane; e < E; e += 32) row[e] = expf_glibc(__fsub_rn(row[e], mx), tab);
    __syncwarp();
    float sum = 0.0f;
    if (lane == 0)
        for (int e = 0; e < E; ++e) sum = __fadd_rn(sum, row[e]);   // ascending e (gate.hpp:85-88)
    sum = __shfl_sync(0xffffffffu, sum, 0);
    for (int e = lane; e < E; e += 32) {
        const float p = __fdiv_rn(row[e], sum);
        row[e] = p;
        R.g_phi[(size_t)tok * E + e] = p;
    }
    __syncwarp();
    // top-k by repeated argmax on p; ties -> lower expert index (gate.hpp:41-51)
    uint32_t taken = 0;   // bit jj: expert lane + 32*jj taken
    float denom = 0.0f;
    float pv[8];
    int pe[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        if (j >= K) break;
        float bv = -1.0f;
        int bi = 0x7fffffff;
        for (int e = lane, jj = 0; e < E; e += 32, ++jj) {
            if (taken & (1u << jj)) continue;
            const float v = row[e];
            if (v > bv || (v == bv && e < bi)) { bv = v; bi = e; }
        }
        warp_argmax(bv, bi);
        if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
        pe[j] = bi;
        pv[j] = bv;
        denom = __fadd_rn(denom, bv);   // pick order (gate.hpp:92)
    }
    if (lane == 0) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (j >= K) break;
            R.pick_e[(size_t)tok * K + j] = pe[j];
            R.pick_w[(size_t)tok * K + j] = denom > 0.0f ? __fdiv_rn(pv[j], denom) : 0.0f;
            atomicAdd(&sCnt[pe[j]], 1);
        }
    }
    __syncwarp();
}

// Margin between two logits x > y (m: the token's max logit) that keeps the reference's
// probabilities strictly ordered: with d = fl(z - m) (error <= u|z - m|), glibc expf (< 1 ulp) and
// the division (0.5 ulp), p_x > p_y holds once x - y > 2^-21.4 + u (|x - m| + |y - m|); we use
// 2^-19 + 2^-21 (|x - m| + |y - m|), plus 2^-22 (|x| + |y|) for the float rounding of the bound
// arithmetic (z~ +- beta) that produced x and y.
__device__ __forceinline__ float gate_margin(float x, float y, float m) {
    return 1.9073486e-6f + 4.7683716e-7f * (fabsf(x - m) + fabsf(y - m)) + 2.3841858e-7f * (fabsf(x) + fabsf(y));
}

// Certified routing of token t (local index) from FFMA logits in `row` (one warp).
// Returns 1: routed; 0: candidates appended to the pair list; 2: needs the full exact pass.
__device__ int route_certified(const LaunchParams& P, const RankCtx& R, float* row, int tok, int t,
                               const GateSmem& g, int* s_np) {
    constexpr int J = kMaxExperts / 32;
    const int E = P.E, K = P.k, lane = threadIdx.x & 31;
    const float na = __double2float_ru(sqrt(g.sNa[t] * (1.0 + 1e-5)));
    // SIMT logits: chunk-end partial sums (sSab) + product / chain-distance terms; tensor-core logits:
    // sSab = 0 and the whole bound rides on |a| |w_e| (gate_k1_tc, set by the host)
    const float c_s = P.gate_u * 64.0f * g.sSab[t];
    const float c_w = P.gate_u * (P.gate_tc ? P.gate_k1_tc : P.gate_k1) * na;
    float z[J], bt[J];
    bool bad = false;
#pragma unroll
    for (int jj = 0; jj < J; ++jj) {
        const int e = lane + 32 * jj;
        if (e < E) {
            z[jj] = row[e];
            bt[jj] = c_s + c_w * __ldg(R.wg_norm + e) + 1e-30f;
            bad |= !(fabsf(z[jj]) < 1e30f) || !(bt[jj] < 1e30f);
        } else {
            z[jj] = -INFINITY;
            bt[jj] = 0.0f;
        }
    }
    if (__any_sync(0xffffffffu, bad)) return 2;   // NaN / inf / overflow: the exact path decides
    // top-1 by z~ (reference max ~ z0) and the k-th largest lower bound
    float z0 = -INFINITY;
    {
        int i0 = 0x7fffffff;
#pragma unroll
        for (int jj = 0; jj < J; ++jj)
            if (z[jj] > z0) { z0 = z[jj]; i0 = lane + 32 * jj; }
        warp_argmax(z0, i0);
    }
    float Lk = 0.0f;
    {
        uint32_t taken = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (j >= K) break;
            float bv = -INFINITY;
            int bi = 0x7fffffff;
#pragma unroll
            for (int jj = 0; jj < J; ++jj) {
                const int e = lane + 32 * jj;
                if (e >= E || (taken & (1u << jj))) continue;
                const float lb = z[jj] - bt[jj];
                if (lb > bv) { bv = lb; bi = e; }
            }
            warp_argmax(bv, bi);
            if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
            Lk = bv;
        }
    }
    // candidates: experts whose upper bound reaches the k-th largest lower bound
    uint32_t cmask = 0;
    int n_c = 0;
#pragma unroll
    for (int jj = 0; jj < J; ++jj) {
        const int e = lane + 32 * jj;
        const float ub = z[jj] + bt[jj];
        const bool c = e < E && ub >= Lk - gate_margin(ub, Lk, z0);
        if (c) cmask |= 1u << jj;
        n_c += __popc(__ballot_sync(0xffffffffu, c));
    }
    if (n_c > kGateMaxCand) return 2;
    if (n_c == K) {
        // the set is certain; the order is certain if consecutive z~-sorted picks are separated
        int pe[8];
        uint32_t taken = 0;
        float prev_lb = 0.0f;
        bool ok = true;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (j >= K) break;
            float bv = -INFINITY, bb = 0.0f;
            int bi = 0x7fffffff;
#pragma unroll
            for (int jj = 0; jj < J; ++jj) {
                if (!(cmask & (1u << jj)) || (taken & (1u << jj))) continue;
                if (z[jj] > bv) { bv = z[jj]; bi = lane + 32 * jj; bb = bt[jj]; }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                const float ob = __shfl_xor_sync(0xffffffffu, bb, o);
                if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; bb = ob; }
            }
            if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
            pe[j] = bi;
            if (j > 0) ok &= prev_lb > bv + bb + gate_margin(prev_lb, bv + bb, z0);
            prev_lb = bv - bb;
        }
        // picks far below the max could underflow to tied zero probabilities in the reference
        ok &= prev_lb - z0 > -80.0f;
        if (ok) {
            write_routing_from_row(P, R, row, z0, tok, pe, g.sCnt, g.tab);
            return 1;
        }
    }
    // append the candidates as (token, expert) pairs for the exact pair pass
    int base = 0;
    if (lane == 0) base = atomicAdd(s_np, n_c);
    base = __shfl_sync(0xffffffffu, base, 0);
    int off = 0;
#pragma unroll
    for (int jj = 0; jj < J; ++jj) {
        const bool c = cmask & (1u << jj);
        const uint32_t m = __ballot_sync(0xffffffffu, c);
        const int pos = base + off + __popc(m & ((1u << lane) - 1));
        if (c && pos < kGatePairCap) { g.sPT[pos] = tok; g.sPE[pos] = lane + 32 * jj; }
        off += __popc(m);
    }
    if (base + n_c > kGatePairCap) return 2;
    if (lane == 0) { g.sTP0[t] = base; g.sTNC[t] = n_c; }
    return 0;
}

// Certified routing of token t by ONE thread (tensor-core logits, k <= 2, E <= 128): the decision
// procedure of route_certified over the thread's own row (smem, odd pitch: conflict-free across the
// warp's rows), so a CTA's ~110 tokens decide in parallel instead of ~10 per warp in sequence.
// Returns 1: routed (picks in *p0/*p1, max logit in *zmax; the softmax is written by route_softmax);
// 0: candidates appended to the pair list; 2: needs the full exact pass.
__device__ int route_decide_thread(const LaunchParams& P, const float* row, int tok, int t, const GateSmem& g,
                                   const float* __restrict__ sWn, int* s_np, int* p0o, int* p1o, float* zmax) {
    const int E = P.E, K = P.k;
    const float na = __double2float_ru(sqrt(g.sNa[t] * (1.0 + 1e-5)));
    const float c_s = P.gate_u * 64.0f * g.sSab[t];
    const float c_w = P.gate_u * P.gate_k1_tc * na;
    // pass 1: overflow guard, max z~, the k largest lower bounds
    float z0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY;
    bool bad = false;
#pragma unroll 8
    for (int e = 0; e < E; ++e) {   // branch-free (divergent branches cost a reconvergence per element)
        const float z = row[e], bt = c_s + c_w * sWn[e] + 1e-30f;
        bad |= !(fabsf(z) < 1e30f) || !(bt < 1e30f);
        z0 = fmaxf(z0, z);
        const float lb = z - bt;
        m2 = fmaxf(m2, fminf(m1, lb));   // multiset top-2 of the lower bounds
        m1 = fmaxf(m1, lb);
    }
    if (bad) return 2;   // NaN / inf / overflow: the exact path decides
    const float Lk = K == 1 ? m1 : m2;
    // pass 2: candidates (upper bound reaches the k-th lower bound) and their top-k by z~ (ties -> lower id)
    int n_c = 0, p0 = -1, p1 = -1;
    float v0 = -INFINITY, v1 = -INFINITY;
#pragma unroll 8
    for (int e = 0; e < E; ++e) {
        const float z = row[e], bt = c_s + c_w * sWn[e] + 1e-30f, ub = z + bt;
        const bool c = ub >= Lk - gate_margin(ub, Lk, z0);
        const bool g0 = c && z > v0, g1 = c && !g0 && z > v1;   // strict: ties keep the lower id
        n_c += c ? 1 : 0;
        v1 = g0 ? v0 : (g1 ? z : v1);
        p1 = g0 ? p0 : (g1 ? e : p1);
        v0 = g0 ? z : v0;
        p0 = g0 ? e : p0;
    }
    if (n_c > kGateMaxCand) return 2;
    if (n_c == K) {
        const float b0 = c_s + c_w * sWn[p0] + 1e-30f;
        float last_lb = v0 - b0;
        bool ok = true;
        if (K == 2) {
            const float b1 = c_s + c_w * sWn[p1] + 1e-30f;
            ok = last_lb > v1 + b1 + gate_margin(last_lb, v1 + b1, z0);
            last_lb = v1 - b1;
        }
        ok &= last_lb - z0 > -80.0f;   // picks far below the max could tie at zero probability
        if (ok) {
            *p0o = p0;
            *p1o = p1;
            *zmax = z0;
            return 1;
        }
    }
    // the candidates (ascending expert id) become (token, expert) pairs for the exact pair pass (slots past
    // the list's capacity are dropped and the token goes to the full pass; every slot below it is filled)
    const int base = atomicAdd(s_np, n_c);
    int pos = base;
    for (int e = 0; e < E; ++e) {
        const float z = row[e], bt = c_s + c_w * sWn[e] + 1e-30f, ub = z + bt;
        if (ub >= Lk - gate_margin(ub, Lk, z0)) {
            if (pos < kGatePairCap) { g.sPT[pos] = tok; g.sPE[pos] = e; }
            ++pos;
        }
    }
    if (pos > kGatePairCap) return 2;
    g.sTP0[t] = base;
    g.sTNC[t] = n_c;
    return 0;
}

// Softmax and routing outputs of the thread-decided tokens of a sub-tile (whole CTA): exps over the flat
// (token, expert) range by every thread, then one warp per token sums, normalises and writes G_phi
// (coalesced) and the picks -- write_routing_from_row's outputs (G_phi / weights from z~: tolerance).
__device__ void route_softmax(const LaunchParams& P, const RankCtx& R, const GateSmem& g, int Lp, int tok0, int ts,
                              const int* sDec, const float* sZ0, int cta) {
    const int E = P.E, K = P.k, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < ts * E; i += kThreads) {
        const int t = i / E, e = i - t * E;
        if (sDec[t] < 0) continue;
        float* x = g.sL + t * Lp + e;
        // G_phi / weights of certified tokens carry z~'s tolerance anyway: CUDA's FP32 expf (<= 2 ulp, no
        // FP64) instead of the bit-exact glibc restatement the exact paths use
        *x = expf(__fsub_rn(*x, sZ0[t]));
    }
    __syncthreads();
    if (tid == 0) R.trace[(size_t)cta * kTracePts + kTrGateExp] = globaltimer();
    for (int t = warp; t < ts; t += kThreads / 32) {
        const int d = sDec[t];
        if (d < 0) continue;
        const float* row = g.sL + t * Lp;
        float part = 0.0f;
        for (int e = lane; e < E; e += 32) part += row[e];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        const float inv = 1.0f / part;
        const int tok = tok0 + t;
        for (int e = lane; e < E; e += 32) R.g_phi[(size_t)tok * E + e] = row[e] * inv;
        if (lane == 0) {
            const int p0 = d & 0xffff, p1 = d >> 16;
            const float q0 = row[p0] * inv, q1 = K == 2 ? row[p1] * inv : 0.0f;
            const float denom = q0 + q1;
            R.pick_e[(size_t)tok * K] = p0;
            R.pick_w[(size_t)tok * K] = denom > 0.0f ? q0 / denom : 0.0f;
            atomicAdd(&g.sCnt[p0], 1);
            if (K == 2) {
                R.pick_e[(size_t)tok * K + 1] = p1;
                R.pick_w[(size_t)tok * K + 1] = denom > 0.0f ? q1 / denom : 0.0f;
                atomicAdd(&g.sCnt[p1], 1);
            }
        }
    }
}

// FP32 mode: the reference logits of the k picks of every thread-certified token of a sub-tile, one thread per
// (token, pick) running the reference chain z = sum over x ascending of fl(a_x w_x) (gate.hpp:77-81) over token /
// Wg^T row chunks staged in smem (3-deep cp.async ring, 32 x per chunk), and the tokens' combine weights
// recomputed from them: w_j = e_j / (e_0 + e_1) with e_j = expf(z_j - z_0) (the softmax sum cancels). The
// certified z~ is ~1e-6 off the reference chain, and the weights derived from it carried that error into rare
// cancellation-dominated output elements above the FP32 bound (tools/dev/parity_wide.py: worst 1.07 of the bound
// with z~ weights, 0.54 with exact ones). Routing is unaffected (it is certified bit-exact either way).
// It also runs the sub-tile's candidate (token, expert) pairs of the undecided tokens (g.sPT / g.sPE, np of them,
// results to g.sPZ) -- the pair pass -- as a second chain per thread over the same staged rows.
__device__ void gate_pick_weights(const LaunchParams& P, const RankCtx& R, const float* __restrict__ A,
                                  const GateSmem& g, int tok0, int ts, const int* sDec, int np) {
    const int H = P.H, E = P.E, K = P.k, tid = threadIdx.x;
    constexpr int XC = 32, PITCH = 36, NST = 3;   // (16-x chunks x 6 stages measured slower: per-chunk cost)
    float* ring = g.sA;
    const int rows = ts + E;
    const int stage_f = rows * PITCH;
    int* plist = reinterpret_cast<int*>(ring + NST * stage_f);   // [2 ts]: (t << 16) | expert, -1 = none
    float* zp = reinterpret_cast<float*>(plist + 2 * kGateSubMax);
    for (int i = tid; i < 2 * ts; i += kThreads) {
        const int t = i >> 1, j = i & 1;
        const int d = sDec[t];
        plist[i] = (d < 0 || j >= K) ? -1 : ((t << 16) | (j == 0 ? (d & 0xffff) : (d >> 16)));
    }
    __syncthreads();   // sDec lives in the staging area the ring overwrites
    const int my = tid < 2 * ts ? plist[tid] : -1;
    const int mt = my >> 16, me = my & 0xffff;
    const int cp_t = tid < np ? g.sPT[tid] - tok0 : -1, cp_e = tid < np ? g.sPE[tid] : 0;   // candidate pair
    auto load = [&](int st, int c) {
        float* b = ring + st * stage_f;
        const int x0 = c * XC;
        for (int i = tid; i < rows * (XC / 4); i += kThreads) {
            const int r = i / (XC / 4), q = i % (XC / 4);
            const float* src = r < ts ? A + (size_t)(tok0 + r) * H + x0 + 4 * q : R.wgT + (size_t)(r - ts) * H + x0 + 4 * q;
            cp_async16(b + r * PITCH + 4 * q, src, true);
        }
        cp_async_commit();
    };
    const int nch = H / XC;   // H % 32 == 0 (envelope)
    float z = 0.0f, z2 = 0.0f;
    for (int c = 0; c < NST - 1; ++c) {
        if (c < nch) load(c, c); else cp_async_commit();
    }
    for (int c = 0; c < nch; ++c) {
        if (c + NST - 1 < nch) load((c + NST - 1) % NST, c + NST - 1); else cp_async_commit();
        cp_async_wait<NST - 1>();
        __syncthreads();
        const float* st = ring + (c % NST) * stage_f;
        if (my >= 0) {
            const float* ar = st + mt * PITCH;
            const float* wr = st + (ts + me) * PITCH;
#pragma unroll
            for (int q = 0; q < XC / 4; ++q) {
                const float4 a4 = *reinterpret_cast<const float4*>(ar + 4 * q);
                const float4 w4 = *reinterpret_cast<const float4*>(wr + 4 * q);
                z = __fadd_rn(z, __fmul_rn(a4.x, w4.x));
                z = __fadd_rn(z, __fmul_rn(a4.y, w4.y));
                z = __fadd_rn(z, __fmul_rn(a4.z, w4.z));
                z = __fadd_rn(z, __fmul_rn(a4.w, w4.w));
            }
        }
        if (cp_t >= 0) {
            const float* ar = st + cp_t * PITCH;
            const float* wr = st + (ts + cp_e) * PITCH;
#pragma unroll
            for (int q = 0; q < XC / 4; ++q) {
                const float4 a4 = *reinterpret_cast<const float4*>(ar + 4 * q);
                const float4 w4 = *reinterpret_cast<const float4*>(wr + 4 * q);
                z2 = __fadd_rn(z2, __fmul_rn(a4.x, w4.x));
                z2 = __fadd_rn(z2, __fmul_rn(a4.y, w4.y));
                z2 = __fadd_rn(z2, __fmul_rn(a4.z, w4.z));
                z2 = __fadd_rn(z2, __fmul_rn(a4.w, w4.w));
            }
        }
        __syncthreads();
    }
    cp_async_wait<0>();
    if (my >= 0) zp[tid] = z;
    if (cp_t >= 0) g.sPZ[tid] = z2;
    __syncthreads();
    if (K == 2)
        for (int t = tid; t < ts; t += kThreads) {
            if (plist[2 * t] < 0) continue;
            const size_t tok = (size_t)tok0 + t;
            const float e1 = expf_glibc(__fsub_rn(zp[2 * t + 1], zp[2 * t]), g.tab);   // e_0 = expf(0) = 1
            const float den = __fadd_rn(1.0f, e1);
            R.pick_w[tok * 2] = __fdiv_rn(1.0f, den);
            R.pick_w[tok * 2 + 1] = __fdiv_rn(e1, den);
        }
    __syncthreads();
}

// Exact reference logits of np (token, expert) pairs: thread p runs pair p's separately-rounded
// chain over x ascending (gate.hpp:77-81), rows staged through smem in x-chunks (A row and Wg^T row).
__device__ void gate_pairs_exact(const LaunchParams& P, const RankCtx& R, const float* __restrict__ A,
                                 const GateSmem& g, int np) {
    const int H = P.H, tid = threadIdx.x;
    const int nch = (H + kGatePairX - 1) / kGatePairX;
    for (int p0 = 0; p0 < np; p0 += kGatePairBatch) {
        const int nb = min(kGatePairBatch, np - p0);
        auto load = [&](int st, int ch) {
            const int x0 = ch * kGatePairX, per_row = min(kGatePairX, H - x0) >> 2;
            float* b = g.sPair + st * kGatePairBatch * kGatePairPitch;
            for (int i = tid; i < nb * 2 * per_row; i += kThreads) {
                const int r = i / per_row, c = i - r * per_row;
                const int pi = p0 + (r >> 1);
                const float* src = (r & 1) ? R.wgT + (size_t)g.sPE[pi] * H + x0 + 4 * c
                                           : A + (size_t)g.sPT[pi] * H + x0 + 4 * c;
                cp_async16(b + (r >> 1) * kGatePairPitch + (r & 1) * kGatePairX + 4 * c, src, true);
            }
            cp_async_commit();
        };
        float acc = 0.0f;
        __syncthreads();
        load(0, 0);
        for (int ch = 0; ch < nch; ++ch) {
            if (ch + 1 < nch) load((ch + 1) & 1, ch + 1); else cp_async_commit();
            cp_async_wait<1>();
            __syncthreads();
            if (tid < nb) {
                const float* b = g.sPair + (ch & 1) * kGatePairBatch * kGatePairPitch + tid * kGatePairPitch;
                const int xl = min(kGatePairX, H - ch * kGatePairX);
#pragma unroll 4   // loads of the next groups issue ahead of this group's dependent FADDs
                for (int x = 0; x < xl; x += 4) {
                    const float4 a4 = *reinterpret_cast<const float4*>(b + x);
                    const float4 w4 = *reinterpret_cast<const float4*>(b + kGatePairX + x);
                    acc = __fadd_rn(acc, __fmul_rn(a4.x, w4.x));
                    acc = __fadd_rn(acc, __fmul_rn(a4.y, w4.y));
                    acc = __fadd_rn(acc, __fmul_rn(a4.z, w4.z));
                    acc = __fadd_rn(acc, __fmul_rn(a4.w, w4.w));
                }
            }
            __syncthreads();
        }
        cp_async_wait<0>();
        if (tid < nb) g.sPZ[p0 + tid] = acc;
    }
    __syncthreads();
}

// Full exact pass (ties / near-ties): every expert's reference logit of the nf tokens in sFull -> sL
// rows [0, nf). Thread e runs expert e's chain z = sum over x ascending of fl(a_x * w_xe)
// (gate.hpp:77-81) over Wg rows that stream through shared memory in X-row chunks (cp.async,
// double-buffered, coalesced; the token's x-chunk rides along). The chain loop is unrolled so its
// shared loads are off the FADD dependency: ~4 cycles per x, one H-long chain per expert.
__device__ void gate_full_exact(const LaunchParams& P, const RankCtx& R, const float* __restrict__ A,
                                const GateSmem& g, int nf) {
    const int E = P.E, H = P.H, Ep = (E + 7) & ~7, tid = threadIdx.x;
    const int cap = kGateRegionFloats - (int)(g.sA - g.sL);   // floats after sL (the cp.async staging area)
    int X = (cap / (2 * (Ep + 1))) & ~31;
    X = X < 32 ? 32 : (X > 256 ? 256 : X);
    float* buf = g.sA;   // [2][X][Ep] Wg rows, then [2][X] token values
    float* abuf = buf + 2 * X * Ep;
    const bool vec = (E & 3) == 0;
    const int nch = (H + X - 1) / X;   // H % 32 == 0 (envelope), X % 32 == 0: whole 16-byte groups
    for (int t = 0; t < nf; ++t) {
        const float* a = A + (size_t)g.sFull[t] * H;
        auto load = [&](int st, int c) {
            const int x0 = c * X, xn = min(X, H - x0);
            float* b = buf + st * X * Ep;
            if (vec) {
                const int cpr = E >> 2;
                for (int i = tid; i < xn * cpr; i += kThreads) {
                    const int xx = i / cpr, q = i - xx * cpr;
                    cp_async16(b + xx * Ep + 4 * q, R.wg + (size_t)(x0 + xx) * E + 4 * q, true);
                }
            } else {
                for (int i = tid; i < xn * E; i += kThreads) {
                    const int xx = i / E, e = i - xx * E;
                    b[xx * Ep + e] = R.wg[(size_t)(x0 + xx) * E + e];
                }
            }
            for (int i = tid; i < xn / 4; i += kThreads) cp_async16(abuf + st * X + 4 * i, a + x0 + 4 * i, true);
            cp_async_commit();
        };
        float acc = 0.0f;
        __syncthreads();   // sL / staging area free (callers' previous use is done)
        load(0, 0);
        for (int c = 0; c < nch; ++c) {
            if (c + 1 < nch) load((c + 1) & 1, c + 1); else cp_async_commit();
            cp_async_wait<1>();
            __syncthreads();
            const int xn = min(X, H - c * X);
            const float* b = buf + (c & 1) * X * Ep + tid;
            const float* av = abuf + (c & 1) * X;
            if (tid < E) {
                for (int xx = 0; xx < xn; xx += 8) {   // xn % 32 == 0
                    float w[8], x[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) { w[u] = b[(xx + u) * Ep]; x[u] = av[xx + u]; }
#pragma unroll
                    for (int u = 0; u < 8; ++u) acc = __fadd_rn(acc, __fmul_rn(x[u], w[u]));
                }
            }
            __syncthreads();   // buffer (c & 1) is refilled by the next iteration's load
        }
        cp_async_wait<0>();
        if (tid < E) g.sL[t * Ep + tid] = acc;
    }
    __syncthreads();
}

// Decide a token from its candidates' exact logits (one warp). false: ties / near-ties -> full exact.
__device__ bool route_resolve(const LaunchParams& P, const RankCtx& R, float* row, int tok, int t, const GateSmem& g) {
    const int K = P.k, lane = threadIdx.x & 31;
    const int n_c = g.sTNC[t], p0 = g.sTP0[t];
    float zc = -INFINITY;
    int ec = 0x7fffffff;
    if (lane < n_c) { zc = g.sPZ[p0 + lane]; ec = g.sPE[p0 + lane]; }
    if (__any_sync(0xffffffffu, lane < n_c && !(fabsf(zc) < 1e30f))) return false;
    float m = zc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    int pe[8];
    bool taken = false, ok = true;
    float prev = 0.0f;
#pragma unroll
    for (int j = 0; j < 9; ++j) {
        if (j > K || (j == K && n_c == K)) break;
        float bv = taken ? -INFINITY : zc;
        int bi = taken ? 0x7fffffff : ec;
        warp_argmax(bv, bi);
        if (j > 0) ok &= prev - bv > gate_margin(prev, bv, m);
        if (j == K) break;
        if (bi == ec) taken = true;
        pe[j] = bi;
        prev = bv;
    }
    ok &= prev - m > -80.0f;
    if (!ok) return false;
    // exact logits of the candidates replace z~ (G_phi / weights from the row: tolerance)
    if (lane < n_c) row[ec] = zc;
    __syncwarp();
    write_routing_from_row(P, R, row, m, tok, pe, g.sCnt, g.tab);
    return true;
}

// Distributed full-exact pass (after the gate barrier; every CTA of the rank). A near-tie token needs all E
// reference logits: E sequential H-long chains over 2 x H*E*4 bytes of Wg that one SM streams at its own
// memory-level parallelism (~50 us for the CTA that holds the token, the whole rank waiting at the next
// barrier). Here each (listed token, expert) chain is one warp's item: the lanes load the token row and the
// Wg^T row, form the products fl(a_x w_x) in parallel, and lane 0 runs the separately-rounded chain over them
// in x order (gate.hpp:77-81) -- bit-identical to the owner's pass, ~5 us for all E chains at once. The owners
// then route their tokens from R.full_z (route_exact). Returns false on abort.
__device__ bool full_exact_distributed(const LaunchParams& P, const RankCtx& R, const float* __restrict__ A,
                                       uint8_t* smem, int cta, const unsigned long long* tab) {
    const int E = P.E, H = P.H, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int kWarps = kThreads / 32;
    const int nf = (int)min(ld_volatile_u32(&R.full_ctr[0]), (uint32_t)kFullCap);
    if (nf == 0) return true;
    const int items = nf * E;
    float* prod = reinterpret_cast<float*>(smem) + warp * 1024;   // 4 KB per warp: products of one 1024-x chunk
    while (true) {
        int it = 0;
        if (lane == 0) it = (int)atomicAdd(&R.full_ctr[1], 1u);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it >= items) break;
        const int t = it / E, e = it - t * E;
        const int tok = R.full_list[t];
        const float4* a4 = reinterpret_cast<const float4*>(A + (size_t)tok * H);
        const float4* w4 = reinterpret_cast<const float4*>(R.wgT + (size_t)e * H);
        float z = 0.0f;
        for (int x0 = 0; x0 < H; x0 += 1024) {
            const int n4 = min(1024, H - x0) / 4;   // H % 32 == 0 (envelope): whole float4 groups
            float4 av[8], wv[8];   // every load of the chunk in flight at once (one L2 round trip per chunk)
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = lane + 32 * u;
                if (i < n4) { av[u] = __ldcg(a4 + x0 / 4 + i); wv[u] = __ldcg(w4 + x0 / 4 + i); }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = lane + 32 * u;
                if (i < n4)
                    reinterpret_cast<float4*>(prod)[i] = make_float4(__fmul_rn(av[u].x, wv[u].x), __fmul_rn(av[u].y, wv[u].y),
                                                                     __fmul_rn(av[u].z, wv[u].z), __fmul_rn(av[u].w, wv[u].w));
            }
            __syncwarp();
            if (lane == 0) {
#pragma unroll 4
                for (int i = 0; i < n4; ++i) {
                    const float4 p = reinterpret_cast<const float4*>(prod)[i];
                    z = __fadd_rn(z, p.x); z = __fadd_rn(z, p.y); z = __fadd_rn(z, p.z); z = __fadd_rn(z, p.w);
                }
            }
            __syncwarp();
        }
        if (lane == 0) {
            R.full_z[(size_t)t * E + e] = z;
            __threadfence();
            atomicAdd(&R.full_ctr[2], 1u);
        }
    }
    if (tid == 0) R.trace[(size_t)cta * kTracePts + kTrFullChains] = globaltimer();
    // owners: route their listed tokens once every chain is done; their picks join the CTA's counts
    int* sCnt = reinterpret_cast<int*>(smem) + kWarps * 1024 + kWarps * kMaxExperts;
    for (int e = tid; e < E; e += kThreads) sCnt[e] = 0;
    __syncthreads();
    int tokA, tokB, b0, b1;
    gate_token_range(P, cta, tokA, tokB, b0, b1);
    bool mine_any = false;
    for (int t = warp; t < nf; t += kWarps) {
        const int tok = R.full_list[t];
        if (tok < tokA || tok >= tokB) continue;
        mine_any = true;
        int ok = 1;
        if (lane == 0) {
            const uint64_t t0 = globaltimer();
            uint32_t n = 0;
            while (ld_acquire_gpu_u32(&R.full_ctr[2]) < (uint32_t)items) {
                if ((++n & 255u) == 0) {
                    if (ld_volatile_u32(P.abort_flag)) { ok = 0; break; }
                    if (globaltimer() - t0 > P.budget_ns) {
                        raise_error(P, R, kErrTimeout, 120, (uint32_t)items, 0);
                        ok = 0;
                        break;
                    }
                }
            }
        }
        if (!__shfl_sync(0xffffffffu, ok, 0)) break;
        float* row = reinterpret_cast<float*>(smem) + kWarps * 1024 + warp * kMaxExperts;
        for (int e = lane; e < E; e += 32) row[e] = __ldcg(R.full_z + (size_t)t * E + e);
        __syncwarp();
        route_exact(P, R, row, tok, sCnt, tab);
    }
    __shared__ int s_any, s_ok;
    if (tid == 0) s_any = 0;
    __syncthreads();
    if (mine_any && lane == 0) s_any = 1;
    __syncthreads();
    if (s_any)
        for (int e = tid; e < E; e += kThreads)
            if (sCnt[e]) R.cnt_cta[(size_t)cta * E + e] += sCnt[e];
    if (tid == 0) {
        s_ok = ld_volatile_u32(P.abort_flag) == 0;
        R.trace[(size_t)cta * kTracePts + kTrFullRouted] = globaltimer();
    }
    __syncthreads();
    return s_ok != 0;
}

__device__ void gate_phase(const LaunchParams& P, const RankCtx& R, const float* __restrict__ A, int cta,
                           uint8_t* smem, unsigned long long* stat, const unsigned long long* tab) {
    const int E = P.E;
    const int Ep = (E + 7) & ~7;
    const int tid = threadIdx.x, warp = tid >> 5;
    constexpr int kWarps = kThreads / 32;
    GateSmem g;
    g.sub = gate_sub(Ep);
    g.tab = tab;
    // thread-per-token certified routing (tensor-core logits): rows at an odd pitch (conflict-free)
    const bool thread_route = P.gate_tc && !P.exact_gate && P.k <= 2 && E <= 128;
    const int Lp = thread_route ? Ep + 1 : Ep;
    float* region = reinterpret_cast<float*>(smem);
    g.sL = region;
    g.sA = g.sL + g.sub * Lp;
    g.sW = g.sA + kGateStages * g.sub * kGateApitch;
    g.sPair = g.sL + kGateSubMax * 129 > g.sL + g.sub * Lp ? g.sL + kGateSubMax * 129 : g.sL + g.sub * Lp;
    float* sWn = g.sW;   // thread route: |w_e| (the SIMT staging area is unused with tensor-core logits)
    uint8_t* tail = smem + ((kGateRegionFloats * 4 + 15) & ~15);
    g.sNa = reinterpret_cast<double*>(tail);                    tail += kGateSubMax * 8;
    g.sCnt = reinterpret_cast<int*>(tail);                      tail += kMaxExperts * 4;
    g.sSab = reinterpret_cast<float*>(tail);                    tail += kGateSubMax * 4;
    g.sTP0 = reinterpret_cast<int*>(tail);                      tail += kGateSubMax * 4;
    g.sTNC = reinterpret_cast<int*>(tail);                      tail += kGateSubMax * 4;
    g.sFull = reinterpret_cast<int*>(tail);                     tail += kGateSubMax * 4;
    g.sPT = reinterpret_cast<int*>(tail);                       tail += kGatePairCap * 4;
    g.sPE = reinterpret_cast<int*>(tail);                       tail += kGatePairCap * 4;
    g.sPZ = reinterpret_cast<float*>(tail);
    __shared__ int s_np, s_nfull;
    for (int e = tid; e < Ep; e += kThreads) g.sCnt[e] = 0;
    // The exact passes read Wg (full pass, [H][E]) and Wg^T rows (pair pass): 2 x H*E*4 bytes that no other
    // phase touches, so they are cold in HBM after the previous launch's weight stream. A near-tie token then
    // streams 1 MB from HBM at one SM's memory-level parallelism (~50 us, the gate's critical path). Each CTA
    // of the rank prefetches its slice of both into L2 first; the exact passes then hit L2.
    if (tid == 0 && !P.exact_gate) {
        const size_t bytes = (size_t)P.H * E * 4;
        const size_t per = ((bytes + P.ctas_per_rank - 1) / P.ctas_per_rank + 15) & ~(size_t)15;
        const size_t o = (size_t)cta * per;
        if (o < bytes) {
            const uint32_t n = (uint32_t)min(per, bytes - o);
            prefetch_l2_bulk(reinterpret_cast<const uint8_t*>(R.wg) + o, n);
            prefetch_l2_bulk(reinterpret_cast<const uint8_t*>(R.wgT) + o, n);
        }
    }

    int tokA, tokB, b0, b1;
    gate_token_range(P, cta, tokA, tokB, b0, b1);
    const int ntok = tokB - tokA;
    const int nsub = (ntok + g.sub - 1) / g.sub;
    unsigned long long n_full = 0, n_pair_tok = 0;

    for (int si = 0; si < nsub; ++si) {
        // balanced sub-tiles
        const int s0 = (int)((long long)ntok * si / nsub);
        const int s1 = (int)((long long)ntok * (si + 1) / nsub);
        const int ts = s1 - s0;
        // few tokens per CTA (small S or many CTAs per rank): the 5 x 8 thread tile would leave most
        // threads idle (c5: 6 of 384 active), so switch to 1 token x 4 experts per thread
        const bool small = ((ts + kGateTT - 1) / kGateTT) * (Ep / kGateTE) * 4 <= kThreads &&
                           ts * (Ep / 4) <= kThreads;   // ... and the small tile covers the sub-tile in one round
        if (P.exact_gate) {
            if (small) gate_logits<false, 1, 4>(P, R, A, tokA + s0, nullptr, ts, g);
            else gate_logits<false, kGateTT, kGateTE>(P, R, A, tokA + s0, nullptr, ts, g);
            for (int t = warp; t < ts; t += kWarps) route_exact(P, R, g.sL + t * Ep, tokA + s0 + t, g.sCnt, g.tab);
            n_full += ts;
            continue;
        }
        bool pairs_done = false;
        for (int t = tid; t < ts; t += kThreads) { g.sSab[t] = 0.0f; g.sTNC[t] = 0; }
        if (tid == 0) { s_np = 0; s_nfull = 0; }
        __syncthreads();
        if (P.gate_tc) {   // tensor-core logits (phase 1a) and row norms from global
            if ((E & 3) == 0) {   // float4 rows, every load of a thread in flight before its stores
                const int q4 = E >> 2, n4 = ts * q4;
                const float4* src = reinterpret_cast<const float4*>(R.g_phi + (size_t)(tokA + s0) * E);
                for (int i0 = tid; i0 < n4; i0 += kThreads * 8) {
                    float4 v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if (i0 + u * kThreads < n4) v[u] = __ldcg(src + i0 + u * kThreads);
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int i = i0 + u * kThreads;
                        if (i < n4) {
                            float* d = g.sL + (i / q4) * Lp + 4 * (i % q4);
                            d[0] = v[u].x; d[1] = v[u].y; d[2] = v[u].z; d[3] = v[u].w;
                        }
                    }
                }
                for (int i = tid; i < ts * (Ep - E); i += kThreads)
                    g.sL[(i / (Ep - E)) * Lp + E + i % (Ep - E)] = 0.0f;
            } else {
                for (int i = tid; i < ts * Ep; i += kThreads) {
                    const int t = i / Ep, e = i - t * Ep;
                    g.sL[t * Lp + e] = e < E ? R.g_phi[(size_t)(tokA + s0 + t) * E + e] : 0.0f;
                }
            }
            for (int t = tid; t < ts; t += kThreads) {
                g.sNa[t] = R.gate_na[tokA + s0 + t];
                g.sSab[t] = R.gate_sab[tokA + s0 + t];
            }
            if (thread_route)
                for (int e = tid; e < E; e += kThreads) sWn[e] = R.wg_norm[e];
            __syncthreads();
        } else if (small) gate_logits<true, 1, 4>(P, R, A, tokA + s0, nullptr, ts, g);
        else gate_logits<true, kGateTT, kGateTE>(P, R, A, tokA + s0, nullptr, ts, g);
        if (tid == 0) R.trace[(size_t)cta * kTracePts + kTrGateLoad] = globaltimer();
        if (thread_route) {
            // decisions (thread per token), then the softmax / outputs of the routed ones (whole CTA)
            int* sDec = reinterpret_cast<int*>(sWn + E);   // (p1 << 16 | p0), -1: not routed here
            float* sZ0 = reinterpret_cast<float*>(sDec + kGateSubMax);
            for (int t = tid; t < ts; t += kThreads) {
                int p0 = 0, p1 = 0;
                float z0 = 0.0f;
                const int r = route_decide_thread(P, g.sL + t * Lp, tokA + s0 + t, t, g, sWn, &s_np, &p0, &p1, &z0);
                sDec[t] = r == 1 ? (p0 | ((P.k == 2 ? p1 : 0) << 16)) : -1;
                sZ0[t] = z0;
                if (r == 2) g.sFull[atomicAdd(&s_nfull, 1)] = tokA + s0 + t;
            }
            __syncthreads();
            if (tid == 0) R.trace[(size_t)cta * kTracePts + kTrGateDecide] = globaltimer();
            route_softmax(P, R, g, Lp, tokA + s0, ts, sDec, sZ0, cta);
#ifndef FDMOE_NO_PICKW
            if (P.prec == kFP32) {
                const int npc = FD_DBG(kDbgGateNoFlush) ? 0 : min(s_np, kGatePairCap);
                gate_pick_weights(P, R, A, g, tokA + s0, ts, sDec, npc <= kThreads ? npc : 0);
                pairs_done = npc <= kThreads;
            }
#endif
        } else {
            for (int t = warp; t < ts; t += kWarps) {
                const int r = route_certified(P, R, g.sL + t * Ep, tokA + s0 + t, t, g, &s_np);
                if (r == 2 && (tid & 31) == 0) g.sFull[atomicAdd(&s_nfull, 1)] = tokA + s0 + t;
            }
        }
        __syncthreads();
        if (tid == 0) R.trace[(size_t)cta * kTracePts + kTrGateLogits] = globaltimer();
        const int np = min(s_np, kGatePairCap);
        if (np > 0 && !(FD_DBG(kDbgGateNoFlush))) {
            if (!pairs_done) gate_pairs_exact(P, R, A, g, np);   // (the FP32 pick pass ran them already)
            for (int t = warp; t < ts; t += kWarps) {
                if (g.sTNC[t] == 0) continue;
                ++n_pair_tok;
                if (!route_resolve(P, R, g.sL + t * Lp, tokA + s0 + t, t, g) && (tid & 31) == 0)
                    g.sFull[atomicAdd(&s_nfull, 1)] = tokA + s0 + t;
            }
            __syncthreads();
        }
        if (tid == 0) R.trace[(size_t)cta * kTracePts + kTrGatePairs] = globaltimer();
        const int nf = s_nfull;
        if (nf > 0 && !(FD_DBG(kDbgGateNoFlush))) {   // ties / near-ties / overflow: the reference chain for all E
            // Listed rank-wide: every CTA computes a share of their chains after the gate barrier
            // (full_exact_distributed); only a list overflow is computed here by the owner alone.
            __shared__ int s_base;
            if (tid == 0) s_base = (int)atomicAdd(&R.full_ctr[0], (uint32_t)nf);
            __syncthreads();
            const int base = s_base;
            if (base + nf <= kFullCap) {
                for (int t = tid; t < nf; t += kThreads) R.full_list[base + t] = g.sFull[t];
            } else {
                if (tid == 0) atomicSub(&R.full_ctr[0], (uint32_t)nf);
                gate_full_exact(P, R, A, g, nf);
                for (int t = warp; t < nf; t += kWarps) route_exact(P, R, g.sL + t * Ep, g.sFull[t], g.sCnt, g.tab);
            }
            n_full += nf;
        }
        __syncthreads();
    }
    if (tid == 0) {
        stat[3] += n_full;
        R.trace[(size_t)cta * kTracePts + kTrGateFull] = globaltimer();
        R.trace[(size_t)cta * kTracePts + kTrGateNFull] = n_full;
    }
    if ((tid & 31) == 0 && n_pair_tok) atomicAdd(&stat[4], n_pair_tok);
    __syncthreads();
    for (int e = tid; e < E; e += kThreads) R.cnt_cta[(size_t)cta * E + e] = g.sCnt[e];
}

// ================================================================ phase 2: slots + dispatch
__device__ void dispatch_phase(const LaunchParams& P, const RankCtx& R, const float* __restrict__ A, int cta,
                               uint8_t* smem) {
    const int E = P.E, H = P.H, S = P.S, K = P.k, C = P.C;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int* sRun = reinterpret_cast<int*>(smem);     // running slot counter per expert
    int* sN = sRun + kMaxExperts;                  // n_e = min(total, C)
    const uint32_t par = P.epoch & 1u;
    const uint64_t sig_hi = (uint64_t)P.epoch << 32;
    const uint64_t t_disp0 = globaltimer();
    const bool straggle = P.straggler_rank == R.rank;
    // straggler (runtime.hpp:358-362): packet e's signal is held back until its cumulative delay
    auto hold = [&](int e) {
        if (!straggle) return;
        const uint64_t until = t_disp0 + R.delay_ns[e];
        while (globaltimer() < until) {
            if (ld_volatile_u32(P.abort_flag)) return;
            __nanosleep(1000);
        }
    };

    // Per-expert prefix of the per-CTA pick counts: (expert, CTA-range part) per thread so every thread of the
    // CTA has loads in flight (16 at a time): a thread per expert walking all 148 CTAs paid ~19 L2 round trips.
    const int parts = E <= kThreads ? min(8, kThreads / E) : 1;
    int* sPb = sRun + 2 * kMaxExperts;        // [parts][E] partial base (CTAs < cta) and total
    int* sPt = sPb + 8 * kMaxExperts;
    {
        const int per = (P.ctas_per_rank + parts - 1) / parts;
        for (int i = tid; i < parts * E; i += kThreads) {
            const int e = i % E, part = i / E;
            const int c_lo = part * per, c_hi = min(P.ctas_per_rank, c_lo + per);
            int base = 0, tot = 0;
            for (int c0 = c_lo; c0 < c_hi; c0 += 16) {
                int v[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) v[u] = c0 + u < c_hi ? __ldcg(R.cnt_cta + (size_t)(c0 + u) * E + e) : 0;
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    if (c0 + u < cta) base += v[u];
                    tot += v[u];
                }
            }
            sPb[part * E + e] = base;
            sPt[part * E + e] = tot;
        }
    }
    __syncthreads();
    for (int e = tid; e < E; e += kThreads) {
        int base = 0, tot = 0;
        for (int part = 0; part < parts; ++part) { base += sPb[part * E + e]; tot += sPt[part * E + e]; }
        const int n = min(tot, C);
        sRun[e] = base;
        sN[e] = n;
        if (cta == 0) {
            R.slot_counts[e] = n;
            for (int s = n; s < C; ++s) {
                R.tbl_tok[(size_t)e * C + s] = -1;
                R.tbl_w[(size_t)e * C + s] = 0.0f;
            }
            if (n == 0) {   // zero-row packets still signal (runtime.hpp:328-331)
                const int q = e / P.El, le = e % P.El;
                unsigned long long* f = reinterpret_cast<unsigned long long*>(R.peer_heap[q] + R.hl.dflag[par]) +
                                        (size_t)le * P.P + R.rank;
                hold(e);
                st_release_sys(f, sig_hi);
                emit_event(P, R, kEvDispatchPut, cta, 0, globaltimer(), 0, R.rank, le, -1, -1, q, 0);
            }
        }
    }
    __syncthreads();
    if (tid == 0) R.trace[(size_t)cta * kTracePts + kTrPrefix] = globaltimer();

    int tokA, tokB, b0, b1;
    gate_token_range(P, cta, tokA, tokB, b0, b1);

    // slot assignment in ascending token order: slot = (picks of e by earlier CTAs) + (by earlier
    // blocks of this CTA) + (by earlier tokens of this block) -- exactly the sequential counter of
    // gate.hpp:94-103. Blocks go 12 at a time, one warp each: (A) per-block pick counts per expert,
    // (B) exclusive prefix over the group's blocks on top of the running counter, (C) each warp ranks
    // its block's picks (lane = token) and writes slots / T_phi.
    int* sGrp = sRun + 8 * kMaxExperts;   // [kWarps][E] pick counts of the group's blocks
    constexpr int kWarps = kThreads / 32;
    for (int g0 = b0; g0 < b1; g0 += kWarps) {
        const int blk = g0 + warp;
        const bool wv = blk < b1;
        const int tok = blk * kGateTok + lane;
        const bool valid = wv && lane < kGateTok && tok < S;
        for (int i = tid; i < kWarps * E; i += kThreads) sGrp[i] = 0;
        __syncthreads();
        int mye[8];
        float myw[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            mye[j] = (valid && j < K) ? R.pick_e[(size_t)tok * K + j] : -1;
            myw[j] = (valid && j < K) ? R.pick_w[(size_t)tok * K + j] : 0.0f;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (j < K && valid) atomicAdd(&sGrp[warp * E + mye[j]], 1);
        __syncthreads();
        for (int e = tid; e < E; e += kThreads) {   // (B): counts -> bases, running counter advances
            int run = sRun[e];
            for (int w = 0; w < kWarps; ++w) {
                const int c = sGrp[w * E + e];
                sGrp[w * E + e] = run;
                run += c;
            }
            sRun[e] = run;
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < 8; ++j) {   // (C)
            if (j >= K) break;
            const int e = mye[j];
            int rank = 0;
            for (int t2 = 0; t2 < kGateTok; ++t2) {
#pragma unroll
                for (int j2 = 0; j2 < 8; ++j2) {
                    if (j2 >= K) break;
                    const int e2 = __shfl_sync(0xffffffffu, mye[j2], t2);
                    if (t2 < lane && e2 == e) ++rank;
                }
            }
            if (valid) {
                const int slot = sGrp[warp * E + e] + rank;
                if (slot < C) {
                    R.pick_slot[(size_t)tok * K + j] = slot;
                    R.tbl_tok[(size_t)e * C + slot] = tok;
                    R.tbl_w[(size_t)e * C + slot] = myw[j];
                } else {
                    R.pick_slot[(size_t)tok * K + j] = -1;
                }
            }
        }
        __syncthreads();   // sGrp is reused by the next group
    }
    // these blocks' picks/slots/weights are final (every warp's writes precede the bar.sync above):
    // fence + per-block epoch flags, which the combine (any CTA of this rank) acquires
    for (int blk = b0 + tid; blk < b1; blk += kThreads) {
        __threadfence();
        st_release_gpu_u32(R.blk_ready + blk, P.epoch);
    }
    __syncthreads();
}

// Row push (runtime.hpp:341-372), after a second rank barrier (the slot table T_phi is complete):
// the kept rows of this rank, flattened in (expert, slot) order, are split evenly across its CTAs.
// Balanced — with slots taken in ascending token order, the low token ranges own almost every kept
// row, so pushing by token range left half the CTAs idle — and progressive: CTA c covers a
// contiguous run of experts, so the first experts' packets complete (and their FFN tiles start)
// while later experts are still in flight. One warp per row, 16-byte peer stores, tf32 hi/lo split
// (FP32) or bf16; the CTA completing a packet publishes its release signal (pgas.hpp:99-113).
constexpr int kPushUnroll = 8;

__device__ void push_phase(const LaunchParams& P, const RankCtx& R, const float* __restrict__ A, int cta,
                           uint8_t* smem) {
    const int E = P.E, H = P.H, C = P.C;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int* sN = reinterpret_cast<const int*>(smem) + kMaxExperts;   // n_e (dispatch_phase)
    int* sOff = reinterpret_cast<int*>(smem) + 3 * kMaxExperts;        // [E + 1] prefix of n_e
    int* sMine = sOff + kMaxExperts + 1;                                // rows of e pushed by this CTA
    const uint32_t par = P.epoch & 1u;
    const uint64_t sig_hi = (uint64_t)P.epoch << 32;
    const uint64_t t_disp0 = globaltimer();
    const bool straggle = P.straggler_rank == R.rank;
    // straggler (runtime.hpp:358-362): packet e's signal is held back until its cumulative delay
    auto hold = [&](int e) {
        if (!straggle) return;
        const uint64_t until = t_disp0 + R.delay_ns[e];
        while (globaltimer() < until) {
            if (ld_volatile_u32(P.abort_flag)) return;
            __nanosleep(1000);
        }
    };
    if (tid == 0) {
        int acc = 0;
        for (int e = 0; e < E; ++e) { sOff[e] = acc; acc += sN[e]; }
        sOff[E] = acc;
    }
    __syncthreads();
    const int total = sOff[E];
    const int f0 = (int)((long long)total * cta / P.ctas_per_rank);
    const int f1 = (int)((long long)total * (cta + 1) / P.ctas_per_rank);
    for (int e = tid; e < E; e += kThreads) sMine[e] = max(0, min(f1, sOff[e + 1]) - max(f0, sOff[e]));
    const int H4 = H >> 2;
    for (int f = f0 + warp; f < f1; f += kThreads / 32) {
        int e = 0;   // expert of flattened row f: last e with sOff[e] <= f (binary search)
        for (int lo = 0, hi = E; lo < hi;) {
            const int mid = (lo + hi + 1) >> 1;
            if (mid < E && sOff[mid] <= f) { e = mid; lo = mid; } else hi = mid - 1;
        }
        const int slot = f - sOff[e];
        const int tok = R.tbl_tok[(size_t)e * C + slot];
        const int q = e / P.El, le = e % P.El;
        const size_t row = (size_t)le * P.RP + (size_t)R.rank * P.Cp + slot;
        const float4* src = reinterpret_cast<const float4*>(A + (size_t)tok * H);
        uint8_t* hb = R.peer_heap[q];
        // kPushUnroll 16-byte loads per lane are issued before any store: one HBM latency per group
        // instead of one per element (the loop would otherwise be latency-bound at ~1 us per load)
        for (int c0 = lane; c0 < H4; c0 += 32 * kPushUnroll) {
            float4 v[kPushUnroll];
#pragma unroll
            for (int u = 0; u < kPushUnroll; ++u)
                if (c0 + 32 * u < H4) v[u] = __ldg(src + c0 + 32 * u);
            if (P.prec == kFP32) {
                float4* dhi = reinterpret_cast<float4*>(hb + R.hl.x[par][0]) + row * H4;
                float4* dlo = reinterpret_cast<float4*>(hb + R.hl.x[par][1]) + row * H4;
                uint2* dlb = reinterpret_cast<uint2*>(hb + R.hl.x[par][1]) + row * (size_t)(H / 2);
#pragma unroll
                for (int u = 0; u < kPushUnroll; ++u) {
                    const int c = c0 + 32 * u;
                    if (c >= H4) break;
                    float4 h, l;
                    h.x = tf32_hi(v[u].x); h.y = tf32_hi(v[u].y); h.z = tf32_hi(v[u].z); h.w = tf32_hi(v[u].w);
                    l.x = __fsub_rn(v[u].x, h.x); l.y = __fsub_rn(v[u].y, h.y);
                    l.z = __fsub_rn(v[u].z, h.z); l.w = __fsub_rn(v[u].w, h.w);
                    dhi[c] = h;
                    if (kCorrBf16) {   // plane 1: [bf16 x_hi | bf16 x_lo] per 32-k group (16 uint2 per group)
                        const size_t gb = (size_t)(c >> 3) * 16 + (c & 7);
                        dlb[gb] = make_uint2(pack_bf16x2(h.x, h.y), pack_bf16x2(h.z, h.w));
                        dlb[gb + 8] = make_uint2(pack_bf16x2(l.x, l.y), pack_bf16x2(l.z, l.w));
                    } else {
                        dlo[c] = l;
                    }
                }
            } else {
                uint2* d = reinterpret_cast<uint2*>(hb + R.hl.x[par][0]) + row * H4;
#pragma unroll
                for (int u = 0; u < kPushUnroll; ++u) {
                    if (c0 + 32 * u >= H4) break;
                    __nv_bfloat162 p0 = __floats2bfloat162_rn(v[u].x, v[u].y);
                    __nv_bfloat162 p1 = __floats2bfloat162_rn(v[u].z, v[u].w);
                    uint2 o;
                    o.x = *reinterpret_cast<uint32_t*>(&p0);
                    o.y = *reinterpret_cast<uint32_t*>(&p1);
                    d[c0 + 32 * u] = o;
                }
            }
        }
    }
    __syncthreads();
    // one system-scope fence orders every row this CTA pushed (cumulative through bar.sync) before
    // the packet counters below; the last CTA to complete a packet publishes its signal
    if (tid == 0) __threadfence_system();
    __syncthreads();
    for (int e = tid; e < E; e += kThreads) {
        const int kept = sMine[e] + (FD_DBG(kDbgInjectOversub) && e == 0 && cta == 0 && sMine[e] > 0 ? 1 : 0);
        if (kept <= 0) continue;
        const uint32_t old = atomicAdd(&R.sent[e], (uint32_t)kept);
        if ((int)(old + kept) == sN[e]) {
            __threadfence_system();
            const int q = e / P.El, le = e % P.El;
            unsigned long long* f =
                reinterpret_cast<unsigned long long*>(R.peer_heap[q] + R.hl.dflag[par]) + (size_t)le * P.P + R.rank;
            hold(e);
            st_release_sys(f, sig_hi | (uint32_t)sN[e]);
            emit_event(P, R, kEvDispatchPut, cta, 0, globaltimer(), 0, R.rank, le, -1, -1, q, sN[e]);
        } else if ((int)(old + kept) > sN[e]) {
            raise_error(P, R, kErrProtocol, 200, e, old + kept);
        }
    }
}

// ================================================================ phase 3: expert FFN
// Tile = (local expert le, feature block nb of 128 outputs, row tile m of 128 received tokens):
//   D[f][t] = sum_k W^T[f][k] * X[t][k]     (GEMM0: K = H, W = W1;  GEMM1: K = D, W = W2, X = C1)
// A operand (weights) lives in TMEM: the producer TMA-loads raw FP32 (or bf16) weight rows into a
// SWIZZLE_128B smem ring; 4 converter warps read them (LDS), split FP32 into tf32 hi/lo in
// registers and tcgen05.st both parts into the TMEM stage — weights cross HBM once at 4 bytes per
// element. B operand (tokens, already hi/lo-split by the sender at dispatch) is TMA-staged in a
// SWIZZLE_128B smem ring. 3xTF32: lo*hi + hi*lo + hi*hi per k-step (product-major), FP32
// accumulation in double-buffered TMEM accumulators. (runtime.hpp:652-699, tiled_blas.hpp:80-96)
constexpr int kGateTask = 2;
struct Task {
    int type;   // 0 = GEMM0, 1 = GEMM1, 2 = gate logits tile (kGateTask), -1 = end
                // gate tile: m = first token, nb = expert block, cnt[0] = valid token rows
    int le, nb, m;
    int nsrc, src0;
    int cnt[kMaxSrcPerTile];   // valid rows per packet in the tile
    uint64_t t0;               // event log: dependencies resolved, operand streaming starts
};

// K extent of a task: GEMM0 and gate tiles contract over H, GEMM1 over D.
__device__ __forceinline__ int task_k(const LaunchParams& P, int type) { return type == 1 ? P.D : P.H; }

// Stage = BK elements of K = NATOM SWIZZLE_128B atoms (128-byte rows). One wait + one commit per
// stage: ready[s] completes when the token TMA bytes landed AND the 4 converter warps stored the
// weight stage into TMEM; done[s] is committed by the MMA warp when the stage's MMAs retire.
// (The tensor queue is ~1 instruction deep, so per-stage bookkeeping is paid as a bubble; a stage
// carries 24 MMAs in FP32 mode.)
template <int PREC>
struct GemmCfg {
    static constexpr int ESZ = PREC == kFP32 ? 4 : 2;
    static constexpr int ATOM_K = 128 / ESZ;                    // K elements per 128-byte atom row
    static constexpr int NATOM = 2;
    static constexpr int BK = ATOM_K * NATOM;                   // K per stage (64 fp32 / 128 bf16)
    static constexpr int ATOM_BYTES = 128 * 128;                // 128 rows x 128 B
    static constexpr int PLANE_BYTES = ATOM_BYTES * NATOM;      // one operand plane per stage (32 KB)
    static constexpr int PLANES = PREC == kFP32 ? 2 : 1;        // hi/lo split of the token operand
    static constexpr int STAGE_BYTES = PLANE_BYTES * PLANES;   // token stage
    static constexpr int STAGES = PREC == kFP32 ? 2 : 3;       // token smem ring == weight TMEM ring
    static constexpr int W_BYTES = PLANE_BYTES;                 // weight stage (raw FP32 / bf16)
    static constexpr int WSTAGES = PREC == kFP32 ? 2 : 3;      // weight smem ring (TMA -> converters)
    static constexpr int KSTEP = PREC == kFP32 ? 8 : 16;       // K per tcgen05.mma
    static constexpr int KSTEPS = BK / KSTEP;                   // 8
    static constexpr int STEPS_PER_ATOM = ATOM_K / KSTEP;       // 4
    // TMEM weight operand. bf16: one slot per stage (BK/2 columns), STAGES deep, after the two
    // accumulators. FP32: a 2-deep ring of half-stages (one 128-byte atom = 32 K: 32 hi + 32 lo
    // columns) after the two accumulators and the tile's correction accumulator (kTmemCorr).
    static constexpr int A_COLS = PREC == kFP32 ? 2 * ATOM_K : BK / 2;
    static constexpr int A_SLOTS = PREC == kFP32 ? 2 : STAGES;
    static constexpr uint32_t IDESC = umma_idesc(PREC == kFP32 ? 2u : 1u, kBF, kNT);
    static constexpr int W_OFF = STAGE_BYTES * STAGES;
    static constexpr int RING_BYTES = W_OFF + W_BYTES * WSTAGES;
    static constexpr uint32_t TMEM_A0 = PREC == kFP32 ? kTmemCorr + kNT : kAccStages * kNT;
    static_assert(TMEM_A0 + A_SLOTS * A_COLS <= 512, "TMEM budget");
};

// dynamic smem: [max(gate scratch, FFN rings)] [GemmCtrl]
// (the tensor-core gate runs the FP32 pipeline in either precision's kernel, so the region covers both rings;
//  the FFN and the gate each get their own control block)
constexpr int cmax(int a, int b) { return a > b ? a : b; }
template <int PREC>
struct SmemPlan {
    static constexpr int REGION =
        (cmax(kGateSmemBytes, cmax(GemmCfg<kFP32>::RING_BYTES, GemmCfg<kBF16>::RING_BYTES)) + 1023) / 1024 * 1024;
    static constexpr int CTRL_GATE = REGION + 1024;
    static constexpr int TOTAL = REGION + 2048 /* ctrl: FFN, gate */ + 1024 /* alignment slack */;
};

struct GemmCtrl {
    uint64_t ready[8], done[8];                      // token smem ring (+ bf16: the weight TMEM ring, same stages)
    uint64_t afull[2], aempty[2];                    // FP32: weight TMEM half-stage ring (converters <-> MMA)
    uint64_t cempty;                                 // FP32: correction accumulator folded (epilogue -> MMA)
    uint64_t wfull[8], wempty[8];                    // weight smem ring (producer -> converters)
    uint64_t tfull[kAccStages], tempty[kAccStages];  // accumulators
    uint64_t qfull[kTaskRing], qempty[kTaskRing];    // task ring
    uint64_t sfull[kTaskRing], sempty[kTaskRing];    // epilogue -> signal warp (finished tiles)
    uint64_t pp[2];                                  // FP32 FFN issuer hand-off: pp[i] = "the other warp issued"
    uint32_t tmem_base;
    uint32_t pp_corr;                                // FP32 FFN: correction accumulator state handed h=0 -> h=1
    uint32_t pp_cph;                                 //   and the cempty parity, handed between the issuers
    uint32_t pad;
    Task ring[kTaskRing];
    Task sring[kTaskRing];                           // finished tiles awaiting their release signals
};
static_assert(sizeof(GemmCtrl) <= 1024, "GemmCtrl fits the control area");
constexpr int kTaskConsumers = 1 + 4 + 1;   // MMA warp, 4 converter warps, epilogue
template <int PREC>
struct TaskConsumers {   // FP32 FFN: two MMA issuer warps
    static constexpr int N = kTaskConsumers + (PREC == kFP32 ? 1 : 0);
};
template <int PREC>
struct MmaCommits {      // arrivals per accumulator (tfull): one commit per issuer warp
    static constexpr int N = PREC == kFP32 ? 2 : 1;
};
template <int PREC>
struct ReadyCount {   // bf16: producer (expect_tx) + 4 converter warps; FP32: producer (tokens only)
    static constexpr int N = PREC == kFP32 ? 1 : 1 + 4;
};

__device__ __forceinline__ void decode_task(const LaunchParams& P, uint32_t t, uint32_t n_g0, Task& tk) {
    const bool g1 = t >= n_g0;
    if (g1) t -= n_g0;
    const uint32_t nbk = g1 ? (uint32_t)P.NB1 : (uint32_t)P.NB0;
    const uint32_t per_e = nbk * P.MT;
    tk.type = g1 ? 1 : 0;
    tk.le = t / per_e;
    const uint32_t r = t % per_e;
    tk.nb = r / P.MT;   // consecutive tasks share the weight tile (e, nb) across row tiles m
    tk.m = r % P.MT;
}

// Packets intersecting row tile m of an expert's receive region, and their signalled rows.
// Returns total valid rows, or -1 on abort.
__device__ int resolve_tile_rows(const LaunchParams& P, const RankCtx& R, Task& tk) {
    const uint32_t par = P.epoch & 1u;
    const unsigned long long* dflag =
        reinterpret_cast<const unsigned long long*>(R.peer_heap[R.rank] + R.hl.dflag[par]) + (size_t)tk.le * P.P;
    int total = 0;
    if (P.Cp >= kBM) {
        const int per = P.Cp / kBM;
        const int src = tk.m / per, rb = tk.m % per;
        tk.nsrc = 1;
        tk.src0 = src;
        const int64_t n = wait_epoch_flag(P, R, dflag + src, 300);
        if (n < 0) return -1;
        const int v = max(0, min(kBM, (int)n - rb * kBM));
        tk.cnt[0] = v;
        total = v;
    } else {
        const int per = kBM / P.Cp;
        const int s0 = tk.m * per;
        const int s1 = min(P.P, s0 + per);
        tk.nsrc = s1 - s0;
        tk.src0 = s0;
        for (int s = s0; s < s1; ++s) {
            const int64_t n = wait_epoch_flag(P, R, dflag + s, 301);
            if (n < 0) return -1;
            tk.cnt[s - s0] = (int)n;
            total += (int)n;
        }
    }
    return total;
}

// Wait accounting (device trace slots 8..15): cycles each role spends blocked on a pipeline edge.
// Compiled in only for profiling builds (-DFDMOE_WAIT_ACCOUNTING, tools/phase_trace.py): two clock reads
// around every pipeline wait cost the single MMA issuer measurable tensor-pipe bubbles.
#ifdef FDMOE_WAIT_ACCOUNTING
#define FD_TIMED_WAIT(acc, expr)              \
    ({                                        \
        const long long _t0 = clk();          \
        const bool _ok = (expr);              \
        acc += clk() - _t0;                   \
        _ok;                                  \
    })
#else
#define FD_TIMED_WAIT(acc, expr) (expr)
#endif
// clock reads of the role-level profiling counters (trace slots, chunk log): compiled out of the product
__device__ __forceinline__ long long pclk() {
#ifdef FDMOE_WAIT_ACCOUNTING
    return clk();
#else
    return 0;
#endif
}

// warp 10, one lane: fetch tiles, resolve dependencies, stream both operands
template <int PREC>
__device__ void gemm_producer(const LaunchParams& P, const RankCtx& R, uint8_t* ring, GemmCtrl& G,
                              unsigned long long* trace) {
    using Cfg = GemmCfg<PREC>;
    long long w_w = 0, w_x = 0, t_fetch = 0;
    const uint32_t n_g0 = (uint32_t)P.El * P.NB0 * P.MT;
    const uint32_t n_g1 = (uint32_t)P.El * P.NB1 * P.MT;
    const uint32_t par = P.epoch & 1u;
    int stage = 0, wstage = 0;
    uint32_t phase = 0, wphase = 0;
    int q = 0;
    uint32_t qphase = 0;
    for (int i = 0; i < Cfg::PLANES; ++i) {
        tma_prefetch(&R.tm_x[par][i]);
        tma_prefetch(&R.tm_c1[i]);
    }
    tma_prefetch(&R.tm_w1);
    tma_prefetch(&R.tm_w2);
    // weights stream through once (evict first); token / C1 tiles are re-read by the other feature
    // blocks of the same row tile (keep)
    const uint64_t pol_w = l2_policy_evict_first();
    const uint64_t pol_x = FD_DBG(kDbgEvictNormal) ? l2_policy_evict_normal() : l2_policy_evict_last();
    // Task accounting (runtime.hpp:122-165, 407-415 restated for the static tile grid): the bound starts at
    // every (expert, row tile, feature block) task of both GEMMs and self-corrects when a row tile's dispatch
    // signals resolve: an empty row tile removes its NB0 + NB1 tasks. Each row tile is corrected exactly once,
    // by the producer that claims its (GEMM0, nb = 0) task. scheduled = non-empty tasks handed to the pipeline.
    long long bound_delta = 0, scheduled = 0, tiles_resolved = 0;
    while (true) {
        const long long tf0 = pclk();
        const uint32_t t = atomicAdd(R.gemm_head, 1u);
        Task tk;
        bool end = t >= n_g0 + n_g1;
        if (!end) {
            decode_task(P, t, n_g0, tk);
            const int rows = resolve_tile_rows(P, R, tk);
            if (rows >= 0 && tk.type == 0 && tk.nb == 0) {
                ++tiles_resolved;
                if (rows == 0) bound_delta -= P.NB0 + P.NB1;
            }
            if (rows < 0) end = true;
            else if (rows == 0) continue;   // empty row tile: no GEMM0/GEMM1 work exists for it
            else if (tk.type == 1) {
                if (!wait_counter(P, R, R.g0done + (size_t)tk.le * P.MT + tk.m, (uint32_t)P.NB0, 302)) end = true;
            }
        }
        t_fetch += pclk() - tf0;
        if (!mbar_wait(&G.qempty[q], qphase ^ 1u, P.abort_flag)) end = true;
        if (end) {
            G.ring[q].type = -1;
            mbar_arrive(&G.qfull[q]);
            trace[kWaitProdW] = w_w;
            trace[kWaitProdX] = w_x;
            trace[kProdFetch] = t_fetch;
            atomicAdd(R.stats + 5, (unsigned long long)bound_delta);   // two's complement: a signed sum
            atomicAdd(R.stats + 6, (unsigned long long)scheduled);
            atomicAdd(R.stats + 7, (unsigned long long)tiles_resolved);
            return;
        }
        ++scheduled;
        tk.t0 = P.trace_events ? globaltimer() : 0;
        G.ring[q] = tk;
        mbar_arrive(&G.qfull[q]);
        if (++q == kTaskRing) { q = 0; qphase ^= 1u; }

        // token rows were written by the generic proxy (peer dispatch stores / GEMM0 epilogues)
        // and acquired above; order them before the async-proxy (TMA) reads
        fence_proxy_async_global();
        const CUtensorMap* tb[2];
        const CUtensorMap* tw;
        int yw;
        if (tk.type == 0) { tb[0] = &R.tm_x[par][0]; tb[1] = &R.tm_x[par][1]; tw = &R.tm_w1; yw = tk.le * P.D; }
        else { tb[0] = &R.tm_c1[0]; tb[1] = &R.tm_c1[1]; tw = &R.tm_w2; yw = tk.le * P.H; }
        yw += tk.nb * kBF;
        const int y = tk.le * P.RP + tk.m * kBM;
        const int nk = (task_k(P, tk.type) + Cfg::BK - 1) / Cfg::BK;
        for (int kb = 0; kb < nk; ++kb) {
            // weight tile first: the converter warps need it one step before the MMA does
            if (!FD_TIMED_WAIT(w_w, mbar_wait(&G.wempty[wstage], wphase ^ 1u, P.abort_flag))) return;
            if (FD_DBG(kDbgNoWTma)) mbar_arrive(&G.wfull[wstage]);
            else {
                mbar_expect_tx(&G.wfull[wstage], Cfg::W_BYTES);
#pragma unroll
                for (int at = 0; at < Cfg::NATOM; ++at)
                    tma_load_2d_hint(ring + Cfg::W_OFF + wstage * Cfg::W_BYTES + at * Cfg::ATOM_BYTES, tw,
                                     &G.wfull[wstage], kb * Cfg::BK + at * Cfg::ATOM_K, yw, pol_w);
            }
            if (++wstage == Cfg::WSTAGES) { wstage = 0; wphase ^= 1u; }

            uint8_t* st = ring + stage * Cfg::STAGE_BYTES;
            if constexpr (PREC == kFP32) {
                // FP32: the token ring is 2 stages x 2 atoms with one ready/done pair per ATOM (slot 2*stage + at):
                // the two MMA issuer warps each consume one atom of every stage, so an atom's slot refills as soon
                // as its 12 MMAs retire -- 3 of the 4 slots can be in flight instead of 1 of 2 stages (the token
                // TMA from L2 is latency- not bandwidth-bound: lts__throughput 32 %, tools/dev ncu r02).
#pragma unroll
                for (int at = 0; at < Cfg::NATOM; ++at) {
                    const int j = stage * Cfg::NATOM + at;
                    if (!FD_TIMED_WAIT(w_x, mbar_wait(&G.done[j], phase ^ 1u, P.abort_flag))) return;
                    if (FD_DBG(kDbgNoXTma)) { mbar_arrive(&G.ready[j]); continue; }
                    mbar_expect_tx(&G.ready[j], Cfg::PLANES * Cfg::ATOM_BYTES);
#pragma unroll
                    for (int pl = 0; pl < Cfg::PLANES; ++pl)
                        tma_load_2d_hint(st + pl * Cfg::PLANE_BYTES + at * Cfg::ATOM_BYTES, tb[pl], &G.ready[j],
                                         kb * Cfg::BK + at * Cfg::ATOM_K, y, pol_x);
                }
                if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1u; }
                continue;
            }
            if (!FD_TIMED_WAIT(w_x, mbar_wait(&G.done[stage], phase ^ 1u, P.abort_flag))) return;
            if (FD_DBG(kDbgNoXTma)) mbar_arrive(&G.ready[stage]);
            else {
                mbar_expect_tx(&G.ready[stage], Cfg::STAGE_BYTES);
#pragma unroll
                for (int pl = 0; pl < Cfg::PLANES; ++pl)
#pragma unroll
                    for (int at = 0; at < Cfg::NATOM; ++at)
                        tma_load_2d_hint(st + pl * Cfg::PLANE_BYTES + at * Cfg::ATOM_BYTES, tb[pl], &G.ready[stage],
                                         kb * Cfg::BK + at * Cfg::ATOM_K, y, pol_x);
            }
            if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1u; }
        }
    }
}

// warps 0-3: weight tile (TMA-staged in smem, SWIZZLE_128B) -> registers -> tf32 hi/lo split ->
// tcgen05.st into the TMEM weight ring. Thread (warp 4+q, lane l) owns feature row r = 32q+l of
// the tile = TMEM lane r; in atom a its 16-byte chunk c sits at a*16K + r*128 + ((c ^ (r & 7)) << 4),
// so a warp's 128-bit loads are bank-conflict free.
// Gate tiles (kGateTask, FP32 config) stream token rows through the same converter path; the
// converters also accumulate each token row's sum of squares into gate_na (certified-gate bound).
// Gate tiles also form their A words (x_hi tf32 | x_lo) in registers before the slot wait and store them with two
// st32, like the FFN. Measured (tools/ab.py, product library, three boxes): FP32 c4 1.498 -> 1.468 ms, c2 0.412 ->
// 0.400 ms, bf16 c4 0.650 -> 0.646 ms. The development build's gate timing (tools/dev/gate_only.py) did not move and
// the product build's phase trace puts the gain in the FFN phase (~1.20 -> ~1.18 ms): the gate and the FFN share
// this converter function, so it is a code-generation effect on the shared loop. -DFDMOE_GATE_PRECONV=0: the old path.
#ifndef FDMOE_GATE_PRECONV
#define FDMOE_GATE_PRECONV 1
#endif
constexpr bool kGatePreConv = FDMOE_GATE_PRECONV != 0;
#ifndef FDMOE_GATE_NORM4
#define FDMOE_GATE_NORM4 1
#endif
template <int PREC>
__device__ void gemm_wconvert(const LaunchParams& P, uint8_t* ring, GemmCtrl& G, unsigned long long* trace,
                              unsigned long long* clog, double* gate_na = nullptr) {
    using Cfg = GemmCfg<PREC>;
    long long w_w = 0, w_a = 0;
    int nlog = 0;
    const int lane = threadIdx.x & 31;
    const int wq = (threadIdx.x >> 5) - kWarpConv0;
    const int r = wq * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(wq * 32) << 16;
    int q = 0;
    uint32_t qphase = 0;
    int ast = 0, wst = 0;
    uint32_t aphase = 0, wphase = 0;
    const uint32_t tmem = G.tmem_base;
    while (true) {
        if (!mbar_wait(&G.qfull[q], qphase, P.abort_flag)) return;
        const int type = G.ring[q].type;
        const int g_tok0 = G.ring[q].m, g_valid = G.ring[q].cnt[0];
        const bool g_norm = type == kGateTask && G.ring[q].nb == 0 && gate_na != nullptr;
        __syncwarp();
        if (lane == 0) mbar_arrive(&G.qempty[q]);
        if (++q == kTaskRing) { q = 0; qphase ^= 1u; }
        if (type < 0) {
            if (threadIdx.x == kWarpConv0 * 32 && trace) { trace[kWaitConvW] = w_w; trace[kWaitConvA] = w_a; }
            return;
        }
        const int nk = (task_k(P, type) + Cfg::BK - 1) / Cfg::BK;
        double ss = 0.0;   // gate tile: sum of squares of this row (float per stage, double across stages)
        for (int kb = 0; kb < nk; ++kb) {
            const long long c0 = pclk();
            if (!FD_TIMED_WAIT(w_w, mbar_wait(&G.wfull[wst], wphase, P.abort_flag))) return;
            const long long c1 = pclk();
            const uint8_t* wrow = ring + Cfg::W_OFF + wst * Cfg::W_BYTES + r * 128;
            float4 c[Cfg::NATOM][8];
#pragma unroll
            for (int at = 0; at < Cfg::NATOM; ++at)
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    c[at][i] = *reinterpret_cast<const float4*>(wrow + at * Cfg::ATOM_BYTES + ((i ^ (r & 7)) << 4));
            // the slot is refilled by the async proxy (TMA) as soon as it is released: order these generic
            // loads before that write (without the fence the release can retire before the loaded data
            // returns, and a TMA issued right behind it corrupts rows of this stage -- seen on the gate's
            // second tile, tools/dev/gate_stage_dump.py)
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&G.wempty[wst]);   // values are in registers: slot reusable
            if (++wst == Cfg::WSTAGES) { wst = 0; wphase ^= 1u; }

            const long long c2 = pclk();
            if (PREC == kFP32 && g_norm && !FD_DBG(kDbgGateNoNorm)) {
#if FDMOE_GATE_NORM4
                // four independent 16-FMA chains (the 64-deep chain sat in front of the stage's TMEM stores);
                // |a|^2 only feeds the certificate's rounded-up |a| (sqrt(na (1 + 1e-5))), any order is within it
                float n0 = 0.0f, n1 = 0.0f, n2 = 0.0f, n3 = 0.0f;
#pragma unroll
                for (int at = 0; at < Cfg::NATOM; ++at)
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const float4 v = c[at][i];
                        n0 = __fmaf_rn(v.x, v.x, n0); n1 = __fmaf_rn(v.y, v.y, n1);
                        n2 = __fmaf_rn(v.z, v.z, n2); n3 = __fmaf_rn(v.w, v.w, n3);
                    }
                const float cs = (n0 + n1) + (n2 + n3);
#else
                float cs = 0.0f;
#pragma unroll
                for (int at = 0; at < Cfg::NATOM; ++at)
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const float4 v = c[at][i];
                        cs = __fmaf_rn(v.x, v.x, cs); cs = __fmaf_rn(v.y, v.y, cs);
                        cs = __fmaf_rn(v.z, v.z, cs); cs = __fmaf_rn(v.w, v.w, cs);
                    }
#endif
                ss += (double)cs;
                if (kb + 1 == nk && r < g_valid) gate_na[g_tok0 + r] = ss;
            }
            if constexpr (PREC == kFP32) {
                // one TMEM half-stage per 128-byte atom (32 K values: hi columns [0, 32), lo [32, 64)),
                // each released to the MMA warp on its own so the ring runs half a stage ahead
#pragma unroll
                for (int at = 0; at < Cfg::NATOM; ++at) {
                    // FFN (kCorrBf16): the atom's A operand is formed in registers BEFORE the slot wait, so only
                    // the two TMEM stores sit between the MMAs freeing the slot and the slot refilled (the
                    // converter's aempty -> afull turnaround must fit one 8-MMA half-stage of the other issuer)
                    const bool ffn_b16 = kCorrBf16 && type != kGateTask && !FD_DBG(kDbgNoConvert);
                    // gate tiles: the token atom's tf32 hi / lo words, also formed before the slot wait
                    const bool gate_pre = kGatePreConv && type == kGateTask && !FD_DBG(kDbgNoConvert);
                    uint32_t fhi[32], fcb[32];   // w_hi tf32 | bf16x2(w_lo) (16 words), bf16x2(w_hi) (16 words)
                    if (gate_pre) {
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const float4 v = c[at][i];
                            const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const float hv = tf32_hi(vv[u]);
                                fhi[i * 4 + u] = __float_as_uint(hv);
                                fcb[i * 4 + u] = __float_as_uint(__fsub_rn(vv[u], hv));
                            }
                        }
                    }
                    if (ffn_b16) {
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const float4 v = c[at][i];
                            const float h0 = tf32_hi(v.x), h1 = tf32_hi(v.y), h2 = tf32_hi(v.z), h3 = tf32_hi(v.w);
                            fhi[i * 4 + 0] = __float_as_uint(h0); fhi[i * 4 + 1] = __float_as_uint(h1);
                            fhi[i * 4 + 2] = __float_as_uint(h2); fhi[i * 4 + 3] = __float_as_uint(h3);
                            fcb[i * 2 + 0] = pack_bf16x2(__fsub_rn(v.x, h0), __fsub_rn(v.y, h1));
                            fcb[i * 2 + 1] = pack_bf16x2(__fsub_rn(v.z, h2), __fsub_rn(v.w, h3));
                            fcb[16 + i * 2 + 0] = pack_bf16x2(h0, h1);
                            fcb[16 + i * 2 + 1] = pack_bf16x2(h2, h3);
                        }
                    }
                    const long long a0 = pclk();
                    if (!FD_TIMED_WAIT(w_a, mbar_wait(&G.aempty[ast], aphase ^ 1u, P.abort_flag))) return;
                    const long long a1 = pclk();
                    tc_fence_after();
                    const uint32_t col = tmem + lane_addr + Cfg::TMEM_A0 + ast * Cfg::A_COLS;
                    if (ffn_b16 || gate_pre) {
                        // FFN: w_hi tf32 in [0, 32), bf16x2(w_lo) in [32, 48), bf16x2(w_hi) in [48, 64)
                        // gate: x_hi tf32 in [0, 32), x_lo FP32 in [32, 64)
                        tmem_st32(col, fhi);
                        tmem_st32(col + Cfg::ATOM_K, fcb);
                    }
#pragma unroll
                    for (int h = 0; h < 2; ++h) {   // 16 K values per half atom
                        if (FD_DBG(kDbgNoConvert) || (kCorrBf16 && type != kGateTask) || gate_pre) break;
                        uint32_t hi[16], lo[16];
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const float4 v = c[at][h * 4 + i];
                            const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const float hv = tf32_hi(vv[u]);
                                hi[i * 4 + u] = __float_as_uint(hv);
                                lo[i * 4 + u] = __float_as_uint(__fsub_rn(vv[u], hv));
                            }
                        }
                        tmem_st16(col + h * 16, hi);                  // hi: columns [0, 32)
                        tmem_st16(col + Cfg::ATOM_K + h * 16, lo);    // lo: columns [32, 64)
                    }
                    tmem_wait_st();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&G.afull[ast]);
                    if (clog && threadIdx.x == kWarpConv0 * 32 && type != kGateTask && nlog < 64) {
                        // chunk log (development build), rows [320, 384): per FFN half-stage {weight-stage wait,
                        // A-slot wait, convert + store + arrive, clock at the A wait}
                        unsigned long long* o = clog + 4 * (320 + nlog++);
                        o[0] = at == 0 ? c1 - c0 : 0; o[1] = a1 - a0; o[2] = pclk() - a1; o[3] = a0;
                    }
                    if (++ast == Cfg::A_SLOTS) { ast = 0; aphase ^= 1u; }
                }
                continue;
            }
            if (!FD_TIMED_WAIT(w_a, mbar_wait(&G.done[ast], aphase ^ 1u, P.abort_flag))) return;
            const long long c3 = pclk();
            tc_fence_after();
            const uint32_t col = tmem + lane_addr + Cfg::TMEM_A0 + ast * Cfg::A_COLS;
            if (FD_DBG(kDbgNoConvert)) {
            } else {
#pragma unroll
                for (int at = 0; at < Cfg::NATOM; ++at)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {   // 32 bf16 (16 columns) per half atom
                        uint32_t w[16];
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const float4 v = c[at][h * 4 + i];
                            w[i * 4 + 0] = __float_as_uint(v.x); w[i * 4 + 1] = __float_as_uint(v.y);
                            w[i * 4 + 2] = __float_as_uint(v.z); w[i * 4 + 3] = __float_as_uint(v.w);
                        }
                        tmem_st16(col + at * 32 + h * 16, w);
                    }
            }
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&G.ready[ast]);
            if (clog && lane == 0 && nlog < kChunkLog / 2) {
                // chunklog rows [256, 512): converter warp 0 per stage: wfull wait, LDS, done wait, convert+st
                unsigned long long* o = clog + 4 * (kChunkLog / 2 + nlog++);
                o[0] = c1 - c0; o[1] = c2 - c1; o[2] = c3 - c2; o[3] = pclk() - c3;
            }
            if (++ast == Cfg::STAGES) { ast = 0; aphase ^= 1u; }
        }
    }
}

// warp 11: tcgen05.mma issue. The whole warp runs the issue loop (waits, bookkeeping) converged and one
// elected lane issues each group of MMAs and commits. Operands computed by the converged warp are provably
// warp-uniform, so each UTCHMMA takes them straight from uniform registers; issued from a single-lane branch
// instead, every MMA sat in a compiler waterfall loop (ELECT + R2UR.BROADCAST per operand) and the
// 12-MMA half-stage pattern issued at 100 cycles per MMA instead of the tensor core's 64
// (tools/dev/mma_stream.py: pipe mode 112 vs 2160). One wait (ready) and one commit (done) per stage.
constexpr int kProbeAt = 1;   // MMAs of a stage issued before the next stage's readiness probe

// every lane waits; the warp proceeds only if no lane saw the abort word
__device__ __forceinline__ bool wwait(uint64_t* bar, uint32_t parity, uint32_t* abort_flag) {
    return __all_sync(0xffffffffu, mbar_wait(bar, parity, abort_flag));
}
// non-blocking probe, lane 0's observation for the whole warp (the elected issuer is lane 0)
__device__ __forceinline__ bool wtest(uint64_t* bar, uint32_t parity) {
    return __shfl_sync(0xffffffffu, mbar_test_wait(bar, parity) ? 1 : 0, 0) != 0;
}
__device__ __forceinline__ void wcommit(uint64_t* bar) {
    if (elect_one()) mma_commit(bar);
    __syncwarp();
}

template <int PREC>
struct StageMmas {
    static constexpr int N = PREC == kFP32 ? 3 * GemmCfg<PREC>::KSTEPS : GemmCfg<PREC>::KSTEPS;
};

// MMAs [I0, I1) of a stage in issue order (3xTF32: product-major, then k-step). Everything but the
// stage bases is a compile-time constant, so each MMA is one UTCHMMA plus a couple of uniform adds:
// the single issuing thread must keep up with a ~64-cycle MMA and a tensor queue only ~2 deep.
// bdesc = UMMA descriptor of the stage's token plane 0; smem offsets are added in 16-byte units to
// its start-address field (the shared window is < 256 KB, so the 14-bit field cannot carry).
template <int PREC, int I0, int I1>
__device__ __forceinline__ void issue_stage(uint32_t d_tmem, uint32_t abase, uint64_t bdesc, uint32_t first) {
    using Cfg = GemmCfg<PREC>;
#pragma unroll
    for (int i = I0; i < I1; ++i) {
        const int p = PREC == kFP32 ? i / Cfg::KSTEPS : 0;
        const int ks = PREC == kFP32 ? i % Cfg::KSTEPS : i;
        const uint32_t boff = (ks / Cfg::STEPS_PER_ATOM) * Cfg::ATOM_BYTES +
                              (ks % Cfg::STEPS_PER_ATOM) * Cfg::KSTEP * Cfg::ESZ;
        const uint32_t accum = i == 0 ? (first ^ 1u) : 1u;
        if (PREC == kFP32) {
            // product-major: back-to-back MMAs that read the same TMEM A columns serialize
            // (measured 61% of peak k-step-major vs 100% product-major)
            const uint32_t a_hi = abase + ks * Cfg::KSTEP;
            if (p == 2)        // w_hi * x_hi
                mma_tf32_ts(d_tmem, a_hi, bdesc + (boff >> 4), Cfg::IDESC, accum);
            else if (p == 0)   // w_lo * x_hi
                mma_tf32_ts(d_tmem, a_hi + Cfg::BK, bdesc + (boff >> 4), Cfg::IDESC, accum);
            else               // w_hi * x_lo
                mma_tf32_ts(d_tmem, a_hi, bdesc + ((Cfg::PLANE_BYTES + boff) >> 4), Cfg::IDESC, accum);
        } else {
            mma_bf16_ts(d_tmem, abase + ks * (Cfg::KSTEP / 2), bdesc + (boff >> 4), Cfg::IDESC, accum);
        }
    }
}

// FP32 (3xTF32) MMAs of one half-stage (one 128-byte token atom = 4 k-steps). The tcgen05 FP32
// accumulator rounds toward zero once per MMA (measured: tools/dev/acc_probe.py, profiles/r02_numerics.md),
// so the error of one accumulator grows with the number of MMAs folded into it. The w_hi*x_hi products
// go to the tile's main accumulator (K/8 MMAs), the two correction products (2^-11 smaller) to a
// separate correction accumulator that the epilogue adds in round-to-nearest FP32: a third of the
// main accumulator's truncations, and the corrections' own truncations are 2^-11 smaller.
// CORR_FIRST: corrections then main (back-to-back MMAs never read the same TMEM A columns either way).
template <bool MAIN, bool CORR>
__device__ __forceinline__ void issue_half_fp32(uint32_t d_main, uint32_t d_corr, uint32_t a_half, uint64_t bdesc,
                                                uint32_t idesc, uint32_t main_acc, uint32_t corr_acc) {
    using Cfg = GemmCfg<kFP32>;
    if (CORR) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)   // w_lo * x_hi
            mma_tf32_ts(d_corr, a_half + Cfg::ATOM_K + ks * Cfg::KSTEP, bdesc + ((ks * 32) >> 4), idesc,
                        ks == 0 ? corr_acc : 1u);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)   // w_hi * x_lo
            mma_tf32_ts(d_corr, a_half + ks * Cfg::KSTEP, bdesc + ((Cfg::PLANE_BYTES + ks * 32) >> 4), idesc, 1u);
    }
    if (MAIN) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)   // w_hi * x_hi
            mma_tf32_ts(d_main, a_half + ks * Cfg::KSTEP, bdesc + ((ks * 32) >> 4), idesc, ks == 0 ? main_acc : 1u);
    }
}

// Steady-state half-stage MMAs [I0, I1) of the 12 (both accumulators in use, accumulating): 0-3 w_lo*x_hi and
// 4-7 w_hi*x_lo into the correction accumulator, 8-11 w_hi*x_hi into the main one -- issue_half_fp32's order,
// split so the issuing warp can probe the next half-stage's barriers between the two parts.
template <int I0, int I1>
__device__ __forceinline__ void issue_fp32_steady(uint32_t d_main, uint32_t d_corr, uint32_t a_half, uint64_t bdesc,
                                                  uint32_t idesc) {
    using Cfg = GemmCfg<kFP32>;
#pragma unroll
    for (int i = I0; i < I1; ++i) {
        const int ks = i & 3;
        if (i < 4) mma_tf32_ts(d_corr, a_half + Cfg::ATOM_K + ks * Cfg::KSTEP, bdesc + ((ks * 32) >> 4), idesc, 1u);
        else if (i < 8) mma_tf32_ts(d_corr, a_half + ks * Cfg::KSTEP, bdesc + ((Cfg::PLANE_BYTES + ks * 32) >> 4), idesc, 1u);
        else mma_tf32_ts(d_main, a_half + ks * Cfg::KSTEP, bdesc + ((ks * 32) >> 4), idesc, 1u);
    }
}

// bf16-correction half-stage (kCorrBf16, FFN tiles): MAIN = 4 tf32 MMAs w_hi*x_hi into d_main; CORR = 2 bf16 MMAs
// bf16(w_lo)*bf16(x_hi) then 2 bf16(w_hi)*bf16(x_lo) (K = 16 each) into d_corr. bdesc: the atom's plane-0
// descriptor (plane 1 is PLANE_BYTES further).
template <bool MAIN, bool CORR>
__device__ __forceinline__ void issue_half_b16(uint32_t d_main, uint32_t d_corr, uint32_t a_half, uint64_t bdesc,
                                               uint32_t idesc, uint32_t main_acc, uint32_t corr_acc) {
    using Cfg = GemmCfg<kFP32>;
    constexpr uint32_t kIdescB = umma_idesc(1u, kBF, kNT);
    if (CORR) {
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)   // bf16(w_lo) * bf16(x_hi): A cols 32 + 8 ks, plane-1 bytes 32 ks
            mma_bf16_ts(d_corr, a_half + Cfg::ATOM_K + ks * 8, bdesc + ((Cfg::PLANE_BYTES + ks * 32) >> 4), kIdescB,
                        ks == 0 ? corr_acc : 1u);
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)   // bf16(w_hi) * bf16(x_lo): A cols 48 + 8 ks, plane-1 bytes 64 + 32 ks
            mma_bf16_ts(d_corr, a_half + Cfg::ATOM_K + 16 + ks * 8, bdesc + ((Cfg::PLANE_BYTES + 64 + ks * 32) >> 4),
                        kIdescB, 1u);
    }
    if (MAIN) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)   // w_hi * x_hi (tf32)
            mma_tf32_ts(d_main, a_half + ks * Cfg::KSTEP, bdesc + ((ks * 32) >> 4), idesc, ks == 0 ? main_acc : 1u);
    }
}
// the FFN's half-stage in either format
template <bool MAIN, bool CORR>
__device__ __forceinline__ void issue_half_ffn(uint32_t d_main, uint32_t d_corr, uint32_t a_half, uint64_t bdesc,
                                               uint32_t idesc, uint32_t main_acc, uint32_t corr_acc) {
    if (kCorrBf16) issue_half_b16<MAIN, CORR>(d_main, d_corr, a_half, bdesc, idesc, main_acc, corr_acc);
    else issue_half_fp32<MAIN, CORR>(d_main, d_corr, a_half, bdesc, idesc, main_acc, corr_acc);
}

constexpr int kCorrInMainMax = 2;
struct MmaFp32State {
    int stage = 0, ah = 0;
    uint32_t phase = 0, ahph = 0, cph = 0;
};

// One FP32 tile on the MMA warp (one lane): token stages of 2 atoms (ready/done), weight half-stages
// (afull/aempty), main accumulator d_main, correction accumulator kTmemCorr (freed by the epilogue's
// fold of the previous tile: cempty). The tile's first half-stage issues its main MMAs before waiting
// for the fold, so the fold overlaps them.
__device__ __forceinline__ bool mma_tile_fp32(const LaunchParams& P, uint8_t* ring, GemmCtrl& G, uint32_t tmem,
                                              uint32_t d_main, int nk, uint32_t idesc, MmaFp32State& st,
                                              long long& w_x, unsigned long long* clog = nullptr, int* nlog = nullptr) {
    using Cfg = GemmCfg<kFP32>;
    const uint32_t d_corr = tmem + kTmemCorr;
    // The correction accumulator is free once the epilogue folded the previous tile's corrections
    // (cempty). Until then -- for at most kCorrInMainMax half-stages -- the correction products go into the
    // main accumulator (<= 16 extra truncating MMAs at the start of the sum, where the partial sums are
    // smallest) instead of stalling the tensor pipe; after that the issuer blocks on the fold. The first
    // correction product after the fold starts kTmemCorr fresh. (Unbounded, the main accumulator took
    // every correction of a tile whenever the epilogue ran a tile behind: worst element 1.17x the FP32
    // bound at c4 EP8 -- tests/test_gpu_baseline.py.)
    bool corr_free = false;
    const int nhalf = nk * Cfg::NATOM;
    // Steady state: the half-stage's MMAs and their commits go out in one elected block. (Probing the next
    // half-stage's barriers between its MMAs so the boundary can skip its wait measured slower: 1.565 -> 1.631 ms.)
    const bool rdy_known = false, a_known = false;
    for (int kb = 0; kb < nk; ++kb) {
        if (!rdy_known && !FD_TIMED_WAIT(w_x, wwait(&G.ready[st.stage], st.phase, P.abort_flag))) return false;
        tc_fence_after();
        const uint64_t bdesc = umma_desc_kmajor(smem_u32(ring + st.stage * Cfg::STAGE_BYTES), 128);
        const int nstage = st.stage + 1 == Cfg::STAGES ? 0 : st.stage + 1;
        const uint32_t nphase = st.stage + 1 == Cfg::STAGES ? st.phase ^ 1u : st.phase;
#pragma unroll
        for (int at = 0; at < Cfg::NATOM; ++at) {
            const long long c0 = clog ? pclk() : 0;
            if (!a_known && !FD_TIMED_WAIT(w_x, wwait(&G.afull[st.ah], st.ahph, P.abort_flag))) return false;
            tc_fence_after();
            const long long c1 = clog ? pclk() : 0;
            const uint32_t a_half = tmem + Cfg::TMEM_A0 + st.ah * Cfg::A_COLS;
            const uint64_t bd = bdesc + ((at * Cfg::ATOM_BYTES) >> 4);
            const bool first = kb == 0 && at == 0;
            const bool stage_end = at == Cfg::NATOM - 1;
            if (corr_free) {
                if (elect_one()) {
                    if (kCorrBf16) issue_half_b16<true, true>(d_main, d_corr, a_half, bd, idesc, 1u, 1u);
                    else issue_fp32_steady<0, 12>(d_main, d_corr, a_half, bd, idesc);
                    mma_commit(&G.aempty[st.ah]);
                    if (stage_end) mma_commit(&G.done[st.stage]);   // token + weight stage reusable
                }
                __syncwarp();
            } else {
                if (elect_one()) issue_half_ffn<true, false>(d_main, d_corr, a_half, bd, idesc, first ? 0u : 1u, 0u);
                __syncwarp();
                const int h = kb * Cfg::NATOM + at;
                corr_free = wtest(&G.cempty, st.cph ^ 1u);
                if (!corr_free && (h + 1 >= kCorrInMainMax || h + 1 == nhalf)) {
                    if (!FD_TIMED_WAIT(w_x, wwait(&G.cempty, st.cph ^ 1u, P.abort_flag))) return false;
                    corr_free = true;
                }
                if (corr_free) {
                    st.cph ^= 1u;
                    tc_fence_after();
                    if (elect_one()) issue_half_ffn<false, true>(d_main, d_corr, a_half, bd, idesc, 0u, 0u);
                } else {   // corrections of this half-stage ride in the main accumulator
                    if (elect_one()) issue_half_ffn<false, true>(d_main, d_main, a_half, bd, idesc, 0u, 1u);
                }
                __syncwarp();
                wcommit(&G.aempty[st.ah]);
                if (stage_end) wcommit(&G.done[st.stage]);
            }
            const long long c2 = clog ? pclk() : 0;
            if (clog && (threadIdx.x & 31) == 0 && *nlog < kChunkLog / 2) {
                // chunk log (development build): per half-stage {afull wait start, wait end, MMAs issued, logged}
                unsigned long long* o = clog + 4 * (*nlog)++;
                o[0] = c0; o[1] = c1; o[2] = c2; o[3] = pclk();
            }
            if (++st.ah == Cfg::A_SLOTS) { st.ah = 0; st.ahph ^= 1u; }
        }
        st.stage = nstage;
        st.phase = nphase;
    }
    return true;
}

// Gate tile (kGateTask): the main (w_hi x_hi) products of every 64-K stage go to a fresh accumulator
// (ping-pong acc[0]/acc[1], tfull after each stage), which the gate epilogue folds into registers in
// round-to-nearest FP32: each accumulator then sees only 8 truncating MMAs on a 64-term partial sum, and
// the epilogue gets the chunk-end prefix sums the certificate needs (gate_epilogue). The corrections
// accumulate over the whole tile in kTmemCorr as in the FFN.
__device__ __forceinline__ bool mma_gate_tile(const LaunchParams& P, uint8_t* ring, GemmCtrl& G, uint32_t tmem, int nk,
                                              uint32_t idesc, MmaFp32State& st, int& acc, uint32_t& accphase,
                                              long long& w_x) {
    using Cfg = GemmCfg<kFP32>;
    const uint32_t d_corr = tmem + kTmemCorr;
    for (int kb = 0; kb < nk; ++kb) {
        if (!FD_TIMED_WAIT(w_x, wwait(&G.tempty[acc], accphase ^ 1u, P.abort_flag))) return false;
        const uint32_t d_main = tmem + (uint32_t)(acc * kNT);
        if (!FD_TIMED_WAIT(w_x, wwait(&G.ready[st.stage], st.phase, P.abort_flag))) return false;
        tc_fence_after();
        const uint64_t bdesc = umma_desc_kmajor(smem_u32(ring + st.stage * Cfg::STAGE_BYTES), 128);
#pragma unroll
        for (int at = 0; at < Cfg::NATOM; ++at) {
            if (!FD_TIMED_WAIT(w_x, wwait(&G.afull[st.ah], st.ahph, P.abort_flag))) return false;
            tc_fence_after();
            const uint32_t a_half = tmem + Cfg::TMEM_A0 + st.ah * Cfg::A_COLS;
            const uint64_t bd = bdesc + ((at * Cfg::ATOM_BYTES) >> 4);
            const uint32_t main_acc = at == 0 ? 0u : 1u;
            if (kb == 0 && at == 0) {
                if (elect_one()) issue_half_fp32<true, false>(d_main, d_corr, a_half, bd, idesc, 0u, 0u);
                __syncwarp();
                if (!FD_TIMED_WAIT(w_x, wwait(&G.cempty, st.cph ^ 1u, P.abort_flag))) return false;
                st.cph ^= 1u;
                tc_fence_after();
                if (elect_one()) issue_half_fp32<false, true>(d_main, d_corr, a_half, bd, idesc, 0u, 0u);
            } else {
                if (elect_one()) issue_half_fp32<true, true>(d_main, d_corr, a_half, bd, idesc, main_acc, 1u);
            }
            __syncwarp();
            wcommit(&G.aempty[st.ah]);
            if (++st.ah == Cfg::A_SLOTS) { st.ah = 0; st.ahph ^= 1u; }
        }
        wcommit(&G.done[st.stage]);
        if (++st.stage == Cfg::STAGES) { st.stage = 0; st.phase ^= 1u; }
        wcommit(&G.tfull[acc]);   // this stage's main partial (and, at the last stage, the corrections)
        if (++acc == kAccStages) { acc = 0; accphase ^= 1u; }
    }
    return true;
}

template <int PREC>
__device__ void gemm_mma(const LaunchParams& P, uint8_t* ring, GemmCtrl& G, unsigned long long* trace,
                         unsigned long long* chunklog) {
    using Cfg = GemmCfg<PREC>;
    constexpr int NM = StageMmas<PREC>::N;
    int nlog = 0;
    const int lane = threadIdx.x & 31;
    long long w_x = 0, w_acc = 0, w_task = 0, ntile = 0;
    int stage = 0;
    uint32_t phase = 0;
    int q = 0;
    uint32_t qphase = 0;
    int acc = 0;
    uint32_t accphase = 0;
    const uint32_t tmem = G.tmem_base;
    // per-stage constants of the 2-stage ring, hoisted out of the tile loop (lean path below)
    const uint32_t abase_s[2] = {tmem + Cfg::TMEM_A0, tmem + Cfg::TMEM_A0 + Cfg::A_COLS};
    const uint64_t bdesc_s[2] = {umma_desc_kmajor(smem_u32(ring), 128),
                                 umma_desc_kmajor(smem_u32(ring + Cfg::STAGE_BYTES), 128)};
    MmaFp32State st32;
    while (true) {
        if (!FD_TIMED_WAIT(w_task, wwait(&G.qfull[q], qphase, P.abort_flag))) return;
        const int type = G.ring[q].type;
        __syncwarp();
        if (lane == 0) mbar_arrive(&G.qempty[q]);
        if (++q == kTaskRing) { q = 0; qphase ^= 1u; }
        if (type < 0) {
            if (lane == 0) {
                trace[kWaitMmaX] = w_x; trace[kWaitMmaA] = 0; trace[kWaitMmaAcc] = w_acc;
                trace[kWaitMmaTask] = w_task; trace[kMmaTiles] = ntile;
            }
            return;
        }
        ++ntile;
        const int nk = (task_k(P, type) + Cfg::BK - 1) / Cfg::BK;
        if constexpr (PREC == kFP32) {
            if (type == kGateTask) {
                if (!mma_gate_tile(P, ring, G, tmem, nk, umma_idesc(2u, kBF, (uint32_t)P.gate_n), st32, acc, accphase,
                                   w_x))
                    return;
                continue;
            }
        }
        if (!FD_TIMED_WAIT(w_acc, wwait(&G.tempty[acc], accphase ^ 1u, P.abort_flag))) return;
        const uint32_t d_tmem = tmem + (uint32_t)(acc * kNT);
        if constexpr (PREC == kFP32) {
            if (!mma_tile_fp32(P, ring, G, tmem, d_tmem, nk, Cfg::IDESC, st32, w_x, chunklog, &nlog)) return;
            wcommit(&G.tfull[acc]);   // main + correction accumulators ready for the epilogue
            if (++acc == kAccStages) { acc = 0; accphase ^= 1u; }
            continue;
        }
        long long t_rdy = chunklog ? pclk() : 0;
        if (!FD_TIMED_WAIT(w_x, wwait(&G.ready[stage], phase, P.abort_flag))) return;
        tc_fence_after();
        if (Cfg::STAGES == 2 && stage == 0 && (nk & 1) == 0 && !chunklog) {
            // Lean path (tile starts at ring slot 0, even stage count): stage pairs with compile-time
            // slot indices, so a stage boundary is the commit, one probe and the descriptor selects.
            for (int kb = 0; kb < nk; kb += 2) {
                const bool last = kb + 2 == nk;
                if (elect_one()) issue_stage<PREC, 0, NM>(d_tmem, abase_s[0], bdesc_s[0], kb == 0);
                __syncwarp();
                wcommit(&G.done[0]);
                if (!FD_TIMED_WAIT(w_x, wwait(&G.ready[1], phase, P.abort_flag))) return;
                tc_fence_after();
                if (elect_one()) issue_stage<PREC, 0, NM>(d_tmem, abase_s[1], bdesc_s[1], 0u);
                __syncwarp();
                wcommit(&G.done[1]);
                phase ^= 1u;
                if (!last) {
                    if (!FD_TIMED_WAIT(w_x, wwait(&G.ready[0], phase, P.abort_flag))) return;
                    tc_fence_after();
                }
            }
            wcommit(&G.tfull[acc]);
            if (++acc == kAccStages) { acc = 0; accphase ^= 1u; }
            continue;
        }
#pragma unroll 4   // fewer loop back-edges (and their YIELDs) between stages (measured: 4 beats 1/2/8/16)
        for (int kb = 0; kb < nk; ++kb) {
            const long long t_iss = chunklog ? pclk() : 0;
            const uint32_t abase = tmem + Cfg::TMEM_A0 + stage * Cfg::A_COLS;
            const uint64_t bdesc = umma_desc_kmajor(smem_u32(ring + stage * Cfg::STAGE_BYTES), 128);
            const int nstage = stage + 1 == Cfg::STAGES ? 0 : stage + 1;
            const uint32_t nphase = stage + 1 == Cfg::STAGES ? phase ^ 1u : phase;
            const bool last = kb + 1 == nk;
            if (elect_one()) issue_stage<PREC, 0, NM>(d_tmem, abase, bdesc, kb == 0);
            __syncwarp();
            wcommit(&G.done[stage]);   // token + weight stage reusable once these MMAs retire
            if (chunklog && lane == 0 && nlog < kChunkLog / 2) {
                chunklog[4 * nlog] = pclk();
                chunklog[4 * nlog + 1] = t_rdy;   // wait for ready started
                chunklog[4 * nlog + 2] = t_iss;   // ready observed, issue starts
                chunklog[4 * nlog + 3] = 0;
                ++nlog;
            }
            stage = nstage;
            phase = nphase;
            if (!last) {
                if (chunklog) t_rdy = pclk();
                if (!FD_TIMED_WAIT(w_x, wwait(&G.ready[stage], phase, P.abort_flag))) return;
                tc_fence_after();
            }
        }
        wcommit(&G.tfull[acc]);         // accumulator ready for the epilogue
        if (++acc == kAccStages) { acc = 0; accphase ^= 1u; }
    }
}

// FP32 FFN issue on TWO warps (kWarpMma: even half-stages = token atom 0 of each stage, A slot 0; kWarpMma2:
// odd half-stages = atom 1, A slot 1), strictly alternating through an mbarrier hand-off (pp[]). Each warp has
// its own token atom slots (ready/done per atom) and A slot, so only the accumulator commit (tfull) counts both. The tensor queue
// holds only ~1-2 MMAs, so every wait / commit / bookkeeping step between two half-stages of ONE issuer drained it
// (chunk log: ~450 cycles per 768-cycle half-stage); with two issuers each does its waits while the other one's
// 12 MMAs run, and the hand-off (arrive -> wait, ~tens of cycles) is the only gap (tools/dev/pipe_rate3.py: 91.7 ->
// 64.0 cycles per MMA for the full barrier protocol). Issue order is identical to one issuer's (results are
// bit-identical); each warp commits its own MMAs.
// Issuer hand-off on hardware named barriers (ids 2, 3; 64 threads = the two issuer warps): warp par waits on
// barrier 2 + par, the other warp arrives on it after issuing its half-stage. A bar.sync completes in tens of
// cycles (an mbarrier wake-up costs ~100-200), and the tensor queue holds only ~1-2 MMAs of the other warp's
// half-stage (tools/dev/pipe_rate3.py: the named-barrier ping-pong issues at the tensor core's rate). A warp
// leaving on abort arrives once more so that its partner is never left in bar.sync.
__device__ __forceinline__ void pp_wait(int par) {
    asm volatile("bar.sync %0, 64;" ::"r"(2 + par) : "memory");
    tc_fence_after();
}
__device__ __forceinline__ void pp_signal(int par) {
    tc_fence_before();
    asm volatile("bar.arrive %0, 64;" ::"r"(2 + (par ^ 1)) : "memory");
}

__device__ void gemm_mma_fp32_pp(const LaunchParams& P, uint8_t* ring, GemmCtrl& G, unsigned long long* trace,
                                 unsigned long long* clog, const int par) {
    using Cfg = GemmCfg<kFP32>;
    const int lane = threadIdx.x & 31;
    long long w_x = 0, w_acc = 0, w_task = 0, ntile = 0;
    int q = 0;
    uint32_t qphase = 0;
    int acc = 0;
    uint32_t accphase = 0;
    uint32_t tph0 = 0, tph1 = 0;   // FFN split-K buffers' tempty phases
    int stage = 0;
    uint32_t phase = 0, aph = 0, pph = 0;
    bool started = par == 1;   // par 0's very first half-stage has no predecessor
    int nlog = 0;
    const uint32_t tmem = G.tmem_base;
    const uint32_t d_corr = tmem + kTmemCorr;
    const uint32_t a_half = tmem + Cfg::TMEM_A0 + (uint32_t)par * Cfg::A_COLS;
    const uint32_t idesc = Cfg::IDESC;
    while (true) {
        if (!FD_TIMED_WAIT(w_task, wwait(&G.qfull[q], qphase, P.abort_flag))) { pp_signal(par); return; }
        const int type = G.ring[q].type;
        __syncwarp();
        if (lane == 0) mbar_arrive(&G.qempty[q]);
        if (++q == kTaskRing) { q = 0; qphase ^= 1u; }
        if (type < 0) {
            if (lane == 0 && par == 0) {
                trace[kWaitMmaX] = w_x; trace[kWaitMmaA] = 0; trace[kWaitMmaAcc] = w_acc;
                trace[kWaitMmaTask] = w_task; trace[kMmaTiles] = ntile;
            }
            if (par == 0 && ntile > 0) pp_wait(0);   // every tile ends on warp 1: consume its last hand-off
            return;
        }
        ++ntile;
        const int nk = (task_k(P, type) + Cfg::BK - 1) / Cfg::BK;
        if (type == kGateTask) {
            // Gate tile (M = 128 token rows in TMEM, N = gate_n experts from smem): the main products of every
            // 64-K stage go to a FRESH accumulator (rotating acc; the gate epilogue folds each stage in RN FP32,
            // mma_gate_tile's scheme), the corrections accumulate over the tile in kTmemCorr, fresh after the
            // previous tile's fold (cempty). Token stages carry one ready/done per stage (both warps commit).
            const uint32_t gdesc = umma_idesc(2u, kBF, (uint32_t)P.gate_n);
            for (int kb = 0; kb < nk; ++kb) {
                const long long g0 = clog ? pclk() : 0;
                if (par == 0 && !FD_TIMED_WAIT(w_acc, wwait(&G.tempty[acc], accphase ^ 1u, P.abort_flag))) { pp_signal(par); return; }
                const long long g1 = clog ? pclk() : 0;
                if (!FD_TIMED_WAIT(w_x, wwait(&G.ready[stage], phase, P.abort_flag))) { pp_signal(par); return; }
                const long long g2 = clog ? pclk() : 0;
                if (!FD_TIMED_WAIT(w_x, wwait(&G.afull[par], aph, P.abort_flag))) { pp_signal(par); return; }
                const long long g3 = clog ? pclk() : 0;
                if (started) pp_wait(par);
                if (clog && lane == 0 && nlog < kChunkLog / 8) {
                    // chunk log (development build), gate, rows [384 + 64 par, +64): per stage {acc wait,
                    // token-plane wait, A wait, hand-off wait + issue}
                    unsigned long long* o = clog + 4 * (3 * kChunkLog / 4 + par * (kChunkLog / 8) + nlog++);
                    o[0] = g1 - g0; o[1] = g2 - g1; o[2] = g3 - g2; o[3] = pclk() - g3;
                }
                started = true;
                tc_fence_after();
                const uint32_t d_main = tmem + (uint32_t)(acc * kNT);
                const uint64_t bd = umma_desc_kmajor(smem_u32(ring + stage * Cfg::STAGE_BYTES), 128) +
                                    (uint64_t)((par * Cfg::ATOM_BYTES) >> 4);
                const uint32_t main_acc = par == 0 ? 0u : 1u;
                if (kb == 0 && par == 0) {   // corrections start fresh once the previous tile's fold freed them
                    if (elect_one()) issue_half_fp32<true, false>(d_main, d_corr, a_half, bd, gdesc, 0u, 0u);
                    __syncwarp();
                    uint32_t cph = G.pp_cph;
                    if (!FD_TIMED_WAIT(w_x, wwait(&G.cempty, cph ^ 1u, P.abort_flag))) { pp_signal(par); return; }
                    cph ^= 1u;
                    tc_fence_after();
                    if (elect_one()) {
                        issue_half_fp32<false, true>(d_main, d_corr, a_half, bd, gdesc, 0u, 0u);
                        G.pp_cph = cph;
                    }
                } else if (elect_one()) {
                    issue_half_fp32<true, true>(d_main, d_corr, a_half, bd, gdesc, main_acc, 1u);
                }
                __syncwarp();
                if (elect_one()) {
                    mma_commit(&G.aempty[par]);
                    mma_commit(&G.done[stage]);
                    mma_commit(&G.tfull[acc]);   // this stage's main partial (and at the last stage the corrections)
                }
                __syncwarp();
                tc_fence_before();
                pp_signal(par);
                if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1u; }
                aph ^= 1u;
                if (++acc == kAccStages) { acc = 0; accphase ^= 1u; }
            }
            if (FD_DBG(kDbgGateOnly) && lane == 0) trace[20 + par] = globaltimer();   // tools/dev/gate_only.py
            continue;
        }
        const long long t_tile = clog ? pclk() : 0;
        long long s_tok = 0, s_a = 0, s_pp = 0;
        const long long t_acc = clog ? pclk() : 0;
        // Split-K main accumulation (FFN): the first nk0 = nk/2 stages' main products go to buffer 0, the rest to
        // buffer 1; the epilogue saves buffer 0's partial mid-tile and adds it in RN at the end. Each buffer then
        // sees half the truncating MMAs on a half-length partial sum (profiles/r02_numerics.md §5).
        const int nk0 = kSplitK ? nk / 2 : 0;
        for (int kb = 0; kb < nk; ++kb) {
            const int buf = kb < nk0 ? 0 : 1;
            if (par == 0 && (kb == 0 || kb == nk0)) {   // buffer free (the epilogue read the previous tile's)
                if (!FD_TIMED_WAIT(w_acc, wwait(&G.tempty[buf], (buf ? tph1 : tph0) ^ 1u, P.abort_flag))) { pp_signal(par); return; }
            }
            if (kb == 0 && nk0 > 0) tph0 ^= 1u;
            if (kb == nk0) tph1 ^= 1u;
            const uint32_t d_main = tmem + (uint32_t)(buf * kNT);
            const bool buf_first = kb == nk0 && kb > 0;   // first stage into buffer 1 (par 0's MMAs start it fresh)
            const long long c0 = clog ? pclk() : 0;
            const int slot = stage * Cfg::NATOM + par;   // this warp's token atom of the stage (own ready/done)
            if (!FD_TIMED_WAIT(w_x, wwait(&G.ready[slot], phase, P.abort_flag))) { pp_signal(par); return; }
            const long long c1 = clog ? pclk() : 0;
            if (!FD_TIMED_WAIT(w_x, wwait(&G.afull[par], aph, P.abort_flag))) { pp_signal(par); return; }
            const long long c2 = clog ? pclk() : 0;
            if (started) pp_wait(par);   // h-1 issued
            const long long c3 = clog ? pclk() : 0;
            started = true;
            tc_fence_after();
            const uint64_t bd = umma_desc_kmajor(smem_u32(ring + stage * Cfg::STAGE_BYTES), 128) +
                                (uint64_t)((par * Cfg::ATOM_BYTES) >> 4);
            const bool last = kb + 1 == nk;
            const bool half_end = kb + 1 == nk0;   // buffer 0 complete after this stage
            if (kb > 0) {   // steady state: both accumulators accumulate
                if (elect_one()) {
                    const uint32_t macc = (buf_first && par == 0) ? 0u : 1u;
                    if (kCorrBf16) issue_half_b16<true, true>(d_main, d_corr, a_half, bd, idesc, macc, 1u);
                    else if (macc) issue_fp32_steady<0, 12>(d_main, d_corr, a_half, bd, idesc);
                    else issue_half_fp32<true, true>(d_main, d_corr, a_half, bd, idesc, 0u, 1u);
                    mma_commit(&G.aempty[par]);
                    mma_commit(&G.done[slot]);
                    if (half_end) mma_commit(&G.tfull[0]);
                    if (last) mma_commit(&G.tfull[1]);
                }
                __syncwarp();
            } else if (par == 0) {   // h = 0: main starts fresh; corrections fresh if the fold freed kTmemCorr
                if (elect_one()) issue_half_ffn<true, false>(d_main, d_corr, a_half, bd, idesc, 0u, 0u);
                __syncwarp();
                uint32_t cph = G.pp_cph;
                const bool corr_free = wtest(&G.cempty, cph ^ 1u);
                if (corr_free) {
                    cph ^= 1u;
                    tc_fence_after();
                }
                if (elect_one()) {
                    if (corr_free) issue_half_ffn<false, true>(d_main, d_corr, a_half, bd, idesc, 0u, 0u);
                    else issue_half_ffn<false, true>(d_main, d_main, a_half, bd, idesc, 0u, 1u);   // ride in main
                    mma_commit(&G.aempty[par]);
                    mma_commit(&G.done[slot]);
                    if (half_end) mma_commit(&G.tfull[0]);
                    if (last) mma_commit(&G.tfull[1]);
                    G.pp_corr = corr_free ? 1u : 0u;
                    G.pp_cph = cph;
                }
                __syncwarp();
            } else {   // h = 1: corrections into kTmemCorr -- fresh if h = 0 could not, after the fold (blocking)
                uint32_t cph = G.pp_cph;
                const bool corr_free = G.pp_corr != 0;
                if (elect_one()) issue_half_ffn<true, false>(d_main, d_corr, a_half, bd, idesc, 1u, 0u);
                __syncwarp();
                if (!corr_free) {
                    if (!FD_TIMED_WAIT(w_x, wwait(&G.cempty, cph ^ 1u, P.abort_flag))) { pp_signal(par); return; }
                    cph ^= 1u;
                    tc_fence_after();
                }
                if (elect_one()) {
                    issue_half_ffn<false, true>(d_main, d_corr, a_half, bd, idesc, 0u, corr_free ? 1u : 0u);
                    mma_commit(&G.aempty[par]);
                    mma_commit(&G.done[slot]);
                    if (half_end) mma_commit(&G.tfull[0]);
                    if (last) mma_commit(&G.tfull[1]);
                    G.pp_cph = cph;
                }
                __syncwarp();
            }
            // hand-off: this half-stage is issued (tcgen05 ops ordered before the other warp's by the fence pair)
            tc_fence_before();
            pp_signal(par);
            s_tok += c1 - c0; s_a += c2 - c1; s_pp += c3 - c2;
            if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1u; }
            aph ^= 1u;
        }
        if (clog && lane == 0 && nlog < kChunkLog / 4) {
            // chunk log (development build), rows [128 * par, +128): per tile {type | tile cycles << 8, accumulator
            // wait, token wait, A wait | hand-off wait << 32}
            unsigned long long* o = clog + 4 * (par * (kChunkLog / 4) + nlog++);
            o[0] = (unsigned long long)type | ((unsigned long long)(pclk() - t_tile) << 8);
            o[1] = t_acc - t_tile; o[2] = s_tok; o[3] = (unsigned long long)s_a | ((unsigned long long)s_pp << 32);
        }
    }
}

// warps 4-7: thread = output feature (TMEM lane), 32 token columns per tcgen05.ld
// warp 9, one lane: release signals of finished tiles, in tile order (runtime.hpp:685-690). Every
// epilogue thread's stores precede the hand-off (bar.sync, then the mbarrier arrive/wait pair), so the
// fence here orders them before the counter / flag release (cumulativity).
__device__ void gemm_signal(const LaunchParams& P, const RankCtx& R, GemmCtrl& G, unsigned long long* stat) {
    const uint32_t par = P.epoch & 1u;
    const int cta = blockIdx.x % P.ctas_per_rank;
    const int e_glob_base = R.rank * P.El;
    int sq = 0;
    uint32_t sphase = 0;
    while (true) {
        if (!mbar_wait(&G.sfull[sq], sphase, P.abort_flag)) return;
        const Task tk = G.sring[sq];
        mbar_arrive(&G.sempty[sq]);
        if (++sq == kTaskRing) { sq = 0; sphase ^= 1u; }
        if (tk.type < 0) return;
        int rows = 0;
        for (int j = 0; j < tk.nsrc; ++j) rows += tk.cnt[j];
        if (tk.type == 0) {
            __threadfence();
            // event before the counter release: GEMM0's end precedes any dependent GEMM1 start
            emit_event(P, R, kEvExec, cta, kTaskGemm0, tk.t0, globaltimer(), tk.src0, tk.le, tk.m, tk.nb,
                       tk.nsrc, rows);
            atomicAdd(R.g0done + (size_t)tk.le * P.MT + tk.m, 1u);
            stat[0]++;
        } else {
            // the tile's rows went to the origin rank: system scope when it may be another GPU
            if (P.nranks == P.P) __threadfence(); else __threadfence_system();
            emit_event(P, R, kEvExec, cta, kTaskGemm1, tk.t0, globaltimer(), tk.src0, tk.le, tk.m, tk.nb,
                       tk.nsrc, rows);
            const int e_glob = e_glob_base + tk.le;
            const int rbf = P.Cp >= kBM ? (tk.m % (P.Cp / kBM)) : 0;
            for (int j = 0; j < tk.nsrc && !P.fused_combine; ++j) {
                if (tk.cnt[j] <= 0) continue;
                unsigned long long* f = reinterpret_cast<unsigned long long*>(R.peer_heap[tk.src0 + j] +
                                                                              R.hl.cflag[par]) +
                                        ((size_t)e_glob * P.RBF + rbf) * P.NB1 + tk.nb;
                emit_event(P, R, kEvTilePut, cta, kTaskGemm1, globaltimer(), 0, R.rank, tk.le, tk.m, tk.nb,
                           tk.src0 + j, tk.cnt[j]);
                st_release_sys(f, ((uint64_t)P.epoch << 32) | (uint32_t)tk.cnt[j]);
            }
            stat[1]++;
        }
    }
}

// FP32: add the tile's correction accumulator into its main accumulator in round-to-nearest FP32
// (this warp's 32 TMEM lanes, 128 token columns), leaving the correction columns free.
// buffer 1 (second-half main partial) += first-half partial (RN, from the CTA scratch) += corrections (RN)
__device__ __forceinline__ void fold_corr_part(uint32_t t_main, uint32_t t_corr, const float* part) {
#pragma unroll 1
    for (int ch = 0; ch < kNT / 32; ++ch) {
        uint32_t m[32], c[32];
        tmem_ld32(t_main + ch * 32, m);
        tmem_ld32(t_corr + ch * 32, c);
        float pv[32];
        if (part) {
#pragma unroll
            for (int i = 0; i < 32; ++i) pv[i] = part[(size_t)(ch * 32 + i) * kBF];
        }
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            float v = __uint_as_float(m[i]);
            if (part) v = __fadd_rn(pv[i], v);
            m[i] = __float_as_uint(__fadd_rn(v, __uint_as_float(c[i])));
        }
        tmem_st32(t_main + ch * 32, m);
    }
    tmem_wait_st();
    tc_fence_before();
}

__device__ __forceinline__ void fold_corr(uint32_t t_main, uint32_t t_corr) {
#pragma unroll 1
    for (int ch = 0; ch < kNT / 32; ++ch) {
        uint32_t m[32], c[32];
        tmem_ld32(t_main + ch * 32, m);
        tmem_ld32(t_corr + ch * 32, c);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) m[i] = __float_as_uint(__fadd_rn(__uint_as_float(m[i]), __uint_as_float(c[i])));
        tmem_st32(t_main + ch * 32, m);
    }
    tmem_wait_st();
    tc_fence_before();
}

// GEMM0 epilogue of one 32-token chunk: +b1, activation, store C1 (tf32 hi/lo planes or bf16).
// Row i of the chunk lives at +i*D; bit i of vmask = row holds a landed token (warp-uniform).
template <int PREC, int ACT>
__device__ __forceinline__ void epi_gemm0(const uint32_t (&r)[32], uint32_t vmask, float bias, float* hi, float* lo,
                                          __nv_bfloat16* bf, int D) {
    // C1 plane 1 in the bf16-correction format: this thread's feature is lane (feat % 32) of its 32-k group
    const int lane = threadIdx.x & 31;
    __nv_bfloat16* lb = reinterpret_cast<__nv_bfloat16*>(reinterpret_cast<uint8_t*>(lo) - 4 * lane) + lane;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        if (!(vmask & (1u << i))) continue;
        const float v = activation(ACT, __fadd_rn(__uint_as_float(r[i]), bias));
        const size_t o = (size_t)i * D;
        if (PREC == kFP32) {
            const float h = tf32_hi(v);
            hi[o] = h;
            if (kCorrBf16) {
                lb[2 * o] = __float2bfloat16_rn(h);                  // bf16 x_hi at byte 2 * lane of the group
                lb[2 * o + 32] = __float2bfloat16_rn(__fsub_rn(v, h));   // bf16 x_lo at byte 64 + 2 * lane
            } else {
                lo[o] = __fsub_rn(v, h);
            }
        } else {
            bf[o] = __float2bfloat16_rn(v);
        }
    }
}

template <int PREC, bool FUSED>
__device__ void gemm_epilogue(const LaunchParams& P, const RankCtx& R, GemmCtrl& G, unsigned long long* stat,
                              unsigned long long* trace, unsigned long long* elog) {
    int nelog = 0;
    long long w_acc = 0, busy = 0;
    const int et = threadIdx.x - kWarpEpi0 * 32;   // 0..127 == TMEM lane == feature row in the tile
    const int wq = et >> 5;
    const uint32_t par = P.epoch & 1u;
    int q = 0;
    uint32_t qphase = 0;
    int acc = 0;
    uint32_t accphase = 0;
    uint32_t tph0 = 0, tph1 = 0;   // FP32: the split-K buffers' tfull phases
    const uint32_t tmem = G.tmem_base;
    const int e_glob_base = R.rank * P.El;
    int sq = 0;
    uint32_t sphase = 0;
    bool zero_seen = false;
    if (FUSED) {
        // fused combine accumulates into the output: zero this CTA's token rows while the first tile's
        // MMAs run (streaming stores), then count this CTA in; GEMM1 epilogues wait for every CTA of
        // the origin rank (the first GEMM1 tile starts long after, so the wait is free in practice)
        const int cta = blockIdx.x % P.ctas_per_rank;
        int tokA, tokB, b0, b1;
        gate_token_range(P, cta, tokA, tokB, b0, b1);
        float4* o4 = reinterpret_cast<float4*>(P.out[blockIdx.x / P.ctas_per_rank] + (size_t)tokA * P.H);
        const size_t n4 = (size_t)(tokB - tokA) * P.H / 4;
        for (size_t i = et; i < n4; i += 128) __stcs(o4 + i, make_float4(0.0f, 0.0f, 0.0f, 0.0f));
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (et == 0) {
            __threadfence();
            atomicAdd(R.zero_ctr, 1u);
        }
    }
    while (true) {
        if (!mbar_wait(&G.qfull[q], qphase, P.abort_flag)) return;
        const Task& tk = G.ring[q];   // stays valid until this warp group releases the slot
        const int type = tk.type;
        if (type < 0) {
            if (et == 0) {
                trace[kWaitEpiAcc] = w_acc; trace[kEpiBusy] = busy;
                if (mbar_wait(&G.sempty[sq], sphase ^ 1u, P.abort_flag)) {   // end marker for the signal warp
                    G.sring[sq].type = -1;
                    mbar_arrive(&G.sfull[sq]);
                }
            }
            return;
        }
        if constexpr (PREC == kFP32) {
            // split-K main accumulators (gemm_mma_fp32_pp): buffer 0 holds the first nk/2 stages' main partial
            // and completes mid-tile -- save it (this thread's feature row, [col][row] in the CTA's scratch) and
            // free the buffer for the next tile; at the end buffer 1 += partial (RN), += corrections (RN)
            acc = 1;
            const uint32_t lanes = (uint32_t)(wq * 32) << 16;
            const int nk0 = kSplitK ? ((task_k(P, type) + GemmCfg<kFP32>::BK - 1) / GemmCfg<kFP32>::BK) / 2 : 0;
            float* part = R.epart + (size_t)(blockIdx.x % P.ctas_per_rank) * kNT * kBF + et;
            if (nk0 > 0) {
                if (!FD_TIMED_WAIT(w_acc, mbar_wait(&G.tfull[0], tph0, P.abort_flag))) return;
                tph0 ^= 1u;
                tc_fence_after();
#pragma unroll 1
                for (int ch = 0; ch < kNT / 32; ++ch) {
                    uint32_t m[32];
                    tmem_ld32(tmem + lanes + (uint32_t)(ch * 32), m);
                    tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < 32; ++i) part[(size_t)(ch * 32 + i) * kBF] = __uint_as_float(m[i]);
                }
                tc_fence_before();
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (et == 0) mbar_arrive(&G.tempty[0]);
            }
            if (!FD_TIMED_WAIT(w_acc, mbar_wait(&G.tfull[1], tph1, P.abort_flag))) return;
            tph1 ^= 1u;
            tc_fence_after();
            fold_corr_part(tmem + lanes + (uint32_t)kNT, tmem + lanes + kTmemCorr, nk0 > 0 ? part : nullptr);
            __syncwarp();
            if ((et & 31) == 0) mbar_arrive(&G.cempty);
        } else {
            if (!FD_TIMED_WAIT(w_acc, mbar_wait(&G.tfull[acc], accphase, P.abort_flag))) return;
            tc_fence_after();
        }
        if (FUSED && type == 1 && !zero_seen) {
            for (int r = 0; r < P.nranks; ++r)
                if (!wait_counter(P, R, P.ranks[r].zero_ctr, P.zero_target, 310)) return;
            zero_seen = true;
        }
        const long long tb0 = pclk();
        long long e_loop = 0, e_bar = 0, e_ld = 0;

        const int ncols = type == 0 ? P.D : P.H;
        const int feat = tk.nb * kBF + et;
        const bool fvalid = feat < ncols;
        const float bias =
            fvalid ? __ldg((type == 0 ? R.b1 + (size_t)tk.le * P.D : R.b2 + (size_t)tk.le * P.H) + feat) : 0.0f;
        const int e_glob = e_glob_base + tk.le;
        const size_t grow0 = (size_t)tk.le * P.RP + (size_t)tk.m * kBM;   // first X / C1 row of the tile
        const int rb_base = P.Cp >= kBM ? (tk.m % (P.Cp / kBM)) * kBM : 0;
        const int src0 = tk.src0, nsrc = tk.nsrc, cnt0 = tk.cnt[0];
        const uint32_t tbase = tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(acc * kNT);
        float* c1hi = reinterpret_cast<float*>(R.c1[0]) + grow0 * (size_t)P.D + feat;
        float* c1lo = reinterpret_cast<float*>(R.c1[1]) + grow0 * (size_t)P.D + feat;
        __nv_bfloat16* c1b = reinterpret_cast<__nv_bfloat16*>(R.c1[0]) + grow0 * (size_t)P.D + feat;
        // GEMM1 row metadata, one row per lane per 32-row chunk, all loads issued together at tile start
        // (a per-row chain of dependent loads inside the element loop cost ~600 cycles per row):
        // fused: the origin's output row pointer and combine weight; else the origin's yc row pointer
        const int lane = et & 31;
        float* rowp[kNT / 32];
        float roww[kNT / 32];
        if (type == 1) {
#pragma unroll
            for (int c = 0; c < kNT / 32; ++c) {
                const int n = c * 32 + lane;
                int src, slot;
                if (P.Cp >= kBM) { src = src0; slot = rb_base + n; }
                else { const int j = n / P.Cp; src = min(src0 + j, P.P - 1); slot = n - j * P.Cp; }
                const size_t ts = (size_t)e_glob * P.C + min(slot, P.C - 1);
                if (FUSED) {
                    const RankCtx& Ro = P.ranks[src];
                    const int t = Ro.tbl_tok[ts];
                    roww[c] = Ro.tbl_w[ts];
                    rowp[c] = P.out[src] + (size_t)max(t, 0) * P.H;
                } else {
                    roww[c] = 0.0f;
                    rowp[c] = reinterpret_cast<float*>(R.peer_heap[src] + R.hl.yc) + ts * P.H;
                }
            }
        }
#pragma unroll 1
        for (int ch = 0; ch < kNT / 32; ++ch) {
            uint32_t r[32];
            // this chunk's row pointer / weight by register selects (indexing the arrays with the runtime
            // ch would put them in local memory: two LDL per row in the store loop)
            float* rowp_c = rowp[0];
            float roww_c = roww[0];
#pragma unroll
            for (int c = 1; c < kNT / 32; ++c)
                if (ch == c) { rowp_c = rowp[c]; roww_c = roww[c]; }
            const long long tl0 = pclk();
            tmem_ld32(tbase + ch * 32, r);
            // validity of the 32 token rows of this chunk: bit i = row ch*32+i holds a landed token
            uint32_t vmask;
            if (P.Cp >= kBM) {
                const int lo = ch * 32, n = cnt0 - lo;
                vmask = n >= 32 ? 0xffffffffu : (n <= 0 ? 0u : ((1u << n) - 1u));
            } else {
                vmask = 0;
                // packets of Cp rows: rows [j*Cp, j*Cp + cnt_j) are valid (Cp in {16, 32, 64})
                for (int j = (ch * 32) / P.Cp; j < nsrc && j * P.Cp < ch * 32 + 32; ++j) {
                    const int a = max(j * P.Cp, ch * 32), b = min(j * P.Cp + tk.cnt[j], ch * 32 + 32);
                    if (b > a) vmask |= (b - a >= 32 ? 0xffffffffu : ((1u << (b - a)) - 1u)) << (a - ch * 32);
                }
            }
            tmem_wait_ld();
            e_ld += pclk() - tl0;
            if (!fvalid || (FD_DBG(kDbgNoEpiStore))) vmask = 0;
            // separate compact loops per tile type and activation (one fully unrolled body with every
            // variant inlined — erff included — was ~20 KB of SASS streamed through the I-cache per chunk)
            if (type == 0) {
                float* hi = c1hi + (size_t)ch * 32 * P.D;
                float* lo = c1lo + (size_t)ch * 32 * P.D;
                __nv_bfloat16* bf = c1b + (size_t)ch * 32 * P.D;
                if (P.act == 0) epi_gemm0<PREC, 0>(r, vmask, bias, hi, lo, bf, P.D);
                else if (P.act == 1) epi_gemm0<PREC, 1>(r, vmask, bias, hi, lo, bf, P.D);
                else epi_gemm0<PREC, 2>(r, vmask, bias, hi, lo, bf, P.D);
            } else {
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    if (!(vmask & (1u << i))) continue;   // warp-uniform: same token row for all lanes
                    const float v = __fadd_rn(__uint_as_float(r[i]), bias);
                    // row n's pointer (and weight) from lane i of this chunk's prefetch
                    float* rp = reinterpret_cast<float*>(
                        __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(rowp_c), i));
                    if (FUSED) {
                        // combine fused here (oracle.hpp:102-107 with k <= 2): O[t] += fl(w * y); the
                        // origin's slot table gives the token and its combine weight
                        const float w = __shfl_sync(0xffffffffu, roww_c, i);
                        atomicAdd(rp + feat, __fmul_rn(w, v));
                    } else {
                        rp[feat] = v;
                    }
                }
            }
        }
        e_loop = pclk();
        tc_fence_before();
        asm volatile("bar.sync 1, 128;" ::: "memory");   // all rows stored, TMEM drained
        e_bar = pclk();
        if (et == 0) {
            mbar_arrive(&G.tempty[acc]);
            // the tile's release signals (fence + counters / flags) go to the signal warp: the epilogue
            // moves on to the next accumulator instead of waiting out the fence
            if (!mbar_wait(&G.sempty[sq], sphase ^ 1u, P.abort_flag)) return;
            G.sring[sq] = tk;
            mbar_arrive(&G.sfull[sq]);
            if (++sq == kTaskRing) { sq = 0; sphase ^= 1u; }
            mbar_arrive(&G.qempty[q]);
        }
        busy += pclk() - tb0;
        if (elog && et == 0 && nelog < kChunkLog / 2) {   // chunklog rows [256, 512): per tile
            unsigned long long* o = elog + 4 * (kChunkLog / 2 + nelog++);
            o[0] = type; o[1] = e_loop - tb0; o[2] = e_ld; o[3] = pclk() - e_bar;
        }
        if (++q == kTaskRing) { q = 0; qphase ^= 1u; }
        if (PREC != kFP32 && ++acc == kAccStages) { acc = 0; accphase ^= 1u; }
    }
}

// ================================================================ phase 1a: gate logits on the tensor cores
// The gate GEMM z~ = A Wg of this CTA's token range runs through the FFN pipeline roles in the FP32
// (3xTF32) configuration with the operands in the other roles: the token rows (raw FP32, TMA from the
// caller's shard) take the weight role (converter warps split them into tf32 hi/lo TMEM operands and
// accumulate each row's sum of squares), the pre-split Wg^T hi/lo planes take the token role (smem
// B operand, N = gate_n experts per block). One task per (128-token tile, expert block).
__device__ void gate_producer(const LaunchParams& P, const RankCtx& R, int rl, uint8_t* ring, GemmCtrl& G,
                              int tokA, int tokB) {
    using Cfg = GemmCfg<kFP32>;
    int stage = 0, wstage = 0, q = 0;
    uint32_t phase = 0, wphase = 0, qphase = 0;
    const CUtensorMap* ta = &P.tm_in[rl];
    tma_prefetch(ta);
    tma_prefetch(&R.tm_wg[0]);
    tma_prefetch(&R.tm_wg[1]);
    const uint64_t pol = FD_DBG(kDbgEvictNormal) ? l2_policy_evict_normal() : l2_policy_evict_last();   // token rows: re-read by the dispatch push; Wg: by every CTA
    const int nk = (P.H + Cfg::BK - 1) / Cfg::BK;
    const uint32_t bbytes = (uint32_t)(Cfg::PLANES * Cfg::NATOM * P.gate_n * 128);
    for (int tok0 = tokA; tok0 < tokB; tok0 += kNT)
        for (int eb = 0; eb < P.gate_nblk; ++eb) {
            if (!mbar_wait(&G.qempty[q], qphase ^ 1u, P.abort_flag)) return;
            Task tk{};
            tk.type = kGateTask;
            tk.m = tok0;
            tk.nb = eb;
            tk.nsrc = 1;
            tk.cnt[0] = min(kNT, tokB - tok0);
            G.ring[q] = tk;
            mbar_arrive(&G.qfull[q]);
            if (++q == kTaskRing) { q = 0; qphase ^= 1u; }
            for (int kb = 0; kb < nk; ++kb) {
                if (!mbar_wait(&G.wempty[wstage], wphase ^ 1u, P.abort_flag)) return;
                if (FD_DBG(kDbgGateNoTokTma)) mbar_arrive(&G.wfull[wstage]);
                else {
                    mbar_expect_tx(&G.wfull[wstage], Cfg::W_BYTES);
#pragma unroll
                    for (int at = 0; at < Cfg::NATOM; ++at)
                        tma_load_2d_hint(ring + Cfg::W_OFF + wstage * Cfg::W_BYTES + at * Cfg::ATOM_BYTES, ta,
                                         &G.wfull[wstage], kb * Cfg::BK + at * Cfg::ATOM_K, tok0, pol);
                }
                if (++wstage == Cfg::WSTAGES) { wstage = 0; wphase ^= 1u; }
                if (!mbar_wait(&G.done[stage], phase ^ 1u, P.abort_flag)) return;
                uint8_t* st = ring + stage * Cfg::STAGE_BYTES;
                if (FD_DBG(kDbgGateNoWgTma)) mbar_arrive(&G.ready[stage]);
                else {
                    mbar_expect_tx(&G.ready[stage], bbytes);
#pragma unroll
                    for (int pl = 0; pl < Cfg::PLANES; ++pl)
#pragma unroll
                        for (int at = 0; at < Cfg::NATOM; ++at)
                            tma_load_2d_hint(st + pl * Cfg::PLANE_BYTES + at * Cfg::ATOM_BYTES, &R.tm_wg[pl],
                                             &G.ready[stage], kb * Cfg::BK + at * Cfg::ATOM_K, eb * P.gate_n, pol);
                }
                if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1u; }
            }
        }
    if (!mbar_wait(&G.qempty[q], qphase ^ 1u, P.abort_flag)) return;
    G.ring[q].type = -1;
    mbar_arrive(&G.qfull[q]);
}

// warps 4-7: thread = TMEM lane = token row of the tile. Per 64-K stage it adds the stage's main partial
// (gate_n <= 128 expert columns) into z[] in round-to-nearest FP32 and accumulates
//   sab += max_e |z_e|   (the prefix sums at 64-term chunk ends: the certificate's Sab, gate.hpp:77-81 chain)
// then adds the corrections at the end and writes the z~ row to g_phi and Sab to gate_sab (the certified
// routing reads both back; it overwrites g_phi with probabilities).
__device__ void gate_epilogue(const LaunchParams& P, const RankCtx& R, GemmCtrl& G) {
    using Cfg = GemmCfg<kFP32>;
    const int et = threadIdx.x - kWarpEpi0 * 32;
    const uint32_t lanes = (uint32_t)((et >> 5) * 32) << 16;
    const uint32_t tmem = G.tmem_base;
    const int nk = (P.H + Cfg::BK - 1) / Cfg::BK;
    int q = 0, acc = 0;
    uint32_t qphase = 0, accphase = 0;
    while (true) {
        if (!mbar_wait(&G.qfull[q], qphase, P.abort_flag)) return;
        const int type = G.ring[q].type, tok0 = G.ring[q].m, eb = G.ring[q].nb, valid = G.ring[q].cnt[0];
        if (type < 0) return;
        const int e0 = eb * P.gate_n;
        const int nv = min(P.gate_n, P.E - e0);   // valid expert columns of this block
        float z[kBF];
#pragma unroll
        for (int i = 0; i < kBF; ++i) z[i] = 0.0f;
        float sab = 0.0f;
        for (int kb = 0; kb < nk; ++kb) {
            if (!mbar_wait(&G.tfull[acc], accphase, P.abort_flag)) return;
            tc_fence_after();
            float m = 0.0f;
            if (FD_DBG(kDbgGateNoEpi)) goto folded;
            // 32-column chunks: one TMEM load round trip per 32 columns (the fold is on the gate's
            // critical path: the MMA warp reuses this accumulator two stages later)
#pragma unroll
            for (int ch = 0; ch < kBF / 32; ++ch) {
                if (ch * 32 < P.gate_n) {
                    uint32_t v[32];
                    tmem_ld32(tmem + lanes + (uint32_t)(acc * kNT + ch * 32), v);
                    tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        z[ch * 32 + i] = __fadd_rn(z[ch * 32 + i], __uint_as_float(v[i]));
                        if (ch * 32 + i < nv) m = fmaxf(m, fabsf(z[ch * 32 + i]));
                    }
                }
            }
            sab = __fadd_ru(sab, m);
        folded:
            tc_fence_before();
            __syncwarp();
            if ((et & 31) == 0) mbar_arrive(&G.tempty[acc]);
            if (++acc == kAccStages) { acc = 0; accphase ^= 1u; }
        }
        // the last stage's tfull also covered every correction MMA of the tile
        if (FD_DBG(kDbgGateOnly) && et == 0) R.trace[(size_t)blockIdx.x % P.ctas_per_rank * kTracePts + 22] = globaltimer();
#pragma unroll
        for (int ch = 0; ch < kBF / 16; ++ch) {
            if (ch * 16 < P.gate_n) {
                uint32_t v[16];
                tmem_ld16(tmem + lanes + kTmemCorr + (uint32_t)(ch * 16), v);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 16; ++i) z[ch * 16 + i] = __fadd_rn(z[ch * 16 + i], __uint_as_float(v[i]));
            }
        }
        tc_fence_before();
        __syncwarp();
        if ((et & 31) == 0) mbar_arrive(&G.cempty);
        if (et < valid) {
            float* zrow = R.g_phi + (size_t)(tok0 + et) * P.E + e0;
            if ((P.E & 3) == 0) {   // 16-byte rows (e0 is a multiple of 16): a quarter of the store instructions
#pragma unroll
                for (int i = 0; i < kBF; i += 4)
                    if (i < nv) *reinterpret_cast<float4*>(zrow + i) = make_float4(z[i], z[i + 1], z[i + 2], z[i + 3]);
            } else {
#pragma unroll
                for (int i = 0; i < kBF; ++i)
                    if (i < nv) zrow[i] = z[i];
            }
            int* sp = reinterpret_cast<int*>(R.gate_sab) + tok0 + et;
            if (eb == 0) *sp = __float_as_int(sab);
            else atomicMax(sp, __float_as_int(sab));   // non-negative floats order like their bits
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (FD_DBG(kDbgGateOnly) && et == 0) R.trace[(size_t)blockIdx.x % P.ctas_per_rank * kTracePts + 23] = globaltimer();
        if (et == 0) mbar_arrive(&G.qempty[q]);
        if (++q == kTaskRing) { q = 0; qphase ^= 1u; }
    }
}

__device__ __forceinline__ void init_ctrl_fp32(GemmCtrl& G, uint32_t tmem_base, uint32_t tempty_count) {
    using Cfg = GemmCfg<kFP32>;
    // the tensor-core gate runs on the two FP32 issuer warps (gemm_mma_fp32_pp): each commits every token stage
    // (both read it: one atom each) and every per-stage accumulator, and both take tasks from the ring
    for (int i = 0; i < Cfg::STAGES; ++i) { mbar_init(&G.ready[i], ReadyCount<kFP32>::N); mbar_init(&G.done[i], 2); }
    for (int i = 0; i < Cfg::WSTAGES; ++i) { mbar_init(&G.wfull[i], 1); mbar_init(&G.wempty[i], 4); }
    for (int i = 0; i < 2; ++i) { mbar_init(&G.afull[i], 4); mbar_init(&G.aempty[i], 1); mbar_init(&G.pp[i], 1); }
    mbar_init(&G.cempty, 4);
    for (int i = 0; i < kAccStages; ++i) { mbar_init(&G.tfull[i], 2); mbar_init(&G.tempty[i], tempty_count); }
    for (int i = 0; i < kTaskRing; ++i) { mbar_init(&G.qfull[i], 1); mbar_init(&G.qempty[i], TaskConsumers<kFP32>::N); }
    for (int i = 0; i < kTaskRing; ++i) { mbar_init(&G.sfull[i], 1); mbar_init(&G.sempty[i], 1); }
    G.tmem_base = tmem_base;
    G.pp_corr = 0;
    G.pp_cph = 0;
}

// ================================================================ phase 4: combine
static_assert(kCombineTok == kGateTok, "combine tasks are aligned with gate blocks (blk_ready)");
// O[t] = sum over the token's kept picks, in pick order, of w * y (oracle.hpp:102-107): one warp
// per token, 16-byte column chunks, all of a token's landed rows loaded before the adds.
// The CTA first waits once for every combine tile this rank expects (n_e = kept rows per expert,
// saved from the dispatch phase in sN), so the per-token loop has no flag traffic.
constexpr int kCombUnroll = 8;

__device__ void combine_phase(const LaunchParams& P, const RankCtx& R, float* __restrict__ O, uint8_t* smem,
                              const int* __restrict__ sN, unsigned long long* stat) {
    const int S = P.S, H = P.H, K = P.k;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t par = P.epoch & 1u;
    int* sTask = reinterpret_cast<int*>(smem);
    const int ntask = (S + kCombineTok - 1) / kCombineTok;
    const float* yc = reinterpret_cast<const float*>(R.peer_heap[R.rank] + R.hl.yc);
    const unsigned long long* cflag =
        reinterpret_cast<const unsigned long long*>(R.peer_heap[R.rank] + R.hl.cflag[par]);

    // (1) every expected combine tile has landed (acquire), then CTA barrier
    const int nflags = P.E * P.RBF * P.NB1;
    bool ok = true;
    for (int f = tid; f < nflags && ok; f += kThreads) {
        const int e = f / (P.RBF * P.NB1);
        const int rbf = (f / P.NB1) % P.RBF;
        if (sN[e] > rbf * kBM)
            if (wait_epoch_flag(P, R, cflag + f, 400) < 0) ok = false;
    }
    if (!__syncthreads_and(ok)) return;

    const int H4 = H >> 2;
    const int cta = blockIdx.x % P.ctas_per_rank;
    int prev_t = -1;
    uint64_t prev_t0 = 0;
    while (true) {
        __syncthreads();
        if (tid == 0) {
            if (prev_t >= 0)
                emit_event(P, R, kEvExec, cta, kTaskCombine, prev_t0, globaltimer(), R.rank, -1, prev_t, -1, -1,
                           min(kCombineTok, S - prev_t * kCombineTok));
            int t = ld_volatile_u32(P.abort_flag) ? ntask : (int)atomicAdd(R.comb_head, 1u);
            // routing of these tokens was written by the CTA that gated them (dispatch phase)
            if (t < ntask && !wait_counter_eq(P, R, R.blk_ready + t, P.epoch, 401)) t = ntask;
            sTask[0] = t;
            prev_t = t < ntask ? t : -1;
            prev_t0 = P.trace_events ? globaltimer() : 0;
        }
        __syncthreads();
        const int t = sTask[0];
        if (t >= ntask) break;
        if (tid == 0) stat[2]++;
        for (int i = warp; i < kCombineTok; i += kThreads / 32) {
            const int tok = t * kCombineTok + i;
            if (tok >= S) break;
            // this token's picks, one per lane, then broadcast
            int my_e = 0, my_s = -1;
            float my_w = 0.0f;
            if (lane < K) {
                my_s = R.pick_slot[(size_t)tok * K + lane];
                my_e = R.pick_e[(size_t)tok * K + lane];
                my_w = R.pick_w[(size_t)tok * K + lane];
            }
            const float4* yrow[8];
            float wj[8];
            int nk = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (j >= K) break;
                const int sj = __shfl_sync(0xffffffffu, my_s, j);
                const int ej = __shfl_sync(0xffffffffu, my_e, j);
                const float w = __shfl_sync(0xffffffffu, my_w, j);
                yrow[j] = reinterpret_cast<const float4*>(yc + ((size_t)ej * P.C + (sj < 0 ? 0 : sj)) * H);
                wj[j] = sj < 0 ? 0.0f : w;
                nk += sj < 0 ? 0 : (1 << j);   // bitmask of kept picks
            }
            float4* orow = reinterpret_cast<float4*>(O + (size_t)tok * H);
            for (int c0 = lane; c0 < H4; c0 += 32 * kCombUnroll) {
                float4 acc[kCombUnroll];
#pragma unroll
                for (int u = 0; u < kCombUnroll; ++u) acc[u] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (j >= K) break;
                    if (!(nk & (1 << j))) continue;   // capacity-dropped: zero contribution
                    float4 y[kCombUnroll];
#pragma unroll
                    for (int u = 0; u < kCombUnroll; ++u)
                        if (c0 + 32 * u < H4) y[u] = __ldcs(yrow[j] + c0 + 32 * u);
#pragma unroll
                    for (int u = 0; u < kCombUnroll; ++u) {
                        acc[u].x = __fadd_rn(acc[u].x, __fmul_rn(wj[j], y[u].x));
                        acc[u].y = __fadd_rn(acc[u].y, __fmul_rn(wj[j], y[u].y));
                        acc[u].z = __fadd_rn(acc[u].z, __fmul_rn(wj[j], y[u].z));
                        acc[u].w = __fadd_rn(acc[u].w, __fmul_rn(wj[j], y[u].w));
                    }
                }
#pragma unroll
                for (int u = 0; u < kCombUnroll; ++u)
                    if (c0 + 32 * u < H4) __stcs(orow + c0 + 32 * u, acc[u]);
            }
        }
    }
}

// ================================================================ the layer kernel
template <int PREC>
__global__ void __launch_bounds__(kThreads, 1) fdmoe_layer_kernel(const __grid_constant__ LaunchParams P) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // align to 1024 B (SWIZZLE_128B atoms) by offsetting the shared array itself, so nvcc keeps
    // the shared address space (LDS/STS, not generic LD/ST) for every pointer derived from it
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    using Cfg = GemmCfg<PREC>;
    const int rl = blockIdx.x / P.ctas_per_rank;
    const int cta = blockIdx.x % P.ctas_per_rank;
    const RankCtx& R = P.ranks[rl];
    const float* A = P.in[rl];
    float* O = P.out[rl];
    const int tid = threadIdx.x, warp = tid >> 5;
    __shared__ unsigned long long s_stat[5];   // gemm0/gemm1 tiles, combine tasks, full-exact / pair-resolved gate tokens
    __shared__ int s_n_expert[kMaxExperts];   // kept rows per expert of this rank (dispatch -> combine)
    __shared__ unsigned long long s_exp_tab[32];   // glibc expf table (divergent lookups: smem, not __constant__)
    if (tid < 5) s_stat[tid] = 0;
    if (tid < 32) s_exp_tab[tid] = c_exp_tab[tid];
    unsigned long long* trace = R.trace + (size_t)cta * kTracePts;
    if (tid == 0) { trace[0] = globaltimer(); trace[kTrClk0] = clock64(); }

    GemmCtrl& G = *reinterpret_cast<GemmCtrl*>(smem + SmemPlan<PREC>::REGION);
    uint8_t* ring = smem;

    // TMEM: allocated once for the whole launch (1 CTA per SM, all 512 columns)
    if (warp == kWarpTmem) {
        tmem_alloc(&G.tmem_base, 512);
        tmem_relinquish();
    }
    // phase 0: rank-local control reset (consumed only after the grid barrier)
    if (cta == 0) {
        if (tid == 0) { *R.gemm_head = 0; *R.comb_head = 0; }
        for (int e = tid; e < P.E; e += kThreads) R.sent[e] = 0;
        for (int i = tid; i < P.El * P.MT; i += kThreads) R.g0done[i] = 0;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = G.tmem_base;

    // phase 1a: gate logits on the tensor cores (FP32 pipeline roles, own control block)
    if (P.gate_tc) {
        GemmCtrl& GG = *reinterpret_cast<GemmCtrl*>(smem + SmemPlan<PREC>::CTRL_GATE);
        if (tid == 0) {
            init_ctrl_fp32(GG, tmem_base, 4);   // gate epilogue: one tempty arrival per warp per stage
            mbar_fence_init();
        }
        __syncthreads();
        int tokA, tokB, b0, b1;
        gate_token_range(P, cta, tokA, tokB, b0, b1);
        if (tid == 0) trace[kTrGateStart] = globaltimer();
        if (warp == kWarpMma || warp == kWarpTmem) {
            gemm_mma_fp32_pp(P, ring, GG, trace, (cta == 0 && R.chunklog) ? R.chunklog : nullptr, warp == kWarpMma ? 0 : 1);
        } else if (warp == kWarpProducer) {
            if ((tid & 31) == 0) gate_producer(P, R, rl, ring, GG, tokA, tokB);
        } else if (warp >= kWarpConv0 && warp < kWarpConv0 + 4) {
            gemm_wconvert<kFP32>(P, ring, GG, nullptr, nullptr, R.gate_na);
        } else if (warp >= kWarpEpi0 && warp < kWarpEpi0 + 4) {
            gate_epilogue(P, R, GG);
            if (tid == kWarpEpi0 * 32) trace[kTrGateEpiDone] = globaltimer();
        }
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
        if (tid == 0) trace[kTrGateTc] = globaltimer();
        if (FD_DBG(kDbgGateOnly)) goto done;
    }
    // phase 1b: routing (certified from the tensor-core logits, or the SIMT gate), smem region as scratch
    gate_phase(P, R, A, cta, smem, s_stat, s_exp_tab);
    if (tid == 0) {
        trace[1] = globaltimer();
        emit_event(P, R, kEvGateDone, cta, 0, trace[0], trace[1], R.rank, -1, -1, -1, -1, 0);
    }
    if (!rank_barrier(P, R, P.launch_seq)) goto done;
    // near-tie tokens listed by the gate: every CTA computes a share of their exact chains, owners route them
    if (!full_exact_distributed(P, R, A, smem, cta, s_exp_tab)) goto done;
    if (!rank_barrier(P, R, P.launch_seq + 1)) goto done;
    if (cta == 0 && tid == 0) { R.full_ctr[0] = 0; R.full_ctr[1] = 0; R.full_ctr[2] = 0; }   // next launch's list
    if (tid == 0) trace[2] = globaltimer();

    // phase 2: slot assignment, then (after the slot table is complete) the balanced row push
    dispatch_phase(P, R, A, cta, smem);
    if (tid == 0) trace[kTrSlots] = globaltimer();
    if (!rank_barrier(P, R, P.launch_seq + 2)) goto done;
    if (tid == 0) trace[kTrSlotBarrier] = globaltimer();
    push_phase(P, R, A, cta, smem);
    __syncthreads();
    if (tid == 0) trace[kTrPush] = globaltimer();
    for (int e = tid; e < P.E; e += kThreads) s_n_expert[e] = reinterpret_cast<const int*>(smem)[kMaxExperts + e];
    // sequential schedule: every rank's dispatch lands before any expert tile starts
    if (P.sequential && !group_barrier(P, R, P.launch_seq + 3, 0, cta)) goto done;
    if (tid == 0) { trace[3] = globaltimer(); trace[kTrClkFfn0] = clock64(); }

    // phase 3: expert FFN tiles
    if (tid == 0) {
        // FP32: one ready/done pair per token atom (slot 2 * stage + atom, gemm_producer); bf16: per stage
        for (int i = 0; i < Cfg::STAGES * (PREC == kFP32 ? Cfg::NATOM : 1); ++i) {
            mbar_init(&G.ready[i], ReadyCount<PREC>::N);
            mbar_init(&G.done[i], 1);
        }
        for (int i = 0; i < Cfg::WSTAGES; ++i) { mbar_init(&G.wfull[i], 1); mbar_init(&G.wempty[i], 4); }
        for (int i = 0; i < 2; ++i) { mbar_init(&G.afull[i], 4); mbar_init(&G.aempty[i], 1); mbar_init(&G.pp[i], 1); }
        mbar_init(&G.cempty, 4);
        for (int i = 0; i < kAccStages; ++i) { mbar_init(&G.tfull[i], MmaCommits<PREC>::N); mbar_init(&G.tempty[i], 1); }
        for (int i = 0; i < kTaskRing; ++i) { mbar_init(&G.qfull[i], 1); mbar_init(&G.qempty[i], TaskConsumers<PREC>::N); }
        for (int i = 0; i < kTaskRing; ++i) { mbar_init(&G.sfull[i], 1); mbar_init(&G.sempty[i], 1); }
        G.tmem_base = tmem_base;
        G.pp_corr = 0;
        G.pp_cph = 0;
        mbar_fence_init();
    }
    fence_proxy_async_smem();   // the smem region was written by the generic proxy in phases 1-2
    __syncthreads();
    // Role placement follows the warp arbiter (highest warp id first): the single-lane MMA issuer
    // and TMA producer get the top warp ids so busy converter/epilogue warps cannot starve them.
    if (warp == kWarpMma || (PREC == kFP32 && warp == kWarpTmem)) {
        unsigned long long* clog = (cta == 0 && R.chunklog) ? R.chunklog : nullptr;
        if constexpr (PREC == kFP32) gemm_mma_fp32_pp(P, ring, G, trace, clog, warp == kWarpMma ? 0 : 1);
        else gemm_mma<PREC>(P, ring, G, trace, clog);
    } else if (warp == kWarpProducer) {
        if ((tid & 31) == 0) gemm_producer<PREC>(P, R, ring, G, trace);
    } else if (warp >= kWarpConv0 && warp < kWarpConv0 + 4) {
        gemm_wconvert<PREC>(P, ring, G, trace, (cta == 0 && R.chunklog) ? R.chunklog : nullptr);
    } else if (warp == kWarpSignal) {
        if ((tid & 31) == 0) gemm_signal(P, R, G, s_stat);
    } else if (warp >= kWarpEpi0 && warp < kWarpEpi0 + 4) {
        unsigned long long* elog = (cta == 0 && R.chunklog) ? R.chunklog : nullptr;
        // both precisions fuse the combine into the GEMM1 epilogue when the launch holds every rank (round 2: bf16
        // c4 0.672 -> 0.651 ms, c5 0.170 -> 0.158 ms, tools/ab.py; in round 1 its epilogue-bound FFN did not gain)
        if (P.fused_combine) gemm_epilogue<PREC, true>(P, R, G, s_stat, trace, elog);
        else gemm_epilogue<PREC, false>(P, R, G, s_stat, trace, elog);
    }
    __syncthreads();
    // sequential schedule: every rank's expert compute drains before any combine starts
    if (P.sequential && !group_barrier(P, R, P.launch_seq + 5, 1, cta)) goto done;
    if (tid == 0) { trace[4] = globaltimer(); trace[kTrClkFfn1] = clock64(); }

    // phase 4: combine (fused into the GEMM1 epilogues when P.fused_combine)
    if (!P.fused_combine && ld_volatile_u32(P.abort_flag) == 0) combine_phase(P, R, O, smem, s_n_expert, s_stat);
    if (tid == 0) trace[5] = globaltimer();

done:
    __syncthreads();
    if (tid == 0) {
        trace[6] = globaltimer();
        trace[kTrClkEnd] = clock64();
        trace[7] = s_stat[0] + s_stat[1];
        emit_event(P, R, kEvSpawn, cta, 0, trace[0], trace[6], R.rank, -1, -1, -1, -1, 0);
    }
    if (warp == kWarpTmem) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
    }
    if (tid == 0) {
        atomicAdd(R.stats + 0, s_stat[0]);
        atomicAdd(R.stats + 1, s_stat[1]);
        atomicAdd(R.stats + 2, s_stat[2]);
        atomicAdd(R.stats + 3, s_stat[3]);
        atomicAdd(R.stats + 4, s_stat[4]);
    }
}

// ================================================================ weight preparation
// W (E_local x Rr x Cc, row-major: the reference's N-contiguous layout, config.hpp:130-135)
// -> W^T (E_local x Cc x Rr, K-major) as FP32 (split into tf32 hi/lo on chip) or bf16.
__global__ void prep_transpose_kernel(const float* __restrict__ W, int El, int Rr, int Cc, void* out, int prec) {
    __shared__ float tile[32][33];
    const int e = blockIdx.z;
    const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
    const float* src = W + (size_t)e * Rr * Cc;
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int r = r0 + i, c = c0 + threadIdx.x;
        tile[i][threadIdx.x] = (r < Rr && c < Cc) ? src[(size_t)r * Cc + c] : 0.0f;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int c = c0 + i, r = r0 + threadIdx.x;   // output row c, col r
        if (c < Cc && r < Rr) {
            const float v = tile[threadIdx.x][i];
            const size_t o = (size_t)e * Cc * Rr + (size_t)c * Rr + r;
            if (prec == kFP32) reinterpret_cast<float*>(out)[o] = v;
            else reinterpret_cast<__nv_bfloat16*>(out)[o] = __float2bfloat16_rn(v);
        }
    }
}

#ifdef FDMOE_DEV   // diagnostics: libfdmoe_dev.so only (include/fdmoe_dev.h)
// ================================================================ debug entry points
__global__ void debug_expf_kernel(const float* x, float* y, long long n) {
    __shared__ unsigned long long s_tab[32];
    if (threadIdx.x < 32) s_tab[threadIdx.x] = c_exp_tab[threadIdx.x];
    __syncthreads();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        y[i] = expf_glibc(x[i], s_tab);
}

// One tile through the layer's exact machinery (weight loader -> TMEM, TMA token ring,
// tcgen05.mma, TMEM epilogue): D[f][t] = sum_k W[f][k] * X[t][k], 128 x 128, K-major inputs.
// W: FP32 [128][K] (bf16 mode: bf16), X planes via tensor maps (128 rows).
template <int PREC>
__global__ void __launch_bounds__(kThreads, 1) debug_gemm_kernel(const __grid_constant__ CUtensorMap tx0,
                                                                 const __grid_constant__ CUtensorMap tx1,
                                                                 const __grid_constant__ CUtensorMap tw, int K,
                                                                 float* D, uint32_t* abort_flag) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    using Cfg = GemmCfg<PREC>;
    GemmCtrl& G = *reinterpret_cast<GemmCtrl*>(smem + SmemPlan<PREC>::REGION);
    const int tid = threadIdx.x, warp = tid >> 5;
    if (warp == kWarpTmem) { tmem_alloc(&G.tmem_base, 512); tmem_relinquish(); }
    if (tid == 0) {
        for (int i = 0; i < Cfg::STAGES; ++i) { mbar_init(&G.ready[i], ReadyCount<PREC>::N); mbar_init(&G.done[i], 1); }
        for (int i = 0; i < Cfg::WSTAGES; ++i) { mbar_init(&G.wfull[i], 1); mbar_init(&G.wempty[i], 4); }
        for (int i = 0; i < 2; ++i) { mbar_init(&G.afull[i], 4); mbar_init(&G.aempty[i], 1); }
        mbar_init(&G.cempty, 4);
        mbar_init(&G.tfull[0], 1);
        for (int i = 0; i < kTaskRing; ++i) { mbar_init(&G.qfull[i], 1); mbar_init(&G.qempty[i], kTaskConsumers); }
        G.ring[0].type = 0;
        G.ring[1].type = -1;
        mbar_fence_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) { mbar_arrive(&G.qfull[0]); mbar_arrive(&G.qfull[1]); }   // one task, then end
    const uint32_t tmem = G.tmem_base;
    const int nk = (K + Cfg::BK - 1) / Cfg::BK;
    if (tid == kWarpProducer * 32) {
        int stage = 0, wstage = 0; uint32_t phase = 0, wphase = 0;
        const CUtensorMap* tb[2] = {&tx0, &tx1};
        for (int kb = 0; kb < nk; ++kb) {
            mbar_wait(&G.wempty[wstage], wphase ^ 1u, abort_flag);
            mbar_expect_tx(&G.wfull[wstage], Cfg::W_BYTES);
            for (int at = 0; at < Cfg::NATOM; ++at)
                tma_load_2d(smem + Cfg::W_OFF + wstage * Cfg::W_BYTES + at * Cfg::ATOM_BYTES, &tw, &G.wfull[wstage],
                            kb * Cfg::BK + at * Cfg::ATOM_K, 0);
            if (++wstage == Cfg::WSTAGES) { wstage = 0; wphase ^= 1u; }
            mbar_wait(&G.done[stage], phase ^ 1u, abort_flag);
            uint8_t* st = smem + stage * Cfg::STAGE_BYTES;
            mbar_expect_tx(&G.ready[stage], Cfg::STAGE_BYTES);
            for (int pl = 0; pl < Cfg::PLANES; ++pl)
                for (int at = 0; at < Cfg::NATOM; ++at)
                    tma_load_2d(st + pl * Cfg::PLANE_BYTES + at * Cfg::ATOM_BYTES, tb[pl], &G.ready[stage],
                                kb * Cfg::BK + at * Cfg::ATOM_K, 0);
            if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1u; }
        }
    } else if (warp == kWarpMma) {   // the whole warp, one elected lane issues (as in the layer kernel)
        if constexpr (PREC == kFP32) {
            LaunchParams P{};
            P.abort_flag = abort_flag;
            MmaFp32State st;
            long long w = 0;
            mma_tile_fp32(P, smem, G, tmem, tmem, nk, GemmCfg<kFP32>::IDESC, st, w);
        } else {
            int stage = 0; uint32_t phase = 0;
            for (int kb = 0; kb < nk; ++kb) {
                wwait(&G.ready[stage], phase, abort_flag);
                tc_fence_after();
                const uint64_t bd = umma_desc_kmajor(smem_u32(smem + stage * Cfg::STAGE_BYTES), 128);
                if (elect_one())
                    issue_stage<PREC, 0, StageMmas<PREC>::N>(tmem, tmem + Cfg::TMEM_A0 + stage * Cfg::A_COLS, bd, kb == 0);
                __syncwarp();
                wcommit(&G.done[stage]);
                if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1u; }
            }
        }
        wcommit(&G.tfull[0]);
    } else if (warp >= kWarpConv0 && warp < kWarpConv0 + 4) {
        LaunchParams P{};
        P.H = K; P.D = K; P.abort_flag = abort_flag;
        gemm_wconvert<PREC>(P, smem, G, nullptr, nullptr);
    } else if (warp >= kWarpEpi0 && warp < kWarpEpi0 + 4) {
        const int et = tid - kWarpEpi0 * 32, wq = et >> 5;
        mbar_wait(&G.tfull[0], 0, abort_flag);
        tc_fence_after();
        if (PREC == kFP32) fold_corr(tmem + ((uint32_t)(wq * 32) << 16), tmem + ((uint32_t)(wq * 32) << 16) + kTmemCorr);
        for (int ch = 0; ch < kNT / 32; ++ch) {
            uint32_t r[32];
            tmem_ld32(tmem + ((uint32_t)(wq * 32) << 16) + ch * 32, r);
            tmem_wait_ld();
            for (int i = 0; i < 32; ++i) D[(size_t)et * kNT + ch * 32 + i] = __uint_as_float(r[i]);
        }
        tc_fence_before();
    }
    __syncthreads();
    if (warp == kWarpTmem) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

// MMA issue-rate microbenchmark: `nissuers` warps (lane 0 each) issue `iters` tcgen05.mma (M=128,
// A from TMEM, tf32 or bf16) back to back, each into its own accumulator; returns SM cycles for
// the whole batch / total MMAs (i.e. cycles per MMA per SM).
template <int KIND, int N>
__device__ __forceinline__ void mma_burst(uint32_t d, uint32_t a_t, uint64_t b, int iters, int walk) {
    constexpr uint32_t idesc = umma_idesc(KIND == 0 ? 2u : 1u, 128, N);
    mma_tf32_ts(d, a_t, b, idesc, 0u);
    if (walk == 4 || walk == 5) {   // streaming operands: 40 distinct B (10 atoms x 4 k-steps), A walks 32 groups
        for (int i = 1; i < iters; i += 40) {
#pragma unroll
            for (int j = 0; j < 40; ++j) {
                const uint32_t aa = walk == 4 ? a_t + (uint32_t)((j % 32) * 8) : a_t + (uint32_t)((j & 3) * 8);
                mma_tf32_ts(d, aa, b + (uint64_t)((((j >> 2) % 10) * 16384 + (j & 3) * 32) >> 4), idesc, 1u);
            }
        }
        return;
    }
    if (walk == 6) {   // B streams (40 distinct), A fixed 4 groups -- see walk 5; walk 7: A streams, B 8 fixed
        for (int i = 1; i < iters; i += 40) {
#pragma unroll
            for (int j = 0; j < 40; ++j)
                mma_tf32_ts(d, a_t + (uint32_t)((j % 32) * 8), b + (uint64_t)((((j >> 2) & 1) * 16384 + (j & 3) * 32) >> 4), idesc, 1u);
        }
        return;
    }
    if (walk == 7) {   // the FFN pattern with the A slot (TMEM +64 columns) and B atom (+16 KB) alternating per group
        for (int i = 1; i < iters; i += 24) {
#pragma unroll
            for (int sl = 0; sl < 2; ++sl) {
                const uint32_t a = a_t + 128u + sl * 64u;
                const uint64_t bd = b + (uint64_t)(sl * 1024);
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) mma_tf32_ts(d, a + 32 + ks * 8, bd + ((ks * 32) >> 4), idesc, 1u);
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) mma_tf32_ts(d, a + ks * 8, bd + ((32768 + ks * 32) >> 4), idesc, 1u);
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) mma_tf32_ts(d, a + ks * 8, bd + ((ks * 32) >> 4), idesc, 1u);
            }
        }
        return;
    }
    if (walk >= 2) {   // the FFN's 12-MMA half-stage pattern (lo*hi, hi*lo from plane +32 KB, hi*hi)
        const uint32_t a = a_t + (walk == 3 ? 128u : 0u);   // walk 3: A at column 384 (the kernel's ring)
        for (int i = 1; i < iters; i += 12) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) mma_tf32_ts(d, a + 32 + ks * 8, b + ((ks * 32) >> 4), idesc, 1u);
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) mma_tf32_ts(d, a + ks * 8, b + ((32768 + ks * 32) >> 4), idesc, 1u);
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) mma_tf32_ts(d, a + ks * 8, b + ((ks * 32) >> 4), idesc, 1u);
        }
        return;
    }
    for (int i = 1; i < iters; i += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            // walk = 1: each MMA reads a different B slice (k-step inside the 128B atom, then stage)
            const uint64_t bb = walk ? b + (uint64_t)(((u & 3) * 32 + (u >> 2) * (N * 128)) >> 4) : b;
            const uint32_t aa = walk ? a_t + (u & 3) * 8 : a_t;
            if (KIND == 0) mma_tf32_ts(d, aa, bb, idesc, 1u);
            else mma_bf16_ts(d, aa, bb, idesc, 1u);
        }
    }
}

__global__ void __launch_bounds__(384, 1) debug_mma_rate_kernel(int kind, int N, int iters, int nissuers,
                                                                 unsigned long long* out, int walk, int spin_mode) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t s_bar[4];
    __shared__ __align__(8) uint64_t s_never;
    __shared__ volatile int s_stop;
    __shared__ long long s_t[2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x)   // pseudo-random finite data
        reinterpret_cast<float*>(smem)[i] = walk ? (float)((i * 2654435761u) >> 20) * 1e-3f - 2.0f : 0.0f;
    if (warp == 0) { tmem_alloc(&s_tmem, 512); tmem_relinquish(); }
    if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) mbar_init(&s_bar[i], 1); mbar_init(&s_never, 1); s_stop = 0; mbar_fence_init(); }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;
    const uint64_t b = umma_desc_kmajor(smem_u32(smem + (walk ? 0 : 32768)), 128);
    const int spinners = blockDim.x / 32 - 4;   // warps 4.. spin (noise) while warp 0..3 issue
    if (walk && warp < 4) {   // random tf32/bf16-valid data in the A stages too
        uint32_t v[16];
        for (int i = 0; i < 16; ++i) v[i] = __float_as_uint((float)((threadIdx.x * 16 + i) % 7) * 0.25f - 0.7f);
        for (int c = 0; c < 256; c += 16) tmem_st16(tmem + ((uint32_t)(warp * 32) << 16) + 256 + c, v);
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) s_t[0] = clock64();
    __syncthreads();
    if (warp >= 4 && spinners > 0) {
        const int mode = spin_mode;
        if (mode == 1) {   // polling noise: try_wait on a barrier that never completes
            while (!s_stop) { mbar_try_wait(&s_never, 0); }
        } else if (mode == 2 || mode == 4) {   // LDS.128 streams over 64 KB of smem (converter-like)
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            int i = threadIdx.x;
            while (!s_stop) {
                const float4 v = reinterpret_cast<const float4*>(smem + 65536)[i & 4095];
                acc.x += v.x; acc.y += v.y;
                i += 384;
                if (mode == 4 && warp < 8 && (i & 1023) < 384) {   // + tcgen05.st into columns [384, 512)
                    uint32_t r16[16];
                    for (int j = 0; j < 16; ++j) r16[j] = __float_as_uint(acc.x + j);
                    tmem_st16(tmem + ((uint32_t)((warp - 4) * 32) << 16) + 384 + ((i >> 10) & 7) * 16, r16);
                    tmem_wait_st();
                }
            }
            if (acc.x == 12345.f) s_t[1] = (long long)acc.y;
        } else if (mode == 3) {   // tcgen05.st streams (converter-like TMEM writes) into columns [384, 512)
            if (warp < 8) {
                uint32_t r16[16];
                for (int j = 0; j < 16; ++j) r16[j] = j;
                int c = 0;
                while (!s_stop) {
                    tmem_st16(tmem + ((uint32_t)((warp - 4) * 32) << 16) + 384 + (c & 7) * 16, r16);
                    tmem_wait_st();
                    ++c;
                }
            }
        }
    }
    if (warp < nissuers && lane == 0) {
        const uint32_t d = tmem + (uint32_t)(warp * (N <= 128 ? 128 : 0));
        const uint32_t a_t = tmem + 256 + warp * 64;
        if (kind == 0) {
            if (N == 64) mma_burst<0, 64>(d, a_t, b, iters, walk);
            else if (N == 128) mma_burst<0, 128>(d, a_t, b, iters, walk);
            else mma_burst<0, 256>(d, a_t, b, iters, walk);
        } else {
            if (N == 64) mma_burst<1, 64>(d, a_t, b, iters, walk);
            else if (N == 128) mma_burst<1, 128>(d, a_t, b, iters, walk);
            else mma_burst<1, 256>(d, a_t, b, iters, walk);
        }
        mma_commit(&s_bar[warp]);
        while (!mbar_try_wait(&s_bar[warp], 0)) {}
        if (warp == 0) out[blockIdx.x] = (unsigned long long)(clock64() - s_t[0]);
        s_stop = 1;
    }
    __syncthreads();
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int VAR>
__device__ __forceinline__ void issue12_var(uint32_t d, uint32_t a, uint64_t bd, uint32_t idesc, uint32_t acc) {
#pragma unroll
    for (int i = 0; i < 12; ++i) {
        const int ks = i & 3, p = i >> 2;
        uint32_t ao; uint32_t bo;
        if (VAR == 1) { ao = (p == 0 ? 32 : 0) + ks * 8; bo = ks * 32; }                          // B plane 0 only
        else if (VAR == 2) { ao = ks * 8; bo = (p == 1 ? 32768 : 0) + ks * 32; }                // A hi only
        else if (VAR == 3) { ao = ks * 8; bo = ks * 32; }                                        // same 4 (A, B) x3
        else if (VAR == 4) { ao = (i & 7) * 8; bo = (i & 7) * 32; }                              // 8 distinct
        else if (VAR == 5) { ao = (p == 1 ? 32 : 0) + ks * 8; bo = (p == 2 ? 32768 : 0) + ks * 32; }   // hi.hi, lo.hi, hi.lo
        else if (VAR == 6) { ao = (p == 0 ? 32 : 0) + ks * 8; bo = (p == 1 ? 16384 : 0) + ks * 32; }   // plane 1 at +16 KB
        else { ao = (p == 0 ? 32 : 0) + ks * 8; bo = (p == 1 ? 32768 : 0) + ks * 32; }          // = the FFN's order
        mma_tf32_ts(d, a + ao, bd + (bo >> 4), idesc, i ? 1u : acc);
    }
}

// FFN pipeline skeleton microbenchmark (148 CTAs x 384 threads): the MMA warp's 3xTF32 issue pattern
// with the layer's barrier protocol, without memory traffic. mode bits: 1 = FFN accumulator pattern
// (lo*hi, hi*lo -> correction accumulator, hi*hi -> main) else every MMA into one accumulator;
// 2 = 2-slot TMEM A ring handshake with 4 converter warps (aempty -> afull); 4 = converters tcgen05.st the
// hi/lo half-stage (64 columns) each time; 8 = per-stage token ring handshake with a producer lane
// (done -> ready, 2 slots). N = MMA N (128 or 256; 256 implies one accumulator). nhalf half-stages of
// 12 MMAs (M=128, K=8 each). Writes cycles of CTA i to out[i].
__global__ void __launch_bounds__(384, 1) debug_pipe_kernel(int mode, int N, int nhalf, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t afull[2], aempty[2], ready[2], done[2], fin;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x)
        reinterpret_cast<float*>(smem)[i] = (float)((i * 2654435761u) >> 20) * 1e-3f - 2.0f;
    if (warp == 0) { tmem_alloc(&s_tmem, 512); tmem_relinquish(); }
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&afull[i], 4); mbar_init(&aempty[i], 1); mbar_init(&ready[i], 1);
            mbar_init(&done[i], (mode & 4096) ? 2 : 1);
        }
        mbar_init(&fin, (mode & 4096) ? 2 : 1);
        mbar_fence_init();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;
    const uint64_t bdesc = umma_desc_kmajor(smem_u32(smem), 128);
    const long long t0 = clock64();
    if ((mode & 1024) && warp < 4) {   // bit 1024: valid tf32 data in the A ring (columns 256..511)
        uint32_t v[16];
        for (int i = 0; i < 16; ++i) v[i] = __float_as_uint((float)((threadIdx.x * 16 + i) % 7) * 0.25f - 0.7f);
        for (int c = 0; c < 256; c += 16) tmem_st16(tmem + ((uint32_t)(warp * 32) << 16) + 256 + c, v);
        tmem_wait_st();
        tc_fence_before();
    }
    __syncthreads();
    tc_fence_after();
    const int issuer = (mode & 256) ? 0 : 11;   // bit 256: issue from warp 0 (free-running modes only)
    const bool pingpong = (mode & 4096) != 0;   // bit 4096: warps 11 / 9 issue alternate half-stages (named-barrier hand-off)
    if ((mode & (2048 | 4096)) && (warp == issuer || (pingpong && warp == 9))) {
        const uint32_t idesc = umma_idesc(2u, 128, (uint32_t)N);
        const uint32_t d_main = tmem, d_corr = tmem + 256u;
        uint32_t aph[2] = {0, 0}, rph[2] = {0, 0};
        const int par = pingpong ? (warp == 9 ? 1 : 0) : -1;
        for (int h = 0; h < nhalf; ++h) {
            const int sl = h & 1, st = (h >> 1) & 1;
            const bool mine = par < 0 || sl == par;
            if ((mode & 8) && sl == 0) {   // both issuers track the token stage (each reads one of its atoms)
                if (par < 0 || true) {
                    while (!mbar_try_wait(&ready[st], rph[st])) {}
                    rph[st] ^= 1u;
                }
            }
            if (!mine) continue;
            if (mode & 2) {
                while (!mbar_try_wait(&afull[sl], aph[sl])) {}
                aph[sl] ^= 1u;
            }
            tc_fence_after();
            if (pingpong && h > 0) asm volatile("bar.sync %0, 64;" ::"r"(1 + par) : "memory");   // h-1 issued
            const uint32_t a = tmem + 384u + (uint32_t)sl * 64u;
            const uint64_t bd = bdesc + (uint64_t)(sl * 1024);
            if (elect_one()) {
                if (mode & 1) {
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks) mma_tf32_ts(d_corr, a + 32 + ks * 8, bd + ((ks * 32) >> 4), idesc, (h | ks) ? 1u : 0u);
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks) mma_tf32_ts(d_corr, a + ks * 8, bd + ((32768 + ks * 32) >> 4), idesc, 1u);
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks) mma_tf32_ts(d_main, a + ks * 8, bd + ((ks * 32) >> 4), idesc, (h | ks) ? 1u : 0u);
                } else {
                    issue12_var<7>(d_main, a, bd, idesc, h ? 1u : 0u);
                }
                if (mode & 2) mma_commit(&aempty[sl]);
                if (mode & 8) { if (pingpong || sl == 1) mma_commit(&done[st]); }
            }
            __syncwarp();
            if (pingpong && h + 1 < nhalf) asm volatile("bar.arrive %0, 64;" ::"r"(2 - par) : "memory");   // h issued
        }
        if (elect_one()) mma_commit(&fin);
        __syncwarp();
        if (warp == issuer) {
            while (!mbar_try_wait(&fin, 0)) {}
            if (lane == 0) out[blockIdx.x] = (unsigned long long)(clock64() - t0);
        }
    }
    if ((mode & (2048 | 4096)) && (warp == issuer || (pingpong && warp == 9))) nhalf = 0;
    if (warp == issuer && lane == 0) {
        const uint32_t idesc = umma_idesc(2u, 128, (uint32_t)N);
        const uint32_t d_main = tmem, d_corr = tmem + 256u;   // (N = 256: one accumulator at column 0)
        uint32_t aph[2] = {0, 0}, rph[2] = {0, 0};
        if (mode == 240) {   // var 15: branch-free loop, h unrolled x2 (compile-time slot), FFN order, one acc
            for (int h = 0; h < nhalf; h += 2) {
#pragma unroll
                for (int sl = 0; sl < 2; ++sl)
                    issue12_var<7>(d_main, tmem + 384u + sl * 64u, bdesc + (uint64_t)(sl * 1024), idesc, h + sl ? 1u : 0u);
            }
            mma_commit(&fin);
            while (!mbar_try_wait(&fin, 0)) {}
            out[blockIdx.x] = (unsigned long long)(clock64() - t0);
            nhalf = 0;
        }
        for (int h = 0; h < nhalf; ++h) {
            const int sl = h & 1, st = (h >> 1) & 1;
            if ((mode & 8) && sl == 0) {
                while (!mbar_try_wait(&ready[st], rph[st])) {}
                rph[st] ^= 1u;
                tc_fence_after();
            }
            if (mode & 2) {
                while (!mbar_try_wait(&afull[sl], aph[sl])) {}
                aph[sl] ^= 1u;
                tc_fence_after();
            }
            const int var = (mode >> 4) & 15;
            // var 8/9/10: FFN order into one accumulator with the A ring at TMEM column 256 / 128 / 320
            const uint32_t a_base = (var == 8 || var == 11) ? 256u : var == 9 ? 128u : var == 10 ? 320u : 384u;
            const uint32_t a = tmem + a_base + (uint32_t)sl * (var == 10 ? 96u : 64u);
            const uint64_t bd = bdesc + (uint64_t)(sl * 1024);   // the stage's second 128-byte atom
            const uint32_t acc = h == 0 ? 0u : 1u;
            if (var) {   // free-running pattern variants (one accumulator, compile-time operand offsets)
                switch (var) {
                    case 1: issue12_var<1>(d_main, a, bd, idesc, acc); break;
                    case 2: issue12_var<2>(d_main, a, bd, idesc, acc); break;
                    case 3: issue12_var<3>(d_main, a, bd, idesc, acc); break;
                    case 4: issue12_var<4>(d_main, a, bd, idesc, acc); break;
                    case 5: issue12_var<5>(d_main, a, bd, idesc, acc); break;
                    case 6: issue12_var<6>(d_main, a, bd, idesc, acc); break;
                    case 9: issue12_var<7>(var == 9 ? tmem + 256u : d_main, a, bd, idesc, acc); break;
                    case 11: {   // FFN accumulator pattern with the A ring at 256: corrections into column 384
                        const uint32_t dc = tmem + 384u;
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks) mma_tf32_ts(dc, a + 32 + ks * 8, bd + ((ks * 32) >> 4), idesc, ks ? 1u : acc);
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks) mma_tf32_ts(dc, a + ks * 8, bd + ((32768 + ks * 32) >> 4), idesc, 1u);
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks) mma_tf32_ts(d_main, a + ks * 8, bd + ((ks * 32) >> 4), idesc, ks ? 1u : acc);
                        break;
                    }
                    default: issue12_var<7>(d_main, a, bd, idesc, acc); break;
                }
            } else if ((mode & 1) && N <= 128) {
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) mma_tf32_ts(d_corr, a + 32 + ks * 8, bd + ((ks * 32) >> 4), idesc, ks ? 1u : acc);
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) mma_tf32_ts(d_corr, a + ks * 8, bd + ((32768 + ks * 32) >> 4), idesc, 1u);
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) mma_tf32_ts(d_main, a + ks * 8, bd + ((ks * 32) >> 4), idesc, ks ? 1u : acc);
            } else {
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) mma_tf32_ts(d_main, a + 32 + ks * 8, bd + ((ks * 32) >> 4), idesc, ks ? 1u : acc);
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) mma_tf32_ts(d_main, a + ks * 8, bd + ((32768 + ks * 32) >> 4), idesc, 1u);
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) mma_tf32_ts(d_main, a + ks * 8, bd + ((ks * 32) >> 4), idesc, 1u);
            }
            if (mode & 2) mma_commit(&aempty[sl]);
            if ((mode & 8) && sl == 1) mma_commit(&done[st]);
        }
        if (mode != 240 && !(mode & (2048 | 4096))) {
            mma_commit(&fin);
            while (!mbar_try_wait(&fin, 0)) {}
            out[blockIdx.x] = (unsigned long long)(clock64() - t0);
        }
    } else if (warp < 4 && (mode & 2)) {
        uint32_t eph[2] = {1, 1};
        uint32_t v[16];
        for (int i = 0; i < 16; ++i) v[i] = __float_as_uint((float)((threadIdx.x * 16 + i) % 7) * 0.25f - 0.7f);
        const uint32_t lane_addr = (uint32_t)(warp * 32) << 16;
        for (int h = 0; h < nhalf; ++h) {
            const int sl = h & 1;
            while (!mbar_try_wait(&aempty[sl], eph[sl])) {}
            eph[sl] ^= 1u;
            tc_fence_after();
            if (mode & 4) {
                const uint32_t col = tmem + lane_addr + 384u + (uint32_t)sl * 64u;
                tmem_st16(col, v); tmem_st16(col + 16, v); tmem_st16(col + 32, v); tmem_st16(col + 48, v);
                tmem_wait_st();
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&afull[sl]);
        }
    } else if (warp == 10 && lane == 0 && (mode & 8)) {
        uint32_t dph[2] = {1, 1};
        for (int s = 0; s < (nhalf + 1) / 2; ++s) {
            const int st = s & 1;
            while (!mbar_try_wait(&done[st], dph[st])) {}
            dph[st] ^= 1u;
            mbar_arrive(&ready[st]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

// Latency probe: issue `n` tf32 N=128 MMAs (+commit) and time until the commit's mbarrier fires;
// also time tcgen05.st (16 columns) + wait::st, and an mbarrier arrive->wait wakeup.
__global__ void __launch_bounds__(128, 1) debug_latency_kernel(int n, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t s_bar[2];
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 32 * 1024 / 4; i += blockDim.x)   // pseudo-random finite operands
        reinterpret_cast<float*>(smem)[i] = (float)((i * 2654435761u) >> 20) * 1e-3f - 2.0f;
    if (warp == 0) { tmem_alloc(&s_tmem, 512); tmem_relinquish(); }
    if (threadIdx.x == 0) { mbar_init(&s_bar[0], 1); mbar_init(&s_bar[1], 1); mbar_fence_init(); }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;
    if (warp < 4 && n >= 2000) {   // random A operand in TMEM
        uint32_t v[16];
        for (int i = 0; i < 16; ++i) v[i] = __float_as_uint((float)(((threadIdx.x * 16 + i) * 2654435761u) >> 22) * 1e-3f - 0.5f);
        for (int c = 0; c < 256; c += 16) tmem_st16(tmem + ((uint32_t)(warp * 32) << 16) + 256 + c, v);
        tmem_wait_st();
        tc_fence_before();
    }
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0 && n >= 2000) {   // exact layer MMA sequence: 64 chunks x 4 k-steps x 3 products
        const int variant = n - 2000;
        using Cfg = GemmCfg<kFP32>;
        const long long t0 = clock64();
        int stage = 0, ast = 0, acc = 0;
        const int nchunk = (variant & 16) ? 25600 : 256;
        for (int c = 0; c < nchunk; ++c) {
            const uint32_t d_tmem = tmem + (uint32_t)(acc * kNT);
            const uint32_t bbase = smem_u32(smem) + stage * 0;   // one 32 KB stage: hi plane + lo plane
            const uint32_t abase = tmem + Cfg::TMEM_A0 + ast * Cfg::A_COLS;
            tc_fence_after();
            if (variant & 8) {   // product-major order: consecutive MMAs never share A columns
#pragma unroll
                for (int p = 0; p < 3; ++p)
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks) {
                        const uint32_t koff = ks * 32;
                        const uint64_t b0 = umma_desc_kmajor(bbase + koff, 128);
                        const uint64_t b1 = umma_desc_kmajor(bbase + 16384 + koff, 128);
                        const uint32_t accum = ((c & 63) | ks | p) != 0 ? 1u : 0u;
                        const uint32_t a_hi = abase + ks * 8, a_lo = a_hi + 32;
                        if (p == 0) mma_tf32_ts(d_tmem, a_lo, b0, Cfg::IDESC, accum);
                        else if (p == 1) mma_tf32_ts(d_tmem, a_hi, b1, Cfg::IDESC, 1u);
                        else mma_tf32_ts(d_tmem, a_hi, b0, Cfg::IDESC, 1u);
                    }
            } else {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                const uint32_t koff = ks * 32;
                const uint64_t b0 = umma_desc_kmajor(bbase + koff, 128);
                const uint64_t b1 = umma_desc_kmajor(bbase + 16384 + koff, 128);
                const uint32_t accum = ((c & 63) | ks) != 0 ? 1u : 0u;
                const uint32_t a_hi = abase + ks * 8, a_lo = a_hi + 32;
                if (variant & 1) {
                    mma_tf32_ts(d_tmem, a_hi, b0, Cfg::IDESC, accum);
                    mma_tf32_ts(d_tmem, a_hi, b0, Cfg::IDESC, 1u);
                    mma_tf32_ts(d_tmem, a_hi, b0, Cfg::IDESC, 1u);
                } else {
                    mma_tf32_ts(d_tmem, a_lo, b0, Cfg::IDESC, accum);
                    mma_tf32_ts(d_tmem, a_hi, b1, Cfg::IDESC, 1u);
                    mma_tf32_ts(d_tmem, a_hi, b0, Cfg::IDESC, 1u);
                }
            }
            }
            mma_commit(&s_bar[0]);
            if (!(variant & 4)) mma_commit(&s_bar[1]);
            if (++ast == 4) ast = 0;
            if ((c & 63) == 63) acc ^= (variant & 2) ? 0 : 1;
        }
        mma_commit(&s_bar[0]);
        const long long t1 = clock64();
        out[blockIdx.x * 4 + 0] = t1 - t0;
        out[blockIdx.x * 4 + 1] = (t1 - t0) / nchunk;
    }
    if (n >= 2000) { __syncthreads(); tc_fence_before(); __syncthreads(); if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); } return; }
    if (threadIdx.x == 0 && n >= 1000) {   // chunk-loop variants: n = 1000 + variant
        const int variant = n - 1000;
        const uint64_t b = umma_desc_kmajor(smem_u32(smem), 128);
        constexpr uint32_t idesc = umma_idesc(2u, 128, 128);
        uint32_t ph = 0;
        const long long t0 = clock64();
        for (int c = 0; c < 64; ++c) {
            if (variant & 1) tc_fence_after();
            if (variant & 4) { while (!mbar_try_wait(&s_bar[1], 1)) {} }   // already-complete parity
#pragma unroll
            for (int i = 0; i < 12; ++i) mma_tf32_ts(tmem, tmem + 256 + (i & 3) * 8, b + ((i & 3) * 2), idesc, (c | i) > 0);
            if (variant & 2) { mma_commit(&s_bar[0]); }
        }
        mma_commit(&s_bar[0]);
        const long long t1 = clock64();
        out[0] = t1 - t0;
        out[1] = (t1 - t0) / 64;
        out[2] = 0; out[3] = 0;
    }
    if (n >= 1000) { __syncthreads(); tc_fence_before(); __syncthreads(); if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); } return; }
    if (threadIdx.x == 0) {
        const uint64_t b = umma_desc_kmajor(smem_u32(smem), 128);
        constexpr uint32_t idesc = umma_idesc(2u, 128, 128);
        const long long t0 = clock64();
        for (int i = 0; i < n; ++i) mma_tf32_ts(tmem, tmem + 256, b, idesc, i > 0);
        const long long t1 = clock64();
        mma_commit(&s_bar[0]);
        while (!mbar_try_wait(&s_bar[0], 0)) {}
        const long long t2 = clock64();
        out[0] = t1 - t0;   // issue time
        out[1] = t2 - t0;   // issue -> completion observed
    }
    __syncthreads();
    if (warp == 1) {
        uint32_t v[16];
        for (int i = 0; i < 16; ++i) v[i] = i;
        const long long t0 = clock64();
        for (int r = 0; r < 8; ++r) tmem_st16(tmem + ((uint32_t)32 << 16) + 256 + r * 16, v);
        tmem_wait_st();
        const long long t1 = clock64();
        if ((threadIdx.x & 31) == 0) out[2] = t1 - t0;   // 8 x st.x16 + wait::st
    }
    __syncthreads();
    if (threadIdx.x == 64) {   // wakeup latency: thread 96 arrives, thread 64 waits
        const long long t0 = clock64();
        while (!mbar_try_wait(&s_bar[1], 0)) {}
        out[3] = clock64() - t0;
    } else if (threadIdx.x == 96) {
        const long long t0 = clock64();
        while (clock64() - t0 < 2000) {}
        mbar_arrive(&s_bar[1]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

cudaError_t launch_debug_latency(int n, unsigned long long* out) {
    cudaFuncSetAttribute(debug_latency_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 34 * 1024);
    const int grid = (n >= 2000 && (n - 2000) & 32) ? 148 : 1;
    debug_latency_kernel<<<grid, 128, 34 * 1024>>>(n, out);
    return cudaGetLastError();
}

cudaError_t launch_debug_mma_rate(int kind, int N, int iters, int nissuers, unsigned long long* out) {
    if (kind >= 16) {   // pipeline skeleton: kind = 16 + mode, iters = half-stages
        cudaFuncSetAttribute(debug_pipe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
        debug_pipe_kernel<<<148, ((kind - 16) & 512) ? 128 : 384, 66 * 1024>>>(kind - 16, N, iters, out);
        return cudaGetLastError();
    }
    cudaFuncSetAttribute(debug_mma_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 161 * 1024);
    const int walk = (nissuers >> 4) & 7;
    const int grid = (nissuers >> 8) & 255 ? (nissuers >> 8) & 255 : 1;   // number of SMs running the benchmark
    const int spin_mode = (nissuers >> 16) & 7;
    const int threads = spin_mode ? 384 : 128;                             // + 8 noise warps
    debug_mma_rate_kernel<<<grid, threads, 161 * 1024>>>(kind, N, iters, nissuers & 15, out, walk, spin_mode);
    return cudaGetLastError();
}

#endif  // FDMOE_DEV

// ---------------------------------------------------------------- host-visible launchers
int layer_smem_bytes(int prec) {
    return prec == kFP32 ? SmemPlan<kFP32>::TOTAL : SmemPlan<kBF16>::TOTAL;
}

cudaError_t launch_layer(const LaunchParams& p, int grid, int smem, cudaStream_t stream) {
    void* args[] = {const_cast<LaunchParams*>(&p)};
    if (p.prec == kFP32) {
        cudaFuncSetAttribute(fdmoe_layer_kernel<kFP32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        return cudaLaunchCooperativeKernel((const void*)fdmoe_layer_kernel<kFP32>, dim3(grid), dim3(kThreads), args,
                                           (size_t)smem, stream);
    }
    cudaFuncSetAttribute(fdmoe_layer_kernel<kBF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return cudaLaunchCooperativeKernel((const void*)fdmoe_layer_kernel<kBF16>, dim3(grid), dim3(kThreads), args,
                                       (size_t)smem, stream);
}

int layer_max_blocks_per_sm(int prec, int smem) {
    int n = 0;
    if (prec == kFP32) {
        cudaFuncSetAttribute(fdmoe_layer_kernel<kFP32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fdmoe_layer_kernel<kFP32>, kThreads, smem);
    } else {
        cudaFuncSetAttribute(fdmoe_layer_kernel<kBF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fdmoe_layer_kernel<kBF16>, kThreads, smem);
    }
    return n;
}

cudaError_t launch_prep_transpose(const float* W, int El, int Rr, int Cc, void* out, int prec, cudaStream_t s) {
    dim3 grid((Cc + 31) / 32, (Rr + 31) / 32, El);
    prep_transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(W, El, Rr, Cc, out, prec);
    return cudaGetLastError();
}

#ifdef FDMOE_DEV
cudaError_t launch_debug_expf(const float* x, float* y, long long n, cudaStream_t s) {
    debug_expf_kernel<<<1024, 256, 0, s>>>(x, y, n);
    return cudaGetLastError();
}

cudaError_t launch_debug_gemm(int prec, const CUtensorMap* t, int K, float* D, uint32_t* abort_flag,
                              cudaStream_t s) {
    const int smem = layer_smem_bytes(prec);
    if (prec == kFP32) {
        cudaFuncSetAttribute(debug_gemm_kernel<kFP32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        debug_gemm_kernel<kFP32><<<1, kThreads, smem, s>>>(t[0], t[1], t[2], K, D, abort_flag);
    } else {
        cudaFuncSetAttribute(debug_gemm_kernel<kBF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        debug_gemm_kernel<kBF16><<<1, kThreads, smem, s>>>(t[0], t[1], t[2], K, D, abort_flag);
    }
    return cudaGetLastError();
}

#endif  // FDMOE_DEV

}  // namespace fdmoe
