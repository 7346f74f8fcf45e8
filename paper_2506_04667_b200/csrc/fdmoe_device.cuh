// fdmoe_device.cuh — sm_100a PTX wrappers (mbarrier, TMA, tcgen05/TMEM, scoped
// flags) and the launch-parameter structs shared by the host runtime and kernels.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>

namespace fdmoe {

// ---------------------------------------------------------------- constants
// 12 warps. FFN roles: w0-3 weight converters (TMA-staged smem -> registers -> tf32 hi/lo -> TMEM),
// w4-7 epilogue (TMEM -> registers -> bias/activation -> global / peer stores), w8 TMEM allocator,
// w9 signal warp (tile release fences / counters / flags), w10 tile scheduler + TMA producer, w11
// tcgen05.mma issuer (the warp arbiter favours high warp ids, so the single-lane issuers sit on top
// and the epilogue above the converters). A warp reaches TMEM lanes 32*(warp % 4) .. +31 only, so
// each 4-warp group covers all 128 lanes.
constexpr int kThreads = 384;
constexpr int kWarpEpi0 = 4, kWarpConv0 = 0, kWarpTmem = 8, kWarpSignal = 9, kWarpProducer = 10, kWarpMma = 11;
constexpr int kBM = 128;            // tokens per row tile of an expert's receive region
constexpr int kBF = 128;            // output features per FFN tile (MMA M = TMEM lanes)
constexpr int kNT = 128;            // tokens per FFN tile (MMA N = accumulator columns)
constexpr int kAccStages = 2;       // TMEM accumulators: 2 x 128 columns
constexpr uint32_t kTmemCorr = 256; // FP32: the tile's 3xTF32 correction accumulator (columns 256..383)
constexpr int kBN = kBF;            // feature block width used by the flag / task arithmetic
constexpr int kTaskRing = 4;        // producer -> MMA/epilogue task ring
constexpr int kGateTok = 16;        // tokens per gate block (slot-assignment / combine granule)
constexpr int kGateKC = 32;         // K chunk of the exact gate
constexpr int kMaxExperts = 256;    // E_total envelope of the exact SIMT gate
constexpr int kMaxRanks = 64;       // P envelope (peer table size)
constexpr int kMaxSrcPerTile = 8;   // packet_rows >= 16 -> <= 8 packets per 128-row tile
constexpr int kCombineTok = 16;     // tokens per combine task (== kGateTok)
constexpr int kMaxLocalRanks = 8;   // ranks per launch (virtual ranks on one GPU)
constexpr int kTracePts = 40;
constexpr int kFullCap = 256;       // rank-wide full-exact token list capacity (overflow: the owner CTA computes)
constexpr int kGroupBarriers = 2;   // sequential mode: after dispatch, after the expert FFN
constexpr int kChunkLog = 512;       // start, gate, barrier, dispatch, gemm, combine, end, tiles,
                                    // then FFN pipeline wait cycles (see kWait*)
enum WaitSlot : int {
    kWaitMmaX = 8, kWaitMmaA, kWaitMmaAcc, kWaitConvW, kWaitConvA, kWaitProdW, kWaitProdX, kWaitEpiAcc,
    kWaitMmaTask, kProdFetch, kEpiBusy, kMmaTiles,
    kTrPrefix = 20, kTrSlots, kTrSlotBarrier, kTrPush,   // dispatch sub-phases (%globaltimer)
    kTrGateLogits = 24, kTrGatePairs, kTrGateFull, kTrGateNFull,  // gate sub-phases (last sub-tile), full tokens
    kTrGateTc = 28,                                               // tensor-core gate logits done
    kTrGateLoad = 29,                                             // tensor-core logits staged for routing
    kTrGateDecide = 30, kTrGateExp = 31,                          // thread-route decisions / exps done
    kTrClk0 = 32, kTrClkFfn0, kTrClkFfn1, kTrClkEnd,              // clock64 at start / FFN start / FFN end / end
    kTrFullChains = 36, kTrFullRouted = 37,                       // distributed full-exact pass: chains claimed / routed
    kTrGateStart = 38, kTrGateEpiDone = 39                        // tensor-core gate: roles start / epilogue done
};

enum Prec : int { kFP32 = 0, kBF16 = 1 };

// Byte offsets inside one rank's symmetric heap (identical on every rank).
struct HeapLayout {
    uint64_t x[2][2];     // [parity][hi|lo] receive buffer (bf16: [parity][0] only)
    uint64_t yc;          // combine-in rows: [E_total][C][H] fp32
    uint64_t dflag[2];    // [parity] -> [E_local][P] u64 dispatch signals
    uint64_t cflag[2];    // [parity] -> [E_total][RBF][NB1] u64 combine tile signals
    uint64_t gbar;        // [kGroupBarriers][P] u64 group-barrier arrivals (sequential mode)
    uint64_t bytes;
};

// One device event record; layout identical to fdmoe_event (include/fdmoe.h).
struct DevEvent {
    uint64_t t0, t1;
    int32_t kind, cta, type, src, expert, rb, cb, peer;
    int64_t value;
};
enum EvKind : int { kEvSpawn = 0, kEvGateDone, kEvDispatchPut, kEvExec, kEvTilePut, kEvBarrierEnter, kEvBarrierExit };
enum EvTask : int { kTaskGemm0 = 1, kTaskGemm1 = 2, kTaskCombine = 3 };

// Everything one rank's kernel needs. Lives in device global memory (64B aligned
// so the embedded TMA descriptors are valid operands of cp.async.bulk.tensor).
struct alignas(64) RankCtx {
    CUtensorMap tm_x[2][2];    // [parity][hi|lo]  rows = E_local*RP, cols = H
    CUtensorMap tm_c1[2];      // [hi|lo]          rows = E_local*RP, cols = D
    CUtensorMap tm_w1;         // W1^T [E_local*D (+pad)][H], FP32 (split on chip) or bf16, box 128 rows
    CUtensorMap tm_w2;         // W2^T [E_local*H (+pad)][D]
    CUtensorMap tm_wg[2];      // tensor-core gate: Wg^T tf32 [hi|lo] planes [gate_nblk * gate_n][H], box gate_n rows

    uint8_t* peer_heap[kMaxRanks];   // heap base of rank q as mapped here (q == rank: own)
    HeapLayout hl;

    // private scratch
    void* c1[2];               // GEMM0 output (hi|lo or bf16)
    const float* b1;           // [E_local][D]
    const float* b2;           // [E_local][H]
    const float* wg;           // [H][E_total]
    const float* wg_norm;      // [E_total] |Wg[:, e]|_2 rounded up (certified gate)
    const float* wgT;          // [E_total][H] Wg transposed (certified gate's exact pair pass)
    double* gate_na;           // [S] tensor-core gate: sum of squares of each token row (converter warps)
    float* gate_sab;           // [S] tensor-core gate: sum over 64-K chunk ends of max_e |prefix logit|
    float* g_phi;              // [S][E_total]
    int32_t* pick_e;           // [S][k]
    int32_t* pick_slot;        // [S][k]  (-1 = capacity-dropped)
    float* pick_w;             // [S][k]
    int32_t* cnt_cta;          // [ctas][E_total] per-CTA expert pick counts
    int32_t* tbl_tok;          // [E_total][C]
    float* tbl_w;              // [E_total][C]
    int32_t* slot_counts;      // [E_total]
    uint32_t* blk_ready;       // [ceil(S/32)] epoch: routing of this token block is final
    // control block (rank-local)
    unsigned long long* bar;   // grid barrier counter (monotonic across launches)
    uint32_t* gemm_head;
    uint32_t* comb_head;
    uint32_t* sent;            // [E_total] rows dispatched so far (last-arriver signals)
    uint32_t* g0done;          // [E_local][MT] GEMM0 tiles completed per row tile
    uint32_t* err;             // [4] error word: code, where, a, b
    unsigned long long* stats; // [8] gemm0, gemm1, combine tasks, dispatch rows, ...
    unsigned long long* trace; // [ctas][kTracePts] %globaltimer per phase boundary (device trace)
    unsigned long long* chunklog;   // debug: CTA 0 MMA-warp chunk timeline [kChunkLog][4] (null = off)
    const unsigned long long* delay_ns;   // [E_total] straggler: cumulative hold-back of packet e's signal
    DevEvent* ev;              // [ev_cap] device event log (fdmoe_event layout)
    uint32_t* ev_ctr;          // records emitted this launch (reset by the host before the launch)
    uint32_t* zero_ctr;        // fused combine: CTAs whose output rows are zeroed (monotonic)
    uint32_t* full_ctr;        // [3] distributed full-exact pass: tokens listed, chains claimed, chains done
    int32_t* full_list;        // [kFullCap] tokens needing every expert's exact logit (ties / near-ties)
    float* full_z;             // [kFullCap][E_total] their exact logits (reference chain, gate.hpp:77-81)
    float* epart;              // [ctas][128 cols][128 rows] FP32 FFN: the first-half main partial of the CTA's tile
    uint32_t ev_cap;
    int32_t rank;
};

struct LaunchParams {
    CUtensorMap tm_in[kMaxLocalRanks];   // tensor-core gate: each local rank's input shard [S][H] FP32, box 128 rows
    RankCtx* ranks;            // device array, one per rank in this launch
    const float* in[kMaxLocalRanks];
    float* out[kMaxLocalRanks];
    // shape
    int S, H, D, E, El, P, k, C, Cp, RP, MT, RBF, NB0, NB1;
    int act, prec;
    int ctas_per_rank, nranks;
    uint32_t epoch;            // 1-based forward counter (same on every rank)
    unsigned long long launch_seq;   // barrier generation
    unsigned long long budget_ns;    // watchdog budget
    uint32_t* abort_flag;      // per launch-group abort word
    int sequential;            // bulk-synchronous schedule (group barrier after dispatch and after the FFN)
    int trace_events;          // record the device event log
    int straggler_rank;        // rank whose packet signals are held back by delay_ns (-1: none)
    uint32_t zero_target;      // fused combine: zero_ctr value once every CTA of this launch zeroed its rows
    int fused_combine;         // 1: GEMM1 epilogues accumulate w * y straight into the origin's output
                               //    (k <= 2: fl(fl(w0 y0) + fl(w1 y1)) is order-free; all ranks of the
                               //    group on this device; overlapped schedule) -- no combine phase
    int debug;                 // ablation bits (FDMOE_DEBUG env; 0 in production): see kDbg*
    int exact_gate;            // 1: reference-exact logits for every token (bit-exact G_phi, weights)
    float gate_u;              // certified gate: u' = 2^-24 * 1.001
    float gate_k1;             // certified gate: 66 + 2 H gamma_{H+1}
    int gate_tc;               // 1: gate logits on the tensor cores (3xTF32), certified with gate_k1_tc
    int gate_n;                // tensor-core gate: MMA N (experts per block, multiple of 16, <= 128)
    int gate_nblk;             // tensor-core gate: expert blocks of gate_n
    float gate_k1_tc;          // tensor-core gate: |z~ - z_ref| <= gate_u * gate_k1_tc * |a| |w_e|
};
enum DebugBits : int {
    kDbgNoConvert = 1,    // converter warps skip the split + tcgen05.st (MMA reads stale TMEM)
    kDbgNoEpiStore = 4,   // epilogue skips global stores
    kDbgNoXTma = 8,       // producer skips the token TMA (barrier completes without data)
    kDbgNoWTma = 16,      // producer skips the weight TMA
    kDbgGateNoNorm = 32,  // certified gate skips the |a|^2 accumulation (bounds wrong: timing only)
    kDbgGateNoFlush = 64, // certified gate skips the exact pass (routing wrong: timing only)
    kDbgGateNoLoad = 128, // gate skips its cp.async loads (timing only)
    kDbgGateNoMath = 256, // gate skips its dot-product loop (timing only)
    kDbgGateNoWgTma = 512,    // tensor-core gate: producer skips the Wg^T plane TMA (timing only)
    kDbgGateNoTokTma = 1024,  // tensor-core gate: producer skips the token-row TMA (timing only)
    kDbgGateNoEpi = 2048,     // tensor-core gate: epilogue skips the per-stage TMEM fold (timing only)
    kDbgEvictNormal = 4096,   // token / C1 / gate-row loads with evict_normal instead of evict_last (A/B)
    kDbgInjectOversub = 8192, // fault injection: CTA 0 over-counts one kept row of expert 0 (ProtocolError test)
    kDbgSimtGate = 16384,     // A/B: SIMT certified gate logits instead of the tensor-core gate
    kDbgHalfCorr = 32768,     // timing only: the FP32 FFN issues half of its correction MMAs (results wrong)
    kDbgGateOnly = 65536,     // timing only: the launch ends after the tensor-core gate (gate role stamps in 20..23)
};

// Ablation bits are honoured only by the development library (libfdmoe_dev.so, -DFDMOE_DEV);
// the product build compiles every FD_DBG test to false.
#ifdef FDMOE_DEV
#define FD_DBG(bit) ((P.debug & (bit)) != 0)
#else
#define FD_DBG(bit) false
#endif

// Error codes written to RankCtx::err[0] (mirrors the reference's exceptions).
enum DevErr : uint32_t { kErrNone = 0, kErrTimeout = 1, kErrProtocol = 2, kErrAccounting = 3 };

#ifdef __CUDACC__
// ---------------------------------------------------------------- misc PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ long long clk() { return clock64(); }
__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const unsigned long long* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_gpu_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t ld_acquire_gpu_u64(const unsigned long long* p) {
    uint64_t v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Wait with an escape hatch: every 4096 probes check the launch-group abort word and a
// hard 20 s ceiling (a lost TMA completion must not wedge the GPU).
__device__ __forceinline__ bool mbar_wait(uint64_t* bar, uint32_t parity, uint32_t* abort_flag) {
    if (mbar_try_wait(bar, parity)) return true;
    const uint64_t t0 = globaltimer();
    uint32_t n = 0;
    while (!mbar_try_wait(bar, parity)) {
        if ((++n & 4095u) == 0) {
            if (ld_volatile_u32(abort_flag) != 0) return false;
            if (globaltimer() - t0 > 20000000000ull) {
                atomicExch(abort_flag, 1u);
                return false;
            }
        }
    }
    return true;
}

// ---------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* m) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(m) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* m, uint64_t* bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
        ::"r"(smem_u32(dst)), "l"(m), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}

// TMA load with an L2 cache-policy hint (createpolicy): expert weights are read exactly once per
// launch (evict_first), so they should not push the reused token / C1 tiles out of L2.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* m, uint64_t* bar, int x, int y,
                                                 uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4}], [%2], %5;"
        ::"r"(smem_u32(dst)), "l"(m), "r"(smem_u32(bar)), "r"(x), "r"(y), "l"(policy)
        : "memory");
}

// ---------------------------------------------------------------- tcgen05
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
}
__device__ __forceinline__ void tmem_relinquish() {
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(d_tmem), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(d_tmem), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// A operand from TMEM (the expert's weight tile), B from shared memory (tokens).
// elect.sync: true in exactly one lane of the (converged) warp
__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(pred));
    return pred != 0;
}
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
        ::"r"(d_tmem), "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
        ::"r"(d_tmem), "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// 32 lanes x 16 consecutive 32-bit columns from registers (thread t -> its lane's row).
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
        ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
          "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
// 32 lanes x 8 consecutive 32-bit columns from registers.
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
// 32 lanes x 32 consecutive 32-bit columns from registers.
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
        ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
          "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
          "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
          "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ float4 ld_stream_f4(const void* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
// bulk L2 prefetch of [p, p + bytes) (16-byte aligned, bytes % 16 == 0), no completion tracking
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
// 32 lanes x 32 consecutive 32-bit columns: thread t of the warp gets its lane's row.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");
}
// 32 lanes x 16 consecutive 32-bit columns.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// UMMA shared-memory matrix descriptor, K-major operand staged by TMA with
// SWIZZLE_{128,64}B: start>>4 [0,14), LBO>>4 [16,30) (unused for swizzled K-major),
// SBO>>4 [32,46) = 8 rows x swizzle width, version 1 [46,48), layout [61,64).
__device__ __forceinline__ uint64_t umma_desc_kmajor(uint32_t smem_addr, uint32_t swizzle_bytes) {
    const uint64_t layout = swizzle_bytes == 128 ? 2ull : (swizzle_bytes == 64 ? 4ull : 6ull);
    const uint64_t sbo = 8ull * swizzle_bytes;
    return (uint64_t)((smem_addr >> 4) & 0x3FFF) | (1ull << 16) | (((sbo >> 4) & 0x3FFF) << 32) |
           (1ull << 46) | (layout << 61);
}
// Instruction descriptor: D=f32 [4,6)=1, A/B format [7,10)/[10,13) (1=bf16, 2=tf32),
// K-major A/B, N>>3 at [17,23), M>>4 at [24,29).
__host__ __device__ constexpr uint32_t umma_idesc(uint32_t ab_format, uint32_t M, uint32_t N) {
    return (1u << 4) | (ab_format << 7) | (ab_format << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
#endif  // __CUDACC__

}  // namespace fdmoe
