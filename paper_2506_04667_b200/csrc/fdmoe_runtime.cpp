// fdmoe_runtime.cpp — host runtime behind the C ABI: rank/heap setup, peer mapping
// (same-process peers or CUDA IPC), weight repacking, TMA descriptors, and exactly one
// cooperative persistent launch per device per forward (runtime.hpp:802-1002 semantics).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <random>
#include <string>
#include <vector>

#include "fdmoe.h"
#include "fdmoe_internal.h"

using namespace fdmoe;

namespace {

#define CK(expr)                                                                                \
    do {                                                                                        \
        cudaError_t _e = (expr);                                                                \
        if (_e != cudaSuccess)                                                                  \
            return fail(FDMOE_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));     \
    } while (0)

constexpr size_t kAlign = 1024;
size_t align_up(size_t x, size_t a = kAlign) { return (x + a - 1) / a * a; }

// Operator geometry derived from the reference config.
struct Dims {
    int64_t S, H, D, E, El, P, k, C, Cp, RP, MT, RBF, NB0, NB1;
    int64_t rows_x, rows_w1, rows_w2;
    int64_t gate_n, gate_nblk;      // tensor-core gate: experts per MMA block (N), blocks
    int prec, esz, planes;
};

Dims make_dims(const fdmoe_config& c) {
    Dims d{};
    d.S = c.tokens_per_device; d.H = c.embed_dim; d.D = c.ffn_dim; d.E = c.experts_total;
    d.P = c.devices; d.El = d.E / d.P; d.k = c.topk;
    d.C = fdmoe_expert_capacity(&c);
    // rows reserved per (source, expert) packet: 16/32/64/128, else a multiple of 128,
    // so a 128-row tile holds whole packets or whole 128-row pieces of one packet
    if (d.C <= 16) d.Cp = 16;
    else if (d.C <= 32) d.Cp = 32;
    else if (d.C <= 64) d.Cp = 64;
    else d.Cp = (d.C + kBM - 1) / kBM * kBM;
    d.RP = d.P * d.Cp;
    d.MT = (d.RP + kBM - 1) / kBM;
    d.RBF = d.Cp >= kBM ? d.Cp / kBM : 1;
    d.NB0 = (d.D + kBF - 1) / kBF;   // GEMM0 feature blocks
    d.NB1 = (d.H + kBF - 1) / kBF;   // GEMM1 feature blocks
    d.rows_x = std::max(d.El * d.RP, (d.El - 1) * d.RP + d.MT * kBM);
    d.rows_w1 = (d.El - 1) * d.D + d.NB0 * kBF;
    d.rows_w2 = (d.El - 1) * d.H + d.NB1 * kBF;
    d.gate_n = d.E <= kBF ? (d.E + 15) / 16 * 16 : kBF;
    d.gate_nblk = (d.E + d.gate_n - 1) / d.gate_n;
    d.prec = c.precision;
    d.esz = c.precision == FDMOE_FP32 ? 4 : 2;
    d.planes = c.precision == FDMOE_FP32 ? 2 : 1;
    return d;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda needed).
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn get_encode() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    }
    return fn;
}

// K-major 2-D operand: rows x cols, box = (128 bytes of K) x box_rows, SWIZZLE_128B.
fdmoe_status make_tmap(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int esz, int box_rows) {
    EncodeFn enc = get_encode();
    if (!enc) return fail(FDMOE_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const CUtensorMapDataType dt = esz == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t gstride[1] = {(cuuint64_t)(cols * esz)};
    cuuint32_t box[2] = {(cuuint32_t)(128 / esz), (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, dt, 2, const_cast<void*>(base), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(FDMOE_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return FDMOE_OK;
}

struct RankRes {
    int rank = 0, dev = 0;
    uint8_t* heap = nullptr;
    HeapLayout hl{};
    size_t heap_bytes = 0;
    uint8_t* scratch = nullptr;     // one allocation carved below
    size_t scratch_bytes = 0;
    void* c1[2] = {nullptr, nullptr};
    void* w1[2] = {nullptr, nullptr};
    void* w2[2] = {nullptr, nullptr};
    float *b1 = nullptr, *b2 = nullptr, *wg = nullptr, *wg_norm = nullptr, *wgT = nullptr;
    float* wg_split = nullptr;      // tensor-core gate: Wg^T tf32 hi plane, then lo plane, [gate_nblk*gate_n][H] each
    double* gate_na = nullptr;      // [S] token-row sums of squares (tensor-core gate)
    float* gate_sab = nullptr;      // [S] certificate chunk-end prefix sums (tensor-core gate)
    float* g_phi = nullptr;
    int32_t *pick_e = nullptr, *pick_slot = nullptr;
    float* pick_w = nullptr;
    int32_t* cnt_cta = nullptr;
    int32_t* tbl_tok = nullptr;
    float* tbl_w = nullptr;
    int32_t* slot_counts = nullptr;
    uint32_t* blk_ready = nullptr;
    unsigned long long* trace = nullptr;
    unsigned long long* chunklog = nullptr;
    unsigned long long* delay_ns = nullptr;
    DevEvent* ev = nullptr;
    int32_t* full_list = nullptr;
    float* full_z = nullptr;
    float* epart = nullptr;
    uint32_t ev_cap = 0;
    int ctas = 0;
    uint8_t* ctrl = nullptr;        // bar | heads | err | stats | sent | g0done
    float* in_buf = nullptr;
    float* out_buf = nullptr;
    float* in_buf2 = nullptr;       // second shard buffers of the streaming API (allocated on first use)
    float* out_buf2 = nullptr;
    size_t weight_bytes = 0;
    std::vector<uint8_t*> peer;     // heap of every rank as addressable from this rank's device
    std::vector<bool> peer_opened;  // opened through IPC (must be closed)
};

struct Group {
    int dev = 0;
    std::vector<int> members;       // indices into handle->ranks
    RankCtx* d_ctx = nullptr;
    uint32_t* d_abort = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // streaming API (fdmoe_forward_stream): copy-in / copy-out streams and per-slot events
    cudaStream_t s_in = nullptr, s_out = nullptr;
    cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_comp[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
    int ctas_per_rank = 0;
    int smem = 0;
    int num_sms = 0;
    unsigned long long launch_seq = 0;
    uint32_t zero_seq = 0;          // fused-combine launches since the control block was cleared
    cudaStream_t last_stream = nullptr;   // stream of the previous launch (cross-stream ordering)
};

// control block offsets
constexpr size_t kCtrlBar = 0, kCtrlGemm = 8, kCtrlComb = 12, kCtrlErr = 16, kCtrlStats = 32, kCtrlSent = 96;

}  // namespace

struct fdmoe_handle {
    fdmoe_config cfg{};
    Dims dm{};
    int first_rank = 0, n_local = 0;
    std::vector<RankRes> ranks;
    std::vector<Group> groups;
    uint32_t epoch = 0;
    bool weights_set = false;
    bool peers_ready = false;
    bool in_flight = false;
};

namespace {

size_t ctrl_bytes(const Dims& d) { return align_up(kCtrlSent + 4 * d.E + 4 * d.El * d.MT + 64, 256); }
size_t ctrl_ev_ctr(const Dims& d) { return kCtrlSent + 4 * d.E + 4 * d.El * d.MT; }

// Event-log capacity: every task, tile put, packet signal, per-CTA record and barrier of one launch.
uint32_t event_capacity(const Dims& d, int ctas) {
    const int64_t tiles = d.El * d.MT;
    const int64_t n = tiles * (d.NB0 + d.NB1) + tiles * d.NB1 * std::min<int64_t>(d.P, kMaxSrcPerTile) +
                      (d.S + kCombineTok - 1) / kCombineTok + d.E + 2 * (int64_t)ctas + 4 * kGroupBarriers + 1024;
    return (uint32_t)std::min<int64_t>(n, 1 << 26);
}

fdmoe_status alloc_rank(fdmoe_handle* h, RankRes& r, int ctas_per_rank) {
    const Dims& d = h->dm;
    CK(cudaSetDevice(r.dev));
    // ---- symmetric heap (peers write into it)
    HeapLayout hl{};
    size_t off = 0;
    const size_t xplane = align_up((size_t)d.rows_x * d.H * d.esz);
    for (int par = 0; par < 2; ++par)
        for (int pl = 0; pl < 2; ++pl) {
            if (pl < d.planes) { hl.x[par][pl] = off; off += xplane; }
            else hl.x[par][pl] = hl.x[par][0];
        }
    hl.yc = off; off += align_up((size_t)d.E * d.C * d.H * 4);
    for (int par = 0; par < 2; ++par) { hl.dflag[par] = off; off += align_up((size_t)d.El * d.P * 8); }
    for (int par = 0; par < 2; ++par) { hl.cflag[par] = off; off += align_up((size_t)d.E * d.RBF * d.NB1 * 8); }
    hl.gbar = off; off += align_up((size_t)kGroupBarriers * d.P * 8);
    hl.bytes = off;
    r.hl = hl;
    r.heap_bytes = off;
    CK(cudaMalloc(&r.heap, off));
    CK(cudaMemset(r.heap + hl.dflag[0], 0, hl.bytes - hl.dflag[0]));   // all signal words = epoch 0

    // ---- private scratch
    std::vector<std::pair<void**, size_t>> parts;
    const size_t c1plane = (size_t)d.rows_x * d.D * d.esz;
    // expert weights: ONE plane (FP32, split into tf32 hi/lo on chip; or bf16), K-major
    const size_t w1plane = (size_t)d.rows_w1 * d.H * d.esz;
    const size_t w2plane = (size_t)d.rows_w2 * d.D * d.esz;
    for (int pl = 0; pl < d.planes; ++pl) parts.push_back({&r.c1[pl], c1plane});
    parts.push_back({&r.w1[0], w1plane});
    parts.push_back({&r.w2[0], w2plane});
    parts.push_back({(void**)&r.b1, (size_t)d.El * d.D * 4});
    parts.push_back({(void**)&r.b2, (size_t)d.El * d.H * 4});
    parts.push_back({(void**)&r.wg, (size_t)d.H * d.E * 4});
    parts.push_back({(void**)&r.wg_norm, (size_t)d.E * 4});
    parts.push_back({(void**)&r.wgT, (size_t)d.E * d.H * 4});
    parts.push_back({(void**)&r.wg_split, (size_t)2 * d.gate_nblk * d.gate_n * d.H * 4});
    parts.push_back({(void**)&r.gate_na, (size_t)d.S * 8});
    parts.push_back({(void**)&r.gate_sab, (size_t)d.S * 4});
    parts.push_back({(void**)&r.g_phi, (size_t)d.S * d.E * 4});
    parts.push_back({(void**)&r.pick_e, (size_t)d.S * d.k * 4});
    parts.push_back({(void**)&r.pick_slot, (size_t)d.S * d.k * 4});
    parts.push_back({(void**)&r.pick_w, (size_t)d.S * d.k * 4});
    parts.push_back({(void**)&r.cnt_cta, (size_t)ctas_per_rank * d.E * 4});
    parts.push_back({(void**)&r.tbl_tok, (size_t)d.E * d.C * 4});
    parts.push_back({(void**)&r.tbl_w, (size_t)d.E * d.C * 4});
    parts.push_back({(void**)&r.slot_counts, (size_t)d.E * 4});
    parts.push_back({(void**)&r.trace, (size_t)ctas_per_rank * kTracePts * 8});
    parts.push_back({(void**)&r.chunklog, (size_t)kChunkLog * 4 * 8});
    parts.push_back({(void**)&r.delay_ns, (size_t)d.E * 8});
    r.ev_cap = event_capacity(d, ctas_per_rank);
    parts.push_back({(void**)&r.ev, (size_t)r.ev_cap * sizeof(DevEvent)});
    parts.push_back({(void**)&r.blk_ready, (size_t)(d.S + kGateTok - 1) / kGateTok * 4});
    parts.push_back({(void**)&r.full_list, (size_t)kFullCap * 4});
    parts.push_back({(void**)&r.full_z, (size_t)kFullCap * d.E * 4});
    parts.push_back({(void**)&r.epart, (size_t)ctas_per_rank * kNT * kBF * 4});
    parts.push_back({(void**)&r.ctrl, ctrl_bytes(d)});
    parts.push_back({(void**)&r.in_buf, (size_t)d.S * d.H * 4});
    parts.push_back({(void**)&r.out_buf, (size_t)d.S * d.H * 4});
    size_t total = 0;
    for (auto& p : parts) total += align_up(p.second);
    CK(cudaMalloc(&r.scratch, total));
    r.scratch_bytes = total;
    size_t o = 0;
    for (auto& p : parts) { *p.first = r.scratch + o; o += align_up(p.second); }
    r.ctas = ctas_per_rank;
    CK(cudaMemset(r.trace, 0, (size_t)ctas_per_rank * kTracePts * 8));
    CK(cudaMemset(r.ctrl, 0, ctrl_bytes(d)));
    CK(cudaMemset(r.delay_ns, 0, (size_t)d.E * 8));
    CK(cudaMemset(r.blk_ready, 0, (size_t)(d.S + kGateTok - 1) / kGateTok * 4));
    CK(cudaMemset(r.w1[0], 0, w1plane));   // padding rows stay finite
    CK(cudaMemset(r.w2[0], 0, w2plane));
    r.weight_bytes = w1plane + w2plane;
    return FDMOE_OK;
}

fdmoe_status build_ctx(fdmoe_handle* h) {
    const Dims& d = h->dm;
    for (auto& g : h->groups) {
        std::vector<RankCtx> host(g.members.size());
        for (size_t i = 0; i < g.members.size(); ++i) {
            RankRes& r = h->ranks[g.members[i]];
            RankCtx& c = host[i];
            std::memset(&c, 0, sizeof(c));
            fdmoe_status st;
            for (int par = 0; par < 2; ++par)
                for (int pl = 0; pl < 2; ++pl)
                    if ((st = make_tmap(&c.tm_x[par][pl], r.heap + r.hl.x[par][pl], d.rows_x, d.H, d.esz, kBM)))
                        return st;
            for (int pl = 0; pl < 2; ++pl) {
                const int p = pl < d.planes ? pl : 0;
                if ((st = make_tmap(&c.tm_c1[pl], r.c1[p], d.rows_x, d.D, d.esz, kBM))) return st;
            }
            if ((st = make_tmap(&c.tm_w1, r.w1[0], d.rows_w1, d.H, d.esz, kBF))) return st;
            if ((st = make_tmap(&c.tm_w2, r.w2[0], d.rows_w2, d.D, d.esz, kBF))) return st;
            for (int pl = 0; pl < 2; ++pl)
                if ((st = make_tmap(&c.tm_wg[pl], r.wg_split + (size_t)pl * d.gate_nblk * d.gate_n * d.H,
                                    d.gate_nblk * d.gate_n, d.H, 4, (int)d.gate_n)))
                    return st;
            for (int q = 0; q < d.P; ++q) c.peer_heap[q] = r.peer[q];
            c.hl = r.hl;
            c.c1[0] = r.c1[0];
            c.c1[1] = r.c1[d.planes - 1];
            c.b1 = r.b1; c.b2 = r.b2; c.wg = r.wg; c.wg_norm = r.wg_norm; c.wgT = r.wgT;
            c.gate_na = r.gate_na;
            c.gate_sab = r.gate_sab;
            c.g_phi = r.g_phi; c.pick_e = r.pick_e; c.pick_slot = r.pick_slot; c.pick_w = r.pick_w;
            c.cnt_cta = r.cnt_cta; c.tbl_tok = r.tbl_tok; c.tbl_w = r.tbl_w; c.slot_counts = r.slot_counts;
            c.blk_ready = r.blk_ready;
            c.trace = r.trace;
#ifdef FDMOE_DEV
            c.chunklog = getenv("FDMOE_CHUNKLOG") ? r.chunklog : nullptr;
#else
            c.chunklog = nullptr;
#endif
            c.delay_ns = r.delay_ns;
            c.ev = r.ev;
            c.ev_cap = r.ev_cap;
            c.ev_ctr = reinterpret_cast<uint32_t*>(r.ctrl + ctrl_ev_ctr(d));
            c.zero_ctr = reinterpret_cast<uint32_t*>(r.ctrl + ctrl_ev_ctr(d) + 4);
            c.full_ctr = reinterpret_cast<uint32_t*>(r.ctrl + ctrl_ev_ctr(d) + 8);   // [3], inside the 64 spare bytes
            c.full_list = r.full_list;
            c.full_z = r.full_z;
            c.epart = r.epart;
            c.bar = reinterpret_cast<unsigned long long*>(r.ctrl + kCtrlBar);
            c.gemm_head = reinterpret_cast<uint32_t*>(r.ctrl + kCtrlGemm);
            c.comb_head = reinterpret_cast<uint32_t*>(r.ctrl + kCtrlComb);
            c.err = reinterpret_cast<uint32_t*>(r.ctrl + kCtrlErr);
            c.stats = reinterpret_cast<unsigned long long*>(r.ctrl + kCtrlStats);
            c.sent = reinterpret_cast<uint32_t*>(r.ctrl + kCtrlSent);
            c.g0done = reinterpret_cast<uint32_t*>(r.ctrl + kCtrlSent + 4 * d.E);
            c.rank = r.rank;
        }
        CK(cudaSetDevice(g.dev));
        CK(cudaMemcpy(g.d_ctx, host.data(), sizeof(RankCtx) * host.size(), cudaMemcpyHostToDevice));
    }
    return FDMOE_OK;
}

fdmoe_status check_errors(fdmoe_handle* h) {
    for (auto& g : h->groups) {
        CK(cudaSetDevice(g.dev));
        CK(cudaEventSynchronize(g.ev1));          // end of the launch, on whatever stream it ran
        CK(cudaStreamSynchronize(g.stream));      // host-path copies queued behind it
    }
    fdmoe_status worst = FDMOE_OK;
    std::string msg;
    for (auto& g : h->groups) {
        CK(cudaSetDevice(g.dev));
        for (int idx : g.members) {
            RankRes& r = h->ranks[idx];
            uint32_t err[4];
            CK(cudaMemcpy(err, r.ctrl + kCtrlErr, 16, cudaMemcpyDeviceToHost));
            if (err[0] != kErrNone) {
                const char* what = err[0] == kErrTimeout ? "device watchdog: no progress within the deadlock budget"
                                   : err[0] == kErrProtocol ? "protocol error: packet over-subscribed"
                                                            : "accounting mismatch";
                msg += "rank " + std::to_string(r.rank) + ": " + what + " (site " + std::to_string(err[1]) +
                       ", " + std::to_string(err[2]) + ", " + std::to_string(err[3]) + "); ";
                worst = err[0] == kErrProtocol ? FDMOE_ERR_PROTOCOL : FDMOE_ERR_RUNTIME;
            }
        }
    }
    if (worst != FDMOE_OK) {
        // recover: clear error words, abort flags and barrier generations
        for (auto& g : h->groups) {
            cudaSetDevice(g.dev);
            cudaMemset(g.d_abort, 0, 4);
            for (int idx : g.members) {
                cudaMemset(h->ranks[idx].ctrl, 0, ctrl_bytes(h->dm));
            }
            g.launch_seq = 0;
            g.zero_seq = 0;
        }
        return fail(worst, msg);
    }
    return FDMOE_OK;
}

}  // namespace

extern "C" {

fdmoe_status fdmoe_create(const fdmoe_config* cfg, const int32_t* device_ids, int32_t n_local, int32_t first_rank,
                          fdmoe_handle** out) {
    if (!out) return fail(FDMOE_ERR_CONFIG, "null out");
    *out = nullptr;
    fdmoe_status st = fdmoe_config_validate(cfg, 1);
    if (st) return st;
    if (n_local < 1 || first_rank < 0 || first_rank + n_local > cfg->devices)
        return fail(FDMOE_ERR_CONFIG, "local rank range outside [0, devices)");
    auto* h = new fdmoe_handle();
    h->cfg = *cfg;
    h->dm = make_dims(*cfg);
    h->first_rank = first_rank;
    h->n_local = n_local;
    h->ranks.resize(n_local);
    std::map<int, int> dev_group;
    for (int i = 0; i < n_local; ++i) {
        h->ranks[i].rank = first_rank + i;
        h->ranks[i].dev = device_ids ? device_ids[i] : 0;
        auto it = dev_group.find(h->ranks[i].dev);
        if (it == dev_group.end()) {
            dev_group[h->ranks[i].dev] = (int)h->groups.size();
            Group g;
            g.dev = h->ranks[i].dev;
            h->groups.push_back(g);
            it = dev_group.find(h->ranks[i].dev);
        }
        h->groups[it->second].members.push_back(i);
    }
    auto cleanup = [&](fdmoe_status s) { fdmoe_destroy(h); return s; };
    for (auto& g : h->groups) {
        if ((int)g.members.size() > kMaxLocalRanks) return cleanup(fail(FDMOE_ERR_UNSUPPORTED, "more than 8 ranks on one GPU"));
        if (cudaSetDevice(g.dev) != cudaSuccess) return cleanup(fail(FDMOE_ERR_CUDA, "cudaSetDevice failed (no GPU?)"));
        cudaDeviceProp prop;
        if (cudaGetDeviceProperties(&prop, g.dev) != cudaSuccess) return cleanup(fail(FDMOE_ERR_CUDA, "no device"));
        if (prop.major != 10) return cleanup(fail(FDMOE_ERR_UNSUPPORTED, "libfdmoe targets sm_100a (B200)"));
        g.num_sms = prop.multiProcessorCount;
        g.smem = layer_smem_bytes(cfg->precision);
        const int per_sm = layer_max_blocks_per_sm(cfg->precision, g.smem);
        if (per_sm < 1) return cleanup(fail(FDMOE_ERR_CUDA, "layer kernel does not fit on an SM"));
        g.ctas_per_rank = per_sm * g.num_sms / (int)g.members.size();
        if (g.ctas_per_rank < 1) return cleanup(fail(FDMOE_ERR_UNSUPPORTED, "too many ranks for one GPU"));
        if (cudaStreamCreateWithFlags(&g.stream, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreate(&g.ev0) != cudaSuccess || cudaEventCreate(&g.ev1) != cudaSuccess ||
            cudaMalloc(&g.d_ctx, sizeof(RankCtx) * g.members.size()) != cudaSuccess ||
            cudaMalloc(&g.d_abort, 4) != cudaSuccess || cudaMemset(g.d_abort, 0, 4) != cudaSuccess)
            return cleanup(fail(FDMOE_ERR_CUDA, "stream/event/context allocation failed"));
        for (int idx : g.members)
            if ((st = alloc_rank(h, h->ranks[idx], g.ctas_per_rank))) return cleanup(st);
    }
    // same-process peers: direct pointers (enable peer access across distinct devices)
    for (auto& a : h->groups)
        for (auto& b : h->groups)
            if (a.dev != b.dev) {
                cudaSetDevice(a.dev);
                int can = 0;
                cudaDeviceCanAccessPeer(&can, a.dev, b.dev);
                if (!can) return cleanup(fail(FDMOE_ERR_UNSUPPORTED, "devices lack peer access"));
                cudaError_t e = cudaDeviceEnablePeerAccess(b.dev, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                    return cleanup(fail(FDMOE_ERR_CUDA, "cudaDeviceEnablePeerAccess failed"));
                cudaGetLastError();
            }
    for (auto& r : h->ranks) {
        r.peer.assign(cfg->devices, nullptr);
        r.peer_opened.assign(cfg->devices, false);
        for (auto& o : h->ranks) r.peer[o.rank] = o.heap;
    }
    h->peers_ready = (n_local == cfg->devices);
    if (h->peers_ready && (st = build_ctx(h))) return cleanup(st);
    *out = h;
    return FDMOE_OK;
}

fdmoe_status fdmoe_destroy(fdmoe_handle* h) {
    if (!h) return FDMOE_OK;
    for (auto& r : h->ranks) {
        cudaSetDevice(r.dev);
        for (size_t q = 0; q < r.peer_opened.size(); ++q)
            if (r.peer_opened[q]) cudaIpcCloseMemHandle(r.peer[q]);
        if (r.heap) cudaFree(r.heap);
        if (r.scratch) cudaFree(r.scratch);
        if (r.in_buf2) cudaFree(r.in_buf2);
        if (r.out_buf2) cudaFree(r.out_buf2);
    }
    for (auto& g : h->groups) {
        cudaSetDevice(g.dev);
        if (g.stream) cudaStreamDestroy(g.stream);
        if (g.ev0) cudaEventDestroy(g.ev0);
        if (g.ev1) cudaEventDestroy(g.ev1);
        if (g.s_in) cudaStreamDestroy(g.s_in);
        if (g.s_out) cudaStreamDestroy(g.s_out);
        for (int i = 0; i < 2; ++i) {
            if (g.ev_in[i]) cudaEventDestroy(g.ev_in[i]);
            if (g.ev_comp[i]) cudaEventDestroy(g.ev_comp[i]);
            if (g.ev_out[i]) cudaEventDestroy(g.ev_out[i]);
        }
        if (g.d_ctx) cudaFree(g.d_ctx);
        if (g.d_abort) cudaFree(g.d_abort);
    }
    delete h;
    return FDMOE_OK;
}

size_t fdmoe_ipc_size(void) { return sizeof(cudaIpcMemHandle_t) + 8; }

fdmoe_status fdmoe_export_heap(fdmoe_handle* h, void* blob) {
    if (!h || h->n_local != 1) return fail(FDMOE_ERR_CONFIG, "export_heap needs a single-rank handle");
    RankRes& r = h->ranks[0];
    CK(cudaSetDevice(r.dev));
    cudaIpcMemHandle_t mh;
    CK(cudaIpcGetMemHandle(&mh, r.heap));
    std::memcpy(blob, &mh, sizeof(mh));
    const uint64_t bytes = r.heap_bytes;
    std::memcpy(static_cast<uint8_t*>(blob) + sizeof(mh), &bytes, 8);
    return FDMOE_OK;
}

fdmoe_status fdmoe_import_peers(fdmoe_handle* h, const void* blobs, int32_t world) {
    if (!h || h->n_local != 1) return fail(FDMOE_ERR_CONFIG, "import_peers needs a single-rank handle");
    if (world != h->cfg.devices) return fail(FDMOE_ERR_CONFIG, "world size != devices");
    RankRes& r = h->ranks[0];
    CK(cudaSetDevice(r.dev));
    const size_t sz = fdmoe_ipc_size();
    for (int q = 0; q < world; ++q) {
        if (q == r.rank) continue;
        cudaIpcMemHandle_t mh;
        std::memcpy(&mh, static_cast<const uint8_t*>(blobs) + q * sz, sizeof(mh));
        uint64_t bytes;
        std::memcpy(&bytes, static_cast<const uint8_t*>(blobs) + q * sz + sizeof(mh), 8);
        if (bytes != r.heap_bytes) return fail(FDMOE_ERR_CONFIG, "peer heap layout differs (config mismatch)");
        void* p = nullptr;
        CK(cudaIpcOpenMemHandle(&p, mh, cudaIpcMemLazyEnablePeerAccess));
        r.peer[q] = static_cast<uint8_t*>(p);
        r.peer_opened[q] = true;
    }
    h->peers_ready = true;
    return build_ctx(h);
}

fdmoe_status fdmoe_set_weights(fdmoe_handle* h, const float* wg, const float* w1, const float* b1, const float* w2,
                               const float* b2, int32_t where) {
    if (!h) return fail(FDMOE_ERR_CONFIG, "null handle");
    if (!wg || !w1 || !b1 || !w2 || !b2) return fail(FDMOE_ERR_CONFIG, "null weight pointer");
    const Dims& d = h->dm;
    const cudaMemcpyKind kind = where == FDMOE_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    // |Wg[:, e]|_2 for the certified gate, computed in double and rounded up to float
    std::vector<float> wn(d.E), wt((size_t)d.E * d.H), wsplit;
    {
        std::vector<float> hw;
        const float* src = wg;
        if (where != FDMOE_HOST) {
            hw.resize((size_t)d.H * d.E);
            CK(cudaMemcpy(hw.data(), wg, hw.size() * 4, cudaMemcpyDeviceToHost));
            src = hw.data();
        }
        std::vector<double> ss(d.E, 0.0);
        for (int64_t x = 0; x < d.H; ++x)
            for (int64_t e = 0; e < d.E; ++e) {
                ss[e] += (double)src[x * d.E + e] * src[x * d.E + e];
                wt[e * d.H + x] = src[x * d.E + e];
            }
        // tensor-core gate operand: Wg^T split into a tf32 hi plane (round to nearest, as tf32_hi on the
        // device) and the exact remainder plane; expert rows past E are zero
        const size_t plane = (size_t)d.gate_nblk * d.gate_n * d.H;
        wsplit.assign(2 * plane, 0.0f);
        for (int64_t e = 0; e < d.E; ++e)
            for (int64_t x = 0; x < d.H; ++x) {
                const float v = wt[e * d.H + x];
                uint32_t u;
                std::memcpy(&u, &v, 4);
                u = (u + 0x1000u) & 0xFFFFE000u;
                float hi;
                std::memcpy(&hi, &u, 4);
                wsplit[e * d.H + x] = hi;
                wsplit[plane + e * d.H + x] = v - hi;
            }
        for (int64_t e = 0; e < d.E; ++e) {
            const double n = std::sqrt(ss[e]) * (1.0 + 1e-12);
            float f = (float)n;
            if ((double)f < n) f = std::nextafter(f, INFINITY);
            wn[e] = f;
        }
    }
    for (auto& r : h->ranks) {
        CK(cudaSetDevice(r.dev));
        const int64_t e0 = (int64_t)r.rank * d.El;   // config.hpp:66 uniform placement
        const size_t wbytes = (size_t)d.El * d.H * d.D * 4;
        float* tmp = nullptr;
        CK(cudaMalloc(&tmp, wbytes));
        CK(cudaMemcpy(tmp, w1 + e0 * d.H * d.D, wbytes, kind));
        CK(launch_prep_transpose(tmp, (int)d.El, (int)d.H, (int)d.D, r.w1[0], d.prec, 0));
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(tmp, w2 + e0 * d.D * d.H, wbytes, kind));
        CK(launch_prep_transpose(tmp, (int)d.El, (int)d.D, (int)d.H, r.w2[0], d.prec, 0));
        CK(cudaDeviceSynchronize());
        CK(cudaFree(tmp));
        CK(cudaMemcpy(r.b1, b1 + e0 * d.D, (size_t)d.El * d.D * 4, kind));
        CK(cudaMemcpy(r.b2, b2 + e0 * d.H, (size_t)d.El * d.H * 4, kind));
        CK(cudaMemcpy(r.wg, wg, (size_t)d.H * d.E * 4, kind));
        CK(cudaMemcpy(r.wg_norm, wn.data(), (size_t)d.E * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(r.wgT, wt.data(), wt.size() * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(r.wg_split, wsplit.data(), wsplit.size() * 4, cudaMemcpyHostToDevice));
    }
    h->weights_set = true;
    return FDMOE_OK;
}

static fdmoe_status launch_all(fdmoe_handle* h, const float* const* in_dev, float* const* out_dev,
                               void* const* streams, const fdmoe_options* opts) {
    const Dims& d = h->dm;
    if (!h->weights_set) return fail(FDMOE_ERR_CONFIG, "weights not set");
    if (!h->peers_ready) return fail(FDMOE_ERR_CONFIG, "peers not attached (fdmoe_import_peers)");
    const int64_t budget_ms = (opts && opts->deadlock_budget_ms > 0) ? opts->deadlock_budget_ms : 5000;
    const bool sequential = opts && opts->sequential;
    const bool trace_events = opts && opts->trace_events;
    int straggler_rank = -1;
    std::vector<uint64_t> delay;
    if (opts && opts->straggler_kind != FDMOE_STRAGGLER_NONE) {
        if (opts->straggler_kind < 0 || opts->straggler_kind > FDMOE_STRAGGLER_LOGNORMAL)
            return fail(FDMOE_ERR_CONFIG, "unknown straggler kind");
        if (opts->straggler_device < 0 || opts->straggler_device >= d.P)
            return fail(FDMOE_ERR_CONFIG, "straggler device outside [0, devices)");
        straggler_rank = opts->straggler_device;
        delay.resize(d.E);
        fdmoe_status ds = fdmoe_straggler_delays(opts, d.P, d.El, delay.data());
        if (ds) return ds;
    }
    // The kernel reads the input shards while other CTAs already write outputs (the fused combine zeroes
    // and accumulates output rows during the FFN; the separate combine writes them while late packets may
    // still be in flight from peers): in-place forwards are not supported.
    for (auto& g : h->groups)
        for (int idx : g.members) {
            const uint8_t* a = reinterpret_cast<const uint8_t*>(in_dev[idx]);
            const uint8_t* o = reinterpret_cast<const uint8_t*>(out_dev[idx]);
            const size_t bytes = (size_t)d.S * d.H * 4;
            if (!a || !o) return fail(FDMOE_ERR_CONFIG, "null shard pointer");
            if (a < o + bytes && o < a + bytes) return fail(FDMOE_ERR_CONFIG, "input and output shards overlap");
        }
    h->epoch += 1;
    for (auto& g : h->groups) {
        LaunchParams p{};
        p.ranks = g.d_ctx;
        for (size_t i = 0; i < g.members.size(); ++i) {
            p.in[i] = in_dev[g.members[i]];
            p.out[i] = out_dev[g.members[i]];
        }
        p.S = (int)d.S; p.H = (int)d.H; p.D = (int)d.D; p.E = (int)d.E; p.El = (int)d.El; p.P = (int)d.P;
        p.k = (int)d.k; p.C = (int)d.C; p.Cp = (int)d.Cp; p.RP = (int)d.RP; p.MT = (int)d.MT; p.RBF = (int)d.RBF;
        p.NB0 = (int)d.NB0; p.NB1 = (int)d.NB1;
        p.act = h->cfg.activation;
        p.prec = h->cfg.precision;
        p.ctas_per_rank = g.ctas_per_rank;
        p.nranks = (int)g.members.size();
        p.epoch = h->epoch;
        p.launch_seq = g.launch_seq;
        p.budget_ns = (unsigned long long)budget_ms * 1000000ull;
        p.abort_flag = g.d_abort;
        p.sequential = sequential ? 1 : 0;
        p.trace_events = trace_events ? 1 : 0;
        p.straggler_rank = straggler_rank;
        p.fused_combine = (d.k <= 2 && !sequential && (int64_t)g.members.size() == d.P && h->n_local == d.P) ? 1 : 0;
        if (p.fused_combine) p.zero_target = (++g.zero_seq) * (uint32_t)g.ctas_per_rank;
        p.exact_gate = (opts && opts->exact_gate) ? 1 : 0;
        {   // certified-gate bound coefficients (fdmoe_kernel.cu, phase 1)
            const double u = std::ldexp(1.0, -24), n1 = (double)d.H + 1.0;
            p.gate_u = (float)(u * 1.001);
            p.gate_k1 = (float)((66.0 + 2.0 * (double)d.H * (n1 * u / (1.0 - n1 * u))) * 1.001);
        }
        {   // tensor-core gate (fdmoe_kernel.cu phase 1a): 3xTF32 logits folded per 64-K chunk, certified with
            //   |z~ - z_ref| <= u' (64 Sab + k1_tc |a| |w_e|)
            // The reference chain (gate.hpp:77-81): u sum_i |s_i| + u sum |a_x w_x|, with |s_i| <= |P_J-1| + S_J inside
            // chunk J (P: prefix at chunk ends, S_J = sum over the chunk of |a_x w_x|), so <= u (64 Sab + 65 |a||w|)
            // (+ 2H gamma_{H+1} |a||w| for computed-vs-exact partials, + 1 for Sab's own error). Ours: tf32 products
            // 2^-19 = 32u; per 64-K chunk 8 main MMAs, each < 3 ulp of the chunk's magnitude (products truncated 2
            // bits below the accumulator's ulp + final round toward zero: tools/dev/acc_guard.py) -> 48u sum S_J;
            // <= 2H/64 register folds (u each); the 2^-9-scaled correction accumulator (2H/8 MMAs) -> 6u; the
            // corrections' fold u. All terms times |a||w_e| >= sum |a_x||w_xe|.
            bool aligned = true;
            for (size_t i = 0; i < g.members.size(); ++i) aligned &= ((uintptr_t)p.in[i] & 15u) == 0;
            p.gate_tc = (!p.exact_gate && aligned) ? 1 : 0;
            p.gate_n = (int)d.gate_n;
            p.gate_nblk = (int)d.gate_nblk;
            const double u = std::ldexp(1.0, -24), H = (double)d.H, n1 = H + 1.0;
            const double chunks = std::ceil(H / 64.0);
            p.gate_k1_tc = (float)((65.0 + 2.0 * H * (n1 * u / (1.0 - n1 * u)) + 1.0 + 32.0 + 48.0 + chunks + 6.0 + 1.0 +
                                    8.0) * 1.001);
            if (p.gate_tc)
                for (size_t i = 0; i < g.members.size(); ++i) {
                    fdmoe_status ts = make_tmap(&p.tm_in[i], p.in[i], d.S, d.H, 4, kNT);
                    if (ts) return ts;
                }
        }
#ifdef FDMOE_DEV
        const char* dbg = getenv("FDMOE_DEBUG");   // ablation switches (tools/ablate.py): development library only
        p.debug = dbg ? atoi(dbg) : 0;
        if (p.debug & kDbgSimtGate) p.gate_tc = 0;   // A/B: the SIMT certified gate instead of the tensor-core one
#else
        p.debug = 0;
#endif
        CK(cudaSetDevice(g.dev));
        cudaStream_t s = g.stream;
        if (streams && streams[g.members[0]]) s = static_cast<cudaStream_t>(streams[g.members[0]]);
        // Launches share the control block, heaps and C1 of the handle: a launch on another stream than the
        // previous one is ordered behind it (ev1 = end of the previous launch, whatever stream it ran on;
        // a no-op for back-to-back launches on one stream).
        if (h->in_flight && s != g.last_stream) CK(cudaStreamWaitEvent(s, g.ev1, 0));
        g.last_stream = s;
        for (int idx : g.members) {
            RankRes& r = h->ranks[idx];
            if (trace_events) CK(cudaMemsetAsync(r.ctrl + ctrl_ev_ctr(d), 0, 4, s));
            if (r.rank == straggler_rank)
                CK(cudaMemcpyAsync(r.delay_ns, delay.data(), (size_t)d.E * 8, cudaMemcpyHostToDevice, s));
        }
        CK(cudaEventRecord(g.ev0, s));
        CK(launch_layer(p, g.ctas_per_rank * (int)g.members.size(), g.smem, s));
        CK(cudaEventRecord(g.ev1, s));
        g.launch_seq += sequential ? 3 + 2 * kGroupBarriers : 3;   // rank-barrier generations used
    }
    h->in_flight = true;
    return FDMOE_OK;
}

fdmoe_status fdmoe_forward_async(fdmoe_handle* h, const float* const* in_dev, float* const* out_dev,
                                 void* const* streams, const fdmoe_options* opts) {
    if (!h || !in_dev || !out_dev) return fail(FDMOE_ERR_CONFIG, "null argument");
    return launch_all(h, in_dev, out_dev, streams, opts);
}

fdmoe_status fdmoe_sync(fdmoe_handle* h) {
    if (!h) return fail(FDMOE_ERR_CONFIG, "null handle");
    h->in_flight = false;
    return check_errors(h);
}

fdmoe_status fdmoe_forward(fdmoe_handle* h, const float* const* in_shards, float* const* out_shards, int32_t where,
                           const fdmoe_options* opts, fdmoe_routing* routing, fdmoe_stats* stats) {
    if (!h || !in_shards || !out_shards) return fail(FDMOE_ERR_CONFIG, "null argument");
    const Dims& d = h->dm;
    const size_t shard_bytes = (size_t)d.S * d.H * 4;
    std::vector<const float*> in(h->n_local);
    std::vector<float*> out(h->n_local);
    std::vector<unsigned long long> stat0(h->n_local * 8, 0);
    for (int i = 0; i < h->n_local; ++i) {
        RankRes& r = h->ranks[i];
        CK(cudaSetDevice(r.dev));
        if (stats) CK(cudaMemcpy(&stat0[i * 8], r.ctrl + kCtrlStats, 64, cudaMemcpyDeviceToHost));
        if (where == FDMOE_HOST) {
            Group* g = nullptr;
            for (auto& gg : h->groups) if (gg.dev == r.dev) g = &gg;
            CK(cudaMemcpyAsync(r.in_buf, in_shards[i], shard_bytes, cudaMemcpyHostToDevice, g->stream));
            in[i] = r.in_buf;
            out[i] = r.out_buf;
        } else {
            in[i] = in_shards[i];
            out[i] = out_shards[i];
        }
    }
    fdmoe_status st = launch_all(h, in.data(), out.data(), nullptr, opts);
    if (st) return st;
    if (where == FDMOE_HOST) {
        for (int i = 0; i < h->n_local; ++i) {
            RankRes& r = h->ranks[i];
            Group* g = nullptr;
            for (auto& gg : h->groups) if (gg.dev == r.dev) g = &gg;
            CK(cudaSetDevice(r.dev));
            CK(cudaMemcpyAsync(out_shards[i], r.out_buf, shard_bytes, cudaMemcpyDeviceToHost, g->stream));
        }
    }
    h->in_flight = false;
    if ((st = check_errors(h))) return st;
    for (int i = 0; i < h->n_local; ++i) {
        RankRes& r = h->ranks[i];
        CK(cudaSetDevice(r.dev));
        if (routing) {
            fdmoe_routing& ro = routing[i];
            const int64_t S = d.S, E = d.E, C = d.C, K = d.k;
            if (ro.g_phi) CK(cudaMemcpy(ro.g_phi, r.g_phi, (size_t)S * E * 4, cudaMemcpyDeviceToHost));
            if (ro.table_token || ro.table_weight) {
                std::vector<int32_t> tt((size_t)E * C);
                CK(cudaMemcpy(tt.data(), r.tbl_tok, tt.size() * 4, cudaMemcpyDeviceToHost));
                if (ro.table_token) for (size_t j = 0; j < tt.size(); ++j) ro.table_token[j] = tt[j];
                if (ro.table_weight) CK(cudaMemcpy(ro.table_weight, r.tbl_w, (size_t)E * C * 4, cudaMemcpyDeviceToHost));
            }
            if (ro.slot_counts) {
                std::vector<int32_t> sc((size_t)E);
                CK(cudaMemcpy(sc.data(), r.slot_counts, sc.size() * 4, cudaMemcpyDeviceToHost));
                for (int64_t e = 0; e < E; ++e) ro.slot_counts[e] = sc[e];
            }
            std::vector<int32_t> pe((size_t)S * K), ps((size_t)S * K);
            std::vector<float> pw((size_t)S * K);
            CK(cudaMemcpy(pe.data(), r.pick_e, pe.size() * 4, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(ps.data(), r.pick_slot, ps.size() * 4, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(pw.data(), r.pick_w, pw.size() * 4, cudaMemcpyDeviceToHost));
            if (ro.picks_expert) std::memcpy(ro.picks_expert, pe.data(), pe.size() * 4);
            if (ro.picks_slot) std::memcpy(ro.picks_slot, ps.data(), ps.size() * 4);
            if (ro.picks_weight) std::memcpy(ro.picks_weight, pw.data(), pw.size() * 4);
            if (ro.dropped || ro.n_dropped) {
                int64_t nd = 0;
                for (int64_t t = 0; t < S; ++t)
                    for (int64_t j = 0; j < K; ++j)
                        if (ps[t * K + j] < 0) {
                            if (ro.dropped) { ro.dropped[2 * nd] = t; ro.dropped[2 * nd + 1] = pe[t * K + j]; }
                            ++nd;
                        }
                if (ro.n_dropped) *ro.n_dropped = nd;
            }
        }
        if (stats) {
            unsigned long long s1[8];
            CK(cudaMemcpy(s1, r.ctrl + kCtrlStats, 64, cudaMemcpyDeviceToHost));
            fdmoe_stats& so = stats[i];
            std::memset(&so, 0, sizeof(so));
            so.gemm0 = (int64_t)(s1[0] - stat0[i * 8 + 0]);
            so.gemm1 = (int64_t)(s1[1] - stat0[i * 8 + 1]);
            so.combine = (int64_t)(s1[2] - stat0[i * 8 + 2]);
            so.executed = so.gemm0 + so.gemm1 + so.combine;
            // device task accounting (fdmoe_kernel.cu gemm_producer): bound self-corrected per resolved row
            // tile, scheduled = non-empty FFN tasks the producers handed to their pipelines; the combine tasks
            // of the separate phase are static (the fused combine has none)
            const int64_t comb_bound = so.combine ? (d.S + kCombineTok - 1) / kCombineTok : 0;
            const int64_t bdelta = (int64_t)(s1[5] - stat0[i * 8 + 5]);
            so.bound_initial = d.El * d.MT * (d.NB0 + d.NB1) + comb_bound;
            so.bound_final = so.bound_initial + bdelta;
            so.scheduled_final = (int64_t)(s1[6] - stat0[i * 8 + 6]) + so.combine;
            so.enqueued = so.scheduled_final;
            so.tiles_resolved = (int64_t)(s1[7] - stat0[i * 8 + 7]);
            so.launches = 1;
            so.gate_exact_tokens = (int64_t)(s1[3] - stat0[i * 8 + 3]);
            so.gate_pair_tokens = (int64_t)(s1[4] - stat0[i * 8 + 4]);
            for (auto& g : h->groups)
                if (g.dev == r.dev) {
                    float ms = 0.0f;
                    cudaEventElapsedTime(&ms, g.ev0, g.ev1);
                    so.kernel_ms = ms;
                }
        }
    }
    return FDMOE_OK;
}

// Serving loop over host batches: batch b's H2D (stream s_in), layer launch (the group stream) and
// D2H (stream s_out) run on three streams with double-buffered device shards, so the PCIe copies of
// batches b-1 and b+1 overlap the launch of batch b (H2D and D2H overlap each other: PCIe is full
// duplex). Still exactly one kernel launch per device per batch.
fdmoe_status fdmoe_forward_stream(fdmoe_handle* h, int32_t n_batches, const float* const* in_batches,
                                  float* const* out_batches, const fdmoe_options* opts) {
    if (!h || !in_batches || !out_batches || n_batches < 1) return fail(FDMOE_ERR_CONFIG, "null argument");
    const Dims& d = h->dm;
    const size_t shard_bytes = (size_t)d.S * d.H * 4;
    for (auto& g : h->groups) {
        CK(cudaSetDevice(g.dev));
        if (!g.s_in) {
            CK(cudaStreamCreateWithFlags(&g.s_in, cudaStreamNonBlocking));
            CK(cudaStreamCreateWithFlags(&g.s_out, cudaStreamNonBlocking));
            for (int i = 0; i < 2; ++i) {
                CK(cudaEventCreateWithFlags(&g.ev_in[i], cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&g.ev_comp[i], cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&g.ev_out[i], cudaEventDisableTiming));
            }
        }
        for (int idx : g.members) {
            RankRes& r = h->ranks[idx];
            if (!r.in_buf2) CK(cudaMalloc(&r.in_buf2, shard_bytes));
            if (!r.out_buf2) CK(cudaMalloc(&r.out_buf2, shard_bytes));
        }
    }
    const int n = h->n_local;
    std::vector<const float*> din(n);
    std::vector<float*> dout(n);
    for (int b = 0; b < n_batches; ++b) {
        const int slot = b & 1;
        for (auto& g : h->groups) {
            CK(cudaSetDevice(g.dev));
            if (b >= 2) CK(cudaStreamWaitEvent(g.s_in, g.ev_comp[slot], 0));   // launch b-2 done with the slot
            for (int idx : g.members) {
                RankRes& r = h->ranks[idx];
                CK(cudaMemcpyAsync(slot ? r.in_buf2 : r.in_buf, in_batches[(size_t)b * n + idx], shard_bytes,
                                   cudaMemcpyHostToDevice, g.s_in));
            }
            CK(cudaEventRecord(g.ev_in[slot], g.s_in));
            CK(cudaStreamWaitEvent(g.stream, g.ev_in[slot], 0));
            if (b >= 2) CK(cudaStreamWaitEvent(g.stream, g.ev_out[slot], 0));   // D2H of b-2 drained the slot
        }
        for (int i = 0; i < n; ++i) {
            din[i] = slot ? h->ranks[i].in_buf2 : h->ranks[i].in_buf;
            dout[i] = slot ? h->ranks[i].out_buf2 : h->ranks[i].out_buf;
        }
        fdmoe_status st = launch_all(h, din.data(), dout.data(), nullptr, opts);
        if (st) return st;
        for (auto& g : h->groups) {
            CK(cudaSetDevice(g.dev));
            CK(cudaEventRecord(g.ev_comp[slot], g.stream));
            CK(cudaStreamWaitEvent(g.s_out, g.ev_comp[slot], 0));
            for (int idx : g.members) {
                RankRes& r = h->ranks[idx];
                CK(cudaMemcpyAsync(out_batches[(size_t)b * n + idx], slot ? r.out_buf2 : r.out_buf, shard_bytes,
                                   cudaMemcpyDeviceToHost, g.s_out));
            }
            CK(cudaEventRecord(g.ev_out[slot], g.s_out));
        }
    }
    for (auto& g : h->groups) {
        CK(cudaSetDevice(g.dev));
        CK(cudaStreamSynchronize(g.s_out));
    }
    h->in_flight = false;
    return check_errors(h);
}

fdmoe_status fdmoe_get_info(fdmoe_handle* h, fdmoe_info* info) {
    if (!h || !info) return fail(FDMOE_ERR_CONFIG, "null argument");
    std::memset(info, 0, sizeof(*info));
    info->capacity = h->dm.C;
    info->packet_rows = h->dm.Cp;
    info->heap_bytes = (int64_t)h->ranks[0].heap_bytes;
    info->scratch_bytes = (int64_t)h->ranks[0].scratch_bytes;
    info->weight_bytes = (int64_t)h->ranks[0].weight_bytes;
    info->ctas_per_rank = h->groups[0].ctas_per_rank;
    info->smem_bytes = h->groups[0].smem;
    info->num_sms = h->groups[0].num_sms;
    info->ranks_per_launch = (int32_t)h->groups[0].members.size();
    info->fused_combine = (h->dm.k <= 2 && (int64_t)h->groups[0].members.size() == h->dm.P && h->n_local == h->dm.P)
                              ? 1 : 0;
    return FDMOE_OK;
}

fdmoe_status fdmoe_read_trace(fdmoe_handle* h, int32_t local_rank, uint64_t* out, int32_t cap, int32_t* n_ctas) {
    if (!h || local_rank < 0 || local_rank >= h->n_local) return fail(FDMOE_ERR_CONFIG, "bad rank");
    RankRes& r = h->ranks[local_rank];
    CK(cudaSetDevice(r.dev));
    for (auto& g : h->groups) if (g.dev == r.dev) CK(cudaEventSynchronize(g.ev1));
    const int n = std::min(cap / kTracePts, r.ctas);
    CK(cudaMemcpy(out, r.trace, (size_t)n * kTracePts * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemset(r.trace, 0, (size_t)r.ctas * kTracePts * 8));
    if (n_ctas) *n_ctas = r.ctas;
    return FDMOE_OK;
}

fdmoe_status fdmoe_read_events(fdmoe_handle* h, int32_t local_rank, fdmoe_event* out, int64_t cap, int64_t* n,
                               int64_t* dropped) {
    static_assert(sizeof(fdmoe_event) == sizeof(DevEvent), "event record layout");
    if (!h || local_rank < 0 || local_rank >= h->n_local) return fail(FDMOE_ERR_CONFIG, "bad rank");
    RankRes& r = h->ranks[local_rank];
    CK(cudaSetDevice(r.dev));
    for (auto& g : h->groups) if (g.dev == r.dev) CK(cudaEventSynchronize(g.ev1));
    uint32_t cnt = 0;
    CK(cudaMemcpy(&cnt, r.ctrl + ctrl_ev_ctr(h->dm), 4, cudaMemcpyDeviceToHost));
    const int64_t have = std::min<int64_t>(cnt, r.ev_cap);
    const int64_t k = out ? std::min<int64_t>(have, cap) : 0;
    if (k > 0) CK(cudaMemcpy(out, r.ev, (size_t)k * sizeof(DevEvent), cudaMemcpyDeviceToHost));
    if (n) *n = have;
    if (dropped) *dropped = (int64_t)cnt - have;
    return FDMOE_OK;
}

fdmoe_status fdmoe_last_kernel_ms(fdmoe_handle* h, double* ms) {
    if (!h || !ms) return fail(FDMOE_ERR_CONFIG, "null argument");
    double best = 0.0;
    for (auto& g : h->groups) {
        CK(cudaSetDevice(g.dev));
        CK(cudaEventSynchronize(g.ev1));
        float v = 0.0f;
        CK(cudaEventElapsedTime(&v, g.ev0, g.ev1));
        best = std::max(best, (double)v);
    }
    *ms = best;
    return FDMOE_OK;
}

#ifdef FDMOE_DEV   // diagnostics: libfdmoe_dev.so only (include/fdmoe_dev.h)
fdmoe_status fdmoe_read_chunklog(fdmoe_handle* h, uint64_t* out) {
    RankRes& r = h->ranks[0];
    CK(cudaSetDevice(r.dev));
    for (auto& g : h->groups) if (g.dev == r.dev) CK(cudaEventSynchronize(g.ev1));
    CK(cudaMemcpy(out, r.chunklog, (size_t)kChunkLog * 4 * 8, cudaMemcpyDeviceToHost));
    return FDMOE_OK;
}

// ---- diagnostics (tests): device expf and a single-tile tcgen05 GEMM ----------------
fdmoe_status fdmoe_debug_expf(const float* x, float* y, int64_t n) {
    float *dx = nullptr, *dy = nullptr;
    CK(cudaMalloc(&dx, n * 4));
    CK(cudaMalloc(&dy, n * 4));
    CK(cudaMemcpy(dx, x, n * 4, cudaMemcpyHostToDevice));
    CK(launch_debug_expf(dx, dy, n, 0));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(y, dy, n * 4, cudaMemcpyDeviceToHost));
    cudaFree(dx);
    cudaFree(dy);
    return FDMOE_OK;
}

// D[f][t] = sum_k W[f][k] * X[t][k]: W 128 x K (weights, TMEM operand), X 128 x K (tokens, TMA
// operand), host row-major FP32; D 128 x 128. prec as fdmoe_precision.
fdmoe_status fdmoe_debug_gemm(int32_t prec, int32_t K, const float* W, const float* X, float* D) {
    if (K % 64 != 0) return fail(FDMOE_ERR_CONFIG, "K must be a multiple of 64");
    const int esz = prec == FDMOE_FP32 ? 4 : 2;
    auto to_bf16 = [](float f) {
        uint32_t u;
        std::memcpy(&u, &f, 4);
        return (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
    };
    std::vector<uint8_t> wp((size_t)128 * K * esz), xh((size_t)128 * K * esz), xl((size_t)128 * K * esz);
    for (size_t i = 0; i < (size_t)128 * K; ++i) {
        if (prec == FDMOE_FP32) {
            std::memcpy(&wp[i * 4], &W[i], 4);
            uint32_t u;
            std::memcpy(&u, &X[i], 4);
            u = (u + 0x1000u) & 0xFFFFE000u;
            float h;
            std::memcpy(&h, &u, 4);
            const float l = X[i] - h;
            std::memcpy(&xh[i * 4], &h, 4);
            // plane 1 in the FFN's bf16-correction format (fdmoe_kernel.cu kCorrBf16): per row and 32-k group,
            // bf16(x_hi[k]) at byte 2 (k % 32), bf16(x_lo[k]) at byte 64 + 2 (k % 32)
            const size_t row = i / (size_t)K, k = i % (size_t)K, g = row * (size_t)K * 4 + (k / 32) * 128;
            const uint16_t bh = to_bf16(h), bl = to_bf16(l);
            std::memcpy(&xl[g + 2 * (k % 32)], &bh, 2);
            std::memcpy(&xl[g + 64 + 2 * (k % 32)], &bl, 2);
        } else {
            const uint16_t bw = to_bf16(W[i]), bx = to_bf16(X[i]);
            std::memcpy(&wp[i * 2], &bw, 2);
            std::memcpy(&xh[i * 2], &bx, 2);
            std::memcpy(&xl[i * 2], &bx, 2);
        }
    }
    void *dw = nullptr, *dxh = nullptr, *dxl = nullptr;
    CK(cudaMalloc(&dw, wp.size()));
    CK(cudaMalloc(&dxh, xh.size()));
    CK(cudaMalloc(&dxl, xl.size()));
    CK(cudaMemcpy(dw, wp.data(), wp.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dxh, xh.data(), xh.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dxl, xl.data(), xl.size(), cudaMemcpyHostToDevice));
    CUtensorMap tm[3];
    fdmoe_status st;
    if ((st = make_tmap(&tm[0], dxh, 128, K, esz, kNT))) return st;
    if ((st = make_tmap(&tm[1], dxl, 128, K, esz, kNT))) return st;
    if ((st = make_tmap(&tm[2], dw, 128, K, esz, kBF))) return st;
    float* dD = nullptr;
    uint32_t* abort_flag = nullptr;
    CK(cudaMalloc(&dD, 128 * 128 * 4));
    CK(cudaMalloc(&abort_flag, 4));
    CK(cudaMemset(abort_flag, 0, 4));
    CK(launch_debug_gemm(prec, tm, K, dD, abort_flag, 0));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(D, dD, 128 * 128 * 4, cudaMemcpyDeviceToHost));
    cudaFree(dw); cudaFree(dxh); cudaFree(dxl); cudaFree(dD); cudaFree(abort_flag);
    return FDMOE_OK;
}

// Cycles per tcgen05.mma (M=128) issued back to back: kind 0 tf32 / 1 bf16, ts = A from TMEM.
fdmoe_status fdmoe_debug_mma_rate(int32_t kind, int32_t nissuers, int32_t N, int32_t iters, double* cycles_per_mma) {
    unsigned long long* d = nullptr;
    CK(cudaMalloc(&d, 8 * 256));
    CK(cudaMemset(d, 0, 8 * 256));
    CK(launch_debug_mma_rate(kind, N, iters, nissuers, d));
    CK(cudaDeviceSynchronize());
    unsigned long long cs[256];
    CK(cudaMemcpy(cs, d, 8 * 256, cudaMemcpyDeviceToHost));
    unsigned long long c = 0;
    for (int i = 0; i < 256; ++i) c = std::max(c, cs[i]);   // slowest SM
    cudaFree(d);
    *cycles_per_mma = kind >= 16 ? (double)c / ((double)iters * 12.0) : (double)c / ((double)iters * (nissuers & 15));
    return FDMOE_OK;
}

// Latency probe (cycles): [0] issue of n MMAs, [1] issue -> commit completion observed,
// [2] 8 x tcgen05.st.x16 + wait::st, [3] mbarrier wait including a 2000-cycle delayed arrive.
fdmoe_status fdmoe_debug_latency(int32_t n, uint64_t* out4) {
    unsigned long long* d = nullptr;
    CK(cudaMalloc(&d, 32 * 148));
    CK(cudaMemset(d, 0, 32 * 148));
    CK(launch_debug_latency(n, d));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(out4, d, 32, cudaMemcpyDeviceToHost));
    cudaFree(d);
    return FDMOE_OK;
}

#endif  // FDMOE_DEV

}  // extern "C"
