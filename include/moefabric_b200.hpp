// moefabric_b200.hpp — drop-in C++ operator API of the B200 FlashDMoE operator.
//
// Restates the reference's public types and entry point field for field
// (/root/reference/proj/include/moefabric/config.hpp:16-147, gate.hpp:24-151,
//  tiled_blas.hpp:118-121, runtime.hpp:86-117, 802) on top of the C ABI in fdmoe.h,
// so code written against moefabric::forward() switches by changing the include and
// linking libfdmoe.so:
//
//     #include "moefabric_b200.hpp"      // instead of "moefabric/runtime.hpp"
//     moefabric::ForwardResult r = moefabric::forward(cfg, shards, model, opts);
//
// Differences, all documented in INTEGRATION.md: ForwardResult::trace is empty (device
// evidence comes from ncu and fdmoe_read_trace), TaskStats count 128x128 GPU tiles instead of
// bM x bN CPU tasks, MoeConfig gains `precision` (FP32-accurate 3xTF32 by default), and
// ForwardOptions gains `device_ids` (default: every rank on GPU 0 = virtual ranks) and
// `exact_gate` (default false: certified gate — routing bit-exact, G_phi within ~1e-6).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "fdmoe.h"

namespace moefabric {

// config.hpp:16-30
struct ConfigError : std::runtime_error {
    explicit ConfigError(const std::string& w) : std::runtime_error(w) {}
};
struct ProtocolError : std::runtime_error {
    explicit ProtocolError(const std::string& w) : std::runtime_error(w) {}
};
struct RuntimeFault : std::runtime_error {
    explicit RuntimeFault(const std::string& w) : std::runtime_error(w) {}
};
// No reference equivalent: CUDA failure or outside the GPU envelope.
struct DeviceError : std::runtime_error {
    explicit DeviceError(const std::string& w) : std::runtime_error(w) {}
};

namespace detail {
inline void check(fdmoe_status s) {
    if (s == FDMOE_OK) return;
    const std::string m = fdmoe_last_error();
    switch (s) {
        case FDMOE_ERR_CONFIG: throw ConfigError(m);
        case FDMOE_ERR_PROTOCOL: throw ProtocolError(m);
        case FDMOE_ERR_RUNTIME: throw RuntimeFault(m);
        default: throw DeviceError(m);
    }
}
}  // namespace detail

// config.hpp:32-49
enum class Activation : std::uint8_t { relu, gelu, identity };
inline const char* to_string(Activation a) {
    return a == Activation::relu ? "relu" : a == Activation::gelu ? "gelu" : "identity";
}
inline Activation activation_from_string(const std::string& s) {
    if (s == "relu") return Activation::relu;
    if (s == "gelu") return Activation::gelu;
    if (s == "identity") return Activation::identity;
    throw ConfigError("unknown activation: " + s);
}

enum class Precision : std::int32_t { fp32 = FDMOE_FP32, bf16 = FDMOE_BF16 };

// config.hpp:53-87
struct MoeConfig {
    std::int64_t tokens_per_device = 8;
    std::int64_t embed_dim = 8;
    std::int64_t ffn_dim = 8;
    std::int64_t experts_total = 2;
    std::int64_t devices = 1;
    std::int64_t topk = 1;
    double capacity_factor = 1.0;
    std::int64_t tile_rows = 16;
    std::int64_t tile_cols = 8;
    Activation activation = Activation::relu;
    std::uint64_t seed = 0;
    Precision precision = Precision::fp32;   // B200 addition

    std::int64_t local_experts() const { return experts_total / devices; }
    fdmoe_config to_c() const {
        fdmoe_config c{};
        c.tokens_per_device = tokens_per_device; c.embed_dim = embed_dim; c.ffn_dim = ffn_dim;
        c.experts_total = experts_total; c.devices = devices; c.topk = topk;
        c.capacity_factor = capacity_factor; c.tile_rows = tile_rows; c.tile_cols = tile_cols;
        c.activation = static_cast<std::int32_t>(activation);
        c.precision = static_cast<std::int32_t>(precision);
        c.seed = seed;
        return c;
    }
    void validate() const {
        const fdmoe_config c = to_c();
        detail::check(fdmoe_config_validate(&c, 0));
    }
};

inline std::int64_t ceil_div(std::int64_t a, std::int64_t b) { return (a + b - 1) / b; }
inline std::int64_t expert_capacity(const MoeConfig& cfg) {   // config.hpp:94
    const fdmoe_config c = cfg.to_c();
    return fdmoe_expert_capacity(&c);
}
inline std::int64_t padded_capacity(std::int64_t capacity, std::int64_t tile_rows) {   // config.hpp:104
    return fdmoe_padded_capacity(capacity, tile_rows);
}

// config.hpp:109-127
struct TokenMatrix {
    std::int64_t rows = 0;
    std::int64_t cols = 0;
    std::vector<float> data;
    TokenMatrix() = default;
    TokenMatrix(std::int64_t r, std::int64_t c) : rows(r), cols(c), data(static_cast<std::size_t>(r * c), 0.0f) {}
    float& at(std::int64_t r, std::int64_t c) { return data[static_cast<std::size_t>(r * cols + c)]; }
    float at(std::int64_t r, std::int64_t c) const { return data[static_cast<std::size_t>(r * cols + c)]; }
    const float* row(std::int64_t r) const { return data.data() + r * cols; }
    float* row(std::int64_t r) { return data.data() + r * cols; }
    bool all_finite() const {
        for (float v : data)
            if (!std::isfinite(v)) return false;
        return true;
    }
};

// config.hpp:130-147
struct ExpertParams {
    TokenMatrix w1;
    std::vector<float> b1;
    TokenMatrix w2;
    std::vector<float> b2;
};
struct GateWeights {
    TokenMatrix wg;
};
struct ModelWeights {
    GateWeights gate;
    std::vector<ExpertParams> experts;
};

// tiled_blas.hpp:118-121
struct SlotMap {
    std::int64_t token = -1;
    float weight = 0.0f;
};

// gate.hpp:24-37
struct GateOutput {
    TokenMatrix g_phi;
    std::int64_t capacity = 0;
    std::vector<SlotMap> table;
    std::vector<std::int64_t> slot_counts;
    std::vector<std::pair<std::int64_t, std::int64_t>> dropped;
    const SlotMap& slot(std::int64_t e, std::int64_t c) const { return table[static_cast<std::size_t>(e * capacity + c)]; }
    SlotMap& slot(std::int64_t e, std::int64_t c) { return table[static_cast<std::size_t>(e * capacity + c)]; }
};

// gate.hpp:113-151
struct ManifestExpert {
    std::int64_t expert_global = 0;
    std::int64_t count = 0;
    std::vector<std::int64_t> tokens;
};
struct DispatchManifest {
    std::vector<std::vector<ManifestExpert>> per_device;
    std::int64_t total_routed() const {
        std::int64_t n = 0;
        for (const auto& d : per_device)
            for (const auto& m : d) n += m.count;
        return n;
    }
};
inline DispatchManifest dispatch_manifest(const GateOutput& gate, const MoeConfig& cfg) {
    const std::int64_t el = cfg.local_experts();
    DispatchManifest mf;
    mf.per_device.resize(static_cast<std::size_t>(cfg.devices));
    for (std::int64_t d = 0; d < cfg.devices; ++d) {
        auto& dev = mf.per_device[static_cast<std::size_t>(d)];
        dev.resize(static_cast<std::size_t>(el));
        for (std::int64_t le = 0; le < el; ++le) {
            const std::int64_t e = d * el + le;
            ManifestExpert& m = dev[static_cast<std::size_t>(le)];
            m.expert_global = e;
            m.count = gate.slot_counts[static_cast<std::size_t>(e)];
            for (std::int64_t c = 0; c < m.count; ++c) m.tokens.push_back(gate.slot(e, c).token);
        }
    }
    return mf;
}

// runtime.hpp:76-117
enum class ScheduleMode : std::uint8_t { overlapped, sequential };
struct StragglerSpec {
    enum class Kind : std::uint8_t { none, constant, uniform, lognormal };
    Kind kind = Kind::none;
    double a = 0.0, b = 0.0;
    std::int32_t device = 0;
};
struct ForwardOptions {
    std::int32_t processors = 4;
    ScheduleMode mode = ScheduleMode::overlapped;
    StragglerSpec straggler;
    std::int64_t deadlock_budget_ms = 5000;
    std::uint64_t seed = 0;
    std::vector<std::int32_t> device_ids;   // B200 addition: CUDA device per rank (default all 0)
    bool exact_gate = false;                // B200 addition: reference-exact gate logits (fdmoe.h)
    bool trace = true;                      // B200 addition: record the device event log into ForwardResult::trace
};
struct TaskStats {
    std::int64_t gemm0 = 0, gemm1 = 0, combine = 0, enqueued = 0, executed = 0;
    std::int64_t bound_initial = 0, bound_final = 0, scheduled_final = 0, launches = 0;
    std::int64_t total() const { return gemm0 + gemm1 + combine; }
};
// trace.hpp:38-60, recorded on the device (fdmoe_read_events); t0/t1 are ns since the earliest
// event of the launch (%globaltimer), `worker` is the CTA ("cta<N>").
struct TraceEvent {
    std::uint64_t t0 = 0, t1 = 0;
    std::int32_t device = -1;
    char worker[12] = {0};
    const char* event = "";
    const char* task_type = nullptr;  // "gemm0" | "gemm1" | "combine"
    std::int32_t src = -1, expert = -1, rb = -1, cb = -1;
    std::int64_t value = -1;
    std::int32_t peer = -1;
    bool has_task() const { return task_type != nullptr; }
};
namespace detail {
inline const char* event_name(std::int32_t k) {
    static const char* names[] = {"spawn", "gate_done", "dispatch_put", "exec", "tile_put", "barrier_enter",
                                  "barrier_exit"};
    return (k >= 0 && k < 7) ? names[k] : "unknown";
}
inline const char* task_name(std::int32_t t) {
    return t == 1 ? "gemm0" : t == 2 ? "gemm1" : t == 3 ? "combine" : nullptr;
}
}  // namespace detail
struct ForwardResult {
    std::vector<TokenMatrix> outputs;
    std::vector<GateOutput> gates;
    std::vector<DispatchManifest> manifests;
    std::vector<TraceEvent> trace;
    std::vector<std::uint64_t> bytes;
    std::vector<std::uint64_t> bytes_padded;
    std::vector<TaskStats> stats;
    std::uint64_t makespan_ns = 0;
};

/// runtime.hpp:802: the whole MoE layer, one persistent kernel launch per GPU.
inline ForwardResult forward(const MoeConfig& cfg, const std::vector<TokenMatrix>& shards, const ModelWeights& model,
                             const ForwardOptions& opts = {}) {
    cfg.validate();
    if (static_cast<std::int64_t>(shards.size()) != cfg.devices) throw ConfigError("forward: shard count != devices");
    if (static_cast<std::int64_t>(model.experts.size()) != cfg.experts_total)
        throw ConfigError("forward: expert parameter count != experts_total");
    if (opts.processors < 1) throw ConfigError("forward: need at least one processor");
    const std::int64_t S = cfg.tokens_per_device, H = cfg.embed_dim, D = cfg.ffn_dim, E = cfg.experts_total,
                       P = cfg.devices, K = cfg.topk;
    for (std::int64_t d = 0; d < P; ++d)
        if (shards[static_cast<std::size_t>(d)].rows != S || shards[static_cast<std::size_t>(d)].cols != H)
            throw ConfigError("forward: shard " + std::to_string(d) + " is not S x H");
    // flatten the weights into the ABI layout (w1: E x H x D, w2: E x D x H)
    std::vector<float> w1(static_cast<std::size_t>(E * H * D)), w2(static_cast<std::size_t>(E * D * H)),
        b1(static_cast<std::size_t>(E * D)), b2(static_cast<std::size_t>(E * H));
    for (std::int64_t e = 0; e < E; ++e) {
        const ExpertParams& ep = model.experts[static_cast<std::size_t>(e)];
        if (ep.w1.rows != H || ep.w1.cols != D || ep.w2.rows != D || ep.w2.cols != H ||
            static_cast<std::int64_t>(ep.b1.size()) != D || static_cast<std::int64_t>(ep.b2.size()) != H)
            throw ConfigError("forward: expert " + std::to_string(e) + " has wrong shapes");
        std::copy(ep.w1.data.begin(), ep.w1.data.end(), w1.begin() + e * H * D);
        std::copy(ep.w2.data.begin(), ep.w2.data.end(), w2.begin() + e * D * H);
        std::copy(ep.b1.begin(), ep.b1.end(), b1.begin() + e * D);
        std::copy(ep.b2.begin(), ep.b2.end(), b2.begin() + e * H);
    }
    if (model.gate.wg.rows != H || model.gate.wg.cols != E) throw ConfigError("forward: gate weights are not H x E");

    const fdmoe_config c = cfg.to_c();
    std::vector<std::int32_t> dev = opts.device_ids;
    if (dev.empty()) dev.assign(static_cast<std::size_t>(P), 0);
    fdmoe_handle* h = nullptr;
    detail::check(fdmoe_create(&c, dev.data(), static_cast<std::int32_t>(P), 0, &h));
    struct Guard { fdmoe_handle* h; ~Guard() { fdmoe_destroy(h); } } guard{h};
    detail::check(fdmoe_set_weights(h, model.gate.wg.data.data(), w1.data(), b1.data(), w2.data(), b2.data(),
                                    FDMOE_HOST));

    ForwardResult res;
    res.outputs.assign(static_cast<std::size_t>(P), TokenMatrix(S, H));
    const std::int64_t C = expert_capacity(cfg);
    std::vector<const float*> in(static_cast<std::size_t>(P));
    std::vector<float*> out(static_cast<std::size_t>(P));
    std::vector<fdmoe_routing> ro(static_cast<std::size_t>(P));
    std::vector<fdmoe_stats> st(static_cast<std::size_t>(P));
    std::vector<std::vector<std::int64_t>> tt(static_cast<std::size_t>(P)), drop(static_cast<std::size_t>(P));
    std::vector<std::vector<float>> tw(static_cast<std::size_t>(P));
    std::vector<std::int64_t> nd(static_cast<std::size_t>(P));
    res.gates.resize(static_cast<std::size_t>(P));
    for (std::int64_t d = 0; d < P; ++d) {
        const auto i = static_cast<std::size_t>(d);
        in[i] = shards[i].data.data();
        out[i] = res.outputs[i].data.data();
        GateOutput& g = res.gates[i];
        g.capacity = C;
        g.g_phi = TokenMatrix(S, E);
        g.slot_counts.assign(static_cast<std::size_t>(E), 0);
        tt[i].assign(static_cast<std::size_t>(E * C), -1);
        tw[i].assign(static_cast<std::size_t>(E * C), 0.0f);
        drop[i].assign(static_cast<std::size_t>(2 * S * K), 0);
        ro[i] = fdmoe_routing{g.g_phi.data.data(), tt[i].data(), tw[i].data(), g.slot_counts.data(),
                              drop[i].data(), &nd[i], nullptr, nullptr, nullptr};
    }
    fdmoe_options o{};
    o.processors = opts.processors;
    o.sequential = opts.mode == ScheduleMode::sequential ? 1 : 0;
    o.deadlock_budget_ms = opts.deadlock_budget_ms;
    o.exact_gate = opts.exact_gate ? 1 : 0;
    o.trace_events = opts.trace ? 1 : 0;
    o.straggler_kind = static_cast<std::int32_t>(opts.straggler.kind);
    o.straggler_device = opts.straggler.device;
    o.straggler_a = opts.straggler.a;
    o.straggler_b = opts.straggler.b;
    o.seed = opts.seed;
    detail::check(fdmoe_forward(h, in.data(), out.data(), FDMOE_HOST, &o, ro.data(), st.data()));
    if (opts.trace) {
        std::vector<fdmoe_event> evs;
        std::uint64_t base = ~0ull;
        for (std::int64_t d = 0; d < P; ++d) {
            std::int64_t n = 0, dropped = 0;
            detail::check(fdmoe_read_events(h, static_cast<std::int32_t>(d), nullptr, 0, &n, &dropped));
            std::vector<fdmoe_event> buf(static_cast<std::size_t>(n));
            detail::check(fdmoe_read_events(h, static_cast<std::int32_t>(d), buf.data(), n, &n, &dropped));
            for (auto& e : buf) {
                base = std::min<std::uint64_t>(base, e.t0);
                res.trace.emplace_back();
                TraceEvent& t = res.trace.back();
                t.t0 = e.t0;
                t.t1 = e.t1;
                t.device = static_cast<std::int32_t>(d);
                std::snprintf(t.worker, sizeof(t.worker), "cta%d", e.cta);
                t.event = detail::event_name(e.kind);
                t.task_type = e.kind == FDMOE_EV_EXEC ? detail::task_name(e.type) : nullptr;
                t.src = e.src; t.expert = e.expert; t.rb = e.rb; t.cb = e.cb; t.value = e.value; t.peer = e.peer;
            }
        }
        for (auto& t : res.trace) {
            t.t0 -= base;
            if (t.t1) t.t1 -= base;
        }
        std::stable_sort(res.trace.begin(), res.trace.end(),
                         [](const TraceEvent& a, const TraceEvent& b) { return a.t0 < b.t0; });
    }

    double kernel_ms = 0.0;
    for (std::int64_t d = 0; d < P; ++d) {
        const auto i = static_cast<std::size_t>(d);
        GateOutput& g = res.gates[i];
        g.table.resize(static_cast<std::size_t>(E * C));
        for (std::size_t j = 0; j < g.table.size(); ++j) g.table[j] = SlotMap{tt[i][j], tw[i][j]};
        for (std::int64_t j = 0; j < nd[i]; ++j)
            g.dropped.emplace_back(drop[i][static_cast<std::size_t>(2 * j)], drop[i][static_cast<std::size_t>(2 * j + 1)]);
        res.manifests.push_back(dispatch_manifest(g, cfg));
        TaskStats ts;
        ts.gemm0 = st[i].gemm0; ts.gemm1 = st[i].gemm1; ts.combine = st[i].combine;
        ts.enqueued = st[i].enqueued; ts.executed = st[i].executed; ts.bound_initial = st[i].bound_initial;
        ts.bound_final = st[i].bound_final; ts.scheduled_final = st[i].scheduled_final; ts.launches = st[i].launches;
        res.stats.push_back(ts);
        kernel_ms = std::max(kernel_ms, st[i].kernel_ms);
    }
    // pgas.hpp:130-147 accounting from the routing counts (dispatch + combine rows, FP32 units)
    const std::int64_t el = cfg.local_experts();
    res.bytes.assign(static_cast<std::size_t>(P * P), 0);
    for (std::int64_t p = 0; p < P; ++p)
        for (std::int64_t q = 0; q < P; ++q) {
            std::int64_t n = 0;
            for (std::int64_t le = 0; le < el; ++le)
                n += res.gates[static_cast<std::size_t>(p)].slot_counts[static_cast<std::size_t>(q * el + le)] +
                     res.gates[static_cast<std::size_t>(q)].slot_counts[static_cast<std::size_t>(p * el + le)];
            res.bytes[static_cast<std::size_t>(p * P + q)] = static_cast<std::uint64_t>(n * H * 4);
        }
    const std::uint64_t per = 2ull * static_cast<std::uint64_t>(el) *
                              static_cast<std::uint64_t>(padded_capacity(C, cfg.tile_rows)) *
                              static_cast<std::uint64_t>(H) * 4ull;
    res.bytes_padded.assign(static_cast<std::size_t>(P * P), per);
    res.makespan_ns = static_cast<std::uint64_t>(kernel_ms * 1e6);
    return res;
}

}  // namespace moefabric
