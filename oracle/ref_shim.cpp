// ref_shim.cpp — C-ABI shim over the UNMODIFIED reference headers (TEST INFRASTRUCTURE ONLY).
//
// Compiled by oracle/Makefile against /root/reference/proj/include into
// oracle/_ref/libmoefabric_ref.so. It contains no algorithm of its own: it only
// marshals flat arrays into the reference's types and calls
//   moefabric::forward                     (runtime.hpp:802)
//   moefabric::oracle::dense_moe_forward   (oracle.hpp:116)
//   moefabric::gate_forward                (gate.hpp:108)
// so the repo's oracle restatement and the CUDA operator can be checked against
// the reference itself, and bench.py can time the reference's CPU path.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <exception>
#include <string>
#include <vector>

#include "moefabric/gate.hpp"
#include "moefabric/oracle.hpp"
#include "moefabric/runtime.hpp"

using namespace moefabric;

namespace {

thread_local std::string g_err;

MoeConfig make_cfg(const int64_t* v, double cf) {
    MoeConfig c;
    c.tokens_per_device = v[0];
    c.embed_dim = v[1];
    c.ffn_dim = v[2];
    c.experts_total = v[3];
    c.devices = v[4];
    c.topk = v[5];
    c.tile_rows = v[6];
    c.tile_cols = v[7];
    c.activation = static_cast<Activation>(v[8]);
    c.capacity_factor = cf;
    return c;
}

TokenMatrix mat(const float* p, int64_t r, int64_t c) {
    TokenMatrix m(r, c);
    std::memcpy(m.data.data(), p, sizeof(float) * static_cast<size_t>(r * c));
    return m;
}

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Model handle: the reference's ModelWeights built once from flat arrays
// (W1: E x H x D, B1: E x D, W2: E x D x H, B2: E x H, Wg: H x E).
void* ref_model_create(int64_t H, int64_t D, int64_t E, const float* wg, const float* w1,
                       const float* b1, const float* w2, const float* b2) {
    auto* m = new ModelWeights();
    m->gate.wg = mat(wg, H, E);
    m->experts.resize(static_cast<size_t>(E));
    for (int64_t e = 0; e < E; ++e) {
        ExpertParams& ep = m->experts[static_cast<size_t>(e)];
        ep.w1 = mat(w1 + e * H * D, H, D);
        ep.b1.assign(b1 + e * D, b1 + (e + 1) * D);
        ep.w2 = mat(w2 + e * D * H, D, H);
        ep.b2.assign(b2 + e * H, b2 + (e + 1) * H);
    }
    return m;
}

void ref_model_destroy(void* m) { delete static_cast<ModelWeights*>(m); }

// The reference harness's seeded model (harness.hpp:76-97, restated because harness.hpp itself
// needs the absent vendor/ JSON library): Wg, W1 ~ N(0,1)/sqrt(H), W2 ~ N(0,1)/sqrt(D),
// b ~ 0.1 N(0,1), one mt19937_64 stream in this draw order. Lets bench.py's reference arm build its
// inputs without loading the product library.
void* ref_model_synth(const int64_t* cfgv, double cf, uint64_t seed) {
    const MoeConfig cfg = make_cfg(cfgv, cf);
    std::mt19937_64 rng(seed);
    std::normal_distribution<float> dist(0.0f, 1.0f);
    const float s1 = 1.0f / std::sqrt(static_cast<float>(cfg.embed_dim));
    const float s2 = 1.0f / std::sqrt(static_cast<float>(cfg.ffn_dim));
    auto* m = new ModelWeights();
    m->gate.wg = TokenMatrix(cfg.embed_dim, cfg.experts_total);
    for (auto& v : m->gate.wg.data) v = dist(rng) * s1;
    m->experts.resize(static_cast<size_t>(cfg.experts_total));
    for (auto& ep : m->experts) {
        ep.w1 = TokenMatrix(cfg.embed_dim, cfg.ffn_dim);
        for (auto& v : ep.w1.data) v = dist(rng) * s1;
        ep.b1.assign(static_cast<size_t>(cfg.ffn_dim), 0.0f);
        for (auto& v : ep.b1) v = 0.1f * dist(rng);
        ep.w2 = TokenMatrix(cfg.ffn_dim, cfg.embed_dim);
        for (auto& v : ep.w2.data) v = dist(rng) * s2;
        ep.b2.assign(static_cast<size_t>(cfg.embed_dim), 0.0f);
        for (auto& v : ep.b2) v = 0.1f * dist(rng);
    }
    return m;
}

// harness.hpp:99-109: device d's tokens from mt19937_64(seed ^ 0xD1B54A32D192ED03 * (d + 1)).
// out: P x S x H.
void ref_synth_shards(const int64_t* cfgv, double cf, uint64_t seed, float* out) {
    const MoeConfig cfg = make_cfg(cfgv, cf);
    const int64_t n = cfg.tokens_per_device * cfg.embed_dim;
    for (int64_t d = 0; d < cfg.devices; ++d) {
        std::mt19937_64 rng(seed ^ (0xD1B54A32D192ED03ull * (static_cast<uint64_t>(d) + 1)));
        std::normal_distribution<float> dist(0.0f, 1.0f);
        float* a = out + d * n;
        for (int64_t i = 0; i < n; ++i) a[i] = dist(rng);
    }
}

// forward(): cfgv = {S, H, D, E, P, k, bM, bN, act}. shards/out: P x S x H.
// Routing outputs per device: tbl_tok/tbl_w P x E x cap, slot_counts P x E,
// g_phi P x S x E (all nullable). bytes/bytes_padded: P x P. stats: P x 9
// {gemm0, gemm1, combine, enqueued, executed, bound_initial, bound_final,
//  scheduled_final, launches}. Returns 0 or 1 (ConfigError) / 2 (ProtocolError) /
// 3 (RuntimeFault) / 9 (other).
int ref_forward(const int64_t* cfgv, double cf, int processors, int sequential, void* model,
                const float* shards, float* out, int64_t* tbl_tok, float* tbl_w,
                int64_t* slot_counts, float* g_phi, uint64_t* bytes, uint64_t* bytes_padded,
                int64_t* stats, uint64_t* makespan_ns) {
    try {
        const MoeConfig cfg = make_cfg(cfgv, cf);
        const int64_t S = cfg.tokens_per_device, H = cfg.embed_dim, P = cfg.devices,
                      E = cfg.experts_total;
        std::vector<TokenMatrix> sh;
        for (int64_t d = 0; d < P; ++d) sh.push_back(mat(shards + d * S * H, S, H));
        ForwardOptions opts;
        opts.processors = processors;
        opts.mode = sequential ? ScheduleMode::sequential : ScheduleMode::overlapped;
        ForwardResult r = forward(cfg, sh, *static_cast<ModelWeights*>(model), opts);
        const int64_t cap = expert_capacity(cfg);
        for (int64_t d = 0; d < P; ++d) {
            const auto& o = r.outputs[static_cast<size_t>(d)];
            std::memcpy(out + d * S * H, o.data.data(), sizeof(float) * static_cast<size_t>(S * H));
            const GateOutput& g = r.gates[static_cast<size_t>(d)];
            if (tbl_tok)
                for (int64_t i = 0; i < E * cap; ++i) {
                    tbl_tok[d * E * cap + i] = g.table[static_cast<size_t>(i)].token;
                    tbl_w[d * E * cap + i] = g.table[static_cast<size_t>(i)].weight;
                }
            if (slot_counts)
                for (int64_t e = 0; e < E; ++e) slot_counts[d * E + e] = g.slot_counts[static_cast<size_t>(e)];
            if (g_phi)
                std::memcpy(g_phi + d * S * E, g.g_phi.data.data(), sizeof(float) * static_cast<size_t>(S * E));
            if (stats) {
                const TaskStats& s = r.stats[static_cast<size_t>(d)];
                int64_t* st = stats + d * 9;
                st[0] = s.gemm0; st[1] = s.gemm1; st[2] = s.combine; st[3] = s.enqueued;
                st[4] = s.executed; st[5] = s.bound_initial; st[6] = s.bound_final;
                st[7] = s.scheduled_final; st[8] = s.launches;
            }
        }
        if (bytes) std::memcpy(bytes, r.bytes.data(), sizeof(uint64_t) * r.bytes.size());
        if (bytes_padded)
            std::memcpy(bytes_padded, r.bytes_padded.data(), sizeof(uint64_t) * r.bytes_padded.size());
        if (makespan_ns) *makespan_ns = r.makespan_ns;
        return 0;
    } catch (const ConfigError& e) { return fail(e, 1);
    } catch (const ProtocolError& e) { return fail(e, 2);
    } catch (const RuntimeFault& e) { return fail(e, 3);
    } catch (const std::exception& e) { return fail(e, 9); }
}

// oracle::dense_moe_forward on one shard (S x H) -> out (S x H).
int ref_dense_forward(const int64_t* cfgv, double cf, void* model, const float* shard, float* out) {
    try {
        const MoeConfig cfg = make_cfg(cfgv, cf);
        const ModelWeights& m = *static_cast<ModelWeights*>(model);
        TokenMatrix o = oracle::dense_moe_forward(mat(shard, cfg.tokens_per_device, cfg.embed_dim),
                                                  m.gate, m.experts, cfg);
        std::memcpy(out, o.data.data(), sizeof(float) * o.data.size());
        return 0;
    } catch (const ConfigError& e) { return fail(e, 1);
    } catch (const std::exception& e) { return fail(e, 9); }
}

// gate_forward_with_capacity (cap < 0 -> expert_capacity(cfg)). Outputs as in
// orc_gate: tbl E x max(cap,1), slot_counts E, dropped 2*S*k pairs, g_phi S x E.
int ref_gate(const int64_t* cfgv, double cf, int64_t cap, const float* a, const float* wg,
             float* g_phi, int64_t* tbl_tok, float* tbl_w, int64_t* slot_counts,
             int64_t* dropped, int64_t* n_dropped) {
    try {
        const MoeConfig cfg = make_cfg(cfgv, cf);
        GateWeights g;
        g.wg = mat(wg, cfg.embed_dim, cfg.experts_total);
        const int64_t c = cap < 0 ? expert_capacity(cfg) : cap;
        GateOutput o = gate_forward_with_capacity(mat(a, cfg.tokens_per_device, cfg.embed_dim), g, cfg, c);
        std::memcpy(g_phi, o.g_phi.data.data(), sizeof(float) * o.g_phi.data.size());
        for (size_t i = 0; i < o.table.size(); ++i) {
            tbl_tok[i] = o.table[i].token;
            tbl_w[i] = o.table[i].weight;
        }
        for (size_t e = 0; e < o.slot_counts.size(); ++e) slot_counts[e] = o.slot_counts[e];
        for (size_t i = 0; i < o.dropped.size(); ++i) {
            dropped[2 * i] = o.dropped[i].first;
            dropped[2 * i + 1] = o.dropped[i].second;
        }
        *n_dropped = static_cast<int64_t>(o.dropped.size());
        return 0;
    } catch (const ConfigError& e) { return fail(e, 1);
    } catch (const std::exception& e) { return fail(e, 9); }
}

int64_t ref_expert_capacity(const int64_t* cfgv, double cf) { return expert_capacity(make_cfg(cfgv, cf)); }

// The reference's own per-packet straggler draws (runtime.hpp:312-326) in dispatch_tokens' order
// and RNG seeding (runtime.hpp:341-362), accumulated in ms: cum_ms[t * E_local + le].
int ref_straggler_delays(int kind, double a, double b, int device, uint64_t seed, int64_t devices,
                         int64_t local_experts, double* cum_ms) {
    StragglerSpec sp;
    sp.kind = static_cast<StragglerSpec::Kind>(kind);
    sp.a = a;
    sp.b = b;
    sp.device = device;
    std::mt19937_64 rng(seed ^ (0x9E3779B97F4A7C15ull * (static_cast<std::uint64_t>(device) + 1)));
    double cum = 0.0;
    for (int64_t t = 0; t < devices; ++t)
        for (int64_t le = 0; le < local_experts; ++le) {
            const double ms = moefabric::detail::sample_delay_ms(sp, rng);
            if (ms > 0.0) cum += ms;
            cum_ms[t * local_experts + le] = cum;
        }
    return 0;
}

}  // extern "C"
