// fdmoe_abi.cpp — the GPU-free part of the C ABI: configuration validation,
// capacity / layout / task-count arithmetic, and the seeded synthetic inputs.
// Each function restates the reference rule it cites; none of it runs on the hot path.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <string>

#include "fdmoe.h"
#include "fdmoe_internal.h"

namespace fdmoe {
thread_local std::string g_last_error;

fdmoe_status fail(fdmoe_status s, const std::string& msg) {
    g_last_error = msg;
    return s;
}
}  // namespace fdmoe

using fdmoe::fail;

extern "C" {

int32_t fdmoe_abi_version(void) { return FDMOE_ABI_VERSION; }
const char* fdmoe_last_error(void) { return fdmoe::g_last_error.c_str(); }

// config.hpp:68-86, then this operator's envelope.
fdmoe_status fdmoe_config_validate(const fdmoe_config* c, int32_t gpu_envelope) {
    if (!c) return fail(FDMOE_ERR_CONFIG, "null config");
    if (c->tokens_per_device < 1) return fail(FDMOE_ERR_CONFIG, "tokens_per_device must be >= 1");
    if (c->embed_dim < 1) return fail(FDMOE_ERR_CONFIG, "embed_dim must be >= 1");
    if (c->ffn_dim < 1) return fail(FDMOE_ERR_CONFIG, "ffn_dim must be >= 1");
    if (c->devices < 1) return fail(FDMOE_ERR_CONFIG, "devices must be >= 1");
    if (c->experts_total < 1) return fail(FDMOE_ERR_CONFIG, "experts_total must be >= 1");
    if (c->experts_total % c->devices != 0)
        return fail(FDMOE_ERR_CONFIG, "experts_total must be divisible by devices (uniform placement)");
    if (c->topk < 1 || c->topk > c->experts_total) return fail(FDMOE_ERR_CONFIG, "topk must be in [1, experts_total]");
    if (!(c->capacity_factor > 0.0)) return fail(FDMOE_ERR_CONFIG, "capacity_factor must be > 0");
    if (c->tile_rows < 1 || c->tile_cols < 1) return fail(FDMOE_ERR_CONFIG, "tile dims must be >= 1");
    const double prod = (double)c->devices * 4.0 * (double)c->experts_total *
                        (double)(c->tokens_per_device + c->tile_rows) * (double)c->embed_dim;
    if (prod > 9e15) return fail(FDMOE_ERR_CONFIG, "dimension product exceeds addressable size");
    if (c->activation < 0 || c->activation > 2) return fail(FDMOE_ERR_CONFIG, "unknown activation");
    if (c->precision < 0 || c->precision > 1) return fail(FDMOE_ERR_CONFIG, "unknown precision");
    if (gpu_envelope) {
        if (c->experts_total > fdmoe::kMaxExperts)
            return fail(FDMOE_ERR_UNSUPPORTED, "experts_total > 256 is outside the GPU gate envelope");
        if (c->topk > 8) return fail(FDMOE_ERR_UNSUPPORTED, "topk > 8 is outside the GPU envelope");
        if (c->devices > fdmoe::kMaxRanks) return fail(FDMOE_ERR_UNSUPPORTED, "devices > 64");
        if (c->embed_dim % 32 != 0 || c->ffn_dim % 32 != 0)
            return fail(FDMOE_ERR_UNSUPPORTED, "embed_dim and ffn_dim must be multiples of 32 on the GPU path");
        const int64_t C = fdmoe_expert_capacity(c);
        if (C > (int64_t)1 << 24) return fail(FDMOE_ERR_UNSUPPORTED, "capacity too large");
    }
    return FDMOE_OK;
}

// config.hpp:94-101
int64_t fdmoe_expert_capacity(const fdmoe_config* c) {
    const long double q = (long double)c->capacity_factor * (long double)c->tokens_per_device /
                          (long double)c->experts_total;
    const int64_t cap = (int64_t)std::ceil(q - 1e-9L);
    return cap < 1 ? 1 : cap;
}

// config.hpp:104-106
int64_t fdmoe_padded_capacity(int64_t capacity, int64_t tile_rows) {
    return (capacity + tile_rows - 1) / tile_rows * tile_rows;
}

// layout.hpp:106-113
uint64_t fdmoe_size_L(const fdmoe_config* c) {
    const uint64_t s = (uint64_t)c->tokens_per_device, h = (uint64_t)c->embed_dim,
                   e = (uint64_t)c->experts_total, bm = (uint64_t)c->tile_rows;
    if (s >= bm * e) return 16 * s * h;
    return 16 * bm * e * h;
}

// layout.hpp:67-79 (row-major over P x R x B x E x C' x H)
int64_t fdmoe_flat_index(int64_t devices, int64_t local_experts, int64_t slot_capacity, int64_t embed_dim,
                         int64_t p_star, int64_t round, int64_t buffer, int64_t expert, int64_t slot) {
    if (p_star < 0 || p_star >= devices || round < 0 || round >= 2 || buffer < 0 || buffer >= 2 || expert < 0 ||
        expert >= local_experts || slot < 0 || slot >= slot_capacity)
        return -1;
    return ((((p_star * 2 + round) * 2 + buffer) * local_experts + expert) * slot_capacity + slot) * embed_dim;
}

// layout.hpp:91-100
int32_t fdmoe_validate_write(int64_t src, int64_t dst, int64_t p_star, int64_t buffer) {
    if (buffer == 1) return p_star == src ? 0 : 1;
    return src == dst ? 0 : 2;
}

// runtime.hpp:122-145
int64_t fdmoe_gemm_tasks_for_rows(const fdmoe_config* c, int64_t n) {
    if (n <= 0) return 0;
    const int64_t cbf = (c->ffn_dim + c->tile_cols - 1) / c->tile_cols;
    const int64_t cbe = (c->embed_dim + c->tile_cols - 1) / c->tile_cols;
    return (n + c->tile_rows - 1) / c->tile_rows * (cbf + cbe);
}
int64_t fdmoe_combine_tiles_for_rows(const fdmoe_config* c, int64_t n) {
    if (n <= 0) return 0;
    return (n + c->tile_rows - 1) / c->tile_rows * ((c->embed_dim + c->tile_cols - 1) / c->tile_cols);
}
int64_t fdmoe_initial_task_bound(const fdmoe_config* c) {
    const int64_t el = c->experts_total / c->devices;
    const int64_t cp = fdmoe_padded_capacity(fdmoe_expert_capacity(c), c->tile_rows);
    const int64_t cbf = (c->ffn_dim + c->tile_cols - 1) / c->tile_cols;
    const int64_t cbe = (c->embed_dim + c->tile_cols - 1) / c->tile_cols;
    const int64_t worst = (cp / c->tile_rows) * (cbf + cbe);
    return c->devices * el * worst + c->topk * ((c->tokens_per_device + c->tile_rows - 1) / c->tile_rows) * cbe;
}

// harness.hpp:76-97: one mt19937_64 stream, fixed draw order Wg, then per expert W1, b1, W2, b2.
fdmoe_status fdmoe_synth_model(const fdmoe_config* c, uint64_t seed, float* wg, float* w1, float* b1, float* w2,
                               float* b2) {
    const int64_t H = c->embed_dim, D = c->ffn_dim, E = c->experts_total;
    std::mt19937_64 rng(seed);
    std::normal_distribution<float> dist(0.0f, 1.0f);
    const float s1 = 1.0f / std::sqrt(static_cast<float>(H));
    const float s2 = 1.0f / std::sqrt(static_cast<float>(D));
    for (int64_t i = 0; i < H * E; ++i) wg[i] = dist(rng) * s1;
    for (int64_t e = 0; e < E; ++e) {
        float* pw1 = w1 + e * H * D;
        for (int64_t i = 0; i < H * D; ++i) pw1[i] = dist(rng) * s1;
        float* pb1 = b1 + e * D;
        for (int64_t i = 0; i < D; ++i) pb1[i] = 0.1f * dist(rng);
        float* pw2 = w2 + e * D * H;
        for (int64_t i = 0; i < D * H; ++i) pw2[i] = dist(rng) * s2;
        float* pb2 = b2 + e * H;
        for (int64_t i = 0; i < H; ++i) pb2[i] = 0.1f * dist(rng);
    }
    return FDMOE_OK;
}

// harness.hpp:99-109: per-device stream seeded seed ^ (0xD1B54A32D192ED03 * (d + 1)).
fdmoe_status fdmoe_synth_shards(const fdmoe_config* c, uint64_t seed, float* shards) {
    const int64_t S = c->tokens_per_device, H = c->embed_dim;
    for (int64_t d = 0; d < c->devices; ++d) {
        std::mt19937_64 rng(seed ^ (0xD1B54A32D192ED03ull * (static_cast<uint64_t>(d) + 1)));
        std::normal_distribution<float> dist(0.0f, 1.0f);
        float* a = shards + d * S * H;
        for (int64_t i = 0; i < S * H; ++i) a[i] = dist(rng);
    }
    return FDMOE_OK;
}

// Straggler hold-back (runtime.hpp:312-326, 341-362): the straggling device draws one delay per
// (destination, local expert) packet, in that order, from std::mt19937_64(seed ^ 0x9E37...*(dev+1)),
// each distribution constructed afresh per draw as sample_delay_ms does, and sleeps it before the
// packet's put. cum_ns[e] (e = destination * E_local + local expert) is the running sum in ns: the
// earliest time after dispatch start that packet e's signal may be published.
fdmoe_status fdmoe_straggler_delays(const fdmoe_options* o, int64_t devices, int64_t local_experts,
                                    uint64_t* cum_ns) {
    if (!o || !cum_ns) return fail(FDMOE_ERR_CONFIG, "null argument");
    if (o->straggler_kind < FDMOE_STRAGGLER_NONE || o->straggler_kind > FDMOE_STRAGGLER_LOGNORMAL)
        return fail(FDMOE_ERR_CONFIG, "unknown straggler kind");
    if (o->straggler_device < 0 || o->straggler_device >= devices)
        return fail(FDMOE_ERR_CONFIG, "straggler device outside [0, devices)");
    std::mt19937_64 rng(o->seed ^ (0x9E3779B97F4A7C15ull * ((uint64_t)o->straggler_device + 1ull)));
    double cum_ms = 0.0;
    for (int64_t e = 0; e < devices * local_experts; ++e) {
        double ms = 0.0;
        switch (o->straggler_kind) {
            case FDMOE_STRAGGLER_NONE: break;
            case FDMOE_STRAGGLER_CONSTANT: ms = o->straggler_a; break;
            case FDMOE_STRAGGLER_UNIFORM: {
                std::uniform_real_distribution<double> u(o->straggler_a, o->straggler_b);
                ms = u(rng);
                break;
            }
            default: {
                std::lognormal_distribution<double> ln(std::log(std::max(o->straggler_a, 1e-9)), o->straggler_b);
                ms = ln(rng);
            }
        }
        if (ms > 0.0) cum_ms += ms;
        cum_ns[e] = (uint64_t)std::llround(cum_ms * 1e6);
    }
    return FDMOE_OK;
}

}  // extern "C"
