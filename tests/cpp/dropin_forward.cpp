// The reference's C++ entry point, moefabric::forward (runtime.hpp:802), called exactly as a reference
// user calls it -- only the include changes (include/moefabric_b200.hpp) -- on a B200.
// Inputs: the harness generator (harness.hpp:76-109, fdmoe_synth_*). Writes the P output shards and the
// P slot tables (int32 token ids) to argv[1] for tests/test_gpu_faults.py to compare with the
// reference's own forward(); checks the TaskStats invariants here.
#include "moefabric_b200.hpp"

#include <cstdio>
#include <cstring>

int main(int argc, char** argv) {
    if (argc < 2) return 64;
    moefabric::MoeConfig cfg;
    cfg.tokens_per_device = 512;
    cfg.embed_dim = 256;
    cfg.ffn_dim = 512;
    cfg.experts_total = 8;
    cfg.devices = 2;
    cfg.topk = 2;
    cfg.seed = 3;
    const std::int64_t S = cfg.tokens_per_device, H = cfg.embed_dim, D = cfg.ffn_dim, E = cfg.experts_total,
                       P = cfg.devices;

    // the harness's seeded model and shards, in the reference's own types
    std::vector<float> wg(H * E), w1(E * H * D), b1(E * D), w2(E * D * H), b2(E * H), a(P * S * H);
    const fdmoe_config c = cfg.to_c();
    moefabric::detail::check(fdmoe_synth_model(&c, cfg.seed, wg.data(), w1.data(), b1.data(), w2.data(), b2.data()));
    moefabric::detail::check(fdmoe_synth_shards(&c, cfg.seed, a.data()));
    moefabric::ModelWeights model;
    model.gate.wg = moefabric::TokenMatrix(H, E);
    model.gate.wg.data = wg;
    model.experts.resize(E);
    for (std::int64_t e = 0; e < E; ++e) {
        auto& ep = model.experts[e];
        ep.w1 = moefabric::TokenMatrix(H, D);
        std::memcpy(ep.w1.data.data(), w1.data() + e * H * D, H * D * 4);
        ep.w2 = moefabric::TokenMatrix(D, H);
        std::memcpy(ep.w2.data.data(), w2.data() + e * D * H, D * H * 4);
        ep.b1.assign(b1.begin() + e * D, b1.begin() + (e + 1) * D);
        ep.b2.assign(b2.begin() + e * H, b2.begin() + (e + 1) * H);
    }
    std::vector<moefabric::TokenMatrix> shards(P, moefabric::TokenMatrix(S, H));
    for (std::int64_t d = 0; d < P; ++d) std::memcpy(shards[d].data.data(), a.data() + d * S * H, S * H * 4);

    moefabric::ForwardResult r;
    try {
        r = moefabric::forward(cfg, shards, model);
    } catch (const std::exception& ex) {
        std::printf("forward threw: %s\n", ex.what());
        return 1;
    }
    // the reference's failure contract: a bad config throws ConfigError
    try {
        moefabric::MoeConfig bad = cfg;
        bad.experts_total = 6;
        moefabric::forward(bad, shards, model);
        std::printf("bad config accepted\n");
        return 2;
    } catch (const moefabric::ConfigError&) {
    }
    for (std::int64_t d = 0; d < P; ++d) {
        const auto& s = r.stats[d];
        if (!(s.bound_final == s.scheduled_final && s.scheduled_final == s.executed && s.executed > 0 &&
              s.launches == 1)) {
            std::printf("stats mismatch on rank %lld: bound %lld sched %lld exec %lld\n", (long long)d,
                        (long long)s.bound_final, (long long)s.scheduled_final, (long long)s.executed);
            return 3;
        }
    }
    std::printf("stats ok\n");
    FILE* f = std::fopen(argv[1], "wb");
    if (!f) return 4;
    for (std::int64_t d = 0; d < P; ++d) std::fwrite(r.outputs[d].data.data(), 4, S * H, f);
    const std::int64_t C = r.gates[0].capacity;
    for (std::int64_t d = 0; d < P; ++d)
        for (std::int64_t j = 0; j < E * C; ++j) {
            const std::int32_t t = static_cast<std::int32_t>(r.gates[d].table[j].token);
            std::fwrite(&t, 4, 1, f);
        }
    std::fclose(f);
    return 0;
}
