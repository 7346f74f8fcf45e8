"""GPU parity at every BASELINE.json configuration (the reference's oracle_check protocol,
harness.hpp:418-426: per shard, forward() against dense_moe_forward, oracle.hpp:116-120).

* c1, c2 (P = 1, FP32): every output element against the full dense oracle.
* c3 (P = 2, 4; FP32), c4 (the bench shape, P = 1 and P = 8; FP32), c5 (P = 1, 2, 4, 8; bf16): routing
  of EVERY token bit-exact against orc_gate (picks, slots, T_phi, drops), and outputs on sampled token
  rows against orc_ffn_rows (the dense oracle's per-token FFN + combine for those rows, bit-identical
  to orc_dense_forward's rows) — the full dense oracle at these sizes takes minutes to hours per shard.
  EP > 1 runs as virtual ranks on the one GPU: the same single launch and the same cross-rank protocol.

Tolerances (BASELINE.json north_star): FP32 mode |got - want| <= 1e-5 + 1e-4 |want| per element and
normwise <= 1e-4; bf16 mode normwise <= 1e-2. Each case appends its error statistics to
gpurun_out/numerics.jsonl (summarised in profiles/).
"""
import json
import os
import time

import numpy as np
import pytest

import paper_2506_04667_b200 as fd
from oracle import pyoracle as po

pytestmark = pytest.mark.gpu

FP32_REL, FP32_ATOL, BF16_REL = 1e-4, 1e-5, 1e-2
THREADS = os.cpu_count() or 8
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# id: (S per rank, H, D, E_total, P, precision, full oracle?)
CONFIGS = {
    "c1": (1024, 1024, 2048, 8, 1, fd.Precision.fp32, True),
    "c2": (4096, 2048, 2048, 16, 1, fd.Precision.fp32, True),
    "c3_p2": (8192, 2048, 2048, 32, 2, fd.Precision.fp32, False),
    "c3_p4": (8192, 2048, 2048, 32, 4, fd.Precision.fp32, False),
    "c4_p1": (16384, 2048, 2048, 128, 1, fd.Precision.fp32, False),
    "c4_p8": (16384, 2048, 2048, 128, 8, fd.Precision.fp32, False),
    "c5_p1": (2048, 2048, 2048, 16, 1, fd.Precision.bf16, False),
    "c5_p2": (2048, 2048, 2048, 32, 2, fd.Precision.bf16, False),
    "c5_p4": (2048, 2048, 2048, 64, 4, fd.Precision.bf16, False),
    "c5_p8": (2048, 2048, 2048, 128, 8, fd.Precision.bf16, False),
}
N_SAMPLE = 192


def sample_rows(S, seed):
    """Low token ids (they hold the kept picks under cf = 1), the last ids (mostly fully dropped: zero
    rows) and a uniform sample."""
    rng = np.random.default_rng(seed)
    rows = np.concatenate([np.arange(32), np.arange(S - 16, S), rng.choice(S, N_SAMPLE - 48, replace=False)])
    return np.unique(rows)


def error_stats(got, want, prec):
    g = got.astype(np.float64)
    w = want.astype(np.float64)
    err = np.abs(g - w)
    bound = FP32_ATOL + FP32_REL * np.abs(w)
    num = np.sqrt(np.sum(err ** 2))
    den = np.sqrt(np.sum(w ** 2))
    return {"normwise": float(num / den) if den > 0 else float(num), "max_abs": float(err.max()),
            "max_err_over_bound": float((err / bound).max()), "n_bad": int(np.sum(err > bound)),
            "n": int(err.size), "prec": "fp32" if prec == fd.Precision.fp32 else "bf16"}


def record(name, d):
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "numerics.jsonl"), "a") as f:
        f.write(json.dumps({"case": name, **d}) + "\n")
    print(name, json.dumps(d))


def check_routing(cfg, shard, model, gate):
    cap = fd.expert_capacity(cfg)
    want = po.gate(shard, model.wg, cfg.topk, cap)
    assert np.array_equal(gate.slot_counts, want["slot_counts"]), "slot counts differ"
    assert np.array_equal(gate.table_token, want["table_token"][:, :cap]), "T_phi token indices differ"
    assert gate.dropped == want["dropped"], "capacity drops differ"
    assert np.array_equal(gate.picks_expert, want["picks_expert"]), "picks differ"
    assert np.array_equal(gate.picks_slot, want["picks_slot"]), "slots differ"
    return want


def check_outputs(prec, stats):
    if prec == fd.Precision.fp32:
        assert stats["normwise"] <= FP32_REL, stats
        assert stats["n_bad"] == 0, stats
    else:
        assert stats["normwise"] <= BF16_REL, stats


@pytest.mark.parametrize("name", list(CONFIGS))
def test_baseline_config(name):
    S, H, D, E, P, prec, full = CONFIGS[name]
    cfg = fd.MoeConfig(tokens_per_device=S, embed_dim=H, ffn_dim=D, experts_total=E, devices=P, topk=2,
                       capacity_factor=1.0, precision=prec, seed=0)
    model = fd.make_model(cfg)
    shards = fd.make_shards(cfg)
    t0 = time.perf_counter()
    res = fd.forward(cfg, shards, model)
    t_gpu = time.perf_counter() - t0
    for d in range(P):
        want_route = check_routing(cfg, shards[d], model, res.gates[d])
        if full:
            want = po.dense_forward(shards[d], model, cfg, threads=THREADS)
            got = res.outputs[d]
        else:
            rows = sample_rows(S, 17 + d)
            want = po.ffn_rows(shards[d], model, cfg, want_route, rows, threads=THREADS)
            got = res.outputs[d][rows]
            # rows whose picks were all dropped are exactly zero
            all_dropped = np.all(want_route["picks_slot"][rows] < 0, axis=1)
            assert np.all(got[all_dropped] == 0.0)
        st = error_stats(got, want, prec)
        st.update({"rank": d, "rows": "all" if full else int(got.shape[0]), "forward_s": t_gpu})
        record(name, st)
        check_outputs(prec, st)


@pytest.mark.parametrize("name,seed,nrows", [("c2", 1, 4096), ("c3_p4", 0, 3072), ("c4_p1", 1, 6144)])
def test_wide_rows(name, seed, nrows):
    """Beyond the sampled rows: thousands of contiguous token rows (the kept-pick region) at the configurations and
    seeds whose worst elements came closest to the FP32 bound before the split-K main accumulation and the exact
    pick weights (tools/dev/parity_wide.py, profiles/r02_numerics.md §5): every element within the bound."""
    S, H, D, E, P, prec, _ = CONFIGS[name]
    cfg = fd.MoeConfig(tokens_per_device=S, embed_dim=H, ffn_dim=D, experts_total=E, devices=P, topk=2,
                       capacity_factor=1.0, precision=prec, seed=seed)
    model = fd.make_model(cfg)
    shards = fd.make_shards(cfg)
    res = fd.forward(cfg, shards, model)
    for d in range(P):
        want_route = check_routing(cfg, shards[d], model, res.gates[d])
        rows = np.arange(min(nrows, S))
        want = po.ffn_rows(shards[d], model, cfg, want_route, rows, threads=THREADS)
        st = error_stats(res.outputs[d][rows], want, prec)
        st.update({"rank": d, "rows": int(rows.size), "seed": seed})
        record(name + "_wide", st)
        check_outputs(prec, st)
