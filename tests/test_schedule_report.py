"""CPU tests for the §8(f) host-side pieces: ForwardOptions ABI layout, straggler sampling pinned to the
reference's own sampler, the payload/memory report (harness.hpp) and the trace audits (audit.hpp) on
synthetic event streams. The GPU runs of these paths are in test_gpu_schedule.py."""
import json
import os
import subprocess
import tempfile

import numpy as np
import pytest

import paper_2506_04667_b200 as fd
from paper_2506_04667_b200 import audit, report
from paper_2506_04667_b200.trace import EVENT_DTYPE, TraceEvent, busy_fractions, to_trace_events, write_trace_jsonl
from oracle import pyoracle as po

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
needs_ref = pytest.mark.skipif(not po.ref_available(), reason="oracle/_ref not built")


def test_abi_struct_layouts_match_header():
    src = r'''
#include <stddef.h>
#include <stdio.h>
#include "fdmoe.h"
int main() {
    printf("%zu %zu %zu %zu %zu\n", sizeof(fdmoe_options), offsetof(fdmoe_options, straggler_a),
           offsetof(fdmoe_options, seed), sizeof(fdmoe_event), offsetof(fdmoe_event, value));
    return 0;
}
'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "t")
        r = subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        got = [int(x) for x in subprocess.run([exe], capture_output=True, text=True).stdout.split()]
    import ctypes as C
    O = fd._Opts
    assert got == [C.sizeof(O), O.straggler_a.offset, O.seed.offset, EVENT_DTYPE.itemsize,
                   EVENT_DTYPE.fields["value"][1]]
    assert fd.lib().fdmoe_abi_version() == 3


@needs_ref
@pytest.mark.parametrize("kind,a,b,device,seed,P,El", [
    ("constant", 0.25, 0.0, 1, 0, 2, 4),
    ("uniform", 0.1, 0.7, 0, 7, 4, 3),
    ("lognormal", 0.2, 0.5, 3, 12345, 4, 8),
    ("lognormal", 1.0, 1.5, 0, 99, 1, 16),
])
def test_straggler_delays_match_reference_sampler(kind, a, b, device, seed, P, El):
    cfg = fd.MoeConfig(tokens_per_device=8, embed_dim=8, ffn_dim=8, experts_total=P * El, devices=P)
    opts = fd.ForwardOptions(seed=seed, straggler=fd.StragglerSpec(kind, a, b, device))
    got = fd.straggler_delays(cfg, opts)
    code = fd.StragglerSpec._KINDS[kind]
    want_ms = po.ref_straggler_delays(code, a, b, device, seed, P, El)
    want = np.array([int(round(x * 1e6)) for x in want_ms], np.uint64)
    assert np.array_equal(got, want)
    assert np.all(np.diff(got.astype(np.int64)) >= 0)


def test_straggler_rejects_bad_spec():
    cfg = fd.MoeConfig(tokens_per_device=8, embed_dim=8, ffn_dim=8, experts_total=4, devices=2)
    with pytest.raises(fd.ConfigError):
        fd.straggler_delays(cfg, fd.ForwardOptions(straggler=fd.StragglerSpec("constant", 1.0, 0.0, 2)))
    with pytest.raises(fd.ConfigError):
        fd.ForwardOptions(straggler=fd.StragglerSpec("gamma")).to_c()
    with pytest.raises(fd.ConfigError):
        fd.ForwardOptions(mode="eager").to_c()
    assert fd.ForwardOptions(mode=fd.ScheduleMode.sequential).to_c().sequential == 1


def test_memory_table_matches_reference_table3():
    # test_config.cpp:42-58 (EC, max(bM, EC)) and Size(L) = P*2*2*E_local*C'*H*4 (layout.hpp:43-47, 106)
    want = [(4096, 16, 256, 256), (4096, 32, 128, 128), (4096, 64, 64, 128), (4096, 128, 32, 128),
            (8192, 16, 512, 512), (8192, 32, 256, 256), (8192, 64, 128, 128), (8192, 128, 64, 128),
            (16384, 16, 1024, 1024), (16384, 32, 512, 512), (16384, 64, 256, 256), (16384, 128, 128, 128)]
    rows = report.memory_table()
    assert [(r["tokens"], r["experts"], r["capacity"], r["padded"]) for r in rows] == want
    for r in rows:
        assert r["size_mb"] == 2 * 2 * r["experts"] * r["padded"] * 1024 * 4 / 2 ** 20
    txt = report.memory_table_text().splitlines()
    assert txt[0] == "tokens,experts,capacity,padded_capacity,size_L_mb" and len(txt) == 13
    assert txt[-1] == "16384,128,128,128,256.00"


def _fake_result(cfg, counts):
    """ForwardResult carrying only routing counts (gates[d].slot_counts) and stats."""
    gates = []
    for d in range(cfg.devices):
        g = fd.GateOutput(np.zeros((1, 1), np.float32), 0, np.zeros((cfg.experts_total, 0), np.int64),
                          np.zeros((cfg.experts_total, 0), np.float32), np.asarray(counts[d], np.int64), [])
        gates.append(g)
    b = fd.payload_bytes(cfg, [g.slot_counts for g in gates])
    return fd.ForwardResult([], gates, [], [], b, fd.padded_baseline_bytes(cfg), [], 1000)


def test_payload_report_and_csv(tmp_path):
    cfg = fd.MoeConfig(tokens_per_device=64, embed_dim=32, ffn_dim=48, experts_total=4, devices=2, topk=2,
                       tile_rows=16, tile_cols=8)
    counts = [[16, 10, 5, 16], [0, 16, 16, 7]]   # C = 64 / 4 = 16
    res = _fake_result(cfg, counts)
    res.stats = [fd.TaskStats(gemm0=6, gemm1=4, combine=4, launches=1), fd.TaskStats(launches=1)]
    # bytes[p][q] = rows p -> q (dispatch) + rows q -> p (combine), FP32 rows of H
    assert report.remote_total(res.bytes, 2) == 2 * (5 + 16 + 0 + 16) * 32 * 4
    assert int(res.bytes[0]) == 2 * (16 + 10) * 32 * 4
    j = report.report_json(cfg, fd.ForwardOptions(mode="sequential"), [300, 100, 200], res)
    assert j["mode"] == "sequential" and j["latency_ns"]["median"] == 200 and j["latency_ns"]["mean"] == 200
    assert j["bytes"]["padded_remote_total"] == 2 * (2 * 2 * 16 * 32 * 4)
    assert 0 < j["bytes"]["remote_ratio"] < 1
    assert j["tasks"]["total"] == 14
    m = j["memory"]
    assert m["size_L_formula_bytes"] == m["heap_bytes_per_device"] == 2 * 2 * 2 * 2 * 16 * 32 * 4
    json.dumps(j)
    p = tmp_path / "bytes.csv"
    report.write_bytes_csv(str(p), res, 2)
    lines = p.read_text().splitlines()
    assert lines[0] == "src,dst,efficient_bytes,padded_bytes" and len(lines) == 5
    assert lines[2].split(",")[:2] == ["0", "1"]


def _synthetic_trace(cfg, counts, sequential=False, ctas=3):
    """A trace that obeys the protocol: signals, then GEMM0 tiles, then GEMM1, puts, combine."""
    El, P = cfg.local_experts(), cfg.devices
    res = _fake_result(cfg, counts)
    nb0, nb1 = -(-cfg.ffn_dim // 128), -(-cfg.embed_dim // 128)
    recs = [[] for _ in range(P)]
    t = 1000

    def ev(d, kind, t0, t1=0, typ=0, src=-1, expert=-1, rb=-1, cb=-1, peer=-1, value=0, cta=0):
        recs[d].append((t0, t1, kind, cta, typ, src, expert, rb, cb, peer, value))

    for d in range(P):
        for c in range(ctas):
            ev(d, 1, 10, 20, cta=c)
        for e in range(cfg.experts_total):
            ev(d, 2, 100 + e, src=d, expert=e % El, peer=e // El, value=counts[d][e])
    t = 500
    stats = []
    for d in range(P):
        tiles = audit.tile_rows(cfg, res.gates, d)
        for (le, m), (s0, ns, rows) in sorted(tiles.items()):
            for nb in range(nb0):
                ev(d, 3, t, t + 10, 1, s0, le, m, nb, ns, rows); t += 11
        for (le, m), (s0, ns, rows) in sorted(tiles.items()):
            for nb in range(nb1):
                ev(d, 3, t, t + 10, 2, s0, le, m, nb, ns, rows)
                for j in range(ns):
                    ev(d, 4, t + 10, 0, 2, d, le, m, nb, s0 + j, rows)
                t += 11
        stats.append(fd.TaskStats(gemm0=len(tiles) * nb0, gemm1=len(tiles) * nb1,
                                  combine=-(-cfg.tokens_per_device // 16), launches=1))
    t += 100
    for d in range(P):
        for blk in range(-(-cfg.tokens_per_device // 16)):
            ev(d, 3, t, t + 5, 3, d, -1, blk, -1, -1, 16, cta=blk % ctas)
        for c in range(ctas):
            ev(d, 0, 0, t + 50, cta=c)
    if sequential:
        for d in range(P):
            ev(d, 5, 400, value=0); ev(d, 6, 450, value=0)
    arrs = [np.array(r, EVENT_DTYPE) for r in recs]
    res.trace = to_trace_events(arrs)
    res.stats = stats
    return res


@pytest.mark.parametrize("P,E,S", [(2, 4, 64), (4, 8, 40), (1, 3, 300)])
def test_audit_accepts_protocol_trace(P, E, S):
    cfg = fd.MoeConfig(tokens_per_device=S, embed_dim=256, ffn_dim=384, experts_total=E, devices=P, topk=2)
    cap = fd.expert_capacity(cfg)
    rng = np.random.default_rng(P * 100 + E)
    counts = [list(rng.integers(0, cap + 1, size=E)) for _ in range(P)]
    res = _synthetic_trace(cfg, counts, ctas=3)
    rep = audit.full_audit(res, cfg, ctas_per_rank=3)
    assert rep.ok(), rep.problems
    bf = busy_fractions(res.trace)
    assert len(bf) == 3 * P and all(0.0 <= v <= 1.0 for v in bf.values())


def test_audit_flags_violations(tmp_path):
    cfg = fd.MoeConfig(tokens_per_device=64, embed_dim=256, ffn_dim=256, experts_total=4, devices=2, topk=2)
    counts = [[32, 3, 0, 32], [32, 32, 16, 1]]
    base = _synthetic_trace(cfg, counts)
    assert audit.full_audit(base, cfg).ok()

    dup = _synthetic_trace(cfg, counts)
    dup.trace.append(next(e for e in dup.trace if e.event == "exec" and e.task_type == "gemm0"))
    assert any("executed" in p for p in audit.full_audit(dup, cfg).problems)

    late = _synthetic_trace(cfg, counts)
    g0 = next(e for e in late.trace if e.event == "exec" and e.task_type == "gemm0")
    g0.t1 = 10 ** 9
    assert any("gemm0 after gemm1" in p for p in audit.full_audit(late, cfg).problems)

    early = _synthetic_trace(cfg, counts)
    g0 = next(e for e in early.trace if e.event == "exec" and e.task_type == "gemm0")
    g0.t0 = 0
    assert any("before packet" in p for p in audit.full_audit(early, cfg).problems)

    put = _synthetic_trace(cfg, counts)
    next(e for e in put.trace if e.event == "tile_put").t0 = 10 ** 9
    assert any("tile put" in p for p in audit.full_audit(put, cfg).problems)

    acc = _synthetic_trace(cfg, counts)
    acc.stats[0].gemm1 += 1
    assert any("recount" in p for p in audit.full_audit(acc, cfg).problems)

    seq = _synthetic_trace(cfg, counts, sequential=True)
    assert audit.full_audit(seq, cfg, sequential=True).ok()
    assert any("barrier events in an overlapped" in p for p in audit.full_audit(seq, cfg).problems)
    assert any("without barrier" in p for p in audit.full_audit(base, cfg, sequential=True).problems)

    path = tmp_path / "t.jsonl"
    write_trace_jsonl(str(path), base.trace)
    first = json.loads(path.read_text().splitlines()[0])
    assert {"time", "device", "worker", "event"} <= set(first)
    execs = [json.loads(x) for x in path.read_text().splitlines() if '"exec"' in x]
    assert all(x["task"].startswith(x["type"] + ":s") for x in execs)
