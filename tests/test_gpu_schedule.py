"""GPU tests of the §8(f) paths inside the single launch: the bulk-synchronous schedule
(ScheduleMode::sequential, runtime.hpp:885-908), the device event log and its audits (trace.hpp,
audit.hpp), straggler injection (runtime.hpp:312-362) and the payload/memory report."""
import json

import numpy as np
import pytest

import paper_2506_04667_b200 as fd
from paper_2506_04667_b200 import audit, report
from paper_2506_04667_b200.trace import busy_fractions
from oracle import pyoracle as po

pytestmark = pytest.mark.gpu


def _cfg(P, E, S=256, H=128, D=256, k=2, prec=fd.Precision.fp32, seed=11):
    return fd.MoeConfig(tokens_per_device=S, embed_dim=H, ffn_dim=D, experts_total=E, devices=P, topk=k,
                        precision=prec, seed=seed)


def _run(cfg, opts, model=None, shards=None):
    model = model if model is not None else fd.make_model(cfg)
    shards = shards if shards is not None else fd.make_shards(cfg)
    op = fd.Operator(cfg)
    op.set_weights(model)
    res = op.forward(shards, opts)
    info = op.info()
    ms = op.last_kernel_ms()
    op.close()
    return res, info, ms, model, shards


@pytest.mark.parametrize("P,E,S", [(1, 8, 512), (2, 8, 256), (4, 16, 256), (8, 16, 128)])
def test_sequential_mode_matches_overlapped(P, E, S):
    """The bulk-synchronous baseline computes the same layer: routing identical and outputs
    bit-identical (every tile and the combine order are schedule independent)."""
    cfg = _cfg(P, E, S)
    ov, _, _, model, shards = _run(cfg, fd.ForwardOptions())
    sq, _, _, _, _ = _run(cfg, fd.ForwardOptions(mode=fd.ScheduleMode.sequential), model, shards)
    for d in range(P):
        assert np.array_equal(sq.gates[d].table_token, ov.gates[d].table_token)
        assert np.array_equal(sq.outputs[d].view(np.uint32), ov.outputs[d].view(np.uint32))
        want = po.dense_forward(shards[d], model, cfg, threads=8)
        assert fd.max_rel_error([sq.outputs[d]], [want]) <= 1e-4


@pytest.mark.parametrize("sequential", [False, True])
@pytest.mark.parametrize("P,E,S,prec", [(1, 8, 512, fd.Precision.fp32), (2, 8, 256, fd.Precision.fp32),
                                         (4, 16, 384, fd.Precision.bf16), (8, 32, 128, fd.Precision.fp32)])
def test_event_log_passes_audits(P, E, S, prec, sequential, tmp_path):
    cfg = _cfg(P, E, S, prec=prec)
    res, info, _, _, _ = _run(cfg, fd.ForwardOptions(sequential=sequential, trace=True))
    rep = audit.full_audit(res, cfg, sequential=sequential, ctas_per_rank=info["ctas_per_rank"],
                           fused_combine=bool(info["fused_combine"]))
    assert rep.ok(), rep.problems[:5]
    assert (audit.barrier_event_count(res) > 0) == sequential
    bf = busy_fractions(res.trace)
    assert len(bf) == P * info["ctas_per_rank"]
    assert all(0.0 <= v <= 1.0 for v in bf.values())
    assert max(bf.values()) > 0.0
    j = report.report_json(cfg, fd.ForwardOptions(sequential=sequential), [res.makespan_ns], res, info=info)
    json.dumps(j)
    assert j["memory"]["gpu"]["ctas_per_rank"] == info["ctas_per_rank"]
    assert j["tasks"]["total"] == sum(s.total() for s in res.stats)


def test_event_log_repeated_and_off():
    """The log is per launch (reset before each traced launch) and costs nothing when off."""
    cfg = _cfg(2, 8)
    model = fd.make_model(cfg)
    shards = fd.make_shards(cfg)
    op = fd.Operator(cfg)
    op.set_weights(model)
    r1 = op.forward(shards, fd.ForwardOptions(trace=True))
    r2 = op.forward(shards, fd.ForwardOptions(trace=True))
    assert len(r1.trace) == len(r2.trace) > 0
    r3 = op.forward(shards)
    assert r3.trace == []
    assert np.array_equal(r3.outputs[0], r1.outputs[0])
    op.close()


def test_straggler_holds_back_dispatch():
    """A constant per-packet delay on rank 1: its packet signals appear no earlier than the
    cumulative hold-back, the layer takes at least that long, and the results are unchanged."""
    cfg = _cfg(2, 8, S=256)
    base, _, base_ms, model, shards = _run(cfg, fd.ForwardOptions(trace=True))
    spec = fd.StragglerSpec("constant", 0.05, 0.0, 1)
    opts = fd.ForwardOptions(trace=True, straggler=spec)
    hold = fd.straggler_delays(cfg, opts)
    assert int(hold[-1]) == 8 * 50_000
    res, _, ms, _, _ = _run(cfg, opts, model, shards)
    assert ms * 1e6 >= hold[-1] * 0.95
    for d in range(2):
        assert np.array_equal(res.outputs[d].view(np.uint32), base.outputs[d].view(np.uint32))
    # rank 1's gate finishes before its dispatch starts: signals are at least hold[e] after it
    gate_end = max(e.t1 for e in res.trace if e.device == 1 and e.event == "gate_done")
    sig = {(e.peer * cfg.local_experts() + e.expert): e.t0 for e in res.trace
           if e.device == 1 and e.event == "dispatch_put"}
    assert len(sig) == cfg.experts_total
    for e, t in sig.items():
        assert t - gate_end >= int(hold[e]) * 0.95, (e, t - gate_end, int(hold[e]))
    assert audit.full_audit(res, cfg, fused_combine=True).ok()


def test_lognormal_straggler_sequential_slower_than_overlapped():
    """Paper Table 2's ordinal claim on one GPU: with a straggling rank, the bulk-synchronous
    schedule is no faster than the overlapped one."""
    cfg = _cfg(4, 16, S=512, H=256, D=512)
    spec = fd.StragglerSpec("lognormal", 0.02, 0.5, 2)
    ov, _, ov_ms, model, shards = _run(cfg, fd.ForwardOptions(straggler=spec, seed=3))
    sq, _, sq_ms, _, _ = _run(cfg, fd.ForwardOptions(straggler=spec, seed=3, sequential=True), model, shards)
    assert sq_ms >= ov_ms * 0.9
    for d in range(4):
        assert np.array_equal(sq.outputs[d].view(np.uint32), ov.outputs[d].view(np.uint32))


def test_forward_stream_matches_single_launches():
    """fdmoe_forward_stream (copies of neighbouring batches overlapping each launch) computes exactly
    what one synchronous forward per batch computes."""
    import torch
    cfg = _cfg(2, 8, S=256)
    model = fd.make_model(cfg)
    op = fd.Operator(cfg)
    op.set_weights(model)
    batches = [fd.make_shards(cfg, seed=200 + b) for b in range(5)]
    pin = [[torch.from_numpy(a.copy()).pin_memory().numpy() for a in b] for b in batches]
    outs = [[torch.empty(a.shape, dtype=torch.float32).pin_memory().numpy() for a in b] for b in batches]
    op.forward_stream(pin, outs)
    for b, shards in enumerate(batches):
        want = op.forward(shards, routing=False, stats=False).outputs
        for d in range(2):
            assert np.array_equal(outs[b][d].view(np.uint32), want[d].view(np.uint32)), (b, d)
    op.close()
