"""GPU tests of the operator's failure behaviour, task accounting, argument contract and the paths that
need their own processes:

* the device watchdog -> RuntimeFault (runtime.hpp:937-969), then recovery on the same operator;
* an over-subscribed dispatch packet -> ProtocolError (pgas.hpp:101-112), via the development library's
  fault injection in a subprocess, then recovery;
* device task accounting: bound self-corrected on the device == tasks scheduled == tiles executed
  (runtime.hpp:122-165, 407-415, 633-647), and equal to the count recomputed from the routing;
* in-place forwards rejected (ConfigError);
* two processes x one rank on one B200 through CUDA IPC (the torchrun data path), parity vs the oracle;
* the C++ drop-in (include/moefabric_b200.hpp, runtime.hpp:802) compiled and run on the GPU, parity vs
  the reference's own forward() (oracle/_ref) when it is built, else the oracle restatement.
"""
import json
import math
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import paper_2506_04667_b200 as fd
from oracle import pyoracle as po

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "gpu_workers.py")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _check_outputs(got, want, prec=fd.Precision.fp32):
    if prec == fd.Precision.fp32:
        assert np.all(np.abs(got - want) <= 1e-5 + 1e-4 * np.abs(want))
    else:
        assert fd.max_rel_error([got], [want]) <= 1e-2


def test_watchdog_raises_runtime_fault_and_recovers():
    """A straggler holding its dispatch signals past the deadlock budget trips the device watchdog of the
    waiting ranks: RuntimeFault, not a hang. The same operator then runs a clean forward."""
    cfg = fd.MoeConfig(tokens_per_device=256, embed_dim=128, ffn_dim=256, experts_total=8, devices=2, topk=2, seed=9)
    model = fd.make_model(cfg)
    shards = fd.make_shards(cfg)
    op = fd.Operator(cfg)
    op.set_weights(model)
    opts = fd.ForwardOptions(deadlock_budget_ms=40,
                             straggler=fd.StragglerSpec(kind="constant", a=400.0, device=1))
    with pytest.raises(fd.RuntimeFault, match="watchdog"):
        op.forward(shards, opts)
    res = op.forward(shards)
    for d in range(cfg.devices):
        _check_outputs(res.outputs[d], po.dense_forward(shards[d], model, cfg, threads=8))
    op.close()


def test_oversubscribed_packet_raises_protocol_error(tmp_path):
    out = str(tmp_path / "fault.json")
    r = subprocess.run([sys.executable, WORKER, "fault", out], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.load(open(out))
    assert res["first"].startswith("ProtocolError"), res["first"]
    assert "over-subscribed" in res["first"]
    cfg = fd.MoeConfig(tokens_per_device=256, embed_dim=128, ffn_dim=256, experts_total=8, devices=2, topk=2, seed=5)
    model = fd.make_model(cfg)
    shards = fd.make_shards(cfg)
    for d in range(cfg.devices):
        _check_outputs(np.asarray(res["outputs"][d], np.float32), po.dense_forward(shards[d], model, cfg, threads=8))


def _expected_tasks(res, cfg, info):
    """Non-empty (expert, row tile) pairs per destination rank from the routing (the realized task count,
    runtime.hpp:150-163, on the kernel's tile grid)."""
    P, El, Cp = cfg.devices, cfg.local_experts(), info["packet_rows"]
    nb0, nb1 = math.ceil(cfg.ffn_dim / 128), math.ceil(cfg.embed_dim / 128)
    out = []
    for q in range(P):
        tiles = 0
        for le in range(El):
            n = [int(res.gates[p].slot_counts[q * El + le]) for p in range(P)]
            if Cp >= 128:
                tiles += sum(math.ceil(x / 128) for x in n)
            else:
                per = 128 // Cp
                tiles += sum(1 for m in range(0, P, per) if sum(n[m:m + per]) > 0)
        out.append((tiles * nb0, tiles * nb1))
    return out


@pytest.mark.parametrize("P,E,S,cf,prec,seq", [
    (2, 8, 256, 8.0, fd.Precision.fp32, False),    # C' = 256: two row tiles per packet, the second mostly empty
    (4, 16, 256, 4.0, fd.Precision.fp32, True),    # separate combine phase (sequential schedule)
    (8, 32, 128, 1.0, fd.Precision.bf16, False),   # C' = 16: eight packets per row tile
])
def test_device_task_accounting(P, E, S, cf, prec, seq):
    cfg = fd.MoeConfig(tokens_per_device=S, embed_dim=256, ffn_dim=384, experts_total=E, devices=P, topk=2,
                       capacity_factor=cf, precision=prec, seed=13)
    op = fd.Operator(cfg)
    op.set_weights(fd.make_model(cfg))
    res = op.forward(fd.make_shards(cfg), fd.ForwardOptions(sequential=seq))
    info = op.info()
    op.close()
    exp = _expected_tasks(res, cfg, info)
    nb = math.ceil(cfg.ffn_dim / 128) + math.ceil(cfg.embed_dim / 128)
    row_tiles = cfg.local_experts() * math.ceil(info["packet_rows"] * P / 128)
    any_corrected = False
    for d, s in enumerate(res.stats):
        assert (s.gemm0, s.gemm1) == exp[d]
        assert s.bound_final == s.scheduled_final == s.executed, s
        assert s.combine in (0, math.ceil(S / 16))
        assert s.combine == 0 or seq or not info["fused_combine"]
        assert s.bound_initial == row_tiles * nb + s.combine
        assert s.tiles_resolved == row_tiles
        any_corrected |= s.bound_final < s.bound_initial
    if cf >= 8.0:
        assert any_corrected   # empty row tiles removed from the bound on the device


def test_in_place_forward_rejected():
    import torch
    cfg = fd.MoeConfig(tokens_per_device=128, embed_dim=128, ffn_dim=128, experts_total=4, devices=1, topk=2)
    op = fd.Operator(cfg)
    op.set_weights(fd.make_model(cfg))
    x = torch.from_numpy(fd.make_shards(cfg)[0]).cuda()
    with pytest.raises(fd.ConfigError, match="overlap"):
        op.forward_device([x.data_ptr()], [x.data_ptr()])
    with pytest.raises(fd.ConfigError, match="overlap"):   # partial overlap
        op.forward_device([x.data_ptr()], [x.data_ptr() + 4 * 128 * 8])
    y = torch.empty_like(x)
    op.forward_device([x.data_ptr()], [y.data_ptr()])
    op.sync()
    op.close()


@pytest.mark.parametrize("prec", [fd.Precision.fp32, fd.Precision.bf16])
def test_two_process_ipc_forward(prec, tmp_path):
    """Two OS processes, one rank each, on one B200: heaps cross-mapped through CUDA IPC, dispatch rows,
    combine rows and epoch flags cross the process boundary. Overlapped twice (epoch parity flip), then
    sequential; every output checked against the oracle, routing bit-exact, accounting consistent."""
    world, port = 2, _free_port()
    outs = [str(tmp_path / f"r{r}.npz") for r in range(world)]
    env = dict(os.environ, PYTHONPATH=ROOT)
    procs = [subprocess.Popen([sys.executable, WORKER, "ipc", str(r), str(world), str(port), str(int(prec)), outs[r]],
                              cwd=ROOT, env=env, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
             for r in range(world)]
    errs = []
    for p in procs:
        try:
            _, e = p.communicate(timeout=900)
        except subprocess.TimeoutExpired:
            p.kill()
            _, e = p.communicate()
        errs.append(e)
    assert all(p.returncode == 0 for p in procs), [e[-2000:] for e in errs]
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import gpu_workers
    cfg = gpu_workers.ipc_cfg(fd, world, prec)
    model = fd.make_model(cfg)
    shards = fd.make_shards(cfg)
    cap = fd.expert_capacity(cfg)
    for r in range(world):
        z = np.load(outs[r])
        assert int(z["fused"]) == 0   # ranks in different processes: the combine is a separate phase
        want_g = po.gate(shards[r], model.wg, cfg.topk, cap)
        want = po.dense_forward(shards[r], model, cfg, threads=8)
        for i in range(z["outs"].shape[0]):
            assert np.array_equal(z["tabs"][i].reshape(-1), np.asarray(want_g["table_token"]).reshape(-1))
            _check_outputs(z["outs"][i], want, prec)
        assert np.array_equal(z["outs"][0].view(np.uint32), z["outs"][1].view(np.uint32))
        for s in z["stats"]:
            gemm0, gemm1, comb, executed, bound_final, sched = (int(v) for v in s)
            assert bound_final == sched == executed == gemm0 + gemm1 + comb


def test_cpp_dropin_forward_on_gpu(tmp_path):
    """include/moefabric_b200.hpp's moefabric::forward (the reference's runtime.hpp:802 entry point) as a
    compiled C++ program on the GPU: outputs and routing vs the reference's own forward()."""
    exe = str(tmp_path / "dropin")
    lib = os.path.dirname(fd._build.LIB)
    r = subprocess.run(["g++", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "dropin_forward.cpp"), "-o", exe, "-L", lib, "-lfdmoe",
                        "-Wl,-rpath," + lib], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    out = str(tmp_path / "out.bin")
    r = subprocess.run([exe, out], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "stats ok" in r.stdout
    cfg = fd.MoeConfig(tokens_per_device=512, embed_dim=256, ffn_dim=512, experts_total=8, devices=2, topk=2,
                       capacity_factor=1.0, tile_rows=16, tile_cols=8, seed=3)
    S, H, E, P = cfg.tokens_per_device, cfg.embed_dim, cfg.experts_total, cfg.devices
    cap = fd.expert_capacity(cfg)
    raw = np.fromfile(out, np.float32)
    got = raw[:P * S * H].reshape(P, S, H)
    tab = raw[P * S * H:].view(np.int32).reshape(P, E, cap)
    model = fd.make_model(cfg)
    shards = fd.make_shards(cfg)
    for d in range(P):
        want = po.dense_forward(shards[d], model, cfg, threads=8)
        _check_outputs(got[d], want)
        g = po.gate(shards[d], model.wg, cfg.topk, cap)
        assert np.array_equal(tab[d].reshape(-1), np.asarray(g["table_token"]).reshape(-1))
    if po.ref_available():   # the reference's own forward() on the same inputs
        rr = po.ref_forward(cfg, shards, po.RefModel(model, cfg))
        for d in range(P):
            _check_outputs(got[d], rr["outputs"][d])
            assert np.array_equal(tab[d].reshape(-1), rr["table_token"][d].reshape(-1).astype(np.int32))


def test_bench_torchrun_two_processes_one_gpu():
    """bench.py's multi-process path (the driver's SCALE run: one rank per process, CUDA-IPC heaps, peer stores,
    max-over-ranks timing) under torchrun with 2 ranks sharing GPU 0 (FDMOE_BENCH_SHARED_GPU: gloo bootstrap,
    since NCCL refuses two ranks on one device). Checks the bench line, not the (time-sliced) numbers."""
    port = _free_port()
    env = dict(os.environ, FDMOE_BENCH_SHARED_GPU="1", PYTHONPATH=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--tokens", "1024",
           "--experts", "8", "--steps", "3", "--warmup", "3", "--e2e-steps", "2", "--no-bulksync", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["config"]["ep"] == 2
    assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["gpu_launches_per_step"] == 1
