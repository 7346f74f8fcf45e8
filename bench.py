#!/usr/bin/env python3
"""bench.py — MoE-layer forward on B200 (the FlashDMoE hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fdmoe|reference] [--precision fp32|bf16]

Workload (BASELINE.json metric "MoE layer fwd latency (ms) & tokens/s at 16K tok/128 experts, 1-8 B200"):
T = 16384 tokens per GPU, H = I = 2048, E = 128 experts in total, top-2, cf = 1.0, relu, expert-parallel
over N GPUs (E/N experts per GPU), FP32-accurate (3xTF32). Weak scaling: per-GPU token work is fixed.
Inputs are synthetic (harness.hpp:76-109 seeded generator), weights random-init.

One "step" = one full layer forward = ONE persistent kernel launch per GPU.
  value  : whole-job tokens/s with inputs resident in HBM (CUDA events on the launching stream, max over ranks)
  e2e    : same metric through the C-ABI call with host buffers (H2D of the shard + D2H of the output inside
           the timed region, host wall clock, max over ranks)
  roofline: the layer kernel against the measured tensor peak (3xTF32 effective) and HBM (weights once)
  cpu_baseline: the reference's own forward() (oracle/_ref, compiled from /root/reference) on a bounded
           token sample, all host cores, rank 0 only

Under torchrun (N > 1) each rank drives one GPU; the ranks' symmetric heaps are cross-mapped with CUDA IPC
(handles exchanged through torch.distributed) and the kernels exchange tokens with peer stores — NCCL is
used for bootstrap/barriers only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MoE layer fwd latency (ms) & tokens/s at 16K tok/128 experts, 1–8 B200"
S_PER_GPU, H, D, E_TOTAL, TOPK = 16384, 2048, 2048, 128, 2


def peaks():
    p = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback (B200_PROFILING.md)"}
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        m = json.load(open(path))
        p = {"hbm_gbs": float(m["hbm_gbs"]), "bf16_tflops": float(m["bf16_tflops"]),
             "bf16_tflops_sustained": float(m.get("bf16_tflops_sustained", m["bf16_tflops"])),
             "source": "measured (MEASURED_PEAKS.json)"}
    return p


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML while the timed region runs."""

    def __init__(self, dev_index):
        self.samples, self.reasons, self._stop = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8): "hw_slowdown",
            getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4): "sw_power_cap",
            getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80): "hw_power_brake_slowdown",
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in names.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _ref_cfg(cfg_full, tokens, seed=0):
    """A plain config record for oracle/pyoracle (the reference arm never imports the product package)."""
    from types import SimpleNamespace
    return SimpleNamespace(tokens_per_device=tokens, embed_dim=cfg_full.embed_dim, ffn_dim=cfg_full.ffn_dim,
                           experts_total=cfg_full.experts_total, devices=1, topk=cfg_full.topk,
                           capacity_factor=cfg_full.capacity_factor, tile_rows=128, tile_cols=64, activation=0,
                           seed=seed)


_REF_MODELS = {}


def _ref_runner(cfg):
    """The reference's own forward() (runtime.hpp:802) from oracle/_ref with every host core as processor
    threads, on inputs generated inside oracle/_ref by the reference harness's seeded generator
    (harness.hpp:76-109); the oracle port (C restatement, threaded) when the reference was not built."""
    from oracle import pyoracle as po
    cores = os.cpu_count() or 1
    if po.ref_available():
        key = (cfg.embed_dim, cfg.ffn_dim, cfg.experts_total, cfg.seed)
        if key not in _REF_MODELS:   # the 4.3 GB c4 model is generated once per process
            _REF_MODELS.clear()
            _REF_MODELS[key] = po.RefModel(None, cfg)
        rm = _REF_MODELS[key]
        shards = po.ref_synth_shards(cfg)
        return (lambda: po.ref_forward(cfg, shards, rm, processors=cores)), "reference", cores
    from types import SimpleNamespace
    rng = np.random.default_rng(cfg.seed)
    H, D, E = cfg.embed_dim, cfg.ffn_dim, cfg.experts_total
    f = lambda *sh: rng.standard_normal(sh, dtype=np.float32)  # noqa: E731
    model = SimpleNamespace(wg=f(H, E) / np.sqrt(H), w1=f(E, H, D) / np.sqrt(H), b1=0.1 * f(E, D),
                            w2=f(E, D, H) / np.sqrt(D), b2=0.1 * f(E, H))
    shard = f(cfg.tokens_per_device, H)
    return (lambda: po.dense_forward(shard, model, cfg, threads=cores)), "port", cores


def cpu_reference(cfg_full, sample_tokens, steps, warmup, seed=0):
    """The reference's CPU path on a token sample of the same workload (same H, I, E, k, cf; S reduced to
    the sample)."""
    cfg = _ref_cfg(cfg_full, sample_tokens, seed)
    run, kind, cores = _ref_runner(cfg)
    for _ in range(warmup):
        run()
    t0 = time.perf_counter()
    for _ in range(steps):
        run()
    dt = time.perf_counter() - t0
    return {"value": sample_tokens * steps / dt, "unit": "tokens/s", "cores": cores, "kind": kind,
            "sample": f"{sample_tokens} tokens x {steps} forward() calls of the same layer shape "
                      f"(H={cfg.embed_dim}, I={cfg.ffn_dim}, E={cfg.experts_total}, top-{cfg.topk}, cf=1, P=1)",
            "sample_tokens": sample_tokens, "ms_per_step": dt * 1e3 / steps}


def calibrate_sample(cfg_full, budget_s):
    """Token sample size whose reference forward() takes about budget_s seconds on this host."""
    probe = 256
    run, _, _ = _ref_runner(_ref_cfg(cfg_full, probe))
    t0 = time.perf_counter()
    run()
    dt = time.perf_counter() - t0
    n = int(probe * budget_s / max(dt, 1e-3))
    return max(128, min(S_PER_GPU, (n // 128) * 128))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="fdmoe", choices=["fdmoe", "reference"])
    ap.add_argument("--precision", default="fp32", choices=["fp32", "bf16"])
    ap.add_argument("--tokens", type=int, default=S_PER_GPU)
    ap.add_argument("--experts", type=int, default=E_TOTAL)
    ap.add_argument("--e2e-steps", type=int, default=12)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-bulksync", action="store_true")
    args = ap.parse_args()
    assert args.warmup >= 3, "timing rules: at least 3 warm-up steps"

    rank, world, local = dist_env()
    if world != args.gpus and world > 1:
        print(f"warning: WORLD_SIZE={world} != --gpus {args.gpus}; using WORLD_SIZE", file=sys.stderr)
    n = world if world > 1 else args.gpus

    from types import SimpleNamespace
    prec_fp32 = args.precision == "fp32"
    shape = SimpleNamespace(tokens_per_device=args.tokens, embed_dim=H, ffn_dim=D, experts_total=args.experts,
                            topk=TOPK, capacity_factor=1.0)
    workload = (f"c4-shape: T={shape.tokens_per_device} tokens/GPU, H={H}, I={D}, E={shape.experts_total} total "
                f"({shape.experts_total // n}/GPU), top-{TOPK}, cf=1.0, relu, EP={n}, "
                f"{'FP32-accurate 3xTF32' if prec_fp32 else 'bf16'}")
    config = {"workload": workload, "tokens_per_gpu": shape.tokens_per_device, "embed_dim": H, "ffn_dim": D,
              "experts_total": shape.experts_total, "topk": TOPK, "ep": n,
              "l2": "no flush: per-step inputs (134 MB shard + resident expert weights) exceed the 126 MB L2"}

    # ---------------------------------------------------------------- reference arm
    # The reference's own CPU forward() from oracle/_ref only: this branch never imports the product
    # package (inputs come from the reference harness's generator inside oracle/_ref).
    if args.impl == "reference":
        if rank != 0:
            return
        budget = max(2.0, 150.0 / (args.steps + args.warmup))
        sample = calibrate_sample(shape, budget)
        cb = cpu_reference(shape, sample, args.steps, args.warmup)
        ref_config = dict(config, sample_tokens=sample,
                          sample_note=f"each step is the reference forward() on a {sample}-token sample of this "
                                      f"workload (same H, I, E, k, cf); tokens/s = sample tokens / step time")
        line = {"metric": METRIC, "value": cb["value"], "unit": "tokens/s", "n_gpus": 0, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": cb["ms_per_step"], "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": ref_config,
                "impl": "reference",
                "cpu_baseline": {"value": cb["value"], "unit": "tokens/s", "cores": cb["cores"], "kind": cb["kind"],
                                 "sample": cb["sample"]},
                "e2e": {"value": cb["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    # ---------------------------------------------------------------- our arm
    import paper_2506_04667_b200 as fd
    prec = fd.Precision.fp32 if prec_fp32 else fd.Precision.bf16
    cfg = fd.MoeConfig(tokens_per_device=args.tokens, embed_dim=H, ffn_dim=D, experts_total=args.experts,
                       devices=n, topk=TOPK, capacity_factor=1.0, tile_rows=128, tile_cols=64, seed=0,
                       precision=prec)
    import torch
    import torch.distributed as dist
    # FDMOE_BENCH_SHARED_GPU=1 (tests only): every rank on GPU 0 and gloo for the bootstrap, so the multi-process
    # path of this script (CUDA-IPC heaps, cross-process peer stores) runs on a single-GPU box. NCCL refuses two
    # ranks on one device; the contexts time-slice the GPU, so its timings mean nothing.
    shared_gpu = world > 1 and os.environ.get("FDMOE_BENCH_SHARED_GPU") == "1"
    if shared_gpu:
        local = 0
    red_dev = "cpu" if shared_gpu else "cuda"
    torch.cuda.set_device(local)
    if world > 1:
        if shared_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    t_setup = time.perf_counter()
    model = fd.make_model(cfg)
    shards_all = fd.make_shards(cfg)
    if world > 1:
        from paper_2506_04667_b200 import dist as fdist
        op = fd.Operator(cfg, device_ids=[local], first_rank=rank, n_local=1)
        fdist.attach_peers(op)   # bootstrap only: CUDA-IPC heap handles, rank-major
        my = [shards_all[rank]]
    else:
        op = fd.Operator(cfg, device_ids=[0] * n)   # n == 1 here (or virtual ranks if --gpus > 1 w/o torchrun)
        my = shards_all
    op.set_weights(model)
    info = op.info()
    bulk = None
    if not args.no_bulksync:
        from paper_2506_04667_b200.bulksync import BulkSyncMoE
        bulk = BulkSyncMoE(cfg, model, rank=rank if world > 1 else 0, world=world if world > 1 else 1)
    del model
    setup_s = time.perf_counter() - t_setup

    # a dedicated (non-default) stream: the layer kernel is launched on it and the CUDA events that
    # time it are recorded on it (the legacy default stream would not order with the launch)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    assert stream.cuda_stream != 0
    ins = [torch.from_numpy(s).cuda() for s in my]
    outs = [torch.empty_like(x) for x in ins]
    ip = [x.data_ptr() for x in ins]
    opp = [x.data_ptr() for x in outs]
    sp = [stream.cuda_stream] * len(ins)

    for _ in range(args.warmup):
        op.forward_device(ip, opp, sp)
    op.sync()
    torch.cuda.synchronize()
    barrier()

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            op.forward_device(ip, opp, sp)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    op.sync()
    ms = ev0.elapsed_time(ev1) / args.steps
    # in-kernel SM clock of the last timed launch: per-CTA clock64 / %globaltimer deltas (device trace
    # points kTrClk*; NVML's SM-clock reading does not show the power-cap throttling inside a launch)
    kclk = None
    try:
        tr = op.trace(0).astype(np.float64)
        f_launch = (tr[:, 35] - tr[:, 32]) / np.maximum(tr[:, 6] - tr[:, 0], 1.0) * 1e3
        f_ffn = (tr[:, 34] - tr[:, 33]) / np.maximum(tr[:, 4] - tr[:, 3], 1.0) * 1e3
        kclk = {"launch_mhz": round(float(np.median(f_launch)), 1), "ffn_mhz": round(float(np.median(f_ffn)), 1),
                "source": "median over CTAs of clock64 / %globaltimer deltas, last timed launch (device trace)"}
    except Exception as ex:  # noqa: BLE001
        kclk = {"unavailable": str(ex)}
    if world > 1:
        ms = fdist.max_over_ranks(ms, device=red_dev)
    tokens_per_step = cfg.tokens_per_device * n
    value = tokens_per_step / (ms * 1e-3)
    # cross-check: the operator's own events around its launches (same stream)
    st_ms = op.last_kernel_ms()

    # ---------------------------------------------------------------- bulk-synchronous schedule (same launch)
    # ScheduleMode::sequential (runtime.hpp:885-908): group barriers after dispatch and after the FFN;
    # the paper's overlapped-vs-sequential comparison (Table 2) on this configuration
    seq_steps = 3
    seq_opts = fd.ForwardOptions(mode=fd.ScheduleMode.sequential)
    for _ in range(2):
        op.forward_device(ip, opp, sp, opts=seq_opts)
    op.sync()
    barrier()
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(seq_steps):
        op.forward_device(ip, opp, sp, opts=seq_opts)
    ev1.record(stream)
    torch.cuda.synchronize()
    op.sync()
    seq_ms = ev0.elapsed_time(ev1) / seq_steps
    if world > 1:
        seq_ms = fdist.max_over_ranks(seq_ms, device=red_dev)

    # ---------------------------------------------------------------- bulk-synchronous NCCL baseline (§8 f1)
    # separate library kernels + NCCL all_to_all_single for dispatch and combine (bulksync.py): the
    # conventional schedule the single fused launch replaces (runtime.hpp:885-908)
    bulk_ms = None
    if bulk is not None and n == (world if world > 1 else 1):
        xin = ins[0]
        for _ in range(2):
            bulk.forward(xin)
        torch.cuda.synchronize()
        barrier()
        ev0.record(stream)
        for _ in range(seq_steps):
            bulk.forward(xin)
        ev1.record(stream)
        torch.cuda.synchronize()
        bulk_ms = ev0.elapsed_time(ev1) / seq_steps
        if world > 1:
            bulk_ms = fdist.max_over_ranks(bulk_ms, device=red_dev)
        del bulk
        torch.cuda.empty_cache()

    # ---------------------------------------------------------------- end to end through the C ABI (host buffers)
    pinned = [torch.from_numpy(s).pin_memory() for s in my]
    host_in = [p.numpy() for p in pinned]
    outs_h = [torch.empty(s.shape, dtype=torch.float32).pin_memory().numpy() for s in my]
    outs_h2 = [torch.empty(s.shape, dtype=torch.float32).pin_memory().numpy() for s in my]
    # (a) the serving loop (fdmoe_forward_stream): every step copies its shard in, runs the layer and
    #     copies the output back; neighbouring steps' PCIe copies overlap the launch
    batches = [host_in] * args.e2e_steps
    bouts = [outs_h if b % 2 == 0 else outs_h2 for b in range(args.e2e_steps)]
    op.forward_stream(batches[:2], bouts[:2])   # warm
    barrier()
    t0 = time.perf_counter()
    op.forward_stream(batches, bouts)
    e2e_s = (time.perf_counter() - t0) / args.e2e_steps
    # (b) one synchronous fdmoe_forward per step (copy in, launch, copy out back to back)
    op.forward(host_in, routing=False, stats=False)   # warm
    t0 = time.perf_counter()
    for _ in range(3):
        _forward_host(fd, op, host_in, outs_h)
    sync_s = (time.perf_counter() - t0) / 3
    if world > 1:
        e2e_s = fdist.max_over_ranks(e2e_s, device=red_dev)
        sync_s = fdist.max_over_ranks(sync_s, device=red_dev)
    e2e = {"value": tokens_per_step / e2e_s, "unit": "tokens/s",
           "h2d_bytes_per_step": int(sum(x.nbytes for x in host_in)),
           "d2h_bytes_per_step": int(sum(x.nbytes for x in outs_h)), "ms_per_step": e2e_s * 1e3,
           "api": f"fdmoe_forward_stream over {args.e2e_steps} steps (pinned host shards; H2D, launch, D2H "
                  f"per step on three streams)",
           "sync_api_ms_per_step": sync_s * 1e3,
           "sync_api_value": tokens_per_step / sync_s}

    # ---------------------------------------------------------------- roofline of the (single) layer kernel
    pk = peaks()
    El = cfg.experts_total // n
    rows = cfg.tokens_per_device   # rows received per GPU (every (src, expert) packet fills to C)
    gate_flops = 2.0 * cfg.tokens_per_device * H * cfg.experts_total
    ffn_flops = 4.0 * H * D * rows
    flops = gate_flops + ffn_flops
    weight_bytes = El * 2.0 * H * D * 4   # FP32 weights read once (algorithmic)
    # The timed region is a loop of back-to-back launches that runs at the 1 kW power cap (in-kernel SM clock
    # ~1.4-1.5 GHz in the FFN, `clocks.in_kernel`), so the tensor peak is the driver's SUSTAINED cuBLAS figure
    # (measured at ~1.34 GHz under the same cap; B200_PROFILING.md: "the sustained one for a kernel timed inside
    # a long step"); the burst-peak fraction is reported beside it.
    sus = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
    if prec == fd.Precision.fp32:
        tensor_peak = sus / 2.0 / 3.0   # tf32 = bf16/2; FP32-accurate = 3 tf32 products
        tensor_burst = pk["bf16_tflops"] / 2.0 / 3.0
        peak_note = (f"3xTF32 effective = measured bf16 sustained {sus:.1f} / 2 (tf32 rate) / 3 (products); burst "
                     f"{pk['bf16_tflops']:.1f} / 6 = {tensor_burst:.1f} in peak_burst; {pk['source']}")
    else:
        tensor_peak, tensor_burst = sus, pk["bf16_tflops"]
        weight_bytes /= 2
        peak_note = f"bf16 sustained {sus:.1f} (burst {pk['bf16_tflops']:.1f}); HBM copy {pk['hbm_gbs']:.1f}; {pk['source']}"
    t_tensor = flops / (tensor_peak * 1e12)
    t_hbm = weight_bytes / (pk["hbm_gbs"] * 1e9)
    bound = "tensor" if t_tensor >= t_hbm else "hbm"
    achieved_tf = flops / (ms * 1e-3) / 1e12
    achieved_gbs = weight_bytes / (ms * 1e-3) / 1e9
    if bound == "tensor":
        roof = {"bound": "tensor", "achieved": achieved_tf, "peak": tensor_peak, "unit": "TFLOP/s",
                "frac": achieved_tf / tensor_peak, "peak_burst": tensor_burst, "frac_burst": achieved_tf / tensor_burst}
        if prec == fd.Precision.fp32:
            # the FFN's own arithmetic (tf32 main + bf16 corrections) needs 2 tf32 + 2 bf16 MMA
            # slots per 16 k = 4 bf16-equivalent slots, i.e. a tensor ceiling of bf16 / 4 (the gate stays 3xTF32)
            scheme_peak = sus / 4.0
            roof.update({"peak_scheme": scheme_peak, "frac_scheme": achieved_tf / scheme_peak,
                         "scheme_note": "frac = against 3xTF32 (the north-star FP32-accurate mode); frac_scheme = against "
                                        "the tensor ceiling of the kernel's tf32-main + bf16-correction products"})
    else:
        roof = {"bound": "hbm", "achieved": achieved_gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved_gbs / pk["hbm_gbs"]}
    roof.update({"traffic": None, "peak_note": peak_note,
                 "algorithmic": {"flops_per_launch": flops, "gate_flops": gate_flops, "ffn_flops": ffn_flops,
                                 "weight_bytes_per_launch": weight_bytes},
                 "t_tensor_ms": t_tensor * 1e3, "t_hbm_ms": t_hbm * 1e3,
                 "roofline_ms": max(t_tensor, t_hbm) * 1e3,
                 "frac_of_roofline": max(t_tensor, t_hbm) / (ms * 1e-3),
                 "kernel": "fdmoe_layer_kernel (1 launch/GPU/step)"})
    traffic_file = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(traffic_file):
        tr = json.load(open(traffic_file)).get(f"{args.precision}_n{n}")
        if tr:
            roof["traffic"] = tr

    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": n, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 (3xTF32 tcgen05)" if prec == 0 else "bf16",
            "data": "synthetic (seeded harness.hpp generator), random-init experts", "config": config,
            "e2e": e2e, "gpu_launches": args.steps, "gpu_launches_per_step": 1, "roofline": roof,
            "clocks": dict(clk.summary(), in_kernel=kclk), "setup_s": setup_s, "operator_event_ms_last_launch": st_ms,
            "operator": {k: info[k] for k in ("capacity", "packet_rows", "ctas_per_rank", "smem_bytes")},
            "schedules": {"overlapped_ms": ms, "sequential_ms": seq_ms, "sequential_over_overlapped": seq_ms / ms,
                          "sequential_nccl_ms": bulk_ms,
                          "sequential_nccl_over_overlapped": (bulk_ms / ms) if bulk_ms else None,
                          "note": "sequential = ScheduleMode::sequential in the same single launch (group "
                                  "barriers after dispatch and after the FFN); sequential_nccl = bulk-synchronous "
                                  "separate kernels (cuBLAS FP32 SGEMM, TF32 off) + NCCL all_to_all_single for "
                                  "dispatch and combine (bulksync.py); neither is a timed step of `value`"}}
    if rank == 0 and not args.no_cpu_baseline:
        try:
            budget = 15.0
            sample = calibrate_sample(shape, budget)
            cb = cpu_reference(shape, sample, 1, 0)
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "sample_tokens")}
        except Exception as e:  # never let the baseline break the bench line
            line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    if rank == 0:
        print(json.dumps(line))
    op.close()
    if world > 1:
        dist.destroy_process_group()


def _forward_host(fd, op, host_in, outs_h):
    """fdmoe_forward with FDMOE_HOST pointers: H2D shard, the layer launch, D2H output."""
    import ctypes as C
    n = op.n_local
    ip = (C.c_void_p * n)(*[a.ctypes.data for a in host_in])
    opp = (C.c_void_p * n)(*[a.ctypes.data for a in outs_h])
    fd._check(fd.lib().fdmoe_forward(op._h, ip, opp, 0, None, None, None))


if __name__ == "__main__":
    main()
