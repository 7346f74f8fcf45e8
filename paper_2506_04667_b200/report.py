"""Payload / memory report (harness.hpp:153-160, 199-350): P x P efficient vs padded byte matrices,
Size(L) and the Table 3 memory table, per-device task counts, worker busy fractions, as JSON / CSV.

The reference's byte matrices count FP32 rows (pgas.hpp:130-147). This operator moves the same rows,
so `bytes` / `bytes_padded` are those matrices. It also reports what the GPU path really allocates
(symmetric heap, scratch, resident weights: fdmoe_get_info) next to the reference's formulas.
"""
from __future__ import annotations

import csv
import statistics
from typing import List, Optional, Sequence

import numpy as np

from . import (ScheduleMode, expert_capacity, padded_capacity, size_L)
from .trace import busy_fractions

BM, BN = 128, 64


def remote_total(m: Sequence[int], p: int) -> int:
    """harness.hpp:153-160: off-diagonal sum of a P x P byte matrix."""
    return int(sum(int(m[i * p + j]) for i in range(p) for j in range(p) if i != j))


def bytes_matrix(m: Sequence[int], p: int) -> List[List[int]]:
    return [[int(m[i * p + j]) for j in range(p)] for i in range(p)]


def memory_json(cfg, processors: int = 4, info: Optional[dict] = None) -> dict:
    """harness.hpp:242-261 (the reference's bookkeeping formulas), plus the GPU allocation when
    `info` (Operator.info()) is given."""
    p, el, h = cfg.devices, cfg.local_experts(), cfg.embed_dim
    cap = expert_capacity(cfg)
    cp = padded_capacity(cap, cfg.tile_rows)
    row_blocks = -(-cp // cfg.tile_rows)
    cbe, cbf = -(-h // cfg.tile_cols), -(-cfg.ffn_dim // cfg.tile_cols)
    heap = p * 2 * 2 * el * cp * h * 4                      # LayoutSpec::bytes (layout.hpp:43-47)
    flags = (p * el + p * el * row_blocks * cbe) * 8
    scratch = p * el * cp * cfg.ffn_dim * 4
    qcap = p * el * row_blocks * (cbf + 2 * cbe)
    task_descriptor_bytes = 48                              # sizeof(TaskDescriptor) (runtime.hpp:62-74), x86-64 g++
    queues = qcap * (task_descriptor_bytes + 1) + processors * 16
    j = {
        "size_L_formula_bytes": size_L(cfg),
        "heap_bytes_per_device": heap,
        "flag_bytes_per_device": flags,
        "scratch_bytes_per_device": scratch,
        "queue_bytes_per_device": queues,
        "bookkeeping_bytes_per_device": flags + scratch + queues,
    }
    if info is not None:
        j["gpu"] = {"symmetric_heap_bytes": int(info["heap_bytes"]), "scratch_bytes": int(info["scratch_bytes"]),
                    "resident_weight_bytes": int(info["weight_bytes"]), "packet_rows": int(info["packet_rows"]),
                    "ctas_per_rank": int(info["ctas_per_rank"]), "smem_bytes_per_cta": int(info["smem_bytes"])}
    return j


def memory_table() -> List[dict]:
    """harness.hpp:320-338: the twelve reference configurations (H = 1024, bM = 128, FP32, cf = 1)."""
    from . import MoeConfig
    rows = []
    for tokens in (4096, 8192, 16384):
        for experts in (16, 32, 64, 128):
            cfg = MoeConfig(tokens_per_device=tokens, embed_dim=1024, ffn_dim=8, experts_total=experts, devices=1,
                            capacity_factor=1.0, tile_rows=128)
            ec = expert_capacity(cfg)
            rows.append({"tokens": tokens, "experts": experts, "capacity": ec,
                         "padded": padded_capacity(ec, 128), "size_mb": size_L(cfg) / (1024.0 * 1024.0)})
    return rows


def memory_table_text() -> str:
    """harness.hpp:340-350."""
    out = "tokens,experts,capacity,padded_capacity,size_L_mb\n"
    for r in memory_table():
        out += f"{r['tokens']},{r['experts']},{r['capacity']},{r['padded']},{r['size_mb']:.2f}\n"
    return out


def report_json(cfg, opts, pass_ns: Sequence[int], res, processors: int = 4, warmup: int = 0,
                info: Optional[dict] = None) -> dict:
    """harness.hpp:263-300 over a list of per-pass latencies and the last pass's ForwardResult."""
    p = cfg.devices
    srt = sorted(int(x) for x in pass_ns)
    j = {
        "config": {"tokens_per_device": cfg.tokens_per_device, "embed_dim": cfg.embed_dim,
                   "ffn_dim": cfg.ffn_dim, "experts_total": cfg.experts_total, "devices": p,
                   "topk": cfg.topk, "capacity_factor": cfg.capacity_factor, "tile_rows": cfg.tile_rows,
                   "tile_cols": cfg.tile_cols, "activation": ["relu", "gelu", "identity"][int(cfg.activation)]
                   if isinstance(cfg.activation, int) else str(cfg.activation), "seed": cfg.seed,
                   "processors": processors, "precision": "fp32" if int(cfg.precision) == 0 else "bf16"},
        "passes": {"warmup": warmup, "measured": len(srt)},
        "mode": ScheduleMode.sequential if opts is not None and opts.is_sequential() else ScheduleMode.overlapped,
        "latency_ns": {"mean": int(statistics.mean(srt)) if srt else 0,
                       "median": srt[len(srt) // 2] if srt else 0, "per_pass": [int(x) for x in pass_ns]},
    }
    b, bp = np.asarray(res.bytes, np.uint64), np.asarray(res.bytes_padded, np.uint64)
    j["bytes"] = {"efficient": bytes_matrix(b, p), "padded_baseline": bytes_matrix(bp, p),
                  "efficient_remote_total": remote_total(b, p), "padded_remote_total": remote_total(bp, p)}
    if remote_total(bp, p) > 0:
        j["bytes"]["remote_ratio"] = remote_total(b, p) / remote_total(bp, p)
    tasks = [{"gemm0": s.gemm0, "gemm1": s.gemm1, "combine": s.combine, "bound_final": s.bound_final,
              "scheduled": s.scheduled_final, "launches": s.launches} for s in res.stats]
    j["tasks"] = {"per_device": tasks, "total": int(sum(s.total() for s in res.stats))}
    j["workers"] = {"busy_fraction": busy_fractions(res.trace)}
    j["memory"] = memory_json(cfg, processors, info)
    return j


def write_bytes_csv(path: str, res, p: int) -> None:
    """harness.hpp:380-388."""
    with open(path, "w", newline="") as f:
        w = csv.writer(f, lineterminator="\n")
        w.writerow(["src", "dst", "efficient_bytes", "padded_bytes"])
        for i in range(p):
            for jx in range(p):
                w.writerow([i, jx, int(res.bytes[i * p + jx]), int(res.bytes_padded[i * p + jx])])
