"""Multi-process plumbing for one-rank-per-GPU runs (torch.distributed: NCCL on GPUs, gloo on CPU).

Bootstrap only — the data path (dispatch and combine) never touches torch.distributed; it is the
layer kernel's peer stores into the symmetric heaps these helpers attach:

* ``attach_peers(op)``: all-gather every rank's CUDA-IPC heap blob (rank-major) and import them —
  the role of the reference's shared fabric construction (pgas.hpp:56-97, runtime.hpp:837-848).
* ``max_over_ranks(x)``: the latency reduce (max over GPUs).
* ``gather_payload(cfg, slot_counts)``: the reference's ``ForwardResult::bytes`` P x P matrix
  (pgas.hpp:130-135) from every rank's own routing counts.
* ``rank_experts(cfg, rank)``: the contiguous expert block a rank owns (config.hpp:66).
"""
from typing import List, Optional, Sequence

import numpy as np


def _dist():
    import torch.distributed as dist
    if not dist.is_initialized():
        raise RuntimeError("torch.distributed is not initialised (init_process_group first)")
    return dist


def exchange_blobs(blob: bytes, group=None) -> List[bytes]:
    """All-gather one opaque blob per rank; returns them in rank order (all equal length)."""
    dist = _dist()
    out: List[Optional[bytes]] = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(blob), group=group)
    if any(b is None or len(b) != len(blob) for b in out):
        raise RuntimeError("heap blobs differ in size across ranks (library version mismatch?)")
    return out  # type: ignore[return-value]


def attach_peers(op, group=None) -> None:
    """Make every rank's symmetric heap addressable from this rank's kernel."""
    op.import_peers(exchange_blobs(op.export_heap(), group))


def max_over_ranks(x: float, group=None, device=None) -> float:
    import torch
    dist = _dist()
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def gather_slot_counts(counts: np.ndarray, group=None) -> List[np.ndarray]:
    dist = _dist()
    out: List[Optional[np.ndarray]] = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, np.asarray(counts, np.int64), group=group)
    return out  # type: ignore[return-value]


def gather_payload(cfg, counts: np.ndarray, group=None) -> np.ndarray:
    """bytes[p * P + q] exactly as the single-process operator reports it."""
    from . import payload_bytes
    return payload_bytes(cfg, gather_slot_counts(counts, group))


def rank_experts(cfg, rank: int) -> range:
    el = cfg.experts_total // cfg.devices
    return range(rank * el, (rank + 1) * el)


def rank_shards(cfg, ranks: Sequence[int]) -> List[np.ndarray]:
    """The seeded shards (harness.hpp:99-109) of the given ranks."""
    from . import make_shards
    allsh = make_shards(cfg)
    return [allsh[r] for r in ranks]
