"""Device event log → the reference's TraceEvent stream (trace.hpp:17-118, harness.hpp:352-378).

The kernel records one `fdmoe_event` per event (include/fdmoe.h) with %globaltimer nanoseconds when
ForwardOptions(trace=True); `Operator.events()` returns them as a structured array of EVENT_DTYPE.
This module turns the per-rank arrays into `TraceEvent`s, sorted by start time and relative to the
earliest event of the launch (the reference's "ns since pass epoch"), and writes them as JSONL.

GPU meaning of the fields (the reference's CPU worker threads are CTAs here):
  worker   "cta<N>" — the CTA of that rank that emitted the event
  exec     gemm0 / gemm1: one 128-feature x 128-row FFN tile (expert = local expert, rb = row tile of
           the expert's receive region, cb = 128-wide feature block, src = first source packet in the
           tile, peer = packets in the tile, value = rows); t0 = dependencies resolved and operand
           streaming started, t1 = epilogue stored (gemm0: before the row-tile counter release)
           combine: one block of 16 tokens (rb = token block)
  tile_put GEMM1 tile stored into origin `peer`'s combine buffer, just before its release signal
  dispatch_put  a (source, expert) packet's release signal (value = rows; zero-row packets too)
"""
from __future__ import annotations

import dataclasses
import json
from typing import Dict, Iterable, List, Sequence

import numpy as np

EVENT_DTYPE = np.dtype([("t0", "<u8"), ("t1", "<u8"), ("kind", "<i4"), ("cta", "<i4"), ("type", "<i4"),
                        ("src", "<i4"), ("expert", "<i4"), ("rb", "<i4"), ("cb", "<i4"), ("peer", "<i4"),
                        ("value", "<i8")])
assert EVENT_DTYPE.itemsize == 56

EVENT_NAMES = ["spawn", "gate_done", "dispatch_put", "exec", "tile_put", "barrier_enter", "barrier_exit"]
TASK_NAMES = {1: "gemm0", 2: "gemm1", 3: "combine"}


@dataclasses.dataclass
class TraceEvent:
    """trace.hpp:38-60."""
    t0: int = 0
    t1: int = 0
    device: int = -1
    worker: str = ""
    event: str = ""
    task_type: str = None
    src: int = -1
    expert: int = -1
    rb: int = -1
    cb: int = -1
    value: int = -1
    peer: int = -1

    def has_task(self) -> bool:
        return self.task_type is not None


def task_key(e: TraceEvent) -> str:
    """trace.hpp:62-68: stable task identity, independent of timing."""
    return f"{e.task_type or '-'}:s{e.src}:e{e.expert}:r{e.rb}:c{e.cb}"


def to_trace_events(per_rank: Sequence[np.ndarray], first_rank: int = 0) -> List[TraceEvent]:
    """Merge per-rank event arrays (merge_traces, trace.hpp:105-116)."""
    out: List[TraceEvent] = []
    base = min((int(a["t0"].min()) for a in per_rank if len(a)), default=0)
    for i, arr in enumerate(per_rank):
        dev = first_rank + i
        for r in arr:
            kind = int(r["kind"])
            t1 = int(r["t1"])
            out.append(TraceEvent(
                t0=int(r["t0"]) - base, t1=(t1 - base) if t1 else 0, device=dev, worker=f"cta{int(r['cta'])}",
                event=EVENT_NAMES[kind] if 0 <= kind < len(EVENT_NAMES) else "unknown",
                task_type=TASK_NAMES.get(int(r["type"])) if kind == 3 else None,
                src=int(r["src"]), expert=int(r["expert"]), rb=int(r["rb"]), cb=int(r["cb"]),
                value=int(r["value"]), peer=int(r["peer"])))
    out.sort(key=lambda e: e.t0)   # stable
    return out


def event_json(e: TraceEvent) -> dict:
    """harness.hpp:352-371."""
    j = {"time": e.t0}
    if e.t1:
        j["end"] = e.t1
    j.update(device=e.device, worker=e.worker, event=e.event)
    if e.has_task():
        j["type"] = e.task_type
        j["task"] = task_key(e)
    for k in ("src", "expert", "rb", "cb", "value", "peer"):
        v = getattr(e, k)
        if v >= 0:
            j[k] = v
    return j


def write_trace_jsonl(path: str, trace: Iterable[TraceEvent]) -> None:
    """harness.hpp:373-378."""
    with open(path, "w") as f:
        for e in trace:
            f.write(json.dumps(event_json(e)) + "\n")


def busy_fractions(trace: Iterable[TraceEvent]) -> Dict[str, float]:
    """harness.hpp busy_fractions_json: per worker, executed-task time over its lifetime. A CTA's
    FFN tiles are pipelined (the next tile's operands stream while the previous epilogue drains), so
    busy time is the union of its exec intervals."""
    life: Dict[str, tuple] = {}
    spans: Dict[str, list] = {}
    for e in trace:
        key = f"dev{e.device}.{e.worker}"
        if e.event == "spawn":
            life[key] = (e.t0, e.t1)
        elif e.event == "exec":
            spans.setdefault(key, []).append((e.t0, e.t1))
    out = {}
    for key, (a, b) in sorted(life.items()):
        busy, end = 0, -1
        for s, t in sorted(spans.get(key, [])):
            s = max(s, end)
            if t > s:
                busy += t - s
                end = t
        out[key] = busy / (b - a) if b > a else 0.0
    return out
