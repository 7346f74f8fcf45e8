"""Trace audits over a finished forward (audit.hpp:17-191), on the device event log.

The reference audits its CPU task graph; the same properties are checked here at the GPU's task
granularity (an FFN tile is 128 output features x one 128-row tile of an expert's receive region,
a combine task is a block of 16 tokens — trace.py documents the event fields):

  (a) exactly-once      executed tasks == the closed-form recount from the routing alone
                        (audit.hpp:26-82, recount over the receive layout of DESIGN.md §4)
  (b) accounting        TaskStats counters == that recount (audit.hpp:84-100)
  (c) dependency order  every (source, expert) packet's signal precedes the GEMM0 tiles reading it;
                        all GEMM0 tiles of a row tile end before any of its GEMM1 tiles starts; every
                        GEMM1 tile put into an origin precedes that origin's combine tasks
                        (audit.hpp:102-160; with the combine fused into the GEMM1 epilogues there are
                        neither puts nor combine tasks)
  (d) single launch     one launch per rank, every CTA spawned exactly once (audit.hpp:170-186)
  (e) phase gating      sequential mode only: no expert tile starts before every rank's last
                        dispatch signal, no combine starts before every rank's last GEMM1 tile
                        (runtime.hpp:885-908); barrier events appear iff sequential (audit.hpp:199-206)
Timestamps are %globaltimer, one clock per GPU: cross-rank orderings are checked for ranks that
share a device.
"""
from __future__ import annotations

import collections
import dataclasses
from typing import Dict, List, Optional, Sequence, Tuple

from .trace import TraceEvent

BM = 128          # rows per FFN row tile (fdmoe_device.cuh kBM)
BF = 128          # output features per FFN tile (kBF)
COMBINE_TOK = 16  # tokens per combine task (kCombineTok)


@dataclasses.dataclass
class Report:
    problems: List[str] = dataclasses.field(default_factory=list)

    def ok(self) -> bool:
        return not self.problems

    def fail(self, p: str):
        self.problems.append(p)


def packet_rows(capacity: int) -> int:
    """Rows reserved per (source, expert) packet in the receive buffer (fdmoe_runtime.cpp make_dims)."""
    for c in (16, 32, 64):
        if capacity <= c:
            return c
    return -(-capacity // BM) * BM


def tile_rows(cfg, gates, rank: int) -> Dict[Tuple[int, int], Tuple[int, int, int]]:
    """(local expert, row tile) -> (first source, packets, rows) for every non-empty row tile of `rank`,
    from the routing counts alone: packet (src, e) holds gates[src].slot_counts[e] rows."""
    from . import expert_capacity
    P, El = cfg.devices, cfg.local_experts()
    cp = packet_rows(expert_capacity(cfg))
    out = {}
    for le in range(El):
        e = rank * El + le
        counts = [int(gates[s].slot_counts[e]) for s in range(P)]
        if cp >= BM:
            per = cp // BM
            for src in range(P):
                for rb in range(per):
                    n = max(0, min(BM, counts[src] - rb * BM))
                    if n > 0:
                        out[(le, src * per + rb)] = (src, 1, n)
        else:
            per = BM // cp
            for m in range(-(-P // per)):
                s0, s1 = m * per, min(P, m * per + per)
                n = sum(counts[s0:s1])
                if n > 0:
                    out[(le, m)] = (s0, s1 - s0, n)
    return out


def expected_task_keys(cfg, gates, rank: int, fused_combine: bool = False) -> List[str]:
    """Canonical keys of every task `rank` must execute (the closed-form recount). With the combine
    fused into the GEMM1 epilogues there are no separate combine tasks."""
    nb0, nb1 = -(-cfg.ffn_dim // BF), -(-cfg.embed_dim // BF)
    keys = []
    for (le, m), (s0, _, _) in tile_rows(cfg, gates, rank).items():
        keys += [f"gemm0:s{s0}:e{le}:r{m}:c{c}" for c in range(nb0)]
        keys += [f"gemm1:s{s0}:e{le}:r{m}:c{c}" for c in range(nb1)]
    if not fused_combine:
        keys += [f"combine:s{rank}:e-1:r{t}:c-1" for t in range(-(-cfg.tokens_per_device // COMBINE_TOK))]
    return sorted(keys)


def _key(e: TraceEvent) -> str:
    return f"{e.task_type}:s{e.src}:e{e.expert}:r{e.rb}:c{e.cb}"


def check_exactly_once(res, cfg, rep: Report, ranks: Sequence[int], fused_combine: bool = False):
    for d in ranks:
        executed = sorted(_key(e) for e in res.trace if e.device == d and e.event == "exec")
        expected = expected_task_keys(cfg, res.gates, d, fused_combine)
        if executed != expected:
            dup = [k for k, n in collections.Counter(executed).items() if n > 1]
            rep.fail(f"device {d}: executed {len(executed)} tasks, expected {len(expected)}"
                     f" ({len(set(expected) - set(executed))} missing, {len(dup)} duplicated)")


def check_accounting(res, cfg, rep: Report, ranks: Sequence[int], fused_combine: bool = False):
    nb0, nb1 = -(-cfg.ffn_dim // BF), -(-cfg.embed_dim // BF)
    for i, d in enumerate(ranks):
        st = res.stats[i]
        tiles = len(tile_rows(cfg, res.gates, d))
        want = (tiles * nb0, tiles * nb1, 0 if fused_combine else -(-cfg.tokens_per_device // COMBINE_TOK))
        got = (st.gemm0, st.gemm1, st.combine)
        if got != want:
            rep.fail(f"device {d}: stats gemm0/gemm1/combine={got}, recount={want}")


def check_dependencies(res, cfg, rep: Report, ranks: Sequence[int], same_clock: bool = True):
    El = cfg.local_experts()
    g0_end: Dict[tuple, int] = {}
    g1_start: Dict[tuple, int] = {}
    g0_start: Dict[tuple, int] = {}
    put_last: Dict[int, int] = collections.defaultdict(int)      # origin -> last tile put
    comb_first: Dict[int, int] = {}                              # origin -> first combine start
    sig: Dict[tuple, int] = {}                                   # (owner, le, src) -> packet signal
    for e in res.trace:
        if e.event == "exec" and e.task_type == "gemm0":
            k = (e.device, e.expert, e.rb)
            g0_end[k] = max(g0_end.get(k, 0), e.t1)
            g0_start[k] = min(g0_start.get(k, 1 << 62), e.t0)
        elif e.event == "exec" and e.task_type == "gemm1":
            k = (e.device, e.expert, e.rb)
            g1_start[k] = min(g1_start.get(k, 1 << 62), e.t0)
        elif e.event == "exec" and e.task_type == "combine":
            comb_first[e.device] = min(comb_first.get(e.device, 1 << 62), e.t0)
        elif e.event == "tile_put":
            put_last[e.peer] = max(put_last[e.peer], e.t0)
        elif e.event == "dispatch_put":
            sig[(e.peer, e.expert, e.src)] = e.t0
    for k, t in g1_start.items():
        if k not in g0_end:
            rep.fail(f"gemm1 without gemm0 for block {k}")
        elif g0_end[k] > t:
            rep.fail(f"gemm0 after gemm1 start for block {k}")
    if not same_clock:
        return
    for d in ranks:
        for (le, m), (s0, ns, _) in tile_rows(cfg, res.gates, d).items():
            t = g0_start.get((d, le, m))
            if t is None:
                continue
            for src in range(s0, s0 + ns):
                s = sig.get((d, le, src))
                if s is None:
                    rep.fail(f"no dispatch signal for packet src {src} -> device {d} expert {le}")
                elif s > t:
                    rep.fail(f"gemm0 of device {d} expert {le} tile {m} started before packet {src} signalled")
        if d in comb_first and put_last.get(d, 0) > comb_first[d]:
            rep.fail(f"tile put into device {d} after its combine started")


def check_single_launch(res, rep: Report, ranks: Sequence[int], ctas_per_rank: Optional[int] = None):
    for i, d in enumerate(ranks):
        if res.stats and res.stats[i].launches != 1:
            rep.fail(f"device {d}: {res.stats[i].launches} launches")
        spawns = collections.Counter(e.worker for e in res.trace if e.device == d and e.event == "spawn")
        if any(n != 1 for n in spawns.values()):
            rep.fail(f"device {d}: a CTA spawned more than once")
        if ctas_per_rank is not None and len(spawns) != ctas_per_rank:
            rep.fail(f"device {d}: {len(spawns)} CTAs spawned, expected {ctas_per_rank}")


def barrier_event_count(res) -> int:
    """audit.hpp:195-206: barrier events appear iff the pass ran the bulk-synchronous schedule."""
    return sum(1 for e in res.trace if e.event in ("barrier_enter", "barrier_exit"))


def check_phase_gating(res, rep: Report, sequential: bool):
    nb = barrier_event_count(res)
    if not sequential:
        if nb:
            rep.fail(f"{nb} barrier events in an overlapped pass")
        return
    if nb == 0:
        rep.fail("sequential pass without barrier events")
    last_sig = max((e.t0 for e in res.trace if e.event == "dispatch_put"), default=0)
    first_gemm = min((e.t0 for e in res.trace if e.event == "exec" and e.task_type != "combine"), default=1 << 62)
    last_g1 = max((e.t1 for e in res.trace if e.event == "exec" and e.task_type == "gemm1"), default=0)
    first_comb = min((e.t0 for e in res.trace if e.event == "exec" and e.task_type == "combine"), default=1 << 62)
    if first_gemm < last_sig:
        rep.fail("sequential: an expert tile started before the last dispatch signal")
    if first_comb < last_g1:
        rep.fail("sequential: a combine started before the last GEMM1 tile finished")


def full_audit(res, cfg, sequential: bool = False, ranks: Optional[Sequence[int]] = None,
               ctas_per_rank: Optional[int] = None, same_clock: bool = True, fused_combine: bool = False) -> Report:
    """audit.hpp full_audit over a ForwardResult whose trace was recorded (ForwardOptions(trace=True)).
    fused_combine: the launch folded the combine into the GEMM1 epilogues (Operator.info()
    ["fused_combine"] and an overlapped schedule): no combine tasks, no tile puts."""
    fused_combine = fused_combine and not sequential
    ranks = list(range(cfg.devices)) if ranks is None else list(ranks)
    rep = Report()
    if not res.trace:
        rep.fail("empty trace: run the forward with ForwardOptions(trace=True)")
        return rep
    check_exactly_once(res, cfg, rep, ranks, fused_combine)
    if res.stats:
        check_accounting(res, cfg, rep, ranks, fused_combine)
    check_dependencies(res, cfg, rep, ranks, same_clock)
    check_single_launch(res, rep, ranks, ctas_per_rank)
    check_phase_gating(res, rep, sequential)
    return rep
