"""ctypes bindings for the CPU checkers (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
may import this module. It wraps
  * oracle/liboracle.so              — the C restatement (oracle/moe_oracle.c), and
  * oracle/_ref/libmoefabric_ref.so  — the reference's own headers behind a C shim,
built by oracle/Makefile. The product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmoefabric_ref.so")

_orc = None
_ref = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def orc():
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        i64, vp, f32, u32, u64 = C.c_int64, C.c_void_p, C.c_float, C.c_uint32, C.c_uint64
        L.orc_expert_capacity.restype = i64
        L.orc_expert_capacity.argtypes = [i64, i64, C.c_double]
        L.orc_padded_capacity.restype = i64
        L.orc_padded_capacity.argtypes = [i64, i64]
        L.orc_size_L.restype = u64
        L.orc_size_L.argtypes = [i64, i64, i64, i64]
        L.orc_activation.restype = f32
        L.orc_activation.argtypes = [C.c_int, f32]
        L.orc_expf_restated.restype = f32
        L.orc_expf_restated.argtypes = [f32]
        L.orc_expf_libm.restype = f32
        L.orc_expf_libm.argtypes = [f32]
        L.orc_expf_libm_batch.restype = None
        L.orc_expf_libm_batch.argtypes = [vp, vp, i64]
        L.orc_expf_sweep.restype = u64
        L.orc_expf_sweep.argtypes = [u32, u32]
        L.orc_gate.restype = None
        L.orc_gate.argtypes = [vp, vp, i64, i64, i64, i64, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.orc_dense_forward.restype = None
        L.orc_dense_forward.argtypes = [vp, vp, vp, vp, vp, vp, i64, i64, i64, i64, i64, i64, C.c_int, vp, C.c_int]
        L.orc_ffn_rows.restype = None
        L.orc_ffn_rows.argtypes = [vp, vp, vp, vp, vp, i64, i64, i64, C.c_int, vp, vp, vp, vp, i64, vp, C.c_int]
        L.orc_naive_matmul.restype = None
        L.orc_naive_matmul.argtypes = [vp, vp, i64, i64, i64, vp]
        _orc = L
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO + " (build with `make -C oracle` where /root/reference exists)")
        L = C.CDLL(REF_SO)
        i64, vp, i32 = C.c_int64, C.c_void_p, C.c_int
        L.ref_last_error.restype = C.c_char_p
        L.ref_model_create.restype = vp
        L.ref_model_create.argtypes = [i64, i64, i64, vp, vp, vp, vp, vp]
        L.ref_model_destroy.argtypes = [vp]
        L.ref_model_synth.restype = vp
        L.ref_model_synth.argtypes = [vp, C.c_double, C.c_uint64]
        L.ref_synth_shards.restype = None
        L.ref_synth_shards.argtypes = [vp, C.c_double, C.c_uint64, vp]
        L.ref_forward.restype = i32
        L.ref_forward.argtypes = [vp, C.c_double, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.ref_dense_forward.restype = i32
        L.ref_dense_forward.argtypes = [vp, C.c_double, vp, vp, vp]
        L.ref_gate.restype = i32
        L.ref_gate.argtypes = [vp, C.c_double, i64, vp, vp, vp, vp, vp, vp, vp, vp]
        L.ref_expert_capacity.restype = i64
        L.ref_expert_capacity.argtypes = [vp, C.c_double]
        L.ref_straggler_delays.restype = i32
        L.ref_straggler_delays.argtypes = [i32, C.c_double, C.c_double, i32, C.c_uint64, i64, i64, vp]
        _ref = L
    return _ref


def _cfgv(cfg):
    return np.array([cfg.tokens_per_device, cfg.embed_dim, cfg.ffn_dim, cfg.experts_total, cfg.devices,
                     cfg.topk, cfg.tile_rows, cfg.tile_cols, int(cfg.activation)], np.int64)


# ------------------------------------------------------------------ C restatement
def gate(a, wg, k, cap):
    """orc_gate: returns dict(g_phi, table_token (E x max(cap,1)), table_weight, slot_counts,
    dropped [(tok, e)], picks_expert, picks_weight, picks_slot)."""
    a = np.ascontiguousarray(a, np.float32)
    wg = np.ascontiguousarray(wg, np.float32)
    S, H = a.shape
    E = wg.shape[1]
    ca = max(cap, 1)
    out = dict(g_phi=np.empty((S, E), np.float32), table_token=np.empty((E, ca), np.int64),
               table_weight=np.empty((E, ca), np.float32), slot_counts=np.empty(E, np.int64),
               picks_expert=np.empty((S, k), np.int32), picks_weight=np.empty((S, k), np.float32),
               picks_slot=np.empty((S, k), np.int32))
    dropped = np.empty(2 * S * k, np.int64)
    nd = np.zeros(1, np.int64)
    orc().orc_gate(_p(a), _p(wg), S, H, E, k, cap, _p(out["g_phi"]), _p(out["table_token"]),
                   _p(out["table_weight"]), _p(out["slot_counts"]), _p(dropped), _p(nd), _p(out["picks_expert"]),
                   _p(out["picks_weight"]), _p(out["picks_slot"]))
    out["dropped"] = [(int(dropped[2 * i]), int(dropped[2 * i + 1])) for i in range(int(nd[0]))]
    return out


def dense_forward(a, model, cfg, cap: Optional[int] = None, threads: int = 1):
    """orc_dense_forward on one shard."""
    a = np.ascontiguousarray(a, np.float32)
    S, H = a.shape
    if cap is None:
        cap = int(orc().orc_expert_capacity(cfg.tokens_per_device, cfg.experts_total, cfg.capacity_factor))
    out = np.empty((S, H), np.float32)
    orc().orc_dense_forward(_p(a), _p(model.wg), _p(model.w1), _p(model.b1), _p(model.w2), _p(model.b2), S, H,
                            cfg.ffn_dim, cfg.experts_total, cfg.topk, cap, int(cfg.activation), _p(out), threads)
    return out


def ffn_rows(a, model, cfg, routing, rows, threads: int = 1):
    """orc_ffn_rows: output rows of the given token ids, from orc_gate routing (dict from gate())."""
    a = np.ascontiguousarray(a, np.float32)
    rows = np.ascontiguousarray(rows, np.int64)
    out = np.empty((rows.size, a.shape[1]), np.float32)
    pe = np.ascontiguousarray(routing["picks_expert"], np.int32)
    ps = np.ascontiguousarray(routing["picks_slot"], np.int32)
    pw = np.ascontiguousarray(routing["picks_weight"], np.float32)
    orc().orc_ffn_rows(_p(a), _p(model.w1), _p(model.b1), _p(model.w2), _p(model.b2), a.shape[1], cfg.ffn_dim,
                       cfg.topk, int(cfg.activation), _p(pe), _p(ps), _p(pw), _p(rows), rows.size, _p(out),
                       threads)
    return out


def expf_libm(x):
    x = np.ascontiguousarray(x, np.float32)
    y = np.empty_like(x)
    orc().orc_expf_libm_batch(_p(x), _p(y), x.size)
    return y


# ------------------------------------------------------------------ the reference itself
class RefModel:
    def __init__(self, model, cfg, seed: Optional[int] = None):
        """model=None: the reference harness's seeded model built inside the shim (harness.hpp:76-97)."""
        self.cfg = cfg
        if model is None:
            self._h = ref().ref_model_synth(_p(_cfgv(cfg)), cfg.capacity_factor, cfg.seed if seed is None else seed)
        else:
            self._h = ref().ref_model_create(cfg.embed_dim, cfg.ffn_dim, cfg.experts_total, _p(model.wg),
                                             _p(model.w1), _p(model.b1), _p(model.w2), _p(model.b2))

    def __del__(self):
        try:
            ref().ref_model_destroy(self._h)
        except Exception:
            pass


def ref_synth_shards(cfg, seed: Optional[int] = None):
    """harness.hpp:99-109 shards (P x S x H) from the shim."""
    out = np.empty((cfg.devices, cfg.tokens_per_device, cfg.embed_dim), np.float32)
    ref().ref_synth_shards(_p(_cfgv(cfg)), cfg.capacity_factor, cfg.seed if seed is None else seed, _p(out))
    return [out[d] for d in range(cfg.devices)]


def ref_forward(cfg, shards, refmodel: RefModel, processors: int = 4, sequential: bool = False):
    """moefabric::forward (runtime.hpp:802) on the given shards. Returns dict."""
    P, S, H, E = cfg.devices, cfg.tokens_per_device, cfg.embed_dim, cfg.experts_total
    cap = int(ref().ref_expert_capacity(_p(_cfgv(cfg)), cfg.capacity_factor))
    a = np.ascontiguousarray(np.stack(shards), np.float32)
    out = np.empty((P, S, H), np.float32)
    tt = np.empty((P, E, cap), np.int64)
    tw = np.empty((P, E, cap), np.float32)
    sc = np.empty((P, E), np.int64)
    gp = np.empty((P, S, E), np.float32)
    by = np.empty(P * P, np.uint64)
    bp = np.empty(P * P, np.uint64)
    stt = np.empty((P, 9), np.int64)
    mk = np.zeros(1, np.uint64)
    cfgv = _cfgv(cfg)
    rc = ref().ref_forward(_p(cfgv), cfg.capacity_factor, processors, 1 if sequential else 0, refmodel._h, _p(a),
                           _p(out), _p(tt), _p(tw), _p(sc), _p(gp), _p(by), _p(bp), _p(stt), _p(mk))
    if rc != 0:
        raise RuntimeError(f"reference forward failed ({rc}): {ref().ref_last_error().decode()}")
    return dict(outputs=out, table_token=tt, table_weight=tw, slot_counts=sc, g_phi=gp, bytes=by,
                bytes_padded=bp, stats=stt, makespan_ns=int(mk[0]))


def ref_dense_forward(cfg, shard, refmodel: RefModel):
    out = np.empty((cfg.tokens_per_device, cfg.embed_dim), np.float32)
    a = np.ascontiguousarray(shard, np.float32)
    rc = ref().ref_dense_forward(_p(_cfgv(cfg)), cfg.capacity_factor, refmodel._h, _p(a), _p(out))
    if rc != 0:
        raise RuntimeError(ref().ref_last_error().decode())
    return out


def ref_gate(cfg, a, wg, cap: int = -1):
    S, E = cfg.tokens_per_device, cfg.experts_total
    c = int(ref().ref_expert_capacity(_p(_cfgv(cfg)), cfg.capacity_factor)) if cap < 0 else cap
    ca = max(c, 1)
    g = np.empty((S, E), np.float32)
    tt = np.empty((E, ca), np.int64)
    tw = np.empty((E, ca), np.float32)
    sc = np.empty(E, np.int64)
    dr = np.empty(2 * S * cfg.topk, np.int64)
    nd = np.zeros(1, np.int64)
    a = np.ascontiguousarray(a, np.float32)
    wg = np.ascontiguousarray(wg, np.float32)
    rc = ref().ref_gate(_p(_cfgv(cfg)), cfg.capacity_factor, cap, _p(a), _p(wg), _p(g), _p(tt), _p(tw), _p(sc),
                        _p(dr), _p(nd))
    if rc != 0:
        raise RuntimeError(ref().ref_last_error().decode())
    return dict(g_phi=g, table_token=tt, table_weight=tw, slot_counts=sc,
                dropped=[(int(dr[2 * i]), int(dr[2 * i + 1])) for i in range(int(nd[0]))])


def ref_straggler_delays(kind: int, a: float, b: float, device: int, seed: int, devices: int,
                         local_experts: int) -> np.ndarray:
    """The reference's own sample_delay_ms draws (runtime.hpp:312-362), cumulative ms per packet."""
    out = np.zeros(devices * local_experts, np.float64)
    ref().ref_straggler_delays(kind, a, b, device, seed, devices, local_experts, _p(out))
    return out
