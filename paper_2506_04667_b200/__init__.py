"""paper_2506_04667_b200 — B200-native FlashDMoE MoE-layer operator (host mirror).

Python restatement of the reference's operator surface
(/root/reference/proj/include/moefabric/{config,gate,runtime}.hpp) over the C ABI of
libfdmoe.so (include/fdmoe.h). The compute path is the CUDA library only: if
libfdmoe.so is missing or no B200 is visible, calls raise — there is no CPU fallback.

    cfg = MoeConfig(tokens_per_device=4096, embed_dim=2048, ffn_dim=2048,
                    experts_total=16, devices=1, topk=2)
    model = make_model(cfg, seed=0)          # harness.hpp:76-97 restated in C++
    shards = make_shards(cfg, seed=0)        # harness.hpp:99-109
    res = forward(cfg, shards, model)        # runtime.hpp:802 forward()
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
import time
from typing import List, Optional, Sequence

import numpy as np

from . import build as _build

__all__ = [
    "ConfigError", "ProtocolError", "RuntimeFault", "CudaError", "UnsupportedError",
    "Activation", "Precision", "MoeConfig", "ForwardOptions", "GateOutput", "DispatchManifest",
    "TaskStats", "ForwardResult", "ModelWeights", "Operator", "forward", "make_model", "make_shards",
    "expert_capacity", "padded_capacity", "size_L", "flat_index", "validate_write", "lib",
    "gemm_tasks_for_rows", "combine_tiles_for_rows", "initial_task_bound", "dispatch_manifest",
    "payload_bytes", "padded_baseline_bytes", "max_rel_error",
]


# ---------------------------------------------------------------- errors (config.hpp:16-30)
class FdmoeError(RuntimeError):
    pass


class ConfigError(FdmoeError, ValueError):
    pass


class ProtocolError(FdmoeError):
    pass


class RuntimeFault(FdmoeError):
    pass


class CudaError(FdmoeError):
    pass


class UnsupportedError(FdmoeError):
    pass


_ERRS = {1: ConfigError, 2: ProtocolError, 3: RuntimeFault, 4: CudaError, 5: UnsupportedError}


class Activation:
    relu = 0
    gelu = 1
    identity = 2
    _names = {"relu": 0, "gelu": 1, "identity": 2}

    @classmethod
    def parse(cls, s):  # config.hpp:44-49
        if isinstance(s, int):
            return s
        if s not in cls._names:
            raise ConfigError(f"unknown activation: {s}")
        return cls._names[s]


class Precision:
    fp32 = 0   # FP32-accurate 3xTF32
    bf16 = 1


# ---------------------------------------------------------------- ctypes ABI
class _Cfg(C.Structure):
    _fields_ = [("tokens_per_device", C.c_int64), ("embed_dim", C.c_int64), ("ffn_dim", C.c_int64),
                ("experts_total", C.c_int64), ("devices", C.c_int64), ("topk", C.c_int64),
                ("capacity_factor", C.c_double), ("tile_rows", C.c_int64), ("tile_cols", C.c_int64),
                ("activation", C.c_int32), ("precision", C.c_int32), ("seed", C.c_uint64)]


class _Opts(C.Structure):
    _fields_ = [("processors", C.c_int32), ("sequential", C.c_int32), ("deadlock_budget_ms", C.c_int64),
                ("exact_gate", C.c_int32), ("trace_events", C.c_int32), ("straggler_kind", C.c_int32),
                ("straggler_device", C.c_int32), ("straggler_a", C.c_double), ("straggler_b", C.c_double),
                ("seed", C.c_uint64)]


class _Routing(C.Structure):
    _fields_ = [("g_phi", C.c_void_p), ("table_token", C.c_void_p), ("table_weight", C.c_void_p),
                ("slot_counts", C.c_void_p), ("dropped", C.c_void_p), ("n_dropped", C.c_void_p),
                ("picks_expert", C.c_void_p), ("picks_slot", C.c_void_p), ("picks_weight", C.c_void_p)]


class _Stats(C.Structure):
    _fields_ = [("gemm0", C.c_int64), ("gemm1", C.c_int64), ("combine", C.c_int64), ("enqueued", C.c_int64),
                ("executed", C.c_int64), ("bound_initial", C.c_int64), ("bound_final", C.c_int64),
                ("scheduled_final", C.c_int64), ("launches", C.c_int64), ("kernel_ms", C.c_double),
                ("gate_exact_tokens", C.c_int64), ("gate_pair_tokens", C.c_int64),
                ("tiles_resolved", C.c_int64)]


class _Info(C.Structure):
    _fields_ = [("capacity", C.c_int64), ("packet_rows", C.c_int64), ("heap_bytes", C.c_int64),
                ("scratch_bytes", C.c_int64), ("weight_bytes", C.c_int64), ("ctas_per_rank", C.c_int32),
                ("smem_bytes", C.c_int32), ("num_sms", C.c_int32), ("ranks_per_launch", C.c_int32),
                ("fused_combine", C.c_int32)]


EXPORTED_SYMBOLS = [
    "fdmoe_abi_version", "fdmoe_last_error", "fdmoe_config_validate", "fdmoe_expert_capacity",
    "fdmoe_padded_capacity", "fdmoe_size_L", "fdmoe_flat_index", "fdmoe_validate_write",
    "fdmoe_gemm_tasks_for_rows", "fdmoe_combine_tiles_for_rows", "fdmoe_initial_task_bound",
    "fdmoe_synth_model", "fdmoe_synth_shards", "fdmoe_create", "fdmoe_destroy", "fdmoe_ipc_size",
    "fdmoe_export_heap", "fdmoe_import_peers", "fdmoe_set_weights", "fdmoe_forward", "fdmoe_forward_async",
    "fdmoe_sync", "fdmoe_get_info", "fdmoe_last_kernel_ms", "fdmoe_read_trace",
    "fdmoe_read_events", "fdmoe_straggler_delays", "fdmoe_forward_stream",
]

_LIB = None
_DEV_LIB = None
_LIB_PATH = None   # select_library(): tools/ A/B runs of another build; None = the in-tree product library


TRACE_POINTS = 40   # kTracePts (fdmoe_device.cuh)


def select_library(path: str):
    """Tools only: run the operator on another build of the library (e.g. lib/libfdmoe_dev.so for the
    FDMOE_DEBUG ablations and wait accounting, or an A/B build). Must precede the first lib() call."""
    global _LIB_PATH
    if _LIB is not None:
        raise RuntimeError("select_library() after the library was loaded")
    _LIB_PATH = path


def _load(path: str):
    if path in (_build.LIB, _build.DEV_LIB) and (not os.path.exists(path) or _build._stale(path)):
        try:
            _build.build()
        except Exception as e:  # no nvcc on a deployment box: the prebuilt .so must exist
            if not os.path.exists(path):
                raise ImportError(f"{os.path.basename(path)} missing and build failed: {e}") from e
    return C.CDLL(path)


def dev_lib():
    """libfdmoe_dev.so: the include/fdmoe_dev.h diagnostics (device expf, single-tile GEMM, microbenchmarks)."""
    global _DEV_LIB
    if _DEV_LIB is None:
        L = _load(_build.DEV_LIB)
        vp, i32, i64, f32p = C.c_void_p, C.c_int32, C.c_int64, C.c_void_p
        for name, (res, args) in {
            "fdmoe_debug_expf": (i32, [f32p, f32p, i64]),
            "fdmoe_debug_gemm": (i32, [i32, i32, f32p, f32p, f32p]),
            "fdmoe_debug_mma_rate": (i32, [i32, i32, i32, i32, vp]),
            "fdmoe_debug_latency": (i32, [i32, vp]),
            "fdmoe_last_error": (C.c_char_p, []),
        }.items():
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args
        _DEV_LIB = L
    return _DEV_LIB


def dev_check(status: int):
    if status != 0:
        raise _ERRS.get(status, FdmoeError)(dev_lib().fdmoe_last_error().decode(errors="replace"))


def lib():
    """Load libfdmoe.so (building it first if the sources are newer). Raises if it cannot."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = _LIB_PATH or _build.LIB
    L = _load(path)
    vp, i32, i64, u64, f32p = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_void_p
    sig = {
        "fdmoe_abi_version": (i32, []),
        "fdmoe_last_error": (C.c_char_p, []),
        "fdmoe_config_validate": (i32, [C.POINTER(_Cfg), i32]),
        "fdmoe_expert_capacity": (i64, [C.POINTER(_Cfg)]),
        "fdmoe_padded_capacity": (i64, [i64, i64]),
        "fdmoe_size_L": (u64, [C.POINTER(_Cfg)]),
        "fdmoe_flat_index": (i64, [i64] * 9),
        "fdmoe_validate_write": (i32, [i64] * 4),
        "fdmoe_gemm_tasks_for_rows": (i64, [C.POINTER(_Cfg), i64]),
        "fdmoe_combine_tiles_for_rows": (i64, [C.POINTER(_Cfg), i64]),
        "fdmoe_initial_task_bound": (i64, [C.POINTER(_Cfg)]),
        "fdmoe_synth_model": (i32, [C.POINTER(_Cfg), u64, f32p, f32p, f32p, f32p, f32p]),
        "fdmoe_synth_shards": (i32, [C.POINTER(_Cfg), u64, f32p]),
        "fdmoe_create": (i32, [C.POINTER(_Cfg), vp, i32, i32, C.POINTER(vp)]),
        "fdmoe_destroy": (i32, [vp]),
        "fdmoe_ipc_size": (C.c_size_t, []),
        "fdmoe_export_heap": (i32, [vp, vp]),
        "fdmoe_import_peers": (i32, [vp, vp, i32]),
        "fdmoe_set_weights": (i32, [vp, f32p, f32p, f32p, f32p, f32p, i32]),
        "fdmoe_forward": (i32, [vp, vp, vp, i32, C.POINTER(_Opts), vp, vp]),
        "fdmoe_forward_async": (i32, [vp, vp, vp, vp, vp]),
        "fdmoe_sync": (i32, [vp]),
        "fdmoe_get_info": (i32, [vp, C.POINTER(_Info)]),
        "fdmoe_last_kernel_ms": (i32, [vp, vp]),
        "fdmoe_read_trace": (i32, [vp, i32, vp, i32, vp]),
        "fdmoe_read_events": (i32, [vp, i32, vp, i64, vp, vp]),
        "fdmoe_straggler_delays": (i32, [C.POINTER(_Opts), i64, i64, vp]),
        "fdmoe_forward_stream": (i32, [vp, i32, vp, vp, C.POINTER(_Opts)]),
    }
    if hasattr(L, "fdmoe_read_chunklog"):   # development build (select_library)
        sig["fdmoe_read_chunklog"] = (i32, [vp, vp])
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = L
    return L


def _check(status: int):
    if status != 0:
        msg = lib().fdmoe_last_error().decode(errors="replace")
        raise _ERRS.get(status, FdmoeError)(msg)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------- reference types
@dataclasses.dataclass
class MoeConfig:
    """config.hpp:53-87 (plus the GPU FFN precision)."""
    tokens_per_device: int = 8
    embed_dim: int = 8
    ffn_dim: int = 8
    experts_total: int = 2
    devices: int = 1
    topk: int = 1
    capacity_factor: float = 1.0
    tile_rows: int = 16
    tile_cols: int = 8
    activation: int = Activation.relu
    seed: int = 0
    precision: int = Precision.fp32

    def local_experts(self) -> int:
        return self.experts_total // self.devices

    def to_c(self) -> _Cfg:
        return _Cfg(self.tokens_per_device, self.embed_dim, self.ffn_dim, self.experts_total, self.devices,
                    self.topk, float(self.capacity_factor), self.tile_rows, self.tile_cols,
                    Activation.parse(self.activation), int(self.precision), self.seed)

    def validate(self, gpu_envelope: bool = False):
        c = self.to_c()
        _check(lib().fdmoe_config_validate(C.byref(c), 1 if gpu_envelope else 0))


class ScheduleMode:
    """runtime.hpp:76."""
    overlapped = "overlapped"
    sequential = "sequential"


@dataclasses.dataclass
class StragglerSpec:
    """runtime.hpp:78-84: kind none | constant (a ms) | uniform (U(a, b) ms) | lognormal (median a ms,
    sigma b), applied per dispatch packet of rank `device`."""
    kind: str = "none"
    a: float = 0.0
    b: float = 0.0
    device: int = 0

    _KINDS = {"none": 0, "constant": 1, "uniform": 2, "lognormal": 3}

    def kind_code(self) -> int:
        if self.kind not in self._KINDS:
            raise ConfigError(f"unknown straggler kind {self.kind!r}")
        return self._KINDS[self.kind]


@dataclasses.dataclass
class ForwardOptions:
    """runtime.hpp:86-92."""
    processors: int = 4
    sequential: bool = False
    deadlock_budget_ms: int = 5000
    seed: int = 0
    # B200 addition: True = reference-exact gate logits for every token (G_phi and combine weights
    # bit-identical); False = certified gate (routing proven identical per token)
    exact_gate: bool = False
    mode: str = ScheduleMode.overlapped
    straggler: StragglerSpec = dataclasses.field(default_factory=StragglerSpec)
    # B200 addition: record the device event log into ForwardResult.trace (trace.py / audit.py)
    trace: bool = False

    def is_sequential(self) -> bool:
        if self.mode not in (ScheduleMode.overlapped, ScheduleMode.sequential):
            raise ConfigError(f"unknown schedule mode {self.mode!r}")
        return bool(self.sequential) or self.mode == ScheduleMode.sequential

    def to_c(self):
        sp = self.straggler
        return _Opts(self.processors, 1 if self.is_sequential() else 0, self.deadlock_budget_ms,
                     1 if self.exact_gate else 0, 1 if self.trace else 0, sp.kind_code(), sp.device,
                     float(sp.a), float(sp.b), self.seed)


@dataclasses.dataclass
class ModelWeights:
    """config.hpp:130-147 as stacked arrays: wg H x E; w1 E x H x D; b1 E x D; w2 E x D x H; b2 E x H."""
    wg: np.ndarray
    w1: np.ndarray
    b1: np.ndarray
    w2: np.ndarray
    b2: np.ndarray


@dataclasses.dataclass
class GateOutput:
    """gate.hpp:24-37 (table as two arrays E x C; token -1 = empty slot)."""
    g_phi: np.ndarray
    capacity: int
    table_token: np.ndarray
    table_weight: np.ndarray
    slot_counts: np.ndarray
    dropped: List[tuple]
    picks_expert: Optional[np.ndarray] = None
    picks_slot: Optional[np.ndarray] = None
    picks_weight: Optional[np.ndarray] = None


@dataclasses.dataclass
class DispatchManifest:
    """gate.hpp:113-151: per destination device x local expert (expert_global, count, tokens)."""
    per_device: list

    def total_routed(self) -> int:
        return sum(m[1] for d in self.per_device for m in d)


@dataclasses.dataclass
class TaskStats:
    gemm0: int = 0
    gemm1: int = 0
    combine: int = 0
    enqueued: int = 0
    executed: int = 0
    bound_initial: int = 0
    bound_final: int = 0
    scheduled_final: int = 0
    launches: int = 0
    kernel_ms: float = 0.0
    gate_exact_tokens: int = 0
    gate_pair_tokens: int = 0
    tiles_resolved: int = 0

    def total(self) -> int:
        return self.gemm0 + self.gemm1 + self.combine


@dataclasses.dataclass
class ForwardResult:
    """runtime.hpp:108-117. `trace` holds the device event log (trace.TraceEvent list, trace.hpp:38-60)
    when ForwardOptions.trace is set, else []."""
    outputs: List[np.ndarray]
    gates: List[GateOutput]
    manifests: List[DispatchManifest]
    trace: list
    bytes: np.ndarray
    bytes_padded: np.ndarray
    stats: List[TaskStats]
    makespan_ns: int


# ---------------------------------------------------------------- pure functions
def expert_capacity(cfg: MoeConfig) -> int:
    c = cfg.to_c()
    return int(lib().fdmoe_expert_capacity(C.byref(c)))


def padded_capacity(capacity: int, tile_rows: int) -> int:
    return int(lib().fdmoe_padded_capacity(capacity, tile_rows))


def size_L(cfg: MoeConfig) -> int:
    c = cfg.to_c()
    return int(lib().fdmoe_size_L(C.byref(c)))


def flat_index(devices, local_experts, slot_capacity, embed_dim, p_star, rnd, buffer, expert, slot) -> int:
    v = int(lib().fdmoe_flat_index(devices, local_experts, slot_capacity, embed_dim, p_star, rnd, buffer,
                                   expert, slot))
    if v < 0:
        raise IndexError("flat_index: coordinate out of bounds")
    return v


def validate_write(src, dst, p_star, buffer) -> int:
    return int(lib().fdmoe_validate_write(src, dst, p_star, buffer))


def gemm_tasks_for_rows(cfg: MoeConfig, n: int) -> int:
    c = cfg.to_c()
    return int(lib().fdmoe_gemm_tasks_for_rows(C.byref(c), n))


def combine_tiles_for_rows(cfg: MoeConfig, n: int) -> int:
    c = cfg.to_c()
    return int(lib().fdmoe_combine_tiles_for_rows(C.byref(c), n))


def initial_task_bound(cfg: MoeConfig) -> int:
    c = cfg.to_c()
    return int(lib().fdmoe_initial_task_bound(C.byref(c)))


def straggler_delays(cfg: MoeConfig, opts: ForwardOptions) -> np.ndarray:
    """Cumulative per-packet hold-back (ns) of the straggler's dispatch signals (runtime.hpp:312-362):
    entry e = destination * E_local + local expert."""
    out = np.zeros(cfg.experts_total, np.uint64)
    o = opts.to_c()
    _check(lib().fdmoe_straggler_delays(C.byref(o), cfg.devices, cfg.local_experts(), _ptr(out)))
    return out


def make_model(cfg: MoeConfig, seed: Optional[int] = None) -> ModelWeights:
    """harness.hpp:76-97 restated in C++ (bit-identical draws)."""
    H, D, E = cfg.embed_dim, cfg.ffn_dim, cfg.experts_total
    m = ModelWeights(np.empty((H, E), np.float32), np.empty((E, H, D), np.float32), np.empty((E, D), np.float32),
                     np.empty((E, D, H), np.float32), np.empty((E, H), np.float32))
    c = cfg.to_c()
    _check(lib().fdmoe_synth_model(C.byref(c), cfg.seed if seed is None else seed, _ptr(m.wg), _ptr(m.w1),
                                   _ptr(m.b1), _ptr(m.w2), _ptr(m.b2)))
    return m


def make_shards(cfg: MoeConfig, seed: Optional[int] = None) -> List[np.ndarray]:
    """harness.hpp:99-109 restated in C++."""
    a = np.empty((cfg.devices, cfg.tokens_per_device, cfg.embed_dim), np.float32)
    c = cfg.to_c()
    _check(lib().fdmoe_synth_shards(C.byref(c), cfg.seed if seed is None else seed, _ptr(a)))
    return [a[d] for d in range(cfg.devices)]


def dispatch_manifest(gate: GateOutput, cfg: MoeConfig) -> DispatchManifest:
    """gate.hpp:133-151."""
    el = cfg.local_experts()
    per = []
    for d in range(cfg.devices):
        dev = []
        for le in range(el):
            e = d * el + le
            n = int(gate.slot_counts[e])
            dev.append((e, n, [int(t) for t in gate.table_token[e, :n]]))
        per.append(dev)
    return DispatchManifest(per)


def payload_bytes(cfg: MoeConfig, slot_counts: Sequence[np.ndarray]) -> np.ndarray:
    """pgas.hpp:130-135 for this operator: bytes[p][q] = rows p dispatches to q plus rows p returns
    to q (combine), at the reference's FP32 accounting (4 bytes per element)."""
    P, el, H = cfg.devices, cfg.local_experts(), cfg.embed_dim
    n = np.zeros((P, P), np.int64)
    for p in range(P):
        for q in range(P):
            n[p, q] = int(np.sum(slot_counts[p][q * el:(q + 1) * el]))
    return ((n + n.T) * H * 4).astype(np.uint64).reshape(-1)


def padded_baseline_bytes(cfg: MoeConfig) -> np.ndarray:
    """pgas.hpp:140-147."""
    cp = padded_capacity(expert_capacity(cfg), cfg.tile_rows)
    per = 2 * cfg.local_experts() * cp * cfg.embed_dim * 4
    return np.full(cfg.devices * cfg.devices, per, np.uint64)


def max_rel_error(got: Sequence[np.ndarray], want: Sequence[np.ndarray]) -> float:
    """harness.hpp:163-175 normwise relative error."""
    md = max(float(np.max(np.abs(g.astype(np.float64) - w.astype(np.float64)))) for g, w in zip(got, want))
    mr = max(float(np.max(np.abs(w.astype(np.float64)))) for w in want)
    if mr == 0.0:
        return 0.0 if md == 0.0 else md / 1e-30
    return md / mr


# ---------------------------------------------------------------- the operator
class Operator:
    """Persistent operator handle: ranks, symmetric heaps and resident weights.

    ranks: local rank ids (default all cfg.devices ranks in this process);
    device_ids: CUDA device of each local rank (default all on device 0 = virtual ranks).
    """

    def __init__(self, cfg: MoeConfig, device_ids: Optional[Sequence[int]] = None, first_rank: int = 0,
                 n_local: Optional[int] = None):
        self.cfg = cfg
        L = lib()
        n_local = cfg.devices if n_local is None else n_local
        ids = (C.c_int32 * n_local)(*(device_ids if device_ids is not None else [0] * n_local))
        h = C.c_void_p()
        c = cfg.to_c()
        _check(L.fdmoe_create(C.byref(c), C.cast(ids, C.c_void_p), n_local, first_rank, C.byref(h)))
        self._h = h
        self.n_local = n_local
        self.first_rank = first_rank

    def close(self):
        if getattr(self, "_h", None):
            lib().fdmoe_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        i = _Info()
        _check(lib().fdmoe_get_info(self._h, C.byref(i)))
        return {f: getattr(i, f) for f, _ in _Info._fields_}

    # multi-process attach
    def export_heap(self) -> bytes:
        n = lib().fdmoe_ipc_size()
        buf = C.create_string_buffer(n)
        _check(lib().fdmoe_export_heap(self._h, buf))
        return buf.raw

    def import_peers(self, blobs: Sequence[bytes]):
        blob = b"".join(blobs)
        _check(lib().fdmoe_import_peers(self._h, C.c_char_p(blob), len(blobs)))

    def set_weights(self, model: ModelWeights):
        arrs = [np.ascontiguousarray(x, np.float32) for x in (model.wg, model.w1, model.b1, model.w2, model.b2)]
        _check(lib().fdmoe_set_weights(self._h, *[_ptr(a) for a in arrs], 0))

    def set_weights_device(self, wg, w1, b1, w2, b2):
        """Device pointers (ints), e.g. torch tensors' data_ptr()."""
        _check(lib().fdmoe_set_weights(self._h, wg, w1, b1, w2, b2, 1))

    def forward(self, shards: Sequence[np.ndarray], opts: Optional[ForwardOptions] = None, routing: bool = True,
                stats: bool = True) -> ForwardResult:
        cfg, n = self.cfg, self.n_local
        S, H, E, K = cfg.tokens_per_device, cfg.embed_dim, cfg.experts_total, cfg.topk
        ins = [np.ascontiguousarray(s, np.float32) for s in shards]
        for a in ins:
            if a.shape != (S, H):
                raise ConfigError("forward: shard is not S x H")
        outs = [np.empty((S, H), np.float32) for _ in range(n)]
        in_p = (C.c_void_p * n)(*[a.ctypes.data for a in ins])
        out_p = (C.c_void_p * n)(*[a.ctypes.data for a in outs])
        o = opts or ForwardOptions()
        copts = o.to_c()
        cap = expert_capacity(cfg)
        rt = (_Routing * n)()
        keep = []
        if routing:
            for i in range(n):
                arrs = dict(g_phi=np.empty((S, E), np.float32), table_token=np.empty((E, cap), np.int64),
                            table_weight=np.empty((E, cap), np.float32), slot_counts=np.empty(E, np.int64),
                            dropped=np.empty(2 * S * K, np.int64), n_dropped=np.zeros(1, np.int64),
                            picks_expert=np.empty((S, K), np.int32), picks_slot=np.empty((S, K), np.int32),
                            picks_weight=np.empty((S, K), np.float32))
                for k, v in arrs.items():
                    setattr(rt[i], k, v.ctypes.data)
                keep.append(arrs)
        st = (_Stats * n)()
        t0 = time.perf_counter_ns()
        _check(lib().fdmoe_forward(self._h, in_p, out_p, 0, C.byref(copts), rt if routing else None,
                                   st if stats else None))
        t1 = time.perf_counter_ns()
        gates = []
        for i in range(n):
            if not routing:
                break
            a = keep[i]
            nd = int(a["n_dropped"][0])
            dr = a["dropped"][:2 * nd].reshape(-1, 2)
            gates.append(GateOutput(a["g_phi"], cap, a["table_token"], a["table_weight"], a["slot_counts"],
                                    [(int(x), int(y)) for x, y in dr], a["picks_expert"], a["picks_slot"],
                                    a["picks_weight"]))
        stats_l = [TaskStats(*[getattr(st[i], f) for f, _ in _Stats._fields_]) for i in range(n)] if stats else []
        manifests = [dispatch_manifest(g, cfg) for g in gates]
        if routing and n == cfg.devices:
            b = payload_bytes(cfg, [g.slot_counts for g in gates])
        else:
            b = np.zeros(cfg.devices * cfg.devices, np.uint64)
        tr = []
        if o.trace:
            from . import trace as _trace
            tr = _trace.to_trace_events([self.events(i) for i in range(n)], first_rank=self.first_rank)
        return ForwardResult(outs, gates, manifests, tr, b, padded_baseline_bytes(cfg), stats_l, t1 - t0)

    def forward_device(self, in_ptrs: Sequence[int], out_ptrs: Sequence[int], streams: Optional[Sequence[int]] = None,
                       opts: Optional[ForwardOptions] = None):
        """Asynchronous forward on device pointers (one kernel launch per device)."""
        n = self.n_local
        ip = (C.c_void_p * n)(*in_ptrs)
        op = (C.c_void_p * n)(*out_ptrs)
        sp = (C.c_void_p * n)(*(streams or [0] * n))
        copts = (opts or ForwardOptions()).to_c()
        _check(lib().fdmoe_forward_async(self._h, ip, op, sp, C.byref(copts)))

    def forward_stream(self, batches: Sequence[Sequence[np.ndarray]], outs: Sequence[Sequence[np.ndarray]],
                       opts: Optional[ForwardOptions] = None):
        """Serving loop over host batches (each a list of n_local S x H FP32 arrays, ideally pinned):
        copies of neighbouring batches overlap each launch (fdmoe_forward_stream)."""
        n = self.n_local
        S, H = self.cfg.tokens_per_device, self.cfg.embed_dim
        ins = [a for b in batches for a in b]
        os_ = [a for b in outs for a in b]
        if len(ins) != len(batches) * n or len(os_) != len(ins):
            raise ConfigError("forward_stream: every batch needs n_local input and output shards")
        for a in ins + os_:
            if a.shape != (S, H) or a.dtype != np.float32 or not a.flags["C_CONTIGUOUS"]:
                raise ConfigError("forward_stream: shards must be contiguous S x H float32")
        ip = (C.c_void_p * len(ins))(*[a.ctypes.data for a in ins])
        op_ = (C.c_void_p * len(os_))(*[a.ctypes.data for a in os_])
        copts = (opts or ForwardOptions()).to_c()
        _check(lib().fdmoe_forward_stream(self._h, len(batches), ip, op_, C.byref(copts)))

    def sync(self):
        _check(lib().fdmoe_sync(self._h))

    def trace(self, local_rank: int = 0) -> np.ndarray:
        """Per-CTA phase timestamps of the last launch (ns, relative to the earliest CTA start):
        columns start, gate, barrier, dispatch, ffn, combine, end, ffn_tiles; ... 32-35: raw SM clock64 at the
        start, FFN start, FFN end and end (effective SM clock per phase = cycles / ns)."""
        info = self.info()
        buf = np.zeros((info["ctas_per_rank"], TRACE_POINTS), np.uint64)
        n = C.c_int32()
        _check(lib().fdmoe_read_trace(self._h, local_rank, _ptr(buf), buf.size, C.byref(n)))
        t = buf.astype(np.int64)
        t0 = t[:, 0].min()
        t[:, :7] -= t0
        t[:, 20:27] -= t0
        t[:, 28:32] = np.where(t[:, 28:32] > 0, t[:, 28:32] - t0, 0)   # tensor-core gate logits done / staged
        t[:, 36:40] = np.where(t[:, 36:40] > 0, t[:, 36:40] - t0, 0)   # full-exact pass; gate roles start / epilogue done
        return t

    def events(self, local_rank: int = 0) -> np.ndarray:
        """Device event log of the most recent launch run with ForwardOptions(trace=True), as a
        structured array (trace.EVENT_DTYPE, raw %globaltimer ns). Raises if records were lost."""
        from .trace import EVENT_DTYPE
        n, dropped = C.c_int64(), C.c_int64()
        _check(lib().fdmoe_read_events(self._h, local_rank, None, 0, C.byref(n), C.byref(dropped)))
        buf = np.zeros(n.value, EVENT_DTYPE)
        _check(lib().fdmoe_read_events(self._h, local_rank, _ptr(buf), n.value, C.byref(n), C.byref(dropped)))
        if dropped.value:
            raise RuntimeFault(f"event log overflow: {dropped.value} records lost")
        return buf

    def last_kernel_ms(self) -> float:
        """Device time of the most recent layer launch (CUDA events around it, max over devices)."""
        v = C.c_double()
        _check(lib().fdmoe_last_kernel_ms(self._h, C.byref(v)))
        return v.value


def forward(cfg: MoeConfig, shards: Sequence[np.ndarray], model: ModelWeights,
            opts: Optional[ForwardOptions] = None, device_ids: Optional[Sequence[int]] = None) -> ForwardResult:
    """runtime.hpp:802 forward(cfg, shards, model, opts): one-shot operator (creates, runs, destroys)."""
    if len(shards) != cfg.devices:
        raise ConfigError("forward: shard count != devices")
    if model.w1.shape[0] != cfg.experts_total:
        raise ConfigError("forward: expert parameter count != experts_total")
    cfg.validate()
    op = Operator(cfg, device_ids)
    try:
        op.set_weights(model)
        return op.forward(shards, opts)
    finally:
        op.close()
