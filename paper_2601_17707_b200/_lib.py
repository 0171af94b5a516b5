"""ctypes binding of ``libbbc.so`` (the C ABI declared in ``include/bbc.h``).

There is no CPU fallback: if the library is missing or no CUDA device is visible the
counting entry points raise ``DeviceError``.  Status codes map onto the reference's
exceptions (pkg/src/bbcount/errors.py): RANGE -> IndexOutOfRangeError, DUP ->
DuplicateEdgeError(u, v), OVERFLOW -> CountOverflowError, ARG -> ValueError, the rest ->
DeviceError (a BBCountError).
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .errors import CountOverflowError, DeviceError, DuplicateEdgeError, IndexOutOfRangeError

LIB_PATH = Path(__file__).resolve().with_name("libbbc.so")

ALGO_GBBC = 0
ALGO_GBBCPP = 1
SIDE_CHEAPER = -1
SIDE_U = 0
SIDE_V = 1
SIDE_MIN = 2
FLAG_BANDED_ONLY = 1
FLAG_ROUNDS = 4096  # record per-kind round counters (round_counters())

EXPORTED_SYMBOLS = (
    "bbc_graph_create", "bbc_graph_create_device", "bbc_count", "bbc_block_work", "bbc_task_order",
    "bbc_round_counters", "bbc_classify", "bbc_count_2k", "bbc_ingest_text", "bbc_ingest_edges",
    "bbc_ingest_graph", "bbc_ingest_destroy", "bbc_graph_info", "bbc_graph_stream", "bbc_graph_destroy", "bbc_device_count", "bbc_last_error",
    "bbc_last_error_info", "bbc_multi_create", "bbc_multi_count", "bbc_multi_devices", "bbc_multi_graph",
    "bbc_multi_destroy", "bbc_count_multi", "bbc_block_busy_ns", "bbc_enumerate_butterflies",
)


class Opts(ctypes.Structure):
    _fields_ = [("algo", ctypes.c_int32), ("tile_span", ctypes.c_int32), ("blocks", ctypes.c_int32),
                ("warp_max", ctypes.c_int32), ("partial_max", ctypes.c_int32), ("part_index", ctypes.c_int32),
                ("part_count", ctypes.c_int32), ("flags", ctypes.c_int32)]


class Stats(ctypes.Structure):
    _fields_ = [("wedges", ctypes.c_uint64), ("wedges_total", ctypes.c_uint64), ("w_u", ctypes.c_uint64),
                ("w_v", ctypes.c_uint64), ("balanced_hi", ctypes.c_uint64), ("unbalanced_hi", ctypes.c_uint64),
                ("anchor_side", ctypes.c_int32), ("blocks", ctypes.c_int32), ("threads", ctypes.c_int32),
                ("tile_span", ctypes.c_int32), ("tasks", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("preprocess_ms", ctypes.c_float), ("count_ms", ctypes.c_float)]


class SignPolicy(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("at_or_above", ctypes.c_int32), ("threshold", ctypes.c_double),
                ("p_positive", ctypes.c_double), ("seed", ctypes.c_uint64)]


ERR_PARSE, ERR_MISSING, ERR_SIGNVAL, ERR_UNSUPPORTED = 8, 9, 10, 11

_lock = threading.Lock()
_lib = None


def load() -> ctypes.CDLL:
    """Load libbbc.so once; raise DeviceError if it is absent (no silent fallback)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise DeviceError(f"{LIB_PATH} is not built; run `python -m paper_2601_17707_b200._build`")
        L = ctypes.CDLL(str(LIB_PATH))
        P, I32, I64, U64P = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.POINTER(ctypes.c_uint64)
        L.bbc_graph_create.argtypes = [ctypes.c_int, I64, I64, I64, P, P, P, I32, ctypes.POINTER(P)]
        L.bbc_graph_create_device.argtypes = [ctypes.c_int, I64, I64, I64, P, P, P, I32, ctypes.POINTER(P)]
        L.bbc_count.argtypes = [P, ctypes.POINTER(Opts), U64P, ctypes.POINTER(Stats)]
        L.bbc_block_work.argtypes = [P, U64P, I32]
        L.bbc_task_order.argtypes = [P, I32, ctypes.POINTER(ctypes.c_int32), P, I64]
        L.bbc_round_counters.argtypes = [P, U64P]
        L.bbc_block_busy_ns.argtypes = [P, U64P, I32]
        L.bbc_enumerate_butterflies.argtypes = [I32, I64, I64, I64, P, P, P, U64P, P, P, ctypes.c_uint64]
        L.bbc_classify.argtypes = [P, ctypes.POINTER(Opts), U64P, ctypes.POINTER(Stats)]
        L.bbc_count_2k.argtypes = [P, I32, ctypes.POINTER(Opts), U64P, ctypes.POINTER(Stats)]
        L.bbc_ingest_text.argtypes = [ctypes.c_int, ctypes.c_char_p, I64, ctypes.POINTER(SignPolicy),
                                      ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(P)]
        L.bbc_ingest_edges.argtypes = [P, P, P, P]
        L.bbc_ingest_graph.argtypes = [P, I32, ctypes.POINTER(P)]
        L.bbc_ingest_destroy.argtypes = [P]
        L.bbc_ingest_destroy.restype = None
        L.bbc_graph_info.argtypes = [P, ctypes.POINTER(ctypes.c_int64), I32]
        L.bbc_graph_stream.argtypes = [P]
        L.bbc_graph_stream.restype = P
        L.bbc_graph_destroy.argtypes = [P]
        L.bbc_graph_destroy.restype = None
        L.bbc_multi_create.argtypes = [I32, ctypes.POINTER(ctypes.c_int32), I64, I64, I64, P, P, P, I32,
                                       ctypes.POINTER(P)]
        L.bbc_multi_count.argtypes = [P, ctypes.POINTER(Opts), U64P, ctypes.POINTER(Stats)]
        L.bbc_multi_devices.argtypes = [P, ctypes.POINTER(ctypes.c_int32), I32]
        L.bbc_multi_graph.argtypes = [P, I32]
        L.bbc_multi_graph.restype = P
        L.bbc_multi_destroy.argtypes = [P]
        L.bbc_multi_destroy.restype = None
        L.bbc_count_multi.argtypes = [I32, ctypes.POINTER(ctypes.c_int32), I64, I64, I64, P, P, P, I32,
                                      ctypes.POINTER(Opts), U64P, ctypes.POINTER(Stats)]
        L.bbc_device_count.argtypes = []
        L.bbc_last_error.restype = ctypes.c_char_p
        L.bbc_last_error_info.restype = ctypes.c_int64
        for name in ("bbc_graph_create", "bbc_graph_create_device", "bbc_count", "bbc_block_work",
                     "bbc_task_order", "bbc_round_counters", "bbc_classify", "bbc_count_2k", "bbc_graph_info",
                     "bbc_device_count", "bbc_ingest_text", "bbc_ingest_edges", "bbc_ingest_graph",
                     "bbc_multi_create", "bbc_multi_count", "bbc_multi_devices", "bbc_count_multi", "bbc_block_busy_ns", "bbc_enumerate_butterflies"):
            getattr(L, name).restype = ctypes.c_int
        _lib = L
        return L


def device_count() -> int:
    return int(load().bbc_device_count())


def _raise(rc: int) -> None:
    L = load()
    msg = (L.bbc_last_error() or b"").decode()
    info = int(L.bbc_last_error_info())
    if rc == 1:
        raise IndexOutOfRangeError(msg)
    if rc == 2:
        raise DuplicateEdgeError(info >> 32, info & 0xFFFFFFFF)
    if rc == 3:
        raise CountOverflowError(msg)
    if rc == 4:
        if msg.endswith("is not a valid EdgeSign"):
            raise ValueError(msg)
        raise ValueError(msg)
    raise DeviceError(msg or f"libbbc error {rc}")


@dataclass
class CountResult:
    balanced: int     # exact (may exceed 2^64 - 1; callers apply the overflow contract)
    unbalanced: int
    wedges: int       # admitted wedges processed by this call
    wedges_total: int
    w_u: int
    w_v: int
    anchor_side: int
    blocks: int
    threads: int
    tile_span: int
    tasks: int
    preprocess_ms: float
    count_ms: float


def _result(out, st: Stats) -> CountResult:
    return CountResult(balanced=int(out[0]) | (int(st.balanced_hi) << 64),
                       unbalanced=int(out[1]) | (int(st.unbalanced_hi) << 64), wedges=int(st.wedges),
                       wedges_total=int(st.wedges_total), w_u=int(st.w_u), w_v=int(st.w_v),
                       anchor_side=int(st.anchor_side), blocks=int(st.blocks), threads=int(st.threads),
                       tile_span=int(st.tile_span), tasks=int(st.tasks), preprocess_ms=float(st.preprocess_ms),
                       count_ms=float(st.count_ms))


class DeviceGraph:
    """Owning handle of one device-resident graph (bbc_graph*).

    A handle is not re-entrant (include/bbc.h): its accumulators, queue and per-CTA work
    buffer are reused by every call, so calls on one handle are serialised by a lock
    (ctypes releases the GIL during them)."""

    def __init__(self, handle: int, device: int, owned: bool = True):
        self._h = ctypes.c_void_p(handle)
        self._owned = owned
        self._lock = threading.Lock()
        self.device = device
        info = (ctypes.c_int64 * 8)()
        load().bbc_graph_info(self._h, info, 8)
        self.n_u, self.n_v, self.m, self.anchor_side, self.n_anchors, self.w_s, self.w_u, self.w_v = \
            (int(x) for x in info)

    @classmethod
    def from_host(cls, n_u: int, n_v: int, u: np.ndarray, v: np.ndarray, s: np.ndarray, device: int = 0,
                  side_rule: int = SIDE_CHEAPER) -> "DeviceGraph":
        u = np.ascontiguousarray(u, dtype=np.int32)
        v = np.ascontiguousarray(v, dtype=np.int32)
        s = np.ascontiguousarray(s, dtype=np.int8)
        h = ctypes.c_void_p()
        rc = load().bbc_graph_create(device, n_u, n_v, len(u), u.ctypes.data, v.ctypes.data, s.ctypes.data,
                                     side_rule, ctypes.byref(h))
        if rc:
            _raise(rc)
        return cls(h.value, device)

    @classmethod
    def from_device_ptrs(cls, n_u: int, n_v: int, m: int, ptr_u: int, ptr_v: int, ptr_s: int, device: int = 0,
                         side_rule: int = SIDE_CHEAPER) -> "DeviceGraph":
        h = ctypes.c_void_p()
        rc = load().bbc_graph_create_device(device, n_u, n_v, m, ptr_u, ptr_v, ptr_s, side_rule, ctypes.byref(h))
        if rc:
            _raise(rc)
        return cls(h.value, device)

    def count(self, algo: int = ALGO_GBBCPP, tile_span: int = 0, blocks: int = 0, part_index: int = 0,
              part_count: int = 1, flags: int = 0) -> CountResult:
        """flags bit 0 (FLAG_BANDED_ONLY): always take the general banded path (testing)."""
        if self._h is None:
            raise DeviceError("graph handle already closed")
        o = Opts(algo=algo, tile_span=tile_span, blocks=blocks, warp_max=0, partial_max=0, part_index=part_index,
                 part_count=part_count, flags=flags)
        out = (ctypes.c_uint64 * 2)()
        st = Stats()
        with self._lock:
            rc = load().bbc_count(self._h, ctypes.byref(o), out, ctypes.byref(st))
        if rc and rc != 3:
            _raise(rc)
        return _result(out, st)

    CLASS_NAMES = ("coherent_pp_pp", "coherent_pp_mm", "coherent_mm_mm", "incoherent_pm_pm", "mixed_pp_pm",
                   "mixed_pm_mm")

    def classify(self, algo: int = ALGO_GBBCPP, blocks: int = 0, part_index: int = 0,
                 part_count: int = 1, flags: int = 0) -> tuple[dict[str, int], float]:
        """Six-way classification (needs a U-anchored handle): (as_dict() counts, device ms)."""
        if self._h is None:
            raise DeviceError("graph handle already closed")
        o = Opts(algo=algo, blocks=blocks, part_index=part_index, part_count=part_count, flags=flags)
        out = (ctypes.c_uint64 * 12)()
        st = Stats()
        with self._lock:
            rc = load().bbc_classify(self._h, ctypes.byref(o), out, ctypes.byref(st))
        if rc:
            _raise(rc)
        return ({n: int(out[2 * i]) | (int(out[2 * i + 1]) << 64) for i, n in enumerate(self.CLASS_NAMES)},
                float(st.count_ms))

    def count_2k(self, k: int, algo: int = ALGO_GBBCPP, blocks: int = 0, part_index: int = 0,
                 part_count: int = 1, flags: int = 0) -> tuple[int, bool, float]:
        """Balanced (2,k)-bicliques with the size-2 side = this handle's anchor side:
        (count, overflowed past 2^64 - 1, device ms)."""
        if self._h is None:
            raise DeviceError("graph handle already closed")
        o = Opts(algo=algo, blocks=blocks, part_index=part_index, part_count=part_count, flags=flags)
        out = (ctypes.c_uint64 * 2)()
        st = Stats()
        with self._lock:
            rc = load().bbc_count_2k(self._h, k, ctypes.byref(o), out, ctypes.byref(st))
        if rc and rc != 3:
            _raise(rc)
        return int(out[0]) | (int(out[1]) << 64), rc == 3, float(st.count_ms)

    def block_work(self, n: int) -> list[int]:
        buf = (ctypes.c_uint64 * max(n, 1))()
        with self._lock:
            rc = load().bbc_block_work(self._h, buf, n)
        if rc:
            _raise(rc)
        return [int(buf[i]) for i in range(n)]

    def block_busy_ns(self, n: int) -> list[int]:
        """Per-CTA busy time (ns) of the last count (bbc_block_busy_ns)."""
        buf = (ctypes.c_uint64 * max(n, 1))()
        with self._lock:
            rc = load().bbc_block_busy_ns(self._h, buf, n)
        if rc:
            _raise(rc)
        return [int(buf[i]) for i in range(n)]

    def round_counters(self) -> dict[str, int]:
        """Rounds of the last count run with FLAG_ROUNDS, by kind."""
        buf = (ctypes.c_uint64 * 8)()
        rc = load().bbc_round_counters(self._h, buf)
        if rc:
            _raise(rc)
        return dict(zip(("bitmap", "bitmap_redone", "tile", "hash", "groups", "wedges", "setups"),
                        (int(x) for x in buf)))

    def task_order(self, algo: int) -> tuple[np.ndarray, np.ndarray]:
        """(anchor ids, admitted wedges) in the dispatch order of ``algo``."""
        n = self.n_anchors
        ids = np.empty(max(n, 1), dtype=np.int32)
        work = np.empty(max(n, 1), dtype=np.uint64)
        with self._lock:
            rc = load().bbc_task_order(self._h, algo, ids.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                       work.ctypes.data, n)
        if rc:
            _raise(rc)
        return ids[:n], work[:n]

    def stream(self) -> int:
        return int(load().bbc_graph_stream(self._h) or 0)

    def close(self) -> None:
        with self._lock:
            if self._h is not None and self._h.value and self._owned:
                load().bbc_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class MultiGraph:
    """Owning handle of a graph replicated on several GPUs of this process (bbc_multi*):
    sharded upload + NCCL all-gather + replicated build; counts are start-vertex
    partitions summed by one NCCL all-reduce (include/bbc.h, bbc_multi_*)."""

    def __init__(self, n_u: int, n_v: int, u: np.ndarray, v: np.ndarray, s: np.ndarray, devices: list[int],
                 side_rule: int = SIDE_CHEAPER):
        u = np.ascontiguousarray(u, dtype=np.int32)
        v = np.ascontiguousarray(v, dtype=np.int32)
        s = np.ascontiguousarray(s, dtype=np.int8)
        devs = (ctypes.c_int32 * len(devices))(*devices)
        h = ctypes.c_void_p()
        rc = load().bbc_multi_create(len(devices), devs, n_u, n_v, len(u), u.ctypes.data, v.ctypes.data,
                                     s.ctypes.data, side_rule, ctypes.byref(h))
        if rc:
            _raise(rc)
        self._h = h
        self._lock = threading.Lock()
        self.devices = list(devices)
        self.replicas = [DeviceGraph(load().bbc_multi_graph(h, i), d, owned=False) for i, d in enumerate(devices)]
        r0 = self.replicas[0]
        self.n_u, self.n_v, self.m, self.anchor_side, self.n_anchors, self.w_s, self.w_u, self.w_v = (
            r0.n_u, r0.n_v, r0.m, r0.anchor_side, r0.n_anchors, r0.w_s, r0.w_u, r0.w_v)

    def count(self, algo: int = ALGO_GBBCPP, tile_span: int = 0, blocks: int = 0, flags: int = 0) -> CountResult:
        if self._h is None:
            raise DeviceError("multi-GPU handle already closed")
        o = Opts(algo=algo, tile_span=tile_span, blocks=blocks, flags=flags)
        out = (ctypes.c_uint64 * 2)()
        st = Stats()
        with self._lock:
            rc = load().bbc_multi_count(self._h, ctypes.byref(o), out, ctypes.byref(st))
        if rc and rc != 3:
            _raise(rc)
        return _result(out, st)

    def close(self) -> None:
        with self._lock:
            for r in getattr(self, "replicas", []):
                r._h = None
            if self._h is not None and self._h.value:
                load().bbc_multi_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Ingested:
    """Owning handle of a device-side ingestion (bbc_ingest*): the deduplicated signed edges
    with dense first-occurrence ids, resident on the device."""

    def __init__(self, handle: int, device: int, n_u: int, n_v: int, m: int):
        self._h = ctypes.c_void_p(handle)
        self.device, self.n_u, self.n_v, self.m = device, n_u, n_v, m

    def edges(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        u = np.empty(max(self.m, 1), dtype=np.int32)
        v = np.empty(max(self.m, 1), dtype=np.int32)
        s = np.empty(max(self.m, 1), dtype=np.int8)
        rc = load().bbc_ingest_edges(self._h, u.ctypes.data, v.ctypes.data, s.ctypes.data)
        if rc:
            _raise(rc)
        return u[:self.m], v[:self.m], s[:self.m]

    def device_graph(self, side_rule: int = SIDE_CHEAPER) -> "DeviceGraph":
        h = ctypes.c_void_p()
        rc = load().bbc_ingest_graph(self._h, side_rule, ctypes.byref(h))
        if rc:
            _raise(rc)
        return DeviceGraph(h.value, self.device)

    def close(self) -> None:
        if self._h is not None and self._h.value:
            load().bbc_ingest_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ingest_text(data: bytes, policy: SignPolicy, device: int = 0) -> tuple[int, "Ingested | None", int]:
    """(status, handle or None, 1-based line of the first problem) of bbc_ingest_text."""
    counts = (ctypes.c_int64 * 3)()
    h = ctypes.c_void_p()
    rc = load().bbc_ingest_text(device, data, len(data), ctypes.byref(policy), counts, ctypes.byref(h))
    if rc:
        return rc, None, int(load().bbc_last_error_info())
    return 0, Ingested(h.value, device, int(counts[0]), int(counts[1]), int(counts[2])), 0


def enumerate_butterflies(n_u: int, n_v: int, u, v, s, device: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """Every butterfly on the device (bbc_enumerate_butterflies): (ids int32[B, 4] as
    (u1, u2, v1, v2) in lexicographic order, negative-sign bits uint8[B])."""
    u = np.ascontiguousarray(u, dtype=np.int32)
    v = np.ascontiguousarray(v, dtype=np.int32)
    s = np.ascontiguousarray(s, dtype=np.int8)
    L = load()
    cnt = ctypes.c_uint64(0)
    rc = L.bbc_enumerate_butterflies(device, n_u, n_v, len(u), u.ctypes.data, v.ctypes.data, s.ctypes.data,
                                     ctypes.byref(cnt), None, None, 0)
    if rc:
        _raise(rc)
    b = int(cnt.value)
    ids = np.empty((max(b, 1), 4), dtype=np.int32)
    bits = np.empty(max(b, 1), dtype=np.uint8)
    if b:
        rc = L.bbc_enumerate_butterflies(device, n_u, n_v, len(u), u.ctypes.data, v.ctypes.data, s.ctypes.data,
                                         ctypes.byref(cnt), ids.ctypes.data, bits.ctypes.data, b)
        if rc:
            _raise(rc)
    return ids[:b], bits[:b]
