"""ctypes wrapper of ``oracle/bbc_oracle.c`` -- TEST INFRASTRUCTURE ONLY.

The CPU restatement of the reference bucket engine (pkg/src/bbcount/buckets.py:166-197,
graph.py:99-129, 230-235) used as the parity checker in tests/, by
``__graft_entry__.smoke()`` and as bench.py's CPU baseline / ``--impl reference`` arm.
The product package must never import this module.

Parity pinned: tests/test_oracle_golden.py checks it against the golden vectors in
tests/golden/, which tests/golden/make_golden.py produced with the reference package.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().with_name("liboracle.so")
_lib = None

E_RANGE, E_DUP, E_OVERFLOW, E_ARG = 1, 2, 3, 4


class OracleError(Exception):
    def __init__(self, code: int, info: int):
        super().__init__(f"oracle error {code} (info {info})")
        self.code = code
        self.info = info


def _load():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            import subprocess
            import sys

            subprocess.run([sys.executable, "-c", "from paper_2601_17707_b200 import _build; _build.build_oracle()"],
                           check=True, cwd=str(LIB_PATH.parent.parent))
        L = ctypes.CDLL(str(LIB_PATH))
        P = ctypes.c_void_p
        L.bbc_oracle_graph_build.restype = ctypes.c_int
        L.bbc_oracle_graph_build.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, P, P, P,
                                             ctypes.POINTER(P), ctypes.POINTER(ctypes.c_int64)]
        L.bbc_oracle_count.restype = ctypes.c_int
        L.bbc_oracle_count.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int64, P]
        L.bbc_oracle_graph_free.argtypes = [P]
        L.bbc_oracle_graph_free.restype = None
        L.bbc_oracle_count_sorted.restype = ctypes.c_int
        L.bbc_oracle_count_sorted.argtypes = [P, ctypes.c_int, ctypes.c_int, P]
        L.bbc_oracle_count_2k.restype = ctypes.c_int
        L.bbc_oracle_count_2k.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, P]
        L.bbc_oracle_classify.restype = ctypes.c_int
        L.bbc_oracle_classify.argtypes = [P, ctypes.c_int, P]
        L.bbc_oracle_admitted_total.restype = ctypes.c_uint64
        L.bbc_oracle_admitted_total.argtypes = [P, ctypes.c_int]
        _lib = L
    return _lib


@dataclass
class OracleResult:
    balanced: int
    unbalanced: int
    admitted: int
    scanned: int
    side: int

    @property
    def total(self) -> int:
        return self.balanced + self.unbalanced


class OracleGraph:
    """Validated CPU adjacency (reference graph.py:99-129 semantics)."""

    def __init__(self, n_u: int, n_v: int, u, v, s):
        self.n_u, self.n_v = int(n_u), int(n_v)
        u = np.ascontiguousarray(u, dtype=np.int32)
        v = np.ascontiguousarray(v, dtype=np.int32)
        s = np.ascontiguousarray(s, dtype=np.int8)
        self.m = len(u)
        h = ctypes.c_void_p()
        info = ctypes.c_int64(0)
        rc = _load().bbc_oracle_graph_build(n_u, n_v, len(u), u.ctypes.data, v.ctypes.data, s.ctypes.data,
                                            ctypes.byref(h), ctypes.byref(info))
        if rc:
            raise OracleError(rc, int(info.value))
        self._h = h

    def count(self, side: int = -1, threads: int | None = None, stride: int = 1) -> OracleResult:
        """side: 0 = U, 1 = V, -1 = reference min_side; stride > 1 samples anchors a % stride == 0."""
        if threads is None:
            threads = len(os.sched_getaffinity(0))
        out = (ctypes.c_uint64 * 8)()
        rc = _load().bbc_oracle_count(self._h, side, threads, stride, out)
        if rc not in (0, E_OVERFLOW):
            raise OracleError(rc, 0)
        return OracleResult(balanced=int(out[0]) | (int(out[1]) << 64), unbalanced=int(out[2]) | (int(out[3]) << 64),
                            admitted=int(out[4]), scanned=int(out[5]), side=int(out[6]))

    def count_sorted(self, side: int = -1, threads: int | None = None) -> OracleResult:
        """The reference's sort_neighbors traversal (buckets.py:87-111, early exit at the
        anchor's rank): same counts, scanned = admitted + one stop per record."""
        out = (ctypes.c_uint64 * 8)()
        rc = _load().bbc_oracle_count_sorted(self._h, side, threads or len(os.sched_getaffinity(0)), out)
        if rc not in (0, E_OVERFLOW):
            raise OracleError(rc, 0)
        return OracleResult(balanced=int(out[0]) | (int(out[1]) << 64), unbalanced=int(out[2]) | (int(out[3]) << 64),
                            admitted=int(out[4]), scanned=int(out[5]), side=int(out[6]))

    def count_2k(self, k: int, side: int, threads: int | None = None) -> tuple[int, bool]:
        """Balanced (2,k)-bicliques with the size-2 side ``side`` (buckets.py:64-154):
        (total, overflowed past 2^64 - 1)."""
        out = (ctypes.c_uint64 * 8)()
        rc = _load().bbc_oracle_count_2k(self._h, side, k, threads or len(os.sched_getaffinity(0)), out)
        if rc not in (0, E_OVERFLOW):
            raise OracleError(rc, 0)
        return int(out[0]) | (int(out[1]) << 64), rc == E_OVERFLOW

    CLASS_NAMES = ("coherent_pp_pp", "coherent_pp_mm", "coherent_mm_mm", "incoherent_pm_pm", "mixed_pp_pm",
                   "mixed_pm_mm")

    def classify(self, threads: int | None = None) -> dict[str, int]:
        """Six-way butterfly classification (oracle.py:172-197), as_dict() keys."""
        out = (ctypes.c_uint64 * 20)()
        rc = _load().bbc_oracle_classify(self._h, threads or len(os.sched_getaffinity(0)), out)
        if rc not in (0, E_OVERFLOW):
            raise OracleError(rc, 0)
        return {n: int(out[8 + 2 * i]) | (int(out[9 + 2 * i]) << 64) for i, n in enumerate(self.CLASS_NAMES)}

    def admitted_total(self, side: int) -> int:
        return int(_load().bbc_oracle_admitted_total(self._h, side))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _load().bbc_oracle_graph_free(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def count(n_u, n_v, u, v, s, side: int = -1, threads: int | None = None) -> OracleResult:
    g = OracleGraph(n_u, n_v, u, v, s)
    try:
        return g.count(side, threads)
    finally:
        g.close()
