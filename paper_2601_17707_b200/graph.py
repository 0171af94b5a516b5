"""Immutable signed bipartite graph (drop-in for pkg/src/bbcount/graph.py).

Storage is array-based instead of the reference's list-of-lists: the edges sorted by
(u, v) as int32/int32/int8 numpy arrays plus CSR offsets for both directions.  This is
what the device upload consumes directly (``include/bbc.h`` bbc_graph_create); the
reference's list attributes (``adj_u``, ``signs_u``, ``deg_u``, ``prank_u`` ...) are
materialised lazily for callers that use them.

Semantics kept from the reference:
  * ``build`` validates per edge in input order, u before v (graph.py:108-114), accepts
    ``EdgeSign`` members or +1/-1 (``EdgeSign(sign)``, graph.py:114), sorts by (u, v) and
    raises ``DuplicateEdgeError(u, v)`` at the first equal pair (graph.py:116-121);
  * priority rank = position in ascending (degree, index) order per side
    (graph.py:93-97, 230-235); ``priority_less`` compares (degree, global id)
    (graph.py:163-172) with global ids U-first (graph.py:140-143);
  * ``min_side`` = smaller partition, ties to U (graph.py:174-176);
  * ``fanout``, ``stats``, flip helpers as graph.py:178-217.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from .errors import DuplicateEdgeError, EmptySideError, IndexOutOfRangeError


class EdgeSign(enum.Enum):
    """Polarity of one edge; the value is used in sign products (graph.py:18-25)."""

    POSITIVE = 1
    NEGATIVE = -1

    def flipped(self) -> "EdgeSign":
        return EdgeSign.NEGATIVE if self is EdgeSign.POSITIVE else EdgeSign.POSITIVE


class Side(enum.Enum):
    U = "u"
    V = "v"

    def other(self) -> "Side":
        return Side.V if self is Side.U else Side.U


@dataclass(frozen=True)
class VertexRef:
    """A (side, index) vertex handle; indices are dense and 0-based per side."""

    side: Side
    index: int


@dataclass(frozen=True)
class GraphStats:
    """Smaller partition size, its average degree, density (graph.py:44-50)."""

    n_min: int
    d_min_avg: float
    density: float


def _sign_value(sign) -> int:
    if isinstance(sign, EdgeSign):
        return sign.value
    return EdgeSign(sign).value  # raises ValueError for anything but +1 / -1


def _priority_ranks(deg: np.ndarray) -> np.ndarray:
    order = np.argsort(deg, kind="stable")  # ascending degree, ties by ascending index
    ranks = np.empty(len(deg), dtype=np.int64)
    ranks[order] = np.arange(len(deg), dtype=np.int64)
    return ranks


class SignedBipartiteGraph:
    """Two-sided adjacency structure with per-edge signs, array-backed."""

    __slots__ = ("u_count", "v_count", "edge_count", "_eu", "_ev", "_es", "_off_u", "_perm_v", "_off_v",
                 "_deg_u", "_deg_v", "_lazy", "_device_cache", "__weakref__")

    def __init__(self, u_count: int, v_count: int, eu: np.ndarray, ev: np.ndarray, es: np.ndarray):
        """Arrays must be validated and sorted by (u, v); use ``build``/``from_arrays``."""
        self.u_count = int(u_count)
        self.v_count = int(v_count)
        self.edge_count = int(len(eu))
        self._eu = np.ascontiguousarray(eu, dtype=np.int32)
        self._ev = np.ascontiguousarray(ev, dtype=np.int32)
        self._es = np.ascontiguousarray(es, dtype=np.int8)
        self._deg_u = np.bincount(self._eu, minlength=self.u_count).astype(np.int64)
        self._deg_v = np.bincount(self._ev, minlength=self.v_count).astype(np.int64)
        self._off_u = np.zeros(self.u_count + 1, dtype=np.int64)
        np.cumsum(self._deg_u, out=self._off_u[1:])
        self._off_v = np.zeros(self.v_count + 1, dtype=np.int64)
        np.cumsum(self._deg_v, out=self._off_v[1:])
        # V-side lists: stable by v keeps ascending u (graph.py:128 "already sorted")
        self._perm_v = np.argsort(self._ev, kind="stable")
        self._lazy: dict = {}
        self._device_cache: dict = {}

    # -- construction -------------------------------------------------------

    @classmethod
    def build(cls, u_count: int, v_count: int, edges) -> "SignedBipartiteGraph":
        """Build from an iterable of (u, v, sign); validates ranges, rejects duplicates."""
        edges = list(edges)
        m = len(edges)
        u = np.empty(m, dtype=np.int64)
        v = np.empty(m, dtype=np.int64)
        s = np.empty(m, dtype=np.int8)
        for i, (a, b, sign) in enumerate(edges):
            if not 0 <= a < u_count:
                raise IndexOutOfRangeError(f"u index {a} out of range [0, {u_count})")
            if not 0 <= b < v_count:
                raise IndexOutOfRangeError(f"v index {b} out of range [0, {v_count})")
            u[i] = a
            v[i] = b
            s[i] = _sign_value(sign)
        return cls._from_valid(u_count, v_count, u, v, s)

    @classmethod
    def from_arrays(cls, u_count: int, v_count: int, u, v, sign) -> "SignedBipartiteGraph":
        """Vectorised ``build`` for large graphs: u, v integer arrays, sign in {+1, -1}."""
        u = np.asarray(u)
        v = np.asarray(v)
        s = np.asarray(sign)
        if not (u.shape == v.shape == s.shape) or u.ndim != 1:
            raise ValueError("u, v and sign must be 1-D arrays of equal length")
        bad_u = (u < 0) | (u >= u_count)
        bad_v = (v < 0) | (v >= v_count)
        bad_s = (s != 1) & (s != -1)
        bad = np.flatnonzero(bad_u | bad_v | bad_s)
        if len(bad):
            i = int(bad[0])
            if bad_u[i]:
                raise IndexOutOfRangeError(f"u index {int(u[i])} out of range [0, {u_count})")
            if bad_v[i]:
                raise IndexOutOfRangeError(f"v index {int(v[i])} out of range [0, {v_count})")
            raise ValueError(f"{int(s[i])} is not a valid EdgeSign")
        return cls._from_valid(u_count, v_count, u.astype(np.int64), v.astype(np.int64), s.astype(np.int8))

    @classmethod
    def _from_valid(cls, u_count, v_count, u, v, s) -> "SignedBipartiteGraph":
        if u_count >= 2**31 or v_count >= 2**31:
            raise ValueError("partition sizes must be below 2^31")
        key = (u.astype(np.int64) << 32) | v.astype(np.int64)
        order = np.argsort(key, kind="stable")
        key = key[order]
        if len(key) > 1:
            dup = np.flatnonzero(key[1:] == key[:-1])
            if len(dup):
                k = int(key[dup[0]])
                raise DuplicateEdgeError(k >> 32, k & 0xFFFFFFFF)
        return cls(u_count, v_count, (key >> 32).astype(np.int32), (key & 0xFFFFFFFF).astype(np.int32),
                   s[order])

    # -- array views (device upload) ------------------------------------------

    def edge_arrays(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """(u:int32, v:int32, sign:int8) sorted by (u, v); read-only views."""
        return self._eu, self._ev, self._es

    # -- reference list attributes (lazy) ---------------------------------------

    def _lists(self, side: Side):
        key = ("lists", side)
        if key not in self._lazy:
            if side is Side.U:
                off, nbr, sg = self._off_u, self._ev, self._es
            else:
                off, nbr, sg = self._off_v, self._eu[self._perm_v], self._es[self._perm_v]
            nl, sl = nbr.tolist(), sg.tolist()
            o = off.tolist()
            self._lazy[key] = ([nl[o[i]:o[i + 1]] for i in range(len(o) - 1)],
                               [sl[o[i]:o[i + 1]] for i in range(len(o) - 1)])
        return self._lazy[key]

    @property
    def adj_u(self) -> list[list[int]]:
        return self._lists(Side.U)[0]

    @property
    def signs_u(self) -> list[list[int]]:
        return self._lists(Side.U)[1]

    @property
    def adj_v(self) -> list[list[int]]:
        return self._lists(Side.V)[0]

    @property
    def signs_v(self) -> list[list[int]]:
        return self._lists(Side.V)[1]

    @property
    def deg_u(self) -> list[int]:
        return self._deg_u.tolist()

    @property
    def deg_v(self) -> list[int]:
        return self._deg_v.tolist()

    def degree_array(self, side: Side) -> np.ndarray:
        return self._deg_u if side is Side.U else self._deg_v

    def _prank(self, side: Side) -> np.ndarray:
        key = ("prank", side)
        if key not in self._lazy:
            self._lazy[key] = _priority_ranks(self.degree_array(side))
        return self._lazy[key]

    @property
    def prank_u(self) -> list[int]:
        return self._prank(Side.U).tolist()

    @property
    def prank_v(self) -> list[int]:
        return self._prank(Side.V).tolist()

    # -- basic queries ------------------------------------------------------------

    def side_count(self, side: Side) -> int:
        return self.u_count if side is Side.U else self.v_count

    def _check(self, ref: VertexRef) -> None:
        if not 0 <= ref.index < self.side_count(ref.side):
            raise IndexOutOfRangeError(f"{ref.side.name} index {ref.index} out of range")

    def degree(self, ref: VertexRef) -> int:
        self._check(ref)
        return int(self.degree_array(ref.side)[ref.index])

    def global_id(self, ref: VertexRef) -> int:
        """U keeps its index, V is offset by u_count (graph.py:140-143)."""
        self._check(ref)
        return ref.index if ref.side is Side.U else self.u_count + ref.index

    def neighbors(self, ref: VertexRef) -> list[int]:
        self._check(ref)
        if ref.side is Side.U:
            return self._ev[self._off_u[ref.index]:self._off_u[ref.index + 1]].tolist()
        sl = self._perm_v[self._off_v[ref.index]:self._off_v[ref.index + 1]]
        return self._eu[sl].tolist()

    def edge_sign(self, u: int, v: int) -> EdgeSign | None:
        """Sign of edge (u, v), or None when absent."""
        lo, hi = self._off_u[u], self._off_u[u + 1]
        i = lo + int(np.searchsorted(self._ev[lo:hi], v))
        if i < hi and self._ev[i] == v:
            return EdgeSign(int(self._es[i]))
        return None

    # -- priority / side selection ------------------------------------------------

    def priority_less(self, a: VertexRef, b: VertexRef) -> bool:
        da, db = self.degree(a), self.degree(b)
        if da != db:
            return da < db
        return self.global_id(a) < self.global_id(b)

    def min_side(self) -> Side:
        """The smaller partition (ties go to U)."""
        return Side.U if self.u_count <= self.v_count else Side.V

    def fanout(self, u: VertexRef) -> int:
        """Sum of neighbour degrees plus own degree (graph.py:178-182)."""
        self._check(u)
        other = self._deg_v if u.side is Side.U else self._deg_u
        return int(other[np.asarray(self.neighbors(u), dtype=np.int64)].sum()) + self.degree(u)

    def fanouts(self, side: Side) -> np.ndarray:
        """``fanout`` of every vertex of ``side`` (vectorised)."""
        if side is Side.U:
            per_edge = self._deg_v[self._ev]
            own, idx = self._deg_u, self._eu
        else:
            per_edge = self._deg_u[self._eu]
            own, idx = self._deg_v, self._ev
        return np.bincount(idx, weights=per_edge, minlength=len(own)).astype(np.int64) + own

    def stats(self) -> GraphStats:
        if self.u_count == 0 or self.v_count == 0:
            raise EmptySideError("stats need both partitions nonempty")
        n_min = min(self.u_count, self.v_count)
        return GraphStats(n_min=n_min, d_min_avg=float(Fraction(self.edge_count, n_min)),
                          density=float(Fraction(self.edge_count, self.u_count * self.v_count)))

    def side_arrays(self, side: Side):
        """(adjacency, signs, priority ranks, count) for one side (graph.py:195-199)."""
        adj, sg = self._lists(side)
        return adj, sg, self._prank(side).tolist(), self.side_count(side)

    def with_flipped_vertex(self, ref: VertexRef) -> "SignedBipartiteGraph":
        self._check(ref)
        touch = (self._eu == ref.index) if ref.side is Side.U else (self._ev == ref.index)
        s = np.where(touch, -self._es, self._es).astype(np.int8)
        return SignedBipartiteGraph(self.u_count, self.v_count, self._eu, self._ev, s)

    def with_all_flipped(self) -> "SignedBipartiteGraph":
        return SignedBipartiteGraph(self.u_count, self.v_count, self._eu, self._ev, (-self._es).astype(np.int8))

    def with_all_positive(self) -> "SignedBipartiteGraph":
        """Same structure, every sign +1 (its balanced count is the total count)."""
        return SignedBipartiteGraph(self.u_count, self.v_count, self._eu, self._ev, np.ones_like(self._es))

    def edges(self) -> list[tuple[int, int, EdgeSign]]:
        return [(a, b, EdgeSign(c)) for a, b, c in zip(self._eu.tolist(), self._ev.tolist(), self._es.tolist())]

    def __repr__(self) -> str:
        return f"SignedBipartiteGraph(|U|={self.u_count}, |V|={self.v_count}, |E|={self.edge_count})"


def build(u_count: int, v_count: int, edges) -> SignedBipartiteGraph:
    """Module-level alias for SignedBipartiteGraph.build (graph.py:238-241)."""
    return SignedBipartiteGraph.build(u_count, v_count, edges)
