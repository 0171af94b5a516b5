"""Counting entry points of the drop-in API, all running on the B200 CUDA path.

Reference entry points kept (signatures, argument meaning, errors):

  count_balanced_parallel(g, workers, inline_below)   buckets.py:213-246  (M-BBC)
  count_balanced_2k_serial(g, k, anchor_side, ...)    buckets.py:64-154   (BB2K, k = 2)
  count_balanced_tiled(g, TileConfig)                 tiled.py:107-168    (G-BBC)
  count_balanced_dynamic(g, blocks, thresholds, mode) tiled.py:182-292    (G-BBC++)
  count_balanced_bruteforce(g) -> (balanced, total)   oracle.py:116-124
  sign_product_total(g)                               oracle.py:127-134
  classify_butterflies(g) -> ButterflyClassCounts     oracle.py:172-197

plus ``count_signed_butterflies(g, ...) -> (balanced, unbalanced)``, the unbalanced count
the reference only exposes through its brute-force oracle.

Every engine hands the graph to ``libbbc.so`` (device preprocessing K1-K5 and the
G-BBC / G-BBC++ kernels); nothing here counts on the host.  The device CSR is built once
per (graph, device, side rule) and cached on the immutable graph object.

Mapping of the reference's parallelism knobs onto the device:
  * ``workers`` (fork-pool size) -> number of GPUs in this process, clamped to the
    visible devices; the edge list is uploaded in shards and all-gathered over NVLink,
    every GPU builds the CSR, counts its start-vertex partition, and the exact sums are
    added by one NCCL all-reduce (``bbc_multi_*``, csrc/bbc_multi.cu);
  * ``TileConfig.tile_size`` -> end-vertex tile span of the shared-memory counters,
    ``TileConfig.block_count`` -> CTAs of the static G-BBC grid;
  * ``block_count`` of the dynamic engine -> persistent CTAs claiming from the global
    atomic queue; ``thresholds`` -> the regime bands reported in the histogram;
  * ``inline_below`` has no device meaning (there is no cheaper in-process path) and is
    only validated.
"""

from __future__ import annotations

import enum
import heapq
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import CountOverflowError, DeviceError, InvalidKError, InvalidThresholdsError, NoWorkError, U64_MAX
from .graph import EdgeSign, Side, SignedBipartiteGraph

DEFAULT_INLINE_BELOW = 250_000
DEFAULT_TILE_SIZE = 128
DEFAULT_WARP_MAX = 32
DEFAULT_PARTIAL_MAX = 512


# -- small host-side types (buckets.py:30-57, tiled.py:42-104) -------------------------

class WedgeKind(enum.Enum):
    SYMMETRIC = "symmetric"
    ASYMMETRIC = "asymmetric"


def wedge_kind(sign_uv: EdgeSign, sign_vw: EdgeSign) -> WedgeKind:
    """Symmetric iff the two edge signs are equal (device: sign bit of word ^ s(u,v))."""
    return WedgeKind.SYMMETRIC if sign_uv is sign_vw else WedgeKind.ASYMMETRIC


@dataclass
class WedgeCounters:
    """Instrumentation filled by ``count_balanced_2k_serial`` from device counters.

    ``admitted_per_anchor`` holds, per anchor id, the wedges admitted by the reference's
    filter prank[w] < prank[u] (buckets.py:96-153); every admitted wedge lands in a
    bucket, so ``bucket_sums_per_anchor`` equals it.  ``scanned`` counts the list entries
    the reference traversal examines (see count_balanced_2k_serial).
    """

    admitted_per_anchor: list[int] = field(default_factory=list)
    bucket_sums_per_anchor: list[int] = field(default_factory=list)
    scanned: int = 0

    @property
    def admitted(self) -> int:
        return sum(self.admitted_per_anchor)


def wedge_scan_bound(g: SignedBipartiteGraph, side: Side) -> int:
    """Sum over centres of deg^2 (buckets.py:53-57)."""
    d = g.degree_array(side.other()).astype(object)
    return int(sum(x * x for x in d.tolist()))


def admitted_wedges(g: SignedBipartiteGraph, side: Side) -> int:
    """W_S = sum over the centre side of C(deg, 2): admitted wedges for any once-per-pair filter."""
    d = g.degree_array(side.other())
    return int(sum(int(x) * (int(x) - 1) // 2 for x in d.tolist()))


class CooperationRegime(enum.Enum):
    WARP = "warp"
    PARTIAL_BLOCK = "partial_block"
    FULL_BLOCK = "full_block"


@dataclass(frozen=True)
class TileConfig:
    """tile_size bounds the per-tile counter span; block_count the CTAs (tiled.py:48-59)."""

    tile_size: int = DEFAULT_TILE_SIZE
    block_count: int = 1

    def __post_init__(self):
        if self.tile_size < 1:
            raise ValueError(f"tile_size must be >= 1, got {self.tile_size}")
        if self.block_count < 1:
            raise ValueError(f"block_count must be >= 1, got {self.block_count}")


@dataclass
class ScheduleReport:
    """Per-run load accounting (tiled.py:62-89), measured on the device.

    per_block_work: admitted wedges processed by each CTA; task_order: anchor ids in
    dispatch order; regime_histogram: anchors per cooperation band (dynamic engine only).
    """

    per_block_work: list[int]
    max_over_mean: float
    task_order: list[int]
    regime_histogram: dict[CooperationRegime, int] | None = None

    @property
    def total_work(self) -> int:
        return sum(self.per_block_work)

    def to_json_dict(self) -> dict:
        out: dict = {"per_block_work": self.per_block_work, "max_over_mean": self.max_over_mean,
                     "task_order": self.task_order}
        if self.regime_histogram is not None:
            out["regime_histogram"] = {r.value: n for r, n in self.regime_histogram.items()}
        return out


def _max_over_mean(work: list[int]) -> float:
    total = sum(work)
    if total == 0:
        return 1.0
    return max(work) / (total / len(work))


def load_imbalance(report: ScheduleReport) -> float:
    """max / mean of per_block_work; NoWorkError when there is none (tiled.py:100-104)."""
    if report.total_work == 0:
        raise NoWorkError("schedule report has no work")
    return _max_over_mean(report.per_block_work)


def regime_for_degree(degree: int, warp_max: int = DEFAULT_WARP_MAX,
                      partial_max: int = DEFAULT_PARTIAL_MAX) -> CooperationRegime:
    """WARP below warp_max, FULL_BLOCK above partial_max, PARTIAL_BLOCK between (tiled.py:171-179)."""
    if degree < warp_max:
        return CooperationRegime.WARP
    if degree <= partial_max:
        return CooperationRegime.PARTIAL_BLOCK
    return CooperationRegime.FULL_BLOCK


# -- device plumbing ---------------------------------------------------------------------

_SIDE_RULE = {None: _lib.SIDE_CHEAPER, Side.U: _lib.SIDE_U, Side.V: _lib.SIDE_V}


def device_graph(g: SignedBipartiteGraph, device: int = 0, side: Side | None = None) -> _lib.DeviceGraph:
    """The device CSR of ``g`` (built on first use, cached on the graph)."""
    key = (device, side)
    dg = g._device_cache.get(key)
    if dg is None:
        if _lib.device_count() <= device:
            raise DeviceError(f"CUDA device {device} is not available; the counter has no CPU fallback")
        u, v, s = g.edge_arrays()
        dg = _lib.DeviceGraph.from_host(g.u_count, g.v_count, u, v, s, device, _SIDE_RULE[side])
        g._device_cache[key] = dg
    return dg


def _devices(n: int) -> list[int]:
    avail = _lib.device_count()
    if avail < 1:
        raise DeviceError("no CUDA device visible; the counter has no CPU fallback")
    return list(range(min(max(n, 1), avail)))


def multi_graph(g: SignedBipartiteGraph, devices: list[int], side: Side | None = None) -> _lib.MultiGraph:
    """The graph replicated on ``devices`` (sharded upload + NCCL all-gather + replicated
    build, csrc/bbc_multi.cu), built on first use and cached on the graph."""
    key = ("multi", tuple(devices), side)
    mg = g._device_cache.get(key)
    if mg is None:
        u, v, s = g.edge_arrays()
        mg = _lib.MultiGraph(g.u_count, g.v_count, u, v, s, devices, _SIDE_RULE[side])
        g._device_cache[key] = mg
    return mg


def _count(g: SignedBipartiteGraph, devices: list[int], algo: int, side: Side | None = None, tile_span: int = 0,
           blocks: int = 0) -> tuple[int, int, list[_lib.CountResult]]:
    """Exact (balanced, unbalanced): one device, or start-vertex partitions over several
    GPUs summed by one NCCL all-reduce inside libbbc (bbc_multi_count)."""
    if len(devices) == 1:
        r = device_graph(g, devices[0], side).count(algo, tile_span, blocks)
    else:
        r = multi_graph(g, devices, side).count(algo, tile_span, blocks)
    return r.balanced, r.unbalanced, [r]


def _checked(balanced: int) -> int:
    if balanced > U64_MAX:
        raise CountOverflowError("balanced count exceeded 64-bit range")
    return balanced


# -- engines -----------------------------------------------------------------------------

def count_signed_butterflies(g: SignedBipartiteGraph, devices: int = 1, algo: str = "gbbc++",
                             anchor_side: Side | None = None) -> tuple[int, int]:
    """(balanced, unbalanced) butterfly counts on ``devices`` GPUs of this process.

    ``algo`` is "gbbc++" (dynamic queue) or "gbbc" (static); ``anchor_side`` None picks the
    side with fewer admitted wedges.  CountOverflowError if either exceeds 2^64 - 1.
    """
    if devices < 1:
        raise ValueError(f"devices must be >= 1, got {devices}")
    code = {"gbbc++": _lib.ALGO_GBBCPP, "gbbc": _lib.ALGO_GBBC}.get(algo)
    if code is None:
        raise ValueError(f"unknown algo {algo!r}")
    bal, unb, _ = _count(g, _devices(devices), code, anchor_side)
    if bal > U64_MAX or unb > U64_MAX:
        raise CountOverflowError("butterfly count exceeded 64-bit range")
    return bal, unb


def count_balanced_parallel(g: SignedBipartiteGraph, workers: int, inline_below: int = DEFAULT_INLINE_BELOW) -> int:
    """Balanced butterflies with start vertices split over ``workers`` GPUs (buckets.py:213-246)."""
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    bal, _, _ = _count(g, _devices(workers), _lib.ALGO_GBBCPP)
    return _checked(bal)


def _reference_work(g: SignedBipartiteGraph, side: Side) -> np.ndarray:
    """Admitted visits per anchor of ``side`` under the reference models' id filter w > u
    (tiled.py:143-156, 221-233): for each edge (u, c), the entries of c's id-sorted list
    above u.  Schedule accounting only -- the count itself always comes from the device."""
    eu, ev, _ = g.edge_arrays()  # sorted by (u, v)
    if side is Side.U:
        # position of u in v's list (V lists ascend in u): the stable order of ev
        perm = np.argsort(ev, kind="stable")
        pos = np.empty(len(ev), dtype=np.int64)
        off_v = np.zeros(g.v_count + 1, dtype=np.int64)
        np.cumsum(g.degree_array(Side.V), out=off_v[1:])
        pos[perm] = np.arange(len(ev), dtype=np.int64) - off_v[ev[perm]]
        per_edge = g.degree_array(Side.V)[ev] - 1 - pos
        idx, n = eu, g.u_count
    else:
        off_u = np.zeros(g.u_count + 1, dtype=np.int64)
        np.cumsum(g.degree_array(Side.U), out=off_u[1:])
        pos = np.arange(len(eu), dtype=np.int64) - off_u[eu]  # v's position in u's list
        per_edge = g.degree_array(Side.U)[eu] - 1 - pos
        idx, n = ev, g.v_count
    return np.bincount(idx, weights=per_edge, minlength=n).astype(np.int64)


def count_balanced_2k_serial(g: SignedBipartiteGraph, k: int, anchor_side: Side = Side.U,
                             sort_neighbors: bool = False, counters: WedgeCounters | None = None) -> int:
    """Balanced (2,k)-biclique count with the size-2 side on ``anchor_side`` (buckets.py:64-154).

    k = 2 (balanced butterflies) runs the count kernel anchored on ``anchor_side``; k > 2
    runs the same kernel with C(b1,k) + C(b2,k) closings (buckets.py:146) on the same
    device CSR.  ``sort_neighbors`` only changes what the reference's instrumentation
    counts as scanned (device lists are always rank-sorted).  CountOverflowError above
    2^64 - 1, like the reference.

    ``counters`` is filled as the reference fills it (buckets.py:96-153): per anchor id,
    the wedges admitted by its filter prank[w] < prank[u] -- derived from the device's
    per-anchor work under the mirrored filter: sum over c in N(u) of (deg c - 1) minus
    the device's admitted count -- and ``scanned`` = sum over centres of deg^2 (every
    list fully scanned, buckets.py:53-57) or, with ``sort_neighbors``, admitted plus one
    early-exit stop per anchor-side edge (:106-107).
    """
    if k < 2:
        raise InvalidKError(f"k must be >= 2, got {k}")
    if g.side_count(anchor_side) == 0:
        return 0
    if k > 2:
        _devices(1)
        bal, overflow, _ = device_graph(g, 0, anchor_side).count_2k(k)
        if overflow:
            raise CountOverflowError(f"balanced (2,{k}) count exceeded 64-bit range")
    else:
        bal, _, _ = _count(g, _devices(1), _lib.ALGO_GBBCPP, anchor_side)
    if counters is not None:
        dg = device_graph(g, 0, anchor_side)
        ids, work = dg.task_order(_lib.ALGO_GBBC)
        mirrored = np.zeros(g.side_count(anchor_side), dtype=np.int64)
        mirrored[ids] = work.astype(np.int64)
        deg = g.degree_array(anchor_side)
        centre_sum = g.fanouts(anchor_side) - deg  # sum over c in N(u) of deg c
        per = centre_sum - deg - mirrored
        counters.admitted_per_anchor.extend(per.tolist())
        counters.bucket_sums_per_anchor.extend(per.tolist())
        if sort_neighbors:
            counters.scanned += int(per.sum()) + g.edge_count
        else:
            counters.scanned += wedge_scan_bound(g, anchor_side)
    return _checked(bal)


def count_balanced_tiled(g: SignedBipartiteGraph, cfg: TileConfig) -> tuple[int, ScheduleReport]:
    """G-BBC (tiled.py:107-168): the count from the device's static round-robin kernel
    (BBC_ALGO_GBBC, a full persistent grid and the native shared-memory tiles -- the
    count is independent of the tiling); the report as the reference defines it for
    ``cfg``: anchors of min_side in id order, block b doing anchors b, b + B, ...,
    per_block_work = admitted visits under the id filter w > u (tiled.py:137-156)."""
    blocks = cfg.block_count
    side = g.min_side()
    n = g.side_count(side)
    if n == 0:
        return 0, ScheduleReport([0] * blocks, 1.0, [])
    bal, _, _ = _count(g, _devices(1), _lib.ALGO_GBBC, side)
    per_anchor = _reference_work(g, side)
    work = np.bincount(np.arange(n) % blocks, weights=per_anchor, minlength=blocks).astype(np.int64).tolist()
    return _checked(bal), ScheduleReport(work, _max_over_mean(work), list(range(n)))


def count_balanced_dynamic(g: SignedBipartiteGraph, block_count: int,
                           thresholds: tuple[int, int] = (DEFAULT_WARP_MAX, DEFAULT_PARTIAL_MAX),
                           mode: str = "threads") -> tuple[int, ScheduleReport]:
    """G-BBC++ (tiled.py:182-292) on min_side: task_order = anchors by (-fanout, id)
    (:213-214), the regime histogram by anchor degree (:215-216).

    ``mode="threads"``: ``block_count`` persistent CTAs claim descending-work anchors from
    the device's global atomic queue, and per_block_work is each CTA's admitted wedges
    measured on the device (the split varies run to run, the count and the total work
    do not -- as with the reference's threads).  ``mode="replay"``: the count from a
    full-grid launch and the reference's deterministic least-loaded-claims-next replay
    (:243-258) of the fanout order with the id-filter work per anchor.
    """
    warp_max, partial_max = thresholds
    if warp_max >= partial_max:
        raise InvalidThresholdsError(f"warp_max {warp_max} must be below partial_max {partial_max}")
    if block_count < 1:
        raise ValueError(f"block_count must be >= 1, got {block_count}")
    if mode not in ("threads", "replay"):
        raise ValueError(f"unknown mode {mode!r}")
    side = g.min_side()
    n = g.side_count(side)
    histogram = {r: 0 for r in CooperationRegime}
    if n == 0:
        return 0, ScheduleReport([0] * block_count, 1.0, [], histogram)
    deg = g.degree_array(side)
    histogram[CooperationRegime.WARP] = int((deg < warp_max).sum())
    histogram[CooperationRegime.FULL_BLOCK] = int((deg > partial_max).sum())
    histogram[CooperationRegime.PARTIAL_BLOCK] = n - histogram[CooperationRegime.WARP] - \
        histogram[CooperationRegime.FULL_BLOCK]
    fan = g.fanouts(side)
    order = np.lexsort((np.arange(n), -fan)).tolist()
    if mode == "threads":
        dg = device_graph(g, _devices(1)[0], side)
        r = dg.count(_lib.ALGO_GBBCPP, blocks=block_count)
        bal = r.balanced
        work = dg.block_work(block_count)
    else:
        bal, _, _ = _count(g, _devices(1), _lib.ALGO_GBBCPP, side)
        per_anchor = _reference_work(g, side).tolist()
        work = [0] * block_count
        clocks = [(0, b) for b in range(block_count)]
        for u in order:
            clock, b = heapq.heappop(clocks)
            work[b] += per_anchor[u]
            heapq.heappush(clocks, (clock + per_anchor[u], b))
    return _checked(bal), ScheduleReport(work, _max_over_mean(work), order, histogram)


def count_balanced_bruteforce(g: SignedBipartiteGraph) -> tuple[int, int]:
    """(balanced, total) butterflies (oracle.py:116-124); total = balanced + unbalanced."""
    bal, unb = count_signed_butterflies(g)
    return bal, bal + unb


def sign_product_total(g: SignedBipartiteGraph) -> int:
    """Sum over butterflies of the product of the four signs = balanced - unbalanced."""
    bal, unb = count_signed_butterflies(g)
    return bal - unb


@dataclass(frozen=True)
class Butterfly:
    """Canonical 4-cycle (oracle.py:19-28): u1 < u2, v1 < v2; signs in the order
    (u1-v1, u1-v2, u2-v1, u2-v2)."""

    u1: int
    u2: int
    v1: int
    v2: int
    signs: tuple[EdgeSign, EdgeSign, EdgeSign, EdgeSign]


def enumerate_butterflies(g: SignedBipartiteGraph):
    """Yield every butterfly once, in (u1, u2, v1, v2) lexicographic order
    (oracle.py:73-107), enumerated on the device (csrc/bbc_enum.cu: wedges through each
    centre, stable radix sort by vertex pair, C(r, 2) butterflies per run of r common
    centres).  Materialises all of them: a test-scale API, like the reference's."""
    if g.u_count == 0 or g.v_count == 0 or g.edge_count == 0:
        return
    _devices(1)
    u, v, s = g.edge_arrays()
    ids, bits = _lib.enumerate_butterflies(g.u_count, g.v_count, u, v, s, 0)
    P, N = EdgeSign.POSITIVE, EdgeSign.NEGATIVE
    for (u1, u2, v1, v2), b in zip(ids.tolist(), bits.tolist()):
        yield Butterfly(u1, u2, v1, v2, (N if b & 1 else P, N if b & 2 else P, N if b & 4 else P, N if b & 8 else P))


def is_balanced(b: Butterfly) -> bool:
    """Even number of negative edges (oracle.py:110-113)."""
    return sum(1 for s in b.signs if s is EdgeSign.NEGATIVE) % 2 == 0


def count_balanced_2k_bruteforce(g: SignedBipartiteGraph, k: int, anchor_side: Side = Side.U) -> int:
    """Balanced (2,k)-bicliques with the size-2 side on ``anchor_side`` (oracle.py:137-169).

    A (2,k)-biclique is balanced iff every butterfly in it is, i.e. iff its k centres all
    make wedges of one kind with the pair -- exactly C(b1,k) + C(b2,k) per pair, which the
    device's (2,k) kernel computes (same result as the reference's subset enumeration).
    """
    return count_balanced_2k_serial(g, k, anchor_side)


@dataclass
class ButterflyClassCounts:
    """Six-way split by the two wedges through v1, v2 (endpoints u1, u2) -- the reference's
    oracle.ButterflyClassCounts (oracle.py:31-64), filled from the device."""

    coherent_pp_pp: int = 0
    coherent_pp_mm: int = 0
    coherent_mm_mm: int = 0
    incoherent_pm_pm: int = 0
    mixed_pp_pm: int = 0
    mixed_pm_mm: int = 0

    def total(self) -> int:
        return (self.coherent_pp_pp + self.coherent_pp_mm + self.coherent_mm_mm
                + self.incoherent_pm_pm + self.mixed_pp_pm + self.mixed_pm_mm)

    def balanced(self) -> int:
        """Coherent plus incoherent: exactly the balanced butterflies."""
        return self.coherent_pp_pp + self.coherent_pp_mm + self.coherent_mm_mm + self.incoherent_pm_pm

    def as_dict(self) -> dict[str, int]:
        return {
            "coherent_pp_pp": self.coherent_pp_pp,
            "coherent_pp_mm": self.coherent_pp_mm,
            "coherent_mm_mm": self.coherent_mm_mm,
            "incoherent_pm_pm": self.incoherent_pm_pm,
            "mixed_pp_pm": self.mixed_pp_pm,
            "mixed_pm_mm": self.mixed_pm_mm,
        }


def classify_butterflies(g: SignedBipartiteGraph, devices: int = 1, algo: str = "gbbc++") -> ButterflyClassCounts:
    """Tally the six wedge-pattern classes over all butterflies (oracle.py:172-197).

    Runs the classification kernel (csrc/bbc_ext.cu) on a U-anchored device CSR (the
    classes pair U vertices over V centres, oracle.py:176-178), with start vertices split
    over ``devices`` GPUs of this process and the exact sums added.
    """
    if devices < 1:
        raise ValueError(f"devices must be >= 1, got {devices}")
    code = {"gbbc++": _lib.ALGO_GBBCPP, "gbbc": _lib.ALGO_GBBC}.get(algo)
    if code is None:
        raise ValueError(f"unknown algo {algo!r}")
    if g.u_count == 0 or g.v_count == 0:
        return ButterflyClassCounts()
    devs = _devices(devices)
    graphs = [device_graph(g, d, Side.U) for d in devs]
    results: list = [None] * len(graphs)
    errors: list = []

    def run(i: int) -> None:
        try:
            results[i] = graphs[i].classify(code, part_index=i, part_count=len(graphs))[0]
        except BaseException as e:  # re-raised on the caller's thread
            errors.append(e)

    threads = [threading.Thread(target=run, args=(i,)) for i in range(len(graphs))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    total = {k: sum(r[k] for r in results) for k in results[0]}
    return ButterflyClassCounts(**total)
