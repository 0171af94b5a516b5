"""Host-side behaviour of the drop-in API (CPU only): graph construction and validation,
ingest, schedule types, argument validation of the engines, and the no-fallback contract.
Mirrors the reference's own unit tests (pkg/tests/test_graph.py, test_ingest.py,
test_tiled.py) for the parts that do not count."""

import io
import random

import numpy as np
import pytest

import fixtures
from paper_2601_17707_b200 import (
    CooperationRegime,
    DeviceError,
    DuplicateEdgeError,
    EdgeSign,
    EmptySideError,
    ExplicitSign,
    IndexOutOfRangeError,
    InvalidKError,
    InvalidSignValueError,
    InvalidThresholdsError,
    MalformedLineError,
    MissingValueError,
    NoWorkError,
    RandomBernoulli,
    RatingThreshold,
    RawEdge,
    ScheduleReport,
    Side,
    SignedBipartiteGraph,
    TileConfig,
    VertexRef,
    WedgeKind,
    admitted_wedges,
    apply_sign_policy,
    build,
    checked_u64,
    count_balanced_2k_serial,
    count_balanced_dynamic,
    count_balanced_parallel,
    dedup_latest,
    dump_edge_list,
    load_graph,
    load_imbalance,
    parse_edge_list,
    regime_for_degree,
    wedge_kind,
    wedge_scan_bound,
)


# -- graph (graph.py semantics) ----------------------------------------------------------

def test_build_complete_2x2():
    g = fixtures.complete_graph(2, 2).graph()
    assert g.edge_count == 4 and g.deg_u == [2, 2] and g.deg_v == [2, 2]


def test_build_empty_and_lists():
    g = build(1, 1, [])
    assert g.edge_count == 0 and g.adj_u == [[]] and g.adj_v == [[]]


def test_duplicate_rejected_regardless_of_sign_first_in_uv_order():
    with pytest.raises(DuplicateEdgeError) as e:
        build(3, 3, [(2, 2, 1), (1, 0, 1), (2, 2, -1), (1, 0, -1)])
    assert (e.value.u, e.value.v) == (1, 0)


@pytest.mark.parametrize("edge,msg", [((2, 0, 1), "u index 2 out of range"), ((0, 2, 1), "v index 2 out of range"),
                                      ((-1, 0, 1), "u index -1"), ((0, -1, 1), "v index -1")])
def test_index_out_of_range(edge, msg):
    with pytest.raises(IndexOutOfRangeError, match=msg):
        build(2, 2, [edge])


def test_invalid_sign_raises_value_error():
    with pytest.raises(ValueError):
        build(2, 2, [(0, 0, 0)])
    with pytest.raises(ValueError):
        SignedBipartiteGraph.from_arrays(2, 2, [0], [0], [3])


def test_from_arrays_matches_build():
    rng = random.Random(5)
    for _ in range(20):
        f = fixtures.random_graph(rng, 12, 12, 0.4)
        g1 = build(f.n_u, f.n_v, f.edges())
        g2 = SignedBipartiteGraph.from_arrays(f.n_u, f.n_v, f.u, f.v, f.s)
        assert g1.edges() == g2.edges()
        assert g1.adj_v == g2.adj_v and g1.signs_v == g2.signs_v
        assert g1.prank_u == g2.prank_u and g1.prank_v == g2.prank_v


def test_adjacency_symmetry_and_sorting():
    rng = random.Random(91)
    for _ in range(30):
        g = fixtures.random_graph(rng, 12, 12, 0.4).graph()
        for u in range(g.u_count):
            assert g.adj_u[u] == sorted(g.adj_u[u])
            for v, s in zip(g.adj_u[u], g.signs_u[u]):
                assert g.signs_v[v][g.adj_v[v].index(u)] == s
        for v in range(g.v_count):
            assert g.adj_v[v] == sorted(g.adj_v[v])
        assert sum(g.deg_u) == g.edge_count == sum(g.deg_v)


def test_priority_ranks_are_degree_then_id():
    rng = random.Random(7)
    for _ in range(20):
        g = fixtures.random_graph(rng, 15, 15, 0.3).graph()
        for side, deg, prank in ((Side.U, g.deg_u, g.prank_u), (Side.V, g.deg_v, g.prank_v)):
            order = sorted(range(len(deg)), key=lambda i: (deg[i], i))
            assert [prank[i] for i in order] == list(range(len(deg)))


def test_priority_less_and_global_id():
    g = build(2, 3, [(0, 0, 1), (1, 0, 1), (1, 1, 1), (1, 2, 1)])
    assert g.priority_less(VertexRef(Side.U, 0), VertexRef(Side.U, 1))
    c = fixtures.complete_graph(3, 3).graph()
    assert c.priority_less(VertexRef(Side.U, 2), VertexRef(Side.V, 0))
    assert not c.priority_less(VertexRef(Side.U, 1), VertexRef(Side.U, 1))
    assert c.global_id(VertexRef(Side.V, 1)) == 4


def test_min_side_fanout_stats():
    g = build(3, 3, [(0, 0, 1), (1, 0, 1), (1, 1, 1), (2, 0, 1), (2, 1, 1), (2, 2, 1)])
    assert [g.fanout(VertexRef(Side.U, u)) for u in range(3)] == [4, 7, 9]
    assert g.fanouts(Side.U).tolist() == [4, 7, 9]
    assert build(2, 2, []).min_side() is Side.U and build(3, 2, []).min_side() is Side.V
    s = build(145, 1201, [(i // 1201, i % 1201, 1) for i in range(27083)]).stats()
    assert s.n_min == 145 and f"{s.d_min_avg:.4g}" == "186.8"
    assert s.density == pytest.approx(27083 / 174145, rel=1e-12)
    with pytest.raises(EmptySideError):
        build(0, 2, []).stats()


def test_flips_and_edge_sign():
    g = fixtures.dense_mixed_4x4().graph()
    assert g.edge_sign(2, 0) is EdgeSign.NEGATIVE and g.edge_sign(0, 0) is EdgeSign.POSITIVE
    f = g.with_flipped_vertex(VertexRef(Side.U, 2))
    assert f.edge_sign(2, 0) is EdgeSign.POSITIVE and f.edge_sign(2, 1) is EdgeSign.NEGATIVE
    a = g.with_all_flipped()
    assert all(a.edge_sign(u, v) is s.flipped() for u, v, s in g.edges())
    assert all(s is EdgeSign.POSITIVE for _, _, s in g.with_all_positive().edges())


# -- ingest (ingest.py semantics) --------------------------------------------------------

def test_parse_edge_list_ids_and_comments():
    r = parse_edge_list("% c\n# c\n\na x 1\nb x -1 7\na y 0.5\n")
    assert r.u_ids == {"a": 0, "b": 1} and r.v_ids == {"x": 0, "y": 1}
    assert r.edges[1] == RawEdge("b", "x", -1.0, 7)


@pytest.mark.parametrize("text", ["a\n", "a b c d e\n", "a b zz\n", "a b 1 t\n"])
def test_parse_malformed(text):
    with pytest.raises(MalformedLineError) as e:
        parse_edge_list("ok ok 1\n" + text)
    assert e.value.line_number == 2


def test_sign_policies():
    edges = [RawEdge("a", "b", 1), RawEdge("a", "c", 0), RawEdge("a", "d", -1)]
    assert [s for *_, s, _ in apply_sign_policy(edges, ExplicitSign())] == [
        EdgeSign.POSITIVE, EdgeSign.NEGATIVE, EdgeSign.NEGATIVE]
    with pytest.raises(InvalidSignValueError):
        apply_sign_policy([RawEdge("a", "b", 2)], ExplicitSign())
    with pytest.raises(MissingValueError):
        apply_sign_policy([RawEdge("a", "b")], ExplicitSign())
    strict = RatingThreshold(6, at_or_above_is_positive=False)
    assert [s for *_, s, _ in apply_sign_policy([RawEdge("a", "b", 6), RawEdge("a", "c", 7)], strict)] == [
        EdgeSign.NEGATIVE, EdgeSign.POSITIVE]
    with pytest.raises(ValueError):
        RandomBernoulli(1.5, 0)
    with pytest.raises(TypeError):
        apply_sign_policy(edges, object())


def test_bernoulli_reproducible_and_calibrated():
    edges = [RawEdge(str(i), str(i % 997)) for i in range(20_000)]
    a = apply_sign_policy(edges, RandomBernoulli(0.7, seed=20260810))
    b = apply_sign_policy(edges, RandomBernoulli(0.7, seed=20260810))
    assert a == b
    frac = sum(s is EdgeSign.POSITIVE for _, _, s, _ in a) / len(a)
    assert abs(frac - 0.7) < 0.015


def test_bernoulli_known_answers():
    """Pinned against the reference's keyed blake2b draw (ingest.py:118-123)."""
    import hashlib

    for seed, ordinal in ((0, 0), (42, 7), (20260810, 123456)):
        d = hashlib.blake2b(ordinal.to_bytes(8, "little"), key=seed.to_bytes(8, "little"), digest_size=8).digest()
        unit = int.from_bytes(d, "little") / 2.0**64
        got = apply_sign_policy([RawEdge("u", "v")] * (ordinal + 1), RandomBernoulli(0.5, seed))[ordinal][2]
        assert got is (EdgeSign.POSITIVE if unit < 0.5 else EdgeSign.NEGATIVE)


def test_dedup_latest_and_load_roundtrip():
    signed = [("a", "x", EdgeSign.POSITIVE, None), ("a", "x", EdgeSign.NEGATIVE, 5),
              ("b", "x", EdgeSign.POSITIVE, 3), ("a", "x", EdgeSign.POSITIVE, 5), ("b", "x", EdgeSign.NEGATIVE, 1)]
    assert dedup_latest(signed) == [("a", "x", EdgeSign.POSITIVE), ("b", "x", EdgeSign.POSITIVE)]
    g = load_graph("a x 1\na y -1\nb x 1\n")
    out = io.StringIO()
    dump_edge_list(g, out)
    assert out.getvalue().splitlines() == ["0 0 1", "0 1 -1", "1 0 1"]


# -- schedule types and engine argument validation --------------------------------------

@pytest.mark.parametrize("degree,expected", [(10, CooperationRegime.WARP), (31, CooperationRegime.WARP),
                                             (32, CooperationRegime.PARTIAL_BLOCK),
                                             (512, CooperationRegime.PARTIAL_BLOCK),
                                             (513, CooperationRegime.FULL_BLOCK)])
def test_regime_bands(degree, expected):
    assert regime_for_degree(degree) is expected


def test_load_imbalance_and_report_shape():
    assert load_imbalance(ScheduleReport([10, 10, 10], 1.0, [])) == 1.0
    assert load_imbalance(ScheduleReport([30, 10, 20], 1.5, [])) == 1.5
    with pytest.raises(NoWorkError):
        load_imbalance(ScheduleReport([0, 0], 1.0, []))
    r = ScheduleReport([1], 1.0, [0], {c: 0 for c in CooperationRegime})
    assert set(r.to_json_dict()) == {"per_block_work", "max_over_mean", "task_order", "regime_histogram"}
    assert "regime_histogram" not in ScheduleReport([1], 1.0, [0]).to_json_dict()


def test_argument_validation_happens_before_device_use():
    g = fixtures.complete_graph(2, 2).graph()
    with pytest.raises(ValueError):
        TileConfig(0, 1)
    with pytest.raises(ValueError):
        TileConfig(4, 0)
    with pytest.raises(ValueError):
        count_balanced_parallel(g, 0)
    with pytest.raises(InvalidKError):
        count_balanced_2k_serial(g, 1)
    with pytest.raises(InvalidThresholdsError):
        count_balanced_dynamic(g, 1, thresholds=(512, 32))
    with pytest.raises(ValueError):
        count_balanced_dynamic(g, 0)
    with pytest.raises(ValueError):
        count_balanced_dynamic(g, 1, mode="bogus")


def test_no_cpu_fallback_without_gpu(native_built):
    from conftest import has_gpu

    if has_gpu():
        pytest.skip("a GPU is visible")
    with pytest.raises(DeviceError):
        count_balanced_parallel(fixtures.complete_graph(2, 2).graph(), 1)


def test_wedge_helpers():
    P, N = EdgeSign.POSITIVE, EdgeSign.NEGATIVE
    assert wedge_kind(P, P) is WedgeKind.SYMMETRIC and wedge_kind(N, N) is WedgeKind.SYMMETRIC
    assert wedge_kind(P, N) is WedgeKind.ASYMMETRIC
    g = fixtures.complete_graph(5, 4).graph()
    assert wedge_scan_bound(g, Side.U) == 100 and admitted_wedges(g, Side.U) == 40
    assert checked_u64(2**64 - 1) == 2**64 - 1


def test_synth_generator_deterministic_and_distinct(native_built):
    from paper_2601_17707_b200 import synth

    cfg = synth.CONFIGS[2].scaled(0.002)
    a = synth.generate(cfg)
    b = synth.generate(cfg)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    key = a[0].astype(np.int64) * cfg.n_v + a[1]
    assert len(np.unique(key)) == cfg.m
    assert (a[0] < cfg.n_u).all() and (a[1] < cfg.n_v).all() and set(np.unique(a[2])) <= {-1, 1}


def _policy(p):
    if p[0] == "explicit":
        return ExplicitSign()
    if p[0] == "rating":
        return RatingThreshold(p[1], p[2])
    return RandomBernoulli(p[1], p[2])


def test_host_loader_matches_reference_ingest_vectors(golden):
    """The host loader against the reference's load_graph on the same texts
    (tests/golden/make_golden.py --ingest)."""
    from paper_2601_17707_b200 import synth

    for name, (seed, n, nu, nv, kind, pol) in fixtures.INGEST_CASES.items():
        text = fixtures.ingest_text(seed, n, nu, nv, kind)
        rec = golden["ingest"][name]
        assert len(text) == rec["text_len"], name
        g = load_graph(text, _policy(pol))
        u, v, s = g.edge_arrays()
        assert (g.u_count, g.v_count, g.edge_count) == (rec["n_u"], rec["n_v"], rec["m"]), name
        assert synth.edge_digest(u, v, s) == rec["digest"], name
