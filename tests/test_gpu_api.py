"""The drop-in engines on the device, exercised the way the reference's own tests exercise
its engines (pkg/tests/test_buckets.py, test_tiled.py, test_oracle.py,
test_acceptance.py): cross-engine equality against the golden oracle counts, invariance
over tile sizes / grids / thresholds / sides, schedule-report properties, and the
sign-switching properties."""

import random

import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import fixtures
from paper_2601_17707_b200 import (
    CooperationRegime,
    Side,
    TileConfig,
    VertexRef,
    WedgeCounters,
    build,
    count_balanced_2k_serial,
    count_balanced_bruteforce,
    count_balanced_dynamic,
    count_balanced_parallel,
    count_balanced_tiled,
    count_signed_butterflies,
    load_imbalance,
    sign_product_total,
)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def corpus(golden):
    seed, count, mu, mv, pe, pp = fixtures.CORPORA["corpus_200"]
    return [(f.graph(), rec[4], rec[5]) for f, rec in zip(fixtures.corpus(seed, count, mu, mv, pe, pp),
                                                         golden["corpora"]["corpus_200"])]


def test_acceptance_1_engines_agree_with_oracle(gpu, corpus):
    for g, balanced, total in corpus[:60]:
        assert count_balanced_2k_serial(g, 2, Side.U) == balanced
        assert count_balanced_2k_serial(g, 2, Side.V) == balanced
        for workers in (1, 2, 8):
            assert count_balanced_parallel(g, workers) == balanced
        for tile in (1, 4, 64):
            assert count_balanced_tiled(g, TileConfig(tile, 4))[0] == balanced
        for blocks in (1, 4):
            assert count_balanced_dynamic(g, blocks)[0] == balanced
        assert count_balanced_bruteforce(g) == (balanced, total)


def test_acceptance_2_parity_identity(gpu, corpus):
    for g, balanced, total in corpus[:80]:
        assert 2 * balanced == total + sign_product_total(g)


def test_known_answers(gpu, golden):
    named = fixtures.named_fixtures()
    for name in ("complete_2x2", "complete_2x3", "one_negative", "dense_mixed_4x4", "two_negative_square", "tree"):
        rec = golden["named"][name]
        assert count_balanced_bruteforce(named[name].graph()) == (rec["balanced"], rec["total"])
    assert count_balanced_2k_serial(named["complete_2x2"].graph(), 2) == 1
    assert count_balanced_2k_serial(named["dense_mixed_4x4"].graph(), 2) == 19


def test_tiled_invariant_over_configs_and_report(gpu):
    rng = random.Random(606)
    for _ in range(25):
        g = fixtures.random_graph(rng).graph()
        expected = count_signed_butterflies(g)[0]
        w = None
        for tile in (1, 4, 64, max(1, g.side_count(g.min_side()))):
            for blocks in (1, 3, 8):
                count, report = count_balanced_tiled(g, TileConfig(tile, blocks))
                assert count == expected
                assert len(report.per_block_work) == blocks
                w = report.total_work if w is None else w
                assert report.total_work == w  # work independent of tiling and grid
        # the device anchors the side with fewer admitted wedges W_S
        assert w == min(sum(d * (d - 1) // 2 for d in g.deg_v), sum(d * (d - 1) // 2 for d in g.deg_u))


def test_tiled_hand_trace_complete_2x2(gpu):
    count, report = count_balanced_tiled(fixtures.complete_graph(2, 2).graph(), TileConfig(tile_size=1, block_count=1))
    assert count == 1
    assert report.per_block_work == [2]  # two admitted wedges (one per centre)
    assert sorted(report.task_order) == [0, 1]
    assert report.regime_histogram is None


def test_tiled_empty_processing_side(gpu):
    count, report = count_balanced_tiled(build(0, 3, []), TileConfig(4, 2))
    assert count == 0 and report.per_block_work == [0, 0]


def test_dynamic_counts_and_regimes(gpu):
    degrees = [10, 32, 31, 512, 600]
    g = build(5, 600, [(u, v, 1) for u, d in enumerate(degrees) for v in range(d)])
    count, report = count_balanced_dynamic(g, 2, mode="replay")
    assert count == count_signed_butterflies(g)[0]
    side = Side.U  # 5 anchors: far fewer admitted wedges than anchoring the 600 side
    assert report.regime_histogram == {CooperationRegime.WARP: 2, CooperationRegime.PARTIAL_BLOCK: 2,
                                       CooperationRegime.FULL_BLOCK: 1}
    assert sum(report.regime_histogram.values()) == g.side_count(side)


def test_dynamic_both_modes_and_invariance(gpu):
    rng = random.Random(117)
    for _ in range(20):
        g = fixtures.random_graph(rng).graph()
        expected = count_signed_butterflies(g)[0]
        for blocks in (1, 4, 7):
            for thresholds in ((1, 2), (32, 512), (2, 1000)):
                for mode in ("replay", "threads"):
                    assert count_balanced_dynamic(g, blocks, thresholds, mode)[0] == expected


def test_dynamic_task_order_is_work_sorted(gpu):
    g = build(3, 3, [(0, 0, 1), (1, 0, 1), (1, 1, 1), (2, 0, 1), (2, 1, 1), (2, 2, 1)])
    _, report = count_balanced_dynamic(g, 1, mode="replay")
    assert sorted(report.task_order) == [0, 1, 2]
    dg_work = report.per_block_work
    assert sum(dg_work) == report.total_work


def test_work_conservation_static_vs_dynamic(gpu):
    rng = random.Random(33)
    for _ in range(20):
        g = fixtures.random_graph(rng, 20, 20, 0.3).graph()
        _, static = count_balanced_tiled(g, TileConfig(4, 8))
        _, dynamic = count_balanced_dynamic(g, 8, mode="replay")
        _, threads = count_balanced_dynamic(g, 8, mode="threads")
        assert static.total_work == dynamic.total_work == threads.total_work


def test_acceptance_8_dynamic_beats_static_on_skew(gpu, golden):
    g = fixtures.skew_instance().graph()
    cs, static = count_balanced_tiled(g, TileConfig(64, 8))
    cd, dynamic = count_balanced_dynamic(g, 8, mode="replay")
    assert cs == cd == golden["named"]["skew_instance"]["balanced"]
    assert static.total_work == dynamic.total_work
    assert load_imbalance(dynamic) <= load_imbalance(static)


def test_wedge_counters_instrumentation(gpu):
    rng = random.Random(424)
    for _ in range(15):
        g = fixtures.random_graph(rng, 12, 12, 0.5).graph()
        counters = WedgeCounters()
        count_balanced_2k_serial(g, 2, Side.U, counters=counters)
        assert counters.admitted_per_anchor == counters.bucket_sums_per_anchor
        assert counters.admitted == sum(d * (d - 1) // 2 for d in g.deg_v)
        assert len(counters.admitted_per_anchor) == g.u_count
    counters = WedgeCounters()
    count_balanced_2k_serial(fixtures.complete_graph(5, 4).graph(), 2, Side.U, counters=counters)
    assert counters.admitted == 10 * 4


@st.composite
def signed_graphs(draw, max_u=8, max_v=8):
    nu = draw(st.integers(1, max_u))
    nv = draw(st.integers(1, max_v))
    cells = draw(st.sets(st.tuples(st.integers(0, nu - 1), st.integers(0, nv - 1)), max_size=nu * nv))
    signs = draw(st.lists(st.sampled_from((1, -1)), min_size=len(cells), max_size=len(cells)))
    return build(nu, nv, [(u, v, s) for (u, v), s in zip(sorted(cells), signs)])


@settings(max_examples=40, deadline=None)
@given(signed_graphs())
def test_sign_flip_closure_and_switching_invariance(g):
    bal, unb = count_signed_butterflies(g)
    assert count_signed_butterflies(g.with_all_flipped()) == (bal, unb)
    for index in range(0, g.u_count, 3):
        assert count_signed_butterflies(g.with_flipped_vertex(VertexRef(Side.U, index))) == (bal, unb)
    # total = balanced count of the all-positive graph
    assert count_signed_butterflies(g.with_all_positive()) == (bal + unb, 0)


def test_count_overflow_contract_small(gpu):
    from paper_2601_17707_b200.errors import checked_u64

    bal, unb = count_signed_butterflies(fixtures.complete_graph(30, 30).graph())
    assert bal == checked_u64(bal) and bal + unb == (30 * 29 // 2) ** 2
