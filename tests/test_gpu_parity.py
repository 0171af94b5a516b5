"""Parity of the CUDA path (through the C ABI / drop-in API) with the reference's golden
vectors and the CPU oracle.  Bit-exact: every count is an integer."""

import numpy as np
import pytest

import fixtures
from paper_2601_17707_b200 import _lib, synth
from paper_2601_17707_b200._lib import ALGO_GBBC, ALGO_GBBCPP, SIDE_CHEAPER, SIDE_MIN, SIDE_U, SIDE_V, DeviceGraph

pytestmark = pytest.mark.gpu

ALGOS = (ALGO_GBBC, ALGO_GBBCPP)


def dev_counts(f_or_arrays, side=SIDE_CHEAPER, algo=ALGO_GBBCPP, tile_span=0, blocks=0):
    n_u, n_v, u, v, s = f_or_arrays.arrays() if hasattr(f_or_arrays, "arrays") else f_or_arrays
    g = DeviceGraph.from_host(n_u, n_v, u, v, s, 0, side)
    try:
        r = g.count(algo, tile_span, blocks)
        return r
    finally:
        g.close()


def test_named_fixtures_all_sides_and_algos(gpu, golden):
    for name, f in fixtures.named_fixtures().items():
        rec = golden["named"][name]
        for side in (SIDE_CHEAPER, SIDE_U, SIDE_V, SIDE_MIN):
            for algo in ALGOS:
                r = dev_counts(f, side, algo)
                assert (r.balanced, r.unbalanced) == (rec["balanced"], rec["unbalanced"]), (name, side, algo)


def test_named_fixtures_tile_spans_and_grids(gpu, golden):
    for name in ("dense_mixed_4x4", "skew_instance", "degree_bands", "complete_5x4", "star_u"):
        f = fixtures.named_fixtures()[name]
        rec = golden["named"][name]
        for tile in (1, 3, 4, 64, 1000):
            for blocks in (1, 3, 8, 300):
                for algo in ALGOS:
                    r = dev_counts(f, SIDE_CHEAPER, algo, tile, blocks)
                    assert (r.balanced, r.unbalanced) == (rec["balanced"], rec["unbalanced"]), (name, tile, blocks)


def test_smoke_graph(gpu, golden):
    rec = golden["named"]["smoke_graph"]
    f = fixtures.smoke_graph()
    for side in (SIDE_CHEAPER, SIDE_U, SIDE_V):
        for algo in ALGOS:
            r = dev_counts(f, side, algo)
            assert (r.balanced, r.unbalanced) == (rec["balanced"], rec["unbalanced"])


@pytest.mark.parametrize("corpus", list(fixtures.CORPORA))
def test_corpora(gpu, golden, corpus):
    seed, count, mu, mv, pe, pp = fixtures.CORPORA[corpus]
    for i, (f, rec) in enumerate(zip(fixtures.corpus(seed, count, mu, mv, pe, pp), golden["corpora"][corpus])):
        algo = ALGOS[i % 2]
        side = (SIDE_CHEAPER, SIDE_U, SIDE_V)[i % 3]
        r = dev_counts(f, side, algo, tile_span=(0, 4, 7)[i % 3])
        assert (r.balanced, r.balanced + r.unbalanced) == (rec[4], rec[5]), (corpus, i)


@pytest.mark.parametrize("key", ["1@1", "2@0.01", "2@0.05", "3@0.002", "4@0.0002", "5@small"])
def test_synthetic_configs_vs_reference(gpu, golden, key):
    rec = golden["configs"][key]
    cfg = synth.golden_config(key)
    u, v, s = synth.generate(cfg)
    assert synth.edge_digest(u, v, s) == rec["digest"]
    for side in (SIDE_CHEAPER, SIDE_U, SIDE_V):
        for algo in ALGOS:
            g = DeviceGraph.from_host(cfg.n_u, cfg.n_v, u, v, s, 0, side)
            # every cold-range strategy: default, general banded path, hash rounds (8192),
            # forced bitmap rounds (normal / tiny repeat queue: overflow + narrowing),
            # tiles only (128), sweep-closed tiles (2048), two launches (64)
            # (1024: band boundaries by binary search instead of the table)
            for flags in (0, _lib.FLAG_BANDED_ONLY, 8192, 512, 512 | 256, 128, 128 | 2048, 64, 1024, 1024 | 512,
                          1024 | 8192):
                r = g.count(algo, flags=flags)
                assert (r.balanced, r.unbalanced) == (rec["balanced"], rec["unbalanced"]), (key, side, algo, flags)
                assert r.wedges == r.wedges_total == (rec["w_u"] if g.anchor_side == 0 else rec["w_v"])
            assert (g.w_u, g.w_v) == (rec["w_u"], rec["w_v"])
            g.close()


@pytest.mark.parametrize("key", ["2@0.05", "3@0.002"])
def test_small_tiles_exercise_tiling(gpu, golden, key):
    rec = golden["configs"][key]
    cfg = synth.golden_config(key)
    arrays = (cfg.n_u, cfg.n_v, *synth.generate(cfg))
    for tile in (512, 4096, 20000):
        r = dev_counts(arrays, SIDE_CHEAPER, ALGO_GBBCPP, tile)
        assert (r.balanced, r.unbalanced) == (rec["balanced"], rec["unbalanced"]), tile


def test_partitions_sum_to_whole(gpu, golden):
    rec = golden["configs"]["2@0.05"]
    cfg = synth.golden_config("2@0.05")
    u, v, s = synth.generate(cfg)
    g = DeviceGraph.from_host(cfg.n_u, cfg.n_v, u, v, s)
    for parts in (2, 3, 8):
        for algo in ALGOS:
            rs = [g.count(algo, part_index=p, part_count=parts) for p in range(parts)]
            assert sum(r.balanced for r in rs) == rec["balanced"]
            assert sum(r.unbalanced for r in rs) == rec["unbalanced"]
            assert sum(r.wedges for r in rs) == g.w_s
    g.close()


def test_device_resident_inputs(gpu, golden):
    torch = pytest.importorskip("torch")
    rec = golden["configs"]["1@1"]
    cfg = synth.golden_config("1@1")
    u, v, s = synth.generate(cfg)
    du, dv, ds = (torch.from_numpy(x).cuda() for x in (u, v, s))
    torch.cuda.synchronize()
    g = DeviceGraph.from_device_ptrs(cfg.n_u, cfg.n_v, len(u), du.data_ptr(), dv.data_ptr(), ds.data_ptr())
    r = g.count()
    assert (r.balanced, r.unbalanced) == (rec["balanced"], rec["unbalanced"])
    g.close()


def test_device_validation_errors(gpu):
    from paper_2601_17707_b200 import DuplicateEdgeError, IndexOutOfRangeError

    with pytest.raises(IndexOutOfRangeError, match=r"u index 2 out of range \[0, 2\)"):
        DeviceGraph.from_host(2, 2, np.array([0, 2]), np.array([0, 0]), np.array([1, 1]))
    with pytest.raises(IndexOutOfRangeError, match=r"v index -1 out of range"):
        DeviceGraph.from_host(2, 2, np.array([0, 1]), np.array([0, -1]), np.array([1, 1]))
    with pytest.raises(DuplicateEdgeError) as e:
        DeviceGraph.from_host(3, 3, np.array([2, 1, 2, 1]), np.array([2, 0, 2, 0]), np.array([1, 1, -1, -1]))
    assert (e.value.u, e.value.v) == (1, 0)
    with pytest.raises(ValueError, match="is not a valid EdgeSign"):
        DeviceGraph.from_host(2, 2, np.array([0]), np.array([0]), np.array([0]))
