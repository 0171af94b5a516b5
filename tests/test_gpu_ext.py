"""SURVEY.md 8(f) rows on the GPU: six-way classification (oracle.classify_butterflies,
oracle.py:172-197) and balanced (2,k)-bicliques (count_balanced_2k_serial, buckets.py:64-154)
against the reference's golden vectors (tests/golden, produced by make_golden.py --ext) and,
at sizes the reference cannot reach, against the CPU oracle.  Bit-exact."""

import numpy as np
import pytest

import fixtures
import paper_2601_17707_b200 as bbc
from oracle.oracle import OracleGraph
from paper_2601_17707_b200 import synth
from paper_2601_17707_b200._lib import ALGO_GBBC, ALGO_GBBCPP, SIDE_U, SIDE_V, DeviceGraph

pytestmark = pytest.mark.gpu

ALGOS = (ALGO_GBBC, ALGO_GBBCPP)


def check_ext(arrays, rec, where, algos=ALGOS, flags=(0,)):
    n_u, n_v, u, v, s = arrays
    if not (n_u and n_v):
        return
    gu = DeviceGraph.from_host(n_u, n_v, u, v, s, 0, SIDE_U)
    gv = DeviceGraph.from_host(n_u, n_v, u, v, s, 0, SIDE_V)
    try:
        for algo in algos:
            for fl in flags:  # 2: no classification hash rounds, 1024: no band table
                if "classes" in rec:
                    assert gu.classify(algo, flags=fl)[0] == rec["classes"], (where, algo, fl)
                for key, val in rec.get("b2k", {}).items():
                    k, g = int(key[1]), (gu if key.endswith("_u") else gv)
                    assert g.count_2k(k, algo, flags=fl)[:2] == (val, False), (where, key, algo, fl)
            if "balanced" in rec:  # (2,2) is the balanced count on either side
                for g in (gu, gv):
                    assert g.count_2k(2, algo)[:2] == (rec["balanced"], False), (where, algo)
    finally:
        gu.close()
        gv.close()


def test_named_fixtures(gpu, golden):
    for name, f in fixtures.named_fixtures().items():
        check_ext(f.arrays(), golden["named"][name], name)


@pytest.mark.parametrize("corpus", list(fixtures.CORPORA))
def test_corpora(gpu, golden, corpus):
    seed, count, mu, mv, pe, pp = fixtures.CORPORA[corpus]
    graphs = fixtures.corpus(seed, count, mu, mv, pe, pp)
    for i, (f, rec) in enumerate(zip(graphs, golden["corpora_ext"][corpus])):
        check_ext(f.arrays(), rec, (corpus, i), algos=(ALGOS[i % 2],))


@pytest.mark.parametrize("key", ["1@1", "5@small"])
def test_configs_vs_reference(gpu, golden, key):
    cfg = synth.golden_config(key)
    check_ext((cfg.n_u, cfg.n_v, *synth.generate(cfg)), golden["configs"][key], key, flags=(0, 2, 1024))


@pytest.mark.parametrize("key", ["2@0.05", "3@0.002", "4@0.0002"])
def test_scaled_configs_vs_oracle(gpu, key):
    cfg = synth.golden_config(key)
    arrays = (cfg.n_u, cfg.n_v, *synth.generate(cfg))
    o = OracleGraph(*arrays)
    rec = {"classes": o.classify(), "b2k": {f"k{k}_{'uv'[side]}": o.count_2k(k, side)[0]
                                           for k in (3, 4) for side in (0, 1)}}
    check_ext(arrays, rec, key, flags=(0, 2, 1024))


def test_wide_layouts_vs_oracle(gpu):
    """Anchors above the packed layouts' degree limits: classification C32 (deg > 1023,
    sweep closing) and (2,k) W32 (deg > 65535)."""
    rng = np.random.default_rng(7)
    # 5 U vertices of degree ~1500 over 2000 V vertices, random signs
    u, v = np.nonzero(rng.random((5, 2000)) < 0.75)
    s = np.where(rng.random(len(u)) < 0.3, -1, 1).astype(np.int8)
    arrays = (5, 2000, u.astype(np.int32), v.astype(np.int32), s)
    o = OracleGraph(*arrays)
    check_ext(arrays, {"classes": o.classify(), "b2k": {"k3_u": o.count_2k(3, 0)[0], "k5_u": o.count_2k(5, 0)[0]}},
              "wide-classify")
    # 3 U vertices x 70000 V (complete, mixed signs): (2,k) counters beyond u16
    n_v = 70_000
    u = np.repeat(np.arange(3, dtype=np.int32), n_v)
    v = np.tile(np.arange(n_v, dtype=np.int32), 3)
    s = np.where((u + v) % 7 == 0, -1, 1).astype(np.int8)
    arrays = (3, n_v, u, v, s)
    o = OracleGraph(*arrays)
    check_ext(arrays, {"b2k": {"k3_u": o.count_2k(3, 0)[0]}}, "wide-2k")


# config 2 at full size, U anchors: the round-1/2 classification kernel's counts (band
# tiles + a packed-count hash, an independent implementation of the same closings)
CONFIG2_CLASSES = {"coherent_pp_pp": 863675101, "coherent_pp_mm": 316150114, "coherent_mm_mm": 28869038,
                   "incoherent_pm_pm": 632121112, "mixed_pp_pm": 1478163755, "mixed_pm_mm": 270259568}


def test_config2_full_classification(gpu):
    """Hash rounds (default) and band tiles only (flags 2), both algorithms, agree at full
    size; the classes sum to the reference's balanced / unbalanced counts."""
    cfg = synth.golden_config("2@1")
    g = DeviceGraph.from_host(cfg.n_u, cfg.n_v, *synth.generate(cfg), 0, SIDE_U)
    try:
        for algo, fl in ((ALGO_GBBCPP, 0), (ALGO_GBBC, 0), (ALGO_GBBCPP, 2)):
            assert g.classify(algo, flags=fl)[0] == CONFIG2_CLASSES, (algo, fl)
        c = CONFIG2_CLASSES  # balanced = same-parity wedge pairs; the reference's config-2 counts
        assert c["coherent_pp_pp"] + c["coherent_pp_mm"] + c["coherent_mm_mm"] + c["incoherent_pm_pm"] == 1840815365
        assert c["mixed_pp_pm"] + c["mixed_pm_mm"] == 1748423323
    finally:
        g.close()


def test_partitions_sum(gpu):
    cfg = synth.golden_config("2@0.01")
    g = DeviceGraph.from_host(cfg.n_u, cfg.n_v, *synth.generate(cfg), 0, SIDE_U)
    whole = g.classify()[0]
    parts = [g.classify(part_index=i, part_count=3)[0] for i in range(3)]
    assert {k: sum(p[k] for p in parts) for k in whole} == whole
    w3 = g.count_2k(3)[0]
    assert sum(g.count_2k(3, part_index=i, part_count=4)[0] for i in range(4)) == w3
    g.close()


def test_overflow_and_errors(gpu):
    u = np.repeat(np.arange(2, dtype=np.int32), 200)
    v = np.tile(np.arange(200, dtype=np.int32), 2)
    s = np.ones(400, dtype=np.int8)
    g = DeviceGraph.from_host(2, 200, u, v, s, 0, SIDE_U)
    assert g.count_2k(3)[:2] == (1313400, False)  # C(200, 3)
    assert g.count_2k(30)[1] is True  # C(200, 30) > 2^64
    with pytest.raises(ValueError):
        g.count_2k(1)
    g.close()
    gv = DeviceGraph.from_host(2, 200, u, v, s, 0, SIDE_V)
    with pytest.raises(ValueError):
        gv.classify()  # classification needs U anchors
    gv.close()


def test_drop_in_api(gpu, golden):
    """The reference-facing engines: classify_butterflies / count_balanced_2k_serial."""
    for name in ("dense_mixed_4x4", "degree_bands", "classify_pp_pm", "complete_5x4"):
        f = fixtures.named_fixtures()[name]
        rec = golden["named"][name]
        g = bbc.SignedBipartiteGraph.from_arrays(*f.arrays())
        cls = bbc.classify_butterflies(g)
        assert cls.as_dict() == rec["classes"] and cls.balanced() == rec["balanced"] and cls.total() == rec["total"]
        for key, val in rec["b2k"].items():
            side = bbc.Side.U if key.endswith("_u") else bbc.Side.V
            assert bbc.count_balanced_2k_serial(g, int(key[1]), side) == val, (name, key)
    g = bbc.SignedBipartiteGraph.from_arrays(2, 200, np.repeat(np.arange(2), 200), np.tile(np.arange(200), 2),
                                             np.ones(400, dtype=np.int8))
    with pytest.raises(bbc.CountOverflowError):
        bbc.count_balanced_2k_serial(g, 30, bbc.Side.U)
    with pytest.raises(bbc.InvalidKError):
        bbc.count_balanced_2k_serial(g, 1)
