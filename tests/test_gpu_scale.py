"""Full-size BASELINE configs on the device: bit-exact against the reference where a
golden value exists (tests/golden/golden.json "k@1"), and size-independent invariants
everywhere else: anchoring U == anchoring V, G-BBC == G-BBC++, fast == general path,
start-vertex partitions sum to the whole, and total = balanced count of the all-positive
graph (the identity the reference's own engines provide at scale)."""

import numpy as np
import pytest

from paper_2601_17707_b200 import _lib, synth
from paper_2601_17707_b200._lib import ALGO_GBBC, ALGO_GBBCPP, SIDE_U, SIDE_V, DeviceGraph

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg2():
    cfg = synth.CONFIGS[2]
    return cfg, synth.generate(cfg)


def test_config2_invariants_and_reference(gpu, golden, cfg2):
    cfg, (u, v, s) = cfg2
    results = {}
    for side in (SIDE_U, SIDE_V):
        g = DeviceGraph.from_host(cfg.n_u, cfg.n_v, u, v, s, 0, side)
        for algo in (ALGO_GBBC, ALGO_GBBCPP):
            r = g.count(algo)
            results[(side, algo)] = (r.balanced, r.unbalanced)
            assert r.wedges == g.w_s
        if side == SIDE_V:
            parts = [g.count(ALGO_GBBCPP, part_index=p, part_count=4) for p in range(4)]
            assert (sum(p.balanced for p in parts), sum(p.unbalanced for p in parts)) == results[(side, ALGO_GBBCPP)]
        g.close()
    assert len(set(results.values())) == 1
    bal, unb = results[(SIDE_V, ALGO_GBBCPP)]
    rec = golden["configs"].get("2@1")
    if rec is not None:
        assert synth.edge_digest(u, v, s) == rec["digest"]
        assert (bal, unb) == (rec["balanced"], rec["unbalanced"])
    # total via the all-positive graph, counted by the device
    gp = DeviceGraph.from_host(cfg.n_u, cfg.n_v, u, v, np.ones_like(s))
    rp = gp.count()
    gp.close()
    assert rp.unbalanced == 0 and rp.balanced == bal + unb


def test_config2_general_path_matches_fast_path(gpu, cfg2):
    cfg, (u, v, s) = cfg2
    g = DeviceGraph.from_host(cfg.n_u, cfg.n_v, u, v, s)
    a = g.count(ALGO_GBBCPP)
    b = g.count(ALGO_GBBCPP, flags=_lib.FLAG_BANDED_ONLY)
    g.close()
    assert (a.balanced, a.unbalanced) == (b.balanced, b.unbalanced)


@pytest.mark.parametrize("key", ["3@0.05", "5@0.05"])
def test_other_configs_scaled_invariants(gpu, key):
    cfg = synth.golden_config(key) if key in synth.GOLDEN_SMALL else None
    if cfg is None:
        cid, f = key.split("@")
        base = synth.CONFIGS[int(cid)]
        cfg = base.scaled(float(f)) if int(cid) != 5 else synth.SynthConfig("uniform_20k_2m", 20_000, 20_000,
                                                                            2_000_000, seed=5)
    u, v, s = synth.generate(cfg)
    out = set()
    for side in (SIDE_U, SIDE_V):
        g = DeviceGraph.from_host(cfg.n_u, cfg.n_v, u, v, s, 0, side)
        for algo in (ALGO_GBBC, ALGO_GBBCPP):
            r = g.count(algo)
            out.add((r.balanced, r.unbalanced))
        g.close()
    assert len(out) == 1


def test_wide_sparse_ranges_all_cold_strategies_agree(gpu):
    """Config 4's recipe at 1/10 size (2.5 M anchors, cold rank ranges of millions): the
    key-hash rounds (default there), bitmap rounds only (flags bit 1), counter tiles only
    (bit 7), forced hash rounds (bit 13) and the general banded path give one answer, on
    both sides and for every partition."""
    cfg = synth.CONFIGS[4].scaled(0.1)
    u, v, s = synth.generate(cfg)
    g = DeviceGraph.from_host(cfg.n_u, cfg.n_v, u, v, s)
    out = {f: g.count(ALGO_GBBCPP, flags=f) for f in (0, 2, 128, 8192, _lib.FLAG_BANDED_ONLY)}
    ref = (out[0].balanced, out[0].unbalanced)
    assert all((r.balanced, r.unbalanced) == ref for r in out.values()), {f: (r.balanced, r.unbalanced)
                                                                         for f, r in out.items()}
    assert all(r.wedges == g.w_s for r in out.values())
    parts = [g.count(ALGO_GBBC, part_index=p, part_count=3) for p in range(3)]
    assert (sum(p.balanced for p in parts), sum(p.unbalanced for p in parts)) == ref
    g.close()
    gu = DeviceGraph.from_host(cfg.n_u, cfg.n_v, u, v, s, 0, SIDE_U if g.anchor_side == 1 else SIDE_V)
    r = gu.count()
    assert (r.balanced, r.unbalanced) == ref
    gu.close()


@pytest.mark.slow
def test_config3_full_size_invariants(gpu):
    """Hub-heavy config 3 at full size (100 M edges, planted degree-1e6 hubs on both sides):
    sides, algorithms and partitions agree; total = all-positive balanced count."""
    cfg = synth.CONFIGS[3]
    u, v, s = synth.generate(cfg)
    res = set()
    for side in (SIDE_U, SIDE_V):
        g = DeviceGraph.from_host(cfg.n_u, cfg.n_v, u, v, s, 0, side)
        for algo in (ALGO_GBBC, ALGO_GBBCPP):
            r = g.count(algo)
            res.add((r.balanced, r.unbalanced))
        g.close()
    assert len(res) == 1
    bal, unb = res.pop()
    gp = DeviceGraph.from_host(cfg.n_u, cfg.n_v, u, v, np.ones_like(s))
    rp = gp.count()
    gp.close()
    assert rp.unbalanced == 0 and rp.balanced == bal + unb
