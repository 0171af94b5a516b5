"""Full-size BASELINE configs on the device, bit-exact against the CPU oracle's goldens.

tests/golden/full/<key>.json were produced by tests/golden/make_full_golden.py: the
oracle's sort_neighbors traversal (reference buckets.py:87-111, closing of
buckets.py:166-197) over the same synthetic arrays, at full BASELINE size.  That
traversal is pinned against the reference package's own vectors in
tests/test_oracle_golden.py, including config 2 at full size, where the reference's
count_balanced_parallel ran for 50 minutes.  Each case checks the regenerated edges'
digest first, then the (balanced, unbalanced) pair on both anchor sides and both
scheduling algorithms where affordable.
"""

import json
from pathlib import Path

import numpy as np
import pytest

from paper_2601_17707_b200 import _lib, synth
from paper_2601_17707_b200._lib import ALGO_GBBC, ALGO_GBBCPP, SIDE_U, SIDE_V, DeviceGraph

pytestmark = pytest.mark.gpu

FULL = Path(__file__).resolve().parent / "golden" / "full"
EXTRA = {"u1000": synth.SynthConfig("uniform_20k_20m", 20_000, 20_000, 20_000_000, seed=55)}


def full_golden(key):
    p = FULL / f"{key}.json"
    if not p.exists():
        pytest.fail(f"missing golden {p} (run tests/golden/make_full_golden.py)")
    return json.loads(p.read_text())


def arrays_for(key):
    cfg = EXTRA[key] if key in EXTRA else synth.CONFIGS[int(key.split("@")[0])]
    u, v, s = synth.generate(cfg)
    return cfg, u, v, s


def check(key, sides=(SIDE_U, SIDE_V), algos=(ALGO_GBBC, ALGO_GBBCPP), extra_flags=()):
    rec = full_golden(key)
    cfg, u, v, s = arrays_for(key)
    assert synth.edge_digest(u, v, s) == rec["digest"], key
    want = (rec["balanced"], rec["unbalanced"])
    for side in sides:
        g = DeviceGraph.from_host(cfg.n_u, cfg.n_v, u, v, s, 0, side)
        try:
            assert (g.w_u, g.w_v) == (rec["w_u"], rec["w_v"])
            for algo in algos:
                r = g.count(algo)
                assert (r.balanced, r.unbalanced) == want, (key, side, algo)
                assert r.wedges == g.w_s
            for fl in extra_flags:
                r = g.count(ALGO_GBBCPP, flags=fl)
                assert (r.balanced, r.unbalanced) == want, (key, side, "flags", fl)
        finally:
            g.close()


def test_config2_full_vs_golden(gpu):
    check("2@1", algos=(ALGO_GBBCPP,))


def test_config5_full_vs_golden(gpu):
    """Uniform 200k x 200k, 200 M edges: every anchor of degree ~1000 runs the general
    multi-batch W16 path."""
    check("5@1", sides=(SIDE_U,), algos=(ALGO_GBBC, ALGO_GBBCPP))


def test_uniform_deg1000_vs_golden(gpu):
    """Config 5's regime (deg ~1000, multi-batch W16, 4-8 bands per anchor) at 20 M edges,
    including the table-free search mode and the general banded path only."""
    check("u1000", extra_flags=(_lib.FLAG_BANDED_ONLY, 1024))


@pytest.mark.slow
def test_config3_full_vs_golden(gpu):
    """Hub-heavy config 3: planted degree-1e6 hubs on both sides, so the U-anchored graph
    runs its hub anchors through the W32 layout (deg > 65,535)."""
    check("3@1")


@pytest.mark.slow
def test_config4_full_vs_golden(gpu):
    """Power-law config 4 at 1 B edges (key-hash cold rounds over 25 M-rank ranges)."""
    check("4@1", sides=(SIDE_V,), algos=(ALGO_GBBCPP,))


def test_w32_layout_k2_vs_oracle(gpu):
    """The k = 2 count through the W32 layout (anchor degree > 65,535) against the oracle:
    3 U vertices x 70,000 V vertices with mixed signs, plus sparse noise so that the hub
    anchors share end vertices with low-degree ones."""
    from oracle.oracle import OracleGraph

    n_v = 70_000
    rng = np.random.default_rng(11)
    hu = np.repeat(np.arange(3, dtype=np.int32), n_v)
    hv = np.tile(np.arange(n_v, dtype=np.int32), 3)
    keep = rng.random(len(hu)) < 0.97
    nu = 3 + rng.integers(0, 2000, 60_000).astype(np.int32)
    nv = rng.integers(0, n_v, 60_000).astype(np.int32)
    key = np.unique(nu.astype(np.int64) << 32 | nv.astype(np.int64))
    u = np.concatenate([hu[keep], (key >> 32).astype(np.int32)])
    v = np.concatenate([hv[keep], (key & 0xffffffff).astype(np.int32)])
    s = np.where(rng.random(len(u)) < 0.35, -1, 1).astype(np.int8)
    n_u = 2003
    assert np.bincount(u).max() > 65_535  # U anchors take the W32 layout
    o = OracleGraph(n_u, n_v, u, v, s).count_sorted()
    want = (o.balanced, o.unbalanced)
    for side in (SIDE_U, SIDE_V):
        g = DeviceGraph.from_host(n_u, n_v, u, v, s, 0, side)
        try:
            for algo in (ALGO_GBBC, ALGO_GBBCPP):
                for fl in (0, _lib.FLAG_BANDED_ONLY, 1024):
                    r = g.count(algo, flags=fl)
                    assert (r.balanced, r.unbalanced) == want, (side, algo, fl)
        finally:
            g.close()
