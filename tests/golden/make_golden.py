"""Produce the golden vectors in tests/golden/ by running the REFERENCE package.

Run in the build container (the reference is mounted read-only at /root/reference and is
absent on the GPU box, which only reads the committed JSON):

    python tests/golden/make_golden.py            # fixtures, corpora, config 1, scaled configs
    python tests/golden/make_golden.py --full 2   # config 2 at full size (long: ~30 min)
    python tests/golden/make_golden.py --ext      # classification + (2,k) vectors (8(f))
    python tests/golden/make_golden.py --ingest   # loader vectors (8(f) rank 3)

Every count here comes from the reference's own engines (pkg/src/bbcount):
  balanced  = count_balanced_parallel(g, workers)        (buckets.py:213-246)
  total     = count_balanced_bruteforce(g)[1]             (oracle.py:116-124) when small, else
              count_balanced_parallel(all-positive copy)  (total = balanced count with every
              sign +1, a reference-side identity checked on every small fixture below)
  unbalanced = total - balanced
Fixture graphs are built with the reference's own test fixtures (pkg/tests/conftest.py etc.)
and their edges digested, so tests/fixtures.py can prove it regenerates identical graphs.
"""

from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

sys.dont_write_bytecode = True
REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path[:0] = [REF_SRC, REF_TESTS, str(ROOT), str(ROOT / "tests")]

import random  # noqa: E402

import numpy as np  # noqa: E402

import bbcount  # noqa: E402  (the reference)
import conftest as ref_conftest  # noqa: E402  (reference fixtures)
import test_acceptance as ref_acceptance  # noqa: E402
import test_tiled as ref_tiled  # noqa: E402

import fixtures  # noqa: E402  (our regenerated fixtures)
from paper_2601_17707_b200 import synth  # noqa: E402

WORKERS = len(os.sched_getaffinity(0))


def sorted_digest(u, v, s) -> str:
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    order = np.lexsort((v, u))
    return synth.edge_digest(u[order], v[order], np.asarray(s)[order])


def ref_digest(g) -> str:
    e = g.edges()
    return sorted_digest([x[0] for x in e], [x[1] for x in e], [x[2].value for x in e])


def all_positive(g):
    return bbcount.build(g.u_count, g.v_count, [(u, v, 1) for u, v, _ in g.edges()])


def ref_counts(g, brute: bool) -> dict:
    balanced = bbcount.count_balanced_parallel(g, WORKERS)
    if brute:
        b2, total = bbcount.count_balanced_bruteforce(g)
        assert b2 == balanced
        assert bbcount.count_balanced_parallel(all_positive(g), 1) == total  # identity used at scale
    else:
        total = bbcount.count_balanced_parallel(all_positive(g), WORKERS)
    return {"balanced": balanced, "total": total, "unbalanced": total - balanced}


def named(out: dict) -> None:
    ref = {
        "complete_2x2": ref_conftest.complete_graph(2, 2),
        "complete_2x3": ref_conftest.complete_graph(2, 3),
        "complete_5x4": ref_conftest.complete_graph(5, 4),
        "complete_3x3": ref_conftest.complete_graph(3, 3),
        "complete_6x6_neg": ref_conftest.complete_graph(6, 6, -1),
        "two_negative_square": ref_conftest.graph_from_rows(["+-", "-+"]),
        "one_negative": bbcount.build(2, 2, [(0, 0, -1), (0, 1, 1), (1, 0, 1), (1, 1, 1)]),
        "dense_mixed_4x4": ref_conftest.dense_mixed_4x4(),
        "skew_instance": ref_tiled.skew_instance(),
        "tree": bbcount.build(3, 2, [(0, 0, 1), (1, 0, 1), (1, 1, 1), (2, 1, 1)]),
        "empty_1x1": bbcount.build(1, 1, []),
        "empty_u": bbcount.build(0, 3, []),
        "single_edge": bbcount.build(1, 1, [(0, 0, -1)]),
        "star_u": bbcount.build(1, 50, [(0, b, 1 if b % 3 else -1) for b in range(50)]),
        "classify_pp_pp": ref_conftest.graph_from_rows(["++", "++"]),
        "classify_pp_mm": ref_conftest.graph_from_rows(["+-", "+-"]),
        "classify_mm_mm": ref_conftest.graph_from_rows(["--", "--"]),
        "classify_pm_pm": ref_conftest.graph_from_rows(["++", "--"]),
        "classify_pp_pm": ref_conftest.graph_from_rows(["++", "+-"]),
        "classify_pm_mm": ref_conftest.graph_from_rows(["--", "-+"]),
        "degree_bands": bbcount.build(5, 600, [(a, b, 1 if (a + b) % 5 else -1)
                                               for a, d in enumerate([10, 32, 31, 512, 600]) for b in range(d)]),
    }
    mine = fixtures.named_fixtures()
    for name, g in ref.items():
        rec = {"n_u": g.u_count, "n_v": g.v_count, "m": g.edge_count, "digest": ref_digest(g)}
        if g.u_count and g.v_count:
            rec.update(ref_counts(g, brute=True))
            rec["classes"] = bbcount.classify_butterflies(g).as_dict()
        else:
            rec.update({"balanced": 0, "total": 0, "unbalanced": 0})
        f = mine[name]
        assert sorted_digest(f.u, f.v, f.s) == rec["digest"], name
        out["named"][name] = rec
    # smoke graph (140k edges) from the reference acceptance suite
    g = ref_acceptance._smoke_graph(20260810)
    rec = {"n_u": g.u_count, "n_v": g.v_count, "m": g.edge_count, "digest": ref_digest(g)}
    rec.update(ref_counts(g, brute=False))
    f = fixtures.smoke_graph(20260810)
    assert sorted_digest(f.u, f.v, f.s) == rec["digest"]
    out["named"]["smoke_graph"] = rec


def corpora(out: dict) -> None:
    for name, (seed, count, mu, mv, pe, pp) in fixtures.CORPORA.items():
        rng = random.Random(seed)
        ref_graphs = [ref_conftest.random_graph(rng, mu, mv, pe, pp) for _ in range(count)]
        mine = fixtures.corpus(seed, count, mu, mv, pe, pp)
        recs = []
        for g, f in zip(ref_graphs, mine):
            d = ref_digest(g)
            assert sorted_digest(f.u, f.v, f.s) == d
            r = ref_counts(g, brute=True)
            recs.append([g.u_count, g.v_count, g.edge_count, d, r["balanced"], r["total"]])
        out["corpora"][name] = recs


def synth_configs(out: dict, which: list[str]) -> None:
    for key in which:
        cfg = synth.golden_config(key)
        cfg_id = int(key.split("@")[0])
        t0 = time.time()
        u, v, s = synth.generate(cfg)
        g = bbcount.build(cfg.n_u, cfg.n_v, list(zip(u.tolist(), v.tolist(), s.tolist())))
        t_build = time.time() - t0
        brute = cfg.m <= 25_000
        t0 = time.time()
        rec = {"config": cfg_id, "key": key, "name": cfg.name, "n_u": cfg.n_u, "n_v": cfg.n_v, "m": cfg.m,
               "digest": synth.edge_digest(u, v, s)}
        rec.update(ref_counts(g, brute=brute))
        side = g.min_side()
        rec["min_side"] = side.value
        rec["w_u"] = sum(d * (d - 1) // 2 for d in g.deg_v)
        rec["w_v"] = sum(d * (d - 1) // 2 for d in g.deg_u)
        if brute:
            rec["serial_u"] = bbcount.count_balanced_2k_serial(g, 2, bbcount.Side.U)
            rec["serial_v"] = bbcount.count_balanced_2k_serial(g, 2, bbcount.Side.V)
        rec["ref_seconds"] = {"build": round(t_build, 2), "count": round(time.time() - t0, 2), "workers": WORKERS}
        out["configs"][key] = rec
        print(f"config {key}: {rec}", flush=True)


def extensions(out: dict) -> None:
    """six-way classification (oracle.classify_butterflies,
    oracle.py:172-197) and balanced (2,k)-bicliques for k = 3, 4 (count_balanced_2k_serial,
    buckets.py:64-154, both anchor sides; cross-checked with count_balanced_2k_bruteforce,
    oracle.py:137-169, where small)."""
    def b2k(g, brute: bool) -> dict:
        rec = {}
        for k in (3, 4):
            for side in (bbcount.Side.U, bbcount.Side.V):
                val = bbcount.count_balanced_2k_serial(g, k, side)
                if brute:
                    assert bbcount.count_balanced_2k_bruteforce(g, k, side) == val
                rec[f"k{k}_{side.value}"] = val
        return rec

    ref_named = {name: None for name in out["named"]}
    mine = fixtures.named_fixtures()
    for name in ref_named:
        if name == "smoke_graph":
            continue
        f = mine[name]
        rec = out["named"][name]
        g = bbcount.build(f.n_u, f.n_v, list(zip(f.u.tolist(), f.v.tolist(), f.s.tolist())))
        assert ref_digest(g) == rec["digest"]
        if g.u_count and g.v_count:
            rec["b2k"] = b2k(g, brute=g.edge_count <= 400)
    for name, (seed, count, mu, mv, pe, pp) in fixtures.CORPORA.items():
        rng = random.Random(seed)
        ref_graphs = [ref_conftest.random_graph(rng, mu, mv, pe, pp) for _ in range(count)]
        ext = []
        for g in ref_graphs:
            cls = bbcount.classify_butterflies(g).as_dict()
            ext.append({"classes": cls, "b2k": b2k(g, brute=g.edge_count <= 60)})
        out.setdefault("corpora_ext", {})[name] = ext
    for key in ("1@1", "5@small"):
        cfg = synth.golden_config(key)
        u, v, s = synth.generate(cfg)
        g = bbcount.build(cfg.n_u, cfg.n_v, list(zip(u.tolist(), v.tolist(), s.tolist())))
        t0 = time.time()
        rec = out["configs"][key]
        rec["classes"] = bbcount.classify_butterflies(g).as_dict()
        rec["b2k"] = b2k(g, brute=False)
        print(f"config {key} extensions in {time.time() - t0:.1f}s: {rec['classes']} {rec['b2k']}", flush=True)


def ingest(out: dict) -> None:
    """Loader vectors: the reference's load_graph (ingest.py:185-191)
    on deterministic texts from tests/fixtures.ingest_text, recorded as sorted-edge digests."""
    def policy(p):
        if p[0] == "explicit":
            return bbcount.ExplicitSign()
        if p[0] == "rating":
            return bbcount.RatingThreshold(p[1], p[2])
        return bbcount.RandomBernoulli(p[1], p[2])

    rec = {}
    for name, (seed, n, nu, nv, kind, pol) in fixtures.INGEST_CASES.items():
        text = fixtures.ingest_text(seed, n, nu, nv, kind)
        g = bbcount.load_graph(text, policy(pol))
        rec[name] = {"n_u": g.u_count, "n_v": g.v_count, "m": g.edge_count, "digest": ref_digest(g),
                     "text_len": len(text)}
    out["ingest"] = rec


def main() -> None:
    path = HERE / "golden.json"
    out = json.loads(path.read_text()) if path.exists() else {}
    out.setdefault("named", {})
    out.setdefault("corpora", {})
    out.setdefault("configs", {})
    out["generator"] = "tests/golden/make_golden.py (reference bbcount 0.1.0 at /root/reference/pkg/src)"
    if "--ingest" in sys.argv:
        ingest(out)
    elif "--ext" in sys.argv:
        extensions(out)
    elif "--full" in sys.argv:
        cfg_id = int(sys.argv[sys.argv.index("--full") + 1])
        synth_configs(out, [f"{cfg_id}@1"])
    else:
        named(out)
        corpora(out)
        synth_configs(out, list(synth.GOLDEN_SMALL))
    path.write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    print("wrote", path)


if __name__ == "__main__":
    main()
