"""Device-side ingestion (csrc/bbc_ingest.cu) against the reference's
load_graph vectors (tests/golden, make_golden.py --ingest) and the host pipeline: same dense
ids, same deduplicated signed edges, same exceptions at the same lines."""

import random

import pytest

import fixtures
import paper_2601_17707_b200 as bbc
from paper_2601_17707_b200 import _lib, synth

pytestmark = pytest.mark.gpu


def _policy(p):
    if p[0] == "explicit":
        return bbc.ExplicitSign()
    if p[0] == "rating":
        return bbc.RatingThreshold(p[1], p[2])
    return bbc.RandomBernoulli(p[1], p[2])


def _same(g1, g2):
    assert (g1.u_count, g1.v_count, g1.edge_count) == (g2.u_count, g2.v_count, g2.edge_count)
    a, b = g1.edge_arrays(), g2.edge_arrays()
    assert synth.edge_digest(*a) == synth.edge_digest(*b)


def test_reference_vectors(gpu, golden):
    for name, (seed, n, nu, nv, kind, pol) in fixtures.INGEST_CASES.items():
        text = fixtures.ingest_text(seed, n, nu, nv, kind)
        h = bbc.ingest_device(text, _policy(pol))
        assert h is not None, name  # these texts stay on the device path
        rec = golden["ingest"][name]
        u, v, s = h.edges()
        assert (h.n_u, h.n_v, h.m) == (rec["n_u"], rec["n_v"], rec["m"]), name
        g = bbc.SignedBipartiteGraph.from_arrays(h.n_u, h.n_v, u, v, s)
        assert synth.edge_digest(*g.edge_arrays()) == rec["digest"], name
        h.close()


def test_matches_host_pipeline_edge_order_and_counts(gpu):
    for seed in range(8):
        text = fixtures.ingest_text(100 + seed, 1500, 40 + seed, 30, "explicit", dup=0.35)
        host = bbc.load_graph(text)
        h = bbc.ingest_device(text)
        u, v, s = h.edges()
        # dedup_latest output order (first occurrence of the pair) is kept
        parsed = bbc.parse_edge_list(text)
        ded = bbc.dedup_latest(bbc.apply_sign_policy(parsed.edges, bbc.ExplicitSign()))
        want = [(parsed.u_ids[a], parsed.v_ids[b], sg.value) for a, b, sg in ded]
        assert list(zip(u.tolist(), v.tolist(), s.tolist())) == want
        _same(host, bbc.SignedBipartiteGraph.from_arrays(h.n_u, h.n_v, u, v, s))
        h.close()


def test_counts_through_the_device_graph(gpu):
    text = fixtures.ingest_text(7, 20000, 300, 200, "rating", dup=0.1)
    pol = bbc.RatingThreshold(3.5)
    h = bbc.ingest_device(text, pol)
    dg = h.device_graph()  # no host round trip
    r = dg.count()
    host = bbc.load_graph(text, pol)
    assert (r.balanced, r.unbalanced) == bbc.count_signed_butterflies(host)
    dg.close()
    h.close()


@pytest.mark.parametrize("text, exc, line", [
    ("a b 1\nc\n", bbc.MalformedLineError, 2),
    ("a b 1\n\n% x\nc d 1 2 3\n", bbc.MalformedLineError, 4),
    ("a b 1\nc d\n", bbc.MissingValueError, None),
    ("a b 1\nc d 2\n", bbc.InvalidSignValueError, None),
])
def test_errors_match_host(gpu, text, exc, line):
    with pytest.raises(exc) as e_dev:
        bbc.load_graph_device(text)
    with pytest.raises(exc) as e_host:
        bbc.load_graph(text)
    assert str(e_dev.value) == str(e_host.value)
    if line is not None:
        assert e_dev.value.line_number == line


def test_unsupported_inputs_take_the_host_pipeline(gpu):
    for text in ("a b 1_0\n", "a b 1\nxé y 1\n", "a b 1 1_000\n", "a b 1e400\n", "a b inf\n",
                 "a b 0.1234567890123456789\n"):
        assert bbc.ingest_device(text) is None or text == "a b 1e400\n"
    # the graph is still the host pipeline's
    text = "a b 1\nxé y -1\nxé b 1\n"
    _same(bbc.load_graph_device(text), bbc.load_graph(text))


def test_random_texts_vs_host(gpu):
    rng = random.Random(5)
    for i in range(30):
        kind = rng.choice(["explicit", "rating", "bare"])
        text = fixtures.ingest_text(1000 + i, rng.randrange(1, 400), rng.randrange(1, 30), rng.randrange(1, 30), kind,
                                    dup=rng.random() * 0.6, ts=rng.random())
        pol = {"explicit": bbc.ExplicitSign(), "rating": bbc.RatingThreshold(rng.choice([1.0, 3.5, 4.0])),
               "bare": bbc.RandomBernoulli(rng.random(), rng.randrange(2**64))}[kind]
        _same(bbc.load_graph_device(text, pol), bbc.load_graph(text, pol))


def test_empty_and_comment_only(gpu):
    for text in ("", "\n\n", "% only\n# comments\n"):
        g = bbc.load_graph_device(text)
        assert (g.u_count, g.v_count, g.edge_count) == (0, 0, 0)
    assert _lib.device_count() > 0
