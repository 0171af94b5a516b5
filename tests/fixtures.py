"""Graph fixtures of the reference test-suite, regenerated without the reference.

Each generator consumes ``random.Random`` exactly as the reference fixture it mirrors, so
it yields the same edges; tests/golden/fixtures.json stores a digest of every fixture as
produced BY THE REFERENCE (tests/golden/make_golden.py), and tests/test_oracle_golden.py
checks the regenerated edges against it before any count is compared.

Mirrors (paths under /root/reference/pkg/tests):
  random_graph           conftest.py:8-14
  complete_graph         conftest.py:17-18
  graph_from_rows        conftest.py:21-32
  dense_mixed_4x4        conftest.py:35-43 (paper Fig. 1(b))
  skew_instance          test_tiled.py:161-176
  smoke_graph            test_acceptance.py:157-175
  corpus(seed, ...)      test_acceptance.py:36-40 (corpus_200 = corpus(20260810, 200))
Graphs are returned as plain ``(n_u, n_v, u, v, s)`` int arrays so the same fixture feeds
the CUDA path, the C-ABI and the oracle.
"""

from __future__ import annotations

import random

import numpy as np

from paper_2601_17707_b200.synth import edge_digest


class Fx:
    """A fixture graph: partition sizes and edge arrays (u, v, sign in {+1, -1})."""

    def __init__(self, n_u: int, n_v: int, edges: list[tuple[int, int, int]], name: str = ""):
        self.n_u, self.n_v, self.name = n_u, n_v, name
        self.u = np.array([e[0] for e in edges], dtype=np.int32)
        self.v = np.array([e[1] for e in edges], dtype=np.int32)
        self.s = np.array([e[2] for e in edges], dtype=np.int8)

    @property
    def m(self) -> int:
        return len(self.u)

    def arrays(self):
        return self.n_u, self.n_v, self.u, self.v, self.s

    def digest(self) -> str:
        return edge_digest(self.u, self.v, self.s)

    def edges(self):
        return list(zip(self.u.tolist(), self.v.tolist(), self.s.tolist()))

    def graph(self):
        from paper_2601_17707_b200 import SignedBipartiteGraph

        return SignedBipartiteGraph.from_arrays(self.n_u, self.n_v, self.u, self.v, self.s)


def random_graph(rng: random.Random, max_u: int = 30, max_v: int = 30, p_edge: float = 0.2,
                 p_pos: float = 0.5) -> Fx:
    nu = rng.randint(1, max_u)
    nv = rng.randint(1, max_v)
    edges = []
    for a in range(nu):
        for b in range(nv):
            if rng.random() < p_edge:
                edges.append((a, b, 1 if rng.random() < p_pos else -1))
    return Fx(nu, nv, edges, "random")


def complete_graph(nu: int, nv: int, sign: int = 1) -> Fx:
    return Fx(nu, nv, [(a, b, sign) for a in range(nu) for b in range(nv)], f"complete_{nu}x{nv}")


def graph_from_rows(rows: list[str], name: str = "rows") -> Fx:
    edges = []
    for a, row in enumerate(rows):
        for b, ch in enumerate(row):
            if ch in "+-":
                edges.append((a, b, 1 if ch == "+" else -1))
    return Fx(len(rows), len(rows[0]) if rows else 0, edges, name)


def dense_mixed_4x4() -> Fx:
    return graph_from_rows(["++++", "++++", "-+++", "--++"], "dense_mixed_4x4")


def skew_instance() -> Fx:
    edges = []
    for i in range(1, 41):
        edges += [(0, i - 1, 1), (i, i - 1, 1)]
    groups = [list(range(2 + 4 * j, 6 + 4 * j)) for j in range(9)] + [[38, 39, 40]]
    for j, members in enumerate(groups):
        edges += [(a, 40 + j, 1) for a in members]
    edges += [(0, 50 + p, 1) for p in range(400)]
    return Fx(41, 450, edges, "skew_instance")


def smoke_graph(seed: int = 20260810) -> Fx:
    rng = random.Random(seed)
    n_u, n_v, hubs = 400, 3000, 250
    edges, seen = [], set()
    for b in range(hubs):
        for a in range(n_u):
            seen.add((a, b))
            edges.append((a, b, 1 if rng.random() < 0.7 else -1))
    while len(edges) < 140_000:
        a = rng.randrange(n_u)
        b = rng.randrange(hubs, n_v)
        if (a, b) not in seen:
            seen.add((a, b))
            edges.append((a, b, 1 if rng.random() < 0.7 else -1))
    return Fx(n_u, n_v, edges, "smoke_graph")


def corpus(seed: int, count: int, max_u: int = 30, max_v: int = 30, p_edge: float = 0.2,
           p_pos: float = 0.5) -> list[Fx]:
    rng = random.Random(seed)
    return [random_graph(rng, max_u, max_v, p_edge, p_pos) for _ in range(count)]


def named_fixtures() -> dict[str, Fx]:
    return {
        "complete_2x2": complete_graph(2, 2),
        "complete_2x3": complete_graph(2, 3),
        "complete_5x4": complete_graph(5, 4),
        "complete_3x3": complete_graph(3, 3),
        "complete_6x6_neg": complete_graph(6, 6, -1),
        "two_negative_square": graph_from_rows(["+-", "-+"]),
        "one_negative": Fx(2, 2, [(0, 0, -1), (0, 1, 1), (1, 0, 1), (1, 1, 1)], "one_negative"),
        "dense_mixed_4x4": dense_mixed_4x4(),
        "skew_instance": skew_instance(),
        "tree": Fx(3, 2, [(0, 0, 1), (1, 0, 1), (1, 1, 1), (2, 1, 1)], "tree"),
        "empty_1x1": Fx(1, 1, [], "empty_1x1"),
        "empty_u": Fx(0, 3, [], "empty_u"),
        "single_edge": Fx(1, 1, [(0, 0, -1)], "single_edge"),
        "star_u": Fx(1, 50, [(0, b, 1 if b % 3 else -1) for b in range(50)], "star_u"),
        "classify_pp_pp": graph_from_rows(["++", "++"]),
        "classify_pp_mm": graph_from_rows(["+-", "+-"]),
        "classify_mm_mm": graph_from_rows(["--", "--"]),
        "classify_pm_pm": graph_from_rows(["++", "--"]),
        "classify_pp_pm": graph_from_rows(["++", "+-"]),
        "classify_pm_mm": graph_from_rows(["--", "-+"]),
        "degree_bands": Fx(5, 600, [(a, b, 1 if (a + b) % 5 else -1) for a, d in enumerate([10, 32, 31, 512, 600])
                                    for b in range(d)], "degree_bands"),
    }


CORPORA = {
    # name: (seed, count, max_u, max_v, p_edge, p_pos)
    "corpus_200": (20260810, 200, 30, 30, 0.2, 0.5),
    "dense_40": (1717, 60, 40, 40, 0.5, 0.5),
    "skewed_sign_30": (2929, 80, 30, 30, 0.3, 0.85),
    "tall_thin": (4141, 60, 60, 8, 0.4, 0.5),
}


# ---- edge-list texts for the loaders (device ingestion) --------

def ingest_text(seed: int, n_lines: int, n_u: int, n_v: int, kind: str = "explicit", dup: float = 0.2,
                ts: float = 0.5) -> str:
    """Deterministic edge-list text in the reference's input format (ingest.py:80-115):
    comment and blank lines, string labels, repeated (u, v) pairs with and without
    timestamps, values as signs ("1", "-1", "0", "1.0", "+1", "-0") or ratings."""
    rng = random.Random(seed)
    lines = ["% generated edge list", "# second comment", ""]
    pairs: list[tuple[str, str]] = []
    for _ in range(n_lines):
        r = rng.random()
        if r < 0.02:
            lines.append(rng.choice(["", "   ", "% note", "#x y z", "\t"]))
            continue
        if pairs and r < 0.02 + dup:
            a, b = rng.choice(pairs)
        else:
            a = rng.choice(["u", "user", "U_", ""]) + str(rng.randrange(n_u))
            b = rng.choice(["v", "item", "V-", ""]) + str(rng.randrange(n_v))
            pairs.append((a, b))
        if kind == "explicit":
            val = rng.choice(["1", "-1", "0", "1.0", "+1", "-0", "1e0", "-1.000"])
        elif kind == "rating":
            val = rng.choice(["1", "2", "3", "3.5", "4", "5", "4.25", "2.5e0", "10"])
        else:
            val = rng.choice(["", "1", "7"])
        sep = rng.choice([" ", "\t", "  ", " \t "])
        parts = [a, b] + ([val] if val else [])
        if val and rng.random() < ts:
            parts.append(str(rng.randrange(-5, 50)))
        lines.append(rng.choice(["", " ", "\t"]) + sep.join(parts) + rng.choice(["", " ", "\r", "\t"]))
    return "\n".join(lines) + rng.choice(["", "\n"])


INGEST_CASES = {
    # name: (seed, n_lines, n_u, n_v, kind, policy)  policy: ("explicit",) | ("rating", t, at_or_above)
    #                                                        | ("bernoulli", p, seed)
    "explicit_small": (11, 200, 20, 15, "explicit", ("explicit",)),
    "explicit_dups": (12, 3000, 60, 40, "explicit", ("explicit",)),
    "rating_at_or_above": (13, 2000, 50, 80, "rating", ("rating", 3.5, True)),
    "rating_strict": (14, 2000, 50, 80, "rating", ("rating", 4.0, False)),
    "bernoulli": (15, 2500, 70, 70, "bare", ("bernoulli", 0.7, 20260810)),
    "bernoulli_big_seed": (16, 500, 30, 30, "bare", ("bernoulli", 0.35, 2**64 + 12345)),
}
