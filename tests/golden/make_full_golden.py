"""Full-size BASELINE goldens for configs 2-5 from the CPU oracle (TEST INFRASTRUCTURE).

Generates config k at its BASELINE size (paper_2601_17707_b200.synth, the same arrays the
GPU path uploads), builds the oracle graph (reference graph.py:99-129 semantics), and
counts with the oracle's sort_neighbors traversal (reference buckets.py:87-111 with the
_pair_subtotal buckets and closing of buckets.py:166-197; `bbc_oracle_count_sorted`).
The oracle is pinned by tests/test_oracle_golden.py against the vectors the reference
package itself produced (including config 2 at full size, which this script re-derives
as a check of the sorted traversal at scale).

Writes tests/golden/full/<key>.json (key k@1, or a name from EXTRA) with the counts, W_U / W_V, the edge digest and the
run's provenance (host, cores, wall time).  Run in the build container (no GPU):

    python tests/golden/make_full_golden.py 5 3 4 u1000
"""

from __future__ import annotations

import json
import os
import platform
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.oracle import OracleGraph  # noqa: E402
from paper_2601_17707_b200 import synth  # noqa: E402

OUT = Path(__file__).resolve().parent / "full"

# Extra shapes checked at full size: a dense uniform graph whose anchors all have degree
# ~1000 (config 5's regime -- the general multi-batch path with 4-8 bands per anchor --
# at a size the oracle counts in seconds).
EXTRA = {
    "u1000": synth.SynthConfig("uniform_20k_20m", 20_000, 20_000, 20_000_000, seed=55),
}


def config_for(key: str):
    return EXTRA[key] if key in EXTRA else synth.CONFIGS[int(key.split("@")[0])]


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def run(key: str, threads: int) -> dict:
    cfg = config_for(key)
    t0 = time.time()
    u, v, s = synth.generate(cfg)
    digest = synth.edge_digest(u, v, s)
    t_gen = time.time() - t0
    t0 = time.time()
    g = OracleGraph(cfg.n_u, cfg.n_v, u, v, s)
    del u, v, s
    t_build = time.time() - t0
    w_u, w_v = g.admitted_total(0), g.admitted_total(1)
    side = 0 if w_u <= w_v else 1
    print(f"{key}: m={cfg.m} W_U={w_u:.4e} W_V={w_v:.4e} gen {t_gen:.0f}s build {t_build:.0f}s; "
          f"counting side {'UV'[side]} on {threads} threads", flush=True)
    t0 = time.time()
    r = g.count_sorted(side=side, threads=threads)
    t_count = time.time() - t0
    g.close()
    assert r.admitted == (w_u if side == 0 else w_v)
    rec = {
        "key": key, "name": cfg.name, "n_u": cfg.n_u, "n_v": cfg.n_v, "m": cfg.m, "digest": digest,
        "balanced": r.balanced, "unbalanced": r.unbalanced, "w_u": w_u, "w_v": w_v,
        "oracle_side": "uv"[side], "admitted": r.admitted, "scanned": r.scanned,
        "provenance": {
            "generator": "tests/golden/make_full_golden.py (oracle/bbc_oracle.c bbc_oracle_count_sorted)",
            "host": platform.node(), "cpu": cpu_model(), "threads": threads,
            "gen_s": round(t_gen, 1), "build_s": round(t_build, 1), "count_s": round(t_count, 1),
            "date": time.strftime("%Y-%m-%d %H:%M:%S"),
        },
    }
    print(json.dumps(rec), flush=True)
    return rec


def main() -> None:
    threads = len(os.sched_getaffinity(0))
    OUT.mkdir(exist_ok=True)
    for key in sys.argv[1:]:
        key = key if key in EXTRA or "@" in key else f"{key}@1"
        rec = run(key, threads)
        (OUT / f"{key}.json").write_text(json.dumps(rec, indent=1) + "\n")


if __name__ == "__main__":
    main()
