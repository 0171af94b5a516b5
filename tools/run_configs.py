"""Time the count on BASELINE configs (full or scaled): generation, device build, count."""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2601_17707_b200 import _lib, synth  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("keys", nargs="+", help="config keys like 3@1, 4@0.25, 5@1")
p.add_argument("--reps", type=int, default=2)
p.add_argument("--flags", type=int, default=0)
p.add_argument("--algo", type=int, default=1)
p.add_argument("--extra-flags", type=int, nargs="*", help="time each of these flag sets in turn")
a = p.parse_args()
for key in a.keys:
    cfg = synth.golden_config(key)
    t0 = time.time()
    u, v, s = synth.generate(cfg)
    tg = time.time() - t0
    t0 = time.time()
    g = _lib.DeviceGraph.from_host(cfg.n_u, cfg.n_v, u, v, s)
    tb = time.time() - t0
    for f in a.extra_flags or [a.flags]:
        for _ in range(a.reps):
            r = g.count(a.algo, flags=f)
        if len(a.extra_flags or []) > 1:
            print(f"  flags {f}: count_ms={r.count_ms:.2f} W={r.wedges:.4e}", flush=True)
        if f & _lib.FLAG_ROUNDS:
            print("  rounds", g.round_counters(), flush=True)
    print(f"{key} {cfg.name}: m={cfg.m} side={'UV'[g.anchor_side]} W={r.wedges_total:.4e} bal={r.balanced} "
          f"unb={r.unbalanced} gen={tg:.1f}s build={tb:.2f}s prep_ms={r.preprocess_ms:.1f} count_ms={r.count_ms:.2f} "
          f"rate={r.wedges_total / max(r.count_ms, 1e-6) * 1e3:.3e}/s", flush=True)
    g.close()
    del u, v, s
