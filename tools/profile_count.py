"""Run the count kernel a few times on a config (for ncu / compute-sanitizer captures)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2601_17707_b200 import _lib, synth  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="2@1")
p.add_argument("--reps", type=int, default=2)
p.add_argument("--algo", type=int, default=_lib.ALGO_GBBCPP)
p.add_argument("--tile", type=int, default=0)
p.add_argument("--flags", type=int, default=0)
a = p.parse_args()
cfg = synth.golden_config(a.config)
u, v, s = synth.generate(cfg)
g = _lib.DeviceGraph.from_host(cfg.n_u, cfg.n_v, u, v, s)
for _ in range(a.reps):
    r = g.count(a.algo, a.tile, flags=a.flags)
    print(f"{cfg.name}: balanced={r.balanced} unbalanced={r.unbalanced} W={r.wedges} count_ms={r.count_ms:.3f} "
          f"prep_ms={r.preprocess_ms:.3f} rate={r.wedges / r.count_ms * 1e3:.3e}/s", flush=True)
if a.flags & _lib.FLAG_ROUNDS:
    print("rounds", g.round_counters(), flush=True)
