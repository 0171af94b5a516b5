"""Time the 8(f) kernels (classification on U anchors, (2,k) on both sides) on a config,
next to the C oracle on the same graph (threads = host cores)."""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2601_17707_b200 import _lib, synth  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="2@1")
p.add_argument("--reps", type=int, default=2)
p.add_argument("--oracle", action="store_true")
a = p.parse_args()
cfg = synth.golden_config(a.config)
u, v, s = synth.generate(cfg)
for side, name in ((_lib.SIDE_U, "U"), (_lib.SIDE_V, "V")):
    g = _lib.DeviceGraph.from_host(cfg.n_u, cfg.n_v, u, v, s, 0, side)
    W = g.w_s
    if side == _lib.SIDE_U:
        for _ in range(a.reps):
            cls, ms = g.classify()
        print(f"{cfg.name} classify (U anchors): {ms:.2f} ms, W={W:.4e}, {W / ms * 1e3:.3e} wedges/s {cls}", flush=True)
    for k in (2, 3):
        for _ in range(a.reps):
            val, ovf, ms = g.count_2k(k)
        print(f"{cfg.name} (2,{k}) side {name}: {ms:.2f} ms, {W / ms * 1e3:.3e} wedges/s, count={val}", flush=True)
    g.close()
if a.oracle:
    from oracle.oracle import OracleGraph

    o = OracleGraph(cfg.n_u, cfg.n_v, u, v, s)
    t = time.time()
    print("oracle classify", o.classify(), f"{time.time() - t:.1f}s", flush=True)
