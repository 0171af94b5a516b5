"""Time the device loader (load_graph on the GPU) against the host pipeline on an edge-list
text made from a BASELINE config ("u<id> v<id> +-1" lines, 10 % duplicated pairs with
timestamps)."""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2601_17707_b200 as bbc  # noqa: E402
from paper_2601_17707_b200 import synth  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="2@1")
p.add_argument("--host-lines", type=int, default=200_000)
a = p.parse_args()
cfg = synth.golden_config(a.config)
u, v, s = synth.generate(cfg)
m = len(u)
rng = np.random.default_rng(0)
dup = rng.random(m) < 0.1
ts = rng.integers(0, 1000, m)
cols = [np.char.add("u", u.astype(str)), np.char.add("v", v.astype(str)), s.astype(str)]
base = np.char.add(np.char.add(np.char.add(cols[0], " "), np.char.add(cols[1], " ")), cols[2])
line = np.where(dup, np.char.add(np.char.add(base, " "), ts.astype(str)), base)
extra = np.char.add(np.char.add(base[dup], " "), (ts[dup] + 1).astype(str))  # later duplicates win
text = "\n".join(line.tolist() + extra.tolist()) + "\n"
data = text.encode("ascii")
print(f"{cfg.name}: {m + int(dup.sum())} lines, {len(text) / 1e6:.1f} MB", flush=True)
for rep in range(3):
    t0 = time.perf_counter()
    h = bbc.ingest_device(data)
    t1 = time.perf_counter()
    print(f"device ingest: {t1 - t0:.3f} s ({(m + dup.sum()) / (t1 - t0):.3e} lines/s), n_u={h.n_u} n_v={h.n_v} "
          f"m={h.m}", flush=True)
    if rep < 2:
        h.close()
dg = h.device_graph()
r = dg.count()
print(f"count on the ingested graph: balanced={r.balanced} unbalanced={r.unbalanced} ({r.count_ms:.2f} ms)")
sample = "\n".join(text.split("\n", a.host_lines)[:a.host_lines]) + "\n"
t0 = time.perf_counter()
bbc.load_graph(sample)
t1 = time.perf_counter()
print(f"host pipeline: {a.host_lines} lines in {t1 - t0:.2f} s ({a.host_lines / (t1 - t0):.3e} lines/s)")
