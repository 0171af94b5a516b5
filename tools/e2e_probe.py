"""Repeated host-array builds + counts through the C ABI (e2e latency breakdown)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2601_17707_b200 import _lib, synth  # noqa: E402

cfg = synth.golden_config(sys.argv[1] if len(sys.argv) > 1 else "2@1")
u, v, s = synth.generate(cfg)
pu, pv, ps = (torch.from_numpy(x).pin_memory() for x in (u, v, s))
for i in range(5):
    t0 = time.perf_counter()
    g = _lib.DeviceGraph.from_host(cfg.n_u, cfg.n_v, pu.numpy(), pv.numpy(), ps.numpy())
    t1 = time.perf_counter()
    r = g.count()
    t2 = time.perf_counter()
    g.close()
    t3 = time.perf_counter()
    print(f"build {1e3*(t1-t0):.1f} ms (device prep {r.preprocess_ms:.1f}) count {1e3*(t2-t1):.1f} ms "
          f"(kernel {r.count_ms:.1f}) destroy {1e3*(t3-t2):.1f} ms", flush=True)
