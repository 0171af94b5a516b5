"""A/B of prebuilt libbbc variants (e.g. BBC_NVCC_EXTRA builds copied to build/ab/*.so) on
the same synthetic graphs: each config is generated once (saved under /tmp), then every
variant runs in its own process (ctypes cannot unload a library).

    python tools/lib_ab.py --libs build/ab/a.so build/ab/b.so --configs 2@1 4@1 --reps 3
"""
import argparse
import json
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def child(lib: str, npz: str, reps: int, algo: int, flags: int, op: str) -> None:
    import numpy as np

    from paper_2601_17707_b200 import _lib

    _lib.LIB_PATH = Path(lib).resolve()
    d = np.load(npz)
    if op == "classify":  # six-way classification on U anchors
        g = _lib.DeviceGraph.from_host(int(d["n_u"]), int(d["n_v"]), d["u"], d["v"], d["s"], 0, _lib.SIDE_U)
        ms = []
        for _ in range(reps):
            cls, t = g.classify(algo, flags=flags)
            ms.append(t)
        print(json.dumps({"balanced": sorted(cls.items()), "unbalanced": 0, "ms": sorted(ms)}), flush=True)
        return
    g = _lib.DeviceGraph.from_host(int(d["n_u"]), int(d["n_v"]), d["u"], d["v"], d["s"])
    ms = []
    for _ in range(reps):
        r = g.count(algo, 0, flags=flags)
        ms.append(r.count_ms)
    print(json.dumps({"balanced": r.balanced, "unbalanced": r.unbalanced, "ms": sorted(ms),
                      "prep_ms": r.preprocess_ms}), flush=True)


def main() -> None:
    p = argparse.ArgumentParser()
    p.add_argument("--libs", nargs="+", required=True)
    p.add_argument("--configs", nargs="+", default=["2@1"])
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--algo", type=int, default=1)
    p.add_argument("--flags", type=int, default=0)
    p.add_argument("--op", default="count", choices=("count", "classify"))
    p.add_argument("--child", nargs=2)
    a = p.parse_args()
    if a.child:
        child(a.child[0], a.child[1], a.reps, a.algo, a.flags, a.op)
        return
    import numpy as np

    from paper_2601_17707_b200 import synth

    tmp = Path(tempfile.mkdtemp(prefix="lib_ab_"))
    for key in a.configs:
        cfg = synth.golden_config(key)
        u, v, s = synth.generate(cfg)
        npz = tmp / f"{key}.npz"
        np.savez(npz, u=u, v=v, s=s, n_u=cfg.n_u, n_v=cfg.n_v)
        del u, v, s
        res = {}
        for lib in a.libs:
            out = subprocess.run([sys.executable, __file__, "--libs", lib, "--child", lib, str(npz), "--reps",
                                  str(a.reps), "--algo", str(a.algo), "--flags", str(a.flags), "--op", a.op],
                                 capture_output=True, text=True)
            line = [x for x in out.stdout.splitlines() if x.startswith("{")]
            res[lib] = json.loads(line[-1]) if line else {"error": out.stderr[-400:]}
            print(key, Path(lib).name, json.dumps(res[lib]), flush=True)
        counts = {json.dumps((r.get("balanced"), r.get("unbalanced"))) for r in res.values()}
        print(key, "counts agree" if len(counts) == 1 else f"COUNTS DIFFER {counts}", flush=True)
        npz.unlink()


if __name__ == "__main__":
    main()
