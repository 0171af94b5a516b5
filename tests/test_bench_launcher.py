"""bench.py's multi-GPU launcher on CPU: `python bench.py --gpus 2` without torchrun must
re-execute itself under torch.distributed.run, rendezvous on 127.0.0.1 and print exactly
one JSON line from rank 0 (`--launcher-selftest` swaps the count for a gloo all-reduce,
so no GPU is needed)."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("n", [2, 3])
def test_bench_spawns_n_ranks_and_prints_one_line(n):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", str(n), "--launcher-selftest"],
                       capture_output=True, text=True, timeout=300, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    rec = json.loads(lines[0])
    assert rec == {"selftest": "launcher", "n_gpus": n, "gpus_requested": n, "rank_sum": n * (n + 1) // 2}


def test_reference_arm_needs_no_launcher():
    """--impl reference with --gpus N runs on the launching process only (rank 0)."""
    src = (ROOT / "bench.py").read_text()
    assert src.index('if args.impl == "reference"') < src.index("return spawn(args)")
