"""Executed warp instructions and stall samples per code region, from an ncu source page
(--page source --csv --print-source cuda,sass).  Regions are the functions / lambdas /
structs of each source file, found by their definition lines.

    python tools/ncu_regions.py src.csv [top]
"""
import csv
import re
import sys
from collections import defaultdict
from pathlib import Path

_defs: dict[str, list] = {}


def defs_of(path: str) -> list:
    if path not in _defs:
        d = []
        p = Path(path)
        if p.exists():
            for i, line in enumerate(p.read_text().splitlines(), 1):
                m = (re.match(r"^(?:__device__|__global__|static __device__)[^(]*?\b(\w+)\(", line)
                     or re.match(r"^\s*auto (\w+) = \[&\]", line) or re.match(r"^struct (\w+)", line))
                if m:
                    d.append((i, m.group(1)))
        _defs[path] = sorted(d)
    return _defs[path]


def region(path: str, ln: int) -> str:
    name = "top"
    for i, n in defs_of(path):
        if i <= ln:
            name = n
    return f"{Path(path).name}:{name}"


def regions(rows: list) -> tuple[dict, dict]:
    """(instructions, stall samples) per file:region from the rows of a source page."""
    inst, samp = defaultdict(int), defaultdict(int)
    cur = None
    for r in rows:
        if len(r) >= 2 and r[0] in ("File Path", "File Name"):
            cur = r[1]
            continue
        if not r or r[0] == "Line No" or len(r) < 8 or r[2] != "-" or not cur:
            continue
        try:
            ln = int(r[0])
            s, n = int(r[4] or 0), int(r[7] or 0)
        except ValueError:
            continue
        key = region(cur, ln)
        inst[key] += n
        samp[key] += s
    return inst, samp


if __name__ == "__main__":
    src_csv = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    inst, samp = regions(list(csv.reader(open(src_csv))))
    ti, ts = sum(inst.values()) or 1, sum(samp.values()) or 1
    print(f"total warp instructions {ti:.4g}, samples {ts}")
    for k in sorted(inst, key=lambda k: -inst[k])[:top]:
        print(f"{k:40s} inst {100 * inst[k] / ti:5.1f}%  samples {100 * samp[k] / ts:5.1f}%")
