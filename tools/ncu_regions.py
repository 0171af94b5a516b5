"""Executed warp instructions and stall samples per code region of bbc_count.cu, from an
ncu source page (--page source --csv --print-source cuda,sass).  Regions are the
functions / lambdas of the file, found by their definition lines."""
import csv
import re
import sys
from collections import defaultdict

src_csv, cu = sys.argv[1], sys.argv[2]
defs = []
for i, line in enumerate(open(cu), 1):
    m = re.match(r"^(?:__device__|__global__)[^(]*?\b(\w+)\(", line) or re.match(r"^\s*auto (\w+) = \[&\]", line)
    if m:
        defs.append((i, m.group(1)))
defs.sort()


def region(ln):
    name = "top"
    for i, n in defs:
        if i <= ln:
            name = n
    return name


rows = list(csv.reader(open(src_csv)))
inst, samp = defaultdict(int), defaultdict(int)
cur = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1]
        continue
    if not r or r[0] == "Line No" or len(r) < 8 or r[2] != "-" or not cur or not cur.endswith(cu.split("/")[-1]):
        continue
    try:
        ln = int(r[0])
        s, n = int(r[4] or 0), int(r[7] or 0)
    except ValueError:
        continue
    inst[region(ln)] += n
    samp[region(ln)] += s
ti, ts = sum(inst.values()) or 1, sum(samp.values()) or 1
print(f"total warp instructions {ti:.4g}, samples {ts}")
for k in sorted(inst, key=lambda k: -inst[k]):
    print(f"{k:22s} inst {100 * inst[k] / ti:5.1f}%  samples {100 * samp[k] / ts:5.1f}%")
