"""Summarise an ncu source page (--page source --csv --print-source cuda,sass): top CUDA
lines by warp-stall samples with executed instructions and the dominant stall reasons."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = next(r for r in rows if r and r[0] == "Line No")
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
lines = []
for r in rows:
    if len(r) != len(hdr) or r[0] == "Line No" or r[2] != "-":
        continue
    try:
        samples = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        inst = int(r[ix["Instructions Executed"]] or 0)
    except ValueError:
        continue
    stalls = sorted(((int(r[ix[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
    lines.append((samples, inst, r[0], r[1].strip()[:70], stalls))
tot = sum(x[0] for x in lines) or 1
toti = sum(x[1] for x in lines) or 1
print(f"total samples {tot}, warp instructions {toti}")
for s, i, ln, src, st in sorted(lines, reverse=True)[:top]:
    print(f"{100*s/tot:5.1f}% inst {100*i/toti:5.1f}%  L{ln:>4} {src:70s} {' '.join(f'{n}:{100*c/max(s,1):.0f}%' for c, n in st if c)}")
