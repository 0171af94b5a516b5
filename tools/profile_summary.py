"""Summarise an ncu --set full report of k_count into a JSON file under profiles/.

    python tools/profile_summary.py gpurun_out/prof_X.ncu-rep profiles/<name>.json [--wedges W --edges E --anchors S]

Records the north_star evidence counters: duration, DRAM bytes (traffic), achieved DRAM
GB/s, L2 hit rate, shared-memory atomic instructions / wavefronts / bank conflicts and
pipe utilisation, warp execution efficiency, issue-slot utilisation, occupancy, and the
top source lines by stall samples (from --page source).
"""

import argparse
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__bytes_read.sum.per_second": "dram_read_per_s",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "smsp__inst_executed_op_shared_atom.sum": "shared_atom_inst",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum": "shared_atom_wavefronts",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum": "shared_atom_bank_conflicts",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum.pct_of_peak_sustained_elapsed": "shared_atom_pipe_pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "warp_exec_efficiency_threads",
    "sm__inst_executed.sum": "warp_inst",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__block_size": "block_size",
    "launch__grid_size": "grid_size",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
}
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0,
         "Gbyte/s": 1e9, "Tbyte/s": 1e12, "Mbyte/s": 1e6}


def raw_metrics(rep: str) -> list[dict]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    launches = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else ""}
        for i, h in enumerate(hdr):
            if h in WANT:
                try:
                    v = float(vals[i].replace(",", ""))
                except ValueError:
                    continue
                d[WANT[h]] = v * SCALE.get(units[i], 1.0)
        launches.append(d)
    return launches


def hot_lines(rep: str, top: int = 12) -> tuple[list[dict], dict]:
    """Top source lines by stall samples (all files) and instructions / samples per region."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    import ncu_regions

    inst, samp = ncu_regions.regions(rows)
    ti, ts = sum(inst.values()) or 1, sum(samp.values()) or 1
    regs = {k: {"inst_pct": round(100 * inst[k] / ti, 1), "samples_pct": round(100 * samp[k] / ts, 1)}
            for k in sorted(inst, key=lambda k: -inst[k])[:20]}
    lines, cur, ix, stall_cols = [], None, None, []
    for r in rows:
        if len(r) >= 2 and r[0] in ("File Path", "File Name"):
            cur = Path(r[1]).name
            continue
        if r and r[0] == "Line No":
            ix = {h: i for i, h in enumerate(r)}
            stall_cols = [h for h in r if h.startswith("stall_") and "Not Issued" not in h]
            continue
        if ix is None or len(r) != len(ix) or r[2] != "-":
            continue
        try:
            s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
            n = int(r[ix["Instructions Executed"]] or 0)
        except ValueError:
            continue
        st = sorted(((int(r[ix[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:2]
        lines.append((s, n, f"{cur}:{r[0]}", r[1].strip()[:90], st))
    return ([{"line": ln, "samples_pct": round(100 * s / ts, 1), "inst_pct": round(100 * n / ti, 1), "source": src,
              "stalls": {k: round(100 * c / max(s, 1)) for c, k in st}}
             for s, n, ln, src, st in sorted(lines, reverse=True)[:top]], regs)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("report")
    p.add_argument("out")
    p.add_argument("--wedges", type=int, default=0)
    p.add_argument("--edges", type=int, default=0)
    p.add_argument("--anchors", type=int, default=0)
    p.add_argument("--peak-gbs", type=float, default=6538.6)
    p.add_argument("--note", default="")
    a = p.parse_args()
    launches = raw_metrics(a.report)
    k = next((x for x in launches if "k_count" in x.get("kernel", "")), launches[0] if launches else {})
    summary = {"report": Path(a.report).name, "kernel": k.get("kernel"), "metrics": k, "note": a.note}
    if a.wedges and k.get("duration"):
        alg = 4 * a.wedges + 12 * a.edges + 8 * a.anchors
        summary["algorithmic_bytes"] = alg
        summary["traffic_bytes"] = k.get("dram_read", 0) + k.get("dram_write", 0)
        summary["achieved_algorithmic_gbs"] = alg / k["duration"] / 1e9
        summary["frac_of_measured_hbm_peak"] = summary["achieved_algorithmic_gbs"] / a.peak_gbs
        summary["wedges_per_s_under_profiler"] = a.wedges / k["duration"]
    summary["hot_lines"], summary["regions"] = hot_lines(a.report)
    Path(a.out).write_text(json.dumps(summary, indent=1) + "\n")
    print(json.dumps({x: summary.get(x) for x in ("kernel", "traffic_bytes", "achieved_algorithmic_gbs",
                                                    "frac_of_measured_hbm_peak")}, indent=1))


if __name__ == "__main__":
    main()
