#!/usr/bin/env python
"""Benchmark: admitted wedges/sec of balanced/unbalanced butterfly counting on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

Workload (BASELINE.json configs[1]): synthetic Chung-Lu signed bipartite graph, |U| = 1M,
|V| = 500k, 20M distinct edges, 30 % negative (paper_2601_17707_b200/synth.py, seed 2).
A "step" is one full count of the graph (G-BBC++ kernel incl. closing) with the CSR
resident in HBM; with N ranks (torchrun, or `--gpus N` alone, which re-executes itself
under torch.distributed.run) rank r uploads edge shard r, the shards are all-gathered
over NVLink, every rank builds the replicated CSR, counts its share of the start
vertices, and the counters are summed with one NCCL all-reduce.

JSON line (rank 0): value = W_S / (max over ranks of the device-timed step), W_S the
admitted wedges of the whole graph; `e2e` = the same metric through the public C ABI
from pinned HOST edge arrays (upload + device preprocessing + count + result read-back
per step); `roofline` for the count kernel; `cpu_baseline` = the CPU oracle port
(oracle/bbc_oracle.c, restating the reference's bucket engine) on this host's cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "wedges/sec and end-to-end count time (device-timed) at 1/2/4/8 B200 vs CPU reference"
UNIT = "wedges/s"
L2_FLUSH_BYTES = 512 << 20


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", type=int, default=2)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--algo", choices=("gbbc++", "gbbc"), default="gbbc++")
    p.add_argument("--e2e-steps", type=int, default=None)
    p.add_argument("--cpu-seconds", type=float, default=15.0, help="CPU baseline sample budget")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-extensions", action="store_true", help="skip the 8(f) classification / (2,k) timings")
    p.add_argument("--ext-configs", default="3,5,4",
                   help="other BASELINE configs timed in `extensions` (G-BBC vs G-BBC++, roofline); '' = none")
    p.add_argument("--launcher-selftest", action="store_true",
                   help="spawn/rendezvous check only (gloo, no GPU): rank 0 prints one JSON line")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def spawn(args) -> int:
    """`bench.py --gpus N` without a launcher: re-exec under torch.distributed.run with N
    ranks on 127.0.0.1 (one process per GPU); rank 0 prints the JSON line."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # communicator logging: the ranks NCCL saw
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(ROOT / "bench.py"), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def launcher_selftest(args) -> int:
    """The launcher without a GPU: gloo rendezvous, one all-reduce, one JSON line."""
    import torch
    import torch.distributed as dist

    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    t = torch.tensor([rank + 1], dtype=torch.int64)
    if world > 1:
        dist.all_reduce(t)
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"selftest": "launcher", "n_gpus": world, "gpus_requested": args.gpus,
                          "rank_sum": int(t.item())}), flush=True)
    return 0


def config_dict(cfg, w_u: int, w_v: int, algo: str, world: int) -> dict:
    """The workload description both arms print (same keys and values)."""
    side = "U" if w_u <= w_v else "V"
    return {"workload": cfg.name, "n_u": cfg.n_u, "n_v": cfg.n_v, "edges": cfg.m, "p_neg": cfg.p_neg,
            "gamma": cfg.gamma_u, "seed": cfg.seed, "anchor_side": side, "W_S": min(w_u, w_v), "W_U": w_u,
            "W_V": w_v, "algo": algo,
            "parallelism": f"start-vertex partition x{world}, CSR replicated (sharded upload + all-gather), "
                           f"counter all-reduce",
            "l2": f"{L2_FLUSH_BYTES >> 20} MiB buffer overwritten between timed steps"}


def measured_peaks() -> dict:
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = Path("/tmp") / f"bbc_clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.QUERY}",
                                          "--format=csv,noheader,nounits", "-lms", "50"], stdout=self.fh,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self) -> dict:
        if self.proc is None or not self.path.exists():
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = [r.split(", ") for r in self.path.read_text().strip().splitlines() if r.strip()]
        rows = [r for r in rows if len(r) >= 9]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].strip().lower() == "active"})
        loaded = [x for x in sm if x > 0.5 * max(mx or [1])] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return ""


def cpu_port_rate(n_u, n_v, u, v, s, budget_s: float, steps: int = 1, warmup: int = 0) -> dict:
    """Time the oracle port (reference bucket engine restated in C) on a bounded anchor sample."""
    from oracle.oracle import OracleGraph

    threads = len(os.sched_getaffinity(0))
    g = OracleGraph(n_u, n_v, u, v, s)
    probe_stride = 997
    t0 = time.perf_counter()
    r = g.count(side=-1, threads=threads, stride=probe_stride)
    t_probe = max(time.perf_counter() - t0, 1e-3)
    est_full = t_probe * probe_stride
    stride = max(1, int(est_full / max(budget_s, 1e-3)) + 1)
    rates, secs, adm = [], [], 0
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        r = g.count(side=-1, threads=threads, stride=stride)
        dt = time.perf_counter() - t0
        if i >= warmup:
            rates.append(r.admitted / dt)
            secs.append(dt)
            adm = r.admitted
    g.close()
    return {"value": statistics.median(rates), "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"anchors a with a % {stride} == 0 on the reference's min_side ({adm} admitted wedges, "
                      f"reference filter prank[w] < prank[u]); graph build excluded as in cli.py:215",
            "cpu": cpu_model(), "stride": stride, "sample_wedges": adm, "step_s": statistics.median(secs)}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2601_17707_b200 import synth

    cfg = synth.CONFIGS[args.config]
    u, v, s = synth.generate(cfg)
    budget = max(2.0, 150.0 / max(args.steps + args.warmup, 1))
    cb = cpu_port_rate(cfg.n_u, cfg.n_v, u, v, s, budget, steps=args.steps, warmup=args.warmup)
    from oracle.oracle import OracleGraph

    og = OracleGraph(cfg.n_u, cfg.n_v, u, v, s)
    w_u, w_v = og.admitted_total(0), og.admitted_total(1)
    og.close()
    w_ref = w_u if cfg.n_u <= cfg.n_v else w_v  # the reference's min_side (graph.py:174-176)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["step_s"] * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic", "config": config_dict(cfg, w_u, w_v, args.algo, args.gpus),
            "cpu_baseline": cb, "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0},
            "full_graph_ms_extrapolated": w_ref / cb["value"] * 1e3,
            "note": "reference = oracle/bbc_oracle.c, a C restatement of the reference's Python bucket engine "
                    "(buckets.py:166-197) pinned to its golden vectors, on every host core; each step counts the "
                    "anchor sample named in cpu_baseline.sample (ms_per_step is that sample's time, value its "
                    "admitted wedges / s); the Python package is absent on this box"}
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(args)
    if args.launcher_selftest:
        return launcher_selftest(args)
    import torch
    import torch.distributed as dist

    from paper_2601_17707_b200 import _lib, synth
    from paper_2601_17707_b200.distributed import build_replicated, shard_bounds

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = synth.CONFIGS[args.config]
    u, v, s = synth.generate(cfg)  # input preparation (host), never timed
    m = cfg.m
    lo, hi = shard_bounds(m, rank, world)

    # ---- device-resident inputs: preprocessing once, then K timed count steps ----
    # rank r uploads edge shard r; the shards are all-gathered over NVLink and every rank
    # builds the replicated CSR (the first build is the cold call: context, pools)
    t0 = time.perf_counter()
    g, keep = build_replicated(cfg.n_u, cfg.n_v, m, u[lo:hi], v[lo:hi], s[lo:hi], local)
    cold_first_call_ms = (time.perf_counter() - t0) * 1e3
    g.close()
    g, keep = build_replicated(cfg.n_u, cfg.n_v, m, u[lo:hi], v[lo:hi], s[lo:hi], local)
    du, dv, ds = keep
    warm_preprocess_ms = g.count(_lib.ALGO_GBBCPP, part_index=rank, part_count=world).preprocess_ms
    algo = _lib.ALGO_GBBCPP if args.algo == "gbbc++" else _lib.ALGO_GBBC
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")
    from paper_2601_17707_b200.distributed import from_limbs, to_limbs

    red = torch.zeros(8, dtype=torch.int64, device="cuda")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def step():
        flush.fill_(1)  # overwrite L2 between steps (outside the timed events)
        torch.cuda.synchronize()
        r = g.count(algo, part_index=rank, part_count=world)
        ms = r.count_ms
        if world > 1:
            # one NCCL all-reduce of the two 128-bit counts as 32-bit limbs (exact)
            red.copy_(torch.tensor(to_limbs([r.balanced, r.unbalanced]), dtype=torch.int64))
            ev0.record()
            dist.all_reduce(red)
            ev1.record()
            ev1.synchronize()
            ms += ev0.elapsed_time(ev1)
            bal, unb = from_limbs(red.tolist())
        else:
            bal, unb = r.balanced, r.unbalanced
        return ms, bal, unb, r

    for _ in range(args.warmup):
        step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    times, results = [], None
    with ClockSampler(local) as clocks:
        wall0 = time.perf_counter()
        for _ in range(args.steps):
            ms, bal, unb, r = step()
            times.append(ms)
            results = (bal, unb, r)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        wall = time.perf_counter() - wall0
    total_ms = sum(times)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    bal, unb, r = results
    w_s = g.w_s
    ms_per_step = total_ms / args.steps
    value = w_s / (ms_per_step * 1e-3)
    count_ms_local = sum(times) / args.steps

    # ---- end-to-end through the public API from pinned host buffers ----
    # N = 1: bbc_graph_create(host arrays) + bbc_count; N > 1: this rank's shard uploaded,
    # NCCL all-gather, bbc_graph_create_device, bbc_count of the partition, all-reduce
    pu = torch.from_numpy(u[lo:hi] if world > 1 else u).pin_memory()
    pv = torch.from_numpy(v[lo:hi] if world > 1 else v).pin_memory()
    ps = torch.from_numpy(s[lo:hi] if world > 1 else s).pin_memory()
    e2e_steps = args.e2e_steps or args.steps
    e2e_times = []
    for i in range(args.warmup + e2e_steps):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        if world > 1:
            h, tmp = build_replicated(cfg.n_u, cfg.n_v, m, pu, pv, ps, local)
            r2 = h.count(algo, part_index=rank, part_count=world)
            red.copy_(torch.tensor(to_limbs([r2.balanced, r2.unbalanced]), dtype=torch.int64))
            dist.all_reduce(red)
            from_limbs(red.tolist())
            del tmp
        else:
            h = ctypes_create(pu, pv, ps, cfg, local)
            r2 = h.count(algo)
        dt = time.perf_counter() - t0
        h.close()
        if i >= args.warmup:
            e2e_times.append(dt)
    e2e_s = statistics.median(e2e_times)
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_launch = 11  # own kernels per e2e step: 10 preprocessing + 1 count (CUB sort/scan kernels excluded)

    # ---- roofline of the count kernel ----
    peaks = measured_peaks()
    peak = float(peaks.get("hbm_gbs", 6650.0))
    n_s = g.n_anchors
    alg_bytes = 4 * w_s + 12 * m + 8 * n_s
    achieved = alg_bytes / world / (count_ms_local * 1e-3) / 1e9  # per GPU: each counts ~1/world of the wedges
    traffic, traffic_src = None, None
    profs = sorted((ROOT / "profiles").glob(f"r*_k_count_config{args.config}.json"))
    if profs:  # dram__bytes_read.sum + dram__bytes_write.sum of the latest committed ncu capture
        try:
            traffic = json.loads(profs[-1].read_text()).get("traffic_bytes")
            traffic_src = f"profiles/{profs[-1].name}"
        except Exception:
            traffic = None

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u32", "data": "synthetic",
        "config": config_dict(cfg, g.w_u, g.w_v, args.algo, world),
        "counts": {"balanced": bal, "unbalanced": unb, "total": bal + unb},
        "count_ms": ms_per_step,
        "preprocess_ms": warm_preprocess_ms,
        "cold_first_call_ms": cold_first_call_ms,
        "wall_s_timed_region": wall,
        "gpu_launches": args.steps,
        "e2e": {"value": w_s / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 9 * m,
                "d2h_bytes_per_step": (64 + 8 + 32 + 8 * r.blocks) * world, "end_to_end_count_ms": e2e_s * 1e3,
                "gpu_launches_per_step": e2e_launch,
                "path": "bbc_graph_create(host arrays) + bbc_count" if world == 1 else
                        "per rank: pinned shard upload, NCCL all-gather, bbc_graph_create_device, bbc_count "
                        "(partition), NCCL all-reduce (max over ranks)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_source": traffic_src, "algorithmic_bytes": alg_bytes,
                     "bytes_model": "4*W_S + 12*|E| + 8*|S| (BASELINE.md 2)",
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)" if peaks else "fallback 6650"},
        "clocks": clocks.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_port_rate(cfg.n_u, cfg.n_v, u, v, s, args.cpu_seconds)
    g.close()
    if world == 1 and not args.no_extensions:
        line["extensions"] = extensions(cfg, du, dv, ds, local)
        ext_cfgs = [int(x) for x in args.ext_configs.split(",") if x.strip()]
        if ext_cfgs:
            del du, dv, ds, keep
            line["extensions"]["configs"] = {str(k): other_config(k, peak, local) for k in ext_cfgs
                                             if k != args.config}
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def extensions(cfg, du, dv, ds, device) -> dict:
    """SURVEY.md 8(f) rows on the same workload, device-timed (one warm-up + one timed run):
    six-way classification (U anchors, oracle.py:172-197) and balanced (2,3)-bicliques
    (count_balanced_2k_serial k = 3, buckets.py:64-154) with the size-2 side V."""
    from paper_2601_17707_b200 import _lib

    out = {}
    gu = _lib.DeviceGraph.from_device_ptrs(cfg.n_u, cfg.n_v, cfg.m, du.data_ptr(), dv.data_ptr(), ds.data_ptr(),
                                           device, _lib.SIDE_U)
    gu.classify()
    cls, ms = gu.classify()
    out["classify"] = {"ms": ms, "wedges": gu.w_s, "wedges_per_s": gu.w_s / (ms * 1e-3), "anchor_side": "U",
                       "classes": cls}
    gu.close()
    gv = _lib.DeviceGraph.from_device_ptrs(cfg.n_u, cfg.n_v, cfg.m, du.data_ptr(), dv.data_ptr(), ds.data_ptr(),
                                           device, _lib.SIDE_V)
    gv.count_2k(3)
    val, ovf, ms = gv.count_2k(3)
    out["bicliques_k3"] = {"ms": ms, "wedges": gv.w_s, "wedges_per_s": gv.w_s / (ms * 1e-3), "anchor_side": "V",
                           "count": val, "overflow": ovf}
    gv.close()
    out["loader"] = loader_rate(du, dv, ds)
    return out


def other_config(k: int, peak: float, device: int) -> dict:
    """Another BASELINE config under the bench's clock: G-BBC (static round-robin) and
    G-BBC++ (dynamic queue) device-timed counts (one warm-up, median of three), the
    per-CTA load ratios max/mean of each, measured on the device -- of admitted wedges
    (bbc_block_work, ScheduleReport.max_over_mean, tiled.py:92-97) and of busy time
    (bbc_block_busy_ns: what a persistent grid actually waits on) -- and the roofline
    fraction."""
    import torch

    from paper_2601_17707_b200 import _lib, synth

    cfg = synth.CONFIGS[k]
    t0 = time.perf_counter()
    u, v, s = synth.generate(cfg)
    gen_s = time.perf_counter() - t0
    g = _lib.DeviceGraph.from_host(cfg.n_u, cfg.n_v, u, v, s, device)
    del u, v, s
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")
    out = {"workload": cfg.name, "edges": cfg.m, "anchor_side": "UV"[g.anchor_side], "W_S": g.w_s,
           "W_U": g.w_u, "W_V": g.w_v, "gen_s": gen_s}
    alg_bytes = 4 * g.w_s + 12 * cfg.m + 8 * g.n_anchors
    for name, code in (("gbbc", _lib.ALGO_GBBC), ("gbbc++", _lib.ALGO_GBBCPP)):
        times = []
        for i in range(4):
            flush.fill_(1)
            torch.cuda.synchronize()
            r = g.count(code)
            if i:
                times.append(r.count_ms)
        work = g.block_work(r.blocks)
        busy = g.block_busy_ns(r.blocks)
        mean = sum(work) / max(len(work), 1)
        bmean = sum(busy) / max(len(busy), 1)
        ms = statistics.median(times)
        out[name] = {"count_ms": ms, "wedges_per_s": g.w_s / (ms * 1e-3), "balanced": r.balanced,
                     "unbalanced": r.unbalanced, "cta_work_max_over_mean": max(work) / mean if mean else 1.0,
                     "cta_busy_max_over_mean": max(busy) / bmean if bmean else 1.0, "blocks": r.blocks,
                     "roofline_frac": alg_bytes / (ms * 1e-3) / 1e9 / peak}
    out["counts_agree"] = (out["gbbc"]["balanced"], out["gbbc"]["unbalanced"]) == \
        (out["gbbc++"]["balanced"], out["gbbc++"]["unbalanced"])
    g.close()
    return out


def loader_rate(du, dv, ds, lines: int = 2_000_000, host_lines: int = 50_000) -> dict:
    """Device load_graph on the first `lines` edges of the workload
    written as text ("u<id> v<id> +-1"), wall time incl. the text upload, next to the host
    pipeline on a smaller prefix."""
    import numpy as np

    import paper_2601_17707_b200 as bb

    u, v, s = (x[:lines].cpu().numpy() for x in (du, dv, ds))
    text = "\n".join(np.char.add(np.char.add(np.char.add(np.char.add("u", u.astype(str)), " v"),
                                             np.char.add(v.astype(str), " ")), s.astype(str)).tolist()) + "\n"
    data = text.encode("ascii")
    times = []
    for _ in range(3):
        t0 = time.perf_counter()
        h = bb.ingest_device(data)
        times.append(time.perf_counter() - t0)
        h.close()
    dev = statistics.median(times)
    sample = "\n".join(text.split("\n", host_lines)[:host_lines]) + "\n"
    t0 = time.perf_counter()
    bb.load_graph(sample)
    host = time.perf_counter() - t0
    return {"lines": int(len(u)), "bytes": len(data), "device_s": dev, "device_lines_per_s": len(u) / dev,
            "host_lines_per_s": host_lines / host, "host_sample_lines": host_lines}


def ctypes_create(pu, pv, ps, cfg, device):
    from paper_2601_17707_b200 import _lib

    import ctypes

    h = ctypes.c_void_p()
    rc = _lib.load().bbc_graph_create(device, cfg.n_u, cfg.n_v, cfg.m, pu.data_ptr(), pv.data_ptr(), ps.data_ptr(),
                                      _lib.SIDE_CHEAPER, ctypes.byref(h))
    if rc:
        _lib._raise(rc)
    return _lib.DeviceGraph(h.value, device)


if __name__ == "__main__":
    sys.exit(main())
