#!/usr/bin/env python
"""Benchmark: FP64 Tikhonov-Toeplitz solves/sec on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c5|c1|c3|c4|c5b]
                    [--impl ours|reference] [--refine R] [--batch B]

One process per GPU (torchrun for N > 1, NCCL).  A step solves one batch of
the config's synthetic systems per rank (weak scaling: fixed work per rank);
with N > 1 the solutions are gathered to rank 0 inside the step (the path's
only collective).  Default workload = BASELINE configs[1] (config 2: T 8192 x
4096, l2 with beta = 0.1, 64 right-hand sides sharing T).

Printed JSON (rank 0): the contract keys plus
  e2e          same metric through the public API with host buffers
               (DeviceBatch.stage -> run -> fetch, H2D/D2H inside the timing)
  roofline     the dominant kernel class: leaf classes FP64-bound against the
               FP64 FMA peak measured by tr_fp64_peak(); FFT / combine /
               update HBM-bound against MEASURED_PEAKS.json hbm_gbs
  roofline_hbm the batched-FFT class against the measured HBM peak (tracked from round 1)
  roofline_solve  the whole solve against SURVEY 8(d)'s summed roofline
  chain        the sequential absorption chain: conditions per
               solve and the leaf time per absorbed condition
  kernels      per-class device time from CUDA events (separate pass)
  cpu_baseline the oracle port of the reference, timed on this host's cores
  clocks       nvidia-smi samples taken during the timed region
  gpu_launches kernels this library launched inside the timed region
`--impl reference` times the reference algorithm (oracle/toepreg_oracle.py,
a bit-exact numpy restatement of toepreg) on the host cores instead.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import multiprocessing as mp
import os
import platform
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402

METRIC = "FP64 Tikhonov-Toeplitz solves/sec"


# ---------------------------------------------------------------- workloads
def make_workload(cfg: str, rank: int, batch: int, world: int = 1):
    """Raw problem dict + count for this rank.

    c2 (the default): the 64 right-hand sides of ONE config-2 instance are
    split contiguously over the ranks (strong scaling: 64 / N per rank); c5:
    ``batch`` independent systems per rank, items rank*batch... (weak
    scaling); single-system configs run one replica per rank (item = rank)."""
    from paper_1302_6945_b200 import workloads as wl
    from paper_1302_6945_b200.dist import shard_range
    if cfg == "c2":
        total = batch or 64
        raw = wl.c2_rect(nrhs=total, seed=0, item=0)
        lo, hi = shard_range(total, rank, world)
        raw = dict(raw, b=raw["b"][lo:hi], x_true=raw["x_true"][lo:hi])
        return raw, hi - lo, "c2: T 8192x4096 real (l2, beta=0.1), shared by %d RHS (%d on this rank)" % (
            total, hi - lo)
    if cfg == "c5":
        b = batch or 256
        raw = wl.c5_random(n=16384, count=b, seed=0, first=rank * b)
        return raw, b, "c5: %d independent square systems n=16384 (l2, beta=0.1) per rank" % b
    if cfg == "c1":
        raw = wl.c1_blur(256, seed=0, item=rank)
        return raw, 1, "c1: Gaussian blur n=256 (l2, lambda=1e-2)"
    if cfg == "c4":
        raw = wl.c4_nufft(seed=0, item=rank)
        return raw, 1, "c4: NUFFT gramian m=8192 n=16384 (L=0.01 I)"
    if cfg == "c5b":
        raw = wl.c5_random(n=1 << 22, count=1, seed=0, first=rank)
        return raw, 1, "c5b: one square system n=2^22 (l2, beta=0.1)"
    if cfg == "c3":
        # BASELINE config 3: one instance, lambda swept over four values -- the
        # four systems (same T and b, L scaled) are one batch of independent solves
        lams = (1e-3, 1e-2, 1e-1, 1.0)
        raws = [wl.c3_firstdiff(n=65536, lam=l, seed=0, item=rank) for l in lams]
        return raws, len(raws), "c3: general n=65536, first-difference L, lambda in {1e-3, 1e-2, 1e-1, 1} (one batch of 4)"
    raise SystemExit(f"unknown config {cfg}")


def problems_from(raw, count, mod=None):
    if mod is None:
        import paper_1302_6945_b200 as mod
    from paper_1302_6945_b200 import workloads as wl
    if isinstance(raw, (list, tuple)):  # one raw problem per system
        return [wl.to_problem(r, mod) for r in raw]
    if count == 1 and np.asarray(raw.get("b", raw.get("normal_rhs"))).ndim == 1:
        return [wl.to_problem(raw, mod)]
    return [wl.to_problem(raw, mod, i) for i in range(count)]


# ---------------------------------------------------------------- CPU side
# The reference's CPU path (the oracle port: a bit-exact numpy restatement of
# toepreg, one core per solve as the reference itself) in a persistent pool
# of one process per core.  Each worker synthesises the workload ONCE in its
# initializer; a timed step only runs solves.
_CPU_PROBS = None


def _cpu_init(cfg, batch):
    global _CPU_PROBS
    os.environ["OMP_NUM_THREADS"] = "1"
    import toepreg_oracle as O  # noqa: F401  (import cost outside the timing)
    raw, count, _ = make_workload(cfg, 0, batch)
    _CPU_PROBS = problems_from(raw, count)


def _cpu_solve(i):
    import toepreg_oracle as O
    prob = _CPU_PROBS[i % len(_CPU_PROBS)]
    t0 = time.perf_counter()
    O.solve(prob)
    return time.perf_counter() - t0


class CpuReference:
    def __init__(self, cfg, batch, cores):
        self.cores = cores
        self.pool = mp.get_context("spawn").Pool(cores, initializer=_cpu_init, initargs=(cfg, batch))
        self.pool.map(abs, range(cores))  # workers up and initialised (untimed)

    def step(self, nsolve):
        """Solve `nsolve` systems (items 0..nsolve-1 of the workload);
        returns (wall s, per-solve seconds)."""
        t0 = time.perf_counter()
        singles = self.pool.map(_cpu_solve, range(nsolve), chunksize=1)
        return time.perf_counter() - t0, singles

    def close(self):
        self.pool.terminate()
        self.pool.join()


def cpu_step_size(cfg, count, cores):
    """Systems per CPU step: the whole workload when it is at most 8 solves
    per core (c2: all 64 right-hand sides), else one per core."""
    return count if count <= 8 * cores else cores


# ---------------------------------------------------------------- clocks
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except (ValueError, IndexError):
                continue
            for name, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def hbm_peak_gbs():
    """HBM copy bandwidth from the driver-written MEASURED_PEAKS.json, else
    the profiling recipe's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        for k in ("hbm_gbs", "hbm_copy_gbs", "hbm_GBps"):
            if k in d:
                return float(d[k]), f"MEASURED_PEAKS.json:{k}"
    except (OSError, ValueError):
        pass
    return 7700.0, "B200_PROFILING.md fallback"


def ncu_traffic(cfg, cls):
    """dram__bytes_read+write per launch of the class, averaged over the
    class's launches in the committed ncu launch list of the same bench
    command (profiles/traffic.json, written by tools/profile_summary.py for the
    latest capture), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)[cfg][cls]["dram_bytes_per_launch"]
    except (OSError, ValueError, KeyError):
        return None


# ---------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--refine", type=int, default=1)
    ap.add_argument("--refine-cg", type=int, default=256)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference(args, rank)

    import torch
    import torch.distributed as dist
    import paper_1302_6945_b200 as tb
    from paper_1302_6945_b200 import _lib
    from paper_1302_6945_b200.dist import gather_solutions

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = _lib.load()

    raw, count, label = make_workload(args.config, rank, args.batch, world)
    total_systems = (args.batch or 64) if args.config == "c2" else count * world
    probs = problems_from(raw, count)
    cfg = tb.SolverConfig(refine=args.refine, refine_cg=args.refine_cg)
    db = tb.DeviceBatch(probs, cfg).stage()
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    def step(fetch_host=False, stage=False):
        if stage:
            db.stage()
        db.run(with_diag=False)
        if world > 1:
            gather_solutions(db.x, total_systems, dst=0)
        if fetch_host:
            db.x_host.copy_(db.x, non_blocking=True)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    # ---- device-resident timed region ----
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = lib.tr_launch_count()
    torch.cuda.profiler.start()  # ncu --profile-from-start off sees the timed region only
    with ClockSampler(local) as clk:
        for a, b in evs:
            flush.fill_(1)  # L2 flush (256 MiB write) between timed steps
            a.record(stream)
            step()
            b.record(stream)
        torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    launches = lib.tr_launch_count() - launches0
    if world > 1:
        dist.barrier()
    dev_ms = sum(a.elapsed_time(b) for a, b in evs)
    t = torch.tensor([dev_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    value = total_systems * args.steps / (ms_total / 1e3)

    # ---- end to end through the public API with host buffers ----
    e_evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
             for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for a, b in e_evs:
        flush.fill_(1)
        a.record(stream)
        step(fetch_host=True, stage=True)
        b.record(stream)
    torch.cuda.synchronize()
    e_ms = sum(a.elapsed_time(b) for a, b in e_evs)
    te = torch.tensor([e_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = total_systems * args.steps / (float(te.item()) / 1e3)

    # ---- per-kernel-class timing pass (CUDA events around each launch) ----
    lib.tr_kernel_timing(1)
    nk = 2
    for _ in range(nk):
        step()
    torch.cuda.synchronize()
    kst = _lib.kernel_stats()
    lib.tr_kernel_timing(0)
    peak = C.c_double()
    lib.tr_fp64_peak(C.byref(peak))
    info = tb.plan_info(probs[0], cfg)

    if world > 1:
        dist.barrier()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # roofline of the dominant class: algorithmic work (the library counts
    # minimal bytes / useful flops per launch) / its event time
    tot_k = sum(v[0] for v in kst.values()) or 1.0
    dom = max(kst, key=lambda k: kst[k][0])
    hbm_peak, hbm_src = hbm_peak_gbs()
    ms, nl, by, fl = kst[dom]
    if dom in ("leaf_pivot", "leaf_build", "leaf_check", "leaf_exact"):
        ach = fl / (ms * 1e-3) / 1e12
        roof = {"kernel": dom, "bound": "fp64", "achieved": ach, "peak": peak.value,
                "unit": "TFLOP/s", "peak_source": "measured FP64 FMA burst (tr_fp64_peak); "
                                                  "MEASURED_PEAKS.json has no FP64 entry"}
    else:
        ach = by / (ms * 1e-3) / 1e9
        roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": hbm_peak,
                "unit": "GB/s", "peak_source": hbm_src}
    roof["frac"] = ach / roof["peak"] if roof["peak"] else None
    roof["traffic"] = ncu_traffic(args.config, dom)
    roof["algorithmic_bytes_per_launch"] = by / max(nl, 1)
    roof["algorithmic_flops_per_launch"] = fl / max(nl, 1)
    roof["avg_launch_ms"] = ms / max(nl, 1)
    roof["share_of_step"] = ms / tot_k

    # the HBM-bound class the round-1 review tracks (batched FFT), whatever the dominant class is
    roof_hbm = None
    if "fft" in kst and kst["fft"][0] > 0:
        fms, fnl, fby, ffl = kst["fft"]
        fach = fby / (fms * 1e-3) / 1e9
        roof_hbm = {"kernel": "fft", "bound": "hbm", "achieved": fach, "peak": hbm_peak, "unit": "GB/s",
                    "peak_source": hbm_src, "frac": fach / hbm_peak if hbm_peak else None,
                    "traffic": ncu_traffic(args.config, "fft"),
                    "algorithmic_bytes_per_launch": fby / max(fnl, 1), "avg_launch_ms": fms / max(fnl, 1),
                    "share_of_step": fms / tot_k}
    # whole solve against SURVEY 8(d)'s summed per-class roofline (T_roof per solve at 37 TFLOP/s
    # FP64 and 6.449 TB/s: the table's "roofline solves/s/GPU" column)
    roof_table = {"c1": 5.5e5, "c2": 2.24e4, "c3": 667.0, "c4": 6.49e3, "c5": 6.49e3, "c5b": 17.5}
    roof_solve = None
    if args.config in roof_table:
        rs = roof_table[args.config] * world
        roof_solve = {"roofline_solves_per_s": rs, "frac": value / rs,
                      "source": "SURVEY 8(d): sum over kernel classes of max(flops / FP64 peak, bytes / HBM peak)"}

    # the sequential absorption chain: every condition of a solve passes
    # through one leaf sweep in order (SURVEY 8(d) chain bound C x t_step);
    # groups of <= 148 systems (solver.cu batch_groups) run one after the
    # other in this eager timing pass, their systems in parallel
    raw0 = raw[0] if isinstance(raw, (list, tuple)) else raw
    rows = 3 if raw0.get("variant", "") == "general" else 2
    n_cond = rows * info["order"]
    groups = 1 if count < 32 else (3 if count <= 148 else min(8, -(-count // 148)))  # solver.cu batch_groups
    leaf_ms = sum(kst[k][0] for k in ("leaf_pivot", "leaf_build", "leaf_check", "leaf_exact") if k in kst) / nk
    leaf_launches = kst.get("leaf_pivot", (0, 0))[1] / nk
    solves = max(1.0, round(leaf_launches / max(groups * info["leaves"], 1)))
    chain = {"conditions_per_solve": n_cond, "groups": groups, "direct_solves_per_system": solves,
             "leaf_ms_per_step": leaf_ms,
             "ns_per_condition": leaf_ms * 1e6 / (groups * solves * n_cond),
             "bound": "latency of the pivot chain (one CTA per system and leaf)"}

    out = {
        "metric": METRIC,
        "value": value,
        "unit": "solves/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": max(args.warmup, 3),
        "ms_per_step": ms_total / args.steps,
        "higher_is_better": True,
        "scaling": "strong" if args.config == "c2" else "weak",
        "vs_baseline": None,
        "dtype": "c128 (fp64)",
        "data": "synthetic (seeded BASELINE-config generators, paper_1302_6945_b200/workloads.py)",
        "config": {"workload": label, "config": args.config, "systems_per_rank": count,
                   "order_N": info["order"], "leaves": info["leaves"], "leaf_conditions": info["max_leaf_conditions"],
                   "refine": args.refine, "refine_cg_max_iterations": args.refine_cg, "parallelism": f"dp{world} (systems sharded, gather x to rank 0)",
                   "l2": "256 MiB device write between timed steps (outside the per-step events)",
                   "timing": "CUDA events per step on the launching stream, summed; max over ranks"},
        "e2e": {"value": e2e_value, "unit": "solves/s", "h2d_bytes_per_step": db.h2d_bytes,
                "d2h_bytes_per_step": db.d2h_bytes,
                "path": "DeviceBatch.stage (pinned H2D) -> run -> x D2H"},
        "roofline": roof,
        "roofline_hbm": roof_hbm,
        "roofline_solve": roof_solve,
        "chain": chain,
        "kernels": {k: {"ms_per_step": v[0] / nk, "launches_per_step": v[1] / nk,
                        "share": v[0] / tot_k,
                        "alg_GBps": v[2] / (v[0] * 1e-3) / 1e9 if v[0] else None,
                        "alg_TFLOPs": v[3] / (v[0] * 1e-3) / 1e12 if v[0] else None}
                    for k, v in kst.items() if v[1]},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        ref = CpuReference(args.config, args.batch, cores)
        nsolve = cpu_step_size(args.config, count, cores)
        wall, singles = ref.step(nsolve)
        ref.close()
        out["cpu_baseline"] = {"value": nsolve / wall, "unit": "solves/s", "cores": cores, "kind": "port",
                               "sample": f"{nsolve} of the {count} systems of {args.config} solved by the "
                                         f"oracle (bit-exact numpy restatement of toepreg) in a pool of "
                                         f"{cores} single-threaded processes, inputs built before timing; "
                                         f"{wall:.1f} s wall, 1-core mean {statistics.mean(singles):.2f} s/solve "
                                         f"(cores / mean = {cores / statistics.mean(singles):.2f} solves/s); "
                                         f"{platform.processor() or 'x86_64'}"}
    print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


def run_reference(args, rank):
    """The reference algorithm (oracle port, bit-exact with toepreg) on the
    host cores; rank 0 only (other ranks exit without work)."""
    if rank != 0:
        return
    raw, count, label = make_workload(args.config, 0, args.batch)
    cores = os.cpu_count() or 1
    ref = CpuReference(args.config, args.batch, cores)
    nsolve = cpu_step_size(args.config, count, cores)
    for _ in range(max(args.warmup, 0)):
        ref.step(nsolve)
    walls, singles = [], []
    for _ in range(args.steps):
        w, s1 = ref.step(nsolve)
        walls.append(w)
        singles.extend(s1)
    ref.close()
    total = sum(walls)
    value = nsolve * args.steps / total
    mean1 = statistics.mean(singles)
    out = {
        "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "strong" if args.config == "c2" else "weak",
        "vs_baseline": None, "dtype": "c128 (fp64)",
        "data": "synthetic (seeded BASELINE-config generators)", "impl": "reference",
        "config": {"workload": label, "config": args.config, "systems_per_step": nsolve,
                   "same_config": nsolve == count},
        "cpu_baseline": {"value": value, "unit": "solves/s", "cores": cores, "kind": "port",
                         "sample": f"{nsolve} systems per step in a persistent pool of {cores} "
                                   f"single-threaded processes (inputs built once per worker, untimed); "
                                   f"1-core mean {mean1:.3f} s/solve, cores / mean = {cores / mean1:.2f} solves/s"},
        "latency_1core_s": mean1,
        "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
