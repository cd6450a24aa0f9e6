#!/usr/bin/env python3
"""Benchmark: triangle projections/sec of the Dykstra sweep (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--tile-b 40]
    python bench.py --impl reference ...        # CPU reference arm (oracle port)

Default workload: BASELINE config 3 (n = 4000 Chung-Lu), the largest config
BASELINE.json assigns to one GPU.
A "step" is one full Dykstra pass (all 3*C(n,3) metric rows in the paper's
tiled order + the pair phase) over the config's seeded synthetic instance.
``value`` = K * 3*C(n,3) * N / t with t the device time (CUDA events on the
library's stream) of the K timed passes, max over ranks; L2 is flushed
(256 MiB write) before every timed pass.  ``e2e`` is the same metric through
the public ``solve()`` API from host arrays (instance upload, every pass,
per-pass stats and the final x/f/duals download inside the wall-clock).
Multi-GPU (torchrun) defaults to BASELINE config 4 (n = 10000) sharded over
all ranks (one instance, strong scaling); an explicit --config
without --sharded runs independent replicas, one per GPU (weak scaling).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "triangle projections/sec (whole box)"
UNIT = "projections/s"


def rows_per_pass(n):
    return 3 * (n * (n - 1) * (n - 2) // 6)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def _nvml_loop(self, h, nv):
        bits = (nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self.stop.is_set():
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            flags = ", ".join("Active" if r & bt else "Not Active" for bt in bits)
            self.lines.append(f"{sm}, {mx}, {r:#x}, {flags}")
            self.stop.wait(0.005)

    def __enter__(self):
        # in-process NVML sampling every 5 ms (the timed region is ~0.1-1 s);
        # nvidia-smi -lms 50 as the fallback when NVML is not importable
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            self.stop = threading.Event()
            self.thread = threading.Thread(target=self._nvml_loop, args=(h, nv), daemon=True)
            self.thread.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 2.0:
                time.sleep(0.001)
            self.n0 = len(self.lines)
            self.nvml = True
            return self
        except Exception:
            self.nvml = False
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._drain, daemon=True)
            self.thread.start()
            # nvidia-smi takes a few hundred ms to start: wait for its first
            # sample so the (short) timed region is sampled from its start
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.01)
            self.n0 = len(self.lines)
        except OSError:
            self.proc = None
        return self

    def _drain(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if getattr(self, "nvml", False):
            n = len(self.lines)
            t0 = time.time()
            while len(self.lines) <= n and time.time() - t0 < 0.5:
                time.sleep(0.001)
            self.stop.set()
            self.thread.join(timeout=2)
            return
        if self.proc is not None:
            # at least one sample taken after the region started
            t0 = time.time()
            while len(self.lines) <= getattr(self, "n0", 0) and time.time() - t0 < 2.0 and self.proc.poll() is None:
                time.sleep(0.005)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        # samples from the timed region (the first one was taken before it)
        for ln in (self.lines[getattr(self, "n0", 0):] or self.lines):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(config, b):
    """DRAM bytes (read + write) of one pass's tile_round_kernel launches from
    the committed ncu capture (profiles/ncu_tile_kernel.json), if any -- the
    same unit as ``achieved`` (a pass's algorithmic bytes over its time)."""
    path = os.path.join(ROOT, "profiles", "ncu_tile_kernel.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        e = d.get(f"config{config}_b{b}", {})
        if "dram_bytes_per_pass" in e:
            return e["dram_bytes_per_pass"]
        return None
    except (OSError, ValueError):
        return None


def ncu_counters(config, b):
    """Pipe / hit-rate counters of the committed full captures (one first-family
    round and the dataflow launch): FP64 pipe, shared-memory pipe, L2 / L1 hit
    rates, issue slots; None without a capture for this config."""
    path = os.path.join(ROOT, "profiles", "ncu_tile_kernel.json")
    try:
        with open(path) as fh:
            e = json.load(fh).get(f"config{config}_b{b}", {})
        out = {k: e[k] for k in ("first_family_round", "dataflow_launch", "source") if e.get(k)}
        return out if len(out) > 1 else None
    except (OSError, ValueError):
        return None


def workload_name(spec, b):
    return (f"config{list_index(spec)}: n={spec.n} {spec.name}, gamma={spec.gamma:g}, "
            f"lambda={spec.lam:g}, tiled b={b}")


def list_index(spec):
    from paper_1901_10084_b200.instances import CONFIGS
    for k, v in CONFIGS.items():
        if v is spec:
            return k
    return 0


def cpu_info():
    """CPU model and core counts of the host (reported beside every CPU rate)."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        import psutil
        phys = psutil.cpu_count(logical=False)
    except ImportError:
        phys = None
    return {"cpu_model": model, "physical_cores": phys, "logical_cpus": os.cpu_count()}


def p1_round_limit(n, b, target_rows):
    """Smallest prefix of the tiled rounds holding >= target_rows metric rows."""
    from paper_1901_10084_b200 import schedule
    acc = 0
    for r, rnd in enumerate(schedule.tiled_rounds(n, b)):
        acc += 3 * rnd.size
        if acc >= target_rows:
            return r + 1, acc
    return 0, acc


def cpu_sample(inst, b, passes_warm, passes_timed, threads, p1_rows=0):
    """Time the CPU oracle (a C port of the reference kernels, threaded like
    the reference's worker pool) on a bounded sample of the workload.
    With ``p1_rows`` also a single-thread (P = 1) rate over the first rounds
    of the next pass, started from the warmed x/f (no stored duals: the CPU
    cost is the row visits, exact steps are < 0.1% of them)."""
    from oracle import oracle
    oracle.build()
    o = oracle.OracleSolver(inst.n, inst.d_flat, inst.w_flat, inst.epsilon, b=b, workers=threads)
    for _ in range(passes_warm):
        o.run_pass()
    t0 = time.perf_counter()
    for _ in range(passes_timed):
        o.run_pass()
    dt = time.perf_counter() - t0
    p1 = None
    if p1_rows:
        limit, _ = p1_round_limit(inst.n, b, p1_rows)
        x, f = o.state()
        o1 = oracle.OracleSolver(inst.n, inst.d_flat, inst.w_flat, inst.epsilon, b=b, workers=1)
        o1.set_state(x, f)
        rows, t1 = o1.timed_rounds(limit)
        o1.close()
        p1 = {"value": rows / t1, "unit": UNIT, "cores": 1,
              "sample": f"first {limit} rounds of pass {passes_warm + passes_timed + 1} "
                        f"({rows:.3e} metric rows, {t1:.1f} s) from the warmed x/f, 1 thread"}
    o.close()
    return passes_timed * rows_per_pass(inst.n) / dt, dt, p1


def run_reference(args):
    """Reference arm: the CPU oracle (C port of the reference's numba kernels,
    threaded like its worker pool) on all host threads.  A bounded sample so
    the run ends in minutes at config 3: min(W, 1) warm-up passes, then
    min(K, 3) timed full passes."""
    ws, rank, _ = dist_env()
    if ws > 1 and rank != 0:
        return 0
    from paper_1901_10084_b200 import instances
    cfg = args.config or 3
    spec = instances.CONFIGS[cfg]
    inst = instances.config_instance(cfg)
    threads = args.cpu_threads or os.cpu_count() or 1
    warm = min(args.warmup, 1) if inst.n > 1500 else args.warmup
    timed = min(args.steps, 3) if inst.n > 1500 else args.steps
    rate, dt, _ = cpu_sample(inst, args.tile_b, warm, timed, threads)
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT,
        "n_gpus": args.gpus, "steps": timed, "warmup": warm,
        "ms_per_step": dt / timed * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, BASELINE config shape)",
        "config": {"workload": workload_name(spec, args.tile_b), "n": inst.n, "tile_b": args.tile_b,
                   "parallelism": f"{threads} CPU threads"},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                         **cpu_info(),
                         "sample": f"passes {warm + 1}..{warm + timed} of the config (after {warm} "
                                   f"warm-up passes; requested --steps {args.steps} --warmup "
                                   f"{args.warmup}, capped to bound the CPU run), oracle/ C port "
                                   "of _kernels.metric_units_pass + pair_pass"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def run_gpu(args):
    import torch
    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    from paper_1901_10084_b200 import instances, schedule
    from paper_1901_10084_b200.solver import DeviceSession, SolverConfig, solve

    if not args.config:  # defaults: config 3 on one GPU, config 4 sharded over N > 1
        args.config = 4 if ws > 1 else 3
        args.sharded = args.sharded or ws > 1
    spec = instances.CONFIGS[args.config]
    inst = instances.config_instance(args.config)
    n, b = inst.n, args.tile_b
    rows = rows_per_pass(n)
    copies = 1 if args.sharded else ws  # instances the job solves

    # ---- end to end through the public API (host buffers), run first: the
    # session's device buffers are allocated inside the timed region --------
    total = args.warmup + args.steps
    if ws > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    if args.sharded:
        from paper_1901_10084_b200.distributed import ShardedSession
        shs = ShardedSession(inst, b, device=local)
        stats = shs.run(total)
        xs, fs = shs.state()
        dk, dv = shs.duals()
        shs.close()

        class _Sol:  # the fields the JSON line reads
            pass
        sol = _Sol()
        sol.stats = [type("S", (), {"primal_objective": s_.primal_objective,
                                    "max_violation": s_.max_violation}) for s_ in stats]
        sol.duals = type("D", (), {"nnz": staticmethod(lambda: len(dk))})
    else:
        sol = solve(inst, SolverConfig(tile_size=b, fixed_passes=total, device=local))
    t_e2e = time.perf_counter() - t0
    if ws > 1:
        tt = torch.tensor([t_e2e], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_e2e = float(tt[0])
    m = inst.npairs
    h2d = 8 * 4 * m  # d, w, reg_x, reg_f
    d2h = total * 64 + 8 * 2 * m + 16 * m + 16 * sol.duals.nnz()
    # pass 1 is cheaper than the others (no stored duals yet, no exact steps
    # from duals): timed, but its rows are not counted
    e2e = {"value": copies * (total - 1) * rows / t_e2e, "unit": UNIT,
           "h2d_bytes_per_step": h2d / total, "d2h_bytes_per_step": d2h / total,
           "wall_s": t_e2e, "passes": total, "passes_counted": total - 1,
           "note": "first call in the process (cold device-buffer cache: every cudaMalloc inside); "
                   "rows of passes 2..W+K counted, all passes timed"}

    # ---- device-resident timing ------------------------------------------------
    if args.sharded:  # one instance over all ranks (strong scaling)
        from paper_1901_10084_b200.distributed import ShardedSession
        sess = ShardedSession(inst, b, device=local).session
    else:             # one instance per rank (replicas, weak scaling)
        sess = DeviceSession(inst, "tiled", b, device=local)
    nnz_hist = [0]
    for _ in range(args.warmup):
        nnz_hist.append(sess.run(1)[0].nnz_metric)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t_dev, metric_ms, pair_ms, launches, nnz_io = 0.0, 0.0, 0.0, 0, 0
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            sess.flush_l2()
            st = sess.run(1)[0]
            t_dev += st.wall_time
            m_ms, p_ms, nl = sess.timing()
            metric_ms += m_ms
            pair_ms += p_ms
            launches += nl
            nnz_io += nnz_hist[-1] + st.nnz_metric  # duals read + written
            nnz_hist.append(st.nnz_metric)
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
        tt = torch.tensor([t_dev, metric_ms], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_dev, metric_ms = float(tt[0]), float(tt[1])
    xchg = sess.exchange_volume() if args.sharded else (0, 0)
    sess.close()
    value = copies * args.steps * rows / t_dev

    # ---- roofline of the dominant kernel (tile_round_kernel) ------------------
    tx = schedule.touched_pairs(n, b)
    metric_bytes = args.steps * 16 * tx + 12 * nnz_io  # x read+write per touched pair, 12 B/dual
    achieved = metric_bytes / (metric_ms * 1e-3) / 1e9
    peak, peak_src = measured_peak()
    if args.sharded:  # metric_bytes covers the whole instance: compare with the whole box
        peak *= ws
        peak_src += f" x {ws} GPUs"
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": ncu_traffic(args.config, b),
                "traffic_unit": "DRAM bytes per pass (ncu, all tile_round_kernel launches of pass 4)",
                "kernel": "tile_round_kernel", "peak_source": peak_src,
                "frac_of_8TBs_nominal": achieved / 8000.0,
                "algorithmic_bytes_per_pass": 16 * tx + 12 * nnz_io / max(args.steps, 1),
                "T_x": tx, "metric_phase_share": metric_ms / (t_dev * 1e3),
                "launches_per_pass": launches / max(args.steps, 1),
                "barrier_levels_per_pass": schedule.critical_levels(n, b),
                "ns_per_barrier_level": metric_ms * 1e6 / args.steps / schedule.critical_levels(n, b)}
    roofline["ncu_counters"] = ncu_counters(args.config, b)
    if args.sharded:  # NVLink exchange of this rank (not part of B_pass)
        roofline["exchange"] = {"scheme": "footprint blocks to the next toucher's rank (grouped send/recv)",
                                "sent_bytes_per_pass_rank": 8 * xchg[0],
                                "received_bytes_per_pass_rank": 8 * xchg[1],
                                "all_gather_bytes_per_pass_rank": 8 * tx * (ws - 1) / ws}
    # whole pass (SURVEY 8(d) B_pass): + 72 B per pair for the pair phase
    pass_bytes = metric_bytes + args.steps * 72 * (n * (n - 1) // 2)
    roofline["whole_pass"] = {"bytes_per_pass": pass_bytes / args.steps,
                              "achieved": pass_bytes / t_dev / 1e9,
                              "frac": pass_bytes / t_dev / 1e9 / peak}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        threads = args.cpu_threads or os.cpu_count() or 1
        warm, timed = (2, 3) if n <= 1500 else (1, 1)
        rate, dt, p1 = cpu_sample(inst, b, warm, timed, threads, p1_rows=2.0e9 if n > 1500 else 2.0e8)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port", **cpu_info(),
               "sample": f"passes {warm + 1}..{warm + timed} of the same instance after {warm} "
                         f"warm-up passes ({dt:.1f} s), oracle/ C port of the reference kernels, "
                         f"{threads} threads",
               "p1": p1}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_dev / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong" if args.sharded else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator with the BASELINE config shape)",
            "config": {"workload": workload_name(spec, b), "n": n, "tile_b": b,
                       "passes_in_config": spec.passes,
                       "l2": "flushed (256 MiB write) before every timed pass",
                       "parallelism": (f"sharded x{ws} (one instance)" if args.sharded else
                                       "replicas" if ws > 1 else "1 GPU")},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clk.summary(),
            "final": {"primal": sol.stats[-1].primal_objective,
                      "max_violation": sol.stats[-1].max_violation, "nnz": sol.duals.nnz()},
        }
        print(json.dumps(line))
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=0,
                    help="BASELINE config (default 3: the largest one-GPU config; "
                         "4 sharded under torchrun)")
    ap.add_argument("--tile-b", type=int, default=40)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="one instance over all ranks (strong scaling) instead of replicas")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
