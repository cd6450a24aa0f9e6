"""Summarise a round's ncu outputs (gpurun_out/) into profiles/<tag>_*.

  python tools/summarize_profiles.py r02a 3     (tag, BASELINE config of the captures)
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def read_ncu_csv(path):
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[start:])))
    hdr = rows[0]
    return [dict(zip(hdr, r)) for r in rows[1:] if len(r) == len(hdr)]


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


def launches(tag):
    rows = read_ncu_csv(os.path.join(OUT, f"launches_{tag}.csv"))
    per = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"].split("(")[0]
        unit = r["Metric Unit"]
        v = num(r["Metric Value"]) * (1e-3 if unit == "ns" else (1.0 if unit == "us" else 1e3))
        per[k][0] += 1
        per[k][1] += v
    tot = sum(v[1] for v in per.values())
    lines = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, (c, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {c} | {t:.1f} | {t / tot * 100:.2f}% |")
    return "\n".join(lines), per, tot


def tile_dram(tag):
    rows = read_ncu_csv(os.path.join(OUT, f"tile_dram_{tag}.csv"))
    per = defaultdict(dict)
    for r in rows:
        per[r["ID"]][r["Metric Name"]] = (num(r["Metric Value"]), r["Metric Unit"])
    def b(v):
        val, unit = v
        return val * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    n = len(per)
    rd = sum(b(d["dram__bytes_read.sum"]) for d in per.values())
    wr = sum(b(d["dram__bytes_write.sum"]) for d in per.values())
    lts = sum(b(d["lts__t_bytes.sum"]) for d in per.values())
    dur = sum(d["gpu__time_duration.sum"][0] * (1e-3 if d["gpu__time_duration.sum"][1] == "ns" else 1)
              for d in per.values())
    inst = sum(d["smsp__inst_executed.sum"][0] for d in per.values())
    return {"launches": n, "dram_read_bytes": rd, "dram_write_bytes": wr,
            "dram_bytes_per_launch": (rd + wr) / max(n, 1), "l2_bytes_per_launch": lts / max(n, 1),
            "dram_bytes_per_pass": rd + wr, "l2_bytes_per_pass": lts,
            "duration_us_total": dur, "warp_instructions_total": inst}


def full_summary(tag, name="tile"):
    rep = os.path.join(OUT, f"prof_{name}_{tag}.ncu-rep")
    if not os.path.exists(rep):
        return {}
    txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[0]
    keep = ["Duration", "Elapsed Cycles", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate",
            "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
            "Dynamic Shared Memory Per Block", "Block Size", "Grid Size", "Achieved Active Warps Per SM",
            "Warp Cycles Per Issued Instruction", "Executed Instructions", "No Eligible",
            "Eligible Warps Per Scheduler", "Achieved Occupancy"]
    out = {}
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") in keep:
            out[d["Metric Name"]] = f'{d["Metric Value"]} {d["Metric Unit"]}'.strip()
    return out


def raw_metrics(tag, name="tile"):
    """FP64-pipe, shared-memory pipe and hit-rate counters of a full capture
    (`--page raw`): the figures SURVEY 8(d) asks to report beside DRAM GB/s."""
    rep = os.path.join(OUT, f"prof_{name}_{tag}.ncu-rep")
    if not os.path.exists(rep):
        return {}
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return {}
    hdr, units, vals = rows[0], rows[1], rows[2]
    want = {"sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct_of_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed": "fp64_pipe_pct_of_elapsed",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "shared_pipe_pct_of_elapsed",
            "lts__t_sector_hit_rate.pct": "l2_hit_pct",
            "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
            "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
            "smsp__warps_eligible.avg.per_cycle_active": "eligible_warps_per_scheduler",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct"}
    out = {}
    for h, u, v in zip(hdr, units, vals):
        if h in want:
            try:
                out[want[h]] = float(v.replace(",", ""))
            except ValueError:
                pass
    return out


def main(tag, config=3):
    os.makedirs(PROF, exist_ok=True)
    table, per, tot = launches(tag)
    dram = tile_dram(tag)
    full = full_summary(tag)
    full_df = full_summary(tag, "df")
    raw, raw_df = raw_metrics(tag), raw_metrics(tag, "df")

    def stalls(name):
        rep = os.path.join(OUT, f"prof_{name}_{tag}.ncu-rep")
        if not os.path.exists(rep):
            return ""
        return subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep, "25"],
                              capture_output=True, text=True).stdout
    stall, stall_df = stalls("tile"), stalls("df")
    with open(os.path.join(PROF, f"{tag}_ncu_summary.md"), "w") as fh:
        fh.write(f"# ncu summary, round {tag}\n\n")
        fh.write("## Launch list of `python bench.py --steps 3 --warmup 3 --no-cpu` "
                 "(`--metrics gpu__time_duration.sum --clock-control none`; cold-cache, serialised)\n\n")
        fh.write(table + "\n\n")
        fh.write(f"## tile_round_kernel, every launch of pass 4 (config {config}, b=40): DRAM bytes\n\n")
        fh.write("```\n" + json.dumps(dram, indent=2) + "\n```\n\n")
        for title, f, st, rw in (("a first-family round (round 10 of pass 3: hub rows in its longest tile)", full, stall, raw),
                                 ("the dataflow launch of pass 3 (the second family)", full_df, stall_df, raw_df)):
            if not f:
                continue
            fh.write(f"## Full capture (`--set full`): {title}\n\n```\n")
            for k, v in f.items():
                fh.write(f"{k:40s} {v}\n")
            fh.write("```\n\n")
            if rw:
                fh.write("Pipe and hit-rate counters (`--page raw`):\n\n```\n")
                for k, v in sorted(rw.items()):
                    fh.write(f"{k:40s} {v:.3f}\n")
                fh.write("```\n\n")
            fh.write("Per-source-line instruction share and stall samples:\n\n```\n" + st + "```\n\n")
    path = os.path.join(PROF, "ncu_tile_kernel.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    data[f"config{config}_b40"] = {"dram_bytes_per_pass": dram["dram_bytes_per_pass"],
                                   "l2_bytes_per_pass": dram["l2_bytes_per_pass"],
                                   "dram_bytes_per_launch": dram["dram_bytes_per_launch"],
                                   "l2_bytes_per_launch": dram["l2_bytes_per_launch"],
                                   "launches_measured": dram["launches"],
                                   "first_family_round": raw,
                                   "dataflow_launch": raw_df,
                                   "source": f"{tag}_ncu_summary.md"}
    with open(os.path.join(PROF, "ncu_tile_kernel.json"), "w") as fh:
        json.dump(data, fh, indent=2)
    print(open(os.path.join(PROF, f"{tag}_ncu_summary.md")).read()[:3000])


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 3)
