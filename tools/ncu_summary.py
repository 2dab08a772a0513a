"""Summarize ncu captures from gpurun_out/ into profiles/<round>/ (committed).

  python tools/ncu_summary.py r01

Writes one text summary per `prof_<kernel>.ncu-rep`, a launch-share table
from `launches.csv`, and profiles/ncu_summary.json (DRAM bytes per launch,
read by bench.py for roofline.traffic).
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

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
]

UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9,
              "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
              "s": 1}


def raw(rep):
    r = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(r.stdout)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def to_si(v, u):
    try:
        return float(v.replace(",", "")) * UNIT_SCALE.get(u, 1)
    except ValueError:
        return None


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    # optional second argument: write the summaries there (e.g. inside
    # gpurun_out/ on the GPU box, so the large .ncu-rep files can be dropped)
    dst = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles", tag)
    os.makedirs(dst, exist_ok=True)
    summary = {}
    for f in sorted(os.listdir(OUT)):
        if not (f.startswith("prof_") and f.endswith(".ncu-rep")):
            continue
        kern = f[len("prof_"):-len(".ncu-rep")]
        # prof_<config>__<kernel>.ncu-rep -> key "<config>:<kernel>" (per-config traffic for bench.py)
        key = kern.replace("__", ":", 1) if "__" in kern else kern
        cfg = key.split(":")[0] if ":" in key else "c3"
        bpl = 4 if cfg in ("c1", "c2") else 8
        d = raw(os.path.join(OUT, f))
        lines = [f"# ncu --set full, kernel {kern} (one launch of the bench workload, --batch {bpl})"]
        for k in KEYS:
            if k in d:
                lines.append(f"{k:90s} {d[k][0]:>16s} {d[k][1]}")
        with open(os.path.join(dst, f"ncu_{kern}.txt"), "w") as fh:
            fh.write("\n".join(lines) + "\n")
        rd = to_si(*d["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in d else None
        wr = to_si(*d["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in d else None
        dur = to_si(*d["gpu__time_duration.sum"]) if "gpu__time_duration.sum" in d else None
        grid = to_si(*d["launch__grid_size"]) if "launch__grid_size" in d else None
        summary[key] = {"dram_bytes_per_launch": (rd or 0) + (wr or 0), "duration_s": dur, "grid": grid,
                        "blocks_per_launch": bpl, "source": f"profiles/{tag}/ncu_{kern}.txt"}
    lc = os.path.join(OUT, "launches.csv")
    if os.path.exists(lc):
        tot = defaultdict(float)
        cnt = defaultdict(int)
        with open(lc) as fh:
            txt = fh.read()
        start = txt.find('"ID"')
        for r in csv.DictReader(io.StringIO(txt[start:])):
            if r.get("Metric Name") != "gpu__time_duration.sum":
                continue
            name = r["Kernel Name"].split("(")[0]
            tot[name] += to_si(r["Metric Value"], r["Metric Unit"]) or 0
            cnt[name] += 1
        s = sum(tot.values())
        with open(os.path.join(dst, "launch_shares.txt"), "w") as fh:
            fh.write("# ncu --metrics gpu__time_duration.sum --clock-control none over bench.py --steps 2 --warmup 1 "
                     "--batch 8 (cold-cache, serialized: compare shares)\n")
            for k in sorted(tot, key=lambda x: -tot[x]):
                fh.write(f"{k:60s} launches {cnt[k]:5d}  total {tot[k]*1e3:10.3f} ms  share {100*tot[k]/s:6.2f}%\n")
    with open(os.path.join(dst if len(sys.argv) > 2 else os.path.join(ROOT, "profiles"), "ncu_summary.json"),
              "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
