#!/usr/bin/env python
"""Summarise ncu artefacts into profiles/ (committed evidence).

  python scripts/ncu_summary.py rep <file.ncu-rep> <label> <out.txt>   key metrics of one capture
  python scripts/ncu_summary.py list <launches.csv> <out.csv>          our launches + shares
Also merges dram bytes per launch into profiles/ncu_traffic.json (read by bench.py).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__cycles_elapsed.avg", "smsp__cycles_active.avg", "sm__cycles_active.avg",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_static", "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "launch__waves_per_multiprocessor", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_drain_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [{h: (v, u) for h, u, v in zip(hdr, units, r)} for r in rows[2:]]


def to_bytes(v, u):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    return float(v.replace(",", "")) * scale


def cmd_rep(rep, label, out):
    recs = raw(rep)
    lines = [f"# ncu --set full summary: {label}  (source: {os.path.basename(rep)})"]
    traffic_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        traffic = json.load(open(traffic_path))
    except Exception:
        traffic = {}
    for r in recs:
        name = r.get("Kernel Name", ("?", ""))[0]
        lines.append(f"kernel: {name}")
        for k in KEYS:
            if k in r:
                v, u = r[k]
                lines.append(f"  {k} = {v} {u}")
        if "dram__bytes_read.sum" in r:
            b = to_bytes(*r["dram__bytes_read.sum"]) + to_bytes(*r["dram__bytes_write.sum"])
            lines.append(f"  traffic_bytes (read+write) = {b:.0f}")
            traffic[label] = b
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(traffic_path, "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)
    print("\n".join(lines))


def cmd_list(path, out):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    recs = [(r[ik], float(r[iv].replace(",", "")), r[im]) for r in rows[1:] if len(r) > iv]
    tot = sum(v for _, v, _ in recs)
    with open(out, "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised)\n")
        f.write("kernel,duration,unit,share_of_listed\n")
        for k, v, u in recs:
            f.write(f"\"{k}\",{v},{u},{v / tot:.4f}\n")
    agg = {}
    for k, v, _ in recs:
        agg[k] = agg.get(k, 0) + v
    for k, v in agg.items():
        print(f"{v / tot:7.3%}  {k}")


if __name__ == "__main__":
    if sys.argv[1] == "rep":
        cmd_rep(sys.argv[2], sys.argv[3], sys.argv[4])
    else:
        cmd_list(sys.argv[2], sys.argv[3])
