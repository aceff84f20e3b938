"""Summarise ncu outputs into profiles/ (run here, no GPU needed).

  python tools/ncu_summary.py launches <launches.csv> <out.md>
  python tools/ncu_summary.py full <report.ncu-rep> <out.txt> [traffic.json]
"""
import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr = None
    recs = []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            unit = d.get("Metric Unit", "ns")
            v = float(d["Metric Value"].replace(",", ""))
            ns = v * {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(unit, 1)
            recs.append((d["Kernel Name"], ns, d.get("Grid Size", ""), d.get("Block Size", "")))
    agg = OrderedDict()
    for name, ns, g, b in recs:
        short = name.split("(")[0]
        a = agg.setdefault(short, [0, 0.0])
        a[0] += 1
        a[1] += ns
    total = sum(v[1] for v in agg.values())
    lines = [f"# Launch list summary ({path})", "",
             "Cold-cache, serialised per-launch device times (ncu gpu__time_duration.sum,",
             "--clock-control none). Compare SHARES, not absolutes.", "",
             "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {n} | {ns / 1e3:.1f} | {100 * ns / total:.1f}% |")
    lines += ["", f"total {total / 1e3:.1f} us over {len(recs)} launches", "",
              "## Every launch", "", "| # | kernel | us | grid | block |", "|---|---|---|---|---|"]
    for i, (name, ns, g, b) in enumerate(recs):
        lines.append(f"| {i} | `{name[:70]}` | {ns / 1e3:.1f} | {g} | {b} |")
    open(out, "w").write("\n".join(lines) + "\n")


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "launch__occupancy_limit_shared_mem", "sm__cycles_elapsed.avg.per_second",
        "smsp__average_warp_latency_issue_stalled_barrier",
        "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_wait",
        "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
        "smsp__pcsamp_warps_issue_stalled_mio_throttle", "smsp__pcsamp_warps_issue_stalled_selected",
        "smsp__pcsamp_warps_issue_stalled_not_selected", "smsp__pcsamp_warps_issue_stalled_dispatch_stall",
        "smsp__pcsamp_warps_issue_stalled_lg_throttle", "smsp__pcsamp_warps_issue_stalled_membar",
        "smsp__pcsamp_warps_issue_stalled_sleeping", "smsp__pcsamp_warps_issue_stalled_no_instructions",
        "smsp__pcsamp_warps_issue_stalled_drain", "smsp__pcsamp_warps_issue_stalled_imc_miss",
        "smsp__pcsamp_warps_issue_stalled_branch_resolving", "smsp__pcsamp_sample_count"]


def full(path, out, traffic_out=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full summary ({path})", ""]
    launches_ = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        launches_.append(d)
        lines.append(f"## launch {d.get('ID')} `{d.get('Kernel Name', '')[:90]}` grid {d.get('Grid Size')} "
                     f"block {d.get('Block Size')}")
        for k in KEYS:
            if k in d:
                lines.append(f"- {k} = {d[k]} {u.get(k, '')}")
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")
    if traffic_out and launches_:
        def num(x):
            return float(str(x).replace(",", ""))
        u = dict(zip(hdr, units))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
        tb = []
        for d in launches_:
            rd = num(d["dram__bytes_read.sum"]) * scale.get(u["dram__bytes_read.sum"], 1)
            wr = num(d["dram__bytes_write.sum"]) * scale.get(u["dram__bytes_write.sum"], 1)
            tb.append(rd + wr)
        alu = [num(d.get("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 0))
               for d in launches_]
        dram = [num(d.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 0))
                for d in launches_]
        dur = [num(d["gpu__time_duration.sum"]) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1,
                                                     "msecond": 1e3, "ms": 1e3}.get(u["gpu__time_duration.sum"], 1)
               for d in launches_]
        json.dump({"source": path, "kernel": launches_[0].get("Kernel Name", "")[:80],
                   "kernels": [d.get("Kernel Name", "")[:60] for d in launches_],
                   "duration_us_per_launch": [round(x, 3) for x in dur],
                   "dram_bytes_per_launch": int(sum(tb) / len(tb)),
                   "per_launch": [int(x) for x in tb],
                   "alu_pipe_pct_per_launch": alu, "dram_pct_per_launch": dram},
                  open(traffic_out, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
