"""Summarise ncu evidence for profiles/ (run here, on the CPU box).

  python scripts/ncu_summary.py rep <file.ncu-rep> [--workload NAME] [--dof N]
      -> key metrics of each profiled launch (DRAM bytes, duration, throughputs,
         occupancy, top stall reasons) as JSON
  python scripts/ncu_summary.py launches <launches.csv>
      -> per-kernel launch counts, mean duration and share of the listed time
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__bytes.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__block_size",
    "launch__grid_size", "launch__shared_mem_per_block_dynamic", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
]

UNIT = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "Tbyte/s": 1e12, "Gbyte/s": 1e9,
        "Mbyte/s": 1e6, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9}


def _num(v, unit):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    return x * UNIT.get(unit, 1.0) if unit in UNIT else x


def rep(path, workload=None, dof=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[head.index("Kernel Name")]}
        for k in KEYS:
            if k in head:
                i = head.index(k)
                d[k] = _num(r[i], units[i])
        stalls = {}
        for i, k in enumerate(head):
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
                try:
                    stalls[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(r[i])
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        d["stall_share_top"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda t: -t[1])[:6]}
        rd, wr = d.get("dram__bytes_read.sum"), d.get("dram__bytes_write.sum")
        if isinstance(rd, float) and isinstance(wr, float):
            d["dram_bytes_per_launch"] = rd + wr
            if dof:
                d["dram_bytes_per_dof"] = (rd + wr) / dof
                d["algorithmic_bytes_per_launch"] = 16.0 * dof
        res.append(d)
    return {"report": path, "workload": workload, "dof_per_launch": dof, "launches": res}


def launches(path):
    txt = open(path).read()
    i = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[i:])))
    head = rows[0]
    kn, mv = head.index("Kernel Name"), head.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[1:]:
        if len(r) > mv:
            agg[r[kn].split("(")[0]].append(float(r[mv].replace(",", "")))
    total = sum(sum(v) for v in agg.values())
    return {k: {"launches": len(v), "mean_ns": sum(v) / len(v), "share_of_listed": sum(v) / total}
            for k, v in sorted(agg.items(), key=lambda t: -sum(t[1]))}


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    args = dict(zip(sys.argv[3::2], sys.argv[4::2]))
    if mode == "rep":
        print(json.dumps(rep(path, args.get("--workload"), float(args["--dof"]) if "--dof" in args else None),
                         indent=1))
    else:
        print(json.dumps(launches(path), indent=1))
