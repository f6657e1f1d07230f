"""Summarise ncu reports (gpurun_out/*.ncu-rep, launches.csv) into profiles/.

usage: python tools/ncu_summary.py <key>=<report.ncu-rep>[#launch] ... [--launches launches.csv]
                                   [--algo <key>=<bytes>] [--out profiles/ncu_summary.json]
Writes/merges JSON keyed by <key> with the metrics the roofline needs
(duration, dram bytes read/write, throughput %, registers, occupancy).
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "dram__bytes.sum.per_second": "dram_bw",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__shared_mem_per_block_dynamic": "dyn_smem",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pct",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_active_pct",
    "sm__inst_executed_pipe_tma.sum": "tma_inst",
    "launch__func_name": "kernel",
    "Kernel Name": "kernel_name",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9, "second": 1,
        "byte/second": 1, "Gbyte/second": 1e9, "Tbyte/second": 1e12, "Mbyte/second": 1e6,
        "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "ms": 1e-3, "us": 1e-6, "ns": 1e-9,
        "s": 1, "Tbyte/s": 1e12, "Gbyte/s": 1e9, "Mbyte/s": 1e6, "Kbyte/block": 1e3}


def raw(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {}
        for i, h in enumerate(hdr):
            if h.endswith("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"):
                h = "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"
            if h in METRICS:
                v = vals[i]
                u = units[i] if i < len(units) else ""
                try:
                    f = float(v.replace(",", ""))
                    d[METRICS[h]] = f * UNIT.get(u, 1)
                except ValueError:
                    d[METRICS[h]] = v
        res.append(d)
    return res


def main():
    args = sys.argv[1:]
    out = Path("profiles/ncu_summary.json")
    algo = {}
    flops = {}
    launches = None
    reps = []
    i = 0
    while i < len(args):
        a = args[i]
        if a == "--out":
            out = Path(args[i + 1])
            i += 2
            continue
        if a == "--launches":
            launches = args[i + 1]
            i += 2
            continue
        if a == "--algo":
            k, v = args[i + 1].split("=")
            algo[k] = float(v)
            i += 2
            continue
        if a == "--flops":
            k, v = args[i + 1].split("=")
            flops[k] = float(v)
            i += 2
            continue
        reps.append(a.split("=", 1))
        i += 1
    data = json.loads(out.read_text()) if out.exists() else {}
    for key, rep in reps:
        idx = 0
        if "#" in rep:  # report#launch-index
            rep, idx = rep.split("#")
            idx = int(idx)
        rs = raw(rep)
        d = rs[idx]
        d["dram_bytes_per_launch"] = d.get("dram_read", 0) + d.get("dram_write", 0)
        if key in algo:
            d["algorithmic_bytes"] = algo[key]
            d["traffic_over_algorithmic"] = d["dram_bytes_per_launch"] / algo[key]
            d["achieved_algorithmic_gbs_under_ncu"] = algo[key] / d["duration"] / 1e9
        if key in flops:
            d["algorithmic_flops"] = flops[key]
            d["achieved_tflops_under_ncu"] = flops[key] / d["duration"] / 1e12
        d["report"] = Path(rep).name
        data[key] = d
    if launches:
        rows = list(csv.reader(open(launches)))
        # skip ncu preamble lines
        start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
        hdr = rows[start]
        ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
        agg = {}
        for r in rows[start + 1:]:
            if len(r) <= vi:
                continue
            name = r[ki]
            short = name.split("(")[0][:90]
            t = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1)
            a = agg.setdefault(short, [0, 0.0])
            a[0] += 1
            a[1] += t
        tot = sum(v[1] for v in agg.values())
        data["launch_list"] = {k: {"launches": v[0], "total_s": v[1], "share": v[1] / tot}
                               for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}
    out.parent.mkdir(exist_ok=True)
    out.write_text(json.dumps(data, indent=1))
    print(json.dumps(data, indent=1)[:3000])


if __name__ == "__main__":
    main()
