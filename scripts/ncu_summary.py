#!/usr/bin/env python3
"""Summarise ncu captures into profiles/: key per-launch metrics of the
dominant kernel (time, DRAM bytes, L2 traffic/hit rate, tensor activity,
SM active share) and the launch list's per-kernel time shares.

  python scripts/ncu_summary.py <tag> <workload-name>=<prof.ncu-rep> ... [--launches launches.csv]
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_srcunit_tex_op_read.sum",
    "sm__cycles_active.avg", "gpc__cycles_elapsed.max", "gpc__cycles_elapsed.max.per_second",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__cluster_dim_x",
]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    m = {}
    for h, u, v in zip(hdr, units, vals):
        if h in KEYS:
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                continue
            m[h] = x * UNIT_SCALE.get(u, 1) if u in UNIT_SCALE else x
            m[h + ".unit"] = "byte" if u in UNIT_SCALE else u
    m["kernel"] = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else ""
    return m


def launch_shares(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = {}
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name = r[ki].split("(")[0][:80]
        tot[name] = tot.get(name, 0.0) + v
    s = sum(tot.values())
    return {k: {"time_ns": v, "share": v / s} for k, v in sorted(tot.items(), key=lambda kv: -kv[1])}


def main():
    tag = sys.argv[1]
    args = sys.argv[2:]
    launches = None
    if "--launches" in args:
        i = args.index("--launches")
        launches = args[i + 1]
        args = args[:i] + args[i + 2:]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    summary_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summary = json.load(open(summary_path)) if os.path.exists(summary_path) else {}
    for a in args:
        wl, rep = a.split("=", 1)
        m = raw_metrics(rep)
        m["dram_bytes_per_launch"] = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        m["sm_active_share_of_elapsed"] = m.get("sm__cycles_active.avg", 0) / max(1, m.get("gpc__cycles_elapsed.max", 1))
        m["source"] = f"{tag}: ncu --set full --clock-control none ({os.path.basename(rep)})"
        summary[wl] = m
        print(wl, json.dumps(m, indent=1))
    if launches:
        summary.setdefault("_launch_lists", {})[tag] = launch_shares(launches)
    json.dump(summary, open(summary_path, "w"), indent=1)


if __name__ == "__main__":
    main()
