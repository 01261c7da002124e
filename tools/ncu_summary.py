#!/usr/bin/env python3
"""Summarise an ncu report (or a launch-list CSV) for profiles/.

  python tools/ncu_summary.py full  gpurun_out/prof.ncu-rep  > profiles/r01_k1_full.md
  python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/r01_launches.md
  python tools/ncu_summary.py traffic gpurun_out/prof.ncu-rep venice   # -> profiles/ncu_traffic.json
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import Counter, defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
    "smsp__cycles_active.avg", "sm__cycles_elapsed.avg", "lts__t_bytes.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active",
    "smsp__warps_eligible.avg.per_cycle_active",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def full(rep):
    kernels, units = raw(rep)
    print(f"# ncu --set full summary: `{os.path.basename(rep)}`\n")
    for k in kernels:
        name = k.get("Kernel Name", "?")
        print(f"## {name[:140]}\n")
        print("| metric | value | unit |\n|---|---|---|")
        for key in KEYS:
            if key in k:
                print(f"| {key} | {k[key]} | {units.get(key, '')} |")
        rd, wr = num(k.get("dram__bytes_read.sum")), num(k.get("dram__bytes_write.sum"))
        ru, wu = units.get("dram__bytes_read.sum", ""), units.get("dram__bytes_write.sum", "")
        print(f"\nDRAM traffic per launch: read {rd} {ru} + write {wr} {wu}\n")
        stalls = {kk: num(v) for kk, v in k.items() if kk.startswith("smsp__pcsamp_warps_issue_stalled")
                  and not kk.endswith("not_issued") and num(v)}
        if stalls:
            tot = sum(stalls.values())
            print("Top stall reasons (pc sampling):\n")
            for kk, v in sorted(stalls.items(), key=lambda x: -x[1])[:8]:
                print(f"- {kk.replace('smsp__pcsamp_warps_issue_stalled_', '')}: {100 * v / tot:.1f}%")
            print()


def traffic(rep, workload, pattern="k_stats"):
    kernels, units = raw(rep)
    k = next(x for x in kernels if pattern in x.get("Kernel Name", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = num(k["dram__bytes_read.sum"]) * scale.get(units["dram__bytes_read.sum"], 1)
    wr = num(k["dram__bytes_write.sum"]) * scale.get(units["dram__bytes_write.sum"], 1)
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        "ncu_traffic.json")
    data = {}
    if os.path.exists(path):
        data = json.load(open(path))
    data[workload] = int(rd + wr)  # K1 DRAM read + write bytes per launch
    json.dump(data, open(path, "w"), indent=1, sort_keys=True)
    print(json.dumps(data))


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    idx = {k: i for i, k in enumerate(hdr)}
    per = defaultdict(list)
    for r in rows[hdr_i + 1:]:
        if len(r) < len(hdr) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        per[r[idx["Kernel Name"]]].append((num(r[idx["Metric Value"]]), r[idx["Metric Unit"]]))
    total = sum(v for lst in per.values() for v, _ in lst)
    print(f"# ncu launch list `{os.path.basename(path)}` (gpu__time_duration.sum, --clock-control none)\n")
    print("Per-launch times are cold-cache and serialised: compare SHARES, not absolutes.\n")
    print("| kernel | launches | total | share | mean |\n|---|---|---|---|---|")
    for name, lst in sorted(per.items(), key=lambda x: -sum(v for v, _ in x[1])):
        s = sum(v for v, _ in lst)
        print(f"| {name[:90]} | {len(lst)} | {s:.1f} {lst[0][1]} | {100 * s / total:.1f}% | "
              f"{s / len(lst):.1f} {lst[0][1]} |")


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "full":
        full(sys.argv[2])
    elif mode == "traffic":
        traffic(sys.argv[2], sys.argv[3])
    else:
        launches(sys.argv[2])
