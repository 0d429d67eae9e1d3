"""Summarise an ncu report: key SOL/scheduler metrics, stall reasons and the instruction mix."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]


def run(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


KEEP = ['Duration', 'SM Frequency', 'DRAM Throughput', 'Memory Throughput', 'Compute (SM) Throughput',
        'Executed Ipc Active', 'Issue Slots Busy', 'Executed Instructions', 'L1/TEX Cache Throughput',
        'L2 Hit Rate', 'Eligible Warps Per Scheduler', 'No Eligible', 'Warp Cycles Per Issued Instruction',
        'Registers Per Thread', 'Achieved Active Warps Per SM', 'Block Size', 'Grid Size',
        'Dynamic Shared Memory Per Block']
rows = list(csv.reader(io.StringIO(run("--page", "details", "--csv"))))
hdr = rows[0]
kern = None
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get("Kernel Name") != kern:
        kern = d.get("Kernel Name")
        print("==", kern[:120])
    if d.get("Metric Name") in KEEP:
        print(f"  {d['Metric Name']:40s} {d['Metric Unit']:14s} {d['Metric Value']}")
raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
h, u = raw[0], raw[1]
for vals in raw[2:]:
    stalls = []
    for name, val in zip(h, vals):
        if name.startswith("smsp__pcsamp_warps_issue_stalled") and not name.endswith("not_issued"):
            try:
                stalls.append((float(val.replace(",", "")), name.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
        if name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
                    "gpu__time_duration.sum", "lts__t_bytes.sum", "lts__t_sectors_srcunit_tex.sum",
                    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.sum",
                    "smsp__inst_executed.avg.per_cycle_active", "sm__cycles_elapsed.avg.per_second",
                    "l1tex__t_bytes.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
                    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"):
            print(f"  {name:40s} {vals[h.index(name)]} {u[h.index(name)]}")
    tot = sum(x for x, _ in stalls) or 1
    print("  stalls:", ", ".join(f"{n} {x / tot * 100:.0f}%" for x, n in sorted(stalls, reverse=True)[:8]))
sass = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "sass"))))
if len(sass) > 2:
    hh = sass[1]
    ix = {k: i for i, k in enumerate(hh)}
    ops = collections.Counter()
    tot = 0
    for r in sass[2:]:
        try:
            c = int(r[ix["Instructions Executed"]] or 0)
        except (ValueError, IndexError):
            continue
        toks = r[ix["Source"]].split()
        if not toks or c == 0:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        ops[op.split(".")[0]] += c
        tot += c
    print("  instruction mix:", ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in ops.most_common(14)))
