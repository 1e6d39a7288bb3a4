"""Summarise an ncu report: key metrics + SASS opcode mix + top stall lines."""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
keys = ["Duration", "Elapsed Cycles", "DRAM Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Active Warps Per SM", "No Eligible", "Warp Cycles Per Issued Instruction",
        "L2 Hit Rate", "Memory Throughput", "Executed Instructions"]
for row in csv.reader(io.StringIO(det)):
    if len(row) > 3 and row[-3] in keys:
        print(f"  {row[-3]:40s} {row[-1]:>14s} {row[-2]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if len(rr) >= 3:
    hdr, units, vals = rr[0], rr[1], rr[2]
    for k in ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
              "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]:
        for i, h in enumerate(hdr):
            if h == k:
                print(f"  {k:60s} {vals[i]:>16s} {units[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
if len(rows) > 2:
    hdr = rows[1]
    iS, iE, iW = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    ops, st = collections.Counter(), collections.Counter()
    tot = 0
    for r in rows[2:]:
        if len(r) <= iE:
            continue
        m = re.match(r'(@!?U?P\w+\s+)?([A-Z0-9_]+)', r[iS].strip())
        if not m:
            continue
        n = int(r[iE] or 0)
        tot += n
        ops[m.group(2)] += n
        st[m.group(2)] += int(r[iW] or 0)
    print("  warp-instructions executed:", tot)
    for op, n in ops.most_common(16):
        print(f"    {op:10s} {n:12d} {100*n/tot:5.1f}%  stall-samples {st[op]}")
