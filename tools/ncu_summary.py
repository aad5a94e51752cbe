"""Summarise an ncu report: key throughput metrics, stall reasons, SASS op mix."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
m = dict(zip(raw[0], raw[2]))
keys = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem"]
for k in keys:
    print(f"{k:65s} {m.get(k, '?')}")
print("-- stalls (per issue)")
for k in sorted(m):
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
        try:
            v = float(m[k])
        except ValueError:
            continue
        if v > 0.05:
            print(f"  {v:7.3f} {k[34:-23]}")
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
h = src[1]
iS, iE = h.index("Source"), h.index("Instructions Executed")
cnt = collections.Counter()
tot = 0
for r in src[2:]:
    if len(r) <= iE or not r[iE]:
        continue
    n = int(r[iE])
    toks = r[iS].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    cnt[op.split(".")[0]] += n
    tot += n
print("-- op mix (warp instructions)", tot)
for op, n in cnt.most_common(18):
    print(f"  {op:8s} {n:12d} {100 * n / tot:5.1f}%")
