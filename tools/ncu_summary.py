"""Summarise an ncu report: headline metrics + stall reasons, overall and per
hot SASS block (grouped by execution count). Usage: ncu_summary.py rep.ncu-rep"""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
want = ["Duration", "Elapsed Cycles", "SM Frequency", "Issue Slots Busy", "Issued Ipc Active",
        "Eligible Warps Per Scheduler", "No Eligible", "Registers Per Thread", "DRAM Throughput",
        "L2 Cache Throughput", "L1/TEX Cache Throughput", "Achieved Active Warps Per SM",
        "Avg. Active Threads Per Warp", "Executed Instructions", "Memory Throughput"]
for row in csv.reader(io.StringIO(raw)):
    if len(row) > 14 and row[-3] in want:
        print(f"{row[4][:40]:40s} {row[-3]:32s} {row[-1]:>14s} {row[-2]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr, data = rows[hdr_i], [r for r in rows[hdr_i + 1:] if len(r) == len(rows[hdr_i])]
iE = hdr.index("Instructions Executed"); iS = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
for r in data:
    for i in stall_cols:
        tot[hdr[i]] += int(r[i] or 0)
S = sum(tot.values()) or 1
print("stalls overall:", ", ".join(f"{k[6:]} {100*v/S:.1f}%" for k, v in tot.most_common(8)))
groups = collections.defaultdict(lambda: [0, 0, collections.Counter(), collections.Counter()])
for r in data:
    e = int(r[iE] or 0)
    g = groups[e]
    g[0] += 1; g[1] += int(r[iS] or 0)
    op = r[1].split()
    op = op[1] if op and op[0].startswith("@") else (op[0] if op else "?")
    g[3][op.split(".")[0]] += 1
    for i in stall_cols:
        g[2][hdr[i]] += int(r[i] or 0)
print("hot blocks (exec count, #instr, samples%, top stalls, top ops):")
for e, (n, smp, st, ops) in sorted(groups.items(), key=lambda x: -x[1][1])[:10]:
    print(f"  exec {e:>9d} n={n:4d} samples {100*smp/S:5.1f}%  " +
          ", ".join(f"{k[6:]} {v}" for k, v in st.most_common(4)) + "  | " +
          " ".join(f"{k}:{v}" for k, v in ops.most_common(8)))
