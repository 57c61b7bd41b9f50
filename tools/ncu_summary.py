"""Summarise an ncu report: key metrics + hottest SASS basic blocks (dev tool)."""
import csv, subprocess, sys, io

rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
want = ("Duration", "Executed Instructions", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "DRAM Throughput", "Memory Throughput", "Executed Ipc Active", "Issue Slots Busy", "L1/TEX Hit Rate",
        "Block Limit Registers", "Block Limit Shared Mem", "Dynamic Shared Memory Per Block", "Grid Size",
        "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler", "Avg. Active Threads Per Warp")
for row in csv.DictReader(io.StringIO(det)):
    if row.get("Metric Name") in want:
        print(f"{row['Metric Name']:40s} {row['Metric Value']} {row['Metric Unit']}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
if len(r) > 2:
    hdr, vals = r[0], r[2]
    for k, v in zip(hdr, vals):
        if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
            print(f"{k:40s} {v} {r[1][hdr.index(k)]}")
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                      text=True).stdout
rows = list(csv.reader(io.StringIO(sass)))
h = rows[1]; data = rows[2:]
iS = h.index("Source"); iE = h.index("Instructions Executed"); iW = h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(x[iE] or 0) for x in data); totw = sum(int(x[iW] or 0) for x in data)
print("total warp instr", tot, "stall samples", totw)
blocks = []; cur = None
for k, x in enumerate(data):
    e = int(x[iE] or 0); w = int(x[iW] or 0)
    if cur and cur[2] == e:
        cur[1] = k; cur[3] += e; cur[4] += w
    else:
        cur = [k, k, e, e, w, x[iS].strip()[:60]]; blocks.append(cur)
blocks.sort(key=lambda b: -b[3])
for b in blocks[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{b[0]:5d}-{b[1]:5d} n={b[1]-b[0]+1:4d} exec={b[2]:9d} {b[3]/tot*100:5.1f}% stall={b[4]/max(totw,1)*100:5.1f}% {b[5]}")
