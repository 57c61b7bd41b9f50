"""Dev tool: per-CUDA-source-line instruction and stall totals of an ncu report.

  python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, lines = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("", "Function Name"):
        try:
            ie = int(r[7] or 0)
            st = int(r[4]) if r[4] not in ("-", "") else 0
        except ValueError:
            continue
        lines.append((ie, st, f"{fname}:{r[0]}", r[1].strip()))
tot_i = sum(x[0] for x in lines) or 1
tot_s = sum(x[1] for x in lines) or 1
print(f"total warp instructions {tot_i}, stall samples {tot_s}")
for ie, st, loc, src in sorted(lines, key=lambda x: -x[1])[:top]:
    print(f"instr {ie / tot_i * 100:5.1f}%  stall {st / tot_s * 100:5.1f}%  {loc:22s} {src[:90]}")
