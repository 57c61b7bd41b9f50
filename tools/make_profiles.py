"""Summarise a round's GPU evidence (gpurun_out/) into profiles/ (tracked).

  python tools/make_profiles.py r01

Reads gpurun_out/{launches_R.csv, sweep_R.ncu-rep, finish_R.ncu-rep,
bench_R.json, bench_ref_R.json} written by tools/gpu_round.sh and writes:
  profiles/R_launches.csv            ncu launch list (gpu__time_duration.sum per launch)
  profiles/R_launch_summary.txt      per-kernel mean duration, count and share
  profiles/R_sweep_ncu_summary.txt   key metrics + hottest SASS blocks (sweep)
  profiles/R_finish_ncu_summary.txt  same for the step tail
  profiles/ncu_sweep_R.json          DRAM bytes per sweep launch (bench.py roofline.traffic)
  profiles/R_bench.json, R_bench_reference.json  the bench lines of that run
"""
import collections
import csv
import io
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
R = sys.argv[1] if len(sys.argv) > 1 else "r01"
G, P = ROOT / "gpurun_out", ROOT / "profiles"
P.mkdir(exist_ok=True)


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def num(x):
    return float(str(x).replace(",", ""))


# launch list
src = G / f"launches_{R}.csv"
if src.exists():
    shutil.copy(src, P / f"{R}_launches.csv")
    rows = [r for r in csv.reader(open(src)) if len(r) > 10]
    h = rows[0]
    iN, iV = h.index("Kernel Name"), h.index("Metric Value")
    per = collections.defaultdict(list)
    for r in rows[1:]:
        per[r[iN].split("(")[0]].append(num(r[iV]) / 1e3)
    total = sum(sum(v) for v in per.values())
    with open(P / f"{R}_launch_summary.txt", "w") as f:
        f.write(f"# ncu launch list of `python bench.py --steps 20 --warmup 3 --no-cpu-baseline` "
                f"(--clock-control none, cold caches, serialised)\n")
        f.write(f"{'count':>5} {'mean us':>9} {'total us':>10} {'share':>6}  kernel\n")
        for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            f.write(f"{len(v):5d} {sum(v) / len(v):9.2f} {sum(v):10.1f} {sum(v) / total:6.1%}  {k}\n")
        sw = next((v for k, v in per.items() if "k_joint_sweep" in k), None) or \
            per.get("void sg::k_small_sweep<5, 3>", [])
        fin = per.get("sg::k_step_tail_joint", []) or per.get("sg::k_step_finish", [])
        if sw and fin:
            a, b = sum(sw) / len(sw), sum(fin) / len(fin)
            f.write(f"\nper step (graph replay = 1 sweep + 1 step tail): sweep {a:.1f} us + tail {b:.1f} us; "
                    f"sweep share {a / (a + b):.1%}\n")

for name in ("sweep", "finish"):
    rep = G / f"{name}_{R}.ncu-rep"
    if rep.exists():
        txt = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"), str(rep), "20"],
                             capture_output=True, text=True).stdout
        (P / f"{R}_{name}_ncu_summary.txt").write_text(
            f"# ncu --set full --clock-control none --import-source on, one launch ({rep.name})\n" + txt)

rep = G / f"sweep_{R}.ncu-rep"
if rep.exists():
    m = raw_metrics(rep)
    rd, wr = num(m["dram__bytes_read.sum"][0]), num(m["dram__bytes_write.sum"][0])
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd *= scale.get(m["dram__bytes_read.sum"][1], 1)
    wr *= scale.get(m["dram__bytes_write.sum"][1], 1)
    dur = num(m["gpu__time_duration.sum"][0]) * (1e-3 if m["gpu__time_duration.sum"][1] == "nsecond" else 1)
    kname = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv", "--metrics", "gpu__time_duration.sum"],
                           capture_output=True, text=True).stdout
    kernel = ("k_joint_sweep<3, 2> (sg_joint_sweep)" if "k_joint_sweep" in kname else
              "k_small_sweep<5, 3> (sg_small_sweep)")
    (P / f"ncu_sweep_{R}.json").write_text(json.dumps({
        "kernel": kernel, "cases": 1_000_000, "m": 10,
        "command": "python bench.py --steps 5 --warmup 3 --no-cpu-baseline (step graph replay, 2-bit observation block)",
        "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
        "duration_us_under_ncu": dur, "algorithmic_bytes_per_launch": 75_000_000,
        "note": "traffic = dram__bytes_read.sum + dram__bytes_write.sum of one launch; the lane words, pattern "
                "bytes, case ids and the observation block (range check) are read once, the lane words "
                "written back (writes land in L2 and are not evicted within the launch).",
    }, indent=1) + "\n")

for name in ("big",):
    rep = G / f"{name}_{R}.ncu-rep"
    if rep.exists():
        txt = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"), str(rep), "20"],
                             capture_output=True, text=True).stdout
        (P / f"{R}_sweep_big_ncu_summary.txt").write_text(
            f"# ncu --set full --clock-control none --import-source on, one k_sweep_big launch on C4 ({rep.name})\n"
            + txt)
if (G / f"pytest_gpu_{R}.log").exists():
    shutil.copy(G / f"pytest_gpu_{R}.log", P / f"{R}_pytest_gpu.log")
for src, dst in ((f"bench_{R}.json", f"{R}_bench.json"), (f"bench_ref_{R}.json", f"{R}_bench_reference.json"),
                 (f"bench_numpy_{R}.json", f"{R}_bench_numpy.json"), (f"bench_c3_{R}.json", f"{R}_bench_c3.json"),
                 (f"bench_c4_{R}.json", f"{R}_bench_c4.json"), (f"bench_c5_{R}.json", f"{R}_bench_c5.json"),
                 (f"bench_c2s_{R}.json", f"{R}_bench_c2s.json")):
    if (G / src).exists():
        lines = [l for l in (G / src).read_text().splitlines() if l.startswith("{")]
        if lines:
            (P / dst).write_text(lines[-1] + "\n")
print(sorted(p.name for p in P.iterdir()))
