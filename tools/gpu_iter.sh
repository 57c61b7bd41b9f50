#!/bin/bash
# Dev loop on one B200: parity tests of the joint path, the bench line, the
# launch list and (optional) one ncu --set full capture of a kernel.
#   tools/gpu_iter.sh TAG [kernel-regex]
set -u
O=gpurun_out; T=${1:-it}; K=${2:-}
timeout 600 python -m pytest tests/test_gpu_joint.py -x -q > $O/pt_$T.log 2>&1; echo "joint tests rc=$?"; tail -2 $O/pt_$T.log
timeout 300 python bench.py --no-cpu-baseline > $O/bench_$T.json 2> $O/bench_$T.err; echo "bench rc=$?"
python - "$O/bench_$T.json" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r = d["roofline"]
print(f"step {d['ms_per_step']*1e3:.1f} us  sweep {r['kernel_ms']*1e3:.1f} us  frac {r['frac']:.3f}  "
      f"value {d['value']:.3e}  e2e {d['e2e']['value']:.3e} ({d['e2e']['ms_per_step']*1e3:.1f} us)")
PY
L="python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches_$T.csv $L > $O/ncu_l_$T.log 2>&1
python tools/launch_table.py $O/launches_$T.csv > $O/lt_$T.txt 2>/dev/null; head -7 $O/lt_$T.txt
if [ -n "$K" ]; then
  F="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --eager"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K --launch-skip 4 --launch-count 1 \
    -o $O/full_$T -f $F > $O/ncu_full_$T.log 2>&1; echo "ncu full rc=$?"
fi
