#!/bin/bash
# A/B of library variants on the streamed C2 workload (c2s): us per step.
for L in "$@"; do
  if [ "$L" = default ]; then unset SAMEGIBBS_LIB; else export SAMEGIBBS_LIB=$PWD/$L; fi
  timeout 600 python bench.py --workload c2s --no-cpu-baseline --steps 100 --c2s-cases 20000000 > gpurun_out/abs.json 2>gpurun_out/abs.err || { echo "$L c2s FAILED"; tail -3 gpurun_out/abs.err; continue; }
  python - "$L" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/abs.json").read().strip().splitlines()[-1])
print(f"{sys.argv[1]:48s} step {d['ms_per_step']*1e3:7.1f} us  value {d['value']:.3e}")
PY
done
