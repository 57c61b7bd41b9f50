#!/bin/bash
# A/B of library variants on the headline bench (joint path): parity tests + step / sweep time.
#   tools/ab_joint.sh default paper_1511_06416_b200/lib_variant_X.so ...
for L in "$@"; do
  if [ "$L" = default ]; then unset SAMEGIBBS_LIB; else export SAMEGIBBS_LIB=$PWD/$L; fi
  timeout 600 python -m pytest tests/test_gpu_joint.py -x -q > gpurun_out/ab_pt.log 2>&1 || { echo "$L: joint tests FAILED"; tail -5 gpurun_out/ab_pt.log; }
  timeout 300 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/ab.json 2>gpurun_out/ab.err || { echo "$L bench FAILED"; tail -3 gpurun_out/ab.err; continue; }
  python - "$L" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
print(f"{sys.argv[1]:44s} step {d['ms_per_step']*1e3:6.1f} us  sweep {d['roofline']['kernel_ms']*1e3:6.1f} us  "
      f"frac {d['roofline']['frac']:.3f}  e2e {d['e2e']['ms_per_step']*1e3:6.1f} us")
PY
done
