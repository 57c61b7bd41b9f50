#!/bin/bash
# A/B of library variants on the bit-exact numpy-stream C2 bench: parity tests + step / sweep time.
#   tools/ab_numpy.sh default paper_1511_06416_b200/lib_variant_X.so ...
for L in "$@"; do
  if [ "$L" = default ]; then unset SAMEGIBBS_LIB; else export SAMEGIBBS_LIB=$PWD/$L; fi
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/abn_pt.log 2>&1 || { echo "$L: parity tests FAILED"; tail -5 gpurun_out/abn_pt.log; }
  timeout 300 python bench.py --rng numpy --no-cpu-baseline --steps 20 > gpurun_out/abn.json 2>gpurun_out/abn.err || { echo "$L bench FAILED"; tail -3 gpurun_out/abn.err; continue; }
  python - "$L" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/abn.json").read().strip().splitlines()[-1])
print(f"{sys.argv[1]:44s} step {d['ms_per_step']*1e3:7.1f} us  sweep {d['roofline']['kernel_ms']*1e3:7.1f} us  frac {d['roofline']['frac']:.4f}")
PY
done
