#!/bin/bash
# A/B of library variants: bench line digest + warm sweep time per variant.
# usage: tools/ab.sh lib1.so lib2.so ...   (in-tree default lib = "default")
for L in "$@"; do
  if [ "$L" = default ]; then unset SAMEGIBBS_LIB; else export SAMEGIBBS_LIB=$PWD/$L; fi
  python bench.py --no-cpu-baseline --steps 100 > gpurun_out/ab.json 2>gpurun_out/ab.err || { echo "$L FAILED"; tail -3 gpurun_out/ab.err; continue; }
  python - "$L" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
print(f"{sys.argv[1]:28s} step {d['ms_per_step']*1e3:6.1f} us  sweep(cold) {d['roofline']['kernel_ms']*1e3:6.1f} us  "
      f"value {d['value']/1e9:6.1f} G  e2e {d['e2e']['value']/1e9:6.1f} G")
PY
  python tools/time_finish.py 2>/dev/null | tail -2 | sed "s/^/   /"
done
