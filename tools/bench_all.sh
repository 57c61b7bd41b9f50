#!/bin/bash
# One digest line per workload (no CPU baseline).
for W in ${@:-c2 c3 c4}; do
  python bench.py --workload $W --no-cpu-baseline --steps 50 > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err || { echo "$W FAILED"; tail -5 gpurun_out/bench_$W.err; continue; }
  python - $W <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/bench_{sys.argv[1]}.json").read().strip().splitlines()[-1])
r = d["roofline"]
print(f"{sys.argv[1]} step {d['ms_per_step']*1e3:8.1f} us  value {d['value']:.3e}  sweep {r['kernel_ms']*1e3:8.1f} us  "
      f"frac {r['frac']:.3f}  e2e {d['e2e']['value']:.3e}  {d['kernel_path']}")
PY
done
