#!/bin/bash
# Lane-kernel draw variant check (build with -DSG_LANE_UNIFIED=3 or 4 to A/B): C3 parity + bench.
set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q > $O/pt_lane.log 2>&1; echo "tests rc=$?"; tail -2 $O/pt_lane.log
for w in c3 c3; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > $O/${w}_bench4.json 2> $O/${w}_bench4.err; echo "$w bench rc=$?"
  python -c "import json; d=json.loads(open('$O/${w}_bench4.json').read().strip().splitlines()[-1]); print('$w', d['ms_per_step'], d['e2e']['ms_per_step'])"
done
