#!/bin/bash
# Packed uploads on the generic graphs: parity + C4/C3 bench lines (e2e).
set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_joint.py tests/test_gpu_api.py -x -q > $O/pt_e2e.log 2>&1; echo "tests rc=$?"; tail -3 $O/pt_e2e.log
for w in c4 c3; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > $O/${w}_bench3.json 2> $O/${w}_bench3.err; echo "$w bench rc=$?"
  python -c "import json; d=json.loads(open('$O/${w}_bench3.json').read().strip().splitlines()[-1]); print('$w', d['ms_per_step'], d['e2e'])"
done
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > $O/c2_bench3.json 2> $O/c2_bench3.err; echo "c2 rc=$?"
python -c "import json; d=json.loads(open('$O/c2_bench3.json').read().strip().splitlines()[-1]); print('c2', d['ms_per_step'], d['e2e']['ms_per_step'])"
