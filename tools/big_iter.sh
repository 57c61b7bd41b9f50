#!/bin/bash
# Tally rewrite check on one B200: parity of the chunked tally + the large-network
# configs, C4/C3 bench lines, one ncu capture of k_sweep_big.
set -u
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_api.py tests/test_gpu_stats.py -x -q > $O/pt_tally.log 2>&1; echo "tests rc=$?"; tail -3 $O/pt_tally.log
for w in c4 c3 c5; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > $O/${w}_bench2.json 2> $O/${w}_bench2.err; echo "$w bench rc=$?"
  python -c "import json,sys; d=json.loads(open('$O/${w}_bench2.json').read().strip().splitlines()[-1]); print('$w', d['ms_per_step'], d['value'], d['e2e']['ms_per_step'])"
done
F="python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline --eager"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_sweep_big" --launch-skip 2 --launch-count 1 -o $O/full_big -f $F > $O/ncu_big.log 2>&1; echo "ncu rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_c4.csv python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "launches rc=$?"
