#!/bin/bash
for L in "$@"; do
  if [ "$L" = default ]; then unset SAMEGIBBS_LIB; else export SAMEGIBBS_LIB=$PWD/$L; fi
  echo "== $L"; python bench.py --workload c5 --steps 8 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 step ms', round(d['ms_per_step'],1), 'value', '%.3e' % d['value'])"
done
