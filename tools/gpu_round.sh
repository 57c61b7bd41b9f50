#!/bin/bash
# Round-end GPU evidence: tests, bench lines, launch list and one full ncu capture
# of the sweep kernel.  Each ncu command runs only after the same command exited 0.
set -u
O=gpurun_out; R=${1:-r01}
python -m pytest tests -m gpu -x -q > $O/pytest_gpu_$R.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu_$R.log
python bench.py > $O/bench_$R.json 2> $O/bench_$R.err; echo "bench rc=$?"
python bench.py --no-fuse --no-cpu-baseline > $O/bench_nofuse_$R.json 2>&1; echo "nofuse rc=$?"
L="python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
if $L > $O/plain_launch_$R.log 2>&1; then
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_$R.csv $L \
    > $O/ncu_launch_$R.log 2>&1; echo "ncu launches rc=$?"
fi
F="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --eager --no-fuse"
if $F > $O/plain_full_$R.log 2>&1; then
  ncu --set full --clock-control none --import-source on -k regex:k_small_sweep --launch-skip 4 --launch-count 1 \
    -o $O/sweep_$R -f $F > $O/ncu_full_$R.log 2>&1; echo "ncu full rc=$?"
fi
