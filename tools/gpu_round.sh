#!/bin/bash
# Round-end GPU evidence: tests, bench lines, launch list and full ncu captures
# of the sweep and step-tail kernels.  Each ncu command runs only after the
# same command exited 0 without ncu.   usage: tools/gpu_round.sh r01
set -u
O=gpurun_out; R=${1:-r01}
python -m pytest tests -m gpu -x -q > $O/pytest_gpu_$R.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu_$R.log
python bench.py > $O/bench_$R.json 2> $O/bench_$R.err; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_$R.json 2> $O/bench_ref_$R.err; echo "ref rc=$?"
L="python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
if $L > $O/plain_launch_$R.log 2>&1; then
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_$R.csv $L \
    > $O/ncu_launch_$R.log 2>&1; echo "ncu launches rc=$?"
fi
F="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --eager"
if $F > $O/plain_full_$R.log 2>&1; then
  ncu --set full --clock-control none --import-source on -k regex:${SWEEP_K:-k_joint_sweep} --launch-skip 4 \
    --launch-count 1 -o $O/sweep_$R -f $F > $O/ncu_full_$R.log 2>&1; echo "ncu sweep rc=$?"
  ncu --set full --clock-control none --import-source on -k regex:${TAIL_K:-k_step_tail_joint} --launch-skip 4 \
    --launch-count 1 -o $O/finish_$R -f $F > $O/ncu_finish_$R.log 2>&1; echo "ncu finish rc=$?"
fi
