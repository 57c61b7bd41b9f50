#!/bin/bash
# Round-end GPU evidence: tests, bench lines, launch list and full ncu captures
# of the sweep and step-tail kernels (as they run in the replayed step graph).
# Each ncu command runs only after the same command exited 0 without ncu.
#   usage: tools/gpu_round.sh r02
set -u
O=gpurun_out; R=${1:-r02}
python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu_$R.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu_$R.log
python bench.py > $O/bench_$R.json 2> $O/bench_$R.err; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_$R.json 2> $O/bench_ref_$R.err; echo "ref rc=$?"
python bench.py --rng numpy --steps 20 --no-cpu-baseline > $O/bench_numpy_$R.json 2>&1; echo "numpy rc=$?"
for w in c3 c4; do python bench.py --workload $w --steps 10 > $O/bench_${w}_$R.json 2>&1; echo "$w rc=$?"; done
python bench.py --workload c5 > $O/bench_c5_$R.json 2>&1; echo "c5 rc=$?"
python bench.py --workload c2s --no-cpu-baseline > $O/bench_c2s_$R.json 2>&1; echo "c2s rc=$?"
L="python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
if $L > $O/plain_launch_$R.log 2>&1; then
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_$R.csv $L \
    > $O/ncu_launch_$R.log 2>&1; echo "ncu launches rc=$?"
fi
F="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
if $F > $O/plain_full_$R.log 2>&1; then
  ncu --set full --clock-control none --import-source on -k regex:${SWEEP_K:-k_joint_sweep} --launch-skip 8 \
    --launch-count 1 -o $O/sweep_$R -f $F > $O/ncu_full_$R.log 2>&1; echo "ncu sweep rc=$?"
  ncu --set full --clock-control none --import-source on -k regex:${TAIL_K:-k_step_tail_joint} --launch-skip 8 \
    --launch-count 1 -o $O/finish_$R -f $F > $O/ncu_finish_$R.log 2>&1; echo "ncu finish rc=$?"
fi
B="python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline --eager"
if $B > $O/plain_big_$R.log 2>&1; then
  ncu --set full --clock-control none --import-source on -k regex:k_sweep_big --launch-skip 3 --launch-count 1 \
    -o $O/big_$R -f $B > $O/ncu_big_$R.log 2>&1; echo "ncu big rc=$?"
fi
