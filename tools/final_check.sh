set -u
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_final.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke_final.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke_final.log
timeout 600 python bench.py > $O/bench_final.json 2> $O/bench_final.err; echo "bench rc=$?"; tail -c 400 $O/bench_final.json
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
$B > $O/plain_launch_final.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_final.csv $B > $O/ncu_launch_final.log 2>&1; echo "ncu rc=$?"
