python -m pytest tests/test_gpu_configs.py tests/test_gpu_large.py -q -x -p no:cacheprovider > gpurun_out/big_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/big_tests.log
python bench.py --workload c4 --steps 10 --no-cpu-baseline > gpurun_out/c4_r2f.json 2> gpurun_out/c4_r2f.err; echo "c4 rc=$?"
python bench.py --workload c3 --steps 10 --no-cpu-baseline > gpurun_out/c3_r2f.json 2> gpurun_out/c3_r2f.err; echo "c3 rc=$?"
B="python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline --eager"
$B > gpurun_out/plain_big.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_sweep_big --launch-skip 3 --launch-count 1 -o gpurun_out/big_k3 -f $B > gpurun_out/ncu_big_list.log 2>&1; echo "ncu rc=$?"
