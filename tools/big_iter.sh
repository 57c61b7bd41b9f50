python -m pytest tests/test_gpu_configs.py tests/test_gpu_large.py -q -x -p no:cacheprovider > gpurun_out/bft_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/bft_tests.log
python bench.py --workload c4 --steps 10 --no-cpu-baseline > gpurun_out/bft_c4.json 2> gpurun_out/bft_c4.err; echo "c4 rc=$?"
B="python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline --eager"
$B > gpurun_out/plain_big.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_sweep_big --launch-skip 3 --launch-count 1 -o gpurun_out/big_it -f $B > gpurun_out/ncu_big_it.log 2>&1; echo "ncu rc=$?"
