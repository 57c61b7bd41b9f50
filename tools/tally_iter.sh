python -m pytest tests/test_gpu_configs.py tests/test_gpu_large.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/tally_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/tally_tests.log
bash tools/bench_all.sh c3 c4
