set -u
O=gpurun_out
timeout 300 python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline > $O/c4_bench.json 2> $O/c4_bench.err; echo "bench rc=$?"; tail -c 600 $O/c4_bench.json
F="python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline --eager"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_tally_chunked|k_sweep_big" --launch-skip 2 --launch-count 2 -o $O/full_c4 -f $F > $O/ncu_c4.log 2>&1; echo "ncu rc=$?"; tail -3 $O/ncu_c4.log
