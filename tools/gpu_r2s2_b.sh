# bucket build: quick check, grid/parity tests, bench, C2 launch list
timeout 300 python tools/one_solve.py 20 4 > gpurun_out/s2b_one.log 2>&1; echo rc=$? >> gpurun_out/s2b_one.log
timeout 900 python -m pytest tests/test_gpu_grid_build.py tests/test_gpu_parity.py tests/test_gpu_ties.py -q -x 2>&1 | tail -15 > gpurun_out/s2b_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-candidate-kernel --no-cpu-baseline --no-configs > gpurun_out/s2b_bench.json 2> gpurun_out/s2b_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/s2b_launches_c2.csv python tools/one_solve.py 20 4 > gpurun_out/s2b_ncu1.log 2>&1
cat gpurun_out/s2b_one.log gpurun_out/s2b_tests.log
