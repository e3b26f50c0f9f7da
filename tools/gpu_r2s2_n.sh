# PDL chain: check, A/B bench, suite
timeout 300 python tools/one_solve.py 20 4 > gpurun_out/s2n_one.log 2>&1; echo rc=$? >> gpurun_out/s2n_one.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-candidate-kernel --no-cpu-baseline --no-configs > gpurun_out/s2n_bench.json 2> gpurun_out/s2n_bench.err
PSG_NO_PDL=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-candidate-kernel --no-cpu-baseline --no-configs > gpurun_out/s2n_bench_nopdl.json 2> gpurun_out/s2n_bench_nopdl.err
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/s2n_suite.log
cat gpurun_out/s2n_one.log gpurun_out/s2n_suite.log
