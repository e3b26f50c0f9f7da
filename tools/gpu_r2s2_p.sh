# ILP build kernels + bigger scan tiles: check, warm launch list, bench, suite
timeout 300 python tools/one_solve.py 20 4 > gpurun_out/s2p_one.log 2>&1; echo rc=$? >> gpurun_out/s2p_one.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/s2p_launches.csv python tools/one_solve.py 20 4 > gpurun_out/s2p_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/s2p_launches.csv > gpurun_out/s2p_launches.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-candidate-kernel --no-cpu-baseline --no-configs > gpurun_out/s2p_bench.json 2> gpurun_out/s2p_bench.err
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/s2p_suite.log
cat gpurun_out/s2p_one.log gpurun_out/s2p_launches.txt gpurun_out/s2p_suite.log
