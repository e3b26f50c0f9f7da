# bucket build v2: quick check, launch list, full gpu suite, bench
timeout 300 python tools/one_solve.py 20 4 > gpurun_out/s2l_one.log 2>&1; echo rc=$? >> gpurun_out/s2l_one.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/s2l_launches_c2.csv python tools/one_solve.py 20 4 > gpurun_out/s2l_ncu1.log 2>&1
python tools/launch_summary.py gpurun_out/s2l_launches_c2.csv > gpurun_out/s2l_launches_c2.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-candidate-kernel --no-cpu-baseline --no-configs > gpurun_out/s2l_bench.json 2> gpurun_out/s2l_bench.err
cat gpurun_out/s2l_one.log gpurun_out/s2l_launches_c2.txt gpurun_out/s2l_suite.log
