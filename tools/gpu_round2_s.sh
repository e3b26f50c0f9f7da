timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -5 > gpurun_out/r2s_suite.log
timeout 900 python bench.py > gpurun_out/r2s_bench.json 2> gpurun_out/r2s_bench.err
python bench.py --steps 20 --warmup 5 --no-configs --no-cpu-baseline --no-candidate-kernel > gpurun_out/r2s_bench_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2s_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-configs --no-cpu-baseline --no-candidate-kernel > gpurun_out/r2s_ncu.log 2>&1
tail -3 gpurun_out/r2s_suite.log
