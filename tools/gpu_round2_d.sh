# round 2, call D: fused C2 pipeline (presample -> counting projection -> fix+bootstrap LB -> select)
set -x
timeout 600 python tools/bench_configs.py c1 c2 c3 c4 c5 > gpurun_out/r2d_configs.jsonl 2> gpurun_out/r2d_configs.err
cat gpurun_out/r2d_configs.jsonl; tail -5 gpurun_out/r2d_configs.err
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -40 > gpurun_out/r2d_suite.log
tail -3 gpurun_out/r2d_suite.log
python tools/one_solve.py 20 4 > gpurun_out/r2d_one.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2d_launches_c2.csv python tools/one_solve.py 20 4 > gpurun_out/r2d_ncu1.log 2>&1
