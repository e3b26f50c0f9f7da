# round 2, call B: full GPU suite, bench, C2 launch list + ncu of the latency-bound kernels
set -x
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -40 > gpurun_out/r2b_suite.log
timeout 900 python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
python tools/one_solve.py 20 4 > gpurun_out/r2b_one.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2b_launches_c2.csv python tools/one_solve.py 20 4 > gpurun_out/r2b_ncu1.log 2>&1
python tools/one_solve.py 20 2 > gpurun_out/r2b_one2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_grid_scan2|k_grid_bootstrap|k_setup|k_cell_fix<|k_cell_place|k_cell_count|k_scan_lookback|k_recheck" -s 9 -c 9 -o gpurun_out/r2b_c2small python tools/one_solve.py 20 2 > gpurun_out/r2b_ncu2.log 2>&1
tail -3 gpurun_out/r2b_suite.log
head -c 3000 gpurun_out/r2b_bench.json
