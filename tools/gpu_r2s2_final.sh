# round-2 final validation: suite, smoke, full bench, C2 launch list, ncu of the projection
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/fin3_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin3_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/fin3_bench.json 2> gpurun_out/fin3_bench.err
timeout 600 python tools/one_solve.py 20 4 > gpurun_out/fin3_one.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/fin3_launches_c2.csv python tools/one_solve.py 20 4 > gpurun_out/fin3_ncu1.log 2>&1
python tools/launch_summary.py gpurun_out/fin3_launches_c2.csv > gpurun_out/fin3_launches_c2.txt
timeout 600 ncu --set full --clock-control none -k regex:k_project_tc -s 1 -c 1 -o gpurun_out/fin3_proj python tools/one_solve.py 20 2 > gpurun_out/fin3_ncu2.log 2>&1
cat gpurun_out/fin3_suite.log gpurun_out/fin3_smoke.log
