# HEAD validation: suite, smoke, full bench (default flags), launch list of the C2 bench
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/s2v_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2v_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/s2v_bench.json 2> gpurun_out/s2v_bench.err
timeout 600 python tools/one_solve.py 20 4 > gpurun_out/s2v_one.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/s2v_launches_c2.csv python tools/one_solve.py 20 4 > gpurun_out/s2v_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/s2v_launches_c2.csv > gpurun_out/s2v_launches_c2.txt
cat gpurun_out/s2v_suite.log gpurun_out/s2v_smoke.log
