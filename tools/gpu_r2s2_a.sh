# round 2, session 2: validate HEAD (suite, smoke, bench)
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/s2a_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2a_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/s2a_bench.json 2> gpurun_out/s2a_bench.err
cat gpurun_out/s2a_suite.log gpurun_out/s2a_smoke.log
