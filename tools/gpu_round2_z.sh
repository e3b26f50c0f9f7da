timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/r2z_suite.log
timeout 900 python bench.py > gpurun_out/r2z_bench.json 2> gpurun_out/r2z_bench.err
cat gpurun_out/r2z_suite.log
