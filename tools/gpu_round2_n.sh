timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -15 > gpurun_out/r2n_suite.log
timeout 900 python bench.py > gpurun_out/r2n_bench.json 2> gpurun_out/r2n_bench.err
tail -3 gpurun_out/r2n_suite.log
