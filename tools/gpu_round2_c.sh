# round 2, call C: GPU suite after the virtual window rows + exact rescan; C3 timing
set -x
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -40 > gpurun_out/r2c_suite.log
timeout 600 python tools/bench_configs.py c3 c2 > gpurun_out/r2c_configs.jsonl 2> gpurun_out/r2c_configs.err
tail -3 gpurun_out/r2c_suite.log
cat gpurun_out/r2c_configs.jsonl
