timeout 900 python -m pytest tests -q -m gpu -x -k "c4 or frnn or multiprocess or c5_recipe or dense" 2>&1 | tail -5 > gpurun_out/r2m_suite.log
timeout 900 python bench.py > gpurun_out/r2m_bench.json 2> gpurun_out/r2m_bench.err
python tools/stage_probe.py c5 2 > gpurun_out/r2m_c5.json 2>&1
tail -3 gpurun_out/r2m_suite.log
