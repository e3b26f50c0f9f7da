timeout 1200 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "not c5_full" 2>&1 | tail -2 > gpurun_out/ai.log
timeout 900 python tools/perf_sweep.py 2>&1 | grep -E "d=  8|d= 16|d=  3|d= 32|d= 64" >> gpurun_out/ai.log
cat gpurun_out/ai.log
