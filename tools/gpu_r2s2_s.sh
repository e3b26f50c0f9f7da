PSG_TRACE=1 timeout 600 python tools/c4_list_probe.py 2>&1 | grep -E "csr|frnn|^list|^count" | tail -14 > gpurun_out/s2s_c4.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "csr or c4" 2>&1 | tail -5 > gpurun_out/s2s_tests.log
cat gpurun_out/s2s_c4.log gpurun_out/s2s_tests.log
