timeout 600 python tools/c4_list_probe.py > gpurun_out/s2r_c4.log 2>&1
PSG_CSR_RADIX=1 timeout 600 python tools/c4_list_probe.py > gpurun_out/s2r_c4_radix.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "csr or c4" 2>&1 | tail -5 > gpurun_out/s2r_tests.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c4" 2>&1 | tail -5 >> gpurun_out/s2r_tests.log
cat gpurun_out/s2r_c4.log gpurun_out/s2r_c4_radix.log gpurun_out/s2r_tests.log
