set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_ties.py "tests/test_gpu_fullsize.py" -x -q -m gpu -k "ties or c5 or identical or duplicates or flat or repeated" 2>&1 | tail -30 > gpurun_out/r1_new.log
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -30 > gpurun_out/r1_suite.log
timeout 1500 python tools/c5_fullsize.py gpurun_out/c5_fullsize.json 24 > gpurun_out/r1_c5.log 2>&1
tail -5 gpurun_out/r1_new.log gpurun_out/r1_suite.log gpurun_out/r1_c5.log
