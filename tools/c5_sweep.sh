python -m pytest tests -m gpu -x -q -k "dense or sharded or gram or c5 or mixture or fullsize" > gpurun_out/dense_tests.log 2>&1; echo rc=$? >> gpurun_out/dense_tests.log
PSG_TRACE=1 python tools/one_c5.py 16777216 3 2>&1 | grep -v "stage\|enqueued" > gpurun_out/c5_sweep.log 2>&1
