python -m pytest tests -m gpu -x -q -k "dense or sharded or gram or c5 or mixture" > gpurun_out/dense_tests.log 2>&1; echo rc=$? >> gpurun_out/dense_tests.log
for k in 8 7 6; do
  echo "keys=$k" >> gpurun_out/c5_sweep.log
  PSG_TRACE=1 PSG_DENSE_KEYS=$k timeout 300 python tools/one_c5.py 16777216 2 >> gpurun_out/c5_sweep.log 2>&1
done
