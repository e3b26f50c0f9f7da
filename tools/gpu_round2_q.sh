python tools/stage_probe.py c5 2 > gpurun_out/r2q_c5.json 2>&1
timeout 900 python -m pytest tests -q -m gpu -x -k "c5 or dense or sharded" 2>&1 | tail -3 > gpurun_out/r2q_suite.log
python tools/one_c5.py 1048576 2 > gpurun_out/r2q_c5_20.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_dense_gram -s 1 -c 1 -o gpurun_out/r2q_gram python tools/one_c5.py 1048576 2 > gpurun_out/r2q_ncu.log 2>&1
cat gpurun_out/r2q_suite.log
