rm -f gpurun_out/r2w_probe.jsonl
for c in c1 c2 c3 c5; do python tools/stage_probe.py $c 3 >> gpurun_out/r2w_probe.jsonl 2>>gpurun_out/r2w_probe.err; done
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > gpurun_out/r2w_suite.log
python tools/one_solve.py 20 4 > gpurun_out/r2w_one.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2w_launches_c2.csv python tools/one_solve.py 20 4 > gpurun_out/r2w_ncu1.log 2>&1
cat gpurun_out/r2w_suite.log
