rm -f gpurun_out/r2j_probe.jsonl
python tools/stage_probe.py c5 3 >> gpurun_out/r2j_probe.jsonl 2>>gpurun_out/r2j_probe.err
for o in 0.15 0.5 1.0; do PSG_OCC=$o python tools/stage_probe.py c2 3 >> gpurun_out/r2j_probe.jsonl 2>>gpurun_out/r2j_probe.err; done
python tools/stage_probe.py c2 3 >> gpurun_out/r2j_probe.jsonl 2>>gpurun_out/r2j_probe.err
python tools/one_solve.py 20 4 > gpurun_out/r2j_one.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2j_launches_c2.csv python tools/one_solve.py 20 4 > gpurun_out/r2j_ncu1.log 2>&1
