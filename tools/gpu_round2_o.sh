python tools/c3_oneshot_probe.py > gpurun_out/r2o_c3.json 2>&1
PSG_TRACE=1 python tools/c3_oneshot_probe.py > gpurun_out/r2o_c3_trace.log 2>&1
python tools/stage_probe.py c5 2 > gpurun_out/r2o_c5.json 2>&1
cat gpurun_out/r2o_c3.json
