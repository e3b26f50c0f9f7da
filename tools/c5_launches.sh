ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python tools/one_c5.py 16777216 3 > gpurun_out/ncu_c5.log 2>&1
