timeout 300 python tools/one_solve.py 20 4 > gpurun_out/s2o_one.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 200 --csv --log-file gpurun_out/s2o_launches_warm.csv python tools/one_solve.py 20 4 > gpurun_out/s2o_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/s2o_launches_warm.csv
