# launch list of the bench command + one full capture of the FRNN small-d scan
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_frnn_scan_small -s 1 -c 1 -o gpurun_out/frnn_small -f python tools/one_c4.py 2 > gpurun_out/ncu_frnn.log 2>&1
