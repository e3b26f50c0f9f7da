python -m pytest tests -m gpu -x -q -k "frnn or neighbor or fixed_radius or cli or sweep" > gpurun_out/frnn_tests.log 2>&1; echo rc=$? >> gpurun_out/frnn_tests.log
python tools/one_c4.py 5 > gpurun_out/frnn_sweep.log 2>&1
python tools/bench_configs.py c4 >> gpurun_out/frnn_sweep.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_frnn_cells -s 1 -c 1 -o gpurun_out/frnn_cells -f python tools/one_c4.py 2 > gpurun_out/ncu_frnn.log 2>&1
