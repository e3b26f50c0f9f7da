# FRNN scan: GPU parity subset + C4 timings (count+hash and the sorted list)
python -m pytest tests -m gpu -x -q -k "frnn or neighbor or fixed_radius or cli" > gpurun_out/frnn_tests.log 2>&1; echo rc=$? >> gpurun_out/frnn_tests.log
python tools/one_c4.py 5 > gpurun_out/frnn_sweep.log 2>&1
python tools/bench_configs.py c4 >> gpurun_out/frnn_sweep.log 2>&1
