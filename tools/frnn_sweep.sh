python -m pytest tests -m gpu -x -q -k "frnn or neighbor or fixed_radius or cli or sweep" > gpurun_out/frnn_tests.log 2>&1; echo rc=$? >> gpurun_out/frnn_tests.log
python tools/one_c4.py 7 > gpurun_out/frnn_sweep.log 2>&1
