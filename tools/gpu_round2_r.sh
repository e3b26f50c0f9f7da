python tools/stage_probe.py c5 2 > gpurun_out/r2r_c5.json 2>&1
timeout 900 python -m pytest tests -q -m gpu -x -k "c5 or dense or sharded or parity" 2>&1 | tail -3 > gpurun_out/r2r_suite.log
PSG_LIB_PATH=$PWD/tools/dbg/libpairscan_b200_tl.so python tools/one_c5.py 4194304 2 > gpurun_out/r2r_tl.log 2>&1
cat gpurun_out/r2r_suite.log
