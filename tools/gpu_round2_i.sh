PSG_LIB_PATH=$PWD/tools/dbg/libpairscan_b200_dbg.so PSG_TRACE=1 PSG_NO_GRAPH=1 timeout 600 python tools/stage_probe.py c5 1 > gpurun_out/r2i_c5_dbg.log 2>&1
tail -20 gpurun_out/r2i_c5_dbg.log
