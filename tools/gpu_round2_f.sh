set -x
PSG_TRACE=1 PSG_NO_GRAPH=1 python tools/stage_probe.py c3 1 > gpurun_out/r2f_c3_new.log 2>&1
PSG_OLD_BOOT=1 PSG_TRACE=1 PSG_NO_GRAPH=1 python tools/stage_probe.py c3 1 > gpurun_out/r2f_c3_old.log 2>&1
PSG_OLD_BOOT=1 python tools/stage_probe.py c5 2 > gpurun_out/r2f_c5_old.log 2>&1
PSG_OLD_BOOT=1 python tools/stage_probe.py c2 3 > gpurun_out/r2f_c2_old.log 2>&1
python tools/stage_probe.py c2 3 > gpurun_out/r2f_c2_new.log 2>&1
