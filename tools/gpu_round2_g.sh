PSG_TRACE=1 PSG_NO_GRAPH=1 PSG_NO_FUSED_COUNT=1 PSG_OLD_BOOT=1 python tools/stage_probe.py c3 1 > gpurun_out/r2g_c3_a.log 2>&1
PSG_TRACE=1 PSG_NO_GRAPH=1 PSG_NO_FUSED_COUNT=1 python tools/stage_probe.py c3 1 > gpurun_out/r2g_c3_b.log 2>&1
