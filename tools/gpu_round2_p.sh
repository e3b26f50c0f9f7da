PSG_LIB_PATH=$PWD/tools/dbg/libpairscan_b200_tl.so python tools/one_c5.py 4194304 2 > gpurun_out/r2p_tl.log 2>&1
grep -c "^TL" gpurun_out/r2p_tl.log
python tools/one_c5.py 4194304 2 > gpurun_out/r2p_c5_22.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_hmma.sum,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_dense_gram -c 2 --csv --log-file gpurun_out/r2p_gram_metrics.csv python tools/one_c5.py 4194304 2 > gpurun_out/r2p_ncu.log 2>&1
