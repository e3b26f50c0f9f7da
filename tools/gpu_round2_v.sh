python tools/one_solve.py 20 2 > gpurun_out/r2v_one.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"presample|cell_fix|boot_select|scan_lookback" -c 8 -o gpurun_out/r2v_c2 python tools/one_solve.py 20 2 > gpurun_out/r2v_ncu.log 2>&1
tail -3 gpurun_out/r2v_ncu.log
