python tools/one_solve.py 20 2 > gpurun_out/r2k_one.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_presample|k_cell_fix<|k_grid_scan2|k_cell_place" -s 4 -c 4 -o gpurun_out/r2k_c2 python tools/one_solve.py 20 2 > gpurun_out/r2k_ncu.log 2>&1
tail -3 gpurun_out/r2k_ncu.log
