# ncu full capture of the bucket build kernels (second solve)
timeout 300 python tools/one_solve.py 20 2 > gpurun_out/s2d_one.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bucket -s 3 -c 3 -o gpurun_out/s2d_bucket python tools/one_solve.py 20 2 > gpurun_out/s2d_ncu.log 2>&1
tail -3 gpurun_out/s2d_ncu.log
