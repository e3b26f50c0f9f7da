# ncu full capture of the bucket build kernels (second solve)
timeout 300 python tools/one_solve.py 20 2 > gpurun_out/s2k_one.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bucket_build -s 1 -c 1 -o gpurun_out/s2k_bucket python tools/one_solve.py 20 2 > gpurun_out/s2k_ncu.log 2>&1
tail -3 gpurun_out/s2k_ncu.log
