python tools/one_c5.py 4194304 3 > gpurun_out/c5_small.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_dense_gram -s 1 -c 1 -o gpurun_out/gram8 -f python tools/one_c5.py 4194304 2 > gpurun_out/ncu_gram.log 2>&1
