timeout 300 python tools/c4_list_probe.py > gpurun_out/s2t_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:k_group -c 4 -o gpurun_out/s2t_group python tools/c4_list_probe.py > gpurun_out/s2t_ncu.log 2>&1
tail -2 gpurun_out/s2t_ncu.log
