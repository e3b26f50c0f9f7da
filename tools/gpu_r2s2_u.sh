timeout 300 python tools/c4_list_probe.py > gpurun_out/s2u_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_group|k_frnn|k_radix|k_bucket" --csv --log-file gpurun_out/s2u_launches.csv python tools/c4_list_probe.py > gpurun_out/s2u_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/s2u_launches.csv
