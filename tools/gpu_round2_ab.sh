rm -f gpurun_out/r2ab_probe.jsonl
for k in 1 2; do python tools/stage_probe.py c2 5 >> gpurun_out/r2ab_probe.jsonl 2>>gpurun_out/r2ab_probe.err; done
