set -x
rm -f gpurun_out/r2ad_*
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2ad_smi.txt
for lv in 0 1 2; do PSG_GRAPH_PROF=$lv timeout 300 python tools/stage_probe.py c2 5 >> gpurun_out/r2ad_probe.jsonl 2>>gpurun_out/r2ad_probe.err; done
timeout 300 python tools/stage_probe.py c1 5 >> gpurun_out/r2ad_probe.jsonl 2>>gpurun_out/r2ad_probe.err
PSG_GRAPH_PROF=0 timeout 300 python tools/stage_probe.py c3 5 >> gpurun_out/r2ad_probe.jsonl 2>>gpurun_out/r2ad_probe.err
timeout 900 python bench.py > gpurun_out/r2ad_bench.json 2> gpurun_out/r2ad_bench.err
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r2ad_suite.log 2>&1
tail -3 gpurun_out/r2ad_suite.log
tail -c 3000 gpurun_out/r2ad_bench.json
