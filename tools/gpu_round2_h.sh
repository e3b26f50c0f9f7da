set -x
rm -f gpurun_out/r2h_probe.jsonl
for c in c1 c2 c3 c5; do python tools/stage_probe.py $c 3 >> gpurun_out/r2h_probe.jsonl 2>gpurun_out/r2h_probe.err; done
PSG_TRACE=1 PSG_NO_GRAPH=1 python tools/stage_probe.py c3 2 > gpurun_out/r2h_c3_trace.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -30 > gpurun_out/r2h_suite.log
