rm -f gpurun_out/r2ac_probe.jsonl
for c in c1 c2 c3; do python tools/stage_probe.py $c 3 >> gpurun_out/r2ac_probe.jsonl 2>>gpurun_out/r2ac_probe.err; PSG_GRAPH_STAGES=1 python tools/stage_probe.py $c 3 >> gpurun_out/r2ac_probe.jsonl 2>>gpurun_out/r2ac_probe.err; done
echo
cat gpurun_out/r2ac_suite.log
