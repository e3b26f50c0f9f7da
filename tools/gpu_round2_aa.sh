rm -f gpurun_out/r2aa_probe.jsonl
for c in c1 c2 c3; do python tools/stage_probe.py $c 5 >> gpurun_out/r2aa_probe.jsonl 2>>gpurun_out/r2aa_probe.err; done
timeout 1200 python -m pytest tests -q -m gpu -x -k "parity or ties or fullsize or sharded or cli" 2>&1 | tail -3 > gpurun_out/r2aa_suite.log
cat gpurun_out/r2aa_suite.log
