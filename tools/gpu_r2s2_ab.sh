out=gpurun_out/s2ab.txt; rm -f $out
for k in 1 2; do PSG_GRAPH_PROF=0 timeout 300 python tools/stage_probe.py c2 10 | python -c "
import json,sys; d=json.load(sys.stdin); t=sorted(r['total_ms'] for r in d['runs'])
print('c2 graph', t[len(t)//2], t[0], d['answer'])" >> $out; done
PSG_GRAPH_PROF=0 timeout 300 python tools/stage_probe.py c3 6 | python -c "
import json,sys; d=json.load(sys.stdin); t=sorted(r['total_ms'] for r in d['runs'])
print('c3 graph', t[len(t)//2], t[0], d['answer'])" >> $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ties.py tests/test_gpu_grid_build.py tests/test_gpu_keys.py -q -x 2>&1 | tail -2 >> $out
python tools/one_solve.py 20 2 > gpurun_out/o.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_grid_scan2 --csv --log-file gpurun_out/s2ab_scan.csv python tools/one_solve.py 20 2 > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/s2ab_scan.csv >> $out
cat $out
