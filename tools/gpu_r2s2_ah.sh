timeout 1500 python -m pytest tests -q -x -m gpu 2>&1 | tail -4 > gpurun_out/ah.log
for k in 1 2; do for e in "" "PSG_ORDERED_GRID=1"; do env $e PSG_GRAPH_PROF=0 timeout 300 python tools/stage_probe.py c2 12 | python -c "
import json,sys; d=json.load(sys.stdin); t=sorted(r['total_ms'] for r in d['runs'])
print('$e' or 'arrival', 'median', t[len(t)//2], 'min', t[0], d['answer'][:2], d['runs'][-1]['window_pairs'])" >> gpurun_out/ah.log; done; done
cat gpurun_out/ah.log
