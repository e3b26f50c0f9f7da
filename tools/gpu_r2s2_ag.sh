timeout 900 python -m pytest tests/test_gpu_keys.py -q -x 2>&1 | tail -3 > gpurun_out/ag_keys.log
timeout 900 python -m pytest tests -q -x -m gpu -k "motif or window or c3 or znorm or walk" 2>&1 | tail -2 >> gpurun_out/ag_keys.log
for e in "" "PSG_WINDOW_CC=1"; do env $e PSG_GRAPH_PROF=0 python tools/stage_probe.py c3 8 > gpurun_out/ag_c3.json; env $e python tools/c3_oneshot_probe.py > gpurun_out/ag_c3o.json; python -c "
import json; g=json.load(open('gpurun_out/ag_c3.json')); t=sorted(r['total_ms'] for r in g['runs']); d=json.load(open('gpurun_out/ag_c3o.json'))
print('$e' or 'tc', 'graph', t[len(t)//2], 'one_shot', d['one_shot_s']*1e3, g['answer'])" >> gpurun_out/ag_keys.log; done
cat gpurun_out/ag_keys.log
