timeout 1200 python -m pytest tests -q -x -m gpu -k "c5 or dense or mixture or cluster or ties" 2>&1 | tail -3 > gpurun_out/ae_t.log
PSG_GRAPH_PROF=0 timeout 600 python tools/stage_probe.py c5 2 > gpurun_out/ae_c5.json 2>&1
python -c "
import json; g=json.load(open('gpurun_out/ae_c5.json')); print([r['total_ms'] for r in g['runs']], g['answer'], [r['dense_tiles'] for r in g['runs']])"
cat gpurun_out/ae_t.log
