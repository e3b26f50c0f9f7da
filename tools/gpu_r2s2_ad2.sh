timeout 1500 python -m pytest tests -q -x -m gpu 2>&1 | tail -3 > gpurun_out/ad2_suite.log
PSG_GRAPH_PROF=0 python tools/stage_probe.py c3 8 > gpurun_out/ad2_c3.json
PSG_GRAPH_PROF=0 python tools/stage_probe.py c2 8 > gpurun_out/ad2_c2.json
python tools/c3_oneshot_probe.py > gpurun_out/ad2_c3o.json
python - <<'PY'
import json
for f in ("ad2_c3.json","ad2_c2.json"):
    g=json.load(open("gpurun_out/"+f)); t=sorted(r['total_ms'] for r in g['runs']); print(f, t[len(t)//2], g['answer'])
d=json.load(open("gpurun_out/ad2_c3o.json")); print("c3 one-shot", d["one_shot_s"]*1e3)
PY
cat gpurun_out/ad2_suite.log
