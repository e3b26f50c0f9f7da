for o in 0.25 1.0 1.5 2.0 3.0; do
  PSG_OCC=$o python tools/c3_oneshot_probe.py > gpurun_out/occ_c3_$o.json 2>&1
  PSG_OCC=$o PSG_GRAPH_PROF=0 python tools/stage_probe.py c3 6 > gpurun_out/occ_c3g_$o.json 2>&1
done
python - <<'PY'
import json
for o in ("0.25","1.0","1.5","2.0","3.0"):
    d=json.load(open(f"gpurun_out/occ_c3_{o}.json")); g=json.load(open(f"gpurun_out/occ_c3g_{o}.json"))
    t=sorted(r['total_ms'] for r in g['runs'])
    print(o, "one_shot %.2f first %.2f third %.2f graph_med %.3f" % (d['one_shot_s']*1e3, d['1']['first_solve_s']*1e3, d['1']['third_s']*1e3, t[len(t)//2]), g['answer'])
PY
