python tools/c3_oneshot_probe.py > gpurun_out/s2x_c3.json 2>&1
for o in 0.5 0.85 1.5; do PSG_OCC=$o python tools/c3_oneshot_probe.py > gpurun_out/s2x_c3_occ$o.json 2>&1; done
python - <<'PY'
import json
for f in ["s2x_c3.json","s2x_c3_occ0.5.json","s2x_c3_occ0.85.json","s2x_c3_occ1.5.json"]:
    try:
        d=json.load(open("gpurun_out/"+f))
        print(f, "one_shot %.2f ms" % (d["one_shot_s"]*1e3), "create %.2f first %.2f second %.2f third %.2f" % tuple(d["1"][k]*1e3 for k in ("create_s","first_solve_s","second_s","third_s")), d["one_shot_stages"])
    except Exception as e: print(f, "ERR", open("gpurun_out/"+f).read()[-300:])
PY
