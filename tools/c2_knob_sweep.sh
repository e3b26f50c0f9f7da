# C2 graph-replay totals (PSG_GRAPH_PROF=0) across the grid occupancy and the bootstrap evaluation count
out=gpurun_out/c2_knobs.jsonl; rm -f $out
for occ in 0.25 0.35 0.5 0.75; do
  PSG_GRAPH_PROF=0 PSG_OCC=$occ timeout 300 python tools/stage_probe.py c2 8 | python -c "
import json,sys; d=json.load(sys.stdin); t=sorted(r['total_ms'] for r in d['runs'])
print(json.dumps({'occ': $occ, 'median_ms': t[len(t)//2], 'min_ms': t[0], 'answer': d['answer']}))" >> $out
done
for ev in 1024 2048 8192; do
  PSG_GRAPH_PROF=0 PSG_BOOT_EVALS=$ev timeout 300 python tools/stage_probe.py c2 8 | python -c "
import json,sys; d=json.load(sys.stdin); t=sorted(r['total_ms'] for r in d['runs'])
print(json.dumps({'boot_evals': $ev, 'median_ms': t[len(t)//2], 'min_ms': t[0]}))" >> $out
done
cat $out
timeout 300 python tools/c4_list_probe.py > gpurun_out/c4_probe_blockmax.log 2>&1; cat gpurun_out/c4_probe_blockmax.log
PSG_GRAPH_PROF=2 timeout 300 python tools/stage_probe.py c3 3 > gpurun_out/c3_probe_blockmax.json 2>&1; tail -c 600 gpurun_out/c3_probe_blockmax.json
