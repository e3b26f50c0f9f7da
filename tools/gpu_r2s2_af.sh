for k in 1 2 3; do for e in "" "PSG_NO_PDL=1"; do env $e PSG_GRAPH_PROF=0 timeout 300 python tools/stage_probe.py c2 12 | python -c "
import json,sys; d=json.load(sys.stdin); t=sorted(r['total_ms'] for r in d['runs'])
print('$e' or 'pdl', 'median', t[len(t)//2], 'min', t[0], d['answer'][:2])"; done; done
