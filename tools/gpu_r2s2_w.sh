out=gpurun_out/s2w.jsonl; rm -f $out
for k in 1 2; do PSG_GRAPH_PROF=0 timeout 300 python tools/stage_probe.py c2 10 | python -c "
import json,sys; d=json.load(sys.stdin); t=sorted(r['total_ms'] for r in d['runs'])
print(json.dumps({'median_ms': t[len(t)//2], 'min_ms': t[0], 'answer': d['answer']}))" >> $out; done
timeout 600 python bench.py --steps 20 --warmup 5 --no-candidate-kernel --no-cpu-baseline --no-configs > gpurun_out/s2w_bench.json 2> gpurun_out/s2w_bench.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ties.py tests/test_gpu_grid_build.py -q -x 2>&1 | tail -3 >> $out
cat $out; python -c "import json; d=json.load(open('gpurun_out/s2w_bench.json')); print(d['ms_per_step'], d['roofline']['frac'])"
