for occ in 0.08 0.15 0.25 0.4 0.7; do
  echo "occ=$occ $(PSG_OCC=$occ python bench.py --steps 20 --no-candidate-kernel --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readline()); print(d["ms_per_step"], d["kernel_ms_per_step"], d["correct"])')" >> gpurun_out/occ_sweep.log
done
