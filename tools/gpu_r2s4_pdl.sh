# A/B: the projection's mainloop starting under k_presample (PDL, epilogue-only wait) against PSG_NO_PDL=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_grid_build.py tests/test_gpu_keys.py -q -x -m gpu 2>&1 | tail -3 > gpurun_out/pdl_suite.log
for i in 1 2 3; do
  timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-configs --no-candidate-kernel --e2e-steps 2 2> /dev/null | python -c "import sys,json; j=json.loads(sys.stdin.readlines()[-1]); print('pdl', j['ms_per_step'], j['roofline']['frac'])" >> gpurun_out/pdl_ab.log
  PSG_NO_PDL=1 timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-configs --no-candidate-kernel --e2e-steps 2 2> /dev/null | python -c "import sys,json; j=json.loads(sys.stdin.readlines()[-1]); print('nopdl', j['ms_per_step'], j['roofline']['frac'])" >> gpurun_out/pdl_ab.log
done
cat gpurun_out/pdl_suite.log gpurun_out/pdl_ab.log
