python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python tools/bench_configs.py c1 c2 c3 c4 c5 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 3 --warmup 3 --no-candidate-kernel --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
