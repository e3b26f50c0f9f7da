timeout 900 python -m pytest tests -q -m gpu -x -k "sharded" 2>&1 | tail -3 > gpurun_out/r2u_suite.log
PSG_BENCH_GLOO=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/r2u_bench2.json 2> gpurun_out/r2u_bench2.err
cat gpurun_out/r2u_suite.log; python -c "import json;d=json.loads(open('gpurun_out/r2u_bench2.json').read().strip().splitlines()[-1]);print(d['correct'], d['ms_per_step'], d['c5_scaling'])"
