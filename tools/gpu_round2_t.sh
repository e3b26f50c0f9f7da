PSG_BENCH_GLOO=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/r2t_bench2.json 2> gpurun_out/r2t_bench2.err
timeout 900 python -m pytest tests -q -m gpu -x -k "dense or c5 or ties or fullsize or parity" 2>&1 | tail -3 > gpurun_out/r2t_suite.log
cat gpurun_out/r2t_suite.log; tail -c 1500 gpurun_out/r2t_bench2.json
