set -x
for c in c1 c2 c3; do python tools/stage_probe.py $c 3 >> gpurun_out/r2e_probe.jsonl; PSG_NO_GRAPH=1 python tools/stage_probe.py $c 2 >> gpurun_out/r2e_probe.jsonl; done
for e in 1024 4096 32768 1000000; do PSG_BOOT_EVALS=$e python tools/stage_probe.py c5 2 >> gpurun_out/r2e_probe.jsonl; done
PSG_NO_GRAPH=1 python tools/stage_probe.py c5 1 >> gpurun_out/r2e_probe.jsonl
