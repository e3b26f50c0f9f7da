for k in 1 2; do
python tools/stage_probe.py c2 5 >> gpurun_out/r2x_probe.jsonl 2>&1
PSG_LIB_PATH=$PWD/tools/dbg/libpairscan_b200_b4.so python tools/stage_probe.py c2 5 >> gpurun_out/r2x_probe.jsonl 2>&1
done
