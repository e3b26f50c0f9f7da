# grid occupancy (mean points per cell) vs C1/C2/C3 device solve times
for occ in 0.15 0.25 0.35; do
  echo "occ=$occ" >> gpurun_out/occ_sweep.log
  PSG_OCC=$occ python tools/bench_configs.py c1 c2 c3 2>/dev/null | cut -c1-160 >> gpurun_out/occ_sweep.log
done
