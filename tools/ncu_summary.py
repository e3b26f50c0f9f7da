"""Summarise an ncu report (details page) into a few lines per kernel."""
import csv, subprocess, sys
want = ('Duration', 'Memory Throughput', 'DRAM Throughput', 'L1/TEX Hit Rate', 'L2 Hit Rate', 'Achieved Occupancy',
        'Theoretical Occupancy', 'Registers Per Thread', 'Issued Ipc Active', 'Warp Cycles Per Issued Instruction',
        'Executed Instructions', 'Avg. Active Threads Per Warp', 'Branch Efficiency', 'L1/TEX Cache Throughput',
        'L2 Cache Throughput', 'Compute (SM) Throughput', 'Block Limit Registers', 'Block Limit Shared Mem')
out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'details', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
K, M, U, V = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Unit'), h.index('Metric Value')
I = h.index('ID')
cur = None
for r in rows[1:]:
    if len(r) <= V:
        continue
    if r[M] in want:
        key = (r[I], r[K][:70])
        if key != cur:
            print('==', key[0], key[1]); cur = key
        print(f'   {r[M]:40s} {r[V]} {r[U]}')
