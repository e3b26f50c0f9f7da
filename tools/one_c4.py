"""C4 FRNN count + hash on a resident point set, for profiling."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1407_5609_b200 as psg
R_C4 = float.fromhex("0x1.902ce9269f6dp-7")
cube = psg.gen.uniform(4, 1 << 22, 3)
pc = psg.PointSet.from_flat(cube, 3)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    r = psg.fixed_radius_neighbors(pc, R_C4, 10, 10.0, 1, 0, want_lists=False)
print(r.pair_count, r.pair_hash, psg.last_profile()["stage_list"])
