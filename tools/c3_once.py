import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, paper_1407_5609_b200 as psg
s, _ = psg.gen.walk_motif(3, 1 << 20, 256)
s64 = s.astype(np.float64)
for _ in range(2):
    m = psg.motif(s64, 256)
print(m)
