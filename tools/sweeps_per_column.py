import sys, os, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2101_03652_b200 as P
g = P.generate_rmat(22, 16, 3)
s = P.sample_sources(np.diff(g.out_offsets()), 256, 3)
outs, cs = P.power_push_batch(g, s[:64], 0.2, 1e-8, keep=False)
sw = sorted(o.sweeps for o in outs)
print("sweeps per column:", sw)
print("levels", sorted(o.local_levels for o in outs)[:5], "max_sweeps", cs.max_sweeps)
