"""Writes an R-MAT transpose for the gather-engine probes (default the configs[2]
graph, R-MAT 22/16 seed 3; `dump_transpose.py FILE SCALE EF SEED` for others):
u64 n, u64 m, u64 in_off[n+1], u32 in_nbr[m] (design probe, not product)."""
import sys
import numpy as np
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(
    __import__("os").path.dirname(__import__("os").path.abspath(__file__)))))
import paper_2101_03652_b200 as P

args = sys.argv[2:5]
scale, ef, seed = (int(a) for a in args) if len(args) == 3 else (22, 16, 3)
g = P.generate_rmat(scale, ef, seed)
off, nbr = g.transpose()
with open(sys.argv[1] if len(sys.argv) > 1 else "/tmp/transpose.bin", "wb") as f:
    np.array([g.n(), g.m()], np.uint64).tofile(f)
    np.asarray(off, np.uint64).tofile(f)
    np.asarray(nbr, np.uint32).tofile(f)
print("wrote", g.n(), g.m())
