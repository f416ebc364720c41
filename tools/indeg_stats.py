import sys, numpy as np
sys.path.insert(0, '.')
import paper_2101_03652_b200 as P
g = P.generate_rmat(22, 16, 3)
d = np.bincount(g.out_neighbors(), minlength=g.n())
m = d.sum()
for lo, hi in [(1, 32), (33, 384), (385, 4096), (4097, 1 << 30)]:
    sel = (d >= lo) & (d <= hi)
    print(f"in-degree {lo}-{hi}: rows {sel.sum()} edges {d[sel].sum() / m:.3f}")
