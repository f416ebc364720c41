"""Edge share of the top out-degree nodes (how much of the pull gather a
per-sweep hub stage could serve from shared memory)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_03652_b200 as P  # noqa: E402

g = P.generate_rmat(22, 16, 3)
d = np.sort(np.diff(g.out_offsets()).astype(np.int64))[::-1]
m = d.sum()
for t in (16, 64, 256, 1024, 4096, 16384, 65536):
    print(f"top {t:6d} nodes: {d[:t].sum() / m:.3f} of edges")
