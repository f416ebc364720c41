"""One 64-source block of configs[2] under different epoch counts and local-phase
queue limits (A/B helper for the delta sweeps): device / local / sweep ms, sweeps."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_03652_b200 as P  # noqa: E402

g = P.generate_rmat(22, 16, 3)
n = g.n()
s = P.sample_sources(np.diff(g.out_offsets()), 256, 3)[:64]
P.power_push_batch(g, s, 0.2, 1e-8, keep=False)
for epochs, div in [(8, 4), (1, 4), (2, 4), (4, 4), (16, 4), (8, 8), (8, 16), (8, 32), (8, 128), (8, 1024)]:
    outs, cs = P.power_push_batch(g, s, 0.2, 1e-8, epoch_num=epochs, scan_threshold=n // div, keep=False)
    print(json.dumps({"epochs": epochs, "scan_threshold": f"n/{div}", "device_ms": round(cs.device_ms, 2),
                      "local_ms": round(cs.local_ms, 2), "sweep_ms": round(cs.sweep_ms, 2),
                      "sweeps": cs.max_sweeps, "r_sum_max": max(o.achieved_r_sum for o in outs)}))
