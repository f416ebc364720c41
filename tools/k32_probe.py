"""One 32-source block on the configs[2] graph (what each rank runs under
bench.py --gpus 8): device ms and sweeps, for A/B under PPRG_* env."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_03652_b200 as P  # noqa: E402

g = P.generate_rmat(22, 16, 3)
s = P.sample_sources(np.diff(g.out_offsets()), 256, 3)[:32]
P.power_push_batch(g, s, 0.2, 1e-8, keep=False)
outs, cs = P.power_push_batch(g, s, 0.2, 1e-8, keep=False)
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("PPRG_")},
                  "device_ms": cs.device_ms, "sweep_ms": cs.sweep_ms, "sweeps": cs.max_sweeps,
                  "r_sum_max": max(o.achieved_r_sum for o in outs)}))
