"""One SpeedPPR batch (configs[3] shape) for a kernel launch list under ncu.

ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/spp_launches.csv python tools/profile_speedppr.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_03652_b200 as P  # noqa: E402

scale = int(os.environ.get("SPP_LOG2N", "22"))
n = 1 << scale
g = P.generate_chung_lu(n, 146 * n // 4, 4)
s = P.sample_sources(np.diff(g.out_offsets()), 64, 4)
idx = P.build_index(g, 0.2, 4)
for _ in range(int(os.environ.get("SPP_REPS", "1"))):
    outs, cs = P.speedppr_batch(g, s, P.QueryConfig(epsilon=0.5, seed=4), idx, keep=False)
    print("device_ms", cs.device_ms, "local", cs.local_ms, "sweep", cs.sweep_ms, "final", cs.final_ms,
          "walks", np.mean([o.walks for o in outs]), "dead", len(g.dead_ends()), "max_sweeps", cs.max_sweeps,
          "sweeps", [o.sweeps for o in outs][:16], "levels", [o.local_levels for o in outs][:16])
