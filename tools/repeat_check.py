"""Bit-identity of repeated evaluations on the large path (cfg 3 blocks, short grid, sequential schedule):
REPS evaluations in fresh engines, with and without the sparse-generator kernels.

python tools/repeat_check.py [n_slices] [reps]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2309_05884_b200 import systems  # noqa: E402
from paper_2309_05884_b200.engine import GrapeEngine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
s = systems.config(3, n_slices=n, builder="gpu")
u = s.controls(9)
for flag in os.environ.get("REPEAT_MODES", "1,0").split(","):
    os.environ["SQOC_SPARSE"] = flag
    outs = []
    for r in range(reps):
        eng = GrapeEngine(s, max_batch=1)
        eng.set_schedule("sequential")
        F, g = eng.objective(u)
        F2, g2 = eng.objective(u)  # second call on the same engine
        outs += [(float(F), np.array(g)), (float(F2), np.array(g2))]
        eng.close()
    F0, g0 = outs[0]
    dF = [abs(F - F0) for F, _ in outs]
    dg = [float(np.abs(g - g0).max() / np.abs(g0).max()) for _, g in outs]
    print(json.dumps({"sparse": flag, "n_slices": n, "evaluations": len(outs), "max_abs_dF": max(dF),
                      "max_rel_dgrad": max(dg), "blips": [i for i, x in enumerate(dg) if x > 1e-15],
                      "dgrad": dg if len(dg) <= 12 else None}))
