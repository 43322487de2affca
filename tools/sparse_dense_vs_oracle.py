"""cfg 3 blocks on a short grid: the sequential schedule with and without the sparse-generator kernels
(SQOC_SPARSE) against the CPU oracle -- which side moves when the two disagree.

python tools/sparse_dense_vs_oracle.py [n_slices]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import grape_oracle  # noqa: E402
from paper_2309_05884_b200 import systems  # noqa: E402
from paper_2309_05884_b200.engine import GrapeEngine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
s = systems.config(3, n_slices=n, builder="gpu")
u = s.controls(9)
out = {}
for flag in ("0", "1"):
    os.environ["SQOC_SPARSE"] = flag
    eng = GrapeEngine(s, max_batch=1)
    eng.set_schedule("sequential")
    out[flag] = eng.objective(u)
    eng.close()
rel = lambda a, b: float(np.abs(a - b).max() / np.abs(b).max())  # noqa: E731
if os.environ.get("SKIP_ORACLE"):
    print(json.dumps({"n_slices": n, "dense_vs_sparse": [abs(float(out["0"][0]) - float(out["1"][0])),
                                                         rel(out["0"][1], out["1"][1])],
                      "per_slice": (np.abs(out["0"][1] - out["1"][1]).max(0) / np.abs(out["1"][1]).max()).tolist()}))
    sys.exit(0)
Fo, go, _ = grape_oracle.objective(s, u)
print(json.dumps({"n_slices": n, "dense_vs_oracle": [abs(float(out["0"][0]) - Fo), rel(out["0"][1], go)],
                  "sparse_vs_oracle": [abs(float(out["1"][0]) - Fo), rel(out["1"][1], go)],
                  "dense_vs_sparse": [abs(float(out["0"][0]) - float(out["1"][0])), rel(out["0"][1], out["1"][1])]}))
