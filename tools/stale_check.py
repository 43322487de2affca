"""Does an evaluation on the large path depend on what the previous evaluation left in the workspaces?
Engine A evaluates u1 and then u2; engine B evaluates u2 twice (the repeat is the steady-state value).
A's u2 result must equal B's bit for bit.

python tools/stale_check.py [n_slices] [trials]
"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2309_05884_b200 import systems  # noqa: E402
from paper_2309_05884_b200.engine import GrapeEngine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
trials = int(sys.argv[2]) if len(sys.argv) > 2 else 8
s = systems.config(3, n_slices=n, builder="gpu")
u1, u2 = s.controls(9), s.controls(10)
res = []
for t in range(trials):
    a = GrapeEngine(s, max_batch=1)
    a.set_schedule("sequential")
    a.objective(u1)
    Fa, ga = a.objective(u2)
    a.close()
    b = GrapeEngine(s, max_batch=1)
    b.set_schedule("sequential")
    Fb1, gb1 = b.objective(u2)
    Fb2, gb2 = b.objective(u2)
    b.close()
    sc = np.abs(gb2).max()
    res.append({"after_other_u": float(np.abs(np.array(ga) - np.array(gb2)).max() / sc),
                "first_vs_repeat": float(np.abs(np.array(gb1) - np.array(gb2)).max() / sc)})
print(json.dumps({"n_slices": n, "trials": res}))
