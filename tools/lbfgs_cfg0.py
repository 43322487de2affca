"""BASELINE cfg 0 end to end: one objective+gradient evaluation, then 50 L-BFGS iterations
(scipy L-BFGS-B on the host; every F/grad on the GPU), with the same driver over the CPU
oracle port for comparison.  Prints one JSON line."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_05884_b200 import qoc, systems  # noqa: E402
from paper_2309_05884_b200.engine import GrapeEngine  # noqa: E402


class OracleEngine:
    def __init__(self, s):
        from oracle import grape_oracle

        self.s, self.o = s, grape_oracle

    def objective(self, u):
        F, g, _ = self.o.objective(self.s, u)
        return F, g


import scipy.optimize  # noqa: E402,F401  (imported before the timed regions: qoc imports it lazily)

s = systems.config(0)
u0 = s.controls(0)
out = {"config": "cfg0: n=6 ring, A1 d=13, state transfer, N_t=100; 50 L-BFGS-B iterations"}
for name, eng in (("gpu", GrapeEngine(s, max_batch=1)), ("cpu_oracle_port", OracleEngine(s))):
    eng.objective(u0)  # warm
    t0 = time.perf_counter()
    F0, _ = eng.objective(u0)
    t_eval = time.perf_counter() - t0
    t0 = time.perf_counter()
    res = qoc.optimize_lbfgs(eng, u0, maxiter=50)
    t_opt = time.perf_counter() - t0
    out[name] = {"first_eval_ms": t_eval * 1e3, "F0": float(F0), "lbfgs_wall_s": t_opt,
                 "evaluations": res.evaluations, "iterations": len(res.trace), "F_final": res.trace[-1],
                 "ms_per_eval_in_loop": t_opt / max(1, res.evaluations) * 1e3}
out["F_final_diff"] = abs(out["gpu"]["F_final"] - out["cpu_oracle_port"]["F_final"])
print(json.dumps(out))
