"""cfg 1 optimisation on the GPU: 4096 seeds, batched device-resident L-BFGS (optim.py)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_05884_b200 import optim, systems  # noqa: E402
from paper_2309_05884_b200.engine import GrapeEngine  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 50
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
s = systems.config(1)
eng = GrapeEngine(s, max_batch=batch)
u0 = torch.from_numpy(s.controls(0, batch=batch)).cuda()
fun = optim.DeviceObjective(eng)
fun(u0)
torch.cuda.synchronize()
t0 = time.perf_counter()
res = optim.lbfgs_maximize(fun, u0, iterations=iters)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
print(json.dumps({"config": "cfg1, 4096 seeds, batched device L-BFGS", "iterations": iters, "batch": batch,
                  "wall_s": wall, "evaluations": res.evaluations,
                  "seed_evals_per_s": res.evaluations * batch / wall,
                  "mean_F_first_last": [res.history[0], res.history[-1]],
                  "min_F_final": float(res.F.min()), "max_F_final": float(res.F.max()),
                  "history_every_10": res.history[::10]}))
