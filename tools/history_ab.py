"""Same-box A/B of the fused tiny kernel's HBM histories on the cfg 1 step.

python tools/history_ab.py [reps]
For each history mode (none / x / chain / auto) times the whole cfg 1 evaluation (4096 seeds, N_t=1000)
with CUDA events, and reports the device memory the histories reserve (torch.cuda.mem_get_info before /
after the first evaluation).  Modes are interleaved over `reps` rounds so clock drift hits all alike.
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2309_05884_b200 import systems  # noqa: E402
from paper_2309_05884_b200.engine import GrapeEngine  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
s = systems.config(1)
batch = systems.CONFIG_BATCH[1]
u = torch.from_numpy(s.controls(0, batch=batch)).cuda()
F = torch.empty(batch, dtype=torch.float64, device="cuda")
g = torch.empty_like(u)
modes = ["off", "x", "chain", "auto"]
res = {m: {"ms": []} for m in modes}
engines = {}
for m in modes:
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    eng = GrapeEngine(s, max_batch=batch)
    eng.set_tiny_history(m)
    eng.evaluate_device(u.data_ptr(), batch, F.data_ptr(), g.data_ptr())
    torch.cuda.synchronize()
    res[m]["reserved_gb"] = (free0 - torch.cuda.mem_get_info()[0]) / 1e9
    res[m]["used"] = eng.last_tiny_history
    res[m]["F0"] = F[0].item()
    res[m]["g_ref"] = g[:2].clone()
    eng.close()
for r in range(reps):
    for m in modes:
        eng = GrapeEngine(s, max_batch=batch)
        eng.set_tiny_history(m)
        eng.evaluate_device(u.data_ptr(), batch, F.data_ptr(), g.data_ptr())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.evaluate_device(u.data_ptr(), batch, F.data_ptr(), g.data_ptr())
        e1.record()
        torch.cuda.synchronize()
        res[m]["ms"].append(e0.elapsed_time(e1))
        eng.close()
refs = {m: res[m].pop("g_ref") for m in modes}
for m in modes:
    res[m]["max_dgrad_vs_off_rows01"] = float((refs[m] - refs["off"]).abs().max())
    res[m]["median_ms"] = float(np.median(res[m]["ms"]))
print(json.dumps(res))
