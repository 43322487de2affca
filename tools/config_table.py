"""Per-config device timing table (all five BASELINE configs) -> JSON lines.

python tools/config_table.py [cfg ...]   (run on the GPU box; CPU baselines from bench.cpu_reference)
Timing: CUDA events on the caller's stream around sqoc_eval (device pointers), after warm-up.
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2309_05884_b200 import systems  # noqa: E402
from paper_2309_05884_b200.engine import GrapeEngine  # noqa: E402

CASES = {
    "0": dict(cfg=0, batch=1, reps=20, warm=3),
    "0b": dict(cfg=0, batch=4096, reps=3, warm=2),
    "1": dict(cfg=1, batch=4096, reps=3, warm=2),
    "2": dict(cfg=2, batch=1, reps=5, warm=2),
    "3": dict(cfg=3, batch=1, reps=1, warm=0),
    "4": dict(cfg=4, batch=1, reps=1, warm=1),
    "4a1": dict(cfg=4, batch=1, reps=5, warm=2, full=False),
}


def run(name, cfg, batch, reps, warm, full=True, cpu=True):
    kw = {} if full else {"full": False}
    s = systems.config(cfg, **kw)
    t0 = time.time()
    eng = GrapeEngine(s, max_batch=batch)
    setup = time.time() - t0
    u = torch.from_numpy(s.controls(0, batch=batch)).cuda()
    F = torch.empty(batch, dtype=torch.float64, device="cuda")
    g = torch.empty_like(u)
    for _ in range(max(warm, 1) if reps > 1 else warm):
        eng.evaluate_device(u.data_ptr(), batch, F.data_ptr(), g.data_ptr())
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.evaluate_device(u.data_ptr(), batch, F.data_ptr(), g.data_ptr())
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    flops = s.flops_per_eval() * batch
    row = {
        "case": name, "config": bench.CONFIG_NAMES[cfg] + ("" if full else " [A1 block d=224]"),
        "blocks": [b.dim for b in s.blocks], "batch": batch, "ms_per_eval_batch": ms,
        "evals_per_s": batch / ms * 1e3, "tflops_convention": flops / ms / 1e9,
        "frac_of_fp64_peak": flops / ms / 1e9 / bench.FP64_PEAK_TFLOPS, "schedule": eng.last_schedule,
        "plan": eng.last_plan if eng.large_blocks else None, "launches": eng.last_launches, "setup_s": setup,
        "F0": float(F[0].item()),
    }
    eng.close()
    if cpu and full:
        v, cores, sample = bench.cpu_reference(cfg, seconds_budget=10.0)
        row["cpu_evals_per_s"] = v
        row["cpu_cores"] = cores
        row["cpu_sample"] = sample
        row["speedup_vs_cpu"] = row["evals_per_s"] / v
    print(json.dumps(row), flush=True)


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        run(n, **CASES[n])
