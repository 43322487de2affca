"""Device timing of one large-block config with the per-GEMM event accounting (sqoc_last_gemm_stats).

python tools/gemm_stats.py CFG N_SLICES [schedule] [reps]
Prints step ms, GEMM ms (sum of per-launch event pairs), GEMM units per slice (complex MACs / sum d^3 / N),
the convention frac (8 N G sum d^3 / step / 36.9 TF) and the executed-DMMA pipe fraction.
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2309_05884_b200 import systems  # noqa: E402
from paper_2309_05884_b200.engine import GrapeEngine  # noqa: E402

PEAK = 36.9
cfg = int(sys.argv[1])
n_sl = int(sys.argv[2])
sched = sys.argv[3] if len(sys.argv) > 3 else "auto"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
s = systems.config(cfg, n_slices=n_sl, builder="gpu") if cfg in (2, 3) else systems.config(cfg, n_slices=n_sl)
eng = GrapeEngine(s)
eng.set_schedule(sched)
u = torch.from_numpy(s.controls(0)).cuda()
F = torch.empty(1, dtype=torch.float64, device="cuda")
g = torch.empty_like(u)
st = torch.cuda.current_stream()
eng.evaluate_device(u.data_ptr(), 1, F.data_ptr(), g.data_ptr(), stream=st.cuda_stream)
eng.set_timing(True)
ts, gs = [], []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    eng.evaluate_device(u.data_ptr(), 1, F.data_ptr(), g.data_ptr(), stream=st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
    gs.append(eng.gemm_stats())
ms = float(np.median(ts))
gst = gs[-1]
sd3 = sum(float(b.dim) ** 3 for b in s.blocks)
G = 22 if s.objective == "gate" else 8
conv = 8.0 * n_sl * G * sd3
execd = 2.0 * gst["real_fma_per_complex_mac"] * gst["complex_macs"]
print(json.dumps({
    "cfg": cfg, "n_slices": n_sl, "schedule": eng.last_schedule, "plan": eng.last_plan, "step_ms": ms,
    "gemm_ms": gst["ms"], "gemm_launches": gst["launches"], "units_per_slice": gst["complex_macs"] / sd3 / n_sl,
    "frac_convention_step": conv / (ms / 1e3) / 1e12 / PEAK,
    "frac_convention_gemm": conv / (gst["ms"] / 1e3) / 1e12 / PEAK,
    "dmma_pipe_frac_gemm": execd / (gst["ms"] / 1e3) / 1e12 / PEAK,
    "F": F.item(), "steps_ms": ts}))
