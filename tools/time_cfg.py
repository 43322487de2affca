"""Quick device timing of one config through the C ABI (device pointers)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2309_05884_b200 import systems
from paper_2309_05884_b200.engine import GrapeEngine

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
batch = int(sys.argv[2]) if len(sys.argv) > 2 else systems.CONFIG_BATCH[cfg]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
kw = {"n_slices": int(sys.argv[4])} if len(sys.argv) > 4 else {}
s = systems.config(cfg, **kw)
eng = GrapeEngine(s, max_batch=batch)
if len(sys.argv) > 5:
    eng.set_schedule(sys.argv[5])
u = torch.from_numpy(s.controls(0, batch=batch)).cuda()
F = torch.empty(batch, dtype=torch.float64, device="cuda")
g = torch.empty_like(u)
eng.evaluate_device(u.data_ptr(), batch, F.data_ptr(), g.data_ptr())
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); eng.evaluate_device(u.data_ptr(), batch, F.data_ptr(), g.data_ptr()); e1.record()
    torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
ms = min(ts)
fl = s.flops_per_eval() * batch
print(f"cfg{cfg} batch={batch} dims={[b.dim for b in s.blocks]}: {ms:.3f} ms/eval-batch, {batch/ms*1e3:.1f} evals/s, "
      f"{fl/ms/1e9:.2f} TFLOP/s (G-convention), launches={eng.last_launches}, F[0]={F[0].item():.6f}, "
      f"schedule={eng.last_schedule}, plan={eng.last_plan}")
