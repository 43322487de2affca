"""Per-sector device timing of the cfg 1 tiny kernels, each sector launched alone.

python tools/sector_times.py [n_slices] [batch] [dims...]

Prints, per sector d: launch ms (CUDA events, min of 3), problems resident per SM and
SM-ms per problem (launch ms x 148 / batch, i.e. the machine share one problem costs when
the sectors are packed concurrently), and SM-ms per problem / d^3.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2309_05884_b200 import systems
from paper_2309_05884_b200.engine import GrapeEngine

n_sl = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
want = [int(x) for x in sys.argv[3:]]
full = systems.config(1, n_slices=n_sl)
sms = torch.cuda.get_device_properties(0).multi_processor_count
tot = 0.0
for bi, blk in enumerate(full.blocks):
    if want and blk.dim not in want:
        continue
    s = systems.GrapeSystem(f"sector{blk.dim}", full.n_qubits, [blk], "gate", full.T, n_sl, [full.targets[bi]])
    eng = GrapeEngine(s, max_batch=batch)
    # the CTA size the multi-sector step uses (a single-block engine would pick 4-warp CTAs);
    # SECTOR_CTA=auto times the single-block default instead
    if os.environ.get("SECTOR_CTA", "full") == "full":
        eng.set_tiny_cta_warps(0)
    u = torch.from_numpy(s.controls(0, batch=batch)).cuda()
    F = torch.empty(batch, dtype=torch.float64, device="cuda")
    g = torch.empty_like(u)
    eng.evaluate_device(u.data_ptr(), batch, F.data_ptr(), g.data_ptr())
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.evaluate_device(u.data_ptr(), batch, F.data_ptr(), g.data_ptr())
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    smms = ms * sms / batch
    tot += smms * batch / sms
    print(f"d={blk.dim:2d}: {ms:8.3f} ms  SM-ms/problem {smms:.4f}  per d^3 {smms / blk.dim ** 3 * 1e3:.3f}e-3  "
          f"hist={eng.last_tiny_history}", flush=True)
    eng.close()
    del eng
    torch.cuda.empty_cache()
print(f"packed estimate (sum of SM-ms / {sms} SMs): {tot:.2f} ms")
