"""Device time of the GPU fidelity replay (trotter.cu) per step at several n, and of the fused
multi-step apply; CUDA events on the launching stream; prints JSON lines."""

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_05884_b200 import trotter  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
    for n in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "6,8,10,11,12").split(",")]:
        cfg = trotter.TrotterModel(n, 1.0, (0.2,))
        bx, by = trotter.benchmark_controls(cfg, steps, 0.05)
        plan = trotter.PerQubitPlan(cfg, 0.05)
        bxd, byd = torch.as_tensor(bx).cuda(), torch.as_tensor(by).cuda()
        fids = torch.empty(steps, dtype=torch.float64, device="cuda")
        st = torch.cuda.current_stream()
        plan.replay_device(bxd.data_ptr(), byd.data_ptr(), min(steps, 50), 1, fids.data_ptr(), st.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        plan.replay_device(bxd.data_ptr(), byd.data_ptr(), steps, 100, fids.data_ptr(), st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        dim = 1 << n
        print(json.dumps({"n": n, "steps": steps, "replay_ms": ms, "us_per_step": 1e3 * ms / steps,
                          "launches": plan.last_launches,
                          "algorithmic_GBps": 4 * dim * dim * 16 * steps / (ms / 1e3) / 1e9}), flush=True)
        plan.close()


if __name__ == "__main__":
    main()
