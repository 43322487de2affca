"""A/B of the large-path GEMM operand staging (sqoc_set_gemm_staging: 0 per-tile cp.async kernel, 1 persistent warp-specialised TMA kernel)
on the same GPU: device ms per slice of GEMM work and the F / gradient deltas
against cp.async.  Prints one JSON line per (workload, mode)."""

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_05884_b200 import _lib, systems  # noqa: E402
from paper_2309_05884_b200.engine import GrapeEngine  # noqa: E402


def run(name, s, sched, modes, reps=2):
    lib = _lib.load()
    u = s.controls(4)
    ref = None
    for mode in modes:
        assert lib.sqoc_set_gemm_staging(mode) == 0
        eng = GrapeEngine(s, max_batch=1)
        eng.set_schedule(sched)
        eng.objective(u)
        eng.set_timing(True)
        ms, gms = [], []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            F, g = eng.objective(u)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
            gms.append(eng.gemm_stats())
        eng.close()
        if ref is None:
            ref = (F, g)
        st = gms[-1]
        print(json.dumps({"workload": name, "mode": mode, "ms": float(np.median(ms)),
                          "ms_per_slice": float(np.median(ms)) / s.n_slices, "gemm_ms": st["ms"],
                          "launches": st["launches"],
                          "executed_dmma_frac": 2 * 3 * st["complex_macs"] / (st["ms"] / 1e3) / 1e12 / 36.9,
                          "dF": abs(F - ref[0]), "dg_rel": float(np.abs(g - ref[1]).max() / np.abs(ref[1]).max())}),
              flush=True)
    lib.sqoc_set_gemm_staging(1)


if __name__ == "__main__":
    modes = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "0,1").split(",")]
    which = sys.argv[2] if len(sys.argv) > 2 else "3,2,4"
    tag = os.environ.get("SQOC_PT_VARIANT", "")
    if "3" in which:
        run(f"cfg3 N=6 sequential {tag}", systems.config(3, n_slices=6, builder="gpu"), "sequential", modes)
    if "2" in which:
        run(f"cfg2 N=500 history {tag}", systems.config(2, builder="gpu"), "auto", modes)
    if "4" in which:
        run(f"cfg4 full N=4 state-vector {tag}", systems.config(4, n_slices=4, full=True), "state-vector", modes)
