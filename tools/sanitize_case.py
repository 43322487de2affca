"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck):
tiny kernel (gate + state), large path (sequential, history + chunked scans, state-vector),
slice-chunk boundary API, 3M and 4M GEMMs."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_05884_b200 import _lib, parallel, systems  # noqa: E402
from paper_2309_05884_b200.engine import GrapeEngine  # noqa: E402

lib = _lib.load()
s = systems.config(1, n=8, n_slices=6)          # S_n sectors d = 9, 7, 5, 3, 1 (tiny, gate)
GrapeEngine(s, max_batch=3).objective(s.controls(0, batch=3))
s = systems.config(1, n=12, n_slices=4)         # all S_12 sectors, fused kernel + chain-history backward
GrapeEngine(s, max_batch=20).objective(s.controls(0, batch=20))
from paper_2309_05884_b200 import gpu_basis  # noqa: E402

gb = gpu_basis.GpuDnBasis(6)                    # on-GPU D_n basis + compression
gb.blocks()
gb.compress(systems.ring_heisenberg(6))
gb.close()
s = systems.config(0, n_slices=5)               # d = 13 state (tiny)
GrapeEngine(s, max_batch=2).objective(s.controls(0, batch=2))
for mults in (3, 4):
    lib.sqoc_set_complex_gemm(mults)
    g = systems.gate_ring(8, 0.1 * 66, 66)      # mixed tiny + large blocks, N >= 64 -> chunked scans
    for sched in ("sequential", "history"):
        e = GrapeEngine(g, max_batch=1)
        e.set_schedule(sched)
        e.objective(g.controls(1))
    st = systems.state_transfer_ring(6, 0.4, 4, full=True)   # d = 64 state
    for sched in ("sequential", "history", "state-vector"):
        e = GrapeEngine(st, max_batch=1)
        e.set_schedule(sched)
        e.objective(st.controls(2))
lib.sqoc_set_complex_gemm(3)
g = systems.config(2, n_slices=6)
F, grad = parallel.emulate_ranks(g, 2, lambda x: GrapeEngine(x, max_batch=1), g.controls(3))
print("sanitize case ok", F)
