"""Host restatement vs on-GPU D_n basis + compression wall times.

python tools/basis_times.py [n ...]   -> one JSON line per n
"""
import json
import sys
import time

sys.path.insert(0, ".")
from paper_2309_05884_b200 import gpu_basis, pauli, symmetry, systems

for n in [int(a) for a in sys.argv[1:]] or [10, 12, 14]:
    ops = (systems.ring_heisenberg(n), *systems.global_controls(n))
    t0 = time.perf_counter()
    host = symmetry.dn_full_basis(n)
    t1 = time.perf_counter()
    full = [pauli.realize(o) for o in ops]
    hm = [[systems.hermitian_part(b.compress(f)) for b in host] for f in full]
    t2 = time.perf_counter()
    gpu_basis.GpuDnBasis(3).close()  # CUDA context / library warm-up
    t3 = time.perf_counter()
    gb = gpu_basis.GpuDnBasis(n)
    t4 = time.perf_counter()
    gm = [gb.compress(o) for o in ops]
    t5 = time.perf_counter()
    blocks = gb.blocks()
    t6 = time.perf_counter()
    err = max(abs(systems.hermitian_part(g) - h).max() for gl, hl in zip(gm, hm) for g, h in zip(gl, hl))
    same = [b.keys for b in blocks] == [b.keys for b in host]
    gb.close()
    print(json.dumps({"n": n, "dims": [b.dim for b in host], "host_basis_s": round(t1 - t0, 3),
                      "host_compress_s": round(t2 - t1, 3), "gpu_basis_s": round(t4 - t3, 4),
                      "gpu_compress_s": round(t5 - t4, 4), "gpu_export_columns_s": round(t6 - t5, 3),
                      "same_column_order": same, "max_abs_diff_generators": float(err)}), flush=True)
