"""Host-side owner of one GRAPE problem on the GPU (wraps sqoc_create / sqoc_eval).

``GrapeEngine(system).objective(u) -> (F, grad)`` is the BASELINE API; the
reference-shaped ``qoc.gradient`` adapter is in ``qoc.py``.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


def spectral_norm_bound(h: np.ndarray) -> float:
    """Upper bound of ||H||_2 for a Hermitian generator (host setup, not the hot path).

    Dense eigvalsh up to d = 2048, Lanczos (ARPACK, largest magnitude) above; a
    relative margin of 1e-6 covers the iteration tolerance.
    """
    h = np.asarray(h)
    if h.shape[0] <= 2048:  # dense tridiagonalisation: 0.25 s at d = 1161 against 0.4-0.8 s for Lanczos
        return float(np.abs(np.linalg.eigvalsh(h)).max()) * (1 + 1e-12) + 1e-300
    from scipy.sparse.linalg import eigsh

    lam = eigsh(h, k=1, which="LM", return_eigenvectors=False, tol=1e-10)
    return float(np.abs(lam).max()) * (1 + 1e-6)


def block_norm_bounds(blk) -> tuple:
    """(||H0||_2, ||H_1||_2, ...) bounds of one block, computed once and kept on the block object
    (the engines of sharded ranks and of the correctness gate share the system's blocks)."""
    cached = getattr(blk, "_sqoc_norm_bounds", None)
    if cached is None:
        cached = tuple(spectral_norm_bound(m) for m in (blk.h0, *blk.hk))
        try:
            blk._sqoc_norm_bounds = cached
        except AttributeError:
            pass
    return cached


def _cplx(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex128))


class GrapeEngine:
    """Device-resident generators/targets of a ``systems.GrapeSystem``-like object.

    Required attributes of ``system``: ``blocks`` (each with ``h0``, ``hk``),
    ``objective`` ('gate'|'state'), ``targets``, ``initial`` (state), ``dt``,
    ``n_slices``, and optionally ``block_weights()``.
    """

    def __init__(self, system, max_batch: int = 1, device: int = 0, spectral_bounds: bool = True):
        self.lib = _lib.load()
        self.system = system
        self.K = len(system.blocks[0].hk)
        self.N = int(system.n_slices)
        self.nblocks = len(system.blocks)
        self.max_batch = int(max_batch)
        self.device = device
        gate = system.objective == "gate"
        dims = [int(b.h0.shape[0]) for b in system.blocks]
        self.dims = dims
        keep = []

        def dptr(arr):
            arr = np.ascontiguousarray(arr)
            keep.append(arr)
            return arr.ctypes.data_as(ctypes.POINTER(ctypes.c_double))

        h0 = (ctypes.POINTER(ctypes.c_double) * self.nblocks)()
        hk = (ctypes.POINTER(ctypes.c_double) * self.nblocks)()
        tg = (ctypes.POINTER(ctypes.c_double) * self.nblocks)()
        ini = (ctypes.POINTER(ctypes.c_double) * self.nblocks)()
        for b, blk in enumerate(system.blocks):
            d = dims[b]
            if len(blk.hk) != self.K:
                raise ValueError("all blocks need the same number of controls")
            h0[b] = dptr(_cplx(blk.h0).view(np.float64))
            hk[b] = dptr(np.concatenate([_cplx(h).reshape(-1) for h in blk.hk]).view(np.float64))
            t = _cplx(system.targets[b])
            if t.shape != ((d, d) if gate else (d,)):
                raise ValueError(f"target of block {b} has shape {t.shape}")
            tg[b] = dptr(t.view(np.float64))
            if not gate:
                ini[b] = dptr(_cplx(system.initial[b]).view(np.float64))
        w = getattr(system, "block_weights", None)
        weights = None if w is None else np.ascontiguousarray(w(), dtype=np.float64)
        dims_arr = (ctypes.c_int * self.nblocks)(*dims)
        handle = ctypes.c_void_p()
        rc = self.lib.sqoc_create(
            ctypes.byref(handle), device, self.nblocks, dims_arr, self.K, h0, hk,
            _lib.OBJ_GATE if gate else _lib.OBJ_STATE, None if gate else ini, tg,
            None if weights is None else weights.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
            self.N, float(system.dt), self.max_batch,
        )
        _lib.check(rc, "sqoc_create")
        self.handle = handle
        if spectral_bounds and max(dims) > self.lib.sqoc_tiny_max_dim():
            bounds = np.array([block_norm_bounds(blk) for blk in system.blocks])
            _lib.check(self.lib.sqoc_set_norm_bounds(self.handle, np.ascontiguousarray(bounds).ctypes.data_as(
                ctypes.POINTER(ctypes.c_double))), "sqoc_set_norm_bounds")

    def close(self):
        if getattr(self, "handle", None):
            self.lib.sqoc_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def large_blocks(self) -> list:
        tiny_max = self.lib.sqoc_tiny_max_dim()
        return [b for b, d in enumerate(self.dims) if d > tiny_max]

    SCHEDULES = {"auto": -1, "sequential": 0, "history": 1, "state-vector": 2, "matrix-free": 3}

    def set_schedule(self, name: str) -> None:
        """Large-block schedule: 'auto', 'sequential' (O(sum d^2) memory) or 'history' (slice-batched)."""
        _lib.check(self.lib.sqoc_set_schedule(self.handle, self.SCHEDULES[name]), "sqoc_set_schedule")

    @property
    def last_schedule(self) -> str:
        return {-1: "none", 0: "sequential", 1: "history", 2: "state-vector", 3: "matrix-free"}[
            self.lib.sqoc_last_schedule(self.handle)]

    TINY_SCHEDULES = {"auto": -1, "fused": 0, "slice-parallel": 1}

    def set_tiny_schedule(self, name: str) -> None:
        """Tiny blocks: 'auto', 'fused' (throughput) or 'slice-parallel' (latency)."""
        _lib.check(self.lib.sqoc_set_tiny_schedule(self.handle, self.TINY_SCHEDULES[name]), "sqoc_set_tiny_schedule")

    @property
    def last_tiny_schedule(self) -> str:
        return {-1: "none", 0: "fused", 1: "slice-parallel"}[self.lib.sqoc_last_tiny_schedule(self.handle)]

    TINY_HISTORY = {"auto": -1, "off": 0, "x": 1, "on": 1, "chain": 2}

    def set_tiny_history(self, mode: str) -> None:
        """Fused tiny schedule histories: 'auto', 'off' (recompute), 'x' (X_{j-1} per slice) or
        'chain' (X and the propagator chain per slice)."""
        _lib.check(self.lib.sqoc_set_tiny_history(self.handle, self.TINY_HISTORY[mode]), "sqoc_set_tiny_history")

    def set_tiny_cta_warps(self, warps: int) -> None:
        """Fused tiny kernel warps per CTA: -1 auto, 0 full (one CTA per SM), > 0 a cap."""
        _lib.check(self.lib.sqoc_set_tiny_cta_warps(self.handle, int(warps)), "sqoc_set_tiny_cta_warps")

    @property
    def last_tiny_history(self) -> str:
        return {-1: "none", 0: "off", 1: "x", 2: "chain"}[self.lib.sqoc_last_tiny_history(self.handle)]

    @property
    def last_plan(self) -> dict:
        nb, s, m = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _lib.check(self.lib.sqoc_last_plan(self.handle, ctypes.byref(nb), ctypes.byref(s), ctypes.byref(m)),
                   "sqoc_last_plan")
        return {"taylor_degree": nb.value, "squarings": s.value, "action_terms": m.value}

    def set_timing(self, on: bool) -> None:
        _lib.check(self.lib.sqoc_set_timing(self.handle, 1 if on else 0), "sqoc_set_timing")

    def block_times_ms(self) -> list:
        """Device time of each block's work in the last evaluation (needs set_timing(True))."""
        out = []
        for b in range(self.nblocks):
            ms = ctypes.c_double()
            _lib.check(self.lib.sqoc_block_time_ms(self.handle, b, ctypes.byref(ms)), "sqoc_block_time_ms")
            out.append(ms.value)
        return out

    def gemm_stats(self) -> dict:
        """Large-block GEMMs of the last evaluation: device ms (needs set_timing(True)), complex
        MACs issued, launches, and the real FMAs per complex MAC of the GEMM algorithm (3M / 4M)."""
        ms, macs, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
        _lib.check(self.lib.sqoc_last_gemm_stats(self.handle, ctypes.byref(ms), ctypes.byref(macs), ctypes.byref(n)),
                   "sqoc_last_gemm_stats")
        return {"ms": ms.value, "complex_macs": macs.value, "launches": n.value,
                "real_fma_per_complex_mac": self.lib.sqoc_complex_gemm_mults()}

    @property
    def last_launches(self) -> int:
        return self.lib.sqoc_last_launch_count(self.handle)

    def evaluate(self, u, want_tau: bool = False):
        """Host arrays in/out. u: (K, N) or (B, K, N). Returns F, grad (, tau)."""
        u = np.ascontiguousarray(np.asarray(u, dtype=np.float64))
        single = u.ndim == 2
        ub = u[None] if single else u
        if ub.shape[1:] != (self.K, self.N):
            raise ValueError(f"u must have shape (B, {self.K}, {self.N}), got {u.shape}")
        if not np.all(np.isfinite(ub)):
            raise ValueError("control samples must be finite")
        B = ub.shape[0]
        F = np.empty(B)
        grad = np.empty_like(ub)
        tau = np.empty((B, self.nblocks), dtype=np.complex128)
        rc = self.lib.sqoc_eval(self.handle, ub.ctypes.data, B, F.ctypes.data, grad.ctypes.data,
                                tau.ctypes.data, _lib.MEM_HOST, None)
        _lib.check(rc, "sqoc_eval")
        if single:
            F, grad, tau = F[0], grad[0], tau[0]
        return (F, grad, tau) if want_tau else (F, grad)

    def objective(self, u):
        """objective(u) -> (F, grad): the BASELINE host API."""
        return self.evaluate(u)

    # ---- slice-chunk sharding (parallel.py): torch tensors on this device ----
    @property
    def torch_device(self):
        import torch

        return torch.device("cuda", self.device)

    def objective_t(self, u_t):
        """Ordinary evaluation on device tensors: u_t (K, N) -> (F (1,), grad (K, N)) on this device."""
        import torch

        u_t = u_t.to(self.torch_device, torch.float64).contiguous()
        F = torch.empty(1, dtype=torch.float64, device=self.torch_device)
        grad = torch.empty_like(u_t)
        st = torch.cuda.current_stream(self.torch_device).cuda_stream
        self.evaluate_device(u_t.data_ptr(), 1, F.data_ptr(), grad.data_ptr(), stream=st)
        return F, grad

    def chunk_size(self) -> int:
        """Doubles in one packed chunk product (sum_b 2 d_b^2)."""
        n = ctypes.c_longlong()
        _lib.check(self.lib.sqoc_chunk_size(self.handle, ctypes.byref(n)), "sqoc_chunk_size")
        return n.value

    def chunk_forward_t(self, u_t):
        """Packed U_{N-1} ... U_0 of every block (float64 [2 sum d^2] on this device) for this problem's
        slices; u_t (K, N) float64 on this device.  Runs on torch's current stream."""
        import torch

        u_t = u_t.to(self.torch_device, torch.float64).contiguous()
        out = torch.empty(self.chunk_size(), dtype=torch.float64, device=self.torch_device)
        st = torch.cuda.current_stream(self.torch_device).cuda_stream
        _lib.check(self.lib.sqoc_chunk_forward(self.handle, u_t.data_ptr(), out.data_ptr(), _lib.MEM_DEVICE,
                                               st or None), "sqoc_chunk_forward")
        return out

    def chunk_backward_t(self, u_t, gathered, n_chunks: int, chunk: int):
        """(F (1,), grad (K, N_local)) device tensors of this chunk from the gathered products
        [n_chunks, 2 sum d^2] (boundary values formed on the device)."""
        import torch

        u_t = u_t.to(self.torch_device, torch.float64).contiguous()
        gathered = gathered.contiguous()
        F = torch.empty(1, dtype=torch.float64, device=self.torch_device)
        grad = torch.empty_like(u_t)
        st = torch.cuda.current_stream(self.torch_device).cuda_stream
        _lib.check(self.lib.sqoc_chunk_backward(self.handle, u_t.data_ptr(), gathered.data_ptr(), int(n_chunks),
                                                int(chunk), F.data_ptr(), grad.data_ptr(), None, _lib.MEM_DEVICE,
                                                st or None), "sqoc_chunk_backward")
        return F, grad

    def carry_stats(self) -> dict:
        """Last chunk backward: device ms of the boundary values (needs set_timing(True)) and carry launches."""
        ms, n = ctypes.c_double(), ctypes.c_int()
        _lib.check(self.lib.sqoc_last_carry_stats(self.handle, ctypes.byref(ms), ctypes.byref(n)),
                   "sqoc_last_carry_stats")
        return {"ms": ms.value, "launches": n.value}

    def evaluate_host_ptr(self, u_ptr: int, batch: int, F_ptr: int, grad_ptr: int):
        """Host pointers (e.g. pinned torch tensors); copies happen inside the call."""
        rc = self.lib.sqoc_eval(self.handle, u_ptr, batch, F_ptr or None, grad_ptr or None, None, _lib.MEM_HOST, None)
        _lib.check(rc, "sqoc_eval")

    def evaluate_device(self, u_ptr: int, batch: int, F_ptr: int, grad_ptr: int, tau_ptr: int = 0,
                        stream: int = 0):
        """Device pointers in/out (e.g. torch ``data_ptr()``); blocking."""
        rc = self.lib.sqoc_eval(self.handle, u_ptr, batch, F_ptr or None, grad_ptr or None, tau_ptr or None,
                                _lib.MEM_DEVICE, stream or None)
        _lib.check(rc, "sqoc_eval")
