"""Multi-GPU sharding of one fidelity+gradient evaluation (host side).

Two partitionings:

* seed-DP (cfg 0 batches, cfg 1): independent control vectors per rank, no
  data-path collective -- ``bench.py`` runs it directly.
* slice chunks (cfg 3, cfg 4): rank g owns slices [s_g, e_g).  The only exchange
  is the scan carry: every rank forms its chunk product C_g = U_{e-1}...U_s per
  block, an all-gather shares the P chunk products (sum_b d_b^2 complex per rank),
  and each rank derives its boundary values

      L_g = C_{g-1} ... C_0            X before its first slice = L_g X_0
      R_g = C_{P-1} ... C_{g+1}        Lambda after its last slice = R_g^dag V
      X_N = C_{P-1} ... C_0            tau_b = <V_b, X_N X_0>

  with 2(P-1) redundant carry GEMMs per block, then runs the backward sweep on its
  own slices only.  A second all-gather assembles the gradient.

The math is written against a small engine interface (``chunk_product(u)``,
``eval_chunk(u, x_start, lam_end, tau)``) so the same host logic runs with the GPU
engine (``GrapeEngine``, one rank per GPU over NCCL) and, in the CPU tests, with
an oracle-backed engine over gloo.
"""

from __future__ import annotations

import copy

import numpy as np


def chunk_bounds(n_slices: int, world: int) -> list:
    """Contiguous, balanced slice ranges [(s_g, e_g)] for g = 0..world-1."""
    edges = np.linspace(0, n_slices, world + 1).round().astype(int)
    return [(int(edges[g]), int(edges[g + 1])) for g in range(world)]


def local_system(system, s: int, e: int):
    """The same physical system restricted to slices [s, e) (same dt)."""
    loc = copy.copy(system)
    loc.n_slices = e - s
    loc.T = system.dt * (e - s)
    return loc


def gate_view(system):
    """Gate-objective twin of a system (chunk products need d x d propagation)."""
    g = copy.copy(system)
    g.objective = "gate"
    g.targets = [np.eye(b.dim, dtype=np.complex128) for b in system.blocks]
    g.initial = []
    return g


def carries(products: list, rank: int):
    """(L_g, R_g, X_N) for one block from the gathered chunk products [C_0 .. C_{P-1}]."""
    d = products[0].shape[0]
    left = np.eye(d, dtype=np.complex128)
    for c in products[:rank]:
        left = c @ left
    right = np.eye(d, dtype=np.complex128)
    for c in products[rank + 1:]:
        right = c @ right
    full = products[rank] @ left
    full = right @ full
    return left, right, full


def boundary_values(system, gathered: list, rank: int):
    """Per-block (x_start, lam_end, tau) for `rank` from gathered[g][b] = C_g,b."""
    xs, ls, taus = [], [], []
    for b in range(len(system.blocks)):
        left, right, full = carries([gathered[g][b] for g in range(len(gathered))], rank)
        tgt = np.asarray(system.targets[b], dtype=np.complex128)
        if system.objective == "gate":
            xs.append(left)
            ls.append(right.conj().T @ tgt)
            taus.append(np.vdot(tgt, full))
        else:
            psi0 = np.asarray(system.initial[b], dtype=np.complex128)
            xs.append(left @ psi0)
            ls.append(right.conj().T @ tgt)
            taus.append(np.vdot(tgt, full @ psi0))
    return xs, ls, np.array(taus)


class Comm:
    """Minimal communicator: all-gather of numpy arrays (torch.distributed underneath)."""

    def __init__(self, group=None, device=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.device = device
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def allgather(self, arr: np.ndarray) -> list:
        import torch

        t = torch.from_numpy(np.ascontiguousarray(arr))
        if self.device is not None:
            t = t.to(self.device)
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return [o.cpu().numpy() for o in out]


class ShardedObjective:
    """objective(u) -> (F, grad) for the full grid, evaluated by slice chunks over ranks."""

    def __init__(self, system, comm, engine_factory, rank: int | None = None, world: int | None = None):
        self.system = system
        self.comm = comm
        self.rank = comm.rank if rank is None else rank
        world = comm.world if world is None else world
        self.bounds = chunk_bounds(system.n_slices, world)
        s, e = self.bounds[self.rank]
        self.s, self.e = s, e
        loc = local_system(system, s, e)
        self.eng = engine_factory(loc)
        self.prod = self.eng if system.objective == "gate" else engine_factory(gate_view(loc))

    # the three stages (separable so a single process can emulate P ranks on one GPU)
    def stage_product(self, u) -> np.ndarray:
        u_loc = np.ascontiguousarray(np.asarray(u, dtype=np.float64)[:, self.s:self.e])
        mine = self.prod.chunk_product(u_loc)  # C_g,b
        return np.concatenate([c.reshape(-1) for c in mine])

    def stage_local(self, u, all_products: list):
        dims = [b.dim for b in self.system.blocks]
        gathered = []
        for buf in all_products:
            parts, o = [], 0
            for d in dims:
                parts.append(buf[o:o + d * d].reshape(d, d))
                o += d * d
            gathered.append(parts)
        xs, ls, taus = boundary_values(self.system, gathered, self.comm_rank)
        u_loc = np.ascontiguousarray(np.asarray(u, dtype=np.float64)[:, self.s:self.e])
        F, g_loc = self.eng.eval_chunk(u_loc, xs, ls, taus)
        width = max(e - s for s, e in self.bounds)
        pad = np.zeros((g_loc.shape[0], width))
        pad[:, :g_loc.shape[1]] = g_loc
        return F, pad

    def assemble(self, padded: list) -> np.ndarray:
        return np.concatenate([p[:, :e - s] for p, (s, e) in zip(padded, self.bounds)], axis=1)

    @property
    def comm_rank(self) -> int:
        return self.rank

    def objective(self, u):
        allp = self.comm.allgather(self.stage_product(u))  # the scan-carry exchange
        F, pad = self.stage_local(u, allp)
        return F, self.assemble(self.comm.allgather(pad))


def emulate_ranks(system, world: int, engine_factory, u):
    """Run the P-rank slice-chunk algorithm in one process (no collective): used on a
    single GPU to check the sharded path against the unsharded one."""
    ranks = [ShardedObjective(system, None, engine_factory, rank=g, world=world) for g in range(world)]
    allp = [r.stage_product(u) for r in ranks]
    outs = [r.stage_local(u, allp) for r in ranks]
    F = outs[0][0]
    grad = ranks[0].assemble([o[1] for o in outs])
    return F, grad
