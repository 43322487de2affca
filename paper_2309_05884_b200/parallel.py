"""Multi-GPU sharding of one fidelity+gradient evaluation (host side).

The reference walks the slices strictly in order (forward ``qoc.py:128-134``, backward
``qoc.py:156-167``).  Two partitionings replace that on P ranks (one process per GPU):

* seed-DP (cfg 0 batches, cfg 1): independent control vectors per rank, no data-path
  collective -- ``bench.py`` runs it directly.
* block groups x slice chunks (cfg 2, 3, 4): ranks form a G x C grid, rank = g * C + c.
  Block group g owns a d^3-balanced subset of the symmetry blocks; chunk c owns the
  contiguous slices [s_c, e_c).  Per rank, all on its own GPU:

      sqoc_chunk_forward   C_c,b = U_{e_c-1} ... U_{s_c} of every owned block (packed)
      all-gather           the C chunk products of the block group (NCCL, device to device:
                           the only data that crosses GPUs for the scan carry)
      sqoc_chunk_backward  boundary values on the device -- X_end = C_c..C_0,
                           Lam_end = C_{c+1}^dag..C_{C-1}^dag V (gate), psi / chi carries (state),
                           the full-grid tau_b -- then the backward sweep of the chunk only
      all-gather           one row per rank [F_part, grad_part (K x N)] -- 8 KB at cfg 3 -- summed
                           in rank order on every rank (deterministic: fixed order, no atomics)

  F_part is the weighted sum over the group's blocks, contributed by chunk 0 only; grad_part
  holds the group's contribution to the chunk's slices.  With one chunk per group (C = 1, block
  groups only -- cfg 2's ~100-dim blocks, whose slice-batched history schedule beats any chunking)
  each rank runs the ordinary evaluation of its blocks and only the row exchange remains.  Carry cost: C - 1 batched GEMM launches
  per rank (c left + C - 1 - c right), against ~24 GEMM-units per slice of local work.

The algorithm is written against a two-method engine interface on torch tensors
(``chunk_forward_t(u) -> packed``, ``chunk_backward_t(u, gathered, C, c) -> (F, grad)``), so the
same host logic drives ``GrapeEngine`` on CUDA tensors over NCCL and, in the CPU tests, the
oracle-backed ``OracleChunkEngine`` on CPU tensors over gloo.
"""

from __future__ import annotations

import copy

import numpy as np


def chunk_bounds(n_slices: int, world: int) -> list:
    """Contiguous, balanced slice ranges [(s_c, e_c)] for c = 0..world-1."""
    edges = np.linspace(0, n_slices, world + 1).round().astype(int)
    return [(int(edges[g]), int(edges[g + 1])) for g in range(world)]


def block_groups(dims, n_groups: int) -> list:
    """d^3-balanced partition of the blocks into n_groups (longest-processing-time first; ties to the
    lowest group).  Each group lists its global block indices in ascending order."""
    if n_groups < 1 or n_groups > len(dims):
        raise ValueError(f"need 1 <= block groups <= {len(dims)} blocks, got {n_groups}")
    load = [0.0] * n_groups
    groups = [[] for _ in range(n_groups)]
    for b in sorted(range(len(dims)), key=lambda i: (-float(dims[i]) ** 3, i)):
        g = min(range(n_groups), key=lambda k: (load[k], k))
        groups[g].append(b)
        load[g] += float(dims[b]) ** 3
    return [sorted(g) for g in groups]


def local_system(system, s: int, e: int, blocks=None):
    """The same physical system restricted to slices [s, e) (same dt) and, optionally, a subset of
    the blocks (keeping the full system's weights, so F and the gradient stay additive)."""
    loc = copy.copy(system)
    loc.n_slices = e - s
    loc.T = system.dt * (e - s)
    if blocks is not None:
        w = np.asarray(system.block_weights(), dtype=np.float64)
        loc.blocks = [system.blocks[b] for b in blocks]
        loc.targets = [system.targets[b] for b in blocks]
        loc.initial = [system.initial[b] for b in blocks] if system.initial else []
        loc.weights = w[list(blocks)]
    return loc


class Comm:
    """torch.distributed underneath: flat all-gathers of tensors (NCCL on CUDA tensors stays on
    the devices; gloo on CPU tensors in the tests) and the block-group sub-communicators."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def new_group(self, ranks):
        return self.dist.new_group(ranks=list(ranks))

    def all_gather(self, t, group=None, size=None):
        """[size, *t.shape] stacked in rank order of `group` (default: the whole communicator)."""
        import torch

        size = self.world if size is None else size
        t = t.contiguous()
        out = torch.empty(size * t.numel(), dtype=t.dtype, device=t.device)
        self.dist.all_gather_into_tensor(out, t.reshape(-1), group=group if group is not None else self.group)
        return out.view(size, *t.shape)


class ShardedObjective:
    """objective(u) -> (F, grad) for the full grid and all blocks, evaluated on a
    (block groups x slice chunks) grid of ranks."""

    def __init__(self, system, comm, engine_factory, n_block_groups: int = 1, rank: int | None = None,
                 world: int | None = None):
        self.system = system
        self.comm = comm
        self.rank = comm.rank if rank is None else rank
        self.world = comm.world if world is None else world
        if self.world % n_block_groups:
            raise ValueError(f"{self.world} ranks do not split into {n_block_groups} block groups")
        self.G = n_block_groups
        self.C = self.world // n_block_groups
        self.g, self.c = divmod(self.rank, self.C)
        self.groups = block_groups([b.dim for b in system.blocks], self.G)
        self.bounds = chunk_bounds(system.n_slices, self.C)
        self.s, self.e = self.bounds[self.c]
        self.K = system.n_controls
        self.eng = engine_factory(local_system(system, self.s, self.e, self.groups[self.g]))
        self.chunk_group = None
        self.timing = False
        self.stage_ms = {}
        if comm is not None and self.C < self.world:
            # every rank creates every sub-group, in the same order (torch.distributed contract)
            for g in range(self.G):
                grp = comm.new_group(range(g * self.C, (g + 1) * self.C))
                if g == self.g:
                    self.chunk_group = grp

    # ---- the stages (separable so one process can emulate the grid of ranks on one GPU) ----
    def local_u(self, u_t):
        return u_t[:, self.s:self.e].contiguous()

    def stage_forward(self, u_t):
        if self.C == 1:  # block groups only: the ordinary evaluation (any schedule) runs in stage_backward
            self.last_launches = 0
            return None
        out = self.eng.chunk_forward_t(self.local_u(u_t))
        self.last_launches = getattr(self.eng, "last_launches", 0)
        return out

    def stage_backward(self, u_t, gathered):
        """This rank's row [F_part, grad_part (K x N) flattened] from its group's gathered products."""
        import torch

        if self.C == 1:
            F, g_loc = self.eng.objective_t(self.local_u(u_t))
        else:
            F, g_loc = self.eng.chunk_backward_t(self.local_u(u_t), gathered, self.C, self.c)
        self.last_launches = getattr(self, "last_launches", 0) + getattr(self.eng, "last_launches", 0)
        N = self.system.n_slices
        row = torch.zeros(1 + self.K * N, dtype=torch.float64, device=g_loc.device)
        if self.c == 0:
            row[0] = F.reshape(())
        row[1:].view(self.K, N)[:, self.s:self.e] = g_loc
        return row

    @staticmethod
    def reduce_rows(rows):
        """Sum of the ranks' rows in rank order (fixed association: bitwise-reproducible)."""
        acc = rows[0].clone()
        for r in range(1, rows.shape[0]):
            acc += rows[r]
        return acc

    def objective_t(self, u_t):
        """Device tensors in and out: u (K, N) on this rank's device -> (F (), grad (K, N)).
        With ``timing`` on, ``stage_ms`` holds the device time of each stage on torch's current stream
        (forward, exchange, backward incl. the on-device carries, gradient reduction)."""
        ev = self._events() if self.timing else None
        if ev:
            ev[0].record()
        packed = self.stage_forward(u_t)
        if ev:
            ev[1].record()
        gathered = None
        if self.C > 1:  # the scan-carry exchange
            gathered = self.comm.all_gather(packed, group=self.chunk_group, size=self.C)
        if ev:
            ev[2].record()
        row = self.stage_backward(u_t, gathered)
        if ev:
            ev[3].record()
        tot = self.reduce_rows(self.comm.all_gather(row))
        if ev:
            ev[4].record()
            ev[4].synchronize()
            names = ("forward", "exchange", "backward", "reduce")
            self.stage_ms = {n: ev[i].elapsed_time(ev[i + 1]) for i, n in enumerate(names)}
        return tot[0], tot[1:].view(self.K, self.system.n_slices)

    def _events(self):
        import torch

        if not hasattr(self, "_ev"):
            self._ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        return self._ev

    def objective(self, u):
        """Host arrays: u (K, N) -> (F float, grad (K, N) ndarray)."""
        import torch

        u_t = torch.as_tensor(np.ascontiguousarray(u, dtype=np.float64)).to(self.eng.torch_device)
        F, g = self.objective_t(u_t)
        return float(F.item()), g.cpu().numpy()


def emulate_ranks(system, world: int, engine_factory, u, n_block_groups: int = 1):
    """The (block groups x chunks) algorithm on `world` ranks in one process, no collective: every
    rank's stages run through its own engine and the exchanges become local stacks.  On one GPU this
    runs the exact device path (chunk ABI, device carries) of a multi-GPU evaluation."""
    import torch

    ranks = [ShardedObjective(system, None, engine_factory, n_block_groups, rank=r, world=world)
             for r in range(world)]
    dev = ranks[0].eng.torch_device
    u_t = torch.as_tensor(np.ascontiguousarray(u, dtype=np.float64)).to(dev)
    packed = [r.stage_forward(u_t) for r in ranks]
    C = ranks[0].C
    rows = []
    for r in ranks:
        gathered = torch.stack(packed[r.g * C:(r.g + 1) * C]) if C > 1 else None
        rows.append(r.stage_backward(u_t, gathered))
    tot = ShardedObjective.reduce_rows(torch.stack(rows))
    K, N = ranks[0].K, system.n_slices
    for r in ranks:
        r.eng.close()
    return float(tot[0].item()), tot[1:].view(K, N).cpu().numpy()
