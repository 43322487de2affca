"""Slice-chunk sharding host logic: world-size-2 gloo processes on CPU, oracle-backed engines."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import grape_oracle as O
from paper_2309_05884_b200 import parallel, systems


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _systems():
    return {
        "gate": systems.gate_ring(6, 10.0 * 13 / 100, 13, seed=2),
        "state": systems.state_transfer_ring(4, 10.0 * 11 / 100, 11, seed=1, full=True),
    }


def _worker(rank, world, port, kind, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = _systems()[kind]
        u = s.controls(3)
        obj = parallel.ShardedObjective(s, parallel.Comm(), O.OracleChunkEngine)
        F, g = obj.objective(u)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), F=F, g=g)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["gate", "state"])
def test_two_rank_gloo_matches_unsharded_oracle(kind):
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_worker, args=(2, _free_port(), kind, tmp), nprocs=2, join=True)
        s = _systems()[kind]
        Fo, go, _ = O.objective(s, s.controls(3))
        for r in range(2):
            res = np.load(os.path.join(tmp, f"r{r}.npz"))
            assert abs(float(res["F"]) - Fo) <= 1e-12
            np.testing.assert_allclose(res["g"], go, atol=1e-12 * np.abs(go).max())


@pytest.mark.parametrize("world", [1, 3, 4])
def test_emulated_ranks_match_unsharded_oracle(world):
    for s in _systems().values():
        u = s.controls(7)
        F, g = parallel.emulate_ranks(s, world, O.OracleChunkEngine, u)
        Fo, go, _ = O.objective(s, u)
        assert abs(F - Fo) <= 1e-12
        np.testing.assert_allclose(g, go, atol=1e-12 * np.abs(go).max())


def test_chunk_bounds_cover_grid():
    for n, p in [(500, 8), (7, 3), (200, 8), (5, 5)]:
        b = parallel.chunk_bounds(n, p)
        assert b[0][0] == 0 and b[-1][1] == n
        assert all(b[i][1] == b[i + 1][0] for i in range(p - 1))
        assert max(e - s for s, e in b) - min(e - s for s, e in b) <= 1
