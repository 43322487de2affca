"""Random dense systems over every tiny-kernel dimension and several DMMA-path sizes, both
objectives, K = 2, both tiny schedules -- against the CPU oracle."""

import numpy as np
import pytest

from oracle import grape_oracle as O
from paper_2309_05884_b200 import systems
from paper_2309_05884_b200.engine import GrapeEngine

pytestmark = pytest.mark.gpu


def random_system(d, objective, n_slices, seed):
    rng = np.random.default_rng(seed)

    def herm(scale):
        a = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
        return systems.hermitian_part(a) * scale / max(1.0, np.sqrt(d))

    blk = systems.Block(f"rand{d}", herm(1.0), [herm(0.5), herm(0.5)], None)
    if objective == "gate":
        targets = [systems.haar_unitary(rng, d)]
        initial = []
    else:
        targets = [systems.haar_state(rng, d)]
        initial = [systems.haar_state(rng, d)]
    return systems.GrapeSystem(f"rand{d}", 0, [blk], objective, 0.05 * n_slices, n_slices, targets, initial)


@pytest.mark.parametrize("d", list(range(1, 17)) + [17, 24, 33, 64, 65])
@pytest.mark.parametrize("objective", ["gate", "state"])
def test_random_dense_block(d, objective):
    s = random_system(d, objective, 9, seed=100 + d)
    u = np.random.default_rng(d).uniform(-1, 1, (3, 2, 9))
    hist = {"fused-recompute": "off", "fused-x": "x", "fused-chain": "chain"}
    schedules = list(hist) + ["slice-parallel"] if d <= 16 else ["auto"]
    for sched in schedules:
        eng = GrapeEngine(s, max_batch=3)
        if d <= 16:
            eng.set_tiny_schedule("fused" if sched.startswith("fused") else sched)
            if sched in hist:
                eng.set_tiny_history(hist[sched])
        F, g = eng.objective(u)
        if sched in hist:
            assert eng.last_tiny_history == hist[sched]
        for b in range(3):
            Fo, go, _ = O.objective(s, u[b])
            assert abs(F[b] - Fo) <= 1e-10, (d, objective, sched)
            # d = 1 has F = 1 and an exactly-zero gradient: rounding noise ~1e-18 is judged
            # against an absolute floor of 1e-14 (1e-8 of a unit-scale gradient entry 1e-6)
            assert np.abs(g[b] - go).max() <= 1e-8 * max(np.abs(go).max(), 1e-6), (d, objective, sched)
