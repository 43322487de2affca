"""qoc.gradient's engine cache is keyed on the matrices' contents (CPU; the engine is faked)."""

import numpy as np

from paper_2309_05884_b200 import qoc


class FakeEngine:
    made = []

    def __init__(self, system, max_batch=1):
        self.system = system
        self.closed = False
        FakeEngine.made.append(self)

    def objective(self, u):
        h0 = self.system.blocks[0].h0
        return float(h0[0, 0].real), np.zeros_like(u)

    def close(self):
        self.closed = True


class Duck:
    def __init__(self, h0):
        self.h0 = h0
        self.hx = np.eye(2, dtype=np.complex128)
        self.hy = np.eye(2, dtype=np.complex128)


def test_cache_distinguishes_backends_with_reused_ids(monkeypatch):
    monkeypatch.setattr(qoc, "GrapeEngine", FakeEngine)
    qoc._ENGINE_CACHE.clear()
    FakeEngine.made.clear()
    psi0 = np.array([1, 0], dtype=np.complex128)
    psif = np.array([0, 1], dtype=np.complex128)
    b = np.zeros(3)
    # inline temporaries: CPython typically reuses the same id for each of them
    ps = [qoc.gradient(psi0, psif, b, b, Duck(np.diag([float(j), 0.0]).astype(np.complex128)), 0.1)[2]
          for j in range(5)]
    assert ps == [0.0, 1.0, 2.0, 3.0, 4.0]  # every backend got its own matrices' engine
    assert len(FakeEngine.made) == 5
    # same contents -> cache hit
    qoc.gradient(psi0, psif, b, b, Duck(np.diag([2.0, 0.0]).astype(np.complex128)), 0.1)
    assert len(FakeEngine.made) == 5


def test_cache_evicts_and_closes_lru(monkeypatch):
    monkeypatch.setattr(qoc, "GrapeEngine", FakeEngine)
    qoc._ENGINE_CACHE.clear()
    FakeEngine.made.clear()
    psi0 = np.array([1, 0], dtype=np.complex128)
    b = np.zeros(2)
    for j in range(qoc._ENGINE_CACHE_MAX + 3):
        qoc.gradient(psi0, psi0, b, b, Duck(np.diag([float(j), 1.0]).astype(np.complex128)), 0.1)
    assert len(qoc._ENGINE_CACHE) == qoc._ENGINE_CACHE_MAX
    assert [e.closed for e in FakeEngine.made[:3]] == [True, True, True]
    assert not any(e.closed for e in FakeEngine.made[3:])
    qoc._ENGINE_CACHE.clear()
