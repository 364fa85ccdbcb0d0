"""Randomised parity (-m gpu): many small CNF shapes — mixed widths 1..12 with duplicate
literals and tautologies, every batch padding class (W < 4 scalar sweep, W % 4 == 0
vector sweep, whole 1024-member chunks with the TMA update and k_sweep) — one step from
identical iterates plus a short free-running trajectory, each against the fp64 oracle."""
import numpy as np
import pytest

from paper_2603_28796_b200 import instances as I
from tests import parity

pytestmark = pytest.mark.gpu

BATCHES = [1, 31, 64, 96, 128, 200, 1000, 1024, 2048]


@pytest.fixture(scope="module")
def G():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2603_28796_b200 import galois
    galois.lib()
    return galois


def random_instance(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(2, 600))
    m = int(rng.integers(1, 6 * n))
    clauses = []
    for _ in range(m):
        w = int(rng.choice([1, 2, 3, 3, 3, 4, 5, 8, 12]))
        vs = rng.integers(1, n + 1, size=w)                     # duplicates / tautologies allowed
        clauses.append([int(v) if rng.random() < 0.5 else -int(v) for v in vs])
    return I.from_clauses(f"fuzz{seed}", n, clauses), rng


@pytest.mark.parametrize("seed", range(32))
def test_random_shapes(G, seed):
    inst, rng = random_instance(seed)
    batch = BATCHES[seed % len(BATCHES)]
    t = int(rng.choice([0, 3]))
    res = parity.one_step(G, inst, batch, t, seed=seed)
    assert res["tie_x"] + res["tie_r"] <= 3
    rep = parity.run_trajectory(G, inst, batch, 6, seed=seed)   # ends at the first SAT check
    assert rep.best_gpu == rep.best_oracle, (rep.best_gpu, rep.best_oracle)
