"""Single-launch small-instance run (k_small_run, used by galois_engine_run when a CTA's
32 members fit shared memory) against the per-step kernels (-m gpu).

The per-step path is forced by turning profiling on (its per-kernel records need the
per-step kernels). Both run the same quad_update(), so the iterates, best record, bits,
counts and losses must be bit-identical — also after a SAT, where a grid barrier at each
check stops every CTA exactly where the per-step engine stops."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2603_28796_b200 import instances as I

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2603_28796_b200 import galois
    galois.lib()
    return galois


def _run(G, inst, B, T, seed, per_step, pre=0, state=True, **kw):
    cnf = G.Cnf.from_instance(inst)
    eng = G.Engine(cnf, B, T, 0.5, seed, **kw)
    if per_step:
        eng.set_profiling(True)
    if pre:
        eng.enqueue(pre)
    rc = eng.run()
    best = eng.best_assignment()
    counts, _ = eng.unsat_counts()
    info = eng.info()
    out = dict(rc=rc, best=(best["unsat"], best["step"], best["global_b"]), values=best["values"], counts=counts,
               info=info)
    if state:
        out["iterate"] = eng.get_iterate()
        out["loss"] = eng.get_loss()
        out["bits"] = eng.get_bits()
    eng.free()
    cnf.free()
    return out


def _same(a, b, state=True):
    assert a["rc"] == b["rc"]
    assert a["best"] == b["best"]
    np.testing.assert_array_equal(a["values"], b["values"])
    np.testing.assert_array_equal(a["counts"], b["counts"])
    assert a["info"] == b["info"]
    if state:
        for x, y in zip(a["iterate"], b["iterate"]):
            np.testing.assert_array_equal(x, y)
        np.testing.assert_array_equal(a["loss"], b["loss"])
        for x, y in zip(a["bits"], b["bits"]):
            np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("K,B", [(1, 1000), (3, 1024), (4, 96)])
def test_small_run_equals_per_step(G, K, B):
    """No SAT in the budget: every member's iterate (z, m, v, t), the best record and its
    bits, the counts of the last check, Lambda and the bit planes are identical."""
    inst = I.random_ksat(300, 1290, 3, 5)
    a = _run(G, inst, B, 40, 7, per_step=True, check_interval=K)
    b = _run(G, inst, B, 40, 7, per_step=False, check_interval=K)
    assert a["rc"] == G.BUDGET
    _same(a, b)


def test_small_run_after_enqueue(G):
    """run() after steps already enqueued on the per-step path continues from there."""
    inst = I.random_ksat(200, 852, 3, 3)
    a = _run(G, inst, 512, 30, 1, per_step=True, pre=7)
    b = _run(G, inst, 512, 30, 1, per_step=False, pre=7)
    _same(a, b)


@pytest.mark.parametrize("variant", [dict(tau=0.5), dict(optimizer=1), dict(cubes=[3, 17, 40])])
def test_small_run_variants(G, variant):
    """tau != 1 (logistic path), SGD and cube pins use the same quad_update variants."""
    inst = I.random_ksat(120, 510, 3, 4)
    a = _run(G, inst, 256, 25, 2, per_step=True, **variant)
    b = _run(G, inst, 256, 25, 2, per_step=False, **variant)
    _same(a, b)


@pytest.mark.parametrize("seed", [0, 2, 3])
def test_small_run_first_sat(G, seed):
    """C1 shape: the first satisfying (step, member), its bits (a model of the CNF, checked
    by the oracle), the step count, every member's iterate and last-check count equal the
    per-step engine's."""
    inst = I.random_ksat(50, 213, 3, seed)
    a = _run(G, inst, 1024, 100, 0, per_step=True)
    b = _run(G, inst, 1024, 100, 0, per_step=False)
    _same(a, b)                                   # iterates and counts too: the stop is exact
    f = O.Cnf(inst.n, inst.offsets, inst.lits)
    assert O.unsat_count(f, b["values"]) == b["best"][0]
    if b["rc"] == G.SAT:
        assert b["counts"][b["best"][2]] == 0


def test_small_run_not_used_when_large(G):
    """Instances whose 32-member state exceeds shared memory take the per-step path (same
    results either way; this only checks that run() works at the boundary sizes)."""
    inst = I.random_ksat(600, 2556, 3, 1)         # 600 x 384 B + E > 200 KB: per-step
    a = _run(G, inst, 64, 10, 0, per_step=True)
    b = _run(G, inst, 64, 10, 0, per_step=False)
    _same(a, b)


def test_small_run_planted_sat_k_interval(G):
    """A planted instance solved mid-run with a check interval: stop step, record and state
    identical (the barrier sits only at check steps)."""
    inst = I.random_ksat(60, 255, 3, 13, planted=True)
    for K in (1, 3):
        a = _run(G, inst, 2048, 40, 21, per_step=True, check_interval=K)
        b = _run(G, inst, 2048, 40, 21, per_step=False, check_interval=K)
        _same(a, b)
