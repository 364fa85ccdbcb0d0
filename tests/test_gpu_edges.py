"""Edge cases of the CUDA path against the oracle (-m gpu): empty formulas, contradictions,
very long clauses, unused variables, tiny and ragged batches, call-order and argument
errors."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2603_28796_b200 import instances as I
from tests import parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2603_28796_b200 import galois
    galois.lib()
    return galois


def test_no_clauses_is_sat_at_t0(G):
    """m = 0: every assignment satisfies the (empty) conjunction; the t = 0 check finds
    u* = 0 at member 0 and the engine stops before any update."""
    cnf = G.Cnf(5, np.zeros(1, np.int64), np.zeros(0, np.int32))
    eng = G.Engine(cnf, 64, 10, 0.5, 0)
    assert eng.run() == G.SAT
    best = eng.best_assignment()
    assert (best["unsat"], best["step"], best["global_b"]) == (0, 0, 0)
    assert eng.info()["steps_done"] == 0
    eng.free()


@pytest.mark.parametrize("batch", [64, 1024])
def test_contradiction_never_sat(G, batch):
    """(x1) and (not x1): every member leaves exactly one clause unsatisfied at every check;
    the whole trajectory equals the oracle's and the run ends on the budget."""
    inst = I.from_clauses("contra", 1, [[1], [-1]])
    rep = parity.run_trajectory(G, inst, batch, 20, seed=4, stop_on_sat=False)
    assert rep.best_gpu == rep.best_oracle == (1, 0, 0)
    cnf = G.Cnf.from_instance(inst)
    eng = G.Engine(cnf, batch, 20, 0.5, 4)
    assert eng.run() == G.BUDGET
    counts, _ = eng.unsat_counts()
    assert (counts == 1).all()
    eng.free()


@pytest.mark.parametrize("batch", [96, 1024])
def test_long_clause(G, batch):
    """A 300-literal clause next to 3-clauses (widths far beyond the sweep's register cache
    and the update's 32-row stage: streamed pieces) from identical iterates."""
    rng = np.random.default_rng(3)
    clauses = [list(map(int, (rng.choice(400, 300, replace=False) + 1) * np.where(rng.random(300) < .5, -1, 1)))]
    r3 = I.random_ksat(400, 1200, 3, 9)
    clauses += [r3.lits[r3.offsets[c]:r3.offsets[c + 1]].tolist() for c in range(r3.m)]
    inst = I.from_clauses("long", 400, clauses)
    res = parity.one_step(G, inst, batch, 2)
    assert res["tie_x"] + res["tie_r"] <= 2


def test_unused_variables_do_not_move(G):
    """A variable with no occurrence has G = 0 every step: Adam's moments stay 0 and its
    logit keeps its initial value exactly (no gradient flows to it)."""
    # x1 and not x1 keep every member unsatisfied (no SAT stop); x4..x6 never occur
    inst = I.from_clauses("unused", 6, [[1], [-1], [2, -3], [3, 2, -1]])
    cnf = G.Cnf.from_instance(inst)
    eng = G.Engine(cnf, 64, 8, 0.5, 1, debug=True)
    z0, _, _, _ = eng.get_iterate()
    for _ in range(8):
        eng.step()
    z, m, v, t = eng.get_iterate()
    assert t == 8
    np.testing.assert_array_equal(z[:, 3:], z0[:, 3:])
    assert not m[:, 3:].any() and not v[:, 3:].any()
    eng.free()


@pytest.mark.parametrize("batch", [1, 33, 1025])
def test_tiny_and_ragged_batches(G, batch):
    """B = 1 (one member in a 32-wide word), 33 (two words, one member in the second) and
    1025 (a 1024-member chunk plus one member): padding members never leak into counts."""
    inst = I.random_ksat(40, 170, 3, 6)
    rep = parity.run_trajectory(G, inst, batch, 12, seed=5, stop_on_sat=False)
    assert rep.best_gpu == rep.best_oracle
    assert len(rep.resyncs) <= 2


def test_local_slice_beyond_int32_is_rejected(G):
    """A local batch slice of 2^31 members or more (the slice is indexed in int32) is
    rejected with E_ARG at preparation, before any allocation."""
    inst = I.random_ksat(30, 120, 3, 1)
    cnf = G.Cnf.from_instance(inst)
    eng = G.Engine(cnf, 2 ** 31 + 4096, 3, 0.5, 0)
    with pytest.raises(G.GaloisError) as e:
        eng.step()
    assert e.value.code == G.E_ARG
    eng.free()
    cnf.free()


def test_call_order_and_arguments(G):
    inst = I.random_ksat(30, 120, 3, 1)
    cnf = G.Cnf.from_instance(inst)
    for bad in (dict(batch=0, steps=5, lr=0.5), dict(batch=32, steps=-1, lr=0.5), dict(batch=32, steps=5, lr=0.0),
                dict(batch=32, steps=5, lr=float("nan"))):
        with pytest.raises(G.GaloisError) as e:
            G.Engine(cnf, bad["batch"], bad["steps"], bad["lr"], 0)
        assert e.value.code == G.E_ARG
    eng = G.Engine(cnf, 32, 3, 0.5, 0)
    rc = G.OK
    for _ in range(3):
        rc = eng.step()
        if rc == G.SAT:
            break
    if rc != G.SAT:
        assert eng.step() == G.BUDGET                  # budget spent: no further step
    with pytest.raises(G.GaloisError) as e:            # setters only before the first step
        G._check(G.lib().galois_engine_set_check_interval(eng.handle, 2))
    assert e.value.code == G.E_STATE
    first = eng.best_assignment()
    assert eng.run() in (G.SAT, G.BUDGET)              # idempotent after the end
    assert eng.best_assignment()["unsat"] == first["unsat"]
    f = O.Cnf(inst.n, inst.offsets, inst.lits)
    assert O.unsat_count(f, first["values"]) == first["unsat"]
    eng.free()


def test_graph_replay_equals_plain_launches(G):
    """run() replays CUDA graphs of 8 captured steps when the budget is long (>= 256 steps
    left): the result must be bit-identical to enqueueing the same steps one by one
    (Lambda parity buffers, step counters and the stop flag all live on the device)."""
    inst = I.random_ksat(60, 420, 3, 11)              # ratio 7: UNSAT, runs the whole budget
    out = []
    for mode in ("graph", "plain"):
        cnf = G.Cnf.from_instance(inst)
        eng = G.Engine(cnf, 2048, 300, 0.5, 2)
        if mode == "graph":
            rc = eng.run()
        else:
            eng.enqueue(300)
            rc = eng.run()                             # nothing left: settles and reports
        best = eng.best_assignment()
        counts, _ = eng.unsat_counts()
        z, _, _, t = eng.get_iterate()
        out.append((rc, best["unsat"], best["step"], best["global_b"], counts.copy(), z.copy(), t))
        eng.free()
    a, b = out
    assert a[0] == b[0] == G.BUDGET and a[1:4] == b[1:4] and a[6] == b[6] == 300
    np.testing.assert_array_equal(a[4], b[4])
    np.testing.assert_array_equal(a[5], b[5])


@pytest.mark.parametrize("batch,field", [(64, "z"), (2048, "z"), (2048, "m")])
def test_nonfinite_iterate_poisons(G, batch, field):
    """SPEC: a NaN/Inf iterate is a hard error. An injected NaN logit (or an
    infinite first moment, which drives z to -inf) makes the update raise the device's non-finite flag; the step
    returns E_NONFINITE, and the handle is poisoned (every later call E_STATE)."""
    import numpy as np
    inst = I.random_ksat(100, 420, 3, 1)
    cnf = G.Cnf.from_instance(inst)
    eng = G.Engine(cnf, batch, 10, 0.5, 0)
    z, m, v, _ = eng.get_iterate()
    if field == "z":
        z[batch // 2, 17] = np.nan
    else:
        m[batch // 2, 17] = np.inf
    eng.set_iterate(z, m, v, 0)
    with pytest.raises(G.GaloisError) as e:
        eng.step()
    assert e.value.code == G.E_NONFINITE
    with pytest.raises(G.GaloisError) as e:
        eng.info()
    assert e.value.code == G.E_STATE
    eng.free()
    cnf.free()
