"""Lanes (galois_engine_set_lanes): the local slice split into concurrent engines over
consecutive member ranges gives the undivided engine's results exactly (-m gpu).

Members are independent restarts whose RNG counters use the global member
index, so every member's trajectory, the best record (u*, t*, b*) and its assignment
must be bit-identical to the undivided engine's."""
import numpy as np
import pytest

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


def _solve(G, inst, batch, steps, seed, drive="run", **kw):
    cnf = G.Cnf.from_instance(inst)
    eng = G.Engine(cnf, batch, steps, 0.5, seed, **kw)
    if drive == "run":
        rc = eng.run()
    else:                                   # bench-style: enqueue in pieces, then query
        rc = None
        for k in drive:
            eng.enqueue(k)
    best = eng.best_assignment()
    counts, b0 = eng.unsat_counts()
    info = eng.info()
    eng.free()
    cnf.free()
    return rc, (best["unsat"], best["step"], best["global_b"]), best["values"], counts, info


@pytest.mark.parametrize("K,lanes,B", [(1, 2, 3000), (4, 3, 3000), (1, 4, 4096), (2, 2, 2100)])
def test_lanes_equal_undivided(G, K, lanes, B):
    """No SAT in the budget: best (u, t, b), its bits, every member's last count and the
    step count equal the undivided engine's (ragged last lanes: 3000 = 1024 + 1024 + 952
    runs the short lane on the W < 32 kernels; 2100 = 2048 + 52)."""
    inst = I.random_ksat(300, 1290, 3, 5)
    full = _solve(G, inst, B, 40, 7, check_interval=K)
    part = _solve(G, inst, B, 40, 7, check_interval=K, lanes=lanes)
    assert full[0] == part[0] == G.BUDGET
    assert full[1] == part[1]
    np.testing.assert_array_equal(full[2], part[2])
    np.testing.assert_array_equal(full[3], part[3])
    assert full[4] == part[4]


def test_lanes_graph_chunks(G):
    """A run long enough for the CUDA-graph chunks (>= 256 steps) on every lane."""
    inst = I.random_ksat(2000, 8520, 3, 11)
    full = _solve(G, inst, 4096, 300, 3)
    part = _solve(G, inst, 4096, 300, 3, lanes=2)
    assert full[0] == part[0]
    assert full[1] == part[1]
    np.testing.assert_array_equal(full[2], part[2])
    np.testing.assert_array_equal(full[3], part[3])
    assert full[4] == part[4]


def test_lanes_enqueue_pieces(G):
    """The bench's driving: enqueue(k) several times, then query (the aggregate is formed
    again after every enqueue)."""
    inst = I.random_ksat(1000, 4260, 3, 2)
    full = _solve(G, inst, 4096, 60, 1, drive=(5, 20, 35))
    part = _solve(G, inst, 4096, 60, 1, drive=(5, 20, 35), lanes=4)
    assert full[1] == part[1]
    np.testing.assert_array_equal(full[2], part[2])
    np.testing.assert_array_equal(full[3], part[3])
    assert full[4] == part[4]


@pytest.mark.parametrize("lanes", [2, 4])
def test_lanes_first_sat(G, lanes):
    """SAT stop: the first satisfying (step, member) of the undivided batch, its bits and
    the step count; the winner's lane reports the undivided engine's count for its member."""
    inst = I.random_ksat(50, 213, 3, 0)
    full = _solve(G, inst, 4096, 100, 0)
    part = _solve(G, inst, 4096, 100, 0, lanes=lanes)
    assert full[0] == part[0] == G.SAT
    assert full[1] == part[1] and full[1][0] == 0
    np.testing.assert_array_equal(full[2], part[2])
    assert full[4]["steps_done"] == part[4]["steps_done"] and part[4]["stopped"]
    b = full[1][2]
    assert part[3][b] == full[3][b] == 0


def test_lanes_step_api(G):
    """galois_engine_step on a split engine: OK per step, then BUDGET, same results."""
    inst = I.random_ksat(300, 1290, 3, 5)
    out = []
    for lanes in (1, 2):
        cnf = G.Cnf.from_instance(inst)
        eng = G.Engine(cnf, 2048, 6, 0.5, 4, lanes=lanes)
        rcs = [eng.step() for _ in range(7)]
        out.append((rcs, eng.best_assignment(), eng.unsat_counts()[0]))
        eng.free()
        cnf.free()
    assert out[0][0] == out[1][0] == [G.OK] * 6 + [G.BUDGET]
    assert out[0][1]["unsat"] == out[1][1]["unsat"] and out[0][1]["global_b"] == out[1][1]["global_b"]
    np.testing.assert_array_equal(out[0][2], out[1][2])


def test_lanes_theta_sel_pool_and_cubes(G):
    """f1/f3 on a split engine: select_member, the candidate pool and the cube variables of
    any member equal the undivided engine's (every member stays resident in its lane)."""
    inst = I.random_ksat(300, 1290, 3, 5)
    out = []
    for lanes in (1, 3):
        cnf = G.Cnf.from_instance(inst)
        eng = G.Engine(cnf, 3000, 25, 0.5, 3, lanes=lanes)
        assert eng.run() == G.BUDGET
        sel = [eng.select_member(r) for r in (0, 1)]
        b0 = sel[0]["global_b"]
        pool = eng.candidate_pool(b0, 16, 0.02, 5)
        cubes = eng.cube_variables(2500, 7)              # a member of the last lane
        out.append((sel, pool, cubes))
        eng.free()
        cnf.free()
    (s0, p0, c0), (s1, p1, c1) = out
    for r in (0, 1):
        assert s0[r]["global_b"] == s1[r]["global_b"] and s0[r]["unsat"] == s1[r]["unsat"]
        np.testing.assert_array_equal(s0[r]["z"], s1[r]["z"])
    np.testing.assert_array_equal(p0["values"], p1["values"])
    np.testing.assert_array_equal(p0["units"], p1["units"])
    np.testing.assert_array_equal(c0, c1)


def test_lanes_cubes_pins(G):
    """Cube pins (alpha = b mod 2^d) follow the global member index into every lane."""
    inst = I.random_ksat(200, 852, 3, 9)
    pins = [3, 17, 40, 41, 99]
    full = _solve(G, inst, 4096, 30, 2, cubes=pins)
    part = _solve(G, inst, 4096, 30, 2, cubes=pins, lanes=4)
    assert full[1] == part[1]
    np.testing.assert_array_equal(full[2], part[2])
    np.testing.assert_array_equal(full[3], part[3])


def test_lanes_gating_and_kernel_times(G):
    inst = I.random_ksat(300, 1290, 3, 5)
    cnf = G.Cnf.from_instance(inst)
    with pytest.raises(G.GaloisError) as e:
        G.Engine(cnf, 4096, 10, 0.5, 0, lanes=0)
    assert e.value.code == G.E_ARG
    small = G.Engine(cnf, 1024, 4, 0.5, 0, lanes=2)        # one lane's worth: undivided
    small.run()
    small.get_iterate()
    small.free()
    eng = G.Engine(cnf, 4096, 10, 0.5, 0, lanes=2)
    eng.enqueue(2)
    ref = G.Engine(cnf, 4096, 10, 0.5, 0)
    ref.enqueue(2)
    # the test hooks act on every lane: the same iterate, bits and Lambda as undivided
    for a, b in zip(eng.get_iterate(), ref.get_iterate()):
        np.testing.assert_array_equal(a, b)
    for a, b in zip(eng.get_bits(), ref.get_bits()):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(eng.get_loss(), ref.get_loss())
    for b in (0, 2047, 2048, 4095):
        x, y = eng.get_member(b), ref.get_member(b)
        for k in ("z", "m", "v", "x_next", "r"):
            np.testing.assert_array_equal(x[k], y[k])
        assert (x["t"], x["unsat"], x["check_t"]) == (y["t"], y["unsat"], y["check_t"])
    ref.free()
    eng.set_profiling(True)
    eng.kernel_times()
    eng.enqueue(3)
    kt = eng.kernel_times()
    # per step and lane: one sweep and one update
    assert kt["forward"][1] == 2 * 3 and kt["update"][1] == 2 * 3
    eng.free()
    cnf.free()


@pytest.mark.parametrize("K", [1, 3])
def test_lanes_over_nccl(G, K):
    """Lanes requested together with an NCCL communicator (a 1-rank one here): the engine
    stays undivided (concurrent collectives on several communicators of one device are not
    guaranteed to progress, galois.h set_lanes); best, its bits (broadcast from the owner)
    and the counts equal the undivided engine's, with and without SAT."""
    inst = I.random_ksat(300, 1290, 3, 5)
    full = _solve(G, inst, 3000, 40, 7, check_interval=K)
    comm = _solve(G, inst, 3000, 40, 7, check_interval=K, lanes=3, nccl_id=G.galois_comm_unique_id())
    assert full[1] == comm[1]
    np.testing.assert_array_equal(full[2], comm[2])
    np.testing.assert_array_equal(full[3], comm[3])
    assert full[4] == comm[4]
    sat = I.random_ksat(50, 213, 3, 0)
    f2 = _solve(G, sat, 4096, 100, 0)
    c2 = _solve(G, sat, 4096, 100, 0, lanes=2, nccl_id=G.galois_comm_unique_id())
    assert f2[0] == c2[0] == G.SAT and f2[1] == c2[1]
    np.testing.assert_array_equal(f2[2], c2[2])
