"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle (-m gpu)."""
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


# --------------------------------------------------------------------------- a1 / a2
def test_cnf_load_device_validation(G):
    with pytest.raises(G.GaloisError) as e:
        G.Cnf(3, np.array([0, 2, 1, 3], np.int64), np.array([1, 2, 3], np.int32))
    assert e.value.code == G.E_OFFSETS
    with pytest.raises(G.GaloisError) as e:
        G.Cnf(3, np.array([0, 2, 3], np.int64), np.array([1, 4, 3], np.int32))
    assert e.value.code == G.E_VAR_RANGE
    with pytest.raises(G.GaloisError) as e:
        G.Cnf(3, np.array([0, 2, 3], np.int64), np.array([1, 0, 3], np.int32))
    assert e.value.code == G.E_VAR_RANGE
    with pytest.raises(G.GaloisError) as e:
        G.Cnf(3, np.array([0, 2, 2, 3], np.int64), np.array([1, -2, 3], np.int32))
    assert e.value.code == G.E_EMPTY_CLAUSE
    c = G.Cnf(3, np.array([0], np.int64), np.zeros(0, np.int32))       # zero clauses is fine
    assert c.info()["m"] == 0


@pytest.mark.parametrize("which", ["small", "3sat", "industrial", "wide_n"])
def test_csc_is_stable_counting_sort(G, which):
    """a2: the device transpose equals numpy's stable argsort of the literal codes
    (variable, sign, slot order) — bit-exact, including several radix passes."""
    inst = {"small": lambda: I.from_clauses("t", 5, [[1, -2, 5], [-5, 3, 4], [-1, 3, 3]]),
            "3sat": lambda: I.random_ksat(3000, 12000, 3, 1),
            "industrial": lambda: I.industrial(40_000, 160_000, 3),
            "wide_n": lambda: I.random_ksat(200_000, 300_000, 4, 2)}[which]()
    c = G.Cnf.from_instance(inst)
    code_off, occ = c.csc()
    lits = inst.lits.astype(np.int64)
    code = (np.abs(lits) - 1) * 2 + (lits < 0)
    np.testing.assert_array_equal(occ, np.argsort(code, kind="stable"))
    np.testing.assert_array_equal(code_off, np.concatenate([[0], np.cumsum(np.bincount(code, minlength=2 * inst.n))]))
    info = c.info()
    deg = I.degrees(inst)
    assert info["max_degree"] == deg.max()
    assert info["max_width"] == np.diff(inst.offsets).max()
    assert info["num_hubs"] == int((deg > 256).sum())


# --------------------------------------------------------------------------- a3-a8
@pytest.mark.parametrize("batch", [32, 64, 100, 224, 256, 2048])
def test_init_and_t0_check(G, batch):
    """a3 + a8 at t = 0: z0 = theta_1 - theta_0 from the same Philox counters, R_0, the
    exact unsat counts and the best at t = 0."""
    inst = I.random_ksat(50, 213, 3, 0)
    rep = parity.run_trajectory(G, inst, batch, steps=0)
    assert rep.best_gpu == rep.best_oracle


@pytest.mark.parametrize("t", [0, 1, 7, 40])
@pytest.mark.parametrize("which", ["3sat", "mixed", "dups"])
def test_one_step_identical_iterate(G, which, t):
    """a4-a8 from identical iterates: X, R bit-exact (outside the tie zone), Lambda and G
    exact, g1 within relative 1e-5, z/m/v within 1e-5."""
    inst = {"3sat": lambda: I.random_ksat(60, 255, 3, 3),
            "mixed": lambda: I.industrial(300, 1500, 4),
            "dups": lambda: I.from_clauses("dups", 6, [[1, 1, -2], [2, -3, 3], [4, 5, 6, -1, 2, 3, 4, 5, 6, -6],
                                                        [-4], [5, -5], [1, 2, 3, 4, 5, 6, -1, -2, -3, -4]])}[which]()
    res = parity.one_step(G, inst, 96, t)
    assert res["tie_x"] + res["tie_r"] <= 2


@pytest.mark.parametrize("batch", [1000, 1024, 2048, 3000])
def test_one_step_tma_path(G, batch):
    """Batches that pad to whole 1024-member chunks run the TMA-staged update kernel; its
    three signal paths (E rows staged in one piece for degree <= 48, streamed through
    further 48-row pieces up to degree 256 — bit-sliced counts for long pieces — and hub
    partials above) must all equal the oracle."""
    inst = I.industrial(2500, 30_000, 21, occ_exp=0.9)
    deg = I.degrees(inst)
    assert (deg <= 48).any() and ((deg > 48) & (deg <= 256)).any() and (deg > 256).any()
    res = parity.one_step(G, inst, batch, 4)
    assert res["tie_x"] + res["tie_r"] <= 3


@pytest.mark.parametrize("k,batch", [(5, 1024), (7, 2048)])
def test_wide_clause_sweep(G, k, batch):
    """Average width >= 4.5 selects the sweep's wide shape (6 counter planes, no register
    cache, 4 CTAs per SM): one step from identical iterates and a 12-step trajectory
    (Lambda, G, unsat counts, best) against the oracle."""
    inst = I.random_ksat(120, {5: 2400, 7: 9000}[k], k, 8)
    res = parity.one_step(G, inst, batch, 3)
    assert res["tie_x"] + res["tie_r"] <= 3
    rep = parity.run_trajectory(G, inst, batch, 12, seed=2, stop_on_sat=False)
    assert rep.best_gpu == rep.best_oracle


def test_trajectory_50_steps(G):
    """North star: per-step trajectories within 1e-4 for 50 steps on small instances."""
    inst = I.random_ksat(50, 213, 3, 5)
    rep = parity.run_trajectory(G, inst, 128, 50, seed=3, stop_on_sat=False)
    assert rep.steps == 50
    assert len(rep.resyncs) <= 3, rep.resyncs
    assert rep.best_gpu == rep.best_oracle


def test_trajectory_mixed_widths_check_interval(G):
    inst = I.industrial(400, 1800, 7)
    rep = parity.run_trajectory(G, inst, 64, 30, seed=11, check_interval=4, stop_on_sat=False)
    assert rep.best_gpu == rep.best_oracle


def test_first_sat_matches_oracle_C1(G):
    """configs[0]: 3-SAT n=50, m=213, B=1024, 100 steps: the first satisfying member and
    step found by the engine are the oracle's."""
    inst = I.random_ksat(50, 213, 3, 0)
    rep = parity.run_trajectory(G, inst, 1024, 100, seed=0)
    assert rep.best_gpu == rep.best_oracle, rep


def test_run_equals_stepwise(G):
    """galois_engine_run (chunked, device stop flag) gives the same best and step count
    as stepping one call at a time; a SAT stop freezes the engine."""
    inst = I.random_ksat(40, 160, 3, 2, planted=True)
    out = []
    for mode in ("run", "step"):
        cnf = G.Cnf.from_instance(inst)
        eng = G.Engine(cnf, 512, 60, 0.5, 4)
        if mode == "run":
            rc = eng.run()
        else:
            rc = G.OK
            while rc == G.OK:
                rc = eng.step()
        best = eng.best_assignment()
        info = eng.info()
        out.append((rc, best["unsat"], best["step"], best["global_b"], info["steps_done"], info["stopped"]))
        f = O.Cnf(inst.n, inst.offsets, inst.lits)
        assert O.unsat_count(f, best["values"]) == best["unsat"]
        eng.free()
    assert out[0] == out[1]
    if out[0][0] == G.SAT:
        assert out[0][1] == 0 and out[0][4] == out[0][2]


def test_batch_independence_and_determinism(G):
    """Member b's trajectory does not depend on B (global RNG counters) and repeats are
    bit-identical."""
    inst = I.random_ksat(80, 336, 3, 6)
    states = []
    for B in (64, 64, 160):
        cnf = G.Cnf.from_instance(inst)
        eng = G.Engine(cnf, B, 12, 0.5, 9)
        for _ in range(12):
            eng.step()
        z, m, v, t = eng.get_iterate()
        x, r = eng.get_bits()
        states.append((z[:64], m[:64], v[:64], x[:64], r[:64]))
        eng.free()
    for a, b in zip(states[0], states[1]):
        np.testing.assert_array_equal(a, b)
    for a, b in zip(states[0], states[2]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("batch", [256, 2048])
def test_nccl_path_single_rank(G, batch):
    """a9 through NCCL on one GPU: a 1-rank communicator (ncclCommInitRank from our own
    ncclUniqueId; MIN all-reduce of the best key each check; k_finalize; broadcast of the
    winner's bits) gives exactly the single-process results."""
    inst = I.random_ksat(60, 255, 3, 13, planted=True)
    outs = []
    for nid in (None, G.galois_comm_unique_id()):
        cnf = G.Cnf.from_instance(inst)
        eng = G.Engine(cnf, batch, 40, 0.5, 21, rank=0, world=1, nccl_id=nid)
        rc = eng.run()
        best = eng.best_assignment()
        u, _ = eng.unsat_counts()
        z = eng.get_iterate()[0]
        outs.append((rc, best["unsat"], best["step"], best["global_b"], best["values"].tobytes(), u.tobytes(),
                     z.tobytes()))
        eng.free()
    assert outs[0] == outs[1]


@pytest.mark.parametrize("batch,n", [(96, 300), (2048, 5000)])
def test_selection_pool_and_cubes(G, batch, n):
    """NEXT f1/f3: theta_sel (min and max loss), the candidate pool (Eq.10), the top-|S|
    unit literals (Eq.11) and the lowest-confidence cube variables (Lemma 1) against the
    oracle on the engine's own logits. Integer decisions taken in floating point (the
    sample bit, the |S|-th confidence, |z| order) may differ only inside the fp32 tie zone."""
    inst = I.industrial(n, 4 * n, 31)
    cnf = G.Cnf.from_instance(inst)
    eng = G.Engine(cnf, batch, 12, 0.5, 5)
    eng.run()
    counts, b0 = eng.unsat_counts()
    z_all = eng.get_iterate()[0]
    for rule in (0, 1):
        sel = eng.select_member(rule)
        assert (sel["global_b"], sel["unsat"]) == O.select_member(counts, b0, rule)
        np.testing.assert_array_equal(sel["z"], z_all[sel["global_b"] - b0])
    b = eng.select_member(1)["global_b"]
    z = z_all[b - b0].astype(np.float64)
    N, rho = 24, 0.01
    pool = eng.candidate_pool(b, N, rho, pool_seed=77)
    xo, co = O.pool(z, N, 1.0, 77)
    ell_zone = np.abs(np.log(co / (1 - co)))          # |a| of the oracle's decision
    diff = pool["values"] != xo
    assert not (diff & (ell_zone > 1e-5 * (1 + np.abs(z)))).any()
    np.testing.assert_allclose(pool["confidence"], co, rtol=2e-6, atol=0)
    S = pool["S"]
    for k in range(N):
        gpu_units = list(pool["units"][k])
        ora_units = O.top_confident_units(xo[k], co[k], rho)
        assert len(gpu_units) == S == len(ora_units)
        if gpu_units != ora_units:
            # only near-equal confidences at the |S|-th place may swap
            thr = np.sort(co[k])[::-1][S - 1]
            for u in set(gpu_units) ^ set(ora_units):
                assert abs(co[k][abs(u) - 1] - thr) < 1e-6
    for d in (1, 7, 16):
        vars_ = eng.cube_variables(b, d)
        assert list(vars_) == O.lowest_confidence_vars(z, d)     # same fp32 z on both sides: exact
    eng.free()
    cnf.free()


def test_pool_large_S_units_only(G):
    """f1 at the shape of the paper's largest instance: |S| above one CTA's
    shared-memory sort (global-memory bitonic sort) and the units-only pool, drawn over the
    original variables of a normalised CNF in candidate groups; against the oracle's Eq.10-11
    on the same fp32 logits and against the full draw (identical units)."""
    inst = I.industrial(20_000, 80_000, 13)
    cnf0 = G.Cnf.from_instance(inst)
    cnf = cnf0.normalize(3)
    assert cnf.original_vars() == inst.n < cnf.n
    eng = G.Engine(cnf, 64, 8, 0.5, 3)
    eng.run()
    sel = eng.select_member(0)
    b, z = sel["global_b"], sel["z"][:inst.n].astype(np.float64)
    N, rho = 5, 0.3
    full = eng.candidate_pool(b, N, rho, pool_seed=9)
    part = eng.candidate_pool(b, N, rho, pool_seed=9, arrays=False)
    S = full["S"]
    assert S == part["S"] == 6000 > 4096
    np.testing.assert_array_equal(full["units"], part["units"])
    xo, co = O.pool(z, N, 1.0, 9)
    for k in range(N):
        gpu_units = list(full["units"][k])
        ora_units = O.top_confident_units(xo[k], co[k], rho)
        assert len(gpu_units) == S == len(ora_units)
        if gpu_units != ora_units:
            thr = np.sort(co[k])[::-1][S - 1]
            for u in set(gpu_units) ^ set(ora_units):
                assert abs(co[k][abs(u) - 1] - thr) < 1e-6
            # the order is descending confidence (ties to the lower index) up to fp32 ties
            cg = co[k][np.abs(gpu_units) - 1]
            assert (np.diff(cg) <= 1e-6).all()
    eng.free()
    cnf.free()
    cnf0.free()


def test_cubes(G):
    """Lemma 1 cube pins: pinned variables follow alpha = b mod 2^d, never move, and the
    engine matches the oracle with pins."""
    inst = I.random_ksat(60, 250, 3, 8)
    cubes = I.top_degree_vars(inst, 5)
    rep = parity.run_trajectory(G, inst, 64, 15, seed=2, cubes=cubes, stop_on_sat=False)
    assert rep.best_gpu == rep.best_oracle
    cnf = G.Cnf.from_instance(inst)
    eng = G.Engine(cnf, 64, 5, 0.5, 2, cubes=cubes)
    z0 = eng.get_iterate()[0]
    for _ in range(5):
        eng.step()
    z, _, _, _ = eng.get_iterate()
    x, r = eng.get_bits()
    idx = np.array(cubes) - 1
    np.testing.assert_array_equal(z[:, idx], z0[:, idx])
    for b in range(64):
        expect = [(b >> k) & 1 for k in range(5)]
        assert list(r[b, idx]) == expect and list(x[b, idx]) == expect


def test_sgd_and_tau(G):
    inst = I.random_ksat(50, 200, 3, 9)
    parity.one_step(G, inst, 64, 3, optimizer=1, lr=0.2)
    parity.one_step(G, inst, 64, 3, tau=0.5)
    rep = parity.run_trajectory(G, inst, 64, 20, seed=1, tau=1.7, stop_on_sat=False)
    assert rep.best_gpu == rep.best_oracle


@pytest.mark.parametrize("t", [0, 5])
def test_soft_mode_one_step(G, t):
    """SOFT mode: fp32 relaxed forward/backward vs the fp64 oracle."""
    inst = I.industrial(200, 900, 5)
    parity.one_step(G, inst, 64, t, mode=1)


def test_hub_path_exact(G):
    """Variables with > 256 occurrences are reduced through deterministic chunked
    partials; their signal G must still equal the oracle's exactly."""
    inst = I.industrial(3000, 60_000, 12, occ_exp=1.0)
    deg = I.degrees(inst)
    assert (deg > 256).sum() >= 2
    res = parity.one_step(G, inst, 64, 2)
    assert res["tie_x"] + res["tie_r"] <= 2


def test_full_size_sampled_C2(G):
    """configs[1] at full size in the bench launch configuration (B = 4096): one step, then
    the sampled members' Lambda, unsat counts and bits against the oracle computed for
    those members only (global RNG counters make members independent)."""
    inst = I.random_ksat(10_000, 42_000, 3, 0)
    f = O.Cnf(inst.n, inst.offsets, inst.lits)
    cnf = G.Cnf.from_instance(inst)
    eng = G.Engine(cnf, 4096, 50, 0.5, 0, debug=True)
    eng.step()
    lam = eng.get_loss()
    u, _ = eng.unsat_counts()
    x, r = eng.get_bits()
    Gg, _ = eng.get_grad()
    for b in (0, 1, 31, 32, 1000, 2047, 4095):
        st = O.State.init(inst.n, b, 1, 0)
        out = O.step(f, parity.oracle_cfg(0), st)
        ties = np.abs(out["a"][0]) <= 1e-5 * (1 + np.abs(st.reduced()[0][0]))
        if not ties.any():
            assert lam[b] == out["lam"][0]
            np.testing.assert_array_equal(Gg[b], out["G"][0].astype(np.int32))
        zo = st.reduced()[0][0]
        safe = np.abs(zo) > 1e-4 * np.maximum(1, np.abs(zo))
        np.testing.assert_array_equal(r[b][safe], out["r"][0][safe])
        if safe.all() and not ties.any():
            assert u[b] == out["unsat"][0]
    eng.free()


# ------------------------------------------------------------ f2: chain normalisation
def _oracle_normalize(inst, k):
    from oracle import normalize as N
    clauses = [inst.lits[inst.offsets[c]:inst.offsets[c + 1]].tolist() for c in range(inst.m)]
    return N.normalize(inst.n, clauses, k)


@pytest.mark.parametrize("which,k", [("appendix", 3), ("industrial", 3), ("industrial", 4),
                                     ("industrial", 8), ("wide", 5), ("wide", 32), ("narrow", 3)])
def test_normalize_matches_oracle(G, which, k):
    """f2 (Eq.6-9): the device chain encoding equals the oracle's phi'
    clause for clause, literal for literal (same auxiliary numbering), bit-exact."""
    inst = {"appendix": lambda: I.from_clauses("b", 4, [[1, -2, 3, 4], [-1, 3]]),
            "industrial": lambda: I.industrial(30_000, 120_000, 5),
            "wide": lambda: I.industrial(5_000, 20_000, 9, wmin=1, wmax=80, width_exp=0.5),
            "narrow": lambda: I.random_ksat(20_000, 80_000, 2, 3)}[which]()
    n2, phi2 = _oracle_normalize(inst, k)
    out = G.Cnf.from_instance(inst).normalize(k)
    assert out.n == n2 and out.num_aux == n2 - inst.n and out.m == len(phi2)
    off, lits = out.csr()
    np.testing.assert_array_equal(off, np.arange(len(phi2) + 1, dtype=np.int64) * k)
    np.testing.assert_array_equal(lits, np.array(phi2, np.int32).reshape(-1))
    info = out.info()
    assert info["max_width"] == k


def test_normalize_rejects_bad_k(G):
    c = G.Cnf.from_instance(I.random_ksat(10, 20, 3, 0))
    for k in (0, 2, 33):
        with pytest.raises(G.GaloisError):
            c.normalize(k)


def test_normalize_then_solve(G):
    """The paper's pipeline: normalise a planted mixed-width formula to 3-CNF,
    run the engine on phi', and project the best model to the original variables: it
    satisfies phi (Eq.9), checked by the oracle's exact counter on phi."""
    inst = I.industrial(200, 500, 4, planted=True, wmax=10)
    out = G.Cnf.from_instance(inst).normalize(3)
    eng = G.Engine(out, 1024, 200, 0.5, 1)
    rc = eng.run()
    best = eng.best_assignment()
    eng.free()
    assert rc == G.SAT and best["unsat"] == 0
    f = O.Cnf(inst.n, inst.offsets, inst.lits)
    assert O.unsat_count(f, best["values"][:inst.n]) == 0


def test_normalized_trajectory(G):
    """The normalised phi' of the solve test through the step-by-step parity harness for
    30 steps (north_star: trajectories within 1e-4). Longer runs of this instance leave
    the 1e-4 band: fp32-vs-fp64 drift grows ~x1.15/step through Adam's normalisation
    (a numpy fp32 emulation fed the oracle's own G drifts 1.9e-4 by step 34; DESIGN.md
    §Parity), so the first-SAT comparison lives on C1 (test_first_sat_matches_oracle_C1)."""
    n2, phi2 = _oracle_normalize(I.industrial(200, 500, 4, planted=True, wmax=10), 3)
    rep = parity.run_trajectory(G, I.from_clauses("phi'", n2, phi2), 1024, 30, seed=1, stop_on_sat=False)
    assert rep.best_gpu == rep.best_oracle, rep
    assert len(rep.resyncs) <= 8, rep.resyncs


def test_normalized_steps_31_to_50_identical_iterates(G):
    """Steps 31-50 of the same phi' (north_star's 50-step horizon), compared one step at a
    time from identical iterates (reading of the 50-step tolerance past the
    fp32 drift horizon): the engine runs its first 30 steps alone, then before each of
    steps 31..50 the sampled members' fp32 iterates go to the oracle, and X, Lambda, R,
    the unsat count of the previous rounding and z/m/v are held to the one-step bounds."""
    n2, phi2 = _oracle_normalize(I.industrial(200, 500, 4, planted=True, wmax=10), 3)
    inst = I.from_clauses("phi'", n2, phi2)
    cnf = G.Cnf.from_instance(inst)
    eng = G.Engine(cnf, 1024, 50, 0.5, 1)
    eng.enqueue(30)
    members = (0, 1, 7, 100, 333, 512, 777, 1023)
    rep = parity.stepwise_sampled(G, inst, eng, members, 20, seed=1)
    assert rep["compared"] >= len(members) * 20 - 4, rep
    eng.free()
    cnf.free()


# ------------------------------------------------------------------ f4: sub-batching
def _solve(G, inst, batch, steps, seed, **kw):
    cnf = G.Cnf.from_instance(inst)
    eng = G.Engine(cnf, batch, steps, 0.5, seed, **kw)
    rc = eng.run()
    best = eng.best_assignment()
    counts, b0 = eng.unsat_counts()
    info = eng.info()
    eng.free()
    return rc, (best["unsat"], best["step"], best["global_b"]), best["values"], counts, info


@pytest.mark.parametrize("K,sub", [(1, 1024), (4, 992), (3, 32)])
def test_subbatch_equals_full_batch(G, K, sub):
    """f4: windows of sub members give the full-batch result exactly — best
    (u, t, b), its bits, every member's last count and the step count (no SAT here,
    every window runs the whole budget; ragged last window)."""
    inst = I.random_ksat(300, 1290, 3, 5)
    B, T = 3000 if sub >= 512 else 200, 40
    full = _solve(G, inst, B, T, 7, check_interval=K)
    part = _solve(G, inst, B, T, 7, check_interval=K, sub_batch=sub)
    assert full[0] == part[0] == G.BUDGET
    assert full[1] == part[1]
    np.testing.assert_array_equal(full[2], part[2])
    np.testing.assert_array_equal(full[3], part[3])
    assert full[4] == part[4]


@pytest.mark.parametrize("sub", [256, 1024])
def test_subbatch_first_sat(G, sub):
    """SAT stop across windows: the first satisfying (step, member) of the full batch,
    its bits and the step count (windows after the SAT run at most t* steps)."""
    inst = I.random_ksat(50, 213, 3, 0)
    full = _solve(G, inst, 4096, 100, 0)
    part = _solve(G, inst, 4096, 100, 0, sub_batch=sub)
    assert full[0] == part[0] == G.SAT
    assert full[1] == part[1] and full[1][0] == 0
    np.testing.assert_array_equal(full[2], part[2])
    assert full[4]["steps_done"] == part[4]["steps_done"] and part[4]["stopped"]


def test_subbatch_cubes_and_nccl(G):
    """Windows keep global member indices: cube pins (alpha = b mod 2^d) and the NCCL
    MIN path (1-rank communicator) give the unwindowed result."""
    inst = I.random_ksat(200, 852, 3, 9)
    pins = [3, 17, 40, 41, 99]
    full = _solve(G, inst, 2048, 30, 2, cubes=pins)
    part = _solve(G, inst, 2048, 30, 2, cubes=pins, sub_batch=640)
    assert full[1] == part[1]
    np.testing.assert_array_equal(full[3], part[3])
    nid = G.galois_comm_unique_id()
    comm = _solve(G, inst, 2048, 30, 2, cubes=pins, sub_batch=640, nccl_id=nid)
    assert comm[1] == full[1]
    np.testing.assert_array_equal(comm[2], full[2])


def test_subbatch_gating_and_sizing(G):
    import torch
    inst = I.random_ksat(1000, 4200, 3, 1)
    cnf = G.Cnf.from_instance(inst)
    with pytest.raises(G.GaloisError):
        G.Engine(cnf, 4096, 10, 0.5, 0, sub_batch=100)          # not a multiple of 32
    eng = G.Engine(cnf, 4096, 10, 0.5, 0, sub_batch=1024)
    with pytest.raises(G.GaloisError) as e:
        eng.step()
    assert e.value.code == G.E_STATE
    eng.free()
    per = cnf.bytes_per_member()
    assert per >= 12 * inst.n + inst.lits.size // 8
    # exact window sizing (galois_engine_window_bytes mirrors prepare's allocation)
    wb = cnf.window_bytes(992, 10)
    assert per * 992 <= wb < cnf.window_bytes(1024, 10)
    assert cnf.sub_batch_for(wb, 10) == 992
    assert cnf.sub_batch_for(wb - 1, 10) == 960
    assert cnf.window_bytes(32, 1000) - cnf.window_bytes(32, 0) >= 1000 * 8 - 256   # adam constants per step
    assert cnf.window_bytes(32, 10) >= 32 * 12 * inst.n + 8 * inst.n + 4 * inst.L   # z/m/v, compact X/R, E at W = 1
    with pytest.raises(G.GaloisError):
        cnf.sub_batch_for(1000, 10)                                          # not even 32 members
    # the resident footprint scales with sub_batch, not B
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    big = G.Engine(cnf, 1 << 20, 1, 0.5, 0, sub_batch=2048)
    big.info()
    used = free0 - torch.cuda.mem_get_info()[0]
    big.free()
    assert used < 4 * per * 2048 + (64 << 20), used


def test_subbatch_theta_sel_and_pool(G):
    """f4 + f1: a sub-batched run keeps theta_sel (min and max of every member's last count)
    and its final iterate, so select_member, the candidate pool and the cube variables
    equal those of the resident batch (no SAT stop: every window runs the budget)."""
    inst = I.random_ksat(300, 1290, 3, 5)
    out = []
    for sub in (0, 1024):
        cnf = G.Cnf.from_instance(inst)
        eng = G.Engine(cnf, 3000, 25, 0.5, 3, sub_batch=sub)
        assert eng.run() == G.BUDGET
        sel = [eng.select_member(r) for r in (0, 1)]
        b0 = sel[0]["global_b"]
        pool = eng.candidate_pool(b0, 16, 0.02, 5)
        cubes = eng.cube_variables(b0, 7)
        out.append((sel, pool, cubes))
        eng.free()
    (s0, p0, c0), (s1, p1, c1) = out
    for r in (0, 1):
        assert s0[r]["global_b"] == s1[r]["global_b"] and s0[r]["unsat"] == s1[r]["unsat"]
        np.testing.assert_array_equal(s0[r]["z"], s1[r]["z"])
    np.testing.assert_array_equal(p0["values"], p1["values"])
    np.testing.assert_array_equal(p0["units"], p1["units"])
    np.testing.assert_array_equal(c0, c1)
