"""Pins of the fp64 oracle against things other than itself (-m "not gpu").

Each test names what it pins and where that comes from: the paper's printed numbers
(tests/golden/*.json, each with its citation), closed forms, library routines
(scipy distributions, torch.optim.Adam, torch autograd of Eq.3-5), and brute force
over all 2^n assignments (oracle/bruteforce.py).
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import bruteforce as BF
from oracle import oracle as O
from paper_2603_28796_b200 import instances as I

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def random_cnf(rng, n, m, wmin=1, wmax=4, distinct=True):
    clauses = []
    for _ in range(m):
        w = int(rng.integers(wmin, wmax + 1))
        if distinct:
            vs = rng.choice(n, size=min(w, n), replace=False) + 1
        else:
            vs = rng.integers(1, n + 1, size=w)
        signs = np.where(rng.random(len(vs)) < 0.5, -1, 1)
        clauses.append([int(s * v) for s, v in zip(signs, vs)])
    return clauses


# ----------------------------------------------------------------------------- RNG
def test_philox_known_answers():
    """Random123 KAT vectors (tests/golden/philox4x32_10_kat.json)."""
    for vec in golden("philox4x32_10_kat.json")["vectors"]:
        out = O.philox4x32_10([int(x, 16) for x in vec["ctr"]], [int(x, 16) for x in vec["key"]])
        assert [f"{int(x):08x}" for x in out] == vec["out"]


def test_uniform_is_open_and_complement_exact():
    """u = (k + 1/2) 2^-23 from the low 23 bits; u + (1-u) == 1 exactly (reading R2)."""
    for w in [0, 1, 511, 512, 0x7FFFFF, 0x800000, 0x7FFFFFFF, 0x80000000, 0xFFFFFE00, 0xFFFFFFFF, 0x12345678]:
        u, ub = O.uniform(w), O.uniform_complement(w)
        k = w & 0x7FFFFF
        assert u == (k + 0.5) / 2 ** 23
        assert u + ub == 1.0
        assert 0.0 < u < 1.0 and 0.0 < ub < 1.0
        # both are exact in binary32 (24 significant bits)
        assert float(np.float32(u)) == u and float(np.float32(ub)) == ub


def test_logistic_noise_distribution():
    """ell = ln u - ln(1-u) is Logistic(0,1) = the law of g1 - g0 for iid Gumbel(0,1)
    (Eq.3; reading R2): KS test against scipy's logistic, variance pi^2/3."""
    from scipy import stats
    ell = O.noise(200, 0, 400, seed=7, t=3).ravel()
    assert abs(ell.mean()) < 0.03
    assert abs(ell.var() / (math.pi ** 2 / 3) - 1) < 0.03
    assert stats.kstest(ell, "logistic").pvalue > 1e-3
    # the difference of two independent Gumbel(0,1) draws has the same law
    rng = np.random.default_rng(0)
    g = rng.gumbel(size=(2, 200000))
    assert stats.ks_2samp(ell, g[1] - g[0]).pvalue > 1e-3


def test_logistic_noise_closed_form():
    """ell(k) = ln((2k+1) / (2^24 - 2k - 1)) for the 23-bit k of the selected word."""
    seed, v, b, t = 12345, 3, 9, 5
    w = O.philox4x32_10([v, b >> 2, t, 1], [seed & 0xFFFFFFFF, seed >> 32])
    k = int(w[b & 3]) & 0x7FFFFF
    expect = math.log((2 * k + 1) / (2 ** 24 - 2 * k - 1))
    assert abs(O.lib().oracle_logistic_noise(v, b, t, seed) - expect) < 1e-12


def test_init_logits_standard_normal():
    """theta ~ N(0,1) i.i.d. (P:137 'independently and randomly initialized'; reading R1)."""
    from scipy import stats
    th = O.init_logits(300, 0, 300, seed=11)
    for j in (0, 1):
        x = th[..., j].ravel()
        assert abs(x.mean()) < 0.02 and abs(x.var() - 1) < 0.03
        assert stats.kstest(x, "norm").pvalue > 1e-3
    assert abs(np.corrcoef(th[..., 0].ravel(), th[..., 1].ravel())[0, 1]) < 0.02


def test_init_is_per_global_member():
    """Member b's draws depend on the global index only (sharding invariance)."""
    a = O.init_logits(17, 0, 12, seed=3)
    b = O.init_logits(17, 5, 7, seed=3)
    np.testing.assert_array_equal(a[5:], b)


# ---------------------------------------------------------------- clause polynomial
@pytest.mark.parametrize("w", list(range(1, 17)))
def test_clause_polynomial_boolean_exhaustive(w):
    """Eq.2 on Boolean inputs equals Boolean OR, for all 2^w inputs."""
    m = 2 ** w
    bits = ((np.arange(m)[:, None] >> np.arange(w)[None, :]) & 1).astype(np.float64)
    f = O.Cnf(w, np.arange(0, m * w + 1, w), np.tile(np.arange(1, w + 1), m))
    U, E = O.clause_products(f, bits.ravel())
    any_true = bits.any(axis=1)
    np.testing.assert_array_equal(U, (~any_true).astype(np.float64))       # U = 1 iff all false
    # E_i = 1 iff every OTHER slot is false
    others_true = bits.sum(axis=1, keepdims=True) - bits
    np.testing.assert_array_equal(E.reshape(m, w), (others_true == 0).astype(np.float64))


def test_relaxed_or_printed_value():
    """two literals at 0.5 give 1 - 0.5*0.5 = 0.75."""
    g = golden("relaxed_or.json")
    f = O.Cnf.from_clauses(2, [[1, 2]])
    U, _ = O.clause_products(f, np.array(g["s"]))
    assert 1 - U[0] == g["C"]


def test_three_term_expansion():
    """a or b or c = a + b + c - ab - bc - ca + abc on random reals."""
    rng = np.random.default_rng(1)
    f = O.Cnf.from_clauses(3, [[1, 2, 3]])
    for _ in range(200):
        a, b, c = rng.random(3)
        U, E = O.clause_products(f, np.array([a, b, c]))
        assert abs((1 - U[0]) - (a + b + c - a * b - b * c - c * a + a * b * c)) < 1e-14
        assert abs(E[0] - (1 - b) * (1 - c)) < 1e-15
        assert abs(E[1] - (1 - a) * (1 - c)) < 1e-15
        assert abs(E[2] - (1 - a) * (1 - b)) < 1e-15


def test_exclusive_product_with_true_slots():
    """E must not be formed by division: with s_i = 1 the siblings' E are 0 and E_i is
    the product of the others (product annihilation)."""
    f = O.Cnf.from_clauses(3, [[1, 2, 3]])
    U, E = O.clause_products(f, np.array([1.0, 0.0, 0.0]))
    assert U[0] == 0.0 and list(E) == [1.0, 0.0, 0.0]


# ------------------------------------------------------------ Appendix B example
@pytest.mark.parametrize("polarity", ["phi_prime_eq7", "phi_prime_as_printed"])
@pytest.mark.parametrize("z5", [0, 1])
def test_appendix_b_forward(polarity, z5):
    """x_hat = (1,0,0,1) gives C = (1,1,0) and L = -2 on phi' (either polarity of
    the second clause, reading R16; the auxiliary z1 = x5 either value)."""
    g = golden("appendix_b.json")
    f = O.Cnf.from_clauses(g["n_normalized"], g[polarity])
    x = np.array(g["x_hat"] + [z5], dtype=np.float64)
    lam, U, E, G = O.member_signal(f, x)
    assert list(1 - U) == g["C"]
    assert lam - f.m == g["loss"]          # L = sum U - m = -sum C
    assert O.unsat_count(f, x.astype(np.uint8)) == 1


def test_appendix_b_original_formula():
    g = golden("appendix_b.json")
    f = O.Cnf.from_clauses(g["n_original"], g["phi"])
    lam, U, E, G = O.member_signal(f, np.array(g["x_hat"], dtype=np.float64))
    assert lam == 1.0                      # (not x1 or x3) is violated by (1,0,0,1)


@pytest.mark.parametrize("z5,G_expect", [(0, [-1, 0, 2, 0, 0]), (1, [-1, 0, 2, 1, 0])])
def test_appendix_b_backward(z5, G_expect):
    """Straight-through signal on the paper's example (derived by hand from Eq.2/Eq.4):
    clause 3 (not x1 or x3 or x3) is all-false, so G_1 = -1 and G_3 = +2 (x3 appears
    twice); clause 2 gives x4 the signal z5. With p = (0.7, 0.3, 0.2, 0.9):
    dL/dtheta_{.,1} = -G p q = (+0.21, 0, -0.32, ...)."""
    g = golden("appendix_b.json")
    f = O.Cnf.from_clauses(5, g["phi_prime_eq7"])
    lam, U, E, G = O.member_signal(f, np.array(g["x_hat"] + [z5], dtype=np.float64))
    np.testing.assert_array_equal(G, G_expect)
    p = np.array(g["y_second_entries"] + [0.5])
    grad1 = -G * p * (1 - p)
    assert abs(grad1[0] - 0.21) < 1e-15 and abs(grad1[2] + 0.32) < 1e-15


def test_spec_backward_example():
    """(x1 or x2), x_hat = (0,0), p = 0.4 -> dL/dtheta_{1,1} = -0.24."""
    g = golden("spec_backward_example.json")
    f = O.Cnf.from_clauses(g["n"], g["clauses"])
    lam, U, E, G = O.member_signal(f, np.array(g["x_hat"], dtype=np.float64))
    p = np.array(g["p"])
    np.testing.assert_allclose(-G * p * (1 - p), g["dL_dtheta1"], rtol=0, atol=1e-15)


# --------------------------------------------------------------- brute force pins
@pytest.mark.parametrize("seed", range(6))
def test_checker_and_loss_vs_bruteforce(seed):
    """For every x in {0,1}^n (n <= 12): the exact checker equals the naive Boolean
    count, the ST loss Lambda equals it too, and Lambda = 0 iff x satisfies the
    CNF (north_star). Duplicated literals and tautologies included (reading R12)."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 13))
    clauses = random_cnf(rng, n, int(rng.integers(1, 4 * n)), 1, 5, distinct=(seed % 2 == 0))
    f = O.Cnf.from_clauses(n, clauses)
    for x in BF.all_assignments(n):
        u = BF.naive_unsat(clauses, x)
        assert O.unsat_count(f, np.array(x, np.uint8)) == u
        lam, U, E, G = O.member_signal(f, np.array(x, dtype=np.float64))
        assert lam == u
        assert (lam == 0) == (u == 0)


@pytest.mark.parametrize("seed", range(6))
def test_flip_delta_identity(seed):
    """ST signal structure (brute force + closed form): for duplicate-free clauses,
    G_v(x) = (2 x_v - 1) (u(x xor e_v) - u(x)) for every x and v, i.e. the signal is
    WalkSAT's break - make count. Pins E, the sign sigma and the per-variable sum."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(3, 11))
    clauses = random_cnf(rng, n, int(rng.integers(1, 5 * n)), 1, 5, distinct=True)
    f = O.Cnf.from_clauses(n, clauses)
    for x in BF.all_assignments(n):
        _, _, _, G = O.member_signal(f, np.array(x, dtype=np.float64))
        u = BF.naive_unsat(clauses, x)
        for v in range(n):
            y = list(x)
            y[v] ^= 1
            assert G[v] == (2 * x[v] - 1) * (BF.naive_unsat(clauses, y) - u)


def test_sec41_example():
    """(x1 or not x2) and (not x1 or x3) is satisfied by (T,F,T)."""
    g = golden("sec41_example.json")
    f = O.Cnf.from_clauses(g["n"], g["clauses"])
    assert O.unsat_count(f, np.array(g["model"], np.uint8)) == 0
    assert BF.naive_unsat(g["clauses"], g["model"]) == 0


def test_contradiction_never_satisfied():
    f = O.Cnf.from_clauses(1, [[1], [-1]])
    assert O.unsat_count(f, np.array([0], np.uint8)) == 1
    assert O.unsat_count(f, np.array([1], np.uint8)) == 1


# -------------------------------------------------------------- gradient pins
def _soft_loss(clauses, p):
    """L = -sum_c C_c with C = 1 - prod(1 - s), s = p or 1 - p (Eq.2, Eq.5) — plain numpy."""
    total = 0.0
    for c in clauses:
        prod = 1.0
        for l in c:
            s = p[abs(l) - 1] if l > 0 else 1.0 - p[abs(l) - 1]
            prod *= (1.0 - s)
        total -= (1.0 - prod)
    return total


@pytest.mark.parametrize("seed", range(4))
def test_soft_gradient_central_differences(seed):
    """SOFT mode: the analytic dL/dtheta_{b,v,1} of the oracle matches
    central finite differences of L(theta) at fixed noise, h = 1e-5, with the absolute
    term the survey's C.3 derives (|fd - g| <= 1e-6 |g| + 1e-12 (m+1)/h)."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 16))
    clauses = random_cnf(rng, n, int(rng.integers(1, 4 * n)), 1, 5, distinct=(seed % 2 == 0))
    f = O.Cnf.from_clauses(n, clauses)
    cfg = O.Config(mode=1, seed=seed, tau=[1.0, 0.7, 1.3, 2.0][seed])
    nb = 3
    st = O.State(rng.normal(size=(nb, n, 2)) * 1.5)
    th0 = st.theta.copy()
    out = O.step(f, cfg, st)                        # grad1 evaluated at th0, noise t = 1
    ell = O.noise(n, 0, nb, cfg.seed, 1)
    h = 1e-5
    m = len(clauses)
    for b in range(nb):
        for v in range(n):
            for j, sgn in ((1, 1.0), (0, -1.0)):
                vals = []
                for d in (+h, -h):
                    th = th0[b].copy()
                    th[v, j] += d
                    p = 1.0 / (1.0 + np.exp(-(th[:, 1] - th[:, 0] + ell[b]) / cfg.tau))
                    vals.append(_soft_loss(clauses, p))
                fd = (vals[0] - vals[1]) / (2 * h)
                g = sgn * out["grad1"][b, v]        # dL/dtheta_0 = -dL/dtheta_1
                assert abs(fd - g) <= 1e-6 * abs(g) + 1e-12 * (m + 1) / h, (b, v, j, fd, g)


def _torch_paper_step(clauses, n, theta, opt, ell, tau):
    """Eq.3-5 in PyTorch, the paper's implementation language, with autograd
    doing the backward: y = softmax((Theta + g)/tau) with g = (0, ell), the ST one-hot
    x = y_hard - y.detach() + y (ties to class 1), s = x[.,1] for a positive literal and
    x[.,0] for a negated one, C = 1 - prod(1 - s), L = -sum C, then Adam."""
    import torch
    nb = theta.shape[0]
    g = torch.stack([torch.zeros_like(ell), ell], dim=-1)
    y = torch.softmax((theta + g) / tau, dim=-1)
    hard1 = (y[..., 1] >= y[..., 0]).to(y.dtype)
    y_hard = torch.stack([1 - hard1, hard1], dim=-1)
    x = y_hard - y.detach() + y
    loss = torch.zeros(nb, dtype=theta.dtype)
    for c in clauses:
        prod = torch.ones(nb, dtype=theta.dtype)
        for l in c:
            s = x[:, abs(l) - 1, 1] if l > 0 else x[:, abs(l) - 1, 0]
            prod = prod * (1 - s)
        loss = loss - (1 - prod)
    opt.zero_grad()
    loss.sum().backward()
    grad = theta.grad.detach().clone()
    opt.step()
    return loss.detach(), hard1.detach(), grad


@pytest.mark.parametrize("seed,tau", [(0, 1.0), (1, 1.0), (2, 0.5)])
def test_straight_through_adam_trajectory_vs_torch_autograd(seed, tau):
    """The oracle's closed-form ST gradient + two-logit Adam equals, step by step, the
    paper's method written in PyTorch autograd + torch.optim.Adam(lr=0.5) (App. A):
    theta, the hard samples and the losses over 25 steps, in fp64."""
    import torch
    rng = np.random.default_rng(seed)
    n = 12
    clauses = random_cnf(rng, n, 50, 2, 4, distinct=(seed != 1))
    f = O.Cnf.from_clauses(n, clauses)
    cfg = O.Config(seed=seed, tau=tau)
    nb = 6
    st = O.State.init(n, 0, nb, cfg.seed)
    theta = torch.tensor(st.theta.copy(), dtype=torch.float64, requires_grad=True)
    opt = torch.optim.Adam([theta], lr=cfg.lr, betas=(cfg.beta1, cfg.beta2), eps=cfg.eps)
    for t in range(1, 26):
        ell = torch.tensor(O.noise(n, 0, nb, cfg.seed, t))
        loss, hard1, grad = _torch_paper_step(clauses, n, theta, opt, ell, tau)
        out = O.step(f, cfg, st)
        np.testing.assert_array_equal(out["xhat"], hard1.numpy().astype(np.uint8))
        np.testing.assert_allclose(out["lam"] - len(clauses), loss.numpy(), rtol=0, atol=1e-12)
        # (theta drifts apart by ~1e-8, see below, so the gradients agree to ~1e-8 relative)
        np.testing.assert_allclose(out["grad1"], grad[..., 1].numpy(), rtol=1e-6, atol=1e-12)
        np.testing.assert_allclose(-out["grad1"], grad[..., 0].numpy(), rtol=1e-6, atol=1e-12)
        # torch's softmax backward forms y1 (d1 - y0 d0 - y1 d1), which cancels when
        # y1 -> 1 (relative error ~ 1e-16 / y0); Adam's normalisation turns that into an
        # absolute theta difference of order lr * 1e-8. A wrong term would be O(lr).
        np.testing.assert_allclose(st.theta, theta.detach().numpy(), rtol=0, atol=1e-7)


def test_plain_gradient_step_vs_torch_sgd():
    """optimizer = 1 is theta <- theta - lr g, i.e. torch.optim.SGD(lr)."""
    import torch
    rng = np.random.default_rng(5)
    n = 10
    clauses = random_cnf(rng, n, 40, 2, 3)
    f = O.Cnf.from_clauses(n, clauses)
    cfg = O.Config(seed=5, optimizer=1, lr=0.3)
    st = O.State.init(n, 0, 4, cfg.seed)
    theta = torch.tensor(st.theta.copy(), dtype=torch.float64, requires_grad=True)
    opt = torch.optim.SGD([theta], lr=cfg.lr)
    for t in range(1, 11):
        ell = torch.tensor(O.noise(n, 0, 4, cfg.seed, t))
        _torch_paper_step(clauses, n, theta, opt, ell, cfg.tau)
        O.step(f, cfg, st)
        np.testing.assert_allclose(st.theta, theta.detach().numpy(), rtol=1e-12, atol=1e-13)


def test_adam_first_step_closed_form():
    """from zero moments, Adam's first step is -lr g / (|g| + eps) per logit."""
    rng = np.random.default_rng(9)
    n = 8
    f = O.Cnf.from_clauses(n, random_cnf(rng, n, 30, 2, 3))
    cfg = O.Config(seed=9)
    st = O.State.init(n, 0, 5, cfg.seed)
    th0 = st.theta.copy()
    out = O.step(f, cfg, st)
    g1 = out["grad1"]
    np.testing.assert_allclose(st.theta[..., 1] - th0[..., 1], -cfg.lr * g1 / (np.abs(g1) + cfg.eps),
                               rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(st.theta[..., 0] - th0[..., 0], cfg.lr * g1 / (np.abs(g1) + cfg.eps),
                               rtol=1e-12, atol=1e-15)


def test_zero_gradient_leaves_theta_unchanged():
    """g = 0 everywhere leaves theta unchanged (empty formula)."""
    f = O.Cnf(5, np.zeros(1, np.int64), np.zeros(0, np.int32))
    st = O.State.init(5, 0, 3, 1)
    th0 = st.theta.copy()
    for _ in range(3):
        out = O.step(f, O.Config(seed=1), st)
        assert (out["lam"] == 0).all() and (out["unsat"] == 0).all()
    np.testing.assert_array_equal(st.theta, th0)


def test_reduced_form_is_exact():
    """Reading R24: the engine's reduced iterate (z = theta_1 - theta_0, m_1, v_1) evolves
    exactly like the two-logit form, because g_0 = -g_1 keeps m_0 = -m_1, v_0 = v_1."""
    rng = np.random.default_rng(3)
    n = 15
    f = O.Cnf.from_clauses(n, random_cnf(rng, n, 60, 2, 4))
    cfg = O.Config(seed=3)
    a = O.State.init(n, 0, 8, cfg.seed)
    z, m, v = a.reduced()
    b = O.State.from_reduced(z, m, v, 0)
    for _ in range(30):
        oa = O.step(f, cfg, a)
        ob = O.step(f, cfg, b)
        np.testing.assert_array_equal(oa["xhat"], ob["xhat"])
        np.testing.assert_allclose(a.reduced()[0], b.reduced()[0], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(a.mom[..., 0], -a.mom[..., 1], rtol=0, atol=0)
        np.testing.assert_allclose(a.vel[..., 0], a.vel[..., 1], rtol=0, atol=0)


# --------------------------------------------------------------- run-level pins
def test_unit_clause_sanity():
    """phi = (x1), B = 4: after training theta_{1,1} > theta_{1,0} for all members."""
    f = O.Cnf.from_clauses(1, [[1]])
    st = O.State.init(1, 0, 4, 0)
    for _ in range(10):
        O.step(f, O.Config(seed=0), st)
    assert (st.theta[:, 0, 1] > st.theta[:, 0, 0]).all()


def test_empty_formula_sat_at_t0():
    f = O.Cnf(3, np.zeros(1, np.int64), np.zeros(0, np.int32))
    res = O.run(f, O.Config(), 0, 4, T=5)
    assert res["best_unsat"] == 0 and res["best_t"] == 0 and res["best_b"] == 0 and res["steps"] == 0


def test_lambda_equals_checker_on_sample_and_bounds():
    """Loss bounds: 0 <= Lambda_b <= m, integer in ST mode, equal to the exact
    unsat count of the hard sample x_hat."""
    inst = I.random_ksat(40, 170, 3, 4)
    f = O.Cnf(inst.n, inst.offsets, inst.lits)
    st = O.State.init(inst.n, 0, 16, 4)
    for _ in range(5):
        out = O.step(f, O.Config(seed=4), st)
        for b in range(16):
            assert out["lam"][b] == O.unsat_count(f, out["xhat"][b])
        assert ((out["lam"] >= 0) & (out["lam"] <= f.m)).all()


@pytest.mark.parametrize("k", [3, 5, 7])
def test_t0_statistics(k):
    """Closed form at t = 0 on uniform random k-SAT: E[u/m] = 2^-k for an unbiased random
    assignment; the mean density of the exclusive products E is 2^(1-k)."""
    inst = I.random_ksat(400, 4000, k, 1)
    f = O.Cnf(inst.n, inst.offsets, inst.lits)
    cfg = O.Config(seed=2)
    st = O.State.init(inst.n, 0, 64, cfg.seed)
    r, u = O.round_and_check(f, cfg, st)
    assert abs(u.mean() / f.m - 2.0 ** -k) < 0.15 * 2.0 ** -k
    dens = []
    for b in range(16):
        _, _, E, _ = O.member_signal(f, r[b].astype(np.float64))
        dens.append(E.mean())
    assert abs(np.mean(dens) - 2.0 ** (1 - k)) < 0.1 * 2.0 ** (1 - k)


def test_cube_pins_lemma1():
    """Lemma 1: with d pins and B = 2^d members, every full assignment is
    consistent with exactly one member's cube; pinned variables keep their value and
    their logits never move."""
    d, n = 4, 12
    rng = np.random.default_rng(8)
    clauses = random_cnf(rng, n, 40, 2, 3)
    f = O.Cnf.from_clauses(n, clauses)
    pins = [1, 4, 7, 10]
    cfg = O.Config(seed=8, pins=pins)
    st = O.State.init(n, 0, 2 ** d, cfg.seed)
    th0 = st.theta.copy()
    for _ in range(4):
        out = O.step(f, cfg, st)
        cubes = {tuple(out["r"][b, pins]) for b in range(2 ** d)}
        assert len(cubes) == 2 ** d
        np.testing.assert_array_equal(out["xhat"][:, pins], out["r"][:, pins])
        for b in range(2 ** d):
            assert tuple(out["r"][b, pins]) == tuple((b >> r) & 1 for r in range(d))
    np.testing.assert_array_equal(st.theta[:, pins], th0[:, pins])
    for x in BF.all_assignments(d):
        owners = [b for b in range(2 ** d) if all(((b >> r) & 1) == x[r] for r in range(d))]
        assert len(owners) == 1


def test_run_matches_stepwise_best_and_determinism():
    """run() is the step loop with checks at t = 0, K, 2K, ..., T and the lexicographic
    (u, t, b) best; two runs are bit-identical, and members are independent of
    the slice they run in (sharding invariance)."""
    inst = I.random_ksat(30, 128, 3, 2)
    f = O.Cnf(inst.n, inst.offsets, inst.lits)
    cfg = O.Config(seed=6)
    T, K, nb = 12, 3, 10
    res = O.run(f, cfg, 0, nb, T, K)
    res2 = O.run(f, cfg, 0, nb, T, K)
    assert (res["best_unsat"], res["best_t"], res["best_b"]) == (res2["best_unsat"], res2["best_t"], res2["best_b"])
    np.testing.assert_array_equal(res["state"].theta, res2["state"].theta)
    st = O.State.init(inst.n, 0, nb, cfg.seed)
    _, u = O.round_and_check(f, cfg, st)
    best = (int(u.min()), 0, int(np.argmin(u)))
    for t in range(1, T + 1):
        out = O.step(f, cfg, st)
        if t % K == 0 or t == T:
            b = int(np.argmin(out["unsat"]))
            if out["unsat"][b] < best[0]:
                best = (int(out["unsat"][b]), t, b)
        if best[0] == 0:
            break
    assert best == (res["best_unsat"], res["best_t"], res["best_b"])
    lo = O.run(f, cfg, 0, 4, T, K)["state"].theta
    hi = O.run(f, cfg, 4, 6, T, K)["state"].theta
    if res["best_unsat"] > 0:
        np.testing.assert_array_equal(np.concatenate([lo, hi]), res["state"].theta)


def test_planted_instances_are_satisfied_by_their_model():
    for inst in (I.random_ksat(60, 250, 3, 1, planted=True), I.industrial(300, 1200, 2, planted=True)):
        f = O.Cnf(inst.n, inst.offsets, inst.lits)
        assert O.unsat_count(f, inst.planted) == 0


def test_industrial_large_generator_laws():
    """PL's generator (instances.industrial_large, the paper's largest size P:559): widths in
    [2, 30] with P(w) ~ w^-2.5, distinct variables within a clause, literals in range, both
    signs, occurrence counts falling with the pre-permutation rank (P(i) ~ i^-0.8), and the
    same formula for the same seed."""
    n, m = 200_000, 840_000
    a = I.industrial_large(n, m, 7)
    b = I.industrial_large(n, m, 7)
    np.testing.assert_array_equal(a.offsets, b.offsets)
    np.testing.assert_array_equal(a.lits, b.lits)
    w = np.diff(a.offsets)
    assert w.min() >= 2 and w.max() <= 30 and a.m == m
    ws = np.arange(2, 31)
    pw = ws ** -2.5 / (ws ** -2.5).sum()
    freq = np.bincount(w, minlength=31)[2:] / m
    assert np.abs(freq - pw).max() < 3e-3
    v = np.abs(a.lits)
    assert v.min() >= 1 and v.max() <= n and (a.lits < 0).mean() == pytest.approx(0.5, abs=2e-3)
    cid = np.repeat(np.arange(m), w)
    key = cid * (n + 1) + v
    assert np.unique(key).size == key.size                          # no variable twice in a clause
    deg = np.sort(I.degrees(a))[::-1]
    # rank-frequency of a ~ i^-0.8 law: the top 1 % of variables carry far more than 1 %
    top = deg[: n // 100].sum() / deg.sum()
    assert 0.2 < top < 0.6, top


# --------------------------------------------- f1 / f3: pool, partial assignments, cubes
def test_extract_partial_spec_example():
    """SPEC extract_partial: top-|S| by descending confidence, Eq.11 literals."""
    g = golden("spec_pool_examples.json")
    assert O.top_confident_units(g["x"], g["conf"], g["rho"]) == g["units"]
    assert len(O.top_confident_units([1] * 100, [0.7] * 100, 0.0005)) == 1      # |S| floors at 1
    assert O.top_confident_units([1, 0, 1], [0.8, 0.8, 0.8], 1.0) == [1, -2, 3]   # ties -> lower index


def test_branch_vars_spec_example():
    """SPEC select_branch_vars: lowest noise-free confidence, ties lower index."""
    g = golden("spec_pool_examples.json")
    th = np.array(g["theta"], dtype=np.float64)
    assert O.lowest_confidence_vars(th[:, 1] - th[:, 0], g["d"]) == g["vars"]
    assert O.lowest_confidence_vars(np.zeros(6), 3) == [1, 2, 3]                   # all equal -> first d


def test_pool_statistics_and_saturation():
    """Eq.10: with z = 0 the samples are fair coins and the confidence
    sigma(|ell|) = max(U, 1-U) for U uniform has mean 3/4 (closed form); with z = +20
    every candidate is all-true with confidence ~1; pools are deterministic."""
    x, c = O.pool(np.zeros(500), 40, 1.0, 17)
    assert abs(x.mean() - 0.5) < 0.01 and abs(c.mean() - 0.75) < 0.005
    assert (c >= 0.5).all() and (c <= 1.0).all()
    x2, c2 = O.pool(np.zeros(500), 40, 1.0, 17)
    np.testing.assert_array_equal(x, x2)
    x3, _ = O.pool(np.zeros(500), 40, 1.0, 18)
    assert (x3 != x).any()
    xs, cs = O.pool(np.full(300, 20.0), 10, 1.0, 3)
    # |ell| <= ln(2^24) = 16.6 with 23-bit uniforms, so a >= 3.4: all true, confidence ~1
    assert xs.all() and (cs > 0.96).all() and cs.mean() > 0.9999


def test_select_member_rules():
    """theta_sel: min loss and max loss, ties to the lower member."""
    counts = np.array([5, 2, 7, 2, 7])
    assert O.select_member(counts, 100, 0) == (101, 2)
    assert O.select_member(counts, 100, 1) == (102, 7)


# ------------------------------------------------- clause normalisation (NEXT f2)
from oracle import normalize as N  # noqa: E402


def test_normalize_appendix_b():
    """Appendix B: phi -> phi' with z_1 = x_5; Eq.7's polarity (R16)."""
    g = golden("appendix_b.json")
    n2, phi2 = N.normalize(g["n_original"], g["phi"], 3)
    assert n2 == g["n_normalized"] and phi2 == g["phi_prime_eq7"]


@pytest.mark.parametrize("u", range(1, 12))
def test_normalize_eq7_shape(u):
    """Eq.7: a u-literal clause (u > 3) becomes u-2 clauses with u-3
    auxiliaries f_1..f_{u-3}; the first is (l1 l2 f1), the last (-f_{u-3} l_{u-1} l_u);
    u <= 3 is padded by duplication."""
    lits = [(-1) ** i * (i + 1) for i in range(u)]
    n2, phi2 = N.normalize(u, [lits], 3)
    assert all(len(c) == 3 for c in phi2)
    if u <= 3:
        assert n2 == u and phi2 == [lits + [lits[-1]] * (3 - u)]
        return
    assert n2 - u == u - 3 and len(phi2) == u - 2
    f = list(range(u + 1, n2 + 1))
    assert phi2[0] == [lits[0], lits[1], f[0]]
    assert phi2[-1] == [-f[-1], lits[-2], lits[-1]]
    for j in range(1, u - 3):
        assert phi2[j] == [-f[j - 1], lits[j + 1], f[j]]


def _models(n, clauses):
    return {tuple(x) for x in BF.all_assignments(n) if BF.naive_unsat(clauses, x) == 0}


@pytest.mark.parametrize("k", [3, 4, 5])
@pytest.mark.parametrize("seed", range(5))
def test_normalize_projection_bruteforce(k, seed):
    """Eq.9, strengthened: for every x over the original variables,
    x |= phi  <=>  some extension (x, f) |= phi'; and the first n bits of every model of
    phi' are a model of phi. Exhaustive on small random formulas, widths 1..8."""
    rng = np.random.default_rng(100 * k + seed)
    n = int(rng.integers(2, 7))
    clauses = random_cnf(rng, n, int(rng.integers(1, 4)), 1, 8, distinct=False)
    n2, phi2 = N.normalize(n, clauses, k)
    assert all(len(c) == k for c in phi2)
    assert n2 - n <= 12
    m1 = _models(n, clauses)
    m2 = _models(n2, phi2)
    assert {x[:n] for x in m2} == m1


@pytest.mark.parametrize("k", [3, 4, 7])
def test_normalize_literal_conservation(k):
    """Every original literal occurs exactly once in its chain, in order,
    plus only auxiliaries and padding duplicates; each auxiliary occurs once positive,
    once negative (the chain link)."""
    rng = np.random.default_rng(k)
    n = 40
    clauses = random_cnf(rng, n, 60, 1, 20, distinct=True)
    n2, phi2 = N.normalize(n, clauses, k)
    flat = [l for c in phi2 for l in c]
    aux = [l for l in flat if abs(l) > n]
    assert sorted(set(abs(l) for l in aux)) == list(range(n + 1, n2 + 1))
    for v in range(n + 1, n2 + 1):
        assert aux.count(v) == 1 and aux.count(-v) == 1
    expect_aux = sum(max(0, -(-(len(c) - 2) // (k - 2)) - 1) if len(c) > k else 0 for c in clauses)
    assert n2 - n == expect_aux
    # originals in order, dropping padding duplicates of the last literal of each chain
    pos = 0
    for c in clauses:
        got = []
        while len(got) < len(c):
            got.extend(l for l in phi2[pos] if abs(l) <= n)
            pos += 1
        assert got[:len(c)] == c and all(l == c[-1] for l in got[len(c):])
    assert pos == len(phi2)
