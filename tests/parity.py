"""GPU-vs-oracle parity harness (used by the -m gpu tests and __graft_entry__.smoke()).

The CUDA engine (through the C ABI) and the fp64 oracle are run on the same seeded
instance and compared step by step:
  * integers bit-exact: sample bits X_t, rounding bits R_t, Lambda_b (ST), the signal
    G (ST), unsat counts, best (u*, t*, b*);
  * fp32 vs fp64: gradient g1 within relative 1e-5 from identical iterates, z within
    1e-4 max(1, |z|) along free-running trajectories (north_star's tolerances).
Where floating point decides a bit, both sides decide [a >= 0] but in different precision;
a mismatch is accepted only inside the tie zone |a_oracle| <= tie,
and that member's oracle iterate is then re-synchronised from the engine (exact map,
oracle.State.from_reduced). Every accepted tie is counted and reported.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from oracle import oracle as O


@dataclass
class Report:
    steps: int = 0
    ties_x: int = 0
    ties_r: int = 0
    resyncs: List[tuple] = field(default_factory=list)
    max_z_err: float = 0.0
    max_g1_rel: float = 0.0
    best_gpu: Optional[tuple] = None
    best_oracle: Optional[tuple] = None


def oracle_cfg(seed, mode=0, tau=1.0, lr=0.5, optimizer=0, pins=()):
    return O.Config(mode=mode, optimizer=optimizer, lr=lr, tau=tau, seed=seed, pins=[p - 1 for p in pins])


def z_tol(z, rel):
    return rel * np.maximum(1.0, np.abs(z))


def compare_bits(name, gpu, ora, margin, tie_zone):
    """gpu, ora: uint8 [nb, n]; margin: |a| of the oracle's decision. Returns the mask of
    members that had an accepted tie; raises on a mismatch outside the tie zone."""
    diff = gpu != ora
    if not diff.any():
        return np.zeros(gpu.shape[0], bool)
    bad = diff & ~(margin <= tie_zone)
    if bad.any():
        b, v = np.argwhere(bad)[0]
        raise AssertionError(f"{name} bit mismatch at member {b} var {v}: gpu {gpu[b, v]} oracle {ora[b, v]} "
                             f"margin {margin[b, v]:.3e} > tie zone {np.broadcast_to(tie_zone, margin.shape)[b, v]:.3e}")
    return diff.any(axis=1)


def run_trajectory(G, inst, batch, steps, seed=0, *, mode=0, tau=1.0, lr=0.5, optimizer=0, cubes=(),
                   check_interval=1, z_rel=1e-4, compare_every=1, stop_on_sat=True) -> Report:
    """Free-running trajectory parity (re-sync only at accepted ties)."""
    f = O.Cnf(inst.n, inst.offsets, inst.lits)
    cfg = oracle_cfg(seed, mode, tau, lr, optimizer, cubes)
    cnf = G.Cnf.from_instance(inst)
    eng = G.Engine(cnf, batch, steps, lr, seed, mode=mode, tau=tau, optimizer=optimizer, cubes=cubes,
                   debug=True, check_interval=check_interval)
    rep = Report()
    st = O.State.init(inst.n, 0, batch, seed)
    z0, _, _, t0 = eng.get_iterate()
    assert t0 == 0
    zo = st.reduced()[0]
    err = np.abs(z0 - zo)
    assert (err <= 1e-6 * np.maximum(1, np.abs(zo))).all(), f"init z error {err.max()}"
    x_next, r = eng.get_bits()
    ro, uo = O.round_and_check(f, cfg, st)
    ties = compare_bits("R_0", r, ro, np.abs(zo), z_tol(zo, 1e-6))
    u_gpu, _ = eng.unsat_counts()
    ok = ~ties
    np.testing.assert_array_equal(u_gpu[ok], uo[ok])
    best_o = (int(uo.min()), 0, int(np.argmin(uo)))
    for t in range(1, steps + 1):
        if stop_on_sat and best_o[0] == 0:
            break
        x_used = x_next
        z_pre = st.reduced()[0]
        rc = eng.step()
        out = O.step(f, cfg, st)
        rep.steps = t
        # sample bits of this step: [a >= 0] with a = (z + ell)/tau
        tie_x = compare_bits(f"X_{t}", x_used, out["xhat"], np.abs(out["a"]), z_tol(z_pre, z_rel) / tau)
        rep.ties_x += int(tie_x.sum())
        zg, mg, vg, tg = eng.get_iterate()
        assert tg == t, (tg, t)
        zo = st.reduced()[0]
        x_next, r = eng.get_bits()
        tie_r = compare_bits(f"R_{t}", r, out["r"], np.abs(zo), z_tol(zo, z_rel))
        rep.ties_r += int(tie_r.sum())
        same = ~(tie_x | tie_r)
        if mode == 0:
            lam = eng.get_loss()
            np.testing.assert_array_equal(lam[~tie_x], out["lam"][~tie_x])
            Gg, g1 = eng.get_grad()
            np.testing.assert_array_equal(Gg[~tie_x], out["G"][~tie_x].astype(np.int32))
        zerr = np.abs(zg - zo)[same]
        if zerr.size:
            rep.max_z_err = max(rep.max_z_err, float(zerr.max()))
            assert (zerr <= z_tol(zo[same], z_rel)).all(), f"z drift at step {t}: {zerr.max()}"
        is_check = (t % check_interval == 0) or t == steps
        if is_check:
            u_gpu, _ = eng.unsat_counts()
            np.testing.assert_array_equal(u_gpu[same], out["unsat"][same])
        # re-sync members with accepted ties from the engine (exact map)
        for b in np.nonzero(~same)[0]:
            rs = O.State.from_reduced(zg[b:b + 1], mg[b:b + 1], vg[b:b + 1], t)
            st.theta[b] = rs.theta[0]; st.mom[b] = rs.mom[0]; st.vel[b] = rs.vel[0]
            rep.resyncs.append((t, int(b)))
            if is_check:
                # the engine's count on its own bits must equal the exact count of those bits
                assert u_gpu[b] == O.unsat_count(f, r[b]), "checker mismatch on re-synced member"
                out["unsat"][b] = u_gpu[b]
        if is_check:
            b = int(np.argmin(out["unsat"]))
            if out["unsat"][b] < best_o[0]:
                best_o = (int(out["unsat"][b]), t, b)
        if rc == G.SAT:
            break
    best = eng.best_assignment()
    rep.best_gpu = (best["unsat"], best["step"], best["global_b"])
    rep.best_oracle = best_o
    assert O.unsat_count(f, best["values"]) == best["unsat"], "best bits do not reproduce the best count"
    eng.free()
    cnf.free()
    return rep


def one_step(G, inst, batch, t, seed=0, *, mode=0, tau=1.0, lr=0.5, optimizer=0, cubes=(), steps=None,
             warm=3, rng_seed=1):
    """Identical-iterate parity: put the same (fp32-representable) iterate into both
    sides at step t, advance one step, compare everything with tight tolerances."""
    steps = max(steps or 0, t + 1)
    f = O.Cnf(inst.n, inst.offsets, inst.lits)
    cfg = oracle_cfg(seed, mode, tau, lr, optimizer, cubes)
    cnf = G.Cnf.from_instance(inst)
    eng = G.Engine(cnf, batch, steps, lr, seed, mode=mode, tau=tau, optimizer=optimizer, cubes=cubes, debug=True)
    rng = np.random.default_rng(rng_seed)
    z = (rng.normal(size=(batch, inst.n)) * 2.5).astype(np.float32)
    m = (rng.normal(size=(batch, inst.n)) * 0.3).astype(np.float32)
    v = (np.abs(rng.normal(size=(batch, inst.n))) * 0.2).astype(np.float32) if t > 0 else np.zeros_like(m)
    if t == 0:
        m[:] = 0
    eng.set_iterate(z, m, v, t)
    st = O.State.from_reduced(z, m, v, t)
    x_used, _ = eng.get_bits()
    eng.step()
    out = O.step(f, cfg, st)
    # identical z; only ell differs (lg2.approx, |d ell| <~ 2.3e-7 + 2.4e-7 |ell|)
    tie_x = compare_bits("X", x_used, out["xhat"], np.abs(out["a"]), (1e-6 + 1e-6 * np.abs(z)) / tau)
    x_next, r = eng.get_bits()
    zg, mg, vg, tg = eng.get_iterate()
    assert tg == t + 1
    zo, mo, vo = st.reduced()
    res = dict(tie_x=int(tie_x.sum()))

    def _where(bad, *arrs):
        b, v = np.argwhere(bad)[0]
        return f"member {b} var {v}: " + ", ".join(f"{a[b, v]!r}" for a in arrs)

    okx = ~tie_x[:, None] & np.ones((1, inst.n), bool)
    Gg, g1 = eng.get_grad()
    lam = eng.get_loss()
    go = out["grad1"]
    e = np.exp(-np.abs(out["a"]))
    pq = e / (1 + e) ** 2
    if mode == 0:
        np.testing.assert_array_equal(Gg[~tie_x], out["G"][~tie_x].astype(np.int32))
        np.testing.assert_array_equal(lam[~tie_x], out["lam"][~tie_x])
        dg = 1e-5 * np.abs(go) + 1e-30            # north_star: relative 1e-5 (fp32 vs fp64)
        nz = okx & (go != 0)
        res["max_g1_rel"] = float((np.abs(g1 - go)[nz] / np.abs(go)[nz]).max()) if nz.any() else 0.0
    else:
        # SOFT: fp32 sums of reals; absolute bound on the scale A_v = sum |E| <= degree
        deg = np.bincount(np.abs(inst.lits) - 1, minlength=inst.n).astype(np.float64)
        dg = 1e-5 * (deg[None, :] + 1.0) * pq / tau + 1e-30
        assert (np.abs(lam - out["lam"]) <= 1e-5 * (inst.m + 1)).all(), "soft lambda mismatch"
    bad_g = (np.abs(g1 - go) > dg) & okx
    assert not bad_g.any(), "g1 mismatch " + _where(bad_g, g1, go, out["G"], out["a"])
    # propagate the gradient tolerance through the optimiser (first-order error bounds)
    m_prev = m.astype(np.float64); v_prev = v.astype(np.float64)
    tol_m = tol_v = None
    if optimizer == 0:
        b1, b2, eps = 0.9, 0.999, 1e-8
        tol_m = 1e-6 * (b1 * np.abs(m_prev) + (1 - b1) * np.abs(go)) + (1 - b1) * dg + 1e-30
        tol_v = 1e-6 * (b2 * v_prev + (1 - b2) * go * go) + (1 - b2) * 2 * np.abs(go) * dg + 1e-30
        c1 = lr / (1 - b1 ** (t + 1)); c2 = 1 / np.sqrt(1 - b2 ** (t + 1))
        denom = np.sqrt(vo) * c2 + eps
        dz = np.abs(2 * c1 * mo / denom)
        tol_z = 2 * c1 * tol_m / denom + dz * 0.5 * tol_v / np.maximum(vo, 1e-300) + 1e-6 * dz \
            + 1e-6 * np.maximum(1, np.abs(zo))
    else:
        tol_z = 2 * lr * dg + 1e-6 * np.abs(2 * lr * go) + 1e-6 * np.maximum(1, np.abs(zo))
    tie_r = compare_bits("R", r, out["r"], np.abs(zo), tol_z)
    res["tie_r"] = int(tie_r.sum())
    okm = ~(tie_x | tie_r)[:, None] & np.ones((1, inst.n), bool)
    if tol_m is not None:
        bad_m = (np.abs(mg - mo) > tol_m) & okm
        assert not bad_m.any(), "m mismatch " + _where(bad_m, mg, mo, m, go, out["G"])
        bad_v = (np.abs(vg - vo) > tol_v) & okm
        assert not bad_v.any(), "v mismatch " + _where(bad_v, vg, vo, v, go)
    bad_z = (np.abs(zg - zo) > tol_z) & okm
    if bad_z.any():
        ratio = np.where(okm, np.abs(zg - zo) / tol_z, 0)
        b, v_ = np.unravel_index(np.argmax(ratio), ratio.shape)
        raise AssertionError(f"z mismatch: {int(bad_z.sum())} elements, worst ratio {ratio[b, v_]:.2f} at "
                             f"member {b} var {v_}: zg {zg[b, v_]!r} zo {zo[b, v_]!r} z {z[b, v_]!r} m {m[b, v_]!r} "
                             f"v {v[b, v_]!r} mo {mo[b, v_]!r} vo {vo[b, v_]!r} g {go[b, v_]!r} a {out['a'][b, v_]!r}")
    res["x_next"] = x_next
    res["out"] = out
    res["eng_state"] = (zg, mg, vg)
    eng.free()
    cnf.free()
    return res
