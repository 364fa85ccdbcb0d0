"""Seeded synthetic CNF generators (recipe in DESIGN.md §Inputs).

This module holds NO arithmetic of the method: it only draws clauses. It is the one
module shared by the tests, bench.py and the oracle harness (the oracle itself and
the CUDA path never import each other).  Every generator uses numpy's
Generator(PCG64(seed)).

Shapes follow the paper's workloads: uniform random k-SAT near the phase transition
(configs C1-C3 of BASELINE.json) and industrial-like instances with power-law
variable occurrence and mixed clause widths (Table 2's instance shapes, P:402-496;
config C4), plus a cube split over the highest-degree variables (Lemma 1, P:245-253;
config C5).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np


@dataclass
class Instance:
    """Clause-major CSR: clause c = lits[offsets[c]:offsets[c+1]] (DIMACS, 1-based)."""
    name: str
    n: int
    offsets: np.ndarray            # int64 [m+1]
    lits: np.ndarray               # int32 [L]
    planted: Optional[np.ndarray] = None   # uint8 [n] hidden model of a planted instance
    pins: List[int] = field(default_factory=list)  # 1-based cube variables (C5)

    @property
    def m(self) -> int:
        return len(self.offsets) - 1

    @property
    def L(self) -> int:
        return int(self.offsets[-1])

    def clauses(self) -> List[List[int]]:
        return [self.lits[self.offsets[c]:self.offsets[c + 1]].tolist() for c in range(self.m)]


def from_clauses(name: str, n: int, clauses: Sequence[Sequence[int]]) -> Instance:
    offsets = np.zeros(len(clauses) + 1, dtype=np.int64)
    if clauses:
        offsets[1:] = np.cumsum([len(c) for c in clauses])
    lits = np.array([l for c in clauses for l in c], dtype=np.int32)
    return Instance(name, n, offsets, lits)


def _distinct_rows(rng: np.random.Generator, m: int, k: int, n: int) -> np.ndarray:
    """m rows of k distinct variables (0-based), uniform, in draw order."""
    if k > n:
        raise ValueError("clause width exceeds variable count")
    rows = rng.integers(0, n, size=(m, k), dtype=np.int64)
    while True:
        s = np.sort(rows, axis=1)
        bad = np.nonzero((s[:, 1:] == s[:, :-1]).any(axis=1))[0] if k > 1 else np.zeros(0, np.int64)
        if bad.size == 0:
            return rows
        rows[bad] = rng.integers(0, n, size=(bad.size, k), dtype=np.int64)


def _signed(rng: np.random.Generator, vars0: np.ndarray) -> np.ndarray:
    neg = rng.random(vars0.shape) < 0.5
    return np.where(neg, -(vars0 + 1), vars0 + 1).astype(np.int32)


def _satisfied_by(lits: np.ndarray, x: np.ndarray) -> np.ndarray:
    """Boolean: does each row of literals contain a literal true under x (generation-time
    rejection of planted instances only)."""
    v = np.abs(lits) - 1
    val = x[v].astype(bool)
    return np.where(lits > 0, val, ~val).any(axis=1)


def random_ksat(n: int, m: int, k: int, seed: int = 0, planted: bool = False) -> Instance:
    """G1 (and G2 when planted): each clause draws k distinct variables uniformly, each
    literal negated with probability 1/2. Planted: a hidden x* is drawn first and clauses
    it falsifies are rejected (so the instance is SAT by construction; easier than an
    unplanted one)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    xstar = rng.integers(0, 2, size=n, dtype=np.uint8) if planted else None
    out = np.zeros((0, k), dtype=np.int32)
    while out.shape[0] < m:
        need = m - out.shape[0]
        draw = int(need * (1.2 if planted else 1.0)) + 8 if planted else need
        rows = _signed(rng, _distinct_rows(rng, draw, k, n))
        if planted:
            rows = rows[_satisfied_by(rows, xstar)]
        out = np.concatenate([out, rows[:need]], axis=0)
    offsets = np.arange(0, m * k + 1, k, dtype=np.int64)
    name = f"{'planted-' if planted else ''}{k}sat-n{n}-m{m}-s{seed}"
    return Instance(name, n, offsets, out.reshape(-1).astype(np.int32), xstar)


def industrial(n: int, m: int, seed: int = 0, planted: bool = False,
               wmin: int = 2, wmax: int = 30, width_exp: float = 2.5, occ_exp: float = 0.8) -> Instance:
    """G3: scale-free industrial-like CNF (after Ansotegui, Bonet, Levy, IJCAI 2009).
    Width w ~ P(w) ∝ w^-2.5 on [2, 30]; variables i.i.d. with P(i) ∝ i^-0.8, within-clause
    duplicates resampled; a seeded permutation of variable ids; fair-coin signs.
    Planted: reject clauses falsified by a hidden x*."""
    rng = np.random.Generator(np.random.PCG64(seed))
    ws = np.arange(wmin, wmax + 1)
    pw = ws.astype(np.float64) ** (-width_exp)
    pw /= pw.sum()
    pv = np.arange(1, n + 1, dtype=np.float64) ** (-occ_exp)
    cdf = np.cumsum(pv)
    cdf /= cdf[-1]
    perm = rng.permutation(n)
    xstar = rng.integers(0, 2, size=n, dtype=np.uint8) if planted else None

    def draw_vars(count):
        idx = np.searchsorted(cdf, rng.random(count), side="right")
        return np.minimum(idx, n - 1).astype(np.int64)

    widths_all: List[np.ndarray] = []
    lits_all: List[np.ndarray] = []
    have = 0
    while have < m:
        need = m - have
        draw = need if not planted else int(need * 1.1) + 16
        w = rng.choice(ws, size=draw, p=pw)
        off = np.zeros(draw + 1, dtype=np.int64)
        off[1:] = np.cumsum(w)
        cid = np.repeat(np.arange(draw, dtype=np.int64), w)
        vars0 = draw_vars(int(off[-1]))
        # resample within-clause duplicates (keep the first occurrence in draw order)
        while True:
            key = cid * n + vars0
            order = np.argsort(key, kind="stable")
            ks = key[order]
            dup_sorted = np.zeros(ks.size, dtype=bool)
            dup_sorted[1:] = ks[1:] == ks[:-1]
            dup = order[dup_sorted]
            if dup.size == 0:
                break
            vars0[dup] = draw_vars(dup.size)
        vars0 = perm[vars0]
        lits = _signed(rng, vars0)
        if planted:
            v = np.abs(lits) - 1
            val = xstar[v].astype(bool)
            true_lit = np.where(lits > 0, val, ~val).astype(np.int64)
            sat = np.add.reduceat(true_lit, off[:-1]) > 0
            keep = np.nonzero(sat)[0][:need]
            w = w[keep]
            lits = _gather_clauses(lits, off, keep)
        else:
            w = w[:need]
        widths_all.append(np.asarray(w, dtype=np.int64))
        lits_all.append(np.asarray(lits, dtype=np.int32))
        have += len(w)
    widths = np.concatenate(widths_all)[:m]
    lits = np.concatenate(lits_all)[: int(widths.sum())]
    offsets = np.zeros(m + 1, dtype=np.int64)
    offsets[1:] = np.cumsum(widths)
    name = f"{'planted-' if planted else ''}industrial-n{n}-m{m}-s{seed}"
    return Instance(name, n, offsets, lits.astype(np.int32), xstar)


def industrial_large(n: int, m: int, seed: int = 0, wmin: int = 2, wmax: int = 30,
                     width_exp: float = 2.5, occ_exp: float = 0.8) -> Instance:
    """G3 at the paper's largest scale (48,505,464 variables, 130,975,382 clauses —
    reading R17), vectorised by width so it draws ~0.5G literals in minutes: widths
    P(w) ∝ w^-2.5 on [2, 30] in random clause order; variables by the inverse CDF of the
    continuous law f(x) ∝ x^-0.8 on [1, n + 1) (index floor(x) - 1: G3's discrete
    P(i) ∝ i^-0.8 up to the discretisation of the density), rows with a repeated variable
    redrawn whole; a seeded permutation of variable ids; fair-coin signs. Not the same
    stream as `industrial` (C4 stays as it is)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    ws = np.arange(wmin, wmax + 1)
    pw = ws.astype(np.float64) ** (-width_exp)
    pw /= pw.sum()
    widths = rng.choice(ws, size=m, p=pw).astype(np.int64)
    offsets = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(widths, out=offsets[1:])
    lits = np.empty(int(offsets[-1]), dtype=np.int32)
    top = float(n + 1) ** (1.0 - occ_exp) - 1.0
    expo = 1.0 / (1.0 - occ_exp)
    perm = rng.permutation(n).astype(np.int32)

    def draw(shape):
        x = (1.0 + rng.random(shape) * top) ** expo
        return np.minimum(x.astype(np.int64) - 1, n - 1)

    for w in ws:
        idx = np.nonzero(widths == w)[0]
        if idx.size == 0:
            continue
        rows = draw((idx.size, int(w)))
        while True:
            srt = np.sort(rows, axis=1)
            bad = np.nonzero((srt[:, 1:] == srt[:, :-1]).any(axis=1))[0]
            if bad.size == 0:
                break
            rows[bad] = draw((bad.size, int(w)))
        signs = np.where(rng.random(rows.shape) < 0.5, -1, 1).astype(np.int32)
        vals = (perm[rows] + 1) * signs
        pos = offsets[idx][:, None] + np.arange(int(w), dtype=np.int64)[None, :]
        lits[pos.ravel()] = vals.ravel()
        del rows, srt, signs, vals, pos
    return Instance(f"industrial-large-n{n}-m{m}-s{seed}", n, offsets, lits)


def _gather_clauses(lits: np.ndarray, off: np.ndarray, keep: np.ndarray) -> np.ndarray:
    w = off[keep + 1] - off[keep]
    starts = np.repeat(off[keep], w)
    within = np.arange(int(w.sum()), dtype=np.int64) - np.repeat(np.cumsum(w) - w, w)
    return lits[starts + within]


def degrees(inst: Instance) -> np.ndarray:
    return np.bincount(np.abs(inst.lits).astype(np.int64) - 1, minlength=inst.n)


def top_degree_vars(inst: Instance, d: int) -> List[int]:
    """The d highest-degree variables (1-based), ties to the lower index, ascending."""
    deg = degrees(inst)
    order = np.lexsort((np.arange(inst.n), -deg))
    return sorted(int(v) + 1 for v in order[:d])


def cube_split(n: int = 100_000, m: int = 426_000, d: int = 16, seed: int = 0,
               planted: bool = False) -> Instance:
    """G4: random 3-SAT plus d cube pins on the d highest-degree variables (reading R14);
    member b takes cube alpha = b mod 2^d (Lemma 1)."""
    inst = random_ksat(n, m, 3, seed, planted=planted)
    inst.pins = top_degree_vars(inst, d)
    inst.name = f"cube{d}-" + inst.name
    return inst


# --------------------------------------------------------------------------- #
# BASELINE.json configs                                      #
# --------------------------------------------------------------------------- #

CONFIGS = {
    # name: (generator thunk, batch, steps)
    "C1": (lambda: random_ksat(50, 213, 3, 0), 1024, 100),
    "C2": (lambda: random_ksat(10_000, 42_000, 3, 0), 4096, 50),
    "C3a": (lambda: random_ksat(2_000, 42_000, 5, 0), 16_384, 50),
    "C3b": (lambda: random_ksat(500, 43_895, 7, 0), 16_384, 50),
    "C4": (lambda: industrial(1_000_000, 4_200_000, 0), 1024, 50),
    "C5": (lambda: cube_split(100_000, 426_000, 16, 0), 65_536, 50),
}


def config(name: str):
    gen, batch, steps = CONFIGS[name]
    return gen(), batch, steps
