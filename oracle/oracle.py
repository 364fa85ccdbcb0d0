"""ctypes wrapper of the fp64 CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py — never by the product package.
It shares no code with the CUDA path.  See oracle.c's header for the citations.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c with plain gcc -O2 (no fast-math) and OpenMP."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-D_DEFAULT_SOURCE", "-fPIC", "-shared",
                               "-fopenmp", "-Wall", "-Wno-unknown-pragmas", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Cnf(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("m", ctypes.c_int64),
                ("offsets", ctypes.c_void_p), ("lits", ctypes.c_void_p)]


class _Config(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("optimizer", ctypes.c_int32),
                ("lr", ctypes.c_double), ("tau", ctypes.c_double),
                ("beta1", ctypes.c_double), ("beta2", ctypes.c_double), ("eps", ctypes.c_double),
                ("seed", ctypes.c_uint64), ("num_pins", ctypes.c_int32),
                ("pin_vars", ctypes.c_void_p)]


class _StepOut(ctypes.Structure):
    _fields_ = [("a", ctypes.c_void_p), ("xhat", ctypes.c_void_p), ("lam", ctypes.c_void_p),
                ("G", ctypes.c_void_p), ("grad1", ctypes.c_void_p), ("r", ctypes.c_void_p),
                ("unsat", ctypes.c_void_p)]


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        _lib.oracle_philox4x32_10.argtypes = [P, P, P]
        _lib.oracle_uniform.argtypes = [ctypes.c_uint32]
        _lib.oracle_uniform.restype = ctypes.c_double
        _lib.oracle_uniform_complement.argtypes = [ctypes.c_uint32]
        _lib.oracle_uniform_complement.restype = ctypes.c_double
        _lib.oracle_init_logits.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64, P]
        _lib.oracle_logistic_noise.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64]
        _lib.oracle_logistic_noise.restype = ctypes.c_double
        _lib.oracle_noise.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64,
                                      ctypes.c_int32, P]
        _lib.oracle_clause_products.argtypes = [P, P, P, P]
        _lib.oracle_member_signal.argtypes = [P, P, P, P, P, P]
        _lib.oracle_member_signal.restype = ctypes.c_double
        _lib.oracle_unsat_count.argtypes = [P, P]
        _lib.oracle_unsat_count.restype = ctypes.c_int64
        _lib.oracle_step.argtypes = [P, P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, P, P, P, P]
        _lib.oracle_round_and_check.argtypes = [P, P, ctypes.c_int64, ctypes.c_int64, P, P, P]
        _lib.oracle_run.argtypes = [P, P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                    P, P, P, P, P, P, P, P]
        _lib.oracle_run.restype = ctypes.c_int32
        _lib.oracle_pool.argtypes = [P, ctypes.c_int32, ctypes.c_int32, ctypes.c_double, ctypes.c_uint64, P, P]
        _lib.oracle_num_threads.restype = ctypes.c_int32
        _lib.oracle_set_num_threads.argtypes = [ctypes.c_int32]
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


class Cnf:
    """A CNF in clause-major CSR form: clause c = lits[offsets[c]:offsets[c+1]],
    DIMACS-signed 1-based literals."""

    def __init__(self, n: int, offsets, lits):
        self.n = int(n)
        self.offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        self.lits = np.ascontiguousarray(lits, dtype=np.int32)
        self.m = len(self.offsets) - 1
        self._c = _Cnf(self.n, self.m, self.offsets.ctypes.data, self.lits.ctypes.data)

    @classmethod
    def from_clauses(cls, n: int, clauses: Sequence[Sequence[int]]) -> "Cnf":
        offsets = np.zeros(len(clauses) + 1, dtype=np.int64)
        offsets[1:] = np.cumsum([len(c) for c in clauses])
        lits = np.array([l for c in clauses for l in c], dtype=np.int32)
        return cls(n, offsets, lits)

    @property
    def L(self) -> int:
        return int(self.offsets[-1])

    def ref(self):
        return ctypes.byref(self._c)


@dataclass
class Config:
    mode: int = 0          # 0 straight-through (paper), 1 fully soft (debug)
    optimizer: int = 0     # 0 Adam, 1 plain gradient step
    lr: float = 0.5
    tau: float = 1.0
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    seed: int = 0
    pins: Sequence[int] = ()   # 0-based variables, ascending

    def _c(self):
        self._pins = np.ascontiguousarray(sorted(self.pins), dtype=np.int32)
        return _Config(self.mode, self.optimizer, self.lr, self.tau, self.beta1, self.beta2,
                       self.eps, self.seed & 0xFFFFFFFFFFFFFFFF, len(self._pins),
                       self._pins.ctypes.data if len(self._pins) else None)


def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def uniform(word: int) -> float:
    return lib().oracle_uniform(int(word) & 0xFFFFFFFF)


def uniform_complement(word: int) -> float:
    return lib().oracle_uniform_complement(int(word) & 0xFFFFFFFF)


def init_logits(n: int, b0: int, nb: int, seed: int) -> np.ndarray:
    theta = np.zeros((nb, n, 2), dtype=np.float64)
    lib().oracle_init_logits(n, b0, nb, seed & 0xFFFFFFFFFFFFFFFF, _ptr(theta))
    return theta


def noise(n: int, b0: int, nb: int, seed: int, t: int) -> np.ndarray:
    ell = np.zeros((nb, n), dtype=np.float64)
    lib().oracle_noise(n, b0, nb, seed & 0xFFFFFFFFFFFFFFFF, t, _ptr(ell))
    return ell


def clause_products(f: Cnf, s: np.ndarray):
    s = np.ascontiguousarray(s, dtype=np.float64)
    U = np.zeros(f.m, dtype=np.float64)
    E = np.zeros(f.L, dtype=np.float64)
    lib().oracle_clause_products(f.ref(), _ptr(s), _ptr(U), _ptr(E))
    return U, E


def member_signal(f: Cnf, xval: np.ndarray):
    """Returns (Lambda, U[m], E[L], G[n]) for one member with variable values xval."""
    xval = np.ascontiguousarray(xval, dtype=np.float64)
    s = np.zeros(max(f.L, 1)); U = np.zeros(max(f.m, 1)); E = np.zeros(max(f.L, 1)); G = np.zeros(max(f.n, 1))
    lam = lib().oracle_member_signal(f.ref(), _ptr(xval), _ptr(s), _ptr(U), _ptr(E), _ptr(G))
    return lam, U[:f.m], E[:f.L], G[:f.n]


def unsat_count(f: Cnf, r) -> int:
    r = np.ascontiguousarray(r, dtype=np.uint8)
    return int(lib().oracle_unsat_count(f.ref(), _ptr(r)))


class State:
    """Oracle iterate for members b0 .. b0+nb-1: Theta, Adam moments ([nb][n][2], fp64)
    and the step counter t."""

    def __init__(self, theta: np.ndarray, mom=None, vel=None, t: int = 0, b0: int = 0):
        self.theta = np.ascontiguousarray(theta, dtype=np.float64)
        self.mom = np.zeros_like(self.theta) if mom is None else np.ascontiguousarray(mom, dtype=np.float64)
        self.vel = np.zeros_like(self.theta) if vel is None else np.ascontiguousarray(vel, dtype=np.float64)
        self.t = int(t)
        self.b0 = int(b0)

    @property
    def nb(self) -> int:
        return self.theta.shape[0]

    @classmethod
    def init(cls, n: int, b0: int, nb: int, seed: int) -> "State":
        return cls(init_logits(n, b0, nb, seed), b0=b0)

    @classmethod
    def from_reduced(cls, z, m, v, t: int, b0: int = 0) -> "State":
        """Exact map from the engine's reduced iterate (z = theta_1 - theta_0, m = m_1,
        v = v_1; layout [nb][n]) to the two-logit form: theta_1 = z/2, theta_0 = -z/2,
        m_0 = -m_1, v_0 = v_1 (every quantity depends on theta only through z, and
        Adam is odd in g; reading R24)."""
        z = np.asarray(z, dtype=np.float64); m = np.asarray(m, dtype=np.float64)
        v = np.asarray(v, dtype=np.float64)
        theta = np.stack([-z / 2, z / 2], axis=-1)
        mom = np.stack([-m, m], axis=-1)
        vel = np.stack([v, v], axis=-1)
        return cls(theta, mom, vel, t, b0)

    def reduced(self):
        return (self.theta[..., 1] - self.theta[..., 0], self.mom[..., 1].copy(), self.vel[..., 1].copy())

    def copy(self) -> "State":
        return State(self.theta.copy(), self.mom.copy(), self.vel.copy(), self.t, self.b0)


def step(f: Cnf, cfg: Config, st: State) -> dict:
    """Advance st by one step (t -> t+1) in place; returns the step's records."""
    nb, n = st.nb, f.n
    out = dict(a=np.zeros((nb, n)), xhat=np.zeros((nb, n), np.uint8), lam=np.zeros(nb),
               G=np.zeros((nb, n)), grad1=np.zeros((nb, n)), r=np.zeros((nb, n), np.uint8),
               unsat=np.zeros(nb, np.int64))
    so = _StepOut(*[out[k].ctypes.data for k in ("a", "xhat", "lam", "G", "grad1", "r", "unsat")])
    c = cfg._c()
    st.t += 1
    lib().oracle_step(f.ref(), ctypes.byref(c), st.b0, nb, st.t, _ptr(st.theta), _ptr(st.mom),
                      _ptr(st.vel), ctypes.byref(so))
    return out


def round_and_check(f: Cnf, cfg: Config, st: State):
    nb, n = st.nb, f.n
    r = np.zeros((nb, n), np.uint8)
    u = np.zeros(nb, np.int64)
    c = cfg._c()
    lib().oracle_round_and_check(f.ref(), ctypes.byref(c), st.b0, nb, _ptr(st.theta), _ptr(r), _ptr(u))
    return r, u


def run(f: Cnf, cfg: Config, b0: int, nb: int, T: int, K: int = 1) -> dict:
    n = f.n
    theta = np.zeros((nb, n, 2)); mom = np.zeros_like(theta); vel = np.zeros_like(theta)
    bu = ctypes.c_int64(); bt = ctypes.c_int32(); bb = ctypes.c_int64()
    best_r = np.zeros(max(n, 1), np.uint8)
    last = np.zeros(max(nb, 1), np.int64)
    c = cfg._c()
    steps = lib().oracle_run(f.ref(), ctypes.byref(c), b0, nb, T, K, _ptr(theta), _ptr(mom), _ptr(vel),
                             ctypes.byref(bu), ctypes.byref(bt), ctypes.byref(bb), _ptr(best_r), _ptr(last))
    return dict(steps=int(steps), best_unsat=int(bu.value), best_t=int(bt.value), best_b=int(bb.value),
                best_r=best_r[:n].copy(), last_unsat=last[:nb].copy(),
                state=State(theta, mom, vel, int(steps), b0))


# ------------------------------------------------- what the CPU stage consumes (f1, f3)
def select_member(counts: np.ndarray, b0: int, rule: int = 0):
    """theta_sel (P:102 min loss / P:210 max loss) over exact unsat counts, ties to the
    lower member. Returns (global member, count)."""
    counts = np.asarray(counts)
    best = None
    for i, u in enumerate(counts):
        key = (u, i) if rule == 0 else (-u, i)
        if best is None or key < best[0]:
            best = (key, i)
    i = best[1]
    return b0 + i, int(counts[i])


def pool(z, N: int, tau: float, pool_seed: int):
    """Eq.10: N samples of the reduced logits z (fp64) -> (x [N][n] uint8, conf [N][n])."""
    z = np.ascontiguousarray(z, dtype=np.float64)
    n = len(z)
    x = np.zeros((N, n), np.uint8)
    c = np.zeros((N, n), np.float64)
    lib().oracle_pool(_ptr(z), n, N, tau, pool_seed & 0xFFFFFFFFFFFFFFFF, _ptr(x), _ptr(c))
    return x, c


def top_confident_units(x, conf, rho: float):
    """Eq.11 / SPEC extract_partial: |S| = max(1, ceil(rho n)); variables by descending
    confidence, ties to the lower index; literal +v if x_v = 1 else -v (1-based)."""
    x = np.asarray(x); conf = np.asarray(conf)
    n = len(conf)
    S = max(1, int(np.ceil(rho * n - 1e-9)))
    order = sorted(range(n), key=lambda v: (-conf[v], v))[:S]
    return [v + 1 if x[v] else -(v + 1) for v in order]


def lowest_confidence_vars(z, d: int, tau: float = 1.0):
    """Lemma 1 branching (SPEC select_branch_vars): the d variables with the
    lowest noise-free confidence max(y0, y1) = sigma(|z|/tau), ties to the lower index,
    returned 1-based ascending."""
    z = np.asarray(z, dtype=np.float64)
    # sigma is strictly increasing, so ordering by confidence is ordering by |z| / tau; the
    # key |z| keeps the order exact where sigma would round to 1.0 (|z| > ~37)
    order = sorted(range(len(z)), key=lambda v: (abs(z[v]), v))[:d]
    return sorted(v + 1 for v in order)


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def set_num_threads(k: int) -> None:
    lib().oracle_set_num_threads(int(k))
