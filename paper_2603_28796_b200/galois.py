"""Thin ctypes binding of libgalois (include/galois.h): argument marshalling only.

Every step of the method runs in the CUDA kernels behind the C ABI; this module only
converts numpy arrays to pointers and status codes to exceptions. It never falls back
to a CPU path: if libgalois.so is missing or cannot be loaded, every call raises.

Functions keep the C names (galois_cnf_load, galois_engine_create, ...); the classes
Cnf and Engine wrap the handles for convenience.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GALOIS_LIB") or os.path.join(_PKG, "libgalois.so")   # override: A/B builds

OK, BUDGET, SAT = 0, 1, 10
E_ARG, E_VAR_RANGE, E_OFFSETS, E_EMPTY_CLAUSE = -1, -2, -3, -4
E_OOM, E_CUDA, E_NCCL, E_NONFINITE, E_STATE = -5, -6, -7, -8, -9
STATUS_NAMES = {0: "OK", 1: "BUDGET", 10: "SAT", -1: "E_ARG", -2: "E_VAR_RANGE", -3: "E_OFFSETS",
                -4: "E_EMPTY_CLAUSE", -5: "E_OOM", -6: "E_CUDA", -7: "E_NCCL", -8: "E_NONFINITE",
                -9: "E_STATE"}
NUM_KERNEL_CLASSES = 6
KERNEL_CLASSES = ("forward", "update", "check", "best", "hub_partial", "init")

EXPORTED = (
    "galois_cnf_load", "galois_cnf_info", "galois_cnf_get_csc", "galois_cnf_free",
    "galois_engine_create", "galois_engine_step", "galois_engine_run", "galois_engine_enqueue",
    "galois_best_assignment", "galois_unsat_counts", "galois_engine_info", "galois_engine_free",
    "galois_last_error", "galois_engine_set_mode", "galois_engine_set_hparams",
    "galois_engine_set_check_interval", "galois_engine_set_cubes", "galois_engine_set_comm",
    "galois_engine_set_stream", "galois_engine_set_debug", "galois_engine_set_profiling",
    "galois_comm_unique_id", "galois_engine_get_iterate", "galois_engine_set_iterate",
    "galois_engine_get_grad", "galois_engine_get_loss", "galois_engine_get_bits",
    "galois_engine_kernel_times", "galois_select_member", "galois_candidate_pool", "galois_cube_variables",
    "galois_cnf_normalize", "galois_cnf_get_csr", "galois_engine_set_subbatch", "galois_engine_set_lanes", "galois_engine_bytes_per_member",
    "galois_engine_set_graphs", "galois_engine_get_member", "galois_cnf_original_vars", "galois_candidate_pool_size",
    "galois_device_free_bytes", "galois_engine_window_bytes", "galois_engine_max_sub_batch",
)


class GaloisError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code


_lib = None


def lib() -> ctypes.CDLL:
    """Load libgalois.so (built by paper_2603_28796_b200.build / __graft_entry__.build)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2603_28796_b200.build` "
                               "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        P, I32, I64, U64, F = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
        sig = {
            "galois_cnf_load": [I32, I64, P, P, P],
            "galois_cnf_info": [P, P, P, P, P, P, P],
            "galois_cnf_get_csc": [P, P, P],
            "galois_cnf_free": [P],
            "galois_engine_create": [P, I64, I32, F, U64, P],
            "galois_engine_step": [P],
            "galois_engine_run": [P],
            "galois_engine_enqueue": [P, I32],
            "galois_best_assignment": [P, P, P, P, P],
            "galois_unsat_counts": [P, P, P],
            "galois_engine_info": [P, P, P, P, P],
            "galois_engine_free": [P],
            "galois_last_error": [],
            "galois_engine_set_mode": [P, I32],
            "galois_engine_set_hparams": [P, F, F, F, F, I32],
            "galois_engine_set_check_interval": [P, I32],
            "galois_engine_set_cubes": [P, I32, P],
            "galois_engine_set_comm": [P, I32, I32, P],
            "galois_engine_set_stream": [P, P],
            "galois_engine_set_debug": [P, I32],
            "galois_engine_set_profiling": [P, I32],
            "galois_comm_unique_id": [P],
            "galois_engine_get_iterate": [P, P, P, P, P],
            "galois_engine_set_iterate": [P, P, P, P, I32],
            "galois_engine_get_grad": [P, P, P],
            "galois_engine_get_loss": [P, P],
            "galois_engine_get_bits": [P, P, P],
            "galois_engine_kernel_times": [P, P, P],
            "galois_select_member": [P, I32, P, P, P],
            "galois_candidate_pool": [P, I64, I32, F, U64, P, P, P, P],
            "galois_cube_variables": [P, I64, I32, P],
            "galois_cnf_normalize": [P, I32, P, P],
            "galois_cnf_get_csr": [P, P, P],
            "galois_engine_set_subbatch": [P, I32],
            "galois_engine_set_lanes": [P, I32],
            "galois_engine_bytes_per_member": [P, I32, P],
            "galois_device_free_bytes": [I32, P],
            "galois_engine_window_bytes": [P, I32, I32, I32, I32, P],
            "galois_engine_max_sub_batch": [P, I32, I32, I32, I64, P],
            "galois_engine_set_graphs": [P, I32],
            "galois_engine_get_member": [P, I64, P, P, P, P, P, P, P, P, P, P],
            "galois_cnf_original_vars": [P, P],
            "galois_candidate_pool_size": [P, F, P],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        L.galois_cnf_free.restype = None
        L.galois_engine_free.restype = None
        L.galois_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


def last_error() -> str:
    return lib().galois_last_error().decode()


def _check(rc: int, allowed=(OK,)) -> int:
    if rc in allowed:
        return rc
    raise GaloisError(rc, last_error())


def _p(a: Optional[np.ndarray]):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


# ----------------------------------------------------------------- C-named functions
def galois_cnf_load(num_vars: int, num_clauses: int, clause_offsets: np.ndarray, literals: np.ndarray):
    off = np.ascontiguousarray(clause_offsets, dtype=np.int64)
    lits = np.ascontiguousarray(literals, dtype=np.int32)
    h = ctypes.c_void_p()
    rc = lib().galois_cnf_load(int(num_vars), int(num_clauses), _p(off), _p(lits) if lits.size else None,
                               ctypes.byref(h))
    _check(rc)
    return h


def galois_engine_create(cnf, batch: int, steps: int, lr: float, seed: int):
    h = ctypes.c_void_p()
    _check(lib().galois_engine_create(cnf, int(batch), int(steps), float(lr), int(seed) & (2 ** 64 - 1),
                                      ctypes.byref(h)))
    return h


def galois_engine_step(eng) -> int:
    return _check(lib().galois_engine_step(eng), (OK, SAT, BUDGET))


def galois_engine_run(eng) -> int:
    return _check(lib().galois_engine_run(eng), (SAT, BUDGET))


def galois_engine_enqueue(eng, max_steps: int) -> int:
    return _check(lib().galois_engine_enqueue(eng, int(max_steps)), (OK, BUDGET))


def galois_comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().galois_comm_unique_id(buf))
    return buf.raw


def galois_device_free_bytes(device: int = 0) -> int:
    out = ctypes.c_int64()
    _check(lib().galois_device_free_bytes(int(device), ctypes.byref(out)))
    return out.value


# ------------------------------------------------------------------------- classes
class Cnf:
    """A CNF resident on the current CUDA device (CSR + CSC + hub table)."""

    def __init__(self, n: int, offsets, lits):
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        self.n = int(n)
        self.m = len(offsets) - 1
        self.handle = galois_cnf_load(self.n, self.m, offsets, lits)

    @classmethod
    def from_instance(cls, inst) -> "Cnf":
        return cls(inst.n, inst.offsets, inst.lits)

    def info(self) -> dict:
        n, m, L = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64()
        w, d, h = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        _check(lib().galois_cnf_info(self.handle, ctypes.byref(n), ctypes.byref(m), ctypes.byref(L),
                                     ctypes.byref(w), ctypes.byref(d), ctypes.byref(h)))
        return dict(n=n.value, m=m.value, L=L.value, max_width=w.value, max_degree=d.value, num_hubs=h.value)

    def normalize(self, k: int = 3) -> "Cnf":
        """Fixed-width chain normalisation on the device (Eq.6-9); returns the new CNF
        (n + num_aux variables) with attribute num_aux."""
        h = ctypes.c_void_p()
        aux = ctypes.c_int32()
        _check(lib().galois_cnf_normalize(self.handle, int(k), ctypes.byref(h), ctypes.byref(aux)))
        out = Cnf.__new__(Cnf)
        out.handle = h
        info = out.info()
        out.n, out.m, out.num_aux = info["n"], info["m"], aux.value
        return out

    def original_vars(self) -> int:
        out = ctypes.c_int32()
        _check(lib().galois_cnf_original_vars(self.handle, ctypes.byref(out)))
        return out.value

    def pool_size(self, rho: float) -> int:
        out = ctypes.c_int32()
        _check(lib().galois_candidate_pool_size(self.handle, float(rho), ctypes.byref(out)))
        return out.value

    def bytes_per_member(self, mode: int = 0) -> int:
        out = ctypes.c_int64()
        _check(lib().galois_engine_bytes_per_member(self.handle, int(mode), ctypes.byref(out)))
        return out.value

    def window_bytes(self, members: int, steps: int, mode: int = 0, cubes: bool = False) -> int:
        out = ctypes.c_int64()
        _check(lib().galois_engine_window_bytes(self.handle, int(mode), int(members), int(steps), int(cubes),
                                                ctypes.byref(out)))
        return out.value

    def sub_batch_for(self, budget_bytes: int, steps: int, mode: int = 0, cubes: bool = False) -> int:
        """Largest multiple of 32 members whose engine fits budget_bytes (f4; the library's
        galois_engine_max_sub_batch)."""
        out = ctypes.c_int32()
        _check(lib().galois_engine_max_sub_batch(self.handle, int(mode), int(steps), int(cubes), int(budget_bytes),
                                                 ctypes.byref(out)))
        return out.value

    def csr(self):
        info = self.info()
        off = np.zeros(info["m"] + 1, np.int64)
        lits = np.zeros(max(info["L"], 1), np.int32)
        _check(lib().galois_cnf_get_csr(self.handle, _p(off), _p(lits)))
        return off, lits[:info["L"]]

    def csc(self):
        info = self.info()
        code_off = np.zeros(2 * self.n + 1, np.int32)
        occ = np.zeros(max(info["L"], 1), np.int32)
        _check(lib().galois_cnf_get_csc(self.handle, _p(code_off), _p(occ)))
        return code_off, occ[:info["L"]]

    def free(self):
        if getattr(self, "handle", None):
            lib().galois_cnf_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Engine:
    """One rank's slice of the batch (see include/galois.h)."""

    def __init__(self, cnf: Cnf, batch: int, steps: int, lr: float = 0.5, seed: int = 0, *,
                 mode: int = 0, tau: float = 1.0, beta1: float = 0.9, beta2: float = 0.999,
                 eps: float = 1e-8, optimizer: int = 0, check_interval: int = 1,
                 cubes: Sequence[int] = (), debug: bool = False, stream=None,
                 rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None, sub_batch: int = 0,
                 lanes: int = 1, graphs: int = 0):
        self.cnf = cnf
        self.n = cnf.n
        # this rank's slice (galois.h: b_per = roundup(ceil(B / world), 32)), to size host
        # arrays without galois_engine_info (which would run a pending check)
        per = -(-int(batch) // int(world))
        per = -(-per // 32) * 32
        self.local_batch = max(0, min(per, int(batch) - per * int(rank)))
        self.handle = galois_engine_create(cnf.handle, batch, steps, lr, seed)
        L = lib()
        if mode:
            _check(L.galois_engine_set_mode(self.handle, int(mode)))
        if (tau, beta1, beta2, eps, optimizer) != (1.0, 0.9, 0.999, 1e-8, 0):
            _check(L.galois_engine_set_hparams(self.handle, tau, beta1, beta2, eps, int(optimizer)))
        if check_interval != 1:
            _check(L.galois_engine_set_check_interval(self.handle, int(check_interval)))
        if len(cubes):
            c = np.ascontiguousarray(cubes, dtype=np.int32)
            _check(L.galois_engine_set_cubes(self.handle, len(c), _p(c)))
        if debug:
            _check(L.galois_engine_set_debug(self.handle, 1))
        if stream is not None:
            _check(L.galois_engine_set_stream(self.handle, ctypes.c_void_p(int(stream))))
        if sub_batch:
            _check(L.galois_engine_set_subbatch(self.handle, int(sub_batch)))
        if lanes != 1:
            _check(L.galois_engine_set_lanes(self.handle, int(lanes)))
        if graphs:
            _check(L.galois_engine_set_graphs(self.handle, int(graphs)))
        if world > 1 or nccl_id is not None:
            buf = ctypes.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None
            _check(L.galois_engine_set_comm(self.handle, int(rank), int(world), buf))

    # -- driving
    def step(self) -> int:
        return galois_engine_step(self.handle)

    def run(self) -> int:
        return galois_engine_run(self.handle)

    def enqueue(self, max_steps: int) -> int:
        return galois_engine_enqueue(self.handle, max_steps)

    def set_profiling(self, on: bool = True):
        _check(lib().galois_engine_set_profiling(self.handle, 1 if on else 0))

    # -- results
    def info(self) -> dict:
        lb, b0, t, st = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32()
        _check(lib().galois_engine_info(self.handle, ctypes.byref(lb), ctypes.byref(b0), ctypes.byref(t),
                                        ctypes.byref(st)))
        return dict(local_batch=lb.value, first_global_b=b0.value, steps_done=t.value, stopped=bool(st.value))

    def best_assignment(self):
        vals = np.zeros(self.n, np.uint8)
        u, b, t = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int32()
        _check(lib().galois_best_assignment(self.handle, _p(vals), ctypes.byref(u), ctypes.byref(b),
                                            ctypes.byref(t)))
        return dict(values=vals, unsat=u.value, global_b=b.value, step=t.value)

    def unsat_counts(self):
        nb = self.local_batch
        out = np.zeros(max(nb, 1), np.int32)
        b0 = ctypes.c_int64()
        _check(lib().galois_unsat_counts(self.handle, _p(out), ctypes.byref(b0)))
        return out[:nb], b0.value

    def get_iterate(self):
        nb = self.local_batch
        z = np.zeros((nb, self.n), np.float32); m = np.zeros_like(z); v = np.zeros_like(z)
        t = ctypes.c_int32()
        _check(lib().galois_engine_get_iterate(self.handle, _p(z), _p(m), _p(v), ctypes.byref(t)))
        return z, m, v, t.value

    def set_iterate(self, z, m, v, t: int):
        z = np.ascontiguousarray(z, np.float32); m = np.ascontiguousarray(m, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        _check(lib().galois_engine_set_iterate(self.handle, _p(z), _p(m), _p(v), int(t)))

    def get_member(self, global_b: int, grad: bool = False):
        """One member's z, m, v (float32 [n]), sample bits x_next and rounding r (uint8 [n]),
        t, its count at the last check that ran (unsat, check_t; no pending check is run),
        and with grad=True (debug engines) G (int32) and g1 (float32)."""
        n = self.n
        z = np.zeros(n, np.float32); m = np.zeros_like(z); v = np.zeros_like(z)
        x = np.zeros(n, np.uint8); r = np.zeros(n, np.uint8)
        G = np.zeros(n, np.int32) if grad else None
        g1 = np.zeros(n, np.float32) if grad else None
        t, u, ct = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        _check(lib().galois_engine_get_member(self.handle, int(global_b), _p(z), _p(m), _p(v), _p(x), _p(r),
                                              _p(G), _p(g1), ctypes.byref(t), ctypes.byref(u), ctypes.byref(ct)))
        out = dict(z=z, m=m, v=v, x_next=x, r=r, t=t.value, unsat=u.value, check_t=ct.value)
        if grad:
            out.update(G=G, g1=g1)
        return out

    def get_grad(self):
        nb = self.local_batch
        G = np.zeros((nb, self.n), np.int32); g1 = np.zeros((nb, self.n), np.float32)
        _check(lib().galois_engine_get_grad(self.handle, _p(G), _p(g1)))
        return G, g1

    def get_loss(self):
        nb = self.local_batch
        lam = np.zeros(max(nb, 1), np.float64)        # exact counts (ST) beyond 2^24
        _check(lib().galois_engine_get_loss(self.handle, _p(lam)))
        return lam[:nb]

    def get_bits(self):
        nb = self.local_batch
        x = np.zeros((nb, self.n), np.uint8); r = np.zeros((nb, self.n), np.uint8)
        _check(lib().galois_engine_get_bits(self.handle, _p(x), _p(r)))
        return x, r

    # -- what the CPU stage consumes (f1, f3)
    def select_member(self, rule: int = 0):
        """theta_sel: rule 0 = min loss, 1 = max loss at the last check."""
        b, u = ctypes.c_int64(), ctypes.c_int32()
        z = np.zeros(self.n, np.float32)
        _check(lib().galois_select_member(self.handle, int(rule), ctypes.byref(b), ctypes.byref(u), _p(z)))
        return dict(global_b=b.value, unsat=u.value, z=z)

    def candidate_pool(self, global_b: int, N: int = 100, rho: float = 0.0005, pool_seed: int = 0,
                       arrays: bool = True):
        """Eq.10-11: N samples of member global_b, their confidences and top-|S| unit literals
        (arrays=False: the unit lists only; values / confidence stay on the device)."""
        n = self.n
        S = self.cnf.pool_size(rho)                   # |S| (Eq.11) from the library
        x = np.zeros((N, n), np.uint8) if arrays else None
        c = np.zeros((N, n), np.float32) if arrays else None
        u = np.zeros((N, S), np.int32)
        s_out = ctypes.c_int32()
        _check(lib().galois_candidate_pool(self.handle, int(global_b), int(N), float(rho),
                                           int(pool_seed) & (2 ** 64 - 1), _p(x), _p(c), _p(u),
                                           ctypes.byref(s_out)))
        assert s_out.value == S
        return dict(values=x, confidence=c, units=u, S=S)

    def cube_variables(self, global_b: int, d: int):
        """Lemma 1 branching: the d least confident variables (1-based, ascending)."""
        out = np.zeros(d, np.int32)
        _check(lib().galois_cube_variables(self.handle, int(global_b), int(d), _p(out)))
        return out

    def kernel_times(self):
        ms = np.zeros(NUM_KERNEL_CLASSES, np.float64)
        cnt = np.zeros(NUM_KERNEL_CLASSES, np.int64)
        _check(lib().galois_engine_kernel_times(self.handle, _p(ms), _p(cnt)))
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(KERNEL_CLASSES)}

    def free(self):
        if getattr(self, "handle", None):
            lib().galois_engine_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
