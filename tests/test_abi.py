"""The C-ABI library loads and exports every symbol include/galois.h declares, and the
host-side argument checks fail with the documented status codes (-m "not gpu")."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from tests.conftest import ROOT, cuda_available

HEADER = os.path.join(ROOT, "include", "galois.h")


@pytest.fixture(scope="module")
def G():
    from paper_2603_28796_b200 import build, galois
    build.build()
    galois.lib()
    return galois


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(galois_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_north_star_calls():
    names = header_functions()
    for required in ("galois_cnf_load", "galois_engine_create", "galois_engine_step", "galois_engine_run",
                     "galois_best_assignment", "galois_unsat_counts"):
        assert required in names


def test_library_exports_every_declared_symbol(G):
    names = header_functions()
    out = subprocess.run(["nm", "-D", "--defined-only", G.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (galois_\w+)", out))
    assert set(names) <= exported, set(names) - exported
    assert set(G.EXPORTED) == set(names)
    for name in names:
        assert hasattr(G.lib(), name)


def test_library_is_sm100a_only(G):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", G.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(80|86|89|90)\b", out)


def test_last_error_starts_empty_and_reports(G):
    lib = G.lib()
    h = ctypes.c_void_p()
    off = np.array([0, 1], np.int64)
    lits = np.array([1], np.int32)
    rc = lib.galois_cnf_load(0, 1, off.ctypes.data, lits.ctypes.data, ctypes.byref(h))
    assert rc == G.E_ARG and "num_vars" in G.last_error()
    assert not h.value


def test_host_argument_checks(G):
    lib = G.lib()
    h = ctypes.c_void_p()
    off = np.array([0, 2, 3], np.int64)
    lits = np.array([1, -2, 2], np.int32)
    assert lib.galois_cnf_load(2, 2, off.ctypes.data, lits.ctypes.data, None) == G.E_ARG
    assert lib.galois_cnf_load(2, 2, None, lits.ctypes.data, ctypes.byref(h)) == G.E_ARG
    bad0 = np.array([1, 2, 3], np.int64)
    assert lib.galois_cnf_load(2, 2, bad0.ctypes.data, lits.ctypes.data, ctypes.byref(h)) == G.E_OFFSETS
    assert lib.galois_cnf_load(2, -1, off.ctypes.data, lits.ctypes.data, ctypes.byref(h)) == G.E_ARG
    assert lib.galois_cnf_load(2, 2, off.ctypes.data, None, ctypes.byref(h)) == G.E_ARG
    e = ctypes.c_void_p()
    assert lib.galois_engine_create(None, 4, 1, ctypes.c_double(0.5), 0, ctypes.byref(e)) == G.E_ARG
    assert lib.galois_engine_step(None) == G.E_ARG
    assert lib.galois_engine_run(None) == G.E_ARG
    assert lib.galois_best_assignment(None, None, None, None, None) == G.E_ARG
    assert lib.galois_unsat_counts(None, None, None) == G.E_ARG
    lib.galois_engine_free(None)
    lib.galois_cnf_free(None)


@pytest.mark.skipif(cuda_available(), reason="checks the no-device error path")
def test_no_device_fails_loudly(G):
    """Without a GPU the product path fails with E_CUDA — there is no CPU fallback."""
    with pytest.raises(G.GaloisError) as ei:
        G.Cnf(2, np.array([0, 2], np.int64), np.array([1, -2], np.int32))
    assert ei.value.code == G.E_CUDA and "no CUDA device" in str(ei.value)


def test_binding_refuses_missing_library(G, monkeypatch, tmp_path):
    monkeypatch.setattr(G, "_lib", None)
    monkeypatch.setattr(G, "LIB_PATH", str(tmp_path / "libgalois.so"))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        G.lib()
