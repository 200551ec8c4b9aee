"""ctypes wrappers for oracle/eloc_oracle.c (TEST INFRASTRUCTURE ONLY)."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "eloc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the C oracle (plain gcc, OpenMP over rows)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        L.oracle_row_hits.argtypes = [ctypes.c_int, P, P, ctypes.c_double, ctypes.c_int, P,
                                      ctypes.c_int64, P, ctypes.c_int64, P, P, P]
        L.oracle_row_hits.restype = ctypes.c_int
        L.oracle_eloc.argtypes = [ctypes.c_int, P, P, ctypes.c_double, ctypes.c_int, P, P,
                                  ctypes.c_int64, P, P, ctypes.c_int64, P, P, ctypes.c_int]
        L.oracle_eloc.restype = ctypes.c_int
        L.oracle_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _ints(h1, h2):
    h1 = np.ascontiguousarray(h1, dtype=np.float64)
    h2 = np.ascontiguousarray(h2, dtype=np.float64)
    return h1, h2, h1.shape[0]


def row_hits(h1, h2, e_core, x, keys=None, n_qubits=None, max_hits=1 << 22):
    """{x' in T : <x'|H|x>} for one row x (uint64[2]).  keys=None -> exact mode
    (T = all 2^N states, index = x').  Returns (idx[int64], H[float64])."""
    h1, h2, n = _ints(h1, h2)
    x = np.ascontiguousarray(x, dtype=np.uint64).reshape(2)
    exact = keys is None
    if exact:
        n_keys = 1 << (2 * n if n_qubits is None else n_qubits)
        kp = None
    else:
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        n_keys = len(keys)
        kp = _p(keys)
    cap = min(max_hits, n_keys)
    idx = np.empty(cap, dtype=np.int64)
    hv = np.empty(cap, dtype=np.float64)
    nh = np.zeros(1, dtype=np.int64)
    rc = lib().oracle_row_hits(n, _p(h1), _p(h2), float(e_core), int(exact), kp, n_keys, _p(x),
                               cap, _p(idx), _p(hv), _p(nh))
    if rc != 0:
        raise RuntimeError(f"oracle_row_hits failed: {rc}")
    return idx[: nh[0]].copy(), hv[: nh[0]].copy()


def eloc(h1, h2, e_core, rows, row_logpsi, keys=None, logpsi=None, n_threads=0, with_scale=False):
    """E_loc (Eq. 4) for explicit rows.  keys=None -> exact mode with logpsi
    indexed by configuration.  Returns complex128 [n_rows] (and, with
    with_scale, the per-row tolerance scale sum |H_xx'| |psi(x')/psi(x)|)."""
    h1, h2, n = _ints(h1, h2)
    rows = np.ascontiguousarray(rows, dtype=np.uint64).reshape(-1, 2)
    row_logpsi = np.ascontiguousarray(row_logpsi, dtype=np.float64).reshape(-1, 2)
    logpsi = np.ascontiguousarray(logpsi, dtype=np.float64).reshape(-1, 2)
    exact = keys is None
    if exact:
        kp, n_keys = None, len(logpsi)
    else:
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        kp, n_keys = _p(keys), len(keys)
        assert len(logpsi) == n_keys
    out = np.empty((len(rows), 2), dtype=np.float64)
    scale = np.empty(len(rows), dtype=np.float64)
    rc = lib().oracle_eloc(n, _p(h1), _p(h2), float(e_core), int(exact), kp, _p(logpsi), n_keys,
                           _p(rows), _p(row_logpsi), len(rows), _p(out), _p(scale), int(n_threads))
    if rc != 0:
        raise RuntimeError(f"oracle_eloc failed: {rc}")
    e = out[:, 0] + 1j * out[:, 1]
    return (e, scale) if with_scale else e


def num_threads() -> int:
    return int(lib().oracle_num_threads())
