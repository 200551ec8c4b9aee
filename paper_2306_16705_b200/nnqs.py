"""Thin ctypes binding of libnnqs (include/nnqs.h), same names as the C-ABI.

Argument marshalling only: every step of the path runs in libnnqs (host C++
compress, sm_100a kernels).  Device buffers are torch tensors (PyTorch is the
plumbing: device memory, streams); host buffers are numpy arrays.  There is no
CPU fallback: importing this module without the built library raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libnnqs.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libnnqs.so not found at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(the CUDA path has no fallback)")

_lib = ctypes.CDLL(LIB_PATH)
P = ctypes.c_void_p
I64 = ctypes.c_int64
_sig = {
    "nnqs_last_error": ([], ctypes.c_char_p),
    "nnqs_version": ([], ctypes.c_char_p),
    "nnqs_ham_compress": ([P, P, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_int, P], ctypes.c_int),
    "nnqs_ham_from_pauli": ([P, P, P, P, I64, ctypes.c_int, ctypes.c_double, ctypes.c_int, P], ctypes.c_int),
    "nnqs_ham_info": ([P, P, P, P, P], ctypes.c_int),
    "nnqs_ham_export": ([P, P, P, P, P], ctypes.c_int),
    "nnqs_ham_free": ([P], ctypes.c_int),
    "nnqs_options_default": ([P], None),
    "nnqs_table_prepare": ([P, ctypes.c_int, P, P, I64, P, P], ctypes.c_int),
    "nnqs_table_prepare_ex": ([P, ctypes.c_int, P, P, I64, P, P, P], ctypes.c_int),
    "nnqs_table_set_algorithm": ([P, ctypes.c_int], ctypes.c_int),
    "nnqs_table_free": ([P], ctypes.c_int),
    "nnqs_table_info": ([P, P, P, P], ctypes.c_int),
    "nnqs_local_energy": ([P, P, I64, P, P, I64, P, P, P, P, P], ctypes.c_int),
    "nnqs_local_energy_check": ([P, I64, P], ctypes.c_int),
    "nnqs_chunk_work": ([P, I64, P, P, P], ctypes.c_int),
    "nnqs_debug_counters": ([P, ctypes.c_int], ctypes.c_int),
    "nnqs_grad_weights": ([P, P, I64, P, P, P], ctypes.c_int),
    "nnqs_energy_chunk_partials": ([P, P, I64, P, P, P], ctypes.c_int),
    "nnqs_energy_combine": ([P, I64, ctypes.c_int, P, P], ctypes.c_int),
    "nnqs_energy_reduce": ([P, P, I64, P, P], ctypes.c_int),
    "nnqs_coupled_debug": ([P, P, P, I64, I64, P, P, P, P, P, P], ctypes.c_int),
    "nnqs_coupled_debug_rows": ([P, P, I64, I64, I64, P, P, P, P, P, P], ctypes.c_int),
    "nnqs_bas_layer": ([P, P, P, I64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, P, P,
                        P, P], ctypes.c_int),
}
class Options(ctypes.Structure):
    """nnqs_options (include/nnqs.h): per-table algorithm and list thresholds."""
    _fields_ = [("algorithm", ctypes.c_int32), ("thr_single", ctypes.c_int32), ("thr_double", ctypes.c_int32),
                ("thr_rowheavy", ctypes.c_int32), ("literal_kernel", ctypes.c_int32),
                ("reserved", ctypes.c_int32 * 11)]


for _name, (_args, _res) in _sig.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res

REDUCE_CHUNK = 1024
NNQS_OK, NNQS_E_ARG, NNQS_E_SIZE, NNQS_E_SYMMETRY, NNQS_E_TABLE = 0, -1, -2, -3, -4
NNQS_E_ZERO_PSI, NNQS_E_CUDA, NNQS_E_NOMEM, NNQS_E_EMPTY, NNQS_E_ODD_Y = -5, -6, -7, -8, -9


class NNQSError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def nnqs_last_error() -> str:
    return _lib.nnqs_last_error().decode()


def nnqs_version() -> str:
    return _lib.nnqs_version().decode()


def _check(rc: int):
    if rc != NNQS_OK:
        raise NNQSError(rc, nnqs_last_error())


def _np_ptr(a):
    return None if a is None else a.ctypes.data_as(P)


def _dev_ptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return P(t.data_ptr())


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return P(stream.cuda_stream)


class Hamiltonian:
    """Owning wrapper of an nnqs_ham handle (immutable after creation)."""

    def __init__(self, handle: P):
        self._h = handle

    @property
    def handle(self):
        return self._h

    def info(self):
        nq = ctypes.c_int()
        k, nh, b = I64(), I64(), I64()
        _check(_lib.nnqs_ham_info(self._h, ctypes.byref(nq), ctypes.byref(k), ctypes.byref(nh), ctypes.byref(b)))
        return {"n_qubits": nq.value, "n_groups": k.value, "n_terms": nh.value, "device_bytes": b.value}

    def export(self):
        inf = self.info()
        K, Nh = inf["n_groups"], inf["n_terms"]
        x = np.empty((K, 2), dtype=np.uint64)
        off = np.empty(K + 1, dtype=np.int64)
        z = np.empty((Nh, 2), dtype=np.uint64)
        d = np.empty(Nh, dtype=np.float64)
        _check(_lib.nnqs_ham_export(self._h, _np_ptr(x), _np_ptr(off), _np_ptr(z), _np_ptr(d)))
        return x, off, z, d

    def close(self):
        if self._h:
            _lib.nnqs_ham_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Table:
    """Owning wrapper of an nnqs_table handle."""

    def __init__(self, handle: P, mode: int, n: int):
        self._t = handle
        self.mode = mode
        self.n = n

    @property
    def handle(self):
        return self._t

    def info(self):
        n, s, b = I64(), ctypes.c_double(), I64()
        _check(_lib.nnqs_table_info(self._t, ctypes.byref(n), ctypes.byref(s), ctypes.byref(b)))
        return {"n": n.value, "shift": s.value, "device_bytes": b.value}

    def close(self):
        if self._t:
            _lib.nnqs_table_free(self._t)
            self._t = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ C-ABI names
def nnqs_ham_compress(h1, h2, n_spin_orbitals: int, e_core: float, tol: float = 0.0, device: int = 0) -> Hamiltonian:
    h1 = np.ascontiguousarray(h1, dtype=np.float64)
    h2 = np.ascontiguousarray(h2, dtype=np.float64)
    n = n_spin_orbitals // 2
    if h1.size != n * n or h2.size != n ** 4:
        raise ValueError("h1/h2 sizes do not match n_spin_orbitals")
    out = P()
    _check(_lib.nnqs_ham_compress(_np_ptr(h1), _np_ptr(h2), int(n_spin_orbitals), float(e_core), float(tol),
                                  int(device), ctypes.byref(out)))
    return Hamiltonian(out)


def nnqs_ham_from_pauli(xmask, zmask, coeff, n_qubits: int, tol: float = 0.0, device: int = 0) -> Hamiltonian:
    xmask = np.ascontiguousarray(xmask, dtype=np.uint64).reshape(-1, 2)
    zmask = np.ascontiguousarray(zmask, dtype=np.uint64).reshape(-1, 2)
    coeff = np.asarray(coeff, dtype=np.complex128).reshape(-1)
    cre = np.ascontiguousarray(coeff.real)
    cim = np.ascontiguousarray(coeff.imag)
    out = P()
    _check(_lib.nnqs_ham_from_pauli(_np_ptr(xmask), _np_ptr(zmask), _np_ptr(cre), _np_ptr(cim), len(cre),
                                    int(n_qubits), float(tol), int(device), ctypes.byref(out)))
    return Hamiltonian(out)


def nnqs_options_default() -> Options:
    o = Options()
    _lib.nnqs_options_default(ctypes.byref(o))
    return o


def nnqs_table_prepare(ham: Hamiltonian, mode: int, keys, logpsi, stream=None, algorithm: int | None = None,
                       thr_single: int = 0, thr_double: int = 0, thr_rowheavy: int = 0,
                       literal_kernel: int = 0) -> Table:
    """keys: CUDA int64/uint64 [n, 2] (mode 0) or None (mode 1); logpsi CUDA float64 [n, 2].
    Keyword options fill nnqs_options (0 = the library default) -> nnqs_table_prepare_ex."""
    n = int(logpsi.shape[0])
    out = P()
    if algorithm is None and not (thr_single or thr_double or thr_rowheavy or literal_kernel):
        _check(_lib.nnqs_table_prepare(ham.handle, int(mode), _dev_ptr(keys), _dev_ptr(logpsi), n, _stream(stream),
                                       ctypes.byref(out)))
    else:
        o = Options()
        o.algorithm = int(algorithm or 0)
        o.thr_single, o.thr_double, o.thr_rowheavy = int(thr_single), int(thr_double), int(thr_rowheavy)
        o.literal_kernel = int(literal_kernel)
        _check(_lib.nnqs_table_prepare_ex(ham.handle, int(mode), _dev_ptr(keys), _dev_ptr(logpsi), n,
                                          ctypes.byref(o), _stream(stream), ctypes.byref(out)))
    return Table(out, mode, n)


def nnqs_table_set_algorithm(table: Table, algorithm: int):
    """NNQS_ALGO_AUTO (0) or NNQS_ALGO_LITERAL (1) for this table."""
    _check(_lib.nnqs_table_set_algorithm(table.handle, int(algorithm)))


def nnqs_local_energy(ham: Hamiltonian, table: Table, row_begin: int = 0, rows=None, row_logpsi=None,
                      n_rows: int | None = None, eloc_out=None, counts=None, partials_out=None, stats_out=None,
                      stream=None):
    """E_loc (device f64[n_rows][2]).  counts (device i64[n_rows]) + partials_out (device
    f64[ceil(n_rows/1024)][3]): the fused first pass of Eq. (6) per 1024-row chunk."""
    import torch
    if n_rows is None:
        n_rows = int(rows.shape[0]) if rows is not None else table.n - row_begin
    if eloc_out is None:
        dev = (rows if rows is not None else row_logpsi)
        device = dev.device if dev is not None else torch.device("cuda", torch.cuda.current_device())
        eloc_out = torch.empty((n_rows, 2), dtype=torch.float64, device=device)
    _check(_lib.nnqs_local_energy(ham.handle, table.handle, int(row_begin), _dev_ptr(rows), _dev_ptr(row_logpsi),
                                  int(n_rows), _dev_ptr(eloc_out), _dev_ptr(counts), _dev_ptr(partials_out),
                                  _dev_ptr(stats_out), _stream(stream)))
    return eloc_out


ALGO_AUTO, ALGO_LITERAL = 0, 1


def nnqs_debug_counters(reset: bool = True):
    """Section cycle counters of the structured kernel (libnnqs built with -DNNQS_PROFILE)."""
    out = np.zeros(16, dtype=np.uint64)
    _check(_lib.nnqs_debug_counters(out.ctypes.data, int(bool(reset))))
    return out


def nnqs_chunk_work(table: Table, chunk: int = REDUCE_CHUNK, stream=None, with_floor: bool = False):
    """Host int64[ceil(n/chunk)] work estimate per chunk of table rows (see include/nnqs.h);
    with_floor: (work, floor), floor = the largest single-row latency floor per chunk."""
    import numpy as np
    nch = (table.n + chunk - 1) // chunk if chunk > 0 else 0   # chunk <= 0: the library reports NNQS_E_ARG
    out = np.zeros(max(nch, 1), dtype=np.int64)
    fl = np.zeros(max(nch, 1), dtype=np.int64)
    _check(_lib.nnqs_chunk_work(table.handle, int(chunk), out.ctypes.data, fl.ctypes.data if with_floor else None,
                                _stream(stream)))
    return (out[:nch], fl[:nch]) if with_floor else out[:nch]


def nnqs_local_energy_check(eloc, stream=None):
    _check(_lib.nnqs_local_energy_check(_dev_ptr(eloc), int(eloc.shape[0]), _stream(stream)))


def nnqs_energy_chunk_partials(eloc, counts, mean_dev=None, partials=None, stream=None):
    import torch
    n = int(eloc.shape[0])
    chunks = (n + REDUCE_CHUNK - 1) // REDUCE_CHUNK
    if partials is None:
        partials = torch.empty((max(chunks, 1), 3), dtype=torch.float64, device=eloc.device)
    _check(_lib.nnqs_energy_chunk_partials(_dev_ptr(eloc), _dev_ptr(counts), n, _dev_ptr(mean_dev),
                                           _dev_ptr(partials), _stream(stream)))
    return partials


def nnqs_energy_combine(partials, pass_: int, out_dev=None, n_chunks: int | None = None, stream=None):
    import torch
    if out_dev is None:
        out_dev = torch.empty(4, dtype=torch.float64, device=partials.device)
    nc = int(partials.shape[0]) if n_chunks is None else int(n_chunks)
    _check(_lib.nnqs_energy_combine(_dev_ptr(partials), nc, int(pass_), _dev_ptr(out_dev), _stream(stream)))
    return out_dev


def nnqs_grad_weights(eloc, counts, energy_dev, ab_out=None, stream=None):
    """Eq. (7) weights (a_u, b_u) as a device f64[n][2]; energy_dev = (mean_re, mean_im, W, ...)."""
    import torch
    n = int(eloc.shape[0])
    if ab_out is None:
        ab_out = torch.empty((n, 2), dtype=torch.float64, device=eloc.device)
    _check(_lib.nnqs_grad_weights(_dev_ptr(eloc), _dev_ptr(counts), n, _dev_ptr(energy_dev), _dev_ptr(ab_out),
                                  _stream(stream)))
    return ab_out


def nnqs_bas_layer(keys, counts, probs, orbital: int, n_orbitals: int, n_up: int, n_dn: int, seed: int,
                   stream=None):
    """One BAS layer (include/nnqs.h): keys CUDA int64 [m, 2], counts CUDA int64 [m],
    probs CUDA float64 [m, 4] -> (child keys [m', 2], child counts [m']) on the same device."""
    import torch
    m = int(keys.shape[0])
    dev = keys.device
    ko = torch.empty((max(4 * m, 1), 2), dtype=torch.int64, device=dev)
    co = torch.empty(max(4 * m, 1), dtype=torch.int64, device=dev)
    mo = ctypes.c_int64(0)
    _check(_lib.nnqs_bas_layer(_dev_ptr(keys), _dev_ptr(counts), _dev_ptr(probs), m, int(orbital), int(n_orbitals),
                               int(n_up), int(n_dn), ctypes.c_uint64(int(seed) & (2**64 - 1)), _dev_ptr(ko),
                               _dev_ptr(co), ctypes.byref(mo), _stream(stream)))
    return ko[: mo.value], co[: mo.value]


def nnqs_energy_reduce(eloc, counts, stream=None):
    """Returns (mean complex, var, W) -- Eq. (6) with counts (synchronises)."""
    out = np.zeros(4, dtype=np.float64)
    _check(_lib.nnqs_energy_reduce(_dev_ptr(eloc), _dev_ptr(counts), int(eloc.shape[0]), _np_ptr(out),
                                   _stream(stream)))
    return complex(out[0], out[1]), float(out[2]), float(out[3])


def nnqs_coupled_debug(ham: Hamiltonian, table: Table, rows_host, max_pairs: int = 1 << 20):
    rows_host = np.ascontiguousarray(rows_host, dtype=np.uint64).reshape(-1, 2)
    rid = np.empty(max_pairs, dtype=np.int64)
    gid = np.empty(max_pairs, dtype=np.int64)
    xp = np.empty((max_pairs, 2), dtype=np.uint64)
    tix = np.empty(max_pairs, dtype=np.int64)
    hv = np.empty(max_pairs, dtype=np.float64)
    n = I64()
    _check(_lib.nnqs_coupled_debug(ham.handle, table.handle, _np_ptr(rows_host), len(rows_host), int(max_pairs),
                                   _np_ptr(rid), _np_ptr(gid), _np_ptr(xp), _np_ptr(tix), _np_ptr(hv),
                                   ctypes.byref(n)))
    m = n.value
    return rid[:m], gid[:m], xp[:m], tix[:m], hv[:m]


def nnqs_coupled_debug_rows(ham: Hamiltonian, table: Table, row_begin: int, n_rows: int, max_pairs: int = 1 << 20):
    """Every hit the production launch sequence evaluates for table rows [row_begin, row_begin+n_rows):
    (row table index, group id, x' key, x' table index, H_xx')."""
    rid = np.empty(max_pairs, dtype=np.int64)
    gid = np.empty(max_pairs, dtype=np.int64)
    xp = np.empty((max_pairs, 2), dtype=np.uint64)
    tix = np.empty(max_pairs, dtype=np.int64)
    hv = np.empty(max_pairs, dtype=np.float64)
    n = I64()
    _check(_lib.nnqs_coupled_debug_rows(ham.handle, table.handle, int(row_begin), int(n_rows), int(max_pairs),
                                        _np_ptr(rid), _np_ptr(gid), _np_ptr(xp), _np_ptr(tix), _np_ptr(hv),
                                        ctypes.byref(n)))
    m = n.value
    return rid[:m], gid[:m], xp[:m], tix[:m], hv[:m]


EXPORTED = [n for n in _sig]
