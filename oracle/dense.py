"""Dense / sparse small-N tools of the oracle (TEST INFRASTRUCTURE ONLY).

* fermionic_sparse_H  -- H[x', x] = <x'|H|x> for all 2^N x, from the C oracle's
                         term-by-term rows (Eq. 9 + JW sign rules)
* kron_dense_H        -- the same operator built independently from explicit
                         Kronecker products a_j = Z x ... x Z x sigma^- x I ... (N <= 8)
* sector_basis / ground_state -- FCI in the (n_alpha, n_beta) sector
                         (number conservation; Table 1 'FCI')
* pauli_recovery      -- the grouped Pauli table of Fig. 6(c) / Algorithm 1
                          recovered by a Walsh-Hadamard
                         transform of each flip-diagonal of H:
                         d(X, Z) = 2^-N sum_x (-1)^{popc(x & Z)} H[x ^ X, x]
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import rows as R


def fermionic_sparse_H(h1, h2, e_core, n_qubits=None):
    n = h1.shape[0]
    N = 2 * n if n_qubits is None else n_qubits
    dim = 1 << N
    I, J, V = [], [], []
    for x in range(dim):
        idx, hv = R.row_hits(h1, h2, e_core, np.array([x, 0], dtype=np.uint64), keys=None, n_qubits=N)
        I.append(idx)
        J.append(np.full(len(idx), x, dtype=np.int64))
        V.append(hv)
    return sp.csr_matrix((np.concatenate(V), (np.concatenate(I), np.concatenate(J))), shape=(dim, dim))


def kron_dense_H(h1, h2, e_core):
    """Independent construction from explicit Kronecker-product ladder operators.
    Qubit 0 is the least-significant bit of the basis index, so the Kronecker
    product runs from qubit N-1 (leftmost factor) down to qubit 0."""
    n = h1.shape[0]
    N = 2 * n
    Z = sp.csr_matrix(np.diag([1.0, -1.0]))
    Id = sp.identity(2, format="csr")
    sm = sp.csr_matrix(np.array([[0.0, 1.0], [0.0, 0.0]]))   # |0><1|

    def a(j):
        op = None
        for k in range(N - 1, -1, -1):
            f = Z if k < j else (sm if k == j else Id)
            op = f if op is None else sp.kron(op, f, format="csr")
        return op

    A = [a(j) for j in range(N)]
    Ad = [m.T.tocsr() for m in A]
    dim = 1 << N
    H = e_core * sp.identity(dim, format="csr")
    for p in range(n):
        for q in range(n):
            if h1[p, q] == 0.0:
                continue
            for s in range(2):
                H = H + h1[p, q] * (Ad[2 * p + s] @ A[2 * q + s])
    for p in range(n):
        for q in range(n):
            for r in range(n):
                for s_ in range(n):
                    v = h2[p, q, r, s_]
                    if v == 0.0:
                        continue
                    for sg in range(2):
                        for tau in range(2):
                            H = H + 0.5 * v * (Ad[2 * p + sg] @ Ad[2 * r + tau] @ A[2 * s_ + tau] @ A[2 * q + sg])
    return H.toarray()


def sector_basis(n_orb, n_alpha, n_beta):
    """Configurations (ints) with n_alpha even-qubit and n_beta odd-qubit bits set."""
    out = []
    for x in range(1 << (2 * n_orb)):
        a = sum((x >> (2 * p)) & 1 for p in range(n_orb))
        b = sum((x >> (2 * p + 1)) & 1 for p in range(n_orb))
        if a == n_alpha and b == n_beta:
            out.append(x)
    return np.array(out, dtype=np.int64)


def sector_hamiltonian(h1, h2, e_core, keys):
    """Dense H restricted to a sorted key table (sample-mode rows)."""
    m = len(keys)
    H = np.zeros((m, m))
    for j in range(m):
        idx, hv = R.row_hits(h1, h2, e_core, keys[j], keys=keys)
        H[idx, j] = hv
    return H


def ground_state(h1, h2, e_core, keys):
    """Lowest eigenpair of H restricted to the given (sector) table; global sign
    fixed so the largest-magnitude component is positive."""
    H = sector_hamiltonian(h1, h2, e_core, keys)
    w, v = np.linalg.eigh(H)
    psi = v[:, 0]
    k = np.argmax(np.abs(psi))
    if psi[k] < 0:
        psi = -psi
    return float(w[0]), psi, H


def fwht(f):
    """Unnormalised Walsh-Hadamard transform: F[Z] = sum_x (-1)^{popc(x&Z)} f[x]."""
    f = np.array(f, dtype=np.float64, copy=True)
    h = 1
    n = len(f)
    while h < n:
        f = f.reshape(-1, 2, h)
        a = f[:, 0, :].copy()
        b = f[:, 1, :].copy()
        f[:, 0, :] = a + b
        f[:, 1, :] = a - b
        f = f.reshape(n)
        h *= 2
    return f


def pauli_recovery(Hs, N, tol):
    """Grouped Pauli table {X: [(Z, d)]} of H (sparse [2^N, 2^N]) with |d| > tol."""
    Hc = sp.coo_matrix(Hs)
    xs = np.unique(Hc.row ^ Hc.col)
    dim = 1 << N
    x = np.arange(dim)
    Hcsr = sp.csr_matrix(Hs)
    table = {}
    for X in xs:
        f = np.asarray(Hcsr[x ^ X, x]).ravel()
        d = fwht(f) / dim
        zs = np.nonzero(np.abs(d) > tol)[0]
        if len(zs):
            table[int(X)] = [(int(z), float(d[z])) for z in zs]
    return table
