"""Seeded molecular-integral inputs (h1, h2 in chemists' notation, e_core).

This module holds INPUT GENERATORS only -- none of the method's arithmetic.
Both the oracle (``oracle/``) and the CUDA path (``paper_2306_16705_b200``)
consume what it produces; neither imports the other.

Conventions (DESIGN.md "Readings" R8): spatial orbitals p = 0..n-1, real
integrals, h2[p,q,r,s] = (pq|rs) with the 8-fold permutational symmetry of
real orbitals; spin orbital (p, sigma) is qubit 2p+sigma (PAPER.md:287,
Sec. 3.3, 0-indexed reading).
"""
from __future__ import annotations

import numpy as np


def h2_sto3g():
    """Minimal-basis H2 at R = 1.4 bohr in the MO basis.

    Values: Szabo & Ostlund, *Modern Quantum Chemistry*, Sec. 3.5.2 / 4.x
    (textbook, external to the paper).  The paper's own H2 example is the
    4-qubit, 2-electron Hamiltonian of Fig. 6(a).
    Returns (h1[2,2], h2[2,2,2,2], e_core, n_alpha, n_beta).
    """
    h1 = np.array([[-1.2528, 0.0], [0.0, -0.4756]])
    J11, J22, J12, K12 = 0.6746, 0.6975, 0.6636, 0.1813
    h2 = np.zeros((2, 2, 2, 2))
    h2[0, 0, 0, 0] = J11
    h2[1, 1, 1, 1] = J22
    h2[0, 0, 1, 1] = h2[1, 1, 0, 0] = J12
    for p, q, r, s in [(0, 1, 0, 1), (0, 1, 1, 0), (1, 0, 0, 1), (1, 0, 1, 0)]:
        h2[p, q, r, s] = K12
    return h1, h2, 1.0 / 1.4, 1, 1


def _pair_index(n):
    """Index of the unordered pair {p, q} (p >= q) in the packed lower triangle."""
    idx = np.zeros((n, n), dtype=np.int64)
    k = 0
    for p in range(n):
        for q in range(p + 1):
            idx[p, q] = idx[q, p] = k
            k += 1
    return idx, k


def synthetic_integrals(n: int, irreps, seed: int, e_core: float = 10.0):
    """Symmetry-masked 'Cholesky-vector' integrals.

    irreps: length-n sequence of abelian irrep labels (ints combined by XOR).
    (pq|rs) = sum_L B^L_pq B^L_rs with B^L symmetric and B^L_pq = 0 unless
    G_p ^ G_q = G_L: 8-fold symmetric, PSD, and exactly zero where the
    point group forbids it.  Every orbit of the 8-fold group is written from
    one canonical value so the symmetry is bit-exact.
    Returns (h1[n,n], h2[n,n,n,n], e_core).
    """
    rng = np.random.default_rng(seed)
    irreps = np.asarray(irreps, dtype=np.int64)
    assert irreps.shape == (n,)
    n_irrep = 1
    while n_irrep <= int(irreps.max()):
        n_irrep *= 2
    L = 2 * n
    pq = np.abs(np.subtract.outer(np.arange(n), np.arange(n)))
    damp = np.exp(-pq / 8.0)
    gpq = irreps[:, None] ^ irreps[None, :]
    pidx, npair = _pair_index(n)
    V = np.zeros((npair, L))
    tril = np.tril_indices(n)
    for l in range(L):
        g_l = l % n_irrep
        B = rng.normal(0.0, 0.3, size=(n, n)) * damp
        B = np.tril(B) + np.tril(B, -1).T
        B[gpq != g_l] = 0.0
        V[pidx[tril], l] = B[tril]
    G = V @ V.T
    G = np.tril(G) + np.tril(G, -1).T          # exact symmetry (pq|rs) = (rs|pq)
    h2 = G[pidx[:, :, None, None], pidx[None, None, :, :]]
    eps = -2.0 + 2.5 * (np.arange(n) + 0.5) / n
    h1 = np.diag(eps) + rng.normal(0.0, 0.05, size=(n, n)) * (gpq == 0)
    h1 = np.tril(h1) + np.tril(h1, -1).T
    return np.ascontiguousarray(h1), np.ascontiguousarray(h2), float(e_core)


def random_dense_integrals(n: int, seed: int, e_core: float = 0.5):
    """Generic real integrals with 8-fold symmetry and no point-group zeros."""
    return synthetic_integrals(n, [0] * n, seed, e_core)


def coulomb_only_integrals(n: int, seed: int, e_core: float = 0.3):
    """h1 diagonal and only (pp|qq) non-zero: H is diagonal in the occupation
    basis (SURVEY.md Sec. 8(c) special cases)."""
    rng = np.random.default_rng(seed)
    h1 = np.diag(rng.normal(-1.0, 0.3, size=n))
    J = rng.uniform(0.2, 0.8, size=(n, n))
    J = np.tril(J) + np.tril(J, -1).T
    h2 = np.zeros((n, n, n, n))
    for p in range(n):
        for q in range(n):
            h2[p, p, q, q] = J[p, q]
    return h1, h2, float(e_core)
