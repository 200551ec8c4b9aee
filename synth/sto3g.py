"""Real-molecule inputs: STO-3G integrals and restricted Hartree-Fock orbitals for
small molecules (INPUT GENERATOR -- none of the local-energy method's arithmetic).

The paper takes h and g from PySCF; PySCF is not installed here, so
this module computes them: contracted Cartesian Gaussians (s and p shells, the
standard STO-3G contractions), overlap / kinetic / nuclear-attraction / electron-
repulsion integrals by the McMurchie-Davidson scheme (Hermite expansion coefficients
E, Hermite Coulomb integrals R with the Boys function), a plain RHF SCF, and the
AO -> MO transformation.  Output: spatial h1[n, n], chemists' (pq|rs) h2[n]^4 and
e_core = the nuclear repulsion, the inputs of nnqs_ham_compress (R8).
"""
from __future__ import annotations

import math
from functools import lru_cache

import numpy as np
from scipy.special import gammainc, gamma

ANG = 1.0 / 0.52917721092          # bohr per angstrom

# STO-3G (Hehre, Stewart, Pople 1969): exponents and contraction coefficients
_STO3G = {
    "H": [("s", [3.42525091, 0.62391373, 0.16885540], [0.15432897, 0.53532814, 0.44463454])],
    "O": [("s", [130.7093200, 23.8088610, 6.4436083], [0.15432897, 0.53532814, 0.44463454]),
          ("s", [5.0331513, 1.1695961, 0.3803890], [-0.09996723, 0.39951283, 0.70011547]),
          ("p", [5.0331513, 1.1695961, 0.3803890], [0.15591627, 0.60768372, 0.39195739])],
    "N": [("s", [99.1061690, 18.0523120, 4.8856602], [0.15432897, 0.53532814, 0.44463454]),
          ("s", [3.7804559, 0.8784966, 0.2857144], [-0.09996723, 0.39951283, 0.70011547]),
          ("p", [3.7804559, 0.8784966, 0.2857144], [0.15591627, 0.60768372, 0.39195739])],
}
_Z = {"H": 1, "N": 7, "O": 8}


def _dfact(n: int) -> int:
    return 1 if n <= 0 else n * _dfact(n - 2)


class Shell:
    def __init__(self, center, lmn, exps, coefs):
        self.A = np.asarray(center, dtype=float)
        self.lmn = lmn
        self.exps = np.asarray(exps, dtype=float)
        L = sum(lmn)
        norm = [(2 * a / math.pi) ** 0.75 * (4 * a) ** (L / 2) /
                math.sqrt(_dfact(2 * lmn[0] - 1) * _dfact(2 * lmn[1] - 1) * _dfact(2 * lmn[2] - 1)) for a in exps]
        self.coefs = np.asarray(coefs, dtype=float) * np.asarray(norm)
        s = sum(ci * cj * _overlap_prim(ai, lmn, self.A, aj, lmn, self.A)
                for ai, ci in zip(self.exps, self.coefs) for aj, cj in zip(self.exps, self.coefs))
        self.coefs /= math.sqrt(s)


def basis(atoms):
    """atoms: [(symbol, (x, y, z) in bohr)] -> list of contracted functions (s, then px py pz)."""
    out = []
    for sym, xyz in atoms:
        for kind, exps, coefs in _STO3G[sym]:
            if kind == "s":
                out.append(Shell(xyz, (0, 0, 0), exps, coefs))
            else:
                for lmn in ((1, 0, 0), (0, 1, 0), (0, 0, 1)):
                    out.append(Shell(xyz, lmn, exps, coefs))
    return out


@lru_cache(maxsize=None)
def _E(i, j, t, Qx, a, b):
    """Hermite expansion coefficient E_t^{ij} of the product of two 1-D Gaussians."""
    p = a + b
    q = a * b / p
    if t < 0 or t > i + j:
        return 0.0
    if i == j == t == 0:
        return math.exp(-q * Qx * Qx)
    if j == 0:
        return (_E(i - 1, j, t - 1, Qx, a, b) / (2 * p) - q * Qx / a * _E(i - 1, j, t, Qx, a, b)
                + (t + 1) * _E(i - 1, j, t + 1, Qx, a, b))
    return (_E(i, j - 1, t - 1, Qx, a, b) / (2 * p) + q * Qx / b * _E(i, j - 1, t, Qx, a, b)
            + (t + 1) * _E(i, j - 1, t + 1, Qx, a, b))


def _overlap_prim(a, lmn1, A, b, lmn2, B):
    p = a + b
    return (_E(lmn1[0], lmn2[0], 0, A[0] - B[0], a, b) * _E(lmn1[1], lmn2[1], 0, A[1] - B[1], a, b)
            * _E(lmn1[2], lmn2[2], 0, A[2] - B[2], a, b) * (math.pi / p) ** 1.5)


def _kinetic_prim(a, lmn1, A, b, lmn2, B):
    l2, m2, n2 = lmn2
    t0 = b * (2 * (l2 + m2 + n2) + 3) * _overlap_prim(a, lmn1, A, b, lmn2, B)
    t1 = -2 * b * b * (_overlap_prim(a, lmn1, A, b, (l2 + 2, m2, n2), B) +
                       _overlap_prim(a, lmn1, A, b, (l2, m2 + 2, n2), B) +
                       _overlap_prim(a, lmn1, A, b, (l2, m2, n2 + 2), B))
    t2 = -0.5 * (l2 * (l2 - 1) * _overlap_prim(a, lmn1, A, b, (l2 - 2, m2, n2), B) +
                 m2 * (m2 - 1) * _overlap_prim(a, lmn1, A, b, (l2, m2 - 2, n2), B) +
                 n2 * (n2 - 1) * _overlap_prim(a, lmn1, A, b, (l2, m2, n2 - 2), B))
    return t0 + t1 + t2


def _boys(n, T):
    if T < 1e-12:
        return 1.0 / (2 * n + 1)
    return 0.5 * T ** (-(n + 0.5)) * gamma(n + 0.5) * gammainc(n + 0.5, T)


def _R(t, u, v, n, p, PCx, PCy, PCz, RPC):
    """Hermite Coulomb integral R^n_{tuv}."""
    T = p * RPC * RPC
    if t == u == v == 0:
        return (-2 * p) ** n * _boys(n, T)
    if t == u == 0:
        val = 0.0
        if v > 1:
            val += (v - 1) * _R(t, u, v - 2, n + 1, p, PCx, PCy, PCz, RPC)
        return val + PCz * _R(t, u, v - 1, n + 1, p, PCx, PCy, PCz, RPC)
    if t == 0:
        val = 0.0
        if u > 1:
            val += (u - 1) * _R(t, u - 2, v, n + 1, p, PCx, PCy, PCz, RPC)
        return val + PCy * _R(t, u - 1, v, n + 1, p, PCx, PCy, PCz, RPC)
    val = 0.0
    if t > 1:
        val += (t - 1) * _R(t - 2, u, v, n + 1, p, PCx, PCy, PCz, RPC)
    return val + PCx * _R(t - 1, u, v, n + 1, p, PCx, PCy, PCz, RPC)


def _nuclear_prim(a, lmn1, A, b, lmn2, B, C):
    p = a + b
    P = (a * A + b * B) / p
    PC = P - C
    RPC = float(np.linalg.norm(PC))
    val = 0.0
    for t in range(lmn1[0] + lmn2[0] + 1):
        for u in range(lmn1[1] + lmn2[1] + 1):
            for v in range(lmn1[2] + lmn2[2] + 1):
                val += (_E(lmn1[0], lmn2[0], t, A[0] - B[0], a, b) * _E(lmn1[1], lmn2[1], u, A[1] - B[1], a, b)
                        * _E(lmn1[2], lmn2[2], v, A[2] - B[2], a, b)
                        * _R(t, u, v, 0, p, PC[0], PC[1], PC[2], RPC))
    return 2 * math.pi / p * val


def _eri_prim(a, l1, A, b, l2, B, c, l3, C, d, l4, D):
    p, q = a + b, c + d
    alpha = p * q / (p + q)
    P = (a * A + b * B) / p
    Q = (c * C + d * D) / q
    PQ = P - Q
    RPQ = float(np.linalg.norm(PQ))
    val = 0.0
    for t in range(l1[0] + l2[0] + 1):
        Et = _E(l1[0], l2[0], t, A[0] - B[0], a, b)
        for u in range(l1[1] + l2[1] + 1):
            Eu = _E(l1[1], l2[1], u, A[1] - B[1], a, b)
            for v in range(l1[2] + l2[2] + 1):
                Ev = _E(l1[2], l2[2], v, A[2] - B[2], a, b)
                for tau in range(l3[0] + l4[0] + 1):
                    Etau = _E(l3[0], l4[0], tau, C[0] - D[0], c, d)
                    for nu in range(l3[1] + l4[1] + 1):
                        Enu = _E(l3[1], l4[1], nu, C[1] - D[1], c, d)
                        for phi in range(l3[2] + l4[2] + 1):
                            Ephi = _E(l3[2], l4[2], phi, C[2] - D[2], c, d)
                            val += (Et * Eu * Ev * Etau * Enu * Ephi * (-1) ** (tau + nu + phi)
                                    * _R(t + tau, u + nu, v + phi, 0, alpha, PQ[0], PQ[1], PQ[2], RPQ))
    return 2 * math.pi ** 2.5 / (p * q * math.sqrt(p + q)) * val


def _contract2(f, sa, sb, *extra):
    return sum(ca * cb * f(a, sa.lmn, sa.A, b, sb.lmn, sb.A, *extra)
               for a, ca in zip(sa.exps, sa.coefs) for b, cb in zip(sb.exps, sb.coefs))


def ao_integrals(atoms):
    """S, T + V (core Hamiltonian), ERI (chemists' (ij|kl)) in the AO basis, E_nuc."""
    bs = basis(atoms)
    n = len(bs)
    S = np.zeros((n, n))
    Hc = np.zeros((n, n))
    for i in range(n):
        for j in range(i + 1):
            S[i, j] = S[j, i] = _contract2(_overlap_prim, bs[i], bs[j])
            t = _contract2(_kinetic_prim, bs[i], bs[j])
            v = sum(-_Z[sym] * _contract2(_nuclear_prim, bs[i], bs[j], np.asarray(xyz, float)) for sym, xyz in atoms)
            Hc[i, j] = Hc[j, i] = t + v
    eri = np.zeros((n, n, n, n))
    for i in range(n):
        for j in range(i + 1):
            for k in range(n):
                for l in range(k + 1):
                    if i * (i + 1) // 2 + j < k * (k + 1) // 2 + l:
                        continue
                    si, sj, sk, sl = bs[i], bs[j], bs[k], bs[l]
                    val = 0.0
                    for a, ca in zip(si.exps, si.coefs):
                        for b, cb in zip(sj.exps, sj.coefs):
                            for c, cc in zip(sk.exps, sk.coefs):
                                for d, cd in zip(sl.exps, sl.coefs):
                                    val += ca * cb * cc * cd * _eri_prim(a, si.lmn, si.A, b, sj.lmn, sj.A,
                                                                         c, sk.lmn, sk.A, d, sl.lmn, sl.A)
                    for (p, q, r, s) in ((i, j, k, l), (j, i, k, l), (i, j, l, k), (j, i, l, k),
                                         (k, l, i, j), (l, k, i, j), (k, l, j, i), (l, k, j, i)):
                        eri[p, q, r, s] = val
    enuc = 0.0
    for x in range(len(atoms)):
        for y in range(x):
            enuc += _Z[atoms[x][0]] * _Z[atoms[y][0]] / np.linalg.norm(np.subtract(atoms[x][1], atoms[y][1]))
    return S, Hc, eri, enuc


def rhf(S, Hc, eri, n_occ, max_iter=200, tol=1e-12):
    """Plain restricted Hartree-Fock (Roothaan-Hall iterations with DIIS)."""
    s, U = np.linalg.eigh(S)
    X = U @ np.diag(s ** -0.5) @ U.T
    F = Hc.copy()
    D = np.zeros_like(S)
    e_old = 0.0
    errs, focks = [], []
    for it in range(max_iter):
        e, C = np.linalg.eigh(X.T @ F @ X)
        C = X @ C
        Cocc = C[:, :n_occ]
        D = 2 * Cocc @ Cocc.T
        J = np.einsum("pqrs,rs->pq", eri, D)
        K = np.einsum("prqs,rs->pq", eri, D)
        F = Hc + J - 0.5 * K
        e_el = 0.5 * np.sum(D * (Hc + F))
        err = F @ D @ S - S @ D @ F
        errs.append(err)
        focks.append(F)
        if len(errs) > 8:
            errs.pop(0)
            focks.pop(0)
        if len(errs) > 2:
            m = len(errs)
            B = -np.ones((m + 1, m + 1))
            B[m, m] = 0.0
            for a in range(m):
                for b in range(m):
                    B[a, b] = np.sum(errs[a] * errs[b])
            rhs = np.zeros(m + 1)
            rhs[m] = -1.0
            c = np.linalg.solve(B, rhs)
            F = sum(c[a] * focks[a] for a in range(m))
        if abs(e_el - e_old) < tol and np.abs(err).max() < 1e-9:
            break
        e_old = e_el
    e, C = np.linalg.eigh(X.T @ F @ X)
    return e_el, X @ C, e


def molecular_integrals(atoms, n_electrons):
    """(h1, h2, e_core, E_HF, mo energies) in the RHF MO basis (all orbitals active)."""
    S, Hc, eri, enuc = ao_integrals(atoms)
    e_el, C, eps = rhf(S, Hc, eri, n_electrons // 2)
    h1 = C.T @ Hc @ C
    h2 = np.einsum("pi,qj,rk,sl,pqrs->ijkl", C, C, C, C, eri, optimize=True)
    return h1, h2, enuc, e_el + enuc, eps


def water(r_oh_angstrom: float = 0.9578, angle_deg: float = 104.5):
    """H2O in the yz plane, O at the origin (the PySCF documentation geometry by default)."""
    th = math.radians(angle_deg) / 2
    r = r_oh_angstrom * ANG
    return [("O", (0.0, 0.0, 0.0)), ("H", (0.0, -r * math.sin(th), r * math.cos(th))),
            ("H", (0.0, r * math.sin(th), r * math.cos(th)))]
