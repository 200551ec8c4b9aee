"""Symbolic Jordan-Wigner transformation with explicit Pauli strings
(TEST INFRASTRUCTURE ONLY).

Eq. (9) -> Eq. (10): every ladder operator becomes
  a_j  = Z_0 ... Z_{j-1} (X_j + i Y_j)/2,   a+_j = Z_0 ... Z_{j-1} (X_j - i Y_j)/2
and products of Pauli strings are taken qubit by qubit with the textbook
single-qubit table (XY = iZ, YZ = iX, ZX = iY, ...), complex coefficients
summed per string (the OpenFermion convention the paper uses).  Then
Algorithm 1 groups the strings by their X/Y flip mask and
fuses coeff <- Re(c) * Re((-i)^{Y_occ}).

This is deliberately a different derivation from anything in the CUDA
library: strings carry Y explicitly and phases are tracked as complex numbers.
"""
from __future__ import annotations

# single-qubit Pauli products: (a, b) -> (phase, c) with a*b = phase * c
_MUL = {
    ("I", "I"): (1, "I"), ("I", "X"): (1, "X"), ("I", "Y"): (1, "Y"), ("I", "Z"): (1, "Z"),
    ("X", "I"): (1, "X"), ("X", "X"): (1, "I"), ("X", "Y"): (1j, "Z"), ("X", "Z"): (-1j, "Y"),
    ("Y", "I"): (1, "Y"), ("Y", "X"): (-1j, "Z"), ("Y", "Y"): (1, "I"), ("Y", "Z"): (1j, "X"),
    ("Z", "I"): (1, "Z"), ("Z", "X"): (1j, "Y"), ("Z", "Y"): (-1j, "X"), ("Z", "Z"): (1, "I"),
}


def _mul_strings(a: dict, b: dict):
    """Product of two Pauli strings stored sparsely as {qubit: 'X'|'Y'|'Z'}."""
    phase = 1
    out = dict(a)
    for q, pb in b.items():
        pa = out.get(q, "I")
        ph, pc = _MUL[(pa, pb)]
        phase *= ph
        if pc == "I":
            out.pop(q, None)
        else:
            out[q] = pc
    return phase, out


def ladder(j: int, dagger: bool):
    """JW image of a_j (dagger=False) or a+_j as [(coeff, string)]."""
    zs = {k: "Z" for k in range(j)}
    sx = dict(zs); sx[j] = "X"
    sy = dict(zs); sy[j] = "Y"
    return [(0.5, sx), ((-0.5j if dagger else 0.5j), sy)]


def _product(ops):
    terms = [(1.0 + 0j, {})]
    for op in ops:
        new = []
        for c1, s1 in terms:
            for c2, s2 in op:
                ph, s = _mul_strings(s1, s2)
                new.append((c1 * c2 * ph, s))
        terms = new
    return terms


def _key(s: dict):
    return tuple(sorted(s.items()))


def pauli_hamiltonian(h1, h2, e_core):
    """Eq. (10): {string_key: complex c} for Eq. (9) with chemists' spatial
    integrals, spin orbital (p,s) -> qubit 2p+s."""
    n = h1.shape[0]
    acc = {(): complex(e_core)}
    lad = {}

    def L(j, d):
        if (j, d) not in lad:
            lad[(j, d)] = ladder(j, d)
        return lad[(j, d)]

    def add(coef, ops):
        for c, s in _product(ops):
            k = _key(s)
            acc[k] = acc.get(k, 0j) + coef * c

    for p in range(n):
        for q in range(n):
            if h1[p, q] != 0.0:
                for s in range(2):
                    add(h1[p, q], [L(2 * p + s, True), L(2 * q + s, False)])
    for p in range(n):
        for q in range(n):
            for r in range(n):
                for s_ in range(n):
                    v = h2[p, q, r, s_]
                    if v == 0.0:
                        continue
                    for sg in range(2):
                        for tau in range(2):
                            P, Q, Rr, S = 2 * p + sg, 2 * q + sg, 2 * r + tau, 2 * s_ + tau
                            if P == Rr or Q == S:
                                continue
                            add(0.5 * v, [L(P, True), L(Rr, True), L(S, False), L(Q, False)])
    return acc


def fused_groups(pauli: dict, tol: float):
    """Algorithm 1: {X_mask: [(Z_mask, fused d)]} with
    pmXY = X|Y positions, pmYZ = Y|Z positions, d = Re(c) * Re((-i)^{Y_occ}).
    Strings with |d| <= tol are dropped (odd Y_occ gives Re((-i)^odd) = 0)."""
    groups = {}
    for k, c in pauli.items():
        xm = zm = 0
        ny = 0
        for q, op in k:
            if op in ("X", "Y"):
                xm |= 1 << q
            if op in ("Y", "Z"):
                zm |= 1 << q
            if op == "Y":
                ny += 1
        d = c.real * ((-1j) ** ny).real
        if abs(d) > tol:
            groups.setdefault(xm, []).append((zm, d))
    for xm in groups:
        groups[xm].sort()
    return groups
