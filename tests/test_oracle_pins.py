"""Pins of the CPU oracle against facts fixed by the paper and by mathematics
(not against itself).  CPU only.

Each test names what it pins; a plausible oracle mistake (dropped term, wrong
JW sign, transposed integral index, word-boundary bug at qubit 64) fails at
least one of them.
"""
import itertools
import math
import os

import numpy as np
import pytest

from oracle import counts, dense, energy, jw
from oracle import rows as R
from synth import configs as C
from synth import integrals as I
from synth import samples as S

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    out = {}
    for line in open(os.path.join(GOLD, name)):
        line = line.strip()
        if line and not line.startswith("#"):
            k, *v = line.split()
            out[k] = v
    return out


# ---------------------------------------------------------------- H2 closed form
def test_h2_fci_closed_form():
    """2x2 CI in the {sigma_g^2, sigma_u^2} basis (Szabo-Ostlund 4.4) vs the
    oracle's sector diagonalisation of its term-by-term H (Eq. 9)."""
    g = {k: float(v[0]) for k, v in _golden("h2_sto3g.txt").items()}
    E1 = 2 * g["h11"] + g["J11"]
    E2 = 2 * g["h22"] + g["J22"]
    K = g["K12"]
    e_closed = 0.5 * ((E1 + E2) - math.sqrt((E2 - E1) ** 2 + 4 * K * K)) + g["e_core"]
    h1, h2, e, na, nb = I.h2_sto3g()
    keys = S.sector_keys(2, na, nb)
    e0, psi, _ = dense.ground_state(h1, h2, e, keys)
    assert abs(e0 - e_closed) < 1e-13
    assert abs(e0 - g["E_fci_textbook"]) < 1e-4


def test_h2_pauli_counts_fig6a():
    """Fig. 6(a): H2, 4 qubits -> 15 strings in 2 flip groups."""
    g = _golden("h2_sto3g.txt")
    h1, h2, e, _, _ = I.h2_sto3g()
    tab = dense.pauli_recovery(dense.fermionic_sparse_H(h1, h2, e), 4, 1e-12)
    assert len(tab) == int(g["K"][0])
    assert sum(len(v) for v in tab.values()) == int(g["N_h"][0])
    assert sorted(tab) == [0, 0b1111]


# ---------------------------------------------------- independent constructions
@pytest.mark.parametrize("which", ["h2", "rand8"])
def test_fermionic_rows_equal_kronecker(which):
    """Term-by-term JW rows (C oracle) == explicit Kronecker-product operators."""
    if which == "h2":
        h1, h2, e, _, _ = I.h2_sto3g()
    else:
        h1, h2, e = I.random_dense_integrals(4, 11)
    Hf = dense.fermionic_sparse_H(h1, h2, e).toarray()
    Hk = dense.kron_dense_H(h1, h2, e)
    assert np.max(np.abs(Hf - Hk)) < 1e-13 * max(1.0, np.max(np.abs(Hk)))


def test_hermitian_and_conserving():
    """H is real symmetric and conserves N_alpha, N_beta."""
    h1, h2, e = I.random_dense_integrals(4, 12)
    H = dense.fermionic_sparse_H(h1, h2, e).tocoo()
    Hd = H.toarray()
    assert np.max(np.abs(Hd - Hd.T)) == 0.0
    a = lambda x: bin(x & 0x5555).count("1")
    b = lambda x: bin(x & 0xAAAA).count("1")
    for i, j in zip(H.row, H.col):
        assert a(int(i)) == a(int(j)) and b(int(i)) == b(int(j))


def test_slater_condon_diagonal():
    """H_xx = e_core + sum_occ h_pp + 1/2 sum_{P!=Q occ} [(pp|qq) - d_s (pq|qp)]."""
    h1, h2, e = I.random_dense_integrals(4, 13)
    Hd = dense.fermionic_sparse_H(h1, h2, e).diagonal()
    for x in range(256):
        occ = [P for P in range(8) if (x >> P) & 1]
        v = e + sum(h1[P // 2, P // 2] for P in occ)
        for P in occ:
            for Q in occ:
                if P != Q:
                    p, q = P // 2, Q // 2
                    v += 0.5 * (h2[p, p, q, q] - (h2[p, q, q, p] if P % 2 == Q % 2 else 0.0))
        assert abs(Hd[x] - v) < 1e-13


def test_coulomb_only_is_diagonal():
    """Only (pp|qq) and diagonal h: E_loc(x) = H_xx for any psi."""
    h1, h2, e = I.coulomb_only_integrals(4, 14)
    H = dense.fermionic_sparse_H(h1, h2, e).toarray()
    assert np.count_nonzero(H - np.diag(np.diag(H))) == 0
    lp = S.random_logpsi(256, 15)
    rows = np.array([[x, 0] for x in range(256)], dtype=np.uint64)
    el = R.eloc(h1, h2, e, rows, lp, keys=None, logpsi=lp)
    assert np.max(np.abs(el - np.diag(H))) < 1e-13


# ------------------------------------------------------------ local energy pins
def test_quadratic_form_exact_mode():
    """sum_x |psi|^2 E_loc(x) / sum |psi|^2 = <psi|H|psi>/<psi|psi> (Eqs. 2-5,
    PAPER.md:129-145) with <psi|H|psi> from the Kronecker-built dense H."""
    h1, h2, e = I.random_dense_integrals(4, 16)
    Hk = dense.kron_dense_H(h1, h2, e)
    lp = S.random_logpsi(256, 17)
    psi = np.exp(lp[:, 0] + 1j * lp[:, 1])
    rows = np.array([[x, 0] for x in range(256)], dtype=np.uint64)
    el = R.eloc(h1, h2, e, rows, lp, keys=None, logpsi=lp)
    p = np.abs(psi) ** 2
    lhs = np.sum(p * el) / np.sum(p)
    rhs = np.vdot(psi, Hk @ psi) / np.vdot(psi, psi)
    assert abs(lhs - rhs) < 1e-12 * abs(rhs)
    assert abs(lhs.imag) < 1e-12 * abs(rhs)


def test_counts_consistent_reduce():
    """Re log psi = 1/2 ln(count) makes the count-weighted mean (Eq. 6) equal the
    exact variational energy (Eq. 2), i.e. the reduce is pinned end to end."""
    h1, h2, e = I.random_dense_integrals(3, 18)
    Hk = dense.kron_dense_H(h1, h2, e)
    rng = np.random.default_rng(19)
    cnt = rng.integers(1, 50, size=64)
    lp = np.stack([0.5 * np.log(cnt), rng.uniform(-np.pi, np.pi, 64)], axis=1)
    psi = np.exp(lp[:, 0] + 1j * lp[:, 1])
    rows = np.array([[x, 0] for x in range(64)], dtype=np.uint64)
    el = R.eloc(h1, h2, e, rows, lp, keys=None, logpsi=lp)
    mean, var, W = energy.energy(el, cnt)
    rhs = np.vdot(psi, Hk @ psi) / np.vdot(psi, psi)
    assert abs(mean - rhs) < 1e-12 * abs(rhs)
    assert W == cnt.sum() and var > 0


def test_ground_state_local_energy_constant():
    """psi = exact sector ground state -> E_loc(x) = E_0 on supp(psi)
    (north star).  C2 (LiH-shaped, 225-dim sector)."""
    mol = C.molecule(2)
    keys = S.sector_keys(mol.n_orb, mol.n_alpha, mol.n_beta)
    e0, psi, H = dense.ground_state(mol.h1, mol.h2, mol.e_core, keys)
    res = np.max(np.abs(H @ psi - e0 * psi))
    amp = np.abs(psi)
    sup = amp > 1e-12 * amp.max()
    lp = np.stack([np.where(sup, np.log(np.where(sup, amp, 1.0)), -np.inf),
                   np.where(psi < 0, np.pi, 0.0)], axis=1)
    el = R.eloc(mol.h1, mol.h2, mol.e_core, keys[sup], lp[sup], keys=keys, logpsi=lp)
    tol = 1e-10 * abs(e0) + 10 * res / amp[sup]
    assert np.all(np.abs(el - e0) <= tol)
    assert np.all(np.abs(el.imag) <= tol)


def test_sample_space_full_sector_equals_exact():
    """T = the whole sector and psi = 0 outside it: sample-aware == exact
    (SPEC.md:259)."""
    mol = C.molecule(2)
    N = mol.n_qubits
    keys = S.sector_keys(mol.n_orb, mol.n_alpha, mol.n_beta)
    lp_t = S.random_logpsi(len(keys), 21)
    lp_full = np.full((1 << N, 2), [-np.inf, 0.0])
    lp_full[keys[:, 0].astype(np.int64)] = lp_t
    sel = np.arange(0, len(keys), 7)
    a = R.eloc(mol.h1, mol.h2, mol.e_core, keys[sel], lp_t[sel], keys=keys, logpsi=lp_t)
    b = R.eloc(mol.h1, mol.h2, mol.e_core, keys[sel], lp_t[sel], keys=None, logpsi=lp_full)
    assert np.max(np.abs(a - b)) < 1e-12 * np.max(np.abs(a))


def test_absent_configurations_contribute_zero():
    """T = {x}: only the diagonal survives."""
    h1, h2, e = I.random_dense_integrals(4, 22)
    Hd = dense.fermionic_sparse_H(h1, h2, e).diagonal()
    for x in (0b00110011, 0b01011010):
        k = np.array([[x, 0]], dtype=np.uint64)
        lp = np.array([[-0.3, 1.1]])
        el = R.eloc(h1, h2, e, k, lp, keys=k, logpsi=lp)
        assert abs(el[0] - Hd[x]) < 1e-13


def test_zero_amplitude_row_is_nan():
    """psi(x) = 0 makes E_loc 0/0 (reading R10)."""
    h1, h2, e, _, _ = I.h2_sto3g()
    lp = S.random_logpsi(16, 23)
    lp[5, 0] = -np.inf
    rows = np.array([[5, 0], [3, 0]], dtype=np.uint64)
    el = R.eloc(h1, h2, e, rows, lp[[5, 3]], keys=None, logpsi=lp)
    assert np.isnan(el[0]) and np.isfinite(el[1])


# ----------------------------------------------------- Pauli table (Fig. 6(c))
@pytest.mark.parametrize("c", [1, 2, 3])
def test_symbolic_jw_equals_walsh_recovery(c):
    """Two derivations of the grouped fused table: symbolic JW + Algorithm 1's
    fusion vs the Walsh-Hadamard transform of the oracle's
    dense H.  Same X set, same Z sets, coefficients within 1e-13."""
    mol = C.molecule(c)
    tol = 1e-12 * max(np.abs(mol.h1).max(), np.abs(mol.h2).max())
    A = jw.fused_groups(jw.pauli_hamiltonian(mol.h1, mol.h2, mol.e_core), tol)
    B = dense.pauli_recovery(dense.fermionic_sparse_H(mol.h1, mol.h2, mol.e_core), mol.n_qubits, tol)
    assert sorted(A) == sorted(B)
    scale = max(abs(d) for v in A.values() for _, d in v)
    for X in A:
        za = [z for z, _ in A[X]]
        zb = [z for z, _ in B[X]]
        assert za == zb
        for (_, da), (_, db) in zip(A[X], B[X]):
            assert abs(da - db) <= 1e-13 * scale
    k, nh = counts.group_counts(mol.irreps)
    assert len(A) == k and sum(len(v) for v in A.values()) == nh


def test_table1_n2_string_count():
    """Table 1: N2 / STO-3G has N_h = 2239 Pauli strings; the
    closed-form count with D2h labels of the 10 N2 orbitals reproduces it."""
    g = _golden("table1_counts.txt")
    mol = C.molecule(4)
    assert mol.n_qubits == int(g["N2"][0])
    assert counts.group_counts(mol.irreps)[1] == int(g["N2"][2])


def test_closed_form_counts_brute_force():
    """Closed-form K', N_h == brute-force enumeration of X/Z masks for random
    labels at n <= 6 (via symbolic JW)."""
    for seed, labels in [(31, [0, 1, 0, 1, 0]), (32, [0, 1, 2, 3, 0, 2])]:
        h1, h2, e = I.synthetic_integrals(len(labels), labels, seed)
        A = jw.fused_groups(jw.pauli_hamiltonian(h1, h2, e), 1e-12 * np.abs(h2).max())
        assert (len(A), sum(len(v) for v in A.values())) == counts.group_counts(labels)
    assert counts.group_counts_fast([p % 2 for p in range(14)]) == counts.group_counts([p % 2 for p in range(14)])


# ------------------------------------------------- words >= 64 (N up to 128)
def _embed(h1, h2, slots, n_big):
    H1 = np.zeros((n_big, n_big))
    H2 = np.zeros((n_big,) * 4)
    for i, p in enumerate(slots):
        for j, q in enumerate(slots):
            H1[p, q] = h1[i, j]
            for k, r in enumerate(slots):
                for l, s in enumerate(slots):
                    H2[p, q, r, s] = h2[i, j, k, l]
    return H1, H2


def _spread(y, slots, frozen):
    x = 0
    for i, p in enumerate(slots):
        for s in range(2):
            if (y >> (2 * i + s)) & 1:
                x |= 1 << (2 * p + s)
    for j in frozen:
        x |= 1 << j
    return np.array([x & ((1 << 64) - 1), x >> 64], dtype=np.uint64)


def test_embedding_across_word_boundary_rows():
    """4 active orbitals at spatial 28, 31, 33, 50 of a 60-orbital system (qubits
    56..101, straddling qubit 64), 21 frozen electrons on qubits 0..20 below
    them (odd, so a JW string that forgot word 0 flips sign): every row
    equals the N = 8 row (frozen electrons below all active sites cancel in
    each JW string)."""
    h1, h2, e = I.random_dense_integrals(4, 24)
    slots, frozen = [28, 31, 33, 50], list(range(21))
    H1, H2 = _embed(h1, h2, slots, 60)
    Hs = dense.fermionic_sparse_H(h1, h2, e).toarray()
    sec = [y for y in range(256) if bin(y & 0x55).count("1") == 2 and bin(y & 0xAA).count("1") == 1]
    keys = np.array([_spread(y, slots, frozen) for y in sec], dtype=np.uint64)
    order = np.lexsort((keys[:, 0], keys[:, 1]))
    keys_s = keys[order]
    for j, y in enumerate(sec):
        idx, hv = R.row_hits(H1, H2, e, keys[j], keys=keys_s)
        got = {sec[order[i]]: v for i, v in zip(idx, hv)}
        want = {yp: Hs[yp, y] for yp in sec if Hs[yp, y] != 0.0}
        assert set(got) == set(want)
        for yp in want:
            assert got[yp] == want[yp] + 0.0 or abs(got[yp] - want[yp]) < 1e-14


def test_embedding_spectrum_with_interleaved_core():
    """Frozen electrons BETWEEN active orbitals turn the embedding into a sign
    gauge: the sector spectrum must still equal the N = 8 one."""
    h1, h2, e = I.random_dense_integrals(4, 25)
    slots, frozen = [20, 40, 45, 59], [7, 60, 61, 62, 85, 117]
    H1, H2 = _embed(h1, h2, slots, 60)
    sec = [y for y in range(256) if bin(y & 0x55).count("1") == 2 and bin(y & 0xAA).count("1") == 2]
    keys = np.array([_spread(y, slots, frozen) for y in sec], dtype=np.uint64)
    keys = keys[np.lexsort((keys[:, 0], keys[:, 1]))]
    w_big = np.linalg.eigvalsh(dense.sector_hamiltonian(H1, H2, e, keys))
    ks = np.array([[y, 0] for y in sec], dtype=np.uint64)
    w_small = np.linalg.eigvalsh(dense.sector_hamiltonian(h1, h2, e, ks))
    assert np.max(np.abs(w_big - w_small)) < 1e-12


# ---------------------------------------------------------------- reduce pins
def test_reduce_spec_examples():
    """all equal -> var 0; weights (3,1), E (0,4) -> mean 1, var 3."""
    m, v, W = energy.energy([2.5 + 0.1j] * 5, [1, 2, 3, 4, 5])
    assert m == 2.5 + 0.1j and v == 0.0 and W == 15
    m, v, W = energy.energy([0.0, 4.0], [3, 1])
    assert m == 1.0 and v == 3.0 and W == 4
    with pytest.raises(ValueError):
        energy.energy([1.0], [0])


# ---------------------------------------------- Eq. (7) gradient weights (NEXT-3)
@pytest.mark.parametrize("which", ["h2", "n4"])
def test_grad_weights_equal_finite_differences(which):
    """Eq. (7): with psi(x) = sqrt(c_x) exp(theta_x + i phi_x)
    over the whole Fock space (integer weights c_x = |psi|^2 at theta = 0), the
    weights a_x, b_x of grad ln|psi(x)| and grad phi(x) are exactly dE/dtheta_x and
    dE/dphi_x of E = <psi|H|psi>/<psi|psi>, H built independently from Kronecker
    ladder operators -- central differences, relative error <= 1e-6."""
    if which == "h2":
        m = C.molecule(1)
        h1, h2, ec = m.h1, m.h2, m.e_core
    else:
        h1, h2, ec = I.synthetic_integrals(4, [0, 1, 0, 1], 77, e_core=3.0)
    N = 2 * h1.shape[0]
    dim = 1 << N
    rng = np.random.default_rng(5)
    c = rng.integers(1, 10, size=dim)
    phi = rng.uniform(-np.pi, np.pi, size=dim)
    H = dense.kron_dense_H(h1, h2, ec)

    def E(theta, ph):
        psi = np.sqrt(c) * np.exp(theta + 1j * ph)
        return float(np.real(np.vdot(psi, H @ psi)) / np.real(np.vdot(psi, psi)))

    lp = np.stack([0.5 * np.log(c), phi], axis=1)
    el = R.eloc(h1, h2, ec, np.array([[x, 0] for x in range(dim)], dtype=np.uint64), lp, keys=None, logpsi=lp)
    a, b = energy.grad_weights(el, c)
    eps = 1e-5
    z = np.zeros(dim)
    for x in rng.choice(dim, size=min(dim, 12), replace=False):
        e = np.zeros(dim)
        e[x] = eps
        da = (E(z + e, phi) - E(z - e, phi)) / (2 * eps)
        db = (E(z, phi + e) - E(z, phi - e)) / (2 * eps)
        scale = max(1e-3, np.max(np.abs(a)), np.max(np.abs(b)))
        assert abs(da - a[x]) <= 1e-6 * scale, (x, da, a[x])
        assert abs(db - b[x]) <= 1e-6 * scale, (x, db, b[x])


def test_grad_weights_constant_eloc_is_zero():
    """Constant E_loc gives exactly zero weights (centred estimator)."""
    a, b = energy.grad_weights(np.full(7, -1.25 + 0.5j), [1, 2, 3, 4, 5, 6, 7])
    assert np.all(a == 0.0) and np.all(b == 0.0)


def test_compressed_layout_memory_reduction():
    """Fig. 6(c) vs 6(b) ("around 40%", "more than 40%"
    on their molecules): with the closed-form K', N_h of the N2-shaped D2h case
    (N_h = 2239 = Table 1) the byte model gives 1 - c/b = 38.4 %, and the same
    model stays within 35-45 % across C2-C5 (one byte per boolean)."""
    D2H = {"ag": 0, "b1g": 1, "b2g": 2, "b3g": 3, "au": 4, "b1u": 5, "b2u": 6, "b3u": 7}
    irr = [D2H[s] for s in ["ag", "b1u", "ag", "b1u", "b3u", "b2u", "ag", "b2g", "b3g", "b1u"]]
    k, nh = counts.group_counts(irr)
    assert (k, nh) == (378, 2239)
    b, c, red = counts.hamiltonian_memory(20, k, nh)
    assert (b, c) == (2239 * 52, 2239 * 28 + 378 * 24)
    assert abs(red - 0.3836) < 1e-3
    for cfg in (2, 3, 5):
        irr = C.molecule(cfg).irreps
        kk, hh = (counts.group_counts_fast if cfg == 5 else counts.group_counts)(irr)
        _, _, r = counts.hamiltonian_memory(2 * len(irr), kk, hh)
        assert 0.35 <= r <= 0.5, (cfg, r)
