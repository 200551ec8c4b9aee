"""Host compress (nnqs_ham_compress, C++ in libnnqs, device=-1 handle) against
the oracle's two independent derivations of the grouped table (Fig. 6(c)):
symbolic JW + Algorithm 1 fusion, and the closed-form counts.  Parity P1/P2:
flip masks and Z masks bit-exact, signs exact, |dd| <= 1e-13 max|d|."""
import numpy as np
import pytest

from oracle import counts, jw
from synth import configs as C


@pytest.fixture(scope="module")
def nnqs():
    import __graft_entry__ as g
    g.build()
    from paper_2306_16705_b200 import nnqs as m
    return m


def _compare(x, off, z, d, ref):
    xs = [int(a) | (int(b) << 64) for a, b in x]
    assert xs == sorted(ref)
    scale = max(abs(v) for lst in ref.values() for _, v in lst)
    for k, X in enumerate(xs):
        zs = [int(a) | (int(b) << 64) for a, b in z[off[k]:off[k + 1]]]
        assert zs == [zz for zz, _ in ref[X]]
        for (_, dr), dg in zip(ref[X], d[off[k]:off[k + 1]]):
            assert np.sign(dr) == np.sign(dg)
            assert abs(dr - dg) <= 1e-13 * scale


@pytest.mark.parametrize("c", [1, 2, 3])
def test_compress_equals_symbolic_jw(nnqs, c):
    m = C.molecule(c)
    h = nnqs.nnqs_ham_compress(m.h1, m.h2, m.n_qubits, m.e_core, device=-1)
    tol = 1e-12 * max(np.abs(m.h1).max(), np.abs(m.h2).max())
    _compare(*h.export(), jw.fused_groups(jw.pauli_hamiltonian(m.h1, m.h2, m.e_core), tol))


@pytest.mark.parametrize("c", [1, 2, 3, 4, 5])
def test_compress_counts_closed_form(nnqs, c):
    """K' and N_h equal the closed forms (C4: Table 1's N2 N_h = 2239)."""
    m = C.molecule(c)
    h = nnqs.nnqs_ham_compress(m.h1, m.h2, m.n_qubits, m.e_core, device=-1)
    inf = h.info()
    assert (inf["n_groups"], inf["n_terms"]) == counts.group_counts_fast(m.irreps)
    if c == 5:
        x, off, z, d = h.export()
        # groups ascending as 128-bit integers, CSR offsets consistent
        hi, lo = x[:, 1], x[:, 0]
        assert np.all((hi[1:] > hi[:-1]) | ((hi[1:] == hi[:-1]) & (lo[1:] > lo[:-1])))
        assert off[0] == 0 and off[-1] == len(d) and np.all(np.diff(off) > 0)
        # every flip mask is a spin-conserving 0/2/4-site excitation pattern
        pc = np.array([bin(int(a)).count("1") + bin(int(b)).count("1") for a, b in x[:2000]])
        assert set(pc) <= {0, 2, 4}


def test_from_pauli_spec_example(nnqs):
    """{c1 ZI, c2 IZ, c3 XX, c4 YY} -> 2 groups, idxs [0,2,4], YY fused = -c4."""
    c1, c2, c3, c4 = 0.3, -0.7, 0.11, 0.25
    X = [[0, 0], [0, 0], [3, 0], [3, 0]]
    Z = [[1, 0], [2, 0], [0, 0], [3, 0]]
    h = nnqs.nnqs_ham_from_pauli(X, Z, [c1, c2, c3, c4], 2, device=-1)
    x, off, z, d = h.export()
    assert list(x[:, 0]) == [0, 3] and list(off) == [0, 2, 4]
    assert list(z[:, 0]) == [1, 2, 0, 3]
    assert list(d) == [c1, c2, c3, -c4]
    h = nnqs.nnqs_ham_from_pauli([[0, 0]], [[0, 0]], [-0.8], 4, device=-1)
    assert h.info()["n_groups"] == 1


@pytest.mark.parametrize("c", [3, 4, 5])
def test_flip_mask_set_equals_symmetry_allowed_set(nnqs, c):
    """P1 at N = 14, 20 and 120: the exported X set is, bit for bit,
    the symmetry-allowed excitation set written out from the irrep labels
    (oracle.counts.flip_masks); at N = 20 its N_h is Table 1's N2 value."""
    m = C.molecule(c)
    h = nnqs.nnqs_ham_compress(m.h1, m.h2, m.n_qubits, m.e_core, device=-1)
    x = h.export()[0]
    got = {int(a) | (int(b) << 64) for a, b in x}
    assert len(got) == len(x)
    assert got == counts.flip_masks(m.irreps)
