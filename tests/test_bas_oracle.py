"""Pins of the BAS oracle (oracle/bas.py) against what the paper and probability fix
(-m "not gpu"): the binomial draws follow Binomial(n, p) (scipy's pmf, moments),
multinomial splits conserve the weight and respect Eq. (12)'s mask, a full BAS run
reproduces the autoregressive distribution it samples (Fig. 3(b)), and the
parallel partition reproduces the serial samples exactly.  Also the
product's host-side partition (sampler.partition) and the ansatz's normalisation."""
import numpy as np
import pytest
from scipy import stats

from oracle import bas


@pytest.mark.parametrize("n,p", [(7, 0.3), (60, 0.1), (25, 0.45), (50, 0.93), (1000, 0.3)])
def test_binomial_matches_pmf(n, p):
    N = 20000
    xs = np.array([bas.binomial(n, p, bas.Uniforms(11, n % 64, j, 7)) for j in range(N)])
    pm = stats.binom.pmf(np.arange(n + 1), n, p) * N
    h = np.bincount(xs, minlength=n + 1)
    sel = pm > 5
    obs = np.append(h[sel], h[~sel].sum())
    exp = np.append(pm[sel], pm[~sel].sum())
    if exp[-1] < 1:
        obs, exp = obs[:-1], exp[:-1] * obs[:-1].sum() / exp[:-1].sum()
    chi = ((obs - exp) ** 2 / exp).sum()
    assert stats.chi2.sf(chi, len(obs) - 1) > 1e-4
    assert xs.min() >= 0 and xs.max() <= n


@pytest.mark.parametrize("n,p", [(10**6, 0.5), (10**12, 0.25), (10**12, 2e-12), (10**9, 0.999)])
def test_binomial_large_n_moments(n, p):
    """BTRS and inversion with counts up to the paper's N_s = 10^12."""
    N = 4000
    xs = np.array([bas.binomial(n, p, bas.Uniforms(3, 1, j, 5)) for j in range(N)], dtype=float)
    m, v = n * p, n * p * (1 - p)
    assert abs(xs.mean() - m) <= 5 * np.sqrt(v / N)
    assert abs(xs.var() - v) <= 6 * v * np.sqrt(2 / N)


def test_binomial_edges():
    U = bas.Uniforms(0, 0, 0, 0)
    assert bas.binomial(0, 0.3, U) == 0 and bas.binomial(5, 0.0, U) == 0 and bas.binomial(5, 1.0, U) == 5


def test_split_conserves_and_masks():
    """Eq. (12) + reachability (R24): 2 orbitals, one up and one down electron.
    Root at orbital 1: every outcome is feasible; after '11' on orbital 1 only '00'."""
    rng = np.random.default_rng(0)
    for w in (1, 7, 1000, 10**12):
        pr = rng.random(4)
        c = bas.split_node(0, w, pr, 1, 1, 1, 9)
        assert sum(c) == w and min(c) >= 0
        c = bas.split_node(bas.child_key(0, 3, 1), w, pr, 0, 1, 1, 9)
        assert c == [w, 0, 0, 0]            # orbital 0 must stay empty: outcome 0
    with pytest.raises(ValueError):
        bas.split_node(0, 5, [1.0, 0.0, 0.0, 0.0], 0, 1, 1, 1)   # only infeasible outcomes


def _product_conditional(table):
    def cond(nodes, orbital):
        return [table[orbital] for _ in nodes]
    return cond


def _exact_distribution(table, n, n_up, n_dn):
    """pi(x) = prod_i pi~(x_i | x_>i) over every sector configuration, by enumeration."""
    out = {}

    def rec(key, orbital, p):
        if orbital < 0:
            out[key] = p
            return
        na = bin(key & int("01" * 64, 2)).count("1")
        nb = bin(key & int("10" * 64, 2)).count("1")
        ok = bas.feasible(na, nb, orbital, n_up, n_dn)
        q = [table[orbital][o] if ok[o] else 0.0 for o in range(4)]
        s = sum(q)
        for o in range(4):
            if q[o] > 0:
                rec(bas.child_key(key, o, orbital), orbital - 1, p * q[o] / s)
    rec(0, n - 1, 1.0)
    return out


def test_bas_reproduces_the_autoregressive_distribution():
    """N=6 qubits (3 orbitals), (n_up, n_dn) = (1, 2): N_s = 10^6 samples; the
    frequencies are within 0.005 total variation of the enumerated pi (SPEC's check)."""
    rng = np.random.default_rng(4)
    table = {i: list(rng.random(4) + 0.05) for i in range(3)}
    ns = 10**6
    got = bas.sample(_product_conditional(table), 3, 1, 2, ns, seed=21)
    exact = _exact_distribution(table, 3, 1, 2)
    assert sum(c for _, c in got) == ns
    keys = [k for k, _ in got]
    assert keys == sorted(keys) and set(keys) <= set(exact)
    freq = {k: c / ns for k, c in got}
    tv = 0.5 * sum(abs(freq.get(k, 0.0) - p) for k, p in exact.items())
    assert tv < 0.005


def test_parallel_bas_equals_serial():
    """replay until the layer is wider than the threshold, split it into
    contiguous parts of about equal weight, finish each part: the union is the serial
    sample set (per-node seeding)."""
    rng = np.random.default_rng(8)
    n = 6
    table = {i: list(rng.random(4) + 0.01) for i in range(n)}
    serial = bas.sample(_product_conditional(table), n, 3, 3, 10**9, seed=5)
    for parts in (2, 3, 4):
        union = []
        for r in range(parts):
            union += bas.sample(_product_conditional(table), n, 3, 3, 10**9, seed=5, split=(4, parts, r))
        assert union == serial


def test_product_partition_matches_oracle():
    from paper_2306_16705_b200.sampler import partition
    rng = np.random.default_rng(1)
    for _ in range(200):
        w = rng.integers(0, 50, size=int(rng.integers(1, 40)))
        P = int(rng.integers(1, 6))
        assert partition(w, P) == bas.partition(list(w), P)


def test_ansatz_normalised_over_sector():
    """|psi|^2 = prod of masked conditionals sums to 1 over the sector (Eq. 8, 12)."""
    import torch
    from paper_2306_16705_b200.ansatz import QiankunNet
    from synth import samples as S
    for n, nu, nd in ((2, 1, 1), (6, 2, 2), (5, 3, 1)):
        m = QiankunNet(n, nu, nd, seed=n)
        keys = torch.from_numpy(S.sector_keys(n, nu, nd).view(np.int64))
        lp = m.log_psi(keys)
        assert abs(float(torch.exp(2 * lp[:, 0]).sum()) - 1.0) < 1e-12
