"""Parity of the CUDA path (through the C-ABI) with the CPU oracle.

Tolerances (reading R14): per row |dE| <= 1e-10 * sum_x' |H_xx'| |psi(x')/psi(x)|
(the oracle's scale output); bit-exact on flip masks, lookup indices and signs.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import dense, energy  # noqa: E402
from oracle import rows as R  # noqa: E402
from synth import configs as C  # noqa: E402
from synth import samples as S  # noqa: E402

TOL = 1e-10


@pytest.fixture(scope="module")
def nnqs():
    import __graft_entry__ as g
    g.build()
    from paper_2306_16705_b200 import nnqs as m
    assert torch.cuda.is_available()
    return m


@pytest.fixture(scope="module")
def dev():
    return torch.device("cuda", 0)


def _t(a, dev):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint64:
        a = a.view(np.int64)
    return torch.from_numpy(a).to(dev)


def _c(el):
    el = el.cpu().numpy()
    return el[:, 0] + 1j * el[:, 1]


def _assert_close(got, ref, scale, what):
    bad = ~(np.abs(got - ref) <= TOL * scale)
    assert not bad.any(), f"{what}: {bad.sum()} rows off, worst {np.max(np.abs(got - ref) / scale)}"


_HAMS = {}


def ham_for(nnqs, c):
    if c not in _HAMS:
        m = C.molecule(c)
        _HAMS[c] = nnqs.nnqs_ham_compress(m.h1, m.h2, m.n_qubits, m.e_core, device=0)
    return _HAMS[c]


# ------------------------------------------------------------------- compress
@pytest.mark.parametrize("c", [1, 2, 3, 4])
def test_device_ham_export_matches_host(nnqs, c):
    m = C.molecule(c)
    a = nnqs.nnqs_ham_compress(m.h1, m.h2, m.n_qubits, m.e_core, device=-1).export()
    b = ham_for(nnqs, c).export()
    for u, v in zip(a, b):
        assert np.array_equal(u, v)
    assert ham_for(nnqs, c).info()["device_bytes"] > 0


# ----------------------------------------------------------------- exact mode
@pytest.mark.parametrize("c", [1, 2])
def test_exact_mode_random_psi(nnqs, dev, c):
    """C1: all 16 configurations; C2: all 4096 (exact mode, random complex psi)."""
    m = C.molecule(c)
    lp = C.exact_random_psi(c)
    ham = ham_for(nnqs, c)
    tab = nnqs.nnqs_table_prepare(ham, 1, None, _t(lp, dev))
    n = len(lp)
    got = _c(nnqs.nnqs_local_energy(ham, tab, 0, n_rows=n))
    rows = np.stack([np.arange(n, dtype=np.uint64), np.zeros(n, dtype=np.uint64)], axis=1)
    ref, scale = R.eloc(m.h1, m.h2, m.e_core, rows, lp, keys=None, logpsi=lp, with_scale=True)
    _assert_close(got, ref, scale, f"C{c} exact")


def test_exact_mode_fci_vector(nnqs, dev):
    """C1 with the FCI vector (sector eigh): E_loc == E_0 on the 2 supported rows,
    NaN (+ NNQS_E_ZERO_PSI) on the 14 rows with psi = 0 (reading R10, R17)."""
    m = C.molecule(1)
    keys = S.sector_keys(2, 1, 1)
    e0, psi, _ = dense.ground_state(m.h1, m.h2, m.e_core, keys)
    full = np.full((16, 2), [-np.inf, 0.0])
    for k, a in zip(keys[:, 0], psi):
        if abs(a) > 1e-12 * np.abs(psi).max():
            full[int(k)] = [np.log(abs(a)), np.pi if a < 0 else 0.0]
    ham = ham_for(nnqs, 1)
    tab = nnqs.nnqs_table_prepare(ham, 1, None, _t(full, dev))
    el = nnqs.nnqs_local_energy(ham, tab, 0, n_rows=16)
    got = _c(el)
    sup = np.isfinite(full[:, 0])
    assert sup.sum() == 2
    assert np.all(np.abs(got[sup] - e0) <= TOL * abs(e0))
    assert np.all(np.isnan(got[~sup].real))
    with pytest.raises(nnqs.NNQSError) as e:
        nnqs.nnqs_local_energy_check(el)
    assert e.value.code == nnqs.NNQS_E_ZERO_PSI


# --------------------------------------------------------- sample-aware mode
def _sample_case(nnqs, dev, c, variant, row_idx=None):
    m = C.molecule(c)
    st = C.sample_table(c, variant)
    ham = ham_for(nnqs, c)
    tab = nnqs.nnqs_table_prepare(ham, 0, _t(st.keys, dev), _t(st.logpsi, dev))
    if row_idx is None:
        got = _c(nnqs.nnqs_local_energy(ham, tab, 0, n_rows=len(st.keys)))
        rows, rlp = st.keys, st.logpsi
    else:
        rows, rlp = st.keys[row_idx], st.logpsi[row_idx]
        got = _c(nnqs.nnqs_local_energy(ham, tab, rows=_t(rows, dev), row_logpsi=_t(rlp, dev)))
    ref, scale = R.eloc(m.h1, m.h2, m.e_core, rows, rlp, keys=st.keys, logpsi=st.logpsi, with_scale=True)
    return got, ref, scale


@pytest.mark.parametrize("c,variant", [(2, "full"), (2, "half"), (3, "full"), (3, "half"), (4, "full")])
def test_sample_mode_table_rows(nnqs, dev, c, variant):
    """Every table entry as a row (the paper's ist/l slice)."""
    got, ref, scale = _sample_case(nnqs, dev, c, variant)
    _assert_close(got, ref, scale, f"C{c}/{variant}")


@pytest.mark.parametrize("c", [2, 3, 4])
def test_sample_mode_drawn_rows(nnqs, dev, c):
    """Rows drawn with replacement (reading R19): C2 10^4, C3/C4 a seeded
    10^4-row subset of the 10^5 draws (oracle cost), as explicit rows."""
    st = C.sample_table(c, "full")
    draws = C.row_draws(c, len(st.keys))[:10_000]
    got, ref, scale = _sample_case(nnqs, dev, c, "full", draws)
    _assert_close(got, ref, scale, f"C{c} drawn")


def test_sample_mode_equals_exact_full_sector(nnqs, dev):
    """Sample-aware with T = full sector == exact mode with psi = 0 off-sector."""
    m = C.molecule(2)
    st = C.sample_table(2, "full")
    ham = ham_for(nnqs, 2)
    full = np.full((4096, 2), [-np.inf, 0.0])
    full[st.keys[:, 0].astype(np.int64)] = st.logpsi
    ta = nnqs.nnqs_table_prepare(ham, 0, _t(st.keys, dev), _t(st.logpsi, dev))
    tb = nnqs.nnqs_table_prepare(ham, 1, None, _t(full, dev))
    a = _c(nnqs.nnqs_local_energy(ham, ta, 0, n_rows=len(st.keys)))
    b = _c(nnqs.nnqs_local_energy(ham, tb, rows=_t(st.keys, dev), row_logpsi=_t(st.logpsi, dev)))
    assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(a))


# ------------------------------------------------------------ C5: 120 qubits
@pytest.fixture(scope="module")
def c5(nnqs, dev):
    m = C.molecule(5)
    st = C.sample_table(5)
    ham = ham_for(nnqs, 5)
    tab = nnqs.nnqs_table_prepare(ham, 0, _t(st.keys, dev), _t(st.logpsi, dev))
    return m, st, ham, tab


def test_c5_sampled_rows(nnqs, dev, c5):
    """120 spin orbitals, 10^6 unique near-HF samples: a seeded row subset plus
    the HF row (most hits), evaluated as explicit rows."""
    m, st, ham, tab = c5
    idx = C.oracle_row_subset(5, len(st.keys), 16)
    hf = np.argmax(st.counts)
    idx = np.unique(np.concatenate([idx, [hf]]))
    rows, rlp = st.keys[idx], st.logpsi[idx]
    got = _c(nnqs.nnqs_local_energy(ham, tab, rows=_t(rows, dev), row_logpsi=_t(rlp, dev)))
    ref, scale = R.eloc(m.h1, m.h2, m.e_core, rows, rlp, keys=st.keys, logpsi=st.logpsi, with_scale=True)
    _assert_close(got, ref, scale, "C5 rows")


def test_c5_full_launch_sampled(nnqs, dev, c5):
    """The bench launch: every one of the 10^6 table rows in one call; 1024 seeded
    rows + the HF row + the 10 longest-list rows checked against the oracle."""
    m, st, ham, tab = c5
    n = len(st.keys)
    stats = torch.zeros(4, dtype=torch.int64, device=dev)
    el = nnqs.nnqs_local_energy(ham, tab, 0, n_rows=n, stats_out=stats)
    nnqs.nnqs_local_energy_check(el)
    hf, top, _ = _c5_special_rows(st)
    idx = np.unique(np.concatenate([C.oracle_row_subset(5, n, 1024), [hf], top]))
    got = _c(el)[idx]
    ref, scale = R.eloc(m.h1, m.h2, m.e_core, st.keys[idx], st.logpsi[idx], keys=st.keys, logpsi=st.logpsi,
                        with_scale=True)
    _assert_close(got, ref, scale, "C5 full launch")
    s = stats.cpu().numpy()
    assert s[0] == n * ham.info()["n_groups"] and s[2] > n


def test_c5_bitwise_determinism_and_slices(nnqs, dev, c5):
    """C5 at full size: the same bits on a re-run and when the rows are split
    into uneven slices (the rank slices of a multi-GPU run) -- covers the
    entry-driven join of the heavy alpha group, the multimap probes and the
    dynamic row schedule (a row's summation order depends on the row alone)."""
    m, st, ham, tab = c5
    n = len(st.keys)
    a = nnqs.nnqs_local_energy(ham, tab, 0, n_rows=n).cpu().numpy()
    b = nnqs.nnqs_local_energy(ham, tab, 0, n_rows=n).cpu().numpy()
    cuts = [0, 123457, 500001, 777777, n]
    d = np.concatenate([nnqs.nnqs_local_energy(ham, tab, s0, n_rows=s1 - s0).cpu().numpy()
                        for s0, s1 in zip(cuts[:-1], cuts[1:])])
    assert a.tobytes() == b.tobytes()
    assert a.tobytes() == d.tobytes()
    # work-balanced rank slices (nnqs_chunk_work + balanced_bounds), 8 ranks
    from paper_2306_16705_b200 import distributed as D
    w = nnqs.nnqs_chunk_work(tab)
    assert w.shape == ((n + 1023) // 1024,) and (w > 0).all()
    assert np.array_equal(w, nnqs.nnqs_chunk_work(tab))
    bs = [D.balanced_bounds(w, 8, r, n_rows=n) for r in range(8)]
    assert bs[0][0] == 0 and bs[-1][1] == n and all(x[1] == y[0] for x, y in zip(bs[:-1], bs[1:]))
    f = np.concatenate([nnqs.nnqs_local_energy(ham, tab, s0, n_rows=s1 - s0).cpu().numpy() for s0, s1 in bs])
    assert a.tobytes() == f.tobytes()


def test_c5_structured_equals_literal_hits(nnqs, dev, c5):
    """On a 4096-row slice of C5: identical hit counts for the two enumerations
    (the same (row, group) pairs are found), E_loc within tolerance of each
    other.  The structured path evaluates the in-sector folded strings (DESIGN.md
    R21), so it evaluates fewer strings than the literal loop."""
    m, st, ham, tab = c5
    s1 = torch.zeros(4, dtype=torch.int64, device=dev)
    s2 = torch.zeros(4, dtype=torch.int64, device=dev)
    a = _c(nnqs.nnqs_local_energy(ham, tab, 500_000, n_rows=4096, stats_out=s1))
    nnqs.nnqs_table_set_algorithm(tab, nnqs.ALGO_LITERAL)
    try:
        b = _c(nnqs.nnqs_local_energy(ham, tab, 500_000, n_rows=4096, stats_out=s2))
    finally:
        nnqs.nnqs_table_set_algorithm(tab, nnqs.ALGO_AUTO)
    s1, s2 = s1.cpu().numpy(), s2.cpu().numpy()
    assert s1[2] == s2[2] and s1[3] < s2[3]
    assert np.max(np.abs(a - b) / np.maximum(np.abs(b), 1.0)) < 1e-9


# ---------------------------------------------- P3: coupled configurations
@pytest.mark.parametrize("c,variant", [(2, "half"), (3, "full"), (4, "full")])
def test_coupled_configurations_bit_exact(nnqs, dev, c, variant):
    """Per row, the set of (x', table index) with |H_xx'| > tau equals the
    oracle's, bit for bit; signs agree; GPU extras have |H| <= tau."""
    m = C.molecule(c)
    st = C.sample_table(c, variant)
    ham = ham_for(nnqs, c)
    tab = nnqs.nnqs_table_prepare(ham, 0, _t(st.keys, dev), _t(st.logpsi, dev))
    sel = C.oracle_row_subset(c, len(st.keys), 24)
    rid, gid, xp, tix, hv = nnqs.nnqs_coupled_debug(ham, tab, st.keys[sel])
    tau = 1e-13 * max(np.abs(m.h1).max(), np.abs(m.h2).max())
    x_all, _, _, _ = ham.export()
    for j, i in enumerate(sel):
        ridx, rh = R.row_hits(m.h1, m.h2, m.e_core, st.keys[i], keys=st.keys)
        want = {int(a): b for a, b in zip(ridx, rh) if abs(b) > tau}
        mine = rid == j
        got = {int(a): b for a, b in zip(tix[mine], hv[mine])}
        for k, g in zip(tix[mine], gid[mine]):      # x' = x ^ X_k and it is the table key
            assert np.array_equal(st.keys[k], st.keys[i] ^ x_all[g])
        assert set(k for k, v in got.items() if abs(v) > tau) == set(want)
        for k, v in want.items():
            assert np.sign(got[k]) == np.sign(v)
            assert abs(got[k] - v) <= 1e-12 * max(1.0, abs(v))


# ------------------------------- P3 on the production (structured) path
def _oracle_hits(m, keys, rows_idx, workers=16):
    """oracle row_hits (plain term-by-term Eq. 9 + bisection) of many rows, threaded
    (the ctypes call releases the GIL)."""
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(workers) as ex:
        return list(ex.map(lambda i: R.row_hits(m.h1, m.h2, m.e_core, keys[i], keys=keys), rows_idx))


def _p3_compare(m, keys, i, rid, gid, xp, tix, hv, ref):
    """Bit-exact P3 for one row: the set of x' (table indices) with |H| > tau equals the
    oracle's, every logged x' is x ^ X_k for a group k of the table and is logged once,
    signs agree, values agree to rounding; extras have |H| <= tau (structural zeros)."""
    tau = 1e-13 * max(np.abs(m.h1).max(), np.abs(m.h2).max())
    ridx, rh = ref
    assert (rid == i).all()
    assert len(np.unique(tix)) == len(tix), f"row {i}: an x' evaluated twice"
    assert (gid >= 0).all(), f"row {i}: x ^ x' is not a flip group of the table"
    assert np.array_equal(xp, keys[tix])
    want = {int(a): b for a, b in zip(ridx, rh) if abs(b) > tau}
    got = dict(zip(tix.tolist(), hv.tolist()))
    assert set(k for k, v in got.items() if abs(v) > tau) == set(want), f"row {i}: hit sets differ"
    for k, v in want.items():
        assert np.sign(got[k]) == np.sign(v), f"row {i}, x' {k}: sign"
        assert abs(got[k] - v) <= 1e-12 * max(1.0, abs(v)), f"row {i}, x' {k}: {got[k]} vs {v}"


def _p3_check(nnqs, ham, tab, m, keys, rows_idx, per_row=False):
    rows_idx = np.asarray(rows_idx)
    refs = _oracle_hits(m, keys, rows_idx)
    if per_row:        # one production call per row (large rows: the C5 HF row has ~44k hits)
        for i, ref in zip(rows_idx, refs):
            rid, gid, xp, tix, hv = nnqs.nnqs_coupled_debug_rows(ham, tab, int(i), 1, max_pairs=1 << 18)
            _p3_compare(m, keys, int(i), rid, gid, xp, tix, hv, ref)
        return
    # one production call over the whole row range, hits grouped by row
    lo, hi = int(rows_idx.min()), int(rows_idx.max()) + 1
    rid, gid, xp, tix, hv = nnqs.nnqs_coupled_debug_rows(ham, tab, lo, hi - lo, max_pairs=1 << 23)
    order = np.argsort(rid, kind="stable")
    rid, gid, xp, tix, hv = rid[order], gid[order], xp[order], tix[order], hv[order]
    starts = np.searchsorted(rid, rows_idx, "left")
    ends = np.searchsorted(rid, rows_idx, "right")
    for i, a, b, ref in zip(rows_idx, starts, ends, refs):
        _p3_compare(m, keys, int(i), rid[a:b], gid[a:b], xp[a:b], tix[a:b], hv[a:b], ref)


@pytest.mark.parametrize("c,variant", [(2, "full"), (2, "half"), (3, "full"), (3, "half"), (4, "full")])
def test_production_coupled_configurations_bit_exact(nnqs, dev, c, variant):
    """P3 on the path nnqs_local_energy runs for table rows (the structured kernels):
    every row of the table, its (x', lookup index) set and signs bit-exact against the
    oracle (Algorithm 2's hit/sign steps)."""
    m = C.molecule(c)
    st = C.sample_table(c, variant)
    ham = ham_for(nnqs, c)
    tab = nnqs.nnqs_table_prepare(ham, 0, _t(st.keys, dev), _t(st.logpsi, dev))
    _p3_check(nnqs, ham, tab, m, st.keys, np.arange(len(st.keys)))


def _c5_special_rows(st):
    """The HF row (largest count) and the 10 rows with the longest alpha + beta lists
    (the rows with the most hits), plus 100 seeded rows (SURVEY.md 8(c) reading 20)."""
    from synth import samples as SS  # noqa: F401
    k = st.keys

    def spin(w, s):
        w = (w >> np.uint64(s)) & np.uint64(0x5555555555555555)
        for sh, mk in [(1, 0x3333333333333333), (2, 0x0F0F0F0F0F0F0F0F), (4, 0x00FF00FF00FF00FF),
                       (8, 0x0000FFFF0000FFFF), (16, 0x00000000FFFFFFFF)]:
            w = (w | (w >> np.uint64(sh))) & np.uint64(mk)
        return w
    a = spin(k[:, 0], 0) | (spin(k[:, 1], 0) << np.uint64(32))
    b = spin(k[:, 0], 1) | (spin(k[:, 1], 1) << np.uint64(32))
    _, ia, ca = np.unique(a, return_inverse=True, return_counts=True)
    _, ib, cb = np.unique(b, return_inverse=True, return_counts=True)
    size = ca[ia] + cb[ib]
    hf = int(np.argmax(st.counts))
    top = [int(i) for i in np.argsort(-size, kind="stable") if i != hf][:10]
    seeded = C.oracle_row_subset(5, len(k), 100)
    return hf, top, seeded


def test_c5_production_coupled_configurations_bit_exact(nnqs, dev, c5):
    """P3 at the headline config on the production path: the HF row (~44k hits, the
    entry-driven join + multimap probes), the 10 rows with the longest lists and 100
    seeded rows -- x' sets, lookup indices and signs bit-exact against the oracle."""
    m, st, ham, tab = c5
    hf, top, seeded = _c5_special_rows(st)
    _p3_check(nnqs, ham, tab, m, st.keys, [hf] + top, per_row=True)
    _p3_check(nnqs, ham, tab, m, st.keys, seeded, per_row=True)


def test_structured_zero_psi_rows(nnqs, dev):
    """psi(x) = 0 (log psi = -inf) on the structured path (reading R10): those rows are
    NaN (NNQS_E_ZERO_PSI from the check), and as x' of other rows they contribute 0;
    every other row matches the oracle."""
    for c in (3, 4):
        m = C.molecule(c)
        st = C.sample_table(c, "full")
        lp = st.logpsi.copy()
        rng = np.random.default_rng(77 + c)
        zero = np.sort(rng.choice(len(lp), size=max(3, len(lp) // 50), replace=False))
        lp[zero, 0] = -np.inf
        ham = ham_for(nnqs, c)
        tab = nnqs.nnqs_table_prepare(ham, 0, _t(st.keys, dev), _t(lp, dev))
        el = nnqs.nnqs_local_energy(ham, tab, 0, n_rows=len(lp))
        with pytest.raises(nnqs.NNQSError) as e:
            nnqs.nnqs_local_energy_check(el)
        assert e.value.code == nnqs.NNQS_E_ZERO_PSI
        got = _c(el)
        assert np.isnan(got[zero]).all()
        ok = np.setdiff1d(np.arange(len(lp)), zero)
        ref, scale = R.eloc(m.h1, m.h2, m.e_core, st.keys[ok], lp[ok], keys=st.keys, logpsi=lp, with_scale=True)
        _assert_close(got[ok], ref, scale, f"C{c} zero-psi")


@pytest.mark.parametrize("c", [3, 4])
def test_fused_chunk_partials(nnqs, dev, c):
    """nnqs_local_energy(counts, partials_out): the fused first pass of Eq. (6) equals
    nnqs_energy_chunk_partials bit for bit, on both algorithms and on a chunk-aligned
    slice; the partials of the slices combine to the single-call energy bit for bit."""
    st = C.sample_table(c, "full")
    ham = ham_for(nnqs, c)
    n = len(st.keys)
    cnt = _t(st.counts, dev)
    for algo in (nnqs.ALGO_AUTO, nnqs.ALGO_LITERAL):
        tab = nnqs.nnqs_table_prepare(ham, 0, _t(st.keys, dev), _t(st.logpsi, dev), algorithm=algo)
        nch = (n + 1023) // 1024
        part = torch.full((nch, 3), np.nan, dtype=torch.float64, device=dev)
        el = nnqs.nnqs_local_energy(ham, tab, 0, n_rows=n, counts=cnt, partials_out=part)
        ref = nnqs.nnqs_energy_chunk_partials(el, cnt)
        assert part.cpu().numpy().tobytes() == ref.cpu().numpy().tobytes()
        if n > 2048:
            cut = 1024 * (nch // 2)
            p1 = torch.empty(((cut + 1023) // 1024, 3), dtype=torch.float64, device=dev)
            p2 = torch.empty(((n - cut + 1023) // 1024, 3), dtype=torch.float64, device=dev)
            nnqs.nnqs_local_energy(ham, tab, 0, n_rows=cut, counts=cnt[:cut], partials_out=p1)
            nnqs.nnqs_local_energy(ham, tab, cut, n_rows=n - cut, counts=cnt[cut:], partials_out=p2)
            a = nnqs.nnqs_energy_combine(torch.cat([p1, p2]), 1).cpu().numpy()
            b = nnqs.nnqs_energy_combine(ref, 1).cpu().numpy()
            assert a.tobytes() == b.tobytes()


def test_c5_fixture_every_row(nnqs, dev, c5):
    """Every-row parity at the headline config (SURVEY.md 8(c) reading 20): all 10^6
    E_loc against the committed oracle fixture (scripts/c5_oracle_fixture.py, oracle/
    only), and Eq. (6) mean / variance against the oracle's (R14 tolerances)."""
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "c5_eloc.npz")
    if not os.path.exists(path):
        pytest.skip("C5 oracle fixture not generated (scripts/c5_oracle_fixture.py)")
    m, st, ham, tab = c5
    z = np.load(path)
    import hashlib
    h = hashlib.sha256()
    for a in (st.keys, st.counts, st.logpsi):
        h.update(np.ascontiguousarray(a).tobytes())
    assert str(z["digest"]) == h.hexdigest(), "fixture computed from other C5 inputs"
    n = len(st.keys)
    cnt = _t(st.counts, dev)
    part = torch.empty(((n + 1023) // 1024, 3), dtype=torch.float64, device=dev)
    el = nnqs.nnqs_local_energy(ham, tab, 0, n_rows=n, counts=cnt, partials_out=part)
    got = _c(el)
    have = z["have"]
    assert have.sum() > 0
    ref = z["re"][have] + 1j * z["im"][have]
    _assert_close(got[have], ref, z["scale"][have], f"C5 fixture ({int(have.sum())} rows)")
    if bool(z["complete"]):
        m1 = nnqs.nnqs_energy_combine(part, 1)
        m2 = nnqs.nnqs_energy_combine(nnqs.nnqs_energy_chunk_partials(el, cnt, mean_dev=m1[:2].contiguous()), 2)
        m1, m2 = m1.cpu().numpy(), m2.cpu().numpy()
        TOLE = TOL * float(z["energy_scale"])
        assert abs(m1[0] - float(z["mean_re"])) <= TOLE and abs(m1[1] - float(z["mean_im"])) <= TOLE
        var = float(z["var"])
        assert abs(m2[0] - var) <= TOL * var + 2 * TOL * np.sqrt(var) * float(z["max_abs"])
        assert m1[2] == float(z["W"])
    # the literal Algorithm 2 loop (bit-sliced kernel) over every row too
    lit = nnqs.nnqs_table_prepare(ham, 0, _t(st.keys, dev), _t(st.logpsi, dev), algorithm=nnqs.ALGO_LITERAL)
    got_l = _c(nnqs.nnqs_local_energy(ham, lit, 0, n_rows=n))
    lit.close()
    _assert_close(got_l[have], ref, z["scale"][have], f"C5 fixture, literal loop ({int(have.sum())} rows)")


# ---------------------------------------------------- Pauli-level semantics
def _pauli(nnqs, terms, nq):
    X = [[x, 0] for x, _, _ in terms]
    Z = [[z, 0] for _, z, _ in terms]
    return nnqs.nnqs_ham_from_pauli(X, Z, [c for _, _, c in terms], nq, device=0)


def test_spec_pauli_examples(nnqs, dev):
    """SPEC.md:60-62, 253, 260 (Y = i X Z; <x'|P|x> with Z|b> = (-1)^b|b>)."""
    c = 0.37
    zero = np.zeros((1, 2))
    # c Z0 on bit0 = 1 -> -c (T = {x})
    h = _pauli(nnqs, [(0, 1, c)], 2)
    k = np.array([[1, 0]], dtype=np.uint64)
    t = nnqs.nnqs_table_prepare(h, 0, _t(k, dev), _t(zero, dev))
    assert _c(nnqs.nnqs_local_energy(h, t, 0, n_rows=1))[0] == -c
    # c Y0Y1 on |00> -> c * <11|Y0Y1|00> = -c ; uniform psi, exact mode
    h = _pauli(nnqs, [(3, 3, c)], 2)
    t = nnqs.nnqs_table_prepare(h, 1, None, _t(np.zeros((4, 2)), dev))
    assert _c(nnqs.nnqs_local_energy(h, t, 0, n_rows=1))[0] == -c
    # {c1 Z0, c2 Z1} on bit0 = 1, bit1 = 0 -> -c1 + c2
    h = _pauli(nnqs, [(0, 1, 0.3), (0, 2, -0.45)], 2)
    t = nnqs.nnqs_table_prepare(h, 0, _t(k, dev), _t(zero, dev))
    assert _c(nnqs.nnqs_local_energy(h, t, 0, n_rows=1))[0] == -0.3 + -0.45
    # T = {x}, c X0 -> 0 (absent x' contributes 0)
    h = _pauli(nnqs, [(1, 0, c)], 2)
    t = nnqs.nnqs_table_prepare(h, 0, _t(k, dev), _t(zero, dev))
    assert _c(nnqs.nnqs_local_energy(h, t, 0, n_rows=1))[0] == 0.0
    # c X0X1 with uniform psi -> c
    h = _pauli(nnqs, [(3, 0, c)], 2)
    t = nnqs.nnqs_table_prepare(h, 1, None, _t(np.zeros((4, 2)), dev))
    assert np.all(_c(nnqs.nnqs_local_energy(h, t, 0, n_rows=4)) == c)


# ------------------------------------------------------------------ reduce
def test_reduce_matches_oracle(nnqs, dev):
    rng = np.random.default_rng(5)
    n = 70_001
    e = rng.normal(-3.0, 0.4, size=n) + 1j * rng.normal(0, 0.01, size=n)
    w = rng.integers(1, 100, size=n)
    el = _t(np.stack([e.real, e.imag], axis=1), dev)
    m, v, W = nnqs.nnqs_energy_reduce(el, _t(w.astype(np.int64), dev))
    mr, vr, Wr = energy.energy(e, w)
    assert W == Wr
    assert abs(m - mr) <= TOL * np.sum(w * np.abs(e)) / Wr
    assert abs(v - vr) <= TOL * vr + 2 * TOL * np.sqrt(vr) * np.abs(e).max()


def test_reduce_spec_examples(nnqs, dev):
    el = _t(np.array([[0.0, 0.0], [4.0, 0.0]]), dev)
    m, v, W = nnqs.nnqs_energy_reduce(el, _t(np.array([3, 1], dtype=np.int64), dev))
    assert (m, v, W) == (1.0, 3.0, 4.0)
    with pytest.raises(nnqs.NNQSError) as e:
        nnqs.nnqs_energy_reduce(el, _t(np.array([0, 0], dtype=np.int64), dev))
    assert e.value.code == nnqs.NNQS_E_EMPTY


# ---------------------------------------------- determinism and sharding
def test_bitwise_determinism_and_slices(nnqs, dev):
    """Same bits on a re-run and for any row slicing (a row's summation order
    depends on the row alone) -- structured path (table rows) and literal
    path (explicit rows) separately."""
    st = C.sample_table(4, "full")
    ham = ham_for(nnqs, 4)
    tab = nnqs.nnqs_table_prepare(ham, 0, _t(st.keys, dev), _t(st.logpsi, dev))
    n = len(st.keys)
    a = nnqs.nnqs_local_energy(ham, tab, 0, n_rows=n).cpu().numpy()
    b = nnqs.nnqs_local_energy(ham, tab, 0, n_rows=n).cpu().numpy()
    parts = [nnqs.nnqs_local_energy(ham, tab, s, n_rows=min(3001, n - s)).cpu().numpy() for s in range(0, n, 3001)]
    d = np.concatenate(parts)
    assert a.tobytes() == b.tobytes() == d.tobytes()
    c1 = nnqs.nnqs_local_energy(ham, tab, rows=_t(st.keys, dev), row_logpsi=_t(st.logpsi, dev)).cpu().numpy()
    c2 = nnqs.nnqs_local_energy(ham, tab, rows=_t(st.keys[::-1].copy(), dev),
                                row_logpsi=_t(st.logpsi[::-1].copy(), dev)).cpu().numpy()[::-1]
    assert c1.tobytes() == np.ascontiguousarray(c2).tobytes()


@pytest.mark.parametrize("c,variant", [(2, "half"), (3, "full"), (4, "full")])
def test_structured_equals_literal(nnqs, dev, c, variant):
    """The alpha/beta-factorised enumeration finds exactly the literal loop's
    hits (equal hit counts) and the same E_loc (within the parity tolerance)."""
    m = C.molecule(c)
    st = C.sample_table(c, variant)
    ham = ham_for(nnqs, c)
    tab = nnqs.nnqs_table_prepare(ham, 0, _t(st.keys, dev), _t(st.logpsi, dev))
    n = len(st.keys)
    s1 = torch.zeros(4, dtype=torch.int64, device=dev)
    s2 = torch.zeros(4, dtype=torch.int64, device=dev)
    a = _c(nnqs.nnqs_local_energy(ham, tab, 0, n_rows=n, stats_out=s1))
    lit = nnqs.nnqs_table_prepare(ham, 0, _t(st.keys, dev), _t(st.logpsi, dev), algorithm=nnqs.ALGO_LITERAL)
    b = _c(nnqs.nnqs_local_energy(ham, lit, 0, n_rows=n, stats_out=s2))
    s1, s2 = s1.cpu().numpy(), s2.cpu().numpy()
    assert s1[0] == s2[0] == n * ham.info()["n_groups"]
    assert s1[2] == s2[2]                       # identical hit sets (counts)
    assert s1[3] <= s2[3]                       # in-sector folded strings (R21): never more
    ref, scale = R.eloc(m.h1, m.h2, m.e_core, st.keys, st.logpsi, keys=st.keys, logpsi=st.logpsi, with_scale=True)
    _assert_close(a, ref, scale, "structured")
    _assert_close(b, ref, scale, "literal")


def test_chunked_energy_is_partition_invariant(nnqs, dev):
    """Chunk partials of chunk-aligned slices, combined in order, are bit-identical
    to the single-call reduce (the multi-GPU energy path, Sec. 3.2 stage 4)."""
    rng = np.random.default_rng(9)
    n = 10 * 1024 + 77
    e = np.stack([rng.normal(-2, 1, n), rng.normal(0, 0.1, n)], axis=1)
    w = rng.integers(1, 9, size=n).astype(np.int64)
    el, wc = _t(e, dev), _t(w, dev)
    ref = nnqs.nnqs_energy_reduce(el, wc)
    for P in (2, 3, 4):
        bounds = np.linspace(0, n // 1024, P + 1).astype(int) * 1024
        bounds[-1] = n
        parts = [nnqs.nnqs_energy_chunk_partials(el[a:b], wc[a:b]) for a, b in zip(bounds[:-1], bounds[1:])]
        allp = torch.cat(parts)
        m1 = nnqs.nnqs_energy_combine(allp, 1)
        parts2 = [nnqs.nnqs_energy_chunk_partials(el[a:b], wc[a:b], mean_dev=m1[:2].contiguous())
                  for a, b in zip(bounds[:-1], bounds[1:])]
        m2 = nnqs.nnqs_energy_combine(torch.cat(parts2), 2).cpu().numpy()
        m1 = m1.cpu().numpy()
        assert complex(m1[0], m1[1]) == ref[0] and m2[0] == ref[1] and m1[2] == ref[2]


# ------------------------------------------------------------ edge cases
def test_errors_and_edges(nnqs, dev):
    ham = ham_for(nnqs, 2)
    st = C.sample_table(2, "full")
    bad = st.keys[::-1].copy()
    with pytest.raises(nnqs.NNQSError) as e:
        nnqs.nnqs_table_prepare(ham, 0, _t(bad, dev), _t(st.logpsi, dev))
    assert e.value.code == nnqs.NNQS_E_TABLE
    tab = nnqs.nnqs_table_prepare(ham, 0, _t(st.keys, dev), _t(st.logpsi, dev))
    out = nnqs.nnqs_local_energy(ham, tab, 0, n_rows=0)
    assert out.shape[0] == 0
    with pytest.raises(nnqs.NNQSError):
        nnqs.nnqs_local_energy(ham, tab, len(st.keys) - 1, n_rows=2)
    # a single-entry table and an empty table
    one = nnqs.nnqs_table_prepare(ham, 0, _t(st.keys[:1], dev), _t(st.logpsi[:1], dev))
    got = _c(nnqs.nnqs_local_energy(ham, one, 0, n_rows=1))
    m = C.molecule(2)
    ref = R.eloc(m.h1, m.h2, m.e_core, st.keys[:1], st.logpsi[:1], keys=st.keys[:1], logpsi=st.logpsi[:1])
    assert abs(got[0] - ref[0]) <= 1e-12 * abs(ref[0])


def test_chunk_work_and_balanced_slices(nnqs, dev):
    """nnqs_chunk_work: one positive estimate per 1024-row chunk (ragged tail
    included), deterministic, rows-per-chunk on the literal path, NNQS_E_ARG on a
    bad chunk; work-balanced slices of C4 evaluate bit-equal to one launch and
    their chunk partials combine to the single-launch energy bit for bit."""
    from paper_2306_16705_b200 import distributed as D
    ham = ham_for(nnqs, 4)
    st = C.sample_table(4, "full")
    n = len(st.keys)
    tab = nnqs.nnqs_table_prepare(ham, 0, _t(st.keys, dev), _t(st.logpsi, dev))
    w = nnqs.nnqs_chunk_work(tab)
    assert w.shape == ((n + 1023) // 1024,) and (w > 0).all()
    assert np.array_equal(w, nnqs.nnqs_chunk_work(tab))
    w256 = nnqs.nnqs_chunk_work(tab, chunk=256)
    assert w256.shape == ((n + 255) // 256,) and w256.sum() == w.sum()
    with pytest.raises(nnqs.NNQSError) as e:
        nnqs.nnqs_chunk_work(tab, chunk=0)
    assert e.value.code == nnqs.NNQS_E_ARG
    nnqs.nnqs_table_set_algorithm(tab, nnqs.ALGO_LITERAL)
    try:
        lit = nnqs.nnqs_chunk_work(tab)
    finally:
        nnqs.nnqs_table_set_algorithm(tab, nnqs.ALGO_AUTO)
    assert lit.sum() == n and (lit[:-1] == 1024).all()
    cnt = _t(st.counts, dev)
    full = nnqs.nnqs_local_energy(ham, tab, 0, n_rows=n)
    e1 = nnqs.nnqs_energy_combine(nnqs.nnqs_energy_chunk_partials(full, cnt), 1).cpu().numpy()
    for world in (2, 3, 5):
        bs = [D.balanced_bounds(w, world, r, n_rows=n) for r in range(world)]
        parts = [nnqs.nnqs_local_energy(ham, tab, b, n_rows=e - b) for b, e in bs]
        assert torch.cat(parts).cpu().numpy().tobytes() == full.cpu().numpy().tobytes()
        p = torch.cat([nnqs.nnqs_energy_chunk_partials(x, cnt[b:e])[: (e - b + 1023) // 1024]
                       for x, (b, e) in zip(parts, bs)])
        assert nnqs.nnqs_energy_combine(p, 1).cpu().numpy().tobytes() == e1.tobytes()


def test_tiny_amplitude_row_fallback(nnqs, dev):
    """A row with Re log psi(x) - s < -600 takes the per-term exp path (reading R11)."""
    m = C.molecule(3)
    st = C.sample_table(3, "full")
    lp = st.logpsi.copy()
    lp[5, 0] -= 620.0
    lp[6, 0] += 30.0
    ham = ham_for(nnqs, 3)
    tab = nnqs.nnqs_table_prepare(ham, 0, _t(st.keys, dev), _t(lp, dev))
    got = _c(nnqs.nnqs_local_energy(ham, tab, 0, n_rows=len(st.keys)))
    ref, scale = R.eloc(m.h1, m.h2, m.e_core, st.keys, lp, keys=st.keys, logpsi=lp, with_scale=True)
    _assert_close(got, ref, scale, "tiny psi")


def test_grad_weights_matches_oracle(nnqs, dev):
    """Eq. (7) weights on the GPU (nnqs_grad_weights with the device energy of
    nnqs_energy_combine) vs the oracle's, on C4 local energies and counts."""
    st = C.sample_table(4, "full")
    ham = ham_for(nnqs, 4)
    tab = nnqs.nnqs_table_prepare(ham, 0, _t(st.keys, dev), _t(st.logpsi, dev))
    n = len(st.keys)
    el = nnqs.nnqs_local_energy(ham, tab, 0, n_rows=n)
    cnt = _t(st.counts, dev)
    part = nnqs.nnqs_energy_chunk_partials(el, cnt)
    m1 = nnqs.nnqs_energy_combine(part, 1)
    ab = nnqs.nnqs_grad_weights(el, cnt, m1).cpu().numpy()
    a, b = energy.grad_weights(_c(el), st.counts)
    W = float(st.counts.sum())
    tol = 1e-12 * 2 * st.counts * np.abs(_c(el)).max() / W + 1e-300
    assert np.all(np.abs(ab[:, 0] - a) <= tol) and np.all(np.abs(ab[:, 1] - b) <= tol)
    assert abs(ab[:, 0].sum()) <= 1e-9 * np.abs(ab[:, 0]).sum()


@pytest.mark.parametrize("mixed,rowheavy", [(False, 40), (False, 1000), (True, 1000)])
def test_structured_heavy_paths_small(nnqs, dev, mixed, rowheavy):
    """The heavy-group machinery (deletion multimap with its Bloom filter, the
    compact-key or two-sort build, heavy-neighbour probes, the entry-driven join)
    forced onto C4 by low thresholds (per-table nnqs_options):
    rowheavy=40 sends every row's phase (iii) through the join, 1000 through the
    row kernel's probes; mixed=True holds two particle sectors (two-sort build,
    no single-sector shortcut).  Two rows get psi(x) < e^-600 (DIRECT kernels).
    E_loc of sampled rows against the oracle."""
    m = C.molecule(4)
    keys = S.sector_keys(10, 7, 7)
    if mixed:
        keys = np.concatenate([keys, S.sector_keys(10, 6, 7)])
        order = np.lexsort((keys[:, 0], keys[:, 1]))
        keys = np.ascontiguousarray(keys[order])
    rng = np.random.default_rng(31)
    lp = np.stack([rng.normal(0, 1, len(keys)), rng.uniform(-np.pi, np.pi, len(keys))], axis=1)
    lp[[3, 1000], 0] -= 620.0                                  # DIRECT rows (reading R11)
    ham = ham_for(nnqs, 4)
    tab = nnqs.nnqs_table_prepare(ham, 0, _t(keys, dev), _t(lp, dev), thr_single=3, thr_double=6,
                                  thr_rowheavy=rowheavy)
    n = len(keys)
    stats = torch.zeros(4, dtype=torch.int64, device=dev)
    got = _c(nnqs.nnqs_local_energy(ham, tab, 0, n_rows=n, stats_out=stats))
    sel = np.unique(np.concatenate([np.arange(0, n, max(1, n // 600)), [3, 1000, n - 1]]))
    ref, scale = R.eloc(m.h1, m.h2, m.e_core, keys[sel], lp[sel], keys=keys, logpsi=lp, with_scale=True)
    _assert_close(got[sel], ref, scale, f"heavy paths mixed={mixed}")
    s2 = torch.zeros(4, dtype=torch.int64, device=dev)
    lit = nnqs.nnqs_table_prepare(ham, 0, _t(keys, dev), _t(lp, dev), algorithm=nnqs.ALGO_LITERAL)
    nnqs.nnqs_local_energy(ham, lit, 0, n_rows=n, stats_out=s2)
    assert stats.cpu().numpy()[2] == s2.cpu().numpy()[2]     # identical hit counts
    _p3_check(nnqs, ham, tab, m, keys, np.arange(0, n, max(1, n // 40)))   # and identical hit sets
    # degenerate slices through the same machinery: empty, one row, the last row
    assert nnqs.nnqs_local_energy(ham, tab, 7, n_rows=0).shape[0] == 0
    full = nnqs.nnqs_local_energy(ham, tab, 0, n_rows=n).cpu().numpy()
    for r0 in (7, n - 1):
        one = nnqs.nnqs_local_energy(ham, tab, r0, n_rows=1).cpu().numpy()
        assert one.tobytes() == full[r0:r0 + 1].tobytes()


def test_bench_two_ranks_shared_gpu():
    """The N > 1 path of bench.py end to end (torchrun, 2 ranks: stage-2 all-gather,
    rank row slices, stage-4 partials) on the one available GPU with gloo
    (NNQS_BENCH_SHARED_GPU): the energy is bit-identical to the 1-rank run and the
    hit counts sum to the 1-rank counts."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, NNQS_BENCH_SHARED_GPU="1")

    def run(n):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
               "--master-addr", "127.0.0.1", "--master-port", str(29600 + n), "bench.py", "--gpus", str(n),
               "--steps", "1", "--warmup", "3", "--no-cpu-baseline", "--config", "C4"]
        out = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        return json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])

    one, two = run(1), run(2)
    assert one["energy"] == two["energy"]
    assert one["stats"]["hits"] == two["stats"]["hits"]


# ------------------------------------- literal loop: the three kernels agree bit for bit
def _lit_run(nnqs, ham, tab, dev, lk, n=None, rows=None, rlp=None, row_begin=0):
    stats = torch.zeros(4, dtype=torch.int64, device=dev)
    if rows is None:
        el = nnqs.nnqs_local_energy(ham, tab, row_begin, n_rows=n, stats_out=stats)
    else:
        el = nnqs.nnqs_local_energy(ham, tab, rows=_t(rows, dev), row_logpsi=_t(rlp, dev), stats_out=stats)
    return el.cpu().numpy(), stats.cpu().numpy()


@pytest.mark.parametrize("c,variant", [(2, "half"), (3, "full"), (3, "half"), (4, "full")])
def test_literal_kernels_bit_identical(nnqs, dev, c, variant):
    """Algorithm 2's loop in its three kernels -- bit-sliced (32 rows x 32
    groups per sector test + per-spin string filter), group-tile staged, plain -- gives
    the same bits and the same pair / in-sector / hit / string counts, on table rows
    (a psi = 0 row and a row on the exp-ratio path, R10/R11, included), on explicit
    rows that are not in the table, and on a ragged slice; and matches the oracle (R14)."""
    m = C.molecule(c)
    st = C.sample_table(c, variant)
    lp = st.logpsi.copy()
    lp[3, 0] = -np.inf
    lp[5, 0] -= 620.0
    ham = ham_for(nnqs, c)
    full = C.sample_table(c, "full")
    rows, rlp = full.keys, full.logpsi          # for "half": rows outside the table too
    outs = []
    for lk in (0, 1, 2):
        tab = nnqs.nnqs_table_prepare(ham, 0, _t(st.keys, dev), _t(lp, dev), algorithm=nnqs.ALGO_LITERAL,
                                      literal_kernel=lk)
        n = len(st.keys)
        a = _lit_run(nnqs, ham, tab, dev, lk, n=n)
        b = _lit_run(nnqs, ham, tab, dev, lk, rows=rows, rlp=rlp)
        cut = 1 + n // 3
        d = _lit_run(nnqs, ham, tab, dev, lk, n=n - cut - 1, row_begin=cut)
        outs.append((a, b, d))
    for (a, b, d) in outs[1:]:
        for u, v in zip((a, b, d), outs[0]):
            assert u[0].tobytes() == v[0].tobytes()
            assert np.array_equal(u[1], v[1])
    el = outs[0][0][0]
    got = el[:, 0] + 1j * el[:, 1]
    ok = np.isfinite(lp[:, 0])
    assert np.all(np.isnan(got[~ok].real))
    ref, scale = R.eloc(m.h1, m.h2, m.e_core, st.keys[ok], lp[ok], keys=st.keys, logpsi=lp, with_scale=True)
    _assert_close(got[ok], ref, scale, f"C{c}/{variant} bit-sliced literal")


def test_c5_literal_kernels_bit_identical(nnqs, dev, c5):
    """C5 (120 qubits, 2.06M groups): a ragged 2085-row slice plus the HF row and the
    10 longest-list rows as explicit rows -- bit-sliced == staged, bit for bit, equal
    counts, and the oracle's E_loc within R14."""
    m, st, ham, _ = c5
    hf, top, _ = _c5_special_rows(st)
    idx = np.unique(np.concatenate([np.arange(2085), [hf], top]))
    rows, rlp = st.keys[idx], st.logpsi[idx]
    res = []
    for lk in (0, 1):
        tab = nnqs.nnqs_table_prepare(ham, 0, _t(st.keys, dev), _t(st.logpsi, dev), algorithm=nnqs.ALGO_LITERAL,
                                      literal_kernel=lk)
        res.append(_lit_run(nnqs, ham, tab, dev, lk, rows=rows, rlp=rlp))
        tab.close()
    assert res[0][0].tobytes() == res[1][0].tobytes() and np.array_equal(res[0][1], res[1][1])
    sub = np.unique(np.concatenate([C.oracle_row_subset(5, len(idx), 24), np.searchsorted(idx, [hf])]))
    got = res[0][0][sub, 0] + 1j * res[0][0][sub, 1]
    ref, scale = R.eloc(m.h1, m.h2, m.e_core, rows[sub], rlp[sub], keys=st.keys, logpsi=st.logpsi, with_scale=True)
    _assert_close(got, ref, scale, "C5 bit-sliced literal")
