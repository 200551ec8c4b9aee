"""GPU batch autoregressive sampling (nnqs_bas_layer, csrc/bas.cu; sampler.py) against
the BAS oracle (oracle/bas.py), bit for bit: the same prefixes, weights and
conditional probabilities give the same children and counts (integer outputs), for
weights up to the paper's N_s = 10^12; whole BAS runs and their parallel
partition equal the oracle's; the ansatz-driven sampler and one VMC
iteration (stages 1-6) on H2."""
import numpy as np
import pytest
import torch

from oracle import bas

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nnqs():
    import __graft_entry__ as g
    g.build()
    from paper_2306_16705_b200 import nnqs as m
    return m


@pytest.fixture(scope="module")
def dev():
    return torch.device("cuda", 0)


def _keys_t(keys, dev):
    a = np.array([[k & bas.M64, k >> 64] for k in keys], dtype=np.uint64).reshape(-1, 2)
    return torch.from_numpy(a.view(np.int64)).to(dev)


def _keys_int(t):
    a = t.cpu().numpy().view(np.uint64)
    return [int(lo) | (int(hi) << 64) for lo, hi in a]


def _random_layer(rng, n_orb, orbital, n_up, n_dn, m):
    """m distinct feasible prefixes (orbitals above `orbital` filled), ascending."""
    out = set()
    for _ in range(50 * m):
        if len(out) >= m:
            break
        key, na, nb = 0, 0, 0
        for o in range(n_orb - 1, orbital, -1):
            ok = bas.feasible(na, nb, o, n_up, n_dn)
            choice = int(rng.choice([c for c in range(4) if ok[c]]))
            key = bas.child_key(key, choice, o)
            na += choice & 1
            nb += choice >> 1
        out.add(key)
    return sorted(out)


@pytest.mark.parametrize("n_orb,orbital,n_up,n_dn,m", [(6, 3, 3, 3, 40), (30, 17, 8, 7, 500), (60, 40, 15, 15, 800),
                                                       (64, 33, 20, 12, 300)])
def test_layer_equals_oracle(nnqs, dev, n_orb, orbital, n_up, n_dn, m):
    rng = np.random.default_rng(n_orb + orbital)
    keys = _random_layer(rng, n_orb, orbital, n_up, n_dn, m)
    m = len(keys)
    scales = np.array([0, 1, 3, 17, 1000, 10**6, 10**9, 10**12])
    counts = (scales[rng.integers(0, len(scales), m)] * rng.uniform(0.5, 1.0, m)).astype(np.int64)
    probs = rng.random((m, 4))
    probs[rng.random((m, 4)) < 0.1] = 0.0
    probs[:, 0] += 1e-3                       # keep a feasible outcome with mass in most nodes
    seed = 1234567
    want = []
    ok_rows = []
    for j in range(m):
        try:
            bas.split_node(keys[j], int(counts[j]), probs[j], orbital, n_up, n_dn, seed)
            ok_rows.append(j)
        except ValueError:
            pass
    keys = [keys[j] for j in ok_rows]
    counts, probs = counts[ok_rows], probs[ok_rows]
    want = bas.layer(list(zip(keys, counts.tolist())), probs, orbital, n_up, n_dn, seed)
    kt, ct = nnqs.nnqs_bas_layer(_keys_t(keys, dev), torch.from_numpy(counts).to(dev),
                                 torch.from_numpy(np.ascontiguousarray(probs)).to(dev), orbital, n_orb, n_up, n_dn,
                                 seed)
    got = list(zip(_keys_int(kt), ct.cpu().tolist()))
    assert got == want
    assert sum(c for _, c in got) == int(counts.sum())


def test_layer_errors(nnqs, dev):
    k = torch.zeros((1, 2), dtype=torch.int64, device=dev)
    c = torch.ones(1, dtype=torch.int64, device=dev)
    p = torch.tensor([[1.0, 0.0, 0.0, 0.0]], dtype=torch.float64, device=dev)
    with pytest.raises(nnqs.NNQSError):                    # only infeasible mass: caller bug
        nnqs.nnqs_bas_layer(k, c, p, 0, 1, 1, 1, 0)
    with pytest.raises(nnqs.NNQSError):
        nnqs.nnqs_bas_layer(k, c, p, 5, 3, 1, 1, 0)         # orbital outside [0, n)
    kt, ct = nnqs.nnqs_bas_layer(k[:0], c[:0], p[:0], 0, 2, 1, 1, 0)
    assert kt.shape[0] == 0


def _hash_conditional(nodes_keys, orbital):
    """A deterministic synthetic model: probabilities from a hash of (prefix, orbital)."""
    out = np.empty((len(nodes_keys), 4))
    for j, k in enumerate(nodes_keys):
        h = bas.mix(bas.mix(k & bas.M64 ^ (k >> 64) * 31) + orbital)
        out[j] = [0.05 + ((h >> (16 * o)) & 0xFFFF) / 65536.0 for o in range(4)]
    return out


@pytest.mark.parametrize("n_orb,n_up,n_dn,ns", [(4, 2, 2, 10**12), (10, 4, 3, 10**9), (20, 7, 7, 10**5)])
def test_bas_run_equals_oracle(nnqs, dev, n_orb, n_up, n_dn, ns):
    from paper_2306_16705_b200.sampler import bas_sample

    def cond_gpu(keys, orbital):
        return torch.from_numpy(_hash_conditional(_keys_int(keys), orbital)).to(dev)

    def cond_oracle(nodes, orbital):
        return _hash_conditional([k for k, _ in nodes], orbital)

    seed = 77
    want = bas.sample(cond_oracle, n_orb, n_up, n_dn, ns, seed)
    kt, ct, widths = bas_sample(cond_gpu, n_orb, n_up, n_dn, ns, seed, dev)
    got = list(zip(_keys_int(kt), ct.cpu().tolist()))
    assert got == want
    assert widths[-1] == len(want)
    # parallel BAS: every part, concatenated in rank order, is the serial set
    for parts in (2, 3):
        union = []
        for r in range(parts):
            k2, c2, _ = bas_sample(cond_gpu, n_orb, n_up, n_dn, ns, seed, dev, n_parts=parts, part=r, n_u_star=8)
            union += list(zip(_keys_int(k2), c2.cpu().tolist()))
        assert union == want


def test_ansatz_sampler_and_vmc_on_h2(nnqs, dev):
    """QiankunNet-shaped ansatz on H2 (C1): with N_s = 10^12 the sampled frequencies equal
    |psi|^2 to ~1e-6; the VMC energy estimate (stages 1-4) equals <psi|H|psi>/<psi|psi>
    from the oracle's dense H; one full iteration (stages 5-6) moves the parameters."""
    from oracle import dense
    from paper_2306_16705_b200.ansatz import QiankunNet
    from paper_2306_16705_b200.vmc import VMC
    from synth import configs as C
    from synth import samples as S
    mol = C.molecule(1)
    model = QiankunNet(2, 1, 1, seed=3).to(dev)
    ham = nnqs.nnqs_ham_compress(mol.h1, mol.h2, mol.n_qubits, mol.e_core, device=0)
    keys = torch.from_numpy(S.sector_keys(2, 1, 1).view(np.int64)).to(dev)
    with torch.no_grad():
        lp = model.log_psi(keys).cpu().numpy()
    psi = np.exp(lp[:, 0] + 1j * lp[:, 1])
    Hs = dense.sector_hamiltonian(mol.h1, mol.h2, mol.e_core, S.sector_keys(2, 1, 1))
    e_exact = float(np.real(np.vdot(psi, Hs @ psi) / np.vdot(psi, psi)))
    vmc = VMC(ham, model, n_samples=10**12, seed=5, lr=1e-2)
    before = [p.detach().clone() for p in model.parameters()]
    out = vmc.step()
    assert out["W"] == 1e12
    assert abs(out["energy"].real - e_exact) < 1e-4
    assert any(not torch.equal(a, b) for a, b in zip(before, model.parameters()))
    es = [vmc.step()["energy"].real for _ in range(30)]
    assert min(es) < out["energy"].real                   # the optimiser lowers the energy
