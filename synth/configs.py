"""The five BASELINE.json configurations, restated as seeded synthetic inputs
(SURVEY.md Sec. 8(d) 'Configs').

C1  H2 STO-3G, 4 qubits, exact mode over all 16 configurations
C2  LiH-shaped (C2v labels), 12 qubits, exact + sample-space
C3  H2O-shaped (C2v), 14 qubits, sample-space
C4  N2-shaped (D2h), 20 qubits, sample-space (1/2/4/8 GPUs)
C5  synthetic 120-qubit molecule (2 irreps), 10^6 unique near-HF samples

Seeds (config c): integrals 100+c, sample set 200+c, row draws 300+c,
psi noise 400+c, random complex psi 500+c, 50% subsets 600+c, oracle row
subsets 700+c.
"""
from __future__ import annotations

import functools
from dataclasses import dataclass, field

import numpy as np

from . import integrals as I
from . import samples as S

# abelian irrep labels as XOR groups
C2V = {"a1": 0, "b1": 1, "b2": 2, "a2": 3}
D2H = {"ag": 0, "b1g": 1, "b2g": 2, "b3g": 3, "au": 4, "b1u": 5, "b2u": 6, "b3u": 7}


@dataclass
class Molecule:
    name: str
    n_orb: int
    n_alpha: int
    n_beta: int
    h1: np.ndarray
    h2: np.ndarray
    e_core: float
    irreps: list = field(default_factory=list)

    @property
    def n_qubits(self) -> int:
        return 2 * self.n_orb


@functools.lru_cache(maxsize=None)
def molecule(c: int) -> Molecule:
    if c == 1:
        h1, h2, e, na, nb = I.h2_sto3g()
        return Molecule("H2/STO-3G", 2, na, nb, h1, h2, e, [0, 1])
    if c == 2:
        irr = [C2V[s] for s in ["a1", "a1", "a1", "b1", "b2", "a1"]]
        h1, h2, e = I.synthetic_integrals(6, irr, 100 + c, e_core=1.0)
        return Molecule("LiH-shaped/C2v", 6, 2, 2, h1, h2, e, irr)
    if c == 3:
        irr = [C2V[s] for s in ["a1", "a1", "b2", "a1", "b1", "a1", "b2"]]
        h1, h2, e = I.synthetic_integrals(7, irr, 100 + c, e_core=9.0)
        return Molecule("H2O-shaped/C2v", 7, 5, 5, h1, h2, e, irr)
    if c == 4:
        irr = [D2H[s] for s in ["ag", "b1u", "ag", "b1u", "b3u", "b2u", "ag", "b2g", "b3g", "b1u"]]
        h1, h2, e = I.synthetic_integrals(10, irr, 100 + c, e_core=23.0)
        return Molecule("N2-shaped/D2h", 10, 7, 7, h1, h2, e, irr)
    if c == 5:
        irr = [p % 2 for p in range(60)]
        h1, h2, e = I.synthetic_integrals(60, irr, 100 + c, e_core=200.0)
        return Molecule("synthetic-120/2-irrep", 60, 15, 15, h1, h2, e, irr)
    raise ValueError(c)


@dataclass
class SampleTable:
    """A sorted unique-sample table with counts and log-psi (the paper's
    id_lut / wf_lut)."""
    keys: np.ndarray      # uint64 [m, 2]
    counts: np.ndarray    # int64 [m]
    logpsi: np.ndarray    # float64 [m, 2]


@functools.lru_cache(maxsize=None)
def sample_table(c: int, variant: str = "full") -> SampleTable:
    """C2-C4: 'full' = the whole (n_alpha, n_beta) sector, 'half' = a seeded 50%
    subset (exercises misses).  C5: 10^6 unique near-HF samples.
    C1/C2 'exact': the 2^N table is built by exact_psi()."""
    mol = molecule(c)
    if c == 5:
        keys, counts, _ = S.near_hf_samples(60, 15, 15, 1_000_000, 200 + c)
        return SampleTable(keys, counts, S.logpsi_from_counts(keys, counts, 400 + c))
    keys = S.sector_keys(mol.n_orb, mol.n_alpha, mol.n_beta)
    if variant == "half":
        keys = S.subset(keys, 0.5, 600 + c)
    rng = np.random.default_rng(200 + c)
    counts = rng.integers(1, 6, size=len(keys)).astype(np.int64)
    return SampleTable(keys, counts, S.random_logpsi(len(keys), 500 + c, re_scale=0.5))


def exact_random_psi(c: int) -> np.ndarray:
    """Exact mode: complex log psi over all 2^N configurations, no zeros."""
    mol = molecule(c)
    return S.random_logpsi(1 << mol.n_qubits, 500 + c, re_scale=0.5)


def row_draws(c: int, n_table: int) -> np.ndarray:
    """Rows drawn with replacement from the table (SURVEY.md reading 19):
    C2 10^4, C3/C4 10^5."""
    n_rows = {2: 10_000, 3: 100_000, 4: 100_000}[c]
    return S.draw_rows(n_table, n_rows, 300 + c)


def oracle_row_subset(c: int, n_table: int, k: int) -> np.ndarray:
    rng = np.random.default_rng(700 + c)
    return np.sort(rng.choice(n_table, size=min(k, n_table), replace=False))
