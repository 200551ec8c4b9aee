"""Seeded synthetic sample sets: bit-packed keys, counts and complex log-psi.

INPUT GENERATORS only -- none of the method's arithmetic (see synth/integrals.py).

Key layout (Sec. 3.4(5) "encode the boolean tuple into the bits of
a 64-bit integer (in case 64 <= N < 128, we use two integers)"): qubit j is bit
(j mod 64) of word floor(j/64); word0 = qubits 0..63, word1 = qubits 64..127.
Spin orbital (p, alpha) -> qubit 2p, (p, beta) -> qubit 2p+1.
Tables are sorted ascending as 128-bit integers (word1, then word0).
"""
from __future__ import annotations

import itertools

import numpy as np


def _spread32(v: np.ndarray) -> np.ndarray:
    """Interleave zeros: bit i of the low 32 bits of v -> bit 2i."""
    v = v.astype(np.uint64) & np.uint64(0xFFFFFFFF)
    v = (v | (v << np.uint64(16))) & np.uint64(0x0000FFFF0000FFFF)
    v = (v | (v << np.uint64(8))) & np.uint64(0x00FF00FF00FF00FF)
    v = (v | (v << np.uint64(4))) & np.uint64(0x0F0F0F0F0F0F0F0F)
    v = (v | (v << np.uint64(2))) & np.uint64(0x3333333333333333)
    v = (v | (v << np.uint64(1))) & np.uint64(0x5555555555555555)
    return v


def keys_from_strings(alpha: np.ndarray, beta: np.ndarray) -> np.ndarray:
    """alpha/beta occupation strings (uint64, bit p = orbital p, n <= 64) ->
    uint64 keys [m, 2] (word0, word1)."""
    alpha = np.asarray(alpha, dtype=np.uint64)
    beta = np.asarray(beta, dtype=np.uint64)
    lo = _spread32(alpha) | (_spread32(beta) << np.uint64(1))
    hi = _spread32(alpha >> np.uint64(32)) | (_spread32(beta >> np.uint64(32)) << np.uint64(1))
    return np.stack([lo, hi], axis=1)


def sort_unique_keys(keys: np.ndarray):
    """Sort [m,2] keys ascending as 128-bit ints; return (unique_keys, inverse, counts)."""
    order = np.lexsort((keys[:, 0], keys[:, 1]))
    sk = keys[order]
    new = np.ones(len(sk), dtype=bool)
    new[1:] = (sk[1:, 0] != sk[:-1, 0]) | (sk[1:, 1] != sk[:-1, 1])
    uniq = sk[new]
    grp = np.cumsum(new) - 1
    inverse = np.empty(len(keys), dtype=np.int64)
    inverse[order] = grp
    counts = np.bincount(grp, minlength=len(uniq)).astype(np.int64)
    return np.ascontiguousarray(uniq), inverse, counts


def sector_strings(n: int, k: int) -> np.ndarray:
    """All n-bit strings with k bits set, as uint64, ascending."""
    out = []
    for occ in itertools.combinations(range(n), k):
        v = 0
        for p in occ:
            v |= 1 << p
        out.append(v)
    return np.array(sorted(out), dtype=np.uint64)


def sector_keys(n: int, n_alpha: int, n_beta: int) -> np.ndarray:
    """Every determinant of the (n_alpha, n_beta) sector, sorted keys [d, 2]."""
    a = sector_strings(n, n_alpha)
    b = sector_strings(n, n_beta)
    A, B = np.meshgrid(a, b, indexing="ij")
    keys = keys_from_strings(A.ravel(), B.ravel())
    uniq, _, _ = sort_unique_keys(keys)
    return uniq


def _draw_restricted(rng, strings, weight, want_set):
    """For each string, draw an orbital p with probability proportional to
    weight[p] among the orbitals whose bit equals want_set (rejection)."""
    cdf = np.cumsum(weight / weight.sum())
    out = np.empty(len(strings), dtype=np.int64)
    todo = np.arange(len(strings))
    while len(todo):
        p = np.minimum(np.searchsorted(cdf, rng.random(len(todo))), len(cdf) - 1)
        bit = ((strings[todo] >> p.astype(np.uint64)) & np.uint64(1)).astype(bool)
        ok = bit == want_set
        out[todo[ok]] = p[ok]
        todo = todo[~ok]
    return out


def near_hf_samples(n: int, n_alpha: int, n_beta: int, n_unique: int, seed: int,
                    hf_count: int = 1000):
    """Unique near-Hartree-Fock determinants with multiplicities.

    Shaped like the paper's sample sets (N_u/N_s ~ 0.4, mostly counts of 1;
    PAPER.md:226-231 'stores only the unique samples with their weights',
    PAPER.md:452, 533): the HF determinant with count hf_count, plus draws of
    excitation rank r in {1,2,3,4} with P = (0.10, 0.55, 0.25, 0.10); each
    excitation step picks a spin uniformly, a hole among the occupied orbitals
    of that spin with weight exp(-|p - n_s + 1/2|/6) and a particle among the
    empty ones with weight exp(-|p - n_s + 1/2|/10).  Draws continue until
    n_unique distinct determinants exist (the HF one included); counts are the
    multiplicities among the draws kept.
    Returns (keys[n_unique,2] sorted, counts[n_unique] int64, n_samples).
    """
    assert n <= 64
    rng = np.random.default_rng(seed)
    orb = np.arange(n, dtype=np.float64)
    nel = (n_alpha, n_beta)
    hf = [np.uint64((1 << ns) - 1) for ns in nel]
    hf_key = keys_from_strings(np.array([hf[0]]), np.array([hf[1]]))
    chunk = 1 << 17
    parts = [hf_key]
    n_drawn, target = 0, int(2.5 * n_unique)
    while True:
        strings = [np.full(chunk, hf[0], dtype=np.uint64), np.full(chunk, hf[1], dtype=np.uint64)]
        rank = rng.choice(4, size=chunk, p=[0.10, 0.55, 0.25, 0.10]) + 1
        for step in range(4):
            active = rank > step
            spin = rng.integers(0, 2, size=chunk)
            for s in (0, 1):
                sel = np.nonzero(active & (spin == s))[0]
                if len(sel) == 0 or nel[s] == 0 or nel[s] == n:
                    continue
                cur = strings[s][sel]
                dist = np.abs(orb - nel[s] + 0.5)
                hole = _draw_restricted(rng, cur, np.exp(-dist / 6.0), want_set=True)
                part = _draw_restricted(rng, cur, np.exp(-dist / 10.0), want_set=False)
                flip = (np.uint64(1) << hole.astype(np.uint64)) | (np.uint64(1) << part.astype(np.uint64))
                strings[s][sel] = cur ^ flip
        parts.append(keys_from_strings(strings[0], strings[1]))
        n_drawn += chunk
        if n_drawn < target:
            continue
        all_keys = np.concatenate(parts)
        uniq, inverse, _ = sort_unique_keys(all_keys)
        if len(uniq) < n_unique:
            target = int(n_drawn * max(1.05, 1.02 * n_unique / len(uniq)))
            continue
        first = np.full(len(uniq), len(all_keys), dtype=np.int64)
        rev = np.arange(len(all_keys) - 1, -1, -1)
        first[inverse[rev]] = rev          # last write wins -> first occurrence
        cut = np.sort(first)[n_unique - 1]
        keep = inverse[: cut + 1]
        counts_all = np.bincount(keep, minlength=len(uniq))
        chosen = np.nonzero(counts_all)[0]
        ukeys = uniq[chosen]
        counts = counts_all[chosen].astype(np.int64)
        hf_pos = np.nonzero((ukeys[:, 0] == hf_key[0, 0]) & (ukeys[:, 1] == hf_key[0, 1]))[0][0]
        counts[hf_pos] += hf_count - 1
        return np.ascontiguousarray(ukeys), counts, int(counts.sum())


def logpsi_from_counts(keys: np.ndarray, counts: np.ndarray, seed: int, hf_index: int | None = None):
    """log psi = 1/2 ln(count/N_s) + N(0,0.05) + i*pi*Bernoulli(1/2) + i*N(0,0.05)
    (an amplitude consistent with the sampled frequencies plus noise; the
    paper's psi = |psi| e^{i phi}).  Returns float64 [m, 2]."""
    rng = np.random.default_rng(seed)
    ns = counts.sum()
    re = 0.5 * np.log(counts / ns) + rng.normal(0.0, 0.05, size=len(counts))
    im = np.pi * rng.integers(0, 2, size=len(counts)) + rng.normal(0.0, 0.05, size=len(counts))
    if hf_index is not None:
        im[hf_index] = 0.0
    return np.ascontiguousarray(np.stack([re, im], axis=1))


def random_logpsi(m: int, seed: int, re_scale: float = 1.0):
    """Generic complex log-amplitudes with no zeros."""
    rng = np.random.default_rng(seed)
    re = rng.normal(-1.0, re_scale, size=m)
    im = rng.uniform(-np.pi, np.pi, size=m)
    return np.ascontiguousarray(np.stack([re, im], axis=1))


def subset(keys: np.ndarray, frac: float, seed: int) -> np.ndarray:
    """A seeded subset of a sorted table (keeps sort order)."""
    rng = np.random.default_rng(seed)
    m = max(1, int(round(frac * len(keys))))
    pick = np.sort(rng.choice(len(keys), size=m, replace=False))
    return np.ascontiguousarray(keys[pick])


def draw_rows(n_table: int, n_rows: int, seed: int) -> np.ndarray:
    """Row indices into a table, drawn with replacement (SURVEY.md reading 19)."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, n_table, size=n_rows)
