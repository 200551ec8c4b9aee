"""Closed-form flip-group (K') and Pauli-string (N_h) counts of the JW-mapped
Hamiltonian from abelian irrep labels (TEST INFRASTRUCTURE ONLY).

Assumes every symmetry-allowed integral is non-zero (the synthetic generator's
property).  With spin orbitals N = 2n and irreps G_p combined by XOR:
  W2   = 2 * #{p<q : G_p = G_q}                      (2-site same-spin groups)
  Q_ss = 2 * #{p<q<r<s : G_p^G_q^G_r^G_s = 0}        (4-site same-spin groups)
  Q_os = #{(p<q), (r<s) : G_p^G_q = G_r^G_s}         (4-site opposite-spin)
  K'   = 1 + W2 + Q_ss + Q_os
  N_h  = (1 + N + C(N,2)) + 2(N-1) W2 + 6 Q_ss + 4 Q_os
Counting by enumeration (no shortcuts).  Pinned against Table 1's N2 value
N_h = 2239 and against the Walsh-Hadamard recovery of dense H.
"""
from __future__ import annotations

import itertools
from collections import Counter
from math import comb


def group_counts(irreps):
    g = list(irreps)
    n = len(g)
    N = 2 * n
    same_pairs = sum(1 for p, q in itertools.combinations(range(n), 2) if g[p] == g[q])
    w2 = 2 * same_pairs
    q_ss = 2 * sum(1 for p, q, r, s in itertools.combinations(range(n), 4) if g[p] ^ g[q] ^ g[r] ^ g[s] == 0)
    pair_irr = Counter(g[p] ^ g[q] for p, q in itertools.combinations(range(n), 2))
    q_os = sum(c * c for c in pair_irr.values())
    k = 1 + w2 + q_ss + q_os
    nh = (1 + N + comb(N, 2)) + 2 * (N - 1) * w2 + 6 * q_ss + 4 * q_os
    return k, nh


def group_counts_fast(irreps):
    """Same counts for large n (C5): the 4-subset count via irrep histograms."""
    g = list(irreps)
    n = len(g)
    N = 2 * n
    hist = Counter(g)
    same_pairs = sum(c * (c - 1) // 2 for c in hist.values())
    pair_irr = Counter()
    labels = sorted(hist)
    for a in labels:
        for b in labels:
            if a < b:
                pair_irr[a ^ b] += hist[a] * hist[b]
            elif a == b:
                pair_irr[0] += hist[a] * (hist[a] - 1) // 2
    q_os = sum(c * c for c in pair_irr.values())
    # 4-subsets with XOR 0: count multisets of labels (a<=b<=c<=d) with a^b^c^d == 0
    total = 0
    for combo in itertools.combinations_with_replacement(labels, 4):
        if combo[0] ^ combo[1] ^ combo[2] ^ combo[3]:
            continue
        ways = 1
        for lab, m in Counter(combo).items():
            ways *= comb(hist[lab], m)
        total += ways
    q_ss = 2 * total
    w2 = 2 * same_pairs
    return 1 + w2 + q_ss + q_os, (1 + N + comb(N, 2)) + 2 * (N - 1) * w2 + 6 * q_ss + 4 * q_os


def flip_masks(irreps):
    """The set of flip masks X (as 128-bit ints) of the JW-mapped Eq. (9) with every
    symmetry-allowed integral non-zero, written out from the excitation classes
    (spin orbital (p, sigma) -> qubit 2p + sigma): X = 0; a same-spin pair (p, q) with
    G_p = G_q (one-body h_pq and the two-body terms with one index pair equal); a
    same-spin quad with G_p^G_q^G_r^G_s = 0; an up pair x a down pair with equal pair
    irreps.  Enumeration, no shortcuts: the P1 reference at N = 20 and 120."""
    g = list(irreps)
    n = len(g)
    out = {0}
    for s in (0, 1):
        for p, q in itertools.combinations(range(n), 2):
            if g[p] == g[q]:
                out.add((1 << (2 * p + s)) | (1 << (2 * q + s)))
        for p, q, r, t in itertools.combinations(range(n), 4):
            if g[p] ^ g[q] ^ g[r] ^ g[t] == 0:
                out.add((1 << (2 * p + s)) | (1 << (2 * q + s)) | (1 << (2 * r + s)) | (1 << (2 * t + s)))
    pairs = {}
    for p, q in itertools.combinations(range(n), 2):
        pairs.setdefault(g[p] ^ g[q], []).append((1 << (2 * p)) | (1 << (2 * q)))
    for lab, ups in pairs.items():
        downs = [m << 1 for m in ups]
        for u in ups:
            for d in downs:
                out.add(u | d)
    return out


def hamiltonian_memory(n_qubits: int, n_groups: int, n_terms: int):
    """Fig. 6(b) vs 6(c) storage (Fig. 9 at PAPER.md:500-504), with
    one byte per boolean entry (reading: the figure's "boolean tuples"):
      (b) per Pauli string: XY tuple (N) + YZ tuple (N) + Y count (int32) + coefficient (f64)
      (c) per string: YZ tuple (N) + fused coefficient (f64); per unique XY tuple
          (flip group): the tuple (N) + its idxs entry (int32)
    Returns (bytes_b, bytes_c, reduction = 1 - c/b)."""
    b = n_terms * (2 * n_qubits + 4 + 8)
    c = n_terms * (n_qubits + 8) + n_groups * (n_qubits + 4)
    return b, c, 1.0 - c / b
