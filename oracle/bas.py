"""Oracle of batch autoregressive sampling (BAS) -- TEST INFRASTRUCTURE ONLY.

Plain Python, one node at a time, written from the paper and DESIGN.md
reading R24; shares no code with libnnqs (whose kernel is csrc/bas.cu).

  * BAS (Fig. 3(b)): layer by layer, every unique prefix of
    weight w draws "exactly w samples" of the next local state from its
    conditional distribution; unique children keep their counts, zero-weight
    children are pruned.
  * Two qubits (one spatial orbital) per step, orbitals from n-1 down to 0,
    "the reverse order of the qubits"; outcome o of orbital i sets the
    spin-up qubit 2i to o & 1 and the spin-down qubit 2i+1 to o >> 1 (R7).
  * Number-conservation mask, Eq. (12): outcomes whose running
    up / down electron count exceeds n_up / n_dn are zeroed, then renormalised;
    reading R24 also zeroes outcomes that can no longer reach n_up / n_dn.
  * The multinomial draw (R24): sequential conditional binomials over o = 0, 1, 2
    (c_3 = the rest); Binomial(n, p) by inversion (BINV) when n min(p, 1-p) < 10,
    else Hormann's BTRS; uniforms U_t = floor(mix(base + t * golden) / 2^11) / 2^53
    with base = mix(mix(mix(mix(seed) ^ (i + 1)) ^ key_lo) ^ key_hi), t = 1, 2, ...
    per node, mix = the splitmix64 finaliser.
"""
from __future__ import annotations

import math

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
LOG_FACT_SMALL = [0.0, 0.0, 0.6931471805599453, 1.791759469228055, 3.1780538303479458,
                  4.787491742782046, 6.579251212010101, 8.525161361065415, 10.60460290274525,
                  12.801827480081469]


def mix(z: int) -> int:
    z &= M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


class Uniforms:
    """The node's uniform stream (reading R24)."""

    def __init__(self, seed: int, orbital: int, key_lo: int, key_hi: int):
        self.base = mix(mix(mix(mix(seed) ^ (orbital + 1)) ^ key_lo) ^ key_hi)
        self.t = 0

    def __call__(self) -> float:
        self.t += 1
        return float(mix(self.base + self.t * GOLDEN) >> 11) * 2.0 ** -53


def log_factorial(k: float) -> float:
    """log(k!) for integral k >= 0: exact table below 10, Stirling with two
    correction terms above (the form BTRS uses)."""
    if k < 10.0:
        return LOG_FACT_SMALL[int(k)]
    z = k + 1.0
    return (k + 0.5) * math.log(z) - z + 0.9189385332046727 + (1.0 / 12.0 - 1.0 / (360.0 * z * z)) / z


def binomial(n: int, p: float, U: Uniforms) -> int:
    """Binomial(n, p) draw (reading R24)."""
    if n <= 0 or p <= 0.0:
        return 0
    if p >= 1.0:
        return n
    if p > 0.5:
        return n - _binomial_half(n, 1.0 - p, U)
    return _binomial_half(n, p, U)


def _binomial_half(n: int, p: float, U: Uniforms) -> int:
    nd, q = float(n), 1.0 - p
    if nd * p < 10.0:
        # BINV: walk the CDF from x = 0 with f(0) = q^n, f(x) = f(x-1) ((n+1) s / x - s), s = p/q
        s = p / q
        a = (nd + 1.0) * s
        while True:
            r = math.exp(nd * math.log1p(-p))
            u = U()
            x = 0
            while x <= n and x < 256:
                if u < r:
                    return x
                u -= r
                x += 1
                r *= a / float(x) - s
    # BTRS: W. Hormann, "The generation of binomial random variates" (1993)
    spq = math.sqrt(nd * p * q)
    b = 1.15 + 2.53 * spq
    a = -0.0873 + 0.0248 * b + 0.01 * p
    c = nd * p + 0.5
    vr = 0.92 - 4.2 / b
    alpha = (2.83 + 5.1 / b) * spq
    lpq = math.log(p / q)
    m = math.floor((nd + 1.0) * p)
    h = log_factorial(m) + log_factorial(nd - m)
    while True:
        u = U() - 0.5
        v = U()
        us = 0.5 - abs(u)
        if us == 0.0:
            continue                      # k = +-inf: outside [0, n]
        k = math.floor((2.0 * a / us + b) * u + c)
        if not (0.0 <= k <= nd):
            continue
        if us >= 0.07 and v <= vr:
            return int(k)
        v = math.log(v * alpha / (a / (us * us) + b))
        if v <= h - log_factorial(k) - log_factorial(nd - k) + (k - m) * lpq:
            return int(k)


def feasible(na: int, nb: int, orbital: int, n_up: int, n_dn: int) -> list[bool]:
    """Eq. (12) plus reachability (R24) for the 4 outcomes of `orbital`, given the
    electrons na / nb already placed on the orbitals above it."""
    out = []
    for o in range(4):
        a2, b2 = na + (o & 1), nb + (o >> 1)
        out.append(a2 <= n_up and b2 <= n_dn and a2 + orbital >= n_up and b2 + orbital >= n_dn)
    return out


def split_node(key: int, w: int, probs, orbital: int, n_up: int, n_dn: int, seed: int) -> list[int]:
    """Children counts [c_0..c_3] of one node: the masked multinomial draw of w."""
    na = bin(key & int("01" * 64, 2)).count("1")
    nb = bin(key & int("10" * 64, 2)).count("1")
    ok = feasible(na, nb, orbital, n_up, n_dn)
    q = [float(probs[o]) if ok[o] else 0.0 for o in range(4)]
    tail = [0.0] * 4
    tail[3] = q[3]
    tail[2] = q[2] + tail[3]
    tail[1] = q[1] + tail[2]
    tail[0] = q[0] + tail[1]
    if w > 0 and not tail[0] > 0.0:
        raise ValueError("node without a feasible continuation")
    U = Uniforms(seed, orbital, key & M64, key >> 64)
    c = [0, 0, 0, 0]
    rem = w
    for o in range(3):
        if rem > 0 and q[o] > 0.0:
            c[o] = binomial(rem, q[o] / tail[o], U)
        rem -= c[o]
    c[3] = rem
    return c


def child_key(key: int, o: int, orbital: int) -> int:
    return key | ((o & 1) << (2 * orbital)) | ((o >> 1) << (2 * orbital + 1))


def layer(nodes, probs, orbital: int, n_up: int, n_dn: int, seed: int):
    """nodes: list of (key int, weight); probs: per node 4 floats -> children list."""
    out = []
    for (key, w), pr in zip(nodes, probs):
        for o, c in enumerate(split_node(key, w, pr, orbital, n_up, n_dn, seed)):
            if c > 0:
                out.append((child_key(key, o, orbital), c))
    return out


def sample(conditional, n_orbitals: int, n_up: int, n_dn: int, n_samples: int, seed: int,
           split=None):
    """Full BAS: conditional(nodes, orbital) -> per-node 4 probabilities.  Returns the
    unique samples [(key, count)] ascending.  split=(k_threshold, n_parts, part): the
    parallel BAS of P:280-284 -- replay layers until the width exceeds the threshold,
    keep this part's contiguous slice of that layer (see partition()), finish it."""
    nodes = [(0, int(n_samples))]
    cut = False
    for orbital in range(n_orbitals - 1, -1, -1):
        nodes = layer(nodes, conditional(nodes, orbital), orbital, n_up, n_dn, seed)
        if split is not None and not cut and len(nodes) > split[0]:
            b, e = partition([w for _, w in nodes], split[1])[split[2]]
            nodes = nodes[b:e]
            cut = True
    return nodes


def partition(weights, n_parts: int):
    """Contiguous split of a layer into n_parts with about equal total weight
    ("approximately the same number of samples"): part r starts at the
    first node whose weight prefix reaches r/n_parts of the total."""
    tot = sum(weights)
    bounds, acc, r = [0], 0, 1
    for j, w in enumerate(weights):
        while r < n_parts and acc >= tot * r / n_parts:
            bounds.append(j)
            r += 1
        acc += w
    while len(bounds) < n_parts:
        bounds.append(len(weights))
    bounds.append(len(weights))
    return [(bounds[r], bounds[r + 1]) for r in range(n_parts)]
