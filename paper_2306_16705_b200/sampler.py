"""Batch autoregressive sampling (BAS) on the GPU -- stage 1 of the data-centric
VMC iteration and its parallel partition (Fig. 5).

Every layer is one nnqs_bas_layer call (csrc/bas.cu): the unique prefixes of the
layer, their weights and the model's conditional distribution of the next
spatial orbital go in, the pruned unique children come out.  The
model's conditionals are computed by the caller's `conditional(keys, orbital)`
(e.g. ansatz.QiankunNet.conditionals); this module only drives the layers.

Parallel BAS: all ranks replay the layers with the same seed until the layer is
wider than n_u_star ("the first local sampling step such that ... N_{u,k}
is larger than N_u*"), then rank r keeps a contiguous slice of that layer with
about 1/P of the samples and finishes its subtrees alone.  The node
draws are keyed by (seed, orbital, prefix), so the union of the ranks' samples
is exactly the serial sample set, and concatenated in rank order it is sorted.
"""
from __future__ import annotations

import numpy as np

from . import nnqs


def partition(counts, n_parts: int):
    """Contiguous split of a layer's nodes (weights `counts`, host array) into
    n_parts slices of about equal total weight: slice r starts at the first node
    whose exclusive weight prefix reaches r / n_parts of the total."""
    w = np.asarray(counts, dtype=np.int64)
    excl = np.concatenate([[0], np.cumsum(w)[:-1]]) if len(w) else np.zeros(0, dtype=np.int64)
    tot = int(w.sum())
    starts = [0] + [int(np.searchsorted(excl, tot * r / n_parts, side="left")) for r in range(1, n_parts)]
    starts = [min(s, len(w)) for s in starts]
    return [(starts[r], starts[r + 1] if r + 1 < n_parts else len(w)) for r in range(n_parts)]


def bas_sample(conditional, n_orbitals: int, n_up: int, n_dn: int, n_samples: int, seed: int, device,
               n_parts: int = 1, part: int = 0, n_u_star: int | None = None, stream=None):
    """Unique samples (keys int64 [m, 2], counts int64 [m], on `device`, keys
    ascending) of n_samples draws from the autoregressive model `conditional`.
    n_parts > 1: this rank's share of the parallel BAS (see module doc);
    n_u_star defaults to the paper's 16384 * n_orbitals."""
    import torch
    keys = torch.zeros((1, 2), dtype=torch.int64, device=device)
    counts = torch.full((1,), int(n_samples), dtype=torch.int64, device=device)
    star = 16384 * n_orbitals if n_u_star is None else int(n_u_star)
    cut = n_parts <= 1
    widths = []
    for orbital in range(n_orbitals - 1, -1, -1):
        probs = conditional(keys, orbital).to(torch.float64).contiguous()
        keys, counts = nnqs.nnqs_bas_layer(keys, counts, probs, orbital, n_orbitals, n_up, n_dn, seed,
                                           stream=stream)
        widths.append(int(keys.shape[0]))
        if not cut and keys.shape[0] > star:
            b, e = partition(counts.cpu().numpy(), n_parts)[part]
            keys, counts = keys[b:e].contiguous(), counts[b:e].contiguous()
            cut = True
    return keys, counts, widths
