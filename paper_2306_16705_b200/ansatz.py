"""QiankunNet-shaped wave function ansatz (Fig. 2; hyper-parameters
P:440-441) -- the model side of the VMC iteration, in plain PyTorch (library GEMMs).

  psi(x) = |psi(x)| e^{i phi(x)}  (Eq. 11): a decoder-only transformer gives the
  autoregressive conditionals pi(x_i | x_<i) (Eq. 8) over the 4 states of one spatial
  orbital (two qubits per step, orbitals n-1 ... 0), |psi(x)|^2 = prod_i
  pi~(x_i | x_<i) with pi~ the Eq. (12)-masked, renormalised conditional (the same
  mask the sampler applies, R24); an MLP N x 512 x 512 x 1 on the +-1
  encoded configuration gives the phase.

Random-initialised weights (no trained checkpoints exist here); float64 throughout,
so that the probabilities handed to the sampler and the log psi handed to the
local-energy kernels are the model's exactly.  Keys use the sample-key layout of
include/nnqs.h (qubit 2p = spin-up orbital p, 2p+1 = spin-down).
"""
from __future__ import annotations

import math

import torch
from torch import nn

BOS = 4


def key_tokens(keys: torch.Tensor, n_orbitals: int, upto: int | None = None) -> torch.Tensor:
    """int64 keys [m, 2] -> tokens [m, L] for orbitals n-1, n-2, ... (L = upto or n):
    token = up bit + 2 * down bit of the orbital."""
    L = n_orbitals if upto is None else upto
    orb = torch.arange(n_orbitals - 1, n_orbitals - 1 - L, -1, device=keys.device)
    qa = 2 * orb
    word = (qa // 64).long()
    bit = (qa % 64).long()
    w = torch.where(word[None, :] == 0, keys[:, :1], keys[:, 1:2])
    up = (w >> bit[None, :]) & 1
    dn = (w >> (bit[None, :] + 1)) & 1
    return (up + 2 * dn).long()


class QiankunNet(nn.Module):
    def __init__(self, n_orbitals: int, n_up: int, n_dn: int, d_model: int = 16, n_heads: int = 4,
                 n_layers: int = 2, phase_hidden: int = 512, seed: int = 0):
        super().__init__()
        self.n, self.n_up, self.n_dn = n_orbitals, n_up, n_dn
        g = torch.Generator().manual_seed(seed)
        self.tok = nn.Embedding(5, d_model)
        self.pos = nn.Embedding(n_orbitals + 1, d_model)
        layer = nn.TransformerEncoderLayer(d_model, n_heads, dim_feedforward=4 * d_model, dropout=0.0,
                                           batch_first=True, norm_first=True)
        self.dec = nn.TransformerEncoder(layer, n_layers, enable_nested_tensor=False)
        self.head = nn.Linear(d_model, 4)
        N = 2 * n_orbitals
        self.phase = nn.Sequential(nn.Linear(N, phase_hidden), nn.Tanh(), nn.Linear(phase_hidden, phase_hidden),
                                   nn.Tanh(), nn.Linear(phase_hidden, 1))
        with torch.no_grad():                         # deterministic init from `seed`
            for name, p in self.named_parameters():
                if p.dim() > 1:
                    bound = math.sqrt(6.0 / (p.shape[0] + p.shape[1]))
                    p.copy_(torch.rand(p.shape, generator=g, dtype=torch.float64) * 2 * bound - bound)
                elif "norm" in name and name.endswith("weight"):
                    p.fill_(1.0)
                else:
                    p.zero_()
        self.double()

    def _logits(self, tokens: torch.Tensor) -> torch.Tensor:
        """tokens [m, L] -> logits [m, L + 1, 4]: position l predicts the token of
        orbital n-1-l from the BOS token and the first l tokens (causal)."""
        m, L = tokens.shape
        seq = torch.cat([torch.full((m, 1), BOS, dtype=torch.long, device=tokens.device), tokens], dim=1)
        pos = torch.arange(L + 1, device=tokens.device)
        h = self.tok(seq) + self.pos(pos)[None]
        mask = torch.triu(torch.full((L + 1, L + 1), float("-inf"), device=tokens.device, dtype=h.dtype), 1)
        return self.head(self.dec(h, mask=mask))

    def conditionals(self, keys: torch.Tensor, orbital: int) -> torch.Tensor:
        """pi(x_orbital | orbitals above it) for every prefix key [m, 2] -> [m, 4]
        (unmasked; the sampler applies Eq. 12)."""
        L = self.n - 1 - orbital
        with torch.no_grad():
            lg = self._logits(key_tokens(keys, self.n, L))[:, L]
            return torch.softmax(lg, dim=-1)

    def _masked_logp(self, tokens: torch.Tensor) -> torch.Tensor:
        """log pi~ of every step of full configurations [m, n] -> [m]."""
        lg = self._logits(tokens[:, :-1])                       # [m, n, 4]
        logp = torch.log_softmax(lg, dim=-1)
        up = (tokens & 1)
        dn = (tokens >> 1)
        na = torch.cumsum(up, 1) - up                            # electrons above each orbital
        nb = torch.cumsum(dn, 1) - dn
        o = torch.arange(4, device=tokens.device)
        rem = torch.arange(self.n - 1, -1, -1, device=tokens.device)   # orbitals left below: i
        a2 = na[:, :, None] + (o & 1)[None, None]
        b2 = nb[:, :, None] + (o >> 1)[None, None]
        ok = (a2 <= self.n_up) & (b2 <= self.n_dn) & (a2 + rem[None, :, None] >= self.n_up) & \
             (b2 + rem[None, :, None] >= self.n_dn)
        masked = torch.where(ok, logp, torch.full_like(logp, float("-inf")))
        norm = torch.logsumexp(masked, dim=-1)
        step = torch.gather(masked, 2, tokens[:, :, None])[:, :, 0] - norm
        return step.sum(dim=1)

    def log_psi(self, keys: torch.Tensor) -> torch.Tensor:
        """Complex log psi as float64 [m, 2] = (Re, Im) -- differentiable."""
        tokens = key_tokens(keys, self.n)
        re = 0.5 * self._masked_logp(tokens)
        q = torch.arange(2 * self.n, device=keys.device)
        w = torch.where((q // 64)[None, :] == 0, keys[:, :1], keys[:, 1:2])
        spins = (((w >> (q % 64)[None, :]) & 1) * 2 - 1).to(torch.float64)
        im = self.phase(spins)[:, 0]
        return torch.stack([re, im], dim=1)


def learning_rate(i: int, d_model: int = 16, warmup: int = 4000) -> float:
    """Eq. (13): alpha_i = d_model^-1/2 min(i^-1/2, i S_w^-3/2)."""
    i = max(1, i)
    return d_model ** -0.5 * min(i ** -0.5, i * warmup ** -1.5)
