"""One iteration of the data-centric VMC loop, stages 1-6 of PAPER.md:251 (Sec. 3.2,
Fig. 4), around the local-energy path:

  1) batch autoregressive sampling, parallel over ranks (sampler.bas_sample, the
     nnqs_bas_layer kernel);  2) all-gather of the unique samples and
     their log psi (NCCL);  3) local energies of the rank's own samples
     against the replicated table (nnqs_table_prepare + nnqs_local_energy);
  4) count-weighted energy (Eq. 6) combined over ranks;  5) backward: the Eq. (7)
     estimator as the gradient of S = sum_u a_u Re ln psi_u + b_u Im ln psi_u with
     (a_u, b_u) from nnqs_grad_weights (torch autograd through the ansatz);
  6) all-reduce of the gradients and the AdamW step with the Eq. (13) schedule.

Every rank keeps its own samples throughout ("data-centric"); the model is
replicated.  world == 1 runs the same code without collectives.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import distributed as D
from . import nnqs
from .ansatz import QiankunNet, learning_rate
from .sampler import bas_sample


class VMC:
    def __init__(self, ham: nnqs.Hamiltonian, model: QiankunNet, n_samples: int, seed: int = 0, group=None,
                 n_u_star: int | None = None, lr: float | None = None):
        """lr None: the paper's schedule, Eq. (13); a number: constant learning rate."""
        self.ham, self.model, self.n_samples, self.seed = ham, model, int(n_samples), int(seed)
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if self.world > 1 else 0
        self.n_u_star = n_u_star
        self.it = 0
        d_model = model.tok.embedding_dim
        self.opt = torch.optim.AdamW(model.parameters(), lr=1.0 if lr is None else lr)
        sched = (lambda i: learning_rate(i + 1, d_model)) if lr is None else (lambda i: 1.0)
        self.sched = torch.optim.lr_scheduler.LambdaLR(self.opt, sched)

    def step(self):
        """One VMC iteration; returns a dict with the energy (mean, var, W) and sizes."""
        m = self.model
        dev = next(m.parameters()).device
        seed = self.seed * 1000003 + self.it
        # 1) sampling (this rank's share)
        keys, counts, widths = bas_sample(m.conditionals, m.n, m.n_up, m.n_dn, self.n_samples, seed, dev,
                                          n_parts=self.world, part=self.rank, n_u_star=self.n_u_star)
        lp = m.log_psi(keys)                                  # differentiable
        lpd = lp.detach().contiguous()
        # 2) every rank gets every unique sample (shards are contiguous key ranges)
        if self.world > 1:
            gk, gl = D.gather_samples(keys, lpd, self.group)
            n_before = D.all_gather_varlen(torch.tensor([[keys.shape[0]]], device=dev), self.group)[:, 0]
            row0 = int(n_before[: self.rank].sum())
        else:
            gk, gl, row0 = keys, lpd, 0
        # 3) local energies of this rank's samples
        tab = nnqs.nnqs_table_prepare(self.ham, 0, gk, gl)
        eloc = nnqs.nnqs_local_energy(self.ham, tab, row0, n_rows=keys.shape[0])
        tab.close()
        # 4) energy over all ranks (Eq. 6)
        if self.world > 1:
            en = D.distributed_energy(eloc, counts, self.group)
        else:
            part = nnqs.nnqs_energy_chunk_partials(eloc, counts)
            m1 = nnqs.nnqs_energy_combine(part, 1)
            p2 = nnqs.nnqs_energy_chunk_partials(eloc, counts, mean_dev=m1[:2].contiguous())
            m2 = nnqs.nnqs_energy_combine(p2, 2)
            en = torch.stack([m1[0], m1[1], m2[0], m1[2]])
        # 5) Eq. (7): grad E = sum_u a_u grad Re ln psi_u + b_u grad Im ln psi_u
        ab = nnqs.nnqs_grad_weights(eloc, counts, torch.stack([en[0], en[1], en[3]]).contiguous())
        self.opt.zero_grad(set_to_none=True)
        surrogate = (ab[:, 0] * lp[:, 0] + ab[:, 1] * lp[:, 1]).sum()
        surrogate.backward()
        # 6) gradients summed over ranks (each rank's S covers its own samples)
        if self.world > 1:
            for p in m.parameters():
                if p.grad is not None:
                    dist.all_reduce(p.grad, group=self.group)
        self.opt.step()
        self.sched.step()
        self.it += 1
        e = en.cpu().numpy()
        return {"energy": complex(e[0], e[1]), "var": float(e[2]), "W": float(e[3]),
                "n_unique_local": int(keys.shape[0]), "widths": widths}
