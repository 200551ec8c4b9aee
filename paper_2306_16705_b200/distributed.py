"""Multi-GPU orchestration of the path with torch.distributed (NCCL on B200).

The paper's data-centric scheme (Sec. 3.2): each process
owns a batch of ~N_u/N_p unique samples; stage 2 all-gathers the samples
(MPI_Allgather, N_u N_p (ceil(N/8)+16) bytes), stage 3 evaluates the local
energies of the process's own batch against the replicated lookup table,
stage 4 reduces the energy (MPI_Allreduce, 16 N_p bytes).

Here: stage 2 is one NCCL all_gather_into_tensor of 32-byte records (key u64[2]
| log-psi f64[2]); stage 4 all-gathers per-chunk energy partials (3 f64 per
NNQS_REDUCE_CHUNK rows) and every rank combines them in global chunk order on
the device, so the energy is bit-identical for any number of GPUs as long as
row slices are chunk-aligned (shard_bounds).  This module only moves data;
all arithmetic runs in libnnqs kernels.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

REDUCE_CHUNK = 1024


def shard_bounds(n_rows: int, world: int, rank: int, chunk: int = REDUCE_CHUNK):
    """Contiguous, chunk-aligned slice [begin, end) of n_rows for this rank
    (the paper's ist / batch_size_cur_rank)."""
    n_chunks = (n_rows + chunk - 1) // chunk
    lo = (n_chunks * rank) // world
    hi = (n_chunks * (rank + 1)) // world
    return min(lo * chunk, n_rows), min(hi * chunk, n_rows)


def balanced_bounds(work, world: int, rank: int, chunk: int = REDUCE_CHUNK, n_rows: int | None = None,
                    floor=None):
    """Contiguous, chunk-aligned slice [begin, end) of the table rows for this rank
    with about equal estimated work (nnqs_chunk_work: one int64 per chunk): rank r
    starts at the first chunk whose work prefix reaches r/world of the total.  With
    `floor` (nnqs_chunk_work's per-chunk single-row latency floor) a slice costs
    max(its largest floor, its work) and the slices minimise the largest cost
    (bisection on the bound, then a greedy fill from the left).  Pure integer
    arithmetic on the replicated estimate, so every rank derives the same slices;
    chunk alignment keeps the energy bit-identical to 1 GPU."""
    w = [int(v) for v in work]
    n_chunks = len(w)
    n = n_chunks * chunk if n_rows is None else n_rows
    total = sum(w)
    # floors at most half a fair share never bind (floor + work/2 <= work): the plain split
    if floor is not None and n_chunks and 2 * world * max(int(v) for v in floor) > total:
        st = _floor_bounds(w, [int(v) for v in floor], world)
        return min(st[rank] * chunk, n), (min(st[rank + 1] * chunk, n) if rank + 1 < world else n)
    if total <= 0:
        return shard_bounds(n, world, rank, chunk)

    def start(r):
        if r <= 0:
            return 0
        if r >= world:
            return n_chunks
        target = total * r   # first c with world * prefix(c) >= total * r
        acc = 0
        for c in range(n_chunks):
            if acc * world >= target:
                return c
            acc += w[c]
        return n_chunks

    return min(start(rank) * chunk, n), min(start(rank + 1) * chunk, n)


def _slice_cost(acc: int, mf: int) -> int:
    """A slice's time estimate: its work, or its slowest row plus half its work."""
    return max(acc, mf + acc // 2)


def _reach(w, fl, bound):
    """e[c] = the largest e with cost(w[c:e], max fl[c:e]) <= bound (e = c if chunk c alone
    exceeds it), by two pointers with a sliding-window maximum (cost is monotone in
    the slice), and f[c] = the fewest slices covering chunks [c, n) under the bound."""
    from collections import deque
    n = len(w)
    e = [0] * n
    dq = deque()
    j, acc = 0, 0
    for c in range(n):
        if j < c:
            j, acc = c, 0
            dq.clear()
        while j < n:
            nmf = max(fl[dq[0]] if dq else 0, fl[j])
            if _slice_cost(acc + w[j], nmf) > bound:
                break
            acc += w[j]
            while dq and fl[dq[-1]] <= fl[j]:
                dq.pop()
            dq.append(j)
            j += 1
        e[c] = j
        if j > c:
            acc -= w[c]
            if dq and dq[0] == c:
                dq.popleft()
    inf = 1 << 62          # infeasible: some chunk alone exceeds the bound
    f = [0] * (n + 1)
    for c in range(n - 1, -1, -1):
        f[c] = inf if e[c] == c else min(inf, 1 + f[e[c]])
    return e, f


def _floor_bounds(w, fl, world):
    """Chunk starts of `world` contiguous slices minimising the largest slice cost
    max(work, floor + work/2): bisection on the bound with the exact min-slice count
    (_reach), then a fill that gives every rank about its fair share of the remaining
    work but stops early only where the rest still fits on the remaining ranks under
    the bound (so no slice, the last included, exceeds it)."""
    n_chunks, total = len(w), sum(w)
    lo, hi = 0, max(total, max(fl)) + total
    while lo < hi:
        mid = (lo + hi) // 2
        if _reach(w, fl, mid)[1][0] <= world:
            hi = mid
        else:
            lo = mid + 1
    e, f = _reach(w, fl, lo)
    st, c, rem = [0], 0, total
    for r in range(world - 1):
        R = world - r
        acc = 0
        while c < e[st[-1]] if st[-1] < n_chunks else False:
            nacc = acc + w[c]
            # fair share reached and the rest fits on the R - 1 other ranks: stop here
            if acc > 0 and nacc * R > rem + R - 1 and f[c] <= R - 1:
                break
            acc, c = nacc, c + 1
        rem -= acc
        st.append(c)
    st.append(n_chunks)
    return st


def all_gather_varlen(t: torch.Tensor, group=None, lens=None) -> torch.Tensor:
    """all_gather_into_tensor of per-rank tensors with different first
    dimensions: gather the lengths (unless every rank already knows them: `lens`,
    which saves a collective and a host sync), pad to the maximum, gather, strip."""
    world = dist.get_world_size(group)
    if lens is None:
        n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
        ns = torch.empty(world, dtype=torch.int64, device=t.device)
        dist.all_gather_into_tensor(ns, n, group=group)
        lens = [int(v) for v in ns.cpu()]
    lens = [int(v) for v in lens]
    assert lens[dist.get_rank(group)] == t.shape[0], "lens disagrees with this rank's tensor"
    m = max(lens)
    if t.shape[0] < m:
        pad = torch.zeros((m - t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        t = torch.cat([t, pad])
    out = torch.empty((world * m,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    dist.all_gather_into_tensor(out, t.contiguous(), group=group)
    if all(v == m for v in lens):
        return out
    return torch.cat([out[r * m: r * m + lens[r]] for r in range(world)])


def pack_records(keys: torch.Tensor, logpsi: torch.Tensor) -> torch.Tensor:
    """[m,2] int64 keys + [m,2] float64 log-psi -> [m,4] int64 records (32 B/sample)."""
    return torch.cat([keys.view(torch.int64), logpsi.view(torch.int64)], dim=1).contiguous()


def unpack_records(rec: torch.Tensor):
    keys = rec[:, :2].contiguous()
    logpsi = rec[:, 2:].contiguous().view(torch.float64)
    return keys, logpsi


def gather_samples(local_keys: torch.Tensor, local_logpsi: torch.Tensor, group=None, lens=None):
    """Stage 2: every rank receives every unique sample.  Shards
    are disjoint key ranges in rank order, so the concatenation stays sorted.
    lens: every rank's shard size, if known everywhere (no length exchange)."""
    rec = all_gather_varlen(pack_records(local_keys, local_logpsi), group, lens)
    return unpack_records(rec)


def gather_counts(local_counts: torch.Tensor, group=None, lens=None) -> torch.Tensor:
    """Sample multiplicities of every rank's shard, in rank order (needed when the
    evaluated row slice, balanced_bounds, differs from the owned sample shard)."""
    return all_gather_varlen(local_counts.reshape(-1, 1), group, lens).reshape(-1)


def distributed_energy(eloc_local: torch.Tensor, counts_local: torch.Tensor, group=None, stream=None, p1=None,
                       rows_per_rank=None):
    """Stage 4: count-weighted mean and variance (Eq. 6) over all
    ranks' rows.  p1: this rank's first-pass chunk partials if nnqs_local_energy
    already produced them (its fused epilogue).  rows_per_rank: every rank's row
    count, if known everywhere (saves the two length exchanges and host syncs).
    Returns a device f64[4] = (mean_re, mean_im, var, W)."""
    from . import nnqs
    if p1 is None:
        p1 = nnqs.nnqs_energy_chunk_partials(eloc_local, counts_local, stream=stream)
    clens = None if rows_per_rank is None else [(r + REDUCE_CHUNK - 1) // REDUCE_CHUNK for r in rows_per_rank]
    allp = all_gather_varlen(p1[: _n_chunks(eloc_local)], group, clens)
    m1 = nnqs.nnqs_energy_combine(allp, 1, stream=stream)
    p2 = nnqs.nnqs_energy_chunk_partials(eloc_local, counts_local, mean_dev=m1[:2].contiguous(), stream=stream)
    allp2 = all_gather_varlen(p2[: _n_chunks(eloc_local)], group, clens)
    m2 = nnqs.nnqs_energy_combine(allp2, 2, stream=stream)
    return torch.stack([m1[0], m1[1], m2[0], m1[2]])


def _n_chunks(t: torch.Tensor) -> int:
    return (t.shape[0] + REDUCE_CHUNK - 1) // REDUCE_CHUNK


def comm_bytes_paper(n_u: int, n_qubits: int, n_p: int, n_params: int) -> int:
    """The paper's per-iteration communication volume:
    N_u N_p (ceil(N/8) + 16) + 16 N_p + 8 M N_p bytes."""
    return n_u * n_p * (-(-n_qubits // 8) + 16) + 16 * n_p + 8 * n_params * n_p
