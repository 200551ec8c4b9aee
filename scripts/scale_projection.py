"""Per-rank step times of the P-GPU bench flow, measured one rank at a time on ONE B200.

Only one GPU is available to this run, so the multi-GPU step is measured piecewise: for
P in {1, 2, 4, 8} and every rank r < P, the work rank r does in bench.py's step (the
replicated nnqs_table_prepare over all N_u samples, then nnqs_local_energy on its
chunk-aligned slice (distributed.balanced_bounds on nnqs_chunk_work's
estimate, or distributed.shard_bounds by count), then the energy partials) is timed
with CUDA events on the launching stream, L2 flushed before each repetition, median of
`reps`.  T(P) = max over ranks + the stage-2 all-gather of N_u x 32 B over NVLink (a
bandwidth term, stated, not measured here).  Prints one JSON line (dev/evidence tool).
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import __graft_entry__ as g

g.build()
from paper_2306_16705_b200 import distributed as D
from paper_2306_16705_b200 import nnqs
from synth import configs as C

c = int(sys.argv[1]) if len(sys.argv) > 1 else 5
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
split = sys.argv[3] if len(sys.argv) > 3 else "work"   # "work" (with floors), "work_nofloor", "count"
NVLINK_GBS = 900.0          # per-direction NVLink 5 bandwidth per GPU (B200_PROFILING.md)
dev = torch.device("cuda", 0)
m = C.molecule(c)
st = C.sample_table(c, "full")
n = len(st.keys)
ham = nnqs.nnqs_ham_compress(m.h1, m.h2, m.n_qubits, m.e_core, device=0)
keys = torch.from_numpy(st.keys.view(np.int64)).to(dev)
lp = torch.from_numpy(st.logpsi).to(dev)
cnt = torch.from_numpy(st.counts).to(dev)
stream = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def ev():
    return torch.cuda.Event(enable_timing=True)


def rank_step(b, e):
    """(prepare ms, local-energy ms, step ms) of one rank's step, median of reps."""
    eloc = torch.empty((max(e - b, 1), 2), dtype=torch.float64, device=dev)
    out = []
    for i in range(reps + 1):
        flush.fill_(1)
        a0, a1, a2, a3 = ev(), ev(), ev(), ev()
        a0.record(stream)
        tab = nnqs.nnqs_table_prepare(ham, 0, keys, lp, stream=stream)
        a1.record(stream)
        nnqs.nnqs_local_energy(ham, tab, b, n_rows=e - b, eloc_out=eloc[: e - b], stream=stream)
        a2.record(stream)
        part = nnqs.nnqs_energy_chunk_partials(eloc[: e - b], cnt[b:e], stream=stream)
        nnqs.nnqs_energy_combine(part, 1, stream=stream)
        a3.record(stream)
        a3.synchronize()
        tab.close()
        if i:   # first repetition is a warm-up
            out.append((a0.elapsed_time(a1), a1.elapsed_time(a2), a0.elapsed_time(a3)))
    return tuple(statistics.median(x[k] for x in out) for k in range(3))


tab0 = nnqs.nnqs_table_prepare(ham, 0, keys, lp, stream=stream)
work, floor = nnqs.nnqs_chunk_work(tab0, stream=stream, with_floor=True)
tab0.close()


def bounds(P, r):
    if split == "work":
        return D.balanced_bounds(work, P, r, n_rows=n, floor=floor)
    if split == "work_nofloor":
        return D.balanced_bounds(work, P, r, n_rows=n)
    return D.shard_bounds(n, P, r)


res = {"what": "per-rank step times of the P-GPU bench flow, each rank measured alone on one B200",
       "config": f"C{c}", "split": split, "n_unique": n, "reps": reps, "per_P": {}}
t1 = None
for P in (1, 2, 4, 8):
    ranks = []
    for r in range(P):
        b, e = bounds(P, r)
        pm, lm, sm = rank_step(b, e)
        ranks.append({"rank": r, "rows": e - b, "prepare_ms": round(pm, 3), "local_energy_ms": round(lm, 3),
                      "step_ms": round(sm, 3)})
    gather_ms = 0.0 if P == 1 else n * 32 * (P - 1) / P / (NVLINK_GBS * 1e9) * 1e3
    tmax = max(x["step_ms"] for x in ranks) + gather_ms
    if P == 1:
        t1 = tmax
    res["per_P"][P] = {"ranks": ranks, "allgather_ms_model": round(gather_ms, 3), "T_ms": round(tmax, 3),
                       "local_energies_per_s": n / tmax * 1e3, "efficiency": t1 / (P * tmax)}
    print(f"P={P} T={tmax:.2f} ms eff={t1 / (P * tmax):.3f} ranks="
          + " ".join(f"{x['prepare_ms']:.1f}+{x['local_energy_ms']:.1f}" for x in ranks), file=sys.stderr)
print(json.dumps(res))
