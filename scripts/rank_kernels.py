"""Per-kernel device times (torch.profiler / CUPTI) of the local-energy call on rank r's slice
at P ranks, C5 (dev tool: where does a rank's time go?).  Usage: rank_kernels.py P r [r ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import __graft_entry__ as g

g.build()
from paper_2306_16705_b200 import distributed as D
from paper_2306_16705_b200 import nnqs
from synth import configs as C

P = int(sys.argv[1])
ranks = [int(a) for a in sys.argv[2:]] or list(range(P))
dev = torch.device("cuda", 0)
m = C.molecule(5)
st = C.sample_table(5, "full")
n = len(st.keys)
ham = nnqs.nnqs_ham_compress(m.h1, m.h2, m.n_qubits, m.e_core, device=0)
keys = torch.from_numpy(st.keys.view(np.int64)).to(dev)
lp = torch.from_numpy(st.logpsi).to(dev)
tab = nnqs.nnqs_table_prepare(ham, 0, keys, lp)
work = nnqs.nnqs_chunk_work(tab)
sl = os.environ.get("RANGES")   # explicit "b:e,b:e" row ranges instead of rank slices
items = [tuple(int(v) for v in x.split(":")) for x in sl.split(",")] if sl else ranks
for r in items:
    if sl:
        b, e = r
    else:
        b, e = D.balanced_bounds(work, P, r, n_rows=n) if os.environ.get("SPLIT", "count") == "work" else D.shard_bounds(n, P, r)
    out = torch.empty((e - b, 2), dtype=torch.float64, device=dev)
    nnqs.nnqs_local_energy(ham, tab, b, n_rows=e - b, eloc_out=out)
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        nnqs.nnqs_local_energy(ham, tab, b, n_rows=e - b, eloc_out=out)
        e1.record()
        e1.synchronize()
    tot = {}
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            k = ev.name.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0][:40]
            tot[k] = tot.get(k, 0.0) + ev.device_time / 1e3
    top = sorted(tot.items(), key=lambda kv: -kv[1])[:8]
    print(f"P={P} r={r} rows=[{b},{e}) call={e0.elapsed_time(e1):.2f} ms  "
          + "  ".join(f"{k}={v:.2f}" for k, v in top), flush=True)
