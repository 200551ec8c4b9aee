"""Per-kernel device times (CUPTI) of one nnqs_table_prepare on C5 and its event-timed
duration, to separate GPU-busy time from gaps (host syncs, allocations).  Dev tool."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import __graft_entry__ as g

g.build()
from paper_2306_16705_b200 import nnqs
from synth import configs as C

dev = torch.device("cuda", 0)
m = C.molecule(5)
st = C.sample_table(5, "full")
ham = nnqs.nnqs_ham_compress(m.h1, m.h2, m.n_qubits, m.e_core, device=0)
keys = torch.from_numpy(st.keys.view(np.int64)).to(dev)
lp = torch.from_numpy(st.logpsi).to(dev)
for _ in range(2):
    nnqs.nnqs_table_prepare(ham, 0, keys, lp).close()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    tab = nnqs.nnqs_table_prepare(ham, 0, keys, lp)
    e1.record()
    e1.synchronize()
tot, cnt = {}, {}
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        k = ev.name.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0][:48]
        if "cub::" in k:
            k = "cub " + ("Onesweep" if "Onesweep" in ev.name else "Histogram" if "Histogram" in ev.name else
                          "Scan" if "Scan" in ev.name else "other")
        tot[k] = tot.get(k, 0.0) + ev.device_time / 1e3
        cnt[k] = cnt.get(k, 0) + 1
busy = sum(tot.values())
print(f"prepare elapsed {e0.elapsed_time(e1):.3f} ms, device-busy sum {busy:.3f} ms")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"  {v:8.3f} ms  x{cnt[k]:3d}  {k}")
