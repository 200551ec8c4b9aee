"""One warm nnqs_table_prepare + the Eq. (6) reduce kernels on C5 (the workload for the
ncu DRAM capture of the prepare / reduce kernels).  Dev tool."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2306_16705_b200 import nnqs  # noqa: E402
from synth import configs as C  # noqa: E402

dev = torch.device("cuda", 0)
m = C.molecule(5)
st = C.sample_table(5, "full")
ham = nnqs.nnqs_ham_compress(m.h1, m.h2, m.n_qubits, m.e_core, device=0)
keys = torch.from_numpy(st.keys.view(np.int64)).to(dev)
lp = torch.from_numpy(st.logpsi).to(dev)
cnt = torch.from_numpy(st.counts).to(dev)
nnqs.nnqs_table_prepare(ham, 0, keys, lp).close()          # warm the pool (not profiled: -k below)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("prepare")
tab = nnqs.nnqs_table_prepare(ham, 0, keys, lp)
torch.cuda.nvtx.range_pop()
el = torch.empty((len(st.keys), 2), dtype=torch.float64, device=dev)
nnqs.nnqs_local_energy(ham, tab, 0, n_rows=len(st.keys), eloc_out=el)
part = nnqs.nnqs_energy_chunk_partials(el, cnt)
m1 = nnqs.nnqs_energy_combine(part, 1)
p2 = nnqs.nnqs_energy_chunk_partials(el, cnt, mean_dev=m1[:2].contiguous())
nnqs.nnqs_energy_combine(p2, 2)
torch.cuda.synchronize()
print("done")
