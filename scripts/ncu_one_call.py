"""One nnqs_local_energy call on a config (default C5, all table rows) -- the
workload bench.py profiles with ncu (in the same run) for the per-launch DRAM
traffic and ALU-pipe utilisation of the row kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2306_16705_b200 import nnqs  # noqa: E402
from synth import configs as C  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 5
dev = torch.device("cuda", 0)
m = C.molecule(c)
st = C.sample_table(c)
ham = nnqs.nnqs_ham_compress(m.h1, m.h2, m.n_qubits, m.e_core, device=0)
keys = torch.from_numpy(st.keys.view(np.int64)).to(dev)
lp = torch.from_numpy(st.logpsi).to(dev)
tab = nnqs.nnqs_table_prepare(ham, 0, keys, lp)
out = nnqs.nnqs_local_energy(ham, tab, 0, n_rows=len(st.keys))
torch.cuda.synchronize()
print("one call done", float(out[0, 0]))
