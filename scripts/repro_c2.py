import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__ as g
g.build()
from paper_2306_16705_b200 import nnqs
from synth import configs as C
c = int(sys.argv[1]); variant = sys.argv[2] if len(sys.argv) > 2 else "full"
dev = torch.device("cuda", 0)
m = C.molecule(c); st = C.sample_table(c, variant)
ham = nnqs.nnqs_ham_compress(m.h1, m.h2, m.n_qubits, m.e_core, device=0)
tab = nnqs.nnqs_table_prepare(ham, 0, torch.from_numpy(st.keys.view(np.int64)).to(dev), torch.from_numpy(st.logpsi).to(dev))
torch.cuda.synchronize(); print("prepared")
el = nnqs.nnqs_local_energy(ham, tab, 0, n_rows=len(st.keys)); torch.cuda.synchronize(); print("ok", el[:2])
