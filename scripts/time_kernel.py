"""Quick device timing of nnqs_local_energy on a config (dev tool)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__ as g
g.build()
from paper_2306_16705_b200 import nnqs
from synth import configs as C

c = int(sys.argv[1]) if len(sys.argv) > 1 else 5
nrows = int(sys.argv[2]) if len(sys.argv) > 2 else 0
algo = int(sys.argv[3]) if len(sys.argv) > 3 else 0
lk = int(sys.argv[4]) if len(sys.argv) > 4 else 0      # literal kernel: 0 bit-sliced, 1 staged, 2 plain
dev = torch.device("cuda", 0)
m = C.molecule(c); st = C.sample_table(c)
t = time.time(); ham = nnqs.nnqs_ham_compress(m.h1, m.h2, m.n_qubits, m.e_core, device=0); print("compress", time.time() - t, ham.info())
keys = torch.from_numpy(st.keys.view(np.int64)).to(dev); lp = torch.from_numpy(st.logpsi).to(dev)
tab = nnqs.nnqs_table_prepare(ham, 0, keys, lp, literal_kernel=lk)
nnqs.nnqs_table_set_algorithm(tab, algo)
n = nrows or len(st.keys)
out = torch.empty((n, 2), dtype=torch.float64, device=dev)
stats = torch.zeros(4, dtype=torch.int64, device=dev)
for it in range(3):
    stats.zero_()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); nnqs.nnqs_local_energy(ham, tab, 0, n_rows=n, eloc_out=out, stats_out=stats); e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1)
    s = stats.cpu().numpy()
    print(f"algo={algo} lk={lk} C{c} rows={n} K={ham.info()['n_groups']} {ms:.3f} ms  rows/s={n/ms*1e3:.3e} pairs/s={n*ham.info()['n_groups']/ms*1e3:.3e} stats={s} hits/row={s[2]/n:.1f}")
e0.record(); tab2 = nnqs.nnqs_table_prepare(ham, 0, keys, lp); e1.record(); e1.synchronize(); print("table_prepare ms", e0.elapsed_time(e1))
if os.environ.get("NNQS_PRINT_PROF"):
    nnqs.nnqs_debug_counters(True)
    nnqs.nnqs_local_energy(ham, tab, 0, n_rows=n, eloc_out=out)
    pc = nnqs.nnqs_debug_counters(True).astype(float)
    names = ["diag", "phase_i", "phase_ii", "iii_total", "iii_heavy", "flush", "setup", "row_total", "ss_heavy", "ss_flush"]
    tot = pc[7] or 1.0
    print("section cycles (share of row total):", {k: round(v / tot, 3) for k, v in zip(names, pc[:10])})
