"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
the whole C-ABI path on C2-C4 and a 4096-row C5 slice -- table prepare (order
check, psi_hat, hash, alpha/beta index, deletion multimap), both local-energy
algorithms (the literal loop in its bit-sliced and staged kernels), the fused Eq. (6) chunk partials, the reduce, the Eq. (7) weights
and the production-path hit log.  Exits non-zero on any API error; the
sanitizer's own exit code reports device errors.

  compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_run.py [--c5]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2306_16705_b200 import nnqs  # noqa: E402
from synth import configs as C  # noqa: E402


def t(a, dev):
    a = np.ascontiguousarray(a)
    return torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a).to(dev)


def run(c, n_rows=None, variant="full", **opt):
    dev = torch.device("cuda", 0)
    m = C.molecule(c)
    st = C.sample_table(c, variant)
    ham = nnqs.nnqs_ham_compress(m.h1, m.h2, m.n_qubits, m.e_core, device=0)
    tab = nnqs.nnqs_table_prepare(ham, 0, t(st.keys, dev), t(st.logpsi, dev), **opt)
    n = len(st.keys) if n_rows is None else n_rows
    r0 = 0 if n_rows is None else len(st.keys) // 2 // 1024 * 1024
    cnt = t(st.counts[r0:r0 + n], dev)
    part = torch.empty(((n + 1023) // 1024, 3), dtype=torch.float64, device=dev)
    stats = torch.zeros(4, dtype=torch.int64, device=dev)
    el = nnqs.nnqs_local_energy(ham, tab, r0, n_rows=n, counts=cnt, partials_out=part, stats_out=stats)
    nnqs.nnqs_energy_reduce(el, cnt)
    m1 = nnqs.nnqs_energy_combine(part, 1)
    nnqs.nnqs_grad_weights(el, cnt, m1)
    nnqs.nnqs_coupled_debug_rows(ham, tab, r0, min(n, 64), max_pairs=1 << 20)
    if c < 5:   # literal loop: bit-sliced (default) and staged kernels
        nnqs.nnqs_table_set_algorithm(tab, nnqs.ALGO_LITERAL)
        nnqs.nnqs_local_energy(ham, tab, r0, n_rows=n, counts=cnt, partials_out=part)
        nnqs.nnqs_local_energy(ham, tab, rows=t(st.keys[:64], dev), row_logpsi=t(st.logpsi[:64], dev))
        tl = nnqs.nnqs_table_prepare(ham, 0, t(st.keys, dev), t(st.logpsi, dev), algorithm=nnqs.ALGO_LITERAL,
                                     literal_kernel=1)
        nnqs.nnqs_local_energy(ham, tl, r0, n_rows=n)
        tl.close()
    else:       # the bit-sliced literal kernel on 40 explicit C5 rows (2.06M groups each)
        nnqs.nnqs_table_set_algorithm(tab, nnqs.ALGO_LITERAL)
        nnqs.nnqs_local_energy(ham, tab, rows=t(st.keys[:40], dev), row_logpsi=t(st.logpsi[:40], dev))
    nnqs.nnqs_chunk_work(tab, with_floor=True)
    torch.cuda.synchronize()
    tab.close()
    ham.close()
    print(f"C{c}/{variant} rows={n} ok", flush=True)


def run_bas():
    """BAS layers (csrc/bas.cu) on a synthetic 20-orbital model, 10^5 samples (~10^5 leaves)."""
    import numpy as np
    dev = torch.device("cuda", 0)
    keys = torch.zeros((1, 2), dtype=torch.int64, device=dev)
    counts = torch.full((1,), 10**5, dtype=torch.int64, device=dev)
    rng = np.random.default_rng(3)
    for orbital in range(19, -1, -1):
        probs = torch.from_numpy(rng.random((keys.shape[0], 4)) + 0.01).to(dev)
        keys, counts = nnqs.nnqs_bas_layer(keys, counts, probs, orbital, 20, 7, 7, 11)
    torch.cuda.synchronize()
    print(f"BAS 20 orbitals: {keys.shape[0]} unique samples ok", flush=True)


if __name__ == "__main__":
    run(2, variant="half")
    run(3)
    run(4)
    run(4, thr_single=3, thr_double=6, thr_rowheavy=40)   # multimap, probes and the join on C4
    run_bas()
    if "--c5" in sys.argv:
        run(5, n_rows=4096)
    print("sanitize workload done")
