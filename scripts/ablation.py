"""Fig. 10-style ladder re-measured on one B200:
local-energy time for one call over every row of a sample table, for
  cpu_oracle  -- the oracle (plain term-by-term Eq. 9, sample-aware with a
                 bisection lookup, all host cores): the CPU reference point
  gpu_literal_plain / _staged / _bitsliced -- Algorithm 2 on the GPU: every (row,
                 flip group) pair, sector test, GF(2)-hash lookup of x' (sample-aware +
                 fused + LUT + GPU): one row per thread reading the group table from
                 global memory / group tiles staged in shared memory by bulk copies /
                 32 rows x 32 groups per bit-sliced sector test (bit-identical results)
  gpu_structured -- the alpha/beta-factorised enumeration of the same pairs
Workloads: C4 (N2-shaped, N = 20, the whole 14,400-entry sector as the table;
the paper's C2 run is N = 20 with N_u = 10,553), C3 (H2O-shaped, N = 14) and the
first 2048 rows of C5 (N = 120, 10^6-entry table; the oracle on those rows only).
Writes one JSON object to stdout.  Dev/evidence tool, run on the GPU box.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__ as g  # noqa: E402

g.build()
from oracle import rows as R  # noqa: E402
from paper_2306_16705_b200 import nnqs  # noqa: E402
from synth import configs as C  # noqa: E402


def gpu_time(ham, tab, n, algo, reps=20):
    nnqs.nnqs_table_set_algorithm(tab, algo)
    reps = reps if n * ham.info()["n_groups"] < 10 ** 10 else 2
    out = torch.empty((n, 2), dtype=torch.float64, device="cuda")
    for _ in range(3):
        nnqs.nnqs_local_energy(ham, tab, 0, n_rows=n, eloc_out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        nnqs.nnqs_local_energy(ham, tab, 0, n_rows=n, eloc_out=out)
    e1.record()
    e1.synchronize()
    nnqs.nnqs_table_set_algorithm(tab, nnqs.ALGO_AUTO)
    return e0.elapsed_time(e1) / reps / 1e3, out.cpu().numpy()


def main():
    res = {"what": "local energy over every table row, one call", "device": torch.cuda.get_device_name(0),
           "oracle_threads": R.num_threads(), "workloads": []}
    for c in (3, 4, 5):
        m = C.molecule(c)
        st = C.sample_table(c, "full") if c < 5 else C.sample_table(5)
        n = len(st.keys) if c < 5 else 2048
        ham = nnqs.nnqs_ham_compress(m.h1, m.h2, m.n_qubits, m.e_core, device=0)
        keys_d = torch.from_numpy(st.keys.view(np.int64)).cuda()
        lp_d = torch.from_numpy(st.logpsi).cuda()
        t0 = time.perf_counter()
        ref = R.eloc(m.h1, m.h2, m.e_core, st.keys[:n], st.logpsi[:n], keys=st.keys, logpsi=st.logpsi)
        t_cpu = time.perf_counter() - t0
        secs, els = {"cpu_oracle": t_cpu}, {}
        for name, lk in (("gpu_literal_plain", 2), ("gpu_literal_staged", 1), ("gpu_literal_bitsliced", 0)):
            tab = nnqs.nnqs_table_prepare(ham, 0, keys_d, lp_d, literal_kernel=lk)
            secs[name], els[name] = gpu_time(ham, tab, n, nnqs.ALGO_LITERAL)
            tab.close()
        tab = nnqs.nnqs_table_prepare(ham, 0, keys_d, lp_d)
        secs["gpu_structured"], els["gpu_structured"] = gpu_time(ham, tab, n, nnqs.ALGO_AUTO)
        tab.close()
        scale = np.max(np.abs(ref))
        res["workloads"].append({
            "config": f"C{c}: {m.name}, N={m.n_qubits}, N_u={len(st.keys)}, rows={n}, K'={ham.info()['n_groups']}, "
                      f"N_h={ham.info()['n_terms']}",
            "seconds": secs,
            "speedup_vs_cpu_oracle": {k: t_cpu / v for k, v in secs.items() if k != "cpu_oracle"},
            "literal_kernels_bit_identical": all(els[k].tobytes() == els["gpu_literal_plain"].tobytes()
                                                 for k in els if k.startswith("gpu_literal")),
            "max_abs_diff_vs_oracle_over_max_abs": {
                k: float(np.max(np.abs(v[:, 0] + 1j * v[:, 1] - ref)) / scale) for k, v in els.items()},
        })
    print(json.dumps(res))


if __name__ == "__main__":
    main()
