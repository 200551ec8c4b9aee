"""CPU oracle for the NNQS local-energy hot path -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously correct implementations of what the path computes,
written from PAPER.md (arXiv 2306.16705) and sharing no code with the CUDA
library ``paper_2306_16705_b200``:

  oracle/eloc_oracle.c  H_{xx'} by applying every term of Eq. (9) with the
                        Jordan-Wigner sign rules; E_loc of Eq. (4) in long
                        double (sample-aware, or exact mode)
  oracle/rows.py        ctypes wrappers around it
  oracle/dense.py       dense H (fermionic rows; independent Kronecker
                        build), sector ground state, Walsh-Hadamard Pauli
                        recovery of the grouped table (Fig. 6(c))
  oracle/jw.py          symbolic Jordan-Wigner (Pauli strings with Y) and the
                        fused coefficients of Algorithm 1
  oracle/counts.py      closed-form group / string counts from irrep labels
  oracle/energy.py      count-weighted mean and variance, Eq. (6)

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import anything under ``oracle/``.
"""
