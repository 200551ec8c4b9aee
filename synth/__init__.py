"""Seeded synthetic workloads (integrals, sample sets, log-psi) for the
NNQS local-energy hot path.  Input generators only: no arithmetic of the
method lives here, so both ``oracle/`` and the CUDA path may import it."""
