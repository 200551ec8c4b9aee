"""Count-weighted energy estimate, Eq. (6) over unique
samples with weights -- TEST INFRASTRUCTURE ONLY.

  mean = sum_u w_u E_loc(u) / W,   var = sum_u w_u |E_loc(u) - mean|^2 / W,
  W = sum_u w_u  (population variance, two passes; reading R13)
Sums are exact-rounded with math.fsum.

grad_weights: the Eq. (7) weights,
  a_u = 2 w_u Re(E_loc(u) - mean) / W,  b_u = 2 w_u Im(E_loc(u) - mean) / W,
the coefficients of grad ln|Psi(x_u)| and grad phi(x_u) in
2 Re E_p[(E_loc - E) grad ln Psi*] with ln Psi* = ln|Psi| - i phi.
"""
from __future__ import annotations

import math

import numpy as np


def energy(eloc, counts):
    eloc = np.asarray(eloc, dtype=np.complex128)
    w = np.asarray(counts, dtype=np.int64)
    W = int(w.sum())
    if W == 0:
        raise ValueError("sum of counts is zero")
    mre = math.fsum((float(wi) * e.real for wi, e in zip(w, eloc))) / W
    mim = math.fsum((float(wi) * e.imag for wi, e in zip(w, eloc))) / W
    var = math.fsum(float(wi) * ((e.real - mre) ** 2 + (e.imag - mim) ** 2) for wi, e in zip(w, eloc)) / W
    return complex(mre, mim), var, W


def grad_weights(eloc, counts):
    eloc = np.asarray(eloc, dtype=np.complex128)
    w = np.asarray(counts, dtype=np.int64)
    mean, _, W = energy(eloc, counts)
    a = np.array([2.0 * float(wi) * (e.real - mean.real) / W for wi, e in zip(w, eloc)])
    b = np.array([2.0 * float(wi) * (e.imag - mean.imag) / W for wi, e in zip(w, eloc)])
    return a, b
