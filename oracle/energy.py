"""Count-weighted energy estimate, Eq. (6) over unique
samples with weights -- TEST INFRASTRUCTURE ONLY.

  mean = sum_u w_u E_loc(u) / W,   var = sum_u w_u |E_loc(u) - mean|^2 / W,
  W = sum_u w_u  (population variance, two passes; reading R13)
Sums are exact-rounded with math.fsum.
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
