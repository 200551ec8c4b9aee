"""Every-row C5 oracle fixture (SURVEY.md Sec. 8(c) reading 20): E_loc of all
10^6 table rows of the 120-qubit synthetic config, their R14 tolerance scales,
and the count-weighted energy / variance (Eq. 4; Eq. 6,
PAPER.md:146-149).

Calls only oracle/ (the CPU definition) and synth/ (the seeded inputs) -- never
the CUDA library -- so the stored values are the oracle's.  Resumable: rows are
evaluated in 4096-row parts (written to tests/golden/c5_parts/, git-ignored),
in a seeded order so that a partial run is a uniform sample; `--merge` writes
tests/golden/c5_eloc.npz with a SHA-256 of the inputs it was computed from.

  nice -n 19 python scripts/c5_oracle_fixture.py [--threads T] [--merge]
"""
from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import energy as OE  # noqa: E402
from oracle import rows as OR  # noqa: E402
from synth import configs as C  # noqa: E402

PART = 4096
PARTS_DIR = os.path.join(ROOT, "tests", "golden", "c5_parts")
OUT = os.path.join(ROOT, "tests", "golden", "c5_eloc.npz")


def input_digest(st) -> str:
    h = hashlib.sha256()
    for a in (st.keys, st.counts, st.logpsi):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def part_order(n_parts: int) -> np.ndarray:
    return np.random.default_rng(705).permutation(n_parts)


def run(threads: int, max_parts: int, reverse: bool = False, parts_dir: str = PARTS_DIR) -> None:
    mol = C.molecule(5)
    st = C.sample_table(5)
    n = len(st.keys)
    os.makedirs(parts_dir, exist_ok=True)
    dig = input_digest(st)
    n_parts = (n + PART - 1) // PART
    done = 0
    order = part_order(n_parts)
    for p in (order[::-1] if reverse else order):   # two workers: one from each end
        path = os.path.join(parts_dir, f"part_{p:04d}.npz")
        if os.path.exists(path) or os.path.exists(os.path.join(PARTS_DIR, f"part_{p:04d}.npz")):
            continue
        if done >= max_parts:
            break
        r0, r1 = p * PART, min(n, (p + 1) * PART)
        t0 = time.time()
        e, s = OR.eloc(mol.h1, mol.h2, mol.e_core, st.keys[r0:r1], st.logpsi[r0:r1], keys=st.keys,
                       logpsi=st.logpsi, n_threads=threads, with_scale=True)
        tmp = path + ".tmp.npz"
        np.savez(tmp, r0=r0, r1=r1, re=e.real, im=e.imag, scale=s, digest=dig)
        os.replace(tmp, path)
        done += 1
        have = len([f for f in os.listdir(parts_dir) if f.startswith("part_") and f.endswith(".npz")])
        print(f"part {p} rows [{r0},{r1}) {time.time() - t0:.1f}s  ({have}/{n_parts})", flush=True)


def merge() -> None:
    st = C.sample_table(5)
    n = len(st.keys)
    dig = input_digest(st)
    re = np.full(n, np.nan)
    im = np.full(n, np.nan)
    sc = np.full(n, np.nan)
    have = np.zeros(n, dtype=bool)
    for f in sorted(os.listdir(PARTS_DIR)):
        if not (f.startswith("part_") and f.endswith(".npz")) or ".tmp" in f:
            continue
        z = np.load(os.path.join(PARTS_DIR, f))
        assert str(z["digest"]) == dig, f"{f} was computed from other inputs"
        r0, r1 = int(z["r0"]), int(z["r1"])
        re[r0:r1], im[r0:r1], sc[r0:r1] = z["re"], z["im"], z["scale"]
        have[r0:r1] = True
    complete = bool(have.all())
    extra = {}
    if complete:
        mean, var, W = OE.energy(re + 1j * im, st.counts)
        extra = dict(mean_re=mean.real, mean_im=mean.imag, var=var, W=W,
                     energy_scale=float(np.sum(st.counts * np.abs(re + 1j * im)) / W),
                     max_abs=float(np.max(np.abs(re + 1j * im))))
    np.savez_compressed(OUT, digest=dig, complete=complete, have=have, re=re, im=im, scale=sc, **extra)
    print(f"wrote {OUT}: {int(have.sum())}/{n} rows, complete={complete}", {k: v for k, v in extra.items()})


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--max-parts", type=int, default=1 << 30)
    ap.add_argument("--merge", action="store_true")
    ap.add_argument("--reverse", action="store_true", help="walk the part order from its end (a second worker)")
    ap.add_argument("--parts-dir", default=PARTS_DIR, help="where new parts go (merge reads tests/golden/c5_parts)")
    a = ap.parse_args()
    if a.merge:
        merge()
    else:
        run(a.threads, a.max_parts, a.reverse, a.parts_dir)
