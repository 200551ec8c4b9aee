"""The C-ABI library loads and exports every symbol include/nnqs.h declares
(CPU only: no compute calls that need a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "nnqs.h")


def declared_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(nnqs_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def lib_path():
    import __graft_entry__ as g
    g.build()
    from paper_2306_16705_b200 import nnqs
    return nnqs.LIB_PATH


def test_header_declares_the_north_star_calls():
    fns = declared_functions()
    for name in ("nnqs_ham_compress", "nnqs_local_energy", "nnqs_energy_reduce"):
        assert name in fns


def test_every_declared_symbol_is_exported(lib_path):
    lib = ctypes.CDLL(lib_path)
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    exported = set(l.split()[-1] for l in out.splitlines() if l.strip())
    for name in declared_functions():
        assert name in exported, name
        assert hasattr(lib, name)


def test_binding_covers_the_header(lib_path):
    from paper_2306_16705_b200 import nnqs
    assert set(declared_functions()) == set(nnqs.EXPORTED)
    assert "sm_100a" in nnqs.nnqs_version()


def test_library_is_sm100a(lib_path):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_only_errors_without_gpu(lib_path):
    """Argument validation runs on the host and reports through nnqs_last_error."""
    import numpy as np
    from paper_2306_16705_b200 import nnqs
    with pytest.raises(nnqs.NNQSError) as e:
        nnqs.nnqs_ham_compress(np.zeros((1, 1)), np.zeros((1, 1, 1, 1)), 3, 0.0, device=-1)
    assert e.value.code == nnqs.NNQS_E_SIZE
    h1 = np.array([[0.0, 1.0], [0.5, 0.0]])
    with pytest.raises(nnqs.NNQSError) as e:
        nnqs.nnqs_ham_compress(h1, np.zeros((2, 2, 2, 2)), 4, 0.0, device=-1)
    assert e.value.code == nnqs.NNQS_E_SYMMETRY
    with pytest.raises(nnqs.NNQSError) as e:   # Y0 alone: odd Y count
        nnqs.nnqs_ham_from_pauli([[1, 0]], [[1, 0]], [0.3], 2, device=-1)
    assert e.value.code == nnqs.NNQS_E_ODD_Y


def test_options_layout_and_defaults(lib_path):
    """nnqs_options as the header declares it (16 int32: algorithm, three thresholds,
    literal_kernel, 11 reserved) and the library defaults the binding relies on."""
    from paper_2306_16705_b200 import nnqs
    assert ctypes.sizeof(nnqs.Options) == 64
    src = open(HDR).read()
    for name in ("NNQS_LIT_AUTO 0", "NNQS_LIT_STAGED 1", "NNQS_LIT_PLAIN 2", "int32_t literal_kernel;",
                 "int32_t reserved[11];"):
        assert name in src, name
    o = nnqs.nnqs_options_default()
    assert (o.algorithm, o.literal_kernel) == (0, 0)
    assert (o.thr_single, o.thr_double, o.thr_rowheavy) == (128, 8192, 16384)
    assert list(o.reserved) == [0] * 11
