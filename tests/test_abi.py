"""C-ABI checks that need no GPU: libdoa.so loads, exports every function include/doa.h declares,
and rejects invalid arguments synchronously (validation happens before any CUDA call)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "doa.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(doa_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()           # builds libdoa.so in a fresh checkout, then imports the package
    import paper_2007_14135_b200 as d
    return d


def test_every_declared_symbol_exported(lib):
    names = _declared()
    assert "doa_plan_create" in names and "doa_run" in names and len(names) >= 12
    raw = C.CDLL(lib.binding.LIB_PATH)
    for n in names:
        assert hasattr(raw, n), n
    assert set(names) <= set(lib.binding.EXPORTS)


def test_status_strings(lib):
    assert lib.lib.doa_status_string(0) == b"DOA_OK"
    assert lib.lib.doa_status_string(2) == b"DOA_ERR_UNSUPPORTED"
    assert lib.lib.doa_version() == 1


@pytest.mark.parametrize("args,status", [
    ((1, 0.5, 1, -90.0, 1.0, 181, 1, 1), 1),          # M < 2
    ((65, 0.5, 4, -90.0, 1.0, 181, 1, 1), 2),         # M > 64: unsupported
    ((16, 0.5, 0, -90.0, 1.0, 181, 1, 1), 1),         # D < 1
    ((16, 0.5, 16, -90.0, 1.0, 181, 1, 1), 1),        # D >= M
    ((16, 0.0, 3, -90.0, 1.0, 181, 1, 1), 1),         # d/lambda <= 0
    ((16, 0.5, 3, -90.0, 1.0, 2, 1, 1), 1),           # L < 3
    ((16, 0.5, 3, -90.0, 0.0, 181, 1, 1), 1),         # dtheta <= 0
    ((16, 0.5, 3, -91.0, 1.0, 181, 1, 1), 1),         # theta0 < -90
    ((16, 0.5, 3, -90.0, 1.0, 182, 1, 1), 1),         # grid end > 90
    ((16, 0.5, 3, -90.0, 1.0, 181, 4, 1), 1),         # bad alg
    ((16, 0.5, 3, -90.0, 1.0, 181, 1, 0), 1),         # max_batch < 1
    ((16, 0.5, 3, -90.0, 1.0, 1 << 31, 1, 1), 1),     # L >= 2^31
])
def test_plan_create_validation(lib, args, status):
    h = C.c_void_p(123)
    st = lib.lib.doa_plan_create(C.byref(h), *args)
    assert st == status
    assert h.value is None                              # *plan set to NULL on failure
    assert len(lib.lib.doa_last_error()) > 0


def test_null_plan_rejected(lib):
    assert lib.lib.doa_covariance(None, None, 1, 1, None, None) == 1
    assert lib.lib.doa_eig(None, None, 1, None, None, None, None) == 1
    assert lib.lib.doa_spectrum(None, None, None, 1, None, None, None) == 1
    assert lib.lib.doa_peaks(None, 1, None, None, None, None, None) == 1
    assert lib.lib.doa_run(None, None, 1, 1, None, None, None, None, None, None) == 1
    assert lib.lib.doa_plan_destroy(None) == 0


def test_binding_is_thin(lib):
    # the binding must not contain a compute fallback: no numpy/torch math on the data path
    src = open(lib.binding.__file__).read()
    for bad in ("np.linalg", "torch.linalg", "torch.fft", "import oracle", "from oracle"):
        assert bad not in src


@pytest.mark.parametrize("M,D,naz,nel,daz,dele,status", [
    (1, 1, 360, 1, 1.0, 1.0, 1),      # M < 2
    (17, 2, 360, 1, 1.0, 1.0, 2),     # M > 16: unsupported for general arrays
    (8, 8, 360, 1, 1.0, 1.0, 1),      # D >= M
    (8, 2, 1, 2, 1.0, 1.0, 1),        # L < 3
    (8, 2, 360, 1, 0.0, 1.0, 1),      # daz <= 0 with naz > 1
    (8, 2, 360, 2, 1.0, -1.0, 1),     # del <= 0 with nel > 1
])
def test_plan_create_array_validation(lib, M, D, naz, nel, daz, dele, status):
    import numpy as np
    pos = np.zeros((max(M, 1), 3))
    h = C.c_void_p(7)
    st = lib.lib.doa_plan_create_array(C.byref(h), M, pos.ctypes.data_as(C.POINTER(C.c_double)), D, 0.0, daz,
                                       naz, 90.0, dele, nel, 1, 1, 1)
    assert st == status and h.value is None


@pytest.mark.parametrize("M,dl,D,snr,N,B,ok", [
    (0, 0.5, 1, 10.0, 8, 1, False),            # M < 1
    (65, 0.5, 1, 10.0, 8, 1, False),           # M > 64
    (8, 0.5, 0, 10.0, 8, 1, False),            # D < 1
    (8, 0.5, 64, 10.0, 8, 1, False),           # D > 63
    (8, 0.0, 2, 10.0, 8, 1, False),            # d/lambda <= 0
    (8, 0.5, 2, float("nan"), 8, 1, False),    # non-finite SNR
    (8, 0.5, 2, 10.0, 0, 1, False),            # N < 1
    (8, 0.5, 2, 10.0, 8, -1, False),           # B < 0
    (8, 0.5, 2, 10.0, 8, 0, True),             # B == 0: nothing to do, OK
])
def test_generate_validation(lib, M, dl, D, snr, N, B, ok):
    """doa_generate validates before touching the device (NULL pointers are fine for B == 0)."""
    st = lib.lib.doa_generate(M, dl, D, None, 0, snr, 1, 0, B, N, None, None)
    assert (st == 0) == ok
    if not ok:
        assert st == 1 and len(lib.lib.doa_last_error()) > 0
