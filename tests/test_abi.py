"""The C-ABI library loads on a CPU-only box and exports every symbol the headers declare."""
import ctypes as C
import os
import re

import pytest

from paper_2505_23317_b200 import _lib as L
from paper_2505_23317_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header):
    txt = open(os.path.join(ROOT, "include", header)).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(cfdx?_[a-z_0-9]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    B.build()
    return L.load()


def test_every_declared_symbol_is_exported(lib):
    names = _declared("cfdetr.h") + _declared("cfdetr_debug.h")
    assert "cfd_batch_refine" in names and "cfd_select_regions" in names
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(L.PUBLIC_SYMBOLS) == _declared("cfdetr.h")
    assert sorted(L.DEBUG_SYMBOLS) == _declared("cfdetr_debug.h")


def test_status_strings_and_version(lib):
    assert lib.cfd_status_str(0) == b"ok"
    assert lib.cfd_status_str(-4) == b"capacity exceeded"
    assert b"sm_100a" in lib.cfd_version()


def test_host_side_argument_errors_without_gpu(lib):
    ctx = C.c_void_p()
    assert lib.cfd_create(None, None, None, C.byref(ctx)) == -1
    assert lib.cfd_query(None, 1, None, None, None, None) == -1
    assert lib.cfd_coarse_encode(None, 1, None, None, None, None, None, None, 0, None) == -1
    assert lib.cfd_batch_refine(None, 1, None, None, None, None, None, None, None, None, None, None, 0, None) == -1
    assert lib.cfd_destroy(None) == 0
    assert lib.cfd_set_decoder(None, None, None) == -1
    assert lib.cfd_decode(None, 1, None, None, 1, None, None, None, None, 0, None) == -1
    # debug entry points validate shapes before touching the device
    assert lib.cfdx_gemm(0, 64, 64, None, None, None, 0, None, None, None) == -1
    assert lib.cfdx_gemm(10, 60, 64, 1, 1, 1, 0, 1, None, None) == -1


def test_tuning_option_validation_without_gpu(lib):
    """cfdx_set_option accepts the documented keys/values (cfdetr_debug.h) and rejects others
    (ctx = NULL: the debug entry points' switches)."""
    f = lib.cfdx_set_option
    assert f(None, 0, 6) == -1 and f(None, 0, 0) == -1 and f(None, 0, 2) == -1 and f(None, 0, 4) == -1
    assert f(None, 1, 3) == -1 and f(None, 1, 10) == -1 and f(None, 1, -2) == -1
    assert f(None, 5, -3) == -1 and f(None, 6, 4) == -1 and f(None, 9, 0) == -1 and f(None, 10, 0) == -1
    assert f(None, 8, 0) == -1 and f(None, 12, 0) == -1 and f(None, 20, 0) == -1 and f(None, 26, 0) == -1 and f(None, 24, -1) == -1 and f(None, 24, 5000) == -1
    for key, val in ((0, 1), (1, 8), (2, 0), (3, 0), (4, 0), (5, 300), (7, 0), (11, 0), (19, 0), (17, 74)):
        assert f(None, key, val) == 0
    assert f(None, 21, 5) == -1 and f(None, 22, 2) == -1
    assert f(None, 24, 1024) == 0 and f(None, 24, 256) == 0
    for key, val in ((0, 7), (1, 2), (2, 1), (3, 1), (4, 1), (5, 700), (7, 1), (11, 1), (19, 1), (17, 0),
                     (21, 32), (22, 4), (23, 1), (25, 1)):
        assert f(None, key, val) == 0  # restore the defaults


def test_config_validation_without_gpu(lib):
    cfg = L.cfd_config(640, 640, 32, 16, 256, 8, 6, 1024, 5, 8, 1e-6)
    w = L.cfd_weights()
    ctx = C.c_void_p()
    # weights missing -> ARG before any CUDA call
    assert lib.cfd_create(C.byref(cfg), C.byref(w), None, C.byref(ctx)) == -1
    # geometry checks run before any CUDA call (non-null placeholder weight pointers)
    layers = (L.cfd_layer_weights * 6)(*[L.cfd_layer_weights(*([1] * 12)) for _ in range(6)])
    wf = L.cfd_weights(1, 1, 1, 1, 1, 1, layers)

    def create(*g):
        return lib.cfd_create(C.byref(L.cfd_config(*g)), C.byref(wf), None, C.byref(ctx))
    # dh = 64 (SURVEY §8(b) lists {32, 64}): rejected -- the kernels are built for 64-byte head rows
    assert create(640, 640, 32, 16, 256, 4, 6, 1024, 5, 8, 1e-6) == -3
    assert create(640, 640, 32, 16, 192, 6, 6, 768, 5, 8, 1e-6) == -3     # d not in {64, 128, 256, 512}
    assert create(640, 600, 32, 16, 256, 8, 6, 1024, 5, 8, 1e-6) == -2    # W % Pc != 0
    assert create(640, 640, 32, 12, 256, 8, 6, 1024, 5, 8, 1e-6) == -2    # Pc % Pf != 0
    assert create(640, 640, 32, 16, 256, 8, 6, 1024, 6, 8, 1e-6) == -1    # score_layer >= L
    assert create(4096, 4096, 32, 16, 64, 2, 1, 256, 0, 8, 1e-6) == -3     # Nc = 16384 > 4096


def test_sass_contains_tcgen05_and_tma():
    import subprocess
    out = subprocess.run(["cuobjdump", "-sass", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in out      # tcgen05.mma
    assert "UTMALDG" in out      # TMA loads
    assert "LDTM" in out         # tcgen05.ld
    assert "HMMA" not in out.replace("UTCHMMA", "")  # no legacy mma.sync path
