"""The C-ABI library builds for sm_100a, loads, and exports every symbol that
include/pbvd.h declares (no compute without a GPU)."""
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def lib():
    from paper_1608_00066_b200 import build, _lib
    build.build()
    return _lib.load()


def header_functions():
    txt = (ROOT / "include" / "pbvd.h").read_text()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(pbvd_[a-z_]+)\s*\(", txt)))


def test_header_declares_the_north_star_calls():
    fns = header_functions()
    for f in ("pbvd_create", "pbvd_decode", "pbvd_destroy", "pbvd_decode_blocks"):
        assert f in fns


def test_library_exports_every_declared_symbol(lib):
    from paper_1608_00066_b200 import _lib
    fns = header_functions()
    missing = [f for f in fns if not hasattr(lib, f)]
    assert not missing
    assert set(fns) == set(_lib.EXPORTS)


def test_sass_is_sm100a_and_uses_dpx_and_bulk_copies():
    import subprocess
    so = ROOT / "paper_1608_00066_b200" / "libpbvd.so"
    out = subprocess.run(["cuobjdump", "-sass", str(so)], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", str(so)], capture_output=True,
                                       text=True).stdout
    for op in ("VIADDMNMX", "SHFL.BFLY", "PRMT", "UBLKCP", "LDGSTS"):
        assert op in out, op


def test_pure_host_calls(lib):
    import ctypes
    assert lib.pbvd_strerror(0).decode() == "ok"
    assert "unsupported" in lib.pbvd_strerror(-4).decode()
    sup = lib.pbvd_supported().decode()
    assert "7:2:171,133:2" in sup and "9:3:557,663,711" in sup and "3:2:7,5:1" in sup
    h = ctypes.c_void_p()
    polys = (ctypes.c_uint32 * 2)(0o171, 0o133)
    # argument validation happens before any device call
    assert lib.pbvd_create(ctypes.byref(h), 7, 2, polys, 1, None, 12, 42, 8, 1, 0) == -1  # D % 8
    assert lib.pbvd_create(ctypes.byref(h), 7, 2, polys, 1, None, 512, 0, 8, 1, 0) == -1  # L
    assert lib.pbvd_create(None, 7, 2, polys, 1, None, 512, 42, 8, 1, 0) == -1


def test_create_failures_set_the_last_error(lib):
    """Every pbvd_create failure path leaves a message in pbvd_last_error(NULL)."""
    import ctypes
    h = ctypes.c_void_p()
    polys = (ctypes.c_uint32 * 2)(0o171, 0o133)
    zero = (ctypes.c_uint8 * 4)(0, 0, 0, 0)
    cases = [
        (7, 2, polys, 1, None, 12, 42, 8, 1),      # D % 8
        (7, 2, polys, 1, None, 512, 0, 8, 1),      # L
        (7, 2, polys, 2, zero, 512, 42, 8, 1),     # puncture matrix keeps nothing
        (7, 2, polys, 1, None, 512, 42, 9, 1),     # soft bits
        (7, 2, polys, 1, None, 512, 42, 8, 64),    # unknown flag
    ]
    for c in cases:
        rc = lib.pbvd_create(ctypes.byref(h), *c, 0)
        assert rc == -1, c
        assert lib.pbvd_last_error(None).decode(), c


def test_binding_validates_buffers_before_the_call():
    """the C ABI takes no output length, so the binding rejects
    a too-small, wrongly typed, strided or misplaced buffer itself."""
    import torch
    from paper_1608_00066_b200.decoder import _check_in, _check_out
    x = torch.zeros(64, dtype=torch.int8)
    _check_in(x, "llr", None)
    with pytest.raises(ValueError):
        _check_in(x[::2], "llr", None)                 # strided view
    with pytest.raises(ValueError):
        _check_in(x.to(torch.int16), "llr", None)
    with pytest.raises(ValueError):
        _check_in(x, "llr", 0)                          # host tensor where CUDA is needed
    o = torch.zeros(16, dtype=torch.uint8)
    assert _check_out(o, 16, None) is o
    with pytest.raises(ValueError):
        _check_out(o, 17, None)                         # too small
    with pytest.raises(ValueError):
        _check_out(o.to(torch.int8), 8, None)
    with pytest.raises(ValueError):
        _check_out(o[::2], 4, None)
    with pytest.raises(ValueError):
        _check_out(o, 8, 0)
