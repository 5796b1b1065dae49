"""Host side of the run-time kernels (no GPU): NVRTC compiles the kernel
templates for codes that are not compiled in (pbvd_jit_prebuild), and bad
shapes / arguments are rejected with the documented codes."""
import ctypes

import pytest

import paper_1608_00066_b200 as P
from paper_1608_00066_b200 import _lib


@pytest.fixture(scope="module")
def L():
    from paper_1608_00066_b200 import build
    build.build()
    return _lib.load()


@pytest.mark.parametrize("K,polys", [(4, (0o15, 0o17)), (5, (0o23, 0o33, 0o25, 0o37))])
def test_prebuild_compiles(L, K, polys):
    P.jit_prebuild(K, polys)          # raises PbvdError with the NVRTC log on failure


def test_prebuild_rejects(L):
    arr = (ctypes.c_uint32 * 2)(0o171, 0o133)
    msg = ctypes.create_string_buffer(256)
    assert L.pbvd_jit_prebuild(13, 2, arr, 0, msg, 256) == -1          # K out of range
    assert L.pbvd_jit_prebuild(7, 2, arr, 16, msg, 256) == -4          # no 16-lane shape
    assert b"shape" in msg.value
    assert L.pbvd_jit_prebuild(7, 2, arr, 8, msg, 256) == -4           # 8 states per lane
    bad = (ctypes.c_uint32 * 2)(0o171, 0o400)                          # poly >= 2^K
    assert L.pbvd_jit_prebuild(7, 2, bad, 0, msg, 256) == -1
