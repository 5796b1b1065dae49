"""ctypes binding of the CPU oracle (oracle/pbvd_oracle.c).

TEST INFRASTRUCTURE ONLY: tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs are the only callers.  Nothing
under ``paper_1608_00066_b200/`` imports this module and this module imports
nothing from there.

Every function follows a passage of PAPER.md (``P:n``) or a reading of
SURVEY.md §8(c) (``c-n``, restated in DESIGN.md §3); see the C file.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "pbvd_oracle.c"
_LIB = _HERE / "liborc.so"

TERMINATED = 1
START_ZERO = 2
S_HEAD = 8192  # c-12

_lib = None


def build(force: bool = False) -> Path:
    """Compile the oracle with gcc (plain -O2, no vector intrinsics)."""
    if force or not _LIB.exists() or _LIB.stat().st_mtime < _SRC.stat().st_mtime:
        tmp = _LIB.with_suffix(f".so.{os.getpid()}")
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", str(tmp),
                               str(_SRC), "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(_LIB))
        i64, i32, u32p = ctypes.c_int64, ctypes.c_int, ctypes.POINTER(ctypes.c_uint32)
        vp = ctypes.c_void_p
        L.orc_out.argtypes = [i32, i32, u32p, ctypes.c_uint32, i32]
        L.orc_out.restype = i32
        L.orc_next.argtypes = [i32, ctypes.c_uint32, i32]
        L.orc_next.restype = ctypes.c_uint32
        L.orc_tb_step.argtypes = [i32, ctypes.c_uint32, i32, ctypes.POINTER(ctypes.c_int)]
        L.orc_tb_step.restype = ctypes.c_uint32
        L.orc_llr_count.argtypes = [i32, i32, vp, i64]
        L.orc_llr_count.restype = i64
        L.orc_plan.argtypes = [i64, i64, i32, i32, i64, vp, vp, vp, vp]
        L.orc_plan.restype = i64
        L.orc_decode_range.argtypes = [i32, i32, u32p, i32, vp, vp, i64, i64, i64, i32, i32,
                                       ctypes.c_uint, i64, i64, i32, vp, vp, vp]
        L.orc_decode_range.restype = i64
        L.orc_block_decisions.argtypes = [i32, i32, u32p, i32, vp, vp, i64, i64, i32, i32,
                                          ctypes.c_uint, i64, vp, vp, vp, vp]
        L.orc_block_decisions.restype = i32
        L.orc_full.argtypes = [i32, i32, u32p, i32, vp, vp, i64, i64, ctypes.c_uint, vp, vp]
        L.orc_full.restype = i32
        L.orc_path_metric.argtypes = [i32, i32, u32p, i32, vp, vp, i64, i64, ctypes.c_uint,
                                      vp, vp]
        L.orc_path_metric.restype = i32
        L.orc_ml.argtypes = [i32, i32, u32p, i32, vp, vp, i64, i32, ctypes.c_uint, vp, vp, vp]
        L.orc_ml.restype = i32
        _lib = L
    return _lib


# ----------------------------------------------------------------- helpers

def _polys(polys):
    arr = (ctypes.c_uint32 * len(polys))(*[int(p) for p in polys])
    return arr


def _punct(punct, R):
    """punct: None or an R x P keep matrix (rows in generator-list order)."""
    if punct is None:
        return 1, None, None
    m = np.ascontiguousarray(np.asarray(punct, dtype=np.uint8))
    assert m.ndim == 2 and m.shape[0] == R
    return int(m.shape[1]), m, m.ctypes.data


def _llr(llr):
    a = np.ascontiguousarray(np.asarray(llr, dtype=np.int8))
    return a, a.ctypes.data, int(a.size)


def pack_bits(bits: np.ndarray) -> np.ndarray:
    """LSB-first packing (c-16): bit i -> byte i>>3, bit i&7."""
    return np.packbits(np.asarray(bits, dtype=np.uint8), bitorder="little")


def out(K, R, polys, d, x) -> int:
    """Eq. 2: encoder output bits, bit r = c^(r+1)."""
    return lib().orc_out(K, R, _polys(polys), d, x)


def next_state(K, d, x) -> int:
    """P:133 shift S_2j, S_2j+1 -> S_j / S_{j+2^{v-1}}."""
    return lib().orc_next(K, d, x)


def tb_step(K, state, sp):
    """Alg. 1 K2 step: (predecessor, decoded bit)."""
    bit = ctypes.c_int()
    prev = lib().orc_tb_step(K, state, sp, ctypes.byref(bit))
    return prev, bit.value


def butterfly(K, R, polys, j):
    """(alpha, beta, gamma, theta) of butterfly j by direct Eq. 2 (Eqs. 3-6)."""
    return (out(K, R, polys, 2 * j, 0), out(K, R, polys, 2 * j, 1),
            out(K, R, polys, 2 * j + 1, 0), out(K, R, polys, 2 * j + 1, 1))


def classify(K, R, polys):
    """Group the N/2 butterflies by alpha; Table II
    lists the member *states* {2j, 2j+1} (c-21).  Returns a list of dicts in
    first-appearance order of alpha."""
    groups = {}
    for j in range(1 << (K - 2)):
        a, b, g, t = butterfly(K, R, polys, j)
        e = groups.setdefault(a, {"alpha": a, "beta": b, "gamma": g, "theta": t, "states": []})
        e["states"] += [2 * j, 2 * j + 1]
    return list(groups.values())


def llr_count(R, punct, n_stages) -> int:
    P, _, p = _punct(punct, R)
    return lib().orc_llr_count(R, P, p, n_stages)


def plan(n_info, n_stages, D, L, b):
    """Block b's (t0, t1, lo, hi) and the block count."""
    v = [ctypes.c_int64() for _ in range(4)]
    nb = lib().orc_plan(n_info, n_stages, D, L, b, *[ctypes.addressof(x) for x in v])
    return nb, tuple(x.value for x in v)


def decode(code, llr, n_info, D, L, flags=TERMINATED, punct=None, threads=None,
           b0=0, nblk=None, return_starts=False, return_ties=False, window_stage0=0):
    """Segmented PBVD decode of blocks [b0, b0+nblk).

    `llr` is the whole stream, or (window_stage0 > 0) the soft values from the
    first kept value of stage window_stage0 on.  Returns the unpacked decoded
    bits (uint8 0/1) of those blocks' decoding ranges, plus start states / tie
    count on request."""
    K, polys = code["K"], code["polys"]
    R = len(polys)
    P, pm, pp = _punct(punct, R)
    a, ap, n_llr = _llr(llr)
    nb = -(-n_info // D)
    if nblk is None:
        nblk = nb - b0
    t_first = b0 * D
    t_last = min((b0 + nblk) * D, n_info)
    bits = np.zeros(t_last - t_first, dtype=np.uint8)
    starts = np.zeros(nblk, dtype=np.int32)
    ties = ctypes.c_int64()
    if threads is None:
        threads = os.cpu_count() or 1
    rc = lib().orc_decode_range(K, R, _polys(polys), P, pp, ap, window_stage0, n_llr, n_info, D,
                                L, flags, b0, nblk, threads, bits.ctypes.data, starts.ctypes.data,
                                ctypes.addressof(ties))
    if rc < 0:
        raise ValueError(f"orc_decode_range failed: {rc}")
    res = [bits]
    if return_starts:
        res.append(starts)
    if return_ties:
        res.append(ties.value)
    return res[0] if len(res) == 1 else tuple(res)


def block_decisions(code, llr, n_info, D, L, b, flags=TERMINATED, punct=None):
    """Raw per-edge decisions dec[s-lo][u] of block b, its (lo, hi) and start."""
    K, polys = code["K"], code["polys"]
    R = len(polys)
    P, pm, pp = _punct(punct, R)
    a, ap, n_llr = _llr(llr)
    n_stages = n_info + ((K - 1) if flags & TERMINATED else 0)
    nb, (t0, t1, lo, hi) = plan(n_info, n_stages, D, L, b)
    N = 1 << (K - 1)
    dec = np.zeros((hi - lo, N), dtype=np.uint8)
    lo_o, hi_o, st = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
    rc = lib().orc_block_decisions(K, R, _polys(polys), P, pp, ap, n_llr, n_info, D, L, flags,
                                   b, dec.ctypes.data, ctypes.addressof(lo_o),
                                   ctypes.addressof(hi_o), ctypes.addressof(st))
    if rc != 0:
        raise ValueError(f"orc_block_decisions failed: {rc}")
    return dec, (lo_o.value, hi_o.value), st.value


def full(code, llr, n_info, flags=TERMINATED, punct=None):
    """Textbook full-stream Viterbi (§II); returns (bits, metric)."""
    K, polys = code["K"], code["polys"]
    R = len(polys)
    P, pm, pp = _punct(punct, R)
    a, ap, n_llr = _llr(llr)
    bits = np.zeros(n_info, dtype=np.uint8)
    metric = ctypes.c_int64()
    rc = lib().orc_full(K, R, _polys(polys), P, pp, ap, n_llr, n_info, flags, bits.ctypes.data,
                        ctypes.addressof(metric))
    if rc != 0:
        raise ValueError(f"orc_full failed: {rc}")
    return bits, metric.value


def path_metric(code, llr, n_info, bits, flags=TERMINATED, punct=None) -> int:
    """Sum of canonical BMs (c-4) along the encoder path of `bits`."""
    K, polys = code["K"], code["polys"]
    R = len(polys)
    P, pm, pp = _punct(punct, R)
    a, ap, n_llr = _llr(llr)
    b = np.ascontiguousarray(np.asarray(bits, dtype=np.uint8))
    m = ctypes.c_int64()
    rc = lib().orc_path_metric(K, R, _polys(polys), P, pp, ap, n_llr, n_info, flags,
                               b.ctypes.data, ctypes.addressof(m))
    if rc != 0:
        raise ValueError(f"orc_path_metric failed: {rc}")
    return m.value


def ml(code, llr, n_info, flags=TERMINATED, punct=None):
    """Brute-force ML: (min metric, number of minimisers, lowest minimiser)."""
    K, polys = code["K"], code["polys"]
    R = len(polys)
    P, pm, pp = _punct(punct, R)
    a, ap, n_llr = _llr(llr)
    best = ctypes.c_int64()
    nbest = ctypes.c_int64()
    bits = np.zeros(n_info, dtype=np.uint8)
    rc = lib().orc_ml(K, R, _polys(polys), P, pp, ap, n_llr, n_info, flags,
                      ctypes.addressof(best), ctypes.addressof(nbest), bits.ctypes.data)
    if rc != 0:
        raise ValueError(f"orc_ml failed: {rc}")
    return best.value, nbest.value, bits
