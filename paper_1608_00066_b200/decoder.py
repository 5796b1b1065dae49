"""Python binding of the C ABI with the same names: ``Decoder`` wraps a
``pbvd_t`` handle.  Torch provides device memory and streams only; every
decode step runs in libpbvd.so's sm_100a kernels (no CPU fallback)."""
from __future__ import annotations

import ctypes
import weakref

import torch

from . import _lib


class PbvdError(RuntimeError):
    pass


def _check(rc, h=None, what=""):
    if rc < 0:
        L = _lib.load()
        msg = L.pbvd_strerror(rc).decode()
        # h None: the thread's last pbvd_create failure (pbvd_last_error(NULL))
        detail = L.pbvd_last_error(h).decode()
        if detail:
            msg += ": " + detail
        raise PbvdError(f"{what} failed ({rc}): {msg}")
    return rc


def supported():
    """[(K, R, polys, lanes)] compiled into the library."""
    out = []
    for ent in _lib.load().pbvd_supported().decode().strip(";").split(";"):
        K, R, polys, lanes = ent.split(":")
        out.append((int(K), int(R), tuple(int(p, 8) for p in polys.split(",")), int(lanes)))
    return out


def jit_prebuild(K, polys, lanes=0):
    """pbvd_jit_prebuild: NVRTC-build (no GPU needed) and disk-cache the kernels
    pbvd_create would build at run time for a code that is not compiled in."""
    L = _lib.load()
    arr = (ctypes.c_uint32 * len(polys))(*[int(p) for p in polys])
    msg = ctypes.create_string_buffer(8192)
    rc = L.pbvd_jit_prebuild(int(K), len(polys), arr, int(lanes), msg, len(msg))
    if rc < 0:
        raise PbvdError(f"pbvd_jit_prebuild failed ({rc}): {L.pbvd_strerror(rc).decode()}: "
                        f"{msg.value.decode(errors='replace')}")


def probe_acs_balanced(device: int = 0):
    """pbvd_probe_acs_balanced: (measured ACS/s of the pipe-balanced minimal
    sequence, kernel ms)."""
    L = _lib.load()
    a, m = ctypes.c_double(), ctypes.c_double()
    _check(L.pbvd_probe_acs_balanced(int(device), ctypes.byref(a), ctypes.byref(m)), None,
           "pbvd_probe_acs_balanced")
    return a.value, m.value


def probe_acs_peak(device: int = 0):
    """pbvd_probe_acs_peak: (measured ACS/s of the all-ALU minimal sequence,
    kernel ms)."""
    L = _lib.load()
    a, m = ctypes.c_double(), ctypes.c_double()
    _check(L.pbvd_probe_acs_peak(int(device), ctypes.byref(a), ctypes.byref(m)), None,
           "pbvd_probe_acs_peak")
    return a.value, m.value


def _check_in(t: torch.Tensor, name: str, cuda_device: int | None):
    """int8, contiguous, on cuda:cuda_device (None: on the host)."""
    if t.dtype != torch.int8 or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous int8 tensor")
    if cuda_device is None:
        if t.is_cuda:
            raise ValueError(f"{name} must be a host (CPU) tensor")
    elif not t.is_cuda or t.device.index != cuda_device:
        raise ValueError(f"{name} must be on cuda:{cuda_device}")


def _check_out(out: torch.Tensor, nbytes: int, cuda_device: int | None):
    """The C ABI takes no output length: a caller-supplied out must be a
    contiguous uint8 tensor on the right device with >= nbytes elements."""
    if out.dtype != torch.uint8 or not out.is_contiguous():
        raise ValueError("out must be a contiguous uint8 tensor")
    if out.numel() < nbytes:
        raise ValueError(f"out holds {out.numel()} bytes, the call writes {nbytes}")
    if cuda_device is None:
        if out.is_cuda:
            raise ValueError("out must be a host (CPU) tensor")
    elif not out.is_cuda or out.device.index != cuda_device:
        raise ValueError(f"out must be on cuda:{cuda_device}")
    return out


class Decoder:
    """pbvd_create(...) -- see include/pbvd.h for the meaning of every argument.

    punct: None or an R x P keep matrix (rows in generator order)."""

    def __init__(self, K, polys, D, L, punct=None, soft_bits=8, terminated=True, device=0,
                 lanes=0, fused=True, allow_catastrophic=False, start_zero=False):
        self._L = _lib.load()
        self._streams = weakref.WeakSet()
        self.K, self.polys, self.D, self.L = int(K), tuple(int(p) for p in polys), int(D), int(L)
        self.R = len(self.polys)
        self.punct = None if punct is None else tuple(tuple(int(x) for x in row) for row in punct)
        self.terminated = bool(terminated)
        self.start_zero = bool(start_zero)
        self.device = int(device)
        arr = (ctypes.c_uint32 * self.R)(*self.polys)
        if self.punct is None:
            P, pp = 1, None
        else:
            P = len(self.punct[0])
            flat = [self.punct[r][p] for r in range(self.R) for p in range(P)]
            pp = (ctypes.c_uint8 * len(flat))(*flat)
        h = ctypes.c_void_p()
        rc = self._L.pbvd_create(ctypes.byref(h), self.K, self.R, arr, P, pp, self.D, self.L,
                                 int(soft_bits),
                                 (_lib.PBVD_TERMINATED if terminated else 0)
                                 | (_lib.PBVD_ALLOW_CATASTROPHIC if allow_catastrophic else 0)
                                 | (_lib.PBVD_START_ZERO if start_zero else 0),
                                 self.device)
        _check(rc, None, "pbvd_create")
        self._h = h
        if lanes:
            self.set_lanes(lanes)
        if not fused:
            self.set_fused(False)

    # --------------------------------------------------------------- sizes
    def llr_count(self, n_info):
        return _check(self._L.pbvd_llr_count(self._h, int(n_info)), self._h, "pbvd_llr_count")

    def stage_count(self, n_info):
        return _check(self._L.pbvd_stage_count(self._h, int(n_info)), self._h, "pbvd_stage_count")

    def block_count(self, n_info):
        return _check(self._L.pbvd_block_count(self._h, int(n_info)), self._h, "pbvd_block_count")

    # -------------------------------------------------------------- decode
    def _live(self):
        if not getattr(self, "_h", None):
            raise PbvdError("decoder is closed")

    def _range_bytes(self, n_info_total, block0, nblocks):
        t0 = int(block0) * self.D
        t1 = min((int(block0) + int(nblocks)) * self.D, int(n_info_total))
        return max(0, (t1 - t0 + 7) // 8)

    def _stream(self, stream):
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        return ctypes.c_void_p(stream.cuda_stream)

    def decode(self, llr: torch.Tensor, n_info: int, out: torch.Tensor | None = None,
               stream=None) -> torch.Tensor:
        """pbvd_decode: int8 CUDA tensor -> packed uint8 CUDA tensor (async)."""
        self._live()
        _check_in(llr, "llr", self.device)
        nbytes = (int(n_info) + 7) // 8
        if out is None:
            out = torch.empty(nbytes, dtype=torch.uint8, device=llr.device)
        _check_out(out, nbytes, self.device)
        rc = self._L.pbvd_decode(self._h, llr.data_ptr(), llr.numel(), out.data_ptr(),
                                 int(n_info), self._stream(stream))
        _check(rc, self._h, "pbvd_decode")
        return out

    def decode_blocks(self, llr_window: torch.Tensor, window_stage0: int, n_info_total: int,
                      block0: int, nblocks: int, out: torch.Tensor | None = None,
                      stream=None) -> torch.Tensor:
        """pbvd_decode_blocks: decode blocks [block0, block0+nblocks) from a window."""
        self._live()
        _check_in(llr_window, "llr_window", self.device)
        nbytes = self._range_bytes(n_info_total, block0, nblocks)
        if out is None:
            out = torch.empty(nbytes, dtype=torch.uint8, device=llr_window.device)
        _check_out(out, nbytes, self.device)
        rc = self._L.pbvd_decode_blocks(self._h, llr_window.data_ptr(), int(window_stage0),
                                        llr_window.numel(), int(n_info_total), int(block0),
                                        int(nblocks), out.data_ptr(), self._stream(stream))
        _check(rc, self._h, "pbvd_decode_blocks")
        return out

    def decode_blocks_mirrored(self, llr_window: torch.Tensor, window_stage0: int,
                               n_info_total: int, block0: int, nblocks: int, out: torch.Tensor,
                               mirror_ptrs, stream=None) -> torch.Tensor:
        """pbvd_decode_blocks_mirrored: decode_blocks whose traceback also stores
        the bits at every address in mirror_ptrs (ints: device pointers, e.g.
        other ranks' gather buffers opened through CUDA IPC)."""
        self._live()
        _check_in(llr_window, "llr_window", self.device)
        _check_out(out, self._range_bytes(n_info_total, block0, nblocks), self.device)
        arr = (ctypes.c_void_p * max(1, len(mirror_ptrs)))(*[int(x) for x in mirror_ptrs])
        rc = self._L.pbvd_decode_blocks_mirrored(
            self._h, llr_window.data_ptr(), int(window_stage0), llr_window.numel(),
            int(n_info_total), int(block0), int(nblocks), out.data_ptr(), arr, len(mirror_ptrs),
            self._stream(stream))
        _check(rc, self._h, "pbvd_decode_blocks_mirrored")
        return out

    def decode_host(self, llr: torch.Tensor, n_info: int, out: torch.Tensor | None = None,
                    n_streams: int = 3, window_stage0: int = 0, block0: int = 0,
                    nblocks: int | None = None) -> torch.Tensor:
        """pbvd_decode_host: host int8 window (pinned for overlap) -> host packed bits.

        Defaults decode the whole stream; a shard passes its window and range."""
        self._live()
        _check_in(llr, "llr", None)
        if nblocks is None:
            nblocks = self.block_count(n_info) - int(block0)
        nbytes = self._range_bytes(n_info, block0, nblocks)
        if out is None:
            out = torch.empty(nbytes, dtype=torch.uint8, pin_memory=llr.is_pinned())
        _check_out(out, nbytes, None)
        rc = self._L.pbvd_decode_host(self._h, llr.data_ptr(), int(window_stage0), llr.numel(),
                                      int(n_info), int(block0), int(nblocks), out.data_ptr(),
                                      int(n_streams))
        _check(rc, self._h, "pbvd_decode_host")
        return out

    # ------------------------------------------------------------- tuning
    def open_stream(self) -> "StreamDecoder":
        """pbvd_stream_open: a continuous-stream decoder on this handle (closed
        with it: close() closes every stream still open first)."""
        self._live()
        sd = StreamDecoder(self)
        self._streams.add(sd)
        return sd

    def set_lanes(self, lanes: int):
        _check(self._L.pbvd_set_lanes(self._h, int(lanes)), self._h, "pbvd_set_lanes")

    @property
    def lanes(self) -> int:
        return self._L.pbvd_get_lanes(self._h)

    def set_fused(self, fused: bool):
        """True: one kernel (forward + in-warp traceback); False: the paper's
        two kernels (pbvd_set_fused)."""
        _check(self._L.pbvd_set_fused(self._h, int(bool(fused))), self._h, "pbvd_set_fused")

    @property
    def fused(self) -> bool:
        return bool(self._L.pbvd_get_fused(self._h))

    def set_workspace_limit(self, nbytes: int):
        _check(self._L.pbvd_set_workspace_limit(self._h, int(nbytes)), self._h,
               "pbvd_set_workspace_limit")

    def set_profiling(self, enable: bool = True):
        _check(self._L.pbvd_set_profiling(self._h, int(bool(enable))), self._h,
               "pbvd_set_profiling")

    def kernel_times(self):
        """(forward ms, traceback ms, launches) of the last decode (sync first)."""
        f, t, n = ctypes.c_float(), ctypes.c_float(), ctypes.c_int()
        _check(self._L.pbvd_kernel_times(self._h, ctypes.byref(f), ctypes.byref(t),
                                         ctypes.byref(n)), self._h, "pbvd_kernel_times")
        return f.value, t.value, n.value

    def info(self) -> dict:
        i = _lib.PbvdInfo()
        _check(self._L.pbvd_get_info(self._h, ctypes.byref(i)), self._h, "pbvd_get_info")
        return {k: getattr(i, k) for k, _ in _lib.PbvdInfo._fields_}

    def close(self):
        for sd in list(getattr(self, "_streams", ())):
            sd.close()
        if getattr(self, "_h", None):
            self._L.pbvd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class StreamDecoder:
    """pbvd_stream_*: decode one stream whose soft values arrive in pieces.

    push(llr) returns the packed bits of every block completed by this piece
    (a CUDA uint8 tensor, possibly empty); finish() returns the rest.  Their
    concatenation equals Decoder.decode of the whole stream."""

    def __init__(self, dec: Decoder):
        self._dec, self._L = dec, dec._L
        h = ctypes.c_void_p()
        _check(self._L.pbvd_stream_open(dec._h, ctypes.byref(h)), dec._h, "pbvd_stream_open")
        self._s = h
        self._rx = 0          # kept soft values pushed
        self._emitted = 0     # bits returned so far
        R, punct = dec.R, dec.punct
        if punct is None:
            self._P, self._cum, self._kp = 1, [0], R
        else:
            self._P = len(punct[0])
            self._cum, k = [], 0
            for p in range(self._P):
                self._cum.append(k)
                k += sum(int(punct[r][p] != 0) for r in range(R))
            self._kp = k

    def _stages(self, k):
        """Complete stages among the first k kept values (upper bound on bits)."""
        full, rem = divmod(k, self._kp)
        return full * self._P + sum(1 for p in range(1, self._P + 1)
                                    if (self._cum[p] if p < self._P else self._kp) <= rem)

    def _out(self, n_more, device):
        nbits = max(0, self._stages(self._rx + n_more) - self._emitted)
        return torch.empty((nbits + 7) // 8 + 1, dtype=torch.uint8, device=device)

    def _live(self):
        if not getattr(self, "_s", None):
            raise PbvdError("stream is closed (or its decoder was closed)")

    def push(self, llr: torch.Tensor, stream=None) -> torch.Tensor:
        self._live()
        _check_in(llr, "llr", self._dec.device)
        out = self._out(llr.numel(), llr.device)
        n = ctypes.c_int64()
        rc = self._L.pbvd_stream_push(self._s, llr.data_ptr(), llr.numel(), out.data_ptr(),
                                      out.numel(), ctypes.byref(n), self._dec._stream(stream))
        _check(rc, self._dec._h, "pbvd_stream_push")
        self._rx += llr.numel()
        self._emitted += n.value
        return out[: n.value // 8]

    def finish(self, stream=None):
        """-> (packed bits of the remaining blocks, their bit count)."""
        self._live()
        out = self._out(0, torch.device("cuda", self._dec.device))
        n = ctypes.c_int64()
        rc = self._L.pbvd_stream_finish(self._s, out.data_ptr(), out.numel(), ctypes.byref(n),
                                        self._dec._stream(stream))
        self._rx = self._emitted = 0
        _check(rc, self._dec._h, "pbvd_stream_finish")
        return out[: (n.value + 7) // 8], n.value

    def close(self):
        if getattr(self, "_s", None):
            self._L.pbvd_stream_close(self._s)
            self._s = None
            self._dec._streams.discard(self)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
