"""Synthetic convolutionally-coded BPSK/AWGN streams (input generation only).

The workloads follow the paper's experiments -- CCSDS (2,1,7) code
g = 171,133, 8-bit soft quantisation (Fig. 4 caption P:385),
AWGN -- and BASELINE.json's five configs.  Conventions (SURVEY.md §8(c),
restated in DESIGN.md §3):

* generator polynomials are octal with bit K-1 the input tap g_{K-1} (c-2);
* the encoder register holds the last v = K-1 inputs, the newest at the MSB
  (c-1), so coded bit r at stage t is XOR_k g^(r)_{v-k} x_{t-k};
* a terminated stream appends v zero tail bits (c-13);
* puncturing keeps punct[r][t mod P] (c-18), anchored at stage 0 and applied
  to the tail stages too;
* BPSK maps 0 -> +1 (c-5); sigma^2 = 1 / (2 R_eff 10^(EbN0/10)) (c-19);
* soft values: clamp(round_half_even(y * 2^f), -127, 127) with f = 5 (c-6);
  hard values: +1 if y >= 0 else -1 (c-7);
* output layout: int8, [stage][r], punctured positions omitted (c-17).

Reproducibility: info bits are drawn in chunks of 2^20 bits and noise in
chunks of 2^20 stages, each chunk from its own seeded torch.Generator, so any
window of a stream (a multi-GPU shard plus its halo) is bit-identical to the
same slice of the whole stream generated on the same device type.
"""
from __future__ import annotations

import math

import torch

CODES = {
    "k3": {"K": 3, "polys": (0o7, 0o5)},                 # textbook (7,5)
    "k7": {"K": 7, "polys": (0o171, 0o133)},             # CCSDS / 802.11
    "k9": {"K": 9, "polys": (0o557, 0o663, 0o711)},      # rate-1/3, 256 states
}

# Keep matrices, rows in generator-list order (171, 133): 802.11 defines row A
# on 133 and row B on 171 (c-18).
PUNCT = {
    "1/2": None,
    "2/3": ((1, 0), (1, 1)),
    "3/4": ((1, 0, 1), (1, 1, 0)),
}

# BASELINE.json configs -- n_info, D, L, Eb/N0, seed.
CONFIGS = {
    "C1": {"code": "k3", "punct": "1/2", "hard": True, "n_info": 4096, "D": 256, "L": 16,
           "ebn0": 4.0, "seed": 1},
    "C2": {"code": "k7", "punct": "1/2", "hard": False, "n_info": 1 << 24, "D": 512, "L": 42,
           "ebn0": 4.0, "seed": 2},
    "C3a": {"code": "k7", "punct": "2/3", "hard": False, "n_info": 1 << 26, "D": 512, "L": 42,
            "ebn0": 4.0, "seed": 3},
    "C3b": {"code": "k7", "punct": "3/4", "hard": False, "n_info": 1 << 26, "D": 512, "L": 42,
            "ebn0": 4.0, "seed": 4},
    "C4": {"code": "k9", "punct": "1/2", "hard": False, "n_info": 1 << 24, "D": 1024, "L": 64,
           "ebn0": 3.0, "seed": 5},
    "C5": {"code": "k7", "punct": "1/2", "hard": False, "n_info": 1 << 32, "D": 512, "L": 42,
           "ebn0": 4.0, "seed": 6},
}

BIT_CHUNK = 1 << 20
NOISE_CHUNK = 1 << 20


def _keep(punct, R):
    if punct is None:
        return None
    m = torch.tensor(punct, dtype=torch.uint8)
    assert m.shape[0] == R
    return m


def llr_count(R, punct, s) -> int:
    """Kept values in stages [0, s)."""
    if punct is None:
        return s * R
    P = len(punct[0])
    per = sum(sum(row) for row in punct)
    part = sum(punct[r][p] for r in range(R) for p in range(s % P))
    return (s // P) * per + part


def n_stages_of(code, n_info, terminated=True) -> int:
    return n_info + (code["K"] - 1 if terminated else 0)


def code_rate(code, punct) -> float:
    """Info bits per transmitted coded bit."""
    R = len(code["polys"])
    if punct is None:
        return 1.0 / R
    P = len(punct[0])
    return P / sum(sum(row) for row in punct)


def sigma_for(ebn0_db, rate) -> float:
    return math.sqrt(1.0 / (2.0 * rate * 10.0 ** (ebn0_db / 10.0)))


def _gen(device, seed, chunk, salt):
    g = torch.Generator(device=device)
    g.manual_seed((int(seed) * 1000003 + int(chunk) * 7919 + salt) % (1 << 62))
    return g


def info_bits(seed, start, n, device="cpu") -> torch.Tensor:
    """Info bits [start, start+n) of stream `seed` (uint8 0/1)."""
    out = torch.empty(n, dtype=torch.uint8, device=device)
    if n <= 0:
        return out
    c0, c1 = start // BIT_CHUNK, (start + n - 1) // BIT_CHUNK
    for c in range(c0, c1 + 1):
        bits = torch.randint(0, 2, (BIT_CHUNK,), generator=_gen(device, seed, c, 11),
                             device=device, dtype=torch.uint8)
        a = max(start, c * BIT_CHUNK)
        b = min(start + n, (c + 1) * BIT_CHUNK)
        out[a - start:b - start] = bits[a - c * BIT_CHUNK:b - c * BIT_CHUNK]
    return out


def encode(x_ext: torch.Tensor, K: int, polys) -> torch.Tensor:
    """Encoder outputs for x_ext = [x_{s0-v} .. x_{s1-1}] -> [s1-s0, R] uint8.

    Stage t's coded bit r is XOR_{k=0..v} g^(r)_{v-k} x_{t-k} (Eq. 2 with the
    register convention c-1)."""
    v = K - 1
    n = x_ext.numel() - v
    R = len(polys)
    out = torch.zeros((n, R), dtype=torch.uint8, device=x_ext.device)
    for r, g in enumerate(polys):
        acc = torch.zeros(n, dtype=torch.uint8, device=x_ext.device)
        for k in range(v + 1):
            if (int(g) >> (v - k)) & 1:
                acc ^= x_ext[v - k:v - k + n]
        out[:, r] = acc
    return out


def _piece(code, n_info, sigma, seed, s0, s1, punct, hard, device, frac_bits, cs, ce):
    """Soft values of stages [s0, s1) inside noise chunk [cs, ce)."""
    K, polys = code["K"], code["polys"]
    R, v = len(polys), K - 1
    a, b = max(0, s0 - v), min(n_info, s1)
    x = torch.zeros(s1 - s0 + v, dtype=torch.uint8, device=device)
    if b > a:
        x[a - (s0 - v):b - (s0 - v)] = info_bits(seed, a, b - a, device)
    coded = encode(x, K, polys)                                  # [s1-s0, R]
    sym = 1.0 - 2.0 * coded.to(torch.float32)                    # BPSK 0 -> +1
    keep = _keep(punct, R)
    if keep is not None:
        P = keep.shape[1]
        cols = torch.arange(s0, s1, device=device) % P
        sym = sym[keep.to(device)[:, cols].t().bool()]
    else:
        sym = sym.reshape(-1)
    k0, k1 = llr_count(R, punct, cs), llr_count(R, punct, ce)
    c = cs // NOISE_CHUNK
    z = torch.randn(k1 - k0, generator=_gen(device, seed, c, 23), device=device)
    lo = llr_count(R, punct, s0) - k0
    y = sym + sigma * z[lo:lo + sym.numel()]
    if hard:
        return torch.where(y >= 0, 1, -1).to(torch.int8)
    return torch.clamp(torch.round(y * (1 << frac_bits)), -127, 127).to(torch.int8)


def make_window(code, n_info, ebn0_db, seed, s0, s1, punct=None, hard=False, terminated=True,
                device="cpu", frac_bits=5, out=None):
    """int8 soft values of stages [s0, s1) of the stream (kept positions only),
    i.e. exactly llr[llr_count(s0) : llr_count(s1)] of the whole stream.
    Generated piecewise (one noise chunk at a time) so any size fits."""
    R = len(code["polys"])
    n_stages = n_stages_of(code, n_info, terminated)
    assert 0 <= s0 <= s1 <= n_stages
    sigma = sigma_for(ebn0_db, code_rate(code, punct))
    n = llr_count(R, punct, s1) - llr_count(R, punct, s0)
    if out is None:
        out = torch.empty(n, dtype=torch.int8, device=device)
    assert out.numel() == n
    base = llr_count(R, punct, s0)
    for c in range(s0 // NOISE_CHUNK, (s1 - 1) // NOISE_CHUNK + 1 if s1 > s0 else 0):
        cs, ce = c * NOISE_CHUNK, min((c + 1) * NOISE_CHUNK, n_stages)
        a, b = max(s0, cs), min(s1, ce)
        if b <= a:
            continue
        piece = _piece(code, n_info, sigma, seed, a, b, punct, hard, device, frac_bits, cs, ce)
        i = llr_count(R, punct, a) - base
        out[i:i + piece.numel()] = piece
    return out


def make_stream(code, n_info, ebn0_db, seed, punct=None, hard=False, terminated=True,
                device="cpu", frac_bits=5):
    """(info bits uint8 [n_info], llr int8 [llr_count(n_stages)])."""
    n_stages = n_stages_of(code, n_info, terminated)
    info = info_bits(seed, 0, n_info, device)
    llr = make_window(code, n_info, ebn0_db, seed, 0, n_stages, punct, hard, terminated,
                      device, frac_bits)
    return info, llr
