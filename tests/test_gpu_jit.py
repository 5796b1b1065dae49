"""GPU parity of the run-time (NVRTC) kernels: codes that are not compiled
into libpbvd.so (SURVEY §8(f) NEXT 4 -- any generator polynomials, K 3..12,
R 2..4, degenerate groupings) decoded through the C ABI and compared with the
CPU oracle bit for bit.  The oracle is code-generic (it evaluates Eq. 2,
P:128-133, per edge), so these codes are pinned exactly like the compiled
ones."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

# (name, K, polys, punct, D, L, n_info, ebn0, flags-catastrophic)
JIT_CODES = [
    ("k7-133-171", 7, (0o133, 0o171), None, 512, 42, 20000, 3.0),         # CCSDS, swapped order
    ("k5-gsm", 5, (0o23, 0o33), None, 256, 30, 15000, 3.0),               # GSM TCH/FS
    ("k9-is95", 9, (0o561, 0o753), None, 512, 64, 12000, 3.0),            # IS-95 / CDMA2000
    ("k9-r3-perm", 9, (0o711, 0o557, 0o663), None, 1024, 64, 10000, 2.0),  # C4 code, permuted
    ("k7-r4", 7, (0o117, 0o127, 0o155, 0o171), None, 256, 42, 10000, 1.0),  # rate 1/4
    ("k4", 4, (0o15, 0o17), None, 128, 24, 9000, 3.0),                    # 8 states
    ("k6", 6, (0o53, 0o75), None, 256, 36, 9000, 3.0),                    # 32 states
    ("k8", 8, (0o247, 0o371), None, 512, 48, 9000, 3.0),                  # 128 states
    ("k3-r3", 3, (0o5, 0o7, 0o7), None, 64, 16, 6000, 2.0),               # rank-2 grouping (dup poly)
    ("k7-133-171-3/4", 7, (0o133, 0o171), ((1, 1, 0), (1, 0, 1)), 512, 42, 12000, 4.0),
    ("k10", 10, (0o1467, 0o1751), None, 256, 50, 6000, 3.0),              # 512 states, 8 lanes
    ("k11", 11, (0o3345, 0o3613), None, 256, 56, 5000, 3.0),              # 1024 states, 16 lanes
    ("k12", 12, (0o5723, 0o6265), None, 256, 60, 5000, 3.0),              # 2048 states, a pair per warp
    ("k12-r3", 12, (0o5723, 0o6265, 0o7173), None, 128, 60, 3000, 2.0),
]


@pytest.fixture(scope="module")
def pbvd():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1608_00066_b200 import build
    build.build()
    # NVRTC-build every code of this module in parallel processes first (a
    # cache hit is a no-op): ~1 min on 16 cores instead of ~7 min one by one
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    subprocess.run([sys.executable, str(root / "tools" / "jit_prebuild.py")], cwd=root,
                   capture_output=True, timeout=1800)
    import paper_1608_00066_b200 as P
    return P


def _check(P, orc, code, punct, n_info, D, L, ebn0, seed, lanes=0, allow=False, term=True):
    info, llr = synth.make_stream(code, n_info, ebn0, seed, punct, False, term)
    flags = orc.TERMINATED if term else 0
    want = orc.pack_bits(orc.decode(code, llr.numpy(), n_info, D, L, flags=flags, punct=punct))
    d = llr.cuda()
    for fused in (True, False):
        dec = P.Decoder(code["K"], code["polys"], D, L, punct=punct, terminated=term,
                        lanes=lanes, fused=fused, allow_catastrophic=allow)
        assert dec.info()["jit"] == 1
        got = dec.decode(d, n_info).cpu().numpy()
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, f"fused={fused} lanes={lanes}: {bad.size} bytes differ, first {bad[:8]}"
    return info, got


@pytest.mark.parametrize("case", JIT_CODES, ids=lambda c: c[0])
def test_jit_code_bit_exact(pbvd, orc, case):
    name, K, polys, punct, D, L, n_info, ebn0 = case
    code = {"K": K, "polys": polys}
    assert all(tuple(p) != polys for (k, r, p, w) in pbvd.supported() if k == K)
    with pytest.raises(pbvd.PbvdError, match="shape"):
        pbvd.Decoder(K, polys, D, L, punct=punct, lanes=64)
    _check(pbvd, orc, code, punct, n_info, D, L, ebn0, 23)
    # unterminated stream with a partial last block
    _check(pbvd, orc, code, punct, n_info - 5, D, L, ebn0, 29, term=False)


@pytest.mark.parametrize("lanes", [1, 2, 4])
def test_jit_lane_variants(pbvd, orc, lanes):
    """Every lane shape of a 64-state JIT code (1: 64 states per lane ... 4:
    two of six butterfly phases across lanes)."""
    code = {"K": 7, "polys": (0o133, 0o171)}
    _check(pbvd, orc, code, None, 20000, 512, 42, 3.0, 31, lanes=lanes)


def test_jit_catastrophic_override(pbvd, orc):
    """No generator has the g_0 tap: rejected unless PBVD_ALLOW_CATASTROPHIC
    (warning-class); with the flag the decode is still exactly
    the oracle's segmented Viterbi (ties included)."""
    code = {"K": 5, "polys": (0o22, 0o36)}
    with pytest.raises(pbvd.PbvdError, match="ALLOW_CATASTROPHIC"):
        pbvd.Decoder(code["K"], code["polys"], 128, 20)
    _check(pbvd, orc, code, None, 5000, 128, 20, 3.0, 37, allow=True)


def test_jit_full_size_sampled(pbvd, orc):
    """A JIT code at a C2-sized stream (2^24 bits, several waves of warps):
    sampled blocks against the oracle, decode works (BER)."""
    code = {"K": 7, "polys": (0o133, 0o171)}
    n_info, D, L = 1 << 24, 512, 42
    info, llr = synth.make_stream(code, n_info, 4.0, 41, None, False, True, device="cuda")
    dec = pbvd.Decoder(7, code["polys"], D, L)
    got = dec.decode(llr, n_info).cpu().numpy()
    host = llr.cpu().numpy()
    nb = n_info // D
    rng = np.random.default_rng(3)
    for b in sorted(set([0, 1, nb - 1] + list(rng.integers(0, nb, 40)))):
        want = orc.pack_bits(orc.decode(code, host, n_info, D, L, b0=int(b), nblk=1))
        assert (got[b * D // 8:(b + 1) * D // 8] == want).all(), b
    ber = (np.unpackbits(got, bitorder="little")[:n_info] != info.cpu().numpy()).mean()
    assert ber < 1e-4
