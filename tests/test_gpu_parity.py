"""GPU parity: libpbvd.so (through the C ABI) vs the CPU oracle, bit-exact.

Every input is seeded synthetic data from synth/ (DESIGN.md §6); expected
values come only from oracle/."""
import json
from pathlib import Path

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def pbvd():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1608_00066_b200 import build
    build.build()
    import paper_1608_00066_b200 as P
    return P


def gpu_decode(P, code, llr, n_info, D, L, punct=None, terminated=True, lanes=0, fused=True,
               start_zero=False):
    dec = P.Decoder(code["K"], code["polys"], D, L, punct=punct, terminated=terminated,
                    lanes=lanes, fused=fused, start_zero=start_zero)
    d = llr.to("cuda") if not llr.is_cuda else llr
    out = dec.decode(d, n_info)
    torch.cuda.synchronize()
    return out.cpu().numpy(), dec


def unpack(b, n):
    return np.unpackbits(b, bitorder="little")[:n]


def lane_variants(P, code):
    return sorted({l for (K, R, polys, l) in P.supported()
                   if K == code["K"] and tuple(polys) == tuple(code["polys"])})


@pytest.mark.parametrize("case", json.loads((GOLDEN / "survey_appendix_b.json").read_text())["cases"],
                         ids=lambda c: c["name"])
def test_golden_vectors_gpu(pbvd, orc, case):
    if case["D"] % 8:
        pytest.skip("the C ABI requires D % 8 == 0 (blocks own whole output bytes)")
    code = {"K": case["K"], "polys": tuple(int(p, 8) for p in case["polys_octal"])}
    llr = torch.tensor(case["llr"], dtype=torch.int8)
    for lanes in lane_variants(pbvd, code):
        for fused in (True, False):
            got, _ = gpu_decode(pbvd, code, llr, case["n_info"], case["D"], case["L"],
                                case["punct"], case["terminated"], lanes, fused)
            assert got.tobytes().hex() == case["packed_hex"], (lanes, fused)


SMALL = [
    # code, punct, hard, n_info, D, L, terminated, ebn0
    ("k3", "1/2", True, 4096, 256, 16, True, 4.0),            # C1 exactly
    ("k3", "1/2", True, 5000, 64, 20, False, 2.0),
    ("k7", "1/2", False, 20000, 512, 42, True, 4.0),
    ("k7", "1/2", False, 33333, 128, 42, True, 2.0),
    ("k7", "1/2", False, 9000, 64, 100, True, 3.0),           # D < L: several head blocks
    ("k7", "1/2", False, 12345, 512, 42, False, 3.0),         # partial last block, no tail
    ("k7", "2/3", False, 20000, 512, 42, True, 4.0),
    ("k7", "3/4", False, 20011, 512, 42, True, 4.0),
    ("k7", "3/4", False, 7777, 96, 30, False, 3.0),
    ("k9", "1/2", False, 30000, 1024, 64, True, 3.0),
    ("k9", "1/2", False, 9999, 256, 40, False, 2.0),
    ("k7", "1/2", False, 40, 8, 8, True, 1.0),
    ("k7", "1/2", False, 8, 8, 42, True, 1.0),                # a single block
]


@pytest.mark.parametrize("cfg", SMALL, ids=lambda c: "-".join(map(str, c)))
def test_small_streams_bit_exact(pbvd, orc, cfg):
    name, pk, hard, n_info, D, L, term, ebn0 = cfg
    code, punct = synth.CODES[name], synth.PUNCT[pk]
    info, llr = synth.make_stream(code, n_info, ebn0, 17, punct, hard, term)
    flags = orc.TERMINATED if term else 0
    want = orc.pack_bits(orc.decode(code, llr.numpy(), n_info, D, L, flags=flags, punct=punct))
    for lanes in lane_variants(pbvd, code):
        for fused in (True, False):
            got, _ = gpu_decode(pbvd, code, llr, n_info, D, L, punct, term, lanes, fused)
            assert got.shape == want.shape
            bad = np.nonzero(got != want)[0]
            assert bad.size == 0, (f"lanes={lanes} fused={fused}: {bad.size} bytes differ, "
                                   f"first at {bad[:8]}")


@pytest.mark.parametrize("K,D,L", [(7, 8, 8), (7, 16, 16), (7, 64, 64), (7, 64, 128), (7, 8, 16),
                                   (3, 16, 16), (9, 32, 64)])
def test_L_multiple_of_D(pbvd, orc, K, D, L):
    """L % D == 0: block L/D spans from stage 0, so it is a head block with
    the known start state (reading c-12), not an interior block with zero
    initial metrics.  Low SNR and several seeds, so the two starting rules
    would give different bits (51 of 200 streams differ)."""
    code = synth.CODES[{3: "k3", 7: "k7", 9: "k9"}[K]]
    for seed in range(1, 9):
        n_info = 6 * max(D, L) + 8 * seed
        info, llr = synth.make_stream(code, n_info, 0.5, 100 + seed)
        want = orc.pack_bits(orc.decode(code, llr.numpy(), n_info, D, L))
        for fused in (True, False):
            got, _ = gpu_decode(pbvd, code, llr, n_info, D, L, fused=fused)
            assert (got == want).all(), (seed, fused, np.nonzero(got != want)[0][:8])


@pytest.mark.parametrize("cfg", SMALL[:11], ids=lambda c: "-".join(map(str, c)))
def test_start_zero_bit_exact(pbvd, orc, cfg):
    """PBVD_START_ZERO, the paper's own traceback start ("state S_0";
    Alg. 1 K2 state = 0): every block traces back from state 0.  Against
    the oracle's START_ZERO (pinned in tests/test_oracle.py)."""
    name, pk, hard, n_info, D, L, term, ebn0 = cfg
    code, punct = synth.CODES[name], synth.PUNCT[pk]
    info, llr = synth.make_stream(code, n_info, ebn0 - 2.0, 23, punct, hard, term)
    flags = (orc.TERMINATED if term else 0) | orc.START_ZERO
    want = orc.pack_bits(orc.decode(code, llr.numpy(), n_info, D, L, flags=flags, punct=punct))
    for lanes in lane_variants(pbvd, code):
        for fused in (True, False):
            got, _ = gpu_decode(pbvd, code, llr, n_info, D, L, punct, term, lanes, fused,
                                start_zero=True)
            bad = np.nonzero(got != want)[0]
            assert bad.size == 0, (lanes, fused, bad[:8])


@pytest.mark.parametrize("K,D,L", [(7, 64, 6), (7, 64, 10), (9, 128, 8), (3, 32, 3)])
def test_start_zero_differs_from_min_pm(pbvd, orc, K, D, L):
    """At short L and low SNR the two traceback starts give different bits
    (Fig. 4's S_0 curve lies above the min-PM one), so
    the flag is really taken -- and each GPU start equals the oracle's."""
    code = synth.CODES[{3: "k3", 7: "k7", 9: "k9"}[K]]
    n_info = 40 * D
    info, llr = synth.make_stream(code, n_info, 1.0, 77)
    outs = {}
    for sz in (False, True):
        flags = orc.TERMINATED | (orc.START_ZERO if sz else 0)
        want = orc.pack_bits(orc.decode(code, llr.numpy(), n_info, D, L, flags=flags))
        for fused in (True, False):
            got, _ = gpu_decode(pbvd, code, llr, n_info, D, L, fused=fused, start_zero=sz)
            assert (got == want).all(), (sz, fused)
        outs[sz] = want
    assert (outs[True] != outs[False]).any()


def test_saturated_and_extreme_inputs(pbvd, orc):
    """int8 extremes (-128 included) and all-erasure input (every ACS ties)."""
    code = synth.CODES["k7"]
    n_info, D, L = 5000, 256, 42
    n = orc.llr_count(2, None, n_info + 6)
    rng = np.random.default_rng(5)
    cases = [rng.choice([-128, 127], size=n), np.zeros(n), rng.integers(-128, 128, size=n)]
    for arr in cases:
        llr = torch.tensor(arr.astype(np.int8))
        want = orc.pack_bits(orc.decode(code, llr.numpy(), n_info, D, L))
        for lanes in lane_variants(pbvd, code):
            for fused in (True, False):
                got, _ = gpu_decode(pbvd, code, llr, n_info, D, L, lanes=lanes, fused=fused)
                assert (got == want).all(), (lanes, fused)


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_config_full_size_bit_exact(pbvd, orc, cfg):
    """BASELINE configs C1 and C2 at full size, every bit against the oracle."""
    c = synth.CONFIGS[cfg]
    code, punct = synth.CODES[c["code"]], synth.PUNCT[c["punct"]]
    info, llr = synth.make_stream(code, c["n_info"], c["ebn0"], c["seed"], punct, c["hard"],
                                  device="cuda")
    want = orc.pack_bits(orc.decode(code, llr.cpu().numpy(), c["n_info"], c["D"], c["L"],
                                    punct=punct))
    for fused in (True, False):
        got, _ = gpu_decode(pbvd, code, llr, c["n_info"], c["D"], c["L"], punct, fused=fused)
        assert (got == want).all(), fused
    # and the decoder actually decodes: BER in the expected range
    ber = (unpack(got, c["n_info"]) != info.cpu().numpy()).mean()
    assert ber < (2e-2 if c["hard"] else 1e-4)


def test_compute_sanitizer_memcheck_clean(pbvd):
    """memcheck over a small decode of each kernel family (edge blocks, lane
    stages, punctured input) reports no error and stays bit-exact."""
    import shutil
    import subprocess
    import sys
    from pathlib import Path
    import os
    if os.environ.get("PBVD_SANITIZER_TEST") != "1":
        # the GPU pool refuses compute-sanitizer runs (they have left GPUs
        # needing a reset); the builder-run captures are in profiles/*_sanitizers.txt
        pytest.skip("compute-sanitizer runs are closed on this GPU pool (opt in: PBVD_SANITIZER_TEST=1)")
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not Path(cs).exists():
        pytest.skip("compute-sanitizer not available")
    root = Path(__file__).resolve().parents[1]
    for args in (["k7", "3000", "64", "20", "2"], ["k7", "2000", "96", "30", "4", "3/4"],
                 ["k9", "1500", "64", "20", "8"], ["k7", "3000", "64", "20", "2", "1/2", "0"],
                 ["k3", "3000", "64", "20", "1"]):
        r = subprocess.run([cs, "--tool", "memcheck", "--error-exitcode", "9", sys.executable,
                            str(root / "tools" / "debug_case.py"), *args],
                           capture_output=True, text=True, timeout=600, cwd=root)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
        assert "bad bytes: 0" in r.stdout


@pytest.mark.parametrize("fused", [True, False])
def test_odd_aligned_soft_pointer(pbvd, orc, fused):
    """The R = 2 forward kernel reads a stage's two soft bytes with one 16-bit
    load; a caller buffer at an odd address is realigned by the library and
    decodes bit-exactly (whole stream and a block-range window)."""
    code = synth.CODES["k7"]
    n_info, D, L = 20000, 512, 42
    info, llr = synth.make_stream(code, n_info, 3.0, 77)
    want = orc.pack_bits(orc.decode(code, llr.numpy(), n_info, D, L))
    buf = torch.empty(llr.numel() + 1, dtype=torch.int8, device="cuda")
    buf[1:].copy_(llr.cuda())
    odd = buf[1:]
    assert odd.data_ptr() % 2 == 1
    dec = pbvd.Decoder(code["K"], code["polys"], D, L, fused=fused)
    got = dec.decode(odd, n_info).cpu().numpy()
    assert (got == want).all()
    # a block range from an odd window start (stage 2*D - L)
    b0, nb = 2, 10
    lo = b0 * D - L
    hi = (b0 + nb) * D + L
    win = buf[1 + 2 * lo: 1 + 2 * hi]
    part = dec.decode_blocks(win, lo, n_info, b0, nb).cpu().numpy()
    assert (part == want[b0 * D // 8:(b0 + nb) * D // 8]).all()
