"""Pins of the CPU oracle against what the paper and the mathematics fix
(never against the CUDA path).  See DESIGN.md §4 for the pin table."""
import json
import math
import zlib
from pathlib import Path

import numpy as np
import pytest
import torch

import synth

GOLDEN = Path(__file__).resolve().parent / "golden"
K7 = synth.CODES["k7"]
K3 = synth.CODES["k3"]
K9 = synth.CODES["k9"]


def bits_of(s):
    return np.array([int(c) for c in s], dtype=np.uint8)


def vec(c, R):
    """alpha as printed in Table II, [c(1) c(2) ...] -> our bit r = c^(r+1)."""
    return sum(int(ch) << r for r, ch in enumerate(c))


# ------------------------------------------------------------------ trellis

def test_table2_reproduced(orc):
    """Table II: groups, their (alpha, beta, gamma, theta) and
    member states for the (2,1,7) code of P:376."""
    doc = json.loads((GOLDEN / "paper_table2.json").read_text())
    polys = tuple(int(p, 8) for p in doc["polys_octal"])
    got = {g["alpha"]: g for g in orc.classify(doc["K"], 2, polys)}
    assert len(got) == 4                      # N_c = 2^R groups
    for row in doc["groups"]:
        g = got[vec(row["alpha"], 2)]
        assert g["beta"] == vec(row["beta"], 2)
        assert g["gamma"] == vec(row["gamma"], 2)
        assert g["theta"] == vec(row["theta"], 2)
        assert sorted(g["states"]) == row["states"]


@pytest.mark.parametrize("code", [K3, K7, K9, {"K": 5, "polys": (0o23, 0o35)},
                                  {"K": 7, "polys": (0o133, 0o171, 0o165)},
                                  {"K": 6, "polys": (0o53, 0o75)}])
def test_eqs_4_to_6_closed_forms(orc, code):
    """Eqs. 4-6: beta = g_{K-1} ^ alpha, gamma = alpha ^ g_0,
    theta = g_{K-1} ^ alpha ^ g_0, for every butterfly -- the oracle's direct
    Eq. 2 evaluation must satisfy the paper's closed forms."""
    K, polys = code["K"], code["polys"]
    R = len(polys)
    gK = sum(((p >> (K - 1)) & 1) << r for r, p in enumerate(polys))
    g0 = sum((p & 1) << r for r, p in enumerate(polys))
    for j in range(1 << (K - 2)):
        a, b, g, t = orc.butterfly(K, R, polys, j)
        assert b == gK ^ a and g == a ^ g0 and t == gK ^ a ^ g0
        # Eq. 3: alpha depends only on D_{K-2}..D_1 of S_2j (x = 0, D_0 = 0)
        d = 2 * j
        expect = 0
        for r, p in enumerate(polys):
            bit = 0
            for i in range(1, K - 1):
                bit ^= ((d >> i) & 1) & ((p >> i) & 1)
            expect |= bit << r
        assert a == expect
    # equal group sizes (cosets of the linear map j -> alpha)
    sizes = {len(gr["states"]) for gr in orc.classify(K, R, polys)}
    assert len(sizes) == 1


def test_shift_and_ccsds_output(orc):
    """S_2j, S_2j+1 -> S_j (x=0), S_{j+2^{v-1}} (x=1); CCSDS state 0,
    x = 1 gives c = 11 (only the x term of Eq. 2 survives)."""
    for j in range(32):
        for b in (0, 1):
            assert orc.next_state(7, 2 * j + b, 0) == j
            assert orc.next_state(7, 2 * j + b, 1) == j + 32
    assert orc.out(7, 2, K7["polys"], 0, 1) == 0b11
    assert orc.out(7, 2, K7["polys"], 0, 0) == 0


def test_encoder_worked_example(orc):
    """the (7,5) code encodes 1011, terminated, to
    11 10 00 01 01 11.  Checked for the oracle's trellis walk and for the
    (independent) generator encoder."""
    want = "111000010111"
    info = [1, 0, 1, 1]
    d, got = 0, ""
    for x in info + [0, 0]:
        c = orc.out(3, 2, K3["polys"], d, x)
        got += f"{c & 1}{(c >> 1) & 1}"
        d = orc.next_state(3, d, x)
    assert got == want
    x_ext = torch.tensor([0, 0] + info + [0, 0], dtype=torch.uint8)
    enc = synth.encode(x_ext, 3, K3["polys"])
    assert "".join(str(int(b)) for b in enc.reshape(-1)) == want


def test_branch_metric_example(orc):
    """lambda = (+5, -3) gives BM(10) = 5, BM(01) = -3,
    BM(11) = 2, BM(00) = 0 (canonical BM, c-4).  The (7,5) path 1,0 from
    state 0 emits 11 then 10; the path 1,1 emits 11 then 01."""
    llr = np.array([5, -3, 5, -3], dtype=np.int8)
    assert orc.path_metric(K3, llr, 2, [0, 0], flags=0) == 0            # 00, 00
    assert orc.path_metric(K3, llr, 2, [1, 0], flags=0) == 2 + 5        # 11, 10
    assert orc.path_metric(K3, llr, 2, [1, 1], flags=0) == 2 - 3        # 11, 01


def test_traceback_step_example(orc):
    """Alg. 1 K2 / SPEC S:220: K = 7, state 37, sp = 1 ->
    predecessor 2*(37 mod 32)+1 = 11, emitted bit (37 >> 5) & 1 = 1."""
    assert orc.tb_step(7, 37, 1) == (11, 1)
    assert orc.tb_step(7, 37, 0) == (10, 1)
    assert orc.tb_step(7, 5, 1) == (11, 0)


def test_plan_examples(orc):
    """SPEC S:200-202 / P:93: 1536 stages, D=512, L=42 -> 3 blocks,
    interior span 596; 1000 stages, D=512 -> 2 blocks, last decodes 488."""
    nb, (t0, t1, lo, hi) = orc.plan(1536, 1536, 512, 42, 1)
    assert nb == 3 and (t0, t1, lo, hi) == (512, 1024, 470, 1066) and hi - lo == 596
    nb, (t0, t1, lo, hi) = orc.plan(1536, 1536, 512, 42, 0)
    assert (lo, hi) == (0, 554)
    nb, (t0, t1, lo, hi) = orc.plan(1000, 1000, 512, 42, 1)
    assert nb == 2 and t1 - t0 == 488 and hi == 1000
    nb, _ = orc.plan(512, 512, 512, 42, 0)
    assert nb == 1


# ----------------------------------------------------------------- decoder

def _golden_cases():
    return json.loads((GOLDEN / "survey_appendix_b.json").read_text())["cases"]


@pytest.mark.parametrize("case", _golden_cases(), ids=lambda c: c["name"])
def test_golden_vectors(orc, case):
    """exact bits, packed bytes, start states and
    tie counts under the readings c-1..c-22."""
    code = {"K": case["K"], "polys": tuple(int(p, 8) for p in case["polys_octal"])}
    flags = orc.TERMINATED if case["terminated"] else 0
    llr = np.array(case["llr"], dtype=np.int8)
    bits, starts, ties = orc.decode(code, llr, case["n_info"], case["D"], case["L"], flags=flags,
                                    punct=case["punct"], return_starts=True, return_ties=True)
    assert "".join(map(str, bits)) == case["decoded"]
    assert orc.pack_bits(bits).tobytes().hex() == case["packed_hex"]
    assert list(starts) == case["starts"]
    assert ties == case["ties"]
    fb, _ = orc.full(code, llr, case["n_info"], flags=flags, punct=case["punct"])
    assert "".join(map(str, fb)) == case["full_va"]
    assert int((bits != bits_of(case["info"])).sum()) == case["errors"]


ML_CASES = [
    (K3, None, False), (K3, None, True), (K7, None, False), (K7, None, True),
    (K7, synth.PUNCT["3/4"], False), (K7, synth.PUNCT["2/3"], False), (K9, None, False),
]


@pytest.mark.parametrize("code,punct,hard", ML_CASES)
@pytest.mark.parametrize("terminated", [True, False])
def test_full_viterbi_is_ml(orc, code, punct, hard, terminated):
    """§II: Viterbi is the ML sequence estimator.  On micro-frames the
    full-stream metric equals the brute-force minimum over all 2^k words and
    the bits equal the minimiser whenever it is unique."""
    # a stable seed (hash() of a str is randomised per process: PYTHONHASHSEED)
    rng = np.random.default_rng(zlib.crc32(repr((code["K"], hard, terminated, punct)).encode()))
    flags = orc.TERMINATED if terminated else 0
    R = len(code["polys"])
    for trial in range(12):
        k = int(rng.integers(3, 11))
        n_stages = k + (code["K"] - 1 if terminated else 0)
        n = orc.llr_count(R, punct, n_stages)
        if hard:
            llr = rng.choice([-1, 1], size=n).astype(np.int8)
        else:
            llr = rng.integers(-128, 128, size=n).astype(np.int8)
        best, nbest, mlbits = orc.ml(code, llr, k, flags=flags, punct=punct)
        fb, metric = orc.full(code, llr, k, flags=flags, punct=punct)
        assert metric == best
        assert orc.path_metric(code, llr, k, fb, flags=flags, punct=punct) == best
        if nbest == 1:
            assert (fb == mlbits).all()
        # one segmented block spanning everything is textbook Viterbi
        seg = orc.decode(code, llr, k, D=k, L=5, flags=flags, punct=punct, threads=1)
        assert (seg == fb).all()


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3a", "C3b", "C4"])
def test_noiseless_recovery(orc, cfg):
    """A noiseless codeword is recovered exactly by every block (the
    zero-distance path is the unique minimum for a non-catastrophic code),
    including D < L head blocks, a partial last block and no termination."""
    c = synth.CONFIGS[cfg]
    code, punct = synth.CODES[c["code"]], synth.PUNCT[c["punct"]]
    R = len(code["polys"])
    for n_info, D, L, term in [(3000, c["D"], c["L"], True), (1001, 64, 40, True),
                               (777, c["D"] // 4, c["L"], False)]:
        info, llr = synth.make_stream(code, n_info, 200.0, 9, punct, c["hard"], term)
        flags = orc.TERMINATED if term else 0
        bits = orc.decode(code, llr.numpy(), n_info, D, L, flags=flags, punct=punct)
        if term:
            assert (bits == info.numpy()).all()
        else:  # unterminated: last block has no merge margin; all others exact
            last0 = ((n_info - 1) // D) * D
            assert (bits[:last0] == info.numpy()[:last0]).all()


def test_pbvd_matches_full_va_at_5k(orc):
    """§III.A: with L about 5K the truncation/merge error is
    negligible -- at 4 dB over 10^6 bits the segmented decoder (D=512,
    L=42 = 6K) differs from full-stream Viterbi in < 0.1 x BER bits."""
    n = 1_000_000
    info, llr = synth.make_stream(K7, n, 4.0, 77)
    seg = orc.decode(K7, llr.numpy(), n, 512, 42)
    fb, _ = orc.full(K7, llr.numpy(), n)
    ber = (fb != info.numpy()).mean()
    diff = (seg != fb).mean()
    assert diff <= 0.1 * max(ber, 1e-6)


def test_generator_windows_are_slices():
    """Input generator: any window (a shard with halos) equals the same slice
    of the whole stream; llr_count matches the oracle's count."""
    code, punct = K7, synth.PUNCT["3/4"]
    n_info = 5000
    info, llr = synth.make_stream(code, n_info, 3.0, 5, punct)
    R = 2
    for s0, s1 in [(0, 100), (1234, 2222), (4990, n_info + 6)]:
        w = synth.make_window(code, n_info, 3.0, 5, s0, s1, punct)
        a, b = synth.llr_count(R, punct, s0), synth.llr_count(R, punct, s1)
        assert torch.equal(w, llr[a:b])
    from oracle import oracle
    assert oracle.llr_count(R, punct, n_info + 6) == llr.numel()


# ------------------------------------------------------ BER vs union bound

# Bit-weight spectrum B_d of the (171,133) code, d = 10..22 (SURVEY.md
# Appendix A item 2; the standard published spectrum).
B_D = {10: 36, 12: 211, 14: 1404, 16: 11633, 18: 77433, 20: 502690, 22: 3322763}


def union_bound(ebn0_db, rate=0.5):
    g = 10 ** (ebn0_db / 10)
    return sum(b * 0.5 * math.erfc(math.sqrt(d * rate * g)) for d, b in B_D.items())


@pytest.mark.slow
@pytest.mark.parametrize("ebn0,n_bits", [(4.0, 20_000_000), (4.5, 70_000_000)])
def test_ber_matches_union_bound(orc, ebn0, n_bits):
    """Soft-decision K=7 BER of the segmented decoder lies within
    [0.55, 1.25] x the union bound built from the code's distance spectrum
    (the bound is tight at these SNRs; 8-bit quantisation loses < 0.2 dB)."""
    errs, total = 0, 0
    chunk = 10_000_000
    seed = 1000 + int(ebn0 * 10)
    for i in range(0, n_bits, chunk):
        n = min(chunk, n_bits - i)
        info, llr = synth.make_stream(K7, n, ebn0, seed + i, None)
        bits = orc.decode(K7, llr.numpy(), n, 512, 42)
        errs += int((bits != info.numpy()).sum())
        total += n
    assert errs >= 150
    ratio = (errs / total) / union_bound(ebn0)
    assert 0.55 <= ratio <= 1.25, (errs, ratio)


# ---------------------------------------------- traceback start rules (c-10)
# The paper's own rule starts the traceback "from a random state (state S_0,
# for example)" with "no state estimation" (Alg. 1 K2 line
# `state = 0`); the build's default is the min-PM state.  Both
# are pinned here by brute force over every path of a block's window, with an
# encoder written out in the test (Eq. 2) -- independent of the oracle.

def _window_paths(code, n_stages, start_states):
    """Every input sequence x_ext = [initial state bits (v), inputs (n)] whose
    initial state is in start_states: (inputs [M, n], coded bits [M, n, R])."""
    K, polys = code["K"], code["polys"]
    v, R = K - 1, len(polys)
    n = n_stages
    seqs = ((np.arange(1 << (v + n))[:, None] >> np.arange(v + n)[None, :]) & 1).astype(np.uint8)
    # x_ext[k] for k < v is x_{-v+k}; the state before stage 0 is
    # (x_{-1} .. x_{-v}) with x_{-1} the MSB (c-1: next = (x << (v-1)) | (d >> 1))
    init = sum(seqs[:, v - 1 - i].astype(np.int64) << (v - 1 - i) for i in range(v))
    seqs = seqs[np.isin(init, list(start_states))]
    coded = np.zeros((seqs.shape[0], n, R), dtype=np.int64)
    for r, g in enumerate(polys):
        for k in range(v + 1):            # c_r(t) = XOR_k g_{v-k} x_{t-k}   (Eq. 2)
            if (g >> (v - k)) & 1:
                coded[:, :, r] ^= seqs[:, v - k:v - k + n]
    return seqs[:, v:], coded


def _end_state(inputs, v):
    # state after the last stage: the last v inputs, newest in the MSB
    n = inputs.shape[1]
    return sum(inputs[:, n - 1 - i].astype(np.int64) << (v - 1 - i) for i in range(v))


def _brute_block(code, lam, start_states, end_zero):
    """Minimum of M(path) = sum_s sum_r c_r lam_r (reading c-4) over the
    window's paths; -> (unique?, inputs of the minimiser)."""
    inputs, coded = _window_paths(code, lam.shape[0], start_states)
    if end_zero:
        keep = _end_state(inputs, code["K"] - 1) == 0
        inputs, coded = inputs[keep], coded[keep]
    metric = (coded * lam[None, :, :]).sum(axis=(1, 2))
    best = metric.min()
    hit = np.nonzero(metric == best)[0]
    return hit.size == 1, inputs[hit[0]]


@pytest.mark.parametrize("start_zero", [False, True])
def test_start_rules_interior_block_brute_force(orc, start_zero):
    """An interior block (lo > 0: all-zero initial metrics, P:93 -- any start
    state) decodes the bits of the minimum-metric window path that ends in
    the min-PM state or, with START_ZERO, in state S_0."""
    code, D, L = K3, 8, 2
    v = code["K"] - 1
    rng = np.random.default_rng(2024 + int(start_zero))
    flags = orc.START_ZERO if start_zero else 0
    checked = 0
    for trial in range(40):
        n_info = 5 * D
        llr = rng.integers(-128, 128, size=2 * n_info).astype(np.int8)
        bits = orc.decode(code, llr, n_info, D, L, flags=flags, threads=1)
        for b in (1, 2, 3):                        # interior: lo = bD - L > 0
            t0, lo, hi = b * D, b * D - L, b * D + D + L
            lam = llr[2 * lo:2 * hi].reshape(-1, 2).astype(np.int64)
            unique, x = _brute_block(code, lam, range(1 << v), start_zero)
            if unique:
                checked += 1
                assert (bits[t0:t0 + D] == x[t0 - lo:t0 - lo + D]).all(), (trial, b)
    assert checked >= 60


def test_start_zero_single_block_is_constrained_ml(orc):
    """One head block spanning an unterminated stream (known start state 0,
    c-12) with the S_0 start decodes the ML word among those ending in state
    0, i.e. whose last v bits are 0."""
    for code in (K3, {"K": 4, "polys": (0o13, 0o15)}):
        v = code["K"] - 1
        rng = np.random.default_rng(7 + code["K"])
        checked = 0
        for trial in range(30):
            n = 11
            llr = rng.integers(-128, 128, size=2 * n).astype(np.int8)
            got = orc.decode(code, llr, n, D=16, L=3, flags=orc.START_ZERO, threads=1)
            unique, x = _brute_block(code, llr.reshape(-1, 2).astype(np.int64), [0], True)
            if unique:
                checked += 1
                assert (got == x).all() and not x[n - v:].any(), trial
        assert checked >= 20


def test_start_rules_differ_and_start_zero_recovers_noiseless(orc):
    """The S_0 branch matters (bits differ from min-PM at short L and low
    SNR), and with L = 5K ("typically equal to 5K") it recovers a
    noiseless codeword exactly, like min-PM."""
    code = K7
    n_info, D = 20000, 512
    info, llr = synth.make_stream(code, n_info, 1.0, 31)
    a = orc.decode(code, llr.numpy(), n_info, D, 8)
    b = orc.decode(code, llr.numpy(), n_info, D, 8, flags=orc.TERMINATED | orc.START_ZERO)
    assert (a != b).sum() > 0
    for cfg in ("C1", "C2", "C3a", "C4"):
        c = synth.CONFIGS[cfg]
        code, punct = synth.CODES[c["code"]], synth.PUNCT[c["punct"]]
        info, llr = synth.make_stream(code, 5000, 200.0, 3, punct, c["hard"])
        got = orc.decode(code, llr.numpy(), 5000, c["D"] // 2, 5 * code["K"],
                         flags=orc.TERMINATED | orc.START_ZERO, punct=punct)
        assert (got == info.numpy()).all(), cfg
