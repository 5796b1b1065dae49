"""Continuous-stream decoding (pbvd_stream_*): soft
values pushed in pieces of random length (empty, one value, mid-stage,
many blocks at once) decode to exactly the oracle's segmented PBVD of the
whole stream -- the halo carried across calls must give every
block the geometry of the one-shot decode."""
import ctypes

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pbvd():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1608_00066_b200 import build
    build.build()
    import paper_1608_00066_b200 as P
    return P


def pieces(n, rng):
    """Random cut points: mostly mid-sized, with empty, 1-value and huge pieces."""
    cuts, pos = [0], 0
    while pos < n:
        r = rng.random()
        step = 0 if r < 0.05 else 1 if r < 0.15 else int(rng.integers(2, 3000)) if r < 0.9 \
            else int(rng.integers(3000, 60000))
        pos = min(n, pos + step)
        cuts.append(pos)
    return cuts


CASES = [
    # code, punct, n_info, D, L, terminated, ebn0
    ("k7", "1/2", 100000, 512, 42, True, 3.0),
    ("k7", "3/4", 30011, 96, 30, False, 4.0),
    ("k7", "2/3", 40000, 512, 42, True, 4.0),
    ("k9", "1/2", 40000, 1024, 64, True, 2.0),
    ("k7", "1/2", 9000, 64, 100, True, 3.0),     # D < L: several head blocks
    ("k3", "1/2", 4096, 256, 16, True, 4.0),
    ("k7", "1/2", 300, 512, 42, True, 3.0),      # shorter than one block
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "-".join(map(str, c)))
def test_stream_pieces_equal_one_shot(pbvd, orc, case):
    name, pk, n_info, D, L, term, ebn0 = case
    code, punct = synth.CODES[name], synth.PUNCT[pk]
    hard = name == "k3"
    info, llr = synth.make_stream(code, n_info, ebn0, 51, punct, hard, term)
    flags = orc.TERMINATED if term else 0
    want = orc.pack_bits(orc.decode(code, llr.numpy(), n_info, D, L, flags=flags, punct=punct))
    dec = pbvd.Decoder(code["K"], code["polys"], D, L, punct=punct, terminated=term)
    d = llr.cuda()
    rng = np.random.default_rng(n_info)
    sd = dec.open_stream()
    for rep in range(2):                       # the object takes a second stream after finish
        cuts = pieces(d.numel(), rng)
        outs, nbits = [], 0
        for a, b in zip(cuts[:-1], cuts[1:]):
            o = sd.push(d[a:b].clone())        # clone: the caller's buffer is not kept
            assert o.numel() * 8 % D == 0
            outs.append(o)
            nbits += o.numel() * 8
        tail, nt = sd.finish()
        assert nbits + nt == n_info
        got = torch.cat(outs + [tail]).cpu().numpy()
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, f"rep {rep}: {bad.size} bytes differ, first {bad[:8]}"
    sd.close()


def test_stream_output_too_small_consumes_nothing(pbvd, orc):
    code = synth.CODES["k7"]
    n_info, D, L = 5000, 512, 42
    info, llr = synth.make_stream(code, n_info, 3.0, 57)
    want = orc.pack_bits(orc.decode(code, llr.numpy(), n_info, D, L))
    dec = pbvd.Decoder(7, code["polys"], D, L)
    Lb = dec._L
    s = ctypes.c_void_p()
    assert Lb.pbvd_stream_open(dec._h, ctypes.byref(s)) == 0
    d = llr.cuda()
    out = torch.zeros(want.size + 8, dtype=torch.uint8, device="cuda")
    n = ctypes.c_int64()
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    half = d.numel() // 2
    # the first half completes blocks: a 0-byte buffer is refused and nothing is consumed
    assert Lb.pbvd_stream_push(s, d.data_ptr(), half, out.data_ptr(), 0, ctypes.byref(n), stream) == -5
    assert Lb.pbvd_stream_push(s, d.data_ptr(), half, out.data_ptr(), out.numel(), ctypes.byref(n),
                               stream) == 0
    k = n.value // 8
    assert k > 0
    assert Lb.pbvd_stream_push(s, d.data_ptr() + half, d.numel() - half, out.data_ptr() + k,
                               out.numel() - k, ctypes.byref(n), stream) == 0
    k += n.value // 8
    assert Lb.pbvd_stream_finish(s, out.data_ptr() + k, out.numel() - k, ctypes.byref(n), stream) == 0
    assert k * 8 + n.value == n_info
    Lb.pbvd_stream_close(s)
    assert (out[: want.size].cpu().numpy() == want).all()


def test_stream_finish_mid_stage_is_an_error(pbvd):
    code = synth.CODES["k7"]
    dec = pbvd.Decoder(7, code["polys"], 512, 42)
    sd = dec.open_stream()
    sd.push(torch.zeros(2 * 1000 + 1, dtype=torch.int8, device="cuda"))
    with pytest.raises(pbvd.PbvdError, match="inside a stage"):
        sd.finish()
    first = sd.push(torch.zeros(2 * 1000, dtype=torch.int8, device="cuda"))   # a new stream works
    out, n = sd.finish()
    assert first.numel() * 8 + n == 1000 - 6
