"""Full-size BASELINE configs on the GPU, in the launch configuration bench.py
times (default lanes, whole-stream pbvd_decode), checked against the oracle
on sampled blocks (every block the oracle can afford: the first and last
blocks of the stream plus a seeded random sample), and shard / determinism
invariants that must hold at any size."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1608_00066_b200 import build
    build.build()
    import paper_1608_00066_b200 as P
    return P


def sampled_parity(orc, code, punct, llr_dev, n_info, D, L, got_packed, nsample, seed):
    """Oracle on whole blocks: first 4, last 4 and `nsample` random ones."""
    nb = -(-n_info // D)
    rng = np.random.default_rng(seed)
    blocks = sorted(set(list(range(min(4, nb))) + list(range(max(0, nb - 4), nb)) +
                        list(rng.integers(0, nb, size=nsample))))
    R = len(code["polys"])
    K = code["K"]
    n_stages = n_info + K - 1
    got_bits = got_packed  # packed uint8 tensor on the host
    for b in blocks:
        t0, t1 = b * D, min(b * D + D, n_info)
        lo = max(0, t0 - L)
        hi = n_stages if b == nb - 1 else min(n_stages, t1 + L)
        k0, k1 = synth.llr_count(R, punct, lo), synth.llr_count(R, punct, hi)
        win = llr_dev[k0:k1].cpu().numpy()
        want = orc.decode(code, win, n_info, D, L, punct=punct, b0=b, nblk=1,
                          window_stage0=lo, threads=1)
        got = np.unpackbits(got_bits[t0 // 8:(t1 + 7) // 8], bitorder="little")[:t1 - t0]
        assert (got == want).all(), f"block {b}"
    return len(blocks)


@pytest.mark.parametrize("cfg", ["C3a", "C3b", "C4"])
def test_config_full_size_sampled(P, orc, cfg):
    c = synth.CONFIGS[cfg]
    code, punct = synth.CODES[c["code"]], synth.PUNCT[c["punct"]]
    info, llr = synth.make_stream(code, c["n_info"], c["ebn0"], c["seed"], punct, c["hard"],
                                  device="cuda")
    dec = P.Decoder(code["K"], code["polys"], c["D"], c["L"], punct=punct)
    out = dec.decode(llr, c["n_info"])
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    n = sampled_parity(orc, code, punct, llr, c["n_info"], c["D"], c["L"], got, 400, 7)
    assert n > 400
    bits = np.unpackbits(got, bitorder="little")[:c["n_info"]]
    ber = (bits != info.cpu().numpy()).mean()
    assert ber < 1e-3


def test_c5_full_stream_sampled(P, orc):
    """2^32 info bits (8 GiB of soft values) in survivor-workspace waves."""
    c = synth.CONFIGS["C5"]
    code, punct = synth.CODES[c["code"]], None
    n_info = c["n_info"]
    n_stages = n_info + code["K"] - 1
    llr = synth.make_window(code, n_info, c["ebn0"], c["seed"], 0, n_stages, punct,
                            device="cuda")
    dec = P.Decoder(code["K"], code["polys"], c["D"], c["L"])
    dec.set_profiling(True)
    out = dec.decode(llr, n_info)
    torch.cuda.synchronize()
    f, t, launches = dec.kernel_times()
    assert launches > 2            # the stream runs in several waves
    got = out.cpu().numpy()
    sampled_parity(orc, code, punct, llr, n_info, c["D"], c["L"], got, 300, 11)
    info_tail = synth.info_bits(c["seed"], n_info - (1 << 20), 1 << 20, "cuda").cpu().numpy()
    tail = np.unpackbits(got[-(1 << 17):], bitorder="little")
    assert (tail != info_tail).mean() < 1e-4


@pytest.mark.parametrize("cfg,nshards", [("C2", 3), ("C3b", 4), ("C4", 2)])
def test_block_range_shards_equal_one_shot(P, cfg, nshards):
    """pbvd_decode_blocks over contiguous ranges, each from its own soft window
    (the multi-GPU decomposition), equals the one-shot decode byte for byte."""
    from paper_1608_00066_b200 import shard as S
    c = synth.CONFIGS[cfg]
    code, punct = synth.CODES[c["code"]], synth.PUNCT[c["punct"]]
    n_info = min(c["n_info"], 1 << 22)
    info, llr = synth.make_stream(code, n_info, c["ebn0"], c["seed"], punct, c["hard"],
                                  device="cuda")
    dec = P.Decoder(code["K"], code["polys"], c["D"], c["L"], punct=punct)
    whole = dec.decode(llr, n_info).cpu()
    parts = []
    R = len(code["polys"])
    for r in range(nshards):
        sh = S.plan(n_info, c["D"], c["L"], code["K"], True, nshards, r)
        k0, k1 = synth.llr_count(R, punct, sh.stage0), synth.llr_count(R, punct, sh.stage1)
        win = llr[k0:k1].clone()          # a separate buffer, as on another GPU
        parts.append(dec.decode_blocks(win, sh.stage0, n_info, sh.block0, sh.nblocks).cpu())
    assert torch.equal(torch.cat(parts), whole)


def test_deterministic_and_lane_invariant(P):
    c = synth.CONFIGS["C2"]
    code = synth.CODES["k7"]
    n_info = 1 << 22
    info, llr = synth.make_stream(code, n_info, 3.0, 123, device="cuda")
    outs = []
    for lanes in (1, 2, 4, 2):
        dec = P.Decoder(code["K"], code["polys"], c["D"], c["L"], lanes=lanes)
        outs.append(dec.decode(llr, n_info).cpu())
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


def test_host_pipeline_matches_device_path(P):
    """pbvd_decode_host (pinned host buffers, multi-stream) == pbvd_decode."""
    code = synth.CODES["k7"]
    for n_info, D, L in [(1 << 21, 512, 42), (100_003, 64, 30)]:
        info, llr = synth.make_stream(code, n_info, 3.5, 9)
        dec = P.Decoder(code["K"], code["polys"], D, L)
        dev = dec.decode(llr.cuda(), n_info).cpu()
        host = dec.decode_host(llr.pin_memory(), n_info, n_streams=3)
        assert torch.equal(host, dev)


@pytest.mark.parametrize("fused", [True, False])
def test_many_waves_equal_one_wave(P, fused):
    """A small survivor-workspace limit splits the decode into many waves
    (interior-block groups, edges riding with the first / last); the bits are
    identical to a one-wave decode."""
    code = synth.CODES["k7"]
    n_info = 1 << 22
    info, llr = synth.make_stream(code, n_info, 3.0, 31, device="cuda")
    ref = P.Decoder(code["K"], code["polys"], 512, 42, fused=fused)
    want = ref.decode(llr, n_info).cpu()
    dec = P.Decoder(code["K"], code["polys"], 512, 42, fused=fused)
    dec.set_workspace_limit(8 << 20)
    dec.set_profiling(True)
    got = dec.decode(llr, n_info).cpu()
    torch.cuda.synchronize()
    _, _, launches = dec.kernel_times()
    assert launches >= 8
    assert torch.equal(got, want)
