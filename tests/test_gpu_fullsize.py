"""Full-size BASELINE configs on the GPU, in the launch configuration bench.py
times (default lanes, whole-stream pbvd_decode), checked against the oracle
on every block (the oracle on all host cores, in block-range chunks), and
shard / determinism invariants that must hold at any size."""
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


def every_bit_parity(orc, code, punct, llr_dev, n_info, D, L, got_packed, chunk_blocks=1 << 18):
    """Every block against the oracle (SURVEY §8(c.iii) "GPU == oracle ...
    every block"), in block-range chunks so host memory stays bounded: each
    chunk's soft window (its spans, L-stage halos included) is copied from
    the device and decoded by the oracle on all host cores."""
    nb = -(-n_info // D)
    R, K = len(code["polys"]), code["K"]
    n_stages = n_info + K - 1
    for b0 in range(0, nb, chunk_blocks):
        nblk = min(chunk_blocks, nb - b0)
        lo = max(0, b0 * D - L)
        hi = n_stages if b0 + nblk == nb else min(n_stages, (b0 + nblk) * D + L)
        k0, k1 = synth.llr_count(R, punct, lo), synth.llr_count(R, punct, hi)
        win = llr_dev[k0:k1].cpu().numpy()
        want = orc.pack_bits(orc.decode(code, win, n_info, D, L, punct=punct, b0=b0, nblk=nblk,
                                        window_stage0=lo))
        t0, t1 = b0 * D, min((b0 + nblk) * D, n_info)
        got = got_packed[t0 // 8:(t1 + 7) // 8]
        diff = np.flatnonzero(got != want)
        assert diff.size == 0, f"blocks [{b0}, {b0 + nblk}): {diff.size} bytes differ, first at " \
                               f"byte {t0 // 8 + diff[0]} (block {(t0 + 8 * diff[0]) // D})"
    return nb


@pytest.mark.parametrize("cfg", ["C3a", "C3b", "C4"])
def test_config_full_size_every_bit(P, orc, cfg):
    c = synth.CONFIGS[cfg]
    code, punct = synth.CODES[c["code"]], synth.PUNCT[c["punct"]]
    info, llr = synth.make_stream(code, c["n_info"], c["ebn0"], c["seed"], punct, c["hard"],
                                  device="cuda")
    dec = P.Decoder(code["K"], code["polys"], c["D"], c["L"], punct=punct)
    out = dec.decode(llr, c["n_info"])
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    nb = every_bit_parity(orc, code, punct, llr, c["n_info"], c["D"], c["L"], got)
    assert nb == dec.block_count(c["n_info"])
    # plus the property that holds at any size: the decode recovers the info bits
    bits = np.unpackbits(got, bitorder="little")[:c["n_info"]]
    ber = (bits != info.cpu().numpy()).mean()
    assert ber < 1e-3


def test_c5_full_stream_every_bit(P, orc):
    """2^32 info bits (8 GiB of soft values; 40 GB of survivors through a
    4 GiB workspace whose regions the jobs of ONE fused launch recycle), all
    8,388,608 blocks against the oracle (~80 s of host cores)."""
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
    assert launches == 1           # one launch; its jobs recycle the workspace's regions
    got = out.cpu().numpy()
    del out
    nb = every_bit_parity(orc, code, punct, llr, n_info, c["D"], c["L"], got, chunk_blocks=1 << 20)
    assert nb == 1 << 23
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


@pytest.mark.parametrize("n_streams", [1, 3])
def test_host_pipeline_matches_oracle(P, orc, n_streams):
    """pbvd_decode_host (pinned host buffers, multi-stream H2D / decode / D2H,
    §IV.C) against the oracle, every bit: the C2 stream, a ragged
    D = 64 stream and a punctured one (segments of any size)."""
    cases = [("k7", "1/2", 1 << 24, 512, 42, 4.0, 1), ("k7", "1/2", 100_003, 64, 30, 3.5, 9),
             ("k7", "3/4", 3_000_001, 512, 42, 4.0, 5), ("k9", "1/2", 1 << 20, 1024, 64, 3.0, 2)]
    for cname, pname, n_info, D, L, ebn0, seed in cases:
        code, punct = synth.CODES[cname], synth.PUNCT[pname]
        info, llr = synth.make_stream(code, n_info, ebn0, seed, punct)
        dec = P.Decoder(code["K"], code["polys"], D, L, punct=punct)
        host = dec.decode_host(llr.pin_memory(), n_info, n_streams=n_streams).numpy()
        want = orc.pack_bits(orc.decode(code, llr.numpy(), n_info, D, L, punct=punct))
        assert np.array_equal(host, want), (cname, pname, n_info)


@pytest.mark.parametrize("fused,ws_mib,pname", [(True, 4, "1/2"), (True, 1, "1/2"), (True, 1, "3/4"),
                                                 (False, 4, "1/2"), (False, 4, "2/3")])
def test_small_workspace_matches_oracle(P, orc, fused, ws_mib, pname):
    """A survivor workspace smaller than the stream: the fused kernel runs ONE
    launch whose jobs recycle the workspace's regions (job gw -> region
    gw % regions once the region's previous job has traced back; 1 MiB = 6
    regions for 256 jobs), the two-kernel path runs many waves (interior-block
    groups, edges riding with the first / last).  Both are bit-exact against
    the oracle and against the one-wave decode."""
    code, punct = synth.CODES["k7"], synth.PUNCT[pname]
    n_info = 1 << 22
    info, llr = synth.make_stream(code, n_info, 3.0, 31, punct)
    want = orc.pack_bits(orc.decode(code, llr.numpy(), n_info, 512, 42, punct=punct))
    d_llr = llr.cuda()
    ref = P.Decoder(code["K"], code["polys"], 512, 42, punct=punct, fused=fused)
    one = ref.decode(d_llr, n_info).cpu().numpy()
    dec = P.Decoder(code["K"], code["polys"], 512, 42, punct=punct, fused=fused)
    dec.set_workspace_limit(ws_mib << 20)
    dec.set_profiling(True)
    got = dec.decode(d_llr, n_info)
    for _ in range(2):            # repeated launches reset the region counters
        got = dec.decode(d_llr, n_info, out=got)
    got = got.cpu().numpy()
    torch.cuda.synchronize()
    _, _, launches = dec.kernel_times()
    assert launches == 1 if fused else launches >= 16
    assert np.array_equal(one, want)
    assert np.array_equal(got, want)
