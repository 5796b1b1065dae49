"""Multi-GPU sharding logic on CPU: world-size-2 gloo process group, each
rank decodes its block range from its own soft window (here with the oracle
standing in for the GPU kernel) and the packed bits are gathered; the result
must equal the single-process decode bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from paper_1608_00066_b200 import shard as S


def test_plan_covers_stream_exactly():
    for n_info, D, L, world in [(20000, 512, 42, 2), (20000, 512, 42, 8), (1000, 64, 100, 3),
                                (4096, 256, 16, 4), (777, 8, 42, 5)]:
        shards = [S.plan(n_info, D, L, 7, True, world, r) for r in range(world)]
        assert shards[0].bit0 == 0 and shards[-1].bit1 == n_info
        for a, b in zip(shards, shards[1:]):
            assert a.bit1 == b.bit0 and a.block0 + a.nblocks == b.block0
        for sh in shards:
            if sh.nblocks:
                assert sh.stage0 == max(0, sh.block0 * D - L)
                assert sh.bit0 % 8 == 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    code, punct, n_info, D, L = cfg
    sh = S.plan(n_info, D, L, code["K"], True, world, rank)
    win = synth.make_window(code, n_info, 3.0, 11, sh.stage0, sh.stage1, punct)
    bits = O.decode(code, win.numpy(), n_info, D, L, punct=punct, b0=sh.block0,
                    nblk=sh.nblocks, window_stage0=sh.stage0, threads=1)
    local = torch.from_numpy(O.pack_bits(bits))
    full = S.gather_bits(local, sh, n_info, D)
    if rank == 0:
        q.put(full.numpy().tobytes())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_info", [16384, 10000])
def test_gloo_two_ranks_equal_single_decode(orc, n_info):
    code, punct, D, L = synth.CODES["k7"], synth.PUNCT["3/4"], 512, 42
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, (code, punct, n_info, D, L), q))
             for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    info, llr = synth.make_stream(code, n_info, 3.0, 11, punct)
    want = orc.pack_bits(orc.decode(code, llr.numpy(), n_info, D, L, punct=punct))
    assert np.frombuffer(got, dtype=np.uint8).tobytes() == want.tobytes()
