"""bench.py contract on one GPU: the N = 1 JSON line, and the N > 1 control
flow (block-range shards, barrier, max-over-ranks timing, final gather) with
two torchrun ranks sharing cuda:0 over gloo (PBVD_BENCH_BACKEND=gloo; the
real multi-GPU run uses NCCL)."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches",
        "clocks", "parity")


def _line(out):
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


@pytest.fixture(scope="module")
def gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_bench_single_gpu_contract(gpu):
    r = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3",
                        "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    for k in KEYS:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["parity"]["bit_exact"]
    assert d["parity"]["blocks_checked"] == d["parity"]["blocks_total"] == 32768   # every block
    assert d["clocks"]["samples"] >= 5 and d["clocks"]["sm_mhz"]
    assert d["roofline"]["bound"] == "alu" and 0 < d["roofline"]["frac"] < 1
    assert d["e2e"]["matches_device_path"] and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 3


def test_bench_two_ranks_gloo(gpu):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, PBVD_BENCH_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        str(port), "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3",
                        "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True,
                       timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _line(r.stdout)
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0
    # rank 0 checked the GATHERED stream, both ranks' blocks, against the oracle
    assert d["parity"]["bit_exact"] and d["parity"]["blocks_checked"] == 65536
    assert d["t_G"]["decode_ms"] > 0 and d["t_G"]["gather_ms"] >= 0
    assert "x2" in d["config"]["parallelism"]
    # the default gather: fused into the traceback over CUDA IPC, verified
    # against an NCCL/gloo all_gather after the warm-up (else it falls back)
    assert d["run"]["gather"].startswith("fused"), d["run"]["gather"]


def test_mirrored_outputs_match_oracle(gpu, orc):
    """pbvd_decode_blocks_mirrored: the traceback's stores land identically in
    every destination (here: two more local buffers at odd 4-byte offsets),
    for fused and two-kernel mode and a range with edge blocks -- every
    destination equal to the oracle's bits."""
    sys.path.insert(0, str(ROOT))
    import synth
    import paper_1608_00066_b200 as P
    code = synth.CODES["k7"]
    n_info, D, L = 100000, 512, 42
    info, llr = synth.make_stream(code, n_info, 3.0, 61, device="cuda")
    want = torch.from_numpy(orc.pack_bits(orc.decode(code, llr.cpu().numpy(), n_info, D, L))).cuda()
    for fused in (True, False):
        dec = P.Decoder(7, code["polys"], D, L, fused=fused)
        nb = dec.block_count(n_info)
        out = torch.zeros(want.numel(), dtype=torch.uint8, device="cuda")
        m1 = torch.zeros(want.numel() + 4, dtype=torch.uint8, device="cuda")
        m2 = torch.zeros(want.numel() + 8, dtype=torch.uint8, device="cuda")
        dec.decode_blocks_mirrored(llr, 0, n_info, 0, nb, out,
                                   [m1.data_ptr() + 4, m2.data_ptr() + 8])
        torch.cuda.synchronize()
        assert torch.equal(out, want)
        assert torch.equal(m1[4:], want) and torch.equal(m2[8:], want)
        with pytest.raises(P.PbvdError):       # not congruent mod 4
            dec.decode_blocks_mirrored(llr, 0, n_info, 0, nb, out, [m1.data_ptr() + 1])


def test_mirrored_outputs_with_recycled_regions(gpu, orc):
    """The mirrored kernel on a range larger than its survivor workspace
    (1 MiB: 6 regions for 128 jobs, so its jobs recycle regions within the one
    launch): every destination equal to the oracle's bits."""
    sys.path.insert(0, str(ROOT))
    import synth
    import paper_1608_00066_b200 as P
    code = synth.CODES["k7"]
    n_info, D, L = 1 << 21, 512, 42
    info, llr = synth.make_stream(code, n_info, 3.0, 67, device="cuda")
    want = torch.from_numpy(orc.pack_bits(orc.decode(code, llr.cpu().numpy(), n_info, D, L))).cuda()
    dec = P.Decoder(7, code["polys"], D, L)
    dec.set_workspace_limit(1 << 20)
    dec.set_profiling(True)
    nb = dec.block_count(n_info)
    out = torch.zeros(want.numel(), dtype=torch.uint8, device="cuda")
    m1 = torch.zeros(want.numel() + 4, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        dec.decode_blocks_mirrored(llr, 0, n_info, 0, nb, out, [m1.data_ptr() + 4])
    torch.cuda.synchronize()
    assert dec.kernel_times()[2] == 1          # one launch, regions recycled
    assert torch.equal(out, want) and torch.equal(m1[4:], want)


def test_ipc_export_open_roundtrip(gpu):
    """pbvd_ipc_export of a pointer inside a torch allocation gives the
    allocation's handle and the pointer's offset (the bench's peer gather
    maps other ranks' buffers with these); a process cannot open its own
    handle, so here only the export side and the error path are checked."""
    sys.path.insert(0, str(ROOT))
    import ctypes
    from paper_1608_00066_b200 import _lib
    L = _lib.load()
    t = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
    hnd = ctypes.create_string_buffer(_lib.PBVD_IPC_HANDLE_BYTES)
    off0, off1 = ctypes.c_int64(), ctypes.c_int64()
    assert L.pbvd_ipc_export(ctypes.c_void_p(t.data_ptr()), hnd, ctypes.byref(off0)) == 0
    assert L.pbvd_ipc_export(ctypes.c_void_p(t.data_ptr() + 4096), hnd, ctypes.byref(off1)) == 0
    assert off1.value - off0.value == 4096
    host = ctypes.create_string_buffer(64)
    assert L.pbvd_ipc_export(host, hnd, ctypes.byref(off0)) < 0        # not device memory


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs two GPUs (the driver's multi-GPU box)")
@pytest.mark.parametrize("gather", ["peer", "nccl"])
def test_bench_two_gpus_nccl(gather):
    """bench.py --gpus 2 on two devices over NCCL: the cross-device gather --
    fused into the decode over CUDA IPC / NVLink, or the NCCL all_gather --
    and rank 0's oracle check of the whole gathered stream."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, PBVD_BENCH_GATHER=gather)
    env.pop("PBVD_BENCH_BACKEND", None)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        str(port), "bench.py", "--gpus", "2", "--steps", "5", "--warmup", "3",
                        "--no-cpu-baseline", "--no-e2e"], cwd=ROOT, capture_output=True,
                       text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _line(r.stdout)
    assert d["n_gpus"] == 2 and d["parity"]["bit_exact"]
    assert d["parity"]["blocks_checked"] == d["parity"]["blocks_total"] == 65536
    if gather == "peer":
        assert d["run"]["gather"].startswith("fused"), d["run"]["gather"]
    else:
        assert d["run"]["gather"].startswith("NCCL")
