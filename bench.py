#!/usr/bin/env python
"""Benchmark of the PBVD hot path on B200 (contract: see DESIGN.md §7).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C2]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference          # the CPU oracle arm

A step = one pass of the whole hot path (block plan, soft
input fetch + depuncture, branch metrics, ACS, normalisation, decision
packing/store, min-PM start, traceback, output packing, and the final gather
for N > 1) over one batch of synthetic input already resident in HBM.
Default workload: BASELINE config C2 (K=7 (171,133), rate 1/2, 8-bit soft,
2^24 info bits, D=512, L=42) per GPU; for N GPUs the stream has N x 2^24
bits and rank r decodes its contiguous block range (weak scaling).
`--workload C5` runs the 2^32-bit stream sharded over the GPUs (strong).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

METRIC = json.loads((ROOT / "BASELINE.json").read_text())["metric"]
UNIT = "Gb/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C2", choices=list(synth.CONFIGS))
    ap.add_argument("--lanes", type=int, default=0)
    ap.add_argument("--kernels", default="fused", choices=["fused", "two"],
                    help="fused: one forward+traceback kernel (default); two: the paper's "
                         "forward and traceback kernels (pbvd_set_fused)")
    ap.add_argument("--e2e-steps", type=int, default=9)
    ap.add_argument("--cpu-seconds", type=float, default=8.0,
                    help="target wall time of the cpu_baseline oracle sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


# ------------------------------------------------------------------ helpers

def eq8_model(D, L, nblocks, U1, B, S_k, n_streams=3):
    """The paper's Eq. 8 throughput model and its transfer-bound
    counterpart for this pipeline (paper_1608_00066_b200/model.py), with the
    segmentation pbvd_decode_host uses (max(4, min(4 n_streams, nblocks/16384))
    equal segments plus a 4096-block last one, pbvd.cu), the measured H2D rate B
    and S_k = the device-timed value."""
    from paper_1608_00066_b200 import model as M
    last = 4096 if nblocks >= 4 * 4096 else 0
    nseg = max(4, min(4 * n_streams, (nblocks - last) // 16384)) + (1 if last else 0)
    seg = -(-nblocks // nseg)
    nseg = -(-nblocks // seg)
    out = M.model(D, L, seg, nseg, U1, 1 / 8, B, S_k)
    out["note"] = ("eq8 = Eq. 8 in its dimensionally consistent form (compute-bound premise); "
                   "transfer_bound = every H2D batch on the critical path; model = min")
    return out


def workload(name, world):
    c = dict(synth.CONFIGS[name])
    c["name"] = name
    code, punct = synth.CODES[c["code"]], synth.PUNCT[c["punct"]]
    if name == "C5":
        n_total, scaling = c["n_info"], "strong"
    else:
        n_total, scaling = c["n_info"] * world, "weak"
    return c, code, punct, n_total, scaling


def describe(c, code, n_total, world):
    K, R = code["K"], len(code["polys"])
    polys = ",".join(f"{p:o}" for p in code["polys"])
    soft = "hard" if c["hard"] else "soft 8-bit"
    return (f"{c['name']}: K={K} ({polys}) rate {c['punct'] if c['punct'] != '1/2' else '1/' + str(R)}"
            f" {soft} AWGN {c['ebn0']} dB, {n_total} info bits over {world} GPU(s), "
            f"D={c['D']} L={c['L']}, terminated")


def workload_config(c, code, n_total, world):
    """The bench line's `config`: the workload, the same in both arms."""
    return {"workload": describe(c, code, n_total, world), "n_info_total": n_total,
            "D": c["D"], "L": c["L"], "parallelism": f"block-range shards x{world}",
            "l2": "GPU arm: L2 flushed (256 MiB memset) before every timed step"}


class ClockSampler:
    """Samples SM clock and throttle reasons through NVML (every `period` s)
    while running; mark() brackets the timed region, whose samples are also
    summarised on their own."""

    def __init__(self, device_index, period=0.001):
        self.period, self.samples, self.reasons = period, [], set()
        self.marks = []
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover - no NVML
            self.nv, self.err = None, str(e)

    def _run(self):
        nv = self.nv
        names = {
            "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
            "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
            "display_clock_setting": 0x100,
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def mark(self):
        self.marks.append(len(self.samples))

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        timed = self.samples[self.marks[0]:self.marks[1]] if len(self.marks) >= 2 else []
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples),
                "period_ms": self.period * 1e3,
                "window": "warm-up + timed steps + profiled pass",
                "timed_sm_mhz": float(statistics.median(timed)) if timed else None,
                "timed_samples": len(timed)}


# ---- ACS roofline derived from unit counts and clocks ----
# Minimal instruction sequence per warp-level packed output (one 16x2 register
# = one state of two blocks, x 32 lanes = 64 ACS), the kernel's d-scheme:
#   VIADDMNMX.S16x2 (ALU) + 15/16 packing instr (PRMT 1/2 + LOP3 7/16, ALU)
#   + other-candidate add + decision add + half of the shared E - O
#     (2.5 two-operand adds, each on the ALU or the FMA pipe)
# Pipe model (B300_MICROARCH.md "Pipe rates"): ALU and FMA reciprocal
# throughput 2 cycles per SM sub-partition each, issue 1 instr/cycle.
ALU_ONLY = 1.0 + 0.5 + 7.0 / 16.0
FLEX = 2.5


def acs_sol_cycles():
    """min over the ALU/FMA split of max(issue, 2*ALU, 2*FMA) cycles per
    packed output; returns (cycles, fraction of the flexible adds on FMA)."""
    best = None
    for i in range(0, 1001):
        f = i / 1000.0
        alu = ALU_ONLY + FLEX * (1.0 - f)
        fma = FLEX * f
        c = max(alu + fma, 2.0 * alu, 2.0 * fma)
        if best is None or c < best[0]:
            best = (c, f)
    return best


def acs_peak_per_s(n_sm, sm_mhz):
    c, _ = acs_sol_cycles()
    return n_sm * 4 * sm_mhz * 1e6 * 64.0 / c


def acs_per_block_span(n_info, D, L, K, terminated, b0, nblk):
    """Sum over blocks of (forward span) x N: the ACS the step performs."""
    N = 1 << (K - 1)
    n_stages = n_info + ((K - 1) if terminated else 0)
    nb = -(-n_info // D)
    total = 0
    # interior blocks all have span D + 2L; edge blocks are counted exactly
    first_int = L // D + 1          # lo = bD - L > 0 (lo == 0 is a head block)
    last_int = min(nb - 2, (n_stages - L - D) // D if n_stages - L - D >= 0 else -1)
    lo_i, hi_i = max(first_int, b0), min(last_int + 1, b0 + nblk)
    n_int = max(0, hi_i - lo_i)
    total += n_int * (D + 2 * L) * N
    for b in list(range(b0, min(lo_i, b0 + nblk))) + list(range(max(hi_i, b0), b0 + nblk)):
        t0 = b * D
        t1 = min(t0 + D, n_info)
        lo = max(0, t0 - L)
        hi = n_stages if b == nb - 1 else min(n_stages, t1 + L)
        total += (hi - lo) * N
    return total


def load_traffic(workload, fused):
    """dram bytes per launch of the dominant kernel from the committed ncu
    summary (profiles/latest_fwd_ncu.json), if it was captured on this
    workload and kernel mode; else None."""
    p = ROOT / "profiles" / "latest_fwd_ncu.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            ent = d.get("captures", {}).get(f"{workload}:{'fused' if fused else 'two'}")
            if ent:
                return ent.get("dram_bytes_per_launch"), ent
        except Exception:
            pass
    return None, None


def cpu_oracle_sample(code, punct, c, llr_host, n_info, target_s, ws0=0, b_first=0,
                      max_blocks=None):
    """Time the oracle, as it stands, on a bounded sample of blocks."""
    from oracle import oracle as O
    threads = os.cpu_count() or 1
    flags = O.TERMINATED
    nb = -(-n_info // c["D"])
    if max_blocks is not None:
        nb = min(nb, b_first + max_blocks)
    # calibrate on a small sample, then size the measured one
    cal = min(nb - b_first, max(threads * 4, 64))
    t = time.perf_counter()
    O.decode(code, llr_host, n_info, c["D"], c["L"], flags=flags, punct=punct, threads=threads,
             b0=b_first, nblk=cal, window_stage0=ws0)
    dt = max(time.perf_counter() - t, 1e-4)
    nblk = int(min(nb - b_first, max(cal, cal * target_s / dt)))
    t = time.perf_counter()
    O.decode(code, llr_host, n_info, c["D"], c["L"], flags=flags, punct=punct, threads=threads,
             b0=b_first, nblk=nblk, window_stage0=ws0)
    dt = time.perf_counter() - t
    bits = min((b_first + nblk) * c["D"], n_info) - b_first * c["D"]
    # and on one core (1 thread and all cores), a smaller sample
    n1 = max(1, min(nblk, nblk // max(1, threads)))
    t = time.perf_counter()
    O.decode(code, llr_host, n_info, c["D"], c["L"], flags=flags, punct=punct, threads=1,
             b0=b_first, nblk=n1, window_stage0=ws0)
    dt1 = time.perf_counter() - t
    bits1 = min((b_first + n1) * c["D"], n_info) - b_first * c["D"]
    return {"value": bits / dt / 1e9, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"{nblk} of {nb} blocks ({bits} info bits) of the same stream, "
                      f"{threads} pthreads, {dt:.2f} s wall",
            "value_1_core": bits1 / dt1 / 1e9,
            "sample_1_core": f"{n1} blocks, 1 thread, {dt1:.2f} s"}


def bench_parity(code, punct, c, n_total, world, got, dev):
    """Oracle parity of a decoded stream `got` (packed, the whole n_total
    bits): every block up to 2^28 bits, else sampled runs in every rank's
    block range (see run_ours)."""
    from oracle import oracle as O
    from paper_1608_00066_b200 import shard as S
    O.build()
    D, L, K = c["D"], c["L"], code["K"]
    R = len(code["polys"])
    nb = -(-n_total // D)
    n_stages = n_total + K - 1
    runs = []
    if n_total <= (1 << 28):
        runs = [(b0, min(1 << 18, nb - b0)) for b0 in range(0, nb, 1 << 18)]
    else:
        rng = np.random.default_rng(12345)
        for r in range(world):
            sh = S.plan(n_total, D, L, K, True, world, r)
            b0, b1 = sh.block0, sh.block0 + sh.nblocks
            mid = int(rng.integers(b0, max(b0 + 1, b1 - 64)))
            runs += [(b0, min(64, b1 - b0)), (max(b0, b1 - 64), min(64, b1 - b0)),
                     (mid, min(64, b1 - mid))]
    checked, ok = 0, True
    for b0, nblk in runs:
        lo = max(0, b0 * D - L)
        hi = n_stages if b0 + nblk == nb else min(n_stages, (b0 + nblk) * D + L)
        win = synth.make_window(code, n_total, c["ebn0"], c["seed"], lo, hi, punct, c["hard"],
                                device=dev).cpu().numpy()
        want = O.pack_bits(O.decode(code, win, n_total, D, L, punct=punct, b0=b0, nblk=nblk,
                                    window_stage0=lo))
        t0 = b0 * D
        seg = got[t0 // 8:t0 // 8 + want.size]
        ok &= bool(np.array_equal(seg, want))
        checked += nblk
    return {"blocks_checked": checked, "blocks_total": nb, "bit_exact": ok,
            "scope": ("every block" if checked == nb else
                      f"first/last/random 64-block runs of each of the {world} ranks' ranges") +
                     (" of the gathered stream" if world > 1 else "")}


# ------------------------------------------------------------------ arms

def run_reference(args):
    """The oracle arm: the CPU oracle as it stands on this host's cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    world = max(1, args.gpus)
    c, code, punct, n_total, scaling = workload(args.workload, world)
    # one rank's share of the stream, generated on the host
    from paper_1608_00066_b200 import shard as S
    sh = S.plan(n_total, c["D"], c["L"], code["K"], True, world, 0)
    llr = synth.make_window(code, n_total, c["ebn0"], c["seed"], sh.stage0, sh.stage1, punct,
                            c["hard"], device="cpu").numpy()
    from oracle import oracle as O
    O.build()
    # bounded sample per step, sized once so the whole run takes ~2 minutes
    per_step = max(0.1, min(2.0, 120.0 / max(1, args.steps + args.warmup)))
    threads = os.cpu_count() or 1
    nb_shard = sh.nblocks
    cal = min(nb_shard, max(threads * 4, 64))
    t = time.perf_counter()
    O.decode(code, llr, n_total, c["D"], c["L"], punct=punct, threads=threads, b0=sh.block0,
             nblk=cal, window_stage0=sh.stage0)
    dt = max(time.perf_counter() - t, 1e-4)
    nblk = int(min(nb_shard, max(cal, cal * per_step / dt)))
    bits = min((sh.block0 + nblk) * c["D"], n_total) - sh.block0 * c["D"]
    vals, secs = [], []
    for i in range(args.warmup + args.steps):
        t = time.perf_counter()
        O.decode(code, llr, n_total, c["D"], c["L"], punct=punct, threads=threads,
                 b0=sh.block0, nblk=nblk, window_stage0=sh.stage0)
        dt = time.perf_counter() - t
        if i >= args.warmup:
            vals.append(bits / dt / 1e9)
            secs.append(dt)
    v = statistics.median(vals)
    cb = {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
          "sample": f"{nblk} of {sh.nblocks} blocks ({bits} info bits) of the same stream per "
                    f"step, {threads} pthreads"}
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.median(secs) * 1e3,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "int32",
        "data": "synthetic", "config": workload_config(c, code, n_total, world),
        "run": {"impl": "CPU oracle (oracle/pbvd_oracle.c), per-edge ACS, all host cores"},
        "cpu_baseline": cb,
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch.distributed as dist
    from paper_1608_00066_b200 import build
    build.build()
    import paper_1608_00066_b200 as P
    from paper_1608_00066_b200 import shard as S

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # NCCL over NVLink for real runs; PBVD_BENCH_BACKEND=gloo exercises the
    # N > 1 control flow with several ranks on one GPU (tests only)
    backend = os.environ.get("PBVD_BENCH_BACKEND", "nccl")
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    cdev = dev if backend == "nccl" else torch.device("cpu")   # collective tensors

    c, code, punct, n_total, scaling = workload(args.workload, world)
    D, L, K = c["D"], c["L"], code["K"]
    sh = S.plan(n_total, D, L, K, True, world, rank)
    llr = synth.make_window(code, n_total, c["ebn0"], c["seed"], sh.stage0, sh.stage1, punct,
                            c["hard"], device=dev)
    dec = P.Decoder(K, code["polys"], D, L, punct=punct, terminated=True, device=local,
                    lanes=args.lanes, fused=(args.kernels == "fused"))
    dec.set_profiling(True)
    out = torch.empty(sh.nbytes, dtype=torch.uint8, device=dev)
    gathered = None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2

    # N > 1: the gather of the decoded bits (a10).  Default: fused into
    # the traceback -- every rank's gather buffer is mapped into every other
    # rank through CUDA IPC (pbvd_ipc_export / pbvd_ipc_open: peer access
    # over NVLink) and the decode kernel stores each output word to all of
    # them (pbvd_decode_blocks_mirrored); checked against an NCCL all_gather
    # after the warm-up, with the NCCL all_gather as the fallback
    # (PBVD_BENCH_GATHER=nccl forces it; config.gather says which ran and why).
    gather_mode = "none" if world == 1 else os.environ.get("PBVD_BENCH_GATHER", "peer")
    gather_note = ""
    gbuf, mirrors, peer = None, [], None
    if gather_mode == "peer":
        try:
            gbuf = torch.zeros((n_total + 7) // 8, dtype=torch.uint8, device=dev)
            peer = S.PeerGather(gbuf)
            mirrors = peer.mirrors(sh)
            out = gbuf[sh.bit0 // 8:sh.bit0 // 8 + sh.nbytes]
        except Exception as ex:  # pragma: no cover - depends on the box
            gather_note = f"peer gather setup failed ({ex})"
            print(gather_note + "; NCCL all_gather instead", file=sys.stderr)
            gather_mode, peer, gbuf = "nccl", None, None
            out = torch.empty(sh.nbytes, dtype=torch.uint8, device=dev)
    elif gather_mode == "nccl":
        gather_note = "forced by PBVD_BENCH_GATHER=nccl"
    done_flag = torch.zeros(1, dtype=torch.int32, device=cdev)
    align_flag = torch.zeros(1, dtype=torch.int32, device=cdev)

    def decode_part():
        if gather_mode == "peer":
            dec.decode_blocks_mirrored(llr, sh.stage0, n_total, sh.block0, sh.nblocks, out,
                                       mirrors)
        else:
            dec.decode_blocks(llr, sh.stage0, n_total, sh.block0, sh.nblocks, out=out)

    def gather_part():
        if gather_mode == "peer":
            # every rank's stores into this buffer are complete once every
            # rank's decode kernel has retired: a one-word all_reduce queued
            # behind the decode on each rank's stream
            dist.all_reduce(done_flag)
            return gbuf
        if world > 1:
            return S.gather_bits(out.to(cdev), sh, n_total, D)
        return out

    def step():
        decode_part()
        return gather_part()

    # measured throughput of the all-ALU ACS sequence (pbvd_probe_acs_peak):
    # reported beside the derived roofline as a cross-check
    probe_acs, _ = P.probe_acs_peak(local)
    probe_bal, _ = P.probe_acs_balanced(local)

    clk = ClockSampler(local, period=0.001)
    clk.__enter__()               # sampled from the warm-up through the profiled pass
    for _ in range(args.warmup):
        flush.zero_()
        gathered = step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if gather_mode == "peer":
        # every rank's buffer must now hold the whole stream: compare with an
        # NCCL all_gather of this rank's own bits; any mismatch -> NCCL path
        ref = S.gather_bits(out.clone().to(cdev), sh, n_total, D)
        good = torch.tensor([int(torch.equal(ref.to(dev), gbuf))], dtype=torch.int32, device=cdev)
        dist.all_reduce(good, op=dist.ReduceOp.MIN)
        if not int(good.item()):
            gather_note = "peer gather check against an NCCL all_gather failed"
            print(gather_note + "; NCCL all_gather instead", file=sys.stderr)
            gather_mode = "nccl"
            out = out.clone()
        torch.cuda.synchronize()
        dist.barrier()

    stream = torch.cuda.current_stream(dev)
    times, dec_times, gat_times, launches = [], [], [], 0
    dec.set_profiling(False)          # no events inside a decode: the timed region is pure
    clk.mark()
    for _ in range(args.steps):
        if world > 1:
            dist.barrier()            # every rank starts the step together
            torch.cuda.synchronize()
        # L2 flush; the host enqueues the decode while the memset runs, so
        # the timed region holds no host launch latency
        flush.zero_()
        if world > 1:
            # device-side start line: one-word all_reduce queued after the
            # flush, so every rank's timed region starts when all GPUs are
            # ready (host wake-up skew after the barrier is not decode time)
            dist.all_reduce(align_flag)
        e0 = torch.cuda.Event(enable_timing=True)
        em = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        decode_part()
        em.record(stream)
        gathered = gather_part()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
        dec_times.append(e0.elapsed_time(em))
        gat_times.append(em.elapsed_time(e1))
        launches += dec.kernel_times()[2]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk.mark()
    # per-kernel times (CUDA events around each launch on the decode stream),
    # a separate pass of the same steps -- the events break the PDL overlap of
    # the two kernels, so they are kept out of the timed region above
    dec.set_profiling(True)
    fwd, tb = [], []
    for _ in range(max(10, min(args.steps, 50))):
        flush.zero_()
        decode_part()
        torch.cuda.synchronize()
        f, t, n = dec.kernel_times()
        fwd.append(f)
        tb.append(t)
    clk.__exit__()
    # max over ranks: of the step total, and of the decode / gather parts
    tms = torch.tensor([sum(times), sum(dec_times), sum(gat_times)], dtype=torch.float64,
                       device=cdev)
    if world > 1:
        dist.all_reduce(tms, op=dist.ReduceOp.MAX)
    total_ms, dec_ms_tot, gat_ms_tot = (float(x) for x in tms.tolist())
    ms_per_step = total_ms / args.steps
    value = n_total / (ms_per_step * 1e-3) / 1e9

    # ---- roofline of the dominant kernel ------------------------------------
    # fused mode: ONE kernel per step (forward + in-warp traceback), timed by
    # CUDA events on the decode stream around each launch (profiled pass)
    acs_step = acs_per_block_span(n_total, D, L, K, True, sh.block0, sh.nblocks)
    fwd_ms = statistics.median(fwd)
    tb_ms = statistics.median(tb)
    achieved = acs_step / (fwd_ms * 1e-3)
    clocks = clk.summary()
    props = torch.cuda.get_device_properties(dev)
    sm_mhz = clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 1965.0
    sol_cycles, sol_f = acs_sol_cycles()
    peak_acs = acs_peak_per_s(props.multi_processor_count, sm_mhz)
    R = len(code["polys"])
    N = 1 << (K - 1)
    span = D + 2 * L
    in_bytes = synth.llr_count(R, punct, sh.stage1) - synth.llr_count(R, punct, sh.stage0)
    nb_rank = sh.nblocks
    dec_bytes = nb_rank * span * N // 8
    dec_read = nb_rank * (span - L - (K - 1)) * N // 8
    out_bytes = sh.nbytes
    # the algorithmic HBM bytes of the fused single-kernel
    # design are the soft input (halo re-reads included) and the packed
    # output -- the survivors never need to leave the chip (~2.5 B/bit for
    # C2); the two-kernel design adds the survivor write and read-back
    # (20.4 B/bit).  `traffic` (ncu) shows what the kernel really moves.
    alg_bytes = in_bytes + out_bytes + (0 if dec.fused else dec_bytes + dec_read)
    fwd_hbm_gbs = alg_bytes / (fwd_ms * 1e-3) / 1e9
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    traffic, _ = load_traffic(args.workload, dec.fused)
    kname = "fwd_kernel<fused>" if dec.fused else "fwd_kernel"
    roofline = {
        "bound": "alu", "achieved": achieved / 1e12, "peak": peak_acs / 1e12, "unit": "Tacs/s",
        "frac": achieved / peak_acs, "traffic": traffic,
        "kernel": f"{kname} (K={K}, lanes={dec.lanes})",
        "peak_source": (f"derived: {props.multi_processor_count} SMs x 4 sub-partitions x "
                        f"{sm_mhz:.0f} MHz (median SM clock under load) x 64 ACS per "
                        f"{sol_cycles:.3f} cycles (minimal 16x2 ACS+decision sequence, "
                        f"ALU/FMA pipes at 0.5 and issue at 1 instr/cycle, "
                        f"{sol_f:.2f} of the two-operand adds on FMA)"),
        "probe_all_alu_tacs": probe_acs / 1e12,
        "probe_balanced_tacs": probe_bal / 1e12,
        "acs_per_launch": acs_step, "kernel_ms": fwd_ms, "tb_kernel_ms": tb_ms,
        "kernel_share_of_step": fwd_ms / ms_per_step,
        "hbm": {"algorithmic_bytes_per_launch": alg_bytes,
                "algorithmic_bytes_per_bit": alg_bytes / max(1, sh.bit1 - sh.bit0),
                "two_kernel_design_bytes_per_launch": in_bytes + out_bytes + dec_bytes + dec_read,
                "dram_bytes_per_launch_ncu": traffic,
                "dram_bytes_per_bit_ncu": (traffic / max(1, sh.bit1 - sh.bit0)) if traffic else None,
                "achieved_gbs": fwd_hbm_gbs,
                "peak_gbs": hbm_peak, "frac": fwd_hbm_gbs / hbm_peak,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback"},
    }

    # ---- parity inside the bench (never timed) -----------------------------
    # rank 0 checks the GATHERED stream (every rank's blocks, N > 1) or its
    # own output (N = 1) against the oracle: every block when the stream has
    # <= 2^28 bits (C2 at N <= 8: a few s on the host cores), else, for each
    # rank's range, its first, last and a seeded random run of 64 blocks,
    # each run's soft window regenerated here from the same seeds
    parity = None
    if rank == 0:
        try:
            parity = bench_parity(code, punct, c, n_total, world,
                                  (gathered if world > 1 else out).cpu().numpy(), dev)
        except Exception as e:  # pragma: no cover
            parity = {"error": str(e)}
    if world > 1:
        dist.barrier()

    # ---- end to end through the C ABI with host buffers ---------------------
    e2e = None
    llr_h = None
    if not args.no_e2e:
        llr_h = torch.empty(llr.shape, dtype=llr.dtype, pin_memory=True)   # one host copy
        llr_h.copy_(llr)
        out_h = torch.empty(sh.nbytes, dtype=torch.uint8).pin_memory()
        # warm-up (untimed): host-lane streams and staging buffers, and the
        # host/PCIe path itself -- freshly pinned buffers copy at ~60 % of the
        # link rate for the first few hundred ms (measured, tools/e2e_check.py),
        # so warm up for >= 1 s, not a fixed count
        t_w, k_w = time.perf_counter(), 0
        while k_w < 5 or time.perf_counter() - t_w < 1.0:
            dec.decode_host(llr_h, n_total, out=out_h, window_stage0=sh.stage0,
                            block0=sh.block0, nblocks=sh.nblocks)
            k_w += 1
        ts = []
        for _ in range(args.e2e_steps):
            if world > 1:
                dist.barrier()
            t = time.perf_counter()
            dec.decode_host(llr_h, n_total, out=out_h, window_stage0=sh.stage0,
                            block0=sh.block0, nblocks=sh.nblocks)
            ts.append(time.perf_counter() - t)
        e2e_s = torch.tensor([statistics.median(ts)], dtype=torch.float64, device=cdev)
        if world > 1:
            dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
        same = bool(torch.equal(out_h, out.cpu()))
        # the PCIe bound of this step: plain pinned copies of the same bytes
        # (H2D of the soft values, D2H of the bits; full duplex, so the
        # slower direction bounds an ideally overlapped pipeline)
        d_in = torch.empty_like(llr_h, device=dev)
        d_out = torch.empty_like(out_h, device=dev)
        ts_in, ts_out = [], []
        for _ in range(3):
            torch.cuda.synchronize()
            t = time.perf_counter()
            d_in.copy_(llr_h, non_blocking=True)
            torch.cuda.synchronize()
            ts_in.append(time.perf_counter() - t)
            t = time.perf_counter()
            out_h.copy_(d_out, non_blocking=True)
            torch.cuda.synchronize()
            ts_out.append(time.perf_counter() - t)
        t_in, t_out = min(ts_in), min(ts_out)
        e2e_v = n_total / float(e2e_s.item()) / 1e9
        bound = n_total / max(t_in, t_out) / 1e9
        e2e = {"value": e2e_v, "unit": UNIT,
               "h2d_bytes_per_step": int(llr_h.numel()), "d2h_bytes_per_step": int(out_h.numel()),
               "host_lanes": dec.info()["host_lanes"],
               "api": "pbvd_decode_host (pinned host buffers, 3 streams)",
               "matches_device_path": same,
               "eq8": eq8_model(D, L, sh.nblocks, in_bytes / max(1, sh.stage1 - sh.stage0),
                                llr_h.numel() / t_in, value * 1e9),
               "pcie": {"h2d_gbs": llr_h.numel() / t_in / 1e9, "d2h_gbs": out_h.numel() / t_out / 1e9,
                        "bound_value": bound, "frac_of_bound": e2e_v / bound}}
        del d_in, d_out

    # ---- CPU baseline: the oracle on this host (rank 0, N == 1) ------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O
        O.build()
        host = llr_h if llr_h is not None else llr.cpu()
        cpu = cpu_oracle_sample(code, punct, c, host.numpy(), n_total, args.cpu_seconds,
                                ws0=sh.stage0, b_first=sh.block0, max_blocks=sh.nblocks)

    if world > 1:
        dist.barrier()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "int16",
            "data": "synthetic (seeded BPSK/AWGN, 8-bit quantised)",
            # config: the workload only (identical in both arms); how this arm
            # ran it is in "run"
            "config": workload_config(c, code, n_total, world),
            "run": {"lanes": dec.lanes,
                       "gather": {"none": "none (1 GPU)",
                                  "peer": "fused into the traceback: stores to every rank's "
                                          "buffer over CUDA IPC / NVLink (completion: one "
                                          "all_reduce word behind the decode)",
                                  "nccl": "NCCL all_gather"}[gather_mode] +
                                 (f" [{gather_note}]" if gather_note else ""),
                       "step_barrier": "dist.barrier + synchronize before every timed step, then a one-word device all_reduce after the L2 flush as the start line of the timed region"
                                       if world > 1 else "none (1 GPU)"},
            "t_G": {"decode_ms": dec_ms_tot / args.steps, "gather_ms": gat_ms_tot / args.steps,
                    "note": "per step, each the max over ranks of its CUDA-event time on the "
                            "decode stream (SURVEY §8(d): max-rank decode + gather)"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clocks, "parity": parity,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.cuda.synchronize()
        dist.barrier()            # no rank still reads or writes a peer buffer
        if peer is not None:
            peer.close()
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
