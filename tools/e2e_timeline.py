"""Timeline of a Python replica of pbvd_decode_host's pipeline (C2): per
segment H2D start/end, decode end, D2H end (CUDA events), to see where the
e2e time above the pure H2D time goes."""
import sys, time
sys.path.insert(0, ".")
import torch, synth, paper_1608_00066_b200 as P
from paper_1608_00066_b200 import shard as S
c = synth.CONFIGS["C2"]; code = synth.CODES["k7"]; n = c["n_info"]; D, L = c["D"], c["L"]
info, llr = synth.make_stream(code, n, c["ebn0"], c["seed"])
llr_h = llr.pin_memory(); out_h = torch.empty((n + 7) // 8, dtype=torch.uint8).pin_memory()
nseg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
ns = 3
decs = [P.Decoder(7, code["polys"], D, L, lanes=int(sys.argv[2]) if len(sys.argv) > 2 else 4)
        for _ in range(ns)]        # one handle (workspace) per stream
streams = [torch.cuda.Stream() for _ in range(ns)]
nb = -(-n // D)
shards = [S.plan(n, D, L, 7, True, nseg, k) for k in range(nseg)]
dbufs = [torch.empty(sh.stage1 * 2 - sh.stage0 * 2, dtype=torch.int8, device="cuda") for sh in shards]
obufs = [torch.empty(sh.nbytes, dtype=torch.uint8, device="cuda") for sh in shards]


def run(record):
    evs = []
    base = torch.cuda.Event(enable_timing=True)
    base.record(torch.cuda.current_stream())
    for k, sh in enumerate(shards):
        s = streams[k % ns]
        s.wait_event(base)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        with torch.cuda.stream(s):
            e[0].record(s)
            dbufs[k].copy_(llr_h[sh.stage0 * 2:sh.stage1 * 2], non_blocking=True)
            e[1].record(s)
            decs[k % ns].decode_blocks(dbufs[k], sh.stage0, n, sh.block0, sh.nblocks, out=obufs[k], stream=s)
            e[2].record(s)
            out_h[sh.bit0 // 8:sh.bit0 // 8 + sh.nbytes].copy_(obufs[k], non_blocking=True)
            e[3].record(s)
        evs.append(e)
    torch.cuda.synchronize()
    if record:
        for k, e in enumerate(evs):
            print(f"  seg {k}: h2d {base.elapsed_time(e[0])*1e3:7.1f}-{base.elapsed_time(e[1])*1e3:7.1f} us  "
                  f"dec end {base.elapsed_time(e[2])*1e3:7.1f}  d2h end {base.elapsed_time(e[3])*1e3:7.1f}")


for _ in range(20):
    run(False)
t = time.perf_counter(); run(False); t = time.perf_counter() - t
print(f"nseg={nseg} wall {t*1e3:.3f} ms  {n/t/1e9:.2f} Gb/s")
run(True)
