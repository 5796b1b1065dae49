"""Quick device timing of pbvd_decode on a BASELINE config (dev tool)."""
import sys, time, torch
sys.path.insert(0, '.')
import synth
from paper_1608_00066_b200 import build
build.build()
import paper_1608_00066_b200 as P

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
c = synth.CONFIGS[cfg]
code, punct = synth.CODES[c["code"]], synth.PUNCT[c["punct"]]
n_info = int(sys.argv[2]) if len(sys.argv) > 2 else c["n_info"]
info, llr = synth.make_stream(code, n_info, c["ebn0"], c["seed"], punct, c["hard"], device="cuda")
import os, itertools
lanes_all = sorted({l for (K, R, p, l) in P.supported() if K == code["K"] and tuple(p) == tuple(code["polys"])})
lanes_sel = [int(x) for x in os.environ.get("QT_LANES", "").split()] or lanes_all
for fused, lanes in itertools.product([int(x) for x in os.environ.get("QT_FUSED", "1").split()], lanes_sel):
    dec = P.Decoder(code["K"], code["polys"], c["D"], c["L"], punct=punct, lanes=lanes, fused=bool(fused))
    dec.set_profiling(True)
    out = dec.decode(llr, n_info)
    torch.cuda.synchronize()
    ts, fw, tb = [], [], []
    for i in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); dec.decode(llr, n_info, out=out); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1)); f, t, n = dec.kernel_times(); fw.append(f); tb.append(t)
    ts.sort(); fw.sort(); tb.sort()
    ms = ts[len(ts)//2]
    ber = (torch.unpackbits if hasattr(torch,'unpackbits') else None)
    dec.set_profiling(False)
    ts2 = []
    for i in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); dec.decode(llr, n_info, out=out); e1.record(); torch.cuda.synchronize()
        ts2.append(e0.elapsed_time(e1))
    ts2.sort()
    ms2 = ts2[len(ts2)//2]
    print(f"{cfg} n_info={n_info} lanes={lanes} fused={fused}: {ms:.3f} ms  {n_info/ms/1e6:.2f} Gb/s  fwd {fw[5]:.3f} ms tb {tb[5]:.3f} ms  launches={n}  | no-prof {ms2:.3f} ms {n_info/ms2/1e6:.2f} Gb/s", flush=True)
