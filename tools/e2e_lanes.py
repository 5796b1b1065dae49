"""e2e (pbvd_decode_host) per lane variant for a BASELINE config: which
variant the host pipeline should use (dev tool)."""
import sys, time
sys.path.insert(0, '.')
import torch, synth
import paper_1608_00066_b200 as P
cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
c = synth.CONFIGS[cfg]; code, punct = synth.CODES[c["code"]], synth.PUNCT[c["punct"]]
n = int(sys.argv[2]) if len(sys.argv) > 2 else c["n_info"]
info, llr = synth.make_stream(code, n, c["ebn0"], c["seed"], punct, c["hard"])
llr_h = llr.pin_memory(); out_h = torch.empty((n + 7) // 8, dtype=torch.uint8).pin_memory()
lanes_all = sorted({l for (K, R, p, l) in P.supported() if K == code["K"] and tuple(p) == tuple(code["polys"])})
for lanes in lanes_all:
    dec = P.Decoder(code["K"], code["polys"], c["D"], c["L"], punct=punct, lanes=lanes)
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 1.0:
        dec.decode_host(llr_h, n, out=out_h)
    ts = []
    for _ in range(9):
        t = time.perf_counter(); dec.decode_host(llr_h, n, out=out_h); ts.append(time.perf_counter() - t)
    ts.sort()
    print(f"{cfg} lanes={lanes}: e2e {ts[4]*1e3:.3f} ms {n/ts[4]/1e9:.2f} Gb/s", flush=True)
