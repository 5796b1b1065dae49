"""e2e (pbvd_decode_host, pinned host buffers) vs the pure H2D time, per
config and stream count: python tools/e2e_quick.py C2 C3a ..."""
import sys, time
sys.path.insert(0, ".")
import torch, synth, paper_1608_00066_b200 as P
for cfg in sys.argv[1:] or ["C2"]:
    c = synth.CONFIGS[cfg]; code, punct = synth.CODES[c["code"]], synth.PUNCT[c["punct"]]
    n = c["n_info"]
    info, llr = synth.make_stream(code, n, c["ebn0"], c["seed"], punct, c["hard"])
    llr_h = llr.pin_memory(); out_h = torch.empty((n + 7) // 8, dtype=torch.uint8).pin_memory()
    dec = P.Decoder(code["K"], code["polys"], c["D"], c["L"], punct=punct)
    ref = dec.decode(llr.cuda(), n).cpu()
    x = torch.empty_like(llr_h, device="cuda"); tt = []
    for _ in range(5):
        torch.cuda.synchronize(); t = time.perf_counter(); x.copy_(llr_h, non_blocking=True)
        torch.cuda.synchronize(); tt.append(time.perf_counter() - t)
    for ns in (2, 3, 4):
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < 1.0:
            dec.decode_host(llr_h, n, out=out_h, n_streams=ns)
        ts = []
        for _ in range(15):
            t = time.perf_counter(); dec.decode_host(llr_h, n, out=out_h, n_streams=ns)
            ts.append(time.perf_counter() - t)
        ts.sort()
        ok = torch.equal(out_h, ref)
        print(f"{cfg} streams={ns}: {ts[7]*1e3:.3f} ms {n/ts[7]/1e9:.2f} Gb/s  h2d alone "
              f"{min(tt)*1e3:.3f} ms  frac {min(tt)/ts[7]:.3f}  same={ok}", flush=True)
