"""e2e host-pipeline sweep over the segment plan (PBVD_HOST_NSEG big
segments + a PBVD_HOST_LAST-block last one; read once per process)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, time; sys.path.insert(0, ".")
import torch, synth, paper_1608_00066_b200 as P
c = synth.CONFIGS[sys.argv[1]]; code, punct = synth.CODES[c["code"]], synth.PUNCT[c["punct"]]; n = c["n_info"]
info, llr = synth.make_stream(code, n, c["ebn0"], c["seed"], punct, c["hard"])
llr_h = llr.pin_memory(); out_h = torch.empty((n + 7) // 8, dtype=torch.uint8).pin_memory()
dec = P.Decoder(code["K"], code["polys"], c["D"], c["L"], punct=punct)
ref = dec.decode(llr.cuda(), n).cpu()
ns = int(sys.argv[2])
t0 = time.perf_counter()
while time.perf_counter() - t0 < 1.5: dec.decode_host(llr_h, n, out=out_h, n_streams=ns)
ts = []
for _ in range(21):
    t = time.perf_counter(); dec.decode_host(llr_h, n, out=out_h, n_streams=ns); ts.append(time.perf_counter() - t)
ts.sort()
import os
print(f"{sys.argv[1]} nseg={os.environ.get('PBVD_HOST_NSEG','-')} last={os.environ.get('PBVD_HOST_LAST','-')} streams={ns}: {ts[10]*1e3:.3f} ms {n/ts[10]/1e9:.2f} Gb/s same={torch.equal(out_h, ref)}", flush=True)
'''
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
for nseg in sys.argv[2].split(",") if len(sys.argv) > 2 else ["2", "3", "4", "6", "8"]:
    for last in sys.argv[3].split(",") if len(sys.argv) > 3 else ["0", "1024", "2048", "4096"]:
        env = dict(os.environ, PBVD_HOST_NSEG=nseg, PBVD_HOST_LAST=last)
        if nseg == "0": env.pop("PBVD_HOST_NSEG")
        if last == "-1": env.pop("PBVD_HOST_LAST")
        subprocess.run([sys.executable, "-c", CODE, cfg, "3"], cwd=ROOT, env=env)
