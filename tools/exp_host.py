"""e2e host pipeline timing sweep (pbvd_decode_host) for C2: lanes (per-warp
latency), stream count; PBVD_HOST_MINSEG / PBVD_HOST_SEGX env knobs."""
import os, sys, time
sys.path.insert(0, '.')
import torch, synth
import paper_1608_00066_b200 as P
c = synth.CONFIGS["C2"]; code = synth.CODES["k7"]; n = c["n_info"]
info, llr = synth.make_stream(code, n, c["ebn0"], c["seed"])
llr_h = llr.pin_memory(); out_h = torch.empty((n + 7) // 8, dtype=torch.uint8).pin_memory()
for lanes in [2, 4, 1]:
    dec = P.Decoder(7, code["polys"], 512, 42, lanes=lanes)
    for ns in [2, 3, 4, 8]:
        dec.decode_host(llr_h, n, out=out_h, n_streams=ns)
        ts = []
        for _ in range(9):
            t = time.perf_counter(); dec.decode_host(llr_h, n, out=out_h, n_streams=ns); ts.append(time.perf_counter() - t)
        ts.sort()
        print(f"lanes={lanes} MINSEG={os.environ.get('PBVD_HOST_MINSEG','8192')} SEGX={os.environ.get('PBVD_HOST_SEGX','2')} streams={ns}: {ts[4]*1e3:.3f} ms  {n/ts[4]/1e9:.2f} Gb/s", flush=True)
