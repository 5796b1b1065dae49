"""C5 (2^32 bits) decode time vs survivor-workspace wave size."""
import sys
sys.path.insert(0, '.')
import torch, synth
import paper_1608_00066_b200 as P
c = synth.CONFIGS["C5"]; code = synth.CODES["k7"]; n = c["n_info"]
llr = synth.make_window(code, n, c["ebn0"], c["seed"], 0, n + 6, None, device="cuda")
out = torch.empty(n // 8, dtype=torch.uint8, device="cuda")
for gb in [1, 2, 4, 8, 16]:
    dec = P.Decoder(7, code["polys"], 512, 42)
    dec.set_workspace_limit(gb << 30)
    dec.decode(llr, n, out=out); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); dec.decode(llr, n, out=out); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    print(f"ws {gb} GiB: {ms:.2f} ms  {n / ms / 1e6:.1f} Gb/s", flush=True)
    del dec
