"""e2e host-pipeline check: decode_host timing before / after a burst of
device load (diagnoses the post-load slowdown seen in bench's e2e)."""
import subprocess, sys, time
sys.path.insert(0, '.')
import torch, synth
import paper_1608_00066_b200 as P
c = synth.CONFIGS["C2"]; code = synth.CODES["k7"]; n = c["n_info"]
info, llr = synth.make_stream(code, n, c["ebn0"], c["seed"])
llr_h = llr.pin_memory(); out_h = torch.empty((n + 7) // 8, dtype=torch.uint8).pin_memory()
dec = P.Decoder(7, code["polys"], 512, 42)
d = llr.cuda(); out = dec.decode(d, n); torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def clocks():
    q = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,pcie.link.gen.current,pcie.link.width.current,clocks_throttle_reasons.active",
                        "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    return q


def e2e(tag, k=9):
    for _ in range(3): dec.decode_host(llr_h, n, out=out_h)
    ts = []
    for _ in range(k):
        t = time.perf_counter(); dec.decode_host(llr_h, n, out=out_h); ts.append(time.perf_counter() - t)
    ts.sort()
    x = torch.empty_like(llr_h, device="cuda")
    torch.cuda.synchronize(); t = time.perf_counter(); x.copy_(llr_h, non_blocking=True); torch.cuda.synchronize()
    h2d = llr_h.numel() / (time.perf_counter() - t) / 1e9
    torch.cuda.synchronize(); t = time.perf_counter(); dec.decode(d, n, out=out); torch.cuda.synchronize()
    dk = (time.perf_counter() - t) * 1e3
    print(f"{tag}: e2e {ts[k//2]*1e3:.3f} ms {n/ts[k//2]/1e9:.2f} Gb/s  h2d {h2d:.1f} GB/s  device decode {dk:.3f} ms | {clocks()}", flush=True)


e2e("fresh")
for burst in range(3):
    t = time.perf_counter()
    while time.perf_counter() - t < 0.5:
        flush.zero_(); dec.decode(d, n, out=out)
    torch.cuda.synchronize()
    e2e(f"after burst {burst}")
    time.sleep(1.0)
    e2e(f"after burst {burst} + 1 s idle")
