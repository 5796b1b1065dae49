import sys, torch
sys.path.insert(0, '.')
import synth
from paper_1608_00066_b200 import build
build.build()
import paper_1608_00066_b200 as P
c = synth.CONFIGS["C2"]; code = synth.CODES["k7"]; n = c["n_info"]
info, llr = synth.make_stream(code, n, c["ebn0"], c["seed"], device="cuda")
dec = P.Decoder(7, code["polys"], c["D"], c["L"])
nb = dec.block_count(n)
out = torch.empty((n + 7) // 8, dtype=torch.uint8, device="cuda")
m1 = torch.empty(out.numel() + 4, dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ts.sort(); return ts[len(ts) // 2]
for r in range(3):
    a = t(lambda: dec.decode_blocks(llr, 0, n, 0, nb, out=out))
    b = t(lambda: dec.decode_blocks_mirrored(llr, 0, n, 0, nb, out, [m1.data_ptr() + 4]))
    print(f"plain {a:.4f} ms  mirrored(1 dest) {b:.4f} ms  ratio {b/a:.4f}")
