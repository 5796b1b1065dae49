"""Small decodes through the newer entry points, each checked against the
oracle -- the workload of the compute-sanitizer pass (tools/sanitize.sh):
mirrored outputs (fused and two-kernel), run-time (JIT) codes incl. K = 12,
the continuous stream, the table depuncture and the host pipeline."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ.setdefault("PBVD_JIT_CACHE", str(ROOT / "paper_1608_00066_b200" / "build" / "jit_cache"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from oracle import oracle as O  # noqa: E402
import paper_1608_00066_b200 as P  # noqa: E402

bad = 0


def check(tag, got, want):
    global bad
    n = int(np.count_nonzero(np.asarray(got) != np.asarray(want)))
    bad += n
    print(f"{tag}: bad bytes {n}", flush=True)


k7 = synth.CODES["k7"]
info, llr = synth.make_stream(k7, 3000, 3.0, 5)
want = O.pack_bits(O.decode(k7, llr.numpy(), 3000, 64, 20))
d = llr.cuda()
for fused in (True, False):
    dec = P.Decoder(7, k7["polys"], 64, 20, fused=fused)
    out = torch.zeros(want.size, dtype=torch.uint8, device="cuda")
    m = torch.zeros(want.size * 2 + 8, dtype=torch.uint8, device="cuda")
    dec.decode_blocks_mirrored(d, 0, 3000, 0, dec.block_count(3000), out,
                               [m.data_ptr(), m.data_ptr() + want.size + 8 - (want.size % 4)])
    torch.cuda.synchronize()
    check(f"mirrored fused={fused}", out.cpu().numpy(), want)
    check(f"mirror 0 fused={fused}", m[:want.size].cpu().numpy(), want)

for K, polys, D, L, n in [(5, (0o23, 0o33), 64, 20, 2000), (12, (0o5723, 0o6265), 64, 60, 600)]:
    code = {"K": K, "polys": polys}
    _, l2 = synth.make_stream(code, n, 3.0, 7)
    w2 = O.pack_bits(O.decode(code, l2.numpy(), n, D, L))
    dec = P.Decoder(K, polys, D, L)
    check(f"jit K={K}", dec.decode(l2.cuda(), n).cpu().numpy(), w2)

p34 = synth.PUNCT["3/4"]
_, l3 = synth.make_stream(k7, 2000, 4.0, 9, p34)
w3 = O.pack_bits(O.decode(k7, l3.numpy(), 2000, 96, 30, punct=p34))
dec = P.Decoder(7, k7["polys"], 96, 30, punct=p34)
check("punctured 3/4", dec.decode(l3.cuda(), 2000).cpu().numpy(), w3)
sd = dec.open_stream()
d3 = l3.cuda()
parts = [sd.push(d3[a:b].clone()) for a, b in ((0, 777), (777, 1501), (1501, d3.numel()))]
tail, _ = sd.finish()
sd.close()
check("stream 3/4", torch.cat(parts + [tail]).cpu().numpy(), w3)

dec = P.Decoder(7, k7["polys"], 64, 20)
check("host pipeline", dec.decode_host(llr.pin_memory(), 3000).numpy(), want)
print("total bad bytes:", bad)
sys.exit(1 if bad else 0)
