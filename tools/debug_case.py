"""Decode one small case on the GPU and compare with the oracle (dev tool)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import synth
from oracle import oracle as O
from paper_1608_00066_b200 import build
build.build()
import paper_1608_00066_b200 as P
name = sys.argv[1] if len(sys.argv) > 1 else "k7"
n_info = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
D = int(sys.argv[3]) if len(sys.argv) > 3 else 64
L = int(sys.argv[4]) if len(sys.argv) > 4 else 20
lanes = int(sys.argv[5]) if len(sys.argv) > 5 else 0
pk = sys.argv[6] if len(sys.argv) > 6 else "1/2"
fused = (sys.argv[7] != "0") if len(sys.argv) > 7 else True
code, punct = synth.CODES[name], synth.PUNCT[pk]
info, llr = synth.make_stream(code, n_info, 3.0, 5, punct)
dec = P.Decoder(code["K"], code["polys"], D, L, punct=punct, lanes=lanes, fused=fused)
got = dec.decode(llr.cuda(), n_info).cpu().numpy()
torch.cuda.synchronize()
want = O.pack_bits(O.decode(code, llr.numpy(), n_info, D, L, punct=punct))
bad = np.nonzero(got != want)[0]
print(name, n_info, D, L, dec.lanes, "bad bytes:", bad.size, bad[:10])
