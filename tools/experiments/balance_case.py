"""Decode one case with the balanced (persistent, job-moving) forward grid and
compare with the oracle; the PBVD_SCHED_* environment forces moves
(tests/test_gpu_balance.py).  usage: balance_case.py code n_info D L lanes punct fused terminated"""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import synth
from oracle import oracle as O
from paper_1608_00066_b200 import build
build.build()
import paper_1608_00066_b200 as P
name, n_info, D, L, lanes, pk = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]), sys.argv[6]
fused = sys.argv[7] != "0"
term = sys.argv[8] != "0"
code, punct = synth.CODES[name], synth.PUNCT[pk]
info, llr = synth.make_stream(code, n_info, 3.0, 11, punct, terminated=term)
want = O.pack_bits(O.decode(code, llr.numpy(), n_info, D, L, flags=(O.TERMINATED if term else 0), punct=punct))
dec = P.Decoder(code["K"], code["polys"], D, L, punct=punct, lanes=lanes, fused=fused,
                terminated=term)
assert dec.balance
d = llr.cuda()
out = dec.decode(d, n_info)
for rep in range(3):           # repeated launches reuse the queue block
    out = dec.decode(d, n_info, out=out)
torch.cuda.synchronize()
got = out.cpu().numpy()
bad = np.nonzero(got != want)[0]
print(name, n_info, D, L, dec.lanes, "fused", fused, "bad bytes:", bad.size, bad[:10])
