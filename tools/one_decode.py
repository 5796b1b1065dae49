"""Run a few decodes of a BASELINE config (for ncu captures)."""
import sys
sys.path.insert(0, '.')
import torch
import synth
from paper_1608_00066_b200 import build
build.build()
import paper_1608_00066_b200 as P
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
lanes = int(sys.argv[3]) if len(sys.argv) > 3 else 0
fused = (sys.argv[4] != "0") if len(sys.argv) > 4 else True
c = dict(synth.CONFIGS[cfg])
if len(sys.argv) > 5:
    c["n_info"] = int(sys.argv[5])
code, punct = synth.CODES[c["code"]], synth.PUNCT[c["punct"]]
info, llr = synth.make_stream(code, c["n_info"], c["ebn0"], c["seed"], punct, c["hard"], device="cuda")
dec = P.Decoder(code["K"], code["polys"], c["D"], c["L"], punct=punct, lanes=lanes, fused=fused)
for _ in range(reps):
    out = dec.decode(llr, c["n_info"])
torch.cuda.synchronize()
print("done", cfg, dec.lanes)
