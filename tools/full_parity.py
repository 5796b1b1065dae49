"""Every bit of full-size BASELINE streams (default C5, 2^32 bits): GPU
decode vs the CPU oracle on all host cores (SURVEY §8(c.iii) "GPU == oracle
... C5: all 8.4 M blocks").  Writes a JSON summary (tools/, not a test:
minutes of CPU time).

    python tools/full_parity.py [out.json] [C5 C3a C3b C4 ...]
"""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from oracle import oracle as O  # noqa: E402
import paper_1608_00066_b200 as P  # noqa: E402

def run(name):
    c = synth.CONFIGS[name]
    code, punct = synth.CODES[c["code"]], synth.PUNCT[c["punct"]]
    n_info, D, L = c["n_info"], c["D"], c["L"]
    n_stages = synth.n_stages_of(code, n_info)
    t0 = time.time()
    llr = synth.make_window(code, n_info, c["ebn0"], c["seed"], 0, n_stages, punct, c["hard"],
                            device="cuda")
    dec = P.Decoder(code["K"], code["polys"], D, L, punct=punct)
    out = dec.decode(llr, n_info)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    host = llr.cpu().numpy()
    del llr, out
    t1 = time.time()
    want = O.pack_bits(O.decode(code, host, n_info, D, L, punct=punct))
    t2 = time.time()
    diff = int(np.count_nonzero(got != want))
    return {"workload": name, "n_info": n_info, "blocks": int(dec.block_count(n_info)),
            "bytes_compared": int(got.size), "bytes_differing": diff, "bit_exact": diff == 0,
            "sha256_gpu": __import__("hashlib").sha256(got.tobytes()).hexdigest(),
            "oracle_cores": os.cpu_count(), "oracle_seconds": round(t2 - t1, 1),
            "gpu_gen_decode_seconds": round(t1 - t0, 1)}


O.build()
names = sys.argv[2:] or ["C5"]
res = []
for nm in names:
    r = run(nm)
    print(json.dumps(r), flush=True)
    res.append(r)
if len(sys.argv) > 1:
    Path(sys.argv[1]).write_text(json.dumps(res, indent=1) + "\n")
