"""GPU BER harness: decoded-bit error rate of the
segmented decoder on the GPU over Eb/N0 and L sweeps, with the info bits of
the seeded synthetic stream as ground truth.

    python tools/ber_sweep.py --code k7 --ebn0 3 4 4.5 5 --L 7 14 28 42 63 \
        --bits 67108864 [--start s0] [--json out.json]

Reproduces the paper's E2 experiments at scale (Fig. 4:
BER vs L at fixed Eb/N0, traceback from the min-PM state) and the BER level
against the union bound from the (171,133) distance spectrum (SURVEY §8(c)
pins).  Each point decodes `--bits` info bits in streams of up to 2^26 bits
(generated on the GPU, distinct seeds), so 10^9-10^10-bit points are a loop.
"""
from __future__ import annotations

import argparse
import json
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import synth  # noqa: E402

# bit-weight spectrum B_d of the K=7 (171,133) code, d = 10..22
B_D = {10: 36, 12: 211, 14: 1404, 16: 11633, 18: 77433, 20: 502690, 22: 3322763}


def union_bound_k7(ebn0_db, rate=0.5):
    g = 10 ** (ebn0_db / 10)
    return sum(b * 0.5 * math.erfc(math.sqrt(d * rate * g)) for d, b in B_D.items())


def ber_point(P, code, ebn0, D, L, n_bits, seed, punct=None, hard=False, chunk=1 << 26):
    """(errors, bits) of the GPU decoder over n_bits info bits."""
    errs, total, k = 0, 0, 0
    dec = P.Decoder(code["K"], code["polys"], D, L, punct=punct)
    while total < n_bits:
        n = min(chunk, n_bits - total)
        n -= n % D if n > D else 0
        info, llr = synth.make_stream(code, n, ebn0, seed + 7919 * k, punct, hard,
                                      device="cuda")
        out = dec.decode(llr, n)
        got = torch.stack([(out >> i) & 1 for i in range(8)], dim=1).reshape(-1)[:n]
        errs += int((got != info).sum().item())
        total += n
        k += 1
    return errs, total


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--code", default="k7", choices=list(synth.CODES))
    ap.add_argument("--punct", default="1/2", choices=list(synth.PUNCT))
    ap.add_argument("--ebn0", type=float, nargs="+", default=[3.0, 4.0, 4.5])
    ap.add_argument("--L", type=int, nargs="+", default=[42])
    ap.add_argument("--D", type=int, default=512)
    ap.add_argument("--bits", type=int, default=1 << 26)
    ap.add_argument("--hard", action="store_true")
    ap.add_argument("--seed", type=int, default=4242)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    from paper_1608_00066_b200 import build
    build.build()
    import paper_1608_00066_b200 as P
    code, punct = synth.CODES[a.code], synth.PUNCT[a.punct]
    rows = []
    for e in a.ebn0:
        for L in a.L:
            errs, n = ber_point(P, code, e, a.D, L, a.bits, a.seed, punct, a.hard)
            row = {"code": a.code, "punct": a.punct, "hard": a.hard, "ebn0": e, "D": a.D, "L": L,
                   "bits": n, "errors": errs, "ber": errs / n}
            if a.code == "k7" and a.punct == "1/2" and not a.hard:
                row["union_bound"] = union_bound_k7(e)
                row["ber_over_ub"] = row["ber"] / row["union_bound"]
            rows.append(row)
            print(json.dumps(row), flush=True)
    if a.json:
        Path(a.json).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
