"""GPU BER harness: decoded-bit error rate of the
segmented decoder on the GPU over Eb/N0 and L sweeps, with the info bits of
the seeded synthetic stream as ground truth.

    python tools/ber_sweep.py --code k7 --ebn0 3 4 4.5 5 --L 7 14 28 42 63 \
        --bits 67108864 [--start minpm|s0|both] [--oracle-blocks 64] [--json out.json]

Reproduces the paper's E2 experiments at scale (Fig. 4:
BER vs L at fixed Eb/N0) for both traceback starts: the paper's own S_0 rule
(Alg. 1 K2 state = 0; PBVD_START_ZERO) and the min-PM state of
P:75 (reading c-10), and the BER level against the union bound from the
(171,133) distance spectrum (SURVEY §8(c) pins).  Each point decodes `--bits`
info bits in streams of up to 2^26 bits (generated on the GPU, distinct
seeds), so 10^9-10^10-bit points are a loop.  Every point carries two 95 %
intervals: Wilson (bit errors as independent Bernoulli trials) and batch
means over the streams (robust to the burstiness of Viterbi errors), and --
as SPEC S:329-337's run_ber does with reference_viterbi -- the first
`--oracle-blocks` blocks of its first stream decoded by the CPU oracle on the
same noisy frames, which must agree bit for bit.
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


def wilson(k, n, z=1.959964):
    """95 % Wilson score interval of a binomial proportion k / n."""
    if n == 0:
        return (0.0, 1.0)
    p = k / n
    den = 1 + z * z / n
    mid = (p + z * z / (2 * n)) / den
    half = z * math.sqrt(p * (1 - p) / n + z * z / (4 * n * n)) / den
    return (max(0.0, mid - half), min(1.0, mid + half))


def batch_ci(errs, bits, z=1.959964):
    """95 % normal interval of the BER from per-stream batch means (each
    stream an independent batch; robust to burst errors).  None if < 4."""
    m = len(errs)
    if m < 4:
        return None
    rates = [e / b for e, b in zip(errs, bits)]
    tot = sum(errs) / sum(bits)
    var = sum((r - tot) ** 2 for r in rates) / (m - 1)
    half = z * math.sqrt(var / m)
    return (max(0.0, tot - half), tot + half)


def ber_point(P, code, ebn0, D, L, n_bits, seed, punct=None, hard=False, chunk=1 << 26,
              start_zero=False, oracle_blocks=0, detail=False):
    """(errors, bits) of the GPU decoder over n_bits info bits; with
    detail=True a dict with per-stream counts, intervals and the oracle check."""
    errs, total, k = 0, 0, 0
    per_e, per_b = [], []
    orc_ok = None
    dec = P.Decoder(code["K"], code["polys"], D, L, punct=punct, start_zero=start_zero)
    while total < n_bits:
        n = min(chunk, n_bits - total)
        n -= n % D if n > D else 0
        info, llr = synth.make_stream(code, n, ebn0, seed + 7919 * k, punct, hard,
                                      device="cuda")
        out = dec.decode(llr, n)
        got = torch.stack([(out >> i) & 1 for i in range(8)], dim=1).reshape(-1)[:n]
        e = int((got != info).sum().item())
        if k == 0 and oracle_blocks > 0:
            from oracle import oracle as O      # test infrastructure: the checker only
            nbk = min(oracle_blocks, -(-n // D))
            hi = min(n + code["K"] - 1, nbk * D + L)
            kk = synth.llr_count(len(code["polys"]), punct, hi)
            flags = O.TERMINATED | (O.START_ZERO if start_zero else 0)
            want = O.decode(code, llr[:kk].cpu().numpy(), n, D, L, flags=flags, punct=punct,
                            b0=0, nblk=nbk)
            orc_ok = bool((got[:want.size].cpu().numpy() == want).all())
        errs += e
        total += n
        per_e.append(e)
        per_b.append(n)
        k += 1
    if not detail:
        return errs, total
    return {"errors": errs, "bits": total, "ber": errs / total, "streams": k,
            "ci95_wilson": wilson(errs, total), "ci95_batch": batch_ci(per_e, per_b),
            "oracle_blocks_bit_exact": orc_ok}


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
    ap.add_argument("--start", default="minpm", choices=["minpm", "s0", "both"])
    ap.add_argument("--chunk", type=int, default=1 << 26)
    ap.add_argument("--oracle-blocks", type=int, default=64)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    from paper_1608_00066_b200 import build
    build.build()
    import paper_1608_00066_b200 as P
    code, punct = synth.CODES[a.code], synth.PUNCT[a.punct]
    rows = []
    starts = {"minpm": [False], "s0": [True], "both": [False, True]}[a.start]
    sys.path.insert(0, str(ROOT))
    for e in a.ebn0:
        for L in a.L:
            for sz in starts:
                # the same seeds for both starts: the two rules see the same frames
                d = ber_point(P, code, e, a.D, L, a.bits, a.seed, punct, a.hard, a.chunk,
                              start_zero=sz, oracle_blocks=a.oracle_blocks, detail=True)
                row = {"code": a.code, "punct": a.punct, "hard": a.hard, "ebn0": e, "D": a.D,
                       "L": L, "start": "s0" if sz else "minpm", **d}
                if a.code == "k7" and a.punct == "1/2" and not a.hard:
                    row["union_bound"] = union_bound_k7(e)
                    row["ber_over_ub"] = row["ber"] / row["union_bound"]
                rows.append(row)
                print(json.dumps(row), flush=True)
    if a.json:
        Path(a.json).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
