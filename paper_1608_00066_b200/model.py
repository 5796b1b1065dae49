"""The paper's end-to-end throughput model (Eq. 8, §IV.C) and its
transfer-bound counterpart, used by bench.py to put the measured e2e number
(pbvd_decode_host) beside the model.  Host arithmetic only.

Eq. 8 as printed, T/P ~ B N_s / ((1 + 2L/D) U1 + N_s / S_k + U2), mixes units
(S_k in bit/s against byte terms).  Rewritten from its own first
line, T/P = D N_t N_s / (T_H2D + N_s T_k + T_D2H) with
T_H2D = (D + 2L) N_t U1 / B, T_k = D N_t / S_k, T_D2H = D N_t U2 / B
(P:290-291), dividing through by D N_t gives the dimensionally consistent

    T/P = B N_s / ((1 + 2L/D) U1 + N_s B / S_k + U2)            (eq8)

(B in bytes/s, U1 bytes per input stage, U2 bytes per decoded bit, S_k in
bit/s).  Its premise is the compute-bound regime: every transfer except the
first H2D batch and the last D2H batch hides behind kernels.  On B200 the
kernels outrun PCIe (C2: S_k ~ 90 Gb/s vs B/U1 ~ 27 Gb/s), so the copies are
the critical path instead:

    T/P = D N_t N_s / (N_s T_H2D + T_k + T_D2H)                (transfer_bound)

with the last batch's kernel and D2H after the final H2D byte.  Our pipeline
sends each stage once (a contiguous window: halo factor 1 + 2L/(D N_t) per
batch instead of 1 + 2L/D), which `halo` selects.
"""
from __future__ import annotations


def t_h2d(D, L, N_t, U1, B, halo="block"):
    """Seconds to copy one batch of N_t blocks' input."""
    stages = (D + 2 * L) * N_t if halo == "block" else D * N_t + 2 * L
    return stages * U1 / B


def t_d2h(D, N_t, U2, B):
    """Seconds to copy one batch's decoded bits."""
    return D * N_t * U2 / B


def eq8(D, L, N_t, N_s, U1, U2, B, S_k, halo="block"):
    """Eq. 8 (dimensionally consistent form): decoded bit/s of N_s batches."""
    T_k = D * N_t / S_k
    return D * N_t * N_s / (t_h2d(D, L, N_t, U1, B, halo) + N_s * T_k + t_d2h(D, N_t, U2, B))


def eq8_printed_limit(D, L, N_s, U1, U2, B):
    """The S_k -> infinity limit of Eq. 8: B N_s / ((1 + 2L/D) U1 + U2)."""
    return B * N_s / ((1 + 2 * L / D) * U1 + U2)


def transfer_bound(D, L, N_t, N_s, U1, U2, B, S_k, halo="window"):
    """The PCIe-bound counterpart: every H2D batch is on the critical path,
    then the last batch's kernel and D2H."""
    T_k = D * N_t / S_k
    return D * N_t * N_s / (N_s * t_h2d(D, L, N_t, U1, B, halo) + T_k + t_d2h(D, N_t, U2, B))


def model(D, L, N_t, N_s, U1, U2, B, S_k):
    """Both forms and the regime they predict (min of the two = the bound of
    a pipeline that overlaps perfectly)."""
    a = eq8(D, L, N_t, N_s, U1, U2, B, S_k, halo="window")
    b = transfer_bound(D, L, N_t, N_s, U1, U2, B, S_k, halo="window")
    return {"eq8_gbs": a / 1e9, "transfer_bound_gbs": b / 1e9, "model_gbs": min(a, b) / 1e9,
            "regime": "transfer" if b < a else "compute",
            "inputs": {"D": D, "L": L, "N_t": N_t, "N_s": N_s, "U1": U1, "U2": U2,
                       "B_gbs": B / 1e9, "S_k_gbs": S_k / 1e9}}
