"""Eq. 8 algebra -- SPEC acceptance 9: limiting cases to
1e-12 relative error and monotonicity on 10^4 random parameter draws."""
import math
import random

from paper_1608_00066_b200 import model as M


def test_eq8_limits():
    for D, L, N_t, N_s in [(512, 42, 10240, 4), (1024, 64, 512, 1), (64, 100, 7, 9)]:
        U1, U2, B = 2.0, 1 / 8, 12e9
        lim = M.eq8_printed_limit(D, L, N_s, U1, U2, B)
        got = M.eq8(D, L, N_t, N_s, U1, U2, B, S_k=1e300)
        assert math.isclose(got, lim, rel_tol=1e-12)
        # L = 0: the halo factor disappears and both halo conventions agree
        a = M.eq8(D, 0, N_t, N_s, U1, U2, B, 1e11, halo="block")
        b = M.eq8(D, 0, N_t, N_s, U1, U2, B, 1e11, halo="window")
        assert math.isclose(a, b, rel_tol=1e-12)
        # N_s = 1: Eq. 8 and the transfer-bound form coincide
        a = M.eq8(D, L, N_t, 1, U1, U2, B, 1e11, halo="window")
        b = M.transfer_bound(D, L, N_t, 1, U1, U2, B, 1e11, halo="window")
        assert math.isclose(a, b, rel_tol=1e-12)


def test_eq8_monotone_random():
    rng = random.Random(9)
    for _ in range(10000):
        D = rng.choice([64, 128, 256, 512, 1024]); L = rng.randint(1, 200)
        N_t = rng.randint(1, 20000); N_s = rng.randint(1, 16)
        U1 = rng.choice([0.5, 1.0, 1.5, 2.0, 3.0]); U2 = 1 / 8
        B = rng.uniform(1e9, 64e9); S_k = rng.uniform(1e8, 2e11)
        base = M.eq8(D, L, N_t, N_s, U1, U2, B, S_k)
        assert M.eq8(D, L, N_t, N_s, U1, U2, B * 1.1, S_k) > base        # faster link
        assert M.eq8(D, L, N_t, N_s, U1, U2, B, S_k * 1.1) > base        # faster kernel
        assert M.eq8(D, L + 1, N_t, N_s, U1, U2, B, S_k) < base          # more halo
        assert base < S_k * (1 + 1e-12) or N_s == 0                      # never beats the kernel
        tb = M.transfer_bound(D, L, N_t, N_s, U1, U2, B, S_k)
        assert tb <= B / U1 * (1 + 1e-12)                                  # never beats the link
        m = M.model(D, L, N_t, N_s, U1, U2, B, S_k)
        assert math.isclose(m["model_gbs"], min(m["eq8_gbs"], m["transfer_bound_gbs"]))
