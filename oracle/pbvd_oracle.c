/*
 * pbvd_oracle.c -- plain, slow, obviously-correct CPU oracle for the
 * parallel block-based Viterbi decoder (PBVD) of Peng et al.,
 * "A Gb/s Parallel Block-based Viterbi Decoder for Convolutional Codes on GPU"
 * (arXiv 1608.00066).  Citations "P:n" are lines of /root/reference/PAPER.md,
 * "S:n" lines of SPEC.md, "c-n" the readings table of SURVEY.md §8(c) which
 * DESIGN.md §3 restates.
 *
 * THIS FILE IS TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  It shares no
 * code, header, table or constant with the CUDA library under
 * paper_1608_00066_b200/ and neither side includes the other.
 *
 * What it computes (step by step, in the paper's order):
 *   - trellis:   Eq. 2 encoder output c(S_d, x) and the shift
 *                S_2j,S_2j+1 -> S_j, S_{j+2^{v-1}}
 *   - grouping:  Eqs. 3-6 and the N_c = 2^R groups;
 *                used only to pin Table II, not in the decoder
 *   - decoder:   per parallel block a per-edge ACS, Eq. 1
 *                (P:72-74), over [t-L, t+D+L) with int32 path metrics, no
 *                grouping, no normalisation; traceback (Alg. 1 K2,
 *                P:216-225) from the minimum-PM state, emitting the
 *                D decoded bits, packed 8 per byte.
 *   - full:      textbook Viterbi over the whole stream (int64), the special
 *                case D >= n_info, used only to validate the oracle.
 *   - ml:        brute-force maximum-likelihood over all 2^k info words, used
 *                only to validate the oracle on tiny inputs.
 *
 * Parity status of each function is listed in DESIGN.md §4 ("pins").
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define ORC_TERMINATED 1u     /* stream ends with v zero tail bits (c-13)      */
#define ORC_START_ZERO 2u     /* traceback from state S_0 instead of min-PM    */
                              /* (P:93 variant, c-10; Fig. 4 study only)       */
#define ORC_S_HEAD 8192       /* known-start sentinel for head blocks (c-12)   */

/* ---------------------------------------------------------------- trellis */

static int parity32(uint32_t x) {
    int p = 0;
    while (x) { p ^= 1; x &= x - 1; }
    return p;
}

/* Eq. 2: c^(r) = x*g_{K-1} ^ D_{K-2}*g_{K-2} ^ ... ^ D_0*g_0,
 * with state d = (D_{v-1} ... D_0)_2.  Generator bit i is g_i, so bit
 * K-1 multiplies the input x and bit i < K-1 multiplies D_i (c-1, c-2).
 * Returns the R output bits packed as bit r = c^(r+1). */
int orc_out(int K, int R, const uint32_t *polys, uint32_t d, int x) {
    uint32_t reg = ((uint32_t)x << (K - 1)) | d;
    int c = 0;
    for (int r = 0; r < R; r++)
        c |= parity32(reg & polys[r]) << r;
    return c;
}

/* S_2j and S_2j+1 shift to S_j (x=0) or S_{j+2^{v-1}} (x=1). */
uint32_t orc_next(int K, uint32_t d, int x) {
    int v = K - 1;
    return ((uint32_t)x << (v - 1)) | (d >> 1);
}

/* One traceback step of Alg. 1 K2: the decoded bit of the
 * current state is (state >> (K-2)) & 1 and, with sp its survivor bit,
 * the predecessor is 2 * (state mod 2^{K-2}) + sp. */
uint32_t orc_tb_step(int K, uint32_t state, int sp, int *bit) {
    *bit = (int)((state >> (K - 2)) & 1u);
    uint32_t j = state % (1u << (K - 2));
    return 2 * j + (uint32_t)sp;
}

/* Eqs. 3-6 for butterfly j: alpha = c(S_2j,0), beta = c(S_2j,1),
 * gamma = c(S_2j+1,0), theta = c(S_2j+1,1), computed by direct evaluation of
 * Eq. 2 (the closed forms of Eqs. 4-6 are checked against these in tests). */
void orc_butterfly(int K, int R, const uint32_t *polys, uint32_t j, int out4[4]) {
    out4[0] = orc_out(K, R, polys, 2 * j, 0);
    out4[1] = orc_out(K, R, polys, 2 * j, 1);
    out4[2] = orc_out(K, R, polys, 2 * j + 1, 0);
    out4[3] = orc_out(K, R, polys, 2 * j + 1, 1);
}

/* ------------------------------------------------------------- input side */

/* Kept soft values in stages [0, s) -- the index of stage s's first kept
 * value in the punctured stream (c-18). */
static int64_t kept_before(int R, int P, const uint8_t *punct, int64_t s) {
    if (P <= 1 || !punct) return s * R;
    int64_t per = 0, part = 0;
    for (int p = 0; p < P; p++)
        for (int r = 0; r < R; r++) {
            per += punct[r * P + p] ? 1 : 0;
            if (p < (int)(s % P)) part += punct[r * P + p] ? 1 : 0;
        }
    return (s / P) * per + part;
}

/* Number of kept soft values in stages [0, n_stages): the keep matrix
 * punct[r*P + p] applies to column p = stage mod P, anchored at stage 0
 * (c-18).  P = 1 / punct = NULL means unpunctured. */
int64_t orc_llr_count(int R, int P, const uint8_t *punct, int64_t n_stages) {
    return kept_before(R, P, punct, n_stages);
}

/* Depuncture stages [s0, s1) reading kept values from llr[i], llr[i+1], ...
 * (llr[i] being the first kept value of stage s0). */
static void depuncture_from(int R, int P, const uint8_t *punct, const int8_t *llr, int64_t i,
                            int64_t s0, int64_t s1, int32_t *lam) {
    for (int64_t s = s0; s < s1; s++)
        for (int r = 0; r < R; r++) {
            int keep = (P <= 1 || !punct) ? 1 : punct[r * P + (int)(s % P)];
            lam[(s - s0) * R + r] = keep ? llr[i++] : 0;
        }
}

/* Depuncture the stage range [s0, s1) into lam[(s-s0)*R + r]: the next kept
 * int8 value, or 0 (erasure) at a punctured position (c-18). */
static void depuncture_range(int R, int P, const uint8_t *punct, const int8_t *llr,
                             int64_t s0, int64_t s1, int32_t *lam) {
    int64_t i = kept_before(R, P, punct, s0);
    depuncture_from(R, P, punct, llr, i, s0, s1, lam);
}

/* Branch metric, canonical integer form (c-4): BM(c) = sum_r c_r*lam_r,
 * to be minimised.  lam > 0 favours coded bit 0 (c-5). */
static int32_t bm(const int32_t *lam_s, int R, int c) {
    int32_t m = 0;
    for (int r = 0; r < R; r++)
        if ((c >> r) & 1) m += lam_s[r];
    return m;
}

/* --------------------------------------------------- block plan */

/* Block b decodes [t0, t1) = [bD, min(bD+D, n_info)); its forward span is
 * [lo, hi) with lo = max(0, t0-L) (truncated block, M = L, c-14) and
 * hi = n_stages for the last block, else min(n_stages, t1+L) (traceback
 * block).  Returns the number of blocks. */
int64_t orc_plan(int64_t n_info, int64_t n_stages, int D, int L, int64_t b,
                 int64_t *t0, int64_t *t1, int64_t *lo, int64_t *hi) {
    int64_t nb = (n_info + D - 1) / D;
    if (b >= 0 && b < nb) {
        *t0 = b * D;
        *t1 = (*t0 + D < n_info) ? *t0 + D : n_info;
        *lo = (*t0 - L > 0) ? *t0 - L : 0;
        if (b == nb - 1) *hi = n_stages;
        else *hi = (*t1 + L < n_stages) ? *t1 + L : n_stages;
    }
    return nb;
}

/* ------------------------------------------------------------- one block */

typedef struct {
    int K, R;
    const uint32_t *polys;
    int P;
    const uint8_t *punct;
    const int8_t *llr;       /* soft values from stage ws0, [stage][r] (c-17) */
    int64_t kb_ws0;          /* kept values before stage ws0 (index of llr[0]) */
    int64_t n_info, n_stages;
    int D, L;
    unsigned flags;
    int64_t b_first;         /* first block of the decoded range           */
    uint8_t *bits;           /* unpacked bits from t0(b_first), 1 per byte */
    int32_t *starts;         /* per-block traceback start state (range)    */
    int64_t *ties;           /* per-block count of exact ACS ties (range)  */
} orc_job;

/* Forward ACS over the span of block b (Eq. 1), per edge, then
 * traceback (Alg. 1 K2).  dec_out, if non-NULL, receives the raw
 * decision bits dec[(s-lo)*N + u] (one byte each) for inspection. */
static int orc_block(const orc_job *J, int64_t b, uint8_t *dec_out) {
    const int K = J->K, R = J->R, v = K - 1, N = 1 << v, half = N >> 1;
    int64_t t0, t1, lo, hi;
    int64_t nb = orc_plan(J->n_info, J->n_stages, J->D, J->L, b, &t0, &t1, &lo, &hi);
    int64_t span = hi - lo;
    int32_t *lam = (int32_t *)malloc(sizeof(int32_t) * (size_t)(span * R));
    int32_t *pm = (int32_t *)malloc(sizeof(int32_t) * N);
    int32_t *pmn = (int32_t *)malloc(sizeof(int32_t) * N);
    uint8_t *dec = dec_out ? dec_out : (uint8_t *)malloc((size_t)span * N);
    int *outs = (int *)malloc(sizeof(int) * N * 2);
    if (!lam || !pm || !pmn || !dec || !outs) return -1;
    depuncture_from(R, J->P, J->punct, J->llr,
                    kept_before(R, J->P, J->punct, lo) - J->kb_ws0, lo, hi, lam);
    for (int d = 0; d < N; d++)
        for (int x = 0; x < 2; x++) outs[d * 2 + x] = orc_out(K, R, J->polys, (uint32_t)d, x);

    /* Initial metrics: "unknown initial state metrics (typically set to zero)"
     * for interior blocks; a head block (lo == 0) starts in the known
     * state 0 (c-12). */
    for (int u = 0; u < N; u++)
        pm[u] = (lo == 0) ? (u == 0 ? 0 : ORC_S_HEAD) : 0;

    int64_t ties = 0;
    for (int64_t s = lo; s < hi; s++) {
        const int32_t *ls = lam + (s - lo) * R;
        for (int u = 0; u < N; u++) {
            int j = u % half, x = u / half;              /* u = j + x*2^{v-1} */
            int32_t m0 = pm[2 * j] + bm(ls, R, outs[(2 * j) * 2 + x]);         /* upper */
            int32_t m1 = pm[2 * j + 1] + bm(ls, R, outs[(2 * j + 1) * 2 + x]); /* lower */
            uint8_t d = (m1 < m0) ? 1 : 0;     /* tie -> upper, bit 0 (c-8) */
            if (m1 == m0) ties++;
            dec[(s - lo) * N + u] = d;
            pmn[u] = d ? m1 : m0;
        }
        memcpy(pm, pmn, sizeof(int32_t) * N);
    }

    /* Start state: min-PM, lowest index on ties (c-10); state 0 for a
     * terminated last block (c-13); or S_0 in the P:93 variant. */
    int32_t st = 0;
    int last = (b == nb - 1);
    if (!((J->flags & ORC_TERMINATED) && last) && !(J->flags & ORC_START_ZERO)) {
        for (int u = 1; u < N; u++)
            if (pm[u] < pm[st]) st = u;
    }
    int64_t first_t0 = J->b_first * (int64_t)J->D;
    J->starts[b - J->b_first] = st;
    J->ties[b - J->b_first] = ties;

    /* Traceback, Alg. 1 K2: emit (state >> (K-2)) & 1 inside the decoding
     * block, then state = 2*(state mod 2^{K-2}) + sp. */
    uint32_t state = (uint32_t)st;
    for (int64_t s = hi - 1; s >= t0; s--) {
        int bit;
        uint32_t prev = orc_tb_step(K, state, dec[(s - lo) * N + state], &bit);
        if (s < t1) J->bits[s - first_t0] = (uint8_t)bit;
        state = prev;
    }
    if (!dec_out) free(dec);
    free(lam); free(pm); free(pmn); free(outs);
    return 0;
}

typedef struct { const orc_job *J; int64_t b0, b1; int rc; } orc_slice;

static void *orc_worker(void *arg) {
    orc_slice *sl = (orc_slice *)arg;
    sl->rc = 0;
    for (int64_t b = sl->b0; b < sl->b1 && sl->rc == 0; b++)
        sl->rc = orc_block(sl->J, b, NULL);
    return NULL;
}

static int check_code(int K, int R, int D, int L, int64_t n_info) {
    return (K < 2 || K > 16 || R < 1 || R > 8 || D < 1 || L < 0 || n_info < 1) ? -1 : 0;
}

/* Segmented PBVD decode of the blocks [b0, b0+nblk) of a stream:
 * every block decoded independently (static split over `threads` pthreads),
 * outputs gathered in stream order.
 *   llr     : n_llr int8 soft values of the punctured stream starting at the
 *             first kept value of stage ws0 ([stage][r] order, punctured
 *             positions omitted, c-17); ws0 = 0 for a whole stream
 *   n_info  : info bits; n_stages = n_info + (TERMINATED ? K-1 : 0)
 *   bits    : unpacked decoded bits of [t0(b0), t1(b0+nblk-1)), one per byte
 *   starts  : optional, nblk int32 start states
 *   ties    : optional, total exact ACS ties (int64)
 * Returns the total block count of the stream, or a negative value. */
int64_t orc_decode_range(int K, int R, const uint32_t *polys, int P, const uint8_t *punct,
                         const int8_t *llr, int64_t ws0, int64_t n_llr, int64_t n_info, int D,
                         int L, unsigned flags, int64_t b0, int64_t nblk, int threads,
                         uint8_t *bits, int32_t *starts, int64_t *ties_total) {
    if (check_code(K, R, D, L, n_info)) return -1;
    int64_t n_stages = n_info + ((flags & ORC_TERMINATED) ? K - 1 : 0);
    int64_t nb = (n_info + D - 1) / D;
    if (b0 < 0 || nblk < 1 || b0 + nblk > nb || ws0 < 0) return -1;
    /* the window [ws0, ...) must hold every span of the range */
    int64_t kb_ws0 = kept_before(R, P, punct, ws0);
    {
        int64_t t0, t1, lo, hi, u0, u1, ulo, uhi;
        orc_plan(n_info, n_stages, D, L, b0, &t0, &t1, &lo, &hi);
        orc_plan(n_info, n_stages, D, L, b0 + nblk - 1, &u0, &u1, &ulo, &uhi);
        if (lo < ws0 || kept_before(R, P, punct, uhi) - kb_ws0 > n_llr) return -3;
    }
    int32_t *st = (int32_t *)malloc(sizeof(int32_t) * (size_t)nblk);
    int64_t *tie = (int64_t *)calloc((size_t)nblk, sizeof(int64_t));
    if (!st || !tie) return -2;
    orc_job J = {K, R, polys, P, punct, llr, kb_ws0, n_info, n_stages, D, L, flags, b0, bits, st,
                 tie};
    if (threads < 1) threads = 1;
    if (threads > nblk) threads = (int)nblk;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * threads);
    orc_slice *sl = (orc_slice *)malloc(sizeof(orc_slice) * threads);
    for (int i = 0; i < threads; i++) {
        sl[i].J = &J;
        sl[i].b0 = b0 + nblk * i / threads;
        sl[i].b1 = b0 + nblk * (i + 1) / threads;
        pthread_create(&th[i], NULL, orc_worker, &sl[i]);
    }
    int rc = 0;
    for (int i = 0; i < threads; i++) { pthread_join(th[i], NULL); rc |= sl[i].rc; }
    if (rc == 0) {
        if (starts) memcpy(starts, st, sizeof(int32_t) * (size_t)nblk);
        if (ties_total) {
            int64_t t = 0;
            for (int64_t b = 0; b < nblk; b++) t += tie[b];
            *ties_total = t;
        }
    }
    free(th); free(sl); free(st); free(tie);
    return rc ? -4 : nb;
}

/* Raw decisions of one block for inspection: dec[(s-lo)*N + u] bytes over
 * its span [lo, hi), plus its start state.  Same routine as the decoder. */
int orc_block_decisions(int K, int R, const uint32_t *polys, int P, const uint8_t *punct,
                        const int8_t *llr, int64_t n_llr, int64_t n_info, int D, int L,
                        unsigned flags, int64_t b, uint8_t *dec, int64_t *lo_out,
                        int64_t *hi_out, int32_t *start) {
    if (check_code(K, R, D, L, n_info)) return -1;
    int64_t n_stages = n_info + ((flags & ORC_TERMINATED) ? K - 1 : 0);
    if (orc_llr_count(R, P, punct, n_stages) != n_llr) return -3;
    int64_t t0, t1, lo, hi;
    int64_t nb = orc_plan(n_info, n_stages, D, L, b, &t0, &t1, &lo, &hi);
    if (b < 0 || b >= nb) return -1;
    uint8_t *bits = (uint8_t *)calloc((size_t)(t1 - t0), 1);
    int32_t st = 0;
    int64_t tie = 0;
    orc_job J = {K, R, polys, P, punct, llr, 0, n_info, n_stages, D, L, flags, b, bits, &st, &tie};
    int rc = orc_block(&J, b, dec);
    *lo_out = lo; *hi_out = hi; *start = st;
    free(bits);
    return rc;
}

/* ------------------------------------------------- full-stream Viterbi (§II) */

/* Textbook Viterbi over the whole stream (§II): start in the known
 * state 0, per-edge ACS (Eq. 1) with int64 metrics, traceback from state 0
 * if TERMINATED else from the min-PM state (lowest index on ties).  This is
 * orc_decode with D >= n_info, written separately so each validates the
 * other.  Writes the unpacked bits (one byte per bit) and the final metric
 * of the decoded path. */
int orc_full(int K, int R, const uint32_t *polys, int P, const uint8_t *punct,
             const int8_t *llr, int64_t n_llr, int64_t n_info, unsigned flags,
             uint8_t *bits, int64_t *metric) {
    const int v = K - 1, N = 1 << v, half = N >> 1;
    int64_t n_stages = n_info + ((flags & ORC_TERMINATED) ? v : 0);
    if (orc_llr_count(R, P, punct, n_stages) != n_llr) return -3;
    int32_t *lam = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n_stages * R));
    if (!lam) return -2;
    depuncture_range(R, P, punct, llr, 0, n_stages, lam);
    const int64_t BIG = (int64_t)1 << 50;
    int64_t *pm = (int64_t *)malloc(sizeof(int64_t) * N);
    int64_t *pmn = (int64_t *)malloc(sizeof(int64_t) * N);
    uint8_t *dec = (uint8_t *)malloc((size_t)(n_stages * N));
    if (!pm || !pmn || !dec) return -2;
    for (int u = 0; u < N; u++) pm[u] = (u == 0) ? 0 : BIG;
    for (int64_t s = 0; s < n_stages; s++) {
        const int32_t *ls = lam + s * R;
        for (int u = 0; u < N; u++) {
            int j = u % half, x = u / half;
            int64_t m0 = pm[2 * j] + bm(ls, R, orc_out(K, R, polys, 2 * j, x));
            int64_t m1 = pm[2 * j + 1] + bm(ls, R, orc_out(K, R, polys, 2 * j + 1, x));
            uint8_t d = (m1 < m0) ? 1 : 0;
            dec[s * N + u] = d;
            pmn[u] = d ? m1 : m0;
        }
        memcpy(pm, pmn, sizeof(int64_t) * N);
    }
    int st = 0;
    if (!(flags & ORC_TERMINATED))
        for (int u = 1; u < N; u++) if (pm[u] < pm[st]) st = u;
    *metric = pm[st];
    uint32_t state = (uint32_t)st;
    for (int64_t s = n_stages - 1; s >= 0; s--) {
        int bit;
        uint32_t prev = orc_tb_step(K, state, dec[s * N + state], &bit);
        if (s < n_info) bits[s] = (uint8_t)bit;
        state = prev;
    }
    free(lam); free(pm); free(pmn); free(dec);
    return 0;
}

/* ------------------------------------------------ brute-force ML (tiny k) */

/* Metric of one info sequence: encode from state 0 by Eq. 2 and the shift of
 * P:133 (plus v zero tail stages if TERMINATED) and sum the canonical BMs. */
static int64_t path_metric(int K, int R, const uint32_t *polys, const int32_t *lam,
                           const uint8_t *bits, int64_t n_info, int64_t n_stages) {
    uint32_t d = 0;
    int64_t m = 0;
    for (int64_t s = 0; s < n_stages; s++) {
        int x = (s < n_info) ? bits[s] : 0;
        m += bm(lam + s * R, R, orc_out(K, R, polys, d, x));
        d = orc_next(K, d, x);
    }
    return m;
}

int orc_path_metric(int K, int R, const uint32_t *polys, int P, const uint8_t *punct,
                    const int8_t *llr, int64_t n_llr, int64_t n_info, unsigned flags,
                    const uint8_t *bits, int64_t *metric) {
    int64_t n_stages = n_info + ((flags & ORC_TERMINATED) ? K - 1 : 0);
    if (orc_llr_count(R, P, punct, n_stages) != n_llr) return -3;
    int32_t *lam = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n_stages * R));
    if (!lam) return -2;
    depuncture_range(R, P, punct, llr, 0, n_stages, lam);
    *metric = path_metric(K, R, polys, lam, bits, n_info, n_stages);
    free(lam);
    return 0;
}

/* Exhaustive ML over all 2^n_info info words (n_info <= 24): the minimum
 * metric, how many words attain it, and the lowest-index minimiser (bit s of
 * the word index = info bit s). */
int orc_ml(int K, int R, const uint32_t *polys, int P, const uint8_t *punct,
           const int8_t *llr, int64_t n_llr, int n_info, unsigned flags,
           int64_t *best_metric, int64_t *n_best, uint8_t *best_bits) {
    if (n_info < 1 || n_info > 24) return -1;
    int64_t n_stages = n_info + ((flags & ORC_TERMINATED) ? K - 1 : 0);
    if (orc_llr_count(R, P, punct, n_stages) != n_llr) return -3;
    int32_t *lam = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n_stages * R));
    if (!lam) return -2;
    depuncture_range(R, P, punct, llr, 0, n_stages, lam);
    uint8_t *bits = (uint8_t *)malloc((size_t)n_info);
    int64_t best = INT64_MAX, cnt = 0, arg = 0;
    for (int64_t w = 0; w < ((int64_t)1 << n_info); w++) {
        for (int s = 0; s < n_info; s++) bits[s] = (uint8_t)((w >> s) & 1);
        int64_t m = path_metric(K, R, polys, lam, bits, n_info, n_stages);
        if (m < best) { best = m; cnt = 1; arg = w; }
        else if (m == best) cnt++;
    }
    for (int s = 0; s < n_info; s++) best_bits[s] = (uint8_t)((arg >> s) & 1);
    *best_metric = best;
    *n_best = cnt;
    free(lam); free(bits);
    return 0;
}
