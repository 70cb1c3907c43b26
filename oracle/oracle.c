/*
 * oracle/oracle.c -- plain, slow, obviously-correct CPU oracle for OPH / GOPH /
 * HOPH / MinWise near-duplicate scoring (arxiv 1805.11254).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / `--impl reference` legs may load this library.
 * The product (paper_1805_11254_b200/) never links, imports or calls it, and
 * this file shares no code, header, table or constant generator with the
 * CUDA path: both are written independently from PAPER.md and DESIGN.md.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n,
 * "Rn" = reading n in DESIGN.md ("Readings of the paper").
 *
 * Everything here is exact integer / rational arithmetic.  The binomial tails
 * of Eq. 10 are evaluated exactly in Python (oracle/binomial.py) and enter as
 * two boolean tables "lower(m) <= eps" and "upper(m) <= eps" (Definition 1,
 * P:278-280); the loops below follow Algorithms 1 and 2 step by step.
 *
 * Parity pins: every function is pinned by tests/test_oracle_*.py (paper
 * worked examples, Table 2, brute force, invariants); see DESIGN.md "Oracle
 * pins".  No function here is "parity unpinned".
 *
 * Build: gcc -O2 -std=c11 -fopenmp -ffp-contract=off -shared -fPIC
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_EMPTY 0xFFFFFFFFu /* the empty-bin marker ("⊗") */

/* record flags */
#define ORC_UNDEFINED 1u /* estimate undefined (k - N_eb = 0) */
#define ORC_EARLY     2u /* terminated before the last group */

/* ------------------------------------------------------------------------ */
/* O1  the permutation psi ("a random permutation psi is generated")   */
/* ------------------------------------------------------------------------ */
/* splitmix64: the counter-based stream that keys psi.     */
static uint64_t splitmix64_next(uint64_t *state)
{
    uint64_t z = (*state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

typedef struct {
    uint64_t V;        /* |V| */
    uint32_t w;        /* word size: max(1, ceil(log2 |V|)) */
    uint64_t mask;     /* 2^w - 1 */
    uint64_t kappa[4]; /* round keys */
    uint64_t mu[4];    /* round multipliers (odd) */
    int identity;      /* psi(x) = x: the paper's worked examples */
} orc_perm;

static void perm_init(orc_perm *P, uint64_t V, uint64_t seed, int identity)
{
    uint32_t w = 0;
    while (w < 64 && (1ull << w) < V) w++;
    if (w == 0) w = 1;
    P->V = V;
    P->w = w;
    P->mask = (w >= 64) ? ~0ull : ((1ull << w) - 1);
    P->identity = identity;
    uint64_t st = seed;
    for (int r = 0; r < 4; r++) {
        P->kappa[r] = splitmix64_next(&st) & P->mask;
        P->mu[r] = (splitmix64_next(&st) & P->mask) | 1ull;
    }
}

/* one pass of the 4-round keyed mix on w-bit words; each step is a bijection
 * of [0, 2^w): xor with a key, multiply by an odd number mod 2^w, xorshift */
static uint64_t perm_pass(const orc_perm *P, uint64_t x)
{
    for (int r = 0; r < 4; r++) {
        x = ((x ^ P->kappa[r]) * P->mu[r]) & P->mask;
        x ^= x >> ((P->w + 1) / 2);
    }
    return x;
}

/* psi: cycle-walk the w-bit bijection until the image lies in [0, |V|) */
uint64_t orc_psi(const orc_perm *P, uint64_t x)
{
    if (P->identity) return x;
    do {
        x = perm_pass(P, x);
    } while (x >= P->V);
    return x;
}

/* exported for tests: psi applied to an array */
void orc_psi_apply(uint64_t V, uint64_t seed, int identity, const uint64_t *x, uint64_t n, uint64_t *out)
{
    orc_perm P;
    perm_init(&P, V, seed, identity);
    for (uint64_t i = 0; i < n; i++) out[i] = orc_psi(&P, x[i]);
}

/* MinWise permutation i ("k independent random permutations"): psi keyed
 * by the i-th output of a splitmix64 stream started at seed ^ "minwise!"      */
static uint64_t minwise_seed(uint64_t seed, uint32_t i)
{
    uint64_t st = seed ^ 0x6D696E7769736521ull;
    uint64_t s = 0;
    for (uint32_t j = 0; j <= i; j++) s = splitmix64_next(&st);
    return s;
}

/* ------------------------------------------------------------------------ */
/* O2  flat layout: bin b covers [floor(b|V|/k), floor((b+1)|V|/k))    */
/* ------------------------------------------------------------------------ */
static uint64_t range_bin_start(uint64_t start, uint64_t len, uint32_t nbins, uint64_t b)
{
    return start + (uint64_t)(((unsigned __int128)b * len) / nbins);
}

/* the unique bin b of the range [start, start+len) split into nbins bins by
 * the floor rule with bin_start(b) <= p < bin_start(b+1)                     */
static uint32_t range_bin_of(uint64_t start, uint64_t len, uint32_t nbins, uint64_t p)
{
    uint64_t b = (uint64_t)(((unsigned __int128)(p - start) * nbins) / len); /* first guess */
    if (b >= nbins) b = nbins - 1;
    while (b + 1 < nbins && range_bin_start(start, len, nbins, b + 1) <= p) b++;
    while (range_bin_start(start, len, nbins, b) > p) b--;
    return (uint32_t)b;
}

/* ------------------------------------------------------------------------ */
/* O3  OPH sketch: per bin the smallest permuted element, stored as
 *     its offset from the bin start ("smallest possible representation");
 *     EMPTY if the bin holds no element.  Output set-major [n_sets][k].     */
/* ------------------------------------------------------------------------ */
void orc_oph_sketch(const uint64_t *offsets, const uint32_t *ids, uint64_t n_sets,
                    uint64_t V, uint32_t k, uint64_t seed, int identity, uint32_t *out)
{
    orc_perm P;
    perm_init(&P, V, seed, identity);
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t s = 0; s < (int64_t)n_sets; s++) {
        uint32_t *F = out + (uint64_t)s * k;
        for (uint32_t b = 0; b < k; b++) F[b] = ORC_EMPTY;
        for (uint64_t e = offsets[s]; e < offsets[s + 1]; e++) {
            uint64_t p = orc_psi(&P, ids[e]);
            uint32_t b = range_bin_of(0, V, k, p);
            uint32_t off = (uint32_t)(p - range_bin_start(0, V, k, b));
            if (F[b] == ORC_EMPTY || off < F[b]) F[b] = off;
        }
    }
}

/* ------------------------------------------------------------------------ */
/* O4  HOPH layout: recursive a:b split of the
 *     remaining space; stop when either part would be <= k', the remainder is
 *     then the final group.  Returns the group count L (0 on error).        */
/* ------------------------------------------------------------------------ */
uint32_t orc_hoph_layout(uint64_t V, uint32_t a, uint32_t b, uint32_t kp,
                         uint32_t max_groups, uint64_t *start, uint64_t *len)
{
    if (a == 0 || b == 0 || kp == 0 || V < 2ull * kp) return 0;
    uint64_t R = V, s = 0;
    uint32_t L = 0;
    for (;;) {
        if (L >= max_groups) return 0;
        uint64_t f = (uint64_t)(((unsigned __int128)a * R) / (a + b));
        uint64_t r = R - f;
        if (f <= kp || r <= kp) { /* final group: the whole remainder */
            start[L] = s;
            len[L] = R;
            L++;
            break;
        }
        start[L] = s;
        len[L] = f;
        L++;
        s += f;
        R = r;
    }
    return L;
}

/* O5  HOPH sketch: the group containing p, then the floor rule
 *     with k' bins inside that group.  Output set-major [n_sets][L*k'].      */
void orc_hoph_sketch(const uint64_t *offsets, const uint32_t *ids, uint64_t n_sets,
                     uint64_t V, uint32_t L, const uint64_t *gstart, const uint64_t *glen,
                     uint32_t kp, uint64_t seed, int identity, uint32_t *out)
{
    orc_perm P;
    perm_init(&P, V, seed, identity);
    uint64_t nb = (uint64_t)L * kp;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t s = 0; s < (int64_t)n_sets; s++) {
        uint32_t *F = out + (uint64_t)s * nb;
        for (uint64_t b = 0; b < nb; b++) F[b] = ORC_EMPTY;
        for (uint64_t e = offsets[s]; e < offsets[s + 1]; e++) {
            uint64_t p = orc_psi(&P, ids[e]);
            uint32_t g = 0;
            while (!(gstart[g] <= p && p < gstart[g] + glen[g])) g++;
            uint32_t b = range_bin_of(gstart[g], glen[g], kp, p);
            uint32_t off = (uint32_t)(p - range_bin_start(gstart[g], glen[g], kp, b));
            uint32_t *slot = &F[(uint64_t)g * kp + b];
            if (*slot == ORC_EMPTY || off < *slot) *slot = off;
        }
    }
}

/* ------------------------------------------------------------------------ */
/* O6  MinWise sketch: fp_i = min over e of pi_i(e).
 *     An empty set has no sketch: flag = 1 and values left EMPTY.           */
/* ------------------------------------------------------------------------ */
void orc_minwise_sketch(const uint64_t *offsets, const uint32_t *ids, uint64_t n_sets,
                        uint64_t V, uint32_t k, uint64_t seed, uint32_t *out, uint8_t *flags)
{
    orc_perm *Pi = (orc_perm *)malloc(sizeof(orc_perm) * (k ? k : 1));
    for (uint32_t i = 0; i < k; i++) perm_init(&Pi[i], V, minwise_seed(seed, i), 0);
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t s = 0; s < (int64_t)n_sets; s++) {
        uint32_t *F = out + (uint64_t)s * k;
        flags[s] = (offsets[s] == offsets[s + 1]) ? 1 : 0;
        for (uint32_t i = 0; i < k; i++) {
            uint64_t m = UINT64_MAX;
            for (uint64_t e = offsets[s]; e < offsets[s + 1]; e++) {
                uint64_t v = orc_psi(&Pi[i], ids[e]);
                if (v < m) m = v;
            }
            F[i] = (m == UINT64_MAX) ? ORC_EMPTY : (uint32_t)m;
        }
    }
    free(Pi);
}

/* ------------------------------------------------------------------------ */
/* O11 exact Jaccard (Eq. 5) by sorted merge; -1 if both empty.       */
/* ------------------------------------------------------------------------ */
double orc_jaccard(const uint32_t *a, uint64_t na, const uint32_t *b, uint64_t nb,
                   uint64_t *inter_out, uint64_t *union_out)
{
    uint64_t i = 0, j = 0, inter = 0;
    while (i < na && j < nb) {
        if (a[i] == b[j]) { inter++; i++; j++; }
        else if (a[i] < b[j]) i++;
        else j++;
    }
    uint64_t uni = na + nb - inter;
    if (inter_out) *inter_out = inter;
    if (union_out) *union_out = uni;
    return uni ? (double)inter / (double)uni : -1.0;
}

/* ------------------------------------------------------------------------ */
/* per-pair records                                                          */
/* ------------------------------------------------------------------------ */
typedef struct {
    uint32_t n_mb;    /* matched bins over the compared bins (Eq. 1, Eq. 3)    */
    uint32_t n_excl;  /* excluded bins over the compared bins (Eq. 2/4, mode)  */
    uint32_t groups;  /* groups compared                                       */
    uint32_t verdict; /* 1 = Similar, 0 = NotSimilar                           */
    uint32_t flags;   /* ORC_UNDEFINED | ORC_EARLY                             */
    uint32_t pad;
    double estimate;  /* the estimator's value; -1 when absent                 */
} orc_rec;

/* matched bin (Eq. 3 with the D1-twice typo read as "both non-empty", R5) */
static int bin_matched(uint32_t x, uint32_t y) { return x != ORC_EMPTY && y != ORC_EMPTY && x == y; }

/* excluded bin: JointEmpty = both empty (Eq. 4); EitherEmpty = either empty
 * (the convention the worked examples need; R6)              */
static int bin_excluded(uint32_t x, uint32_t y, int joint)
{
    return joint ? (x == ORC_EMPTY && y == ORC_EMPTY) : (x == ORC_EMPTY || y == ORC_EMPTY);
}

/* O7 the OPH estimator (Eq. 6) and the threshold verdict R >= T (R1) */
static void oph_verdict(uint32_t n_mb, uint32_t n_excl, uint32_t k, uint32_t t_num, uint32_t t_den, orc_rec *r)
{
    uint32_t den = k - n_excl;
    r->n_mb = n_mb;
    r->n_excl = n_excl;
    if (den == 0) { /* k - N_eb = 0: estimate undefined, never Similar (R7) */
        r->flags |= ORC_UNDEFINED;
        r->verdict = 0;
        r->estimate = -1.0;
        return;
    }
    /* N_mb / den >= t_num / t_den, exactly */
    r->verdict = ((uint64_t)n_mb * t_den >= (uint64_t)t_num * den) ? 1 : 0;
    r->estimate = (double)n_mb / (double)den;
}

/* full OPH comparison of two flat sketches (Eq. 1-6) */
static void pair_full(const uint32_t *q, const uint32_t *s, uint32_t k, uint32_t groups, int joint,
                      uint32_t t_num, uint32_t t_den, orc_rec *r)
{
    uint32_t n_mb = 0, n_excl = 0;
    for (uint32_t b = 0; b < k; b++) {
        n_mb += bin_matched(q[b], s[b]);
        n_excl += bin_excluded(q[b], s[b], joint);
    }
    memset(r, 0, sizeof(*r));
    r->groups = groups;
    oph_verdict(n_mb, n_excl, k, t_num, t_den, r);
}

/* ------------------------------------------------------------------------ */
/* O9  GOPH comparison: Algorithm 1 read per R10-R16.
 *     trace (optional, n entries of 2 x int64): M_ra as num/den per group.   */
/* ------------------------------------------------------------------------ */
static void pair_goph(const uint32_t *q, const uint32_t *s, uint32_t n, uint32_t kp, int joint,
                      uint32_t t_num, uint32_t t_den, const uint8_t *lower_le, const uint8_t *upper_le,
                      orc_rec *r, int64_t *trace)
{
    memset(r, 0, sizeof(*r));
    int64_t M_c = 0;       /* current matched bins (Alg. 1 line 1) */
    uint32_t excl_c = 0;   /* excluded bins so far (reported, not used by the filter) */
    for (uint32_t l = 1; l <= n; l++) {
        /* lines 3-8: count the bins of group l that have equal value (raw count, R14) */
        for (uint32_t b = (l - 1) * kp; b < l * kp; b++) {
            M_c += bin_matched(q[b], s[b]);
            excl_c += bin_excluded(q[b], s[b], joint);
        }
        r->groups = l;
        if (l == n) { /* no early break: full-comparison verdict over all n k' bins (R15) */
            oph_verdict((uint32_t)M_c, excl_c, n * kp, t_num, t_den, r);
            return;
        }
        /* line 11: M_ra = (n k' T - M_c) / (n - l), l = groups compared (R10), T = t_num/t_den */
        int64_t num = (int64_t)n * kp * t_num - M_c * (int64_t)t_den;
        int64_t den = (int64_t)t_den * (n - l);
        if (trace) { trace[2 * (l - 1)] = num; trace[2 * (l - 1) + 1] = den; }
        r->n_mb = (uint32_t)M_c;
        r->n_excl = excl_c;
        r->estimate = -1.0;
        r->flags = ORC_EARLY;
        if (num <= 0) { r->verdict = 1; return; }                 /* requirement met (R16) */
        if (num > (int64_t)kp * den) { r->verdict = 0; return; }  /* infeasible (R16) */
        /* M_a = k' T (line 1); compare M_ra < M_a exactly: num/den < k' t_num / t_den */
        if (num * (int64_t)t_den < (int64_t)kp * t_num * den) {
            int64_t m = num / den;                                 /* floor, num > 0 (R12) */
            if (lower_le[m]) { r->verdict = 1; return; }          /* F <= eps: Similar (R11, R13) */
        } else {
            int64_t m = (num + den - 1) / den;                     /* ceil (R12) */
            if (upper_le[m]) { r->verdict = 0; return; }          /* F <= eps: NotSimilar (R11) */
        }
        r->flags = 0;
    }
}

/* ------------------------------------------------------------------------ */
/* O9e empty-aware GOPH (readings E1-E4).
 *     Algorithm 1 with the binomial trials taken to be the non-excluded bins.
 *     D = k - N_excl over all n k' bins (the empty masks are known before any
 *     value is compared, E1); after l groups D_c = non-excluded bins compared,
 *     R = D - D_c the remaining trials, need = T D - M_c the matches still
 *     needed for the full-OPH verdict (Eq. 6).  Alg. 1's tests (lines 13-26,
 *     R11-R16) run unchanged on the requirement per group of k' trials,
 *     M_ra = k' need / R (E2); with no excluded bin D = n k', R = (n - l) k'
 *     and M_ra is Alg. 1's (n k' T - M_c) / (n - l) exactly.  R = 0 (every
 *     remaining bin excluded) completes the comparison: the full-OPH verdict
 *     and estimate, groups = l (E3).  The last group: the full-OPH verdict.  */
/* ------------------------------------------------------------------------ */
static void pair_goph_e(const uint32_t *q, const uint32_t *s, uint32_t n, uint32_t kp, int joint,
                        uint32_t t_num, uint32_t t_den, const uint8_t *lower_le, const uint8_t *upper_le,
                        orc_rec *r, int64_t *trace)
{
    memset(r, 0, sizeof(*r));
    const uint32_t k = n * kp;
    uint32_t excl_all = 0;
    for (uint32_t b = 0; b < k; b++) excl_all += bin_excluded(q[b], s[b], joint);
    const int64_t D = (int64_t)k - excl_all; /* E1: the pair's trials */
    int64_t M_c = 0;
    uint32_t excl_c = 0;
    for (uint32_t l = 1; l <= n; l++) {
        for (uint32_t b = (l - 1) * kp; b < l * kp; b++) {
            M_c += bin_matched(q[b], s[b]);
            excl_c += bin_excluded(q[b], s[b], joint);
        }
        r->groups = l;
        const int64_t D_c = (int64_t)l * kp - excl_c;
        const int64_t R = D - D_c;
        if (l == n || R == 0) { /* E3: nothing left to compare -- the full-OPH verdict (Eq. 6) */
            oph_verdict((uint32_t)M_c, excl_all, k, t_num, t_den, r);
            return;
        }
        /* E2: M_ra = k' (T D - M_c) / R = num / den with T = t_num / t_den */
        int64_t num = (int64_t)kp * ((int64_t)t_num * D - M_c * (int64_t)t_den);
        int64_t den = (int64_t)t_den * R;
        if (trace) { trace[2 * (l - 1)] = num; trace[2 * (l - 1) + 1] = den; }
        r->n_mb = (uint32_t)M_c;
        r->n_excl = excl_c;
        r->estimate = -1.0;
        r->flags = ORC_EARLY;
        /* Alg. 1 lines 13-26 on M_ra, exactly as pair_goph */
        if (num <= 0) { r->verdict = 1; return; }
        if (num > (int64_t)kp * den) { r->verdict = 0; return; }
        if (num * (int64_t)t_den < (int64_t)kp * t_num * den) {
            int64_t m = num / den;
            if (lower_le[m]) { r->verdict = 1; return; }
        } else {
            int64_t m = (num + den - 1) / den;
            if (upper_le[m]) { r->verdict = 0; return; }
        }
        r->flags = 0;
    }
}

/* ------------------------------------------------------------------------ */
/* O10 HOPH comparison: Algorithm 2 with the mass balance of
 *     nominal group weights (R19, R21).  Weights w_j = r(1-r)^(j-1) for j<L,
 *     w_L = (1-r)^(L-1), r = a/(a+b) (Lemma 3 with l = L), held as
 *     integers c_j = w_j * D over D = (a+b)^(L-1).                           */
/* ------------------------------------------------------------------------ */
typedef __int128 i128;

static i128 i128_gcd(i128 x, i128 y)
{
    if (x < 0) x = -x;
    if (y < 0) y = -y;
    while (y) { i128 t = x % y; x = y; y = t; }
    return x;
}

/* c_j (1-indexed j) */
static void hoph_weights(uint32_t a, uint32_t b, uint32_t L, i128 *c, i128 *D)
{
    i128 ab = (i128)a + b, d = 1;
    for (uint32_t j = 1; j < L; j++) d *= ab;
    *D = d;
    for (uint32_t j = 1; j <= L; j++) {
        i128 w = 1;
        if (j < L) {
            w = a;
            for (uint32_t t = 1; t < j; t++) w *= b;
            for (uint32_t t = j; t < L - 1; t++) w *= ab; /* (a+b)^(L-1-j) */
        } else {
            for (uint32_t t = 1; t < L; t++) w *= b;
        }
        c[j - 1] = w;
    }
}

void orc_hoph_weights(uint32_t a, uint32_t b, uint32_t L, int64_t *c_out, int64_t *D_out)
{
    i128 c[64], D;
    hoph_weights(a, b, L, c, &D);
    for (uint32_t j = 0; j < L; j++) c_out[j] = (int64_t)c[j];
    *D_out = (int64_t)D;
}

/* the HOPH estimator (Lemma 3, R21): per-group OPH estimates
 * M_j / (k' - excl_j) combined with the nominal weights c_j / D; groups with
 * every bin excluded are dropped and the weights renormalised (R22).
 * Verdict: estimate >= T, exactly.                                         */
static void hoph_final(const uint32_t *M, const uint32_t *ex, uint32_t L, uint32_t kp, const i128 *c,
                       uint32_t t_num, uint32_t t_den, orc_rec *r)
{
    i128 num = 0, den = 1, csum = 0; /* sum_j c_j M_j / d_j  =  num / den */
    for (uint32_t j = 0; j < L; j++) {
        uint32_t d = kp - ex[j];
        if (d == 0) continue;
        num = num * d + c[j] * M[j] * den;
        den = den * d;
        i128 g = i128_gcd(num, den);
        if (g > 1) { num /= g; den /= g; }
        csum += c[j];
    }
    r->flags = 0;
    if (csum == 0) {
        r->flags = ORC_UNDEFINED;
        r->verdict = 0;
        r->estimate = -1.0;
        return;
    }
    /* estimate = num / (den csum) >= t_num / t_den */
    r->verdict = (num * t_den >= (i128)t_num * den * csum) ? 1 : 0;
    r->estimate = (double)((long double)num / ((long double)den * (long double)csum));
}

/* exported: the HOPH estimator of one pair of HOPH sketches, no filtering */
void orc_hoph_estimate(const uint32_t *q, const uint32_t *s, uint32_t L, uint32_t kp, uint32_t a, uint32_t b,
                       int joint, uint32_t t_num, uint32_t t_den, orc_rec *r)
{
    i128 c[64], D;
    uint32_t M[64], ex[64];
    hoph_weights(a, b, L, c, &D);
    memset(r, 0, sizeof(*r));
    for (uint32_t j = 0; j < L; j++) {
        M[j] = ex[j] = 0;
        for (uint32_t t = j * kp; t < (j + 1) * kp; t++) {
            M[j] += bin_matched(q[t], s[t]);
            ex[j] += bin_excluded(q[t], s[t], joint);
            r->n_mb += bin_matched(q[t], s[t]);
            r->n_excl += bin_excluded(q[t], s[t], joint);
        }
    }
    r->groups = L;
    hoph_final(M, ex, L, kp, c, t_num, t_den, r);
}

static void pair_hoph(const uint32_t *q, const uint32_t *s, uint32_t L, uint32_t kp, uint32_t a, uint32_t b,
                      int joint, uint32_t t_num, uint32_t t_den, const uint8_t *lower_le,
                      const uint8_t *upper_le, orc_rec *r, int64_t *trace)
{
    i128 c[64], D;
    hoph_weights(a, b, L, c, &D);
    memset(r, 0, sizeof(*r));
    uint32_t M[64], ex[64];
    i128 S = 0;          /* sum_{j<=l} c_j M_j  (achieved mass x D k') */
    i128 W = D;          /* sum_{j>l} c_j       (remaining weight x D) */
    uint32_t nmb = 0, nex = 0;
    for (uint32_t l = 1; l <= L; l++) {
        /* lines 3-8: M_l = matched bins of group l (reset per group, R20) */
        M[l - 1] = 0;
        ex[l - 1] = 0;
        for (uint32_t t = (l - 1) * kp; t < l * kp; t++) {
            M[l - 1] += bin_matched(q[t], s[t]);
            ex[l - 1] += bin_excluded(q[t], s[t], joint);
        }
        nmb += M[l - 1];
        nex += ex[l - 1];
        S += c[l - 1] * M[l - 1];
        W -= c[l - 1];
        r->groups = l;
        r->n_mb = nmb;
        r->n_excl = nex;
        if (l == L) { /* all groups compared: the HOPH estimator verdict */
            hoph_final(M, ex, L, kp, c, t_num, t_den, r);
            return;
        }
        /* line 10: P_r = (T - sum_{j<=l} w_j M_j / k') / sum_{j>l} w_j, and the test
         * uses F(P_r k'); x = P_r k' = (t_num D k' - t_den S) / (t_den W)  (R19, R23) */
        i128 num = (i128)t_num * D * kp - (i128)t_den * S;
        i128 den = (i128)t_den * W;
        if (trace) { trace[2 * (l - 1)] = (int64_t)num; trace[2 * (l - 1) + 1] = (int64_t)den; }
        r->estimate = -1.0;
        r->flags = ORC_EARLY;
        if (num <= 0) { r->verdict = 1; return; }                 /* P_r <= 0 */
        if (num > (i128)kp * den) { r->verdict = 0; return; }     /* P_r > 1  */
        /* P_r < P_a = T  <=>  x < k' T */
        if (num * t_den < (i128)kp * t_num * den) {
            int64_t m = (int64_t)(num / den);
            if (lower_le[m]) { r->verdict = 1; return; }          /* line 12-15 */
        } else {
            int64_t m = (int64_t)((num + den - 1) / den);
            if (upper_le[m]) { r->verdict = 0; return; }          /* line 20-24 */
        }
        r->flags = 0;
    }
}

/* ------------------------------------------------------------------------ */
/* O10e empty-aware HOPH (readings EH1-EH5).
 *     Algorithm 2's mass balance (R19) with each group's trials taken to be
 *     its non-excluded bins d_j = k' - excl_j (known from the empty masks
 *     before any value is compared, EH1).  The groups with d_j > 0 form K; the
 *     final verdict is the HOPH estimator sum_K c_j m_j/d_j / C_K >= T
 *     (R21, R22; C_K = sum_K c_j).  After l groups the achieved mass is
 *     A_l = sum_{j<=l, j in K} c_j m_j / d_j and the usable weight still to
 *     compare is W_l = sum_{j>l, j in K} c_j, so the remaining groups must
 *     reach P_r = (T C_K - A_l) / W_l, and Alg. 2's four tests run unchanged
 *     on x = P_r k' (EH2, EH3).  With no excluded bin d_j = k', C_K = D,
 *     A_l = S_l / k' and x is Alg. 2's (T D k' - S_l) / W_l exactly.  W_l = 0
 *     before group L (every remaining group excluded) completes the comparison:
 *     the final record, groups = l (EH4).  Exact: x = num / den with both
 *     scaled by t_den lcm{d_j : j <= l, j in K}.                             */
/* ------------------------------------------------------------------------ */
static i128 i128_lcm(i128 a, i128 b) { return a / i128_gcd(a, b) * b; }

static void pair_hoph_e(const uint32_t *q, const uint32_t *s, uint32_t L, uint32_t kp, uint32_t a, uint32_t b,
                        int joint, uint32_t t_num, uint32_t t_den, const uint8_t *lower_le,
                        const uint8_t *upper_le, orc_rec *r, int64_t *trace)
{
    i128 c[64], D;
    hoph_weights(a, b, L, c, &D);
    memset(r, 0, sizeof(*r));
    uint32_t M[64], ex[64];
    i128 C_K = 0;                         /* EH1: usable weight of the pair */
    for (uint32_t j = 0; j < L; j++) {
        M[j] = ex[j] = 0;
        for (uint32_t t = j * kp; t < (j + 1) * kp; t++) {
            M[j] += bin_matched(q[t], s[t]);
            ex[j] += bin_excluded(q[t], s[t], joint);
        }
        if (ex[j] < kp) C_K += c[j];
    }
    i128 W = C_K;                         /* usable weight not yet compared */
    i128 lam = 1;                         /* lcm of the compared usable d_j */
    uint32_t nmb = 0, nex = 0;
    for (uint32_t l = 1; l <= L; l++) {
        const uint32_t d = kp - ex[l - 1];
        nmb += M[l - 1];
        nex += ex[l - 1];
        if (d > 0) {
            W -= c[l - 1];
            lam = i128_lcm(lam, (i128)d);
        }
        r->groups = l;
        r->n_mb = nmb;
        r->n_excl = nex;
        if (l == L || W == 0) { /* EH4 / EH5: the HOPH estimator over all groups */
            uint32_t nmb_all = 0, nex_all = 0;
            for (uint32_t j = 0; j < L; j++) { nmb_all += M[j]; nex_all += ex[j]; }
            r->n_mb = nmb_all;
            r->n_excl = nex_all;
            hoph_final(M, ex, L, kp, c, t_num, t_den, r);
            return;
        }
        /* A_l lam = sum_{j<=l, d_j>0} c_j m_j (lam / d_j) */
        i128 A = 0;
        for (uint32_t j = 0; j < l; j++)
            if (ex[j] < kp) A += c[j] * M[j] * (lam / (kp - ex[j]));
        i128 num = (i128)kp * ((i128)t_num * C_K * lam - (i128)t_den * A);
        i128 den = (i128)t_den * lam * W;
        if (trace) { trace[2 * (l - 1)] = (int64_t)num; trace[2 * (l - 1) + 1] = (int64_t)den; }
        r->estimate = -1.0;
        r->flags = ORC_EARLY;
        if (num <= 0) { r->verdict = 1; return; }
        if (num > (i128)kp * den) { r->verdict = 0; return; }
        if (num * t_den < (i128)kp * t_num * den) {
            int64_t m = (int64_t)(num / den);
            if (lower_le[m]) { r->verdict = 1; return; }
        } else {
            int64_t m = (int64_t)((num + den - 1) / den);
            if (upper_le[m]) { r->verdict = 0; return; }
        }
        r->flags = 0;
    }
}

/* ------------------------------------------------------------------------ */
/* MinWise comparison: fraction of equal fingerprints.          */
/* ------------------------------------------------------------------------ */
static void pair_minwise(const uint32_t *q, const uint32_t *s, uint8_t qf, uint8_t sf, uint32_t k,
                         uint32_t t_num, uint32_t t_den, orc_rec *r)
{
    memset(r, 0, sizeof(*r));
    if (qf || sf) { /* the sketch of an empty set is undefined */
        r->flags = ORC_UNDEFINED;
        r->verdict = 0;
        r->estimate = -1.0;
        return;
    }
    uint32_t eq = 0;
    for (uint32_t i = 0; i < k; i++) eq += (q[i] == s[i]);
    r->n_mb = eq;
    r->verdict = ((uint64_t)eq * t_den >= (uint64_t)t_num * k) ? 1 : 0;
    r->estimate = (double)eq / (double)k;
}

/* ------------------------------------------------------------------------ */
/* batch drivers: every (query, set) pair; out is [n_q][n_s] records.        */
/* ------------------------------------------------------------------------ */
void orc_compare_full(const uint32_t *Q, uint64_t n_q, const uint32_t *S, uint64_t n_s, uint32_t k,
                      uint32_t groups, int joint, uint32_t t_num, uint32_t t_den, orc_rec *out)
{
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t qi = 0; qi < (int64_t)n_q; qi++)
        for (uint64_t si = 0; si < n_s; si++)
            pair_full(Q + (uint64_t)qi * k, S + si * k, k, groups, joint, t_num, t_den,
                      &out[(uint64_t)qi * n_s + si]);
}

void orc_compare_goph(const uint32_t *Q, uint64_t n_q, const uint32_t *S, uint64_t n_s, uint32_t n,
                      uint32_t kp, int joint, uint32_t t_num, uint32_t t_den, const uint8_t *lower_le,
                      const uint8_t *upper_le, orc_rec *out, int64_t *trace, int empty_aware)
{
    uint64_t k = (uint64_t)n * kp;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t qi = 0; qi < (int64_t)n_q; qi++)
        for (uint64_t si = 0; si < n_s; si++) {
            uint64_t pi = (uint64_t)qi * n_s + si;
            (empty_aware ? pair_goph_e : pair_goph)(Q + (uint64_t)qi * k, S + si * k, n, kp, joint, t_num, t_den,
                                                    lower_le, upper_le, &out[pi], trace ? trace + 2 * n * pi : NULL);
        }
}

void orc_compare_hoph(const uint32_t *Q, uint64_t n_q, const uint32_t *S, uint64_t n_s, uint32_t L,
                      uint32_t kp, uint32_t a, uint32_t b, int joint, uint32_t t_num, uint32_t t_den,
                      const uint8_t *lower_le, const uint8_t *upper_le, orc_rec *out, int64_t *trace,
                      int empty_aware)
{
    uint64_t k = (uint64_t)L * kp;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t qi = 0; qi < (int64_t)n_q; qi++)
        for (uint64_t si = 0; si < n_s; si++) {
            uint64_t pi = (uint64_t)qi * n_s + si;
            (empty_aware ? pair_hoph_e : pair_hoph)(Q + (uint64_t)qi * k, S + si * k, L, kp, a, b, joint, t_num,
                                                    t_den, lower_le, upper_le, &out[pi],
                                                    trace ? trace + 2 * L * pi : NULL);
        }
}

void orc_compare_minwise(const uint32_t *Q, const uint8_t *qf, uint64_t n_q, const uint32_t *S,
                         const uint8_t *sf, uint64_t n_s, uint32_t k, uint32_t t_num, uint32_t t_den,
                         orc_rec *out)
{
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t qi = 0; qi < (int64_t)n_q; qi++)
        for (uint64_t si = 0; si < n_s; si++)
            pair_minwise(Q + (uint64_t)qi * k, S + si * k, qf[qi], sf[si], k, t_num, t_den,
                         &out[(uint64_t)qi * n_s + si]);
}

int orc_num_threads(void)
{
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}
