// Host side of libophgpu: the C-ABI entry points of include/ophgpu.h, argument
// validation, the HOPH layout, psi keys, and the planner that compiles the
// paper's GOPH / HOPH early-termination rules into exact per-level integer
// thresholds.  No device arithmetic here.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <random>
#include <tuple>
#include <vector>

#include "internal.h"

using namespace ophgpu;
typedef __int128 i128;
typedef unsigned __int128 u128;

namespace {

// ---------------------------------------------------------------- small helpers
uint64_t splitmix64_next(uint64_t &state) {
    uint64_t z = (state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint32_t word_bits(uint64_t V) {  // max(1, ceil(log2 V))
    uint32_t w = 0;
    while (w < 64 && (1ull << w) < V) w++;
    return w == 0 ? 1 : w;
}

// psi keys: splitmix64 stream from seed, kappa_r then mu_r
PsiParams make_psi(uint64_t V, uint64_t seed, uint32_t kind) {
    PsiParams P{};
    const uint32_t w = word_bits(V);
    const uint64_t mask = (w >= 64) ? ~0ull : ((1ull << w) - 1);
    P.V = V;
    P.mask = (uint32_t)mask;
    P.shift = (w + 1) / 2;
    P.hmul = w >= 32 ? 1u : (1u << (32 - w));
    P.hsh = (w >= 32 ? 0u : 32u - w) + P.shift;
    uint64_t st = seed;
    for (int r = 0; r < 4; r++) {
        P.kappa[r] = (uint32_t)(splitmix64_next(st) & mask);
        P.mu[r] = (uint32_t)((splitmix64_next(st) & mask) | 1ull);
    }
    P.identity = kind == OPH_PERM_IDENTITY;
    P.pow2 = (V == (1ull << w));
    return P;
}

RangeBins make_range(uint64_t start, uint64_t len, uint32_t nb) {
    RangeBins R{};
    R.start = start;
    R.len = len;
    if (len % nb == 0) {
        const uint64_t bl = len / nb;
        if ((bl & (bl - 1)) == 0) {
            R.pow2 = 1;
            uint32_t sh = 0;
            while ((1ull << sh) < bl) sh++;
            R.shift = sh;
        }
    }
    return R;
}

uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }
size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

oph_status cuda_status(cudaError_t e) { return e == cudaSuccess ? OPH_OK : OPH_ECUDA; }

// ---------------------------------------------------------------- binomial tails (Eq. 9-10)
// X ~ Bin(K, T) (R8).  lower(m) = P(X <= m), upper(m) = P(X >= m) (R9) in long
// double from log-space terms; "tail <= eps" is certified only when the tail is
// farther than 1e-9 relative from eps (the computed tails are accurate to
// ~1e-15 relative), else OPH_EAMBIGUOUS.
oph_status small_prob_tables(uint32_t K, uint32_t t_num, uint32_t t_den, double eps, std::vector<uint8_t> &lower_le,
                             std::vector<uint8_t> &upper_le) {
    std::vector<long double> pmf(K + 1, 0.0L);
    if (t_num == t_den) {
        pmf[K] = 1.0L;
    } else {
        const long double T = (long double)t_num / (long double)t_den;
        const long double lT = logl(T), l1T = log1pl(-T);
        for (uint32_t j = 0; j <= K; j++)
            pmf[j] = expl(lgammal(K + 1.0L) - lgammal(j + 1.0L) - lgammal(K - j + 1.0L) + j * lT + (K - j) * l1T);
    }
    const long double e = eps;
    auto decide = [&](long double tail, uint8_t &out) -> bool {
        if (fabsl(tail - e) <= 1e-9L * e) return false;
        out = tail <= e;
        return true;
    };
    lower_le.assign(K + 1, 0);
    upper_le.assign(K + 2, 0);
    long double acc = 0.0L;
    for (uint32_t m = 0; m <= K; m++) {
        acc += pmf[m];
        if (!decide(acc, lower_le[m])) return OPH_EAMBIGUOUS;
    }
    acc = 0.0L;
    for (int64_t m = K + 1; m >= 0; m--) {
        if (m <= (int64_t)K) acc += pmf[m];
        if (!decide(acc, upper_le[m])) return OPH_EAMBIGUOUS;
    }
    return OPH_OK;
}

// ---------------------------------------------------------------- the filter rule
enum Decision { kContinue = 0, kSimilar = 1, kNotSimilar = 2 };

// One small-probability decision on x = num / den (den > 0), x = M_ra (GOPH,
// Alg. 1 line 11) or x = P_r k' (HOPH, Alg. 2 line 10):
//   x <= 0 -> Similar; x > k' -> NotSimilar (R16);
//   x <  k'T and P(X <= floor x) <= eps -> Similar    (Alg. 1 lines 13-19, R11, R12)
//   x >= k'T and P(X >= ceil x)  <= eps -> NotSimilar (Alg. 1 lines 20-26)
struct Rule {
    uint32_t kp, t_num, t_den;
    const std::vector<uint8_t> *lower_le, *upper_le;
    Decision operator()(i128 num, i128 den) const {
        if (num <= 0) return kSimilar;
        if (num > (i128)kp * den) return kNotSimilar;
        if (num * (i128)t_den < (i128)kp * t_num * den) {
            const i128 m = num / den;
            return (*lower_le)[(size_t)m] ? kSimilar : kContinue;
        }
        const i128 m = (num + den - 1) / den;
        return (*upper_le)[(size_t)m] ? kNotSimilar : kContinue;
    }
};

// Per-level thresholds on the pair state (GOPH: M_c <= n k'; HOPH: S_l = sum c_j M_j,
// up to D k' ~ 2^75 for the 1:2 split of 2^32): Similar iff state >= acc, NotSimilar
// iff state <= rej.
constexpr u128 kNeverAcc = ~(u128)0;
struct LevelThr {
    u128 acc;  // kNeverAcc: never
    i128 rej;  // -1: never
};

// Compile one level: decide(state) is, by construction, Similar on an upward
// closed set of states and NotSimilar on a downward closed one (x is
// decreasing in the state, the lower tail increasing and the upper tail
// decreasing in x).  Binary search both boundaries, then verify.
template <class F>
bool compile_level(F decide, u128 smax, bool exhaustive, LevelThr &out) {
    out.acc = kNeverAcc;
    out.rej = -1;
    if (decide(smax) == kSimilar) {
        u128 lo = 0, hi = smax;
        while (lo < hi) {
            const u128 mid = lo + (hi - lo) / 2;
            if (decide(mid) == kSimilar) hi = mid; else lo = mid + 1;
        }
        out.acc = lo;
    }
    if (decide(0) == kNotSimilar) {
        u128 lo = 0, hi = smax;
        while (lo < hi) {
            const u128 mid = lo + (hi - lo + 1) / 2;
            if (decide(mid) == kNotSimilar) lo = mid; else hi = mid - 1;
        }
        out.rej = (i128)lo;
    }
    auto check = [&](u128 s) {
        const Decision want = decide(s);
        const Decision got = s >= out.acc ? kSimilar : ((i128)s <= out.rej ? kNotSimilar : kContinue);
        return want == got;
    };
    if (exhaustive) {
        for (u128 s = 0; s <= smax; s++)
            if (!check(s)) return false;
        return true;
    }
    std::mt19937_64 rng(12345);
    for (u128 s = 0; s <= std::min<u128>(smax, 2048); s++)
        if (!check(s)) return false;
    for (int d = -3; d <= 3; d++) {
        if (out.acc != kNeverAcc && (i128)out.acc + d >= 0 && (u128)((i128)out.acc + d) <= smax &&
            !check((u128)((i128)out.acc + d)))
            return false;
        if (out.rej >= 0 && out.rej + d >= 0 && (u128)(out.rej + d) <= smax && !check((u128)(out.rej + d))) return false;
    }
    for (int i = 0; i < 4096; i++) {
        const u128 r = ((u128)rng() << 64) | rng();
        if (!check(r % (smax + 1))) return false;
    }
    return check(smax);
}

struct Plan {
    oph_status st = OPH_OK;
    uint32_t nlev = 0;          // n or L
    uint32_t l0 = 0;            // level the scan ends at
    std::vector<LevelThr> thr;  // thr[l-1] for l = 1..nlev-1
    std::vector<u128> c;        // weights (GOPH: 1)
    u128 lam = 1;               // lcm(1..kp)
};

std::mutex g_plan_mu;
std::map<std::tuple<uint32_t, uint32_t, uint32_t, uint32_t, uint32_t, uint32_t, uint32_t, double>, Plan> g_plans;

u128 lcm_upto(uint32_t kp, bool &overflow) {
    u128 l = 1;
    overflow = false;
    for (uint32_t d = 2; d <= kp; d++) {
        u128 a = l, b = d;
        while (b) { u128 t = a % b; a = b; b = t; }
        const u128 mul = d / (uint32_t)a;
        if (l > (((u128)1) << 120) / mul) { overflow = true; return 0; }
        l *= mul;
    }
    return l;
}

// GOPH (method 1: nlev = n) or HOPH (method 2: nlev = L, ratio a:b)
Plan make_plan(uint32_t method, uint32_t nlev, uint32_t kp, uint32_t a, uint32_t b, uint32_t t_num, uint32_t t_den,
               double eps) {
    const auto key = std::make_tuple(method, nlev, kp, a, b, t_num, t_den, eps);
    {
        std::lock_guard<std::mutex> g(g_plan_mu);
        auto it = g_plans.find(key);
        if (it != g_plans.end()) return it->second;
    }
    Plan P;
    P.nlev = nlev;
    std::vector<uint8_t> lo, up;
    P.st = small_prob_tables(kp, t_num, t_den, eps, lo, up);
    if (P.st != OPH_OK) return P;
    const Rule rule{kp, t_num, t_den, &lo, &up};
    P.c.assign(nlev, 1);
    i128 D = 1;
    if (method == OPH_METHOD_HOPH) {
        // nominal weights w_j = r(1-r)^(j-1), w_L = (1-r)^(L-1), r = a/(a+b) (R21),
        // as integers c_j = w_j D over D = (a+b)^(L-1)
        const i128 ab = (i128)a + b;
        for (uint32_t j = 1; j < nlev; j++) {
            D *= ab;
            if (D > ((i128)1 << 100)) { P.st = OPH_EINVAL; return P; }
        }
        for (uint32_t j = 1; j <= nlev; j++) {
            i128 w = 1;
            if (j < nlev) {
                w = a;
                for (uint32_t t = 1; t < j; t++) w *= b;
                for (uint32_t t = j; t + 1 < nlev; t++) w *= ab;
            } else {
                for (uint32_t t = 1; t < nlev; t++) w *= b;
            }
            P.c[j - 1] = (u128)w;
        }
        // the rule's products (num * t_den, k' * t_num * den) stay below t_num t_den D k'
        if ((i128)t_num * t_den * D * kp >= ((i128)1 << 120)) { P.st = OPH_EINVAL; return P; }
        // the final verdict compares sums over the common denominator lcm(1..k');
        // lam = 0 marks "too large for exact 128-bit arithmetic" (compare_hoph refuses)
        bool of = false;
        P.lam = lcm_upto(kp, of);
        if (of || (u128)t_den * P.lam * (u128)D >= (((u128)1) << 126)) P.lam = 0;
    }
    P.thr.assign(nlev > 0 ? nlev - 1 : 0, LevelThr{kNeverAcc, -1});
    P.l0 = nlev;
    i128 csum = 0;
    for (uint32_t l = 1; l < nlev; l++) {
        csum += (i128)P.c[l - 1];
        const u128 smax = (u128)(csum * kp);
        LevelThr T;
        bool ok;
        if (method == OPH_METHOD_GOPH) {
            // M_ra = (n k' T - M_c) / (n - l) with T = t_num / t_den   (Alg. 1 line 11, R10)
            auto dec = [&](u128 Mc) {
                return rule((i128)nlev * kp * t_num - (i128)Mc * t_den, (i128)t_den * (nlev - l));
            };
            ok = compile_level(dec, smax, true, T);
        } else {
            // x = P_r k' = (T D k' - S_l) / W_l, W_l = D - sum_{j<=l} c_j   (Alg. 2 line 10, R19)
            const i128 W = D - csum;
            auto dec = [&](u128 S) { return rule((i128)t_num * D * kp - (i128)t_den * (i128)S, (i128)t_den * W); };
            ok = compile_level(dec, smax, smax <= (1u << 20), T);
        }
        if (!ok) { P.st = OPH_EINVAL; return P; }
        P.thr[l - 1] = T;
        if (P.l0 == nlev && (T.acc <= smax || T.rej >= 0)) P.l0 = l;
    }
    if (method == OPH_METHOD_HOPH && nlev > 1) P.l0 = 1;  // HOPH: the scan always covers group 1
    std::lock_guard<std::mutex> g(g_plan_mu);
    g_plans[key] = P;
    return P;
}

// AUTO's per-collection decision cache (see probe_pass_run)
struct AutoKey {
    uintptr_t F;
    uint64_t n_sets;
    uint32_t nb, method;
    bool operator<(const AutoKey &o) const {
        return std::tie(F, n_sets, nb, method) < std::tie(o.F, o.n_sets, o.nb, o.method);
    }
};
std::mutex g_auto_mu;
std::map<AutoKey, int> g_auto;

// ---------------------------------------------------------------- validation
oph_status check_sets(const oph_sets *s) {
    if (!s || (s->n_sets && (!s->d_offsets || !s->d_ids)) || s->n_sets >= (1ull << 32)) return OPH_EINVAL;
    return OPH_OK;
}

oph_status check_view(const oph_sketches *v, bool need_empty, bool need_flags) {
    if (!v || !v->d_values || v->ld < v->n_sets || v->ld % 4 || v->n_bins == 0) return OPH_EINVAL;
    if (v->n_sets >= 0xFFFFFFFEull) return OPH_EINVAL;
    if (need_empty && !v->d_empty) return OPH_EINVAL;
    if (need_flags && !v->d_flags) return OPH_EINVAL;
    return OPH_OK;
}

oph_status check_params(const oph_params *p) {
    if (!p || p->t_den == 0 || p->t_num == 0 || p->t_num > p->t_den || !(p->epsilon > 0.0) || !(p->epsilon < 1.0) ||
        p->empty_mode > 1)
        return OPH_EINVAL;
    return OPH_OK;
}

// max bin length of a range must leave two spare uint32 values for the sentinels
bool bins_fit(uint64_t len, uint32_t nb) { return ceil_div(len, nb) <= 0xFFFFFFFEull; }

// ---------------------------------------------------------------- compare workspace
struct Ws {
    uint32_t *QT, *QE, *QM, *QEM;
    uint8_t *qflags;
    unsigned long long *counters;  // [kMaxGroups + 2] level counters, then the PROBE overflow counter
    unsigned long long *table;     // PROBE exact tables [nb][S]
    uint32_t *bloom;               // PROBE filters [ceil(nb/32)][W][32]
    uint32_t *ovf_list;            // PROBE overflow sets [n_sets]
    SurvList list[2];
    uint64_t ldq, cap;
};

constexpr uint32_t kCounters = kMaxGroups + 4 + OPH_STOP_HIST_LEN;  // level counters, PROBE counters, saved histogram
constexpr uint32_t kLevelsPerLaunch = 4;  // GOPH/HOPH levels per survivor-kernel launch

// PROBE exact-table slots per bin for a pass of nq queries: load factor <= 1/4
uint32_t probe_log2S(uint64_t nq) {
    uint32_t l = 4;
    while ((1ull << l) < 4 * nq) l++;
    return l;
}

// Bloom words per bin for a pass of nq queries: >= 16 bits per query, 512 .. 2048
// words (the join kernel is compiled for these three widths)
uint32_t probe_log2W(uint64_t nq) {
    uint32_t l = 9;
    while (l < kJoinMaxLog2W && (1ull << l) * 32 < 16 * nq) l++;
    return l;
}

// queries per PROBE pass: all of them up to kJoinMaxQ, else balanced passes
uint64_t probe_pass(uint64_t ldq) {
    const uint64_t passes = ceil_div(ldq, kJoinMaxQ);
    return ceil_div(ceil_div(ldq, passes), 32) * 32;
}

size_t ws_fixed_bytes(uint64_t n_q, uint64_t n_sets, uint32_t nb) {
    const uint64_t ldq = ceil_div(n_q ? n_q : 1, 32) * 32;
    const uint64_t nw = ceil_div(nb, 32);
    const uint64_t pq = probe_pass(ldq);
    return align256(nb * ldq * 4) + align256(nw * ldq * 4) + align256(n_q * (uint64_t)nb * 4) +
           align256(n_q * nw * 4) + align256(ldq) + align256(kCounters * 8) +
           align256((uint64_t)nb * (1ull << probe_log2S(pq)) * 8) +
           align256(ceil_div(nb, 32) * (1ull << probe_log2W(pq)) * 32 * 4) + align256(n_sets * 4);
}

constexpr uint64_t kSurvBytes = 2 * (4 + 4 + 16 + 4);  // two lists, per entry

Ws carve_ws(void *base, uint64_t n_q, uint64_t n_sets, uint32_t nb, uint64_t cap) {
    Ws w{};
    char *p = (char *)base;
    w.ldq = ceil_div(n_q ? n_q : 1, 32) * 32;
    const uint64_t nw = ceil_div(nb, 32);
    w.QT = (uint32_t *)p; p += align256(nb * w.ldq * 4);
    w.QE = (uint32_t *)p; p += align256(nw * w.ldq * 4);
    w.QM = (uint32_t *)p; p += align256(n_q * (uint64_t)nb * 4);
    w.QEM = (uint32_t *)p; p += align256(n_q * nw * 4);
    w.qflags = (uint8_t *)p; p += align256(w.ldq);
    w.counters = (unsigned long long *)p; p += align256(kCounters * 8);
    const uint64_t pq = probe_pass(w.ldq);
    w.table = (unsigned long long *)p; p += align256((uint64_t)nb * (1ull << probe_log2S(pq)) * 8);
    w.bloom = (uint32_t *)p; p += align256(ceil_div(nb, 32) * (1ull << probe_log2W(pq)) * 32 * 4);
    w.ovf_list = (uint32_t *)p; p += align256(n_sets * 4);
    w.cap = cap;
    for (int i = 0; i < 2; i++) {
        w.list[i].q = (uint32_t *)p; p += align256(cap * 4);
        w.list[i].s = (uint32_t *)p; p += align256(cap * 4);
        w.list[i].state = (u128_t *)p; p += align256(cap * 16);
        w.list[i].nmb = (uint32_t *)p; p += align256(cap * 4);
    }
    return w;
}

size_t surv_region_bytes(uint64_t cap) { return 2 * (align256(cap * 4) * 3 + align256(cap * 16)); }

// BITMAP strategy (bitjoin.cuh): domain and workspace region (after the fixed part)
constexpr uint64_t kBitMaxV = 1ull << 23;
constexpr uint32_t kBitMaxNb = 1023;
bool bitmap_sizes_ok(uint64_t V, uint32_t nb) { return V <= kBitMaxV && nb <= kBitMaxNb; }
// (rows of up to 2,048 query bits: blocks of 2,048 queries for full OPH / GOPH)
size_t bitmap_region_bytes(uint64_t V, uint32_t nb) {
    return align256(V * 4) + align256((1 + (uint64_t)nb * 2048) * 256) + align256(4) + align256(64 * 4) +
           align256(33 * 64 * 4);
}

// largest survivor capacity that fits in ws_bytes
uint64_t cap_from_ws(size_t ws_bytes, size_t fixed) {
    if (ws_bytes <= fixed) return 0;
    uint64_t lo = 0, hi = (ws_bytes - fixed) / kSurvBytes + 1;
    while (lo + 1 < hi) {  // invariant: lo fits, hi does not
        const uint64_t mid = lo + (hi - lo) / 2;
        if (fixed + surv_region_bytes(mid) <= ws_bytes) lo = mid; else hi = mid;
    }
    return lo;
}

// ---------------------------------------------------------------- the BITMAP driver
// Query prep, then per block of 2,048 (or 1,024) queries: the value -> row table (bit_claim /
// bit_fill) and one scan of the collection deciding every level (bit_scan_q_kernel /
// bit_scan_kernel; HOPH: bit_scan_x_kernel).  No host synchronisation, no survivor lists.
oph_status run_bitmap(uint32_t method, const oph_sketches *Qv, const oph_sketches *Sv, uint32_t set_id_base,
                      uint32_t nb, uint32_t nw, uint32_t nlev, uint32_t kp, const Plan &plan, const oph_params *p,
                      oph_results *res, void *d_ws, size_t fixed, cudaStream_t stream) {
    const uint64_t n_q = Qv->n_sets, n_s = Sv->n_sets, V = Qv->vocab_size;
    Ws w = carve_ws(d_ws, n_q, n_s, nb, 0);
    char *bp = (char *)d_ws + fixed;
    BitArgs ba{};
    ba.idx = (uint32_t *)bp; bp += align256(V * 4);
    ba.rows = (uint32_t *)bp; bp += align256((1 + (uint64_t)nb * 2048) * 256);
    ba.nrows = (uint32_t *)bp; bp += align256(4);
    ba.max_eq = (uint32_t *)bp; bp += align256(64 * 4);
    ba.max_eq_pref = (uint32_t *)bp;  // [nw + 1][64], nw <= 32
    ba.vpos = V;

    PrepArgs pa{};
    pa.values = Qv->d_values;
    pa.empty = Qv->d_empty;
    pa.ld_in = Qv->ld;
    pa.n_q = (uint32_t)n_q;
    pa.nb = nb;
    pa.nw = nw;
    pa.remap = 1;
    pa.QT = w.QT;
    pa.QE = w.QE;
    pa.QM = w.QM;
    pa.QEM = w.QEM;
    pa.qflags = w.qflags;
    pa.ldq = w.ldq;
    if (launch_prep(pa, stream) != cudaSuccess) return OPH_ECUDA;

    ba.F = Sv->d_values;
    ba.E = Sv->d_empty;
    ba.n_sets = n_s;
    ba.ld = Sv->ld;
    ba.s_begin = 0;
    ba.QT = w.QT;
    ba.ldq = w.ldq;
    ba.QM = w.QM;
    ba.QEM = w.QEM;
    ba.nb = nb;
    ba.nw = nw;
    // bins in the value -> row table: all for full OPH and GOPH, group 1 for HOPH (its later
    // groups are compared pair by pair from QM)
    ba.nscan = method == OPH_METHOD_HOPH ? std::min<uint32_t>(nb, kp) : nb;
    // bins staged per CTA tile: all (GOPH staging only up to level l0 + 1 measured 13.5 vs
    // 12.9 ms on image-like: the branch-free all-staged lookup wins)
    ba.npre = ba.nscan;
    // short staged tiles (HOPH: one group) need more of them in flight: ~48 KB of staged values
    // per CTA (r02z17 A/B, image-like full OPH: 32 KB 16.02 ms, 48 KB 15.91, 64 KB 15.88, 96 KB
    // 18.10 -- one CTA per SM; GOPH / HOPH flat); OPHGPU_BIT_STAGE_KB overrides the budget
    static const uint32_t stage_bytes =
        getenv("OPHGPU_BIT_STAGE_KB") ? 1024u * (uint32_t)atoi(getenv("OPHGPU_BIT_STAGE_KB")) : 49152u;
    ba.nstage = std::max<uint32_t>(2, std::min<uint32_t>(8, stage_bytes / (ba.npre * 32)));
    ba.kp = kp;
    ba.nbins_total = nb;
    ba.method = method;
    ba.mode_hoph = method == OPH_METHOD_HOPH;
    ba.joint = p->empty_mode == OPH_EMPTY_JOINT;
    ba.t_num = p->t_num;
    ba.t_den = p->t_den;
    ba.nlev = method == OPH_METHOD_FULL ? 1 : nlev;
    ba.level_final = method == OPH_METHOD_FULL ? nb / kp : nlev;
    ba.out.hits = res->d_hits;
    ba.out.cap = res->capacity;
    ba.out.count = res->d_count;
    ba.out.dense = res->mode == OPH_RES_DENSE;
    ba.out.set_id_base = set_id_base;
    ba.out.n_sets = n_s;
    ba.out.hist = res->d_stop_hist;
    ba.scanned = res->d_bins_scanned;
    // full OPH in threshold mode: a set's scan stops once no pair of the block can reach T
    // (R32 / R32b), checked every 32 bins from bin ceil32(9 k / 16) on (288 at k = 512: image-like
    // sweep of the first checkpoint, same box: 256 11.54 ms, 288 11.16, 320 11.96, 352 12.79;
    // every 64 from 288 11.11 -- profiles/r02/full_exit_schedule_r02z32.log);
    // OPHGPU_FULL_EXIT=0 scans every bin (A/B)
    const bool no_exit = getenv("OPHGPU_FULL_EXIT") && atoi(getenv("OPHGPU_FULL_EXIT")) == 0;  // (per call: tests)
    // (OPHGPU_FULL_EXIT_FROM: the first bin count checked, a multiple of 32, A/B; per call: tests)
    const uint32_t exit_from = getenv("OPHGPU_FULL_EXIT_FROM")
                                   ? std::max<uint32_t>(32u, (uint32_t)atoi(getenv("OPHGPU_FULL_EXIT_FROM")) / 32u * 32u)
                                   : std::max<uint32_t>(32u, (9u * nb / 16u + 31u) / 32u * 32u);
    ba.exit_from = (method == OPH_METHOD_FULL && res->mode != OPH_RES_DENSE && !no_exit) ? exit_from : 0u;
    // (OPHGPU_FULL_EXIT_EVERY=64: every other checkpoint, A/B)
    ba.exit_every = getenv("OPHGPU_FULL_EXIT_EVERY") && atoi(getenv("OPHGPU_FULL_EXIT_EVERY")) == 64 ? 64u : 32u;
    // the bins' value ranges: flat = one range of nb bins; HOPH = nlev group ranges of kp bins
    if (method == OPH_METHOD_HOPH) {
        oph_hier_layout lay;
        if (oph_hier_layout_make(V, 1, 1, kp, &lay) != OPH_OK || lay.L != nlev) return OPH_EINCOMPAT;
        ba.bins_per_range = kp;
        for (uint32_t g = 0; g < nlev; g++) ba.ranges[g] = make_range(lay.start[g], lay.len[g], kp);
        for (uint32_t j = 0; j < nlev; j++) ba.c[j] = plan.c[j];
        ba.lam = plan.lam;
    } else {
        ba.bins_per_range = nb;
        ba.ranges[0] = make_range(0, V, nb);
    }
    // level thresholds on the bit-sliced states: GOPH M_c as compiled; HOPH group 1:
    // S_1 = c_1 M_1 = 2^(L-2) M_1, so S_1 >= A <=> M_1 >= ceil(A / 2^(L-2)) and S_1 <= R <=>
    // M_1 <= floor(R / 2^(L-2)); acc128 / rej128: the exact thresholds of the per-pair walk
    for (uint32_t l = 1; method != OPH_METHOD_FULL && l < nlev; l++) {
        const LevelThr &T = plan.thr[l - 1];
        const uint32_t sh = method == OPH_METHOD_HOPH ? nlev - 1 - l : 0;
        const u128 div = (u128)1 << sh;
        u128 A = T.acc == kNeverAcc ? (u128)UINT32_MAX : (T.acc + div - 1) / div;
        ba.acc_cnt[l - 1] = A >= (u128)UINT32_MAX ? UINT32_MAX : (uint32_t)A;
        ba.rej_cnt[l - 1] = T.rej < 0 ? -1 : (int32_t)std::min<i128>(T.rej / (i128)div, (i128)INT32_MAX);
        ba.thr_on[l - 1] = ba.acc_cnt[l - 1] != UINT32_MAX || ba.rej_cnt[l - 1] >= 0;
        ba.acc128[l - 1] = T.acc;
        ba.rej128[l - 1] = T.rej;
    }
    // blocks of 2,048 queries (two words per lane); OPHGPU_BIT_QW=1 forces 1,024 for full OPH /
    // GOPH (A/B)
    static const bool qw1 = getenv("OPHGPU_BIT_QW") && atoi(getenv("OPHGPU_BIT_QW")) == 1;
    ba.qw = qw1 && method != OPH_METHOD_HOPH ? 1 : 2;
    // bit_pipe_kernel (2,048-query rows; nscan / 16 batches per set, even, >= 4): full OPH, and
    // GOPH over levels 1 .. level_b = l0 + 1 (the first level with a decision, and one more:
    // on image-like l0 decides 2/3 of the pairs and l0 + 1 nearly all the rest), the few
    // pairs left walked one by one; the bitmap table and the staged tiles then cover only
    // those levels.  OPHGPU_BIT_PIPE=0 / OPHGPU_GOPH_LB=n: A/B (read per call: tests set them)
    ba.pipe = 0;
    ba.level_b = ba.nlev;
    const char *pipe_env = getenv("OPHGPU_BIT_PIPE");
    if (ba.qw == 2 && method != OPH_METHOD_HOPH && !(pipe_env && atoi(pipe_env) == 0)) {
        auto ok = [](uint32_t bins) { return bins % 32 == 0 && bins >= 64; };
        if (method == OPH_METHOD_FULL) {
            ba.pipe = nb % 64 == 0;  // (ring slots restart with every set: batches % 4 == 0)
        } else {
            const char *lb_env = getenv("OPHGPU_GOPH_LB");
            uint32_t Lb = lb_env ? (uint32_t)atoi(lb_env) : plan.l0 + 1;
            Lb = std::max<uint32_t>(1u, std::min<uint32_t>(Lb, nlev));
            while (Lb < nlev && !ok(Lb * kp)) Lb++;
            if (ok(Lb * kp)) {
                ba.pipe = 1;
                ba.level_b = Lb;
                ba.nscan = ba.npre = Lb * kp;
                ba.nstage = std::max<uint32_t>(2, std::min<uint32_t>(8, stage_bytes / (ba.npre * 32)));
            }
        }
    }
    const uint64_t qb = 1024ull * ba.qw;
    for (uint64_t q0 = 0; q0 < n_q; q0 += qb) {
        ba.qb0 = (uint32_t)q0;
        ba.nqb = (uint32_t)std::min<uint64_t>(qb, n_q - q0);
        if (launch_bit_block(ba, stream) != cudaSuccess) return OPH_ECUDA;
    }
    return OPH_OK;
}

// ---------------------------------------------------------------- the compare driver
oph_status run_compare(uint32_t method, const oph_sketches *Qv, const oph_sketches *Sv, uint32_t set_id_base,
                       uint32_t k_or_L, uint32_t kp, uint32_t a, uint32_t b, const oph_params *p, oph_results *res,
                       void *d_ws, size_t ws_bytes, cudaStream_t stream) {
    const bool mw = method == OPH_METHOD_MINWISE;
    oph_status st;
    if ((st = check_view(Qv, !mw, mw)) || (st = check_view(Sv, !mw, mw)) || (st = check_params(p))) return st;
    if (!res || !res->d_hits || !res->d_count || res->mode > OPH_RES_DENSE) return OPH_EINVAL;
    if (p->strategy > OPH_STRATEGY_BITMAP || p->variant > OPH_VARIANT_EMPTY_AWARE) return OPH_EINVAL;
    // the empty-aware GOPH rule (E1-E4) runs as one register scan of every group
    const bool ea = p->variant == OPH_VARIANT_EMPTY_AWARE;
    if (ea && method != OPH_METHOD_GOPH && method != OPH_METHOD_HOPH) return OPH_EINVAL;
    if (Qv->seed != Sv->seed || Qv->vocab_size != Sv->vocab_size || Qv->n_bins != Sv->n_bins) return OPH_EINCOMPAT;
    const uint32_t nb = Qv->n_bins;
    const uint32_t nw = (uint32_t)ceil_div(nb, 32);
    if (nb > 16384) return OPH_EINVAL;
    if ((uint64_t)set_id_base + Sv->n_sets > 0xFFFFFFFFull) return OPH_EINVAL;
    const uint64_t n_q = Qv->n_sets, n_s = Sv->n_sets;
    if (res->mode == OPH_RES_DENSE && res->capacity < n_q * n_s) return OPH_EINVAL;
    if (n_q == 0 || n_s == 0) return OPH_OK;

    Plan plan;
    uint32_t nlev = 1;
    if (method == OPH_METHOD_GOPH || method == OPH_METHOD_HOPH) {
        nlev = method == OPH_METHOD_GOPH ? k_or_L / kp : k_or_L;
        if (nlev > kMaxGroups) return OPH_EINVAL;
        plan = make_plan(method, nlev, kp, a, b, p->t_num, p->t_den, p->epsilon);
        if (plan.st != OPH_OK) return plan.st;
        if (method == OPH_METHOD_HOPH && nlev > 1 && plan.lam == 0) return OPH_EINVAL;
        if (ea && method == OPH_METHOD_GOPH && (uint64_t)nlev * kp > 512) return OPH_EINVAL;
        if (ea && method == OPH_METHOD_HOPH) {
            // the empty-aware HOPH rule's exact 128-bit states: k'^2 t_num t_den D lcm(1..k') < 2^124
            u128 D = 0;
            for (uint32_t j = 0; j < nlev; j++) D += plan.c[j];
            const long double mag = (long double)kp * kp * p->t_num * p->t_den * (long double)D * (long double)plan.lam;
            if (plan.lam == 0 || nlev < 2 || mag >= 1.0e37L) return OPH_EINVAL;
        }
    }

    const size_t fixed = ws_fixed_bytes(n_q, n_s, nb);

    // BITMAP (bitjoin.cuh): full OPH, GOPH (Algorithm 1) and HOPH with the 1:1 split (group 1
    // bit-sliced, S_1 = c_1 M_1; the later groups per pair on exact 128-bit S_l), |V| <= 2^23,
    // <= 1023 bins
    {
        // (GOPH / HOPH levels must be whole batches of 16 bins: k' % 16 == 0)
        const bool dom = !mw && !ea && bitmap_sizes_ok(Qv->vocab_size, nb) && Sv->ld % 8 == 0 &&
                         (method == OPH_METHOD_FULL || kp % 16 == 0) &&
                         (method != OPH_METHOD_HOPH || (a == 1 && b == 1 && nlev >= 2 && plan.lam));
        const bool fits = ws_bytes >= fixed + bitmap_region_bytes(Qv->vocab_size, nb);
        bool use = false;
        if (p->strategy == OPH_STRATEGY_BITMAP) {
            if (!dom) return OPH_EINVAL;
            if (!fits) return OPH_ENOMEM;
            use = true;
        } else if (p->strategy == OPH_STRATEGY_AUTO && dom && fits && n_q >= 1024) {
            // (a block's scan costs the same for 1 or 2,048 queries: below ~1,024 queries the
            // register scan's Q N k compares are cheaper -- sweep-0.5, full OPH, r02z36: 256 queries
            // 41.6 vs 23.3 ms, 512 queries 42.6 vs 45.8 ms.  GOPH / HOPH on a collection whose
            // pairs mostly survive the bitmap's levels (the sweep: every set a near-duplicate of
            // the hub) walk those pairs one by one and lose to the register scan at any query
            // count -- 512 queries: 225 vs 24.9 ms, 78 vs 6.4 ms; AUTO does not detect that
            // regime)
            // AUTO: where PROBE would not apply, or this collection was found to be a BRUTE one
            const bool probe_ok =
                res->mode != OPH_RES_DENSE &&
                (method == OPH_METHOD_FULL ||
                 (method == OPH_METHOD_GOPH && (plan.l0 == nlev || plan.thr[plan.l0 - 1].rej >= 0)) ||
                 (method == OPH_METHOD_HOPH && (nlev == 1 || plan.thr[0].rej >= 0)));
            int cached = -1;
            {
                std::lock_guard<std::mutex> g(g_auto_mu);
                auto it = g_auto.find(AutoKey{(uintptr_t)Sv->d_values, n_s, nb, method});
                if (it != g_auto.end()) cached = it->second;
            }
            use = !probe_ok || cached == 1;
        }
        if (use) return run_bitmap(method, Qv, Sv, set_id_base, nb, nw, nlev, kp, plan, p, res, d_ws, fixed, stream);
    }
    uint64_t chunk = ceil_div(n_q, 32) * 32;
    uint64_t cap = 0;
    const bool levels = (method == OPH_METHOD_GOPH || method == OPH_METHOD_HOPH) && (plan.l0 < nlev || ea);
    // the empty-aware rule with threshold results and no histogram: the join lists every pair
    // with a matched bin (no other pair can be Similar, E5) and level_e_kernel
    // decides those survivors; otherwise the register scan decides every pair (no lists)
    // AUTO with a remembered BRUTE decision for this collection runs as BRUTE outright
    // (no sample join, no survivor-sized query chunks)
    const AutoKey akey{(uintptr_t)Sv->d_values, n_s, nb, method | (ea ? 16u : 0u)};
    uint32_t strategy = p->strategy;
    if (strategy == OPH_STRATEGY_AUTO) {
        std::lock_guard<std::mutex> g(g_auto_mu);
        auto it = g_auto.find(akey);
        if (it != g_auto.end() && it->second == 1) strategy = OPH_STRATEGY_BRUTE;
    }
    const bool ea_probe = ea && strategy != OPH_STRATEGY_BRUTE && res->mode != OPH_RES_DENSE && !res->d_stop_hist;
    const uint32_t surv_l = ea ? 1u : plan.l0;  // counter / list parity of the scan's survivors
    // BRUTE scans of GOPH / HOPH decide every level in one pass (levels_kernel) when the
    // pair states fit 32 bits and every group's query values fit shared memory; else
    // the scan covers the first decidable level and survivors go through level_kernel
    // (HOPH packs the raw matched-bin count into the counter's low 10 bits: records need it)
    u128 state_max = 0;
    for (uint32_t j = 0; levels && j < nlev; j++) state_max += plan.c[j] * kp;
    const uint32_t msh = method == OPH_METHOD_HOPH ? 10u : 0u;
    // (OPHGPU_NO_MULTI_LEVEL_SCAN set: the survivor path always -- A/B diagnostics and the
    // parity test of that path)
    const bool no_multi = getenv("OPHGPU_NO_MULTI_LEVEL_SCAN") != nullptr;
    const bool multi =
        levels && (uint64_t)nlev * kp <= 512 &&
        (((state_max << msh) < (u128)UINT32_MAX && !no_multi && !ea) || (ea && method == OPH_METHOD_GOPH));
    // the empty-aware HOPH rule without a join list (dense records, histograms, BRUTE): one
    // per-pair walk over every (query, set) pair
    const bool he_all = ea && method == OPH_METHOD_HOPH && !ea_probe;
    // the multi-level scan of a BRUTE or dense call produces no survivor lists: all
    // queries in one chunk (survivor-sized chunks cut its grid into small launches)
    const bool no_lists = multi && !ea_probe && (strategy == OPH_STRATEGY_BRUTE || res->mode == OPH_RES_DENSE);
    if (levels && (!ea || ea_probe) && !no_lists) {
        cap = cap_from_ws(ws_bytes, fixed);
        const uint64_t fit = (cap / n_s) / 32 * 32;
        if (fit < 32) return OPH_ENOMEM;
        chunk = std::min(chunk, fit);
    } else if (ws_bytes < fixed) {
        return OPH_ENOMEM;
    }
    Ws w = carve_ws(d_ws, n_q, n_s, nb, cap);

    PrepArgs pa{};
    pa.values = Qv->d_values;
    pa.empty = mw ? nullptr : Qv->d_empty;
    pa.flags = mw ? Qv->d_flags : nullptr;
    pa.ld_in = Qv->ld;
    pa.n_q = (uint32_t)n_q;
    pa.nb = nb;
    pa.nw = nw;
    pa.remap = !mw;
    pa.QT = w.QT;
    pa.QE = w.QE;
    pa.QM = w.QM;
    pa.QEM = w.QEM;
    pa.qflags = w.qflags;
    pa.ldq = w.ldq;
    cudaError_t e = launch_prep(pa, stream);
    if (e != cudaSuccess) return OPH_ECUDA;

    OutArgs out{};
    out.hits = res->d_hits;
    out.cap = res->capacity;
    out.count = res->d_count;
    out.dense = res->mode == OPH_RES_DENSE;
    out.set_id_base = set_id_base;
    out.n_sets = n_s;
    out.hist = res->d_stop_hist;

    ScanArgs s{};
    s.F = Sv->d_values;
    s.E = mw ? nullptr : Sv->d_empty;
    s.sflags = mw ? Sv->d_flags : nullptr;
    s.n_sets = n_s;
    s.ld = Sv->ld;
    s.QT = w.QT;
    s.QE = w.QE;
    s.qflags = w.qflags;
    s.ldq = w.ldq;
    s.method = method;
    s.joint = p->empty_mode == OPH_EMPTY_JOINT;
    s.t_num = p->t_num;
    s.t_den = p->t_den;
    s.out = out;
    s.w1 = 1;
    s.one = 1;
    s.acc_cnt = UINT32_MAX;
    s.rej_cnt = -1;
    // the scan decides on the raw count of its groups: state = w1 * count, so
    // state >= acc <=> count >= ceil(acc / w1) and state <= rej <=> count <= floor(rej / w1)
    auto set_count_thresholds = [&](u128 w1, const LevelThr &T) {
        s.w1 = w1;
        s.acc_cnt = T.acc == kNeverAcc ? UINT32_MAX
                                       : (uint32_t)std::min<u128>((T.acc + w1 - 1) / w1, (u128)UINT32_MAX);
        s.rej_cnt = T.rej < 0 ? -1 : (int32_t)std::min<i128>(T.rej / (i128)w1, (i128)INT32_MAX);
    };
    s.nbins_total = nb;
    if (method == OPH_METHOD_FULL || mw) {
        s.nscan = nb;
        s.final_ = 1;
        s.level = mw ? 0 : nb / kp;
        s.nw_load = mw ? 0 : nw;
    } else if (ea_probe) {  // list every pair with a matched bin as a survivor
        s.nscan = nb;
        s.level = 1;
        s.final_ = 0;
        s.nw_load = nw;
        s.acc_cnt = UINT32_MAX;
        s.rej_cnt = 0;
    } else if (method == OPH_METHOD_GOPH) {
        s.nscan = plan.l0 * kp;
        s.level = plan.l0;
        s.final_ = plan.l0 == nlev;
        s.nw_load = (uint32_t)(s.final_ ? nw : ceil_div(s.nscan, 32));
        if (!s.final_) set_count_thresholds(1, plan.thr[plan.l0 - 1]);
    } else {  // HOPH: the scan compares group 1
        s.nscan = kp;
        s.level = 1;
        s.final_ = nlev == 1;  // one group: the HOPH estimator is the OPH estimator of it
        s.nw_load = (uint32_t)ceil_div(kp, 32);
        if (!s.final_) set_count_thresholds(plan.c[0], plan.thr[0]);
    }
    if (((size_t)std::min<uint32_t>(s.nscan, 512) + s.nw_load + 1) * 32 * 4 > 227 * 1024) return OPH_EINVAL;

    // PROBE applies to threshold results when a pair with no matched bin is
    // decided NotSimilar at the scanned level (final verdicts: N_mb = 0 is
    // never >= T > 0; otherwise the level must reject state 0)
    const bool probe = ea ? ea_probe : strategy != OPH_STRATEGY_BRUTE && !out.dense && (s.final_ || s.rej_cnt >= 0);

    LevelArgs la{};
    if (levels) {
        la.F = Sv->d_values;
        la.E = Sv->d_empty;
        la.n_sets = n_s;
        la.ld = Sv->ld;
        la.QM = w.QM;
        la.QEM = w.QEM;
        la.nb = nb;
        la.nw = nw;
        la.method = method;
        la.nlev = nlev;
        la.kp = kp;
        la.joint = s.joint;
        la.t_num = p->t_num;
        la.t_den = p->t_den;
        for (uint32_t j = 0; j < nlev; j++) la.c[j] = plan.c[j];
        for (uint32_t l = 1; l < nlev; l++) {
            la.acc[l - 1] = plan.thr[l - 1].acc;
            la.rej[l - 1] = plan.thr[l - 1].rej;
        }
        la.lam = plan.lam;
        la.res = out;
        if (ea) {
            // Alg. 1's tail tests on M_ra reduce to two integers: floor(M_ra) <= m_a <=> M_ra < ma1
            // and ceil(M_ra) >= m_r <=> M_ra > mr1 (lower_le / upper_le are monotone)
            std::vector<uint8_t> lo, up;
            const oph_status ts = small_prob_tables(kp, p->t_num, p->t_den, p->epsilon, lo, up);
            if (ts != OPH_OK) return ts;
            uint32_t ma1 = 0, mr = kp + 1;
            while (ma1 <= kp && lo[ma1]) ma1++;
            while (mr > 0 && up[mr - 1]) mr--;
            for (uint32_t m = 0; m <= kp; m++)
                if (lo[m] != (m < ma1)) return OPH_EINVAL;
            for (uint32_t m = 0; m <= kp + 1; m++)
                if (up[m] != (m >= mr)) return OPH_EINVAL;
            if (mr == 0) return OPH_EINVAL;  // P(X >= 0) = 1 > eps
            la.eaware = 1;
            la.QE = w.QE;
            la.ma1 = ma1;
            la.mr1 = mr - 1;
        }
        // multi-level BRUTE scan (levels_kernel): states as u32 counters, thresholds on them
        la.QT = w.QT;
        la.ldq = w.ldq;
        la.one = 1;
        la.sh = msh;
        for (uint32_t j = 0; j < nlev; j++)
            la.w32[j] = multi ? (uint32_t)((plan.c[j] << msh) | (msh ? 1u : 0u)) : 0u;
        for (uint32_t l = 1; l < nlev; l++) {
            const LevelThr &T = plan.thr[l - 1];
            const u128 A = T.acc == kNeverAcc ? (u128)UINT32_MAX : T.acc << msh;
            la.acc32[l - 1] = A >= (u128)UINT32_MAX ? UINT32_MAX : (uint32_t)A;
            const i128 R1 = T.rej < 0 ? 0 : (T.rej + 1) << msh;
            la.rej1[l - 1] = R1 >= (i128)UINT32_MAX ? UINT32_MAX : (uint32_t)R1;
        }
    }

    unsigned long long *ovf_count = w.counters + kMaxGroups + 2;
    unsigned long long *saved_hits = w.counters + kMaxGroups + 3;  // not cleared per chunk
    unsigned long long *saved_hist = w.counters + kMaxGroups + 4;  // [OPH_STOP_HIST_LEN], likewise

    // the collection scan of queries [q0, q0+nq): BRUTE, or PROBE + its BRUTE list fallback
    // (PROBE in passes of <= kJoinMaxQ queries, each one stream over the collection)
    auto probe_pass_run = [&](uint64_t q0, uint64_t nq) -> cudaError_t {
        cudaError_t e;
        s.q_col0 = (uint32_t)q0;
        s.nq = (uint32_t)nq;
        if ((e = cudaMemsetAsync(ovf_count, 0, 8, stream)) != cudaSuccess) return e;
        const uint32_t log2S = probe_log2S(nq), log2W = probe_log2W(nq);
        if ((e = cudaMemsetAsync(w.table, 0, (size_t)s.nscan * (1ull << log2S) * 8, stream)) != cudaSuccess) return e;
        if ((e = cudaMemsetAsync(w.bloom, 0, (size_t)ceil_div(s.nscan, 32) * (1ull << log2W) * 32 * 4, stream)) !=
            cudaSuccess)
            return e;
        TableArgs ta{};
        ta.QT = w.QT;
        ta.qflags = w.qflags;
        ta.ldq = w.ldq;
        ta.q_col0 = (uint32_t)q0;
        ta.nq = (uint32_t)nq;
        ta.nscan = s.nscan;
        ta.log2S = log2S;
        ta.minwise = mw;
        ta.table = w.table;
        ta.bloom = w.bloom;
        ta.log2W = log2W;
        if ((e = launch_table(ta, stream)) != cudaSuccess) return e;
        ProbeArgs pr{};
        pr.F = s.F;
        pr.E = s.E;
        pr.sflags = s.sflags;
        pr.n_sets = n_s;
        pr.ld = s.ld;
        pr.table = w.table;
        pr.bloom = w.bloom;
        pr.log2S = log2S;
        pr.log2W = log2W;
        pr.nscan = s.nscan;
        pr.QEM = w.QEM;
        pr.qflags = w.qflags;
        pr.nw = nw;
        pr.nbins_total = nb;
        pr.q_col0 = (uint32_t)q0;
        pr.nq = (uint32_t)nq;
        pr.method = method;
        pr.final_ = s.final_;
        pr.level = s.level;
        pr.joint = s.joint;
        pr.t_num = s.t_num;
        pr.t_den = s.t_den;
        pr.w1 = s.w1;
        pr.acc_cnt = s.acc_cnt;
        pr.rej_cnt = s.rej_cnt;
        pr.out = out;
        pr.surv = s.surv;
        pr.surv_count = s.surv_count;
        pr.surv_cap = cap;
        pr.ovf_list = w.ovf_list;
        pr.ovf_count = ovf_count;
        // AUTO probes a leading sample of the sets first; when more than a quarter of it
        // matches too many distinct queries (a high-similarity collection), the rest goes
        // to BRUTE as one contiguous scan instead of the list fallback
        // The decision is only a speed heuristic (every strategy returns the same results), so
        // it is remembered per (collection buffer, size, bins, method, pass size): a repeated call
        // on the same collection skips the sample's host synchronisation -- a probe decision
        // becomes one join over every set.
        uint64_t n1 = strategy == OPH_STRATEGY_AUTO
                          ? std::min<uint64_t>(n_s, std::max<uint64_t>(16384, ceil_div(n_s / 16, 256) * 256))
                          : n_s;
        int cached = -1;  // -1 unknown, 0 probe the rest, 1 BRUTE the rest
        if (n1 < n_s) {
            std::lock_guard<std::mutex> g(g_auto_mu);
            auto it = g_auto.find(akey);
            if (it != g_auto.end()) cached = it->second;
        }
        if (cached == 0) n1 = n_s;
        pr.s_begin = 0;
        pr.s_end = n1;
        if ((e = launch_probe(pr, stream)) != cudaSuccess) return e;
        if (n1 < n_s) {
            bool brute_rest = cached == 1;
            if (cached < 0) {
                unsigned long long ovf = 0;
                if ((e = cudaMemcpyAsync(&ovf, ovf_count, sizeof(ovf), cudaMemcpyDeviceToHost, stream)) != cudaSuccess)
                    return e;
                if ((e = cudaStreamSynchronize(stream)) != cudaSuccess) return e;
                brute_rest = ovf * 4 > n1;
                std::lock_guard<std::mutex> g(g_auto_mu);
                if (g_auto.size() >= 4096) g_auto.clear();  // bounded: stale buffers age out
                g_auto[akey] = brute_rest ? 1 : 0;
            }
            if (brute_rest) {
                if (multi) {
                    LevelArgs lm = la;
                    lm.q_col0 = (uint32_t)q0;
                    lm.nq = (uint32_t)nq;
                    lm.s_begin = n1;
                    if ((e = launch_levels_scan(lm, stream)) != cudaSuccess) return e;
                } else {
                    ScanArgs sr = s;
                    sr.s_begin = n1;
                    if ((e = launch_scan(sr, 32, stream)) != cudaSuccess) return e;
                }
            } else {
                pr.s_begin = n1;
                pr.s_end = n_s;
                if ((e = launch_probe(pr, stream)) != cudaSuccess) return e;
            }
        }
        // sets with too many distinct matched queries: BRUTE over that list (device-side count)
        ScanArgs sl = s;
        sl.set_list = w.ovf_list;
        sl.list_count = ovf_count;
        return launch_scan(sl, 32, stream);
    };
    auto scan_chunk = [&](uint64_t q0, uint64_t nq) -> cudaError_t {
        cudaError_t e;
        s.q_col0 = (uint32_t)q0;
        s.nq = (uint32_t)nq;
        s.surv_cap = cap;
        if (levels) {
            s.surv = w.list[surv_l % 2];
            s.surv_count = w.counters + surv_l;
        }
        if (levels || probe)
            if ((e = cudaMemsetAsync(w.counters, 0, (kMaxGroups + 3) * 8, stream)) != cudaSuccess) return e;
        if (!probe) {
            if (he_all) {
                LevelArgs lm = la;
                lm.q_col0 = (uint32_t)q0;
                lm.nq = (uint32_t)nq;
                lm.implicit = 1;
                return launch_level_e(lm, stream);
            }
            if (!multi) return launch_scan(s, 32, stream);
            LevelArgs lm = la;
            lm.q_col0 = (uint32_t)q0;
            lm.nq = (uint32_t)nq;
            lm.s_begin = 0;
            return launch_levels_scan(lm, stream);
        }
        const uint64_t pq = probe_pass(nq);
        for (uint64_t a0 = q0; a0 < q0 + nq; a0 += pq)
            if ((e = probe_pass_run(a0, std::min<uint64_t>(pq, q0 + nq - a0))) != cudaSuccess) return e;
        return cudaSuccess;
    };
    // later levels, kLevelsPerLaunch per launch, survivors compacted between launches
    // (empty-aware rule: one launch decides every listed pair)
    auto level_chunk = [&]() -> cudaError_t {
        if (ea) {
            la.in = w.list[surv_l % 2];
            la.count_in = w.counters + surv_l;
            return launch_level_e(la, stream);
        }
        // the first launch compacts after kLevelsPerLaunch levels; the few survivors left
        // then finish every remaining level in one launch (HOPH text-like: 2 launches, not 7).
        // The lists ping-pong explicitly: a launch reads list[cur] and appends to the other
        // one (input and output must never alias: the grid-stride walk of the input runs
        // concurrently with other warps' appends).
        uint32_t cur = surv_l % 2;  // the scan appended its survivors to list[surv_l % 2]
        // k' <= 32: one launch of the warp-per-pair walk decides every remaining level
        const bool walk = kp <= 32;
        for (uint32_t l = plan.l0 + 1, first = 1; l <= nlev; first = 0) {
            const uint32_t l_last = (first && !walk) ? std::min(nlev, l + kLevelsPerLaunch - 1) : nlev;
            la.level = l;
            la.level_last = l_last;
            la.in = w.list[cur];
            la.out = w.list[cur ^ 1u];
            cur ^= 1u;
            la.count_in = w.counters + (l - 1);
            la.count_out = w.counters + l_last;
            cudaError_t e = launch_level(la, stream);
            if (e != cudaSuccess) return e;
            l = l_last + 1;
        }
        return cudaSuccess;
    };
    auto safe_range = [&](uint64_t q0, uint64_t q1) -> cudaError_t {
        for (uint64_t a0 = q0; a0 < q1; a0 += chunk) {
            cudaError_t e = scan_chunk(a0, std::min<uint64_t>(chunk, q1 - a0));
            if (e != cudaSuccess) return e;
            if (levels && (!ea || probe) && (e = level_chunk()) != cudaSuccess) return e;
        }
        return cudaSuccess;
    };

    if (levels && probe && chunk < n_q) {
        // PROBE leaves few survivors: try every query at once; if the survivor list overflowed,
        // roll the hit counter back and redo the queries in chunks sized for the worst case
        e = cudaMemcpyAsync(saved_hits, res->d_count, 8, cudaMemcpyDeviceToDevice, stream);
        if (e == cudaSuccess && res->d_stop_hist)
            e = cudaMemcpyAsync(saved_hist, res->d_stop_hist, 8 * OPH_STOP_HIST_LEN, cudaMemcpyDeviceToDevice, stream);
        if (e == cudaSuccess) e = scan_chunk(0, n_q);
        unsigned long long n_surv = 0;
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(&n_surv, w.counters + surv_l, sizeof(n_surv), cudaMemcpyDeviceToHost, stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
        if (e != cudaSuccess) return OPH_ECUDA;
        if (n_surv <= cap) {
            e = level_chunk();
        } else {
            e = cudaMemcpyAsync(res->d_count, saved_hits, 8, cudaMemcpyDeviceToDevice, stream);
            if (e == cudaSuccess && res->d_stop_hist)
                e = cudaMemcpyAsync(res->d_stop_hist, saved_hist, 8 * OPH_STOP_HIST_LEN, cudaMemcpyDeviceToDevice,
                                    stream);
            if (e == cudaSuccess) e = safe_range(0, n_q);
        }
        return e == cudaSuccess ? OPH_OK : OPH_ECUDA;
    }
    return safe_range(0, n_q) == cudaSuccess ? OPH_OK : OPH_ECUDA;
}

}  // namespace

// ======================================================================== C-ABI
extern "C" {

const char *oph_status_string(oph_status s) {
    switch (s) {
        case OPH_OK: return "ok";
        case OPH_EINVAL: return "invalid argument";
        case OPH_EINCOMPAT: return "incompatible sketches (seed, universe or layout differ)";
        case OPH_EOVERFLOW: return "result buffer overflow";
        case OPH_ECUDA: return "CUDA error";
        case OPH_EAMBIGUOUS: return "a binomial tail is within 1e-9 relative of epsilon";
        case OPH_ENOMEM: return "workspace too small";
    }
    return "unknown status";
}

uint64_t oph_sketch_ld(uint64_t n_sets) { return ceil_div(n_sets ? n_sets : 1, 32) * 32; }

oph_status oph_hier_layout_make(uint64_t V, uint32_t a, uint32_t b, uint32_t kp, oph_hier_layout *out) {
    if (!out || a == 0 || b == 0 || kp == 0 || kp > 65535 || V == 0 || V > (1ull << 32) || V < 2ull * kp)
        return OPH_EINVAL;
    std::memset(out, 0, sizeof(*out));
    out->vocab_size = V;
    out->a = a;
    out->b = b;
    out->kprime = kp;
    // recursive a:b split of the remaining space (R17, R18)
    uint64_t R = V, s = 0;
    uint32_t L = 0;
    for (;;) {
        if (L >= OPH_MAX_GROUPS) return OPH_EINVAL;
        const uint64_t f = (uint64_t)(((u128)a * R) / (a + b));
        const uint64_t r = R - f;
        if (f <= kp || r <= kp) {
            out->start[L] = s;
            out->len[L] = R;
            L++;
            break;
        }
        out->start[L] = s;
        out->len[L] = f;
        L++;
        s += f;
        R = r;
    }
    out->L = L;
    return OPH_OK;
}

oph_status oph_validate_sets(const oph_sets *sets, uint64_t V, void *stream) {
    oph_status st;
    if ((st = check_sets(sets))) return st;
    if (V == 0 || V > (1ull << 32)) return OPH_EINVAL;
    if (sets->n_sets == 0) return OPH_OK;
    cudaStream_t s = (cudaStream_t)stream;
    uint32_t *bad = nullptr, h = 0;
    if (cudaMallocAsync((void **)&bad, 4, s) != cudaSuccess) return OPH_ECUDA;
    cudaError_t e = cudaMemsetAsync(bad, 0, 4, s);
    if (e == cudaSuccess) e = launch_validate(sets->d_offsets, sets->d_ids, sets->n_sets, V, bad, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h, bad, 4, cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(bad, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return OPH_ECUDA;
    return h ? OPH_EINVAL : OPH_OK;
}

static bool validate_env() {
    static const bool on = getenv("OPHGPU_VALIDATE") != nullptr;
    return on;
}

oph_status oph_build_sketches(const oph_sets *sets, const oph_perm *perm, const oph_flat_layout *flat, uint32_t *d_oph,
                              uint32_t *d_oph_empty, const oph_hier_layout *hier, uint32_t *d_hoph,
                              uint32_t *d_hoph_empty, uint64_t ld, void *stream) {
    oph_status st;
    if ((st = check_sets(sets))) return st;
    if (!perm || perm->vocab_size == 0 || perm->vocab_size > (1ull << 32) || perm->kind > 1) return OPH_EINVAL;
    if (!flat && !hier) return OPH_EINVAL;
    if (ld < sets->n_sets || ld % 4) return OPH_EINVAL;
    const uint64_t V = perm->vocab_size;
    BuildArgs a{};
    a.offsets = sets->d_offsets;
    a.ids = sets->d_ids;
    a.n_sets = sets->n_sets;
    a.ld = ld;
    a.psi = make_psi(V, perm->seed, perm->kind);
    uint64_t per_set = 0;
    if (flat) {
        if (flat->vocab_size != V || flat->k == 0 || flat->k > 65535 || flat->k > V || !bins_fit(V, flat->k) ||
            !d_oph || !d_oph_empty)
            return OPH_EINVAL;
        a.do_flat = 1;
        a.k = flat->k;
        a.flat = make_range(0, V, flat->k);
        a.oph = d_oph;
        a.oph_empty = d_oph_empty;
        per_set += (flat->k + 31) / 32 * 32 + 1;  // row stride of the build kernel's smem tile
    }
    if (hier) {
        if (hier->vocab_size != V || hier->L == 0 || hier->L > OPH_MAX_GROUPS || hier->kprime == 0 || !d_hoph ||
            !d_hoph_empty)
            return OPH_EINVAL;
        uint64_t s = 0;
        for (uint32_t g = 0; g < hier->L; g++) {  // contiguous cover of [0, V)
            if (hier->start[g] != s || hier->len[g] < hier->kprime || !bins_fit(hier->len[g], hier->kprime))
                return OPH_EINVAL;
            s += hier->len[g];
        }
        if (s != V) return OPH_EINVAL;
        a.do_hier = 1;
        a.L = hier->L;
        a.kp = hier->kprime;
        for (uint32_t g = 0; g < hier->L; g++) a.grp[g] = make_range(hier->start[g], hier->len[g], hier->kprime);
        // fast path: the 1:1 split of a power-of-two universe (group g = [V - V/2^g, V - V/2^(g+1)),
        // the last group the remaining V/2^(L-1)) with a power-of-two kprime
        const uint32_t m = word_bits(V), lk = word_bits(hier->kprime);
        bool halves = V == (1ull << m) && hier->kprime == (1u << lk) && hier->kprime > 1 && hier->L >= 1;
        for (uint32_t g = 0; halves && g < hier->L; g++) {
            const uint64_t len = (g + 1 < hier->L) ? (V >> (g + 1)) : (V >> (hier->L - 1));
            halves = hier->start[g] == V - (V >> g) && hier->len[g] == len && len >= hier->kprime;
        }
        a.hier_pow2_halves = halves;
        a.log2V = m;
        a.log2kp = lk;
        a.hoph = d_hoph;
        a.hoph_empty = d_hoph_empty;
        per_set += ((uint64_t)hier->L * hier->kprime + 31) / 32 * 32 + 1;
    }
    if (per_set * 4 + 16 > 200 * 1024) return OPH_EINVAL;
    if (validate_env() && (st = oph_validate_sets(sets, V, stream)) != OPH_OK) return st;
    return cuda_status(launch_build(a, (cudaStream_t)stream));
}

oph_status minwise_build_sketches(const oph_sets *sets, uint64_t V, uint64_t seed, uint32_t k, uint32_t *d_mw,
                                  uint8_t *d_set_flags, uint64_t ld, void *stream) {
    oph_status st;
    if ((st = check_sets(sets))) return st;
    if (V == 0 || V > (1ull << 32) || k == 0 || k > 65535 || !d_mw || !d_set_flags || ld < sets->n_sets || ld % 4)
        return OPH_EINVAL;
    if (validate_env() && (st = oph_validate_sets(sets, V, stream)) != OPH_OK) return st;
    MinwiseArgs a{};
    a.offsets = sets->d_offsets;
    a.ids = sets->d_ids;
    a.n_sets = sets->n_sets;
    a.ld = ld;
    a.V = V;
    a.seed = seed;
    a.k = k;
    a.w = word_bits(V);
    a.mw = d_mw;
    a.flags = d_set_flags;
    return cuda_status(launch_minwise(a, (cudaStream_t)stream));
}

oph_status oph_workspace_size(uint32_t method, uint64_t n_q, uint64_t n_sets, uint32_t n_bins, uint64_t cap,
                              size_t *bytes) {
    if (!bytes || method > OPH_METHOD_MINWISE || n_bins == 0) return OPH_EINVAL;
    size_t b = ws_fixed_bytes(n_q, n_sets, n_bins);
    if (method == OPH_METHOD_GOPH || method == OPH_METHOD_HOPH) b += surv_region_bytes(std::max<uint64_t>(cap, 32 * n_sets));
    *bytes = b;
    return OPH_OK;
}

oph_status oph_workspace_size_for(uint32_t method, const oph_sketches *q, const oph_sketches *s,
                                  const oph_params *p, uint64_t cap, size_t *bytes) {
    if (!q || !s || !p || !bytes) return OPH_EINVAL;
    oph_status st = oph_workspace_size(method, q->n_sets, s->n_sets, q->n_bins, cap, bytes);
    if (st != OPH_OK) return st;
    if (method != OPH_METHOD_MINWISE && p->variant == OPH_VARIANT_PAPER && bitmap_sizes_ok(q->vocab_size, q->n_bins) &&
        (p->strategy == OPH_STRATEGY_AUTO || p->strategy == OPH_STRATEGY_BITMAP))
        *bytes = std::max(*bytes, ws_fixed_bytes(q->n_sets, s->n_sets, q->n_bins) +
                                      bitmap_region_bytes(q->vocab_size, q->n_bins));
    return OPH_OK;
}

oph_status compare_full(const oph_sketches *q, const oph_sketches *s, uint32_t set_id_base,
                        const oph_flat_layout *layout, const oph_params *p, oph_results *res, void *d_ws,
                        size_t ws_bytes, void *stream) {
    if (!layout || layout->kprime == 0 || layout->k % layout->kprime || !q) return OPH_EINVAL;
    if (q->n_bins != layout->k || q->vocab_size != layout->vocab_size) return OPH_EINCOMPAT;
    return run_compare(OPH_METHOD_FULL, q, s, set_id_base, layout->k, layout->kprime, 1, 1, p, res, d_ws, ws_bytes,
                       (cudaStream_t)stream);
}

oph_status compare_goph(const oph_sketches *q, const oph_sketches *s, uint32_t set_id_base,
                        const oph_flat_layout *layout, const oph_params *p, oph_results *res, void *d_ws,
                        size_t ws_bytes, void *stream) {
    if (!layout || layout->kprime == 0 || layout->k % layout->kprime || !q) return OPH_EINVAL;
    if (q->n_bins != layout->k || q->vocab_size != layout->vocab_size) return OPH_EINCOMPAT;
    return run_compare(OPH_METHOD_GOPH, q, s, set_id_base, layout->k, layout->kprime, 1, 1, p, res, d_ws, ws_bytes,
                       (cudaStream_t)stream);
}

oph_status compare_hoph(const oph_sketches *q, const oph_sketches *s, uint32_t set_id_base,
                        const oph_hier_layout *layout, const oph_params *p, oph_results *res, void *d_ws,
                        size_t ws_bytes, void *stream) {
    if (!layout || layout->L == 0 || layout->L > OPH_MAX_GROUPS || layout->kprime == 0 || !q) return OPH_EINVAL;
    if (q->n_bins != layout->L * layout->kprime || q->vocab_size != layout->vocab_size) return OPH_EINCOMPAT;
    return run_compare(OPH_METHOD_HOPH, q, s, set_id_base, layout->L, layout->kprime, layout->a, layout->b, p, res,
                       d_ws, ws_bytes, (cudaStream_t)stream);
}

oph_status compare_minwise(const oph_sketches *q, const oph_sketches *s, uint32_t set_id_base, const oph_params *p,
                           oph_results *res, void *d_ws, size_t ws_bytes, void *stream) {
    if (!q) return OPH_EINVAL;
    return run_compare(OPH_METHOD_MINWISE, q, s, set_id_base, q->n_bins, 1, 1, 1, p, res, d_ws, ws_bytes,
                       (cudaStream_t)stream);
}

oph_status exact_jaccard_pairs(const oph_sets *queries, const oph_sets *sets, const uint32_t *d_query,
                               const uint32_t *d_set, uint64_t n_pairs, uint32_t *d_inter, uint32_t *d_union,
                               void *stream) {
    oph_status st;
    if ((st = check_sets(queries)) || (st = check_sets(sets))) return st;
    if (n_pairs == 0) return OPH_OK;
    if (!d_query || !d_set || !d_inter || !d_union || !queries->d_offsets || !sets->d_offsets) return OPH_EINVAL;
    JaccardArgs a{};
    a.q_offsets = queries->d_offsets;
    a.s_offsets = sets->d_offsets;
    a.q_ids = queries->d_ids;
    a.s_ids = sets->d_ids;
    a.query = d_query;
    a.set = d_set;
    a.n = n_pairs;
    a.inter = d_inter;
    a.uni = d_union;
    return cuda_status(launch_jaccard(a, (cudaStream_t)stream));
}

// CUB's scan / sort / unique take int item counts: n_bytes + 1 bytes and
// (n_bytes + n_docs) / 2 + 1 tokens must stay below 2^31 - 1
static bool shingle_sizes_ok(uint64_t n_bytes, uint64_t n_docs) {
    return n_bytes + n_docs < (1ull << 31) - 2;
}

oph_status shingle_workspace_size(uint64_t n_bytes, uint64_t n_docs, size_t *bytes) {
    if (!bytes || !shingle_sizes_ok(n_bytes, n_docs)) return OPH_EINVAL;
    *bytes = shingle_temp_bytes(n_bytes, n_docs);
    return OPH_OK;
}

oph_status shingle_text(const uint8_t *d_text, const uint64_t *d_doc_offsets, uint64_t n_docs, uint64_t n_bytes,
                        uint32_t w, uint64_t vocab_size, uint64_t seed, uint64_t *d_set_offsets, uint32_t *d_ids,
                        uint64_t ids_capacity, unsigned long long *d_n_ids, void *d_ws, size_t ws_bytes,
                        void *stream) {
    if (w == 0 || vocab_size == 0 || vocab_size > (1ull << 32) || !shingle_sizes_ok(n_bytes, n_docs))
        return OPH_EINVAL;
    if (!d_doc_offsets || !d_set_offsets || !d_n_ids || (n_bytes && !d_text) || (ids_capacity && !d_ids))
        return OPH_EINVAL;
    if (ws_bytes < shingle_temp_bytes(n_bytes, n_docs) || !d_ws) return OPH_ENOMEM;
    ShingleArgs a{};
    a.text = d_text;
    a.doc_offsets = d_doc_offsets;
    a.n_docs = n_docs;
    a.n_bytes = n_bytes;
    a.w = w;
    a.V = vocab_size;
    a.seed = seed;
    a.set_offsets = d_set_offsets;
    a.ids = d_ids;
    a.ids_cap = ids_capacity;
    a.n_ids = d_n_ids;
    return cuda_status(run_shingle(a, d_ws, ws_bytes, (cudaStream_t)stream));
}

oph_status oph_select_workspace_size(uint64_t n_in, size_t *bytes) {
    if (!bytes || n_in >= (1ull << 31)) return OPH_EINVAL;
    *bytes = select_temp_bytes(n_in);
    return OPH_OK;
}

oph_status topk_or_threshold_results(const oph_hit *d_in, uint64_t n_in, uint32_t mode, uint32_t topk,
                                     uint32_t k_bins, oph_hit *d_out, unsigned long long *d_n_out, void *d_ws,
                                     size_t ws_bytes, void *stream) {
    if ((n_in && (!d_in || !d_out)) || !d_n_out || mode > OPH_SELECT_TOPK || n_in >= (1ull << 31)) return OPH_EINVAL;
    if (mode == OPH_SELECT_TOPK && (k_bins == 0 || k_bins > 32768)) return OPH_EINVAL;
    if (ws_bytes < select_temp_bytes(n_in)) return OPH_ENOMEM;
    return cuda_status(run_select(d_in, n_in, mode, topk, k_bins, d_out, d_n_out, d_ws, ws_bytes, (cudaStream_t)stream));
}

// planner introspection for tests: per-level thresholds (acc, rej) and l0
oph_status oph_plan_thresholds(uint32_t method, uint32_t nlev, uint32_t kp, uint32_t a, uint32_t b, uint32_t t_num,
                               uint32_t t_den, double eps, uint64_t *acc, int64_t *rej, uint32_t *l0, uint64_t *weights) {
    if (method != OPH_METHOD_GOPH && method != OPH_METHOD_HOPH) return OPH_EINVAL;
    if (nlev == 0 || nlev > OPH_MAX_GROUPS || kp == 0 || t_den == 0 || t_num == 0 || t_num > t_den) return OPH_EINVAL;
    Plan P = make_plan(method, nlev, kp, a, b, t_num, t_den, eps);
    if (P.st != OPH_OK) return P.st;
    // 64-bit introspection: plans whose states exceed 64 bits (the 1:2 split of 2^32) report OPH_EOVERFLOW
    for (uint32_t l = 1; l < nlev; l++) {
        const LevelThr &T = P.thr[l - 1];
        if ((T.acc != kNeverAcc && T.acc >= (u128)UINT64_MAX) || T.rej > (i128)INT64_MAX) return OPH_EOVERFLOW;
        acc[l - 1] = T.acc == kNeverAcc ? UINT64_MAX : (uint64_t)T.acc;
        rej[l - 1] = (int64_t)T.rej;
    }
    for (uint32_t j = 0; j < nlev; j++) {
        if (P.c[j] > (u128)UINT64_MAX) return OPH_EOVERFLOW;
        weights[j] = (uint64_t)P.c[j];
    }
    *l0 = P.l0;
    return OPH_OK;
}

}  // extern "C"
