// K7 BITMAP: the collection scan as a value-indexed bitmap join (included by
// ophgpu_kernels.cu).
//
// The counts every method needs are N_mb(q, s) = #{b : F[b][s] == Q'[q][b]}
// over the bins of the groups compared.  For a block of up to 1024 queries:
//   * every bin value is a position p = start(b) + value in [0, |V|) (the
//     bins tile the universe: the floor rule of P:158 / S:38 for the flat
//     layout, the group ranges of P:466 for HOPH), so one table idx[p] of
//     |V| entries (|V| <= 2^23) maps a collection value to the row of the
//     queries holding that value in that bin (0 = none: row 0 is all zeros);
//   * row r is a 1024-bit mask of those queries (32 words, lane = word).
// A warp scores one set against the block: per bin it looks up the set's
// value, broadcasts the row index and every lane adds its word of the row to
// a bit-sliced counter of its 32 queries (carry-save adders, 16 bins per
// batch: ~2.6 LOP3 per lane per bin), i.e. 32 equality tests per lane-word
// instead of 32 ISETP + 32 IMAD per lane in the BRUTE scan.  The bit-sliced
// counts ARE the paper's states: GOPH's M_c (Alg. 1 line 9) and HOPH's
// T_l = S_l / 2^(L-1-l) = 2 T_(l-1) + M_l for the 1:1 weights c_j =
// 2^(L-1-j) (R21).  Level thresholds compiled by the planner are applied as
// bit-sliced comparisons with constants; the rare decided / candidate pairs
// are extracted bit by bit and emitted with the same records as every other
// strategy (bit-exact, R23).
// ---------------------------------------------------------------------------

constexpr uint32_t kBitQB = 1024;     // queries per block: 32 lanes x 32 bits
constexpr uint32_t kBitMaxBins = 1023;  // bins scanned: counts fit 10 bit slices
constexpr uint32_t kBitCS = 10;       // count slices: ones, twos, fours, eights, hi[6]
constexpr int kBitWarps = 8;          // warps per CTA = consecutive sets per CTA tile
constexpr uint32_t kBitMaxStages = 8; // staged CTA tiles in flight (ring of value buffers)
#ifndef OPHGPU_BIT_XRING
#define OPHGPU_BIT_XRING 1
#endif
constexpr bool kBitXRing = OPHGPU_BIT_XRING;  // HOPH scan: row indices via a shared ring (-D...=0: shuffles)

// bin b -> (first position, width) of its value range
__device__ __forceinline__ void bit_bin_range(const BitArgs &a, uint32_t b, uint32_t &start, uint32_t &width) {
    const uint32_t r = b / a.bins_per_range, i = b - r * a.bins_per_range;
    const RangeBins &R = a.ranges[r];
    const uint64_t s0 = (uint64_t)i * R.len / a.bins_per_range;
    const uint64_t s1 = (uint64_t)(i + 1) * R.len / a.bins_per_range;
    start = (uint32_t)(R.start + s0);
    width = (uint32_t)(s1 - s0);
}

// ---- per query block: the value -> row table and the rows
// claim: the first (bin, query) holding a value takes a fresh row (rows are zeroed by
// their claimer; row 0 is the shared all-zero row of "no query has this value")
__global__ void bit_claim_kernel(const __grid_constant__ BitArgs a) {
    const uint64_t n = (uint64_t)a.nscan * a.nqb;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t b = (uint32_t)(i / a.nqb), q = (uint32_t)(i % a.nqb);
        const uint32_t v = a.QT[(uint64_t)b * a.ldq + a.qb0 + q];
        uint32_t st, wd;
        bit_bin_range(a, b, st, wd);
        if (v >= wd) continue;  // the query-side empty bin (kQueryEmpty) matches nothing
        uint32_t *slot = a.idx + st + v;
        if (atomicCAS(slot, 0u, 0xFFFFFFFFu) == 0u) {
            const uint32_t r = atomicAdd(a.nrows, 1u) + 1u;  // row 0 stays the zero row
            uint4 *row = reinterpret_cast<uint4 *>(a.rows + (uint64_t)r * 32 * a.qw);
            for (uint32_t w = 0; w < 8 * a.qw; w++) row[w] = make_uint4(0, 0, 0, 0);
            atomicExch(slot, r);
        }
    }
}

__global__ void bit_fill_kernel(const __grid_constant__ BitArgs a) {
    const uint64_t n = (uint64_t)a.nscan * a.nqb;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t b = (uint32_t)(i / a.nqb), q = (uint32_t)(i % a.nqb);
        const uint32_t v = a.QT[(uint64_t)b * a.ldq + a.qb0 + q];
        uint32_t st, wd;
        bit_bin_range(a, b, st, wd);
        if (v >= wd) continue;
        const uint32_t r = a.idx[st + v];
        atomicOr(a.rows + (uint64_t)r * 32 * a.qw + (q >> 5), 1u << (q & 31u));
    }
}

// max over each word's 32 queries of the query's empty bins (the filter bound of the
// final verdict, see bit_final), and of its empty bins in every prefix [0, 32 c) (the
// full-OPH exit's bound, R32)
__global__ void bit_maxeq_kernel(const __grid_constant__ BitArgs a) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;  // qw CTAs of 1024 threads
    const bool in = q < a.nqb;
    const uint32_t qg = a.qb0 + q;
    uint32_t e = 0;
    if ((q & 31u) == 0) a.max_eq_pref[q >> 5] = 0u;
    for (uint32_t w = 0; w < a.nw; w++) {  // (warp-uniform trip count)
        if (in) e += popc_masked(__ldg(a.QEM + (uint64_t)qg * a.nw + w), 0u, 0, w, a.nbins_total);
        const uint32_t m = __reduce_max_sync(0xFFFFFFFFu, e);
        if ((q & 31u) == 0) a.max_eq_pref[(w + 1) * 64u + (q >> 5)] = m;
    }
    const uint32_t m = __reduce_max_sync(0xFFFFFFFFu, e);
    if ((q & 31u) == 0) a.max_eq[q >> 5] = m;
}

// ---- bit-sliced arithmetic (bit j of every slice word = query 32 lane + j)
// (h, l) = full adder of three words: l = a ^ b ^ c, h = majority
__device__ __forceinline__ void csa(uint32_t &h, uint32_t &l, uint32_t a, uint32_t b, uint32_t c) {
    const uint32_t u = a ^ b;
    h = (a & b) | (u & c);
    l = u ^ c;
}

// add 16 input words (one per bin) to the count: c[0..3] = ones, twos, fours, eights
// (the count mod 16, Harley-Seal), c[4..9] = count >> 4 (ripple add of the sixteens)
__device__ __forceinline__ void csa16(uint32_t (&c)[kBitCS], const uint32_t (&x)[16]) {
    uint32_t twosA, twosB, foursA, foursB, eightsA, eightsB, sixteens;
    csa(twosA, c[0], c[0], x[0], x[1]);
    csa(twosB, c[0], c[0], x[2], x[3]);
    csa(foursA, c[1], c[1], twosA, twosB);
    csa(twosA, c[0], c[0], x[4], x[5]);
    csa(twosB, c[0], c[0], x[6], x[7]);
    csa(foursB, c[1], c[1], twosA, twosB);
    csa(eightsA, c[2], c[2], foursA, foursB);
    csa(twosA, c[0], c[0], x[8], x[9]);
    csa(twosB, c[0], c[0], x[10], x[11]);
    csa(foursA, c[1], c[1], twosA, twosB);
    csa(twosA, c[0], c[0], x[12], x[13]);
    csa(twosB, c[0], c[0], x[14], x[15]);
    csa(foursB, c[1], c[1], twosA, twosB);
    csa(eightsB, c[2], c[2], foursA, foursB);
    csa(sixteens, c[3], c[3], eightsA, eightsB);
#pragma unroll
    for (int i = 4; i < (int)kBitCS; i++) {
        const uint32_t t = c[i] & sixteens;
        c[i] ^= sixteens;
        sixteens = t;
    }
}

// bits whose NS-slice number is >= A (A may differ per lane; A >= 2^NS: none)
template <int NS>
__device__ __forceinline__ uint32_t sliced_ge(const uint32_t *c, uint32_t A) {
    if (A >> NS) return 0u;
    uint32_t gt = 0u, eq = 0xFFFFFFFFu;
#pragma unroll
    for (int i = NS - 1; i >= 0; i--) {
        const uint32_t ai = 0u - ((A >> i) & 1u);
        gt |= eq & c[i] & ~ai;
        eq &= ~(c[i] ^ ai);
    }
    return gt | eq;
}

// the value of bit j of an NS-slice number
template <int NS>
__device__ __forceinline__ uint32_t sliced_get(const uint32_t *c, uint32_t j) {
    uint32_t v = 0;
#pragma unroll
    for (int i = 0; i < NS; i++) v |= ((c[i] >> j) & 1u) << i;
    return v;
}

// excluded bins of a pair among bins [b0, b1) (query-major masks QEM, set masks E)
__device__ __forceinline__ uint32_t bit_excl(const BitArgs &a, uint32_t qg, uint64_t s, uint32_t b0, uint32_t b1) {
    uint32_t ex = 0;
    for (uint32_t w = b0 / 32; w * 32 < b1; w++) {
        const uint32_t qm = __ldg(a.QEM + (uint64_t)qg * a.nw + w), sm = __ldg(a.E + (uint64_t)w * a.ld + s);
        uint32_t x = a.joint ? (qm & sm) : (qm | sm);
        const uint32_t lo = max(b0, 32 * w), hi = min(b1, 32 * w + 32);
        const uint32_t width = hi - lo;
        x &= (width == 32 ? 0xFFFFFFFFu : ((1u << width) - 1u)) << (lo - 32 * w);
        ex += __popc(x);
    }
    return ex;
}

// A count over the scanned bins (FULL: one level, the final verdict; GOPH: levels of k'
// bins with thresholds on M_c).
// The values of a CTA tile (8 consecutive sets) in the first npre bins: per bin row the
// tile's 32-B segment is copied with two 16-B cp.async (L1-bypassing) into
// vbuf[buffer][bin][8]; each issuing lane then arrives on the buffer's mbarrier when its
// copies have landed (cp.async.mbarrier.arrive.noinc; 32 arrivals per fill).  Issued by
// the 32 lanes of the last warp to finish the tile nstage tiles back (a ring of buffers; no
// CTA-wide barrier): one gather request per 16 B of the tile instead of one per set
// value per warp, and the latency hidden behind a whole tile's scan.
__device__ __forceinline__ void bit_tile_load(const BitArgs &a, uint64_t tile, uint32_t *dst, uint64_t *bar,
                                              uint32_t lane) {
    const uint64_t s0 = a.s_begin + tile * kBitWarps + 4u * (lane & 1u);
    for (uint32_t b = lane >> 1; b < a.npre; b += 16) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst + 8 * b + 4 * (lane & 1u))),
                     "l"(a.F + (uint64_t)b * a.ld + s0)
                     : "memory");
    }
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// termination histogram in shared memory (one global add per level per CTA at the end; a
// global add per warp and set serialises on the histogram words in L2)
__device__ __forceinline__ void shist_add(unsigned long long *s_hist, const unsigned long long *g, uint32_t level,
                                          uint32_t n) {
    if (!g) return;
    const uint32_t tot = __reduce_add_sync(0xFFFFFFFFu, n);
    if ((threadIdx.x & 31u) == 0 && tot) atomicAdd(s_hist + level, (unsigned long long)tot);
}
__device__ __forceinline__ void shist_flush(const unsigned long long *s_hist, unsigned long long *g) {
    if (!g) return;
    __syncthreads();
    if (threadIdx.x <= kMaxGroups && s_hist[threadIdx.x]) atomicAdd(g + threadIdx.x, s_hist[threadIdx.x]);
}

// Per-set software pipeline (full OPH, GOPH), blocks of 1,024 queries.
template <int MINB>
__global__ void __launch_bounds__(32 * kBitWarps, MINB) bit_scan_kernel(const __grid_constant__ BitArgs a) {
    __shared__ uint32_t s_start[kBitMaxBins + 1], s_width[kBitMaxBins + 1];
    __shared__ uint64_t s_full[kBitMaxStages];
    __shared__ unsigned long long s_hist[kMaxGroups + 1];
    __shared__ uint32_t s_done[kBitMaxStages];
    extern __shared__ __align__(128) uint32_t s_vals[];  // [2][npre][8]
    for (uint32_t b = threadIdx.x; b < a.nscan; b += blockDim.x) {
        uint32_t st, wd;
        bit_bin_range(a, b, st, wd);
        s_start[b] = st;
        s_width[b] = wd;
    }
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    // this lane's word of the block: queries qb0 + 32 lane + j
    const uint32_t qw0 = 32u * lane;
    const uint32_t qvalid = qw0 >= a.nqb ? 0u : (a.nqb - qw0 >= 32u ? 0xFFFFFFFFu : ((1u << (a.nqb - qw0)) - 1u));
    const uint32_t max_eq = a.max_eq[lane];
    const uint32_t *rows_lane = a.rows + lane;
    const uint32_t nlev_scan = a.method == kGoph ? a.nlev : 1u;
    const uint32_t bins_per_level = a.method == kGoph ? a.kp : a.nscan;
    // (a.n_sets - s_begin and ld are multiples of 8 sets / 32 B: the tiles' 32-B copies are
    // aligned and in bounds; sets past n_sets are never scored)
    const uint64_t ntiles = (a.n_sets - a.s_begin + kBitWarps - 1) / kBitWarps;
    const uint32_t vstride = a.npre * 8u;  // words per buffer
    if (threadIdx.x <= kMaxGroups) s_hist[threadIdx.x] = 0ull;
    if (threadIdx.x == 0) {
        for (uint32_t i = 0; i < a.nstage; i++) {
            mbar_init(&s_full[i], 32);  // the 32 lanes of the filling warp
            s_done[i] = 0u;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 0) {
        for (uint32_t i = 0; i < a.nstage; i++) {
            const uint64_t t = blockIdx.x + (uint64_t)i * gridDim.x;
            if (t < ntiles) bit_tile_load(a, t, s_vals + i * vstride, &s_full[i], lane);
        }
    }

    uint32_t it = 0;  // this CTA's tile counter
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, it++) {
        const uint32_t bi = it % a.nstage;
        const uint64_t s = a.s_begin + tile * kBitWarps + warp;
        const uint32_t *v_cur = s_vals + bi * vstride + warp;  // value of bin b: v_cur[8 b]
        mbar_wait(&s_full[bi], (it / a.nstage) & 1u);
        // the tile is processed; the last warp done with this buffer refills it with tile + nstage
        auto release = [&]() {
            __syncwarp();
            uint32_t last = 0;
            if (lane == 0) {
                __threadfence_block();
                last = atomicAdd(&s_done[bi], 1u) == kBitWarps - 1;
                if (last) s_done[bi] = 0u;
            }
            last = __shfl_sync(0xFFFFFFFFu, last, 0);
            const uint64_t tn = tile + (uint64_t)a.nstage * gridDim.x;
            if (last && tn < ntiles) bit_tile_load(a, tn, s_vals + bi * vstride, &s_full[bi], lane);
        };
        if (s >= a.n_sets) {  // warp-uniform: a tail tile's missing set
            release();
            continue;
        }
        uint32_t c[kBitCS];
#pragma unroll
        for (int i = 0; i < (int)kBitCS; i++) c[i] = 0u;
        uint32_t alive = qvalid;

        // The bins are scanned in batches of 16 (GOPH levels are whole batches: k' is
        // a multiple of 16; full OPH's last batch may be partial).  Per batch: lanes 0-15
        // take the set's value of bins b0 + lane (shared memory) and look up its row (r);
        // rows are then broadcast by shuffle and every lane loads its word (x).  Software
        // pipeline: the row words of batch g+1 and the row indices of g+2 and g+3 are in
        // flight while batch g is counted.
        const uint32_t nbt = (a.nscan + 15u) / 16u;
        const uint32_t bpl = bins_per_level / 16u;  // batches per level (full OPH: unused)
        auto ilook = [&](uint32_t g) -> uint32_t {
            const uint32_t b = 16u * g + lane;
            uint32_t r = 0u;
            if (lane < 16u && b < a.nscan) {
                // bins past the staged prefix (GOPH levels most sets never reach): direct
                const uint32_t v = b < a.npre ? v_cur[8 * b] : __ldg(a.F + (uint64_t)b * a.ld + s);
                if (v < s_width[b]) r = __ldg(a.idx + s_start[b] + v);
            }
            return r;
        };
        auto rload = [&](uint32_t r, uint32_t (&x)[16]) {
#pragma unroll
            for (int u = 0; u < 16; u++) {
                const uint32_t ru = __shfl_sync(0xFFFFFFFFu, r, u);
                x[u] = __ldg(rows_lane + (uint64_t)ru * 32);  // ru = 0 (no row, or past the scan): zero row
            }
        };
        uint32_t x[16], rA, rB;
        {
            const uint32_t r0 = ilook(0);
            rA = ilook(1);
            rB = ilook(2);
            rload(r0, x);
        }
        uint32_t l = 1, jj = 0;  // level of batch g, batch index inside the level
        // one batch: count xc (batch g) while xn (g + 1), r1 (g + 2), v3 (g + 3) load; the two
        // row buffers alternate (a copy between them would wait for the loads in flight)
        // returns true when the set is done
        auto step = [&](uint32_t g, uint32_t (&xc)[16], uint32_t (&xn)[16]) -> bool {
            rload(rA, xn);               // past the scan: rA = 0, the zero row
            rA = rB;
            rB = ilook(g + 3);
            csa16(c, xc);
            const bool level_end = bins_per_level == a.nscan ? g + 1 == nbt : jj + 1 == bpl;
            if (!level_end) {
                jj++;
                return false;
            }
            // ---- decisions at the end of level l
            const bool last = l == nlev_scan;
            uint32_t acc = 0u, dec = 0u;
            if (!last && a.thr_on[l - 1]) {
                const uint32_t A = a.acc_cnt[l - 1];
                const int32_t R = a.rej_cnt[l - 1];
                acc = sliced_ge<kBitCS>(c, A);
                dec = acc | (R >= 0 ? ~sliced_ge<kBitCS>(c, (uint32_t)R + 1u) : 0u);
                acc &= alive;
                dec &= alive;
                shist_add(s_hist, a.out.hist, l, __popc(dec));
                uint32_t want = a.out.dense ? dec : acc;
                while (__any_sync(0xFFFFFFFFu, want != 0u)) {
                    const bool has = want != 0u;
                    const uint32_t j = has ? __ffs(want) - 1 : 0u;
                    want &= want - 1u;
                    const uint32_t qg = a.qb0 + qw0 + j;
                    uint32_t nmb = 0, ex = 0;
                    if (has) {
                        nmb = sliced_get<kBitCS>(c, j);
                        ex = bit_excl(a, qg, s, 0, l * a.kp);
                    }
                    emit(a.out, has, qg, s, nmb, ex, l, (acc >> j) & 1u, OPH_FLAG_EARLY, -1.0f);
                }
                alive &= ~dec;
            }
            if (!last) {
                if (!__any_sync(0xFFFFFFFFu, alive != 0u)) return true;  // every pair of this set is decided
                l++;
                jj = 0;
                return false;
            }
            // ---- the final verdict of every pair still alive
            shist_add(s_hist, a.out.hist, a.level_final, __popc(alive));
            {
                // full-OPH verdict (Eq. 6): den = k - N_excl >= k - (max_q |Eq| + |Es|) (EitherEmpty)
                // or k - min(max_q |Eq|, |Es|) (JointEmpty), so a pair can only be Similar if
                // N_mb >= ceil(t_num den_min / t_den): the candidates, verified exactly
                const uint32_t es_w = lane < a.nw ? __ldg(a.E + (uint64_t)lane * a.ld + s) : 0u;
                const uint32_t es = __reduce_add_sync(0xFFFFFFFFu, popc_masked(0u, es_w, 0, lane, a.nbins_total));
                const uint32_t k = a.nbins_total;
                uint32_t den_min = a.joint ? k - min(max_eq, es) : k - min(k, max_eq + es);
                const uint32_t theta =
                    a.out.dense ? 0u : (uint32_t)(((uint64_t)a.t_num * den_min + a.t_den - 1) / a.t_den);
                uint32_t want = sliced_ge<kBitCS>(c, theta) & alive;
                while (__any_sync(0xFFFFFFFFu, want != 0u)) {
                    const bool has = want != 0u;
                    const uint32_t j = has ? __ffs(want) - 1 : 0u;
                    want &= want - 1u;
                    const uint32_t qg = a.qb0 + qw0 + j;
                    uint32_t ex = 0;
                    for (uint32_t w = 0; w < a.nw; w++) {
                        const uint32_t sw = __shfl_sync(0xFFFFFFFFu, es_w, w);
                        if (has) ex += popc_masked(__ldg(a.QEM + (uint64_t)qg * a.nw + w), sw, a.joint, w, k);
                    }
                    const uint32_t nmb = sliced_get<kBitCS>(c, j);
                    const uint32_t den = k - ex;
                    const bool undef = den == 0;
                    const uint32_t verdict = !undef && (uint64_t)nmb * a.t_den >= (uint64_t)a.t_num * den;
                    emit(a.out, has, qg, s, nmb, ex, a.level_final, verdict, undef ? OPH_FLAG_UNDEFINED : 0u,
                         undef ? -1.0f : (float)nmb / (float)den);
                }
            }
            alive = 0u;
            return true;
        };
        uint32_t xb[16];
        for (uint32_t g = 0; g < nbt; g += 2) {
            if (step(g, x, xb)) break;
            if (g + 1 < nbt && step(g + 1, xb, x)) break;
        }
        release();
    }
    shist_flush(s_hist, a.out.hist);
}

// Full OPH / GOPH with QW query words per lane (QW = 2: blocks of 2,048 queries, rows of
// 256 B read as one 8-B load per lane): per (set, bin) one table lookup and one shuffle /
// address for 2,048 queries instead of 1,024 -- the lookups were a third of the L1
// requests and the shuffles / addresses a third of the issued instructions.
template <int QW, int MINB, bool ALLSTAGED>
__global__ void __launch_bounds__(32 * kBitWarps, MINB) bit_scan_q_kernel(const __grid_constant__ BitArgs a) {
    __shared__ uint32_t s_start[kBitMaxBins + 1], s_width[kBitMaxBins + 1];
    __shared__ uint64_t s_full[kBitMaxStages];
    __shared__ unsigned long long s_hist[kMaxGroups + 1];
    __shared__ uint32_t s_done[kBitMaxStages];
    extern __shared__ __align__(128) uint32_t s_vals[];  // [nstage][npre][8]
    for (uint32_t b = threadIdx.x; b < a.nscan; b += blockDim.x) {
        uint32_t st, wd;
        bit_bin_range(a, b, st, wd);
        s_start[b] = st;
        s_width[b] = wd;
    }
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    // this lane's words of the block: word w holds queries qb0 + 32 (QW lane + w) + j
    uint32_t qw0[QW], qvalid[QW], max_eq[QW];
#pragma unroll
    for (int w = 0; w < QW; w++) {
        qw0[w] = 32u * (QW * lane + w);
        qvalid[w] = qw0[w] >= a.nqb ? 0u : (a.nqb - qw0[w] >= 32u ? 0xFFFFFFFFu : ((1u << (a.nqb - qw0[w])) - 1u));
        max_eq[w] = a.max_eq[QW * lane + w];
    }
    const uint32_t *rows_lane = a.rows + QW * lane;
    const uint32_t nlev_scan = a.method == kGoph ? a.nlev : 1u;
    const uint32_t bins_per_level = a.method == kGoph ? a.kp : a.nscan;
    const uint64_t ntiles = (a.n_sets - a.s_begin + kBitWarps - 1) / kBitWarps;
    const uint32_t vstride = a.npre * 8u;  // words per buffer
    if (threadIdx.x <= kMaxGroups) s_hist[threadIdx.x] = 0ull;
    if (threadIdx.x == 0) {
        for (uint32_t i = 0; i < a.nstage; i++) {
            mbar_init(&s_full[i], 32);  // the 32 lanes of the filling warp
            s_done[i] = 0u;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 0) {
        for (uint32_t i = 0; i < a.nstage; i++) {
            const uint64_t t = blockIdx.x + (uint64_t)i * gridDim.x;
            if (t < ntiles) bit_tile_load(a, t, s_vals + i * vstride, &s_full[i], lane);
        }
    }

    uint32_t it = 0;  // this CTA's tile counter
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, it++) {
        const uint32_t bi = it % a.nstage;
        const uint64_t s = a.s_begin + tile * kBitWarps + warp;
        const uint32_t *v_cur = s_vals + bi * vstride + warp;  // value of bin b: v_cur[8 b]
        mbar_wait(&s_full[bi], (it / a.nstage) & 1u);
        auto release = [&]() {
            __syncwarp();
            uint32_t last = 0;
            if (lane == 0) {
                __threadfence_block();
                last = atomicAdd(&s_done[bi], 1u) == kBitWarps - 1;
                if (last) s_done[bi] = 0u;
            }
            last = __shfl_sync(0xFFFFFFFFu, last, 0);
            const uint64_t tn = tile + (uint64_t)a.nstage * gridDim.x;
            if (last && tn < ntiles) bit_tile_load(a, tn, s_vals + bi * vstride, &s_full[bi], lane);
        };
        if (s >= a.n_sets) {  // warp-uniform: a tail tile's missing set
            release();
            continue;
        }
        uint32_t c[QW][kBitCS];
        uint32_t alive[QW];
#pragma unroll
        for (int w = 0; w < QW; w++) {
            alive[w] = qvalid[w];
#pragma unroll
            for (int i = 0; i < (int)kBitCS; i++) c[w][i] = 0u;
        }
        const uint32_t nbt = (a.nscan + 15u) / 16u;
        const uint32_t bpl = bins_per_level / 16u;
        // (ALLSTAGED: every scanned bin is staged -- full OPH -- so no direct-load path; the
        // lookup is branch-free: lanes past the batch read a staged slot they do not use)
        auto ilook = [&](uint32_t g) -> uint32_t {
            const uint32_t b = 16u * g + lane;
            if (ALLSTAGED) {
                const uint32_t bc = min(b, a.nscan - 1u);
                const uint32_t v = v_cur[8 * bc];
                const bool ok = lane < 16u && b < a.nscan && v < s_width[bc];
                return ok ? __ldg(a.idx + s_start[bc] + v) : 0u;
            }
            uint32_t r = 0u;
            if (lane < 16u && b < a.nscan) {
                const uint32_t v = b < a.npre ? v_cur[8 * b] : __ldg(a.F + (uint64_t)b * a.ld + s);
                if (v < s_width[b]) r = __ldg(a.idx + s_start[b] + v);
            }
            return r;
        };
        auto rload = [&](uint32_t r, uint32_t (&x)[QW][16]) {
#pragma unroll
            for (int u = 0; u < 16; u++) {
                const uint32_t ru = __shfl_sync(0xFFFFFFFFu, r, u);
                if (QW == 2) {
                    const uint2 y = __ldg(reinterpret_cast<const uint2 *>(rows_lane + (uint64_t)ru * 64));
                    x[0][u] = y.x;
                    x[QW - 1][u] = y.y;
                } else {
                    x[0][u] = __ldg(rows_lane + (uint64_t)ru * 32);
                }
            }
        };
        uint32_t x[QW][16], xb[QW][16], rA, rB;
        {
            const uint32_t r0 = ilook(0);
            rA = ilook(1);
            rB = ilook(2);
            rload(r0, x);
        }
        uint32_t l = 1, jj = 0;
        auto step = [&](uint32_t g, uint32_t (&xc)[QW][16], uint32_t (&xn)[QW][16]) -> bool {
            rload(rA, xn);
            rA = rB;
            rB = ilook(g + 3);
#pragma unroll
            for (int w = 0; w < QW; w++) csa16(c[w], xc[w]);
            const bool level_end = bins_per_level == a.nscan ? g + 1 == nbt : jj + 1 == bpl;
            if (!level_end) {
                jj++;
                return false;
            }
            const bool last = l == nlev_scan;
            if (!last && a.thr_on[l - 1]) {
                const uint32_t A = a.acc_cnt[l - 1];
                const int32_t R = a.rej_cnt[l - 1];
#pragma unroll
                for (int w = 0; w < QW; w++) {
                    uint32_t acc = sliced_ge<kBitCS>(c[w], A);
                    uint32_t dec = acc | (R >= 0 ? ~sliced_ge<kBitCS>(c[w], (uint32_t)R + 1u) : 0u);
                    acc &= alive[w];
                    dec &= alive[w];
                    shist_add(s_hist, a.out.hist, l, __popc(dec));
                    uint32_t want = a.out.dense ? dec : acc;
                    while (__any_sync(0xFFFFFFFFu, want != 0u)) {
                        const bool has = want != 0u;
                        const uint32_t j = has ? __ffs(want) - 1 : 0u;
                        want &= want - 1u;
                        const uint32_t qg = a.qb0 + qw0[w] + j;
                        uint32_t nmb = 0, ex = 0;
                        if (has) {
                            nmb = sliced_get<kBitCS>(c[w], j);
                            ex = bit_excl(a, qg, s, 0, l * a.kp);
                        }
                        emit(a.out, has, qg, s, nmb, ex, l, (acc >> j) & 1u, OPH_FLAG_EARLY, -1.0f);
                    }
                    alive[w] &= ~dec;
                }
            }
            if (!last) {
                uint32_t any = 0u;
#pragma unroll
                for (int w = 0; w < QW; w++) any |= alive[w];
                if (!__any_sync(0xFFFFFFFFu, any != 0u)) return true;  // every pair of this set is decided
                l++;
                jj = 0;
                return false;
            }
            // ---- the full-OPH verdict of every pair still alive (Eq. 6): den = k - N_excl >=
            // k - (max_q |Eq| + |Es|) (EitherEmpty) or k - min(max_q |Eq|, |Es|) (JointEmpty), so
            // a pair can only be Similar if N_mb >= ceil(t_num den_min / t_den): the candidates,
            // verified exactly
            const uint32_t es_w = lane < a.nw ? __ldg(a.E + (uint64_t)lane * a.ld + s) : 0u;
            const uint32_t es = __reduce_add_sync(0xFFFFFFFFu, popc_masked(0u, es_w, 0, lane, a.nbins_total));
            const uint32_t k = a.nbins_total;
#pragma unroll
            for (int w = 0; w < QW; w++) {
                shist_add(s_hist, a.out.hist, a.level_final, __popc(alive[w]));
                const uint32_t den_min = a.joint ? k - min(max_eq[w], es) : k - min(k, max_eq[w] + es);
                const uint32_t theta =
                    a.out.dense ? 0u : (uint32_t)(((uint64_t)a.t_num * den_min + a.t_den - 1) / a.t_den);
                uint32_t want = sliced_ge<kBitCS>(c[w], theta) & alive[w];
                while (__any_sync(0xFFFFFFFFu, want != 0u)) {
                    const bool has = want != 0u;
                    const uint32_t j = has ? __ffs(want) - 1 : 0u;
                    want &= want - 1u;
                    const uint32_t qg = a.qb0 + qw0[w] + j;
                    uint32_t ex = 0;
                    for (uint32_t ww = 0; ww < a.nw; ww++) {
                        const uint32_t sw = __shfl_sync(0xFFFFFFFFu, es_w, ww);
                        if (has) ex += popc_masked(__ldg(a.QEM + (uint64_t)qg * a.nw + ww), sw, a.joint, ww, k);
                    }
                    const uint32_t nmb = sliced_get<kBitCS>(c[w], j);
                    const uint32_t den = k - ex;
                    const bool undef = den == 0;
                    const uint32_t verdict = !undef && (uint64_t)nmb * a.t_den >= (uint64_t)a.t_num * den;
                    emit(a.out, has, qg, s, nmb, ex, a.level_final, verdict, undef ? OPH_FLAG_UNDEFINED : 0u,
                         undef ? -1.0f : (float)nmb / (float)den);
                }
                alive[w] = 0u;
            }
            return true;
        };
        for (uint32_t g = 0; g < nbt; g += 2) {
            if (step(g, x, xb)) break;
            if (g + 1 < nbt && step(g + 1, xb, x)) break;
        }
        release();
    }
    shist_flush(s_hist, a.out.hist);
}

// HOPH (1:1): group 1 by the bitmap join in blocks of 2,048 queries (two words per lane) with
// one software pipeline across the warp's sets (items = the two batches of group 1 of its
// sets; the staged tile buffers are released by the lookup stage) -- a set's bitmap work is
// only 2 batches, so a per-set pipeline fill would dominate; then, for the few pairs group 1
// leaves undecided, the later groups one pair at a time by the whole warp (lane = bin:
// ballot counts, exact 128-bit state S_l = sum c_j M_j against the planner's thresholds, the
// HOPH estimator after group L), as level_walk_kernel.
__device__ __forceinline__ void bit_walk_pair(const BitArgs &a, uint32_t qg, uint64_t s, uint32_t m1, uint32_t lane) {
    const bool in_grp = lane < a.kp;
    const uint32_t *qp = a.QM + (uint64_t)qg * a.nb + lane;
    const uint32_t *fp = a.F + (uint64_t)lane * a.ld + s;
    u128_t st = a.c[0] * m1;
    uint32_t nmb = m1;
    for (uint32_t l = 2; l <= a.nlev; l++) {
        const uint32_t g = l - 1;
        const uint32_t qv = in_grp ? __ldg(qp + (uint64_t)g * a.kp) : 0u;
        const uint32_t sv = in_grp ? __ldg(fp + (uint64_t)g * a.kp * a.ld) : 1u;
        const uint32_t M = __popc(__ballot_sync(0xFFFFFFFFu, qv == sv));
        nmb += M;
        st += a.c[g] * M;
        if (l == a.nlev) {
            uint32_t nmb_out = 0, ex_tot = 0, verdict = 0, flags = 0;
            float est = -1.0f;
            u128_t num = 0, csum = 0;
            for (uint32_t gg = 0; gg < a.nlev; gg++) {
                const uint32_t q2 = in_grp ? __ldg(qp + (uint64_t)gg * a.kp) : 0u;
                const uint32_t s2 = in_grp ? __ldg(fp + (uint64_t)gg * a.kp * a.ld) : 1u;
                const uint32_t m = __popc(__ballot_sync(0xFFFFFFFFu, q2 == s2));
                const uint32_t ex = bit_excl(a, qg, s, gg * a.kp, (gg + 1) * a.kp);
                nmb_out += m;
                ex_tot += ex;
                const uint32_t d = a.kp - ex;
                if (d == 0) continue;
                num += a.c[gg] * m * (a.lam / d);
                csum += a.c[gg];
            }
            if (csum == 0) {
                flags = OPH_FLAG_UNDEFINED;
            } else {
                verdict = num * a.t_den >= (u128_t)a.t_num * a.lam * csum;
                est = (float)((double)num / ((double)a.lam * (double)csum));
            }
            if (lane == 0) {
                emit_one(a.out, qg, (uint32_t)s, nmb_out, ex_tot, a.nlev, verdict, flags, est);
                if (a.out.hist) atomicAdd(a.out.hist + a.nlev, 1ull);
            }
            return;
        }
        const bool acc = st >= a.acc128[l - 1];
        const bool rej = !acc && (i128_t)st <= a.rej128[l - 1];
        if (acc || rej) {
            if (a.out.dense || acc) {
                const uint32_t ex = bit_excl(a, qg, s, 0, l * a.kp);
                if (lane == 0) emit_one(a.out, qg, (uint32_t)s, nmb, ex, l, acc ? 1u : 0u, OPH_FLAG_EARLY, -1.0f);
            }
            if (lane == 0 && a.out.hist) atomicAdd(a.out.hist + l, 1ull);
            return;
        }
    }
}

template <int QW, int MINB>
__global__ void __launch_bounds__(32 * kBitWarps, MINB) bit_scan_x_kernel(const __grid_constant__ BitArgs a) {
    __shared__ uint32_t s_start[kBitMaxBins + 1], s_width[kBitMaxBins + 1];
    __shared__ uint64_t s_full[kBitMaxStages];
    __shared__ uint32_t s_done[kBitMaxStages];
    __shared__ __align__(16) uint32_t s_xring[kBitWarps][2][16];  // row indices parked for broadcast
    extern __shared__ __align__(128) uint32_t s_vals[];  // [nstage][npre][8]
    for (uint32_t b = threadIdx.x; b < a.npre; b += blockDim.x) {
        uint32_t st, wd;
        bit_bin_range(a, b, st, wd);
        s_start[b] = st;
        s_width[b] = wd;
    }
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    uint32_t qw0[QW], qvalid[QW];
#pragma unroll
    for (int w = 0; w < QW; w++) {
        qw0[w] = 32u * (QW * lane + w);
        qvalid[w] = qw0[w] >= a.nqb ? 0u : (a.nqb - qw0[w] >= 32u ? 0xFFFFFFFFu : ((1u << (a.nqb - qw0[w])) - 1u));
    }
    const uint32_t *rows_lane = a.rows + QW * lane;
    const uint64_t ntiles = (a.n_sets - a.s_begin + kBitWarps - 1) / kBitWarps;
    const uint32_t vstride = a.npre * 8u;  // words per buffer
    if (threadIdx.x == 0) {
        for (uint32_t i = 0; i < a.nstage; i++) {
            mbar_init(&s_full[i], 32);  // the 32 lanes of the filling warp
            s_done[i] = 0u;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 0) {
        for (uint32_t i = 0; i < a.nstage; i++) {
            const uint64_t t = blockIdx.x + (uint64_t)i * gridDim.x;
            if (t < ntiles) bit_tile_load(a, t, s_vals + i * vstride, &s_full[i], lane);
        }
    }
    const uint32_t nbs = (a.npre + 15u) / 16u;  // batches of group 1 (the staged prefix)
    const uint64_t n_it = (uint64_t)blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const uint64_t nitems = n_it * nbs;

    // ---- stage A: row indices of the next item; releases a tile after its last batch
    uint64_t tiA = 0;
    uint32_t bjA = 0, slotA = 0, phaseA = 0;
    auto stageA = [&]() -> uint32_t {
        uint32_t r = 0u;
        if (tiA >= n_it) return r;
        if (bjA == 0) mbar_wait(&s_full[slotA], phaseA);
        const uint32_t b = 16u * bjA + lane;
        const uint32_t bc = min(b, a.npre - 1u);
        const uint32_t v = s_vals[slotA * vstride + 8u * bc + warp];
        if (lane < 16u && b < a.npre && v < s_width[bc]) r = __ldg(a.idx + s_start[bc] + v);
        if (++bjA == nbs) {
            __syncwarp();
            uint32_t last = 0;
            if (lane == 0) {
                __threadfence_block();
                last = atomicAdd(&s_done[slotA], 1u) == kBitWarps - 1;
                if (last) s_done[slotA] = 0u;
            }
            last = __shfl_sync(0xFFFFFFFFu, last, 0);
            const uint64_t tn = (uint64_t)blockIdx.x + (tiA + a.nstage) * gridDim.x;
            if (last && tn < ntiles) bit_tile_load(a, tn, s_vals + slotA * vstride, &s_full[slotA], lane);
            bjA = 0;
            tiA++;
            if (++slotA == a.nstage) {
                slotA = 0;
                phaseA ^= 1u;
            }
        }
        return r;
    };
    // the 16 row indices of an item (lanes 0-15) reach every lane through the warp's shared
    // ring (one store, 4 broadcast 16-B loads) instead of 16 shuffles (bit_pipe_kernel's way)
    uint32_t xq = 0;
    auto rload = [&](uint32_t r, uint32_t (&x)[QW][16]) {
        uint32_t *rq = &s_xring[threadIdx.x >> 5][xq][0];
        xq ^= 1u;
        if (kBitXRing) {
            if ((threadIdx.x & 31u) < 16u) rq[threadIdx.x & 31u] = r;
            __syncwarp();
        }
        uint4 o = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int u = 0; u < 16; u++) {
            if (kBitXRing && (u & 3) == 0) o = reinterpret_cast<const uint4 *>(rq)[u >> 2];
            const uint32_t ru =
                kBitXRing ? ((u & 3) == 0 ? o.x : (u & 3) == 1 ? o.y : (u & 3) == 2 ? o.z : o.w)
                          : __shfl_sync(0xFFFFFFFFu, r, u);
            if (QW == 2) {
                const uint2 y = __ldg(reinterpret_cast<const uint2 *>(rows_lane + (uint64_t)ru * 64));
                x[0][u] = y.x;
                x[QW - 1][u] = y.y;
            } else {
                x[0][u] = __ldg(rows_lane + (uint64_t)ru * 32);
            }
        }
    };

    // ---- stage C: count item (tiC, bjC); after group 1, decide and walk the undecided pairs
    // (h1: this lane's pairs decided at level 1 -- a global atomic per warp and set on the one
    // histogram word serialised in L2: 4·10^6 same-address adds per image-like call)
    unsigned long long h1 = 0;
    uint64_t tiC = 0;
    uint32_t bjC = 0;
    uint32_t c[QW][kBitCS];
    auto stageC = [&](const uint32_t (&xc)[QW][16]) {
        if (bjC == 0) {
#pragma unroll
            for (int w = 0; w < QW; w++)
#pragma unroll
                for (int i = 0; i < (int)kBitCS; i++) c[w][i] = 0u;
        }
#pragma unroll
        for (int w = 0; w < QW; w++) csa16(c[w], xc[w]);
        if (++bjC < nbs) return;
        bjC = 0;
        const uint64_t s = a.s_begin + ((uint64_t)blockIdx.x + tiC * gridDim.x) * kBitWarps + warp;
        tiC++;
        if (s >= a.n_sets) return;  // warp-uniform: a tail tile's missing set
        // ---- group 1 decided on T_1 = M_1 (6 slices; S_1 = c_1 M_1)
        const uint32_t A = a.acc_cnt[0];
        const int32_t R = a.rej_cnt[0];
#pragma unroll
        for (int w = 0; w < QW; w++) {
            uint32_t acc = sliced_ge<6>(c[w], A) & qvalid[w];
            uint32_t dec = (acc | (R >= 0 ? ~sliced_ge<6>(c[w], (uint32_t)R + 1u) : 0u)) & qvalid[w];
            h1 += __popc(dec);  // (per lane; one global add per warp at the end, not per set)
            uint32_t want = a.out.dense ? dec : acc;
            while (__any_sync(0xFFFFFFFFu, want != 0u)) {
                const bool has = want != 0u;
                const uint32_t j = has ? __ffs(want) - 1 : 0u;
                want &= want - 1u;
                const uint32_t qg = a.qb0 + qw0[w] + j;
                uint32_t nmb = 0, ex = 0;
                if (has) {
                    nmb = sliced_get<6>(c[w], j);
                    ex = bit_excl(a, qg, s, 0, a.kp);
                }
                emit(a.out, has, qg, s, nmb, ex, 1, (acc >> j) & 1u, OPH_FLAG_EARLY, -1.0f);
            }
            // the undecided pairs: the later groups pair by pair, the whole warp per pair
            uint32_t alive = qvalid[w] & ~dec;
            while (__any_sync(0xFFFFFFFFu, alive != 0u)) {
                const uint32_t src = __ffs(__ballot_sync(0xFFFFFFFFu, alive != 0u)) - 1;
                const uint32_t mine = alive != 0u ? __ffs(alive) - 1 : 0u;
                const uint32_t j = __shfl_sync(0xFFFFFFFFu, mine, src);
                const uint32_t m1 = __shfl_sync(0xFFFFFFFFu, sliced_get<6>(c[w], mine), src);
                if (lane == src) alive &= alive - 1u;
                bit_walk_pair(a, a.qb0 + 32u * (QW * src + w) + j, s, m1, lane);
            }
        }
    };

    if (nitems) {
        uint32_t x[QW][16], xb[QW][16], rA, rB;
        {
            const uint32_t r0 = stageA();
            rA = stageA();
            rB = stageA();
            rload(r0, x);
        }
        auto step = [&](uint64_t g, uint32_t (&xc)[QW][16], uint32_t (&xn)[QW][16]) {
            if (g + 1 < nitems) rload(rA, xn);
            rA = rB;
            rB = stageA();
            stageC(xc);
        };
        for (uint64_t g = 0; g < nitems; g += 2) {
            step(g, x, xb);
            if (g + 1 < nitems) step(g + 1, xb, x);
        }
    }
    if (a.out.hist) {
        const unsigned long long tot = __reduce_add_sync(0xFFFFFFFFu, (uint32_t)h1);  // < 2^32 per warp
        if (lane == 0 && tot) atomicAdd(a.out.hist + 1, tot);
    }
}

// GOPH's pairs left after the bitmap part (levels 1 .. level_b): the later levels one pair at
// a time by the whole warp (lane = bin of the level; ballot counts), Algorithm 1's thresholds
// on the running count, the full-OPH verdict (Eq. 6) after level L -- as level_walk_kernel.
__device__ __forceinline__ uint32_t bit_excl_warp(const BitArgs &a, uint32_t qg, uint64_t s, uint32_t nbins,
                                                  uint32_t lane) {
    uint32_t ex = 0;
    for (uint32_t w = lane; w * 32 < nbins; w += 32)
        ex += popc_masked(__ldg(a.QEM + (uint64_t)qg * a.nw + w), __ldg(a.E + (uint64_t)w * a.ld + s), a.joint, w,
                          nbins);
    return __reduce_add_sync(0xFFFFFFFFu, ex);
}

__device__ void bit_walk_goph(const BitArgs &a, uint32_t qg, uint64_t s, uint32_t nmb, uint32_t lane,
                              unsigned long long *hist) {
    const uint32_t *qrow = a.QM + (uint64_t)qg * a.nb;
    for (uint32_t l = a.level_b + 1; l <= a.nlev; l++) {
        uint32_t M = 0;
        for (uint32_t b0 = (l - 1) * a.kp; b0 < l * a.kp; b0 += 32) {
            const uint32_t b = b0 + lane;
            const bool in = b < l * a.kp;
            const uint32_t qv = in ? __ldg(qrow + b) : 0u;
            const uint32_t sv = in ? __ldg(a.F + (uint64_t)b * a.ld + s) : 1u;  // never equal when masked
            M += __popc(__ballot_sync(0xFFFFFFFFu, qv == sv));
        }
        nmb += M;
        if (l == a.nlev) {
            const uint32_t ex = bit_excl_warp(a, qg, s, a.nbins_total, lane);
            const uint32_t den = a.nbins_total - ex;
            const bool undef = den == 0;
            const uint32_t verdict = !undef && (uint64_t)nmb * a.t_den >= (uint64_t)a.t_num * den;
            if (lane == 0) {
                emit_one(a.out, qg, (uint32_t)s, nmb, ex, a.nlev, verdict, undef ? OPH_FLAG_UNDEFINED : 0u,
                         undef ? -1.0f : (float)nmb / (float)den);
                if (hist) atomicAdd(hist + a.nlev, 1ull);
            }
            return;
        }
        if (!a.thr_on[l - 1]) continue;
        const bool acc = nmb >= a.acc_cnt[l - 1];
        const bool rej = !acc && a.rej_cnt[l - 1] >= 0 && nmb <= (uint32_t)a.rej_cnt[l - 1];
        if (acc || rej) {
            if (a.out.dense || acc) {
                const uint32_t ex = bit_excl_warp(a, qg, s, l * a.kp, lane);
                if (lane == 0) emit_one(a.out, qg, (uint32_t)s, nmb, ex, l, acc ? 1u : 0u, OPH_FLAG_EARLY, -1.0f);
            }
            if (lane == 0 && hist) atomicAdd(hist + l, 1ull);
            return;
        }
    }
}

// Full OPH (Eq. 6), and GOPH (Algorithm 1) over its first level_b levels, with 2,048-query
// rows and one software pipeline across the warp's sets (nscan / 16 batches per set, an even
// number >= 4), four stages per batch:
//   A  look the set's 16 values up (value -> row index), 3 batches ahead
//   B  park the 16 row indices in the warp's shared ring, 2 batches ahead (the lookups have
//      landed by then: no stall on them)
//   C  read the ring back (4 broadcast 16-B loads instead of 16 shuffles) and issue the 16
//      row loads (one 8-B load per lane), 1 batch ahead
//   D  count (csa16 on both words); GOPH: at each level end Algorithm 1's thresholds on the
//      bit-sliced counts; after a set's last batch the final verdicts (full OPH; GOPH when
//      level_b = L) or the per-pair walk of the pairs still undecided (GOPH, level_b < L)
// The batch loop is straight-line: the lookahead crosses into the next set only in the last
// three batches of a set (written out after the loop), so no per-batch bookkeeping.  The
// termination histogram is counted in shared memory and added once per CTA; a set's
// empty-bin mask word is fetched at its first batch.
template <int MINB, bool GOPH>
__global__ void __launch_bounds__(32 * kBitWarps, MINB) bit_pipe_kernel(const __grid_constant__ BitArgs a) {
    __shared__ uint2 s_sw[kBitMaxBins + 1];  // per bin: (first position, width)
    __shared__ uint64_t s_full[kBitMaxStages];
    __shared__ uint32_t s_done[kBitMaxStages];
    __shared__ __align__(16) uint32_t s_ring[kBitWarps][4][16];
    __shared__ unsigned long long s_hist[kMaxGroups + 1];
    __shared__ uint32_t s_ceilT[GOPH ? 1 : kBitMaxBins + 2];  // full OPH exit: ceil(T x), x = 0 .. k
    extern __shared__ __align__(128) uint32_t s_vals[];  // [nstage][npre][8]
    for (uint32_t b = threadIdx.x; b < a.nscan; b += blockDim.x) {
        uint32_t st, wd;
        bit_bin_range(a, b, st, wd);
        s_sw[b] = make_uint2(st, wd);
    }
    if (!GOPH && a.exit_from)
        for (uint32_t x = threadIdx.x; x <= a.nbins_total; x += blockDim.x)
            s_ceilT[x] = (uint32_t)(((uint64_t)a.t_num * x + a.t_den - 1) / a.t_den);
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    uint32_t qw0[2], qvalid[2], max_eq[2];
#pragma unroll
    for (int w = 0; w < 2; w++) {
        qw0[w] = 32u * (2 * lane + w);
        qvalid[w] = qw0[w] >= a.nqb ? 0u : (a.nqb - qw0[w] >= 32u ? 0xFFFFFFFFu : ((1u << (a.nqb - qw0[w])) - 1u));
        max_eq[w] = a.max_eq[2 * lane + w];
    }
    const uint2 *rows_lane = reinterpret_cast<const uint2 *>(a.rows) + lane;
    const uint64_t ntiles = (a.n_sets - a.s_begin + kBitWarps - 1) / kBitWarps;
    const uint32_t vstride = a.npre * 8u;
    if (threadIdx.x <= kMaxGroups) s_hist[threadIdx.x] = 0ull;
    if (threadIdx.x == 0) {
        for (uint32_t i = 0; i < a.nstage; i++) {
            mbar_init(&s_full[i], 32);
            s_done[i] = 0u;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 0) {
        for (uint32_t i = 0; i < a.nstage; i++) {
            const uint64_t t = blockIdx.x + (uint64_t)i * gridDim.x;
            if (t < ntiles) bit_tile_load(a, t, s_vals + i * vstride, &s_full[i], lane);
        }
    }
    const uint32_t nbs = a.nscan / 16u;
    // (per-CTA tile counts fit 32 bits)
    const uint32_t n_it = (uint64_t)blockIdx.x < ntiles ? (uint32_t)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0u;
    uint32_t *ring = &s_ring[warp][0][0];
    const uint32_t bl = lane & 15u;
    const uint32_t *vals_lane = s_vals + 8u * bl + warp;  // + slot * vstride + 128 j: bin 16 j + bl
    const uint2 *sw_lane = s_sw + bl;                     // + 16 j

    // A: the row index of this lane's bin of batch j of the set staged in `slot` (lanes 16-31
    // repeat lanes 0-15: same addresses, no extra traffic)
    auto look = [&](uint32_t slot, uint32_t j) -> uint32_t {
        const uint32_t v = vals_lane[slot * vstride + 128u * j];
        const uint2 sw = sw_lane[16u * j];
        return v < sw.y ? __ldg(a.idx + sw.x + v) : 0u;
    };
    // C: the 16 rows of the batch parked in ring slot q
    auto rows = [&](uint32_t q, uint32_t (&x)[2][16]) {
        const uint4 *rp = reinterpret_cast<const uint4 *>(ring + 16u * q);
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const uint4 o = rp[j];
            const uint32_t r4[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const uint2 y = __ldg(rows_lane + (uint64_t)r4[u] * 32u);
                x[0][4 * j + u] = y.x;
                x[1][4 * j + u] = y.y;
            }
        }
    };
    uint32_t c[2][kBitCS];
#pragma unroll
    for (int w = 0; w < 2; w++)
#pragma unroll
        for (int i = 0; i < (int)kBitCS; i++) c[w][i] = 0u;
    uint32_t pend = 0u, n_final = 0u;
    uint32_t n_gathered = 0;  // row batches this warp gathered (oph_results.d_bins_scanned)
    uint32_t alive[2] = {qvalid[0], qvalid[1]};
    uint32_t lev = 1, lend = a.kp / 16u;  // GOPH: the level being counted, the batch it ends at
    uint32_t gb = 0;                      // batches of the warp's earlier sets (ring slots)
    uint64_t s_cur = 0;
    // GOPH: Algorithm 1's decisions at the end of level l < L (as bit_scan_q_kernel)
    auto decide = [&](uint32_t l) {
        const uint32_t A = a.acc_cnt[l - 1];
        const int32_t R = a.rej_cnt[l - 1];
#pragma unroll
        for (int w = 0; w < 2; w++) {
            const uint32_t acc = sliced_ge<kBitCS>(c[w], A) & alive[w];
            const uint32_t dec = (acc | (R >= 0 ? ~sliced_ge<kBitCS>(c[w], (uint32_t)R + 1u) : 0u)) & alive[w];
            const uint32_t tot = __reduce_add_sync(0xFFFFFFFFu, __popc(dec));
            if (lane == 0 && tot) atomicAdd(&s_hist[l], (unsigned long long)tot);
            uint32_t want = a.out.dense ? dec : acc;
            while (__any_sync(0xFFFFFFFFu, want != 0u)) {
                const bool has = want != 0u;
                const uint32_t jj = has ? __ffs(want) - 1 : 0u;
                want &= want - 1u;
                const uint32_t qg = a.qb0 + qw0[w] + jj;
                uint32_t nmb = 0, ex = 0;
                if (has) {
                    nmb = sliced_get<kBitCS>(c[w], jj);
                    ex = bit_excl(a, qg, s_cur, 0, l * a.kp);
                }
                emit(a.out, has, qg, s_cur, nmb, ex, l, (acc >> jj) & 1u, OPH_FLAG_EARLY, -1.0f);
            }
            alive[w] &= ~dec;
        }
    };
    // one batch j: rows of j + 1 issued, the lookup of j + 2 parked, `nl` (the lookup of j + 3)
    // becomes pending, batch j counted
    auto step = [&](uint32_t j, uint32_t (&xc)[2][16], uint32_t (&xn)[2][16], uint32_t nl) {
        // (full OPH: nbs % 4 == 0, the ring slots restart with every set)
        const uint32_t g = GOPH ? gb + j : j;
        rows((g + 1) & 3u, xn);
        if (lane < 16u) ring[16u * ((g + 2) & 3u) + lane] = pend;
        pend = nl;
        __syncwarp();
#pragma unroll
        for (int w = 0; w < 2; w++) csa16(c[w], xc[w]);
        if constexpr (GOPH) {
            if (j + 1 != lend) return;  // warp-uniform
            if (lev < a.nlev && a.thr_on[lev - 1] && s_cur < a.n_sets) decide(lev);
            lev++;
            lend += a.kp / 16u;
        }
    };

    uint32_t x[2][16], xb[2][16];
    uint32_t slot = 0, phase = 0;
    if (n_it) {
        mbar_wait(&s_full[0], 0);
        const uint32_t r0 = look(0, 0), r1 = look(0, 1);
        pend = look(0, 2);
        if (lane < 16u) {
            ring[lane] = r0;
            ring[16u + lane] = r1;
        }
        __syncwarp();
        rows(0, x);
    }
    for (uint32_t it = 0; it < n_it; it++) {
        const uint64_t tile = blockIdx.x + (uint64_t)it * gridDim.x;
        const uint64_t s = a.s_begin + tile * kBitWarps + warp;
        if constexpr (GOPH) s_cur = s;
        uint32_t es_w = 0;
        if (s < a.n_sets) es_w = lane < a.nw ? __ldg(a.E + (uint64_t)lane * a.ld + s) : 0u;
        uint32_t j = 0;
        bool early = false;
        uint32_t theta = 0u;  // full OPH exit: a lower bound on the thresholds of the block's queries
        for (; j + 4 < nbs; j += 2) {
            step(j, x, xb, look(slot, j + 3));
            step(j + 1, xb, x, look(slot, j + 4));
            if constexpr (!GOPH) {
                // R32: after B = 16 (j + 2) bins a pair can still reach T only if its count plus the
                // set's non-empty bins in [B, k) reaches its threshold; theta = ceil(T den_min)
                // with den_min from the largest query-empty count of the lane's two words is a
                // lower bound on it (as in the final filter below; one register: per-word bounds
                // cost spills, 14.55 vs 13.86 ms).  R32b, tighter: the bins in [B, k) add at most
                // R (the set's non-empty bins there) to the count and at least as much to the
                // denominator, so a pair needs M_B >= ceil(T (den_B + R)) - R, den_B >= B - eq_B -
                // es_B (JointEmpty: B - min(eq_B, es_B)) with eq_B the largest query-empty count
                // in [0, B) of the lane's queries (bit_maxeq_kernel's prefix maxima) -- the query's
                // empty bins past B then no longer loosen the bound.  Both bounds are necessary; the
                // larger is used.  No such pair in the block: the set is done -- every pair is
                // NotSimilar, and threshold results emit nothing for them.
                const uint32_t B = 16u * (j + 2);
                if (a.exit_from && B >= a.exit_from && ((B - a.exit_from) & (a.exit_every - 1u)) == 0u && B < a.nbins_total) {
                    const uint32_t k = a.nbins_total;
                    const uint32_t es = __reduce_add_sync(0xFFFFFFFFu, popc_masked(0u, es_w, 0, lane, k));
                    if (theta == 0u) {  // (the lane's two words share one bound: one register)
                        const uint32_t me = max(max_eq[0], max_eq[1]);
                        const uint32_t den_min = a.joint ? k - min(me, es) : k - min(k, me + es);
                        theta = max(1u, s_ceilT[den_min]);
                    }
                    const uint32_t emp = __reduce_add_sync(
                        0xFFFFFFFFu, (lane < a.nw && 32u * lane >= B) ? popc_masked(0u, es_w, 0, lane, k) : 0u);
                    const uint32_t rem = (k - B) - emp;  // the set's non-empty bins not counted yet
                    // (per word: the prefix bounds are loaded per check, no register kept)
                    const uint32_t *pref = a.max_eq_pref + (B >> 5) * 64u + 2u * lane;
                    const uint32_t esB = es - emp;
                    bool cand = false;
#pragma unroll
                    for (int w = 0; w < 2; w++) {
                        const uint32_t eqB = __ldg(pref + w);
                        const uint32_t denB = a.joint ? B - min(eqB, esB) : B - min(B, eqB + esB);
                        const uint32_t th = max(theta, s_ceilT[denB + rem]);
                        cand |= (th <= rem ? qvalid[w] : (sliced_ge<kBitCS>(c[w], th - rem) & qvalid[w])) != 0u;
                    }
                    if (!__any_sync(0xFFFFFFFFu, cand)) {
                        early = true;
                        break;
                    }
                }
            }
        }
        if (!GOPH && early) {
            // release the tile (every lookup this set issued has read its staged value), start
            // the next set's pipeline afresh (its lookups 0-2, rows of batch 0), count the pairs
            // as decided at the last level (the histogram of full OPH, as the paper's method)
            __syncwarp();
            uint32_t last = 0;
            if (lane == 0) {
                __threadfence_block();
                last = atomicAdd(&s_done[slot], 1u) == kBitWarps - 1;
                if (last) s_done[slot] = 0u;
            }
            last = __shfl_sync(0xFFFFFFFFu, last, 0);
            const uint64_t tn = tile + (uint64_t)a.nstage * gridDim.x;
            if (last && tn < ntiles) bit_tile_load(a, tn, s_vals + slot * vstride, &s_full[slot], lane);
            const bool more = it + 1 < n_it;
            if (++slot == a.nstage) {
                slot = 0;
                phase ^= 1u;
            }
            if (more) {
                mbar_wait(&s_full[slot], phase);
                const uint32_t r0 = look(slot, 0), r1 = look(slot, 1);
                pend = look(slot, 2);
                if (lane < 16u) {
                    ring[lane] = r0;
                    ring[16u + lane] = r1;
                }
                __syncwarp();
                rows(0, x);
            }
            if (s < a.n_sets) n_final += __popc(qvalid[0]) + __popc(qvalid[1]);
            if (s < a.n_sets) n_gathered += j + 3;  // row batches issued for this set: 0 .. j + 2
#pragma unroll
            for (int w = 0; w < 2; w++)
#pragma unroll
                for (int i = 0; i < (int)kBitCS; i++) c[w][i] = 0u;
            continue;
        }
        if (s < a.n_sets) n_gathered += nbs;
        // j = nbs - 4: the set's last lookup, then its tile is released and the next one awaited
        step(j, x, xb, look(slot, j + 3));
        {
            __syncwarp();
            uint32_t last = 0;
            if (lane == 0) {
                __threadfence_block();
                last = atomicAdd(&s_done[slot], 1u) == kBitWarps - 1;
                if (last) s_done[slot] = 0u;
            }
            last = __shfl_sync(0xFFFFFFFFu, last, 0);
            const uint64_t tn = tile + (uint64_t)a.nstage * gridDim.x;
            if (last && tn < ntiles) bit_tile_load(a, tn, s_vals + slot * vstride, &s_full[slot], lane);
        }
        const bool more = it + 1 < n_it;
        if (++slot == a.nstage) {
            slot = 0;
            phase ^= 1u;
        }
        if (more) mbar_wait(&s_full[slot], phase);
        step(j + 1, xb, x, more ? look(slot, 0) : 0u);
        step(j + 2, x, xb, more ? look(slot, 1) : 0u);
        step(j + 3, xb, x, more ? look(slot, 2) : 0u);
        // (nbs even: the next set's batch 0 is in x again)
        if (GOPH && a.level_b < a.nlev && s < a.n_sets) {
            // the pairs still undecided after level_b: walked one by one over the later levels
#pragma unroll
            for (int w = 0; w < 2; w++) {
                uint32_t al = alive[w];
                while (__any_sync(0xFFFFFFFFu, al != 0u)) {
                    const uint32_t src = __ffs(__ballot_sync(0xFFFFFFFFu, al != 0u)) - 1;
                    const uint32_t mine = al != 0u ? __ffs(al) - 1 : 0u;
                    const uint32_t jj = __shfl_sync(0xFFFFFFFFu, mine, src);
                    const uint32_t m = __shfl_sync(0xFFFFFFFFu, sliced_get<kBitCS>(c[w], mine), src);
                    if (lane == src) al &= al - 1u;
                    bit_walk_goph(a, a.qb0 + 32u * (2 * src + w) + jj, s, m, lane, a.out.hist ? s_hist : nullptr);
                }
            }
        } else if (s < a.n_sets) {  // warp-uniform: a tail tile's missing set is counted, never scored
            const uint32_t es = __reduce_add_sync(0xFFFFFFFFu, popc_masked(0u, es_w, 0, lane, a.nbins_total));
            const uint32_t k = a.nbins_total;
#pragma unroll
            for (int w = 0; w < 2; w++) {
                const uint32_t al = GOPH ? alive[w] : qvalid[w];
                n_final += __popc(al);
                const uint32_t den_min = a.joint ? k - min(max_eq[w], es) : k - min(k, max_eq[w] + es);
                const uint32_t theta =
                    a.out.dense ? 0u : (uint32_t)(((uint64_t)a.t_num * den_min + a.t_den - 1) / a.t_den);
                uint32_t want = sliced_ge<kBitCS>(c[w], theta) & al;
                while (__any_sync(0xFFFFFFFFu, want != 0u)) {
                    const bool has = want != 0u;
                    const uint32_t jj = has ? __ffs(want) - 1 : 0u;
                    want &= want - 1u;
                    const uint32_t qg = a.qb0 + qw0[w] + jj;
                    uint32_t ex = 0;
                    for (uint32_t ww = 0; ww < a.nw; ww++) {
                        const uint32_t sw = __shfl_sync(0xFFFFFFFFu, es_w, ww);
                        if (has) ex += popc_masked(__ldg(a.QEM + (uint64_t)qg * a.nw + ww), sw, a.joint, ww, k);
                    }
                    const uint32_t nmb = sliced_get<kBitCS>(c[w], jj);
                    const uint32_t den = k - ex;
                    const bool undef = den == 0;
                    const uint32_t verdict = !undef && (uint64_t)nmb * a.t_den >= (uint64_t)a.t_num * den;
                    emit(a.out, has, qg, s, nmb, ex, a.level_final, verdict, undef ? OPH_FLAG_UNDEFINED : 0u,
                         undef ? -1.0f : (float)nmb / (float)den);
                }
            }
        }
#pragma unroll
        for (int w = 0; w < 2; w++) {
            if (GOPH) alive[w] = qvalid[w];
#pragma unroll
            for (int i = 0; i < (int)kBitCS; i++) c[w][i] = 0u;
        }
        if constexpr (GOPH) {
            lev = 1;
            lend = a.kp / 16u;
            gb += nbs;
        }
    }
    if (a.scanned && lane == 0 && n_gathered) atomicAdd(a.scanned, 16ull * n_gathered);
    if (a.out.hist) {
        const uint32_t tot = __reduce_add_sync(0xFFFFFFFFu, n_final);
        if (lane == 0 && tot) atomicAdd(&s_hist[a.level_final], (unsigned long long)tot);
        __syncthreads();
        if (threadIdx.x <= kMaxGroups && s_hist[threadIdx.x]) atomicAdd(a.out.hist + threadIdx.x, s_hist[threadIdx.x]);
    }
}

cudaError_t launch_bit_block(const BitArgs &a, cudaStream_t st) {
    cudaError_t e;
    // the value -> row table of this block: clear, claim rows, set the bits
    if ((e = cudaMemsetAsync(a.idx, 0, (size_t)a.vpos * 4, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(a.nrows, 0, 4, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(a.rows, 0, 128 * a.qw, st)) != cudaSuccess) return e;  // the zero row
    const uint64_t n = (uint64_t)a.nscan * a.nqb;
    const unsigned g = (unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 16);
    bit_claim_kernel<<<g, 256, 0, st>>>(a);
    bit_fill_kernel<<<g, 256, 0, st>>>(a);
    bit_maxeq_kernel<<<a.qw, 1024, 0, st>>>(a);
    // the scan: 8 consecutive sets per CTA tile, grid-stride; 3 CTAs per SM at 1,024-query
    // rows, 2 at 2,048 (two words of counters per lane)
    const uint64_t ntiles = (a.n_sets - a.s_begin + kBitWarps - 1) / kBitWarps;
    // (OPHGPU_BIT_CTAS=2: the full-OPH / GOPH scan at 2 CTAs per SM without register limit, A/B)
    static const bool two = getenv("OPHGPU_BIT_CTAS") && atoi(getenv("OPHGPU_BIT_CTAS")) == 2;
    // (OPHGPU_BIT_CTAS=3: the 2,048-query scan at 3 CTAs per SM, 85 registers, A/B)
    static const bool three = getenv("OPHGPU_BIT_CTAS") && atoi(getenv("OPHGPU_BIT_CTAS")) == 3;
    const int ctas = a.mode_hoph || two || (a.qw == 2 && !three) ? 2 : 3;
    const unsigned grid = (unsigned)std::min<uint64_t>(ntiles, 148ull * ctas * 8);
    const size_t smem = (size_t)a.nstage * a.npre * kBitWarps * 4;
    auto kern = a.mode_hoph ? bit_scan_x_kernel<2, 2>
                : a.pipe    ? (a.method == kGoph ? bit_pipe_kernel<2, true> : bit_pipe_kernel<2, false>)
                            : (a.qw == 2 ? (a.npre == a.nscan ? (three ? bit_scan_q_kernel<2, 3, true>
                                                                       : bit_scan_q_kernel<2, 2, true>)
                                                              : bit_scan_q_kernel<2, 2, false>)
                                         : (two ? bit_scan_kernel<2> : bit_scan_kernel<3>));
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
        return e;
    kern<<<grid, 32 * kBitWarps, smem, st>>>(a);
    return cudaGetLastError();
}
