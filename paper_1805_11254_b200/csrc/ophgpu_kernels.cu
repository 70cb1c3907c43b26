// sm_100a kernels of the OPH / GOPH / HOPH scoring path (arxiv 1805.11254).
//
//   K1 build_kernel     OPH + HOPH sketches from one psi evaluation per element
//                                             SURVEY 8(a) a1-a3
//   K2 minwise_kernel   MinWise sketches, k keyed permutations        a4
//   -- prep_kernel      query preparation: empty remap + both layouts        a5
//   K3 scan_kernel      BRUTE: streaming compare of a register-resident query
//                       block against set tiles; full OPH / MinWise / the
//                       first decidable GOPH level / HOPH level 1          a6-a9
//   K3' table_kernel +  PROBE: hash join of the collection with per-bin Bloom
//       join_kernel     filters in shared memory + exact L2 tables           a6-a9
//   K3'' levels_kernel  BRUTE GOPH / HOPH decided group by group in one pass a7-a8
//   K4 level_kernel     one GOPH/HOPH level over the compacted survivors;
//                       the last level applies the final verdict            a7-a8
//   K6 run_select       threshold / top-k result lists (CUB radix sort)     a10
//   K7 bit_scan_kernel  BITMAP: value-indexed bitmap join, bit-sliced counts
//                       (bitjoin.cuh): full OPH / GOPH / HOPH 1:1         a6-a8
//   -- jaccard_kernel   exact Jaccard of hit pairs (quality check)
//   -- sh_* kernels     text shingling (ingestion before K1)
//
// All decisions are exact integer arithmetic against thresholds the host
// planner compiled from the paper's rules (R23); no floating
// point decides anything.  Layouts: DESIGN.md "Data layout in HBM".
#include <cstdlib>

#include <cub/cub.cuh>

#include "internal.h"

#ifndef EA_B
#define EA_B 16  // queries per thread block of the empty-aware register scan (image-like: 32 208 ms, 16 136, 8 151)
#endif

namespace ophgpu {

__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// ---------------------------------------------------------------------------
// psi: keyed 4-round bijection of [0, 2^w), cycle-walked into [0, |V|)
// (DESIGN.md section 4).  W32: w == 32, the mask is a no-op.
// ---------------------------------------------------------------------------
// w < 32: one round is y = ((x ^ kappa) mu) mod 2^w, x' = y ^ (y >> s).  The bits
// of the 32-bit product above w only reach higher bits through later products,
// so they may stay; only the shift must not pull them down: y >> s =
// (P 2^(32-w) mod 2^32) >> (32 - w + s), an IMAD (the FMA pipe, idle in the
// MinWise build) and one SHF instead of an AND and a SHF on the ALU pipe.  The
// value is masked to w bits once, at the end.  hmul = 2^(32-w) and hsh =
// 32 - w + s come in as runtime values so the multiply stays an IMAD.
template <bool W32>
__device__ __forceinline__ uint32_t psi_pass(const uint32_t (&kappa)[4], const uint32_t (&mu)[4], uint32_t mask,
                                             uint32_t shift, uint32_t hmul, uint32_t hsh, uint32_t x) {
#pragma unroll
    for (int r = 0; r < 4; r++) {
        x = (x ^ kappa[r]) * mu[r];
        if (W32) x ^= x >> shift;
        else x ^= (x * hmul) >> hsh;
    }
    return W32 ? x : (x & mask);
}

template <bool W32>
__device__ __forceinline__ uint32_t psi(const PsiParams &P, uint32_t x) {
    if (P.identity) return x;
    x = psi_pass<W32>(P.kappa, P.mu, P.mask, P.shift, P.hmul, P.hsh, x);
    if (!P.pow2)
        while ((uint64_t)x >= P.V) x = psi_pass<W32>(P.kappa, P.mu, P.mask, P.shift, P.hmul, P.hsh, x);
    return x;
}

// bin and within-bin offset of p in a range cut into nb bins by the floor
// rule: the largest b with floor(b len / nb) <= p - start is
// floor(((p - start + 1) nb - 1) / len).
__device__ __forceinline__ void range_bin(const RangeBins &R, uint32_t nb, uint64_t p, uint32_t &bin, uint32_t &off) {
    const uint64_t x = p - R.start;
    if (R.pow2) {
        bin = (uint32_t)(x >> R.shift);
        off = (uint32_t)(x & ((1ull << R.shift) - 1));
    } else {
        const uint64_t b = ((x + 1) * nb - 1) / R.len;
        bin = (uint32_t)b;
        off = (uint32_t)(x - (b * R.len) / nb);
    }
}

__device__ __forceinline__ uint64_t splitmix64_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// ---------------------------------------------------------------------------
// K1: OPH + HOPH build.  One CTA = SB consecutive sets; their ids are one
// contiguous CSR range, streamed by all 256 threads (a thread tracks the set
// of its element incrementally: elements advance by 256 per iteration).
// Per-set sketches live in shared memory (row stride n+1 words) and are
// minimised with shared atomicMin (EMPTY = 0xFFFFFFFF is the identity of
// min).  HOPH group lookup: for the 1:1 split of a power-of-two universe the
// group of p is its count of leading one bits (capped at L-1) and its bins
// are shifts; other layouts binary-search a group table in shared memory.
// Write-out: 128-bit stores of 4 consecutive sets of one bin row; empty masks
// by warp ballot over 32 bins.
// ---------------------------------------------------------------------------
template <bool W32>
__device__ __forceinline__ void build_one(const BuildArgs &a, const RangeBins *grp, uint32_t *so, uint32_t *sh,
                                          uint32_t kst, uint32_t hst, uint32_t j, uint32_t id) {
    const uint32_t p = psi<W32>(a.psi, id);
    uint32_t bin, off;
    if (a.do_flat) {
        range_bin(a.flat, a.k, p, bin, off);
        // a shared load first: most elements do not lower their bin minimum (for m elements in
        // a bin only ~ln m do), and a load is much cheaper than a shared atomic
        uint32_t *slot = &so[j * kst + bin];
        if (off < *slot) atomicMin(slot, off);
    }
    if (a.do_hier) {
        uint32_t g;
        if (a.hier_pow2_halves) {
            // group g = [V - V/2^g, V - V/2^(g+1)): g = leading ones of p in m bits
            g = min((uint32_t)__clz(~(p << (32 - a.log2V))), a.L - 1);
            const uint32_t e = (g + 1 < a.L) ? a.log2V - 1 - g : a.log2V - (a.L - 1);  // log2 of the group length
            const uint32_t sh_bits = e - a.log2kp;
            const uint32_t x = p & ((e >= 32) ? 0xFFFFFFFFu : ((1u << e) - 1u));
            bin = x >> sh_bits;
            off = x & ((1u << sh_bits) - 1u);
        } else {
            uint32_t g0 = 0, g1 = a.L - 1;  // largest g with start_g <= p
            while (g0 < g1) {
                const uint32_t mid = (g0 + g1 + 1) >> 1;
                if (grp[mid].start <= p) g0 = mid; else g1 = mid - 1;
            }
            g = g0;
            range_bin(grp[g], a.kp, p, bin, off);
        }
        uint32_t *hslot = &sh[j * hst + g * a.kp + bin];
        if (off < *hslot) atomicMin(hslot, off);
    }
}

// The common layout in 32-bit arithmetic (FAST): psi a plain bijection (|V| = 2^w,
// no cycle walking), flat bins of 2^fsh values (bin = p >> fsh), and the 1:1
// HOPH split of 2^log2V with L <= 32 groups, taken from the left-aligned
// t = p << (32 - log2V): g = min(leading ones of t, L - 1); dropping the g ones
// and the 0 after them (L - 1 ones for the last group) leaves the position inside
// the group, left-aligned in y, whose top log2kp bits are the bin and the next
// log2V - sc - log2kp bits the offset.  so_j / sh_j: this set's smem rows.
template <bool W32>
__device__ __forceinline__ void build_one_fast(const BuildArgs &a, uint32_t *so_j, uint32_t *sh_j, uint32_t id) {
    const uint32_t p = psi_pass<W32>(a.psi.kappa, a.psi.mu, a.psi.mask, a.psi.shift, a.psi.hmul, a.psi.hsh, id);
    {
        const uint32_t bin = p >> a.flat.shift, off = p & ((1u << a.flat.shift) - 1u);
        uint32_t *slot = so_j + bin;
        if (off < *slot) atomicMin(slot, off);
    }
    {
        const uint32_t t = p << (32u - a.log2V);
        const uint32_t g = min((uint32_t)__clz(~t), a.L - 1u);
        const uint32_t sc = g + (g + 1u < a.L ? 1u : 0u);
        const uint32_t y = t << sc;
        const uint32_t bin = y >> (32u - a.log2kp);
        const uint32_t off = __funnelshift_rc(y << a.log2kp, 0u, 32u - a.log2V + sc + a.log2kp);
        uint32_t *hslot = sh_j + g * a.kp + bin;
        if (off < *hslot) atomicMin(hslot, off);
    }
}

// write-out of SB sets' sketches (smem rows of `stride` words, stride = 1 mod 32
// so that a lane per bin reads the SB sets conflict-free): a warp takes 32
// consecutive bins; each lane stores its bin's SB values as 128-bit stores of 4
// consecutive sets, and SB ballots give the SB sets' empty-mask words of these
// 32 bins (bit t of word w <=> bin 32 w + t empty), stored by lanes 0..SB-1.
template <int SB>
__device__ __forceinline__ void write_sketch(const uint32_t *src, uint32_t stride, uint32_t nbins, uint32_t nloc,
                                             uint32_t *dst, uint32_t *dst_mask, uint64_t ld, uint64_t s0) {
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const bool full = nloc == SB && SB % 4 == 0;
    if (full && nbins % 32u == 0 && ld < (1ull << 32)) {  // the common tile: straight-line code, 32-bit ld
        const uint32_t ldw = (uint32_t)ld;
        for (uint32_t b0 = warp * 32u; b0 < nbins; b0 += nwarps * 32u) {
            const uint32_t b = b0 + lane;
            uint32_t v[SB];
#pragma unroll
            for (int j = 0; j < SB; j++) v[j] = src[j * stride + b];
            uint32_t *d = dst + (uint64_t)b * ldw + s0;
#pragma unroll
            for (int q = 0; q < SB / 4; q++)
                *reinterpret_cast<uint4 *>(d + 4 * q) = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            uint32_t mine = 0;
#pragma unroll
            for (int j = 0; j < SB; j++) {
                const uint32_t m = __ballot_sync(0xFFFFFFFFu, v[j] == kEmpty);
                mine = lane == (uint32_t)j ? m : mine;
            }
            if (lane < SB) dst_mask[(uint64_t)(b0 >> 5) * ldw + s0 + lane] = mine;
        }
        return;
    }
    for (uint32_t b0 = warp * 32u; b0 < nbins; b0 += nwarps * 32u) {  // warp-uniform
        const uint32_t b = b0 + lane;
        const bool in = b < nbins;
        uint32_t v[SB];
#pragma unroll
        for (int j = 0; j < SB; j++) v[j] = in ? src[j * stride + b] : 0u;
        if (in) {
            uint32_t *d = dst + (uint64_t)b * ld + s0;
            if (full) {
#pragma unroll
                for (int q = 0; q < SB / 4; q++)
                    *reinterpret_cast<uint4 *>(d + 4 * q) = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            } else {
#pragma unroll
                for (int j = 0; j < SB; j++)
                    if ((uint32_t)j < nloc) d[j] = v[j];
            }
        }
        uint32_t mine = 0;
#pragma unroll
        for (int j = 0; j < SB; j++) {
            const uint32_t m = __ballot_sync(0xFFFFFFFFu, v[j] == kEmpty);
            if (lane == (uint32_t)j) mine = m;
        }
        if (lane < nloc) dst_mask[(uint64_t)(b0 >> 5) * ld + s0 + lane] = mine;
    }
}

template <bool W32, int SB, bool FAST>
__global__ void __launch_bounds__(512) build_kernel(const __grid_constant__ BuildArgs a) {
    extern __shared__ __align__(16) uint32_t smem_u32[];
    // group table in shared memory: lanes index it divergently, which would
    // serialise on the constant cache if read from the kernel parameters
    __shared__ RangeBins grp[kMaxGroups];
    __shared__ uint64_t offs[33];
    __shared__ uint32_t loffs[33];  // offsets relative to the tile's first element
    // row strides = 1 mod 32: the write-out reads the SB sets of one bin conflict-free
    const uint32_t kst = (a.k + 31u) / 32u * 32u + 1u;
    const uint32_t nbh = a.L * a.kp;
    const uint32_t hst = (nbh + 31u) / 32u * 32u + 1u;
    uint32_t *so = smem_u32;                                               // [SB][k+1]
    uint32_t *sh = so + (a.do_flat ? (size_t)SB * kst : 0);               // [SB][L*kp+1]
    const uint32_t words = (a.do_flat ? SB * kst : 0) + (a.do_hier ? SB * hst : 0);

    const uint64_t s0 = (uint64_t)blockIdx.x * SB;
    const uint32_t nloc = (uint32_t)min((uint64_t)SB, a.n_sets - s0);
    for (uint32_t i = threadIdx.x; i <= nloc; i += blockDim.x) offs[i] = a.offsets[s0 + i];
    __syncthreads();
    for (uint32_t i = threadIdx.x; i <= nloc; i += blockDim.x) loffs[i] = (uint32_t)(offs[i] - offs[0]);
    if (a.do_hier && !a.hier_pow2_halves)
        for (uint32_t i = threadIdx.x; i < a.L; i += blockDim.x) grp[i] = a.grp[i];
    {
        uint4 *s4 = reinterpret_cast<uint4 *>(smem_u32);
        const uint4 e4 = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
        for (uint32_t i = threadIdx.x; i < (words + 3) / 4; i += blockDim.x) s4[i] = e4;
    }
    __syncthreads();

    const uint64_t e0 = offs[0], e1 = offs[nloc];
    constexpr int kU = FAST ? 8 : 4;  // ids in flight per thread
    uint32_t j = 0;
    if (FAST) {
        // the keys and layout constants in registers (not re-read from the parameter bank per
        // element), shared rows as 32-bit shared addresses, and the bin minima as
        // fire-and-forget shared reductions (red.shared.min: no load, compare and branch per
        // element; an EMPTY slot is the identity of min)
        uint32_t kap[4], mu[4];
#pragma unroll
        for (int r = 0; r < 4; r++) {
            kap[r] = a.psi.kappa[r];
            mu[r] = a.psi.mu[r];
        }
        const uint32_t mask = a.psi.mask, pshift = a.psi.shift, hmul = a.psi.hmul, hsh = a.psi.hsh;
        const uint32_t fsh = a.flat.shift, fmask = (1u << a.flat.shift) - 1u;
        const uint32_t vsh = 32u - a.log2V, Lm1 = a.L - 1u, lkp = a.log2kp, kpw = a.kp;
        const uint32_t osh = 32u - a.log2V + a.log2kp, bsh = 32u - a.log2kp;
        const uint32_t n = (uint32_t)(e1 - e0);
        const uint32_t *ids = a.ids + e0;
        const uint32_t so_base = smem_addr(so), sh_base = smem_addr(sh);
        uint32_t so_j = so_base, sh_j = sh_base;
        for (uint32_t e = threadIdx.x; e < n; e += kU * blockDim.x) {
            uint32_t id[kU];
#pragma unroll
            for (int u = 0; u < kU; u++) id[u] = e + u * blockDim.x < n ? __ldg(ids + e + u * blockDim.x) : 0u;
#pragma unroll
            for (int u = 0; u < kU; u++) {
                const uint32_t eu = e + u * blockDim.x;
                if (eu >= n) break;
                if (loffs[j + 1] <= eu) {  // the set owning element eu (empty sets are skipped)
                    do j++; while (loffs[j + 1] <= eu);
                    so_j = so_base + 4u * j * kst;
                    sh_j = sh_base + 4u * j * hst;
                }
                const uint32_t p = psi_pass<W32>(kap, mu, mask, pshift, hmul, hsh, id[u]);
                const uint32_t fo = p & fmask;
                asm volatile("red.shared.min.u32 [%0], %1;" ::"r"(so_j + 4u * (p >> fsh)), "r"(fo));
                // HOPH 1:1 on 2^log2V: group g = leading ones of the left-aligned p (capped at L-1),
                // then drop them and the 0 after them (not for the last group): bin and offset
                const uint32_t t = p << vsh;
                const uint32_t g = min((uint32_t)__clz(~t), Lm1);
                const uint32_t sc = g + (g < Lm1 ? 1u : 0u);
                const uint32_t y = t << sc;
                const uint32_t hb = y >> bsh;
                const uint32_t ho = __funnelshift_rc(y << lkp, 0u, osh + sc);
                asm volatile("red.shared.min.u32 [%0], %1;" ::"r"(sh_j + 4u * (g * kpw + hb)), "r"(ho));
            }
        }
    } else
    for (uint64_t e = e0 + threadIdx.x; e < e1; e += kU * blockDim.x) {
        uint32_t id[kU];
#pragma unroll
        for (int u = 0; u < kU; u++) {
            const uint64_t eu = e + (uint64_t)u * blockDim.x;
            id[u] = eu < e1 ? __ldg(a.ids + eu) : 0u;
        }
#pragma unroll
        for (int u = 0; u < kU; u++) {
            const uint64_t eu = e + (uint64_t)u * blockDim.x;
            if (eu >= e1) break;
            while (offs[j + 1] <= eu) j++;  // the set owning element eu (empty sets are skipped)
            build_one<W32>(a, grp, so, sh, kst, hst, j, id[u]);
        }
    }
    __syncthreads();

    if (a.do_flat) write_sketch<SB>(so, kst, a.k, nloc, a.oph, a.oph_empty, a.ld, s0);
    if (a.do_hier) write_sketch<SB>(sh, hst, nbh, nloc, a.hoph, a.hoph_empty, a.ld, s0);
}

// K1 (FAST layout, r02): a warp per SPW consecutive sets of the CTA's SB.
//  * The warp streams its sets' contiguous id range (the owning set is a compare
//    against SPW - 1 register boundaries, no per-element shared lookup) with the next
//    batch of ids in flight while the current one is hashed.
//  * HOPH groups 0 .. hder-1 are unions of whole OPH bins: with |V| = 2^m, group g
//    (g < L - 1) bins are 2^(m - g - 1 - log2 k') wide and start at multiples of their
//    width, an OPH bin is 2^(m - log2 k) wide, so for g <= log2 k - log2 k' - 1 every
//    HOPH bin of group g is M_g = 2^(log2 k - log2 k' - 1 - g) consecutive OPH bins.
//    Its minimum offset is that of its first non-empty OPH bin, t 2^fsh + off_t
//    (positions increase with t), exactly the min over its elements (P:143-160 for
//    both layouts: the same psi, min per bin).  So only elements of groups >= hder
//    (the last 2^-hder of the universe) update the HOPH tile: one shared reduction per
//    element instead of two (the kernel is bound by the shared-memory pipe).  The
//    derived bins are written from the OPH tile: a lane reads 4 consecutive OPH bins
//    (one 16-B load; rows are 16-B aligned), takes their min in registers and, for
//    M_g > 4, across M_g / 4 lanes by shuffles.
//  * Each warp initialises and finishes its own sets' rows (no CTA barrier until
//    the bin-major write-out of the SB sets).
// Row strides = 4 mod 32 words (16-B aligned rows; the write-out reads one set's
// consecutive bins per instruction, conflict-free for any stride).
__host__ __device__ inline uint32_t build_warp_stride(uint32_t nbins) { return (nbins + 31u) / 32u * 32u + 4u; }

// count of leading zeros on the ALU / FMA pipes (FLO is a variable-latency op whose
// results queue behind the tile's shared-memory reductions: 36 % short-scoreboard stalls
// in the build, r02z6).  For x < 2^23, 2^23 + x is exact as a float and its exponent field
// is 150 + msb(x); x = u >> 9 when that is non-zero (msb(u) = msb(x) + 9), else u itself:
// clz(u) = 31 - msb(u) = 158 - add - exponent field.  u = 0 gives 158 (>= 32: callers cap).
__device__ __forceinline__ uint32_t clz_alu(uint32_t u) {
    const uint32_t hi = u >> 9;
    const uint32_t x = hi ? hi : u;
    const uint32_t add = hi ? 9u : 0u;
    const float f = __fsub_rn(__uint_as_float(0x4B000000u | x), 8388608.0f);
    return 158u - add - (__float_as_uint(f) >> 23);
}

__device__ __forceinline__ uint32_t derive_cand(uint32_t v, uint32_t t, uint32_t fsh) {
    return v == kEmpty ? kEmpty : ((t << fsh) | v);
}

template <bool W32, int SB, int SPW>
__global__ void __launch_bounds__(32 * SB / SPW) build_warp_kernel(const __grid_constant__ BuildArgs a) {
    extern __shared__ __align__(16) uint32_t smem_u32[];
    const uint32_t kst = build_warp_stride(a.k);
    const uint32_t nbh = a.L * a.kp;
    const uint32_t hst = build_warp_stride(nbh);
    uint32_t *so = smem_u32;               // [SB][kst]
    uint32_t *sh = so + (size_t)SB * kst;  // [SB][hst]
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;

    const uint64_t s0 = (uint64_t)blockIdx.x * SB;
    const uint32_t nloc = (uint32_t)min((uint64_t)SB, a.n_sets - s0);
    const uint32_t j0 = warp * SPW;  // this warp's first local set
    // offsets of the warp's sets (lane t holds offsets[s0 + j0 + t], t <= SPW)
    uint64_t offl = 0;
    if (lane <= (uint32_t)SPW && j0 + lane <= nloc) offl = __ldg(a.offsets + s0 + j0 + lane);
    const uint32_t nmine = j0 < nloc ? min((uint32_t)SPW, nloc - j0) : 0u;
    const uint64_t E0 = __shfl_sync(0xFFFFFFFFu, offl, 0);
    const uint64_t E1 = __shfl_sync(0xFFFFFFFFu, offl, nmine);
    const uint32_t n = nmine ? (uint32_t)(E1 - E0) : 0u;
    uint32_t bnd[SPW];  // local element index where set j0 + t starts (none: past every element)
#pragma unroll
    for (int t = 0; t < SPW; t++) {
        const uint64_t o = __shfl_sync(0xFFFFFFFFu, offl, t);
        bnd[t] = (uint32_t)t <= nmine ? (uint32_t)(o - E0) : 0xFFFFFFFFu;
    }

    // the first batch of ids is in flight while the rows are initialised
    constexpr int kU = 8;
    const uint32_t *ids = a.ids + E0;
    uint32_t idn[kU];
#pragma unroll
    for (int u = 0; u < kU; u++) idn[u] = lane + 32u * u < n ? __ldg(ids + lane + 32u * u) : 0u;

    const uint4 e4 = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
    const uint32_t hinit = a.hder * a.kp;  // derived HOPH bins are written, not initialised (a multiple of 4)
    for (int t = 0; t < SPW; t++) {
        if ((uint32_t)t >= nmine) break;
        uint4 *r = reinterpret_cast<uint4 *>(so + (size_t)(j0 + t) * kst);
        for (uint32_t i = lane; i < kst / 4; i += 32u) r[i] = e4;
        uint4 *h = reinterpret_cast<uint4 *>(sh + (size_t)(j0 + t) * hst);
        for (uint32_t i = hinit / 4 + lane; i < hst / 4; i += 32u) h[i] = e4;
    }
    __syncwarp();

    uint32_t kap[4], mu[4];
#pragma unroll
    for (int r = 0; r < 4; r++) {
        kap[r] = a.psi.kappa[r];
        mu[r] = a.psi.mu[r];
    }
    const uint32_t mask = a.psi.mask, pshift = a.psi.shift, hmul = a.psi.hmul, hsh = a.psi.hsh;
    const uint32_t fsh = a.flat.shift, fmask = (1u << a.flat.shift) - 1u;
    const uint32_t vsh = 32u - a.log2V, Lm1 = a.L - 1u, lkp = a.log2kp, kpw = a.kp;
    const uint32_t osh = 32u - a.log2V + a.log2kp, bsh = 32u - a.log2kp;
    const uint32_t hthr = a.hder ? (0xFFFFFFFFu << (32u - a.hder)) : 0u;  // t >= hthr <=> group >= hder
    const uint32_t so_w = smem_addr(so) + 4u * j0 * kst, sh_w = smem_addr(sh) + 4u * j0 * hst;

    for (uint32_t base = 0; base < n; base += 32u * kU) {
        uint32_t id[kU];
#pragma unroll
        for (int u = 0; u < kU; u++) id[u] = idn[u];
        const uint32_t nb = base + 32u * kU;
        if (nb < n) {
#pragma unroll
            for (int u = 0; u < kU; u++) idn[u] = nb + lane + 32u * u < n ? __ldg(ids + nb + lane + 32u * u) : 0u;
        }
        // one element: both layouts' bin minima (hthr: only groups past the derived ones)
        auto one = [&](uint32_t e, uint32_t x) {
            uint32_t jl = 0;
#pragma unroll
            for (int t = 1; t < SPW; t++) jl += e >= bnd[t] ? 1u : 0u;
            const uint32_t p = psi_pass<W32>(kap, mu, mask, pshift, hmul, hsh, x);
            asm volatile("red.shared.min.u32 [%0], %1;" ::"r"(so_w + 4u * (jl * kst + (p >> fsh))), "r"(p & fmask)
                         : "memory");
            // (branch-free: the HOPH update is predicated on t >= hthr, always true without derivation)
            const uint32_t t = p << vsh;
            const uint32_t g = min(clz_alu(~t), Lm1);
            const uint32_t sc = g + (g < Lm1 ? 1u : 0u);
            const uint32_t y = t << sc;
            const uint32_t hb = y >> bsh;
            const uint32_t ho = __funnelshift_rc(y << lkp, 0u, osh + sc);
            asm volatile(
                "{\n\t.reg .pred q;\n\tsetp.ge.u32 q, %2, %3;\n\t@q red.shared.min.u32 [%0], %1;\n}" ::"r"(
                    sh_w + 4u * (jl * hst + g * kpw + hb)),
                "r"(ho), "r"(t), "r"(hthr)
                : "memory");
        };
        if (nb <= n) {  // a whole batch (warp-uniform): no per-element guard, so the 8 elements'
                        // hashes interleave (the clz of the group lookup is a variable-latency op)
#pragma unroll
            for (int u = 0; u < kU; u++) one(base + lane + 32u * u, id[u]);
        } else {
#pragma unroll
            for (int u = 0; u < kU; u++) {
                const uint32_t e = base + lane + 32u * u;
                if (e < n) one(e, id[u]);
            }
        }
    }
    __syncwarp();

    // derived HOPH groups: lane = 4 OPH bins b .. b+3 < k - k / 2^hder (one group: group
    // boundaries are multiples of k / 2^hder >= k' >= 4); g = leading ones of b (log2 k
    // bits), M_g = 2^lm OPH bins per HOPH bin, aligned
    if (a.hder) {
        const uint32_t log2k = a.log2V - fsh;
        const uint32_t nq4 = (a.k - (a.k >> a.hder)) / 4u;
        const uint32_t M0q = 1u << (log2k - lkp - 1u);  // M_0 (M_0 / 4 lanes per HOPH bin of group 0)
        for (int t = 0; t < SPW; t++) {
            if ((uint32_t)t >= nmine) break;
            const uint4 *r4 = reinterpret_cast<const uint4 *>(so + (size_t)(j0 + t) * kst);
            uint32_t *h = sh + (size_t)(j0 + t) * hst;
            for (uint32_t q0 = 0; q0 < nq4; q0 += 32u) {
                const uint32_t q = q0 + lane, b = 4u * q;
                const bool in = q < nq4;
                const uint4 v = in ? r4[q] : e4;
                const uint32_t g = in ? (uint32_t)__clz(~(b << (32u - log2k))) : 0u;
                const uint32_t lm = log2k - lkp - 1u - g;  // log2 M_g
                const uint32_t M1 = (1u << lm) - 1u;
                const uint32_t c0 = derive_cand(v.x, b & M1, fsh), c1 = derive_cand(v.y, (b + 1u) & M1, fsh);
                const uint32_t c2 = derive_cand(v.z, (b + 2u) & M1, fsh), c3 = derive_cand(v.w, (b + 3u) & M1, fsh);
                uint32_t c = min(min(c0, c1), min(c2, c3));
                for (uint32_t d = 1; 4u * d < M0q; d <<= 1) {  // warp-uniform trip count
                    const uint32_t o = __shfl_xor_sync(0xFFFFFFFFu, c, d);
                    if (4u * d < (1u << lm)) c = min(c, o);
                }
                if (in) {
                    const uint32_t hb = g * kpw + ((b - (a.k - (a.k >> g))) >> lm);
                    if (lm >= 2) {
                        if ((b & M1) == 0u) h[hb] = c;
                    } else if (lm == 1) {
                        *reinterpret_cast<uint2 *>(h + hb) = make_uint2(min(c0, c1), min(c2, c3));
                    } else {
                        *reinterpret_cast<uint4 *>(h + hb) = make_uint4(c0, c1, c2, c3);
                    }
                }
            }
        }
    }
    __syncthreads();
    write_sketch<SB>(so, kst, a.k, nloc, a.oph, a.oph_empty, a.ld, s0);
    write_sketch<SB>(sh, hst, nbh, nloc, a.hoph, a.hoph_empty, a.ld, s0);
}

// ---------------------------------------------------------------------------
// K2: MinWise build.  One CTA = 8 consecutive sets x all k permutations; a
// thread owns permutation i (keys derived on the fly from the counter-based
// splitmix64 stream, R30) and keeps 8 running minima in registers; the
// sets' ids are staged through shared memory in chunks.
// ---------------------------------------------------------------------------
constexpr uint32_t kMwChunk = 8192;

template <bool W32, uint32_t kMwSets>
__global__ void __launch_bounds__(256) minwise_kernel(const __grid_constant__ MinwiseArgs a) {
    __shared__ uint64_t offs[kMwSets + 1];
    __shared__ uint32_t ids[kMwChunk];
    const uint64_t s0 = (uint64_t)blockIdx.x * kMwSets;
    const uint32_t nloc = (uint32_t)min((uint64_t)kMwSets, a.n_sets - s0);
    if (threadIdx.x <= nloc) offs[threadIdx.x] = a.offsets[s0 + threadIdx.x];
    __syncthreads();
    const uint64_t e0 = offs[0], e1 = offs[nloc];
    const uint32_t mask = a.w >= 32 ? 0xFFFFFFFFu : ((1u << a.w) - 1);
    const uint32_t shift = (a.w + 1) / 2;
    const bool pow2 = a.V == (1ull << a.w);
    const uint64_t gamma = 0x9E3779B97F4A7C15ull;

    // permutations i0 + threadIdx.x; grid.y > 1 splits them over CTAs (small collections)
    for (uint32_t i0 = blockIdx.y * blockDim.x; i0 < a.k; i0 += blockDim.x * gridDim.y) {  // uniform over the CTA
        const uint32_t i = i0 + threadIdx.x;
        uint32_t kappa[4], mu[4];
        {
            const uint64_t seed_i = splitmix64_mix((a.seed ^ 0x6D696E7769736521ull) + (uint64_t)(i + 1) * gamma);
#pragma unroll
            for (int r = 0; r < 4; r++) {
                kappa[r] = (uint32_t)splitmix64_mix(seed_i + (uint64_t)(2 * r + 1) * gamma) & mask;
                mu[r] = ((uint32_t)splitmix64_mix(seed_i + (uint64_t)(2 * r + 2) * gamma) & mask) | 1u;
            }
        }
        uint32_t mn[kMwSets];
#pragma unroll
        for (uint32_t j = 0; j < kMwSets; j++) mn[j] = 0xFFFFFFFFu;
        for (uint64_t c0 = e0; c0 < e1; c0 += kMwChunk) {
            const uint32_t cn = (uint32_t)min((uint64_t)kMwChunk, e1 - c0);
            __syncthreads();
            for (uint32_t t = threadIdx.x; t < cn; t += blockDim.x) ids[t] = __ldg(a.ids + c0 + t);
            __syncthreads();
            if (i < a.k) {
#pragma unroll
                for (uint32_t j = 0; j < kMwSets; j++) {
                    if (j >= nloc) break;
                    const uint64_t lo = max(offs[j], c0), hi = min(offs[j + 1], c0 + cn);
                    uint32_t m = mn[j];
                    if (!W32 && pow2) {
                        // w < 32: two elements per step, the pair's minimum and the running one in
                        // one 3-input VIMNMX3 (the ALU pipe bounds this loop; image-like 263 -> 241
                        // ms; the w = 32 loop already fuses its minima and measured slower this way)
                        // (a set outside this chunk has hi < lo: an empty range)
                        uint32_t e = (uint32_t)(lo - c0);
                        const uint32_t end = hi > lo ? (uint32_t)(hi - c0) : e;
                        for (; e + 1 < end; e += 2) {
                            const uint32_t x0 = psi_pass<W32>(kappa, mu, mask, shift, a.hmul, a.hsh, ids[e]);
                            const uint32_t x1 = psi_pass<W32>(kappa, mu, mask, shift, a.hmul, a.hsh, ids[e + 1]);
                            m = min(m, min(x0, x1));
                        }
                        if (e < end) m = min(m, psi_pass<W32>(kappa, mu, mask, shift, a.hmul, a.hsh, ids[e]));
                    } else {
                        for (uint64_t e = lo; e < hi; e++) {
                            uint32_t x = psi_pass<W32>(kappa, mu, mask, shift, a.hmul, a.hsh, ids[e - c0]);
                            if (!pow2)
                                while ((uint64_t)x >= a.V) x = psi_pass<W32>(kappa, mu, mask, shift, a.hmul, a.hsh, x);
                            m = min(m, x);
                        }
                    }
                    mn[j] = m;
                }
            }
        }
        if (i < a.k) {
#pragma unroll
            for (uint32_t j = 0; j < kMwSets; j++)
                if (j < nloc) a.mw[(uint64_t)i * a.ld + s0 + j] = (offs[j] == offs[j + 1]) ? kEmpty : mn[j];
        }
    }
    if (blockIdx.y == 0 && threadIdx.x < nloc) a.flags[s0 + threadIdx.x] = (offs[threadIdx.x] == offs[threadIdx.x + 1]) ? 1 : 0;
}

// ---------------------------------------------------------------------------
// query preparation (row a5): remap the query-side empty bin to a value no
// stored bin holds (so equality alone decides a match, R5), pad to whole
// query blocks, and emit a bin-major copy (scan) and a query-major copy
// (survivor levels).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) prep_kernel(const __grid_constant__ PrepArgs a) {
    // values: 32 (bins) x 32 (queries) tiles through shared memory, so that both the bin-major
    // QT and the query-major QM are written coalesced (the direct QM scatter wrote one 32-B
    // sector per 4-B value: scale-shard HOPH, 16,384 queries x 832 bins, 150 us per call)
    __shared__ uint32_t tile[32][33];
    const uint32_t tx = threadIdx.x & 31u, ty = threadIdx.x >> 5;  // 8 rows of 32
    const uint64_t nqt = (a.ldq + 31) / 32, ntile = (uint64_t)((a.nb + 31) / 32) * nqt;
    for (uint64_t t = blockIdx.x; t < ntile; t += gridDim.x) {
        const uint32_t b0 = (uint32_t)(t / nqt) * 32u;
        const uint64_t q0 = (t % nqt) * 32u;
        for (uint32_t r = ty; r < 32u; r += 8u) {
            const uint32_t b = b0 + r;
            const uint64_t q = q0 + tx;
            uint32_t v = 0u;
            if (b < a.nb && q < a.ldq) {
                if (q < a.n_q) {
                    v = a.values[(uint64_t)b * a.ld_in + q];
                    if (a.remap && v == kEmpty) v = kQueryEmpty;
                } else {
                    v = a.remap ? kQueryEmpty : 0u;
                }
                a.QT[(uint64_t)b * a.ldq + q] = v;
            }
            tile[r][tx] = v;
        }
        __syncthreads();
        for (uint32_t r = ty; r < 32u; r += 8u) {
            const uint64_t q = q0 + r;
            const uint32_t b = b0 + tx;
            if (q < a.n_q && b < a.nb) a.QM[q * a.nb + b] = tile[tx][r];
        }
        __syncthreads();
    }
    if (a.empty) {
        const uint64_t n_w = (uint64_t)a.nw * a.ldq;
        for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < n_w;
             idx += (uint64_t)gridDim.x * blockDim.x) {
            const uint32_t w = (uint32_t)(idx / a.ldq), q = (uint32_t)(idx % a.ldq);
            const uint32_t m = q < a.n_q ? a.empty[(uint64_t)w * a.ld_in + q] : 0u;
            a.QE[idx] = m;
            if (q < a.n_q) a.QEM[(uint64_t)q * a.nw + w] = m;
        }
    }
    if (a.flags)
        for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < a.ldq;
             q += (uint64_t)gridDim.x * blockDim.x)
            a.qflags[q] = q < a.n_q ? a.flags[q] : 1;
}

// ---------------------------------------------------------------------------
// emission helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long warp_append(bool pred, unsigned long long *counter) {
    const unsigned m = __ballot_sync(0xFFFFFFFFu, pred);
    if (m == 0) return ~0ull;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(counter, (unsigned long long)__popc(m));
    base = __shfl_sync(0xFFFFFFFFu, base, leader);
    return base + __popc(m & ((1u << lane) - 1u));
}

// termination-level histogram: add the warp's per-lane counts of pairs decided at
// `level` (warp-uniform; all 32 lanes call)
__device__ __forceinline__ void hist_add(unsigned long long *hist, uint32_t level, uint32_t n) {
    if (!hist) return;
    const uint32_t tot = __reduce_add_sync(0xFFFFFFFFu, n);
    if ((threadIdx.x & 31u) == 0 && tot) atomicAdd(hist + level, (unsigned long long)tot);
}

__device__ __forceinline__ void write_hit(oph_hit *dst, uint32_t q, uint32_t set_id, uint32_t n_mb, uint32_t n_excl,
                                          uint32_t groups, uint32_t verdict, uint32_t flags, float est) {
    uint32_t *d = reinterpret_cast<uint32_t *>(dst);
    d[0] = q;
    d[1] = set_id;
    d[2] = (n_mb & 0xFFFFu) | (n_excl << 16);
    d[3] = (groups & 0xFFu) | ((verdict & 0xFFu) << 8) | ((flags & 0xFFu) << 16);
    d[4] = __float_as_uint(est);
}

// emit one decided pair: dense -> fixed slot; threshold -> append if Similar.
// Must be called by all 32 lanes (warp-aggregated append).
__device__ __forceinline__ void emit(const OutArgs &o, bool valid, uint32_t q, uint64_t s, uint32_t n_mb,
                                     uint32_t n_excl, uint32_t groups, uint32_t verdict, uint32_t flags, float est) {
    if (o.dense) {
        if (valid) write_hit(o.hits + (uint64_t)q * o.n_sets + s, q, o.set_id_base + (uint32_t)s, n_mb, n_excl, groups,
                             verdict, flags, est);
        return;
    }
    const bool h = valid && verdict;
    const unsigned long long idx = warp_append(h, o.count);
    if (h && idx < o.cap) write_hit(o.hits + idx, q, o.set_id_base + (uint32_t)s, n_mb, n_excl, groups, verdict, flags, est);
}

// excluded bins among bins [0, nbins) of a pair, from its two mask columns
__device__ __forceinline__ uint32_t popc_masked(uint32_t qm, uint32_t sm, uint32_t joint, uint32_t w, uint32_t nbins) {
    uint32_t x = joint ? (qm & sm) : (qm | sm);
    const uint32_t lo = 32 * w;
    if (nbins < lo + 32) x &= (nbins <= lo) ? 0u : ((1u << (nbins - lo)) - 1u);
    return __popc(x);
}

// ---------------------------------------------------------------------------
// K3: the collection scan.  CTA = 128 threads; a thread owns SPT consecutive
// sets (one vectorised, coalesced load per bin: a warp reads 32*SPT
// consecutive words of one bin row) and B query counters per set in
// registers; the query block's values sit in shared memory (bin-major, read
// as broadcast 128-bit loads).  grid.x = query blocks (fastest, so CTAs that
// share a set tile run together and hit L2), grid.y = groups of
// tiles_per_cta set tiles.
// ---------------------------------------------------------------------------
template <int SPT>
struct VecT;
template <>
struct VecT<2> {
    using T = uint2;
};
template <>
struct VecT<4> {
    using T = uint4;
};

template <int SPT>
__device__ __forceinline__ void load_vals(const uint32_t *p, uint32_t (&v)[SPT]) {
    static_assert(SPT == 1 || SPT == 2 || SPT == 4, "sets per thread: 1, 2 or 4");
    if constexpr (SPT == 1) {
        v[0] = __ldg(p);  // a gathered (list-mode) set: only 4-byte aligned
    } else if constexpr (SPT == 2) {
        const uint2 x = __ldg(reinterpret_cast<const uint2 *>(p));
        v[0] = x.x;
        v[1] = x.y;
    } else {
        const uint4 x = __ldg(reinterpret_cast<const uint4 *>(p));
        v[0] = x.x;
        v[1] = x.y;
        v[2] = x.z;
        v[3] = x.w;
    }
}

// dst[i] = src[(row0 + i / B) * ldq + col0 + i % B] for i < rows * B: a query block's
// columns of the prepared bin-major query matrix into shared memory, 8 loads in
// flight per thread (the copy is on every CTA's critical path before its first tile)
template <int B>
__device__ __forceinline__ void load_query_block(uint32_t *dst, const uint32_t *src, uint64_t ldq, uint64_t row0,
                                                 uint64_t col0, uint32_t rows) {
    constexpr int kIn = 8;
    const uint32_t n = rows * B;
    for (uint32_t i0 = 0; i0 < n; i0 += kIn * blockDim.x) {
        uint32_t t[kIn];
#pragma unroll
        for (int u = 0; u < kIn; u++) {
            const uint32_t i = i0 + u * blockDim.x + threadIdx.x;
            t[u] = i < n ? __ldg(src + (row0 + i / B) * ldq + col0 + (i % B)) : 0u;
        }
#pragma unroll
        for (int u = 0; u < kIn; u++) {
            const uint32_t i = i0 + u * blockDim.x + threadIdx.x;
            if (i < n) dst[i] = t[u];
        }
    }
}

constexpr uint32_t kScanChunk = 512;  // query bins held in shared memory at once

// c += (v == q) as ISETP (ALU pipe) + predicated IMAD c = c*one + one (FMA
// pipe), `one` a runtime 1 the compiler cannot fold: 2 instructions split
// over both integer pipes.  (The C++ form compiles to 3 instructions, a
// predicated IADD puts both on the ALU pipe, which then bounds the scan.)
__device__ __forceinline__ void acc_eq(uint32_t &c, uint32_t v, uint32_t q, uint32_t one, uint32_t inc) {
    asm("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %1, %2;\n\t@p mad.lo.u32 %0, %0, %3, %4;\n}"
        : "+r"(c)
        : "r"(v), "r"(q), "r"(one), "r"(inc));
}

template <int B, int SPT, int U>
__device__ __forceinline__ void scan_bins(const uint32_t *Fp, uint32_t ldb, const uint32_t *qs, uint32_t b0,
                                          uint32_t nb, uint32_t (&cnt)[SPT][B], uint32_t one, uint32_t inc) {
    // Fp points at a readable column of every row (the caller clamps threads past the
    // last set), so no load is predicated; software pipeline: the U rows of the next
    // group load while this group compares (HBM latency behind ~2*SPT*B*U instructions)
    const char *base = reinterpret_cast<const char *>(Fp);
    auto load_row = [&](uint32_t r, uint32_t (&dst)[SPT]) {
        load_vals<SPT>(reinterpret_cast<const uint32_t *>(base + (uint64_t)(b0 + r) * ldb), dst);
    };
    auto compare_row = [&](const uint32_t (&vr)[SPT], uint32_t row) {
        const uint4 *q4 = reinterpret_cast<const uint4 *>(qs + (size_t)row * B);
#pragma unroll
        for (int q = 0; q < B / 4; q++) {
            const uint4 x = q4[q];
#pragma unroll
            for (int j = 0; j < SPT; j++) {
                acc_eq(cnt[j][4 * q + 0], vr[j], x.x, one, inc);
                acc_eq(cnt[j][4 * q + 1], vr[j], x.y, one, inc);
                acc_eq(cnt[j][4 * q + 2], vr[j], x.z, one, inc);
                acc_eq(cnt[j][4 * q + 3], vr[j], x.w, one, inc);
            }
        }
    };
    uint32_t b = 0;
    if (U <= nb) {
        uint32_t v[U][SPT];
#pragma unroll
        for (int u = 0; u < U; u++) load_row(u, v[u]);
        for (; b + 2 * U <= nb; b += U) {
            uint32_t vn[U][SPT];
#pragma unroll
            for (int u = 0; u < U; u++) load_row(b + U + u, vn[u]);
#pragma unroll
            for (int u = 0; u < U; u++) compare_row(v[u], b + u);
#pragma unroll
            for (int u = 0; u < U; u++)
#pragma unroll
                for (int j = 0; j < SPT; j++) v[u][j] = vn[u][j];
        }
#pragma unroll
        for (int u = 0; u < U; u++) compare_row(v[u], b + u);
        b += U;
    }
    for (; b < nb; b++) {
        uint32_t vr[SPT];
        load_row(b, vr);
        compare_row(vr, b);
    }
}

// The same scan with two 16-bit counters per register (query 2i in the low half,
// 2i + 1 in the high half; nscan <= 65535, so a half never carries): the predicated
// IMAD adds 1 or 1 << 16, still 2 instructions per compare, half the counter
// registers -- more CTAs per SM at every query block.
template <int B, int SPT, int U>
__device__ __forceinline__ void scan_bins_packed(const uint32_t *Fp, uint32_t ldb, const uint32_t *qs, uint32_t b0,
                                                 uint32_t nb, uint32_t (&cp)[SPT][B / 2], uint32_t one, uint32_t hi) {
    // Fp points at a readable column of every row (the caller clamps threads past the
    // last set), so no load is predicated: row r is one IMAD.WIDE.U32 off the base
    const char *base = reinterpret_cast<const char *>(Fp);
    auto load_row = [&](uint32_t r, uint32_t (&dst)[SPT]) {
        load_vals<SPT>(reinterpret_cast<const uint32_t *>(base + (uint64_t)(b0 + r) * ldb), dst);
    };
    auto compare_row = [&](const uint32_t (&vr)[SPT], uint32_t row) {
        const uint4 *q4 = reinterpret_cast<const uint4 *>(qs + (size_t)row * B);
#pragma unroll
        for (int q = 0; q < B / 4; q++) {
            const uint4 x = q4[q];
#pragma unroll
            for (int j = 0; j < SPT; j++) {
                acc_eq(cp[j][2 * q + 0], vr[j], x.x, one, one);
                acc_eq(cp[j][2 * q + 1], vr[j], x.z, one, one);
                acc_eq(cp[j][2 * q + 0], vr[j], x.y, one, hi);
                acc_eq(cp[j][2 * q + 1], vr[j], x.w, one, hi);
            }
        }
    };
    uint32_t b = 0;
    if (U <= nb) {
        // software pipeline: the U rows of the next group load while this group compares
        uint32_t v[U][SPT];
#pragma unroll
        for (int u = 0; u < U; u++) load_row(u, v[u]);
        for (; b + 2 * U <= nb; b += U) {
            uint32_t vn[U][SPT];
#pragma unroll
            for (int u = 0; u < U; u++) load_row(b + U + u, vn[u]);
#pragma unroll
            for (int u = 0; u < U; u++) compare_row(v[u], b + u);
#pragma unroll
            for (int u = 0; u < U; u++)
#pragma unroll
                for (int j = 0; j < SPT; j++) v[u][j] = vn[u][j];
        }
#pragma unroll
        for (int u = 0; u < U; u++) compare_row(v[u], b + u);
        b += U;
    }
    for (; b < nb; b++) {
        uint32_t vr[SPT];
        load_row(b, vr);
        compare_row(vr, b);
    }
}

// CTAs per SM by query block (packed counters, scan_bins_packed):
//   B = 32: 4 (128 registers, 48 B of spills outside the compare loop; 1,862 us on
//           image-like at Q = 32 vs 2,013 at 3 CTAs; unpacked 3 CTAs: 1,871)
//   B = 16: 5 (96 registers; 1,168 -> 913 us on image-like at Q = 16)
//   B = 8 / 4 (HBM-bound): 7 / 8 (72 / 64 registers): the bin-major strip read needs
//           ~32 warps per SM to reach the copy bandwidth (scripts/access_bench.cu:
//           12 / 24 / 32 warps per SM stream 3.1-3.9 / 5.1-5.8 / 6.2-6.7 TB/s,
//           whatever the loads in flight per thread)
template <int B>
constexpr int scan_min_ctas() {
    return B <= 4 ? 8 : (B <= 8 ? 7 : (B <= 16 ? 5 : 4));
}
template <int B, int SPT, bool LIST>
__global__ void __launch_bounds__(128, scan_min_ctas<B>()) scan_kernel(const __grid_constant__ ScanArgs a) {
    static_assert(!LIST || SPT == 1, "list mode scans one gathered set per thread");
    constexpr int U = 4;  // bins in flight per thread
    extern __shared__ __align__(16) uint32_t sm[];
    const uint32_t qs_bins = min(a.nscan, kScanChunk);
    uint32_t *qs = sm;                                  // [qs_bins][B]
    uint32_t *qe = qs + (size_t)qs_bins * B;            // [nw_load][B]
    uint32_t *qf = qe + (size_t)a.nw_load * B;          // [B] MinWise flags

    if (LIST && (uint64_t)blockIdx.y * 128 * SPT >= *a.list_count) return;  // nothing listed for this CTA
    const uint32_t qb0 = blockIdx.x * B;                // chunk-local first query
    const uint64_t col0 = (uint64_t)a.q_col0 + qb0;     // column in the prepared arrays
    const bool one_chunk = a.nscan <= kScanChunk;
    if (one_chunk)
        load_query_block<B>(qs, a.QT, a.ldq, 0, col0, a.nscan);
    if (a.E)
        load_query_block<B>(qe, a.QE, a.ldq, 0, col0, a.nw_load);
    if (a.method == kMinwise)
        for (uint32_t i = threadIdx.x; i < B; i += blockDim.x) qf[i] = a.qflags[col0 + i];
    __syncthreads();

    const uint64_t tile_sets = 128ull * SPT;
    // list mode: items = listed sets; else items = sets [s_begin, n_sets)
    const uint64_t n_items = LIST ? *a.list_count : a.n_sets - a.s_begin;
    const uint64_t ntiles = (n_items + tile_sets - 1) / tile_sets;
    const uint64_t t_first = LIST ? blockIdx.y : (uint64_t)blockIdx.y * a.tiles_per_cta;
    const uint64_t t_end = LIST ? ntiles : min(ntiles, (uint64_t)(blockIdx.y + 1) * a.tiles_per_cta);
    const uint64_t t_step = LIST ? gridDim.y : 1;
    for (uint64_t t = t_first; t < t_end; t += t_step) {
        const uint64_t i0 = t * tile_sets + threadIdx.x * SPT;
        const bool active = i0 < n_items;
        const uint64_t s0 = LIST ? (active ? a.set_list[i0] : 0ull) : a.s_begin + i0;
        uint32_t cp[SPT][B / 2];  // packed counters (scan_bins_packed)
#pragma unroll
        for (int j = 0; j < SPT; j++)
#pragma unroll
            for (int q = 0; q < B / 2; q++) cp[j][q] = 0;
        const uint32_t hi = a.one << 16;

        // threads past the last item read (and never use) the row's last SPT columns
        const uint32_t *Fp = a.F + (active ? s0 : a.ld - SPT);
        const uint32_t ldb = (uint32_t)(a.ld * 4u);  // < 2^32 (launcher)
        if (one_chunk) {
            scan_bins_packed<B, SPT, U>(Fp, ldb, qs, 0, a.nscan, cp, a.one, hi);
        } else {
            for (uint32_t c0 = 0; c0 < a.nscan; c0 += kScanChunk) {
                const uint32_t cn = min(kScanChunk, a.nscan - c0);
                __syncthreads();
                load_query_block<B>(qs, a.QT, a.ldq, c0, col0, cn);
                __syncthreads();
                scan_bins_packed<B, SPT, U>(Fp, ldb, qs, c0, cn, cp, a.one, hi);
            }
        }

        // ---------------- epilogue: decisions and emission, one set column at a time
#define CNT(j, q) ((cp[j][(q) >> 1] >> (((q) & 1) * 16)) & 0xFFFFu)
#pragma unroll
        for (int j = 0; j < SPT; j++) {
            const uint64_t s = s0 + j;
            const bool sv = active && (LIST || s < a.n_sets);
            uint32_t hit_mask = 0, surv_mask = 0, dec_mask = 0;
            if (a.final_) {
                uint32_t ex[B];
#pragma unroll
                for (int q = 0; q < B; q++) ex[q] = 0;
                uint32_t sflag = 0;
                if (a.method == kMinwise) {
                    sflag = sv ? a.sflags[s] : 1u;
                } else {
                    for (uint32_t w = 0; w < a.nw_load; w++) {
                        const uint32_t es = sv ? __ldg(a.E + (uint64_t)w * a.ld + s) : 0u;
#pragma unroll
                        for (int q = 0; q < B; q++) ex[q] += popc_masked(qe[w * B + q], es, a.joint, w, a.nbins_total);
                    }
                }
#pragma unroll
                for (int q = 0; q < B; q++) {
                    const bool valid = sv && (qb0 + q < a.nq);
                    uint32_t den, undef;
                    if (a.method == kMinwise) {
                        den = a.nbins_total;
                        undef = sflag | qf[q];
                    } else {
                        den = a.nbins_total - ex[q];
                        undef = den == 0;
                    }
                    const uint32_t verdict = !undef && (uint64_t)CNT(j, q) * a.t_den >= (uint64_t)a.t_num * den;
                    hit_mask |= (uint32_t)(valid && verdict) << q;
                    dec_mask |= (uint32_t)valid << q;
                }
                hist_add(a.out.hist, a.level, __popc(dec_mask));
                const bool any = __any_sync(0xFFFFFFFFu, a.out.dense ? dec_mask != 0 : hit_mask != 0);
                if (any) {
#pragma unroll
                    for (int q = 0; q < B; q++) {
                        const bool valid = (dec_mask >> q) & 1u;
                        uint32_t den, undef;
                        if (a.method == kMinwise) {
                            den = a.nbins_total;
                            undef = sflag | qf[q];
                        } else {
                            den = a.nbins_total - ex[q];
                            undef = den == 0;
                        }
                        const uint32_t verdict = (hit_mask >> q) & 1u;
                        const float est = undef ? -1.0f : (float)CNT(j, q) / (float)den;
                        // an empty MinWise set has no sketch: nothing is compared
                        const uint32_t nmb = (a.method == kMinwise && undef) ? 0u : CNT(j, q);
                        emit(a.out, valid, (uint32_t)(col0 + q), s, nmb,
                             a.method == kMinwise ? 0u : ex[q], a.level, verdict, undef ? OPH_FLAG_UNDEFINED : 0u, est);
                    }
                }
            } else {
#pragma unroll
                for (int q = 0; q < B; q++) {
                    const bool valid = sv && (qb0 + q < a.nq);
                    const bool acc = CNT(j, q) >= a.acc_cnt, rej = (int32_t)CNT(j, q) <= a.rej_cnt;
                    hit_mask |= (uint32_t)(valid && acc) << q;
                    dec_mask |= (uint32_t)(valid && (acc || rej)) << q;
                    surv_mask |= (uint32_t)(valid && !acc && !rej) << q;
                }
                hist_add(a.out.hist, a.level, __popc(dec_mask));
                const bool any_emit = __any_sync(0xFFFFFFFFu, a.out.dense ? dec_mask != 0 : hit_mask != 0);
                if (any_emit) {
#pragma unroll
                    for (int q = 0; q < B; q++) {
                        const bool e = a.out.dense ? ((dec_mask >> q) & 1u) : ((hit_mask >> q) & 1u);
                        uint32_t ex = 0;
                        if (e)
                            for (uint32_t w = 0; w < a.nw_load; w++)
                                ex += popc_masked(qe[w * B + q], __ldg(a.E + (uint64_t)w * a.ld + s), a.joint, w, a.nscan);
                        emit(a.out, (dec_mask >> q) & 1u, (uint32_t)(col0 + q), s, CNT(j, q), ex, a.level,
                             (hit_mask >> q) & 1u, OPH_FLAG_EARLY, -1.0f);
                    }
                }
                if (__any_sync(0xFFFFFFFFu, surv_mask != 0)) {
#pragma unroll
                    for (int q = 0; q < B; q++) {
                        const bool sp = (surv_mask >> q) & 1u;
                        const unsigned long long idx = warp_append(sp, a.surv_count);
                        if (sp && idx < a.surv_cap) {  // past capacity: counted, the host redoes the chunk
                            a.surv.q[idx] = (uint32_t)(col0 + q);
                            a.surv.s[idx] = (uint32_t)s;
                            a.surv.state[idx] = a.w1 * CNT(j, q);  // S_1 = c_1 M_1 (GOPH: M_c)
                            a.surv.nmb[idx] = CNT(j, q);
                        }
                    }
                }
            }
        }
    }
}

#undef CNT

// ---------------------------------------------------------------------------
// K3' PROBE: the same scan as a hash join, streaming the collection once per
// pass of up to kJoinMaxQ queries.  A query bin matches a set bin only when
// the values are equal, so instead of testing every (query, set, bin) triple
// the pass's query values of each scanned bin go into an exact hash table
// (L2) and a blocked Bloom filter (table_kernel); the join kernel tests every
// set bin against the filter held in shared memory and verifies the rare
// positives in the exact table: work ~ N * bins + matches instead of
// Q * N * bins.  Per set, the matched queries and their counts are collected
// in shared memory; pairs with no matched bin have N_mb = 0 (full OPH /
// MinWise: never Similar for T > 0; GOPH / HOPH: the host only picks PROBE
// when state 0 is rejected at the scanned level), so only listed pairs are
// decided and emitted.  A set that matches more than kJoinList distinct
// queries is handed to the BRUTE scan (list mode).  Threshold results only.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t probe_hash(uint32_t v, uint32_t log2S) {
    return (v * 0x9E3779B1u) >> (32 - log2S);  // Fibonacci hashing
}

// Bloom filter of one bin: 2^log2W words; value v, h = v * golden, sets two
// bits of word h >> (32 - log2W): bit umulhi(v, C) mod 32 (the high half of a
// second product depends on every bit of v; IMAD.HI issues on the FMA pipe)
// and bit h mod 32 (a bijection of v mod 32).
__device__ __forceinline__ uint32_t bloom_bits(uint32_t v, uint32_t h) {
    return __funnelshift_l(0u, 1u, __umulhi(v, 0x85EBCA6Bu)) | __funnelshift_l(0u, 1u, h);
}

// (b1 | b2) & ~word in one LOP3: zero iff both filter bits of v are set in word
__device__ __forceinline__ uint32_t bloom_miss(uint32_t v, uint32_t h, uint32_t word) {
    uint32_t z;
    asm("lop3.b32 %0, %1, %2, %3, 0x54;"
        : "=r"(z)
        : "r"(__funnelshift_l(0u, 1u, __umulhi(v, 0x85EBCA6Bu))), "r"(__funnelshift_l(0u, 1u, h)), "r"(word));
    return z;
}

__global__ void table_kernel(const __grid_constant__ TableArgs a) {
    const uint64_t S = 1ull << a.log2S;
    const uint64_t n = (uint64_t)a.nscan * a.nq;
    for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < n;
         idx += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t b = (uint32_t)(idx / a.nq), q = (uint32_t)(idx % a.nq);
        const uint64_t col = (uint64_t)a.q_col0 + q;
        if (a.minwise && a.qflags[col]) continue;       // an empty query matches nothing
        const uint32_t v = a.QT[(uint64_t)b * a.ldq + col];
        if (!a.minwise && v == kQueryEmpty) continue;   // an empty query bin matches nothing
        const unsigned long long entry = ((unsigned long long)v << 32) | (q + 1u);
        unsigned long long *T = a.table + (uint64_t)b * S;
        uint32_t h = probe_hash(v, a.log2S);
        while (atomicCAS(&T[h], 0ull, entry) != 0ull) h = (h + 1) & (uint32_t)(S - 1);
        const uint32_t hv = v * 0x9E3779B1u;
        atomicOr(a.bloom + ((uint64_t)b << a.log2W) + (hv >> (32 - a.log2W)), bloom_bits(v, hv));
    }
}

// ---- mbarrier / bulk-copy (TMA engine) primitives
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// waits for the phase of the given parity; a protocol bug traps after ~4 s
// (a failed launch) instead of hanging the device
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    if (mbar_try_wait(bar, parity)) return;
    const long long t0 = clock64();
    while (!mbar_try_wait(bar, parity))
        if (clock64() - t0 > 8000000000ll) __trap();
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

constexpr int kJoinWarps = 28;
constexpr int kJoinThreads = 32 * kJoinWarps;
// candidate queue per warp (4-B entries).  Small on purpose: the verification re-reads
// each candidate's value, which is still in L2 only if the flush follows within a few
// tiles (text-like full OPH / MinWise join: 256 entries 90 / 116 us, 128 77 / 87, 64 66 / 74,
// 32 68 / 79), and a 64-entry flush needs 2 loads in flight per lane, not 8
constexpr uint32_t kJoinQCap = 64;
constexpr uint32_t kJoinSPL = 4;                  // sets per lane (one 16-B load per bin row)
constexpr uint32_t kJoinRPT = 8;                  // bin rows per tile
constexpr uint32_t kJoinVals = kJoinSPL * kJoinRPT;  // values per lane per tile (mask bits)
constexpr uint32_t kJoinTile = 32 * kJoinSPL;     // sets per tile
constexpr uint32_t kJoinSlabWords = 16384;  // one filter buffer: 64 KB = SBN bins x W words (W = 512 / 1024 / 2048)
constexpr uint32_t kJoinMaxSlabs = 512;  // nscan <= 16384

// shared-memory carve-up of the join kernel (bytes, 128-B aligned regions)
struct JoinLayout {
    uint32_t bars, tab, lists, ovf, queue, qcount, total;
};
__host__ __device__ inline uint32_t join_align(uint32_t x) { return (x + 127u) & ~127u; }
__host__ __device__ inline JoinLayout join_layout(uint32_t W, uint32_t R, uint32_t nlist) {
    JoinLayout L;
    L.bars = 0;
    L.tab = 128;
    L.lists = L.tab + 2 * kJoinSlabWords * 4;
    L.ovf = join_align(L.lists + nlist * R * 4);
    L.queue = join_align(L.ovf + R / 8);
    L.qcount = L.queue + kJoinWarps * kJoinQCap * 4;  // per slab: tile counter, done counter
    L.total = join_align(L.qcount + 2 * kJoinMaxSlabs * 4);
    return L;
}

// count one more matched bin of query q for the set at local index sl:
// list entry = (q + 1) << 16 | count, 0 = free; a full list flags the set
__device__ __forceinline__ void list_add(uint32_t *lists, uint32_t R, uint32_t nlist, uint32_t *ovf, uint32_t sl,
                                         uint32_t q) {
    const uint32_t key = (q + 1u) << 16;
#pragma unroll
    for (int e = 0; e < kJoinList; e++) {
        if ((uint32_t)e == nlist) break;
        uint32_t *p = lists + e * R + sl;
        uint32_t x = *(volatile uint32_t *)p;
        for (;;) {
            if (x == 0u) {
                const uint32_t old = atomicCAS(p, 0u, key | 1u);
                if (old == 0u) return;
                x = old;
                continue;
            }
            if ((x & 0xFFFF0000u) == key) {
                atomicAdd(p, 1u);
                return;
            }
            break;
        }
    }
    atomicOr(ovf + (sl >> 5), 1u << (sl & 31));
}

// verify n queued filter positives (warp-collective; entry = local set | bin << 16):
// every query whose value of that bin equals the set's value counts one matched
// bin.  The values are re-read from the collection (the tile was just streamed,
// so L2 hits), and each lane issues all its loads before walking any chain.
__device__ __noinline__ void join_flush(const ProbeArgs &a, uint64_t s_lo, uint32_t *lists, uint32_t *ovf,
                                        const uint32_t *queue, uint32_t n) {
    constexpr int kPer = kJoinQCap / 32;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t smask = (1u << a.log2S) - 1u;
    __syncwarp();  // the queue entries of every lane are visible
    uint32_t c[kPer], v[kPer];
#pragma unroll
    for (int r = 0; r < kPer; r++) {
        const uint32_t e = lane + 32u * r;
        c[r] = e < n ? queue[e] : 0xFFFFFFFFu;
        if (c[r] != 0xFFFFFFFFu) v[r] = __ldg(a.F + (uint64_t)(c[r] >> 16) * a.ld + s_lo + (c[r] & 0xFFFFu));
    }
    unsigned long long slot[kPer];
#pragma unroll
    for (int r = 0; r < kPer; r++)
        if (c[r] != 0xFFFFFFFFu)
            slot[r] = __ldg(a.table + ((uint64_t)(c[r] >> 16) << a.log2S) + probe_hash(v[r], a.log2S));
#pragma unroll
    for (int r = 0; r < kPer; r++) {
        if (c[r] == 0xFFFFFFFFu) break;
        const unsigned long long *T = a.table + ((uint64_t)(c[r] >> 16) << a.log2S);
        unsigned long long sl8 = slot[r];
        uint32_t h = probe_hash(v[r], a.log2S);
        while (sl8 != 0ull) {
            if ((uint32_t)(sl8 >> 32) == v[r]) list_add(lists, a.R, a.nlist, ovf, c[r] & 0xFFFFu, (uint32_t)sl8 - 1u);
            h = (h + 1) & smask;
            sl8 = __ldg(T + h);
        }
    }
    __syncwarp();
}

// append the positives of this lane's mask (bit i = set i / RPT, row i % RPT) to the
// warp's queue: a warp prefix sum places every lane's entries (no atomics; the
// fill level qn is warp-uniform, a register).  Lanes with <= 2 positives write
// their own; the rare lane with more (a near-duplicate set: ~25 matched rows)
// is expanded by the whole warp, one bit per lane.  A tile with more positives
// than the queue holds is verified through it in queue-sized rounds.
// queue entry of mask bit i: set sl + i / RPT, bin bin0 + i % RPT
__device__ __forceinline__ uint32_t join_entry(uint32_t sl, uint32_t bin0, uint32_t i) {
    return (sl + i / kJoinRPT) | ((bin0 + i % kJoinRPT) << 16);
}

__device__ __forceinline__ void join_push(const ProbeArgs &a, uint64_t s_lo, uint32_t cm, uint32_t sl, uint32_t bin0,
                                          uint32_t *lists, uint32_t *ovf, uint32_t *queue, uint32_t &qn) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t lt = (1u << lane) - 1u;
    for (;;) {
        const uint32_t c = __popc(cm);
        uint32_t incl = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
            if (lane >= (uint32_t)d) incl += t;
        }
        const uint32_t tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
        if (tot == 0) return;
        if (qn + tot > kJoinQCap && qn) {  // make room
            join_flush(a, s_lo, lists, ovf, queue, qn);
            qn = 0;
        }
        if (qn + tot <= kJoinQCap) {  // the common case: everything fits
            const uint32_t pos = qn + incl - c;
            if (c <= 2u) {
                uint32_t m = cm, p = pos;
                while (m) {
                    queue[p++] = join_entry(sl, bin0, __ffs(m) - 1);
                    m &= m - 1;
                }
            }
            uint32_t heavy = __ballot_sync(0xFFFFFFFFu, c > 2u);
            while (heavy) {
                const uint32_t L = __ffs(heavy) - 1;
                heavy &= heavy - 1;
                const uint32_t m = __shfl_sync(0xFFFFFFFFu, cm, L);
                const uint32_t p = __shfl_sync(0xFFFFFFFFu, pos, L);
                const uint32_t sL = __shfl_sync(0xFFFFFFFFu, sl, L);
                if ((m >> lane) & 1u) queue[p + __popc(m & lt)] = join_entry(sL, bin0, lane);
            }
            qn += tot;
            return;
        }
        // overfull tile (qn == 0, tot > capacity): queue what fits, verify, repeat
        uint32_t pos = incl - c;
        while (cm && pos < kJoinQCap) {
            queue[pos++] = join_entry(sl, bin0, __ffs(cm) - 1);
            cm &= cm - 1;
        }
        join_flush(a, s_lo, lists, ovf, queue, kJoinQCap);
        qn = 0;
    }
}

// One CTA (28 warps, one per SM) owns R consecutive sets.  Per slab of 32
// scanned bins the slab's filters (32 x kJoinW words, bin-major) sit in
// shared memory (double-buffered: the last warp to finish slab j bulk-copies
// slab j + 2, so no CTA-wide barrier between slabs); warps take 32-set tiles
// from a shared counter: lane = one set, one coalesced 4-B load per bin row,
// all 32 rows in flight at once.
template <bool MW, int LOG2W>
__global__ void __launch_bounds__(kJoinThreads, 1) join_kernel(const __grid_constant__ ProbeArgs a) {
    extern __shared__ __align__(128) unsigned char jsm[];
    constexpr uint32_t W = 1u << LOG2W;             // filter words per bin (row offsets are immediates)
    constexpr uint32_t SBN = kJoinSlabWords / W;   // bins per slab: 32 / 16 / 8
    static_assert(SBN % kJoinRPT == 0, "a slab holds whole tile row blocks");
    const uint32_t R = a.R;
    const JoinLayout Ly = join_layout(W, R, a.nlist);
    uint64_t *tfull = reinterpret_cast<uint64_t *>(jsm + Ly.bars);
    uint32_t *tab = reinterpret_cast<uint32_t *>(jsm + Ly.tab);      // [2][32][W]
    uint32_t *lists = reinterpret_cast<uint32_t *>(jsm + Ly.lists);  // [nlist][R]
    uint32_t *ovf = reinterpret_cast<uint32_t *>(jsm + Ly.ovf);      // [R / 32]
    uint32_t *queue = reinterpret_cast<uint32_t *>(jsm + Ly.queue);  // [kJoinWarps][kJoinQCap]
    uint32_t *tctl = reinterpret_cast<uint32_t *>(jsm + Ly.qcount);  // per slab: next tile, warps done

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint64_t s_lo = a.s_begin + (uint64_t)blockIdx.x * R;
    const uint32_t nset = (uint32_t)(min(s_lo + R, a.s_end) - s_lo);
    const uint32_t nslab = (a.nscan + SBN - 1) / SBN;
    const uint32_t slab_bytes = kJoinSlabWords * 4u;

    for (uint32_t x = threadIdx.x; x < a.nlist * R; x += blockDim.x) lists[x] = 0u;
    for (uint32_t x = threadIdx.x; x < R / 32; x += blockDim.x) ovf[x] = 0u;
    for (uint32_t x = threadIdx.x; x < 2 * nslab; x += blockDim.x) tctl[x] = 0u;
    if (threadIdx.x == 0) {
        mbar_init(&tfull[0], 1);
        mbar_init(&tfull[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (uint32_t j = 0; j < 2 && j < nslab; j++) {
            mbar_expect_tx(&tfull[j], slab_bytes);
            bulk_g2s(tab + (size_t)j * kJoinSlabWords, a.bloom + (size_t)j * kJoinSlabWords, slab_bytes, &tfull[j]);
        }
    }
    __syncthreads();

    uint32_t *myq = queue + warp * kJoinQCap;
    uint32_t qn = 0;  // queued positives of this warp (warp-uniform)
    constexpr uint32_t RB = SBN / kJoinRPT;  // tile row blocks per slab
    const uint32_t ntile = (nset + kJoinTile - 1) / kJoinTile * RB;
    const uint32_t ldb = (uint32_t)(a.ld * 4u);  // row stride in bytes
    for (uint32_t j = 0; j < nslab; j++) {
        const uint32_t tb = j & 1u;
        const uint32_t *tabj = tab + (size_t)tb * kJoinSlabWords;
        const uint32_t rows = min(SBN, a.nscan - SBN * j);
        const uint32_t *Fj = a.F + (uint64_t)(SBN * j) * a.ld;
        // tiles are handed out dynamically (a 28-warp SM hides the row-load latency of one
        // warp behind the others' probing; a per-warp double buffer measured slower)
        auto next_tile = [&]() {
            uint32_t t = 0;
            if (lane == 0) t = atomicAdd(&tctl[2 * j], 1u);
            return __shfl_sync(0xFFFFFFFFu, t, 0);
        };
        // tile t: sets [sb * 32 * SPL, +32 * SPL) x rows [rb * RPT, +RPT) of the slab,
        // sb = t / RB, rb = t % RB; lane = SPL adjacent sets (one vector load per row),
        // v[k * RPT + r] = set k, row r
        auto load_tile = [&](uint32_t t, uint32_t (&v)[kJoinVals]) {
            const uint32_t sb = t / RB, rb = t % RB;
            const uint32_t sl = sb * kJoinTile + lane * kJoinSPL;
            const char *Fs = reinterpret_cast<const char *>(Fj + (uint64_t)(rb * kJoinRPT) * a.ld + s_lo + sl);
            // row r at Fs + r * ldb: one IMAD.WIDE.U32 per row (ldb < 2^32, checked by the launcher);
            // default caching (an evict-first hint made the verification re-reads miss L2)
            if ((sb + 1) * kJoinTile <= nset && (rb + 1) * kJoinRPT <= rows) {  // full tile (warp-uniform): no checks
#pragma unroll
                for (int r = 0; r < (int)kJoinRPT; r++) {
                    const uint4 x = __ldg(reinterpret_cast<const uint4 *>(Fs + (uint64_t)((uint32_t)r) * ldb));
                    v[0 * kJoinRPT + r] = x.x;
                    v[1 * kJoinRPT + r] = x.y;
                    v[2 * kJoinRPT + r] = x.z;
                    v[3 * kJoinRPT + r] = x.w;
                }
            } else {
#pragma unroll
                for (int r = 0; r < (int)kJoinRPT; r++)
#pragma unroll
                    for (int k = 0; k < (int)kJoinSPL; k++)
                        v[k * kJoinRPT + r] =
                            (sl + k < nset && rb * kJoinRPT + r < rows)
                                ? __ldg(reinterpret_cast<const uint32_t *>(Fs + (uint64_t)((uint32_t)r) * ldb) + k)
                                : kEmpty;
            }
        };
        auto probe_tile = [&](uint32_t t, const uint32_t (&v)[kJoinVals]) {
            const uint32_t sb = t / RB, rb = t % RB;
            // filter test: h = v * golden; word (h >> 23) of the row's filter; both bits set -> bit of cm
            uint32_t cm = 0;
            const uint32_t *tabr = tabj + rb * kJoinRPT * W;
#pragma unroll
            for (int i = 0; i < (int)kJoinVals; i++) {
                const uint32_t r = (uint32_t)i % kJoinRPT;
                const uint32_t h = v[i] * 0x9E3779B1u;
                const uint32_t word = tabr[r * W + (h >> (32 - LOG2W))];
                const uint32_t z = bloom_miss(v[i], h, word);
                asm("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %1, 0;\n\t@p or.b32 %0, %0, %2;\n}"
                    : "+r"(cm)
                    : "r"(z), "r"(1u << i));
            }
            // rows past the scanned bins and sets past the end: the verification
            // re-reads the value from the collection, so they must not be queued
            // (an empty collection bin that passes the filter -- ~10 % of the
            // positives -- is rejected there: no query inserts the value kEmpty)
            const uint32_t sl = sb * kJoinTile + lane * kJoinSPL;
            if (!((sb + 1) * kJoinTile <= nset && (rb + 1) * kJoinRPT <= rows)) {
#pragma unroll
                for (int i = 0; i < (int)kJoinVals; i++)
                    if (sl + (uint32_t)i / kJoinRPT >= nset || rb * kJoinRPT + (uint32_t)i % kJoinRPT >= rows)
                        cm &= ~(1u << i);
            }
            join_push(a, s_lo, cm, sl, j * SBN + rb * kJoinRPT, lists, ovf, myq, qn);
        };
        mbar_wait(&tfull[tb], (j >> 1) & 1u);  // the slab's filters
        for (uint32_t t = next_tile(); t < ntile; t = next_tile()) {
            uint32_t v[kJoinVals];
            load_tile(t, v);
            probe_tile(t, v);
        }
        // the last warp done with slab j recycles its filter buffer for slab j + 2
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            if (atomicAdd(&tctl[2 * j + 1], 1u) == kJoinWarps - 1) {
                if (j + 2 < nslab) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_expect_tx(&tfull[tb], slab_bytes);
                    bulk_g2s(tab + (size_t)tb * kJoinSlabWords, a.bloom + (size_t)(j + 2) * kJoinSlabWords, slab_bytes,
                             &tfull[tb]);
                }
            }
        }
        __syncwarp();
    }
    if (qn) join_flush(a, s_lo, lists, ovf, myq, qn);
    __syncthreads();  // all counts are in

    // ---------------- epilogue: decide every listed pair (one set per lane)
    for (uint32_t base = warp * 32u; base < R; base += kJoinWarps * 32u) {
        const uint32_t sl = base + lane;
        const uint64_t s = s_lo + sl;
        const bool act = sl < nset && !(MW && a.sflags[s]);
        const bool of = act && ((ovf[sl >> 5] >> (sl & 31)) & 1u);
        {   // overflowing sets go to the BRUTE list scan
            const unsigned long long idx = warp_append(of, a.ovf_count);
            if (of) a.ovf_list[idx] = (uint32_t)s;
        }
        uint32_t n_surv = 0;  // this set's pairs that go on to the next level
#pragma unroll 1
        for (int e = 0; e < (int)a.nlist; e++) {
            const uint32_t x = (act && !of) ? lists[e * R + sl] : 0u;
            const bool has = x != 0u;
            if (!__any_sync(0xFFFFFFFFu, has)) break;
            uint32_t q = 0, m = 0, ex = 0, flags = 0, verdict = 0;
            bool surv = false;
            float est = -1.0f;
            u128_t st = 0;
            if (has) {
                q = (x >> 16) - 1u;
                m = x & 0xFFFFu;
                const uint32_t qg = a.q_col0 + q;
                if (a.final_) {
                    uint32_t den;
                    bool undef;
                    if (MW) {
                        den = a.nbins_total;
                        undef = a.qflags[qg] != 0;
                    } else {
                        for (uint32_t w = 0; w < a.nw; w++)
                            ex += popc_masked(__ldg(a.QEM + (uint64_t)qg * a.nw + w), __ldg(a.E + (uint64_t)w * a.ld + s),
                                              a.joint, w, a.nbins_total);
                        den = a.nbins_total - ex;
                        undef = den == 0;
                    }
                    verdict = !undef && (uint64_t)m * a.t_den >= (uint64_t)a.t_num * den;
                    if (undef) flags = OPH_FLAG_UNDEFINED;
                    else est = (float)m / (float)den;
                } else {
                    st = a.w1 * m;
                    verdict = m >= a.acc_cnt;
                    surv = !verdict && (int32_t)m > a.rej_cnt;
                    flags = OPH_FLAG_EARLY;
                    if (verdict)
                        for (uint32_t w = 0; w * 32 < a.nscan; w++)
                            ex += popc_masked(__ldg(a.QEM + (uint64_t)qg * a.nw + w), __ldg(a.E + (uint64_t)w * a.ld + s),
                                              a.joint, w, a.nscan);
                }
            }
            emit(a.out, has, a.q_col0 + q, s, m, ex, a.level, verdict, flags, est);
            const unsigned long long idx = warp_append(surv, a.surv_count);
            if (surv && idx < a.surv_cap) {  // past capacity: counted, the host redoes the chunk
                a.surv.q[idx] = a.q_col0 + q;
                a.surv.s[idx] = (uint32_t)s;
                a.surv.state[idx] = st;
                a.surv.nmb[idx] = m;
            }
            n_surv += surv;
        }
        // every pair of this set except the survivors is decided at this level: the listed
        // ones above, the unlisted ones (no matched bin) NotSimilar; an overflowing set's
        // pairs are counted by the BRUTE list scan
        hist_add(a.out.hist, a.level, (sl < nset && !of) ? a.nq - n_surv : 0u);
    }
}

// ---------------------------------------------------------------------------
// K4: one GOPH/HOPH level over the survivor list (one thread per surviving
// pair; consecutive survivors mostly share a set, so the bin-row gathers
// coalesce), appending the still-undecided pairs to the next list with
// warp-aggregated atomics.  The last level applies the final verdict.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t group_matches(const LevelArgs &a, uint32_t q, uint32_t s, uint32_t g) {
    const uint32_t *qp = a.QM + (uint64_t)q * a.nb + (uint64_t)g * a.kp;
    const uint32_t *fp = a.F + (uint64_t)g * a.kp * a.ld + s;
    if (a.kp == 32) {  // the configs' k': every load of the group in flight at once (one latency per group)
        uint32_t f[32];
#pragma unroll
        for (int i = 0; i < 32; i++) f[i] = __ldg(fp + (uint64_t)i * a.ld);
        uint32_t m = 0;
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const uint4 x = __ldg(reinterpret_cast<const uint4 *>(qp) + i);  // nb, k' multiples of 4: 16-B aligned
            m += (f[4 * i] == x.x) + (f[4 * i + 1] == x.y) + (f[4 * i + 2] == x.z) + (f[4 * i + 3] == x.w);
        }
        return m;
    }
    uint32_t m = 0;
#pragma unroll 8
    for (uint32_t i = 0; i < a.kp; i++) m += (__ldg(fp + (uint64_t)i * a.ld) == __ldg(qp + i));
    return m;
}

// excluded bins of group g (bins [g kp, (g+1) kp))
__device__ __forceinline__ uint32_t group_excl(const LevelArgs &a, uint32_t q, uint32_t s, uint32_t g) {
    const uint32_t lo = g * a.kp, hi = lo + a.kp;
    uint32_t ex = 0;
    for (uint32_t w = lo / 32; w * 32 < hi; w++) {
        uint32_t x = a.joint ? (__ldg(a.QEM + (uint64_t)q * a.nw + w) & __ldg(a.E + (uint64_t)w * a.ld + s))
                             : (__ldg(a.QEM + (uint64_t)q * a.nw + w) | __ldg(a.E + (uint64_t)w * a.ld + s));
        const uint32_t b0 = max(lo, 32 * w), b1 = min(hi, 32 * w + 32);
        const uint32_t width = b1 - b0;
        const uint32_t mask = (width == 32 ? 0xFFFFFFFFu : ((1u << width) - 1u)) << (b0 - 32 * w);
        ex += __popc(x & mask);
    }
    return ex;
}

// excluded bins among bins [0, nbins) of a pair (= the sum of group_excl over the
// groups they cover): every mask word's pair of loads issued before any is used
__device__ __forceinline__ uint32_t excl_prefix(const LevelArgs &a, uint32_t q, uint32_t s, uint32_t nbins) {
    const uint32_t nw = (nbins + 31) / 32;
    uint32_t ex = 0;
    for (uint32_t w0 = 0; w0 < nw; w0 += 8) {
        uint32_t qm[8], sm[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
            const bool in = w0 + u < nw;
            qm[u] = in ? __ldg(a.QEM + (uint64_t)q * a.nw + w0 + u) : 0u;
            sm[u] = in ? __ldg(a.E + (uint64_t)(w0 + u) * a.ld + s) : 0u;
        }
#pragma unroll
        for (int u = 0; u < 8; u++) ex += popc_masked(qm[u], sm[u], a.joint, w0 + u, nbins);
    }
    return ex;
}

// levels [level, level_last] per launch: a warp walks its 32 survivors level
// by level (lanes that stopped idle), emitting decided pairs at every level;
// pairs still undecided after level_last are compacted into the next list.
__global__ void __launch_bounds__(256) level_kernel(const __grid_constant__ LevelArgs a) {
    const unsigned long long n = *a.count_in;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long base = (unsigned long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < n;
         base += stride) {
        const unsigned long long i = base + (threadIdx.x & 31u);
        bool alive = i < n;
        uint32_t q = 0, s = 0, nmb = 0;
        u128_t st = 0;
        if (alive) {
            q = a.in.q[i];
            s = a.in.s[i];
            st = a.in.state[i];
            nmb = a.in.nmb[i];
        }
        for (uint32_t l = a.level; l <= a.level_last; l++) {
            if (!__any_sync(0xFFFFFFFFu, alive)) break;
            uint32_t M = 0;
            if (alive) {
                M = group_matches(a, q, s, l - 1);
                nmb += M;
                st += a.c[l - 1] * M;
            }
            if (l == a.nlev) {  // the last group: final verdict
                uint32_t verdict = 0, flags = 0, ex_tot = 0;
                float est = -1.0f;
                if (alive) {
                    if (a.method == kGoph) {
                        ex_tot = excl_prefix(a, q, s, a.nb);
                        const uint32_t den = a.nb - ex_tot;
                        if (den == 0) {
                            flags = OPH_FLAG_UNDEFINED;
                        } else {
                            verdict = (uint64_t)nmb * a.t_den >= (uint64_t)a.t_num * den;
                            est = (float)nmb / (float)den;
                        }
                    } else {
                        // HOPH estimator: sum_j c_j m_j / d_j over groups with d_j > 0, exact with
                        // the common denominator lam = lcm(1..kp) (R21, R22)
                        u128_t num = 0, csum = 0;
                        for (uint32_t g = 0; g < a.nlev; g++) {
                            const uint32_t m = (g == l - 1) ? M : group_matches(a, q, s, g);
                            const uint32_t ex = group_excl(a, q, s, g);
                            ex_tot += ex;
                            const uint32_t d = a.kp - ex;
                            if (d == 0) continue;
                            num += a.c[g] * m * (a.lam / d);  // m <= d: num <= D lam (planner-checked)
                            csum += a.c[g];
                        }
                        if (csum == 0) {
                            flags = OPH_FLAG_UNDEFINED;
                        } else {
                            verdict = num * a.t_den >= (u128_t)a.t_num * a.lam * csum;
                            est = (float)((double)num / ((double)a.lam * (double)csum));
                        }
                    }
                }
                emit(a.res, alive, q, s, nmb, ex_tot, a.nlev, verdict, flags, est);
                hist_add(a.res.hist, a.nlev, alive ? 1u : 0u);
                alive = false;
                break;
            }
            const bool acc = alive && st >= a.acc[l - 1];
            const bool rej = alive && !acc && (i128_t)st <= a.rej[l - 1];
            hist_add(a.res.hist, l, (acc || rej) ? 1u : 0u);
            const bool want = a.res.dense ? (acc || rej) : acc;
            if (__any_sync(0xFFFFFFFFu, want)) {
                const uint32_t ex = want ? excl_prefix(a, q, s, l * a.kp) : 0u;
                emit(a.res, acc || rej, q, s, nmb, ex, l, acc ? 1u : 0u, OPH_FLAG_EARLY, -1.0f);
            }
            alive = alive && !acc && !rej;
        }
        const unsigned long long idx = warp_append(alive, a.count_out);
        if (alive) {
            a.out.q[idx] = q;
            a.out.s[idx] = s;
            a.out.state[idx] = st;
            a.out.nmb[idx] = nmb;
        }
    }
}

// ---------------------------------------------------------------------------
// K3'' multi-level BRUTE scan for GOPH / HOPH (Alg. 1 / Alg. 2 group by group in
// registers): the query block's values of every group sit in shared memory; a
// thread owns SPT sets x 32 queries whose counters ARE the pair states (each
// matched bin of group l adds the group weight c_l, GOPH c = 1).  After each
// group the undecided pairs are tested against the level's thresholds; a warp
// stops as soon as none of its pairs is undecided.  Replaces the survivor
// lists when the states fit 32 bits and the groups fit shared memory: a
// high-similarity collection then costs at most one scan instead of per-pair
// gathers at every level.  The HOPH final estimator (per-group counts) is
// recomputed by gathers for the pairs that reach the last group.
// ---------------------------------------------------------------------------
// cnt[q] for a runtime q without demoting the register array to local memory
template <int B>
__device__ __forceinline__ uint32_t pick(const uint32_t (&cnt)[B], uint32_t q) {
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < B; i++) c = ((uint32_t)i == q) ? cnt[i] : c;
    return c;
}

// 4 CTAs/SM (128 registers, no spills; image-like GOPH / HOPH 67.7 / 11.8 -> 63.9 / 11.1 ms vs 3)
template <int SPT>
__global__ void __launch_bounds__(128, 4) levels_kernel(const __grid_constant__ LevelArgs a) {
    constexpr int B = 32, U = 4;
    extern __shared__ __align__(16) uint32_t lsm[];
    const uint32_t nbs = a.nlev * a.kp;  // every bin of every group
    const uint32_t qb0 = blockIdx.x * B;
    const uint64_t col0 = (uint64_t)a.q_col0 + qb0;
    load_query_block<B>(lsm, a.QT, a.ldq, 0, col0, nbs);
    __syncthreads();
    const uint32_t qvalid = qb0 + B <= a.nq ? 0xFFFFFFFFu : ((1u << (a.nq - qb0)) - 1u);
    const bool hoph = a.method == kHoph;
    const uint32_t rawmask = a.sh ? (1u << a.sh) - 1u : 0xFFFFFFFFu;

    const uint64_t tile_sets = 128ull * SPT;
    const uint64_t ntiles = (a.n_sets - a.s_begin + tile_sets - 1) / tile_sets;
    const uint64_t t_end = min(ntiles, (uint64_t)(blockIdx.y + 1) * a.tiles_per_cta);
    for (uint64_t t = (uint64_t)blockIdx.y * a.tiles_per_cta; t < t_end; t++) {
        const uint64_t s0 = a.s_begin + t * tile_sets + threadIdx.x * SPT;
        const bool active = s0 < a.n_sets;
        uint32_t cnt[SPT][B];
        uint32_t alive[SPT];
#pragma unroll
        for (int j = 0; j < SPT; j++) {
            alive[j] = (s0 + j < a.n_sets) ? qvalid : 0u;
#pragma unroll
            for (int q = 0; q < B; q++) cnt[j][q] = 0;
        }
        // threads past the last set read (and never use) the row's last SPT columns
        const uint32_t *Fp = a.F + (active ? s0 : a.ld - SPT);
        const uint32_t ldb = (uint32_t)(a.ld * 4u);  // < 2^32 (launcher)
        for (uint32_t l = 1; l <= a.nlev; l++) {
            uint32_t any = 0;
#pragma unroll
            for (int j = 0; j < SPT; j++) any |= alive[j];
            if (!__any_sync(0xFFFFFFFFu, any != 0u)) break;  // every pair of this warp is decided
            scan_bins<B, SPT, U>(Fp, ldb, lsm + (size_t)(l - 1) * a.kp * B, (l - 1) * a.kp, a.kp, cnt, a.one,
                                 a.w32[l - 1]);
#pragma unroll
            for (int j = 0; j < SPT; j++) {
                const uint32_t s = (uint32_t)(s0 + j);
                if (l < a.nlev) {
                    // ---- early termination at level l (thresholds on the state)
                    uint32_t accm = 0, decm = 0;
#pragma unroll
                    for (int q = 0; q < B; q++) {
                        const bool acc = cnt[j][q] >= a.acc32[l - 1];
                        const bool rej = cnt[j][q] < a.rej1[l - 1];
                        accm |= (uint32_t)acc << q;
                        decm |= (uint32_t)(acc || rej) << q;
                    }
                    accm &= alive[j];
                    decm &= alive[j];
                    hist_add(a.res.hist, l, __popc(decm));
                    const uint32_t want = a.res.dense ? decm : accm;
                    if (__any_sync(0xFFFFFFFFu, want != 0u)) {
#pragma unroll 1
                        for (int q = 0; q < B; q++) {
                            const bool e = (want >> q) & 1u;
                            const uint32_t qg = (uint32_t)(col0 + q);
                            uint32_t ex = 0, nmb = 0;
                            if (e) {
                                ex = excl_prefix(a, qg, s, l * a.kp);
                                nmb = pick<B>(cnt[j], q) & rawmask;  // matched bins over groups 1..l
                            }
                            emit(a.res, e, qg, s, nmb, ex, l, (accm >> q) & 1u, OPH_FLAG_EARLY, -1.0f);
                        }
                    }
                    alive[j] &= ~decm;
                } else {
                    // ---- the last group: the final verdict (GOPH: Eq. 6 over all n k' bins;
                    // HOPH: the nominal-weight estimator, exact over lam = lcm(1..k'))
                    hist_add(a.res.hist, a.nlev, __popc(alive[j]));
                    if (!__any_sync(0xFFFFFFFFu, alive[j] != 0u)) continue;
#pragma unroll 1
                    for (int q = 0; q < B; q++) {
                        const bool al = (alive[j] >> q) & 1u;
                        const uint32_t qg = (uint32_t)(col0 + q);
                        uint32_t verdict = 0, flags = 0, ex_tot = 0, nmb = 0;
                        float est = -1.0f;
                        if (al) {
                            if (!hoph) {
                                nmb = pick<B>(cnt[j], q);
                                ex_tot = excl_prefix(a, qg, s, a.nb);
                                const uint32_t den = a.nb - ex_tot;
                                if (den == 0) {
                                    flags = OPH_FLAG_UNDEFINED;
                                } else {
                                    verdict = (uint64_t)nmb * a.t_den >= (uint64_t)a.t_num * den;
                                    est = (float)nmb / (float)den;
                                }
                            } else {
                                u128_t num = 0, csum = 0;
                                for (uint32_t g = 0; g < a.nlev; g++) {
                                    const uint32_t m = group_matches(a, qg, s, g);
                                    const uint32_t ex = group_excl(a, qg, s, g);
                                    nmb += m;
                                    ex_tot += ex;
                                    const uint32_t d = a.kp - ex;
                                    if (d == 0) continue;
                                    num += a.c[g] * m * (a.lam / d);
                                    csum += a.c[g];
                                }
                                if (csum == 0) {
                                    flags = OPH_FLAG_UNDEFINED;
                                } else {
                                    verdict = num * a.t_den >= (u128_t)a.t_num * a.lam * csum;
                                    est = (float)((double)num / ((double)a.lam * (double)csum));
                                }
                            }
                        }
                        emit(a.res, al, qg, s, nmb, ex_tot, a.nlev, verdict, flags, est);
                    }
                    alive[j] = 0;
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// K3e empty-aware GOPH (E1-E4): Alg. 1 with the
// binomial trials taken to be the pair's non-excluded bins.  The same register
// scan as levels_kernel; a pair's state packs three 10-bit fields,
//   D << 20 | D_c << 10 | M_c   (nb <= 512, so no field carries),
// D = non-excluded bins over all groups (from the empty masks, before any value
// is compared), D_c = non-excluded bins compared so far, M_c = matched bins (the
// scan adds 1 per match).  After group l < n with R = D - D_c remaining trials:
//   R = 0      -> the full-OPH verdict now (E3);
//   else M_ra = k' (T D - M_c) / R = num / den, and Alg. 1's tests on it:
//     Similar    if num <= 0, or num < k' t_num R and floor(M_ra) <= m_a
//                (num < ma1 den, ma1 = m_a + 1 = #{m : P(X <= m) <= eps})
//     NotSimilar if num > k' den, or num >= k' t_num R and ceil(M_ra) >= m_r
//                (num > (m_r - 1) den, m_r = min{m : P(X >= m) <= eps})
// (all products < 2^51 in int64; I = int32_t when the host has bounded them below
// 2^31 -- T with a small denominator, the common case); the last group: the
// full-OPH verdict.
// ---------------------------------------------------------------------------
template <int SPT, typename I, int B>
__global__ void __launch_bounds__(128, 3) levels_e_kernel(const __grid_constant__ LevelArgs a) {
    constexpr int U = 4;
    extern __shared__ __align__(16) uint32_t lsm[];
    const uint32_t nbs = a.nlev * a.kp;  // every bin of every group
    uint32_t *qm = lsm + (size_t)nbs * B;  // [nw][B] query empty masks
    const uint32_t qb0 = blockIdx.x * B;
    const uint64_t col0 = (uint64_t)a.q_col0 + qb0;
    load_query_block<B>(lsm, a.QT, a.ldq, 0, col0, nbs);
    load_query_block<B>(qm, a.QE, a.ldq, 0, col0, a.nw);
    __syncthreads();
    const uint32_t qvalid =
        qb0 + B <= a.nq ? (B == 32 ? 0xFFFFFFFFu : ((1u << (B & 31)) - 1u)) : ((1u << (a.nq - qb0)) - 1u);
    const I kp = (I)a.kp, tn = (I)a.t_num, td = (I)a.t_den, ma1 = (I)a.ma1, mr1 = (I)a.mr1;

    const uint64_t tile_sets = 128ull * SPT;
    const uint64_t ntiles = (a.n_sets - a.s_begin + tile_sets - 1) / tile_sets;
    const uint64_t t_end = min(ntiles, (uint64_t)(blockIdx.y + 1) * a.tiles_per_cta);
    for (uint64_t t = (uint64_t)blockIdx.y * a.tiles_per_cta; t < t_end; t++) {
        const uint64_t s0 = a.s_begin + t * tile_sets + threadIdx.x * SPT;
        const bool active = s0 < a.n_sets;
        uint32_t cnt[SPT][B];
        uint32_t alive[SPT];
        // D of every pair: nb minus the excluded bins over all groups (E1)
#pragma unroll
        for (int j = 0; j < SPT; j++) {
            const uint64_t s = s0 + j;
            alive[j] = (s < a.n_sets) ? qvalid : 0u;
#pragma unroll
            for (int q = 0; q < B; q++) cnt[j][q] = a.nb << 20;
            for (uint32_t w = 0; w < a.nw; w++) {
                const uint32_t es = s < a.n_sets ? __ldg(a.E + (uint64_t)w * a.ld + s) : 0u;
#pragma unroll
                for (int q = 0; q < B; q++) cnt[j][q] -= popc_masked(qm[w * B + q], es, a.joint, w, a.nb) << 20;
            }
        }
        const uint32_t *Fp = a.F + (active ? s0 : a.ld - SPT);
        const uint32_t ldb = (uint32_t)(a.ld * 4u);  // < 2^32 (launcher)
        for (uint32_t l = 1; l <= a.nlev; l++) {
            uint32_t any = 0;
#pragma unroll
            for (int j = 0; j < SPT; j++) any |= alive[j];
            if (!__any_sync(0xFFFFFFFFu, any != 0u)) break;  // every pair of this warp is decided
            scan_bins<B, SPT, U>(Fp, ldb, lsm + (size_t)(l - 1) * a.kp * B, (l - 1) * a.kp, a.kp, cnt, a.one, a.one);
            // D_c += the group's non-excluded bins
            const uint32_t lo = (l - 1) * a.kp, hi = l * a.kp;
            for (uint32_t w = lo / 32; w * 32 < hi; w++) {
                const uint32_t b0 = max(lo, 32 * w), b1 = min(hi, 32 * w + 32);
                const uint32_t gm = (b1 - b0 == 32 ? 0xFFFFFFFFu : ((1u << (b1 - b0)) - 1u)) << (b0 - 32 * w);
                const uint32_t nbw = __popc(gm);
#pragma unroll
                for (int j = 0; j < SPT; j++) {
                    const uint64_t s = s0 + j;
                    const uint32_t es = s < a.n_sets ? __ldg(a.E + (uint64_t)w * a.ld + s) : 0u;
#pragma unroll
                    for (int q = 0; q < B; q++) {
                        const uint32_t x = a.joint ? (qm[w * B + q] & es) : (qm[w * B + q] | es);
                        cnt[j][q] += (nbw - __popc(x & gm)) << 10;
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < SPT; j++) {
                const uint32_t s = (uint32_t)(s0 + j);
                uint32_t accm = 0, decm = 0, donem = 0;  // Similar / decided / complete (E3)
#pragma unroll
                for (int q = 0; q < B; q++) {
                    const uint32_t v = cnt[j][q];
                    const I M = (I)(v & 1023u), Dc = (I)((v >> 10) & 1023u), D = (I)(v >> 20);
                    const I R = D - Dc;
                    bool acc, dec, done = false;
                    if (l == a.nlev || R == 0) {  // the full-OPH verdict
                        acc = D > 0 && M * td >= tn * D;
                        dec = done = true;
                    } else {
                        const I num = kp * (tn * D - td * M), den = td * R;
                        acc = num <= 0 || (num < kp * tn * R && num < ma1 * den);
                        dec = acc || num > kp * den || (num >= kp * tn * R && num > mr1 * den);
                    }
                    accm |= (uint32_t)acc << q;
                    decm |= (uint32_t)dec << q;
                    donem |= (uint32_t)done << q;
                }
                accm &= alive[j];
                decm &= alive[j];
                hist_add(a.res.hist, l, __popc(decm));
                const uint32_t want = a.res.dense ? decm : accm;
                if (__any_sync(0xFFFFFFFFu, want != 0u)) {
#pragma unroll 1
                    for (int q = 0; q < B; q++) {
                        const bool e = (want >> q) & 1u;
                        const uint32_t v = pick<B>(cnt[j], q);
                        const uint32_t M = v & 1023u, Dc = (v >> 10) & 1023u, D = v >> 20;
                        uint32_t flags = OPH_FLAG_EARLY, ex = l * a.kp - Dc;
                        float est = -1.0f;
                        if ((donem >> q) & 1u) {  // complete: the full-OPH record
                            ex = a.nb - D;
                            flags = D == 0 ? OPH_FLAG_UNDEFINED : 0u;
                            if (D) est = (float)M / (float)D;
                        }
                        emit(a.res, e, (uint32_t)(col0 + q), s, M, ex, l, (accm >> q) & 1u, flags, est);
                    }
                }
                alive[j] &= ~decm;
            }
        }
    }
}

cudaError_t launch_levels_scan(const LevelArgs &a0, cudaStream_t st) {
    if (a0.n_sets <= a0.s_begin || a0.nq == 0) return cudaSuccess;
    LevelArgs a = a0;
    constexpr int SPT = 2;
    // the empty-aware scan: 1 set x EB queries per thread -- a pair's stop group depends on its
    // own empty bins, and a warp stops only when all of its pairs have (fewer pairs per warp:
    // image-like 344 ms at 2 x 32, 208 at 1 x 32, 136 at 1 x 16)
    constexpr int EB = EA_B;
    const uint32_t qb = a.eaware ? EB : 32u;
    const size_t smem = ((size_t)a.nlev * a.kp + (a.eaware ? a.nw : 0)) * qb * 4;
    const uint64_t tile_sets = 128ull * (a.eaware ? 1 : SPT);
    const uint32_t qblocks = (a.nq + qb - 1) / qb;
    const uint64_t ntiles = (a.n_sets - a.s_begin + tile_sets - 1) / tile_sets;
    const uint64_t want_y = std::max<uint64_t>(1, (148ull * 4 * 4 + qblocks - 1) / qblocks);
    uint64_t tpc = std::max<uint64_t>(1, (ntiles + want_y - 1) / want_y);
    tpc = std::min<uint64_t>(tpc, 64);
    a.tiles_per_cta = (uint32_t)tpc;
    const uint64_t gy = (ntiles + tpc - 1) / tpc;
    if (gy > 65535 || a.ld * 4 > 0xFFFFFFFFull) return cudaErrorInvalidConfiguration;
    // the empty-aware rule in 32-bit arithmetic when every product is < 2^31
    // (|num|, k' den, ma1 den, k' t_num R <= k' max(t_num, t_den) 512 (k' + 1))
    const bool e32 = (uint64_t)a.kp * std::max(a.t_num, a.t_den) * 512ull * (a.kp + 1ull) < (1ull << 31);
    auto kern = !a.eaware ? levels_kernel<SPT>
                          : (e32 ? levels_e_kernel<1, int32_t, EB> : levels_e_kernel<1, int64_t, EB>);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<dim3(qblocks, (unsigned)gy), 128, smem, st>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Exact Jaccard of (query, set) pairs (Eq. 5): warp per pair.  The smaller set
// A is cut into 32 contiguous slices; lane l binary-searches the first element
// of its slice in the larger set B, then merges the slice with B linearly,
// counting equal ids (ids strictly increasing).  |A u B| = |A| + |B| - |A n B|.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) jaccard_kernel(const __grid_constant__ JaccardArgs a) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t i = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < a.n; i += nwarps) {
        const uint32_t qi = a.query[i], si = a.set[i];
        const uint64_t q0 = a.q_offsets[qi], q1 = a.q_offsets[qi + 1];
        const uint64_t s0 = a.s_offsets[si], s1 = a.s_offsets[si + 1];
        const uint32_t *A = a.q_ids + q0, *B = a.s_ids + s0;
        uint64_t na = q1 - q0, nb = s1 - s0;
        if (na > nb) {
            const uint32_t *t = A;
            A = B;
            B = t;
            const uint64_t u = na;
            na = nb;
            nb = u;
        }
        const uint64_t lo = na * lane / 32, hi = na * (lane + 1) / 32;  // this lane's slice of A
        uint32_t c = 0;
        if (lo < hi) {
            uint64_t l = 0, h = nb;  // first position in B with B[pos] >= A[lo]
            const uint32_t x0 = __ldg(A + lo);
            while (l < h) {
                const uint64_t m = (l + h) >> 1;
                if (__ldg(B + m) < x0) l = m + 1; else h = m;
            }
            uint64_t ia = lo, ib = l;
            while (ia < hi && ib < nb) {
                const uint32_t xa = __ldg(A + ia), xb = __ldg(B + ib);
                c += xa == xb;
                ia += xa <= xb;
                ib += xb <= xa;
            }
        }
        const uint32_t inter = __reduce_add_sync(0xFFFFFFFFu, c);
        if (lane == 0) {
            a.inter[i] = inter;
            a.uni[i] = (uint32_t)(na + nb - inter);
        }
    }
}

cudaError_t launch_jaccard(const JaccardArgs &a, cudaStream_t st) {
    if (a.n == 0) return cudaSuccess;
    const unsigned grid = (unsigned)std::min<uint64_t>((a.n + 7) / 8, 148ull * 16);
    jaccard_kernel<<<grid, 256, 0, st>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
template <int SB>
static cudaError_t launch_build_sb(const BuildArgs &a0, size_t smem, cudaStream_t st, uint32_t threads) {
    const uint64_t grid = (a0.n_sets + SB - 1) / SB;
    const bool fast = a0.do_flat && a0.flat.pow2 && a0.flat.start == 0 && a0.psi.pow2 && !a0.psi.identity &&
                      a0.do_hier && a0.hier_pow2_halves && a0.L <= 32 && a0.log2kp >= 1;
    const bool w32 = a0.psi.mask == 0xFFFFFFFFu;
    BuildArgs a = a0;
    // the warp-per-set kernel (default; OPHGPU_BUILD_V1=1 keeps the element-strided one)
    const char *v1 = getenv("OPHGPU_BUILD_V1");
    const size_t smem_w = (size_t)SB * (build_warp_stride(a0.k) + build_warp_stride(a0.L * a0.kp)) * 4;
    if constexpr (SB == 8 || SB == 16) if (fast && !(v1 && atoi(v1)) && smem_w <= 200 * 1024) {
        const uint32_t log2k = a.log2V - a.flat.shift;
        // derivable leading HOPH groups: g <= log2 k - log2 k' - 1 and g < L - 1; k' >= 4 (4-bin
        // lanes); M_0 <= 128 (M_0 / 4 <= 32 lanes)
        uint32_t hder = 0;
        if (log2k > a.log2kp && a.log2kp >= 2 && log2k - a.log2kp - 1 <= 7) hder = std::min(log2k - a.log2kp, a.L - 1);
        // (measured r02z3: the derivation halves the shared reductions but is not faster -- image-like
        // 3.53 vs 3.49 ms, text-like 0.551 vs 0.538: the build is not bound by the shared-memory
        // pipe (29 % of its wavefront peak) -- so it is an A/B option, OPHGPU_BUILD_DERIVE=1)
        const char *dv = getenv("OPHGPU_BUILD_DERIVE");
        if (!(dv && atoi(dv))) hder = 0;
        a.hder = hder;
        const uint32_t spw = threads == 256 ? 1u : 2u;  // 128 threads: 2 sets per warp at SB 8
        auto kern = w32 ? (spw == 1 ? build_warp_kernel<true, SB, SB / 8> : build_warp_kernel<true, SB, SB / 4>)
                        : (spw == 1 ? build_warp_kernel<false, SB, SB / 8> : build_warp_kernel<false, SB, SB / 4>);
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_w);
        if (e != cudaSuccess) return e;
        kern<<<(unsigned)grid, 32u * SB / (spw == 1 ? SB / 8 : SB / 4), smem_w, st>>>(a);
        return cudaGetLastError();
    }
    auto kern = fast ? (w32 ? build_kernel<true, SB, true> : build_kernel<false, SB, true>)
                     : (w32 ? build_kernel<true, SB, false> : build_kernel<false, SB, false>);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)grid, threads, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_build(const BuildArgs &a, cudaStream_t st) {
    if (a.n_sets == 0) return cudaSuccess;
    const uint32_t per_set = (a.do_flat ? (a.k + 31) / 32 * 32 + 1 : 0) +
                             (a.do_hier ? (a.L * a.kp + 31) / 32 * 32 + 1 : 0);
    // 8 sets per CTA: 36 KB of shared memory at text-like sizes -> 6 CTAs (48 warps) per SM,
    // and a bin row of the tile is one full 32-B sector; fewer for very large sketches
    // (OPHGPU_BUILD_SB / OPHGPU_BUILD_THREADS override the tile for A/B sweeps)
    uint32_t SB = 8, threads = 128;  // (r02 sweep: 128 threads 3.62 / 0.53 ms vs 256: 3.87 / 0.55 on image / text)
    if (const char *e = getenv("OPHGPU_BUILD_SB")) SB = (uint32_t)atoi(e);
    if (const char *e = getenv("OPHGPU_BUILD_THREADS")) threads = (uint32_t)atoi(e);
    if (SB != 1 && SB != 2 && SB != 4 && SB != 8 && SB != 16) SB = 8;
    if (threads != 128 && threads != 256 && threads != 512) threads = 256;
    while (SB > 1 && (size_t)SB * per_set * 4 + 16 > 200 * 1024) SB >>= 1;
    const size_t smem = ((size_t)SB * per_set * 4 + 15) / 16 * 16;
    switch (SB) {
        case 16: return launch_build_sb<16>(a, smem, st, threads);
        case 8: return launch_build_sb<8>(a, smem, st, threads);
        case 4: return launch_build_sb<4>(a, smem, st, threads);
        case 2: return launch_build_sb<2>(a, smem, st, threads);
        default: return launch_build_sb<1>(a, smem, st, threads);
    }
}

cudaError_t launch_minwise(const MinwiseArgs &a, cudaStream_t st) {
    if (a.n_sets == 0) return cudaSuccess;
    // 8 sets per CTA (ids staged once for 8 x k evaluations); a small collection (the
    // queries) one set per CTA with its k permutations split over CTAs of 64 threads,
    // so that it covers the 148 SMs and the largest set's work is spread (the query
    // build sits on the step's critical path: text-like 176 us with 256-thread CTAs)
    const uint32_t sets = a.n_sets >= 148ull * 8 * 4 ? 8u : 1u;
    const uint64_t grid = (a.n_sets + sets - 1) / sets;
    uint32_t threads = a.k >= 256 ? 256 : ((a.k + 31) / 32) * 32;
    uint32_t gy = 1;
    if (sets == 1 && threads > 64) {
        threads = 64;
        gy = (a.k + 63) / 64;
    }
    MinwiseArgs b = a;
    b.hmul = 1u << (32 - std::min<uint32_t>(a.w, 32));  // (w = 32: unused)
    b.hsh = (32 - std::min<uint32_t>(a.w, 32)) + (a.w + 1) / 2;
    if (sets == 8) {
        if (a.w >= 32) minwise_kernel<true, 8><<<(unsigned)grid, threads, 0, st>>>(b);
        else minwise_kernel<false, 8><<<(unsigned)grid, threads, 0, st>>>(b);
    } else {
        if (a.w >= 32) minwise_kernel<true, 1><<<dim3((unsigned)grid, gy), threads, 0, st>>>(b);
        else minwise_kernel<false, 1><<<dim3((unsigned)grid, gy), threads, 0, st>>>(b);
    }
    return cudaGetLastError();
}

cudaError_t launch_prep(const PrepArgs &a, cudaStream_t st) {
    const uint64_t ntile = (uint64_t)((a.nb + 31) / 32) * ((a.ldq + 31) / 32);
    const uint64_t nw = (uint64_t)a.nw * a.ldq;  // (the mask / flag loops are grid-strided too)
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(std::max(ntile, (nw + 255) / 256),
                                                                              148ull * 16));
    prep_kernel<<<grid, 256, 0, st>>>(a);
    return cudaGetLastError();
}

template <int B, int SPT, bool LIST>
static cudaError_t launch_scan_t(const ScanArgs &a0, cudaStream_t st) {
    ScanArgs a = a0;
    const size_t smem = ((size_t)min(a.nscan, kScanChunk) * B + (size_t)a.nw_load * B + B) * 4;
    const uint64_t tile_sets = 128ull * SPT;
    const uint32_t qblocks = (a.nq + B - 1) / B;
    uint64_t gy;
    if (LIST) {  // grid-stride over a device-side list: the count is not known on the host
        gy = std::max<uint64_t>(1, (148ull * 4 + qblocks - 1) / qblocks);
        a.tiles_per_cta = 1;
    } else {
        const uint64_t ntiles = (a.n_sets - a.s_begin + tile_sets - 1) / tile_sets;
        // aim for >= 4 waves of CTAs over 148 SMs, otherwise longest tile runs per CTA;
        // HBM-bound small blocks: one tile per CTA (the hardware's CTA scheduler balances
        // the tail; a tile is 128 SPT sets x every bin, ~0.1 ms at 8 CTAs/SM)
        const uint64_t want_y = std::max<uint64_t>(1, (148ull * 4 * 4 + qblocks - 1) / qblocks);
        uint64_t tpc = B <= 8 ? 1 : std::max<uint64_t>(1, (ntiles + want_y - 1) / want_y);
        tpc = std::min<uint64_t>(tpc, 64);
        if ((ntiles + tpc - 1) / tpc > 65535) tpc = (ntiles + 65534) / 65535;
        a.tiles_per_cta = (uint32_t)tpc;
        gy = (ntiles + tpc - 1) / tpc;
    }
    if (gy > 65535 || a.ld * 4 > 0xFFFFFFFFull) return cudaErrorInvalidConfiguration;
    cudaError_t e =
        cudaFuncSetAttribute(scan_kernel<B, SPT, LIST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    scan_kernel<B, SPT, LIST><<<dim3(qblocks, (unsigned)gy), 128, smem, st>>>(a);
    return cudaGetLastError();
}

// query block B: 32 queries per thread block of registers, fewer when the chunk has
// fewer queries (4 / 8 / 16: less wasted work, fewer registers, more CTAs per SM --
// the small-B end of the HBM-bound -> ALU-bound crossover)
cudaError_t launch_scan(const ScanArgs &a, uint32_t, cudaStream_t st) {
    if (a.n_sets <= a.s_begin || a.nq == 0) return cudaSuccess;
    if (a.set_list) return launch_scan_t<32, 1, true>(a, st);
    if (a.nq <= 4) return launch_scan_t<4, 2, false>(a, st);
    if (a.nq <= 8) return launch_scan_t<8, 2, false>(a, st);
    if (a.nq <= 16) return launch_scan_t<16, 2, false>(a, st);
    return launch_scan_t<32, 2, false>(a, st);
}

cudaError_t launch_table(const TableArgs &a, cudaStream_t st) {
    const uint64_t n = (uint64_t)a.nscan * a.nq;
    if (n == 0) return cudaSuccess;
    const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 16);
    table_kernel<<<grid, 256, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_probe(const ProbeArgs &a0, cudaStream_t st) {
    if (a0.s_end <= a0.s_begin) return cudaSuccess;
    ProbeArgs a = a0;
    const uint64_t n = a.s_end - a.s_begin;
    if (a.log2W < 9 || a.log2W > kJoinMaxLog2W || a.ld * 4 >= (1ull << 32)) return cudaErrorInvalidValue;
    const uint32_t W = 0;  // the layout does not depend on the filter width (64-KB buffers)
    constexpr uint32_t kSmemMax = 227 * 1024;
    // one CTA per SM; sets per CTA: the fewest waves whose per-CTA lists fit next to
    // the filter double buffer, split evenly (multiple of the tile's kJoinTile sets).  Lists
    // of 2 matched queries per set instead of kJoinList when that saves a wave and at most 128
    // bins are scanned (scale shard, GOPH / HOPH: 1.25M sets in one wave instead of two, 0.72 ->
    // 0.70 / 0.68 -> 0.64 ms per call; full OPH's 256 bins give enough sets 3+ spurious
    // single-bin matches that the BRUTE list scan of the overflow, 8 -> 366 us, eats the gain).
    // A set matching more queries goes to that scan either way: the records do not change.
    // OPHGPU_JOIN_LISTS=2|4 forces the choice (A/B).
    auto rmax_for = [&](uint32_t nl) {
        uint32_t r = kJoinTile;
        while (join_layout(W, r + kJoinTile, nl).total <= kSmemMax && r + kJoinTile <= 65504) r += kJoinTile;
        return r;
    };
    auto waves_for = [&](uint32_t rm) { return (n + 148ull * rm - 1) / (148ull * rm); };
    uint32_t nlist = kJoinList;
    uint32_t Rmax = rmax_for(nlist);
    if (a.nscan <= 128 && waves_for(Rmax) > 1 && waves_for(rmax_for(2)) < waves_for(Rmax)) {
        nlist = 2;
        Rmax = rmax_for(2);
    }
    if (const char *e = getenv("OPHGPU_JOIN_LISTS")) {
        const int v = atoi(e);
        if (v == 2 || v == kJoinList) {
            nlist = (uint32_t)v;
            Rmax = rmax_for(nlist);
        }
    }
    const uint64_t waves = waves_for(Rmax);
    const uint32_t R = (uint32_t)((((n + 148 * waves - 1) / (148 * waves)) + kJoinTile - 1) / kJoinTile * kJoinTile);
    a.R = R;
    a.nlist = nlist;
    const size_t smem = join_layout(W, R, nlist).total;
    if (smem > kSmemMax) return cudaErrorInvalidConfiguration;
    const bool mw = a.method == kMinwise;
    auto kern = mw ? join_kernel<true, 9> : join_kernel<false, 9>;
    if (a.log2W == 10) kern = mw ? join_kernel<true, 10> : join_kernel<false, 10>;
    if (a.log2W == 11) kern = mw ? join_kernel<true, 11> : join_kernel<false, 11>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const uint64_t grid = (n + R - 1) / R;
    kern<<<(unsigned)grid, kJoinThreads, smem, st>>>(a);
    return cudaGetLastError();
}

// The empty-aware rule (E1-E4) for listed pairs (the join's pairs with a matched bin,
// E5): one thread per pair walks the groups from the first, gathering each group's
// values and masks, and stops at the pair's decision -- the same arithmetic as
// levels_e_kernel in int64.
__global__ void __launch_bounds__(256) level_e_kernel(const __grid_constant__ LevelArgs a) {
    const unsigned long long n = *a.count_in;
    const int64_t kp = a.kp, tn = a.t_num, td = a.t_den;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    // warp-uniform trip counts: emit() appends with full-warp ballots
    for (unsigned long long base = blockIdx.x * (unsigned long long)blockDim.x + (threadIdx.x & ~31u); base < n;
         base += stride) {
        const unsigned long long i = base + (threadIdx.x & 31u);
        bool alive = i < n;
        uint32_t q = 0, s = 0, ex = 0;
        int64_t D = 0, M = 0, Dc = 0;
        if (alive) {
            q = a.in.q[i];
            s = a.in.s[i];
            uint32_t ex_all = 0;
            for (uint32_t w = 0; w < a.nw; w++)
                ex_all += popc_masked(__ldg(a.QEM + (uint64_t)q * a.nw + w), __ldg(a.E + (uint64_t)w * a.ld + s),
                                      a.joint, w, a.nb);
            D = (int64_t)a.nb - ex_all;
        }
        for (uint32_t l = 1; l <= a.nlev; l++) {
            if (!__any_sync(0xFFFFFFFFu, alive)) break;
            bool dec = false, acc = false, done = false;
            if (alive) {
                M += group_matches(a, q, s, l - 1);
                const uint32_t e = group_excl(a, q, s, l - 1);
                ex += e;
                Dc += kp - e;
                const int64_t R = D - Dc;
                if (l == a.nlev || R == 0) {  // the full-OPH verdict
                    acc = D > 0 && M * td >= tn * D;
                    dec = done = true;
                } else {
                    const int64_t num = kp * (tn * D - td * M), den = td * R;
                    acc = num <= 0 || (num < kp * tn * R && num < (int64_t)a.ma1 * den);
                    dec = acc || num > kp * den || (num >= kp * tn * R && num > (int64_t)a.mr1 * den);
                }
            }
            emit(a.res, dec, q, s, (uint32_t)M, done ? (uint32_t)(a.nb - D) : ex, l, acc,
                 done ? (D == 0 ? OPH_FLAG_UNDEFINED : 0u) : OPH_FLAG_EARLY, (done && D) ? (float)M / (float)D : -1.0f);
            alive = alive && !dec;
        }
    }
}

// The empty-aware HOPH rule (EH1-EH5, oracle pair_hoph_e): per pair, the groups' usable
// bins d_j and the usable weight C_K come from the masks first; then group by group the
// achieved mass A_l = sum_{j<=l, d_j>0} c_j m_j / d_j and the usable weight left W_l give
// x = k' (T C_K - A_l) / W_l, tested with Alg. 2's rules in exact 128-bit integers scaled
// by t_den lcm{d_j compared}; W_l = 0 or the last group: the HOPH estimator.  Pairs come
// from the join's list (those with a matched bin; no other pair can be Similar) or, with
// `implicit`, every (query, set) pair.
__device__ __forceinline__ i128_t i128_gcd_d(i128_t x, i128_t y) {
    while (y != 0) {
        const i128_t t = x % y;
        x = y;
        y = t;
    }
    return x;
}

__global__ void __launch_bounds__(256) level_he_kernel(const __grid_constant__ LevelArgs a) {
    const unsigned long long n = a.implicit ? (unsigned long long)a.nq * a.n_sets : *a.count_in;
    const i128_t kp = a.kp, tn = a.t_num, td = a.t_den;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long base = blockIdx.x * (unsigned long long)blockDim.x + (threadIdx.x & ~31u); base < n;
         base += stride) {
        const unsigned long long i = base + (threadIdx.x & 31u);
        bool alive = i < n;
        uint32_t q = 0, s = 0;
        uint64_t usable = 0;  // bit j: group j has a usable bin
        i128_t CK = 0;
        if (alive) {
            if (a.implicit) {
                q = a.q_col0 + (uint32_t)(i / a.n_sets);
                s = (uint32_t)(i % a.n_sets);
            } else {
                q = a.in.q[i];
                s = a.in.s[i];
            }
            for (uint32_t g = 0; g < a.nlev; g++)
                if (group_excl(a, q, s, g) < a.kp) {
                    usable |= 1ull << g;
                    CK += (i128_t)a.c[g];
                }
        }
        i128_t W = CK, lam = 1, A = 0;  // A = A_l lam
        uint32_t nmb = 0, nex = 0;
        for (uint32_t l = 1; l <= a.nlev; l++) {
            if (!__any_sync(0xFFFFFFFFu, alive)) break;
            bool dec = false, acc = false;
            uint32_t flags = OPH_FLAG_EARLY, n_mb = 0, n_ex = 0;
            float est = -1.0f;
            if (alive) {
                const uint32_t m = group_matches(a, q, s, l - 1);
                const uint32_t e = group_excl(a, q, s, l - 1);
                nmb += m;
                nex += e;
                if ((usable >> (l - 1)) & 1ull) {
                    const i128_t d = (i128_t)(a.kp - e);
                    W -= (i128_t)a.c[l - 1];
                    const i128_t nl = lam / i128_gcd_d(lam, d) * d;  // lcm
                    A = A * (nl / lam) + (i128_t)a.c[l - 1] * m * (nl / d);
                    lam = nl;
                }
                n_mb = nmb;
                n_ex = nex;
                if (l == a.nlev || W == 0) {  // EH4 / EH5: the HOPH estimator over all groups
                    dec = true;
                    u128_t num = 0, csum = 0;
                    n_mb = n_ex = 0;
                    for (uint32_t g = 0; g < a.nlev; g++) {
                        const uint32_t mg = group_matches(a, q, s, g);
                        const uint32_t eg = group_excl(a, q, s, g);
                        n_mb += mg;
                        n_ex += eg;
                        const uint32_t dg = a.kp - eg;
                        if (dg == 0) continue;
                        num += a.c[g] * mg * (a.lam / dg);
                        csum += a.c[g];
                    }
                    flags = 0;
                    if (csum == 0) {
                        flags = OPH_FLAG_UNDEFINED;
                    } else {
                        acc = num * a.t_den >= (u128_t)a.t_num * a.lam * csum;
                        est = (float)((double)num / ((double)a.lam * (double)csum));
                    }
                } else {
                    const i128_t num = kp * (tn * CK * lam - td * A), den = td * lam * W;
                    acc = num <= 0 || (num * td < kp * tn * den && num < (i128_t)a.ma1 * den);
                    dec = acc || num > kp * den || (num * td >= kp * tn * den && num > (i128_t)a.mr1 * den);
                }
            }
            emit(a.res, dec, q, s, n_mb, n_ex, l, acc, flags, est);
            hist_add(a.res.hist, l, dec ? 1u : 0u);
            alive = alive && !dec;
        }
    }
}

cudaError_t launch_level_e(const LevelArgs &a, cudaStream_t st) {
    if (a.method == kHoph) level_he_kernel<<<148 * 4, 256, 0, st>>>(a);
    else level_e_kernel<<<148 * 2, 256, 0, st>>>(a);
    return cudaGetLastError();
}

// The survivor levels, one warp per surviving pair (k' <= 32: lane = bin of a group):
// the values of up to 8 further groups (query side contiguous in QM, set side one gather per
// lane and group) are loaded at once and the levels then decided from registers, so a pair
// costs one memory latency per 8 levels instead of one per level (r01's level_kernel walked
// its 32 pairs level by level in two launches with a compaction between).  Same decisions
// and records as level_kernel.
__device__ __forceinline__ void emit_one(const OutArgs &o, uint32_t q, uint32_t s, uint32_t n_mb, uint32_t n_excl,
                                         uint32_t groups, uint32_t verdict, uint32_t flags, float est) {
    if (o.dense) {
        write_hit(o.hits + (uint64_t)q * o.n_sets + s, q, o.set_id_base + s, n_mb, n_excl, groups, verdict, flags, est);
    } else if (verdict) {
        const unsigned long long idx = atomicAdd(o.count, 1ull);
        if (idx < o.cap) write_hit(o.hits + idx, q, o.set_id_base + s, n_mb, n_excl, groups, verdict, flags, est);
    }
}

// excluded bins of a pair among bins [0, nbins), lane-parallel over the mask words
__device__ __forceinline__ uint32_t excl_warp(const LevelArgs &a, uint32_t q, uint32_t s, uint32_t nbins, uint32_t lane) {
    uint32_t ex = 0;
    for (uint32_t w = lane; w * 32 < nbins; w += 32)
        ex += popc_masked(__ldg(a.QEM + (uint64_t)q * a.nw + w), __ldg(a.E + (uint64_t)w * a.ld + s), a.joint, w, nbins);
    return __reduce_add_sync(0xFFFFFFFFu, ex);
}

__global__ void __launch_bounds__(256) level_walk_kernel(const __grid_constant__ LevelArgs a) {
    constexpr uint32_t kAhead = 8;  // groups loaded at once
    const unsigned long long n = *a.count_in;
    const uint32_t lane = threadIdx.x & 31u;
    const unsigned long long nwarps = (unsigned long long)gridDim.x * (blockDim.x >> 5);
    const bool in_grp = lane < a.kp;
    for (unsigned long long i = blockIdx.x * (unsigned long long)(blockDim.x >> 5) + (threadIdx.x >> 5); i < n;
         i += nwarps) {
        const uint32_t q = a.in.q[i], s = a.in.s[i];
        u128_t st = a.in.state[i];
        uint32_t nmb = a.in.nmb[i];
        const uint32_t *qp = a.QM + (uint64_t)q * a.nb + lane;
        const uint32_t *fp = a.F + (uint64_t)lane * a.ld + s;
        bool done = false;
        for (uint32_t l0 = a.level; l0 <= a.nlev && !done; l0 += kAhead) {
            uint32_t qv[kAhead], sv[kAhead];
#pragma unroll
            for (uint32_t u = 0; u < kAhead; u++) {
                const uint32_t g = l0 - 1 + u;
                const bool ok = in_grp && g < a.nlev;
                qv[u] = ok ? __ldg(qp + (uint64_t)g * a.kp) : 0u;
                sv[u] = ok ? __ldg(fp + (uint64_t)g * a.kp * a.ld) : 1u;  // never equal when masked
            }
#pragma unroll
            for (uint32_t u = 0; u < kAhead; u++) {
                const uint32_t l = l0 + u;
                if (done || l > a.nlev) break;
                const uint32_t M = __popc(__ballot_sync(0xFFFFFFFFu, qv[u] == sv[u]));
                nmb += M;
                st += a.c[l - 1] * M;
                if (l == a.nlev) {  // the last group: final verdict
                    uint32_t verdict = 0, flags = 0, ex_tot = 0, nmb_out = nmb;
                    float est = -1.0f;
                    if (a.method == kGoph) {
                        ex_tot = excl_warp(a, q, s, a.nb, lane);
                        const uint32_t den = a.nb - ex_tot;
                        if (den == 0) {
                            flags = OPH_FLAG_UNDEFINED;
                        } else {
                            verdict = (uint64_t)nmb * a.t_den >= (uint64_t)a.t_num * den;
                            est = (float)nmb / (float)den;
                        }
                    } else {
                        // HOPH estimator over every group (R21, R22), exact over lam = lcm(1..k')
                        u128_t num = 0, csum = 0;
                        nmb_out = 0;
                        for (uint32_t g = 0; g < a.nlev; g++) {
                            const uint32_t qg = in_grp ? __ldg(qp + (uint64_t)g * a.kp) : 0u;
                            const uint32_t sg = in_grp ? __ldg(fp + (uint64_t)g * a.kp * a.ld) : 1u;
                            const uint32_t m = __popc(__ballot_sync(0xFFFFFFFFu, qg == sg));
                            const uint32_t ex = group_excl(a, q, s, g);
                            nmb_out += m;
                            ex_tot += ex;
                            const uint32_t d = a.kp - ex;
                            if (d == 0) continue;
                            num += a.c[g] * m * (a.lam / d);
                            csum += a.c[g];
                        }
                        if (csum == 0) {
                            flags = OPH_FLAG_UNDEFINED;
                        } else {
                            verdict = num * a.t_den >= (u128_t)a.t_num * a.lam * csum;
                            est = (float)((double)num / ((double)a.lam * (double)csum));
                        }
                    }
                    if (lane == 0) {
                        emit_one(a.res, q, s, nmb_out, ex_tot, a.nlev, verdict, flags, est);
                        if (a.res.hist) atomicAdd(a.res.hist + a.nlev, 1ull);
                    }
                    done = true;
                    break;
                }
                const bool acc = st >= a.acc[l - 1];
                const bool rej = !acc && (i128_t)st <= a.rej[l - 1];
                if (acc || rej) {
                    if (a.res.dense || acc) {
                        const uint32_t ex = excl_warp(a, q, s, l * a.kp, lane);
                        if (lane == 0) emit_one(a.res, q, s, nmb, ex, l, acc ? 1u : 0u, OPH_FLAG_EARLY, -1.0f);
                    }
                    if (lane == 0 && a.res.hist) atomicAdd(a.res.hist + l, 1ull);
                    done = true;
                }
            }
        }
    }
}

cudaError_t launch_level(const LevelArgs &a, cudaStream_t st) {
    // grid-stride over a device-side count: one CTA per SM covers sparse
    // survivor lists cheaply and still fills the chip for dense ones
    if (a.kp <= 32 && a.level_last == a.nlev) {
        level_walk_kernel<<<148 * 8, 256, 0, st>>>(a);
        return cudaGetLastError();
    }
    level_kernel<<<148 * 2, 256, 0, st>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K6: result lists.  Threshold: stable radix sort of (query << 32 | set_id).
// Top-k: stable sort by (~estimate_key << 32 | set_id), then stable sort by
// query; estimate_key = floor(n_mb 2^31 / den) is an exact order-preserving
// code of the rational n_mb/den for den <= 2^15 (distinct rationals differ
// by >= 1/(den1 den2) > 2^-31).  Then keep ranks < topk per query.
// ---------------------------------------------------------------------------
struct SelectWs {
    uint64_t *k0, *k1;
    uint32_t *v0, *v1;
    uint32_t *q0, *q1;
    uint64_t *head;
    uint8_t *keep;
    oph_hit *gathered;
    void *cub;
    size_t cub_bytes;
};

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

static size_t cub_bytes_needed(uint64_t n) {
    size_t a = 0, b = 0, c = 0, d = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (uint64_t *)nullptr, (uint64_t *)nullptr, (uint32_t *)nullptr,
                                    (uint32_t *)nullptr, (int)n);
    cub::DeviceRadixSort::SortPairs(nullptr, b, (uint32_t *)nullptr, (uint32_t *)nullptr, (uint32_t *)nullptr,
                                    (uint32_t *)nullptr, (int)n);
    cub::DeviceScan::InclusiveScan(nullptr, c, (uint64_t *)nullptr, (uint64_t *)nullptr, cuda::maximum<uint64_t>{}, (int)n);
    cub::DeviceSelect::Flagged(nullptr, d, (oph_hit *)nullptr, (uint8_t *)nullptr, (oph_hit *)nullptr,
                               (unsigned long long *)nullptr, (int)n);
    return std::max(std::max(a, b), std::max(c, d));
}

size_t select_temp_bytes(uint64_t n) {
    const uint64_t m = n ? n : 1;
    return align_up(8 * m) * 2 + align_up(4 * m) * 4 + align_up(8 * m) + align_up(m) + align_up(sizeof(oph_hit) * m) +
           align_up(cub_bytes_needed(m));
}

static SelectWs carve(void *ws, uint64_t n) {
    const uint64_t m = n ? n : 1;
    char *p = (char *)ws;
    SelectWs w;
    w.k0 = (uint64_t *)p; p += align_up(8 * m);
    w.k1 = (uint64_t *)p; p += align_up(8 * m);
    w.v0 = (uint32_t *)p; p += align_up(4 * m);
    w.v1 = (uint32_t *)p; p += align_up(4 * m);
    w.q0 = (uint32_t *)p; p += align_up(4 * m);
    w.q1 = (uint32_t *)p; p += align_up(4 * m);
    w.head = (uint64_t *)p; p += align_up(8 * m);
    w.keep = (uint8_t *)p; p += align_up(m);
    w.gathered = (oph_hit *)p; p += align_up(sizeof(oph_hit) * m);
    w.cub = p;
    w.cub_bytes = align_up(cub_bytes_needed(m));
    return w;
}

__global__ void sel_keys_threshold(const oph_hit *in, uint64_t n, uint64_t *k, uint32_t *v) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        k[i] = ((uint64_t)in[i].query << 32) | in[i].set_id;
        v[i] = (uint32_t)i;
    }
}

__global__ void sel_keys_topk(const oph_hit *in, uint64_t n, uint32_t k_bins, uint64_t *k, uint32_t *v) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const oph_hit h = in[i];
        const uint32_t den = k_bins - h.n_excl;
        uint64_t ek = 0;
        if (!(h.flags & OPH_FLAG_UNDEFINED) && den > 0 && h.n_mb <= den) ek = ((uint64_t)h.n_mb << 31) / den;
        k[i] = ((uint64_t)(0xFFFFFFFFu - (uint32_t)ek) << 32) | h.set_id;
        v[i] = (uint32_t)i;
    }
}

__global__ void sel_query_keys(const oph_hit *in, const uint32_t *perm, uint64_t n, uint32_t *qk) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const oph_hit h = in[perm[i]];
        qk[i] = (h.flags & OPH_FLAG_UNDEFINED) ? 0xFFFFFFFFu : h.query;
    }
}

__global__ void sel_heads(const uint32_t *qk, uint64_t n, uint64_t *head) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        head[i] = (i == 0 || qk[i] != qk[i - 1]) ? i : 0;
}

__global__ void sel_keep(const uint32_t *qk, const uint64_t *start, uint64_t n, uint32_t topk, uint8_t *keep) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        keep[i] = (qk[i] != 0xFFFFFFFFu) && (i - start[i] < topk);
}

__global__ void sel_gather(const oph_hit *in, const uint32_t *perm, uint64_t n, oph_hit *out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = in[perm[i]];
}

__global__ void sel_set_count(unsigned long long *c, uint64_t n) { *c = n; }

cudaError_t run_select(const oph_hit *in, uint64_t n, uint32_t mode, uint32_t topk, uint32_t k_bins, oph_hit *out,
                       unsigned long long *n_out, void *ws, size_t ws_bytes, cudaStream_t st) {
    if (ws_bytes < select_temp_bytes(n)) return cudaErrorInvalidValue;
    if (n == 0) {
        sel_set_count<<<1, 1, 0, st>>>(n_out, 0);
        return cudaGetLastError();
    }
    SelectWs w = carve(ws, n);
    const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 8);
    size_t tb = w.cub_bytes;
    if (mode == OPH_SELECT_THRESHOLD) {
        sel_keys_threshold<<<grid, 256, 0, st>>>(in, n, w.k0, w.v0);
        cudaError_t e = cub::DeviceRadixSort::SortPairs(w.cub, tb, w.k0, w.k1, w.v0, w.v1, (int)n, 0, 64, st);
        if (e != cudaSuccess) return e;
        sel_gather<<<grid, 256, 0, st>>>(in, w.v1, n, out);
        sel_set_count<<<1, 1, 0, st>>>(n_out, n);
        return cudaGetLastError();
    }
    sel_keys_topk<<<grid, 256, 0, st>>>(in, n, k_bins, w.k0, w.v0);
    cudaError_t e = cub::DeviceRadixSort::SortPairs(w.cub, tb, w.k0, w.k1, w.v0, w.v1, (int)n, 0, 64, st);
    if (e != cudaSuccess) return e;
    sel_query_keys<<<grid, 256, 0, st>>>(in, w.v1, n, w.q0);
    tb = w.cub_bytes;
    e = cub::DeviceRadixSort::SortPairs(w.cub, tb, w.q0, w.q1, w.v1, w.v0, (int)n, 0, 32, st);
    if (e != cudaSuccess) return e;
    sel_heads<<<grid, 256, 0, st>>>(w.q1, n, w.head);
    tb = w.cub_bytes;
    e = cub::DeviceScan::InclusiveScan(w.cub, tb, w.head, w.k0, cuda::maximum<uint64_t>{}, (int)n, st);
    if (e != cudaSuccess) return e;
    sel_keep<<<grid, 256, 0, st>>>(w.q1, w.k0, n, topk, w.keep);
    sel_gather<<<grid, 256, 0, st>>>(in, w.v0, n, w.gathered);
    tb = w.cub_bytes;
    e = cub::DeviceSelect::Flagged(w.cub, tb, w.gathered, w.keep, out, n_out, (int)n, st);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Text shingling (ingestion before the OPH build):
//   1. byte flags: token start = non-whitespace byte at a document start or
//      after whitespace; exclusive scan -> token index
//   2. token starts scattered; per token: document (binary search), FNV-1a 64
//      of its lowercased bytes
//   3. per w-gram start: seeded splitmix64 chain over w token hashes, id = h
//      mod |V|, key = doc << 32 | id (grams crossing a document: key ~0)
//   4. radix sort of the keys, unique, ids + per-document offsets
// Sizes use the bound T = (n_bytes + n_docs) / 2 + 1 tokens, so nothing is
// read back to the host.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool is_ws(uint8_t b) { return b == 32 || (b >= 9 && b <= 13); }

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

struct ShingleWs {
    uint8_t *docstart;   // [n_bytes]
    uint32_t *flag;      // [n_bytes + 1]: token-start flags
    uint32_t *idx;       // [n_bytes + 1]: exclusive scan of flag (idx[n_bytes] = the token count)
    uint64_t *tok_start; // [T]
    uint32_t *tok_doc;   // [T]
    uint64_t *tok_hash;  // [T]
    uint64_t *k0, *k1;   // [T]
    unsigned long long *n_unique;
    void *cub;
    size_t cub_bytes;
};

static uint64_t shingle_T(uint64_t n_bytes, uint64_t n_docs) { return (n_bytes + n_docs) / 2 + 1; }

static size_t shingle_cub_bytes(uint64_t n_bytes, uint64_t T) {
    size_t a = 0, b = 0, c = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, a, (uint32_t *)nullptr, (uint32_t *)nullptr, (int)(n_bytes + 1));
    cub::DeviceRadixSort::SortKeys(nullptr, b, (uint64_t *)nullptr, (uint64_t *)nullptr, (int)T);
    cub::DeviceSelect::Unique(nullptr, c, (uint64_t *)nullptr, (uint64_t *)nullptr, (unsigned long long *)nullptr,
                              (int)T);
    return std::max(a, std::max(b, c));
}

size_t shingle_temp_bytes(uint64_t n_bytes, uint64_t n_docs) {
    const uint64_t T = shingle_T(n_bytes, n_docs);
    return align_up(n_bytes + 1) + 2 * align_up(4 * (n_bytes + 1)) + align_up(8 * T) + align_up(4 * T) +
           align_up(8 * T) * 3 + align_up(8) + align_up(shingle_cub_bytes(n_bytes, T));
}

__global__ void sh_docstart(const uint64_t *doc_offsets, uint64_t n_docs, uint64_t n_bytes, uint8_t *docstart) {
    for (uint64_t d = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; d < n_docs; d += (uint64_t)gridDim.x * blockDim.x)
        if (doc_offsets[d] < n_bytes) docstart[doc_offsets[d]] = 1;
}

__global__ void sh_flags(const uint8_t *text, const uint8_t *docstart, uint64_t n_bytes, uint32_t *flag) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p <= n_bytes;
         p += (uint64_t)gridDim.x * blockDim.x)
        flag[p] = p < n_bytes && !is_ws(text[p]) && (docstart[p] || p == 0 || is_ws(text[p - 1]));
}

__global__ void sh_scatter(const uint32_t *flag, uint64_t n_bytes, const uint32_t *idx, uint64_t *tok_start) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n_bytes;
         p += (uint64_t)gridDim.x * blockDim.x)
        if (flag[p]) tok_start[idx[p]] = p;
}

// per token: its document and the FNV-1a 64 of its lowercased bytes
__global__ void sh_tokens(const __grid_constant__ ShingleArgs a, const uint32_t *idx, const uint64_t *tok_start,
                          uint32_t *tok_doc, uint64_t *tok_hash) {
    const uint64_t n_tok = idx[a.n_bytes];
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n_tok; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t p0 = tok_start[t];
        uint64_t lo = 0, hi = a.n_docs;  // the last document with offsets[d] <= p0
        while (lo + 1 < hi) {
            const uint64_t m = (lo + hi) >> 1;
            if (a.doc_offsets[m] <= p0) lo = m; else hi = m;
        }
        const uint64_t end = a.doc_offsets[lo + 1];
        uint64_t h = 0xCBF29CE484222325ull;
        for (uint64_t p = p0; p < end; p++) {
            uint8_t b = a.text[p];
            if (is_ws(b)) break;
            if (b >= 65 && b <= 90) b += 32;
            h = (h ^ b) * 0x100000001B3ull;
        }
        tok_doc[t] = (uint32_t)lo;
        tok_hash[t] = h;
    }
}

// per gram start t < T: key = doc << 32 | id, or ~0 (no gram: past the tokens or crossing a document)
__global__ void sh_grams(const __grid_constant__ ShingleArgs a, const uint32_t *idx, const uint32_t *tok_doc,
                         const uint64_t *tok_hash, uint64_t T, uint64_t *keys) {
    const uint64_t n_tok = idx[a.n_bytes];
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < T; t += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t key = ~0ull;
        if (t + a.w <= n_tok && tok_doc[t + a.w - 1] == tok_doc[t]) {
            uint64_t h = a.seed;
            for (uint32_t i = 0; i < a.w; i++) h = mix64(h + 0x9E3779B97F4A7C15ull + tok_hash[t + i]);
            key = ((uint64_t)tok_doc[t] << 32) | (uint32_t)(h % a.V);
        }
        keys[t] = key;
    }
}

// ids and per-document offsets from the sorted distinct keys (the last one may be ~0)
__global__ void sh_output(const __grid_constant__ ShingleArgs a, const uint64_t *keys, const unsigned long long *n_unique) {
    uint64_t n = *n_unique;
    if (n && keys[n - 1] == ~0ull) n--;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    for (uint64_t i = tid; i < n && i < a.ids_cap; i += stride) a.ids[i] = (uint32_t)keys[i];
    for (uint64_t d = tid; d <= a.n_docs; d += stride) {
        uint64_t lo = 0, hi = n;  // first key with doc >= d
        while (lo < hi) {
            const uint64_t m = (lo + hi) >> 1;
            if ((keys[m] >> 32) < d) lo = m + 1; else hi = m;
        }
        a.set_offsets[d] = d == a.n_docs ? n : lo;
    }
    if (tid == 0) *a.n_ids = n;
}

cudaError_t run_shingle(const ShingleArgs &a, void *ws, size_t ws_bytes, cudaStream_t st) {
    if (ws_bytes < shingle_temp_bytes(a.n_bytes, a.n_docs)) return cudaErrorInvalidValue;
    const uint64_t T = shingle_T(a.n_bytes, a.n_docs);
    char *p = (char *)ws;
    ShingleWs w;
    w.docstart = (uint8_t *)p; p += align_up(a.n_bytes + 1);
    w.flag = (uint32_t *)p; p += align_up(4 * (a.n_bytes + 1));
    w.idx = (uint32_t *)p; p += align_up(4 * (a.n_bytes + 1));
    w.tok_start = (uint64_t *)p; p += align_up(8 * T);
    w.tok_doc = (uint32_t *)p; p += align_up(4 * T);
    w.tok_hash = (uint64_t *)p; p += align_up(8 * T);
    w.k0 = (uint64_t *)p; p += align_up(8 * T);
    w.k1 = (uint64_t *)p; p += align_up(8 * T);
    w.n_unique = (unsigned long long *)p; p += align_up(8);
    w.cub = p;
    w.cub_bytes = align_up(shingle_cub_bytes(a.n_bytes, T));
    const unsigned gb = (unsigned)std::min<uint64_t>((a.n_bytes + 256) / 256, 148ull * 32);
    const unsigned gt = (unsigned)std::min<uint64_t>((T + 255) / 256, 148ull * 32);
    cudaError_t e;
    if ((e = cudaMemsetAsync(w.docstart, 0, a.n_bytes + 1, st)) != cudaSuccess) return e;
    sh_docstart<<<(unsigned)std::min<uint64_t>((a.n_docs + 255) / 256 + 1, 148ull * 8), 256, 0, st>>>(
        a.doc_offsets, a.n_docs, a.n_bytes, w.docstart);
    sh_flags<<<gb, 256, 0, st>>>(a.text, w.docstart, a.n_bytes, w.flag);
    size_t tb = w.cub_bytes;
    // idx[p] = token starts before p (idx[n_bytes] = the token count)
    if ((e = cub::DeviceScan::ExclusiveSum(w.cub, tb, w.flag, w.idx, (int)(a.n_bytes + 1), st)) != cudaSuccess)
        return e;
    sh_scatter<<<gb, 256, 0, st>>>(w.flag, a.n_bytes, w.idx, w.tok_start);
    sh_tokens<<<gt, 256, 0, st>>>(a, w.idx, w.tok_start, w.tok_doc, w.tok_hash);
    sh_grams<<<gt, 256, 0, st>>>(a, w.idx, w.tok_doc, w.tok_hash, T, w.k0);
    tb = w.cub_bytes;
    if ((e = cub::DeviceRadixSort::SortKeys(w.cub, tb, w.k0, w.k1, (int)T, 0, 64, st)) != cudaSuccess) return e;
    tb = w.cub_bytes;
    if ((e = cub::DeviceSelect::Unique(w.cub, tb, w.k1, w.k0, w.n_unique, (int)T, st)) != cudaSuccess) return e;
    sh_output<<<gt, 256, 0, st>>>(a, w.k0, w.n_unique);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// CSR contract check (debug aid, oph_validate_sets): warp per set, lanes compare
// neighbouring ids; any violation sets *bad.
// ---------------------------------------------------------------------------
__global__ void validate_kernel(const uint64_t *offsets, const uint32_t *ids, uint64_t n_sets, uint64_t V,
                                uint32_t *bad) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t s = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); s < n_sets; s += nwarps) {
        const uint64_t lo = offsets[s], hi = offsets[s + 1];
        bool err = hi < lo;
        if (!err)
            for (uint64_t e = lo + lane; e < hi; e += 32) {
                const uint32_t x = ids[e];
                err |= (uint64_t)x >= V;
                if (e + 1 < hi) err |= ids[e + 1] <= x;
            }
        if (__any_sync(0xFFFFFFFFu, err) && lane == 0) atomicOr(bad, 1u);
    }
}

cudaError_t launch_validate(const uint64_t *offsets, const uint32_t *ids, uint64_t n_sets, uint64_t V, uint32_t *bad,
                            cudaStream_t st) {
    if (n_sets == 0) return cudaSuccess;
    const unsigned grid = (unsigned)std::min<uint64_t>((n_sets + 7) / 8, 148ull * 16);
    validate_kernel<<<grid, 256, 0, st>>>(offsets, ids, n_sets, V, bad);
    return cudaGetLastError();
}

#include "bitjoin.cuh"

}  // namespace ophgpu
