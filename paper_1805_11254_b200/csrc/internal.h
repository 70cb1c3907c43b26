// Private interface between the host planner / C-ABI (ophgpu_host.cu) and the
// sm_100a kernels (ophgpu_kernels.cu).  Not installed, not part of the ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/ophgpu.h"

namespace ophgpu {

constexpr uint32_t kEmpty = 0xFFFFFFFFu;       // collection-side empty bin ("⊗")
constexpr uint32_t kQueryEmpty = 0xFFFFFFFEu;  // query-side empty bin: never equals a stored value
constexpr int kMaxGroups = OPH_MAX_GROUPS;

// psi, keys already derived and masked to w bits.
struct PsiParams {
    uint64_t V;         // |V|
    uint32_t mask;      // 2^w - 1 (w <= 32)
    uint32_t shift;     // ceil(w / 2)
    uint32_t kappa[4];
    uint32_t mu[4];     // odd
    uint32_t identity;  // psi(x) = x
    uint32_t pow2;      // |V| == 2^w: no cycle walking
    uint32_t hmul, hsh; // w < 32: 2^(32-w) and 32 - w + shift (see psi_pass)
};

// One range [start, start+len) cut into nb bins by the floor rule.
struct RangeBins {
    uint64_t start, len;
    uint32_t shift;     // log2(len / nb) when len / nb is an exact power of two ...
    uint32_t pow2;      // ... flagged here (fast path: bin = (p-start) >> shift)
};

struct BuildArgs {
    const uint64_t *offsets;
    const uint32_t *ids;
    uint64_t n_sets, ld;
    PsiParams psi;
    // flat OPH
    uint32_t do_flat, k;
    RangeBins flat;
    uint32_t *oph, *oph_empty;
    // hierarchical
    uint32_t do_hier, L, kp;
    uint32_t hier_pow2_halves;  // 1:1 split of |V| = 2^log2V, kp = 2^log2kp: group = leading ones of p
    uint32_t log2V, log2kp;
    RangeBins grp[kMaxGroups];
    uint32_t *hoph, *hoph_empty;
    uint32_t hder;  // FAST layout: leading HOPH groups derived from the OPH minima (set by launch_build)
};

struct MinwiseArgs {
    const uint64_t *offsets;
    const uint32_t *ids;
    uint64_t n_sets, ld;
    uint64_t V, seed;
    uint32_t k, w;
    uint32_t *mw;
    uint8_t *flags;
    uint32_t hmul, hsh;  // w < 32: 2^(32-w) and 32 - w + ceil(w/2) (set by launch_minwise)
};

typedef unsigned __int128 u128_t;
typedef __int128 i128_t;

// Survivor list (structure of arrays), one per level parity.
struct SurvList {
    uint32_t *q;      // global query index
    uint32_t *s;      // local set index
    u128_t *state;    // M_c (GOPH) or S_l (HOPH: up to D k' ~ 2^75 for the 1:2 split of 2^32)
    uint32_t *nmb;    // raw matched bins so far
};

struct OutArgs {
    oph_hit *hits;
    uint64_t cap;
    unsigned long long *count;
    uint32_t dense;
    uint32_t set_id_base;
    uint64_t n_sets;  // dense row length
    unsigned long long *hist;  // optional termination-level histogram [OPH_STOP_HIST_LEN]
};

enum Method : uint32_t { kFull = 0, kGoph = 1, kHoph = 2, kMinwise = 3 };

struct ScanArgs {
    const uint32_t *F;      // collection values [nb][ld]
    const uint32_t *E;      // collection masks [nw][ld] (null for MinWise)
    const uint8_t *sflags;  // MinWise set flags
    uint64_t n_sets, ld;
    const uint32_t *QT;     // prepared queries, bin-major [nb][ldq]
    const uint32_t *QE;     // query masks [nw][ldq]
    const uint8_t *qflags;  // MinWise query flags [ldq]
    uint64_t ldq;
    uint32_t q_col0;        // first query column of this chunk
    uint32_t nq;            // queries in this chunk
    uint32_t method;
    uint32_t nscan;         // bins scanned (a prefix of the bins)
    uint32_t nw_load;       // mask words held for the epilogue
    uint32_t final_;        // the scan ends with the final verdict
    uint32_t nbins_total;   // k for the final verdict's denominator
    uint32_t joint, t_num, t_den;
    uint32_t level;         // groups compared at the end of the scan
    u128_t w1;              // state = w1 * raw count (HOPH c_1, else 1)
    uint32_t acc_cnt;       // Similar iff raw count >= acc_cnt (state >= acc <=> count >= ceil(acc / w1))
    int32_t rej_cnt;        // NotSimilar iff raw count <= rej_cnt (-1: never)
    uint32_t tiles_per_cta;
    OutArgs out;
    SurvList surv;
    unsigned long long *surv_count;
    uint64_t surv_cap;      // survivor list capacity
    // list mode: the sets to scan are set_list[0 .. *list_count) (PROBE overflow sets)
    const uint32_t *set_list;
    const unsigned long long *list_count;
    uint64_t s_begin;       // range mode: scan sets [s_begin, n_sets) (s_begin even)
    uint32_t one;           // = 1, opaque to the compiler (see acc_eq)
};

// PROBE strategy: per scanned bin b, the chunk's query values are hashed into
// an open-addressing table T_b of 2^log2S slots, slot = value << 32 | (q+1)
// (0 = free, linear probing; duplicates occupy separate slots), and into a
// blocked Bloom filter of 2^log2W 32-bit words per bin, bin-major
// [bin][word] (a slab of 32 bins is the contiguous image the join kernel
// copies into shared memory in one piece).
struct TableArgs {
    const uint32_t *QT;     // prepared queries, bin-major [nb][ldq]
    const uint8_t *qflags;  // MinWise query flags (flagged queries never match)
    uint64_t ldq;
    uint32_t q_col0, nq, nscan, log2S;
    uint32_t minwise;
    unsigned long long *table;  // [nscan][2^log2S]
    uint32_t *bloom;            // [32 * ceil(nscan/32)][2^log2W]
    uint32_t log2W;
};

constexpr int kJoinList = 4;        // distinct matched queries tracked per set before falling back to BRUTE
// queries per join pass: the Bloom filter keeps >= 16 bits per query per bin in
// 64-KB slabs of 32 bins x 512 words (<= 1024 queries), 16 x 1024 (<= 2048) or
// 8 x 2048 (<= 4096)
constexpr uint32_t kJoinMaxQ = 4096;
constexpr uint32_t kJoinMaxLog2W = 11;

struct ProbeArgs {
    const uint32_t *F, *E;
    const uint8_t *sflags;
    uint64_t n_sets, ld;
    const unsigned long long *table;
    const uint32_t *bloom;
    uint32_t log2S, nscan, log2W;
    uint32_t R;             // sets per CTA (multiple of 32; set by launch_probe)
    uint32_t nlist;         // matched-query list entries per set, 2 or kJoinList (set by launch_probe)
    const uint32_t *QEM;    // query masks, query-major [n_q][nw]
    const uint8_t *qflags;  // MinWise query flags, indexed by global query
    uint32_t nw, nbins_total;
    uint32_t q_col0;        // global index of the chunk's first query
    uint32_t nq;            // queries in this pass
    uint32_t method, final_, level, joint, t_num, t_den;
    u128_t w1;              // as ScanArgs
    uint32_t acc_cnt;
    int32_t rej_cnt;
    OutArgs out;
    SurvList surv;
    unsigned long long *surv_count;
    uint64_t surv_cap;
    uint32_t *ovf_list;     // sets that matched more than kJoinList queries
    unsigned long long *ovf_count;
    uint64_t s_begin, s_end;  // the sets [s_begin, s_end) are probed
};

struct LevelArgs {
    const uint32_t *F, *E;
    uint64_t n_sets, ld;
    const uint32_t *QM;     // prepared queries, query-major [n_q][nb]
    const uint32_t *QEM;    // query masks, query-major [n_q][nw]
    uint32_t nb, nw;
    uint32_t method;        // kGoph | kHoph
    uint32_t level;         // first 1-indexed group processed by this launch
    uint32_t level_last;    // last group processed by this launch (<= nlev)
    uint32_t nlev;          // n (GOPH) or L (HOPH)
    uint32_t kp, joint, t_num, t_den;
    u128_t acc[kMaxGroups]; // per-level thresholds on the state, index l-1 (~0: never)
    i128_t rej[kMaxGroups]; // (-1: never)
    u128_t c[kMaxGroups];   // group weights (GOPH: 1)
    u128_t lam;             // lcm(1..kp) for the HOPH final verdict
    SurvList in, out;
    const unsigned long long *count_in;
    unsigned long long *count_out;
    OutArgs res;
    // multi-level BRUTE scan (levels_kernel; states < 2^32): all groups of a query
    // block in one pass, decided group by group
    const uint32_t *QT;     // prepared queries, bin-major [nb][ldq]
    uint64_t ldq;
    uint32_t q_col0, nq;    // query columns [q_col0, q_col0 + nq)
    // the counter of a pair is state << sh | raw matched bins (sh = 10 for HOPH, 0 for GOPH)
    uint32_t sh;
    uint32_t w32[kMaxGroups];    // c_l << sh | (sh ? 1 : 0) (GOPH: 1)
    uint32_t acc32[kMaxGroups];  // Similar iff counter >= acc32 (= A_l << sh; UINT32_MAX: never)
    uint32_t rej1[kMaxGroups];   // NotSimilar iff counter < rej1 (= (R_l + 1) << sh; 0: never)
    uint64_t s_begin;
    uint32_t tiles_per_cta;
    uint32_t one;           // = 1, opaque to the compiler (see acc_eq)
    // empty-aware GOPH (levels_e_kernel, E1-E4)
    uint32_t eaware;
    const uint32_t *QE;     // query empty masks, bin-major [nw][ldq]
    uint32_t ma1;           // #{m : P(X <= m) <= eps}, X ~ Bin(k', T) (0: never Similar by the tail)
    uint32_t mr1;           // min{m : P(X >= m) <= eps} - 1
    // empty-aware HOPH over every pair of queries [q_col0, q_col0 + nq) x the sets (no list)
    uint32_t implicit;
};

// BITMAP strategy (bitjoin.cuh): one block of <= 1024 queries against the collection
struct BitArgs {
    const uint32_t *F, *E;  // collection values [nb][ld], masks [nw][ld]
    uint64_t n_sets, ld, s_begin;  // sets [s_begin, n_sets) are scanned
    const uint32_t *QT;     // prepared queries, bin-major [nb][ldq]
    uint64_t ldq;
    const uint32_t *QM;     // prepared queries, query-major [n_q][nb]
    const uint32_t *QEM;    // query masks, query-major [n_q][nw]
    uint32_t nb, nw, nscan, kp, nlev, nbins_total;
    uint32_t npre;          // bins [0, npre) are staged per CTA tile (the rest read directly)
    uint32_t nstage;        // CTA tiles staged ahead (ring of value buffers, 2 .. 8)
    uint32_t qb0, nqb;      // this block: query columns [qb0, qb0 + nqb), nqb <= 1024 qw
    uint32_t pipe;          // 1: bit_pipe_kernel (full OPH; GOPH over levels 1 .. level_b, then walks)
    uint32_t level_b;       // GOPH levels decided by the bitmap in bit_pipe_kernel (the rest walked)
    uint32_t qw;            // 32-query words per lane: rows of 1024 qw bits (1, or 2 for full OPH / GOPH)
    uint32_t method, mode_hoph, joint, t_num, t_den, level_final;
    // value ranges of the bins: bin b = range b / bins_per_range, floor rule inside it
    uint32_t bins_per_range;
    RangeBins ranges[kMaxGroups];
    uint32_t thr_on[kMaxGroups];    // level l (index l-1) has a threshold
    uint32_t acc_cnt[kMaxGroups];   // Similar iff state >= acc_cnt (GOPH: M_c; HOPH: T_l)
    int32_t rej_cnt[kMaxGroups];    // NotSimilar iff state <= rej_cnt (-1: never)
    u128_t acc128[kMaxGroups];      // HOPH: the planner's thresholds on S_l (the per-pair walk)
    i128_t rej128[kMaxGroups];
    u128_t c[kMaxGroups];           // HOPH weights (final estimator)
    u128_t lam;                     // lcm(1..kp)
    uint32_t *idx;                  // [vpos] position -> row (0: the zero row)
    uint64_t vpos;                  // |V|
    uint32_t *rows;                 // [1 + rows][32] query bitmasks
    uint32_t *nrows;                // rows claimed
    uint32_t *max_eq;               // [32 qw] per query word: max empty bins of its queries
    uint32_t *max_eq_pref;          // [nw + 1][64]: per query word, max over its queries of the empty bins in [0, 32 c)
    uint32_t exit_from;             // full OPH, threshold mode: first bin count checked for a set's exit (0: off)
    uint32_t exit_every;            // then every exit_every bins (32 or 64; exit_from a multiple of 32)
    unsigned long long *scanned;    // optional: adds the (set, bin) rows gathered (oph_results.d_bins_scanned)
    OutArgs out;
};

struct PrepArgs {
    const uint32_t *values;  // caller's query sketches [nb][ld_in]
    const uint32_t *empty;   // [nw][ld_in] or null
    const uint8_t *flags;    // MinWise [n_q] or null
    uint64_t ld_in;
    uint32_t n_q, nb, nw;
    uint32_t remap;          // OPH methods: empty -> kQueryEmpty
    uint32_t *QT, *QE, *QM, *QEM;
    uint8_t *qflags;
    uint64_t ldq;
};

struct JaccardArgs {
    const uint64_t *q_offsets, *s_offsets;
    const uint32_t *q_ids, *s_ids;
    const uint32_t *query, *set;
    uint64_t n;
    uint32_t *inter, *uni;
};

struct ShingleArgs {
    const uint8_t *text;
    const uint64_t *doc_offsets;
    uint64_t n_docs, n_bytes;
    uint32_t w;
    uint64_t V, seed;
    uint64_t *set_offsets;
    uint32_t *ids;
    uint64_t ids_cap;
    unsigned long long *n_ids;
};

// ---- launchers (ophgpu_kernels.cu); all return cudaGetLastError()
cudaError_t launch_build(const BuildArgs &a, cudaStream_t st);
cudaError_t launch_minwise(const MinwiseArgs &a, cudaStream_t st);
cudaError_t launch_prep(const PrepArgs &a, cudaStream_t st);
cudaError_t launch_scan(const ScanArgs &a, uint32_t B, cudaStream_t st);
cudaError_t launch_table(const TableArgs &a, cudaStream_t st);
cudaError_t launch_probe(const ProbeArgs &a, cudaStream_t st);
cudaError_t launch_level(const LevelArgs &a, cudaStream_t st);
cudaError_t launch_level_e(const LevelArgs &a, cudaStream_t st);  // empty-aware rule over a survivor list
cudaError_t launch_levels_scan(const LevelArgs &a, cudaStream_t st);
cudaError_t launch_jaccard(const JaccardArgs &a, cudaStream_t st);
cudaError_t launch_bit_block(const BitArgs &a, cudaStream_t st);
// CSR contract check: *bad (device) |= 1 on a violation
cudaError_t launch_validate(const uint64_t *offsets, const uint32_t *ids, uint64_t n_sets, uint64_t V, uint32_t *bad,
                            cudaStream_t st);
size_t shingle_temp_bytes(uint64_t n_bytes, uint64_t n_docs);
cudaError_t run_shingle(const ShingleArgs &a, void *ws, size_t ws_bytes, cudaStream_t st);
size_t select_temp_bytes(uint64_t n);
cudaError_t run_select(const oph_hit *in, uint64_t n, uint32_t mode, uint32_t topk, uint32_t k_bins, oph_hit *out,
                       unsigned long long *n_out, void *ws, size_t ws_bytes, cudaStream_t st);

}  // namespace ophgpu
