/*
 * ophgpu.h -- C-ABI of the B200-native (sm_100a) OPH / GOPH / HOPH near-duplicate
 * scoring library (arxiv 1805.11254, "Hierarchical One Permutation Hashing").
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, Rn = DESIGN.md
 * reading n.  Problem statement (R1): given a query q and a
 * collection D, return the p in D with sim(q, p) >= T, sim = Jaccard, here
 * estimated from one-permutation-hashing sketches and decided by the paper's
 * comparison rules.
 *
 * Conventions for every entry point
 *  - d_ pointers are DEVICE pointers, owned by the caller (allocate them with
 *    cudaMalloc / torch).  The library never allocates or frees caller memory
 *    and keeps no device state between calls.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  Every call only ENQUEUES work on that stream and returns; the
 *    caller synchronises.  Returned statuses cover argument checking and
 *    launch errors (OPH_ECUDA); device-side result overflow is reported
 *    through the result counters (see oph_results).  The exceptions, each one
 *    host synchronisation of `stream` inside the call:
 *      (1) compare_goph / compare_hoph with the PROBE strategy (or AUTO
 *          choosing it) when the survivor capacity is smaller than
 *          32 x n_sets x the query count: the call first scores every query
 *          at once and reads the survivor count back; only if the list
 *          overflowed does it redo the queries in capacity-sized chunks
 *          (a larger survivor_capacity avoids it);
 *      (2) the first AUTO call on a collection (keyed by its value pointer,
 *          size, bins and method) reads the PROBE sample's overflow count to
 *          choose between PROBE and a register scan; later calls reuse the
 *          decision without synchronising (OPH_STRATEGY_PROBE / BRUTE /
 *          BITMAP never sample);
 *      (3) oph_validate_sets, and the builds when OPHGPU_VALIDATE is set.
 *  - Sketch matrices are BIN-MAJOR uint32: element (bin b, set s) lives at
 *    d_values[b * ld + s], with a row stride ld >= n_sets that is a multiple
 *    of 4 (oph_sketch_ld() gives the canonical one).  An empty bin holds
 *    OPH_EMPTY.  Empty masks are bin-major too: bit (b % 32) of word
 *    d_empty[(b / 32) * ld + s] is set iff bin b of set s is empty.
 *  - Sets are CSR on the device: ids of set s are d_ids[d_offsets[s] ..
 *    d_offsets[s+1]), strictly increasing and < vocab_size.  The
 *    hot path does not check this; oph_validate_sets does (a debug aid), and
 *    with the environment variable OPHGPU_VALIDATE set the two builds run it
 *    first and return OPH_EINVAL on a violation.
 *  - Errors: OPH_EINVAL for bad arguments; OPH_EINCOMPAT when query and
 *    collection sketches differ in permutation seed, universe or layout
 *    (S:62); OPH_EAMBIGUOUS when a binomial tail lies within 1e-9
 *    relative of epsilon (the decision could not be certified);
 *    OPH_ENOMEM when the workspace is too small; OPH_ECUDA for launch errors.
 */
#ifndef OPHGPU_H
#define OPHGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    OPH_OK = 0,
    OPH_EINVAL = 1,
    OPH_EINCOMPAT = 2,
    OPH_EOVERFLOW = 3,
    OPH_ECUDA = 4,
    OPH_EAMBIGUOUS = 5,
    OPH_ENOMEM = 6
} oph_status;

#define OPH_EMPTY 0xFFFFFFFFu /* the empty bin "⊗" */

enum { OPH_PERM_KEYED = 0, OPH_PERM_IDENTITY = 1 };      /* identity: worked examples */
enum { OPH_EMPTY_EITHER = 0, OPH_EMPTY_JOINT = 1 };      /* R6: either-empty (examples) / joint (Eq. 4) */
enum { OPH_RES_THRESHOLD = 0, OPH_RES_DENSE = 1 };       /* compare output mode */
enum { OPH_SELECT_THRESHOLD = 0, OPH_SELECT_TOPK = 1 };  /* topk_or_threshold_results mode */
enum { OPH_METHOD_FULL = 0, OPH_METHOD_GOPH = 1, OPH_METHOD_HOPH = 2, OPH_METHOD_MINWISE = 3 };

#define OPH_FLAG_UNDEFINED 1u /* estimate undefined: k - N_eb = 0 (R7) or empty MinWise set */
#define OPH_FLAG_EARLY 2u     /* GOPH/HOPH stopped before the last group: no estimate */

/* The permutation psi: a keyed 4-round
 * bijection of [0, vocab_size) derived from `seed`, or the identity. */
typedef struct {
    uint64_t vocab_size; /* |V|, 1 .. 2^32 */
    uint64_t seed;
    uint32_t kind;       /* OPH_PERM_KEYED | OPH_PERM_IDENTITY */
    uint32_t pad;
} oph_perm;

/* Flat OPH layout: k bins by the floor rule
 * [floor(b|V|/k), floor((b+1)|V|/k)); GOPH views the k bins as n = k/kprime
 * groups of kprime consecutive bins. */
typedef struct {
    uint64_t vocab_size;
    uint32_t k;      /* 1 .. 65535, k <= vocab_size */
    uint32_t kprime; /* GOPH group size; k % kprime == 0 */
} oph_flat_layout;

#define OPH_MAX_GROUPS 64

/* Hierarchical layout (R17-R18), filled by
 * oph_hier_layout_make: group j covers [start[j], start[j]+len[j]) and is cut
 * into kprime bins by the floor rule. */
typedef struct {
    uint64_t vocab_size;
    uint32_t a, b;   /* split ratio a:b, r = a/(a+b) */
    uint32_t kprime; /* bins per group */
    uint32_t L;      /* number of groups */
    uint64_t start[OPH_MAX_GROUPS];
    uint64_t len[OPH_MAX_GROUPS];
} oph_hier_layout;

/* A set collection in CSR form on the device. */
typedef struct {
    const uint64_t *d_offsets; /* [n_sets + 1] */
    const uint32_t *d_ids;     /* [d_offsets[n_sets]] */
    uint64_t n_sets;
} oph_sets;

/* A read-only view of a sketch matrix (queries or collection). */
typedef struct {
    const uint32_t *d_values; /* [n_bins][ld] */
    const uint32_t *d_empty;  /* [ceil(n_bins/32)][ld] empty masks; NULL for MinWise */
    const uint8_t *d_flags;   /* MinWise only: [n_sets], 1 = empty set (no sketch); else NULL */
    uint64_t n_sets;
    uint64_t ld;              /* row stride (elements), multiple of 4, >= n_sets */
    uint32_t n_bins;          /* k (flat / MinWise) or L*kprime (hierarchical) */
    uint32_t pad;
    uint64_t seed;            /* permutation seed the sketches were built with */
    uint64_t vocab_size;      /* |V| they were built over */
} oph_sketches;

/* Filter parameters: T = t_num / t_den in (0, 1] (R23),
 * epsilon in (0, 1) (Definition 1). */
typedef struct {
    uint32_t t_num, t_den;
    double epsilon;
    uint32_t empty_mode; /* OPH_EMPTY_EITHER | OPH_EMPTY_JOINT */
    uint32_t strategy;   /* OPH_STRATEGY_*: how the collection scan finds matched bins (results identical) */
    uint32_t variant;    /* OPH_VARIANT_*: the filter rule (compare_goph only; 0 elsewhere) */
} oph_params;

/* Filter rule of compare_goph / compare_hoph.
 *   PAPER       : Algorithm 1 as read in DESIGN.md R10-R16: the
 *                 binomial trials of a group are its k' bins.
 *   EMPTY_AWARE : the empty-aware variant (DESIGN.md
 *                 E1-E4): the trials are the pair's non-excluded bins (known
 *                 from the empty masks before any value is compared);
 *                 M_ra = k' (T D - M_c) / R with D the pair's non-excluded
 *                 bins, R those not yet compared; Algorithm 1's tests on M_ra
 *                 unchanged; R = 0 completes the comparison with the full-OPH
 *                 verdict.  Identical to PAPER when no bin is excluded.  Needs
 *                 n k' <= 512 (OPH_EINVAL otherwise).  A pair with no matched
 *                 bin is never Similar under it (E5), so threshold results
 *                 without a termination histogram take the PROBE join (AUTO /
 *                 PROBE) and decide only the listed pairs; dense records, a
 *                 histogram or BRUTE run one register scan over all groups.
 *                 compare_hoph (EH1-EH5): Algorithm 2's mass balance
 *                 with group j's trials its usable bins d_j = k' - excl_j; the
 *                 groups with d_j > 0 (weight C_K) decide: after l groups
 *                 x = k' (T C_K - A_l) / W_l with A_l = sum_{j<=l} c_j m_j / d_j
 *                 and W_l the usable weight left, Algorithm 2's tests on x,
 *                 exact in 128-bit integers; W_l = 0 or the last group: the
 *                 HOPH estimator.  Identical to PAPER when no bin is excluded.
 *                 Threshold results without a histogram take the PROBE join
 *                 (pairs with a matched bin); otherwise every pair is walked.
 *                 EINVAL when k'^2 t_num t_den D lcm(1..k') >= 2^124.
 *   Full OPH and MinWise refuse EMPTY_AWARE (OPH_EINVAL). */
enum { OPH_VARIANT_PAPER = 0, OPH_VARIANT_EMPTY_AWARE = 1 };

/* Collection-scan strategies; every strategy returns
 * identical results.
 *   AUTO : PROBE when it applies (threshold results, and pairs with no matched
 *          bin are decided NotSimilar at the scanned level), else BRUTE.  It
 *          probes a leading sample (1/16 of the sets, >= 16384) first and
 *          scans the rest with BRUTE if more than a quarter of the sample
 *          matched more than 4 distinct queries (one host synchronisation).
 *          The decision is remembered per (collection buffer, n_sets, bins,
 *          method), so repeated calls on a collection neither sample nor
 *          synchronise (a BRUTE decision makes later calls BRUTE outright);
 *          it affects speed only, never results.
 *   BRUTE: every (query, set, bin) equality is tested (register-blocked
 *          query tiles; cost ~ Q N bins; best when most pairs share bins).
 *   PROBE: a hash join in passes of <= 4096 queries, each one stream over
 *          the scanned collection bins: per bin, the pass's query values go
 *          into an exact hash table and a Bloom filter; every set bin tests
 *          the filter (held in shared memory) and the rare positives are
 *          verified in the table, so only matching (query, set, bin) triples
 *          cost more than a filter test (cost ~ N bins + matches; best for
 *          low background similarity).  Sets matching more than 4 distinct
 *          queries are re-scanned by BRUTE.
 *   BITMAP: a value-indexed bitmap join in blocks of 1024 queries: per block, a
 *          table over the |V| bin positions maps a value to the bitmask of the
 *          queries holding it in that bin (built from the query sketches);
 *          per (set, bin) a warp looks the set's value up and adds the mask to
 *          bit-sliced per-query counters (carry-save adders), so 32 equality
 *          tests cost ~3 lane-instructions; GOPH / HOPH thresholds are applied
 *          to the bit-sliced states level by level (no survivor lists; HOPH:
 *          group 1 bit-sliced, the pairs it leaves undecided walked one by
 *          one over the later groups).
 *          Applies to compare_full, compare_goph (Algorithm 1) and compare_hoph
 *          with the 1:1 split when |V| <= 2^23, at most 1023
 *          bins are compared, (GOPH / HOPH) k' is a multiple of 16 and the
 *          collection's row stride ld is a multiple of 8; needs the workspace of oph_workspace_size_for.
 *          AUTO uses it, for batches of >= 1024 queries, wherever it would
 *          otherwise scan BRUTE (and the workspace is large enough); an explicit BITMAP request outside its
 *          domain fails with OPH_EINVAL (OPH_ENOMEM: workspace too small). */
enum { OPH_STRATEGY_AUTO = 0, OPH_STRATEGY_BRUTE = 1, OPH_STRATEGY_PROBE = 2, OPH_STRATEGY_BITMAP = 3 };

/* One scored pair (20 bytes).
 *   full OPH : n_mb = N_mb, n_excl = excluded bins, over all k bins (Eq. 1-4)
 *   GOPH/HOPH: n_mb, n_excl over the groups compared (R28); groups = groups compared
 *   MinWise  : n_mb = equal positions, n_excl = 0, groups = 0
 *   verdict 1 = Similar; estimate = the estimator's value (Eq. 6 / HOPH
 *   estimator P:484 / MinWise fraction), -1 when absent (flags). */
typedef struct {
    uint32_t query;   /* query index in the query view */
    uint32_t set_id;  /* set_id_base + index in the collection view */
    uint16_t n_mb, n_excl;
    uint8_t groups, verdict, flags, pad;
    float estimate;
} oph_hit;

/* Result sink of compare_*.
 *   OPH_RES_THRESHOLD: every Similar pair is appended (unordered) at
 *     d_hits[atomicAdd(d_count, 1)] if that index < capacity; *d_count keeps
 *     counting past capacity, so after synchronising, *d_count > capacity
 *     means truncation (retry with capacity = *d_count; OPH_EOVERFLOW is the
 *     caller-side status for that case).  *d_count is NOT reset by the call:
 *     several calls may append to one sink.
 *   OPH_RES_DENSE: one record per pair at d_hits[query * n_sets + set]
 *     (capacity >= n_queries * n_sets), for parity tests on small inputs.
 *   d_stop_hist (optional, may be NULL): OPH_STOP_HIST_LEN counters; the call
 *     ADDS, for every (query, set) pair it scores, one to entry g where g is
 *     the pair's `groups` field (groups compared when the pair was decided:
 *     GOPH/HOPH early termination, Alg. 1 l / Alg. 2 l; n for
 *     full OPH; 0 for MinWise), so after a call the entries sum to
 *     n_queries * n_sets more than before -- the termination-level histogram
 *     of SURVEY 8(d) (work saved = bins not compared). */
#define OPH_STOP_HIST_LEN (OPH_MAX_GROUPS + 1)
typedef struct {
    oph_hit *d_hits;
    uint64_t capacity;
    unsigned long long *d_count;
    uint32_t mode;
    uint32_t pad;
    unsigned long long *d_stop_hist;
    /* d_bins_scanned (optional, may be NULL; r02): the call ADDS the number of (set, bin)
     * value rows its pipelined BITMAP scan (full OPH; GOPH's levels 1 .. l0+1) gathered,
     * summed over its query blocks of 2,048 -- that scan's algorithmic work (full OPH in
     * threshold mode stops gathering a set's rows once no pair of the block can reach T even
     * if every remaining non-empty bin matched; R32).  Other scans leave it unchanged. */
    unsigned long long *d_bins_scanned;
} oph_results;

/* ---------------------------------------------------------------- host helpers */

/* Human-readable status. */
const char *oph_status_string(oph_status s);

/* Canonical row stride for n_sets columns (n_sets rounded up to a multiple of 32). */
uint64_t oph_sketch_ld(uint64_t n_sets);

/* HOPH layout (host only): recursive a:b split of the
 * remaining space, front part = floor(a R / (a+b)), until either part would be
 * <= kprime; the remainder is the last group.  EINVAL if vocab_size < 2 kprime,
 * vocab_size > 2^32, a or b is 0, or more than 64 groups result. */
oph_status oph_hier_layout_make(uint64_t vocab_size, uint32_t a, uint32_t b, uint32_t kprime,
                                oph_hier_layout *out);

/* Input contract check (debug aid): offsets non-decreasing with
 * offsets[0] = 0 is NOT required, only offsets[s] <= offsets[s+1]; ids of every
 * set strictly increasing and < vocab_size.  One validation kernel, then a
 * host synchronisation of `stream`.  OPH_OK, OPH_EINVAL (violation or bad
 * arguments), OPH_ECUDA. */
oph_status oph_validate_sets(const oph_sets *sets, uint64_t vocab_size, void *stream);

/* ---------------------------------------------------------------- build (rows a1-a3) */

/* OPH and HOPH sketches of every set from ONE evaluation of psi per element
 * (P:143-160).  Either layout may be NULL (then its outputs are
 * ignored).  Outputs (bin-major, stride ld):
 *   d_oph [flat->k][ld], d_oph_empty [ceil(k/32)][ld],
 *   d_hoph [L*kprime][ld], d_hoph_empty [ceil(L*kprime/32)][ld].
 * EINVAL: vocab_size mismatch between perm and layouts, vocab_size == 0 or
 * > 2^32, k == 0 or k > vocab_size, a bin longer than 2^32 - 2 (the empty
 * sentinels need two spare values), ld < n_sets or ld % 4. */
oph_status oph_build_sketches(const oph_sets *sets, const oph_perm *perm,
                              const oph_flat_layout *flat, uint32_t *d_oph, uint32_t *d_oph_empty,
                              const oph_hier_layout *hier, uint32_t *d_hoph, uint32_t *d_hoph_empty,
                              uint64_t ld, void *stream);

/* MinWise sketches: d_mw[i][s] = min over e in set s of
 * pi_i(e), pi_i = psi keyed by seed_i (R30), i < k; d_set_flags[s] = 1 for an
 * empty set (its column is OPH_EMPTY and it never matches).  EINVAL:
 * vocab_size == 0 or > 2^32, k == 0 or k > 65535. */
oph_status minwise_build_sketches(const oph_sets *sets, uint64_t vocab_size, uint64_t seed, uint32_t k,
                                  uint32_t *d_mw, uint8_t *d_set_flags, uint64_t ld, void *stream);

/* ---------------------------------------------------------------- score (rows a5-a9) */

/* Workspace bytes for compare_* with `method` (OPH_METHOD_*), n_queries
 * queries of n_bins bins, and up to `survivor_capacity` pairs carried
 * between GOPH/HOPH levels (ignored for FULL / MINWISE).  compare_goph/hoph
 * process queries in chunks of floor(survivor_capacity / n_sets) queries
 * (rounded down to a multiple of 32, at least 32), so any capacity >=
 * 32 * n_sets is correct and larger capacities only save launches. */
oph_status oph_workspace_size(uint32_t method, uint64_t n_queries, uint64_t n_sets, uint32_t n_bins,
                              uint64_t survivor_capacity, size_t *bytes);

/* Workspace bytes for a compare_* call on these views and parameters: the
 * bytes of oph_workspace_size plus, when the BITMAP strategy can apply
 * (|V| <= 2^23, n_bins <= 1023, not MinWise), its per-block table (|V| x 4 B)
 * and row masks ((1 + n_bins x 1024) x 128 B).  A workspace of only
 * oph_workspace_size bytes keeps every other strategy. */
oph_status oph_workspace_size_for(uint32_t method, const oph_sketches *queries, const oph_sketches *sets,
                                  const oph_params *params, uint64_t survivor_capacity, size_t *bytes);

/* Full-OPH scoring of every (query, set) pair (Eq. 1-6):
 * N_mb = #bins equal and both non-empty (R5), N_excl per empty_mode (R6),
 * Similar <=> k - N_excl > 0 and N_mb / (k - N_excl) >= T (exactly).  Records
 * carry groups = k / kprime.  Workspace: oph_workspace_size(OPH_METHOD_FULL..). */
oph_status compare_full(const oph_sketches *queries, const oph_sketches *sets, uint32_t set_id_base,
                        const oph_flat_layout *layout, const oph_params *params, oph_results *results,
                        void *d_ws, size_t ws_bytes, void *stream);

/* GOPH scoring (Algorithm 1; R10-R16): per pair, groups
 * l = 1..n of kprime bins; M_c = raw matched bins so far; M_ra =
 * (n k' T - M_c)/(n - l); stop Similar if M_ra <= 0, NotSimilar if M_ra > k',
 * Similar if M_ra < k'T and P(X <= floor(M_ra)) <= eps, NotSimilar if
 * M_ra >= k'T and P(X >= ceil(M_ra)) <= eps, X ~ Bin(k', T); after group n
 * the full-OPH verdict.  Every decision is compiled on the host into exact
 * integer thresholds on M_c.  Needs d_empty on both views. */
oph_status compare_goph(const oph_sketches *queries, const oph_sketches *sets, uint32_t set_id_base,
                        const oph_flat_layout *layout, const oph_params *params, oph_results *results,
                        void *d_ws, size_t ws_bytes, void *stream);

/* HOPH scoring (Algorithm 2, mass balance R19, nominal weights
 * R21): per pair, groups l = 1..L; S_l = sum_{j<=l} c_j M_j (c_j = w_j (a+b)^(L-1));
 * x = P_r k' = (T D k' - S_l) / W_l; the four rules of GOPH on x; after
 * group L the HOPH estimator sum_j w_j M_j/(k' - excl_j) (groups with no
 * usable bin dropped, R22) >= T.  EINVAL if (a+b)^(L-1) k' t_num >= 2^62 or
 * t_den lcm(1..k') (a+b)^(L-1) >= 2^126 (exact 128-bit final verdict; k' <= 64
 * at 1:1 on 2^32). */
oph_status compare_hoph(const oph_sketches *queries, const oph_sketches *sets, uint32_t set_id_base,
                        const oph_hier_layout *layout, const oph_params *params, oph_results *results,
                        void *d_ws, size_t ws_bytes, void *stream);

/* MinWise scoring: N_eq = #{i : mw_q[i] == mw_s[i]}, Similar <=>
 * neither set empty and N_eq / k >= T.  Needs d_flags on both views. */
oph_status compare_minwise(const oph_sketches *queries, const oph_sketches *sets, uint32_t set_id_base,
                           const oph_params *params, oph_results *results, void *d_ws, size_t ws_bytes,
                           void *stream);

/* ---------------------------------------------------------------- select (row a10) */

/* Workspace bytes for topk_or_threshold_results on up to n_in records. */
/* Exact Jaccard of (query, set) pairs -- the quality check of the estimators
 * (Eq. 5: J = |A n B| / |A u B|; SURVEY 8(d) "precision/recall vs exact
 * Jaccard", 8(f) rank 2 "GPU sorted-merge verifier for hits").
 *   For pair i: d_inter[i] = |Q_a n S_b|, d_union[i] = |Q_a u S_b| with
 *   a = d_query[i] (index into `queries`) and b = d_set[i] (local index into
 *   `sets`); J is undefined when d_union[i] == 0 (both sets empty).
 *   Ids of each set strictly increasing (the CSR contract); indices in range
 *   (not checked on the device).  One warp per pair: each lane merges a
 *   contiguous slice of the smaller set against the larger from a binary-
 *   searched start.  Asynchronous on `stream`; caller-owned device buffers.
 *   Errors: OPH_EINVAL for NULL arguments (n_pairs == 0 is a no-op). */
oph_status exact_jaccard_pairs(const oph_sets *queries, const oph_sets *sets, const uint32_t *d_query,
                               const uint32_t *d_set, uint64_t n_pairs, uint32_t *d_inter, uint32_t *d_union,
                               void *stream);

/* Text shingling -- the ingestion step before oph_build_sketches (SPEC
 * shingle_text; "convert the words of each document into a set of
 * fingerprints").  Definition:
 * tokens are maximal runs of non-whitespace bytes (ASCII space, \t, \n, \v,
 * \f, \r) with ASCII letters lowercased; tok = FNV-1a 64 of a token; every w
 * consecutive tokens of a document give h_0 = seed, h_i = mix64(h_{i-1} +
 * 0x9E3779B97F4A7C15 + tok_i) (mix64 = the splitmix64 finalizer, mod 2^64),
 * id = h_w mod vocab_size; a document's set is its distinct ids, sorted (a
 * document with fewer than w tokens gets the empty set).
 *   d_text [n_bytes] bytes, document d = bytes [d_doc_offsets[d],
 *   d_doc_offsets[d+1]) with d_doc_offsets[0] = 0 and d_doc_offsets[n_docs]
 *   = n_bytes (caller-owned device memory).
 *   Output: the CSR collection oph_build_sketches takes: d_set_offsets
 *   [n_docs + 1] and d_ids [ids_capacity]; *d_n_ids receives the total id
 *   count (if it exceeds ids_capacity the ids are truncated; retry).
 *   Workspace: shingle_workspace_size(n_bytes, n_docs).  Asynchronous, no
 *   host synchronisation.  Errors: OPH_EINVAL (w == 0, vocab_size == 0 or >
 *   2^32, NULL pointers, n_bytes + n_docs >= 2^31 - 2: the library's scans and
 *   sorts count items in 32-bit ints), OPH_ENOMEM (workspace too small). */
oph_status shingle_workspace_size(uint64_t n_bytes, uint64_t n_docs, size_t *bytes);
oph_status shingle_text(const uint8_t *d_text, const uint64_t *d_doc_offsets, uint64_t n_docs, uint64_t n_bytes,
                        uint32_t w, uint64_t vocab_size, uint64_t seed, uint64_t *d_set_offsets, uint32_t *d_ids,
                        uint64_t ids_capacity, unsigned long long *d_n_ids, void *d_ws, size_t ws_bytes,
                        void *stream);

oph_status oph_select_workspace_size(uint64_t n_in, size_t *bytes);

/* Result lists.  d_in: n_in records (n_in is a
 * HOST value: the caller reads the compare counter first).
 *   OPH_SELECT_THRESHOLD: d_out = the records sorted by (query, set_id).
 *   OPH_SELECT_TOPK: per query the first `topk` records in the order exact
 *     estimate n_mb / (k_bins - n_excl) descending, ties -> smaller set_id
 *     (R27); records flagged UNDEFINED are dropped.  Meant for full-OPH or
 *     MinWise records; requires k_bins <= 32768.
 * *d_n_out (device) receives the number of records written. */
oph_status topk_or_threshold_results(const oph_hit *d_in, uint64_t n_in, uint32_t mode, uint32_t topk,
                                     uint32_t k_bins, oph_hit *d_out, unsigned long long *d_n_out,
                                     void *d_ws, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------- planner introspection */

/* The per-level integer thresholds the planner compiled for GOPH (method
 * OPH_METHOD_GOPH, nlev = n groups) or HOPH (OPH_METHOD_HOPH, nlev = L groups,
 * ratio a:b): for level l = 1..nlev-1 a pair whose state (GOPH: M_c; HOPH:
 * S_l = sum_{j<=l} c_j M_j) is >= acc[l-1] stops Similar, <= rej[l-1] stops
 * NotSimilar (acc = UINT64_MAX / rej = -1: never).  weights[j] = c_{j+1}
 * (GOPH: 1).  *l0 = the level the collection scan ends at.  Host only; for
 * tests and diagnostics.  acc/rej hold nlev-1 entries, weights nlev.  The
 * planner itself works in 128 bits (HOPH 1:2 on |V| = 2^32: L = 45, weights up
 * to 3^44); a plan with a value that does not fit these 64-bit outputs
 * returns OPH_EOVERFLOW here (compare_hoph runs it regardless). */
oph_status oph_plan_thresholds(uint32_t method, uint32_t nlev, uint32_t kprime, uint32_t a, uint32_t b,
                               uint32_t t_num, uint32_t t_den, double epsilon, uint64_t *acc, int64_t *rej,
                               uint32_t *l0, uint64_t *weights);

#ifdef __cplusplus
}
#endif
#endif /* OPHGPU_H */
