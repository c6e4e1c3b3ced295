/*
 * swsearch.h — C ABI of the B200-native Smith-Waterman protein database search.
 *
 * What is computed (§II.A, Eq. 1): for a query S1 = q[1..m]
 * and every database subject S2 = s[1..n], the optimal local alignment score
 *
 *   H(i,j) = max{ 0, H(i-1,j-1) + fsbt(S1[i],S2[j]), E(i,j), F(i,j) }
 *   E(i,j) = max{ E(i-1,j) - alpha, H(i-1,j) - beta }
 *   F(i,j) = max{ F(i,j-1) - alpha, H(i,j-1) - beta }
 *   H(i,0) = H(0,j) = E(0,j) = F(i,0) = 0,   score = max over H,
 *
 * "alpha is the gap extension penalty, beta is the sum of gap open and
 * extension penalties"; the paper's "10-2k" is alpha=2, beta=12
 * (PAPER.md:164).  Results are exact int32 (32-bit lanes): the
 * device computes in packed int16x2 and reruns in int32 every subject whose
 * 16-bit pass could have saturated (DESIGN.md §"Saturation").
 *
 * The workflow follows the paper's four stages (§III, Fig. 2):
 * sw_db_create = the offline index (subjects sorted by length); sw_search =
 * (i) query profile, (ii) alignment on the device, (iii) wait, (iv) rank all
 * scores in descending order (here: exact top-k, ties by ascending id).
 *
 * Conventions (DESIGN.md §"Readings"):
 *  - residue codes: 0..23 = "ARNDCQEGHILKMFPSTWYVBZX*"; code 24 (DUMMY) is
 *    internal padding scoring 0 against everything.  Inputs with
 *    a code >= 24 are rejected (SW_EINVAL).
 *  - matrix: 32x32 int8, row-major, row = QUERY residue, column = SUBJECT
 *    residue: fsbt(S1[i], S2[j]) = matrix[32*q_i + s_j].  Rows and columns
 *    24..31 must be 0 (SW_EINVAL otherwise).
 *  - 0 <= alpha <= beta <= 32767 (SW_EINVAL otherwise); qlen >= 1;
 *    qlen * max(0, max matrix entry) must be < 2^31 (SW_ERANGE otherwise).
 *  - subject lengths >= 0 (a zero-length subject scores 0).
 *  - top-k order: score descending, then global id ascending; slots past the
 *    number of subjects are (id -1, score -1).
 *
 * Ownership / threading: all input pointers are borrowed for the duration of
 * the call (sw_db_create copies and packs the database into device memory it
 * owns).  Output buffers are caller-owned and left untouched on error.  One
 * handle serialises its searches (internal mutex + stream ordering); distinct
 * handles are independent.  All functions return SW_OK (0) or a negative
 * status; sw_last_error() gives a thread-local message for the last failure.
 */
#ifndef SWSEARCH_H
#define SWSEARCH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SW_OK 0
#define SW_EINVAL (-1)    /* invalid argument (message names the argument/position) */
#define SW_ENOMEM (-2)    /* host or device allocation failed */
#define SW_ECUDA (-3)     /* CUDA runtime error (message carries cudaGetErrorString) */
#define SW_ERANGE (-4)    /* int32 score bound qlen * s_max < 2^31 violated */
#define SW_EINTERNAL (-5) /* internal invariant violated */

#define SW_NUM_CODES 24   /* real residue codes 0..23 */
#define SW_DUMMY 24       /* internal padding code */
#define SW_MATRIX_DIM 32

typedef struct sw_db sw_db; /* opaque; owns its device memory */

/*
 * Measurement / test switches (SURVEY.md §8(f) f4 ablations and tile sweeps).
 * Every field 0 = the production design.  They are read once, at
 * sw_db_create / sw_db_load, never from the environment.  The production
 * library libswsearch.so accepts only the defaults (SW_EINVAL otherwise); the
 * ablation build libswsearch_ablation.so (same source, -DSW_ABLATION) carries
 * the extra kernel instances.  Results never depend on any of them.
 */
typedef struct sw_tuning {
  int32_t variant;        /* 0 production; 1 InterSP score profile, 2 IntraQP striped
                             intra-task kernel, 3 static loop schedule (ablation build) */
  int32_t tile_rows;      /* query rows per register tile of the int16x2 pass: 0 = 48; 32, 64 (ablation build) */
  int32_t threads;        /* threads per persistent CTA: 0 = 384; 512 (ablation build) */
  int32_t intra_cols;     /* columns per intra-task wavefront step: 0 = 4; 2 (ablation build) */
  int32_t max_big;        /* inter-task groups wider than a warp's boundary slab that get a slab of
                             their own: 0 = up to 2,048; > 0 at most this many; -1 none (tests) */
  int32_t align_ws_kb;    /* sw_align direction workspace per batch in KiB: 0 = 1 GiB (tests force batching) */
  int32_t pipeline;       /* 1 = the pipelined first pass k_inter16_pipe: query tiles of a group on
                             consecutive warps, tile-edge rows through shared-memory rings (DRAM traffic
                             of the first pass ~50x lower, measured ~11% slower) instead
                             of per-warp global slabs (k_inter16, default) */
  int32_t pipe_chain;     /* warps per pipeline chain: 0 = 3 (one SM sub-partition); 1, 6 or 12
                             (ablation build) */
  int32_t intra_isolate;  /* intra-task kernel: 1 = the warps holding the longest pairs get their SM
                             sub-partition alone, -1 = never, 0 = when the longest pair is the critical
                             path (small databases such as C1) */
  int32_t generic_gaps;   /* 1 = the int16x2 first-pass kernels (inter-task, intra-task wavefront,
                             paired queries) keep alpha, beta in registers even for the paper's 10-2k
                             penalties (alpha 2, beta 12), which otherwise run instances with them as
                             immediates (3.5 % / ~5 % faster; identical results) */
  int32_t intra_chain;    /* intra-task kernel, single-pass queries (m <= 32 x rows per lane): 0 = the
                             pair items of a warp run as one chained stream through the lanes (no fill
                             and drain per item), -1 = one wavefront per item (measurement) */
  int32_t intra_split;    /* with intra_isolate in effect and a single-pass query: 0 = the longest pair of
                             each isolated sub-partition (>= 1,024 columns) is cut into two column segments,
                             the second run speculatively by a second warp and repaired at its start;
                             -1 = one warp per pair (measurement) */
  int32_t launch_chain;   /* resident databases: 0 = launch latency hidden behind the kernel before --
                             up to 262,144 subjects the profile kernel also zeroes the saturation flags
                             and the intra-task pass is launched as its programmatic dependent; up to
                             65,536 the one-CTA flag compaction, the int32 rerun and the one-CTA ranking
                             each follow the kernel before them the same way; -1 = plain stream-ordered
                             launches (measurement).  Results never depend on it. */
} sw_tuning;

typedef struct sw_opts {
  int32_t device;         /* CUDA device ordinal; -1 = the caller's current device */
  int32_t first_stage;    /* lane width of the first pass: 8, 16 (default) or 32 */
  int32_t long_threshold; /* 64-subject groups wider than this many columns are aligned pair
                             by pair by the intra-task wavefront kernel; 0 = library default
                             (max(64, ~one warp's share of the residues)), -1 = none (all
                             inter-task; groups wider than a warp's boundary slab then get
                             slabs of their own, up to 2,048 groups / 8 GiB, the rest stay
                             intra-task).  Results never depend on it. */
  int32_t verbose;        /* 0 = silent */
  int32_t residency;      /* 0 = packed database resident in device memory (default);
                             1 = kept in pinned host memory and streamed to the device
                             in chunks during every search (f2: databases larger than
                             HBM; first_stage 16 or 32; not with sw_search_batch) */
  int32_t chunk_mb;       /* residency 1: device bytes per streamed chunk in MiB
                             (two are allocated); 0 = 512 */
  int32_t max_qlen;       /* per-search device buffers are allocated at create time for
                             queries up to this length: 0 = 8192 (see sw_db_reserve) */
  int32_t max_k;          /* ... and top-k up to this k: 0 = 4096 */
  /* Device-memory hooks, e.g. torch's caching allocator.
   * alloc(bytes, ctx) returns device memory on `device` (NULL = failure ->
   * SW_ENOMEM); free(ptr, ctx) releases it.  Both NULL = cudaMalloc / cudaFree.
   * Every device buffer of the handle comes from them; none is allocated by
   * sw_search_async (buffers are sized at create time / by sw_db_reserve). */
  void* (*alloc)(size_t bytes, void* ctx);
  void (*free)(void* ptr, void* ctx);
  void* alloc_ctx;
  sw_tuning tuning;       /* measurement switches; zero = production */
  int32_t reserved[4];    /* must be 0 */
} sw_opts;

typedef struct sw_stats {
  int64_t cells;          /* qlen * sum of real subject lengths (GCUPS numerator) */
  int64_t n_seqs;         /* subjects searched */
  int64_t n_inter;        /* subjects aligned by the inter-task kernels */
  int64_t n_intra;        /* subjects aligned by the intra-task kernel */
  int64_t n_rerun16;      /* subjects re-aligned at int16 after an int8 first pass */
  int64_t n_rerun32;      /* subjects re-aligned at int32 after saturating at int16 */
  double seconds;         /* wall time of the search call */
  double gcups;           /* cells / seconds / 1e9 */
  float ms_profile, ms_inter, ms_rerun, ms_finalize; /* device times per stage (sw_search only) */
  int32_t first_stage;    /* lane width actually used first */
  int32_t reserved[7];
} sw_stats;

typedef struct sw_db_info {
  int64_t n_seqs, n_residues;   /* real subjects / residues */
  int64_t n_inter, n_intra;     /* split at long_threshold */
  int64_t n_groups;             /* 64-subject interleaved groups of the inter-task layout */
  int64_t packed_bytes;         /* device bytes of packed residues */
  int64_t scratch_bytes;        /* device bytes of DP boundary scratch */
  int64_t launches;             /* CUDA kernels launched by this handle so far */
  int64_t n_searches;           /* searches enqueued so far */
  int64_t n_device_allocs;      /* device allocations made by this handle so far (alloc hook or cudaMalloc) */
  int64_t device_bytes;         /* device bytes currently held by this handle */
  int32_t max_len;              /* longest subject */
  int32_t device;
  int32_t long_threshold;
  int32_t residency;            /* as sw_opts.residency */
  int32_t n_chunks;             /* residency 1: chunks streamed per search */
  int32_t max_qlen, max_k;      /* per-search buffer capacity (sw_opts.max_qlen / max_k, sw_db_reserve) */
  int32_t reserved[1];
} sw_db_info;

/* Fill *opts with defaults (device -1, first_stage 16, long_threshold 0, residency 0,
 * max_qlen 8192, max_k 4096, no allocator hooks, production tuning). */
void sw_opts_default(sw_opts* opts);

/*
 * Build a searchable database (the paper's offline index, and
 * sequence profiles): stable sort by (length, input index),
 * split at long_threshold, pack residues as 5-bit codes (6 per 32-bit word)
 * interleaved over 64-subject groups, upload to the device.
 *   residues   host, n_residues bytes, codes 0..23
 *   offsets    host, n_seqs int64: subject i = residues[offsets[i] .. +lengths[i])
 *   lengths    host, n_seqs int32 >= 0
 *   global_ids host, n_seqs DISTINCT int64 in [0, 2^32-2], or NULL (= 0..n_seqs-1);
 *              used only for top-k ids and the tie-break (a repeated id -> SW_EINVAL)
 *   opts       NULL = defaults
 *   out        receives the handle (NULL on error)
 */
int sw_db_create(const uint8_t* residues, int64_t n_residues, const int64_t* offsets,
                 const int32_t* lengths, int64_t n_seqs, const int64_t* global_ids,
                 const sw_opts* opts, sw_db** out);

/*
 * Persistent packed index (the paper builds "index files"
 * offline that "can be mapped into virtual memory").
 * sw_db_save writes the packed, length-sorted layout (group table, permutation,
 * sorted lengths, global ids, 5-bit words) to `path`; sw_db_load mmaps such a
 * file and uploads it without re-sorting or re-packing.  A truncated, corrupt
 * or foreign file is rejected with SW_EINVAL before any device work.  Searches
 * on a loaded handle are identical to searches on the handle that was saved.
 */
int sw_db_save(sw_db* db, const char* path);
int sw_db_load(const char* path, const sw_opts* opts, sw_db** out);

/*
 * Search one query against every subject; blocks until results are on the host.
 *   query        host, qlen codes 0..23
 *   matrix       host, 32*32 int8 (row = query residue)
 *   k            >= 1
 *   scores       host int32[n_seqs] in input order, or NULL
 *   topk_ids     host int64[k] (global ids), or NULL
 *   topk_scores  host int32[k], or NULL
 *   stats        or NULL
 */
int sw_search(sw_db* db, const uint8_t* query, int32_t qlen, const int8_t* matrix,
              int32_t alpha, int32_t beta, int32_t k, int32_t* scores, int64_t* topk_ids,
              int32_t* topk_scores, sw_stats* stats);

/*
 * As sw_search, but enqueued on `stream` (a cudaStream_t; NULL = legacy default
 * stream) with DEVICE outputs and no host synchronisation.  query/matrix are
 * host pointers, staged by the library.  d_scores int32[n_seqs] (input order),
 * d_topk_ids int64[k], d_topk_scores int32[k]; any may be NULL.
 * Never allocates and never blocks the host (except to recycle one of its
 * eight pinned staging slots when eight searches are still in flight): qlen
 * and k must fit the handle's capacity (sw_opts.max_qlen / max_k or
 * sw_db_reserve), else SW_EINVAL before any device work.  Searches on one
 * handle run in call order whatever streams they are enqueued on.
 */
int sw_search_async(sw_db* db, const uint8_t* query, int32_t qlen, const int8_t* matrix,
                    int32_t alpha, int32_t beta, int32_t k, int32_t* d_scores,
                    int64_t* d_topk_ids, int32_t* d_topk_scores, void* stream);

/*
 * Batched search (the paper's protocol searches 20
 * queries against one database): every query against every
 * subject, results identical to n_queries calls of sw_search.  Queries are
 * paired by length; a pair is aligned in ONE pass with the two queries in the
 * lo/hi halves of int16x2 (the substitution pair is then one word of a pair
 * profile), each query's saturated subjects are rerun in int32.  Pairs whose
 * pair profile would not fit shared memory (longer query > ~2000) and an odd
 * last query run as single searches.  Blocking; host buffers.
 *   queries    host, concatenated codes 0..23; query q = queries[qoffsets[q] .. +qlens[q])
 *   scores     host int32[n_queries][n_seqs] (query-major, input order) or NULL
 *   topk_ids / topk_scores  host [n_queries][k] or NULL
 *   stats      aggregate (cells over all queries; reserved[0] = pairs aligned jointly)
 */
int sw_search_batch(sw_db* db, const uint8_t* queries, const int64_t* qoffsets, const int32_t* qlens,
                    int32_t n_queries, const int8_t* matrix, int32_t alpha, int32_t beta, int32_t k,
                    int32_t* scores, int64_t* topk_ids, int32_t* topk_scores, sw_stats* stats);

/*
 * Traceback of optimal local alignments for chosen subjects (SURVEY.md §8(f)
 * f3; "alignment retrieval" is the paper's future work).  For
 * each subject the device fills Eq. 1 over the whole query x subject matrix in
 * int32 with a 4-bit direction code per cell, then walks back from the end
 * cell.  Deterministic choices (R17-R19): the end cell is the
 * maximal H with the smallest subject position, then the smallest query
 * position; on the walk H prefers diagonal, then E, then F; a gap extends only
 * if that is strictly better than opening.  score equals sw_search's score.
 *   query/matrix/alpha/beta  as sw_search
 *   subjects     host int64[n]: INPUT indices (0 .. n_seqs-1), repeats allowed
 *   out          host sw_alignment[n]
 *   ops          host buffer; alignment t's ops start at out[t].ops_offset and
 *                are out[t].n_ops bytes of 'M' (query residue vs subject residue),
 *                'I' (query residue vs gap) and 'D' (subject residue vs gap),
 *                in alignment order (SAM convention, the query as the read)
 *   ops_cap      bytes of ops; must be >= sum over t of (qlen + length of
 *                subject t), else SW_EINVAL (the message states the need)
 * Coordinates are 0-based and half-open; a score-0 alignment is empty (all 0).
 * Device workspace: qlen/2 bytes per cell of the matrices aligned at once,
 * batched under ~1 GiB (a single larger matrix is allocated alone).
 * Blocking; host buffers.
 */
typedef struct sw_alignment {
  int64_t subject;        /* input index */
  int32_t score;
  int32_t q_begin, q_end; /* query residues [q_begin, q_end) */
  int32_t s_begin, s_end; /* subject residues [s_begin, s_end) */
  int32_t n_ops;
  int32_t reserved;
  int64_t ops_offset;
} sw_alignment;

int sw_align(sw_db* db, const uint8_t* query, int32_t qlen, const int8_t* matrix, int32_t alpha,
             int32_t beta, const int64_t* subjects, int32_t n, sw_alignment* out, char* ops, int64_t ops_cap);

/*
 * Letters -> residue codes (host helper): the 24-letter table
 * "ARNDCQEGHILKMFPSTWYVBZX*" -> 0..23, case-insensitive; letters outside it
 * (J, O, U) -> 22 ('X').  Any other byte -> SW_EINVAL naming its position;
 * `out` (n bytes) is left untouched on error.
 */
int sw_encode(const char* text, int64_t n, uint8_t* out);

/*
 * Merge n_lists top-k lists (host; e.g. one per GPU after an all-gather) into
 * the global top-k by (score desc, id asc).  Entries with id < 0 are ignored.
 *   ids/scores   host, n_lists * k_in entries (list-major)
 *   out_ids/out_scores  host, k_out entries; padded with (-1, -1)
 */
int sw_merge_topk(const int64_t* ids, const int32_t* scores, int32_t n_lists, int32_t k_in,
                  int32_t k_out, int64_t* out_ids, int32_t* out_scores);

/*
 * Grow the per-search device buffers for queries up to max_qlen residues and
 * top-k up to max_k (never shrinks; blocks until the handle is idle).  The
 * blocking calls (sw_search, sw_search_batch, sw_align) grow them on demand;
 * sw_search_async needs them sized beforehand.
 */
int sw_db_reserve(sw_db* db, int32_t max_qlen, int32_t max_k);

int sw_db_get_info(const sw_db* db, sw_db_info* info);

/*
 * Device time (ms, CUDA events on the search's stream) of the four stages of
 * the search enqueued `back` calls ago (1 = the latest; at most 64 back):
 * ms[0] query profile, ms[1] first (int16x2 or int32) pass, ms[2] int32 rerun
 * of saturated subjects, ms[3] scatter + top-k.  Waits for that search.
 */
int sw_db_stage_times(sw_db* db, int32_t back, float* ms);

/* Release the handle and its device memory; NULL is a no-op. */
void sw_db_destroy(sw_db* db);

const char* sw_strerror(int status);
const char* sw_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* SWSEARCH_H */
