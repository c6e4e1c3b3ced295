// sw_api.cu — host side of the C ABI declared in include/swsearch.h.
//
// sw_db_create is the paper's offline indexing ("All subject
// sequences are sorted in ascending order of sequence length") plus its
// sequence-profile layout (consecutive sorted subjects
// interleaved, padded with a dummy residue scoring 0).  sw_search runs the
// four-stage workflow of PAPER.md:55 (Fig. 2) on one B200:
//   (i) query profile -> (ii) inter-task alignment (int16x2 DPX, int32 rerun of
//   flagged subjects) -> (iii) stream-ordered completion -> (iv) ranking
//   (exact top-k by radix select).
//
// One translation unit: this file holds the shared helpers and struct sw_db,
// then includes the ABI in parts -- sw_db.inc (create / save / load / info),
// sw_search.inc (sw_search, sw_search_async, streamed databases),
// sw_batch.inc (f1), sw_align_host.inc (f3) -- and ends with sw_merge_topk.
// Device code (overview in sw_common.cuh; search: sw_common / sw_int16 / sw_pipe / sw_int8 / sw_int32
// / sw_multi / sw_escalate / sw_rank .cuh), sw_align.cuh (f3), sw_ablation.cuh (f4).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <atomic>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <nvtx3/nvToolsExt.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include "../../include/swsearch.h"
#include "sw_common.cuh"
#include "sw_int16.cuh"
#include "sw_pipe.cuh"
#include "sw_int8.cuh"
#include "sw_int32.cuh"
#include "sw_multi.cuh"
#include "sw_escalate.cuh"
#include "sw_rank.cuh"
#include "sw_align.cuh"
#ifdef SW_ABLATION
#include "sw_ablation.cuh"   // f4 kernels: only in the ablation build (libswsearch_ablation.so)
#endif

using swk::GroupDesc;

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

// On a CUDA error: report it and clear the runtime's last-error slot, so a
// non-sticky error (e.g. an invalid launch) is not reported again by the next,
// unrelated cudaGetLastError() of a later call.
#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t _e = (call);                                                              \
    if (_e != cudaSuccess) {                                                              \
      cudaGetLastError();                                                                 \
      return fail(_e == cudaErrorMemoryAllocation ? SW_ENOMEM : SW_ECUDA, "%s: %s (%s:%d)", \
                  #call, cudaGetErrorString(_e), __FILE__, __LINE__);                     \
    }                                                                                     \
  } while (0)

constexpr int kStreamPieces = 16;   // pieces of a streamed search's first chunk
constexpr int kTileRows = 48;        // query rows per register tile (sw_tuning.tile_rows: 32/64 in the ablation build)

#ifdef SW_ABLATION
constexpr bool kAblationBuild = true;
#else
constexpr bool kAblationBuild = false;
#endif

// NVTX range for the host side of a stage (enqueue / wait); header-only nvtx3.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-(device, kernel)
// attribute shared by every handle in the process.  It is only ever RAISED,
// under a process-wide lock, so a concurrent launch on another handle never
// sees it drop below what that launch was set up for.
int raise_smem_limit(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<int, const void*>, size_t>> set;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(SW_ECUDA, "cudaGetDevice failed");
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : set)
    if (e.first.first == dev && e.first.second == fn) {
      if (e.second >= bytes) return SW_OK;
      cudaError_t r = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
      if (r != cudaSuccess) {
        cudaGetLastError();
        return fail(SW_ECUDA, "cudaFuncSetAttribute(%zu B): %s", bytes, cudaGetErrorString(r));
      }
      e.second = bytes;
      return SW_OK;
    }
  cudaError_t r = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(bytes, 1));
  if (r != cudaSuccess) {
    cudaGetLastError();
    return fail(SW_ECUDA, "cudaFuncSetAttribute(%zu B): %s", bytes, cudaGetErrorString(r));
  }
  set.push_back({{dev, fn}, bytes});
  return SW_OK;
}
#define CK_SMEM(fn, bytes)                                      \
  do {                                                          \
    int _rc = raise_smem_limit((const void*)(fn), (bytes));     \
    if (_rc != SW_OK) return _rc;                               \
  } while (0)

template <int T, int NT>
void* inter16_kernel(bool smem, bool big) {
  if (big) return smem ? (void*)swk::k_inter16<T, true, NT, true> : (void*)swk::k_inter16<T, false, NT, true>;
  return smem ? (void*)swk::k_inter16<T, true, NT> : (void*)swk::k_inter16<T, false, NT>;
}
// The shipped shape with the paper's gap penalties as immediates (swk::kFixedAlpha/kFixedBeta;
// profile in shared memory, i.e. m up to ~8,000): sw_common.cuh.
inline void* inter16_kernel_fixed_gaps(bool big) {
  return big ? (void*)swk::k_inter16<kTileRows, true, swk::kInterThreads, true, false, 1>
             : (void*)swk::k_inter16<kTileRows, true, swk::kInterThreads, false, false, 1>;
}
#ifdef SW_ABLATION
// f4 ablation (sw_tuning.variant 3): the paper's static loop schedule instead of the work queue
inline void* inter16_kernel_static(bool smem, bool big) {
  if (big) return smem ? (void*)swk::k_inter16<48, true, 384, true, true> : (void*)swk::k_inter16<48, false, 384, true, true>;
  return smem ? (void*)swk::k_inter16<48, true, 384, false, true> : (void*)swk::k_inter16<48, false, 384, false, true>;
}
#endif

// The int16x2 first-pass instance for a tile height / CTA size (only 48 / 384
// in the production build; sw_db_create rejects the others there).
inline void* inter16_select(int T, int nt, bool smem, bool big, bool static_schedule, bool fixed_gaps) {
  if (fixed_gaps && smem && T == kTileRows && nt == swk::kInterThreads && !static_schedule)
    return inter16_kernel_fixed_gaps(big);
#ifdef SW_ABLATION
  if (static_schedule) return inter16_kernel_static(smem, big);
  if (T == 32) return nt == 512 ? inter16_kernel<32, 512>(smem, big) : inter16_kernel<32, 384>(smem, big);
  if (T == 64) return nt == 512 ? inter16_kernel<64, 512>(smem, big) : inter16_kernel<64, 384>(smem, big);
  if (nt == 512) return inter16_kernel<48, 512>(smem, big);
#else
  (void)T;
  (void)nt;
  (void)static_schedule;
#endif
  return inter16_kernel<48, 384>(smem, big);
}
constexpr int kMaxSmemProfile = 200 * 1024;
constexpr int64_t kFlagZeroInProfiles = 1 << 18;   // databases up to this many subjects: flags zeroed by k_profiles
constexpr size_t kSmemOptin = 227 * 1024 - 4096;  // B200 shared memory per block minus the kernels' static smem

// Ring slots per link of the pipelined first pass for a profile of prof_bytes
// (8, or 4 / 2 for long queries: the more slack between the warps the better), 0 if the profile and the rings do not fit shared
// memory (the slab kernel k_inter16 then runs).
// The pipelined first-pass instance: NS ring slots, CL warps per chain.
template <int CL>
void* pipe_kernel_ns(int ns) {
  if (ns == 8) return (void*)swk::k_inter16_pipe<kTileRows, true, swk::kInterThreads, 8, CL>;
  if (ns == 4) return (void*)swk::k_inter16_pipe<kTileRows, true, swk::kInterThreads, 4, CL>;
  return (void*)swk::k_inter16_pipe<kTileRows, true, swk::kInterThreads, 2, CL>;
}
inline void* pipe_kernel(int ns, int chain) {
#ifdef SW_ABLATION
  if (chain == 1) return pipe_kernel_ns<1>(ns);
  if (chain == 6) return pipe_kernel_ns<6>(ns);
  if (chain == 12) return pipe_kernel_ns<12>(ns);
#else
  (void)chain;
#endif
  return pipe_kernel_ns<3>(ns);
}

inline int pipe_chains(int chain) { return (swk::kInterThreads / 32) / (chain ? chain : 3); }
inline int pipe_slots_for(size_t prof_bytes, int chain = 0) {
  for (int ns : {8, 4, 2})
    if (prof_bytes + swk::pipe_ring_bytes(swk::kInterThreads / 32, ns, pipe_chains(chain)) <= kSmemOptin) return ns;
  return 0;
}

// Shape of the intra-task wavefront's blocked profile: TR rows per lane, the
// fewest that put the query in one 32-lane pass (TR in {4, 6, 8, 12, 16}; longer
// queries take several passes of 16 rows per lane), so few lanes idle.
// (TR in {4, 5, 6, 7, 8, 10, 12, 14, 16}.)
struct IntraShape {
  int tr, nblk, rowstride;
  size_t bytes;
  bool smem;
};
IntraShape intra_shape(int m_pad) {
  const int need = (m_pad + 31) / 32;
  IntraShape sh;
  sh.tr = need <= 4 ? 4 : need <= 8 ? need : need <= 10 ? 10 : need <= 12 ? 12 : need <= 14 ? 14 : 16;
  // Row stride padded to 128 B: lane l reads block l of the row of ITS column's
  // residue, so with a 128-B multiple each quarter-warp of an LDS.128 hits 8
  // distinct 16-B bank groups whatever the residues (m = 144: 464 -> 512 B,
  // 37.8k bank conflicts per 3,303-column pair before, ncu r02_ncu_intra_pair).
  sh.nblk = ((m_pad + sh.tr - 1) / sh.tr + 7) & ~7;
  sh.rowstride = sh.nblk * 16;
  sh.bytes = (size_t)swk::kProfRows * sh.rowstride;
  sh.smem = sh.bytes <= (size_t)kMaxSmemProfile;
  return sh;
}
template <int NC>
void* intra_kernel_nc(const IntraShape& sh) {
  static_assert(NC == 2 || NC == 4 || NC == 8, "columns per step");
  switch (sh.tr) {
    case 4: return sh.smem ? (void*)swk::k_intra16<4, true, NC> : (void*)swk::k_intra16<4, false, NC>;
    case 5: return sh.smem ? (void*)swk::k_intra16<5, true, NC> : (void*)swk::k_intra16<5, false, NC>;
    case 6: return sh.smem ? (void*)swk::k_intra16<6, true, NC> : (void*)swk::k_intra16<6, false, NC>;
    case 7: return sh.smem ? (void*)swk::k_intra16<7, true, NC> : (void*)swk::k_intra16<7, false, NC>;
    case 8: return sh.smem ? (void*)swk::k_intra16<8, true, NC> : (void*)swk::k_intra16<8, false, NC>;
    case 10: return sh.smem ? (void*)swk::k_intra16<10, true, NC> : (void*)swk::k_intra16<10, false, NC>;
    case 12: return sh.smem ? (void*)swk::k_intra16<12, true, NC> : (void*)swk::k_intra16<12, false, NC>;
    case 14: return sh.smem ? (void*)swk::k_intra16<14, true, NC> : (void*)swk::k_intra16<14, false, NC>;
    default: return sh.smem ? (void*)swk::k_intra16<16, true, NC> : (void*)swk::k_intra16<16, false, NC>;
  }
}
// The production shape (4 columns per step, profile in shared memory) with the
// paper's gap penalties as immediates (sw_common.cuh, kFixedAlpha/kFixedBeta).
void* intra_kernel_fixed_gaps(int tr) {
  switch (tr) {
    case 4: return (void*)swk::k_intra16<4, true, 4, 1>;
    case 5: return (void*)swk::k_intra16<5, true, 4, 1>;
    case 6: return (void*)swk::k_intra16<6, true, 4, 1>;
    case 7: return (void*)swk::k_intra16<7, true, 4, 1>;
    case 8: return (void*)swk::k_intra16<8, true, 4, 1>;
    case 10: return (void*)swk::k_intra16<10, true, 4, 1>;
    case 12: return (void*)swk::k_intra16<12, true, 4, 1>;
    case 14: return (void*)swk::k_intra16<14, true, 4, 1>;
    default: return (void*)swk::k_intra16<16, true, 4, 1>;
  }
}
// intra_cols: columns per wavefront step (4 = production; 2 = the previous
// design, ablation build only)
void* intra_kernel(const IntraShape& sh, int intra_cols, bool fixed_gaps) {
  if (fixed_gaps && sh.smem && (intra_cols == 0 || intra_cols == 4)) return intra_kernel_fixed_gaps(sh.tr);
#ifdef SW_ABLATION
  if (intra_cols == 2) return intra_kernel_nc<2>(sh);
#endif
  if (intra_cols == 8) return intra_kernel_nc<8>(sh);
  return intra_kernel_nc<4>(sh);
}

int host_threads() {
  unsigned n = std::thread::hardware_concurrency();
  return (int)std::max(1u, std::min(n, 64u));
}

template <class F>
void parallel_for(int64_t n, F f) {
  int nt = host_threads();
  if (n < 4096 || nt == 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < nt; t++) {
    int64_t a = n * t / nt, b = n * (t + 1) / nt;
    th.emplace_back([=] { f(a, b); });
  }
  for (auto& x : th) x.join();
}

}  // namespace

struct sw_db {
  int device = 0;
  int num_sms = 0;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  int first_stage = 16;
  int long_threshold = -1;
  sw_tuning tuning = {};          // measurement switches, fixed at create / load

  // device memory: the caller's hooks (sw_opts.alloc / free) or cudaMalloc / cudaFree
  void* (*alloc_fn)(size_t, void*) = nullptr;
  void (*free_fn)(void*, void*) = nullptr;
  void* alloc_ctx = nullptr;
  int64_t n_device_allocs = 0, device_bytes = 0;
  std::vector<std::pair<void*, size_t>> live;   // every live device buffer (size for the byte count)

  // capacity of the per-search buffers (sw_opts.max_qlen / max_k, sw_db_reserve)
  int cap_qlen = 0, cap_k = 0;
  // inter/intra split and wide-group slabs: a property of the layout, planned at create
  int split_cut = 0;              // groups with ncols > split_cut go intra-task (pair by pair), slab kernel
  int lb_cut = 0;                 // the same split for the pipelined first pass (load balance only)
  int n_big = 0;                  // inter-task groups wider than a warp slab with a slab of their own
  long long big_cols = 0;         // columns per big slab

  int64_t n_seqs = 0, n_residues = 0, n_inter = 0, n_intra = 0, sum_len = 0;
  int32_t max_len = 0, max_inter_len = 0;
  int64_t n_groups = 0, n_words = 0;
  std::vector<int> group_ncols;   // host copy (ascending): picks the intra-task groups per search

  // f2 host residency: packed words in pinned (mapped) host memory, streamed per search
  bool host_resident = false;
  uint2* h_words = nullptr;
  std::vector<int64_t> h_group_base;                 // n_groups + 1 word offsets
  std::vector<std::pair<int64_t, int64_t>> chunks;   // [g0, g1) per streamed chunk
  int64_t chunk_words = 0;
  uint2* d_chunk[2] = {nullptr, nullptr};
  int* d_stream_cnt = nullptr;                       // int32 reruns per chunk
  long long* h_ready_vals = nullptr;                 // pinned: LLONG_MAX, then each first-chunk piece's start word
  long long* d_ready_from = nullptr;                 // lowest word of the first chunk known to have landed
  std::vector<int64_t> piece_first;                  // first group of each first-chunk piece (descending)
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_consumed[2] = {nullptr, nullptr};

  uint2* d_words = nullptr;
  GroupDesc* d_groups = nullptr;
  int* d_perm = nullptr;          // sorted position -> input index
  int* d_len_sorted = nullptr;    // sorted position -> length
  long long* d_gid = nullptr;     // input index -> global id (nullptr: identity)
  int* d_inv = nullptr;           // input index -> sorted position (built on the first sw_align)
  uint2* d_big = nullptr;         // boundary slabs of the inter-task groups wider than a warp's slab
  size_t big_cap = 0;
  uint2* d_pipe_slab = nullptr;   // k_inter16_pipe: per CTA two round-crossing tile-edge slabs
  long long pipe_slab_cols = 0;
  int8_t* d_profb = nullptr;      // blocked profile of the intra-task wavefront (and f1's second query)
  int8_t* d_profb2 = nullptr;
  size_t profb_cap = 0, profb2_cap = 0;
  int8_t* d_prof_qp = nullptr;    // f4 IntraQP ablation: profile with rows of 32*L bytes
  size_t prof_qp_cap = 0;
  void* aw[10] = {};              // sw_align workspace (grow-only): idx, jobs, res, q, M, prof, dir, bnd, ops, tmp
  size_t aw_cap[10] = {};

  uint2* d_scratch = nullptr;     // DP boundary rows, one slab per resident warp (inter-task kernels)
  uint2* d_scratch_intra = nullptr; // pass boundaries of the intra-task kernel (runs concurrently: own slabs)
  uint2* d_scratch_intra2 = nullptr; // f1: the second query's intra-task pass (allocated on first use)
  long long scratch_cols_intra = 0;
  long long scratch_cols = 0;
  int scratch_slots = 0;

  // per-search buffers
  uint8_t* d_query = nullptr;
  size_t query_cap = 0;
  uint8_t* d_qm = nullptr;      // sw_search's matrix (1,024 B) and query behind it: one H2D copy per search
  size_t qm_cap = 0;
  int8_t* d_matrix = nullptr;
  int8_t* d_prof = nullptr;
  size_t prof_cap = 0;
  int* d_score_sorted = nullptr;
  int* d_scores = nullptr;        // input-order scores for the synchronous API
  unsigned long long* d_keys = nullptr;
  unsigned long long* d_cand = nullptr;
  unsigned long long* d_cand2 = nullptr;
  size_t cand_cap = 0, cand2_cap = 0;   // bytes
  uint8_t* d_flag8 = nullptr;     // per sorted position: saturated in the int8 pass
  uint8_t* d_flag16 = nullptr;    // per sorted position: saturated in the int16 pass
  int* d_list8 = nullptr;         // ascending flagged positions (int8 -> int16)
  int* d_list16 = nullptr;        // ascending flagged positions (int16 -> int32)
  int* d_block_counts = nullptr;  // compaction scratch
  int* d_cnt = nullptr;           // [0] #flagged int8, [1] #flagged int16, [2] #mini-groups
  int64_t n_mini_max = 0;
  int* d_mini_sizes = nullptr;    // words per mini-group -> exclusive scan = bases
  GroupDesc* d_mgroups = nullptr; // mini-group layout of the int8-flagged subjects
  uint2* d_mwords = nullptr;
  uint8_t* d_prof8b = nullptr;    // biased uint8 profile of the int8 stage
  size_t prof8b_cap = 0;
  // f1 batched queries: second query's int8 profile, pair profile, its scores and flags
  int8_t* d_prof_b = nullptr;
  size_t prof_b_cap = 0;
  uint32_t* d_prof2 = nullptr;
  size_t prof2_cap = 0;
  int* d_score_sorted2 = nullptr;
  uint8_t* d_flag_b = nullptr;
  int* d_counters = nullptr;      // work counters: [0] first pass, [2] int32 list, [3] cand count, [4] int16 rerun
  unsigned* d_hist = nullptr;
  swk::SelState* d_sel = nullptr;
  long long* d_topk_ids = nullptr;
  int* d_topk_scores = nullptr;
  size_t topk_cap = 0;
  void* d_cub = nullptr;
  size_t cub_bytes = 0;

  // pinned staging for query + matrix: a ring of slots, each recycled only
  // after its H2D copy has drained (the async path never waits on a search)
  static constexpr int kStage = 8;
  uint8_t* h_stage[kStage] = {};
  cudaEvent_t ev_stage[kStage] = {};
  size_t stage_cap = 0;
  int stage_next = 0;
  cudaEvent_t ev_done = nullptr;
  // stage-boundary events of the last kRing searches (sync and async):
  // [0] start, [1] profile done, [2] first pass done, [3] rerun done, [4] ranking done
  static constexpr int kRing = 64;
  cudaEvent_t ev_ring[kRing][5] = {};
  int64_t n_searches = 0;
  int64_t launches = 0;           // kernels launched by this handle (all searches)
  int last_n_long = 0;            // groups aligned pair-wise by the intra-task path in the last search
  int last_first_stage = 16;      // lane width of the last search's first pass
};

// ---- device memory of a handle: the caller's hooks or cudaMalloc ----
int dalloc(sw_db* db, void** p, size_t bytes) {
  *p = nullptr;
  bytes = std::max<size_t>(bytes, 16);
  if (db->alloc_fn) {
    *p = db->alloc_fn(bytes, db->alloc_ctx);
    if (!*p) return fail(SW_ENOMEM, "device allocation hook returned NULL for %zu bytes", bytes);
  } else {
    cudaError_t e = cudaMalloc(p, bytes);
    if (e != cudaSuccess) {
      *p = nullptr;
      return fail(e == cudaErrorMemoryAllocation ? SW_ENOMEM : SW_ECUDA, "cudaMalloc(%zu): %s", bytes,
                  cudaGetErrorString(e));
    }
  }
  db->n_device_allocs++;
  db->device_bytes += (int64_t)bytes;
  db->live.emplace_back(*p, bytes);
  return SW_OK;
}
template <class T>
int dalloc_t(sw_db* db, T** p, size_t bytes) {
  void* v = nullptr;
  const int rc = dalloc(db, &v, bytes);
  *p = (T*)v;
  return rc;
}
void dfree(sw_db* db, void* p) {
  if (!p) return;
  for (size_t t = 0; t < db->live.size(); t++)
    if (db->live[t].first == p) {
      db->device_bytes -= (int64_t)db->live[t].second;
      db->live[t] = db->live.back();
      db->live.pop_back();
      break;
    }
  if (db->free_fn) db->free_fn(p, db->alloc_ctx);
  else cudaFree(p);
}
// grow-only buffer (blocking paths only: the caller has made the handle idle).
// The new buffer is allocated before the old one is released, so a failed grow
// (SW_ENOMEM) leaves the handle as it was.
template <class T>
int grow(sw_db* db, T** p, size_t* cap, size_t need) {
  if (*p && *cap >= need) return SW_OK;
  T* fresh = nullptr;
  const int rc = dalloc_t(db, &fresh, need);
  if (rc != SW_OK) return rc;
  dfree(db, *p);
  *p = fresh;
  *cap = std::max<size_t>(need, 16);
  return SW_OK;
}
#define CK_RC(expr)                 \
  do {                              \
    const int _rc = (expr);         \
    if (_rc != SW_OK) return _rc;   \
  } while (0)

extern "C" {

#include "sw_db.inc"
#include "sw_search.inc"
#include "sw_batch.inc"
#include "sw_align_host.inc"

int sw_encode(const char* text, int64_t n, uint8_t* out) {
  if (n < 0 || (n > 0 && (!text || !out))) return fail(SW_EINVAL, "sw_encode: bad arguments");
  static const char kAlphabet[] = "ARNDCQEGHILKMFPSTWYVBZX*";
  uint8_t lut[256];
  memset(lut, 255, sizeof lut);
  for (int c = 'A'; c <= 'Z'; c++) lut[c] = lut[c + 32] = 22;   // letters outside the table -> X
  for (int i = 0; i < 24; i++) {
    const unsigned char c = (unsigned char)kAlphabet[i];
    lut[c] = (uint8_t)i;
    if (c >= 'A' && c <= 'Z') lut[c + 32] = (uint8_t)i;
  }
  for (int64_t i = 0; i < n; i++)
    if (lut[(unsigned char)text[i]] == 255)
      return fail(SW_EINVAL, "sw_encode: invalid residue byte 0x%02x at position %lld", (unsigned char)text[i], (long long)i);
  for (int64_t i = 0; i < n; i++) out[i] = lut[(unsigned char)text[i]];
  return SW_OK;
}

#ifdef SW_PIPE_PROF
// Debug build only: read and clear the pipeline's per-warp cycle counters.
int sw_debug_pipe_counters(unsigned long long* out) {
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpyFromSymbol(out, swk::g_pipe_prof, sizeof(swk::g_pipe_prof)));
  static const unsigned long long zero[16][8] = {};
  CK(cudaMemcpyToSymbol(swk::g_pipe_prof, zero, sizeof zero));
  return SW_OK;
}
int sw_debug_intra_counters(unsigned long long* out) {
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpyFromSymbol(out, swk::g_intra_prof, sizeof(swk::g_intra_prof)));
  CK(cudaMemcpyFromSymbol(out + 8, swk::g_intra_first, sizeof(swk::g_intra_first)));
  CK(cudaMemset(nullptr, 0, 0));
  {
    void* p = nullptr;
    CK(cudaGetSymbolAddress(&p, swk::g_intra_first));
    CK(cudaMemset(p, 0, sizeof(swk::g_intra_first)));
  }
  unsigned long long init[8] = {~0ull, 0, 0, 0, 0, 0, 0, 0};
  CK(cudaMemcpyToSymbol(swk::g_intra_prof, init, sizeof init));
  return SW_OK;
}
#endif

// Host merge of per-device top-k lists (the multi-GPU exchange step, DESIGN.md §"Multi-GPU").
int sw_merge_topk(const int64_t* ids, const int32_t* scores, int32_t n_lists, int32_t k_in, int32_t k_out,
                  int64_t* out_ids, int32_t* out_scores) {
  if (n_lists < 0 || k_in < 0 || k_out < 1) return fail(SW_EINVAL, "sw_merge_topk: bad sizes");
  if ((n_lists * (int64_t)k_in > 0 && (!ids || !scores)) || !out_ids || !out_scores)
    return fail(SW_EINVAL, "sw_merge_topk: null pointer");
  std::vector<std::pair<int32_t, int64_t>> all;
  all.reserve((size_t)n_lists * k_in);
  for (int64_t t = 0; t < (int64_t)n_lists * k_in; t++)
    if (ids[t] >= 0) all.emplace_back(scores[t], ids[t]);
  const size_t take = std::min<size_t>(all.size(), (size_t)k_out);
  std::partial_sort(all.begin(), all.begin() + take, all.end(), [](const auto& a, const auto& b) {
    return a.first != b.first ? a.first > b.first : a.second < b.second;
  });
  for (int32_t t = 0; t < k_out; t++) {
    out_ids[t] = (size_t)t < take ? all[t].second : -1;
    out_scores[t] = (size_t)t < take ? all[t].first : -1;
  }
  return SW_OK;
}

}  // extern "C"
