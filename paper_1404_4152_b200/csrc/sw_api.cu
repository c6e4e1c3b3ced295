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
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include "../../include/swsearch.h"
#include "sw_kernels.cuh"
#include "sw_align.cuh"
#include "sw_ablation.cuh"

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

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t _e = (call);                                                              \
    if (_e != cudaSuccess)                                                                \
      return fail(_e == cudaErrorMemoryAllocation ? SW_ENOMEM : SW_ECUDA, "%s: %s (%s:%d)", \
                  #call, cudaGetErrorString(_e), __FILE__, __LINE__);                     \
  } while (0)

constexpr int kTileRows = 48;        // default query rows per register tile (SW_TILE_ROWS overrides: 32/48/64)

int tile_rows_env() {
  const char* e = getenv("SW_TILE_ROWS");
  const int v = e ? atoi(e) : kTileRows;
  return (v == 32 || v == 48 || v == 64) ? v : kTileRows;
}

int threads_env(int def) {
  const char* e = getenv("SW_THREADS");
  const int v = e ? atoi(e) : def;
  return (v == 384 || v == 512) ? v : def;
}

template <int T, int NT>
void* inter16_kernel(bool smem, bool big) {
  if (big) return smem ? (void*)swk::k_inter16<T, true, NT, true> : (void*)swk::k_inter16<T, false, NT, true>;
  return smem ? (void*)swk::k_inter16<T, true, NT> : (void*)swk::k_inter16<T, false, NT>;
}

template <int T>
void* inter16_kernel_nt(bool smem, int nt, bool big) {
  return nt == 512 ? inter16_kernel<T, 512>(smem, big) : inter16_kernel<T, 384>(smem, big);
}
constexpr int kMaxSmemProfile = 200 * 1024;

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
  int8_t* d_prof_qp = nullptr;    // f4 IntraQP ablation: profile with rows of 32*L bytes
  size_t prof_qp_cap = 0;
  void* aw[10] = {};              // sw_align workspace (grow-only): idx, jobs, res, q, M, prof, dir, bnd, ops, tmp
  size_t aw_cap[10] = {};

  uint2* d_scratch = nullptr;     // DP boundary rows, one slab per resident warp (inter-task kernels)
  uint2* d_scratch_intra = nullptr; // pass boundaries of the intra-task kernel (runs concurrently: own slabs)
  long long scratch_cols_intra = 0;
  long long scratch_cols = 0;
  int scratch_slots = 0;

  // per-search buffers
  uint8_t* d_query = nullptr;
  int query_cap = 0;
  int8_t* d_matrix = nullptr;
  int8_t* d_prof = nullptr;
  size_t prof_cap = 0;
  int* d_score_sorted = nullptr;
  int* d_scores = nullptr;        // input-order scores for the synchronous API
  unsigned long long* d_keys = nullptr;
  unsigned long long* d_cand = nullptr;
  unsigned long long* d_cand2 = nullptr;
  int cand_cap = 0;
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
  int topk_cap = 0;
  void* d_cub = nullptr;
  size_t cub_bytes = 0;

  uint8_t* h_stage = nullptr;     // pinned staging for query + matrix
  size_t stage_cap = 0;
  cudaEvent_t ev_stage = nullptr, ev_done = nullptr;
  // stage-boundary events of the last kRing searches (sync and async):
  // [0] start, [1] profile done, [2] first pass done, [3] rerun done, [4] ranking done
  static constexpr int kRing = 64;
  cudaEvent_t ev_ring[kRing][5] = {};
  int64_t n_searches = 0;
  int64_t launches = 0;           // kernels launched by this handle (all searches)
  int last_n_long = 0;            // groups aligned pair-wise by the intra-task path in the last search
  int last_first_stage = 16;      // lane width of the last search's first pass
};

extern "C" {

void sw_opts_default(sw_opts* o) {
  if (!o) return;
  memset(o, 0, sizeof *o);
  o->device = -1;
  o->first_stage = 16;
  o->long_threshold = 0;
}

const char* sw_strerror(int s) {
  switch (s) {
    case SW_OK: return "ok";
    case SW_EINVAL: return "invalid argument";
    case SW_ENOMEM: return "out of memory";
    case SW_ECUDA: return "CUDA error";
    case SW_ERANGE: return "score range exceeds int32 bound";
    case SW_EINTERNAL: return "internal error";
    default: return "unknown status";
  }
}

const char* sw_last_error(void) { return g_last_error.c_str(); }

static void free_db(sw_db* db) {
  if (!db) return;
  cudaSetDevice(db->device);
  if (db->stream) cudaStreamSynchronize(db->stream);
  void* ptrs[] = {db->d_words, db->d_groups, db->d_perm, db->d_len_sorted, db->d_gid, db->d_scratch,
                  db->d_query, db->d_matrix, db->d_prof, db->d_score_sorted, db->d_scores, db->d_keys,
                  db->d_cand, db->d_cand2, db->d_flag8, db->d_flag16, db->d_list8, db->d_list16,
                  db->d_block_counts, db->d_cnt, db->d_mini_sizes, db->d_mgroups, db->d_mwords, db->d_prof8b,
                  db->d_prof_b, db->d_prof2, db->d_score_sorted2, db->d_flag_b, db->d_scratch_intra,
                  db->d_counters, db->d_hist, db->d_sel,
                  db->d_topk_ids, db->d_topk_scores, db->d_cub, db->d_inv, db->d_chunk[0], db->d_chunk[1],
                  db->d_stream_cnt, db->d_prof_qp, db->d_big};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (void* p : db->aw)
    if (p) cudaFree(p);
  if (db->h_words) cudaFreeHost(db->h_words);
  for (int b = 0; b < 2; b++) {
    if (db->ev_copied[b]) cudaEventDestroy(db->ev_copied[b]);
    if (db->ev_consumed[b]) cudaEventDestroy(db->ev_consumed[b]);
  }
  if (db->copy_stream) cudaStreamDestroy(db->copy_stream);
  if (db->h_stage) cudaFreeHost(db->h_stage);
  if (db->ev_stage) cudaEventDestroy(db->ev_stage);
  if (db->ev_done) cudaEventDestroy(db->ev_done);
  for (auto& set : db->ev_ring)
    for (auto& e : set)
      if (e) cudaEventDestroy(e);
  if (db->stream) cudaStreamDestroy(db->stream);
  delete db;
}

void sw_db_destroy(sw_db* db) { free_db(db); }

int sw_db_get_info(const sw_db* db, sw_db_info* info) {
  if (!db || !info) return fail(SW_EINVAL, "sw_db_get_info: null argument");
  memset(info, 0, sizeof *info);
  info->n_seqs = db->n_seqs;
  info->n_residues = db->sum_len;
  info->n_inter = db->n_inter;
  info->n_intra = db->n_intra;
  info->n_groups = db->n_groups;
  info->packed_bytes = db->n_words * (int64_t)sizeof(uint2);
  info->scratch_bytes = ((int64_t)db->scratch_slots * db->scratch_cols +
                         (int64_t)db->num_sms * (swk::kInterThreads / 32) * db->scratch_cols_intra) * 32 * (int64_t)sizeof(uint2);
  info->max_len = db->max_len;
  info->device = db->device;
  info->long_threshold = db->long_threshold;
  info->residency = db->host_resident ? 1 : 0;
  info->n_chunks = (int32_t)db->chunks.size();
  info->launches = db->launches;
  info->n_searches = db->n_searches;
  return SW_OK;
}

int sw_db_stage_times(sw_db* db, int32_t back, float* ms) {
  if (!db || !ms) return fail(SW_EINVAL, "sw_db_stage_times: null argument");
  if (back < 1 || back > sw_db::kRing || back > db->n_searches)
    return fail(SW_EINVAL, "sw_db_stage_times: back must be in [1, min(%d, searches so far)]", sw_db::kRing);
  cudaEvent_t* ev = db->ev_ring[(db->n_searches - back) % sw_db::kRing];
  CK(cudaEventSynchronize(ev[4]));
  for (int t = 0; t < 4; t++) CK(cudaEventElapsedTime(&ms[t], ev[t], ev[t + 1]));
  return SW_OK;
}

static int validate_db(const uint8_t* residues, int64_t n_residues, const int64_t* offsets,
                       const int32_t* lengths, int64_t n_seqs, const int64_t* gids) {
  // ---- validation (host) ----
  if (n_seqs < 0 || n_seqs > 0x7fffffffLL - 64) return fail(SW_EINVAL, "n_seqs out of range: %lld", (long long)n_seqs);
  if (n_residues < 0) return fail(SW_EINVAL, "n_residues < 0");
  if (n_seqs > 0 && (!offsets || !lengths)) return fail(SW_EINVAL, "offsets/lengths must be non-NULL");
  if (n_residues > 0 && !residues) return fail(SW_EINVAL, "residues must be non-NULL");
  std::atomic<int64_t> bad{-1};
  std::atomic<int> bad_kind{0};
  parallel_for(n_seqs, [&](int64_t a, int64_t b) {
    for (int64_t i = a; i < b && bad.load(std::memory_order_relaxed) < 0; i++) {
      const int64_t off = offsets[i];
      const int32_t len = lengths[i];
      if (len < 0 || off < 0 || off > n_residues || (int64_t)len > n_residues - off) {
        bad = i; bad_kind = 1; return;
      }
      const uint8_t* s = residues + off;
      for (int32_t p = 0; p < len; p++)
        if (s[p] >= SW_NUM_CODES) { bad = i; bad_kind = 2; return; }
      if (gids && (gids[i] < 0 || gids[i] > 0xfffffffeLL)) { bad = i; bad_kind = 3; return; }
    }
  });
  if (bad >= 0) {
    const int64_t i = bad;
    if (bad_kind == 1) return fail(SW_EINVAL, "subject %lld: offset %lld / length %d outside residues[0,%lld)", (long long)i, (long long)offsets[i], lengths[i], (long long)n_residues);
    if (bad_kind == 2) return fail(SW_EINVAL, "subject %lld: residue code >= 24", (long long)i);
    return fail(SW_EINVAL, "subject %lld: global id %lld outside [0, 2^32-2]", (long long)i, (long long)gids[i]);
  }
  return SW_OK;
}

static int finish_create(sw_db* db);

static int validate_residency(const sw_opts& o) {
  if (o.residency != 0 && o.residency != 1) return fail(SW_EINVAL, "residency must be 0 or 1 (got %d)", o.residency);
  if (o.residency == 1 && o.first_stage == 8)
    return fail(SW_EINVAL, "residency 1 (streamed) supports first_stage 16 or 32, not 8");
  if (o.chunk_mb < 0 || o.chunk_mb > (1 << 20)) return fail(SW_EINVAL, "chunk_mb out of range (got %d)", o.chunk_mb);
  return SW_OK;
}

static void set_residency(sw_db* db, const sw_opts& o) {
  db->host_resident = o.residency == 1;
  db->chunk_words = (int64_t)(o.chunk_mb > 0 ? o.chunk_mb : 512) * (1 << 20) / (int64_t)sizeof(uint2);
}

static int create_impl(const uint8_t* residues, int64_t n_residues, const int64_t* offsets,
                       const int32_t* lengths, int64_t n_seqs, const int64_t* gids, const sw_opts* o,
                       sw_db* db) {
  db->n_seqs = n_seqs;
  db->n_residues = n_residues;

  // ---- stable sort by (length, input index): counting sort ----
  int32_t max_len = 0;
  int64_t sum_len = 0;
  for (int64_t i = 0; i < n_seqs; i++) {
    max_len = std::max(max_len, lengths[i]);
    sum_len += lengths[i];
  }
  db->max_len = max_len;
  db->sum_len = sum_len;
  std::vector<int> perm(n_seqs);
  {
    std::vector<int64_t> cnt((size_t)max_len + 2, 0);
    for (int64_t i = 0; i < n_seqs; i++) cnt[(size_t)lengths[i] + 1]++;
    for (size_t l = 1; l < cnt.size(); l++) cnt[l] += cnt[l - 1];
    for (int64_t i = 0; i < n_seqs; i++) perm[cnt[(size_t)lengths[i]]++] = (int)i;
  }
  std::vector<int> len_sorted(n_seqs);
  for (int64_t p = 0; p < n_seqs; p++) len_sorted[p] = lengths[perm[p]];

  // ---- one layout for both kernels: the intra-task path reads long groups pair by pair ----
  db->long_threshold = o->long_threshold;
  const int64_t n_inter = n_seqs;
  db->n_inter = n_inter;
  db->n_intra = 0;
  db->max_inter_len = n_inter ? len_sorted[n_inter - 1] : 0;

  // ---- groups of 64 consecutive sorted subjects, 5-bit codes, 6 per word ----
  const int64_t n_groups = (n_inter + swk::kGroup - 1) / swk::kGroup;
  std::vector<GroupDesc> groups(n_groups);
  int64_t base = 0;
  for (int64_t g = 0; g < n_groups; g++) {
    const int64_t first = g * swk::kGroup, last = std::min(first + swk::kGroup, n_inter) - 1;
    groups[g].base = base;
    groups[g].ncols = len_sorted[last];
    groups[g].count = (int)(last - first + 1);
    const int64_t nw = (groups[g].ncols + swk::kResPerWord - 1) / swk::kResPerWord;
    base += nw * 32;
  }
  db->n_groups = n_groups;
  db->n_words = base;
  db->group_ncols.resize(n_groups);
  for (int64_t g = 0; g < n_groups; g++) db->group_ncols[g] = groups[g].ncols;

  db->h_group_base.resize(n_groups + 1);
  for (int64_t g = 0; g < n_groups; g++) db->h_group_base[g] = groups[g].base;
  db->h_group_base[n_groups] = base;
  if (db->host_resident)
    CK(cudaHostAlloc(&db->h_words, std::max<int64_t>(base, 1) * sizeof(uint2), cudaHostAllocMapped | cudaHostAllocPortable));
  else
    CK(cudaMalloc(&db->d_words, std::max<int64_t>(base, 1) * sizeof(uint2)));
  {
    // pack group ranges into two pinned staging buffers, upload overlapped
    // (host residency: pack straight into the pinned host copy, no upload)
    const int64_t kChunkWords = 1 << 24;   // 128 MB of uint2
    uint2* stage[2] = {nullptr, nullptr};
    cudaEvent_t ev[2];
    if (!db->host_resident) {
      CK(cudaHostAlloc(&stage[0], kChunkWords * sizeof(uint2), cudaHostAllocDefault));
      CK(cudaHostAlloc(&stage[1], kChunkWords * sizeof(uint2), cudaHostAllocDefault));
    }
    CK(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
    int64_t g0 = 0;
    int buf = 0;
    bool used[2] = {false, false};
    int rc = SW_OK;
    while (g0 < n_groups && rc == SW_OK) {
      int64_t g1 = g0;
      while (g1 < n_groups) {
        const int64_t end = (g1 + 1 < n_groups ? groups[g1 + 1].base : base);
        if (end - groups[g0].base > kChunkWords && g1 > g0) break;
        if (end - groups[g0].base > kChunkWords) { rc = fail(SW_EINTERNAL, "group larger than staging"); break; }
        g1++;
      }
      if (rc != SW_OK) break;
      if (used[buf]) cudaEventSynchronize(ev[buf]);
      const int64_t wbase = groups[g0].base;
      uint2* st = db->host_resident ? db->h_words + wbase : stage[buf];
      const int64_t wend = (g1 < n_groups ? groups[g1].base : base);
      parallel_for(g1 - g0, [&](int64_t a, int64_t b) {
        for (int64_t gg = g0 + a; gg < g0 + b; gg++) {
          const GroupDesc& G = groups[gg];
          const int nw = (G.ncols + swk::kResPerWord - 1) / swk::kResPerWord;
          uint2* out = st + (G.base - wbase);
          for (int l = 0; l < swk::kGroup; l++) {
            const int64_t p = gg * swk::kGroup + l;
            const uint8_t* s = nullptr;
            int len = 0;
            if (l < G.count) {
              s = residues + offsets[perm[p]];
              len = len_sorted[p];
            }
            for (int w = 0; w < nw; w++) {
              uint32_t word = 0;
              for (int c = 0; c < swk::kResPerWord; c++) {
                const int j = w * swk::kResPerWord + c;
                const uint32_t code = j < len ? s[j] : (uint32_t)swk::kDummy;
                word |= code << (5 * c);
              }
              uint2& dst = out[(int64_t)w * 32 + (l >> 1)];
              if (l & 1) dst.y = word; else dst.x = word;
            }
          }
        }
      });
      if (!db->host_resident) {
        cudaError_t e = cudaMemcpyAsync(db->d_words + wbase, st, (wend - wbase) * sizeof(uint2),
                                        cudaMemcpyHostToDevice, db->stream);
        if (e != cudaSuccess) { rc = fail(SW_ECUDA, "upload: %s", cudaGetErrorString(e)); break; }
      }
      cudaEventRecord(ev[buf], db->stream);
      used[buf] = true;
      buf ^= 1;
      g0 = g1;
    }
    cudaStreamSynchronize(db->stream);
    if (stage[0]) cudaFreeHost(stage[0]);
    if (stage[1]) cudaFreeHost(stage[1]);
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
    if (rc != SW_OK) return rc;
  }
  CK(cudaMalloc(&db->d_groups, std::max<int64_t>(n_groups, 1) * sizeof(GroupDesc)));
  if (n_groups) CK(cudaMemcpy(db->d_groups, groups.data(), n_groups * sizeof(GroupDesc), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&db->d_perm, std::max<int64_t>(n_seqs, 1) * sizeof(int)));
  CK(cudaMalloc(&db->d_len_sorted, std::max<int64_t>(n_seqs, 1) * sizeof(int)));
  if (n_seqs) {
    CK(cudaMemcpy(db->d_perm, perm.data(), n_seqs * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(db->d_len_sorted, len_sorted.data(), n_seqs * sizeof(int), cudaMemcpyHostToDevice));
  }
  if (gids && n_seqs) {
    CK(cudaMalloc(&db->d_gid, n_seqs * sizeof(long long)));
    CK(cudaMemcpy(db->d_gid, gids, n_seqs * sizeof(long long), cudaMemcpyHostToDevice));
  }

  return finish_create(db);
}

// Device buffers that depend only on the layout (shared by create and load).
static int finish_create(sw_db* db) {
  const int64_t n_seqs = db->n_seqs;
  // ---- DP boundary scratch: one slab per resident warp of the persistent kernels ----
  db->scratch_slots = db->num_sms * (swk::kMaxThreads / 32);
  // Inter-task tiles need one boundary column per subject column (capped: longer
  // groups go to the intra-task path); the intra-task wavefronts need 2 x ncols
  // words of the same slab (pass parity).
  {
    const int64_t inter = std::min<int64_t>(((int64_t)db->max_inter_len + swk::kResPerWord) / swk::kResPerWord *
                                            swk::kResPerWord + swk::kResPerWord, swk::kMaxInterCols);
    const int64_t intra = ((int64_t)db->max_len + 15) / 16 + 8;
    db->scratch_cols = std::max(inter, intra);
  }
  CK(cudaMalloc(&db->d_scratch, (size_t)db->scratch_slots * db->scratch_cols * 32 * sizeof(uint2)));
  db->scratch_cols_intra = ((int64_t)db->max_len + 15) / 16 + 2;   // 2 x max_len words per warp
  CK(cudaMalloc(&db->d_scratch_intra,
                (size_t)db->num_sms * (swk::kInterThreads / 32) * db->scratch_cols_intra * 32 * sizeof(uint2)));

  // ---- per-search buffers sized by n ----
  const int64_t n1 = std::max<int64_t>(n_seqs, 1);
  CK(cudaMalloc(&db->d_score_sorted, n1 * sizeof(int)));
  CK(cudaMalloc(&db->d_scores, n1 * sizeof(int)));
  CK(cudaMalloc(&db->d_keys, n1 * sizeof(unsigned long long)));
  CK(cudaMalloc(&db->d_flag8, n1));
  CK(cudaMalloc(&db->d_flag16, n1));
  CK(cudaMalloc(&db->d_list8, n1 * sizeof(int)));
  CK(cudaMalloc(&db->d_list16, n1 * sizeof(int)));
  CK(cudaMalloc(&db->d_block_counts, (n1 / swk::kScanBlock + 2) * sizeof(int)));
  CK(cudaMalloc(&db->d_cnt, 4 * sizeof(int)));
  CK(cudaMemset(db->d_cnt, 0, 4 * sizeof(int)));
  db->n_mini_max = n1 / swk::kGroup + 1;
  if (db->first_stage == 8) {
    // sum over mini-groups of ncols <= 2 max_len + total/64 (sorted members), see DESIGN.md §"int8 stage"
    const int64_t mini_words = db->n_words + (2 * (int64_t)db->max_len / swk::kResPerWord + 2 + db->n_mini_max) * 32;
    CK(cudaMalloc(&db->d_mini_sizes, db->n_mini_max * sizeof(int)));
    CK(cudaMalloc(&db->d_mgroups, db->n_mini_max * sizeof(GroupDesc)));
    CK(cudaMalloc(&db->d_mwords, mini_words * sizeof(uint2)));
  }
  CK(cudaMalloc(&db->d_counters, 8 * sizeof(int)));
  CK(cudaMalloc(&db->d_hist, 256 * sizeof(unsigned)));
  CK(cudaMemset(db->d_hist, 0, 256 * sizeof(unsigned)));
  CK(cudaMalloc(&db->d_sel, sizeof(swk::SelState)));
  CK(cudaMalloc(&db->d_matrix, 32 * 32));
  if (db->host_resident) {
    // chunks of whole groups, at most chunk_words each (a group never splits)
    int64_t maxg = 0;
    for (int64_t g = 0; g < db->n_groups; g++)
      maxg = std::max(maxg, db->h_group_base[g + 1] - db->h_group_base[g]);
    db->chunk_words = std::max(db->chunk_words, std::max<int64_t>(maxg, 1));
    db->chunks.clear();
    for (int64_t g0 = 0; g0 < db->n_groups;) {
      int64_t g1 = g0 + 1;
      while (g1 < db->n_groups && db->h_group_base[g1 + 1] - db->h_group_base[g0] <= db->chunk_words) g1++;
      db->chunks.emplace_back(g0, g1);
      g0 = g1;
    }
    const int64_t cw = std::min(db->chunk_words, std::max<int64_t>(db->n_words, 1));
    CK(cudaMalloc(&db->d_chunk[0], cw * sizeof(uint2)));
    CK(cudaMalloc(&db->d_chunk[1], cw * sizeof(uint2)));
    CK(cudaMalloc(&db->d_stream_cnt, std::max<size_t>(db->chunks.size(), 1) * sizeof(int)));
    CK(cudaMemset(db->d_stream_cnt, 0, std::max<size_t>(db->chunks.size(), 1) * sizeof(int)));
    CK(cudaStreamCreateWithFlags(&db->copy_stream, cudaStreamNonBlocking));
    for (int b = 0; b < 2; b++) {
      CK(cudaEventCreateWithFlags(&db->ev_copied[b], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&db->ev_consumed[b], cudaEventDisableTiming));
    }
  }
  CK(cudaEventCreateWithFlags(&db->ev_stage, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&db->ev_done, cudaEventDisableTiming));
  for (auto& set : db->ev_ring)
    for (auto& e : set) CK(cudaEventCreate(&e));
  return SW_OK;
}

int sw_db_create(const uint8_t* residues, int64_t n_residues, const int64_t* offsets,
                 const int32_t* lengths, int64_t n_seqs, const int64_t* global_ids,
                 const sw_opts* opts, sw_db** out) {
  if (!out) return fail(SW_EINVAL, "out must be non-NULL");
  *out = nullptr;
  sw_opts o;
  sw_opts_default(&o);
  if (opts) o = *opts;
  if (o.first_stage != 8 && o.first_stage != 16 && o.first_stage != 32)
    return fail(SW_EINVAL, "first_stage must be 8, 16 or 32 (got %d)", o.first_stage);
  {
    int rc = validate_residency(o);
    if (rc != SW_OK) return rc;
  }
  {
    int rc = validate_db(residues, n_residues, offsets, lengths, n_seqs, global_ids);
    if (rc != SW_OK) return rc;
  }
  sw_db* db = new (std::nothrow) sw_db;
  if (!db) return fail(SW_ENOMEM, "host allocation");
  if (o.device < 0) {
    if (cudaGetDevice(&db->device) != cudaSuccess) { delete db; return fail(SW_ECUDA, "cudaGetDevice failed"); }
  } else {
    db->device = o.device;
  }
  db->first_stage = o.first_stage;
  set_residency(db, o);
  cudaError_t e = cudaSetDevice(db->device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&db->num_sms, cudaDevAttrMultiProcessorCount, db->device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&db->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    int rc = fail(SW_ECUDA, "device %d: %s", db->device, cudaGetErrorString(e));
    free_db(db);
    return rc;
  }
  int rc = create_impl(residues, n_residues, offsets, lengths, n_seqs, global_ids, &o, db);
  if (rc != SW_OK) {
    std::string msg = g_last_error;
    free_db(db);
    g_last_error = msg;
    return rc;
  }
  *out = db;
  return SW_OK;
}


// ---- f2: persistent packed index (the paper's offline, mmap-able index files) ----
namespace {
struct DbFileHeader {
  char magic[8];            // "SWB200DB"
  uint32_t version;         // 1
  uint32_t header_bytes;
  int64_t n_seqs, n_residues, sum_len;
  int64_t n_groups, n_words;
  int32_t max_len, has_gid;
  int64_t off_groups, off_perm, off_len, off_gid, off_words, file_bytes;
};
constexpr uint32_t kDbFileVersion = 1;
int64_t align64(int64_t x) { return (x + 63) / 64 * 64; }
}  // namespace

int sw_db_save(sw_db* db, const char* path) {
  if (!db || !path) return fail(SW_EINVAL, "sw_db_save: null argument");
  std::lock_guard<std::mutex> lock(db->mu);
  CK(cudaSetDevice(db->device));
  CK(cudaStreamSynchronize(db->stream));
  DbFileHeader h;
  memset(&h, 0, sizeof h);
  memcpy(h.magic, "SWB200DB", 8);
  h.version = kDbFileVersion;
  h.header_bytes = sizeof h;
  h.n_seqs = db->n_seqs;
  h.n_residues = db->n_residues;
  h.sum_len = db->sum_len;
  h.n_groups = db->n_groups;
  h.n_words = db->n_words;
  h.max_len = db->max_len;
  h.has_gid = db->d_gid ? 1 : 0;
  h.off_groups = align64(sizeof h);
  h.off_perm = align64(h.off_groups + h.n_groups * (int64_t)sizeof(GroupDesc));
  h.off_len = align64(h.off_perm + h.n_seqs * 4);
  h.off_gid = align64(h.off_len + h.n_seqs * 4);
  h.off_words = align64(h.off_gid + (h.has_gid ? h.n_seqs * 8 : 0));
  h.file_bytes = h.off_words + h.n_words * (int64_t)sizeof(uint2);
  FILE* f = fopen(path, "wb");
  if (!f) return fail(SW_EINVAL, "sw_db_save: cannot open %s for writing", path);
  int rc = SW_OK;
  auto put = [&](int64_t off, const void* dev, int64_t bytes) {
    if (rc != SW_OK || bytes <= 0) return;
    std::vector<char> buf((size_t)std::min<int64_t>(bytes, 1 << 26));
    for (int64_t done = 0; done < bytes && rc == SW_OK; done += (int64_t)buf.size()) {
      const int64_t c = std::min<int64_t>((int64_t)buf.size(), bytes - done);
      cudaError_t e = cudaMemcpy(buf.data(), (const char*)dev + done, c, cudaMemcpyDefault);
      if (e != cudaSuccess) { rc = fail(SW_ECUDA, "sw_db_save: %s", cudaGetErrorString(e)); return; }
      if (fseeko(f, off + done, SEEK_SET) != 0 || fwrite(buf.data(), 1, c, f) != (size_t)c)
        rc = fail(SW_EINVAL, "sw_db_save: write failed on %s", path);
    }
  };
  if (fwrite(&h, sizeof h, 1, f) != 1) rc = fail(SW_EINVAL, "sw_db_save: write failed on %s", path);
  put(h.off_groups, db->d_groups, h.n_groups * (int64_t)sizeof(GroupDesc));
  put(h.off_perm, db->d_perm, h.n_seqs * 4);
  put(h.off_len, db->d_len_sorted, h.n_seqs * 4);
  if (h.has_gid) put(h.off_gid, db->d_gid, h.n_seqs * 8);
  put(h.off_words, db->host_resident ? (const void*)db->h_words : (const void*)db->d_words,
      h.n_words * (int64_t)sizeof(uint2));
  if (fclose(f) != 0 && rc == SW_OK) rc = fail(SW_EINVAL, "sw_db_save: close failed on %s", path);
  return rc;
}

static int load_impl(const char* map, const DbFileHeader& h, sw_db* db) {
  db->n_seqs = h.n_seqs;
  db->n_residues = h.n_residues;
  db->sum_len = h.sum_len;
  db->max_len = h.max_len;
  db->n_groups = h.n_groups;
  db->n_words = h.n_words;
  db->n_inter = h.n_seqs;
  db->n_intra = 0;
  const GroupDesc* groups = (const GroupDesc*)(map + h.off_groups);
  const int* len_sorted = (const int*)(map + h.off_len);
  db->max_inter_len = h.n_seqs ? len_sorted[h.n_seqs - 1] : 0;
  db->group_ncols.resize(h.n_groups);
  int64_t expect_base = 0;
  for (int64_t g = 0; g < h.n_groups; g++) {   // the table must describe exactly the stored words
    db->group_ncols[g] = groups[g].ncols;
    if (groups[g].base != expect_base || groups[g].ncols < 0 || (g && groups[g].ncols < groups[g - 1].ncols))
      return fail(SW_EINVAL, "sw_db_load: corrupt group table at group %lld", (long long)g);
    expect_base += (int64_t)(groups[g].ncols + swk::kResPerWord - 1) / swk::kResPerWord * 32;
  }
  if (expect_base != h.n_words) return fail(SW_EINVAL, "sw_db_load: group table / word count mismatch");
  db->h_group_base.resize(h.n_groups + 1);
  for (int64_t g = 0; g < h.n_groups; g++) db->h_group_base[g] = groups[g].base;
  db->h_group_base[h.n_groups] = h.n_words;
  if (db->host_resident)
    CK(cudaHostAlloc(&db->h_words, std::max<int64_t>(h.n_words, 1) * sizeof(uint2),
                     cudaHostAllocMapped | cudaHostAllocPortable));
  else
    CK(cudaMalloc(&db->d_words, std::max<int64_t>(h.n_words, 1) * sizeof(uint2)));
  CK(cudaMalloc(&db->d_groups, std::max<int64_t>(h.n_groups, 1) * sizeof(GroupDesc)));
  CK(cudaMalloc(&db->d_perm, std::max<int64_t>(h.n_seqs, 1) * sizeof(int)));
  CK(cudaMalloc(&db->d_len_sorted, std::max<int64_t>(h.n_seqs, 1) * sizeof(int)));
  // pinned double-buffered staging from the mapped file
  const int64_t kChunk = 1 << 27;
  char* stage[2] = {nullptr, nullptr};
  CK(cudaHostAlloc(&stage[0], kChunk, cudaHostAllocDefault));
  CK(cudaHostAlloc(&stage[1], kChunk, cudaHostAllocDefault));
  cudaEvent_t ev[2];
  cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming);
  bool used[2] = {false, false};
  int buf = 0;
  int rc = SW_OK;
  auto up = [&](void* dst, const char* src, int64_t bytes) {
    for (int64_t done = 0; done < bytes && rc == SW_OK; done += kChunk) {
      const int64_t c = std::min(kChunk, bytes - done);
      if (used[buf]) cudaEventSynchronize(ev[buf]);
      memcpy(stage[buf], src + done, c);
      cudaError_t e = cudaMemcpyAsync((char*)dst + done, stage[buf], c, cudaMemcpyHostToDevice, db->stream);
      if (e != cudaSuccess) rc = fail(SW_ECUDA, "sw_db_load: %s", cudaGetErrorString(e));
      cudaEventRecord(ev[buf], db->stream);
      used[buf] = true;
      buf ^= 1;
    }
  };
  up(db->d_groups, map + h.off_groups, h.n_groups * (int64_t)sizeof(GroupDesc));
  up(db->d_perm, map + h.off_perm, h.n_seqs * 4);
  up(db->d_len_sorted, map + h.off_len, h.n_seqs * 4);
  if (h.has_gid) {
    if (cudaMalloc(&db->d_gid, h.n_seqs * sizeof(long long)) != cudaSuccess) rc = fail(SW_ENOMEM, "sw_db_load: gid");
    up(db->d_gid, map + h.off_gid, h.n_seqs * 8);
  }
  if (db->host_resident) {
    const char* src = map + h.off_words;
    char* dst = (char*)db->h_words;
    const int64_t bytes = h.n_words * (int64_t)sizeof(uint2);
    parallel_for((bytes + (1 << 20) - 1) >> 20, [&](int64_t a, int64_t b) {
      const int64_t lo = a << 20, hi = std::min<int64_t>(bytes, b << 20);
      if (hi > lo) memcpy(dst + lo, src + lo, (size_t)(hi - lo));
    });
  } else {
    up(db->d_words, map + h.off_words, h.n_words * (int64_t)sizeof(uint2));
  }
  cudaStreamSynchronize(db->stream);
  cudaFreeHost(stage[0]);
  cudaFreeHost(stage[1]);
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  if (rc != SW_OK) return rc;
  return finish_create(db);
}

int sw_db_load(const char* path, const sw_opts* opts, sw_db** out) {
  if (!out || !path) return fail(SW_EINVAL, "sw_db_load: null argument");
  *out = nullptr;
  sw_opts o;
  sw_opts_default(&o);
  if (opts) o = *opts;
  if (o.first_stage != 8 && o.first_stage != 16 && o.first_stage != 32)
    return fail(SW_EINVAL, "first_stage must be 8, 16 or 32 (got %d)", o.first_stage);
  {
    int rc = validate_residency(o);
    if (rc != SW_OK) return rc;
  }
  const int fd = open(path, O_RDONLY);
  if (fd < 0) return fail(SW_EINVAL, "sw_db_load: cannot open %s", path);
  struct stat sb;
  if (fstat(fd, &sb) != 0 || sb.st_size < (off_t)sizeof(DbFileHeader)) {
    close(fd);
    return fail(SW_EINVAL, "sw_db_load: %s is not a database file (too small)", path);
  }
  void* map = mmap(nullptr, (size_t)sb.st_size, PROT_READ, MAP_PRIVATE, fd, 0);
  close(fd);
  if (map == MAP_FAILED) return fail(SW_EINVAL, "sw_db_load: mmap of %s failed", path);
  DbFileHeader h;
  memcpy(&h, map, sizeof h);
  auto bad = [&](const char* why) {
    munmap(map, (size_t)sb.st_size);
    return fail(SW_EINVAL, "sw_db_load: %s: %s", path, why);
  };
  if (memcmp(h.magic, "SWB200DB", 8) != 0) return bad("bad magic");
  if (h.version != kDbFileVersion || h.header_bytes != sizeof h) return bad("unsupported version");
  if (h.n_seqs < 0 || h.n_seqs > 0x7fffffffLL - 64 || h.n_groups != (h.n_seqs + swk::kGroup - 1) / swk::kGroup ||
      h.n_words < 0 || h.file_bytes != (int64_t)sb.st_size ||
      h.off_words + h.n_words * (int64_t)sizeof(uint2) != h.file_bytes || h.off_groups < (int64_t)sizeof h ||
      h.off_perm < h.off_groups + h.n_groups * (int64_t)sizeof(GroupDesc) || h.off_len < h.off_perm + h.n_seqs * 4 ||
      h.off_gid < h.off_len + h.n_seqs * 4 || h.off_words < h.off_gid + (h.has_gid ? h.n_seqs * 8 : 0))
    return bad("inconsistent header (truncated or corrupt file)");
  sw_db* db = new (std::nothrow) sw_db;
  if (!db) return bad("host allocation");
  db->first_stage = o.first_stage;
  db->long_threshold = o.long_threshold;
  set_residency(db, o);
  cudaError_t e = cudaSuccess;
  if (o.device < 0) e = cudaGetDevice(&db->device);
  else db->device = o.device;
  if (e == cudaSuccess) e = cudaSetDevice(db->device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&db->num_sms, cudaDevAttrMultiProcessorCount, db->device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&db->stream, cudaStreamNonBlocking);
  int rc = e == cudaSuccess ? load_impl((const char*)map, h, db) : fail(SW_ECUDA, "device %d: %s", db->device, cudaGetErrorString(e));
  munmap(map, (size_t)sb.st_size);
  if (rc != SW_OK) {
    std::string msg = g_last_error;
    free_db(db);
    g_last_error = msg;
    return rc;
  }
  *out = db;
  return SW_OK;
}

static int validate_search(const sw_db* db, const uint8_t* query, int32_t qlen, const int8_t* matrix,
                           int32_t alpha, int32_t beta, int32_t k, int* smax_out, int* smin_out) {
  if (!db) return fail(SW_EINVAL, "db is NULL");
  if (!query || !matrix) return fail(SW_EINVAL, "query/matrix must be non-NULL");
  if (qlen < 1) return fail(SW_EINVAL, "qlen must be >= 1 (got %d)", qlen);
  if (k < 1) return fail(SW_EINVAL, "k must be >= 1 (got %d)", k);
  if (alpha < 0 || beta < alpha || beta > 32767)
    return fail(SW_EINVAL, "need 0 <= alpha <= beta <= 32767 (alpha=%d, beta=%d)", alpha, beta);
  for (int i = 0; i < qlen; i++)
    if (query[i] >= SW_NUM_CODES) return fail(SW_EINVAL, "query position %d: residue code %d >= 24", i, query[i]);
  int smax = 0, smin = 0;
  for (int r = 0; r < 32; r++)
    for (int c = 0; c < 32; c++) {
      const int v = matrix[r * 32 + c];
      if ((r >= SW_NUM_CODES || c >= SW_NUM_CODES) && v != 0)
        return fail(SW_EINVAL, "matrix[%d][%d] = %d: rows/columns 24..31 must be 0", r, c, v);
      smax = std::max(smax, v);
      smin = std::min(smin, v);
    }
  if ((int64_t)qlen * smax >= (1LL << 31)) return fail(SW_ERANGE, "qlen * s_max = %lld >= 2^31", (long long)qlen * smax);
  *smax_out = smax;
  *smin_out = smin;
  return SW_OK;
}

static int ensure(void** p, size_t* cap, size_t need) {
  if (*cap >= need && *p) return SW_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  CK(cudaMalloc(p, need));
  *cap = need;
  return SW_OK;
}

// Stage (iv) for one query: scatter the sorted-order scores to input order and
// select the exact top-k by (score desc, global id asc) -- "sort all alignment
// scores in descending order" without sorting all N.
static int rank_enqueue(sw_db* db, const int* score_sorted, int* d_scores, int32_t k, long long* d_tk_ids,
                        int* d_tk_scores, cudaStream_t st, int64_t& nl) {
  const int n = (int)db->n_seqs;
  if (n > 0) {
    const int fb = std::min((n + 255) / 256, db->num_sms * 8);
    swk::k_finalize<<<fb, 256, 0, st>>>(score_sorted, db->d_perm, n, db->d_gid, d_scores, db->d_keys);
    CK(cudaGetLastError());
    nl++;
  }
  if (d_tk_ids || d_tk_scores) {
    const int cnt = std::min<int64_t>(k, n);
    if (cnt > 0) {
      const bool take_all = k >= n;
      if (!take_all) {
        swk::k_sel_init<<<1, 32, 0, st>>>(db->d_sel, (long long)k);
        nl++;
        const int hb = std::min((n + 1023) / 1024, db->num_sms * 4);
        for (int shift = 56; shift >= 0; shift -= 8) {
          swk::k_sel_hist<<<hb, 256, 0, st>>>(db->d_keys, n, db->d_sel, shift, db->d_hist);
          swk::k_sel_pick<<<1, 256, 0, st>>>(db->d_sel, shift, db->d_hist);
          nl += 2;
        }
        CK(cudaGetLastError());
      }
      if (db->cand_cap < cnt) {
        if (db->d_cand) cudaFree(db->d_cand);
        if (db->d_cand2) cudaFree(db->d_cand2);
        db->d_cand = db->d_cand2 = nullptr;
        CK(cudaMalloc(&db->d_cand, (size_t)cnt * sizeof(unsigned long long)));
        CK(cudaMalloc(&db->d_cand2, (size_t)cnt * sizeof(unsigned long long)));
        db->cand_cap = cnt;
      }
      const int cb = std::min((n + 1023) / 1024, db->num_sms * 4);
      CK(cudaMemsetAsync(db->d_counters + 3, 0, sizeof(int), st));   // candidate count (per ranking)
      swk::k_sel_compact<<<cb, 256, 0, st>>>(db->d_keys, n, db->d_sel, take_all ? 1 : 0, db->d_cand,
                                            db->d_counters + 3);
      CK(cudaGetLastError());
      nl += 2;   // compaction + final sort/decode
      if (cnt <= 4096) {
        swk::k_topk_small<<<1, 1024, 0, st>>>(db->d_cand, cnt, k, d_tk_ids, d_tk_scores);
      } else {
        size_t need = 0;
        cub::DeviceRadixSort::SortKeysDescending(nullptr, need, db->d_cand, db->d_cand2, cnt, 0, 64, st);
        int rc = ensure(&db->d_cub, &db->cub_bytes, need);
        if (rc) return rc;
        CK(cub::DeviceRadixSort::SortKeysDescending(db->d_cub, need, db->d_cand, db->d_cand2, cnt, 0, 64, st));
        swk::k_topk_decode<<<(k + 255) / 256, 256, 0, st>>>(db->d_cand2, cnt, k, d_tk_ids, d_tk_scores);
      }
      CK(cudaGetLastError());
    } else {
      swk::k_topk_decode<<<(k + 255) / 256, 256, 0, st>>>(db->d_cand, 0, k, d_tk_ids, d_tk_scores);
      CK(cudaGetLastError());
      nl++;
    }
  }
  return SW_OK;
}

// Enqueue the whole search on `st`.  Outputs: d_scores (input order) may be
// nullptr; top-k always goes to d_tk_ids/d_tk_scores when non-null.
static int search_enqueue(sw_db* db, const uint8_t* query, int32_t qlen, const int8_t* matrix,
                          int32_t alpha, int32_t beta, int32_t k, int smax, int smin, int* d_scores,
                          long long* d_tk_ids, int* d_tk_scores, cudaStream_t st) {
  cudaEvent_t* ev = db->ev_ring[db->n_searches % sw_db::kRing];
  int64_t nl = 0;   // kernel launches of this search
  // ---- stage (i): query + matrix H2D and profile ----
  const int m_pad = (qlen + 7) / 8 * 8;
  const int stride = (m_pad + 31) / 32 * 32 + 8;   // 8-byte skew per residue row (bank spread)
  const size_t prof_bytes = ((size_t)swk::kProfRows * stride + 15) / 16 * 16;
  {
    const size_t need = (size_t)qlen + 1024;
    if (db->stage_cap < need) {
      if (db->h_stage) { cudaEventSynchronize(db->ev_stage); cudaFreeHost(db->h_stage); db->h_stage = nullptr; }
      CK(cudaHostAlloc(&db->h_stage, need, cudaHostAllocDefault));
      db->stage_cap = need;
    } else {
      CK(cudaEventSynchronize(db->ev_stage));   // previous staged copy has drained
    }
    memcpy(db->h_stage, matrix, 1024);
    memcpy(db->h_stage + 1024, query, qlen);
    size_t qcap = (size_t)db->query_cap;
    void* dq = db->d_query;
    int rc = ensure(&dq, &qcap, (size_t)qlen);
    db->d_query = (uint8_t*)dq;
    db->query_cap = (int)qcap;
    if (rc) return rc;
    void* dp = db->d_prof;
    const size_t cap0 = db->prof_cap;
    rc = ensure(&dp, &db->prof_cap, prof_bytes);
    db->d_prof = (int8_t*)dp;
    if (rc) return rc;
    if (db->first_stage == 8 && (db->prof_cap != cap0 || !db->d_prof8b)) {
      if (db->d_prof8b) cudaFree(db->d_prof8b);
      db->d_prof8b = nullptr;
      CK(cudaMalloc(&db->d_prof8b, db->prof_cap));
    }
    CK(cudaMemcpyAsync(db->d_matrix, db->h_stage, 1024, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(db->d_query, db->h_stage + 1024, qlen, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(db->ev_stage, st));
  }
  CK(cudaEventRecord(ev[0], st));
  nl++;
  swk::k_profile<<<64, 256, 0, st>>>(db->d_query, qlen, db->d_matrix, db->d_prof, stride);
  CK(cudaGetLastError());
  CK(cudaMemsetAsync(db->d_counters, 0, 8 * sizeof(int), st));
  CK(cudaMemsetAsync(db->d_cnt, 0, 4 * sizeof(int), st));
  CK(cudaEventRecord(ev[1], st));

  // ---- stage (ii): alignment ----
  const int n = (int)db->n_seqs;
  const bool smem = prof_bytes <= (size_t)kMaxSmemProfile;
  const size_t smem_bytes = smem ? prof_bytes : 0;
  const int grid = db->num_sms;   // one persistent 384-thread CTA per SM
  const int limit16 = 32767 - smax;
  // groups whose inter-task work would exceed ~a warp's average share (or that do
  // not fit the per-warp boundary slab) are aligned pair by pair by the
  // intra-task wavefront kernel (load balance)
  int cut = 0;
  {
    int64_t c;
    const int64_t n_warps = (int64_t)db->num_sms * (swk::kInterThreads / 32);
    if (db->long_threshold > 0) c = db->long_threshold;
    else if (db->long_threshold == 0) c = std::max<int64_t>(128, db->sum_len / (64 * std::max<int64_t>(n_warps, 1)));
    else c = INT64_MAX;
    if (const char* e = getenv("SW_LONG_COLS")) c = atoll(e);
    cut = (int)std::min<int64_t>(c, INT32_MAX);
  }
  // Groups wider than a warp's boundary slab (scratch_cols) stay inter-task with
  // a slab of their own ("big" items: they are the first items of the
  // longest-first queue); at most kMaxBig of them and kBigBytes of slabs, the
  // rest of the widest groups go to the intra-task kernel.
  long long big_cols = 0;
  int n_big = 0;
  {
    int64_t kMaxBig = 2048;
    constexpr int64_t kBigBytes = 8LL << 30;
    if (const char* e = getenv("SW_MAX_BIG")) kMaxBig = std::max<int64_t>(0, atoll(e));   // tests: the fallback
    const auto& gc = db->group_ncols;
    const int64_t b0 = std::upper_bound(gc.begin(), gc.end(), (int)db->scratch_cols) - gc.begin();
    int64_t b1 = std::upper_bound(gc.begin(), gc.end(), cut) - gc.begin();   // inter-task groups: [0, b1)
    if (b1 > b0) {
      b1 = std::min<int64_t>(b1, b0 + kMaxBig);
      while (b1 > b0 && (b1 - b0) * (int64_t)(gc[b1 - 1] + swk::kResPerWord) * 32 * (int64_t)sizeof(uint2) > kBigBytes) b1--;
      cut = b1 > b0 ? gc[b1 - 1] : (int)db->scratch_cols;
      if (b1 < (int64_t)gc.size() && gc[b1] == cut) {          // keep the split on a column count boundary
        while (b1 > b0 && gc[b1 - 1] == cut) b1--;
        cut = b1 > b0 ? gc[b1 - 1] : (int)db->scratch_cols;
      }
      n_big = (int)(b1 - b0);
      big_cols = n_big ? (long long)cut + 2 * swk::kResPerWord : 0;
      if (n_big) {
        void* pb = db->d_big;
        int rc = ensure(&pb, &db->big_cap, (size_t)n_big * big_cols * 32 * sizeof(uint2));
        db->d_big = (uint2*)pb;
        if (rc) return rc;
      }
    } else {
      cut = (int)std::min<int64_t>(cut, db->scratch_cols);
    }
  }
  const int n_long = (int)(db->group_ncols.end() -
                           std::upper_bound(db->group_ncols.begin(), db->group_ncols.end(), cut));
  db->last_n_long = n_long;
  // compaction of a flag byte array (nr positions) into an ascending list of positions
  auto compact = [&](uint8_t* flag, int nr, int* list, int* count, int* tail_groups) -> int {
    const int nb_scan = std::max(1, (nr + swk::kScanBlock - 1) / swk::kScanBlock);
    swk::k_flag_count<<<nb_scan, swk::kScanBlock, 0, st>>>(flag, nr, db->d_block_counts);
    swk::k_scan_exclusive<<<1, swk::kScanBlock, 0, st>>>(db->d_block_counts, nb_scan, count, tail_groups);
    swk::k_flag_scatter<<<nb_scan, swk::kScanBlock, 0, st>>>(flag, nr, db->d_block_counts, list);
    nl += 3;
    CK(cudaGetLastError());
    return SW_OK;
  };
  // f4 ablations (measurement switch, not ABI): 1 = InterSP score profile,
  // 2 = IntraQP striped intra-task kernel (queries up to 2,048 rows)
  int variant = 0;
  if (const char* e = getenv("SW_VARIANT")) variant = strcmp(e, "intersp") == 0 ? 1 : strcmp(e, "intraqp") == 0 ? 2 : 0;
  const int qp_L = ((m_pad + 31) / 32 + 7) / 8 * 8;                  // rows per lane, multiple of 8
  const int qp_stride = 32 * qp_L + 8;
  const size_t qp_bytes = ((size_t)swk::kProfRows * qp_stride + 15) / 16 * 16;
  void* kintra_qp = nullptr;
  if (variant == 2 && qp_L <= 64) {
    void* pq = db->d_prof_qp;
    int rc = ensure(&pq, &db->prof_qp_cap, qp_bytes);
    db->d_prof_qp = (int8_t*)pq;
    if (rc) return rc;
    swk::k_profile<<<64, 256, 0, st>>>(db->d_query, qlen, db->d_matrix, db->d_prof_qp, qp_stride);
    CK(cudaGetLastError());
    nl++;
    switch (qp_L) {
      case 8: kintra_qp = (void*)swk::k_intra16_qp<8, true>; break;
      case 16: kintra_qp = (void*)swk::k_intra16_qp<16, true>; break;
      case 24: kintra_qp = (void*)swk::k_intra16_qp<24, true>; break;
      case 32: kintra_qp = (void*)swk::k_intra16_qp<32, true>; break;
      case 40: kintra_qp = (void*)swk::k_intra16_qp<40, true>; break;
      case 48: kintra_qp = (void*)swk::k_intra16_qp<48, true>; break;
      case 56: kintra_qp = (void*)swk::k_intra16_qp<56, true>; break;
      default: kintra_qp = (void*)swk::k_intra16_qp<64, true>; break;
    }
    CK(cudaFuncSetAttribute(kintra_qp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qp_bytes));
  }
  const int T = tile_rows_env();
  const int nt = threads_env(T == 32 ? 512 : 384);
  // the BIG instantiation (per-item slab choice) only when wide groups stay inter-task
  void* kern16 = T == 32 ? inter16_kernel_nt<32>(smem, nt, n_big > 0) : T == 48 ? inter16_kernel_nt<48>(smem, nt, n_big > 0)
               : inter16_kernel_nt<64>(smem, nt, n_big > 0);
  CK(cudaFuncSetAttribute(kern16, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(smem_bytes, 1)));
  const int intra_tr = m_pad <= 256 ? 8 : 16;   // rows per lane of the intra-task wavefront
  void* kintra = intra_tr == 8 ? (smem ? (void*)swk::k_intra16<8, true> : (void*)swk::k_intra16<8, false>)
                               : (smem ? (void*)swk::k_intra16<16, true> : (void*)swk::k_intra16<16, false>);
  CK(cudaFuncSetAttribute(kintra, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(smem_bytes, 1)));
  // int16x2 pass: the intra-task kernel (long groups, pair items) is launched
  // first and at once lets the inter-task kernel (all other groups) start beside
  // it (programmatic dependent launch on the same stream): its few CTAs reach
  // the SMs first, the persistent inter-task CTAs fill the rest, and the
  // inter-task kernel's last instruction waits for the intra-task grid, so
  // everything after it on the stream sees both.  Both take work longest-first
  // from their own counters.
  auto launch16 = [&](const uint2* words, const GroupDesc* groups, int n_groups_i, const int* n_groups_dev,
                      const int* pos_map, int n_long_r, int* counter_inter, int* counter_intra, int* score_out,
                      uint8_t* flag_out) -> int {
    // only the first-pass layout has big slabs: elsewhere wide groups go intra-task
    int cut_l = (n_groups_dev || variant == 1) ? std::min<int>(cut, (int)db->scratch_cols) : cut;
    if (!n_groups_dev) {
      const int64_t g0 = groups - db->d_groups;
      const auto& gc = db->group_ncols;
      n_long_r = (int)((gc.begin() + g0 + n_groups_i) - std::upper_bound(gc.begin() + g0, gc.begin() + g0 + n_groups_i, cut_l));
    }
    const bool any_long = n_long_r > 0;
    long long scols = db->scratch_cols;
    // the range's inter-task groups wider than a warp slab: the first items of its queue
    long long big_off = db->d_big ? (long long)(db->d_big - db->d_scratch) : 0;   // in uint2, same address space
    int n_big_r = 0;
    if (n_big && !n_groups_dev && variant != 1) {
      const int64_t g0 = groups - db->d_groups, g1 = g0 + n_groups_i;
      const auto& gc = db->group_ncols;
      n_big_r = (int)(std::upper_bound(gc.begin() + g0, gc.begin() + g1, cut) -
                      std::upper_bound(gc.begin() + g0, gc.begin() + g1, (int)db->scratch_cols));
      n_big_r = std::max(0, n_big_r);
    }
    void* kargs_inter[] = {(void*)&words, (void*)&groups, &n_groups_i, (void*)&n_groups_dev, (void*)&pos_map, &cut_l,
                           &db->d_prof, (void*)&m_pad, (void*)&stride, &alpha, &beta, (void*)&limit16, &db->d_scratch,
                           &scols, &counter_inter, &score_out, &flag_out, &big_off, &big_cols, &n_big_r};
    long long scols_intra = db->scratch_cols_intra;
    void* kargs_intra[] = {(void*)&words, (void*)&groups, &n_groups_i, (void*)&n_groups_dev, (void*)&pos_map, &cut_l,
                           &db->d_prof, (void*)&m_pad, (void*)&stride, &alpha, &beta, (void*)&limit16,
                           &db->d_scratch_intra, &scols_intra, &counter_intra, &score_out, &flag_out};
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(nt);
    cfg.dynamicSmemBytes = smem_bytes;
    cfg.stream = st;
    if (any_long) {
      // only as many CTAs as the pair items need (12 warps each): idle CTAs would
      // hold SMs the inter-task kernel could use
      const int64_t items = (int64_t)(n_groups_dev ? n_groups_i : n_long_r) * 32;
      const int grid_intra = (int)std::max<int64_t>(1, std::min<int64_t>(grid, (items + 11) / 12));
      if (kintra_qp && !n_groups_dev) {
        // f4 ablation: striped intra-task kernel (IntraQP) for the pair items
        void* kargs_qp[] = {(void*)&words, (void*)&groups, &n_groups_i, &cut_l, &db->d_prof_qp, (void*)&qp_stride,
                            &alpha, &beta, (void*)&limit16, &counter_intra, &score_out, &flag_out};
        CK(cudaLaunchKernel(kintra_qp, dim3(grid_intra), dim3(swk::kInterThreads), kargs_qp, qp_bytes, st));
      } else {
        CK(cudaLaunchKernel(kintra, dim3(grid_intra), dim3(swk::kInterThreads), kargs_intra, smem_bytes, st));
      }
      nl++;
      cfg.attrs = pdl;
      cfg.numAttrs = 1;
    }
    cfg.gridDim = dim3(grid);
    if (variant == 1 && !n_groups_dev) {
      // f4 ablation: InterSP score profile instead of the query profile (SW_VARIANT=intersp)
      void* kargs_sp[] = {(void*)&words, (void*)&groups, &n_groups_i, &cut_l, &db->d_query, (void*)&qlen,
                          (void*)&m_pad, &db->d_matrix, &alpha, &beta, (void*)&limit16, &db->d_scratch, &scols,
                          &counter_inter, &score_out, &flag_out};
      cfg.blockDim = dim3(swk::kInterThreads);
      cfg.dynamicSmemBytes = 0;
      CK(cudaLaunchKernelExC(&cfg, (void*)swk::k_inter16_sp, kargs_sp));
    } else {
      CK(cudaLaunchKernelExC(&cfg, kern16, kargs_inter));
    }
    nl++;
    return SW_OK;
  };
  // int8 first stage only when every biased byte fits
  const int bias = -std::min(0, smin);
  const bool stage8 = db->first_stage == 8 && beta <= 255 && smax + bias <= 255;
  db->last_first_stage = db->first_stage == 32 ? 32 : (stage8 ? 8 : 16);
  auto k32 = smem ? swk::k_list32<kTileRows, true> : swk::k_list32<kTileRows, false>;
  CK(cudaFuncSetAttribute(k32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(smem_bytes, 1)));
  // First pass + escalation over the groups [g0, g1) whose packed words sit at
  // wb + groups[g].base (the whole resident layout, or one streamed chunk).
  // Positions, scores and flags of the range start at g0 * 64.
  auto run_range = [&](const uint2* wb, int64_t g0, int64_t g1, int* cnt32, bool mark_ev2) -> int {
    const int64_t p0 = g0 * swk::kGroup, p1 = std::min<int64_t>(g1 * swk::kGroup, n);
    const int nr = (int)(p1 - p0);
    const GroupDesc* gr = db->d_groups + g0;
    int* sc = db->d_score_sorted + p0;
    const int* ls = db->d_len_sorted + p0;
    CK(cudaMemsetAsync(db->d_counters, 0, 8 * sizeof(int), st));
    if (db->first_stage != 32) {
      const int n_long_r = (int)((db->group_ncols.begin() + g1) -
                                 std::upper_bound(db->group_ncols.begin() + g0, db->group_ncols.begin() + g1, cut));
      uint8_t* fl = db->d_flag16 + p0;
      int rc = launch16(wb, gr, (int)(g1 - g0), nullptr, nullptr, n_long_r, db->d_counters + 0, db->d_counters + 6, sc,
                        fl);
      if (rc) return rc;
      if (mark_ev2) CK(cudaEventRecord(ev[2], st));
      // escalation 16 -> 32: rerun only the subjects flagged by the int16 pass (count read on device)
      rc = compact(fl, nr, db->d_list16, cnt32, nullptr);
      if (rc) return rc;
      k32<<<grid, swk::kInterThreads, smem_bytes, st>>>(wb, gr, db->d_list16, cnt32, 0, ls, db->d_prof, m_pad, stride,
                                                        alpha, beta, db->d_scratch, db->scratch_cols,
                                                        db->d_counters + 2, sc);
    } else {
      if (mark_ev2) CK(cudaEventRecord(ev[2], st));
      k32<<<grid, swk::kInterThreads, smem_bytes, st>>>(wb, gr, nullptr, nullptr, nr, ls, db->d_prof, m_pad, stride,
                                                        alpha, beta, db->d_scratch, db->scratch_cols,
                                                        db->d_counters + 2, sc);
    }
    CK(cudaGetLastError());
    nl++;
    return SW_OK;
  };
  if (db->n_inter > 0) {
    if (db->first_stage != 32) CK(cudaMemsetAsync(db->d_flag16, 0, (size_t)n, st));
    if (stage8) {
      const int limit8 = 255 - (smax + bias);
      swk::k_profile8b<<<64, 256, 0, st>>>(db->d_query, qlen, db->d_matrix, bias, db->d_prof8b, stride);
      CK(cudaMemsetAsync(db->d_flag8, 0, (size_t)n, st));
      auto k8 = smem ? swk::k_inter8<32, true> : swk::k_inter8<32, false>;
      CK(cudaFuncSetAttribute(k8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(smem_bytes, 1)));
      k8<<<grid, swk::kInterThreads, smem_bytes, st>>>(db->d_words, db->d_groups, (int)db->n_groups, db->d_prof8b,
                                                       m_pad, stride, alpha, beta, bias, limit8, db->d_scratch,
                                                       db->scratch_cols, db->d_counters + 0, db->d_score_sorted,
                                                       db->d_flag8);
      nl += 2;
      CK(cudaGetLastError());
      CK(cudaEventRecord(ev[2], st));
      // escalation 8 -> 16: compact, re-interleave the flagged subjects, int16 pass on the mini layout
      int rc = compact(db->d_flag8, n, db->d_list8, db->d_cnt + 0, db->d_cnt + 2);
      if (rc) return rc;
      const int nmm = (int)db->n_mini_max;
      swk::k_mini_sizes<<<std::min((nmm + 255) / 256, 4096), 256, 0, st>>>(db->d_list8, db->d_cnt + 0,
                                                                          db->d_len_sorted, nmm, db->d_mini_sizes);
      swk::k_scan_exclusive<<<1, swk::kScanBlock, 0, st>>>(db->d_mini_sizes, nmm, nullptr, nullptr);
      swk::k_mini_build<<<std::min((nmm + 7) / 8, 8192), 256, 0, st>>>(db->d_words, db->d_groups, db->d_list8,
                                                                      db->d_cnt + 0, db->d_len_sorted, db->d_mini_sizes,
                                                                      nmm, db->d_mgroups, db->d_mwords);
      nl += 3;
      CK(cudaGetLastError());
      rc = launch16(db->d_mwords, db->d_mgroups, nmm, db->d_cnt + 2, db->d_list8, nmm, db->d_counters + 4,
                    db->d_counters + 7, db->d_score_sorted, db->d_flag16);
      if (rc) return rc;
      rc = compact(db->d_flag16, n, db->d_list16, db->d_cnt + 1, nullptr);
      if (rc) return rc;
      k32<<<grid, swk::kInterThreads, smem_bytes, st>>>(
          db->d_words, db->d_groups, db->d_list16, db->d_cnt + 1, 0, db->d_len_sorted, db->d_prof,
          m_pad, stride, alpha, beta, db->d_scratch, db->scratch_cols, db->d_counters + 2,
          db->d_score_sorted);
      CK(cudaGetLastError());
      nl++;
    } else if (!db->host_resident) {
      int rc = run_range(db->d_words, 0, db->n_groups, db->d_cnt + 1, true);
      if (rc) return rc;
    } else {
      // f2: the packed words stay in pinned host memory; chunks of whole groups are
      // copied on the copy stream into two device buffers while the previous chunk
      // is aligned (double buffering; PAPER.md:55's chunk-by-chunk offload)
      CK(cudaEventRecord(ev[2], st));
      for (size_t c = 0; c < db->chunks.size(); c++) {
        const int b = (int)(c & 1);
        const int64_t g0 = db->chunks[c].first, g1 = db->chunks[c].second;
        const int64_t w0 = db->h_group_base[g0], w1 = db->h_group_base[g1];
        CK(cudaStreamWaitEvent(db->copy_stream, db->ev_consumed[b], 0));
        CK(cudaMemcpyAsync(db->d_chunk[b], db->h_words + w0, (size_t)(w1 - w0) * sizeof(uint2),
                           cudaMemcpyHostToDevice, db->copy_stream));
        CK(cudaEventRecord(db->ev_copied[b], db->copy_stream));
        CK(cudaStreamWaitEvent(st, db->ev_copied[b], 0));
        const uint2* wb = (const uint2*)((uintptr_t)db->d_chunk[b] - (uintptr_t)(w0 * (int64_t)sizeof(uint2)));
        int rc = run_range(wb, g0, g1, db->d_stream_cnt + c, false);
        if (rc) return rc;
        CK(cudaEventRecord(db->ev_consumed[b], st));
      }
    }
  } else {
    CK(cudaEventRecord(ev[2], st));
  }
  CK(cudaEventRecord(ev[3], st));

  // ---- stage (iv): scatter + exact top-k ----
  {
    int rc = rank_enqueue(db, db->d_score_sorted, d_scores, k, d_tk_ids, d_tk_scores, st, nl);
    if (rc) return rc;
  }
  CK(cudaEventRecord(ev[4], st));
  CK(cudaEventRecord(db->ev_done, st));
  db->n_searches++;
  db->launches += nl;
  return SW_OK;
}

int sw_search_async(sw_db* db, const uint8_t* query, int32_t qlen, const int8_t* matrix, int32_t alpha,
                    int32_t beta, int32_t k, int32_t* d_scores, int64_t* d_topk_ids,
                    int32_t* d_topk_scores, void* stream) {
  int smax = 0, smin = 0;
  int rc = validate_search(db, query, qlen, matrix, alpha, beta, k, &smax, &smin);
  if (rc) return rc;
  std::lock_guard<std::mutex> lock(db->mu);
  CK(cudaSetDevice(db->device));
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaStreamWaitEvent(st, db->ev_done, 0));   // serialise with the previous search on this handle
  return search_enqueue(db, query, qlen, matrix, alpha, beta, k, smax, smin, d_scores, (long long*)d_topk_ids,
                        d_topk_scores, st);
}

int sw_search(sw_db* db, const uint8_t* query, int32_t qlen, const int8_t* matrix, int32_t alpha,
              int32_t beta, int32_t k, int32_t* scores, int64_t* topk_ids, int32_t* topk_scores,
              sw_stats* stats) {
  const auto t0 = std::chrono::steady_clock::now();
  int smax = 0, smin = 0;
  int rc = validate_search(db, query, qlen, matrix, alpha, beta, k, &smax, &smin);
  if (rc) return rc;
  std::lock_guard<std::mutex> lock(db->mu);
  CK(cudaSetDevice(db->device));
  {
    if (db->topk_cap < k) {
      if (db->d_topk_ids) cudaFree(db->d_topk_ids);
      if (db->d_topk_scores) cudaFree(db->d_topk_scores);
      db->d_topk_ids = nullptr;
      db->d_topk_scores = nullptr;
      CK(cudaMalloc(&db->d_topk_ids, (size_t)k * sizeof(long long)));
      CK(cudaMalloc(&db->d_topk_scores, (size_t)k * sizeof(int)));
      db->topk_cap = k;
    }
  }
  cudaStream_t st = db->stream;
  rc = search_enqueue(db, query, qlen, matrix, alpha, beta, k, smax, smin, db->d_scores, db->d_topk_ids,
                      db->d_topk_scores, st);
  if (rc) return rc;
  if (scores && db->n_seqs)
    CK(cudaMemcpyAsync(scores, db->d_scores, db->n_seqs * sizeof(int), cudaMemcpyDeviceToHost, st));
  if (topk_ids) CK(cudaMemcpyAsync(topk_ids, db->d_topk_ids, (size_t)k * sizeof(long long), cudaMemcpyDeviceToHost, st));
  if (topk_scores) CK(cudaMemcpyAsync(topk_scores, db->d_topk_scores, (size_t)k * sizeof(int), cudaMemcpyDeviceToHost, st));
  int cnt[4] = {0};
  CK(cudaMemcpyAsync(cnt, db->d_cnt, sizeof cnt, cudaMemcpyDeviceToHost, st));
  std::vector<int> ccnt(db->chunks.size());
  if (db->host_resident && !ccnt.empty())
    CK(cudaMemcpyAsync(ccnt.data(), db->d_stream_cnt, ccnt.size() * sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (db->host_resident) {
    cnt[1] = 0;
    for (int c : ccnt) cnt[1] += c;
  }
  const auto t1 = std::chrono::steady_clock::now();
  if (stats) {
    memset(stats, 0, sizeof *stats);
    stats->cells = (int64_t)qlen * db->sum_len;
    stats->n_seqs = db->n_seqs;
    {
      int64_t n_intra = 0;
      for (int t = 0; t < db->last_n_long; t++) {
        const int64_t g = db->n_groups - 1 - t;
        n_intra += std::min<int64_t>(swk::kGroup, db->n_inter - g * swk::kGroup);
      }
      stats->n_intra = n_intra;
      stats->n_inter = db->n_inter - n_intra;
    }
    stats->n_rerun16 = db->last_first_stage == 8 ? cnt[0] : 0;
    stats->n_rerun32 = db->last_first_stage != 32 ? cnt[1] : 0;
    stats->seconds = std::chrono::duration<double>(t1 - t0).count();
    stats->gcups = stats->seconds > 0 ? (double)stats->cells / stats->seconds / 1e9 : 0.0;
    cudaEvent_t* ev = db->ev_ring[(db->n_searches - 1) % sw_db::kRing];
    float ms = 0;
    cudaEventElapsedTime(&ms, ev[0], ev[1]); stats->ms_profile = ms;
    cudaEventElapsedTime(&ms, ev[1], ev[2]); stats->ms_inter = ms;
    cudaEventElapsedTime(&ms, ev[2], ev[3]); stats->ms_rerun = ms;
    cudaEventElapsedTime(&ms, ev[3], ev[4]); stats->ms_finalize = ms;
    stats->first_stage = db->last_first_stage;
  }
  return SW_OK;
}


// ---- f1: batched queries, two per pass ----
constexpr int kMaxPairStride = kMaxSmemProfile / (4 * swk::kProfRows);   // words per pair-profile row

static int pair_fits(int ma, int mb) {
  const int m_pad = (std::max(ma, mb) + 7) / 8 * 8;
  return (m_pad + 31) / 32 * 32 + 1 <= kMaxPairStride;
}

// Align queries a and b against every subject in ONE inter-task pass (lo/hi
// halves of int16x2 = the two queries, one subject per lane), then rerun each
// query's saturated subjects in int32.  Sorted-order scores land in
// d_score_sorted (a) and d_score_sorted2 (b).
static int pair_enqueue(sw_db* db, const uint8_t* qa, int ma, const uint8_t* qb, int mb, const int8_t* matrix,
                        int alpha, int beta, int smax, cudaStream_t st, int64_t& nl) {
  const int n = (int)db->n_seqs;
  const int m_pad = (std::max(ma, mb) + 7) / 8 * 8;
  const int stride2 = (m_pad + 31) / 32 * 32 + 1;                 // odd word stride: conflict-free LDS.32
  const int mpa = (ma + 7) / 8 * 8, mpb = (mb + 7) / 8 * 8;
  const int sa = (mpa + 31) / 32 * 32 + 8, sb = (mpb + 31) / 32 * 32 + 8;
  const size_t pa = ((size_t)swk::kProfRows * sa + 15) / 16 * 16, pb = ((size_t)swk::kProfRows * sb + 15) / 16 * 16;
  const size_t p2 = (size_t)swk::kProfRows * stride2 * sizeof(uint32_t);
  {
    const size_t need = (size_t)ma + mb + 1024;
    if (db->stage_cap < need) {
      if (db->h_stage) { cudaEventSynchronize(db->ev_stage); cudaFreeHost(db->h_stage); db->h_stage = nullptr; }
      CK(cudaHostAlloc(&db->h_stage, need, cudaHostAllocDefault));
      db->stage_cap = need;
    } else {
      CK(cudaEventSynchronize(db->ev_stage));
    }
    memcpy(db->h_stage, matrix, 1024);
    memcpy(db->h_stage + 1024, qa, ma);
    memcpy(db->h_stage + 1024 + ma, qb, mb);
    size_t qcap = (size_t)db->query_cap;
    void* v = db->d_query;
    int rc = ensure(&v, &qcap, (size_t)ma + mb);
    db->d_query = (uint8_t*)v;
    db->query_cap = (int)qcap;
    if (rc) return rc;
    v = db->d_prof;
    rc = ensure(&v, &db->prof_cap, pa);
    db->d_prof = (int8_t*)v;
    if (rc) return rc;
    v = db->d_prof_b;
    rc = ensure(&v, &db->prof_b_cap, pb);
    db->d_prof_b = (int8_t*)v;
    if (rc) return rc;
    v = db->d_prof2;
    rc = ensure(&v, &db->prof2_cap, p2);
    db->d_prof2 = (uint32_t*)v;
    if (rc) return rc;
    if (!db->d_score_sorted2) CK(cudaMalloc(&db->d_score_sorted2, std::max<int64_t>(n, 1) * sizeof(int)));
    if (!db->d_flag_b) CK(cudaMalloc(&db->d_flag_b, std::max<int64_t>(n, 1)));
    CK(cudaMemcpyAsync(db->d_matrix, db->h_stage, 1024, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(db->d_query, db->h_stage + 1024, (size_t)ma + mb, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(db->ev_stage, st));
  }
  const uint8_t* dqa = db->d_query;
  const uint8_t* dqb = db->d_query + ma;
  swk::k_profile<<<64, 256, 0, st>>>(dqa, ma, db->d_matrix, db->d_prof, sa);
  swk::k_profile<<<64, 256, 0, st>>>(dqb, mb, db->d_matrix, db->d_prof_b, sb);
  swk::k_profile_pair<<<64, 256, 0, st>>>(dqa, ma, dqb, mb, db->d_matrix, db->d_prof2, stride2);
  CK(cudaMemsetAsync(db->d_counters, 0, 8 * sizeof(int), st));
  CK(cudaMemsetAsync(db->d_cnt, 0, 4 * sizeof(int), st));
  CK(cudaMemsetAsync(db->d_flag16, 0, (size_t)std::max(n, 1), st));
  CK(cudaMemsetAsync(db->d_flag_b, 0, (size_t)std::max(n, 1), st));
  nl += 3;
  const int grid = db->num_sms;
  const int limit16 = 32767 - smax;
  if (n > 0) {
    CK(cudaFuncSetAttribute(swk::k_multi16<kTileRows>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p2));
    swk::k_multi16<kTileRows><<<grid, swk::kInterThreads, p2, st>>>(
        db->d_words, db->d_groups, (int)db->n_groups, db->d_prof2, m_pad, stride2, alpha, beta, limit16,
        db->d_scratch, db->scratch_cols, db->d_counters + 0, db->d_score_sorted, db->d_score_sorted2,
        db->d_flag16, db->d_flag_b);
    CK(cudaGetLastError());
    nl++;
    const int nb_scan = std::max(1, (n + swk::kScanBlock - 1) / swk::kScanBlock);
    for (int which = 0; which < 2; which++) {
      uint8_t* flag = which ? db->d_flag_b : db->d_flag16;
      int* cnt = db->d_cnt + (which ? 3 : 1);
      swk::k_flag_count<<<nb_scan, swk::kScanBlock, 0, st>>>(flag, n, db->d_block_counts);
      swk::k_scan_exclusive<<<1, swk::kScanBlock, 0, st>>>(db->d_block_counts, nb_scan, cnt, nullptr);
      swk::k_flag_scatter<<<nb_scan, swk::kScanBlock, 0, st>>>(flag, n, db->d_block_counts, db->d_list16);
      const int mp = which ? mpb : mpa, sw_ = which ? sb : sa;
      const size_t pbytes = which ? pb : pa;
      const bool smem = pbytes <= (size_t)kMaxSmemProfile;
      auto k32 = smem ? swk::k_list32<kTileRows, true> : swk::k_list32<kTileRows, false>;
      CK(cudaFuncSetAttribute(k32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(smem ? pbytes : 0, 1)));
      k32<<<grid, swk::kInterThreads, smem ? pbytes : 0, st>>>(
          db->d_words, db->d_groups, db->d_list16, cnt, 0, db->d_len_sorted, which ? db->d_prof_b : db->d_prof, mp,
          sw_, alpha, beta, db->d_scratch, db->scratch_cols, db->d_counters + (which ? 5 : 2),
          which ? db->d_score_sorted2 : db->d_score_sorted);
      CK(cudaGetLastError());
      nl += 4;
    }
  }
  return SW_OK;
}

int sw_search_batch(sw_db* db, const uint8_t* queries, const int64_t* qoffsets, const int32_t* qlens,
                    int32_t n_queries, const int8_t* matrix, int32_t alpha, int32_t beta, int32_t k,
                    int32_t* scores, int64_t* topk_ids, int32_t* topk_scores, sw_stats* stats) {
  const auto t0 = std::chrono::steady_clock::now();
  if (!db) return fail(SW_EINVAL, "db is NULL");
  if (n_queries < 1 || !queries || !qoffsets || !qlens) return fail(SW_EINVAL, "need n_queries >= 1 and non-NULL query arrays");
  if (db->host_resident)
    return fail(SW_EINVAL, "sw_search_batch needs a device-resident database (residency 0); use sw_search per query");
  int smax = 0, smin = 0;
  for (int q = 0; q < n_queries; q++) {
    if (qoffsets[q] < 0) return fail(SW_EINVAL, "query %d: negative offset", q);
    int rc = validate_search(db, queries + qoffsets[q], qlens[q], matrix, alpha, beta, k, &smax, &smin);
    if (rc) {
      std::string m = g_last_error;
      return fail(rc, "query %d: %s", q, m.c_str());
    }
  }
  std::lock_guard<std::mutex> lock(db->mu);
  CK(cudaSetDevice(db->device));
  cudaStream_t st = db->stream;
  if (db->topk_cap < k) {
    if (db->d_topk_ids) cudaFree(db->d_topk_ids);
    if (db->d_topk_scores) cudaFree(db->d_topk_scores);
    db->d_topk_ids = nullptr;
    db->d_topk_scores = nullptr;
    CK(cudaMalloc(&db->d_topk_ids, (size_t)k * sizeof(long long)));
    CK(cudaMalloc(&db->d_topk_scores, (size_t)k * sizeof(int)));
    db->topk_cap = k;
  }
  const int64_t n = db->n_seqs;
  // queries whose pair profile fits shared memory are paired by length; the rest run singly
  std::vector<int> order;
  for (int q = 0; q < n_queries; q++)
    if (pair_fits(qlens[q], qlens[q])) order.push_back(q);
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return qlens[x] > qlens[y]; });
  if (order.size() % 2) order.push_back(-1);   // odd one out runs singly
  for (int q = 0; q < n_queries; q++)
    if (!pair_fits(qlens[q], qlens[q])) { order.push_back(q); order.push_back(-1); }
  const int n_slots = (int)order.size();
  std::vector<int> cnt_host(4 * (size_t)n_slots, 0);
  int64_t nl = 0, n_rerun32 = 0, n_pairs = 0;
  auto fetch = [&](int q, const int* score_sorted) -> int {
    int rc = rank_enqueue(db, score_sorted, db->d_scores, k, db->d_topk_ids, db->d_topk_scores, st, nl);
    if (rc) return rc;
    if (scores && n) CK(cudaMemcpyAsync(scores + (size_t)q * n, db->d_scores, n * sizeof(int), cudaMemcpyDeviceToHost, st));
    if (topk_ids) CK(cudaMemcpyAsync(topk_ids + (size_t)q * k, db->d_topk_ids, (size_t)k * sizeof(long long), cudaMemcpyDeviceToHost, st));
    if (topk_scores) CK(cudaMemcpyAsync(topk_scores + (size_t)q * k, db->d_topk_scores, (size_t)k * sizeof(int), cudaMemcpyDeviceToHost, st));
    return SW_OK;
  };
  for (int t = 0; t < n_slots; t += 2) {
    const int a = order[t];
    const int b = order[t + 1];
    if (a >= 0 && b >= 0) {
      int rc = pair_enqueue(db, queries + qoffsets[a], qlens[a], queries + qoffsets[b], qlens[b], matrix, alpha, beta,
                            smax, st, nl);
      if (rc) return rc;
      CK(cudaMemcpyAsync(&cnt_host[4 * (size_t)t], db->d_cnt, 4 * sizeof(int), cudaMemcpyDeviceToHost, st));
      if ((rc = fetch(a, db->d_score_sorted))) return rc;
      if ((rc = fetch(b, db->d_score_sorted2))) return rc;
      n_pairs++;
    } else {
      for (int q : {a, b}) {
        if (q < 0) continue;
        int rc = search_enqueue(db, queries + qoffsets[q], qlens[q], matrix, alpha, beta, k, smax, smin, db->d_scores,
                                db->d_topk_ids, db->d_topk_scores, st);
        if (rc) return rc;
        if (scores && n) CK(cudaMemcpyAsync(scores + (size_t)q * n, db->d_scores, n * sizeof(int), cudaMemcpyDeviceToHost, st));
        if (topk_ids) CK(cudaMemcpyAsync(topk_ids + (size_t)q * k, db->d_topk_ids, (size_t)k * sizeof(long long), cudaMemcpyDeviceToHost, st));
        if (topk_scores) CK(cudaMemcpyAsync(topk_scores + (size_t)q * k, db->d_topk_scores, (size_t)k * sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        int c[4];
        CK(cudaMemcpy(c, db->d_cnt, sizeof c, cudaMemcpyDeviceToHost));
        n_rerun32 += c[1];
      }
    }
    CK(cudaStreamSynchronize(st));   // cnt_host (pageable) and the staging buffer are reused per pair
  }
  CK(cudaEventRecord(db->ev_done, st));
  CK(cudaStreamSynchronize(st));
  for (int t = 0; t < n_slots; t += 2) n_rerun32 += cnt_host[4 * (size_t)t + 1] + cnt_host[4 * (size_t)t + 3];
  db->launches += nl;
  const auto t1 = std::chrono::steady_clock::now();
  if (stats) {
    memset(stats, 0, sizeof *stats);
    int64_t qsum = 0;
    for (int q = 0; q < n_queries; q++) qsum += qlens[q];
    stats->cells = qsum * db->sum_len;
    stats->n_seqs = n;
    stats->n_inter = n;
    stats->n_rerun32 = n_rerun32;
    stats->seconds = std::chrono::duration<double>(t1 - t0).count();
    stats->gcups = stats->seconds > 0 ? (double)stats->cells / stats->seconds / 1e9 : 0.0;
    stats->first_stage = 16;
    stats->reserved[0] = (int32_t)n_pairs;   // query pairs aligned in one pass
  }
  return SW_OK;
}

// ---- f3: traceback of optimal alignments for chosen subjects ----
constexpr int kAlignTR = 8;                        // query rows per lane of the traceback wavefront
constexpr int64_t kAlignWorkspace = 1LL << 30;     // direction bytes aligned at once (soft cap)

int sw_align(sw_db* db, const uint8_t* query, int32_t qlen, const int8_t* matrix, int32_t alpha, int32_t beta,
             const int64_t* subjects, int32_t n, sw_alignment* out, char* ops, int64_t ops_cap) {
  int smax = 0, smin = 0;
  int rc = validate_search(db, query, qlen, matrix, alpha, beta, 1, &smax, &smin);
  if (rc) return rc;
  if (n < 0) return fail(SW_EINVAL, "sw_align: n must be >= 0 (got %d)", n);
  if (n == 0) return SW_OK;
  if (!subjects || !out || !ops) return fail(SW_EINVAL, "sw_align: subjects/out/ops must be non-NULL");
  for (int32_t t = 0; t < n; t++)
    if (subjects[t] < 0 || subjects[t] >= db->n_seqs)
      return fail(SW_EINVAL, "sw_align: subjects[%d] = %lld outside [0, %lld)", t, (long long)subjects[t],
                  (long long)db->n_seqs);
  std::lock_guard<std::mutex> lock(db->mu);
  CK(cudaSetDevice(db->device));
  cudaStream_t st = db->stream;
  CK(cudaStreamWaitEvent(st, db->ev_done, 0));
  const int nseq = (int)db->n_seqs;
  if (!db->d_inv) {
    CK(cudaMalloc(&db->d_inv, (size_t)nseq * sizeof(int)));
    swk::k_inverse_perm<<<std::min((nseq + 255) / 256, db->num_sms * 8), 256, 0, st>>>(db->d_perm, nseq, db->d_inv);
    CK(cudaGetLastError());
    db->launches++;
  }
  // ---- locate the subjects in the packed layout; their lengths size everything ----
  const int m_pad = (qlen + 7) / 8 * 8;
  const int stride = (m_pad + 31) / 32 * 32 + 8;
  const size_t prof_bytes = ((size_t)swk::kProfRows * stride + 15) / 16 * 16;
  auto ws = [&](int k, size_t bytes) -> void* {
    return ensure(&db->aw[k], &db->aw_cap[k], std::max<size_t>(bytes, 16)) == SW_OK ? db->aw[k] : nullptr;
  };
  long long* d_idx = (long long*)ws(0, (size_t)n * sizeof(long long));
  swk::AlignJob* d_jobs = (swk::AlignJob*)ws(1, (size_t)n * sizeof(swk::AlignJob));
  int* d_res = (int*)ws(2, (size_t)n * 6 * sizeof(int));
  uint8_t* d_q = (uint8_t*)ws(3, (size_t)qlen);
  int8_t* d_M = (int8_t*)ws(4, 1024);
  int8_t* d_prof = (int8_t*)ws(5, prof_bytes);
  if (!d_idx || !d_jobs || !d_res || !d_q || !d_M || !d_prof) return SW_ENOMEM;
  CK(cudaMemcpyAsync(d_idx, subjects, (size_t)n * sizeof(long long), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_q, query, (size_t)qlen, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_M, matrix, 1024, cudaMemcpyHostToDevice, st));
  swk::k_profile<<<64, 256, 0, st>>>(d_q, qlen, d_M, d_prof, stride);
  swk::k_align_locate<<<(n + 127) / 128, 128, 0, st>>>(d_idx, n, db->d_inv, db->d_len_sorted, db->d_groups, d_jobs);
  CK(cudaGetLastError());
  db->launches += 2;
  std::vector<swk::AlignJob> jobs(n);
  CK(cudaMemcpyAsync(jobs.data(), d_jobs, (size_t)n * sizeof(swk::AlignJob), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  int64_t need = 0;
  for (int32_t t = 0; t < n; t++) need += (int64_t)qlen + jobs[t].n;
  if (ops_cap < need)
    return fail(SW_EINVAL, "sw_align: ops_cap %lld too small, need %lld bytes", (long long)ops_cap, (long long)need);
  char* d_ops = (char*)ws(8, (size_t)need);
  char* d_tmp = (char*)ws(9, (size_t)need);
  if (!d_ops || !d_tmp) return SW_ENOMEM;
  // ---- batches of jobs whose direction matrices fit the workspace ----
  const int64_t rows_blocks = m_pad / kAlignTR;
  int64_t ops_off = 0;
  for (int32_t t = 0; t < n; t++) {
    jobs[t].ops = ops_off;
    jobs[t].tmp = ops_off;
    ops_off += (int64_t)qlen + jobs[t].n;
  }
  const uint2* words_dev = db->d_words;
  if (db->host_resident) {   // streamed database: read the few hits' words from mapped pinned memory
    void* p = nullptr;
    CK(cudaHostGetDevicePointer(&p, db->h_words, 0));
    words_dev = (const uint2*)p;
  }
  const size_t prof_smem = prof_bytes <= (size_t)kMaxSmemProfile ? prof_bytes : 0;
  CK(cudaFuncSetAttribute(swk::k_align<kAlignTR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)std::max<size_t>(prof_smem, 1)));
  int64_t ws_cap = kAlignWorkspace;
  if (const char* e = getenv("SW_ALIGN_WORKSPACE")) ws_cap = std::max<int64_t>(4, atoll(e));   // tests: force batching
  for (int32_t t0 = 0; t0 < n;) {
    int32_t t1 = t0;
    int64_t dsz = 0, bsz = 0;
    while (t1 < n) {
      const int64_t d = rows_blocks * jobs[t1].n, b = 2 * (int64_t)jobs[t1].n;
      if (t1 > t0 && (dsz + d) * 4 > ws_cap) break;
      jobs[t1].dir = dsz;
      jobs[t1].bnd = bsz;
      dsz += d;
      bsz += b;
      t1++;
    }
    uint32_t* d_dir = (uint32_t*)ws(6, (size_t)dsz * sizeof(uint32_t));
    int2* d_bnd = (int2*)ws(7, (size_t)bsz * sizeof(int2));
    if (!d_dir || !d_bnd) return SW_ENOMEM;
    CK(cudaMemcpyAsync(d_jobs + t0, jobs.data() + t0, (size_t)(t1 - t0) * sizeof(swk::AlignJob),
                       cudaMemcpyHostToDevice, st));
    swk::k_align<kAlignTR><<<t1 - t0, 32 * swk::kAlignWarps, prof_smem, st>>>(words_dev, d_jobs + t0, t1 - t0, d_prof, (int)prof_smem,
                                                           stride, qlen, m_pad, alpha, beta, d_dir, d_bnd, d_ops,
                                                           d_tmp, d_res + 6 * t0);
    CK(cudaGetLastError());
    db->launches++;
    CK(cudaStreamSynchronize(st));   // the workspace is reused by the next batch
    t0 = t1;
  }
  std::vector<int> res((size_t)n * 6);
  CK(cudaMemcpyAsync(res.data(), d_res, res.size() * sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(ops, d_ops, (size_t)need, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int32_t t = 0; t < n; t++)
    if (res[6 * t] < 0)
      return fail(SW_EINTERNAL, "sw_align: traceback of subject %lld failed (device pipeline stalled or "
                  "inconsistent direction codes)", (long long)subjects[t]);
  for (int32_t t = 0; t < n; t++) {
    sw_alignment& a = out[t];
    a.subject = subjects[t];
    a.score = res[6 * t];
    a.q_begin = res[6 * t + 1];
    a.q_end = res[6 * t + 2];
    a.s_begin = res[6 * t + 3];
    a.s_end = res[6 * t + 4];
    a.n_ops = res[6 * t + 5];
    a.reserved = 0;
    a.ops_offset = jobs[t].ops;
  }
  return SW_OK;
}

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
