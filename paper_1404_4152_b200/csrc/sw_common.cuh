// sw_common.cuh -- constants, the group descriptor, PRMT/profile/residue helpers, the query profiles, shared pieces of the persistent kernels
//
// The sm_100a device code of the Smith-Waterman database search (overview).
//
// Every kernel computes (part of) Eq. 1 of PAPER.md:31-35 (§II.A):
//   H(i,j) = max{0, H(i-1,j-1) + fsbt(q_i, s_j), E(i,j), F(i,j)}
//   E(i,j) = max{E(i-1,j) - alpha, H(i-1,j) - beta}
//   F(i,j) = max{F(i,j-1) - alpha, H(i,j-1) - beta}
// with E and F clamped at 0 (exact: DESIGN.md §"Clamped gaps", SURVEY.md
// Appendix B1), in linear space.  i runs over the query
// (rows, held in registers per tile), j over the subject (columns, streamed).
//
// Inter-task model: one lane aligns one pair of
// length-sorted subjects, packed as the lo/hi halves of int16x2 registers and
// updated with Blackwell DPX instructions (VIADDMNMX/VIMNMX3 .S16x2).  The
// 16-bit pass flags any subject whose running max could have wrapped
// (DESIGN.md §"Saturation"); flagged subjects are re-aligned in int32.
// The first pass is k_inter16 (sw_int16.cuh: 48-row register tiles, tile-edge
// rows in per-warp global slabs); k_inter16_pipe (sw_pipe.cuh, an option) runs
// the query tiles of a group on consecutive warps of a CTA and passes the
// tile-edge rows through shared-memory rings instead.
// Headers: sw_common (this), sw_int16 (first pass, intra-task wavefront),
// sw_pipe (pipelined first pass), sw_int8, sw_int32 (reruns), sw_multi (f1),
// sw_escalate (compaction), sw_rank (a6), sw_align (f3), sw_ablation (f4).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace swk {

constexpr int kGroup = 64;           // subjects per interleaved group (32 lanes x lo/hi)
constexpr int kResPerWord = 6;       // 5-bit residue codes per 32-bit word
constexpr int kDummy = 24;           // padding code, scores 0
constexpr int kNumCodes = 24;        // real residue codes 0..23
constexpr int kProfRows = 25;        // profile rows: codes 0..23 + DUMMY
constexpr uint32_t kDummyWord = 24u | (24u << 5) | (24u << 10) | (24u << 15) | (24u << 20) | (24u << 25);
constexpr int kInterThreads = 384;   // 12 warps, one persistent CTA per SM (default)
constexpr int kMaxThreads = 512;     // scratch is sized for up to 16 resident warps per SM

struct GroupDesc {
  long long base;   // first uint2 of the group in the packed word array
  int ncols;        // longest member (sorted order: the last member)
  int count;        // members (64 except in the last group)
};

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

// (byte rr of a, byte rr of b) -> sign-extended s16x2 pair; selector nibble bit 3
// replicates the sign of the selected byte (PTX prmt default mode).
__host__ __device__ constexpr uint32_t sel_pair(int rr) {
  return (uint32_t)(rr | ((rr | 8) << 4) | ((4 + rr) << 8) | (((4 + rr) | 8) << 12));
}
// byte rr of a -> sign-extended int32
__host__ __device__ constexpr uint32_t sel_one(int rr) {
  return (uint32_t)(rr | ((rr | 8) << 4) | ((rr | 8) << 8) | ((rr | 8) << 12));
}

// Dynamic shared memory holds the query profile when it fits (SMEM = true).
// Re-deriving the base inside non-inlined helpers keeps their loads LDS.
template <bool SMEM>
__device__ __forceinline__ const int8_t* prof_base(const int8_t* gprof) {
  if constexpr (SMEM) {
    extern __shared__ __align__(16) int8_t dyn_smem[];
    return dyn_smem;
  } else {
    return gprof;
  }
}

__host__ __device__ constexpr uint32_t pack2(int v) {
  return ((uint32_t)v & 0xffffu) | (((uint32_t)v & 0xffffu) << 16);
}

// The gap penalties of every experiment in the paper, "10-2k" (PAPER.md:164,
// §IV.A; reading R4: alpha = 2, beta = 12).  The first-pass kernel has an
// instance with them as immediates (GAPS = 1): the two packed penalties are
// then instruction operands instead of registers, which frees two registers
// and the operand reads of 3 of the 6.5 cell-update instructions per row --
// measured 3.5 % more cells/s on C2 and C5.  Any other (alpha, beta) runs the
// GAPS = 0 instance with the same arithmetic.
constexpr int kFixedAlpha = 2, kFixedBeta = 12;

// ---------------------------------------------------------------------------
// (i) query profile (PAPER.md:55 stage (i); §III.B.2): row r of the
// profile holds fsbt(q_i, r) for every query position i; int8, one row per
// residue code, DUMMY row and padded query positions are 0.
// ---------------------------------------------------------------------------
// Blocked profile of the intra-task wavefront: residue row r holds nblk blocks
// of 16 bytes; block b = fsbt(q_i, r) for query rows i = b*TR .. b*TR+TR-1
// (0 past the query and in the unused bytes).  Row stride = nblk * 16 bytes.
__global__ void k_profile_blk(const uint8_t* __restrict__ q, int m, const int8_t* __restrict__ M,
                              int8_t* __restrict__ profb, int tr, int nblk) {
  const int row = nblk * 16, total = kProfRows * row;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int r = t / row, rem = t - r * row, b = rem >> 4, k = rem & 15, i = b * tr + k;
    int8_t v = 0;
    if (k < tr && i < m && r < kNumCodes) v = M[q[i] * 32 + r];
    profb[t] = v;
  }
}

__global__ void k_profile(const uint8_t* __restrict__ q, int m, const int8_t* __restrict__ M,
                          int8_t* __restrict__ prof, int stride) {
  const int total = kProfRows * stride;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int r = t / stride, i = t - r * stride;
    int8_t v = 0;
    if (i < m && r < kNumCodes) v = M[q[i] * 32 + r];
    prof[t] = v;
  }
}


// Stage (i) of a search in one launch: the query profile, the blocked profile of
// the intra-task wavefront (both as above) and the zeroing of the search's
// work-queue counters (nz ints), which were two kernels and two memsets.
__global__ void k_profiles(const uint8_t* __restrict__ q, int m, const int8_t* __restrict__ M,
                           int8_t* __restrict__ prof, int stride, int8_t* __restrict__ profb, int tr, int nblk,
                           int* __restrict__ zero_a, int nza, int* __restrict__ zero_b, int nzb,
                           uint8_t* __restrict__ zero_c = nullptr, int nzc = 0) {
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  if (t0 < nza) zero_a[t0] = 0;
  if (t0 < nzb) zero_b[t0] = 0;
  for (int t = t0; t < nzc; t += nt) zero_c[t] = 0;   // small databases: the flag bytes (no memset launch)
  const int total = kProfRows * stride;
  for (int t = t0; t < total; t += nt) {
    const int r = t / stride, i = t - r * stride;
    int8_t v = 0;
    if (i < m && r < kNumCodes) v = M[q[i] * 32 + r];
    prof[t] = v;
  }
  const int row = nblk * 16, totb = kProfRows * row;
  for (int t = t0; t < totb; t += nt) {
    const int r = t / row, rem = t - r * row, b = rem >> 4, k = rem & 15, i = b * tr + k;
    int8_t v = 0;
    if (k < tr && i < m && r < kNumCodes) v = M[q[i] * 32 + r];
    profb[t] = v;
  }
}

struct ResCursor {
  uint2 w, wn;
  int c, wi, nwords;
  const uint2* base;   // word wi of this lane at base[wi * 32]
  __device__ __forceinline__ void init(const uint2* b, int nw) {
    base = b;
    nwords = nw;
    c = 0;
    wi = 0;
    const uint2 dd = make_uint2(kDummyWord, kDummyWord);
    w = nw > 0 ? __ldg(b) : dd;
    wn = nw > 1 ? __ldg(b + 32) : dd;
  }
  __device__ __forceinline__ uint32_t lo() const { return (w.x >> (5u * (uint32_t)c)) & 31u; }
  __device__ __forceinline__ uint32_t hi() const { return (w.y >> (5u * (uint32_t)c)) & 31u; }
  __device__ __forceinline__ void next() {
    if (++c == kResPerWord) {
      c = 0;
      ++wi;
      w = wn;
      const uint2 dd = make_uint2(kDummyWord, kDummyWord);
      wn = (wi + 1 < nwords) ? __ldg(base + (wi + 1) * 32) : dd;
    }
  }
};


__device__ __forceinline__ uint2 res_word(const uint2* __restrict__ lw, int c, int nwords) {
  const int w = (int)(__umulhi((unsigned)c, 0xAAAAAAABu) >> 2);   // c / 6
  return w < nwords ? __ldg(lw + (long long)w * 32) : make_uint2(kDummyWord, kDummyWord);
}
__device__ __forceinline__ int res_shift(int c) {
  return 5 * (c - 6 * (int)(__umulhi((unsigned)c, 0xAAAAAAABu) >> 2));
}


__device__ __forceinline__ void load_profile_smem(int8_t* sprof, const int8_t* __restrict__ gprof,
                                                  int stride) {
  const int n16 = (kProfRows * stride + 15) / 16;   // buffers are padded to 16 B
  const uint4* src = reinterpret_cast<const uint4*>(gprof);
  uint4* dst = reinterpret_cast<uint4*>(sprof);
  for (int t = threadIdx.x; t < n16; t += blockDim.x) dst[t] = __ldg(src + t);
  __syncthreads();
}

// (ii) int16x2 pass (first pass, or the rerun of int8-flagged subjects on a
// mini-group layout with pos_map).  Persistent: one CTA per SM; each warp pulls work
// items longest-first from an atomic counter (the device analogue of the
// paper's guided OpenMP schedule over length-sorted sequence profiles,
// PAPER.md:63-65, 73).  Items [0, 32*n_long) are single PAIRS of the n_long
// longest groups, aligned by the intra-task wavefront; the rest are whole
// 64-subject groups, aligned inter-task (one pair per lane).
__device__ __forceinline__ void emit_pair(uint32_t hmax, int g, int slot, int count, int limit,
                                          const int* __restrict__ pos_map, int* __restrict__ score_sorted,
                                          uint8_t* __restrict__ flag) {
  const int lo = (int)(int16_t)(hmax & 0xffffu), hi = (int)(int16_t)(hmax >> 16);
  if (slot < count) {
    const int pos = pos_map ? pos_map[g * kGroup + slot] : g * kGroup + slot;
    score_sorted[pos] = lo;
    if (lo > limit || lo < 0) flag[pos] = 1;
  }
  if (slot + 1 < count) {
    const int pos = pos_map ? pos_map[g * kGroup + slot + 1] : g * kGroup + slot + 1;
    score_sorted[pos] = hi;
    if (hi > limit || hi < 0) flag[pos] = 1;
  }
}

constexpr int kIntraRows = 16;   // rows per lane in the intra-task wavefront
constexpr int kIntra32Cols = 512; // int32 reruns: longer subjects go one per warp (wavefront)
constexpr int kMaxInterCols = 6144; // boundary-slab columns per warp; longer groups go intra-task

// First group (ascending ncols) whose ncols exceeds `cut`: groups at and above it
// go to the intra-task kernel.  Same answer in both kernels.
__device__ __forceinline__ int split_groups(const GroupDesc* __restrict__ groups, int n_groups, int cut) {
  int lo = 0, hi = n_groups;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (groups[mid].ncols > cut) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// Inter-task pass over groups [0, split): whole 64-subject groups, longest first.

}  // namespace swk
