// sw_kernels.cuh — sm_100a device code of the Smith-Waterman database search.
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
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace swk {

constexpr int kGroup = 64;           // subjects per interleaved group (32 lanes x lo/hi)
constexpr int kResPerWord = 6;       // 5-bit residue codes per 32-bit word
constexpr int kDummy = 24;           // padding code, scores 0
constexpr int kNumCodes = 24;        // real residue codes 0..23
constexpr int kProfRows = 25;        // profile rows: codes 0..23 + DUMMY
constexpr uint32_t kDummyWord = 24u | (24u << 5) | (24u << 10) | (24u << 15) | (24u << 20) | (24u << 25);
constexpr int kInterThreads = 384;   // 12 warps, one persistent CTA per SM

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

__device__ __forceinline__ uint32_t pack2(int v) {
  const uint32_t h = (uint32_t)v & 0xffffu;
  return h | (h << 16);
}

// ---------------------------------------------------------------------------
// (i) query profile (PAPER.md:55 stage (i); §III.B.2): row r of the
// profile holds fsbt(q_i, r) for every query position i; int8, one row per
// residue code, DUMMY row and padded query positions are 0.
// ---------------------------------------------------------------------------
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

// ---------------------------------------------------------------------------
// int16x2 tile: rows [i0, i0+R) of the query against all columns of one pair
// of subjects.  Registers: H[r] = H(i0+r, j-1), F[r] = F(i0+r, j); e flows
// down the rows of the current column.  bnd[j] carries (E(i0,j), H(i0-1,j))
// in and (E(i0+R,j), H(i0+R-1,j)) out between tiles (the paper's "tiled SW
// computation").
// Per row: 2 VIADD.16x2 (fma-side pipe) + VIMNMX3 + 2 VIADDMNMX.RELU + 1/2
// VIMNMX3 + PRMT (alu pipe) for two cells.
// ---------------------------------------------------------------------------
template <int R>
__device__ __forceinline__ void tile16(const uint2* __restrict__ gw, int ncols,
                                       const int8_t* __restrict__ prof, int stride, int i0,
                                       uint2* __restrict__ bnd, bool first, bool last,
                                       uint32_t na2, uint32_t nb2, uint32_t& hmax, int lane) {
  uint32_t H[R], F[R];
#pragma unroll
  for (int r = 0; r < R; r++) { H[r] = 0u; F[r] = 0u; }
  if (ncols <= 0) return;
  const int nwords = (ncols + kResPerWord - 1) / kResPerWord;
  uint2 res = __ldg(gw + lane);
  uint2 res_nx = nwords > 1 ? __ldg(gw + 32 + lane) : res;
  uint2 bc = first ? make_uint2(0u, 0u) : bnd[lane];
  uint32_t htop_prev = 0u;   // H(i0-1, j-1)
  int c = 0, w = 0;
  for (int j = 0; j < ncols; j++) {
    uint2 bn = make_uint2(0u, 0u);
    if (!first && j + 1 < ncols) bn = bnd[(j + 1) * 32 + lane];
    const uint32_t sh = 5u * (uint32_t)c;
    const uint32_t rlo = (res.x >> sh) & 31u, rhi = (res.y >> sh) & 31u;
    const int8_t* plo = prof + rlo * stride + i0;
    const int8_t* phi = prof + rhi * stride + i0;
    uint32_t e = bc.x;          // E(i0, j)
    uint32_t diag = htop_prev;  // H(i0-1, j-1)
    htop_prev = bc.y;
    uint32_t hodd = 0u;
#pragma unroll
    for (int k = 0; k < R / 8; k++) {
      const uint2 a = *reinterpret_cast<const uint2*>(plo + 8 * k);
      const uint2 b = *reinterpret_cast<const uint2*>(phi + 8 * k);
#pragma unroll
      for (int rr = 0; rr < 8; rr++) {
        const int r = 8 * k + rr;
        const uint32_t s = prmt(rr < 4 ? a.x : a.y, rr < 4 ? b.x : b.y, sel_pair(rr & 3));
        const uint32_t ds = __vadd2(diag, s);              // H(i-1,j-1) + fsbt (wraps only past LIMIT16)
        const uint32_t h = __vimax3_s16x2(ds, e, F[r]);    // H(i,j) >= 0 since e, F >= 0
        diag = H[r];
        H[r] = h;
        const uint32_t hb = __vadd2(h, nb2);               // H(i,j) - beta
        e = __viaddmax_s16x2_relu(e, na2, hb);             // E(i+1,j)
        F[r] = __viaddmax_s16x2_relu(F[r], na2, hb);       // F(i,j+1)
        if (rr & 1) hmax = __vimax3_s16x2(hmax, hodd, h);
        else hodd = h;
      }
    }
    if (!last) bnd[j * 32 + lane] = make_uint2(e, H[R - 1]);
    bc = bn;
    if (++c == kResPerWord) {
      c = 0;
      ++w;
      res = res_nx;
      if (w + 1 < nwords) res_nx = __ldg(gw + (w + 1) * 32 + lane);
    }
  }
}

template <int T, int R = T - 8>
__device__ __forceinline__ void tile16_rem(int rem, const uint2* gw, int ncols, const int8_t* prof,
                                           int stride, int i0, uint2* bnd, bool first,
                                           uint32_t na2, uint32_t nb2, uint32_t& hmax, int lane) {
  if constexpr (R >= 8) {
    if (rem == R) tile16<R>(gw, ncols, prof, stride, i0, bnd, first, true, na2, nb2, hmax, lane);
    else tile16_rem<T, R - 8>(rem, gw, ncols, prof, stride, i0, bnd, first, na2, nb2, hmax, lane);
  }
}

__device__ __forceinline__ void load_profile_smem(int8_t* sprof, const int8_t* __restrict__ gprof,
                                                  int stride) {
  const int n16 = (kProfRows * stride + 15) / 16;   // buffers are padded to 16 B
  const uint4* src = reinterpret_cast<const uint4*>(gprof);
  uint4* dst = reinterpret_cast<uint4*>(sprof);
  for (int t = threadIdx.x; t < n16; t += blockDim.x) dst[t] = __ldg(src + t);
  __syncthreads();
}

// (ii) inter-task first pass, int16x2.  Persistent: one CTA per SM, each warp
// pulls 64-subject groups longest-first from an atomic counter (the device
// analogue of the paper's guided OpenMP schedule over length-sorted sequence
// profiles).
template <int T, bool SMEM>
__global__ void __launch_bounds__(kInterThreads, 1)
k_inter16(const uint2* __restrict__ words, const GroupDesc* __restrict__ groups, int n_groups,
          const int8_t* __restrict__ gprof, int m_pad, int stride, int alpha, int beta, int limit,
          uint2* __restrict__ scratch, long long scratch_cols, int* __restrict__ counter,
          int* __restrict__ score_sorted, int* __restrict__ flag_count, int* __restrict__ flag_list) {
  extern __shared__ __align__(16) int8_t sprof[];
  const int8_t* prof = gprof;
  if (SMEM) {
    load_profile_smem(sprof, gprof, stride);
    prof = sprof;
  }
  const int lane = threadIdx.x & 31;
  const long long wslot = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  uint2* bnd = scratch + wslot * scratch_cols * 32;
  const uint32_t na2 = pack2(-alpha), nb2 = pack2(-beta);
  const int nfull = m_pad / T, rem = m_pad - nfull * T;
  for (;;) {
    int gi = 0;
    if (lane == 0) gi = atomicAdd(counter, 1);
    gi = __shfl_sync(0xffffffffu, gi, 0);
    if (gi >= n_groups) break;
    const int g = n_groups - 1 - gi;   // groups are stored shortest-first
    const GroupDesc gd = groups[g];
    const uint2* gw = words + gd.base;
    uint32_t hmax = 0u;
    for (int t = 0; t < nfull; t++)
      tile16<T>(gw, gd.ncols, prof, stride, t * T, bnd, t == 0, t == nfull - 1 && rem == 0,
                na2, nb2, hmax, lane);
    if (rem) tile16_rem<T>(rem, gw, gd.ncols, prof, stride, nfull * T, bnd, nfull == 0, na2, nb2, hmax, lane);
    const int slot = 2 * lane;
    const int pos = g * kGroup + slot;
    const int lo = (int)(int16_t)(hmax & 0xffffu), hi = (int)(int16_t)(hmax >> 16);
    if (slot < gd.count) {
      score_sorted[pos] = lo;
      if (lo > limit || lo < 0) flag_list[atomicAdd(flag_count, 1)] = pos;
    }
    if (slot + 1 < gd.count) {
      score_sorted[pos + 1] = hi;
      if (hi > limit || hi < 0) flag_list[atomicAdd(flag_count, 1)] = pos + 1;
    }
  }
}

// ---------------------------------------------------------------------------
// int32 tile, one subject per lane (exact under the ABI bound qlen*s_max < 2^31).
// Used for the rerun of saturated subjects and for first_stage = 32.
// wp: this lane's first packed word; consecutive words are 64 uint32 apart.
// ---------------------------------------------------------------------------
template <int R>
__device__ __forceinline__ void tile32(const uint32_t* __restrict__ wp, int nwords_own, int ncols,
                                       const int8_t* __restrict__ prof, int stride, int i0,
                                       uint2* __restrict__ bnd, bool first, bool last, int alpha,
                                       int beta, int& hmax, int lane) {
  int H[R], F[R];
#pragma unroll
  for (int r = 0; r < R; r++) { H[r] = 0; F[r] = 0; }
  if (ncols <= 0) return;
  uint32_t res = nwords_own > 0 ? __ldg(wp) : kDummyWord;
  uint32_t res_nx = nwords_own > 1 ? __ldg(wp + 64) : kDummyWord;
  uint2 bc = first ? make_uint2(0u, 0u) : bnd[lane];
  int htop_prev = 0;
  int c = 0, w = 0;
  for (int j = 0; j < ncols; j++) {
    uint2 bn = make_uint2(0u, 0u);
    if (!first && j + 1 < ncols) bn = bnd[(j + 1) * 32 + lane];
    const uint32_t rs = (res >> (5u * (uint32_t)c)) & 31u;
    const int8_t* p = prof + rs * stride + i0;
    int e = (int)bc.x;
    int diag = htop_prev;
    htop_prev = (int)bc.y;
    int hodd = 0;
#pragma unroll
    for (int k = 0; k < R / 8; k++) {
      const uint2 a = *reinterpret_cast<const uint2*>(p + 8 * k);
#pragma unroll
      for (int rr = 0; rr < 8; rr++) {
        const int r = 8 * k + rr;
        const int s = (int)prmt(rr < 4 ? a.x : a.y, 0u, sel_one(rr & 3));
        const int h = __vimax3_s32(diag + s, e, F[r]);
        diag = H[r];
        H[r] = h;
        const int hb = h - beta;
        e = __viaddmax_s32_relu(e, -alpha, hb);
        F[r] = __viaddmax_s32_relu(F[r], -alpha, hb);
        if (rr & 1) hmax = __vimax3_s32(hmax, hodd, h);
        else hodd = h;
      }
    }
    if (!last) bnd[j * 32 + lane] = make_uint2((uint32_t)e, (uint32_t)H[R - 1]);
    bc = bn;
    if (++c == kResPerWord) {
      c = 0;
      ++w;
      res = res_nx;
      res_nx = (w + 1 < nwords_own) ? __ldg(wp + (w + 1) * 64) : kDummyWord;
    }
  }
}

template <int T, int R = T - 8>
__device__ __forceinline__ void tile32_rem(int rem, const uint32_t* wp, int nwo, int ncols,
                                           const int8_t* prof, int stride, int i0, uint2* bnd,
                                           bool first, int alpha, int beta, int& hmax, int lane) {
  if constexpr (R >= 8) {
    if (rem == R) tile32<R>(wp, nwo, ncols, prof, stride, i0, bnd, first, true, alpha, beta, hmax, lane);
    else tile32_rem<T, R - 8>(rem, wp, nwo, ncols, prof, stride, i0, bnd, first, alpha, beta, hmax, lane);
  }
}

// int32 pass over a list of sorted positions (list == nullptr: positions
// 0..n_list-1).  Lanes of a warp take consecutive list entries; with a sorted
// list they are neighbours in a group, so word loads stay coalesced.
template <int T, bool SMEM>
__global__ void __launch_bounds__(kInterThreads, 1)
k_list32(const uint2* __restrict__ words, const GroupDesc* __restrict__ groups,
         const int* __restrict__ list, const int* __restrict__ list_count, int n_list,
         const int* __restrict__ len_sorted, const int8_t* __restrict__ gprof, int m_pad, int stride,
         int alpha, int beta, uint2* __restrict__ scratch, long long scratch_cols,
         int* __restrict__ counter, int* __restrict__ score_sorted) {
  extern __shared__ __align__(16) int8_t sprof[];
  const int n = list_count ? *list_count : n_list;
  if (n <= 0) return;
  const int8_t* prof = gprof;
  if (SMEM) {
    load_profile_smem(sprof, gprof, stride);
    prof = sprof;
  }
  const int lane = threadIdx.x & 31;
  const long long wslot = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  uint2* bnd = scratch + wslot * scratch_cols * 32;
  const int nfull = m_pad / T, rem = m_pad - nfull * T;
  for (;;) {
    int chunk = 0;
    if (lane == 0) chunk = atomicAdd(counter, 32);
    chunk = __shfl_sync(0xffffffffu, chunk, 0);
    if (chunk >= n) break;
    const int idx = chunk + lane;
    const int pos = idx < n ? (list ? list[idx] : idx) : -1;
    const int len = pos >= 0 ? len_sorted[pos] : 0;
    int ncols = len;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ncols = max(ncols, __shfl_xor_sync(0xffffffffu, ncols, o));
    const uint32_t* wp = reinterpret_cast<const uint32_t*>(words);
    if (pos >= 0) {
      const int slot = pos & (kGroup - 1);
      wp += 2 * (groups[pos / kGroup].base + (slot >> 1)) + (slot & 1);
    }
    const int nwo = (len + kResPerWord - 1) / kResPerWord;
    int hmax = 0;
    for (int t = 0; t < nfull; t++)
      tile32<T>(wp, nwo, ncols, prof, stride, t * T, bnd, t == 0, t == nfull - 1 && rem == 0, alpha,
                beta, hmax, lane);
    if (rem) tile32_rem<T>(rem, wp, nwo, ncols, prof, stride, nfull * T, bnd, nfull == 0, alpha, beta, hmax, lane);
    if (pos >= 0) score_sorted[pos] = hmax;
  }
}

// ---------------------------------------------------------------------------
// (iv) finalize: scatter to input order and build unique 64-bit ranking keys
// (score << 32 | ~gid): "sort all alignment scores in descending order"
// (PAPER.md:55), ties by ascending global id (reading R7).
// ---------------------------------------------------------------------------
__global__ void k_finalize(const int* __restrict__ score_sorted, const int* __restrict__ perm, int n,
                           const long long* __restrict__ gid, int* __restrict__ scores_out,
                           unsigned long long* __restrict__ keys) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    const int idx = perm[p];
    const int s = score_sorted[p];
    if (scores_out) scores_out[idx] = s;
    const unsigned long long id = gid ? (unsigned long long)gid[idx] : (unsigned long long)idx;
    keys[p] = ((unsigned long long)(unsigned)s << 32) | (0xffffffffull - id);
  }
}

struct SelState {
  unsigned long long prefix, mask;
  long long kk;     // rank (1-based) still to find inside the current prefix
};

// Radix select of the k-th largest key, 8 bits per pass (most significant first).
__global__ void k_sel_hist(const unsigned long long* __restrict__ keys, int n,
                           const SelState* __restrict__ st, int shift, unsigned* __restrict__ hist) {
  __shared__ unsigned sh[256];
  for (int t = threadIdx.x; t < 256; t += blockDim.x) sh[t] = 0;
  __syncthreads();
  const unsigned long long prefix = st->prefix, mask = st->mask;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    const unsigned long long key = keys[p];
    if ((key & mask) == prefix) atomicAdd(&sh[(key >> shift) & 255u], 1u);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 256; t += blockDim.x)
    if (sh[t]) atomicAdd(&hist[t], sh[t]);
}

__global__ void k_sel_pick(SelState* st, int shift, unsigned* hist) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    long long kk = st->kk, above = 0;
    int d = 255;
    for (; d > 0; d--) {
      if (above + (long long)hist[d] >= kk) break;
      above += hist[d];
    }
    st->kk = kk - above;
    st->prefix |= (unsigned long long)d << shift;
    st->mask |= 255ull << shift;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 256; t += blockDim.x) hist[t] = 0;
}

__global__ void k_sel_compact(const unsigned long long* __restrict__ keys, int n,
                              const SelState* __restrict__ st, int take_all,
                              unsigned long long* __restrict__ out, int* __restrict__ count) {
  const unsigned long long thr = take_all ? 0ull : st->prefix;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    const unsigned long long key = keys[p];
    if (key >= thr) out[atomicAdd(count, 1)] = key;
  }
}

// Single-CTA bitonic sort (descending) of cnt <= 4096 keys, then decode.
__global__ void __launch_bounds__(1024) k_topk_small(const unsigned long long* __restrict__ cand,
                                                     int cnt, int k, long long* __restrict__ out_ids,
                                                     int* __restrict__ out_scores) {
  __shared__ unsigned long long s[4096];
  int n2 = 1;
  while (n2 < cnt) n2 <<= 1;
  for (int t = threadIdx.x; t < n2; t += blockDim.x) s[t] = t < cnt ? cand[t] : 0ull;
  __syncthreads();
  for (int size = 2; size <= n2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < n2; t += blockDim.x) {
        const int u = t ^ stride;
        if (u > t) {
          const bool desc = (t & size) == 0;
          const unsigned long long a = s[t], b = s[u];
          if (desc ? (a < b) : (a > b)) { s[t] = b; s[u] = a; }
        }
      }
      __syncthreads();
    }
  }
  for (int t = threadIdx.x; t < k; t += blockDim.x) {
    if (t < cnt) {
      const unsigned long long key = s[t];
      if (out_ids) out_ids[t] = (long long)(0xffffffffull - (key & 0xffffffffull));
      if (out_scores) out_scores[t] = (int)(key >> 32);
    } else {
      if (out_ids) out_ids[t] = -1;
      if (out_scores) out_scores[t] = -1;
    }
  }
}

__global__ void k_topk_decode(const unsigned long long* __restrict__ sorted, int cnt, int k,
                              long long* __restrict__ out_ids, int* __restrict__ out_scores) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < k; t += gridDim.x * blockDim.x) {
    if (t < cnt) {
      const unsigned long long key = sorted[t];
      if (out_ids) out_ids[t] = (long long)(0xffffffffull - (key & 0xffffffffull));
      if (out_scores) out_scores[t] = (int)(key >> 32);
    } else {
      if (out_ids) out_ids[t] = -1;
      if (out_scores) out_scores[t] = -1;
    }
  }
}

}  // namespace swk
