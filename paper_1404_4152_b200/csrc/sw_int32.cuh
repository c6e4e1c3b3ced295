// sw_int32.cuh -- the exact int32 pass: reruns of saturated subjects and first_stage 32 (a4)
// Part of the device code of libswsearch (see sw_common.cuh for the overview).
#pragma once
#include "sw_common.cuh"

namespace swk {

// ---------------------------------------------------------------------------
// int32 tile, one subject per lane (exact under the ABI bound qlen*s_max < 2^31).
// Used for the rerun of saturated subjects and for first_stage = 32.
// wp: this lane's first packed word; consecutive words are 64 uint32 apart.
// ---------------------------------------------------------------------------
// int32 column (one subject per lane), same D formulation as col16.
template <int R>
__device__ __forceinline__ int col32(int (&D)[R], int (&F)[R], int& e, int htop, const int8_t* __restrict__ p,
                                     int alpha, int beta, int& hmax) {
  int hprev = htop, hodd = 0;
  uint2 a = *reinterpret_cast<const uint2*>(p);
#pragma unroll
  for (int k = 0; k < R / 8; k++) {
    uint2 an = a;
    if (k + 1 < R / 8) an = *reinterpret_cast<const uint2*>(p + 8 * (k + 1));
#pragma unroll
    for (int rr = 0; rr < 8; rr++) {
      const int r = 8 * k + rr;
      const int h = __vimax3_s32(D[r], e, F[r]);                  // H(i,j)
      const int sn = (int)prmt(rr < 4 ? a.x : a.y, 0u, sel_one(rr & 3));
      D[r] = hprev + sn;                                          // H(i-1,j) + fsbt(q_i, s_{j+1})
      const int hb = h - beta;
      e = __viaddmax_s32_relu(e, -alpha, hb);
      F[r] = __viaddmax_s32_relu(F[r], -alpha, hb);
      if (rr & 1) hmax = __vimax3_s32(hmax, hodd, h);
      else hodd = h;
      hprev = h;
    }
    a = an;
  }
  return hprev;
}

// residue code of column c for a lane whose packed words are wp[w * 64] (w < nwo)
__device__ __forceinline__ uint32_t res_word32(const uint32_t* __restrict__ wp, int c, int nwo) {
  const int w = (int)(__umulhi((unsigned)c, 0xAAAAAAABu) >> 2);
  return w < nwo ? __ldg(wp + (long long)w * 64) : kDummyWord;
}

// int32 tile, one subject per lane (exact under the ABI bound qlen*s_max < 2^31).
// Used for the rerun of saturated subjects and for first_stage = 32.
template <int R>
__device__ __forceinline__ void tile32(const uint32_t* __restrict__ wp, int nwords_own, int ncols,
                                       const int8_t* __restrict__ prof, int stride, int i0,
                                       uint2* __restrict__ bnd, bool first, bool last, int alpha,
                                       int beta, int& hmax, int lane) {
  if (ncols <= 0) return;
  int D[R], F[R];
#pragma unroll
  for (int r = 0; r < R; r++) { D[r] = 0; F[r] = 0; }
  const int8_t* pr = prof + i0;
  {
    int e0 = 0;
    const uint32_t w0 = nwords_own > 0 ? __ldg(wp) : kDummyWord;
    col32<R>(D, F, e0, 0, pr + (w0 & 31u) * stride, alpha, beta, hmax);
  }
  const uint2 z = make_uint2(0u, 0u);
  uint2 bE = first ? z : bnd[lane];
  uint2 bO = (first || ncols < 2) ? z : bnd[32 + lane];
  uint32_t wA = res_word32(wp, 1, nwords_own), wB = res_word32(wp, 2, nwords_own);
  int j = 0;
  for (; j + 1 < ncols; j += 2) {
    const int shA = res_shift(j + 1), shB = res_shift(j + 2);
    int eA = (int)bE.x, eB = (int)bO.x;
    const int hlA = col32<R>(D, F, eA, (int)bE.y, pr + ((wA >> shA) & 31u) * stride, alpha, beta, hmax);
    const int hlB = col32<R>(D, F, eB, (int)bO.y, pr + ((wB >> shB) & 31u) * stride, alpha, beta, hmax);
    wA = res_word32(wp, j + 3, nwords_own);
    wB = res_word32(wp, j + 4, nwords_own);
    if (!first && j + 2 < ncols) bE = bnd[(j + 2) * 32 + lane];
    if (!first && j + 3 < ncols) bO = bnd[(j + 3) * 32 + lane];
    if (!last) {
      bnd[j * 32 + lane] = make_uint2((uint32_t)eA, (uint32_t)hlA);
      bnd[(j + 1) * 32 + lane] = make_uint2((uint32_t)eB, (uint32_t)hlB);
    }
  }
  if (j < ncols) {
    const int shA = res_shift(j + 1);
    int e = (int)bE.x;
    const int hl = col32<R>(D, F, e, (int)bE.y, pr + ((wA >> shA) & 31u) * stride, alpha, beta, hmax);
    if (!last) bnd[j * 32 + lane] = make_uint2((uint32_t)e, (uint32_t)hl);
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

// Intra-task wavefront for ONE long subject per warp in int32 (rerun of
// saturated long subjects, e.g. the S16 copies): lane l owns rows
// [base + l*TR, base + (l+1)*TR) of a 32*TR-row pass and processes column
// s - l at step s; (E, H, next residue) move to lane l+1 by SHFL.
template <int TR>
__device__ __forceinline__ int intra_single32(const uint32_t* __restrict__ wp, int nwo, int ncols,
                                              const int8_t* __restrict__ prof, int stride, int m_pad,
                                              uint2* __restrict__ gbnd, long long gstride, int alpha, int beta,
                                              int lane) {
  int hmax = 0;
  int pass = 0;
  for (int base = 0; base < m_pad; base += 32 * TR, pass++) {
    const int nact = min(32, (m_pad - base + TR - 1) / TR);
    const bool first = base == 0, last = base + 32 * TR >= m_pad;
    const uint2* gin = gbnd + (long long)(pass & 1) * gstride;
    uint2* gout = gbnd + (long long)((pass + 1) & 1) * gstride;
    const int8_t* pr = prof + base + lane * TR;
    int D[TR], F[TR];
#pragma unroll
    for (int r = 0; r < TR; r++) { D[r] = 0; F[r] = 0; }
    int e_out = 0, h_out = 0;
    uint32_t r_out = 0u;
    uint2 gnext = make_uint2(0u, 0u);
    if (!first && lane == 0) gnext = gin[0];
    __syncwarp();
    for (int s = -1; s < ncols + nact - 1; s++) {
      int e_in = __shfl_up_sync(0xffffffffu, e_out, 1);
      int h_in = __shfl_up_sync(0xffffffffu, h_out, 1);
      uint32_t r_in = __shfl_up_sync(0xffffffffu, r_out, 1);
      const int j = s - lane;
      if (lane == 0) {
        const int c = s + 1;                                       // next column of lane 0
        r_in = (res_word32(wp, c, nwo) >> res_shift(c)) & 31u;
        if (first || j < 0) { e_in = 0; h_in = 0; }
        else {
          e_in = (int)gnext.x;
          h_in = (int)gnext.y;
          gnext = (j + 1 < ncols) ? gin[j + 1] : make_uint2(0u, 0u);
        }
      }
      if (lane < nact && j >= -1 && j < ncols) {
        int e = e_in;
        const int hl = col32<TR>(D, F, e, h_in, pr + r_in * stride, alpha, beta, hmax);
        e_out = e;
        h_out = hl;
        r_out = r_in;
        if (!last && lane == nact - 1 && j >= 0) gout[j] = make_uint2((uint32_t)e, (uint32_t)hl);
      }
    }
    __syncwarp();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) hmax = max(hmax, __shfl_xor_sync(0xffffffffu, hmax, o));
  return hmax;
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
  // programmatic dependent of the flag compaction (small databases): the list
  // and its count are visible after the wait; the ranking behind may launch
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
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
  // A sorted list (reruns) ends with its longest subjects: entries longer than
  // kIntra32Cols are taken one per warp by the intra-task wavefront (first, as
  // the longest work), the rest 32 per warp, one per lane.
  int n_short;
  {
    int lo = 0, hi = n;                               // first entry with len > cut (lists are ascending)
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (len_sorted[list ? list[mid] : mid] > kIntra32Cols) hi = mid;
      else lo = mid + 1;
    }
    n_short = lo;
  }
  const int n_long = n - n_short;
  const int n_items = n_long + (n_short + 31) / 32;
  for (;;) {
    int item = 0;
    if (lane == 0) item = atomicAdd(counter, 1);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= n_items) break;
    if (item < n_long) {
      const int pos = list ? list[n - 1 - item] : n - 1 - item;
      const int len = len_sorted[pos];
      const int slot = pos & (kGroup - 1);
      const uint32_t* wp = reinterpret_cast<const uint32_t*>(words) + 2 * (groups[pos / kGroup].base + (slot >> 1)) + (slot & 1);
      const int hm = intra_single32<kIntraRows>(wp, (len + kResPerWord - 1) / kResPerWord, len, prof, stride, m_pad,
                                                bnd, scratch_cols * 16, alpha, beta, lane);
      if (lane == 0) score_sorted[pos] = hm;
      continue;
    }
    const int chunk = (item - n_long) * 32;
    const int idx = chunk + lane;
    const int pos = idx < n_short ? (list ? list[idx] : idx) : -1;
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


}  // namespace swk
