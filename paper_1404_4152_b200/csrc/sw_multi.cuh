// sw_multi.cuh -- f1: two queries per int16x2 pass
// Part of the device code of libswsearch (see sw_common.cuh for the overview).
#pragma once
#include "sw_common.cuh"

namespace swk {

// ---------------------------------------------------------------------------
// f1 multi-query pass: TWO queries per pass in the lo/hi halves of int16x2, one
// subject per lane.  Both halves read the same subject residue, so the
// substitution pair is a single word of the pair profile
//   prof2[r][i] = (fsbt(qa_i, r), fsbt(qb_i, r))   (int16x2)
// and the PRMT of the single-query kernel disappears (3.5 alu ops per row).
// The row stride is 2 mod 32 words (odd in 8-byte units) and tiles start at even
// rows, so two rows come in one LDS.64 and only residues r, r + 16 share banks.
// ---------------------------------------------------------------------------
template <int R>
__device__ __forceinline__ uint32_t colq(uint32_t (&D)[R], uint32_t (&F)[R], uint32_t& e, uint32_t htop,
                                         const uint32_t* __restrict__ p, uint32_t na2, uint32_t nb2,
                                         uint32_t& hmax) {
  uint32_t hprev = htop, hodd = 0u;
  uint2 pw = make_uint2(0u, 0u);
#pragma unroll
  for (int r = 0; r < R; r++) {
    const uint32_t h = __vimax3_s16x2(D[r], e, F[r]);
    if (!(r & 1)) pw = *reinterpret_cast<const uint2*>(p + r);  // rows r, r+1 in one LDS.64 (p is 8-byte aligned)
    D[r] = __vadd2(hprev, (r & 1) ? pw.y : pw.x);              // H(i-1,j) + (fsbt(qa_i,s_{j+1}), fsbt(qb_i,s_{j+1}))
    const uint32_t hb = __vadd2(h, nb2);
    e = __viaddmax_s16x2_relu(e, na2, hb);
    F[r] = __viaddmax_s16x2_relu(F[r], na2, hb);
    if (r & 1) hmax = __vimax3_s16x2(hmax, hodd, h);
    else hodd = h;
    hprev = h;
  }
  return hprev;
}

template <int R>
__device__ __forceinline__ void tileq(const uint32_t* __restrict__ wp, int nwords, int ncols,
                                      const uint32_t* __restrict__ prof2, int stride2, int i0,
                                      uint2* __restrict__ bnd, bool first, bool last, uint32_t na2, uint32_t nb2,
                                      uint32_t& hmax, int lane) {
  if (ncols <= 0) return;
  uint32_t D[R], F[R];
#pragma unroll
  for (int r = 0; r < R; r++) { D[r] = 0u; F[r] = 0u; }
  const uint32_t* pr = prof2 + i0;
  {
    uint32_t e0 = 0u;
    const uint32_t w0 = nwords > 0 ? __ldg(wp) : kDummyWord;
    colq<R>(D, F, e0, 0u, pr + (w0 & 31u) * stride2, na2, nb2, hmax);
  }
  const uint2 z = make_uint2(0u, 0u);
  uint2 bE = first ? z : bnd[lane];
  uint2 bO = (first || ncols < 2) ? z : bnd[32 + lane];
  uint32_t wA = res_word32(wp, 1, nwords), wB = res_word32(wp, 2, nwords);
  int j = 0;
  for (; j + 1 < ncols; j += 2) {
    const int shA = res_shift(j + 1), shB = res_shift(j + 2);
    uint32_t eA = bE.x, eB = bO.x;
    const uint32_t tA = bE.y, tB = bO.y;
    // next pair's tile-edge rows requested as soon as these are consumed (as in tile16)
    if (!first && j + 2 < ncols) bE = bnd[(j + 2) * 32 + lane];
    if (!first && j + 3 < ncols) bO = bnd[(j + 3) * 32 + lane];
    const uint32_t hlA = colq<R>(D, F, eA, tA, pr + ((wA >> shA) & 31u) * stride2, na2, nb2, hmax);
    const uint32_t hlB = colq<R>(D, F, eB, tB, pr + ((wB >> shB) & 31u) * stride2, na2, nb2, hmax);
    wA = res_word32(wp, j + 3, nwords);
    wB = res_word32(wp, j + 4, nwords);
    if (!last) {
      bnd[j * 32 + lane] = make_uint2(eA, hlA);
      bnd[(j + 1) * 32 + lane] = make_uint2(eB, hlB);
    }
  }
  if (j < ncols) {
    const int shA = res_shift(j + 1);
    uint32_t e = bE.x;
    const uint32_t hl = colq<R>(D, F, e, bE.y, pr + ((wA >> shA) & 31u) * stride2, na2, nb2, hmax);
    if (!last) bnd[j * 32 + lane] = make_uint2(e, hl);
  }
}

template <int T, int R = T - 8>
__device__ __forceinline__ void tileq_rem(int rem, const uint32_t* wp, int nwords, int ncols, const uint32_t* prof2,
                                          int stride2, int i0, uint2* bnd, bool first, uint32_t na2, uint32_t nb2,
                                          uint32_t& hmax, int lane) {
  if constexpr (R >= 8) {
    if (rem == R) tileq<R>(wp, nwords, ncols, prof2, stride2, i0, bnd, first, true, na2, nb2, hmax, lane);
    else tileq_rem<T, R - 8>(rem, wp, nwords, ncols, prof2, stride2, i0, bnd, first, na2, nb2, hmax, lane);
  }
}

// pair profile: prof2[r * stride2 + i] = (fsbt(qa_i, r) lo, fsbt(qb_i, r) hi); rows past a query's end = 0
__global__ void k_profile_pair(const uint8_t* __restrict__ qa, int ma, const uint8_t* __restrict__ qb, int mb,
                               const int8_t* __restrict__ M, uint32_t* __restrict__ prof2, int stride2) {
  const int total = kProfRows * stride2;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int r = t / stride2, i = t - r * stride2;
    int va = 0, vb = 0;
    if (r < kNumCodes) {
      if (i < ma) va = M[qa[i] * 32 + r];
      if (i < mb) vb = M[qb[i] * 32 + r];
    }
    prof2[t] = ((uint32_t)va & 0xffffu) | ((uint32_t)vb << 16);
  }
}

// Items: half-groups (32 subjects, the lo or hi members of a 64-subject group), longest first.
template <int T, int GAPS = 0>
__global__ void __launch_bounds__(kInterThreads, 1)
k_multi16(const uint2* __restrict__ words, const GroupDesc* __restrict__ groups, int n_groups, int cut,
          const uint32_t* __restrict__ gprof2, int m_pad, int stride2, int alpha, int beta, int limit,
          uint2* __restrict__ scratch, long long scratch_cols, int* __restrict__ counter,
          int* __restrict__ score_a, int* __restrict__ score_b, uint8_t* __restrict__ flag_a,
          uint8_t* __restrict__ flag_b) {
  extern __shared__ __align__(16) uint32_t sprof2[];
  __shared__ int s_split;
  {
    if (threadIdx.x == 0) s_split = split_groups(groups, n_groups, cut);   // wider groups: k_intra16 per query
    const int n4 = kProfRows * stride2;
    for (int t = threadIdx.x; t < n4; t += blockDim.x) sprof2[t] = __ldg(gprof2 + t);
    __syncthreads();
  }
  n_groups = s_split;
  const int lane = threadIdx.x & 31;
  const long long wslot = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  uint2* bnd = scratch + wslot * scratch_cols * 32;
  const uint32_t na2 = GAPS == 1 ? pack2(-kFixedAlpha) : pack2(-alpha);    // GAPS: as in k_inter16
  const uint32_t nb2 = GAPS == 1 ? pack2(-kFixedBeta) : pack2(-beta);
  const int nfull = m_pad / T, rem = m_pad - nfull * T;
  const int n_items = 2 * n_groups;
  for (;;) {
    int item = 0;
    if (lane == 0) item = atomicAdd(counter, 1);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= n_items) break;
    const int g = n_groups - 1 - item / 2;
    const int half = 1 - (item & 1);
    const GroupDesc gd = groups[g];
    const int slot = 2 * lane + half;
    if (gd.ncols > scratch_cols) {         // too long for the boundary slab: both queries go to the int32 rerun
      if (slot < gd.count) {
        flag_a[g * kGroup + slot] = 1;
        flag_b[g * kGroup + slot] = 1;
      }
      continue;
    }
    const uint32_t* wp = reinterpret_cast<const uint32_t*>(words) + 2 * (gd.base + lane) + half;
    const int nwords = (gd.ncols + kResPerWord - 1) / kResPerWord;
    uint32_t hmax = 0u;
    for (int t = 0; t < nfull; t++)
      tileq<T>(wp, nwords, gd.ncols, sprof2, stride2, t * T, bnd, t == 0, t == nfull - 1 && rem == 0, na2, nb2,
               hmax, lane);
    if (rem) tileq_rem<T>(rem, wp, nwords, gd.ncols, sprof2, stride2, nfull * T, bnd, nfull == 0, na2, nb2, hmax, lane);
    if (slot < gd.count) {
      const int pos = g * kGroup + slot;
      const int a = (int)(int16_t)(hmax & 0xffffu), b = (int)(int16_t)(hmax >> 16);
      score_a[pos] = a;
      score_b[pos] = b;
      if (a > limit || a < 0) flag_a[pos] = 1;
      if (b > limit || b < 0) flag_b[pos] = 1;
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");   // programmatic dependent of the intra-task passes
}


}  // namespace swk
