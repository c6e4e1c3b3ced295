// sw_int8.cuh -- the optional int8 first stage (a4, biased unsigned bytes)
// Part of the device code of libswsearch (see sw_common.cuh for the overview).
#pragma once
#include "sw_common.cuh"

namespace swk {

// ---------------------------------------------------------------------------
// int8 first stage (biased unsigned bytes): four
// subjects per lane in the bytes of a 32-bit word (pair `lane` of groups 2u and
// 2u+1).  H, E, F hold the true (clamped) values in [0, 255]; substitutions are
// biased by B = -min(0, s_min) so they are unsigned:
//   H = max(satsub(satadd(H(i-1,j-1), s + B), B), E, F)
//   E = max(satsub(E, alpha), satsub(H, beta)),  F likewise.
// Exact until an add saturates, which needs an exactly computed H > LIMIT8 =
// 255 - (s_max + B); those subjects are flagged and re-aligned at int16.
// Byte SIMD is emulated on sm_100a (~7-8 instructions per __vaddus4/__vsubus4/
// __vmaxu4), so this pass is measured, not assumed (DESIGN.md §"int8 stage").
// ---------------------------------------------------------------------------
template <int R>
__device__ __forceinline__ uint32_t col8(uint32_t (&D)[R], uint32_t (&F)[R], uint32_t& e, uint32_t htop,
                                         const uint8_t* __restrict__ p0, const uint8_t* __restrict__ p1,
                                         const uint8_t* __restrict__ p2, const uint8_t* __restrict__ p3,
                                         uint32_t a4, uint32_t b4, uint32_t B4, uint32_t& hmax) {
  uint32_t hprev = htop;
#pragma unroll
  for (int k = 0; k < R / 8; k++) {
    const uint2 q0 = *reinterpret_cast<const uint2*>(p0 + 8 * k);
    const uint2 q1 = *reinterpret_cast<const uint2*>(p1 + 8 * k);
    const uint2 q2 = *reinterpret_cast<const uint2*>(p2 + 8 * k);
    const uint2 q3 = *reinterpret_cast<const uint2*>(p3 + 8 * k);
#pragma unroll
    for (int h2 = 0; h2 < 2; h2++) {           // rows 8k + 4*h2 .. +3
      const uint32_t w0 = h2 ? q0.y : q0.x, w1 = h2 ? q1.y : q1.x;
      const uint32_t w2 = h2 ? q2.y : q2.x, w3 = h2 ? q3.y : q3.x;
      // transpose: row t -> (w0.byte t, w1.byte t, w2.byte t, w3.byte t)
      const uint32_t t01a = prmt(w0, w1, 0x5140u), t23a = prmt(w2, w3, 0x5140u);   // rows 0,1
      const uint32_t t01b = prmt(w0, w1, 0x7362u), t23b = prmt(w2, w3, 0x7362u);   // rows 2,3
      uint32_t sv[4];
      sv[0] = prmt(t01a, t23a, 0x5410u);
      sv[1] = prmt(t01a, t23a, 0x7632u);
      sv[2] = prmt(t01b, t23b, 0x5410u);
      sv[3] = prmt(t01b, t23b, 0x7632u);
#pragma unroll
      for (int t = 0; t < 4; t++) {
        const int r = 8 * k + 4 * h2 + t;
        const uint32_t h = __vmaxu4(__vmaxu4(__vsubus4(D[r], B4), e), F[r]);
        D[r] = __vaddus4(hprev, sv[t]);
        const uint32_t hb = __vsubus4(h, b4);
        e = __vmaxu4(__vsubus4(e, a4), hb);
        F[r] = __vmaxu4(__vsubus4(F[r], a4), hb);
        hmax = __vmaxu4(hmax, h);
        hprev = h;
      }
    }
  }
  return hprev;
}

template <int R>
__device__ __forceinline__ void tile8(const uint2* __restrict__ gw0, const uint2* __restrict__ gw1, int nw0,
                                      int nw1, int ncols, const uint8_t* __restrict__ prof, int stride, int i0,
                                      uint2* __restrict__ bnd, bool first, bool last, uint32_t a4, uint32_t b4,
                                      uint32_t B4, uint32_t& hmax, int lane) {
  if (ncols <= 0) return;
  uint32_t D[R], F[R];
#pragma unroll
  for (int r = 0; r < R; r++) { D[r] = 0u; F[r] = 0u; }
  ResCursor c0, c1;
  c0.init(gw0 + lane, nw0);
  c1.init(gw1 + lane, nw1);
  {
    uint32_t e0 = 0u;
    col8<R>(D, F, e0, 0u, prof + c0.lo() * stride + i0, prof + c0.hi() * stride + i0, prof + c1.lo() * stride + i0,
            prof + c1.hi() * stride + i0, a4, b4, B4, hmax);
    c0.next();
    c1.next();
  }
  const uint2 z = make_uint2(0u, 0u);
  uint2 bc = first ? z : bnd[lane];
  for (int j = 0; j < ncols; j++) {
    uint2 bn = z;
    if (!first && j + 1 < ncols) bn = bnd[(j + 1) * 32 + lane];
    uint32_t e = bc.x;
    const uint32_t hl = col8<R>(D, F, e, bc.y, prof + c0.lo() * stride + i0, prof + c0.hi() * stride + i0,
                                prof + c1.lo() * stride + i0, prof + c1.hi() * stride + i0, a4, b4, B4, hmax);
    if (!last) bnd[j * 32 + lane] = make_uint2(e, hl);
    bc = bn;
    c0.next();
    c1.next();
  }
}

template <int T, int R = T - 8>
__device__ __forceinline__ void tile8_rem(int rem, const uint2* gw0, const uint2* gw1, int nw0, int nw1, int ncols,
                                          const uint8_t* prof, int stride, int i0, uint2* bnd, bool first,
                                          uint32_t a4, uint32_t b4, uint32_t B4, uint32_t& hmax, int lane) {
  if constexpr (R >= 8) {
    if (rem == R) tile8<R>(gw0, gw1, nw0, nw1, ncols, prof, stride, i0, bnd, first, true, a4, b4, B4, hmax, lane);
    else tile8_rem<T, R - 8>(rem, gw0, gw1, nw0, nw1, ncols, prof, stride, i0, bnd, first, a4, b4, B4, hmax, lane);
  }
}

template <int T, bool SMEM>
__global__ void __launch_bounds__(kInterThreads, 1)
k_inter8(const uint2* __restrict__ words, const GroupDesc* __restrict__ groups, int n_groups,
         const uint8_t* __restrict__ gprof, int m_pad, int stride, int alpha, int beta, int bias, int limit,
         uint2* __restrict__ scratch, long long scratch_cols, int* __restrict__ counter,
         int* __restrict__ score_sorted, uint8_t* __restrict__ flag) {
  extern __shared__ __align__(16) int8_t sprof[];
  const uint8_t* prof = gprof;
  if (SMEM) {
    load_profile_smem(sprof, reinterpret_cast<const int8_t*>(gprof), stride);
    prof = reinterpret_cast<const uint8_t*>(sprof);
  }
  const int lane = threadIdx.x & 31;
  const long long wslot = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  uint2* bnd = scratch + wslot * scratch_cols * 32;
  const uint32_t a4 = (uint32_t)alpha * 0x01010101u, b4 = (uint32_t)beta * 0x01010101u,
                 B4 = (uint32_t)bias * 0x01010101u;
  const int nfull = m_pad / T, rem = m_pad - nfull * T;
  const int n_units = (n_groups + 1) / 2;
  for (;;) {
    int item = 0;
    if (lane == 0) item = atomicAdd(counter, 1);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= n_units) break;
    const int u = n_units - 1 - item;                      // longest first
    const int g0 = 2 * u, g1 = 2 * u + 1;
    const GroupDesc d0 = groups[g0];
    GroupDesc d1;
    d1.base = 0;
    d1.ncols = 0;
    d1.count = 0;
    if (g1 < n_groups) d1 = groups[g1];
    const int ncols = max(d0.ncols, d1.ncols);
    if (ncols > scratch_cols) {            // too long for the boundary slab: straight to the int16 rerun
      for (int b = 0; b < 4; b++) {
        const GroupDesc& d = b < 2 ? d0 : d1;
        const int slot = 2 * lane + (b & 1);
        if (slot < d.count) flag[(b < 2 ? g0 : g1) * kGroup + slot] = 1;
      }
      continue;
    }
    const int nw0 = (d0.ncols + kResPerWord - 1) / kResPerWord, nw1 = (d1.ncols + kResPerWord - 1) / kResPerWord;
    const uint2* gw0 = words + d0.base;
    const uint2* gw1 = words + d1.base;
    uint32_t hmax = 0u;
    for (int t = 0; t < nfull; t++)
      tile8<T>(gw0, gw1, nw0, nw1, ncols, prof, stride, t * T, bnd, t == 0, t == nfull - 1 && rem == 0, a4, b4, B4,
               hmax, lane);
    if (rem) tile8_rem<T>(rem, gw0, gw1, nw0, nw1, ncols, prof, stride, nfull * T, bnd, nfull == 0, a4, b4, B4, hmax, lane);
    const int sc[4] = {(int)(hmax & 255u), (int)((hmax >> 8) & 255u), (int)((hmax >> 16) & 255u), (int)(hmax >> 24)};
#pragma unroll
    for (int b = 0; b < 4; b++) {
      const GroupDesc& d = b < 2 ? d0 : d1;
      const int g = b < 2 ? g0 : g1;
      const int slot = 2 * lane + (b & 1);
      if (slot < d.count) {
        const int pos = g * kGroup + slot;
        score_sorted[pos] = sc[b];
        if (sc[b] > limit) flag[pos] = 1;
      }
    }
  }
}

// biased uint8 profile for the int8 stage: prof[r][i] = fsbt(q_i, r) + bias (DUMMY/pad: bias)
__global__ void k_profile8b(const uint8_t* __restrict__ q, int m, const int8_t* __restrict__ M, int bias,
                            uint8_t* __restrict__ prof, int stride) {
  const int total = kProfRows * stride;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int r = t / stride, i = t - r * stride;
    int v = 0;
    if (i < m && r < kNumCodes) v = M[q[i] * 32 + r];
    prof[t] = (uint8_t)(v + bias);
  }
}


}  // namespace swk
