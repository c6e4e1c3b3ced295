// sw_ablation.cuh — f4: the paper's kernel variants re-built on sm_100a as
// ablations of the production kernels.  They compute the
// same Eq. 1 scores (parity-tested) and exist to measure which of the paper's
// design choices transfer to B200; they are selected with SW_VARIANT (a
// measurement switch, not part of the ABI).
//
// InterSP (Fig. 4: "score profile", the paper's fastest
// variant): instead of the query profile, every lane builds, for the next
// subject column, the score profile of its two subjects over the query
// alphabet, SP[a] = (fsbt(a, s_lo), fsbt(a, s_hi)) as int16x2, in its own
// column of a per-warp shared-memory table; each query row then reads
// SP[q_i] with one conflict-free LDS.32 and no PRMT.  The build costs 25 PRMT
// + 25 STS per column, amortized over the tile's rows.
//
// IntraQP (intra-task, query profile, Farrar's striped
// layout with the lazy-F loop): one warp aligns one subject pair (lo/hi halves
// of int16x2); lane v holds the contiguous query segment [v*L, (v+1)*L) in
// registers and all lanes step through their segments together, so the
// vertical gap (E here) entering a segment is at first assumed 0 and then
// corrected by a lazy loop that shifts E one lane down and re-walks rows while
// any lane's incoming E can still raise H.  Replaces the intra-task wavefront.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace swk {

constexpr int kSpRows = 32;          // register-tile height of the InterSP variant (D, F and q offsets in registers)
constexpr int kMtStride = 40;        // bytes per subject row of the transposed int8 matrix in shared memory

// Score profile of the lane's next column: sp[a * 32] (this lane's column) for a = 0..24.
__device__ __forceinline__ void build_sp(uint32_t* __restrict__ sp, const int8_t* __restrict__ mt, uint32_t slo,
                                         uint32_t shi) {
  const uint32_t* lo = reinterpret_cast<const uint32_t*>(mt + slo * kMtStride);
  const uint32_t* hi = reinterpret_cast<const uint32_t*>(mt + shi * kMtStride);
#pragma unroll
  for (int w = 0; w < 7; w++) {
    const uint32_t a = lo[w], b = hi[w];
#pragma unroll
    for (int rr = 0; rr < 4; rr++)
      if (4 * w + rr < kProfRows) sp[(4 * w + rr) * 32] = prmt(a, b, sel_pair(rr));
  }
}

template <int R>
__device__ __forceinline__ uint32_t colsp(uint32_t (&D)[R], uint32_t (&F)[R], uint32_t& e, uint32_t htop,
                                          const uint32_t* __restrict__ sp, const int (&qo)[R], uint32_t na2,
                                          uint32_t nb2, uint32_t& hmax) {
  uint32_t hprev = htop, hodd = 0u;
#pragma unroll
  for (int r = 0; r < R; r++) {
    const uint32_t h = __vimax3_s16x2(D[r], e, F[r]);
    D[r] = __vadd2(hprev, sp[qo[r]]);                          // H(i-1,j) + SP_{j+1}[q_i]
    const uint32_t hb = __vadd2(h, nb2);
    e = __viaddmax_s16x2_relu(e, na2, hb);
    F[r] = __viaddmax_s16x2_relu(F[r], na2, hb);
    if (r & 1) hmax = __vimax3_s16x2(hmax, hodd, h);
    else hodd = h;
    hprev = h;
  }
  return hprev;
}

// One query tile [i0, i0+R) of one group, as tile16 but with the score profile.
template <int R>
__device__ __forceinline__ void tile16sp(const uint2* __restrict__ gw, int ncols, const uint8_t* __restrict__ q,
                                         int m, int i0, uint32_t* __restrict__ sp, const int8_t* __restrict__ mt,
                                         uint2* __restrict__ bnd, bool first, bool last, uint32_t na2, uint32_t nb2,
                                         uint32_t& hmax, int lane) {
  if (ncols <= 0) return;
  uint32_t D[R], F[R];
  int qo[R];
#pragma unroll
  for (int r = 0; r < R; r++) {
    D[r] = 0u;
    F[r] = 0u;
    qo[r] = (i0 + r < m ? (int)__ldg(q + i0 + r) : kDummy) * 32;   // padded rows read the DUMMY entry (0)
  }
  const uint2* lw = gw + lane;
  const int nwords = (ncols + kResPerWord - 1) / kResPerWord;
  {
    const uint2 w0 = lw[0];
    build_sp(sp, mt, w0.x & 31u, w0.y & 31u);
    uint32_t e0 = 0u;
    colsp<R>(D, F, e0, 0u, sp, qo, na2, nb2, hmax);
  }
  const uint2 z = make_uint2(0u, 0u);
  uint2 bc = first ? z : bnd[lane];
  for (int j = 0; j < ncols; j++) {
    const uint2 w = res_word(lw, j + 1, nwords);
    const int sh = res_shift(j + 1);
    build_sp(sp, mt, (w.x >> sh) & 31u, (w.y >> sh) & 31u);      // the lane's own column: no warp sync needed
    const uint2 bn = (!first && j + 1 < ncols) ? bnd[(j + 1) * 32 + lane] : z;
    uint32_t e = bc.x;
    const uint32_t hl = colsp<R>(D, F, e, bc.y, sp, qo, na2, nb2, hmax);
    if (!last) bnd[j * 32 + lane] = make_uint2(e, hl);
    bc = bn;
  }
}

template <int T, int R = T - 8>
__device__ __forceinline__ void tile16sp_rem(int rem, const uint2* gw, int ncols, const uint8_t* q, int m, int i0,
                                             uint32_t* sp, const int8_t* mt, uint2* bnd, bool first, uint32_t na2,
                                             uint32_t nb2, uint32_t& hmax, int lane) {
  if constexpr (R >= 8) {
    if (rem == R) tile16sp<R>(gw, ncols, q, m, i0, sp, mt, bnd, first, true, na2, nb2, hmax, lane);
    else tile16sp_rem<T, R - 8>(rem, gw, ncols, q, m, i0, sp, mt, bnd, first, na2, nb2, hmax, lane);
  }
}

// InterSP ablation of k_inter16: every group inter-task (no intra split), 12
// warps per CTA, shared memory = transposed matrix + 25 x 32 words per warp.
__global__ void __launch_bounds__(kInterThreads, 1)
k_inter16_sp(const uint2* __restrict__ words, const GroupDesc* __restrict__ groups, int n_groups, int cut,
             const uint8_t* __restrict__ q, int m, int m_pad, const int8_t* __restrict__ M, int alpha, int beta,
             int limit, uint2* __restrict__ scratch, long long scratch_cols, int* __restrict__ counter,
             int* __restrict__ score_sorted, uint8_t* __restrict__ flag) {
  __shared__ __align__(16) int8_t mt[kProfRows * kMtStride];
  __shared__ uint32_t sp_all[kInterThreads / 32][kProfRows * 32];
  __shared__ int s_split;
  if (threadIdx.x == 0) s_split = split_groups(groups, n_groups, cut);   // longer groups: k_intra16
  for (int t = threadIdx.x; t < kProfRows * kMtStride; t += blockDim.x) {
    const int s = t / kMtStride, a = t % kMtStride;                 // mt[s][a] = fsbt(a, s); DUMMY row/col = 0
    mt[t] = (s < kNumCodes && a < kNumCodes) ? M[a * 32 + s] : (int8_t)0;
  }
  __syncthreads();
  n_groups = s_split;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* sp = sp_all[warp] + lane;
  uint2* bnd = scratch + ((long long)blockIdx.x * (blockDim.x >> 5) + warp) * scratch_cols * 32;
  const uint32_t na2 = pack2(-alpha), nb2 = pack2(-beta);
  const int nfull = m_pad / kSpRows, rem = m_pad - nfull * kSpRows;
  for (;;) {
    int item = 0;
    if (lane == 0) item = atomicAdd(counter, 1);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= n_groups) break;
    const int g = n_groups - 1 - item;
    const GroupDesc gd = groups[g];
    uint32_t hmax = 0u;
    for (int t = 0; t < nfull; t++)
      tile16sp<kSpRows>(words + gd.base, gd.ncols, q, m, t * kSpRows, sp, mt, bnd, t == 0,
                        t == nfull - 1 && rem == 0, na2, nb2, hmax, lane);
    if (rem)
      tile16sp_rem<kSpRows>(rem, words + gd.base, gd.ncols, q, m, nfull * kSpRows, sp, mt, bnd, nfull == 0, na2, nb2,
                            hmax, lane);
    emit_pair(hmax, g, 2 * lane, gd.count, limit, nullptr, score_sorted, flag);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");   // programmatic dependent of k_intra16 (as k_inter16)
}

// ---------------------------------------------------------------------------
// IntraQP: one column j of the whole query for one subject pair, striped.
//   Hold[k] = H(v*L + k, j-1) in, H(v*L + k, j) out;  Fh[k] = F(., j) in, F(., j+1) out
// ---------------------------------------------------------------------------
template <int L>
__device__ __forceinline__ void col_striped(uint32_t (&Hold)[L], uint32_t (&Fh)[L], const int8_t* __restrict__ plo,
                                            const int8_t* __restrict__ phi, uint32_t na2, uint32_t nb2,
                                            uint32_t& hmax, int lane) {
  uint32_t diag = __shfl_up_sync(0xffffffffu, Hold[L - 1], 1);      // H(v*L - 1, j-1)
  if (lane == 0) diag = 0u;
  uint32_t ev = 0u;                                                 // E entering the segment: fixed below
  uint2 a = *reinterpret_cast<const uint2*>(plo), b = *reinterpret_cast<const uint2*>(phi);
#pragma unroll
  for (int k = 0; k < L; k++) {
    const int rr = k & 7;
    if (rr == 0 && k > 0) {
      a = *reinterpret_cast<const uint2*>(plo + k);
      b = *reinterpret_cast<const uint2*>(phi + k);
    }
    const uint32_t sub = prmt(rr < 4 ? a.x : a.y, rr < 4 ? b.x : b.y, sel_pair(rr & 3));
    const uint32_t h = __vimax3_s16x2(__vadd2(diag, sub), ev, Fh[k]);   // >= 0: ev, Fh >= 0
    diag = Hold[k];
    Hold[k] = h;
    const uint32_t hb = __vadd2(h, nb2);
    Fh[k] = __viaddmax_s16x2_relu(Fh[k], na2, hb);
    ev = __viaddmax_s16x2_relu(ev, na2, hb);
    hmax = __vmaxs2(hmax, h);
  }
  // lazy loop: E leaving lane v-1's segment enters lane v's first row
  for (int wrap = 0; wrap < 32; wrap++) {
    ev = __shfl_up_sync(0xffffffffu, ev, 1);
    if (lane == 0) ev = 0u;
    bool live = true;
#pragma unroll
    for (int k = 0; k < L; k++) {
      // can the incoming E still change H (or the gaps derived from it) at this row?
      // Not if E <= max(H - beta, 0): gaps are clamped at 0, so a
      // zero E is inert (Farrar's test on saturating unsigned lanes).
      const uint32_t hb_old = __vmaxs2(__vadd2(Hold[k], nb2), 0u);
      if (!__any_sync(0xffffffffu, __vcmpgts2(ev, hb_old) != 0u)) { live = false; break; }
      Hold[k] = __vmaxs2(Hold[k], ev);
      hmax = __vmaxs2(hmax, Hold[k]);
      const uint32_t hb = __vadd2(Hold[k], nb2);
      Fh[k] = __vmaxs2(Fh[k], hb);
      ev = __viaddmax_s16x2_relu(ev, na2, hb);
    }
    if (!live) break;
  }
}

// IntraQP ablation of k_intra16: pair items of the long groups, striped.
template <int L, bool SMEM>
__global__ void __launch_bounds__(kInterThreads, 1)
k_intra16_qp(const uint2* __restrict__ words, const GroupDesc* __restrict__ groups, int n_groups, int cut,
             const int8_t* __restrict__ gprof, int stride, int alpha, int beta, int limit,
             int* __restrict__ counter, int* __restrict__ score_sorted, uint8_t* __restrict__ flag) {
  asm volatile("griddepcontrol.launch_dependents;");
  extern __shared__ __align__(16) int8_t sprof[];
  __shared__ int s_split;
  if (threadIdx.x == 0) s_split = split_groups(groups, n_groups, cut);
  __syncthreads();
  const int split = s_split;
  const int n_items = (n_groups - split) * 32;
  if (n_items <= 0) return;
  if (SMEM) load_profile_smem(sprof, gprof, stride);
  const int8_t* prof = prof_base<SMEM>(gprof);
  const int lane = threadIdx.x & 31;
  const uint32_t na2 = pack2(-alpha), nb2 = pack2(-beta);
  const int8_t* pr = prof + lane * L;                                // this lane's query segment
  for (;;) {
    int item = 0;
    if (lane == 0) item = atomicAdd(counter, 1);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= n_items) break;
    const int g = n_groups - 1 - item / 32;
    const int p = 31 - item % 32;
    const GroupDesc gd = groups[g];
    if (2 * p >= gd.count) continue;
    const uint2* pw = words + gd.base + p;
    const int ncols = gd.ncols, nwords = (ncols + kResPerWord - 1) / kResPerWord;
    uint32_t Hold[L], Fh[L], hmax = 0u;
#pragma unroll
    for (int k = 0; k < L; k++) { Hold[k] = 0u; Fh[k] = 0u; }
    uint2 w = make_uint2(kDummyWord, kDummyWord);
    for (int j = 0; j < ncols; j++) {
      const int sh = res_shift(j);
      if (sh == 0) w = j / kResPerWord < nwords ? __ldg(pw + (long long)(j / kResPerWord) * 32) : w;
      col_striped<L>(Hold, Fh, pr + ((w.x >> sh) & 31u) * stride, pr + ((w.y >> sh) & 31u) * stride, na2, nb2,
                     hmax, lane);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) hmax = __vmaxs2(hmax, __shfl_xor_sync(0xffffffffu, hmax, o));
    if (lane == 0) emit_pair(hmax, g, 2 * p, gd.count, limit, nullptr, score_sorted, flag);
  }
}

}  // namespace swk
