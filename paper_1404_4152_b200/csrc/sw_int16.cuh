// sw_int16.cuh -- the int16x2 DPX first pass: cell update, register tiles, inter-task and intra-task kernels (a3, a5)
// Part of the device code of libswsearch (see sw_common.cuh for the overview).
#pragma once
#include "sw_common.cuh"

namespace swk {

// ---------------------------------------------------------------------------
// One column j of R query rows [i0, i0+R) for a pair of subjects (int16x2).
//   in : D[r] = H(i0+r-1, j-1) + fsbt(q_{i0+r}, s_j)   (diagonal term, precomputed)
//        F[r] = F(i0+r, j), e = E(i0, j), htop = H(i0-1, j)
//        plo/phi -> profile rows of the NEXT column's residues (lo/hi subject)
//   out: D[r] = H(i0+r-1, j) + fsbt(q_{i0+r}, s_{j+1}), F[r] = F(i0+r, j+1),
//        e = E(i0+R, j); returns H(i0+R-1, j); hmax folds every H(i, j).
// Per row (two cells): VIMNMX3 + 2 VIADDMNMX.RELU + 1/2 VIMNMX3 + PRMT on the
// alu pipe, 2 VIADD.16x2 on the fma-side pipe (DESIGN.md §"Cell update").
// The diagonal add is done one column ahead so ptxas cannot fuse it into an
// alu-pipe VIADDMNMX, and D is updated in place (no register moves).  (Taking
// E - alpha off the E chain costs a third VIADD.16x2 and measured 3% slower.)
// ---------------------------------------------------------------------------
template <int R, bool A16 = false>
__device__ __forceinline__ uint32_t col16(uint32_t (&D)[R], uint32_t (&F)[R], uint32_t& e, uint32_t htop,
                                          const int8_t* __restrict__ plo, const int8_t* __restrict__ phi,
                                          uint32_t na2, uint32_t nb2, uint32_t& hmax) {
  uint32_t hprev = htop, hodd = 0u;
  if constexpr (A16 && R % 16 == 0) {
    // One LDS.128 per 16 rows per subject (the profile row stride and every full
    // tile's first row are multiples of 16 bytes): half the profile loads.
    uint4 a = *reinterpret_cast<const uint4*>(plo);
    uint4 b = *reinterpret_cast<const uint4*>(phi);
#pragma unroll
    for (int k = 0; k < R / 16; k++) {
      uint4 an = a, bn = b;
      if (k + 1 < R / 16) {
        an = *reinterpret_cast<const uint4*>(plo + 16 * (k + 1));
        bn = *reinterpret_cast<const uint4*>(phi + 16 * (k + 1));
      }
      const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int rr = 0; rr < 16; rr++) {
        const int r = 16 * k + rr;
        const uint32_t h = __vimax3_s16x2(D[r], e, F[r]);
        const uint32_t sn = prmt(aw[rr >> 2], bw[rr >> 2], sel_pair(rr & 3));
        D[r] = __vadd2(hprev, sn);
        const uint32_t hb = __vadd2(h, nb2);
        e = __viaddmax_s16x2_relu(e, na2, hb);
        F[r] = __viaddmax_s16x2_relu(F[r], na2, hb);
        if (rr & 1) hmax = __vimax3_s16x2(hmax, hodd, h);
        else hodd = h;
        hprev = h;
      }
      a = an;
      b = bn;
    }
    return hprev;
  }
  uint2 a = *reinterpret_cast<const uint2*>(plo);
  uint2 b = *reinterpret_cast<const uint2*>(phi);
#pragma unroll
  for (int k = 0; k < R / 8; k++) {
    uint2 an = a, bn = b;
    if (k + 1 < R / 8) {
      an = *reinterpret_cast<const uint2*>(plo + 8 * (k + 1));
      bn = *reinterpret_cast<const uint2*>(phi + 8 * (k + 1));
    }
#pragma unroll
    for (int rr = 0; rr < 8; rr++) {
      const int r = 8 * k + rr;
      const uint32_t h = __vimax3_s16x2(D[r], e, F[r]);          // H(i,j) >= 0 since e, F >= 0
      const uint32_t sn = prmt(rr < 4 ? a.x : a.y, rr < 4 ? b.x : b.y, sel_pair(rr & 3));
      D[r] = __vadd2(hprev, sn);                                 // H(i-1,j) + fsbt(q_i, s_{j+1}); wraps only past LIMIT16
      const uint32_t hb = __vadd2(h, nb2);                       // H(i,j) - beta
      e = __viaddmax_s16x2_relu(e, na2, hb);                     // E(i+1,j) = max(E - alpha, H - beta, 0)
      F[r] = __viaddmax_s16x2_relu(F[r], na2, hb);               // F(i,j+1) = max(F - alpha, H - beta, 0)
      if (rr & 1) hmax = __vimax3_s16x2(hmax, hodd, h);
      else hodd = h;
      hprev = h;
    }
    a = an;
    b = bn;
  }
  return hprev;
}

// Column of R <= 16 rows whose profile bytes for the lane (lo and hi subject)
// are one 16-byte block each (the intra-task "blocked" profile: block b holds
// query rows [b*R, b*R + R), zero-padded).  Same cell update as col16.
template <int R>
__device__ __forceinline__ uint32_t col16b(uint32_t (&D)[R], uint32_t (&F)[R], uint32_t& e, uint32_t htop,
                                           const uint4 a, const uint4 b, uint32_t na2, uint32_t nb2,
                                           uint32_t& hmax) {
  static_assert(R >= 2 && R <= 16, "blocked profile rows");
  uint32_t hprev = htop, hodd = 0u;
#pragma unroll
  for (int r = 0; r < R; r++) {
    const uint32_t wa = r < 4 ? a.x : r < 8 ? a.y : r < 12 ? a.z : a.w;
    const uint32_t wb = r < 4 ? b.x : r < 8 ? b.y : r < 12 ? b.z : b.w;
    const uint32_t h = __vimax3_s16x2(D[r], e, F[r]);
    const uint32_t sn = prmt(wa, wb, sel_pair(r & 3));
    D[r] = __vadd2(hprev, sn);
    const uint32_t hb = __vadd2(h, nb2);
    e = __viaddmax_s16x2_relu(e, na2, hb);
    F[r] = __viaddmax_s16x2_relu(F[r], na2, hb);
    if (r & 1) hmax = __vimax3_s16x2(hmax, hodd, h);
    else hodd = h;
    hprev = h;
  }
  if (R & 1) hmax = __vmaxs2(hmax, hodd);
  return hprev;
}

// Residue cursor over one lane's interleaved packed words (6 codes per word).

// ---------------------------------------------------------------------------
// Inter-task tile: rows [i0, i0+R) of the query against all columns of one
// pair of subjects per lane (32 pairs = one 64-subject group per warp).
// bnd[j] carries (E(i0,j), H(i0-1,j)) in and (E(i0+R,j), H(i0+R-1,j)) out
// between tiles (the paper's "tiled SW computation").
// ---------------------------------------------------------------------------
// Two consecutive columns A = j and B = j+1 interleaved with a one-row skew:
// step r does A(row r) and B(row r-1).  B(row r') only needs D[r'], F[r'] as
// left by A(row r') and B's own E chain, so every step carries two independent
// dependency chains (the fixed-latency "wait" stall of the single-column loop).
template <int R>
__device__ __forceinline__ void col16x2(uint32_t (&D)[R], uint32_t (&F)[R],
                                        uint32_t& eA, uint32_t htopA, const int8_t* __restrict__ ploA,
                                        const int8_t* __restrict__ phiA, uint32_t& eB, uint32_t htopB,
                                        const int8_t* __restrict__ ploB, const int8_t* __restrict__ phiB,
                                        uint32_t na2, uint32_t nb2, uint32_t& hmax, uint32_t& hlA,
                                        uint32_t& hlB) {
  uint32_t hpA = htopA, hpB = htopB, hoA = 0u, hoB = 0u;
  uint2 aA = *reinterpret_cast<const uint2*>(ploA), bA = *reinterpret_cast<const uint2*>(phiA);
  uint2 aB = *reinterpret_cast<const uint2*>(ploB), bB = *reinterpret_cast<const uint2*>(phiB);
  uint2 aBn = aB, bBn = bB;
#pragma unroll
  for (int r = 0; r <= R; r++) {
    if (r < R) {                                   // ---- column A, row r
      const int rr = r & 7;
      if (rr == 0 && r > 0) {
        aA = *reinterpret_cast<const uint2*>(ploA + r);
        bA = *reinterpret_cast<const uint2*>(phiA + r);
      }
      const uint32_t h = __vimax3_s16x2(D[r], eA, F[r]);
      const uint32_t sn = prmt(rr < 4 ? aA.x : aA.y, rr < 4 ? bA.x : bA.y, sel_pair(rr & 3));
      D[r] = __vadd2(hpA, sn);
      const uint32_t hb = __vadd2(h, nb2);
      eA = __viaddmax_s16x2_relu(eA, na2, hb);
      F[r] = __viaddmax_s16x2_relu(F[r], na2, hb);
      if (rr & 1) hmax = __vimax3_s16x2(hmax, hoA, h);
      else hoA = h;
      hpA = h;
    }
    if (r >= 1) {                                  // ---- column B, row r-1
      const int q = r - 1, rr = q & 7;
      if (rr == 0 && q > 0) {
        aB = aBn;
        bB = bBn;
      }
      if (rr == 0 && q + 8 < R) {                  // B's next chunk, one chunk ahead
        aBn = *reinterpret_cast<const uint2*>(ploB + q + 8);
        bBn = *reinterpret_cast<const uint2*>(phiB + q + 8);
      }
      const uint32_t h = __vimax3_s16x2(D[q], eB, F[q]);
      const uint32_t sn = prmt(rr < 4 ? aB.x : aB.y, rr < 4 ? bB.x : bB.y, sel_pair(rr & 3));
      D[q] = __vadd2(hpB, sn);
      const uint32_t hb = __vadd2(h, nb2);
      eB = __viaddmax_s16x2_relu(eB, na2, hb);
      F[q] = __viaddmax_s16x2_relu(F[q], na2, hb);
      if (rr & 1) hmax = __vimax3_s16x2(hmax, hoB, h);
      else hoB = h;
      hpB = h;
    }
  }
  hlA = hpA;
  hlB = hpB;
}

// Packed residue pair (lo, hi codes) of column c of this lane: word c/6, field c%6.

template <int R, bool A16 = (R % 16 == 0)>   // A16: this tile's first profile row is 16-byte aligned
__device__ __forceinline__ void tile16(const uint2* __restrict__ gw, int ncols,
                                       const int8_t* __restrict__ prof, int stride, int i0,
                                       uint2* __restrict__ bnd, bool first, bool last,
                                       uint32_t na2, uint32_t nb2, uint32_t& hmax, int lane) {
  if (ncols <= 0) return;
  uint32_t D[R], F[R];
#pragma unroll
  for (int r = 0; r < R; r++) { D[r] = 0u; F[r] = 0u; }
  const uint2* lw = gw + lane;
  const int nwords = (ncols + kResPerWord - 1) / kResPerWord;
  const int8_t* pr = prof + i0;
  {  // virtual column j = -1 (all-zero boundary): primes D[r] = fsbt(q_{i0+r}, s_0)
    const uint2 w0 = lw[0];
    uint32_t e0 = 0u;
    col16<R, A16>(D, F, e0, 0u, pr + (w0.x & 31u) * stride, pr + (w0.y & 31u) * stride, na2, nb2, hmax);
  }
  // Columns are taken two at a time (A = j, B = j+1).  The residue words of the
  // next pair's "next columns" (j+3, j+4) and its boundary rows (j+2, j+3) are
  // loaded one pair ahead into the registers they are consumed from.
  const uint2 z = make_uint2(0u, 0u);
  uint2 bE = first ? z : bnd[lane];
  uint2 bO = (first || ncols < 2) ? z : bnd[32 + lane];
  uint2 wA = res_word(lw, 1, nwords), wB = res_word(lw, 2, nwords);
  int j = 0;
  for (; j + 1 < ncols; j += 2) {
    const int shA = res_shift(j + 1), shB = res_shift(j + 2);
    uint32_t eA = bE.x, eB = bO.x, hlA, hlB;
    const uint32_t tA = bE.y, tB = bO.y;
    // The next pair's tile-edge rows are requested as soon as this pair's are
    // consumed: both columns (~700 instructions per warp) cover the DRAM latency
    // instead of the tail of the second one (C5 first pass -0.7 %).
    if (!first && j + 2 < ncols) bE = bnd[(j + 2) * 32 + lane];
    if (!first && j + 3 < ncols) bO = bnd[(j + 3) * 32 + lane];
#ifdef SW_INTERLEAVE_COLUMNS
    col16x2<R>(D, F, eA, tA, pr + ((wA.x >> shA) & 31u) * stride, pr + ((wA.y >> shA) & 31u) * stride,
               eB, tB, pr + ((wB.x >> shB) & 31u) * stride, pr + ((wB.y >> shB) & 31u) * stride,
               na2, nb2, hmax, hlA, hlB);
#else
    hlA = col16<R, A16>(D, F, eA, tA, pr + ((wA.x >> shA) & 31u) * stride, pr + ((wA.y >> shA) & 31u) * stride,
                   na2, nb2, hmax);
    hlB = col16<R, A16>(D, F, eB, tB, pr + ((wB.x >> shB) & 31u) * stride, pr + ((wB.y >> shB) & 31u) * stride,
                   na2, nb2, hmax);
#endif
    wA = res_word(lw, j + 3, nwords);
    wB = res_word(lw, j + 4, nwords);
    if (!last) {
      bnd[j * 32 + lane] = make_uint2(eA, hlA);
      bnd[(j + 1) * 32 + lane] = make_uint2(eB, hlB);
    }
  }
  if (j < ncols) {                                 // odd tail column
    const int shA = res_shift(j + 1);
    uint32_t e = bE.x;
    const uint32_t hl = col16<R, A16>(D, F, e, bE.y, pr + ((wA.x >> shA) & 31u) * stride,
                                 pr + ((wA.y >> shA) & 31u) * stride, na2, nb2, hmax);
    if (!last) bnd[j * 32 + lane] = make_uint2(e, hl);
  }
}

template <int T, int R = T - 8>
__device__ __forceinline__ void tile16_rem(int rem, const uint2* gw, int ncols, const int8_t* prof,
                                           int stride, int i0, uint2* bnd, bool first,
                                           uint32_t na2, uint32_t nb2, uint32_t& hmax, int lane) {
  if constexpr (R >= 8) {
    if (rem == R) tile16<R, (T % 16 == 0) && (R % 16 == 0)>(gw, ncols, prof, stride, i0, bnd, first, true, na2, nb2, hmax, lane);
    else tile16_rem<T, R - 8>(rem, gw, ncols, prof, stride, i0, bnd, first, na2, nb2, hmax, lane);
  }
}

// One 64-subject group, all query tiles (inter-task).  Not inlined, so the
// register-hungry tile loop is allocated apart from the persistent queue logic.
template <int T, bool SMEM>
__device__ __forceinline__ uint32_t inter_group16(const uint2* __restrict__ gw, int ncols, const int8_t* __restrict__ gprof,
                                               int stride, int m_pad, uint2* __restrict__ bnd, uint32_t na2,
                                               uint32_t nb2, int lane) {
  const int8_t* prof = prof_base<SMEM>(gprof);
  const int nfull = m_pad / T, rem = m_pad - nfull * T;
  uint32_t hmax = 0u;
  for (int t = 0; t < nfull; t++)
    tile16<T>(gw, ncols, prof, stride, t * T, bnd, t == 0, t == nfull - 1 && rem == 0, na2, nb2, hmax, lane);
  if (rem) tile16_rem<T>(rem, gw, ncols, prof, stride, nfull * T, bnd, nfull == 0, na2, nb2, hmax, lane);
  return hmax;
}

// ---------------------------------------------------------------------------
// Intra-task wavefront for ONE pair of long subjects per warp (north star (c);
// the role of the paper's intra-sequence model, with a
// wavefront instead of Farrar striping).  Lane l owns query rows
// [base + l*TR, base + (l+1)*TR) of a pass of 32*TR rows.  Columns are taken
// two at a time: at step s lane l aligns the column pair k = s - l, i.e.
// columns A = 2k-1 and B = 2k (column -1 is the all-zero boundary that primes
// the diagonal terms), interleaved with a one-row skew so every step carries
// two independent dependency chains; (E, H) of both columns and the next
// residues flow to lane l+1 by SHFL.  The last active lane's output rows are
// kept in gbnd for the next pass.  Returns this lane's running max.
// ---------------------------------------------------------------------------
template <int R>
__device__ __forceinline__ void col16b_x2(uint32_t (&D)[R], uint32_t (&F)[R], uint32_t& eA, uint32_t htopA,
                                          const uint4 a1, const uint4 b1, uint32_t& eB, uint32_t htopB,
                                          const uint4 a2, const uint4 b2, uint32_t na2, uint32_t nb2,
                                          uint32_t& hmax, uint32_t& hlA, uint32_t& hlB) {
  uint32_t hpA = htopA, hpB = htopB, hA = 0u;
#pragma unroll
  for (int r = 0; r <= R; r++) {
    if (r < R) {                                                  // column A, row r
      const uint32_t wa = r < 4 ? a1.x : r < 8 ? a1.y : r < 12 ? a1.z : a1.w;
      const uint32_t wb = r < 4 ? b1.x : r < 8 ? b1.y : r < 12 ? b1.z : b1.w;
      hA = __vimax3_s16x2(D[r], eA, F[r]);
      D[r] = __vadd2(hpA, prmt(wa, wb, sel_pair(r & 3)));         // H(i-1,A) + fsbt(q_i, s_B)
      const uint32_t hb = __vadd2(hA, nb2);
      eA = __viaddmax_s16x2_relu(eA, na2, hb);
      F[r] = __viaddmax_s16x2_relu(F[r], na2, hb);
      hpA = hA;
      if (r == 0) hmax = __vmaxs2(hmax, hA);                     // rows 1.. are folded with column B
    }
    if (r >= 1) {                                                 // column B, row r-1
      const int q = r - 1;
      const uint32_t wa = q < 4 ? a2.x : q < 8 ? a2.y : q < 12 ? a2.z : a2.w;
      const uint32_t wb = q < 4 ? b2.x : q < 8 ? b2.y : q < 12 ? b2.z : b2.w;
      const uint32_t h = __vimax3_s16x2(D[q], eB, F[q]);
      D[q] = __vadd2(hpB, prmt(wa, wb, sel_pair(q & 3)));         // H(i-1,B) + fsbt(q_i, s_{B+1})
      const uint32_t hb = __vadd2(h, nb2);
      eB = __viaddmax_s16x2_relu(eB, na2, hb);
      F[q] = __viaddmax_s16x2_relu(F[q], na2, hb);
      if (r < R) hmax = __vimax3_s16x2(hmax, h, hA);             // H(q, B) and H(r, A)
      else hmax = __vmaxs2(hmax, h);
      hpB = h;
    }
  }
  hlA = hpA;
  hlB = hpB;
}

template <int TR, bool SMEM>
__device__ __forceinline__ uint32_t intra_pair16(const uint2* __restrict__ pw, int ncols,
                                                 const int8_t* __restrict__ gprof, int stride, int m_pad,
                                                 uint2* __restrict__ gbnd, long long gstride,
                                                 uint32_t na2, uint32_t nb2, int lane) {
  const int8_t* prof = prof_base<SMEM>(gprof);
  uint32_t hmax = 0u;
  const int nwords = (ncols + kResPerWord - 1) / kResPerWord;
  const int K = (ncols + 2) / 2;                                        // column pairs (-1,0), (1,2), ...
  int pass = 0;
  for (int base = 0; base < m_pad; base += 32 * TR, pass++) {
    const int nact = min(32, (m_pad - base + TR - 1) / TR);
    const bool first = base == 0, last = base + 32 * TR >= m_pad;
    const uint2* gin = gbnd + (long long)(pass & 1) * gstride;          // written by the previous pass
    uint2* gout = gbnd + (long long)((pass + 1) & 1) * gstride;
    const int8_t* pr = prof + (base / TR + lane) * 16;                 // this lane's 16-byte profile block
    uint32_t D[TR], F[TR];
#pragma unroll
    for (int r = 0; r < TR; r++) { D[r] = 0u; F[r] = 0u; }
    uint32_t eA_out = 0u, hA_out = 0u, eB_out = 0u, hB_out = 0u, r_out = 0u;
    // Lane 0's per-step inputs for pair k (residues of columns 2k and 2k+1, and
    // after the first pass the previous pass's boundary of columns 2k-1, 2k) are
    // fetched by all lanes 32 pairs at a time, one block ahead, and handed over by SHFL.
    auto fetch = [&](int kb, uint32_t& rp, uint2& ga, uint2& gb) {
      const int k = kb + lane;
      const int c0 = 2 * k, c1 = 2 * k + 1;
      const uint2 w0 = res_word(pw, c0, nwords), w1 = res_word(pw, c1, nwords);
      const int s0 = res_shift(c0), s1 = res_shift(c1);
      rp = ((w0.x >> s0) & 31u) | (((w0.y >> s0) & 31u) << 5) | (((w1.x >> s1) & 31u) << 10) |
           (((w1.y >> s1) & 31u) << 15);
      const int ca = 2 * k - 1, cb = 2 * k;
      ga = (!first && ca >= 0 && ca < ncols) ? gin[ca] : make_uint2(0u, 0u);
      gb = (!first && cb < ncols) ? gin[cb] : make_uint2(0u, 0u);
    };
    const int nsteps = K + nact - 1;
    uint32_t rp_cur, rp_nxt;
    uint2 ga_cur, gb_cur, ga_nxt, gb_nxt;
    fetch(0, rp_cur, ga_cur, gb_cur);
    fetch(32, rp_nxt, ga_nxt, gb_nxt);
    __syncwarp();
    for (int sb = 0; sb < nsteps; sb += 32) {
#pragma unroll 1
      for (int t = 0; t < 32; t++) {
        const int s = sb + t;
        if (s >= nsteps) break;
        uint32_t eA = __shfl_up_sync(0xffffffffu, eA_out, 1);
        uint32_t hA = __shfl_up_sync(0xffffffffu, hA_out, 1);
        uint32_t eB = __shfl_up_sync(0xffffffffu, eB_out, 1);
        uint32_t hB = __shfl_up_sync(0xffffffffu, hB_out, 1);
        uint32_t r_in = __shfl_up_sync(0xffffffffu, r_out, 1);
        const uint32_t r0 = __shfl_sync(0xffffffffu, rp_cur, t);
        const uint32_t gax = __shfl_sync(0xffffffffu, ga_cur.x, t), gay = __shfl_sync(0xffffffffu, ga_cur.y, t);
        const uint32_t gbx = __shfl_sync(0xffffffffu, gb_cur.x, t), gby = __shfl_sync(0xffffffffu, gb_cur.y, t);
        const int k = s - lane;
        if (lane == 0) {
          r_in = r0;                                                    // residues of columns 2k, 2k+1
          eA = gax;                                                     // E(base, A), H(base-1, A)
          hA = gay;
          eB = gbx;                                                     // E(base, B), H(base-1, B)
          hB = gby;
        }
        if (lane < nact && k >= 0 && k < K) {
          const uint4 a1 = *reinterpret_cast<const uint4*>(pr + (r_in & 31u) * stride);
          const uint4 b1 = *reinterpret_cast<const uint4*>(pr + ((r_in >> 5) & 31u) * stride);
          const uint4 a2 = *reinterpret_cast<const uint4*>(pr + ((r_in >> 10) & 31u) * stride);
          const uint4 b2 = *reinterpret_cast<const uint4*>(pr + ((r_in >> 15) & 31u) * stride);
          uint32_t hlA, hlB;
          col16b_x2<TR>(D, F, eA, hA, a1, b1, eB, hB, a2, b2, na2, nb2, hmax, hlA, hlB);
          eA_out = eA;
          hA_out = hlA;
          eB_out = eB;
          hB_out = hlB;
          r_out = r_in;
          if (!last && lane == nact - 1) {
            const int ca = 2 * k - 1, cb = 2 * k;
            if (ca >= 0) gout[ca] = make_uint2(eA, hlA);
            if (cb < ncols) gout[cb] = make_uint2(eB, hlB);
          }
        }
      }
      rp_cur = rp_nxt;
      ga_cur = ga_nxt;
      gb_cur = gb_nxt;
      fetch(sb + 64, rp_nxt, ga_nxt, gb_nxt);
    }
    __syncwarp();
  }
  return hmax;
}


// NC columns per wavefront step (NC = 4: twice the work per step of
// intra_pair16, so the per-step SHFL / profile-load / loop latency is paid once
// per four columns).  Column c of step s on lane l is NC*k - 1 + c, k = s - l,
// run with a c-row skew; D, F are shared in place as in col16b_x2.
template <int R, int NC>
__device__ __forceinline__ void col16b_xn(uint32_t (&D)[R], uint32_t (&F)[R], uint32_t (&e)[NC],
                                          uint32_t (&hp)[NC], const uint4 (&pa)[NC], const uint4 (&pb)[NC],
                                          uint32_t na2, uint32_t nb2, uint32_t& hmax) {
  // The running max is folded into two accumulators, alternating per pair of
  // cells, so its dependency chain is half as long as the step's cell count
  // (one chain serialised the latency-bound wavefront).
  uint32_t pend = 0u, hmax2 = 0u;
  int npend = 0, acc = 0;
#pragma unroll
  for (int r = 0; r < R + NC - 1; r++) {
#pragma unroll
    for (int c = 0; c < NC; c++) {
      const int q = r - c;
      if (q >= 0 && q < R) {
        const uint32_t wa = q < 4 ? pa[c].x : q < 8 ? pa[c].y : q < 12 ? pa[c].z : pa[c].w;
        const uint32_t wb = q < 4 ? pb[c].x : q < 8 ? pb[c].y : q < 12 ? pb[c].z : pb[c].w;
        const uint32_t h = __vimax3_s16x2(D[q], e[c], F[q]);
        D[q] = __vadd2(hp[c], prmt(wa, wb, sel_pair(q & 3)));   // H(i-1, col) + fsbt(q_i, s_{col+1})
        const uint32_t hb = __vadd2(h, nb2);
        e[c] = __viaddmax_s16x2_relu(e[c], na2, hb);
        F[q] = __viaddmax_s16x2_relu(F[q], na2, hb);
        hp[c] = h;
        if (npend) {
          if (acc) hmax2 = __vimax3_s16x2(hmax2, pend, h);
          else hmax = __vimax3_s16x2(hmax, pend, h);
          acc ^= 1;
        } else {
          pend = h;
        }
        npend ^= 1;
      }
    }
  }
  hmax = npend ? __vimax3_s16x2(hmax, hmax2, pend) : __vmaxs2(hmax, hmax2);
}

template <int TR, bool SMEM, int NC>
__device__ __forceinline__ uint32_t intra_multi16(const uint2* __restrict__ pw, int ncols,
                                                  const int8_t* __restrict__ gprof, int stride, int m_pad,
                                                  uint2* __restrict__ gbnd, long long gstride,
                                                  uint32_t na2, uint32_t nb2, int lane) {
  static_assert(NC == 2 || NC == 4 || NC == 8, "columns per step");
  constexpr int NR = NC / 2;                                              // residue words (4 codes each)
  const int8_t* prof = prof_base<SMEM>(gprof);
  uint32_t hmax = 0u;
  const int nwords = (ncols + kResPerWord - 1) / kResPerWord;
  const int K = (ncols + NC) / NC;                                        // steps of NC columns from -1
  int pass = 0;
  for (int base = 0; base < m_pad; base += 32 * TR, pass++) {
    const int nact = min(32, (m_pad - base + TR - 1) / TR);
    const bool first = base == 0, last = base + 32 * TR >= m_pad;
    const uint2* gin = gbnd + (long long)(pass & 1) * gstride;
    uint2* gout = gbnd + (long long)((pass + 1) & 1) * gstride;
    const int8_t* pr = prof + (base / TR + lane) * 16;
    uint32_t D[TR], F[TR];
#pragma unroll
    for (int r = 0; r < TR; r++) { D[r] = 0u; F[r] = 0u; }
    uint32_t e_out[NC], h_out[NC], r_out[NR];
#pragma unroll
    for (int c = 0; c < NC; c++) { e_out[c] = 0u; h_out[c] = 0u; }
#pragma unroll
    for (int i = 0; i < NR; i++) r_out[i] = 0u;
    // lane 0's inputs of step k (residues of columns NC*k .. NC*k+NC-1, and the
    // previous pass's boundary of columns NC*k-1 ..), fetched 32 steps at a time
    auto fetch = [&](int kb, uint32_t (&rp)[NR], uint2 (&g)[NC]) {
      const int k = kb + lane;
#pragma unroll
      for (int i = 0; i < NR; i++) {
        const int c0 = NC * k + 2 * i, c1 = c0 + 1;
        const uint2 w0 = res_word(pw, c0, nwords), w1 = res_word(pw, c1, nwords);
        const int s0 = res_shift(c0), s1 = res_shift(c1);
        rp[i] = ((w0.x >> s0) & 31u) | (((w0.y >> s0) & 31u) << 5) | (((w1.x >> s1) & 31u) << 10) |
                (((w1.y >> s1) & 31u) << 15);
      }
#pragma unroll
      for (int c = 0; c < NC; c++) {
        const int col = NC * k - 1 + c;
        g[c] = (!first && col >= 0 && col < ncols) ? gin[col] : make_uint2(0u, 0u);
      }
    };
    const int nsteps = K + nact - 1;
    uint32_t rp_cur[NR], rp_nxt[NR];
    uint2 g_cur[NC], g_nxt[NC];
    fetch(0, rp_cur, g_cur);
    fetch(32, rp_nxt, g_nxt);
    __syncwarp();
    for (int sb = 0; sb < nsteps; sb += 32) {
#pragma unroll 1
      for (int t = 0; t < 32; t++) {
        const int s = sb + t;
        if (s >= nsteps) break;
        uint32_t e[NC], hp[NC], r_in[NR];
#pragma unroll
        for (int c = 0; c < NC; c++) {
          e[c] = __shfl_up_sync(0xffffffffu, e_out[c], 1);
          hp[c] = __shfl_up_sync(0xffffffffu, h_out[c], 1);
        }
#pragma unroll
        for (int i = 0; i < NR; i++) r_in[i] = __shfl_up_sync(0xffffffffu, r_out[i], 1);
#pragma unroll
        for (int i = 0; i < NR; i++) {
          const uint32_t v = __shfl_sync(0xffffffffu, rp_cur[i], t);
          if (lane == 0) r_in[i] = v;
        }
#pragma unroll
        for (int c = 0; c < NC; c++) {
          const uint32_t gx = __shfl_sync(0xffffffffu, g_cur[c].x, t), gy = __shfl_sync(0xffffffffu, g_cur[c].y, t);
          if (lane == 0) { e[c] = gx; hp[c] = gy; }                       // E(base, col), H(base-1, col)
        }
        const int k = s - lane;
        if (lane < nact && k >= 0 && k < K) {
          uint4 pa[NC], pb[NC];
#pragma unroll
          for (int c = 0; c < NC; c++) {
            const uint32_t rr = r_in[c >> 1] >> (10 * (c & 1));
            pa[c] = *reinterpret_cast<const uint4*>(pr + (rr & 31u) * stride);
            pb[c] = *reinterpret_cast<const uint4*>(pr + ((rr >> 5) & 31u) * stride);
          }
          col16b_xn<TR, NC>(D, F, e, hp, pa, pb, na2, nb2, hmax);
#pragma unroll
          for (int c = 0; c < NC; c++) { e_out[c] = e[c]; h_out[c] = hp[c]; }
#pragma unroll
          for (int i = 0; i < NR; i++) r_out[i] = r_in[i];
          if (!last && lane == nact - 1) {
#pragma unroll
            for (int c = 0; c < NC; c++) {
              const int col = NC * k - 1 + c;
              if (col >= 0 && col < ncols) gout[col] = make_uint2(e[c], hp[c]);
            }
          }
        }
      }
#pragma unroll
      for (int i = 0; i < NR; i++) rp_cur[i] = rp_nxt[i];
#pragma unroll
      for (int c = 0; c < NC; c++) g_cur[c] = g_nxt[c];
      fetch(sb + 64, rp_nxt, g_nxt);
    }
    __syncwarp();
  }
  return hmax;
}

// Streamed databases (f2): the first chunk of a search arrives in pieces while
// the first pass already runs; ready_from holds the lowest word index known to
// have landed (written by the copy engine after each piece, longest groups
// first).  A warp waits here until its group's words are in.  nullptr: no wait.
__device__ __forceinline__ void wait_words_ready(const long long* ready_from, long long base) {
  if (ready_from) {
    if ((threadIdx.x & 31) == 0) {
      for (;;) {
        long long v;
        asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(ready_from) : "memory");
        if (v <= base) break;
        __nanosleep(200);
      }
    }
    __syncwarp();
  }
}

// Column segments of ONE pair for the latency-critical longest pairs (single
// pass, NC columns per step): step k covers columns c0 + NC*k - 1 .. c0 + NC*k
// + NC - 2 (column c0 - 1 primes the diagonal terms, as column -1 does in
// intra_multi16).
//   mode 0: from the zero state (the pair's first segment, c0 = 0); the lanes'
//           final rows (D, F) go to `state` (2*TR words per lane, [r][lane]).
//   mode 1: speculative -- from a zero left boundary (H(., c0 - 1) = 0); every
//           kCkSteps steps each lane stores its rows in `ckpt`.
//   mode 2: fix-up -- from the true rows in `state` (the previous segment's
//           end); at every checkpoint each lane compares its rows with the
//           speculative ones, the verdict is AND-ed down the lanes, and once the
//           last lane sees all rows equal, every later column is the
//           speculative run's and the pass stops.
// Eq. 1 is monotone in its left boundary, so the speculative cells are lower
// bounds of the true ones: the segment's maximum is max(speculative, fix-up).
constexpr int kCkSteps = 16;
constexpr int kSplitMinCols = 1024;   // shorter critical pairs run whole on warp 0

template <int TR, bool SMEM, int NC>
__device__ __forceinline__ uint32_t intra_seg16(const uint2* __restrict__ pw, int ncols, int c0, int K,
                                                const int8_t* __restrict__ gprof, int stride, int m_pad,
                                                uint32_t na2, uint32_t nb2, int lane, int mode,
                                                uint32_t* __restrict__ ckpt, uint32_t* __restrict__ state) {
  constexpr int NR = NC / 2;
  const int8_t* pr = prof_base<SMEM>(gprof) + lane * 16;
  const int nwords = (ncols + kResPerWord - 1) / kResPerWord;
  const int nact = min(32, (m_pad + TR - 1) / TR);
  uint32_t D[TR], F[TR];
#pragma unroll
  for (int r = 0; r < TR; r++) {
    D[r] = mode == 2 ? state[r * 32 + lane] : 0u;
    F[r] = mode == 2 ? state[(TR + r) * 32 + lane] : 0u;
  }
  uint32_t hmax = 0u, e_out[NC], h_out[NC], r_out[NR], f_out = 1u;
#pragma unroll
  for (int c = 0; c < NC; c++) { e_out[c] = 0u; h_out[c] = 0u; }
#pragma unroll
  for (int i = 0; i < NR; i++) r_out[i] = 0u;
  auto fetch = [&](int kb, uint32_t (&rp)[NR]) {
    const int k = kb + lane;
#pragma unroll
    for (int i = 0; i < NR; i++) {
      const int a = c0 + NC * k + 2 * i, b = a + 1;
      const uint2 w0 = res_word(pw, a, nwords), w1 = res_word(pw, b, nwords);
      const int s0 = res_shift(a), s1 = res_shift(b);
      rp[i] = ((w0.x >> s0) & 31u) | (((w0.y >> s0) & 31u) << 5) | (((w1.x >> s1) & 31u) << 10) |
              (((w1.y >> s1) & 31u) << 15);
    }
  };
  const int nsteps = K + nact - 1;
  uint32_t rp_cur[NR], rp_nxt[NR];
  fetch(0, rp_cur);
  fetch(32, rp_nxt);
  bool done = false;
  for (int sb = 0; sb < nsteps && !done; sb += 32) {
#pragma unroll 1
    for (int t = 0; t < 32; t++) {
      const int s = sb + t;
      if (s >= nsteps) break;
      uint32_t e[NC], hp[NC], r_in[NR];
#pragma unroll
      for (int c = 0; c < NC; c++) {
        e[c] = __shfl_up_sync(0xffffffffu, e_out[c], 1);
        hp[c] = __shfl_up_sync(0xffffffffu, h_out[c], 1);
      }
#pragma unroll
      for (int i = 0; i < NR; i++) r_in[i] = __shfl_up_sync(0xffffffffu, r_out[i], 1);
      uint32_t f_in = __shfl_up_sync(0xffffffffu, f_out, 1);
#pragma unroll
      for (int i = 0; i < NR; i++) {
        const uint32_t v = __shfl_sync(0xffffffffu, rp_cur[i], t);
        if (lane == 0) r_in[i] = v;
      }
      if (lane == 0) {
        f_in = 1u;
#pragma unroll
        for (int c = 0; c < NC; c++) { e[c] = 0u; hp[c] = 0u; }      // E(0, col) = H(-1, col) = 0
      }
      const int k = s - lane;
      uint32_t conv = 0u;
      if (lane < nact && k >= 0 && k < K) {
        uint4 pa[NC], pb[NC];
#pragma unroll
        for (int c = 0; c < NC; c++) {
          const uint32_t rr = r_in[c >> 1] >> (10 * (c & 1));
          pa[c] = *reinterpret_cast<const uint4*>(pr + (rr & 31u) * stride);
          pb[c] = *reinterpret_cast<const uint4*>(pr + ((rr >> 5) & 31u) * stride);
        }
        col16b_xn<TR, NC>(D, F, e, hp, pa, pb, na2, nb2, hmax);
        if (mode != 0 && (k % kCkSteps) == kCkSteps - 1) {
          uint32_t* ck = ckpt + (long long)(k / kCkSteps) * (2 * TR * 32);
          if (mode == 1) {
#pragma unroll
            for (int r = 0; r < TR; r++) { ck[r * 32 + lane] = D[r]; ck[(TR + r) * 32 + lane] = F[r]; }
          } else {
            bool eq = f_in != 0u;
#pragma unroll
            for (int r = 0; r < TR; r++) eq = eq && ck[r * 32 + lane] == D[r] && ck[(TR + r) * 32 + lane] == F[r];
            f_in = eq ? 1u : 0u;
            conv = (eq && lane == nact - 1) ? 1u : 0u;
          }
        }
      }
#pragma unroll
      for (int c = 0; c < NC; c++) { e_out[c] = e[c]; h_out[c] = hp[c]; }
#pragma unroll
      for (int i = 0; i < NR; i++) r_out[i] = r_in[i];
      f_out = f_in;
      if (mode == 2 && __shfl_sync(0xffffffffu, conv, nact - 1)) {   // all rows equal: the rest is speculative's
        done = true;
        break;
      }
    }
#pragma unroll
    for (int i = 0; i < NR; i++) rp_cur[i] = rp_nxt[i];
    fetch(sb + 64, rp_nxt);
  }
  if (mode == 0) {
#pragma unroll
    for (int r = 0; r < TR; r++) { state[r * 32 + lane] = D[r]; state[(TR + r) * 32 + lane] = F[r]; }
  }
  __syncwarp();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) hmax = __vmaxs2(hmax, __shfl_xor_sync(0xffffffffu, hmax, o));
  return hmax;
}

// Single-pass intra-task items chained through the lanes (m_pad <= 32*TR, NC
// columns per step).  intra_multi16 fills and drains the lane wavefront for every
// pair item: nact - 1 of its K + nact - 1 steps run with idle lanes (C1: ~25 % of
// the steps).  Here lane 0 starts the next item at the step after it finished the
// current one, while the lanes below still finish theirs: the warp runs one
// stream of steps over consecutive items of the work queue.  Each step's control
// word (item index, first / last step) travels down the lanes with the E/H and
// residue values it belongs to; a lane resets its rows at an item's first step,
// and at its last step passes max(own running max, the one from above) on, so
// the last active lane holds the pair's score and emits it.  Items are claimed
// (and their residues decoded, one step per lane) a block of 32 steps ahead.
constexpr uint32_t kCtlVoid = 0xffffffffu, kCtlFirst = 1u << 29, kCtlLast = 1u << 30, kCtlItem = (1u << 29) - 1;

template <int TR, bool SMEM, int NC>
__device__ __forceinline__ void intra_chain16(const uint2* __restrict__ words, const GroupDesc* __restrict__ groups,
                                              int n_groups, int n_items, int first_item, int n_warps,
                                              int* __restrict__ counter, const int* __restrict__ len_sorted,
                                              const long long* __restrict__ ready_from,
                                              const int8_t* __restrict__ gprof, int stride, int m_pad,
                                              uint32_t na2, uint32_t nb2, int limit, const int* __restrict__ pos_map,
                                              int* __restrict__ score_sorted, uint8_t* __restrict__ flag, int lane) {
  static_assert(NC == 4 || NC == 8, "columns per step");
  constexpr int NR = NC / 2;
  const int8_t* pr = prof_base<SMEM>(gprof) + lane * 16;
  const int nact = min(32, (m_pad + TR - 1) / TR);
  // ---- the item stream (warp-uniform): claimed in queue order, mapped to steps
  int next_claim = first_item;              // the dealt first item, then the counter
  int it = -1, itK = 0, itk = 0;            // item being mapped, its steps, next step to map
  int it_ncols = 0, it_nwords = 0;
  const uint2* it_pw = nullptr;
  bool exhausted = false;
  long long mapped = 0;                     // steps mapped so far (stream positions)
  auto claim = [&]() {
    for (;;) {
      int x;
      if (next_claim >= 0) {
        x = next_claim;
        next_claim = -1;
      } else {
        x = 0;
        if (lane == 0) x = n_warps + atomicAdd(counter, 1);
        x = __shfl_sync(0xffffffffu, x, 0);
      }
      if (x >= n_items) { exhausted = true; it = -1; return; }
      const int g = n_groups - 1 - x / 32, p = 31 - x % 32;
      const GroupDesc gd = groups[g];
      if (2 * p >= gd.count) continue;
      wait_words_ready(ready_from, gd.base);
      it = x;
      it_ncols = len_sorted ? len_sorted[(long long)g * kGroup + min(2 * p + 1, gd.count - 1)] : gd.ncols;
      it_nwords = (it_ncols + kResPerWord - 1) / kResPerWord;
      it_pw = words + gd.base + p;
      itK = (it_ncols + NC) / NC;
      itk = 0;
      return;
    }
  };
  // descriptors of the next 32 stream positions: lane t gets position base + t
  auto gen = [&](uint32_t (&rp)[NR], uint32_t& ctl) {
    ctl = kCtlVoid;
#pragma unroll
    for (int i = 0; i < NR; i++) rp[i] = 0u;
    int t0 = 0;
    while (t0 < 32) {
      if (it < 0 || itk >= itK) {
        if (exhausted) break;
        claim();
        if (it < 0) break;
      }
      const int take = min(32 - t0, itK - itk);
      if (lane >= t0 && lane < t0 + take) {
        const int k = itk + lane - t0;
#pragma unroll
        for (int i = 0; i < NR; i++) {
          const int c0 = NC * k + 2 * i, c1 = c0 + 1;
          const uint2 w0 = res_word(it_pw, c0, it_nwords), w1 = res_word(it_pw, c1, it_nwords);
          const int s0 = res_shift(c0), s1 = res_shift(c1);
          rp[i] = ((w0.x >> s0) & 31u) | (((w0.y >> s0) & 31u) << 5) | (((w1.x >> s1) & 31u) << 10) |
                  (((w1.y >> s1) & 31u) << 15);
        }
        ctl = (uint32_t)it | (k == 0 ? kCtlFirst : 0u) | (k == itK - 1 ? kCtlLast : 0u);
      }
      t0 += take;
      itk += take;
      mapped += take;
    }
  };
  uint32_t D[TR], F[TR];
#pragma unroll
  for (int r = 0; r < TR; r++) { D[r] = 0u; F[r] = 0u; }
  uint32_t hmax = 0u, hm_out = 0u, ctl_out = kCtlVoid;
  uint32_t e_out[NC], h_out[NC], r_out[NR];
#pragma unroll
  for (int c = 0; c < NC; c++) { e_out[c] = 0u; h_out[c] = 0u; }
#pragma unroll
  for (int i = 0; i < NR; i++) r_out[i] = 0u;
  uint32_t rp_cur[NR], rp_nxt[NR], ctl_cur, ctl_nxt;
  gen(rp_cur, ctl_cur);
  gen(rp_nxt, ctl_nxt);
  for (long long sb = 0;; sb += 32) {
    // every mapped position has passed the last active lane: done
    if (exhausted && sb >= mapped + nact - 1) break;
#pragma unroll 1
    for (int t = 0; t < 32; t++) {
      uint32_t e[NC], hp[NC], r_in[NR];
#pragma unroll
      for (int c = 0; c < NC; c++) {
        e[c] = __shfl_up_sync(0xffffffffu, e_out[c], 1);
        hp[c] = __shfl_up_sync(0xffffffffu, h_out[c], 1);
      }
#pragma unroll
      for (int i = 0; i < NR; i++) r_in[i] = __shfl_up_sync(0xffffffffu, r_out[i], 1);
      uint32_t ctl = __shfl_up_sync(0xffffffffu, ctl_out, 1);
      uint32_t hm_in = __shfl_up_sync(0xffffffffu, hm_out, 1);
#pragma unroll
      for (int i = 0; i < NR; i++) {
        const uint32_t v = __shfl_sync(0xffffffffu, rp_cur[i], t);
        if (lane == 0) r_in[i] = v;
      }
      {
        const uint32_t v = __shfl_sync(0xffffffffu, ctl_cur, t);
        if (lane == 0) {
          ctl = v;
          hm_in = 0u;
#pragma unroll
          for (int c = 0; c < NC; c++) { e[c] = 0u; hp[c] = 0u; }   // E(0, col) = H(-1, col) = 0
        }
      }
      if (lane < nact && ctl != kCtlVoid) {
        if (ctl & kCtlFirst) {
#pragma unroll
          for (int r = 0; r < TR; r++) { D[r] = 0u; F[r] = 0u; }
          hmax = 0u;
        }
        uint4 pa[NC], pb[NC];
#pragma unroll
        for (int c = 0; c < NC; c++) {
          const uint32_t rr = r_in[c >> 1] >> (10 * (c & 1));
          pa[c] = *reinterpret_cast<const uint4*>(pr + (rr & 31u) * stride);
          pb[c] = *reinterpret_cast<const uint4*>(pr + ((rr >> 5) & 31u) * stride);
        }
        col16b_xn<TR, NC>(D, F, e, hp, pa, pb, na2, nb2, hmax);
        if (ctl & kCtlLast) {
          const uint32_t hm = __vmaxs2(hmax, hm_in);
          if (lane == nact - 1) {
            const int x = (int)(ctl & kCtlItem);
            const int g = n_groups - 1 - x / 32, p = 31 - x % 32;
            emit_pair(hm, g, 2 * p, groups[g].count, limit, pos_map, score_sorted, flag);
          } else {
            hm_out = hm;
          }
        }
      } else {
        ctl = kCtlVoid;
      }
#pragma unroll
      for (int c = 0; c < NC; c++) { e_out[c] = e[c]; h_out[c] = hp[c]; }
#pragma unroll
      for (int i = 0; i < NR; i++) r_out[i] = r_in[i];
      ctl_out = ctl;
    }
#pragma unroll
    for (int i = 0; i < NR; i++) rp_cur[i] = rp_nxt[i];
    ctl_cur = ctl_nxt;
    gen(rp_nxt, ctl_nxt);
  }
  __syncwarp();
}

template <int T, bool SMEM, int NT, bool BIG = false, bool STATIC = false, int GAPS = 0>
__global__ void __launch_bounds__(NT, 1)
k_inter16(const uint2* __restrict__ words, const GroupDesc* __restrict__ groups, int n_groups,
          const int* __restrict__ n_groups_dev, const int* __restrict__ pos_map, int cut,
          const int8_t* __restrict__ gprof, int m_pad, int stride, int alpha, int beta, int limit,
          uint2* __restrict__ scratch, long long scratch_cols, int* __restrict__ counter,
          int* __restrict__ score_sorted, uint8_t* __restrict__ flag, long long big_off,
          long long big_cols, int n_big, const long long* __restrict__ ready_from) {
  extern __shared__ __align__(16) int8_t sprof[];
  __shared__ int s_split;
  if (n_groups_dev) n_groups = *n_groups_dev;   // mini-group layout of a rerun: size known on device only
  if (threadIdx.x == 0) s_split = split_groups(groups, n_groups, cut);
  __syncthreads();
  const int n_items = s_split;
  if (n_items <= 0) {
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    return;
  }
  if (SMEM) load_profile_smem(sprof, gprof, stride);
  const int lane = threadIdx.x & 31;
  const long long own = ((long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * scratch_cols * 32;
  uint2* const own_bnd = scratch + own;
  // GAPS = 1: the paper's penalties as immediates (kFixedAlpha/kFixedBeta; the host launches it only for them)
  const uint32_t na2 = GAPS == 1 ? pack2(-kFixedAlpha) : pack2(-alpha);
  const uint32_t nb2 = GAPS == 1 ? pack2(-kFixedBeta) : pack2(-beta);
  int it_static = 0;
  for (;;) {
    int item = 0;
    if constexpr (STATIC) {
      // f4 ablation of the paper's OpenMP "static" schedule: item w + t*W
      item = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) + it_static++ * gridDim.x * (blockDim.x >> 5);
    } else {
      if (lane == 0) item = atomicAdd(counter, 1);
      item = __shfl_sync(0xffffffffu, item, 0);
    }
    if (item >= n_items) break;
    const int g = n_items - 1 - item;
    const GroupDesc gd = groups[g];
    wait_words_ready(ready_from, gd.base);
    // the n_big longest groups (the first items) are wider than a warp's slab:
    // each has a boundary slab of its own, big_off words from `scratch` (one
    // base pointer keeps the slab accesses of the hot loop __restrict__)
    uint2* bnd = own_bnd;
    if constexpr (BIG) bnd = scratch + (item < n_big ? big_off + (long long)item * big_cols * 32 : own);
    const uint32_t hmax = inter_group16<T, SMEM>(words + gd.base, gd.ncols, gprof, stride, m_pad, bnd, na2, nb2, lane);
    emit_pair(hmax, g, 2 * lane, gd.count, limit, pos_map, score_sorted, flag);
  }
  // Out of work: a programmatic dependent launched behind this grid (the flag
  // compaction of small databases) may become resident now; it waits for this
  // grid's completion before reading anything.
  asm volatile("griddepcontrol.launch_dependents;");
  // Launched as the programmatic dependent of k_intra16 (same stream): do not
  // retire before that grid has completed, so the stream's later work sees its
  // scores.  A no-op when there is no primary grid.
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Intra-task pass over groups [split, n_groups): one subject PAIR per work item,
// longest first, aligned by the lane wavefront.  A kernel of its own (own
// register allocation), launched beside k_inter16.
// len_sorted (first pass only; NULL for rerun layouts): each pair runs to its own
// longer subject's length instead of the group's ncols (the columns past it are
// DUMMY padding, score-neutral).
#ifdef SW_PIPE_PROF
// Debug build only: globaltimer ns of [0] first CTA start (min), [1] last warp end (max),
// [2]/[3] start/end of item 0 (the longest pair), [4] items taken by that warp afterwards.
__device__ unsigned long long g_intra_prof[8];
__device__ unsigned long long g_intra_first[2048][4];   // per warp: first item start, end, ncols, items
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif

template <int TR, bool SMEM, int NC = 2, int GAPS = 0>
__global__ void __launch_bounds__(kInterThreads, 1)
k_intra16(const uint2* __restrict__ words, const GroupDesc* __restrict__ groups, int n_groups,
          const int* __restrict__ n_groups_dev, const int* __restrict__ pos_map, int cut,
          const int8_t* __restrict__ gprof, int m_pad, int stride, int alpha, int beta, int limit,
          uint2* __restrict__ scratch, long long scratch_cols, int* __restrict__ counter,
          int* __restrict__ score_sorted, uint8_t* __restrict__ flag, const int* __restrict__ len_sorted,
          const long long* __restrict__ ready_from, int mode) {
  // mode bit 0: isolate the warps holding the longest pairs; bit 1: no chained stream;
  // bit 2: no split of the critical pairs; bit 3: launched as the programmatic
  // dependent of k_profiles (its CTAs become resident while the profiles are
  // built and wait here for them, the counters and the flags)
  const bool isolate = mode & 1, chain_off = mode & 2, split_off = mode & 4;
  if (mode & 8) asm volatile("griddepcontrol.wait;" ::: "memory");
  // The inter-task kernel may start beside this one (programmatic dependent
  // launch): it only reads what was complete before this grid started (with
  // bit 3, after the wait above: k_profiles has then completed).
  asm volatile("griddepcontrol.launch_dependents;");
  extern __shared__ __align__(16) int8_t sprof[];
  __shared__ int s_split;
  if (n_groups_dev) n_groups = *n_groups_dev;
  if (threadIdx.x == 0) s_split = split_groups(groups, n_groups, cut);
  __syncthreads();
  const int split = s_split;
  const int n_items = (n_groups - split) * 32;
  if (n_items <= 0) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    return;
  }
#ifdef SW_PIPE_PROF
  if (threadIdx.x == 0) atomicMin(&g_intra_prof[0], gtimer());
#endif
  if (SMEM) load_profile_smem(sprof, gprof, stride);
  const int lane = threadIdx.x & 31;
  uint2* bnd = scratch + ((long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * scratch_cols * 32;
  const uint32_t na2 = GAPS == 1 ? pack2(-kFixedAlpha) : pack2(-alpha);    // GAPS: as in k_inter16
  const uint32_t nb2 = GAPS == 1 ? pack2(-kFixedBeta) : pack2(-beta);
  // First items are dealt across the SMs (warp k of CTA b takes item k*gridDim.x + b),
  // so the longest pairs -- the wavefront's critical paths -- do not share an SM;
  // the rest come longest-first from the counter.
  // Latency-bound searches (isolate = 1: the longest pair's wavefront is the
  // critical path of the whole pass, e.g. C1): warp 0 of every CTA, which holds
  // one of the gridDim.x longest pairs, gets its SM sub-partition to itself --
  // warps 4 and 8 (same sub-partition) take no items and the other warps are
  // dealt the first items densely.  Measured on C1: the longest pair 316 -> 229 us
  // (209 us alone on the GPU).
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const bool idle = isolate && w != 0 && (w & 3) == 0;
  const int w_active = isolate ? w - (w > 4) - (w > 8) : w;                  // dense index of this warp
  const int nw_active = isolate ? nw - (nw > 4) - (nw > 8) : nw;
  const int n_warps = gridDim.x * nw_active;
  int item = idle ? n_items : w_active * gridDim.x + blockIdx.x;
  bool finished = idle;                                // takes no (more) items
  // Isolated sub-partition, single-pass query: the longest pair dealt to warp 0
  // is cut into two column segments (about half each): warp 0 runs the first,
  // warp 4 (otherwise idle) the second speculatively from a zero boundary, then
  // repairs its start from warp 0's final rows until they meet the speculative
  // ones (intra_seg16).  Both warps share the sub-partition's issue slots, which
  // the lone latency-bound wavefront leaves half empty.
  if constexpr (NC == 4) {
    if (isolate && (w == 0 || w == 4) && m_pad <= 32 * TR && !split_off) {
      __shared__ uint32_t s_state[2 * 16 * 32 + 1];
      const int it0 = blockIdx.x;                         // warp 0's dealt first item
      int ncols0 = 0, g0 = 0, p0 = 0, cnt0 = 0;
      const uint2* pw0 = nullptr;
      if (it0 < n_items) {
        g0 = n_groups - 1 - it0 / 32;
        p0 = 31 - it0 % 32;
        const GroupDesc gd = groups[g0];
        cnt0 = gd.count;
        if (2 * p0 < gd.count) {
          ncols0 = len_sorted ? len_sorted[(long long)g0 * kGroup + min(2 * p0 + 1, gd.count - 1)] : gd.ncols;
          pw0 = words + gd.base + p0;
        }
      }
      const int c1 = ((ncols0 + 64) / 2 + 7) & ~7;                       // warp 0: columns [0, c1 - 1)
      const int K0 = c1 / 8, K1 = (ncols0 + 1 - c1 + 7) / 8;
      const long long ck_words = (long long)(K1 / kCkSteps + 1) * 2 * TR * 32;
      const long long cap_words = scratch_cols * 32 * 2;                  // warp 4's slab, in 32-bit words
      if (ncols0 >= kSplitMinCols && ck_words <= cap_words) {
        uint32_t* ck = reinterpret_cast<uint32_t*>(scratch + ((long long)blockIdx.x * (blockDim.x >> 5) + 4) *
                                                   scratch_cols * 32);
        wait_words_ready(ready_from, groups[g0].base);
        if (w == 0) {
          const uint32_t h0 = intra_seg16<TR, SMEM, 8>(pw0, ncols0, 0, K0, gprof, stride, m_pad, na2, nb2, lane, 0,
                                                      nullptr, s_state);
          if (lane == 0) s_state[2 * 16 * 32] = h0;
          asm volatile("bar.sync 1, 64;" ::: "memory");
          item = -1;                                      // on to the queue
        } else {
          const uint32_t h1 = intra_seg16<TR, SMEM, 8>(pw0, ncols0, c1, K1, gprof, stride, m_pad, na2, nb2, lane, 1,
                                                      ck, nullptr);
          __threadfence_block();
          asm volatile("bar.sync 1, 64;" ::: "memory");
          const uint32_t h2 = intra_seg16<TR, SMEM, 8>(pw0, ncols0, c1, K1, gprof, stride, m_pad, na2, nb2, lane, 2,
                                                      ck, s_state);
          if (lane == 0)
            emit_pair(__vmaxs2(__vmaxs2(h1, h2), s_state[2 * 16 * 32]), g0, 2 * p0, cnt0, limit, pos_map,
                      score_sorted, flag);
          item = n_items;                                 // warp 4 takes no other item
          finished = true;
        }
      }
    }
  }
  // single-pass queries (m up to 32 * TR rows): the items of a warp run as one
  // chained stream (intra_chain16, 8 columns per step); the isolated critical
  // warps keep the per-item wavefront with 8 columns per step
  if constexpr (NC == 4) {
    if (m_pad <= 32 * TR && !(isolate && w == 0) && !chain_off && !finished) {
      // 8 columns per step: with no fill and drain per item the longer step only
      // amortises its shuffles and loads better (all-intra C2 27.8 -> 26.9 ms)
      intra_chain16<TR, SMEM, 8>(words, groups, n_groups, n_items, item, n_warps, counter, len_sorted, ready_from,
                                 gprof, stride, m_pad, na2, nb2, limit, pos_map, score_sorted, flag, lane);
      item = n_items;
    }
  }
  for (;; item = -1) {
    if (item < 0) {
      if (lane == 0) item = n_warps + atomicAdd(counter, 1);
      item = __shfl_sync(0xffffffffu, item, 0);
    }
    if (item >= n_items) break;
    const int g = n_groups - 1 - item / 32;
    const int p = 31 - item % 32;
    const GroupDesc gd = groups[g];
    if (2 * p >= gd.count) continue;
    wait_words_ready(ready_from, gd.base);
    const int ncols = len_sorted ? len_sorted[(long long)g * kGroup + min(2 * p + 1, gd.count - 1)] : gd.ncols;
#ifdef SW_PIPE_PROF
    const int wid = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (lane == 0) {
      if (g_intra_first[wid][3] == 0) { g_intra_first[wid][0] = gtimer(); g_intra_first[wid][2] = ncols; }
      g_intra_first[wid][3]++;
    }
#endif
    uint32_t hm;
    if constexpr (NC == 2)
      hm = intra_pair16<TR, SMEM>(words + gd.base + p, ncols, gprof, stride, m_pad, bnd, scratch_cols * 16,
                                  na2, nb2, lane);
    else if (NC == 4 && isolate && w == 0)   // the isolated warp: 8 columns per step (lower latency per column)
      hm = intra_multi16<TR, SMEM, 8>(words + gd.base + p, ncols, gprof, stride, m_pad, bnd, scratch_cols * 16,
                                      na2, nb2, lane);
    else
      hm = intra_multi16<TR, SMEM, NC>(words + gd.base + p, ncols, gprof, stride, m_pad, bnd, scratch_cols * 16,
                                       na2, nb2, lane);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) hm = __vmaxs2(hm, __shfl_xor_sync(0xffffffffu, hm, o));
    if (lane == 0) emit_pair(hm, g, 2 * p, gd.count, limit, pos_map, score_sorted, flag);
#ifdef SW_PIPE_PROF
    if (lane == 0 && g_intra_first[wid][3] == 1) g_intra_first[wid][1] = gtimer();
#endif
  }
#ifdef SW_PIPE_PROF
  if (lane == 0) atomicMax(&g_intra_prof[1], gtimer());
#endif
  // When launched as a programmatic dependent (a chain of intra-task passes in
  // sw_search_batch), retire only after the primary grid: a no-op otherwise.
  asm volatile("griddepcontrol.wait;" ::: "memory");
}


}  // namespace swk
