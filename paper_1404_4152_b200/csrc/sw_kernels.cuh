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

__device__ __forceinline__ uint32_t pack2(int v) {
  const uint32_t h = (uint32_t)v & 0xffffu;
  return h | (h << 16);
}

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
template <int R>
__device__ __forceinline__ uint32_t col16(uint32_t (&D)[R], uint32_t (&F)[R], uint32_t& e, uint32_t htop,
                                          const int8_t* __restrict__ plo, const int8_t* __restrict__ phi,
                                          uint32_t na2, uint32_t nb2, uint32_t& hmax) {
  uint32_t hprev = htop, hodd = 0u;
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
__device__ __forceinline__ uint2 res_word(const uint2* __restrict__ lw, int c, int nwords) {
  const int w = (int)(__umulhi((unsigned)c, 0xAAAAAAABu) >> 2);   // c / 6
  return w < nwords ? __ldg(lw + (long long)w * 32) : make_uint2(kDummyWord, kDummyWord);
}
__device__ __forceinline__ int res_shift(int c) {
  return 5 * (c - 6 * (int)(__umulhi((unsigned)c, 0xAAAAAAABu) >> 2));
}

template <int R>
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
    col16<R>(D, F, e0, 0u, pr + (w0.x & 31u) * stride, pr + (w0.y & 31u) * stride, na2, nb2, hmax);
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
#ifdef SW_INTERLEAVE_COLUMNS
    col16x2<R>(D, F, eA, bE.y, pr + ((wA.x >> shA) & 31u) * stride, pr + ((wA.y >> shA) & 31u) * stride,
               eB, bO.y, pr + ((wB.x >> shB) & 31u) * stride, pr + ((wB.y >> shB) & 31u) * stride,
               na2, nb2, hmax, hlA, hlB);
#else
    hlA = col16<R>(D, F, eA, bE.y, pr + ((wA.x >> shA) & 31u) * stride, pr + ((wA.y >> shA) & 31u) * stride,
                   na2, nb2, hmax);
    hlB = col16<R>(D, F, eB, bO.y, pr + ((wB.x >> shB) & 31u) * stride, pr + ((wB.y >> shB) & 31u) * stride,
                   na2, nb2, hmax);
#endif
    wA = res_word(lw, j + 3, nwords);
    wB = res_word(lw, j + 4, nwords);
    if (!first && j + 2 < ncols) bE = bnd[(j + 2) * 32 + lane];
    if (!first && j + 3 < ncols) bO = bnd[(j + 3) * 32 + lane];
    if (!last) {
      bnd[j * 32 + lane] = make_uint2(eA, hlA);
      bnd[(j + 1) * 32 + lane] = make_uint2(eB, hlB);
    }
  }
  if (j < ncols) {                                 // odd tail column
    const int shA = res_shift(j + 1);
    uint32_t e = bE.x;
    const uint32_t hl = col16<R>(D, F, e, bE.y, pr + ((wA.x >> shA) & 31u) * stride,
                                 pr + ((wA.y >> shA) & 31u) * stride, na2, nb2, hmax);
    if (!last) bnd[j * 32 + lane] = make_uint2(e, hl);
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
// [base + l*TR, base + (l+1)*TR) of a pass of 32*TR rows and processes column
// j = s - l at step s; (E, H, next residue) flow to lane l+1 by SHFL.  The
// last active lane's output row is kept in gbnd for the next pass.
// Returns this lane's running max (to be reduced over the warp).
// ---------------------------------------------------------------------------
template <int TR, bool SMEM>
__device__ __forceinline__ uint32_t intra_pair16(const uint2* __restrict__ pw, int ncols,
                                                 const int8_t* __restrict__ gprof, int stride, int m_pad,
                                                 uint2* __restrict__ gbnd, long long gstride,
                                                 uint32_t na2, uint32_t nb2, int lane) {
  const int8_t* prof = prof_base<SMEM>(gprof);
  uint32_t hmax = 0u;
  const int nwords = (ncols + kResPerWord - 1) / kResPerWord;
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
    uint32_t e_out = 0u, h_out = 0u, r_out = 0u;
    // Lane 0's per-step inputs (the residue pair of column s+1 and, after the
    // first pass, the previous pass's boundary of column s) are fetched by all
    // lanes for 32 steps at a time, one block ahead, and handed to lane 0 by
    // SHFL -- no load latency on the wavefront's critical step.
    auto fetch = [&](int sb, uint32_t& rp, uint2& gv) {
      const int c = sb + 1 + lane;                                      // residue column for step sb + lane
      const uint2 w = res_word(pw, c, nwords);
      const int sh = res_shift(c);
      rp = ((w.x >> sh) & 31u) | (((w.y >> sh) & 31u) << 5);
      const int gc = sb + lane;                                         // boundary column for step sb + lane
      gv = (!first && gc >= 0 && gc < ncols) ? gin[gc] : make_uint2(0u, 0u);
    };
    const int nsteps = ncols + nact;                                    // steps s = -1 .. ncols + nact - 2
    uint32_t rp_cur, rp_nxt;
    uint2 gv_cur, gv_nxt;
    fetch(-1, rp_cur, gv_cur);
    fetch(31, rp_nxt, gv_nxt);
    __syncwarp();
    for (int sb = -1; sb < nsteps - 1; sb += 32) {
#pragma unroll 1
      for (int t = 0; t < 32; t++) {
        const int s = sb + t;
        if (s >= nsteps - 1) break;
        uint32_t e_in = __shfl_up_sync(0xffffffffu, e_out, 1);
        uint32_t h_in = __shfl_up_sync(0xffffffffu, h_out, 1);
        uint32_t r_in = __shfl_up_sync(0xffffffffu, r_out, 1);
        const uint32_t r0 = __shfl_sync(0xffffffffu, rp_cur, t);
        const uint32_t g0x = __shfl_sync(0xffffffffu, gv_cur.x, t);
        const uint32_t g0y = __shfl_sync(0xffffffffu, gv_cur.y, t);
        const int j = s - lane;
        if (lane == 0) {
          r_in = r0;                                                    // residues of column j+1
          e_in = g0x;                                                   // E(base, j), H(base-1, j) (0 on pass 0 / j < 0)
          h_in = g0y;
        }
        if (lane < nact && j >= -1 && j < ncols) {
          uint32_t e = e_in;
          const uint4 pa = *reinterpret_cast<const uint4*>(pr + (r_in & 31u) * stride);
          const uint4 pb = *reinterpret_cast<const uint4*>(pr + (r_in >> 5) * stride);
          const uint32_t hl = col16b<TR>(D, F, e, h_in, pa, pb, na2, nb2, hmax);
          e_out = e;
          h_out = hl;
          r_out = r_in;
          if (!last && lane == nact - 1 && j >= 0) gout[j] = make_uint2(e, hl);
        }
      }
      rp_cur = rp_nxt;
      gv_cur = gv_nxt;
      fetch(sb + 64, rp_nxt, gv_nxt);
    }
    __syncwarp();
  }
  return hmax;
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
template <int T, bool SMEM, int NT, bool BIG = false, bool STATIC = false>
__global__ void __launch_bounds__(NT, 1)
k_inter16(const uint2* __restrict__ words, const GroupDesc* __restrict__ groups, int n_groups,
          const int* __restrict__ n_groups_dev, const int* __restrict__ pos_map, int cut,
          const int8_t* __restrict__ gprof, int m_pad, int stride, int alpha, int beta, int limit,
          uint2* __restrict__ scratch, long long scratch_cols, int* __restrict__ counter,
          int* __restrict__ score_sorted, uint8_t* __restrict__ flag, long long big_off,
          long long big_cols, int n_big) {
  extern __shared__ __align__(16) int8_t sprof[];
  __shared__ int s_split;
  if (n_groups_dev) n_groups = *n_groups_dev;   // mini-group layout of a rerun: size known on device only
  if (threadIdx.x == 0) s_split = split_groups(groups, n_groups, cut);
  __syncthreads();
  const int n_items = s_split;
  if (n_items <= 0) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    return;
  }
  if (SMEM) load_profile_smem(sprof, gprof, stride);
  const int lane = threadIdx.x & 31;
  const long long own = ((long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * scratch_cols * 32;
  uint2* const own_bnd = scratch + own;
  const uint32_t na2 = pack2(-alpha), nb2 = pack2(-beta);
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
    // the n_big longest groups (the first items) are wider than a warp's slab:
    // each has a boundary slab of its own, big_off words from `scratch` (one
    // base pointer keeps the slab accesses of the hot loop __restrict__)
    uint2* bnd = own_bnd;
    if constexpr (BIG) bnd = scratch + (item < n_big ? big_off + (long long)item * big_cols * 32 : own);
    const uint32_t hmax = inter_group16<T, SMEM>(words + gd.base, gd.ncols, gprof, stride, m_pad, bnd, na2, nb2, lane);
    emit_pair(hmax, g, 2 * lane, gd.count, limit, pos_map, score_sorted, flag);
  }
  // Launched as the programmatic dependent of k_intra16 (same stream): do not
  // retire before that grid has completed, so the stream's later work sees its
  // scores.  A no-op when there is no primary grid.
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Intra-task pass over groups [split, n_groups): one subject PAIR per work item,
// longest first, aligned by the lane wavefront.  A kernel of its own (own
// register allocation), launched on a second stream beside k_inter16.
template <int TR, bool SMEM>
__global__ void __launch_bounds__(kInterThreads, 1)
k_intra16(const uint2* __restrict__ words, const GroupDesc* __restrict__ groups, int n_groups,
          const int* __restrict__ n_groups_dev, const int* __restrict__ pos_map, int cut,
          const int8_t* __restrict__ gprof, int m_pad, int stride, int alpha, int beta, int limit,
          uint2* __restrict__ scratch, long long scratch_cols, int* __restrict__ counter,
          int* __restrict__ score_sorted, uint8_t* __restrict__ flag) {
  // The inter-task kernel may start beside this one (programmatic dependent
  // launch): it only reads what was complete before this grid started.
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
  if (SMEM) load_profile_smem(sprof, gprof, stride);
  const int lane = threadIdx.x & 31;
  uint2* bnd = scratch + ((long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * scratch_cols * 32;
  const uint32_t na2 = pack2(-alpha), nb2 = pack2(-beta);
  for (;;) {
    int item = 0;
    if (lane == 0) item = atomicAdd(counter, 1);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= n_items) break;
    const int g = n_groups - 1 - item / 32;
    const int p = 31 - item % 32;
    const GroupDesc gd = groups[g];
    if (2 * p >= gd.count) continue;
    uint32_t hm = intra_pair16<TR, SMEM>(words + gd.base + p, gd.ncols, gprof, stride, m_pad, bnd, scratch_cols * 16,
                                         na2, nb2, lane);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) hm = __vmaxs2(hm, __shfl_xor_sync(0xffffffffu, hm, o));
    if (lane == 0) emit_pair(hm, g, 2 * p, gd.count, limit, pos_map, score_sorted, flag);
  }
  // When launched as a programmatic dependent (a chain of intra-task passes in
  // sw_search_batch), retire only after the primary grid: a no-op otherwise.
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

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

// ---------------------------------------------------------------------------
// f1 multi-query pass: TWO queries per pass in the lo/hi halves of int16x2, one
// subject per lane.  Both halves read the same subject residue, so the
// substitution pair is a single word of the pair profile
//   prof2[r][i] = (fsbt(qa_i, r), fsbt(qb_i, r))   (int16x2)
// and the PRMT of the single-query kernel disappears (3.5 alu ops per row).
// The row stride is odd in words, so 32 lanes reading rows of different
// residues hit different banks (LDS.32, conflict-free).
// ---------------------------------------------------------------------------
template <int R>
__device__ __forceinline__ uint32_t colq(uint32_t (&D)[R], uint32_t (&F)[R], uint32_t& e, uint32_t htop,
                                         const uint32_t* __restrict__ p, uint32_t na2, uint32_t nb2,
                                         uint32_t& hmax) {
  uint32_t hprev = htop, hodd = 0u;
#pragma unroll
  for (int r = 0; r < R; r++) {
    const uint32_t h = __vimax3_s16x2(D[r], e, F[r]);
    D[r] = __vadd2(hprev, p[r]);                               // H(i-1,j) + (fsbt(qa_i,s_{j+1}), fsbt(qb_i,s_{j+1}))
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
    const uint32_t hlA = colq<R>(D, F, eA, bE.y, pr + ((wA >> shA) & 31u) * stride2, na2, nb2, hmax);
    const uint32_t hlB = colq<R>(D, F, eB, bO.y, pr + ((wB >> shB) & 31u) * stride2, na2, nb2, hmax);
    wA = res_word32(wp, j + 3, nwords);
    wB = res_word32(wp, j + 4, nwords);
    if (!first && j + 2 < ncols) bE = bnd[(j + 2) * 32 + lane];
    if (!first && j + 3 < ncols) bO = bnd[(j + 3) * 32 + lane];
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
template <int T>
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
  const uint32_t na2 = pack2(-alpha), nb2 = pack2(-beta);
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

// ---------------------------------------------------------------------------
// a4 escalation plumbing: deterministic compaction of flagged sorted positions
// (ascending, hence ascending length) and re-interleaving of the flagged
// subjects into a mini-group layout for the next, wider pass.
// ---------------------------------------------------------------------------
constexpr int kScanBlock = 1024;

__global__ void __launch_bounds__(kScanBlock) k_flag_count(const uint8_t* __restrict__ flag, int n,
                                                           int* __restrict__ block_counts) {
  const int i = blockIdx.x * kScanBlock + threadIdx.x;
  const int f = (i < n && flag[i]) ? 1 : 0;
  const int c = __syncthreads_count(f);
  if (threadIdx.x == 0) block_counts[blockIdx.x] = c;
}

// Exclusive scan of `v[0..nb)` in place by one CTA; total -> *total (and, when
// tail_groups != nullptr, ceil(total/64) -> *tail_groups).
__global__ void __launch_bounds__(kScanBlock) k_scan_exclusive(int* __restrict__ v, int nb, int* __restrict__ total,
                                                              int* __restrict__ tail_groups) {
  __shared__ int sh[kScanBlock];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nb; base += kScanBlock) {
    const int i = base + threadIdx.x;
    const int x = i < nb ? v[i] : 0;
    sh[threadIdx.x] = x;
    __syncthreads();
    for (int off = 1; off < kScanBlock; off <<= 1) {
      const int add = threadIdx.x >= off ? sh[threadIdx.x - off] : 0;
      __syncthreads();
      sh[threadIdx.x] += add;
      __syncthreads();
    }
    if (i < nb) v[i] = carry + sh[threadIdx.x] - x;
    __syncthreads();
    if (threadIdx.x == 0) carry += sh[kScanBlock - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (total) *total = carry;
    if (tail_groups) *tail_groups = (carry + kGroup - 1) / kGroup;
  }
}

__global__ void __launch_bounds__(kScanBlock) k_flag_scatter(const uint8_t* __restrict__ flag, int n,
                                                             const int* __restrict__ block_offsets,
                                                             int* __restrict__ list) {
  __shared__ int warp_sums[kScanBlock / 32];
  const int i = blockIdx.x * kScanBlock + threadIdx.x;
  const int f = (i < n && flag[i]) ? 1 : 0;
  const unsigned bal = __ballot_sync(0xffffffffu, f);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) warp_sums[w] = __popc(bal);
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int k = 0; k < kScanBlock / 32; k++) { const int t = warp_sums[k]; warp_sums[k] = acc; acc += t; }
  }
  __syncthreads();
  if (f) list[block_offsets[blockIdx.x] + warp_sums[w] + __popc(bal & ((1u << lane) - 1u))] = i;
}

// mini-group sizes (words) of a sorted flagged list: ncols = length of the group's last member
__global__ void k_mini_sizes(const int* __restrict__ list, const int* __restrict__ count_ptr,
                             const int* __restrict__ len_sorted, int n_mini_max, int* __restrict__ sizes) {
  const int cnt = *count_ptr;
  for (int gm = blockIdx.x * blockDim.x + threadIdx.x; gm < n_mini_max; gm += gridDim.x * blockDim.x) {
    int words = 0;
    if (gm * kGroup < cnt) {
      const int last = min(gm * kGroup + kGroup, cnt) - 1;
      const int nc = len_sorted[list[last]];
      words = (nc + kResPerWord - 1) / kResPerWord * 32;
    }
    sizes[gm] = words;
  }
}

// one warp per mini-group: descriptor + gather of the members' packed words
__global__ void k_mini_build(const uint2* __restrict__ words, const GroupDesc* __restrict__ groups,
                             const int* __restrict__ list, const int* __restrict__ count_ptr,
                             const int* __restrict__ len_sorted, const int* __restrict__ bases, int n_mini_max,
                             GroupDesc* __restrict__ mgroups, uint2* __restrict__ mwords) {
  const int cnt = *count_ptr;
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int gm = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); gm < n_mini_max && gm * kGroup < cnt; gm += warps) {
    const int first = gm * kGroup, count = min(kGroup, cnt - first);
    const int nc = len_sorted[list[first + count - 1]];
    const int nw = (nc + kResPerWord - 1) / kResPerWord;
    if (lane == 0) {
      GroupDesc d;
      d.base = bases[gm];
      d.ncols = nc;
      d.count = count;
      mgroups[gm] = d;
    }
    const uint32_t* src[2] = {nullptr, nullptr};
    int own_nw[2] = {0, 0};
    for (int h = 0; h < 2; h++) {
      const int slot = 2 * lane + h;
      if (slot < count) {
        const int pos = list[first + slot];
        const int og = pos / kGroup, os = pos % kGroup;
        src[h] = reinterpret_cast<const uint32_t*>(words) + 2 * (groups[og].base + (os >> 1)) + (os & 1);
        own_nw[h] = (len_sorted[pos] + kResPerWord - 1) / kResPerWord;
      }
    }
    uint2* dst = mwords + bases[gm] + lane;
    for (int w = 0; w < nw; w++) {
      uint2 v;
      v.x = w < own_nw[0] ? __ldg(src[0] + (long long)w * 64) : kDummyWord;
      v.y = w < own_nw[1] ? __ldg(src[1] + (long long)w * 64) : kDummyWord;
      dst[(long long)w * 32] = v;
    }
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

__global__ void k_sel_init(SelState* st, long long k) {
  if (threadIdx.x == 0) {
    st->prefix = 0ull;
    st->mask = 0ull;
    st->kk = k;
  }
}

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

__global__ void __launch_bounds__(256) k_sel_pick(SelState* st, int shift, unsigned* hist) {
  // digit d is chosen so that (# keys with digit > d) < kk <= (# keys with digit >= d);
  // suffix sums over the 256 bins by a block-wide scan (descending digit order)
  __shared__ long long suf[256];
  const int t = threadIdx.x;
  const int d = 255 - t;                       // thread t holds digit 255 - t
  long long v = hist[d];
  suf[t] = v;
  __syncthreads();
  for (int off = 1; off < 256; off <<= 1) {
    const long long add = t >= off ? suf[t - off] : 0;
    __syncthreads();
    suf[t] += add;
    __syncthreads();
  }
  const long long kk = st->kk;
  const long long incl = suf[t], excl = incl - v;   // keys with digit >= d, > d
  __syncthreads();
  if (excl < kk && kk <= incl) {
    st->kk = kk - excl;
    st->prefix |= (unsigned long long)d << shift;
    st->mask |= 255ull << shift;
  }
  hist[d] = 0;
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

// Small databases (n <= 65,536, min(k, n) <= 4,096): the whole ranking in ONE
// CTA -- radix select of the k-th largest unique key (8 bits per pass, smem
// histogram), compaction of the k keys above it, bitonic sort, decode --
// instead of the 19-launch multi-CTA path.
__global__ void __launch_bounds__(1024) k_topk_block(const unsigned long long* __restrict__ keys, int n, int k,
                                                     long long* __restrict__ out_ids, int* __restrict__ out_scores) {
  __shared__ unsigned long long s[4096];
  __shared__ unsigned hist[256];
  __shared__ unsigned long long sh_prefix, sh_mask;
  __shared__ long long sh_kk;
  __shared__ int sh_cnt;
  const int cnt = min(k, n);
  unsigned long long thr = 0ull;
  if (k < n) {
    if (threadIdx.x == 0) { sh_prefix = 0ull; sh_mask = 0ull; sh_kk = k; }
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int t = threadIdx.x; t < 256; t += blockDim.x) hist[t] = 0u;
      __syncthreads();
      const unsigned long long prefix = sh_prefix, mask = sh_mask;
      for (int p = threadIdx.x; p < n; p += blockDim.x) {
        const unsigned long long key = keys[p];
        if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
      }
      __syncthreads();
      if (threadIdx.x == 0) {                                  // digit with (# > d) < kk <= (# >= d)
        long long above = 0;
        const long long kk = sh_kk;
        for (int d = 255; d >= 0; d--) {
          const long long c = hist[d];
          if (above < kk && kk <= above + c) {
            sh_kk = kk - above;
            sh_prefix = prefix | ((unsigned long long)d << shift);
            sh_mask = mask | (255ull << shift);
            break;
          }
          above += c;
        }
      }
      __syncthreads();
    }
    thr = sh_prefix;                                           // the k-th largest key (keys are unique)
  }
  if (threadIdx.x == 0) sh_cnt = 0;
  __syncthreads();
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    const unsigned long long key = keys[p];
    if (key >= thr) s[atomicAdd(&sh_cnt, 1)] = key;
  }
  __syncthreads();
  int n2 = 1;
  while (n2 < cnt) n2 <<= 1;
  for (int t = cnt + threadIdx.x; t < n2; t += blockDim.x) s[t] = 0ull;
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
