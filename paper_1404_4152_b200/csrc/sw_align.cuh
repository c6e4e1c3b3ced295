// sw_align.cuh — f3: traceback of optimal local alignments for chosen hits
// (the paper names alignment retrieval as future work,
// PAPER.md:210).  For each requested subject one warp fills Eq. 1
// over the whole query x subject matrix in exact int32 with
// the lane wavefront of the intra-task kernels (lane l owns TR query rows of a
// 32*TR-row pass and handles column s - l at step s), and stores a 4-bit
// direction code per cell:
//   bits 0-1  source of H(i,j): 0 = zero (stop), 1 = diagonal, 2 = E, 3 = F
//             (priority in that order on ties)
//   bit 2     E(i,j) extends E(i-1,j) (E(i-1,j)-alpha > H(i-1,j)-beta)
//   bit 3     F(i,j) extends F(i,j-1)
// Lane 0 then walks back from the end cell (max H; ties -> smallest subject
// position, then smallest query position) -- DESIGN.md readings R17-R19.
// The recurrence is the printed one (E(0,j) = F(i,0) = 0, no clamping), so
// every decision is the one the oracle's full-matrix traceback takes.
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace swk {

struct AlignJob {
  long long word0;   // first packed word (uint2 units) of the subject's group + its lane
  long long dir;     // direction words of this job (DirWord<TR> units): (m_pad/TR) x n
  long long bnd;     // pass boundary (H, E) of this job (int2 units): 2 x n
  long long ops;     // first byte of this job's ops slot (capacity m + n)
  long long tmp;     // first byte of its reversed-ops scratch (capacity m + n)
  int half;          // 0 = lo (.x), 1 = hi (.y) subject of the lane word
  int n;             // subject length
};

// input index -> (packed word, half, length) of each requested subject
__global__ void k_align_locate(const long long* __restrict__ idx, int n_jobs, const int* __restrict__ inv,
                               const int* __restrict__ len_sorted, const GroupDesc* __restrict__ groups,
                               AlignJob* __restrict__ jobs) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_jobs) return;
  const int pos = inv[idx[t]];
  const int slot = pos & (kGroup - 1);
  AlignJob J = {};
  J.word0 = groups[pos / kGroup].base + (slot >> 1);
  J.half = slot & 1;
  J.n = len_sorted[pos];
  jobs[t] = J;
}

// sorted position -> input index  ==>  input index -> sorted position
__global__ void k_inverse_perm(const int* __restrict__ perm, int n, int* __restrict__ inv) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) inv[perm[p]] = p;
}

__device__ __forceinline__ bool better(int h, int j, int i, int bh, int bj, int bi) {
  return h > bh || (h == bh && (j < bj || (j == bj && i < bi)));
}

// warps per hit: one 32*TR-row band each, pipelined along the columns (256 / TR x 32 = 1,024 rows per round)
template <int TR> constexpr int align_warps() { return 64 / TR; }
// direction word of one lane-row-block and column: TR 4-bit codes
template <int TR> using DirWord = typename std::conditional<TR == 8, uint32_t, uint16_t>::type;
constexpr int kRing = 128;           // columns of (H, E) in flight between neighbouring warps (shared memory)

// res[t*6 + ...] = score, q_begin, q_end, s_begin, s_end, n_ops
//
// One CTA of kAlignWarps warps per hit.  The query rows are cut into bands of
// 32*TR rows; in round r warp w fills band r*W + w over all columns with the
// lane wavefront, taking the row above its band from warp w-1 through a
// shared-memory ring (or, for warp 0, from the previous round's last warp
// through global memory) and running ~64 columns behind it.
template <int TR, int kAlignWarps = align_warps<TR>()>
__global__ void __launch_bounds__(32 * kAlignWarps)
k_align(const uint2* __restrict__ words, const AlignJob* __restrict__ jobs, int n_jobs,
        const int8_t* __restrict__ prof, int prof_smem, int stride, int m, int m_pad, int alpha, int beta,
        DirWord<TR>* __restrict__ dir, int2* __restrict__ bnd, char* __restrict__ ops_out,
        char* __restrict__ ops_tmp, int* __restrict__ res) {
  const int t = blockIdx.x;
  if (t >= n_jobs) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const AlignJob J = jobs[t];
  const int n = J.n;
  const uint32_t* wp = reinterpret_cast<const uint32_t*>(words + J.word0) + J.half;   // word w at wp[64 w]
  DirWord<TR>* D = dir + J.dir;
  int2* B = bnd + J.bnd;
  int best = 0, bj = 0x7fffffff, bi = 0x7fffffff;
  int stalled = 0;
  __shared__ int2 ring[kAlignWarps - 1][kRing];
  __shared__ int s_stalled;
  if (threadIdx.x == 0) s_stalled = 0;
  __shared__ volatile int prod[kAlignWarps], cons[kAlignWarps];
  __shared__ int s_best[kAlignWarps][3];
  __shared__ int s_nops;
  // the int8 query profile is staged in shared memory (prof_smem bytes, 0 = read through L1)
  extern __shared__ __align__(16) int8_t s_prof[];
  const int8_t* P = prof;
  if (prof_smem) {
    const uint4* src = reinterpret_cast<const uint4*>(prof);
    uint4* dst = reinterpret_cast<uint4*>(s_prof);
    for (int k = threadIdx.x; k < prof_smem / 16; k += blockDim.x) dst[k] = __ldg(src + k);
    P = s_prof;
  }
  const int band_rows = 32 * TR;
  const int n_bands = (m_pad + band_rows - 1) / band_rows;
  for (int round = 0; n > 0 && round * kAlignWarps < n_bands; round++) {
    __syncthreads();                                             // the previous round is done with the rings
    if (lane == 0) { prod[warp] = 0; cons[warp] = 0; }
    __syncthreads();                                             // also: profile staged, previous round's gout written
    const int band = round * kAlignWarps + warp;
    if (band < n_bands) {
      const int base = band * band_rows;
      const int nact = min(32, (m_pad - base) / TR);
      const bool first = band == 0, last = band == n_bands - 1;
      const bool from_ring = !first && warp > 0, to_ring = !last && warp < kAlignWarps - 1;
      const int2* gin = B + (long long)(round & 1) * n;          // written by the previous round's last warp
      int2* gout = B + (long long)((round + 1) & 1) * n;
      const int i0 = base + lane * TR;
      const int8_t* pr = P + i0;
      int Hc[TR], Fc[TR];                                        // H(i, j-1), F(i, j-1)
#pragma unroll
      for (int r = 0; r < TR; r++) { Hc[r] = 0; Fc[r] = 0; }      // H(i,0) = F(i,0) = 0
      int h_out = 0, e_out = 0, hdiag = 0;                       // hdiag = H(i0-1, j-1)
      uint32_t c_out = 0;                                        // residue of the column this lane just did
      const int nsteps = n + nact - 1;
      for (int sb = 0; sb < nsteps; sb += 32) {
        // lane 0's inputs for steps sb..sb+31: residue of column sb+k and the row above the band
        const int c = sb + lane;
        const uint32_t rc_cur = c < n ? (__ldg(wp + 64 * (c / 6)) >> (5 * (c % 6))) & 31u : 0u;
        int2 gv_cur = make_int2(0, 0);
        if (from_ring) {
          const int need = min(n, sb + 32);
          for (int spin = 0; prod[warp - 1] < need; spin++) {
            if (spin > (1 << 24)) { stalled = 1; break; }         // never expected: reported, not hung
            __nanosleep(20);
          }
          __threadfence_block();
          if (c < n) gv_cur = ring[warp - 1][c % kRing];
          __syncwarp();
          if (lane == 0) cons[warp - 1] = need;                   // these ring slots may be reused
        } else if (!first && c < n) {
          gv_cur = __ldcg(gin + c);
        }
        if (to_ring) {                                           // this block writes columns up to sb
          for (int spin = 0; cons[warp] < sb + 1 - kRing; spin++) {
            if (spin > (1 << 24)) { stalled = 1; break; }
            __nanosleep(20);
          }
        }
#pragma unroll 1
        for (int tt = 0; tt < 32; tt++) {
          const int s = sb + tt;
          if (s >= nsteps) break;
          int h_in = __shfl_up_sync(0xffffffffu, h_out, 1);
          int e_in = __shfl_up_sync(0xffffffffu, e_out, 1);
          uint32_t cc = __shfl_up_sync(0xffffffffu, c_out, 1);
          const uint32_t c0 = __shfl_sync(0xffffffffu, rc_cur, tt);
          const int g0x = __shfl_sync(0xffffffffu, gv_cur.x, tt);
          const int g0y = __shfl_sync(0xffffffffu, gv_cur.y, tt);
          const int j = s - lane;
          if (lane == 0) {                                       // row base-1 of column j, residue s_j
            h_in = g0x;
            e_in = g0y;
            cc = c0;
          }
          if (lane < nact && j >= 0 && j < n) {
            uint2 pv;
            if constexpr (TR == 8) pv = *reinterpret_cast<const uint2*>(pr + cc * stride);
            else pv = make_uint2(*reinterpret_cast<const uint32_t*>(pr + cc * stride), 0u);
            // E(i+1,j) = max(E(i,j) - alpha, H(i,j) - beta) = max(E(i,j) - alpha, Y(i,j) - beta)
            // with Y = max(0, G, F): since alpha <= beta the E - beta term never wins, so the
            // E chain from row to row is one max; H, the direction code and the
            // running max hang off it.  Extension bit of E(i+1,j):
            // E - alpha > H - beta  <=>  alpha < beta  and  E - alpha > Y - beta.
            int dg = hdiag;
            int ec = max(e_in - alpha, h_in - beta);                 // E(i0, j)
            uint32_t ecx = e_in - alpha > h_in - beta ? 4u : 0u;      // its extension bit
            uint32_t nib = 0;
            int eu = 0;
            int cm = 0;                                              // column max over real rows
#pragma unroll
            for (int r = 0; r < TR; r++) {
              const int sub = (int)(int8_t)(((r < 4 ? pv.x : pv.y) >> (8 * (r & 3))) & 0xffu);
              const int G = dg + sub;                                // H(i-1,j-1) + fsbt(q_i, s_j)
              const int fo = Hc[r] - beta, fe = Fc[r] - alpha;
              const int F = max(fe, fo);                             // F(i,j)
              const int Y = max(max(G, F), 0);
              const int H = max(Y, ec);                              // H(i,j)
              const uint32_t src = H == 0 ? 0u : H == G ? 1u : H == ec ? 2u : 3u;
              nib |= (src | ecx | (fe > fo ? 8u : 0u)) << (4 * r);
              if (r == TR - 1) eu = ec;                              // E of the lane's last row
              const int yb = Y - beta, ee = ec - alpha;
              ecx = (alpha < beta && ee > yb) ? 4u : 0u;
              ec = max(ee, yb);                                      // E(i+1,j)
              cm = max(cm, i0 + r < m ? H : 0);
              dg = Hc[r];                                            // H(i, j-1): diagonal of row i+1
              Hc[r] = H;
              Fc[r] = F;
            }
            if (cm > 0 && cm >= best) {                              // rare: locate the first row reaching it
#pragma unroll
              for (int r = 0; r < TR; r++)
                if (i0 + r < m && Hc[r] == cm) {
                  if (better(cm, j, i0 + r, best, bj, bi)) { best = cm; bj = j; bi = i0 + r; }
                  break;
                }
            }
            const int hu = Hc[TR - 1];                               // (H, E) of the last row for the next lane
            D[(long long)(i0 / TR) * n + j] = (DirWord<TR>)nib;
            if (lane == nact - 1 && !last) {
              if (to_ring) ring[warp][j % kRing] = make_int2(hu, eu);
              else gout[j] = make_int2(hu, eu);
            }
            h_out = hu;
            e_out = eu;
            c_out = cc;
            hdiag = h_in;                                          // H(i0-1, j) is the next column's diagonal
          }
        }
        if (to_ring) {                                           // publish columns 0 .. min(sb, n-1)
          __threadfence_block();
          __syncwarp();
          if (lane == 0) prod[warp] = min(n, sb + 1);
        }
      }
      if (to_ring && lane == 0) {
        __threadfence_block();
        prod[warp] = n;
      }
    }
  }
  // end cell: lexicographic (max H, min j, min i) over the CTA
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int h2 = __shfl_xor_sync(0xffffffffu, best, o);
    const int j2 = __shfl_xor_sync(0xffffffffu, bj, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
    if (better(h2, j2, i2, best, bj, bi)) { best = h2; bj = j2; bi = i2; }
  }
  if (lane == 0) { s_best[warp][0] = best; s_best[warp][1] = bj; s_best[warp][2] = bi; }
  if (stalled) s_stalled = 1;
  __syncthreads();                                               // all direction words written and visible
  if (warp != 0) return;
  best = s_best[0][0]; bj = s_best[0][1]; bi = s_best[0][2];
  for (int w = 1; w < kAlignWarps; w++)
    if (better(s_best[w][0], s_best[w][1], s_best[w][2], best, bj, bi)) {
      best = s_best[w][0]; bj = s_best[w][1]; bi = s_best[w][2];
    }
  // walk back (warp 0, all lanes in step): the direction words of row blocks
  // {rb, rb-1} x columns [cj-15, cj] sit in the lanes' registers (lane = 16*dr + dc)
  // and are re-loaded only when the walk leaves that window.
  char* tmp = ops_tmp + J.tmp;
  int i = bi, j = bj, k = 0, state = 0;                          // 0 = H, 1 = E (vertical), 2 = F (horizontal)
  bool bad = s_stalled != 0;
  if (best > 0 && !bad) {
    int wrb = -100, wcj = -100;
    uint32_t win = 0u;
    for (;;) {
      if (state == 0 && (i < 0 || j < 0)) break;
      if (i < 0 || j < 0 || k > m + n) { bad = true; break; }    // inconsistent directions: reported, not hung
      const int rb = i / TR;
      if (rb > wrb || rb < wrb - 1 || j > wcj || j < wcj - 15) {
        wrb = rb;
        wcj = j;
        const int lr = wrb - (lane >> 4), lc = wcj - 15 + (lane & 15);
        win = (lr >= 0 && lc >= 0) ? (uint32_t)__ldcg(D + (long long)lr * n + lc) : 0u;
      }
      const uint32_t w = __shfl_sync(0xffffffffu, win, 16 * (wrb - rb) + (j - (wcj - 15)));
      const uint32_t nib = (w >> (4 * (i % TR))) & 15u;
      if (state == 0) {
        const uint32_t src = nib & 3u;
        if (src == 0u) break;
        if (src == 1u) { if (lane == 0) tmp[k] = 'M'; k++; i--; j--; }
        else state = src == 2u ? 1 : 2;
      } else if (state == 1) {
        if (lane == 0) tmp[k] = 'I';
        k++;
        i--;
        state = (nib & 4u) ? 1 : 0;
      } else {
        if (lane == 0) tmp[k] = 'D';
        k++;
        j--;
        state = (nib & 8u) ? 2 : 0;
      }
    }
  }
  if (lane == 0) {
    int* R = res + 6 * t;
    if (bad) {
      R[0] = -1;                                                 // the host turns this into SW_EINTERNAL
      R[1] = R[2] = R[3] = R[4] = R[5] = 0;
      k = 0;
    } else if (best == 0) {
      R[0] = R[1] = R[2] = R[3] = R[4] = R[5] = 0;
      k = 0;
    } else {
      R[0] = best;
      R[1] = i + 1;
      R[2] = bi + 1;
      R[3] = j + 1;
      R[4] = bj + 1;
      R[5] = k;
    }
    s_nops = k;
  }
  __syncwarp();
  const int nops = s_nops;
  char* out = ops_out + J.ops;
  for (int q = lane; q < nops; q += 32) out[q] = tmp[nops - 1 - q];
}

}  // namespace swk
