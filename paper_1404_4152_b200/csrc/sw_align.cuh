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
#include <cuda_runtime.h>

namespace swk {

struct AlignJob {
  long long word0;   // first packed word (uint2 units) of the subject's group + its lane
  long long dir;     // direction words of this job (uint32 units): (m_pad/TR) x n
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

// res[t*6 + ...] = score, q_begin, q_end, s_begin, s_end, n_ops
template <int TR>
__global__ void __launch_bounds__(32)
k_align(const uint2* __restrict__ words, const AlignJob* __restrict__ jobs, int n_jobs,
        const int8_t* __restrict__ prof, int prof_smem, int stride, int m, int m_pad, int alpha, int beta,
        uint32_t* __restrict__ dir, int2* __restrict__ bnd, char* __restrict__ ops_out,
        char* __restrict__ ops_tmp, int* __restrict__ res) {
  const int t = blockIdx.x;
  if (t >= n_jobs) return;
  const int lane = threadIdx.x;
  const AlignJob J = jobs[t];
  const int n = J.n;
  const uint32_t* wp = reinterpret_cast<const uint32_t*>(words + J.word0) + J.half;   // word w at wp[64 w]
  uint32_t* D = dir + J.dir;
  int2* B = bnd + J.bnd;
  int best = 0, bj = 0x7fffffff, bi = 0x7fffffff;
  // the int8 query profile is staged in shared memory (prof_smem bytes, 0 = read through L1)
  extern __shared__ __align__(16) int8_t s_prof[];
  const int8_t* P = prof;
  if (prof_smem) {
    const uint4* src = reinterpret_cast<const uint4*>(prof);
    uint4* dst = reinterpret_cast<uint4*>(s_prof);
    for (int k = lane; k < prof_smem / 16; k += 32) dst[k] = __ldg(src + k);
    __syncwarp();
    P = s_prof;
  }
  int pass = 0;
  for (int base = 0; n > 0 && base < m_pad; base += 32 * TR, pass++) {
    const int nact = min(32, (m_pad - base) / TR);
    const bool first = base == 0, last = base + 32 * TR >= m_pad;
    const int2* gin = B + (long long)(pass & 1) * n;            // written by the previous pass
    int2* gout = B + (long long)((pass + 1) & 1) * n;
    const int i0 = base + lane * TR;
    const int8_t* pr = P + i0;
    int Hc[TR], Fc[TR];                                          // H(i, j-1), F(i, j-1)
#pragma unroll
    for (int r = 0; r < TR; r++) { Hc[r] = 0; Fc[r] = 0; }        // H(i,0) = F(i,0) = 0
    int h_out = 0, e_out = 0, hdiag = 0;                         // hdiag = H(i0-1, j-1)
    uint32_t c_out = 0;                                          // residue of the column this lane just did
    // lane 0's per-step inputs (residue of column s, boundary row of column s)
    // are fetched 32 steps at a time, one block ahead, and handed over by SHFL
    auto fetch = [&](int sb, uint32_t& rc, int2& gv) {
      const int c = sb + lane;
      rc = c < n ? (__ldg(wp + 64 * (c / 6)) >> (5 * (c % 6))) & 31u : 0u;
      gv = (!first && c < n) ? gin[c] : make_int2(0, 0);
    };
    uint32_t rc_cur, rc_nxt;
    int2 gv_cur, gv_nxt;
    fetch(0, rc_cur, gv_cur);
    fetch(32, rc_nxt, gv_nxt);
    const int nsteps = n + nact - 1;
    for (int sb = 0; sb < nsteps; sb += 32) {
#pragma unroll 1
      for (int tt = 0; tt < 32; tt++) {
        const int s = sb + tt;
        if (s >= nsteps) break;
        int h_in = __shfl_up_sync(0xffffffffu, h_out, 1);
        int e_in = __shfl_up_sync(0xffffffffu, e_out, 1);
        uint32_t c = __shfl_up_sync(0xffffffffu, c_out, 1);
        const uint32_t c0 = __shfl_sync(0xffffffffu, rc_cur, tt);
        const int g0x = __shfl_sync(0xffffffffu, gv_cur.x, tt);
        const int g0y = __shfl_sync(0xffffffffu, gv_cur.y, tt);
        const int j = s - lane;
        if (lane == 0) {                                         // row base-1 of column j, residue s_j
          h_in = g0x;
          e_in = g0y;
          c = c0;
        }
        if (lane < nact && j >= 0 && j < n) {
          const uint2 pv = *reinterpret_cast<const uint2*>(pr + c * stride);
          int hu = h_in, eu = e_in, dg = hdiag;
          uint32_t nib = 0;
#pragma unroll
          for (int r = 0; r < TR; r++) {
            const int sub = (int)(int8_t)(((r < 4 ? pv.x : pv.y) >> (8 * (r & 3))) & 0xffu);
            const int G = dg + sub;                                // H(i-1,j-1) + fsbt(q_i, s_j)
            const int eo = hu - beta, ee = eu - alpha;
            const int E = max(ee, eo);                             // E(i,j)
            const int fo = Hc[r] - beta, fe = Fc[r] - alpha;
            const int F = max(fe, fo);                             // F(i,j)
            const int H = max(max(0, G), max(E, F));
            const uint32_t src = H == 0 ? 0u : H == G ? 1u : H == E ? 2u : 3u;
            nib |= (src | (ee > eo ? 4u : 0u) | (fe > fo ? 8u : 0u)) << (4 * r);
            const int i = i0 + r;
            if (i < m && better(H, j, i, best, bj, bi)) { best = H; bj = j; bi = i; }
            dg = Hc[r];                                            // H(i, j-1): diagonal of row i+1
            Hc[r] = H;
            Fc[r] = F;
            hu = H;
            eu = E;
          }
          D[(long long)(i0 / TR) * n + j] = nib;
          if (!last && lane == nact - 1) gout[j] = make_int2(hu, eu);
          h_out = hu;
          e_out = eu;
          c_out = c;
          hdiag = h_in;                                            // H(i0-1, j) is the next column's diagonal
        }
      }
      rc_cur = rc_nxt;
      gv_cur = gv_nxt;
      fetch(sb + 64, rc_nxt, gv_nxt);
    }
    __syncwarp();
  }
  // end cell: lexicographic (max H, min j, min i) over the warp
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int h2 = __shfl_xor_sync(0xffffffffu, best, o);
    const int j2 = __shfl_xor_sync(0xffffffffu, bj, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
    if (better(h2, j2, i2, best, bj, bi)) { best = h2; bj = j2; bi = i2; }
  }
  __syncwarp();
  __shared__ int s_nops;
  if (lane == 0) {
    int* R = res + 6 * t;
    if (best == 0) {
      R[0] = R[1] = R[2] = R[3] = R[4] = R[5] = 0;
      s_nops = 0;
    } else {
      char* tmp = ops_tmp + J.tmp;
      int i = bi, j = bj, k = 0, state = 0;                      // 0 = H, 1 = E (vertical), 2 = F (horizontal)
      for (;;) {
        if (state == 0 && (i < 0 || j < 0)) break;
        const uint32_t nib = (__ldcg(D + (long long)(i / TR) * n + j) >> (4 * (i % TR))) & 15u;
        if (state == 0) {
          const uint32_t src = nib & 3u;
          if (src == 0u) break;
          if (src == 1u) { tmp[k++] = 'M'; i--; j--; }
          else state = src == 2u ? 1 : 2;
        } else if (state == 1) {
          tmp[k++] = 'I';
          i--;
          state = (nib & 4u) ? 1 : 0;
        } else {
          tmp[k++] = 'D';
          j--;
          state = (nib & 8u) ? 2 : 0;
        }
      }
      R[0] = best;
      R[1] = i + 1;
      R[2] = bi + 1;
      R[3] = j + 1;
      R[4] = bj + 1;
      R[5] = k;
      s_nops = k;
    }
  }
  __syncwarp();
  const int nops = s_nops;
  const char* tmp = ops_tmp + J.tmp;
  char* out = ops_out + J.ops;
  for (int k = lane; k < nops; k += 32) out[k] = tmp[nops - 1 - k];
}

}  // namespace swk
