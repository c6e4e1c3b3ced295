// Substitution-merge variants of the int16x2 cell update with the profile in
// SHARED MEMORY and random residues per column (the k_inter16 tile loop
// without the packed-word decode and boundary traffic).  One lane holds two
// subjects (lo/hi halves); per row the pair (fsbt(q_i, s_lo), fsbt(q_i, s_hi))
// must be formed from two independent table lookups.
//   MODE 0  int8 table, LDS.64 per 8 rows per subject, PRMT (alu) per row (production)
//   MODE 1  32-bit tables LO = zext16(s), HI = s << 16; LDS.64 per 2 rows per
//           subject; D = VIADD2(VIADD2(Hprev, HI), LO): no alu op for the merge
//   MODE 2  one 32-bit zext table, D = VIADD2(IMAD(T_hi, 0x10000, Hprev), T_lo)
//   MODE 3+x mixed: rows (r % 8) < NP use MODE 0, the others MODE 1
//   (round 2, second pass) biased int16 table u = s + beta >= 0 ([25][s16] u16,
//   rows i, i+1 in one word), D = VIADD2(H(i-1) - beta, pair):
//   MODE 5  PRMT per row (0x5410 / 0x7632), no sign replication needed
//   MODE 6  even rows: pair = HFMA2(W_lo, (1.0, 0.0), W_hi << 16) (fma pipe: the
//           fp16 multiply by 1 / 0 is exact on these subnormal bit patterns),
//           odd rows: PRMT 0x7632
//   MODE 7  every row on the fma pipe (odd rows: HFMA2(W_hi, (0.0, 1.0), W_lo >> 16))
//   LW = 16 or 8: LDS.128 per 8 rows or LDS.64 per 4 rows per subject
// Reports Gcell/s (2 cells per lane-row) at 384 threads / SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o merge_ceiling merge_ceiling.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r; asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel)); return r; }
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r; asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c)); return r; }
__device__ __forceinline__ uint32_t hfma2(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r; asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c)); return r; }
__device__ __forceinline__ uint32_t mulhi(uint32_t a, uint32_t b) {
  uint32_t r; asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r; }
__device__ __forceinline__ uint4 lds128(const void* p) {
  uint4 v; asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"((uint32_t)__cvta_generic_to_shared(p))); return v; }
__device__ __forceinline__ uint2 lds64(const void* p) {
  uint2 v; asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"((uint32_t)__cvta_generic_to_shared(p))); return v; }
__host__ __device__ constexpr uint32_t sel_pair(int rr) {
  return (uint32_t)(rr | ((rr | 8) << 4) | ((4 + rr) << 8) | (((4 + rr) | 8) << 12)); }

constexpr int M = 480;          // query rows held in the tables (tile offset i0 cycles over them)

template <int MODE, int NP, int R = 48, int NT = 384>
__global__ void __launch_bounds__(NT, 1) k(uint32_t* out, int ncols, int s8, int s32) {
  extern __shared__ __align__(16) uint8_t sm[];
  int8_t* p8 = (int8_t*)sm;                                   // [25][s8] bytes
  uint32_t* lo32 = (uint32_t*)(sm + ((25 * s8 + 15) / 16) * 16);   // [25][s32]
  uint32_t* hi32 = lo32 + 25 * s32;
  for (int t = threadIdx.x; t < 25 * s8; t += blockDim.x) {
    const int r = t / s8, i = t % s8;
    p8[t] = r == 24 ? 0 : (int8_t)(((r * 7 + i * 13) % 15) - 4);
  }
  for (int t = threadIdx.x; t < 25 * s32; t += blockDim.x) {
    const int r = t / s32, i = t % s32;
    const int v = r == 24 ? 0 : (((r * 7 + i * 13) % 15) - 4);
    lo32[t] = (uint32_t)v & 0xffffu;
    hi32[t] = (uint32_t)v << 16;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t D[R], F[R];
#pragma unroll
  for (int r = 0; r < R; r++) { D[r] = 0; F[r] = 0; }
  uint32_t e = 0, hmax = 0, na2 = 0xfffefffeu, nb2 = 0xfff4fff4u;
  uint32_t w = 0x9e3779b9u * (threadIdx.x + 1 + blockIdx.x * 977);
  const int i0 = R * (blockIdx.x % (M / R));
  for (int j = 0; j < ncols; j++) {
    w = w * 1664525u + 1013904223u;
    const uint32_t rlo = ((w >> 24) * 25u) >> 8, rhi = (((w >> 16) & 255u) * 25u) >> 8;
    const int8_t* a8 = p8 + rlo * s8 + i0;
    const int8_t* b8 = p8 + rhi * s8 + i0;
    const uint32_t* a32 = (MODE == 1 || MODE >= 3 ? lo32 : lo32) + rlo * s32 + i0;
    const uint32_t* b32 = (MODE == 2 ? lo32 : hi32) + rhi * s32 + i0;
    uint32_t hprev = e ^ (uint32_t)j, hodd = 0;
    e = 0;
#pragma unroll
    for (int k8 = 0; k8 < R / 8; k8++) {
      uint2 a, b, la, lb;
      if (MODE == 0 || MODE >= 3) {
        a = *reinterpret_cast<const uint2*>(a8 + 8 * k8);
        b = *reinterpret_cast<const uint2*>(b8 + 8 * k8);
      }
#pragma unroll
      for (int rr = 0; rr < 8; rr++) {
        const int r = 8 * k8 + rr;
        const uint32_t h = __vimax3_s16x2(D[r], e, F[r]);
        const bool use_prmt = MODE == 0 || (MODE >= 3 && rr < NP);
        if (use_prmt) {
          const uint32_t sn = prmt(rr < 4 ? a.x : a.y, rr < 4 ? b.x : b.y, sel_pair(rr & 3));
          D[r] = __vadd2(hprev, sn);
        } else {
          if (!(r & 1) || (MODE >= 3 && rr == NP)) { la = lds64(a32 + (r & ~1)); lb = lds64(b32 + (r & ~1)); }
          const uint32_t lv = (r & 1) ? la.y : la.x, hv = (r & 1) ? lb.y : lb.x;
          if (MODE == 2) D[r] = __vadd2(imad(hv, 0x10000u, hprev), lv);
          else D[r] = __vadd2(__vadd2(hprev, hv), lv);
        }
        const uint32_t hb = __vadd2(h, nb2);
        e = __viaddmax_s16x2_relu(e, na2, hb);
        F[r] = __viaddmax_s16x2_relu(F[r], na2, hb);
        if (rr & 1) hmax = __vimax3_s16x2(hmax, hodd, h);
        else hodd = h;
        hprev = h;
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = hmax ^ e;
}

// Biased int16 table variants (MODE 5..7).  s16 = row stride in u16 units (multiple of 8).
template <int MODE, int LW, int R = 48, int NT = 384>
__global__ void __launch_bounds__(NT, 1) k16(uint32_t* out, int ncols, int s16) {
  extern __shared__ __align__(16) uint8_t sm[];
  uint16_t* t16 = (uint16_t*)sm;                              // [25][s16]
  for (int t = threadIdx.x; t < 25 * s16; t += blockDim.x) {
    const int r = t / s16, i = t % s16;
    t16[t] = (uint16_t)(r == 24 ? 12 : (((r * 7 + i * 13) % 15) - 4) + 12);
  }
  __syncthreads();
  uint32_t D[R], F[R];
#pragma unroll
  for (int r = 0; r < R; r++) { D[r] = 0; F[r] = 0; }
  uint32_t e = 0, hmax = 0;
  const uint32_t na2 = 0xfffefffeu, nb2 = 0xfff4fff4u, one_lo = 0x00003c00u, one_hi = 0x3c000000u;
  uint32_t w = 0x9e3779b9u * (threadIdx.x + 1 + blockIdx.x * 977);
  const int i0 = R * (blockIdx.x % (M / R));
  for (int j = 0; j < ncols; j++) {
    w = w * 1664525u + 1013904223u;
    const uint32_t rlo = ((w >> 24) * 25u) >> 8, rhi = (((w >> 16) & 255u) * 25u) >> 8;
    const uint16_t* a16 = t16 + rlo * s16 + i0;
    const uint16_t* b16 = t16 + rhi * s16 + i0;
    uint32_t hbprev = e ^ (uint32_t)j, hodd = 0;
    e = 0;
    uint32_t A[LW / 4], B[LW / 4];
#pragma unroll
    for (int r = 0; r < R; r++) {
      constexpr int RPL = LW / 2;                            // rows per load
      if (r % RPL == 0) {
        if constexpr (LW == 16) {
          const uint4 x = lds128(a16 + r), y = lds128(b16 + r);
          A[0] = x.x; A[1] = x.y; A[2] = x.z; A[3] = x.w; B[0] = y.x; B[1] = y.y; B[2] = y.z; B[3] = y.w;
        } else {
          const uint2 x = lds64(a16 + r), y = lds64(b16 + r);
          A[0] = x.x; A[1] = x.y; B[0] = y.x; B[1] = y.y;
        }
      }
      const uint32_t wl = A[(r % RPL) / 2], wh = B[(r % RPL) / 2];
      uint32_t pr;
      if (MODE == 5) pr = prmt(wl, wh, (r & 1) ? 0x7632u : 0x5410u);
      else if (!(r & 1)) pr = hfma2(wl, one_lo, imad(wh, 0x10000u, 0u));
      else if (MODE == 6) pr = prmt(wl, wh, 0x7632u);
      else pr = hfma2(wh, one_hi, mulhi(wl, 0x10000u));
      const uint32_t h = __vimax3_s16x2(D[r], e, F[r]);
      D[r] = __vadd2(hbprev, pr);
      const uint32_t hb = __vadd2(h, nb2);
      e = __viaddmax_s16x2_relu(e, na2, hb);
      F[r] = __viaddmax_s16x2_relu(F[r], na2, hb);
      if (r & 1) hmax = __vimax3_s16x2(hmax, hodd, h);
      else hodd = h;
      hbprev = hb;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = hmax ^ e;
}


// MODE 8 (round 2, third pass): PAIR profile of one R-row query tile in shared
// memory, [625 = 25 x 25 residue pairs][SP words], word = (fsbt(q_i, b) << 16) |
// (fsbt(q_i, a) & 0xffff): one LDS.128 per 4 rows per LANE (4 B per lane-row), no
// merge instruction at all.  The first NPAIR rows of the tile use it, the other
// R - NPAIR rows the int8 profile + PRMT (mode 0).  SP = NPAIR + 4 words keeps
// 16-byte alignment and spreads the 625 rows over all eight 16-byte bank groups.
// A production kernel would need every warp of the CTA on the SAME query tile
// (tile-major schedule, table rebuilt per tile).
template <int NPAIR, int R = 48, int NT = 384>
__global__ void __launch_bounds__(NT, 1) kp(uint32_t* out, int ncols, int s8) {
  extern __shared__ __align__(16) uint8_t sm[];
  constexpr int SP = NPAIR + 4;
  int8_t* p8 = (int8_t*)sm;                                          // [25][s8] bytes
  uint32_t* pp = (uint32_t*)(sm + ((25 * s8 + 15) / 16) * 16);       // [625][SP]
  const int i0 = R * (blockIdx.x % (M / R));
  for (int t = threadIdx.x; t < 25 * s8; t += blockDim.x) {
    const int r = t / s8, i = t % s8;
    p8[t] = r == 24 ? 0 : (int8_t)(((r * 7 + i * 13) % 15) - 4);
  }
  for (int t = threadIdx.x; t < 625 * SP; t += blockDim.x) {
    const int pr = t / SP, i = t % SP + i0, ra = pr / 25, rb = pr % 25;
    const int va = ra == 24 ? 0 : (((ra * 7 + i * 13) % 15) - 4), vb = rb == 24 ? 0 : (((rb * 7 + i * 13) % 15) - 4);
    pp[t] = ((uint32_t)va & 0xffffu) | ((uint32_t)vb << 16);
  }
  __syncthreads();
  uint32_t D[R], F[R];
#pragma unroll
  for (int r = 0; r < R; r++) { D[r] = 0; F[r] = 0; }
  uint32_t e = 0, hmax = 0, na2 = 0xfffefffeu, nb2 = 0xfff4fff4u;
  uint32_t w = 0x9e3779b9u * (threadIdx.x + 1 + blockIdx.x * 977);
  for (int j = 0; j < ncols; j++) {
    w = w * 1664525u + 1013904223u;
    const uint32_t rlo = ((w >> 24) * 25u) >> 8, rhi = (((w >> 16) & 255u) * 25u) >> 8;
    const int8_t* a8 = p8 + rlo * s8 + i0;
    const int8_t* b8 = p8 + rhi * s8 + i0;
    const uint32_t* pq = pp + (rlo * 25u + rhi) * SP;
    uint32_t hprev = e ^ (uint32_t)j, hodd = 0;
    e = 0;
#pragma unroll
    for (int k8 = 0; k8 < R / 8; k8++) {
      uint2 a, b;
      uint4 q0, q1;
      if (8 * k8 < NPAIR) { q0 = lds128(pq + 8 * k8); q1 = lds128(pq + 8 * k8 + 4); }
      else {
        a = *reinterpret_cast<const uint2*>(a8 + 8 * k8);
        b = *reinterpret_cast<const uint2*>(b8 + 8 * k8);
      }
#pragma unroll
      for (int rr = 0; rr < 8; rr++) {
        const int r = 8 * k8 + rr;
        const uint32_t h = __vimax3_s16x2(D[r], e, F[r]);
        uint32_t sn;
        if (8 * k8 < NPAIR) {
          const uint4& q = rr < 4 ? q0 : q1;
          sn = (rr & 3) == 0 ? q.x : (rr & 3) == 1 ? q.y : (rr & 3) == 2 ? q.z : q.w;
        } else {
          sn = prmt(rr < 4 ? a.x : a.y, rr < 4 ? b.x : b.y, sel_pair(rr & 3));
        }
        D[r] = __vadd2(hprev, sn);
        const uint32_t hb = __vadd2(h, nb2);
        e = __viaddmax_s16x2_relu(e, na2, hb);
        F[r] = __viaddmax_s16x2_relu(F[r], na2, hb);
        if (rr & 1) hmax = __vimax3_s16x2(hmax, hodd, h);
        else hodd = h;
        hprev = h;
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = hmax ^ e;
}

template <int NPAIR, int R = 48, int NT = 384>
void runp(const char* name, uint32_t* d_out, int nsm) {
  const int ncols = 4096, threads = NT;
  const int s8 = M + 8;
  const size_t smem = ((25 * s8 + 15) / 16) * 16 + 625 * (size_t)(NPAIR + 4) * 4;
  cudaFuncSetAttribute(kp<NPAIR, R, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; rep++) {
    cudaEventRecord(e0); kp<NPAIR, R, NT><<<nsm, threads, smem>>>(d_out, ncols, s8); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (rep && ms < best) best = ms;
  }
  cudaError_t err = cudaGetLastError();
  const double cells = 2.0 * R * ncols * threads * (double)nsm;
  printf("%-34s R=%d NT=%d pair rows %d of %d, smem %zu B  %.1f Gcell/s %s\n", name, R, NT, NPAIR, R, smem,
         cells / (best * 1e-3) / 1e9, err ? cudaGetErrorString(err) : "");
}


// MODE 9: mode 0 (int8 profile + PRMT) with ONE LDS.128 per 16 rows per subject
// instead of LDS.64 per 8 rows (row stride 16 * odd bytes).
template <int R = 48, int NT = 384>
__global__ void __launch_bounds__(NT, 1) k9(uint32_t* out, int ncols, int s8) {
  extern __shared__ __align__(16) uint8_t sm[];
  int8_t* p8 = (int8_t*)sm;
  for (int t = threadIdx.x; t < 25 * s8; t += blockDim.x) {
    const int r = t / s8, i = t % s8;
    p8[t] = r == 24 ? 0 : (int8_t)(((r * 7 + i * 13) % 15) - 4);
  }
  __syncthreads();
  uint32_t D[R], F[R];
#pragma unroll
  for (int r = 0; r < R; r++) { D[r] = 0; F[r] = 0; }
  uint32_t e = 0, hmax = 0, na2 = 0xfffefffeu, nb2 = 0xfff4fff4u;
  uint32_t w = 0x9e3779b9u * (threadIdx.x + 1 + blockIdx.x * 977);
  const int i0 = R * (blockIdx.x % (M / R));
  for (int j = 0; j < ncols; j++) {
    w = w * 1664525u + 1013904223u;
    const uint32_t rlo = ((w >> 24) * 25u) >> 8, rhi = (((w >> 16) & 255u) * 25u) >> 8;
    const int8_t* a8 = p8 + rlo * s8 + i0;
    const int8_t* b8 = p8 + rhi * s8 + i0;
    uint32_t hprev = e ^ (uint32_t)j, hodd = 0;
    e = 0;
#pragma unroll
    for (int k16 = 0; k16 < R / 16; k16++) {
      const uint4 a = lds128(a8 + 16 * k16), b = lds128(b8 + 16 * k16);
      const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int rr = 0; rr < 16; rr++) {
        const int r = 16 * k16 + rr;
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
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = hmax ^ e;
}
template <int R = 48, int NT = 384>
void run9(uint32_t* d_out, int nsm, int s8) {
  const int ncols = 4096, threads = NT;
  const size_t smem = 25 * (size_t)s8;
  cudaFuncSetAttribute(k9<R, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; rep++) {
    cudaEventRecord(e0); k9<R, NT><<<nsm, threads, smem>>>(d_out, ncols, s8); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (rep && ms < best) best = ms;
  }
  cudaError_t err = cudaGetLastError();
  const double cells = 2.0 * R * ncols * threads * (double)nsm;
  printf("mode9 int8+PRMT, LDS.128 per 16 rows  R=%d NT=%d s8=%d  %.1f Gcell/s %s\n", R, NT, s8,
         cells / (best * 1e-3) / 1e9, err ? cudaGetErrorString(err) : "");
}

template <int MODE, int LW, int R = 48, int NT = 384>
void run16(const char* name, uint32_t* d_out, int nsm, int s16) {
  const int ncols = 4096, threads = NT;
  const size_t smem = 25 * (size_t)s16 * 2;
  cudaFuncSetAttribute(k16<MODE, LW, R, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; rep++) {
    cudaEventRecord(e0); k16<MODE, LW, R, NT><<<nsm, threads, smem>>>(d_out, ncols, s16); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (rep && ms < best) best = ms;
  }
  cudaError_t err = cudaGetLastError();
  const double cells = 2.0 * R * ncols * threads * (double)nsm;
  printf("%-34s R=%d NT=%d s16=%d LW=%d  %.1f Gcell/s %s\n", name, R, NT, s16, LW, cells / (best * 1e-3) / 1e9, err ? cudaGetErrorString(err) : "");
}

template <int MODE, int NP = 0, int R = 48, int NT = 384>
void run(const char* name, uint32_t* d_out, int nsm, int s32) {
  const int ncols = 4096, threads = NT;
  const int s8 = M + 8;
  const size_t smem = ((25 * s8 + 15) / 16) * 16 + 2 * 25 * (size_t)s32 * 4;
  cudaFuncSetAttribute(k<MODE, NP, R, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; rep++) {
    cudaEventRecord(e0); k<MODE, NP, R, NT><<<nsm, threads, smem>>>(d_out, ncols, s8, s32); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (rep && ms < best) best = ms;
  }
  cudaError_t err = cudaGetLastError();
  const double cells = 2.0 * R * ncols * threads * (double)nsm;
  printf("%-34s R=%d NT=%d s32=%d  %.1f Gcell/s %s\n", name, R, NT, s32, cells / (best * 1e-3) / 1e9, err ? cudaGetErrorString(err) : "");
}
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* d_out; cudaMalloc(&d_out, 4 * nsm * 512);
  if (getenv("PAIR")) {
    run<0>("mode0 int8+PRMT", d_out, nsm, M + 2);
    runp<0>("mode8 pair profile", d_out, nsm);
    runp<8>("mode8 pair profile", d_out, nsm);
    runp<16>("mode8 pair profile", d_out, nsm);
    runp<24>("mode8 pair profile", d_out, nsm);
    runp<32>("mode8 pair profile", d_out, nsm);
    runp<40>("mode8 pair profile", d_out, nsm);
    runp<48>("mode8 pair profile", d_out, nsm);
    runp<32, 32, 512>("mode8 pair profile", d_out, nsm);
    runp<16, 32, 512>("mode8 pair profile", d_out, nsm);
    runp<40, 40, 384>("mode8 pair profile", d_out, nsm);
    runp<64, 64, 256>("mode8 pair profile", d_out, nsm);
    return 0;
  }
  if (getenv("LDS128")) {
    run<0>("mode0 int8+PRMT", d_out, nsm, M + 2);
    for (int s8 : {496, 528, 560, 592, 624}) run9<48, 384>(d_out, nsm, s8);
    run9<32, 512>(d_out, nsm, 496);
    run9<64, 256>(d_out, nsm, 496);
    return 0;
  }
  if (getenv("INT16")) {
    run<0>("mode0 int8+PRMT", d_out, nsm, M + 2);
    for (int s16 : {M + 8, M + 16, M + 32, M + 64}) {
      run16<5, 16>("mode5 int16 PRMT", d_out, nsm, s16);
      run16<6, 16>("mode6 int16 HFMA2/PRMT", d_out, nsm, s16);
      run16<7, 16>("mode7 int16 HFMA2 all", d_out, nsm, s16);
      run16<5, 8>("mode5 int16 PRMT", d_out, nsm, s16);
      run16<6, 8>("mode6 int16 HFMA2/PRMT", d_out, nsm, s16);
      run16<7, 8>("mode7 int16 HFMA2 all", d_out, nsm, s16);
    }
    return 0;
  }
  if (getenv("TILES")) {
    run<0, 0, 48, 384>("mode0", d_out, nsm, M + 2);
    run<0, 0, 32, 512>("mode0", d_out, nsm, M + 2);
    run<0, 0, 64, 256>("mode0", d_out, nsm, M + 2);
    run<0, 0, 80, 256>("mode0", d_out, nsm, M + 2);
    run<0, 0, 96, 256>("mode0", d_out, nsm, M + 2);
    run<0, 0, 120, 256>("mode0", d_out, nsm, M + 2);
    run<0, 0, 96, 320>("mode0", d_out, nsm, M + 2);
    run<0, 0, 64, 320>("mode0", d_out, nsm, M + 2);
    run<0, 0, 40, 384>("mode0", d_out, nsm, M + 2);
    run<0, 0, 40, 448>("mode0", d_out, nsm, M + 2);
    run<0, 0, 40, 416>("mode0", d_out, nsm, M + 2);
    run<0, 0, 32, 576>("mode0", d_out, nsm, M + 2);
    run<0, 0, 32, 544>("mode0", d_out, nsm, M + 2);
    run<0, 0, 48, 416>("mode0", d_out, nsm, M + 2);
    return 0;
  }
  for (int s32 : {M + 2, M + 4, M + 1 + 1 + 32}) {
    run<0>("mode0 int8+PRMT", d_out, nsm, s32);
    run<1>("mode1 32b VIADD2 x2", d_out, nsm, s32);
    run<2>("mode2 32b IMAD+VIADD2", d_out, nsm, s32);
    run<3, 6>("mode3 mixed 6/8 PRMT", d_out, nsm, s32);
    run<3, 4>("mode3 mixed 4/8 PRMT", d_out, nsm, s32);
    run<3, 2>("mode3 mixed 2/8 PRMT", d_out, nsm, s32);
    run<3, 1>("mode3 mixed 1/8 PRMT", d_out, nsm, s32);
  }
  return 0;
}
