// Ceiling of the int16x2 cell update's instruction mix with no memory traffic:
// the col16 row sequence (VIMNMX3, PRMT, 2 VIADD.16x2, 2 VIADDMNMX.RELU, 1/2
// VIMNMX3) over R register rows, profile bytes taken from registers.
// Reports Gcell/s for 12 warps/SM (the kernel's launch) and 16 warps/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cell_ceiling cell_ceiling.cu
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r; asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel)); return r; }
__host__ __device__ constexpr uint32_t sel_pair(int rr) {
  return (uint32_t)(rr | ((rr | 8) << 4) | ((4 + rr) << 8) | (((4 + rr) | 8) << 12)); }
template <int R, int MODE>
__global__ void __launch_bounds__(384, 1) k(uint32_t* out, const uint32_t* in, int ncols) {
  uint32_t D[R], F[R];
  for (int r = 0; r < R; r++) { D[r] = in[r & 63]; F[r] = 0; }
  uint32_t e = 0, hmax = 0, na2 = 0xfffefffeu, nb2 = 0xfff4fff4u;
  uint32_t a = in[threadIdx.x & 63], b = in[(threadIdx.x + 5) & 63];
  for (int j = 0; j < ncols; j++) {
    uint32_t hprev = e ^ j, hodd = 0;
    e = 0;
    uint32_t pa[R / 4], pb[R / 4];
#pragma unroll
    for (int k = 0; k < R / 4; k++) { pa[k] = a * (2 * k + 3); pb[k] = b * (2 * k + 5); }
#pragma unroll
    for (int r = 0; r < R; r++) {
      const uint32_t h = __vimax3_s16x2(D[r], e, F[r]);
      uint32_t sn;
      if (MODE == 0) sn = prmt(pa[r / 4], pb[r / 4], sel_pair(r & 3));
      else sn = pa[r / 4];                          // no PRMT (pair-profile form)
      D[r] = __vadd2(hprev, sn);
      const uint32_t hb = __vadd2(h, nb2);
      e = __viaddmax_s16x2_relu(e, na2, hb);
      F[r] = __viaddmax_s16x2_relu(F[r], na2, hb);
      if (r & 1) hmax = __vimax3_s16x2(hmax, hodd, h);
      else hodd = h;
      hprev = h;
    }
    a = a * 0x9e3779b9u + j;                        // next column's profile word (IMAD, fma pipe)
    b = b ^ a;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = hmax ^ e;
}
template <int R, int MODE>
void run(const char* name, int threads, uint32_t* d_out, uint32_t* d_in, int nsm) {
  const int ncols = 4096;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 3; rep++) {
    cudaEventRecord(e0); k<R, MODE><<<nsm, threads>>>(d_out, d_in, ncols); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  const double cells = 2.0 * R * ncols * threads * (double)nsm;
  printf("%-28s R=%d threads=%d  %.1f Gcell/s\n", name, R, threads, cells / (best * 1e-3) / 1e9);
}
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  uint32_t *d_out, *d_in; cudaMalloc(&d_out, 4 * nsm * 512); cudaMalloc(&d_in, 4 * 64);
  uint32_t h[64]; for (int i = 0; i < 64; i++) h[i] = 0x01ff02feu * (i + 1); cudaMemcpy(d_in, h, 256, cudaMemcpyHostToDevice);
  run<48, 0>("col16 mix (PRMT)", 384, d_out, d_in, nsm);
  run<32, 0>("col16 mix (PRMT)", 384, d_out, d_in, nsm);
  run<48, 1>("no PRMT", 384, d_out, d_in, nsm);
  return 0;
}
