// Co-issue test: does op B run on a different pipe than the DPX alu op A?
// Independent chains of A and B interleaved 1:1 (and 2:1); combined rate above
// the alu pipe's 64 thread-ops/clk/SM means B issues to another pipe.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_mix2 pipe_mix2.cu
#include <cstdio>
#include <cuda_fp16.h>
#define ITER 2048
#define NCH 6
__device__ __forceinline__ unsigned hmax2(unsigned a, unsigned b) {
  unsigned r; asm volatile("max.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r; }
__device__ __forceinline__ unsigned bmax2(unsigned a, unsigned b) {
  unsigned r; asm volatile("max.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r; }
__device__ __forceinline__ unsigned fmax3u(unsigned a, unsigned b, unsigned c) {
  float r; asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(__uint_as_float(a)), "f"(__uint_as_float(b)), "f"(__uint_as_float(c))); return __float_as_uint(r); }
__device__ __forceinline__ unsigned imad(unsigned a, unsigned b, unsigned c) {
  unsigned r; asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c)); return r; }
__device__ __forceinline__ unsigned vaddmax(unsigned a, unsigned b, unsigned c) { return __viaddmax_s16x2_relu(a, b, c); }
__device__ __forceinline__ unsigned vmax3(unsigned a, unsigned b, unsigned c) { return __vimax3_s16x2_relu(a, b, c); }
__device__ __forceinline__ unsigned fmnmx(unsigned a, unsigned b) {
  float r; asm volatile("max.f32 %0, %1, %2;" : "=f"(r) : "f"(__uint_as_float(a)), "f"(__uint_as_float(b))); return __float_as_uint(r); }
__device__ __forceinline__ unsigned imnmx(unsigned a, unsigned b) {
  unsigned r; asm volatile("max.s32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r; }

template <int OP>
__device__ __forceinline__ unsigned opB(unsigned x, unsigned c, unsigned d) {
  if (OP == 0) return x;                        // none
  if (OP == 1) return hmax2(x, c);
  if (OP == 2) return bmax2(x, c);
  if (OP == 3) return fmax3u(x, c, d);
  if (OP == 4) return fmnmx(x, c);
  if (OP == 5) return imnmx(x, c);
  if (OP == 6) { unsigned r; asm volatile("add.s16x2 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(c)); return r; }
  if (OP == 7) return imad(x, c, d);
  if (OP == 8) return vaddmax(x, c, d);
  return x;
}
template <int B, int NA, int NB>
__global__ void __launch_bounds__(1024, 1) k(unsigned* out, const unsigned* cin) {
  unsigned x[NCH], y[NCH], c1 = cin[1], c2 = cin[2], c3 = cin[3];
  for (int i = 0; i < NCH; i++) { x[i] = cin[(threadIdx.x + i) & 63]; y[i] = cin[(threadIdx.x + 7 * i) & 63]; }
  for (int it = 0; it < ITER; it++) {
#pragma unroll
    for (int i = 0; i < NCH; i++) {
#pragma unroll
      for (int a = 0; a < NA; a++) x[i] = vaddmax(x[i], c1, (a == 0 && B) ? y[i] : c2 ^ a);
#pragma unroll
      for (int b = 0; b < NB; b++) y[i] = opB<B>(y[i], NA ? x[i] : y[(i + 1) % NCH], c3 ^ b);
    }
  }
  unsigned a = 0;
  for (int i = 0; i < NCH; i++) a ^= x[i] ^ y[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = a;
}
template <int B, int NA, int NB>
void run(const char* name, unsigned* d_out, unsigned* d_in, int nsm, int clk_khz) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 3; r++) {
    cudaEventRecord(e0); k<B, NA, NB><<<nsm, 1024>>>(d_out, d_in); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  const double ops = (double)(NA + (B ? NB : 0)) * ITER * NCH * 1024.0 * nsm;
  const double per_clk = ops / (best * 1e-3) / nsm / (clk_khz * 1e3);
  printf("%-26s A:B=%d:%d  %7.2f Tops/s  %6.1f thread-ops/clk/SM (at max clock)\n", name, NA, B ? NB : 0,
         ops / best / 1e9, per_clk);
}
int main() {
  int nsm, clk; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  unsigned *d_out, *d_in; cudaMalloc(&d_out, 4 * nsm * 1024); cudaMalloc(&d_in, 4 * 128);
  unsigned h[128]; for (int i = 0; i < 128; i++) h[i] = 0x00100010u + i * 0x00010001u;
  cudaMemcpy(d_in, h, 512, cudaMemcpyHostToDevice);
  run<0, 1, 1>("viaddmax alone", d_out, d_in, nsm, clk);
  run<1, 1, 1>("viaddmax | hmnmx2", d_out, d_in, nsm, clk);
  run<1, 2, 1>("viaddmax | hmnmx2", d_out, d_in, nsm, clk);
  run<2, 1, 1>("viaddmax | hmnmx2.bf16", d_out, d_in, nsm, clk);
  run<3, 1, 1>("viaddmax | fmnmx3", d_out, d_in, nsm, clk);
  run<4, 1, 1>("viaddmax | fmnmx", d_out, d_in, nsm, clk);
  run<5, 1, 1>("viaddmax | imnmx", d_out, d_in, nsm, clk);
  run<6, 1, 1>("viaddmax | vadd2", d_out, d_in, nsm, clk);
  run<7, 1, 1>("viaddmax | imad", d_out, d_in, nsm, clk);
  run<8, 1, 1>("viaddmax | viaddmax", d_out, d_in, nsm, clk);
  run<1, 0, 1>("hmnmx2 alone", d_out, d_in, nsm, clk);
  run<3, 0, 1>("fmnmx3 alone", d_out, d_in, nsm, clk);
  run<4, 0, 1>("fmnmx alone", d_out, d_in, nsm, clk);
  return 0;
}
