// Which pipe runs HMNMX2 / VIMNMX(2-input) / IMNMX?  Each chain alternates the op under
// test with a dependent HADD2 (fma-side pipe).  Equal rate to HADD2|HADD2 => same pipe.
#include <cstdio>
#include <cuda_fp16.h>
#define ITER 4096
#define NCH 8
__device__ __forceinline__ unsigned hadd2(unsigned a, unsigned b) { __half2 x = *reinterpret_cast<__half2*>(&a), y = *reinterpret_cast<__half2*>(&b); __half2 r = __hadd2(x, y); return *reinterpret_cast<unsigned*>(&r); }
__device__ __forceinline__ unsigned hmax2(unsigned a, unsigned b) { __half2 x = *reinterpret_cast<__half2*>(&a), y = *reinterpret_cast<__half2*>(&b); __half2 r = __hmax2(x, y); return *reinterpret_cast<unsigned*>(&r); }
template <int OP>
__device__ __forceinline__ unsigned op(unsigned x, unsigned c) {
  if (OP == 0) return hadd2(x, c);
  if (OP == 1) return hmax2(x, c);
  if (OP == 2) return __vmaxs2(x, c);
  if (OP == 3) return (unsigned)max((int)x, (int)c);
  if (OP == 4) return __vimax3_s16x2(x, c, c ^ 0x10001u);
  if (OP == 5) return __vadd2(x, c);
  return x;
}
template <int OP>
__global__ void k(unsigned* out, const unsigned* cin) {
  unsigned x[NCH], c1[NCH], c2[NCH];
  for (int i = 0; i < NCH; i++) { x[i] = cin[threadIdx.x % 64 + i]; c1[i] = cin[i + 8]; c2[i] = cin[i + 16]; }
  for (int it = 0; it < ITER; it++) {
#pragma unroll
    for (int i = 0; i < NCH; i++) { x[i] = op<OP>(x[i], c1[i]); x[i] = hadd2(x[i], c2[i]); }
  }
  unsigned a = 0;
  for (int i = 0; i < NCH; i++) a ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = a;
}
template <int OP>
void run(const char* name, unsigned* d_out, unsigned* d_in, int nsm) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int r = 0; r < 2; r++) { cudaEventRecord(e0); k<OP><<<nsm, 1024>>>(d_out, d_in); cudaEventRecord(e1); cudaEventSynchronize(e1); }
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = 2.0 * ITER * NCH * 1024.0 * nsm;
  printf("%-14s|hadd2 : %.2f Tops/s (%.1f thread-ops/clk/SM at 1.9 GHz)\n", name, ops / ms / 1e9, ops / (ms * 1e-3) / nsm / 1.9e9);
}
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned *d_out, *d_in; cudaMalloc(&d_out, 4 * nsm * 1024); cudaMalloc(&d_in, 4 * 128);
  unsigned h[128]; for (int i = 0; i < 128; i++) h[i] = 0x3c003c00u + i * 0x00010001u; cudaMemcpy(d_in, h, 512, cudaMemcpyHostToDevice);
  run<0>("hadd2", d_out, d_in, nsm);
  run<1>("hmax2", d_out, d_in, nsm);
  run<2>("vimnmx.s16x2", d_out, d_in, nsm);
  run<3>("imnmx", d_out, d_in, nsm);
  run<4>("vimnmx3.s16x2", d_out, d_in, nsm);
  run<5>("vadd2", d_out, d_in, nsm);
  return 0;
}
