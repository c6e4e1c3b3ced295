// Does VIADDMNMX/VIMNMX3 .S16x2 keep 64 ops/clk/SM when all three sources are
// distinct, varying registers (as in the SW cell update) rather than loop-invariant?
#include <cstdio>
#include <cstdint>
#define ITER 2048
template <int V>
__global__ void k(uint32_t* out, uint32_t seed) {
  uint32_t x[12];
#pragma unroll
  for (int i = 0; i < 12; i++) x[i] = seed * (threadIdx.x + 3 * i + 1);
  const uint32_t c1 = seed ^ 0x00050005u;
  for (int it = 0; it < ITER; it++) {
#pragma unroll
    for (int i = 0; i < 12; i++) {
      if (V == 0) x[i] = __viaddmax_s16x2(x[i], c1, c1 ^ 0x10001u);                       // invariant sources
      if (V == 1) x[i] = __viaddmax_s16x2(x[i], x[(i + 4) % 12], x[(i + 8) % 12]);       // 3 varying sources
      if (V == 2) x[i] = __vimax3_s16x2(x[i], x[(i + 4) % 12], x[(i + 8) % 12]);
      if (V == 3) x[i] = __viaddmax_s16x2_relu(x[i], c1, x[(i + 6) % 12]);                // E/F update shape
    }
  }
  uint32_t a = 0;
#pragma unroll
  for (int i = 0; i < 12; i++) a ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = a;
}
template <int V>
void run(const char* name, uint32_t* d, int nsm) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int r = 0; r < 2; r++) { cudaEventRecord(e0); k<V><<<nsm * 2, 512>>>(d, 7); cudaEventRecord(e1); cudaEventSynchronize(e1); }
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = 12.0 * ITER * 512 * 2 * nsm;
  printf("%-28s %.2f Tops/s = %.1f thread-ops/clk/SM @1.965GHz\n", name, ops / ms / 1e9, ops / (ms * 1e-3) / nsm / 1.965e9);
}
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* d; cudaMalloc(&d, 4 * nsm * 1024);
  run<0>("viaddmax invariant srcs", d, nsm);
  run<1>("viaddmax 3 varying srcs", d, nsm);
  run<2>("vimax3 3 varying srcs", d, nsm);
  run<3>("viaddmax.relu (x,c,y)", d, nsm);
  return 0;
}
