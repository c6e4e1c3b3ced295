// Dependent-chain latency (cycles) of the cell-update instructions, one warp:
// VIADDMNMX.S16x2, VIMNMX3.S16x2, VIADD.16x2, PRMT, SHFL.UP and the row chain
// of col16 (h = max3(D,e,F); hb = h - beta; e = max(e - alpha, hb)).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dpx_latency dpx_latency.cu
#include <cstdio>
#include <cstdint>
#define N 4096
template <int OP>
__global__ void k(uint32_t* out, uint32_t a, uint32_t b, long long* cyc) {
  uint32_t x = threadIdx.x + a, y = b;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; i++) {
    if (OP == 0) x = __viaddmax_s16x2_relu(x, a, y);
    if (OP == 1) x = __vimax3_s16x2(x, a, y);
    if (OP == 2) x = __vadd2(x, a);
    if (OP == 3) { uint32_t r; asm volatile("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(a), "r"(0x5410u)); x = r; }
    if (OP == 4) x = __shfl_up_sync(0xffffffffu, x, 1) + (threadIdx.x == 0);
    if (OP == 5) {                 // col16 row chain on e
      const uint32_t h = __vimax3_s16x2(y, x, a);
      const uint32_t hb = __vadd2(h, b);
      x = __viaddmax_s16x2_relu(x, 0xfffefffeu, hb);
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
template <int OP>
void run(const char* name, uint32_t* d_out, long long* d_c) {
  long long c = 0;
  for (int r = 0; r < 2; r++) {
    k<OP><<<1, 32>>>(d_out, 3u, 5u, d_c);
    cudaMemcpy(&c, d_c, 8, cudaMemcpyDeviceToHost);
  }
  printf("%-34s %.2f cycles per dependent step\n", name, (double)c / N);
}
int main() {
  uint32_t* d_out; long long* d_c;
  cudaMalloc(&d_out, 4 * 32); cudaMalloc(&d_c, 8);
  run<0>("VIADDMNMX.S16x2.RELU", d_out, d_c);
  run<1>("VIMNMX3.S16x2", d_out, d_c);
  run<2>("VIADD.16x2", d_out, d_c);
  run<3>("PRMT", d_out, d_c);
  run<4>("SHFL.UP (+ IADD)", d_out, d_c);
  run<5>("col16 E chain (VIMNMX3+VIADD+VIADDMNMX)", d_out, d_c);
  return 0;
}
