// B11 microbenchmark: sustained issue rate of the integer/DPX instructions the
// Smith-Waterman cell update uses (SURVEY.md §7 step 5, §8(d) roofline constant P).
// Each thread runs NCH independent dependency chains of one op for ITER iterations.
// Rate is reported as thread-instructions per SM clock per SM, from clock64()
// inside the kernel (clock-independent) and from CUDA events (wall).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITER 4096
#define NCH 8

__device__ __forceinline__ unsigned op_addmax(unsigned a, unsigned b, unsigned c) { return __viaddmax_s16x2(a, b, c); }
__device__ __forceinline__ unsigned op_addmax_relu(unsigned a, unsigned b, unsigned c) { return __viaddmax_s16x2_relu(a, b, c); }
__device__ __forceinline__ unsigned op_max3(unsigned a, unsigned b, unsigned c) { return __vimax3_s16x2_relu(a, b, c); }
__device__ __forceinline__ unsigned op_max2(unsigned a, unsigned b, unsigned c) { return __vmaxs2(a, b ^ c); }
__device__ __forceinline__ unsigned op_vadd2(unsigned a, unsigned b, unsigned c) { return __vadd2(a, b); }
__device__ __forceinline__ unsigned op_prmt(unsigned a, unsigned b, unsigned c) { return __byte_perm(a, b, 0x5410); }
__device__ __forceinline__ unsigned op_iadd3(unsigned a, unsigned b, unsigned c) { return a + b + c; }
__device__ __forceinline__ unsigned op_imad(unsigned a, unsigned b, unsigned c) { return a * b + c; }
__device__ __forceinline__ unsigned op_addmax32(unsigned a, unsigned b, unsigned c) { return (unsigned)__viaddmax_s32((int)a, (int)b, (int)c); }
__device__ __forceinline__ unsigned op_lop3(unsigned a, unsigned b, unsigned c) { return (a & b) ^ c; }
#include <cuda_fp16.h>
__device__ __forceinline__ unsigned op_hmax2(unsigned a, unsigned b, unsigned c) {
  __half2 x = *reinterpret_cast<__half2*>(&a), y = *reinterpret_cast<__half2*>(&b);
  __half2 r = __hmax2(x, y); return *reinterpret_cast<unsigned*>(&r); }
__device__ __forceinline__ unsigned op_hadd2(unsigned a, unsigned b, unsigned c) {
  __half2 x = *reinterpret_cast<__half2*>(&a), y = *reinterpret_cast<__half2*>(&b);
  __half2 r = __hadd2(x, y); return *reinterpret_cast<unsigned*>(&r); }
__device__ __forceinline__ unsigned op_imnmx(unsigned a, unsigned b, unsigned c) { return (unsigned)max((int)a, (int)b); }
__device__ __forceinline__ unsigned op_vimnmx2(unsigned a, unsigned b, unsigned c) { return __vmaxs2(a, b); }
__device__ __forceinline__ unsigned op_fmnmx(unsigned a, unsigned b, unsigned c) { return __float_as_uint(fmaxf(__uint_as_float(a), __uint_as_float(b))); }
__device__ __forceinline__ unsigned op_hmax2relu(unsigned a, unsigned b, unsigned c) {
  __half2 x = *reinterpret_cast<__half2*>(&a), y = *reinterpret_cast<__half2*>(&b); __half2 r = __hfma2_relu(x, y, x); return *reinterpret_cast<unsigned*>(&r); }

template <int OPA, int OPB>
__device__ __forceinline__ unsigned apply(int k, unsigned a, unsigned b, unsigned c) {
  int op = (k & 1) ? OPB : OPA;
  switch (op) {
    case 0: return op_addmax(a, b, c);
    case 1: return op_addmax_relu(a, b, c);
    case 2: return op_max3(a, b, c);
    case 3: return op_max2(a, b, c);
    case 4: return op_vadd2(a, b, c);
    case 5: return op_prmt(a, b, c);
    case 6: return op_iadd3(a, b, c);
    case 7: return op_imad(a, b, c);
    case 8: return op_addmax32(a, b, c);
    case 10: return op_hmax2(a, b, c);
    case 11: return op_hadd2(a, b, c);
    case 12: return op_imnmx(a, b, c);
    case 13: return op_vimnmx2(a, b, c);
    case 14: return op_fmnmx(a, b, c);
    case 15: return op_hmax2relu(a, b, c);
    default: return op_lop3(a, b, c);
  }
}

template <int OPA, int OPB>
__global__ void bench(unsigned* out, long long* cyc, unsigned seed) {
  unsigned x[NCH];
  unsigned b = seed * 0x9e3779b9u + threadIdx.x;
  unsigned c = seed ^ (threadIdx.x * 77u);
#pragma unroll
  for (int k = 0; k < NCH; k++) x[k] = threadIdx.x * 131u + k * 7u + seed;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITER; it++) {
#pragma unroll
    for (int k = 0; k < NCH; k++) x[k] = apply<OPA, OPB>(k, x[k], b, c);
    b += 0x00010001u;  // keep b live & varying (1 extra op per NCH ops)
  }
  __syncthreads();
  long long t1 = clock64();
  unsigned acc = 0;
#pragma unroll
  for (int k = 0; k < NCH; k++) acc ^= x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// LDS.128 rate: each thread reads 16 B from shared memory (conflict-free pattern).
__global__ void bench_lds(unsigned* out, long long* cyc, unsigned seed) {
  __shared__ uint4 sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_uint4(i, i * 3, i ^ seed, i + 7);
  __syncthreads();
  uint4 acc = make_uint4(0, 0, 0, 0);
  unsigned idx = threadIdx.x & 31;
  long long t0 = clock64();
  for (int it = 0; it < ITER; it++) {
#pragma unroll
    for (int k = 0; k < NCH; k++) {
      uint4 v = sm[(idx + k * 32 + (acc.x & 0)) & 2047];
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
    idx = (idx + 256) & 2047;
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x ^ acc.y ^ acc.z ^ acc.w;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OPA, int OPB>
void run(const char* name, int nsm, unsigned* d_out, long long* d_cyc, int threads, int bps, bool lds = false) {
  int grid = nsm * bps;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; rep++) {
    cudaEventRecord(e0);
    if (lds) bench_lds<<<grid, threads>>>(d_out, d_cyc, 3);
    else bench<OPA, OPB><<<grid, threads>>>(d_out, d_cyc, 3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
  }
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long* h = new long long[grid];
  cudaMemcpy(h, d_cyc, grid * sizeof(long long), cudaMemcpyDeviceToHost);
  double mean = 0; long long mx = 0;
  for (int i = 0; i < grid; i++) { mean += h[i]; if (h[i] > mx) mx = h[i]; }
  mean /= grid;
  double ops_per_block = (double)ITER * NCH * threads;  // the op under test (excludes the b+= helper)
  // per SM: bps blocks resident concurrently -> ops per SM per cycle
  double per_sm_clk = ops_per_block * bps / mean;
  double total_ops = ops_per_block * grid;
  double eff_clk_mhz = mean / (ms * 1e-3) / 1e6;
  printf("%-22s threads=%4d bps=%d  %.1f thr-ops/clk/SM (clock64 mean)   wall %.3f ms  %.2f Tops/s  eff_clk %.0f MHz\n",
         name, threads, bps, per_sm_clk, ms, total_ops / (ms * 1e-3) / 1e12, eff_clk_mhz);
  delete[] h;
  if (cudaGetLastError() != cudaSuccess) printf("CUDA error\n");
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("SMs=%d clockRate=%d kHz\n", nsm, clk);
  unsigned* d_out; long long* d_cyc;
  cudaMalloc(&d_out, sizeof(unsigned) * nsm * 8 * 1024);
  cudaMalloc(&d_cyc, sizeof(long long) * nsm * 8);
  int bps = 1;
  run<0, 0>("viaddmax_s16x2", nsm, d_out, d_cyc, 1024, bps);
  run<10, 10>("hmax2", nsm, d_out, d_cyc, 1024, bps);
  run<11, 11>("hadd2", nsm, d_out, d_cyc, 1024, bps);
  run<12, 12>("imnmx", nsm, d_out, d_cyc, 1024, bps);
  run<13, 13>("vimnmx.s16x2", nsm, d_out, d_cyc, 1024, bps);
  run<14, 14>("fmnmx", nsm, d_out, d_cyc, 1024, bps);
  run<15, 15>("hfma2.relu", nsm, d_out, d_cyc, 1024, bps);
  run<0, 10>("addmax16|hmax2", nsm, d_out, d_cyc, 1024, bps);
  run<0, 11>("addmax16|hadd2", nsm, d_out, d_cyc, 1024, bps);
  run<0, 12>("addmax16|imnmx", nsm, d_out, d_cyc, 1024, bps);
  run<0, 14>("addmax16|fmnmx", nsm, d_out, d_cyc, 1024, bps);
  run<0, 4>("addmax16|vadd2", nsm, d_out, d_cyc, 1024, bps);
  run<0, 7>("addmax16|imad", nsm, d_out, d_cyc, 1024, bps);
  run<4, 4>("vadd2", nsm, d_out, d_cyc, 1024, bps);
  run<4, 7>("vadd2|imad", nsm, d_out, d_cyc, 1024, bps);
  run<4, 11>("vadd2|hadd2", nsm, d_out, d_cyc, 1024, bps);
  return 0;
}
