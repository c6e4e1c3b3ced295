// sw_escalate.cuh -- a4 escalation plumbing: flag compaction and mini-group re-interleaving
// Part of the device code of libswsearch (see sw_common.cuh for the overview).
#pragma once
#include "sw_common.cuh"

namespace swk {

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

// Small flag arrays (n <= kCompactBlockMax): count, scan and scatter in ONE CTA
// instead of the three launches above.  Thread t owns the contiguous positions
// [t*S, t*S + S), S = ceil(n / 1024) <= 64, read with independent loads (one
// memory latency, not one per 1,024-flag chunk); one block scan of the per-thread
// counts orders the list.  Same ascending list, total and tail-group count.
constexpr int kCompactBlockMax = 65536;

__global__ void __launch_bounds__(kScanBlock) k_flag_compact_block(const uint8_t* __restrict__ flag, int n,
                                                                   int* __restrict__ list, int* __restrict__ total,
                                                                   int* __restrict__ tail_groups) {
  __shared__ int warp_sums[kScanBlock / 32];
  // programmatic dependent of the first pass (small databases): its flags are
  // complete and visible after the wait; the rerun kernel behind may launch
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int S = (n + kScanBlock - 1) / kScanBlock;
  const int p0 = t * S, p1 = min(n, p0 + S);
  unsigned long long bits = 0ull;                  // bit j: position p0 + j is flagged (S <= 64)
#pragma unroll 16
  for (int p = p0; p < p1; p++)
    if (flag[p]) bits |= 1ull << (p - p0);
  const int c = __popcll(bits);
  int incl = c;                                    // block exclusive scan of c
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_sums[w] = incl;
  __syncthreads();
  if (w == 0) {
    const int x = warp_sums[lane];
    int y = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) y += v;
    }
    warp_sums[lane] = y - x;
    if (lane == 31) {
      if (total) *total = y;
      if (tail_groups) *tail_groups = (y + kGroup - 1) / kGroup;
    }
  }
  __syncthreads();
  int o = warp_sums[w] + incl - c;
  while (bits) {
    const int j = __ffsll((long long)bits) - 1;
    list[o++] = p0 + j;
    bits &= bits - 1;
  }
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


}  // namespace swk
