// sw_rank.cuh -- a6: scatter to input order and exact top-k
// Part of the device code of libswsearch (see sw_common.cuh for the overview).
#pragma once
#include "sw_common.cuh"

namespace swk {

// ---------------------------------------------------------------------------
// (iv) finalize: scatter to input order and build unique 64-bit ranking keys
// (score << 32 | ~gid): "sort all alignment scores in descending order"
// (PAPER.md:55), ties by ascending global id (reading R7).
// ---------------------------------------------------------------------------
__global__ void k_finalize(const int* __restrict__ score_sorted, const int* __restrict__ perm, int n,
                           const long long* __restrict__ gid, int* __restrict__ scores_out,
                           unsigned long long* __restrict__ keys) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    const int idx = perm[p];
    const int s = score_sorted[p];
    if (scores_out) scores_out[idx] = s;
    const unsigned long long id = gid ? (unsigned long long)gid[idx] : (unsigned long long)idx;
    keys[p] = ((unsigned long long)(unsigned)s << 32) | (0xffffffffull - id);
  }
}

struct SelState {
  unsigned long long prefix, mask;
  long long kk;     // rank (1-based) still to find inside the current prefix
};

__global__ void k_sel_init(SelState* st, long long k) {
  if (threadIdx.x == 0) {
    st->prefix = 0ull;
    st->mask = 0ull;
    st->kk = k;
  }
}

// Radix select of the k-th largest key, 8 bits per pass (most significant first).
__global__ void k_sel_hist(const unsigned long long* __restrict__ keys, int n,
                           const SelState* __restrict__ st, int shift, unsigned* __restrict__ hist) {
  __shared__ unsigned sh[256];
  for (int t = threadIdx.x; t < 256; t += blockDim.x) sh[t] = 0;
  __syncthreads();
  const unsigned long long prefix = st->prefix, mask = st->mask;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    const unsigned long long key = keys[p];
    if ((key & mask) == prefix) atomicAdd(&sh[(key >> shift) & 255u], 1u);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 256; t += blockDim.x)
    if (sh[t]) atomicAdd(&hist[t], sh[t]);
}

__global__ void __launch_bounds__(256) k_sel_pick(SelState* st, int shift, unsigned* hist) {
  // digit d is chosen so that (# keys with digit > d) < kk <= (# keys with digit >= d);
  // suffix sums over the 256 bins by a block-wide scan (descending digit order)
  __shared__ long long suf[256];
  const int t = threadIdx.x;
  const int d = 255 - t;                       // thread t holds digit 255 - t
  long long v = hist[d];
  suf[t] = v;
  __syncthreads();
  for (int off = 1; off < 256; off <<= 1) {
    const long long add = t >= off ? suf[t - off] : 0;
    __syncthreads();
    suf[t] += add;
    __syncthreads();
  }
  const long long kk = st->kk;
  const long long incl = suf[t], excl = incl - v;   // keys with digit >= d, > d
  __syncthreads();
  if (excl < kk && kk <= incl) {
    st->kk = kk - excl;
    st->prefix |= (unsigned long long)d << shift;
    st->mask |= 255ull << shift;
  }
  hist[d] = 0;
}

// Keys >= the k-th largest: exactly cap = min(k, n) of them, because keys are
// unique (sw_db_create rejects repeated global ids); the bound check only
// keeps a violated invariant from writing past `out`.
__global__ void k_sel_compact(const unsigned long long* __restrict__ keys, int n,
                              const SelState* __restrict__ st, int take_all,
                              unsigned long long* __restrict__ out, int* __restrict__ count, int cap) {
  const unsigned long long thr = take_all ? 0ull : st->prefix;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    const unsigned long long key = keys[p];
    if (key >= thr) {
      const int slot = atomicAdd(count, 1);
      if (slot < cap) out[slot] = key;
    }
  }
}

// Single-CTA bitonic sort (descending) of cnt <= 4096 keys, then decode.
__global__ void __launch_bounds__(1024) k_topk_small(const unsigned long long* __restrict__ cand,
                                                     int cnt, int k, long long* __restrict__ out_ids,
                                                     int* __restrict__ out_scores) {
  __shared__ unsigned long long s[4096];
  int n2 = 1;
  while (n2 < cnt) n2 <<= 1;
  for (int t = threadIdx.x; t < n2; t += blockDim.x) s[t] = t < cnt ? cand[t] : 0ull;
  __syncthreads();
  for (int size = 2; size <= n2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < n2; t += blockDim.x) {
        const int u = t ^ stride;
        if (u > t) {
          const bool desc = (t & size) == 0;
          const unsigned long long a = s[t], b = s[u];
          if (desc ? (a < b) : (a > b)) { s[t] = b; s[u] = a; }
        }
      }
      __syncthreads();
    }
  }
  for (int t = threadIdx.x; t < k; t += blockDim.x) {
    if (t < cnt) {
      const unsigned long long key = s[t];
      if (out_ids) out_ids[t] = (long long)(0xffffffffull - (key & 0xffffffffull));
      if (out_scores) out_scores[t] = (int)(key >> 32);
    } else {
      if (out_ids) out_ids[t] = -1;
      if (out_scores) out_scores[t] = -1;
    }
  }
}

// Small databases (n <= 65,536, min(k, n) <= 4,096): the whole ranking in ONE
// CTA -- radix select of the k-th largest unique key (8 bits per pass, smem
// histogram), compaction of the k keys above it, bitonic sort, decode --
// instead of the 19-launch multi-CTA path.
// The keys are read eight times (one radix pass per byte); when they fit
// (n <= kTopkSmemKeys) they are staged in dynamic shared memory once, so the
// passes run at shared-memory latency instead of a chain of dependent global
// loads per thread (C1: 22 us per ranking before).
constexpr int kTopkSmemKeys = 12288;              // 96 KB of dynamic shared memory

// Small k (<= 32): k rounds of a block-wide argmax over the unique keys (the
// owner of each round's winner rescans its keys below it); a few us for C1's
// top-10 instead of eight radix passes (~17 us).
// Warp max of 64-bit keys with two REDUX.MAX (high words, then the low words of
// the lanes holding the highest high word) instead of a 10-SHFL butterfly.
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
  const unsigned hi = __reduce_max_sync(0xffffffffu, (unsigned)(v >> 32));
  const unsigned lo = __reduce_max_sync(0xffffffffu, (unsigned)(v >> 32) == hi ? (unsigned)v : 0u);
  return ((unsigned long long)hi << 32) | lo;
}

__device__ __forceinline__ void topk_rounds(const unsigned long long* __restrict__ keys, int n, int k,
                                            long long* __restrict__ out_ids, int* __restrict__ out_scores) {
  __shared__ unsigned long long wbest[32], sel;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5, nw = blockDim.x >> 5;
  unsigned long long best = 0ull;                   // keys are >= 1 (ids <= 2^32 - 2): 0 = none
  for (int p = t; p < n; p += blockDim.x) best = max(best, keys[p]);
  const int cnt = min(k, n);
  for (int r = 0; r < cnt; r++) {
    const unsigned long long v = warp_max_u64(best);
    if (lane == 0) wbest[w] = v;
    __syncthreads();
    if (w == 0) {
      const unsigned long long x = warp_max_u64(lane < nw ? wbest[lane] : 0ull);
      if (lane == 0) {
        sel = x;
        if (out_ids) out_ids[r] = (long long)(0xffffffffull - (x & 0xffffffffull));
        if (out_scores) out_scores[r] = (int)(x >> 32);
      }
    }
    __syncthreads();
    const unsigned long long s = sel;
    if (best == s) {                                // the one thread holding it (unique keys)
      best = 0ull;
      for (int p = t; p < n; p += blockDim.x) {
        const unsigned long long x = keys[p];
        if (x < s && x > best) best = x;
      }
    }
  }
  for (int r = cnt + t; r < k; r += blockDim.x) {
    if (out_ids) out_ids[r] = -1;
    if (out_scores) out_scores[r] = -1;
  }
}

// The whole ranking of n <= 65,536 keys (min(k, n) <= 4,096) by one CTA.
__device__ __forceinline__ void topk_block_impl(const unsigned long long* __restrict__ keys, int n, int k,
                                                long long* __restrict__ out_ids, int* __restrict__ out_scores) {
  if (k <= 32) {
    topk_rounds(keys, n, k, out_ids, out_scores);
    return;
  }
  __shared__ unsigned long long s[4096];
  __shared__ unsigned hist[256];
  __shared__ unsigned long long sh_prefix, sh_mask;
  __shared__ long long sh_kk;
  __shared__ int sh_cnt;
  const int cnt = min(k, n);
  unsigned long long thr = 0ull;
  if (k < n) {
    if (threadIdx.x == 0) { sh_prefix = 0ull; sh_mask = 0ull; sh_kk = k; }
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int t = threadIdx.x; t < 256; t += blockDim.x) hist[t] = 0u;
      __syncthreads();
      const unsigned long long prefix = sh_prefix, mask = sh_mask;
#pragma unroll 4
      for (int p = threadIdx.x; p < n; p += blockDim.x) {
        const unsigned long long key = keys[p];
        if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
      }
      __syncthreads();
      if (threadIdx.x < 32) {                                  // digit with (# > d) < kk <= (# >= d)
        // warp 0: lane l owns digits 255-8l .. 248-8l (descending); exclusive
        // scan of the lane sums gives the count above each lane's first digit
        const int lane = threadIdx.x;
        unsigned c[8];
        unsigned sum = 0;
#pragma unroll
        for (int j = 0; j < 8; j++) {
          c[j] = hist[255 - 8 * lane - j];
          sum += c[j];
        }
        unsigned incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        const long long kk = sh_kk;
        long long above = (long long)(incl - sum);
        if (above < kk && kk <= above + (long long)sum) {      // exactly one lane
#pragma unroll
          for (int j = 0; j < 8; j++) {
            if (above < kk && kk <= above + (long long)c[j]) {
              const int d = 255 - 8 * lane - j;
              sh_kk = kk - above;
              sh_prefix = prefix | ((unsigned long long)d << shift);
              sh_mask = mask | (255ull << shift);
            }
            above += c[j];
          }
        }
      }
      __syncthreads();
    }
    thr = sh_prefix;                                           // the k-th largest key (keys are unique)
  }
  if (threadIdx.x == 0) sh_cnt = 0;
  __syncthreads();
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    const unsigned long long key = keys[p];
    if (key >= thr) {
      const int slot = atomicAdd(&sh_cnt, 1);
      if (slot < cnt) s[slot] = key;   // exactly cnt pass (unique keys); bound kept for safety
    }
  }
  __syncthreads();
  int n2 = 1;
  while (n2 < cnt) n2 <<= 1;
  for (int t = cnt + threadIdx.x; t < n2; t += blockDim.x) s[t] = 0ull;
  __syncthreads();
  for (int size = 2; size <= n2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < n2; t += blockDim.x) {
        const int u = t ^ stride;
        if (u > t) {
          const bool desc = (t & size) == 0;
          const unsigned long long a = s[t], b = s[u];
          if (desc ? (a < b) : (a > b)) { s[t] = b; s[u] = a; }
        }
      }
      __syncthreads();
    }
  }
  for (int t = threadIdx.x; t < k; t += blockDim.x) {
    if (t < cnt) {
      const unsigned long long key = s[t];
      if (out_ids) out_ids[t] = (long long)(0xffffffffull - (key & 0xffffffffull));
      if (out_scores) out_scores[t] = (int)(key >> 32);
    } else {
      if (out_ids) out_ids[t] = -1;
      if (out_scores) out_scores[t] = -1;
    }
  }
}


__global__ void __launch_bounds__(1024) k_topk_block(const unsigned long long* __restrict__ gkeys, int n, int k,
                                                     long long* __restrict__ out_ids, int* __restrict__ out_scores) {
  extern __shared__ unsigned long long skeys[];
  const bool staged = n <= kTopkSmemKeys;
  if (staged) {
#pragma unroll 4
    for (int p = threadIdx.x; p < n; p += blockDim.x) skeys[p] = gkeys[p];
    __syncthreads();
  }
  topk_block_impl(staged ? skeys : gkeys, n, k, out_ids, out_scores);
}

// n <= kTopkSmemKeys: stage (iv) in ONE launch -- k_finalize's scatter and keys
// (into shared memory) followed by the one-CTA top-k (C1: two launches less
// per search than finalize + k_topk_block).
__global__ void __launch_bounds__(1024) k_rank_block(const int* __restrict__ score_sorted, const int* __restrict__ perm,
                                                     int n, const long long* __restrict__ gid,
                                                     int* __restrict__ scores_out, int k,
                                                     long long* __restrict__ out_ids, int* __restrict__ out_scores) {
  extern __shared__ unsigned long long skeys[];
  asm volatile("griddepcontrol.wait;" ::: "memory");   // programmatic dependent of the rerun (small databases)
  // n <= kTopkSmemKeys = 12 x 1024: a thread's loads go out six items at a
  // time before their first use (two rounds of two dependent memory latencies,
  // perm then gid; twelve at a time spill under the 64-register cap)
  constexpr int U = 6;
  for (int p0 = threadIdx.x; p0 < n; p0 += U * 1024) {
    int idx[U], sc[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int p = p0 + u * 1024;
      idx[u] = p < n ? perm[p] : 0;
      sc[u] = p < n ? score_sorted[p] : 0;
    }
    unsigned long long id[U];
#pragma unroll
    for (int u = 0; u < U; u++) id[u] = gid ? (unsigned long long)gid[idx[u]] : (unsigned long long)idx[u];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int p = p0 + u * 1024;
      if (p < n) {
        if (scores_out) scores_out[idx[u]] = sc[u];
        skeys[p] = ((unsigned long long)(unsigned)sc[u] << 32) | (0xffffffffull - id[u]);
      }
    }
  }
  __syncthreads();
  if (out_ids || out_scores) topk_block_impl(skeys, n, k, out_ids, out_scores);
}

__global__ void k_topk_decode(const unsigned long long* __restrict__ sorted, int cnt, int k,
                              long long* __restrict__ out_ids, int* __restrict__ out_scores) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < k; t += gridDim.x * blockDim.x) {
    if (t < cnt) {
      const unsigned long long key = sorted[t];
      if (out_ids) out_ids[t] = (long long)(0xffffffffull - (key & 0xffffffffull));
      if (out_scores) out_scores[t] = (int)(key >> 32);
    } else {
      if (out_ids) out_ids[t] = -1;
      if (out_scores) out_scores[t] = -1;
    }
  }
}


}  // namespace swk
