// sw_pipe.cuh -- the int16x2 first pass with query tiles pipelined over the warps of a CTA (a3)
// Part of the device code of libswsearch (see sw_common.cuh for the overview).
//
// k_inter16 keeps a 48-row query tile in registers and sweeps it over a
// 64-subject group; the (E, H) row at every tile edge goes to a per-warp slab in
// global memory and is read back by the next tile -- 16 B per lane-column per
// edge, 1/6 B per cell, ~106x the algorithmic DRAM bytes.
// The paper names "tiled SW computation ... to significantly reduce the number
// of memory accesses to the intermediate buffers" as the lever (§V).
//
// k_inter16_pipe keeps 11 of every 12 tile edges on chip.  The work of a CTA is
// a sequence of ITEMS (group k, tile t), t = 0 .. T-1 per group it takes, in
// ROUNDS of W = 12: item s = 12 r + w runs on warp w.  Consecutive tiles of a
// group are therefore on consecutive warps; inside a round, tile t's bottom row
// reaches tile t+1 on the next warp through a shared-memory ring (link w ->
// w+1, chunks of C columns, mbarriers for full / empty slots), and the warps
// of a round run a chunk or two apart.  Only the edge that crosses a round --
// warp 11's item to warp 0's item of the next round, a whole item later -- goes
// through a per-CTA global slab (double-buffered by round parity, progress
// counters in shared memory), so the DRAM traffic of the tile edges drops 12x.
// The running max of each subject is forwarded with the last chunk and emitted
// by the group's last tile.  Groups come longest-first from the global counter,
// fetched by the warp running their tile 0 in CTA order (a ticket), so once a
// fetch finds the queue empty every later item is void: void items forward a
// void header, and a warp exits after its first void item.
//
// Arithmetic per cell is col16's (the instruction mix of k_inter16); only where
// the tile-edge rows live changes.  Deadlock freedom: a warp waits only on (a)
// its input (the previous item's data), (b) space in its output ring, freed by
// the next item on the next warp, (c) the fetch ticket or the slab buffer of
// earlier items; every wait is on a lower item index, and the chain of output
// waits ends at warp 11, whose output (the slab) never waits per chunk.
#pragma once
#include "sw_int16.cuh"

namespace swk {

constexpr int kPipeC = 8;                          // columns per ring chunk (mbarrier handshake granularity)
#ifndef SW_PIPE_SLEEP_NS
#define SW_PIPE_SLEEP_NS 64
#endif
#ifndef SW_PIPE_LEAD
#define SW_PIPE_LEAD 2                             // chunks the previous tile is ahead before a tile starts
#endif

struct PipeSlot {
  uint2 d[kPipeC * 32];                            // (E(i0+R, j), H(i0+R-1, j)) per column and lane
  uint32_t hm[32];                                 // running max of the tile's subjects (last chunk only)
  int hdr;                                         // group index of the item, -1 = void
  int pad[3];
};

// Dynamic shared memory after the profile: W x NS ring slots, their 2 x W x NS
// mbarriers, and the chain heads' slab staging rings (kStageCols x 256 B each).
__host__ __device__ constexpr size_t pipe_ring_bytes(int n_warps, int n_slots, int n_chains) {
  return (size_t)n_warps * n_slots * (sizeof(PipeSlot) + 2 * sizeof(unsigned long long)) +
         (size_t)n_chains * 8 * 256;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  const uint32_t a = smem_u32(b);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}

// Ring accesses: volatile asm (kept in program order with the mbarrier asm,
// which carries the "memory" clobber) but no clobber of their own, so the
// read-only profile loads of col16 still schedule freely around them.
__device__ __forceinline__ uint2 lds_u2(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_u2(uint32_t a, uint2 v) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(v.x), "r"(v.y));
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v));
}
__device__ __forceinline__ void mbar_arrive_a(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
// Wait for the phase of the given parity to complete: try_wait (which may park
// the warp for a short system-dependent time), then a short sleep between
// retries so a waiting warp does not spin on the issue slots of the others.
__device__ __forceinline__ bool mbar_test_a(uint32_t a, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(done)
      : "r"(a), "r"(parity)
      : "memory");
  return done != 0;
}
__device__ __forceinline__ void mbar_wait_a(uint32_t a, uint32_t parity) {
  while (!mbar_test_a(a, parity)) __nanosleep(SW_PIPE_SLEEP_NS);
}

// One direction of a ring link as seen by one warp: the link index and the
// chunk counter q (slot q % NS, phase (q / NS) & 1).  Addresses are rebuilt
// from the CTA-uniform ring base (a uniform register), so a link costs two
// registers in the register-bound tile loop.
template <int W, int NS>
struct PipeEnd {
  uint32_t base;                                   // 32-bit shared address of the ring (CTA-uniform)
  uint32_t link, q;
  static constexpr uint32_t kSlot = (uint32_t)sizeof(PipeSlot);
  static constexpr uint32_t kFull = (uint32_t)(W * NS) * kSlot;           // full barriers after the slots
  static constexpr uint32_t kEmpty = kFull + (uint32_t)(W * NS * 8);      // then the empty barriers
  __device__ __forceinline__ uint32_t idx() const { return link * NS + q % NS; }
  __device__ __forceinline__ uint32_t cur() const { return base + idx() * kSlot; }
  __device__ __forceinline__ uint32_t data(int c, int lane) const { return cur() + (uint32_t)(c * 32 + lane) * 8u; }
  __device__ __forceinline__ uint32_t hm(int lane) const {
    return cur() + (uint32_t)offsetof(PipeSlot, hm) + (uint32_t)lane * 4u;
  }
  __device__ __forceinline__ uint32_t hdr() const { return cur() + (uint32_t)offsetof(PipeSlot, hdr); }
  // consumer side
  __device__ __forceinline__ void wait_full() const { mbar_wait_a(base + kFull + idx() * 8u, (q / NS) & 1u); }
  // wait until chunk q + d (d < NS) is also full
  __device__ __forceinline__ void wait_full_ahead(uint32_t d) const {
    const uint32_t qq = q + d;
    mbar_wait_a(base + kFull + (link * NS + qq % NS) * 8u, (qq / NS) & 1u);
  }
  __device__ __forceinline__ void release() { mbar_arrive_a(base + kEmpty + idx() * 8u); q++; }
  // producer side
  __device__ __forceinline__ void wait_empty() const {
    mbar_wait_a(base + kEmpty + idx() * 8u, ((q / NS) & 1u) ^ 1u);
  }
  __device__ __forceinline__ void publish() { mbar_arrive_a(base + kFull + idx() * 8u); q++; }
};

// The round-crossing link (warp W-1 of round r -> warp 0 of round r+1): the
// column data go through a per-CTA global slab (two buffers, by round parity);
// its control lives in static shared memory (CTA-uniform addresses, no
// registers): the round whose item owns a buffer, its group (-1 = void), the
// columns written (ncols + 1 = item done, running max valid), the running max,
// and the last round whose item warp 0 has finished (buffer reuse).
constexpr int kMaxChains = 12;                    // chains per CTA (production: 4, one per SMSP)
__shared__ int sp_round[2 * kMaxChains], sp_hdr[2 * kMaxChains], sp_prog[2 * kMaxChains];
__shared__ int sp_w0_done[kMaxChains], sp_ticket[kMaxChains];
__shared__ uint32_t sp_hm[2 * kMaxChains * 32];
__shared__ int sp_split, sp_done;

#ifdef SW_PIPE_PROF
// Debug build only (tools/pipe_prof.py): cycles per warp position spent in
// [0] item-start waits, [1] chunk input waits, [2] chunk output waits,
// [3] everything (item loop), [4] items, [5] chunks.
__device__ unsigned long long g_pipe_prof[16][8];
#define PP_T0() long long _pp0 = clock64()
#define PP_ADD(slot) atomicAdd(&g_pipe_prof[threadIdx.x >> 5][slot], (unsigned long long)(clock64() - _pp0))
#define PP_CNT(slot) atomicAdd(&g_pipe_prof[threadIdx.x >> 5][slot], 1ull)
#else
#define PP_T0()
#define PP_ADD(slot)
#define PP_CNT(slot)
#endif

__device__ __forceinline__ int vld(const int& x) { return *(const volatile int*)&x; }

// Round-crossing slab input: cp.async (8 B per lane) into a per-chain staging
// ring of kStageCols columns in shared memory, issued kStageCols columns ahead
// of use, so the global (often L2- or DRAM-resident) slab's latency is off the
// chain head's critical path (the head paces the whole chain).
constexpr int kStageCols = 8;
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void vst(int& x, int v) { *(volatile int*)&x = v; }
__device__ __forceinline__ void spin_until_ge(const int& p, int v) {
  while (vld(p) < v) __nanosleep(32);
  __threadfence_block();
}

// One tile (rows [i0, i0+R)) of one group on this warp: the pipeline analogue
// of tile16.  in_mode / out_mode: 0 = none (first / last tile), 1 = shared-memory
// ring, 2 = the round-crossing slab (gin / gout: this lane's column 0).  The
// input row of column j+1 is loaded while column j is aligned.  Folds every H
// into hmax, including the running max handed down from the tiles above.
template <int R, int in_mode, int out_mode, class End>
__device__ __forceinline__ void tile16p(const uint2* __restrict__ gw, int ncols, const int8_t* __restrict__ prof,
                                        int stride, int i0, End& in, End& out, const uint2* gin, uint2* gout,
                                        int sb_in, int sb_out, uint32_t stage, int g, uint32_t na2, uint32_t nb2,
                                        uint32_t& hmax, int lane) {
  uint32_t D[R], F[R];
#pragma unroll
  for (int r = 0; r < R; r++) { D[r] = 0u; F[r] = 0u; }
  const uint2* lw = gw + lane;
  const int nwords = (ncols + kResPerWord - 1) / kResPerWord;
  const int8_t* pr = prof + i0;
  {  // virtual column j = -1 (all-zero boundary): primes D[r] = fsbt(q_{i0+r}, s_0)
    const uint2 w0 = res_word(lw, 0, nwords);
    uint32_t e0 = 0u;
    col16<R>(D, F, e0, 0u, pr + (w0.x & 31u) * stride, pr + (w0.y & 31u) * stride, na2, nb2, hmax);
  }
  // residue words: wA holds column j+1 (the D terms are formed one column
  // ahead), wN the word after it, loaded six columns before it is needed
  uint2 wA = res_word(lw, 0, nwords), wN = res_word(lw, kResPerWord, nwords);
  int nsh = 5;                                     // shift of column j+1 inside wA
  uint2 bn = make_uint2(0u, 0u);                   // input row of the next column
  // slab input (in_mode 2): column x is staged into slot x % kStageCols, one
  // cp.async group per column; progress is checked once per chunk
  if (in_mode == 2) {
    spin_until_ge(sp_prog[sb_in], min(kStageCols, ncols));
#pragma unroll 1
    for (int x = 0; x < kStageCols; x++) {
      if (x < ncols) cp_async8(stage + (uint32_t)x * 256u, gin + (long long)x * 32);
      cp_async_commit();
    }
    cp_async_wait<kStageCols - 1>();               // column 0 has landed
    bn = lds_u2(stage);
  }
  // chunks of kPipeC columns; at least one, since a ring chunk carries the header
  for (int j = 0;;) {
    const int jend = min(j + kPipeC, ncols);
    const bool last_chunk = j + kPipeC >= ncols;
    if (lane == 0) PP_CNT(5);
    {
    PP_T0();
    if (in_mode == 1) {
      in.wait_full();
      if (j < jend) bn = lds_u2(in.data(0, lane));
    } else if (in_mode == 2) {
      spin_until_ge(sp_prog[sb_in], min(jend + kStageCols, ncols));   // every column staged in this chunk
    }
    if (lane == 0) PP_ADD(1);
    }
    {
    PP_T0();
    if (out_mode == 1) out.wait_empty();
    if (lane == 0) PP_ADD(2);
    }
    const uint32_t src = in.data(0, lane) - (uint32_t)j * 256u, dst = out.data(0, lane) - (uint32_t)j * 256u;
    // one column: input row from bn (prefetched), next input row prefetched
    auto column = [&](int jj) {
      const uint2 b = bn;
      if (in_mode == 1) {
        if (jj + 1 < jend) bn = lds_u2(src + (uint32_t)(jj + 1) * 256u);
      } else if (in_mode == 2) {
        cp_async_wait<kStageCols - 2>();           // column jj+1 has landed
        bn = lds_u2(stage + (uint32_t)((jj + 1) % kStageCols) * 256u);
        if (jj + kStageCols < ncols)               // into column jj's slot, just consumed
          cp_async8(stage + (uint32_t)(jj % kStageCols) * 256u, gin + (long long)(jj + kStageCols) * 32);
        cp_async_commit();
      }
      uint32_t e = b.x;
      const uint32_t hl = col16<R>(D, F, e, b.y, pr + ((wA.x >> nsh) & 31u) * stride,
                                   pr + ((wA.y >> nsh) & 31u) * stride, na2, nb2, hmax);
      nsh += 5;
      if (nsh == 5 * kResPerWord) {                // column jj+2 starts the next word
        nsh = 0;
        wA = wN;
        wN = res_word(lw, jj + 2 + kResPerWord, nwords);
      }
      if (out_mode == 1) sts_u2(dst + (uint32_t)jj * 256u, make_uint2(e, hl));
      else if (out_mode == 2) gout[(long long)jj * 32] = make_uint2(e, hl);
    };
#pragma unroll 1
    for (; j < jend; j++) column(j);
    if (in_mode == 1) {
      if (last_chunk) hmax = __vmaxs2(hmax, lds_u32(in.hm(lane)));   // running max of the tiles above
      in.release();
    } else if (in_mode == 2 && last_chunk) {
      spin_until_ge(sp_prog[sb_in], ncols + 1);
      hmax = __vmaxs2(hmax, sp_hm[sb_in * 32 + lane]);
    }
    if (out_mode == 1) {
      if (last_chunk) sts_u32(out.hm(lane), hmax);
      if (lane == 0) sts_u32(out.hdr(), (uint32_t)g);
      out.publish();
    } else if (out_mode == 2) {
      if (last_chunk) sp_hm[sb_out * 32 + lane] = hmax;
      __threadfence_block();
      __syncwarp();
      if (lane == 0) vst(sp_prog[sb_out], last_chunk ? ncols + 1 : jend);
    }
    if (last_chunk) break;
  }
}

// The group's last tile (rem rows, no output): R dispatched at run time.
template <int T, int in_mode, int R = T - 8, class End>
__device__ __forceinline__ void tile16p_rem(int rem, const uint2* gw, int ncols, const int8_t* prof, int stride,
                                            int i0, End& in, End& out, const uint2* gin, int sb_in, uint32_t stage,
                                            int g, uint32_t na2, uint32_t nb2, uint32_t& hmax, int lane) {
  if constexpr (R >= 8) {
    if (rem == R)
      tile16p<R, in_mode, 0>(gw, ncols, prof, stride, i0, in, out, gin, nullptr, sb_in, 0, stage, g, na2, nb2, hmax,
                             lane);
    else
      tile16p_rem<T, in_mode, R - 8, End>(rem, gw, ncols, prof, stride, i0, in, out, gin, sb_in, stage, g, na2, nb2,
                                          hmax, lane);
  }
}

// One item: its tile with the input / output kinds of its position (compile-
// time, so the column loop carries only what it uses).
template <int T, int in_mode, class End>
__device__ __forceinline__ void item16p(int out_mode, bool rem_tile, int rem, const uint2* gw, int ncols,
                                        const int8_t* prof, int stride, int i0, End& in, End& out, const uint2* gin,
                                        uint2* gout, int sb_in, int sb_out, uint32_t stage, int g, uint32_t na2,
                                        uint32_t nb2, uint32_t& hmax, int lane) {
  if (rem_tile)
    tile16p_rem<T, in_mode>(rem, gw, ncols, prof, stride, i0, in, out, gin, sb_in, stage, g, na2, nb2, hmax, lane);
  else if (out_mode == 0)
    tile16p<T, in_mode, 0>(gw, ncols, prof, stride, i0, in, out, gin, gout, sb_in, sb_out, stage, g, na2, nb2, hmax,
                           lane);
  else if (out_mode == 1)
    tile16p<T, in_mode, 1>(gw, ncols, prof, stride, i0, in, out, gin, gout, sb_in, sb_out, stage, g, na2, nb2, hmax,
                           lane);
  else
    tile16p<T, in_mode, 2>(gw, ncols, prof, stride, i0, in, out, gin, gout, sb_in, sb_out, stage, g, na2, nb2, hmax,
                           lane);
}

// Persistent CTA (one per SM) of NT threads = NCH chains of CL warps.  Chain c
// is warps c, c + NCH, c + 2 NCH, ... (with NCH = 4 the three warps of a chain
// share one SM sub-partition, so a warp waiting on its neighbour hands its
// issue slots to the other two instead of idling the scheduler).  Each chain
// runs its own item sequence (rounds of CL items), fetch ticket and
// round-crossing slab.  Dynamic smem: the profile (SMEM), then the ring (W
// links x NS slots: link w = warp w -> warp w + NCH), then its mbarriers
// [full | empty].  slab: per CTA NCH x 2 x slab_cols x 32 uint2 (NCH chains).  Groups
// [0, split) in the longest-first queue `counter`, as k_inter16 (first-pass
// layout only).
template <int T, bool SMEM, int NT, int NS, int CL>
__global__ void __launch_bounds__(NT, 1)
k_inter16_pipe(const uint2* __restrict__ words, const GroupDesc* __restrict__ groups, int n_groups, int cut,
               const int8_t* __restrict__ gprof, int m_pad, int stride, int alpha, int beta, int limit,
               int prof_smem_bytes, uint2* __restrict__ slab, long long slab_cols, int* __restrict__ counter,
               int* __restrict__ score_sorted, uint8_t* __restrict__ flag) {
  constexpr int W = NT / 32;
  constexpr int NCH = W / CL;
  static_assert(NCH * CL == W && NCH <= kMaxChains, "chains");
  extern __shared__ __align__(16) int8_t dyn[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = w % NCH, pos = w / NCH;            // chain and position in it
  PipeSlot* ring = reinterpret_cast<PipeSlot*>(dyn + prof_smem_bytes);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(ring + W * NS);   // [full | empty]
  static_assert(PipeEnd<W, NS>::kFull == (uint32_t)(W * NS * sizeof(PipeSlot)), "ring layout");
  if (threadIdx.x == 0) {
    sp_split = split_groups(groups, n_groups, cut);
    sp_done = 0;
    for (int i = 0; i < kMaxChains; i++) {
      sp_ticket[i] = 0;
      sp_w0_done[i] = -1;
    }
    for (int i = 0; i < 2 * kMaxChains; i++) {
      sp_round[i] = -2;
      sp_prog[i] = 0;
    }
    for (int t = 0; t < 2 * W * NS; t++) mbar_init(&bars[t], 32);   // 32 lanes arrive per phase
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int n_items = sp_split;
  if (n_items <= 0) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    return;
  }
  if (SMEM) load_profile_smem(dyn, gprof, stride);   // ends with __syncthreads
  const int8_t* prof = prof_base<SMEM>(gprof);
  const uint32_t na2 = pack2(-alpha), nb2 = pack2(-beta);
  const int nfull = m_pad / T, rem = m_pad - nfull * T;
  const int n_tiles = nfull + (rem ? 1 : 0);
  using End = PipeEnd<W, NS>;
  End in{smem_u32(ring), (uint32_t)(pos > 0 ? w - NCH : 0), 0u};   // ring link (pos-1) -> pos
  End out{smem_u32(ring), (uint32_t)w, 0u};                         // ring link pos -> pos+1
  uint2* const chain_slab = slab + ((long long)blockIdx.x * NCH + c) * 2 * slab_cols * 32 + lane;
  // staging ring of this chain's head (after the ring's mbarriers): kStageCols x 32 uint2
  const uint32_t stage = smem_u32(bars + 2 * W * NS) + (uint32_t)(c * kStageCols * 256 + lane * 8);
#ifdef SW_PIPE_PROF
  const long long pp_start = clock64();
#endif
  for (int s = pos;; s += CL) {                    // this chain's item sequence
    const int r = s / CL;
    const int k = s / n_tiles;
    const int t = s - k * n_tiles;
    const bool last = t == n_tiles - 1;
    const int in_mode = t == 0 ? 0 : (pos > 0 ? 1 : 2);
    const int out_mode = last ? 0 : (pos < CL - 1 ? 1 : 2);
    const int sb_in = 2 * c + ((r + 1) & 1), sb_out = 2 * c + (r & 1);   // slab buffers of rounds r-1 / r
    int g = -1;
    {
    PP_T0();
    if (in_mode == 0) {
      // fetch in chain order: once a fetch finds the queue empty, every later one would
      if (lane == 0) {
        for (;;) {
          if (vld(sp_done)) break;
          if (vld(sp_ticket[c]) == k) {
            const int item = atomicAdd(counter, 1);
            g = item < n_items ? n_items - 1 - item : -1;
            if (g < 0) vst(sp_done, 1);
            __threadfence_block();
            vst(sp_ticket[c], k + 1);
            break;
          }
          __nanosleep(20);
        }
      }
      g = __shfl_sync(0xffffffffu, g, 0);
    } else if (in_mode == 1) {
      in.wait_full();
      g = (int)lds_u32(in.hdr());
      if (g < 0) in.release();                      // void: one header-only chunk
      else {
        // start SW_PIPE_LEAD chunks behind the previous tile (not right on its
        // heels): the slack absorbs jitter instead of a wait at every chunk
        const int nch = (groups[g].ncols + kPipeC - 1) / kPipeC;
        const int d = min(min(nch, SW_PIPE_LEAD), NS) - 1;
        if (d > 0) in.wait_full_ahead((uint32_t)d);
      }
    } else {
      while (vld(sp_round[sb_in]) != r - 1) __nanosleep(32);
      __threadfence_block();
      g = vld(sp_hdr[sb_in]);
    }
    if (out_mode == 2) {
      // the slab buffer of round r last held round r-2's item, which position
      // 0's item of round r-1 reads: wait until that item is done
      while (vld(sp_w0_done[c]) < r - 1) __nanosleep(32);
      __syncwarp();
      if (lane == 0) {
        vst(sp_prog[sb_out], 0);
        vst(sp_hdr[sb_out], g);
        __threadfence_block();
        vst(sp_round[sb_out], r);
      }
      __syncwarp();
    }
    if (lane == 0) { PP_ADD(0); PP_CNT(4); }
    }
    if (g < 0) {                                    // void: pass it on to the next tile's warp, then stop
      if (out_mode == 1) {
        out.wait_empty();
        if (lane == 0) sts_u32(out.hdr(), (uint32_t)-1);
        out.publish();
      }
      break;
    }
    const GroupDesc gd = groups[g];
    uint32_t hmax = 0u;
    const uint2* gin = chain_slab + (long long)(sb_in & 1) * slab_cols * 32;
    uint2* gout = chain_slab + (long long)(sb_out & 1) * slab_cols * 32;
    const bool rem_tile = last && rem;
    if (in_mode == 0)
      item16p<T, 0>(out_mode, rem_tile, rem, words + gd.base, gd.ncols, prof, stride, t * T, in, out, gin, gout,
                    sb_in, sb_out, stage, g, na2, nb2, hmax, lane);
    else if (in_mode == 1)
      item16p<T, 1>(out_mode, rem_tile, rem, words + gd.base, gd.ncols, prof, stride, t * T, in, out, gin, gout,
                    sb_in, sb_out, stage, g, na2, nb2, hmax, lane);
    else
      item16p<T, 2>(out_mode, rem_tile, rem, words + gd.base, gd.ncols, prof, stride, t * T, in, out, gin, gout,
                    sb_in, sb_out, stage, g, na2, nb2, hmax, lane);
    if (last) emit_pair(hmax, g, 2 * lane, gd.count, limit, nullptr, score_sorted, flag);
    if (pos == 0) {
      __syncwarp();
      __threadfence_block();
      if (lane == 0) vst(sp_w0_done[c], r);
    }
  }
  if (pos == 0 && lane == 0) vst(sp_w0_done[c], 0x7fffffff);   // never again a reader of the slab
#ifdef SW_PIPE_PROF
  if (lane == 0) atomicAdd(&g_pipe_prof[w][3], (unsigned long long)(clock64() - pp_start));
#endif
  // Launched as the programmatic dependent of k_intra16 (same stream): do not
  // retire before that grid has completed.  A no-op without a primary grid.
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

}  // namespace swk
