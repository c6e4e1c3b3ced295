// sw_kernels.cuh — sm_100a device code of the Smith-Waterman database search.
//
// Every kernel computes (part of) Eq. 1 of PAPER.md:31-35 (§II.A):
//   H(i,j) = max{0, H(i-1,j-1) + fsbt(q_i, s_j), E(i,j), F(i,j)}
//   E(i,j) = max{E(i-1,j) - alpha, H(i-1,j) - beta}
//   F(i,j) = max{F(i,j-1) - alpha, H(i,j-1) - beta}
// with E and F clamped at 0 (exact: DESIGN.md §"Clamped gaps", SURVEY.md
// Appendix B1), in linear space.  i runs over the query
// (rows, held in registers per tile), j over the subject (columns, streamed).
//
// Inter-task model: one lane aligns one pair of
// length-sorted subjects, packed as the lo/hi halves of int16x2 registers and
// updated with Blackwell DPX instructions (VIADDMNMX/VIMNMX3 .S16x2).  The
// 16-bit pass flags any subject whose running max could have wrapped
// (DESIGN.md §"Saturation"); flagged subjects are re-aligned in int32.
// The production first pass, k_inter16_pipe (sw_pipe.cuh), runs the query
// tiles of a group on consecutive warps of a CTA and passes tile-edge rows
// through shared-memory rings instead of global memory.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "sw_common.cuh"
#include "sw_int16.cuh"
#include "sw_pipe.cuh"
#include "sw_int8.cuh"
#include "sw_int32.cuh"
#include "sw_multi.cuh"
#include "sw_escalate.cuh"
#include "sw_rank.cuh"
