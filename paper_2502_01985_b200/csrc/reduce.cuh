// Deterministic cross-CTA reduction of fp64 partials.
//
// Every output element red[dst] = sum_b base[b * stride] over nblk per-CTA
// partials is owned by ONE warp: lane l sums b = l, l + 32, ... in a fixed order and
// the warp combines the 32 lane sums with a fixed xor tree, so the result is
// bit-identical run to run (no atomics) while the partial loads of all
// elements proceed in parallel across the grid.
#pragma once
#include "internal.h"

namespace flb {

struct RedDesc {
  const double* base;   // &part[0][offset]
  int stride;           // doubles between consecutive CTA partials
  int nblk;             // number of partials
  int dst;              // index into the output
  int pad;
};

// sum of base[b * stride] over b < nblk by one warp, in a fixed order: lane
// l owns b = l (mod 32) and keeps eight independent chains (b mod 256), so
// eight loads per lane are in flight instead of one dependent chain; the 32
// lane sums meet in a fixed xor tree
__device__ __forceinline__ double warp_sum_strided(const double* __restrict__ base, int stride,
                                                   int nblk, int lane) {
  constexpr int CH = 8;
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; c++) acc[c] = 0.0;
  int b = lane;
  for (; b + 32 * (CH - 1) < nblk; b += 32 * CH) {
    double v[CH];
#pragma unroll
    for (int c = 0; c < CH; c++) v[c] = base[(int64_t)(b + 32 * c) * stride];
#pragma unroll
    for (int c = 0; c < CH; c++) acc[c] += v[c];
  }
#pragma unroll
  for (int c = 0; c < CH - 1; c++)
    if (b + 32 * c < nblk) acc[c] += base[(int64_t)(b + 32 * c) * stride];
  double s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// two elements at once (same fixed order per element as warp_sum_strided):
// twice the loads in flight for the serial last-CTA reductions
__device__ __forceinline__ void warp_sum_strided2(const double* __restrict__ b0, int st0, int n0,
                                                  const double* __restrict__ b1, int st1, int n1,
                                                  int lane, double* s0, double* s1) {
  constexpr int CH = 8;
  double a0[CH], a1[CH];
#pragma unroll
  for (int c = 0; c < CH; c++) a0[c] = a1[c] = 0.0;
  const int nmax = n0 > n1 ? n0 : n1;
  int b = lane;
  for (; b + 32 * (CH - 1) < nmax; b += 32 * CH) {
    double v0[CH], v1[CH];
#pragma unroll
    for (int c = 0; c < CH; c++) {
      const int bb = b + 32 * c;
      v0[c] = bb < n0 ? b0[(int64_t)bb * st0] : 0.0;
      v1[c] = bb < n1 ? b1[(int64_t)bb * st1] : 0.0;
    }
#pragma unroll
    for (int c = 0; c < CH; c++) {
      a0[c] += v0[c];
      a1[c] += v1[c];
    }
  }
#pragma unroll
  for (int c = 0; c < CH - 1; c++) {
    const int bb = b + 32 * c;
    if (bb < n0) a0[c] += b0[(int64_t)bb * st0];
    if (bb < n1) a1[c] += b1[(int64_t)bb * st1];
  }
  double r0 = ((a0[0] + a0[1]) + (a0[2] + a0[3])) + ((a0[4] + a0[5]) + (a0[6] + a0[7]));
  double r1 = ((a1[0] + a1[1]) + (a1[2] + a1[3])) + ((a1[4] + a1[5]) + (a1[6] + a1[7]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    r0 += __shfl_xor_sync(0xffffffffu, r0, o);
    r1 += __shfl_xor_sync(0xffffffffu, r1, o);
  }
  *s0 = r0;
  *s1 = r1;
}

__device__ __forceinline__ double warp_reduce_desc(const RedDesc& d, int lane) {
  return warp_sum_strided(d.base, d.stride, d.nblk, lane);
}

// all warps of the grid walk the descriptor list; returns after writing
__device__ __forceinline__ void reduce_descs(const RedDesc* __restrict__ descs, int n,
                                             double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t e = w0; e < n; e += nw) {
    const RedDesc d = descs[e];
    const double s = warp_reduce_desc(d, lane);
    if (lane == 0) out[d.dst] = s;
  }
}

// last-CTA-done helper: true in exactly one CTA, after every CTA's writes
__device__ __forceinline__ bool last_cta_done(int* counter) {
  __shared__ int is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int total = gridDim.x * gridDim.y * gridDim.z;
    is_last = atomicAdd(counter, 1) == total - 1;
  }
  __syncthreads();
  if (is_last) {
    __threadfence();
    if (threadIdx.x == 0) *counter = 0;
  }
  return is_last;
}

}  // namespace flb
