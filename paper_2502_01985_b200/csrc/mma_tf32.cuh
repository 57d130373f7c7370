// Warp-level tf32 tensor-core helpers (mma.sync m16n8k8) with the 3xTF32
// split used for fp32-class accuracy: x = hi + lo with hi = tf32(x),
// lo = tf32(x - hi); a*b ~= hi_a*hi_b + lo_a*hi_b + hi_a*lo_b.
//
// Fragment ownership (PTX ISA, m16n8k8 .tf32), g = lane>>2, t = lane&3:
//   A 16x8 (row)  a0 (g, t)   a1 (g+8, t)   a2 (g, t+4)   a3 (g+8, t+4)
//   B 8x8  (col)  b0 (k=t, n=g)             b1 (k=t+4, n=g)
//   C 16x8        c0 (g, 2t)  c1 (g, 2t+1)  c2 (g+8, 2t)  c3 (g+8, 2t+1)
#pragma once
#include <stdint.h>

namespace flb {

__device__ __forceinline__ uint32_t tf32_bits(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

struct Split {
  uint32_t hi, lo;
};

__device__ __forceinline__ Split split_tf32(float x) {
  Split s;
  s.hi = tf32_bits(x);
  s.lo = tf32_bits(x - __uint_as_float(s.hi));
  return s;
}

// not volatile: a pure register op, so independent MMAs can be interleaved
__device__ __forceinline__ void mma_tf32(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

constexpr uint32_t kTf32One = 0x3f800000u;  // 1.0f is exact in tf32

}  // namespace flb
