// 5th-generation tensor core (tcgen05) helpers for sm_100a: TMEM allocation,
// shared-memory matrix descriptors, the kind::tf32 instruction descriptor,
// MMA issue / commit and TMEM -> register loads.  Encodings follow the
// sm_100 UMMA descriptor formats (CUTLASS cute/arch/mma_sm100_desc.hpp).
//
// Canonical layouts used here (16-byte units, M = rows of the operand):
//   K-major, no swizzle ("interleave"): 8 x 16B core matrices, contiguous;
//       SBO = stride between 8-row groups, LBO = stride between 16B K chunks.
//   MN-major, no swizzle: core = 4 MN elements x 8 K rows (rows 16B apart);
//       SBO = stride between 4-element MN groups, LBO = stride between 8-row
//       K groups.
//   K-major SWIZZLE_128B: rows of 128B, 8-row atoms of 1024B (SBO), chunk
//       index XOR row%8; a K step of 8 tf32 advances the start by 32B.
//   MN-major SWIZZLE_128B_BASE32B (layout 1, the only MN-major form kind::tf32
//       takes): 32 MN elements per 128B row, K rows 128B apart, 32-byte
//       granule g of row r stored at g ^ (r % 4); LBO = stride between
//       32-element MN groups, SBO = stride between 4-row K groups (512 B for
//       contiguous rows); a K step of 8 advances the start by 1024 B.
//       Measured with fl_tc_probe (profiles/r02_tc_probe.txt), as is the
//       fact that kind::tf32 TRUNCATES fp32 operand bits below the tf32
//       mantissa (an fp32 tile is its own tf32 "hi" part).
#pragma once
#include <stdint.h>

namespace flb {
namespace tc {

enum Layout : uint64_t { kInterleave = 0, kSw128B32 = 1, kSw128 = 2, kSw64 = 4, kSw32 = 6 };

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                              Layout layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fffu);
  d |= (uint64_t)((lbo >> 4) & 0x3fffu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3fffu) << 32;
  d |= (uint64_t)1 << 46;                       // descriptor version (sm_100)
  d |= (uint64_t)layout << 61;
  return d;
}

// kind::tf32, fp32 accumulate; a_mn / b_mn = operand is MN-major
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) |
         ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, bool accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate ? 1u : 0u));
}

// arrive on an mbarrier when every previously issued MMA of this thread is done
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
               : "memory");
}

// one lane of a CONVERGED warp (elect.sync).  Issue tcgen05.mma / commit
// chains inside `if (elect_one())` of a converged warp, not inside
// `if (lane == 0)`: for a lane-0 branch the compiler cannot prove a single
// active thread and wraps every UTC* instruction in its own ELECT / BRA.U.ANY
// loop, which measured ~46 cycles per MMA (profiles/r02_tc_mma_timing.txt);
// under elect.sync the MMAs are emitted back to back.
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// whole-warp TMEM allocation; the base address is written to *dst (smem)
__device__ __forceinline__ void alloc(uint32_t* dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}

// 32 lanes x 16 consecutive 32-bit columns: thread t of the warp gets lane
// (warp%4)*32 + t, columns [col, col+16).  Follow with wait_ld().
__device__ __forceinline__ void ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15},"
      " [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// generic-proxy smem writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_smem_to_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

}  // namespace tc
}  // namespace flb
