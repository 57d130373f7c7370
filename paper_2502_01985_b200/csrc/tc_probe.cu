// Layout probe for MN-major tf32 tcgen05 operands (diagnostics, not a hot
// path).  kind::tf32 accepts MN-major shared-memory operands only in the
// "128B swizzle with 32-byte atoms" layout (descriptor layout 1), which TMA
// produces with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B.  The row-contracting
// products of the fused trainers (K-means one-hot^T [F|1], GNMF [W|F]^T W)
// read their row-major tiles as MN-major operands in that layout, so no
// transposed copy is needed.  This probe:
//   mode 0: TMA-loads a 32 x 32 fp32 tile with that swizzle and dumps the raw
//           shared-memory bytes (the physical layout the epilogues write);
//   mode 1: D[128 x N] = A B with A MN-major: A^T given row-major [K x 128],
//           TMA-loaded as 4 groups of 32 columns; B K-major interleave;
//   mode 2: D[128 x N] = A B with B MN-major: B given row-major [K x N],
//           TMA-loaded as N/32 groups; A K-major interleave.
// Descriptor LBO / SBO / layout are parameters so candidates can be checked.
#include <vector>

#include "internal.h"
#include "tc05.cuh"

namespace flb {

__global__ void __launch_bounds__(128) k_tc_probe(int mode, const __grid_constant__ CUtensorMap tm,
                                                  const float* __restrict__ A,
                                                  const float* __restrict__ B,
                                                  float* __restrict__ D, float* __restrict__ dump,
                                                  int K, int N, int lbo, int sbo, int layout) {
  extern __shared__ __align__(1024) char smem_raw[];
  char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar, mbar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  char* Ts = sm;                      // TMA-loaded operand (<= 4 groups x K x 128 B)
  float* Is = reinterpret_cast<float*>(sm + 65536);   // interleave operand
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_init(&mbar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int groups = mode == 0 ? 1 : mode == 1 ? 4 : N / 32;
  const int rows = mode == 0 ? 32 : K;
  if (tid == 0) {
    mbar_arrive_expect_tx(&bar, (uint32_t)(groups * rows * 128));
    for (int g = 0; g < groups; g++) tma_load_2d(Ts + g * rows * 128, &tm, 32 * g, 0, &bar);
  }
  // interleave operand: mode 1 -> B[K x N] (N rows of K), mode 2 -> A[128 x K]
  if (mode == 1)
    for (int i = tid; i < K * N; i += blockDim.x) {
      const int k = i / N, n = i - k * N;
      Is[(k / 4) * N * 4 + n * 4 + (k & 3)] = B[i];
    }
  if (mode == 2)
    for (int i = tid; i < 128 * K; i += blockDim.x) {
      const int m = i / K, k = i - m * K;
      Is[(k / 4) * 512 + m * 4 + (k & 3)] = A[i];
    }
  tc::fence_smem_to_async();
  mbar_wait(&bar, 0);
  if (mode == 0) {
    for (int i = tid; i < 32 * 32; i += blockDim.x) dump[i] = reinterpret_cast<float*>(Ts)[i];
    return;
  }
  __syncthreads();
  if (warp == 0) tc::alloc(&tbase, 256);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tbase;
  if (tid == 0) {
    const uint32_t t0 = smem_u32(Ts), i0 = smem_u32(Is);
    const uint32_t idesc = tc::idesc_tf32(128, N, mode == 1, mode == 2);
    for (int kk = 0; kk < K / 8; kk++) {
      uint64_t ad, bd;
      const uint64_t mn = tc::smem_desc(t0 + kk * 1024, (uint32_t)lbo, (uint32_t)sbo,
                                        (tc::Layout)layout);
      if (mode == 1) {
        ad = mn;
        bd = tc::smem_desc(i0 + kk * 2 * N * 16, N * 16, 128, tc::kInterleave);
      } else {
        ad = tc::smem_desc(i0 + kk * 2 * 2048, 2048, 128, tc::kInterleave);
        bd = mn;
      }
      tc::mma_tf32(tmem, ad, bd, idesc, kk > 0);
    }
    tc::commit(&mbar);
  }
  mbar_wait(&mbar, 0);
  tc::fence_after();
  for (int c = 0; c < N; c += 16) {
    uint32_t r[16];
    tc::ld16(tmem + ((uint32_t)(32 * warp) << 16) + c, r);
    tc::wait_ld();
    for (int j = 0; j < 16; j++) D[(32 * warp + lane) * N + c + j] = __uint_as_float(r[j]);
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::dealloc(tmem, 256);
}

// Issue-rate probe: one thread per CTA issues `reps` chains of 16 kind::tf32
// MMAs (M x N x 8, operands K-major SW128 or MN-major 128B/32-byte-atom,
// content zero) back to back, round-robin over `nacc` TMEM accumulators,
// and waits for the last; cycles / MMA from clock64 around the whole run.
__device__ __forceinline__ void probe_mma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                               uint32_t idesc, bool accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate ? 1u : 0u));
}

// kind 0: tf32 (K = 8 per MMA), 1: bf16 (K = 16).  Everything the issuing
// lane computes per MMA is a compile-time offset from two base descriptors
// (like the production kernels), so the loop measures the tensor core, not
// the issuing thread.
template <int KIND, bool AMN, bool BMN>
__global__ void __launch_bounds__(128) k_tc_timing(int M, int N, int reps, int nacc,
                                                   double* __restrict__ cyc) {
  extern __shared__ __align__(1024) char smem_raw[];
  char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 3 * 65536 / 16; i += blockDim.x)   // A: 64 KB, B: 128 KB
    reinterpret_cast<float4*>(sm)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (tid == 0) {
    mbar_init(&mbar, 1);
    fence_mbar_init();
  }
  tc::fence_smem_to_async();
  if (warp == 0) tc::alloc(&tbase, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tbase;
  if (warp == 0) {
    const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 65536);
    const uint32_t id = KIND ? ((1u << 4) | (1u << 7) | (1u << 10) | ((AMN ? 1u : 0u) << 15) |
                                ((BMN ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) |
                                ((uint32_t)(M >> 4) << 24))
                             : tc::idesc_tf32(M, N, AMN, BMN);
    // K steps advance by 1024 B (MN-major: 8 rows) or 32 B within a 4-step
    // K-major chunk; the chunk stride is left at zero (content is zero)
    const uint64_t da = AMN ? tc::smem_desc(a0, 16384, 512, tc::kSw128B32)
                            : tc::smem_desc(a0, 16, 1024, tc::kSw128);
    const uint64_t db = BMN ? tc::smem_desc(b0, 16384, 512, tc::kSw128B32)
                            : tc::smem_desc(b0, 16, 1024, tc::kSw128);
    const uint32_t sa = AMN ? 64 : 2, sb = BMN ? 64 : 2;
    __syncwarp();
    const long long c0 = clock64();
    if (tc::elect_one()) {
      for (int r = 0; r < reps; r++) {
#pragma unroll
        for (int kk = 0; kk < 16; kk++) {
          const uint32_t acc = tmem + (uint32_t)(N * (kk % nacc));
          const uint64_t a = da + (uint64_t)((AMN ? kk : (kk & 3)) * sa);
          const uint64_t b = db + (uint64_t)((BMN ? kk : (kk & 3)) * sb);
          if (KIND) probe_mma_bf16(acc, a, b, id, r > 0 || kk >= nacc);
          else tc::mma_tf32(acc, a, b, id, r > 0 || kk >= nacc);
        }
      }
      tc::commit(&mbar);
    }
    __syncwarp();
    mbar_wait(&mbar, 0);
    const long long c1 = clock64();
    if (tc::elect_one()) cyc[blockIdx.x] = (double)(c1 - c0) / (16.0 * reps);
    __syncwarp();
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::dealloc(tmem, 512);
}

}  // namespace flb

using namespace flb;

// cycles per kind::tf32 MMA (mean over `ctas` concurrent CTAs, one per SM)
extern "C" int fl_tc_timing(int32_t M, int32_t N, int32_t a_mn, int32_t b_mn, int32_t reps,
                            int32_t ctas, int32_t nacc, double* cycles) {
  const int kind = (nacc >> 8) & 1;   // nacc | 256: kind::f16 with bf16 operands
  nacc &= 255;
  if ((M != 64 && M != 128) || N < 8 || N > 256 || (N & 7) || reps < 1 || ctas < 1 ||
      ctas > 1024 || nacc < 1 || nacc > 16 || N * nacc > 512 || 16 % nacc) {
    set_error("fl_tc_timing: unsupported shape (M %d, N %d)", M, N);
    return FL_ERR_ARG;
  }
  double* d = nullptr;
  FL_CUDA(cudaMalloc(&d, (size_t)ctas * 8));
  const size_t smem = 1024 + 3 * 65536;
  auto go = [&](auto kern) -> int {
    FL_CUDA(raise_smem_limit(kern, (int)smem));
    kern<<<ctas, 128, smem>>>(M, N, reps, nacc, d);
    return FL_OK;
  };
  int rc;
  const int sel = kind * 4 + (a_mn ? 2 : 0) + (b_mn ? 1 : 0);
  switch (sel) {
    case 0: rc = go(k_tc_timing<0, false, false>); break;
    case 1: rc = go(k_tc_timing<0, false, true>); break;
    case 2: rc = go(k_tc_timing<0, true, false>); break;
    case 3: rc = go(k_tc_timing<0, true, true>); break;
    case 4: rc = go(k_tc_timing<1, false, false>); break;
    case 5: rc = go(k_tc_timing<1, false, true>); break;
    case 6: rc = go(k_tc_timing<1, true, false>); break;
    default: rc = go(k_tc_timing<1, true, true>); break;
  }
  if (rc) return rc;
  FL_CHECK_LAUNCH();
  FL_CUDA(cudaDeviceSynchronize());
  std::vector<double> h((size_t)ctas);
  FL_CUDA(cudaMemcpy(h.data(), d, (size_t)ctas * 8, cudaMemcpyDeviceToHost));
  cudaFree(d);
  double sum = 0.0;
  for (double v : h) sum += v;
  *cycles = sum / ctas;
  return FL_OK;
}

// params = {lbo, sbo, layout}; mode 0: A = the 32 x 32 tile, dump = 1024 floats
extern "C" int fl_tc_probe(int32_t mode, const float* A, const float* B, float* D, float* dump,
                           int32_t K, int32_t N, const int32_t* params) {
  if (mode < 0 || mode > 2 || (mode > 0 && (K < 8 || K > 64 || (K & 7) || N < 32 || N > 128 ||
                                            (N & 31)))) {
    set_error("fl_tc_probe: unsupported shape (mode %d, K %d, N %d)", mode, K, N);
    return FL_ERR_ARG;
  }
  float *dA = nullptr, *dB = nullptr, *dD = nullptr, *dT = nullptr;
  const size_t na = mode == 0 ? 32 * 32 : (size_t)128 * K, nb = mode == 0 ? 1 : (size_t)K * N;
  FL_CUDA(cudaMalloc(&dA, na * 4));
  FL_CUDA(cudaMalloc(&dB, nb * 4));
  FL_CUDA(cudaMalloc(&dD, (size_t)128 * 128 * 4));
  FL_CUDA(cudaMalloc(&dT, 32 * 32 * 4));
  FL_CUDA(cudaMemcpy(dA, A, na * 4, cudaMemcpyDefault));
  if (mode > 0) FL_CUDA(cudaMemcpy(dB, B, nb * 4, cudaMemcpyDefault));
  CUtensorMap tm;
  int rc;
  if (mode == 0) rc = make_tmap_2d(&tm, dA, 32, 32, 128, 32, 32, kSwz128Atom32);
  else if (mode == 1) {
    // A^T row-major [K x 128] is the host's A transposed: upload it that way
    float* at = nullptr;
    FL_CUDA(cudaMalloc(&at, na * 4));
    std::vector<float> h((size_t)128 * K);
    for (int m = 0; m < 128; m++)
      for (int k = 0; k < K; k++) h[(size_t)k * 128 + m] = A[(size_t)m * K + k];
    FL_CUDA(cudaMemcpy(at, h.data(), na * 4, cudaMemcpyHostToDevice));
    cudaFree(dA);
    dA = at;
    rc = make_tmap_2d(&tm, dA, (uint64_t)K, 128, 512, (uint32_t)K, 32, kSwz128Atom32);
  } else {
    rc = make_tmap_2d(&tm, dB, (uint64_t)K, (uint64_t)N, (uint64_t)N * 4, (uint32_t)K, 32,
                      kSwz128Atom32);
  }
  if (rc) return rc;
  const size_t smem = 1024 + 65536 + 65536;
  FL_CUDA(raise_smem_limit(k_tc_probe, (int)smem));
  k_tc_probe<<<1, 128, smem>>>(mode, tm, dA, dB, dD, dT, K, N, params ? params[0] : 16,
                               params ? params[1] : 1024, params ? params[2] : 1);
  FL_CHECK_LAUNCH();
  FL_CUDA(cudaDeviceSynchronize());
  if (mode == 0) FL_CUDA(cudaMemcpy(dump, dT, 32 * 32 * 4, cudaMemcpyDefault));
  else FL_CUDA(cudaMemcpy(D, dD, (size_t)128 * N * 4, cudaMemcpyDefault));
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  cudaFree(dT);
  return FL_OK;
}
