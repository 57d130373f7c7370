// Known-answer self test of the tcgen05 operand layouts the fused trainers
// use (tc05.cuh): one CTA computes D[128 x N] = A[128 x K] B[K x N] with
// kind::tf32 MMAs from shared memory, accumulator in TMEM, read back with
// tcgen05.ld.  Inputs that are exact in tf32 make the answer exact.
//
//   mode 0: A K-major interleave,      B K-major interleave
//   mode 1: A K-major interleave with a padded K-chunk stride and only 32
//           stored rows (D rows >= 32 read neighbouring data and are not
//           checked), B K-major interleave with a padded K-chunk stride --
//           the transposed tiles of the K-means / GNMF row contractions
//   mode 2: A K-major SWIZZLE_128B (K = 32), B K-major interleave
// (kind::tf32 accepts MN-major operands only in the 128B_BASE32B swizzle;
// the kernels use K-major operands throughout.)
#include "internal.h"
#include "tc05.cuh"

namespace flb {

__global__ void __launch_bounds__(128) k_tc_selftest(int mode, const float* __restrict__ A,
                                                     const float* __restrict__ B,
                                                     float* __restrict__ D, int K, int N,
                                                     int lbo_a, int sbo_a, int lbo_b, int sbo_b) {
  extern __shared__ __align__(1024) char smem_raw[];
  char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  float* As = reinterpret_cast<float*>(sm);
  float* Bs = As + 128 * 128;   // A region sized for K <= 128
  for (int i = tid; i < 128 * K; i += blockDim.x) {
    const int m = i / K, k = i - m * K;
    const float v = A[i];
    if (mode == 0) As[(k / 4) * 512 + m * 4 + (k & 3)] = v;
    else if (mode == 1) {
      if (m < 32) As[(k / 4) * 132 + (m / 8) * 32 + (m & 7) * 4 + (k & 3)] = v;   // LBO 528 B
    } else As[m * 32 + (((k >> 2) ^ (m & 7)) << 2) + (k & 3)] = v;
  }
  for (int i = tid; i < K * N; i += blockDim.x) {
    const int k = i / N, n = i - k * N;
    const float v = B[i];
    if (mode == 0 || mode == 2) Bs[(k / 4) * N * 4 + n * 4 + (k & 3)] = v;
    else Bs[(k / 4) * (N * 4 + 4) + (n / 8) * 32 + (n & 7) * 4 + (k & 3)] = v;   // LBO N*16+16
  }
  tc::fence_smem_to_async();
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 0) tc::alloc(&tbase, 256);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tbase;
  if (tid == 0) {
    const uint32_t a0 = smem_u32(As), b0 = smem_u32(Bs);
    const uint32_t idesc = tc::idesc_tf32(128, N, false, false);
    for (int kk = 0; kk < K / 8; kk++) {
      uint64_t ad, bd;
      if (mode == 0) {
        ad = tc::smem_desc(a0 + kk * 2 * 2048, 2048, 128, tc::kInterleave);
        bd = tc::smem_desc(b0 + kk * 2 * N * 16, N * 16, 128, tc::kInterleave);
      } else if (mode == 1) {
        const int la = lbo_a >= 0 ? lbo_a : 528, lb = lbo_b >= 0 ? lbo_b : N * 16 + 16;
        ad = tc::smem_desc(a0 + kk * 2 * la, la, sbo_a >= 0 ? sbo_a : 128, tc::kInterleave);
        bd = tc::smem_desc(b0 + kk * 2 * lb, lb, sbo_b >= 0 ? sbo_b : 128, tc::kInterleave);
      } else {
        ad = tc::smem_desc(a0 + kk * 32, 16, 1024, tc::kSw128);
        bd = tc::smem_desc(b0 + kk * 2 * N * 16, N * 16, 128, tc::kInterleave);
      }
      tc::mma_tf32(tmem, ad, bd, idesc, kk > 0);
    }
    tc::commit(&bar);
  }
  mbar_wait(&bar, 0);
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

}  // namespace flb

using namespace flb;

extern "C" int fl_tc_selftest(int32_t mode, const float* A, const float* B, float* D, int32_t K,
                              int32_t N, const int32_t* lbo_sbo) {
  if (mode < 0 || mode > 2 || K < 8 || K > 128 || (K & 7) || N < 16 || N > 256 || (N & 15) ||
      (mode == 2 && K != 32)) {
    set_error("fl_tc_selftest: unsupported shape (mode %d, K %d, N %d)", mode, K, N);
    return FL_ERR_ARG;
  }
  float *dA, *dB, *dD;
  FL_CUDA(cudaMalloc(&dA, 128 * K * 4));
  FL_CUDA(cudaMalloc(&dB, (size_t)K * N * 4));
  FL_CUDA(cudaMalloc(&dD, (size_t)128 * N * 4));
  FL_CUDA(cudaMemcpy(dA, A, 128 * K * 4, cudaMemcpyDefault));
  FL_CUDA(cudaMemcpy(dB, B, (size_t)K * N * 4, cudaMemcpyDefault));
  const size_t smem = 1024 + 128 * 128 * 4 + 128 * 256 * 4;
  FL_CUDA(raise_smem_limit(k_tc_selftest, (int)smem));
  int ov[4] = {-1, -1, -1, -1};
  if (lbo_sbo)
    for (int i = 0; i < 4; i++) ov[i] = lbo_sbo[i];
  k_tc_selftest<<<1, 128, smem>>>(mode, dA, dB, dD, K, N, ov[0], ov[1], ov[2], ov[3]);
  FL_CHECK_LAUNCH();
  FL_CUDA(cudaDeviceSynchronize());
  FL_CUDA(cudaMemcpy(D, dD, (size_t)128 * N * 4, cudaMemcpyDefault));
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  return FL_OK;
}
