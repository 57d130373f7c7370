// F^T F on the 5th-generation tensor cores (included inside namespace flb by
// crossprod.cu): the stream-block Gram of the factorized crossprod for
// stream blocks of <= 28 columns.  Per 128-row tile ONE M = 128, N = 32 MMA
// chain over the tile's rows computes D = [F | F_lo]^T F with both operands
// read MN-major from row-major tiles (128B / 32-byte-atom swizzle,
// descriptor layout 1, tc05.cuh): the TMA tile is its own tf32 hi part (the
// tensor core truncates) and F_lo is written next to it by the split warps.
// 3xTF32 needs hi^T hi + lo^T hi + hi^T lo; the last term is the transpose
// of the second, so D's two 32-row halves give the Gram as
// G = D_hh + D_lh + D_lh^T at half the MMA work of an N = 64 chain.  TMEM
// accumulates two tiles (256 rows) in fp32, then dedicated fold warps move
// them into fp64 registers (a 512-row window left a 1e-6 relative deviation
// from the fp64 Gram at C2 size, 128 rows 2.5e-7); per-CTA partials are
// reduced in CTA order.  Bound: one read of F (HBM).
//
//   warp 0     producer (TMA of the F tile)
//   warp 1     MMA issuer (one thread)
//   warps 2-5  split: F_lo of each tile (thread = tile row)
//   warps 8-11 fold: the 64 used rows of D into fp64 registers
//   warps 6-7  idle
// m64 selects the M = 64 MMA shape (A = [F | F_lo] exactly, half the shared-
// memory operand reads of M = 128, whose groups 2, 3 are padding): D row i
// then sits in TMEM lane 32 (i / 16) + i % 16 (16 lanes per warp quadrant)
// instead of lane i.
constexpr int R5_TILE = 128;
constexpr int R5_NS = 6;
constexpr int R5_FT = 2;              // fp32 TMEM sums over 256 rows, then fp64
constexpr int R5_THREADS = 384;

struct R5Geom {
  uint32_t stage;   // F (16 KB) | F_lo (16 KB)
  uint32_t o_acc;   // fp64 [32 cols][64 lanes] (+ zero pad to 32 KB), right after the
                    // stages: the M = 128 A operand of the last stage reads it as its
                    // (unused) groups 2, 3
  uint32_t total;
};

__host__ __device__ inline R5Geom r5_geom() {
  R5Geom g{};
  g.stage = 32768;
  g.o_acc = R5_NS * g.stage;
  g.total = g.o_acc + 64 * 64 * 8;
  return g;
}

__device__ __forceinline__ uint32_t r5_b32(int row, int c4) {
  return (uint32_t)(row * 128 + (((c4 >> 1) ^ (row & 3)) << 5) + ((c4 & 1) << 4));
}
__device__ __forceinline__ float r5_lo(float v) {
  return v - __uint_as_float(__float_as_uint(v) & 0xffffe000u);
}

// part[cta][i * pf + j] = sum over the CTA's rows of F[r][i] F[r][j]
__global__ void __launch_bounds__(R5_THREADS, 1)
    k_fgram_t5(const __grid_constant__ CUtensorMap tmF, int pf, int64_t ntiles, R5Geom gm,
               double* __restrict__ part, int m64) {
  extern __shared__ __align__(1024) char smem_raw[];
  char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[R5_NS], empty[R5_NS], lo_ready[R5_NS], acc_full[2], acc_empty[2];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* acc = reinterpret_cast<double*>(sm + gm.o_acc);   // [col][lane] (final combine)
  // the M = 128 operand reads 32 KB past a stage into rows of D that are
  // never used (the last stage reads the combine area): keep it finite
  for (int i = tid; i < 64 * 64; i += blockDim.x) acc[i] = 0.0;
  // F_lo columns past pf are never written by the split: keep them zero
  for (int i = tid; i < R5_NS * 4096; i += blockDim.x)
    reinterpret_cast<float*>(sm + (i >> 12) * gm.stage + 16384)[i & 4095] = 0.f;
  if (tid == 0) {
    for (int s = 0; s < R5_NS; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&lo_ready[s], 128);
    }
    for (int b = 0; b < 2; b++) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], m64 ? 128 : 64);   // the fold warps
    }
    fence_mbar_init();
  }
  tc::fence_smem_to_async();
  if (warp == 0) tc::alloc(&tbase, 64);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tbase;
  const int64_t G = gridDim.x;
  const int64_t base = ntiles / G, rem = ntiles % G;
  const int64_t t0 = blockIdx.x * base + min64(blockIdx.x, rem);
  const int n = (int)(base + (blockIdx.x < rem ? 1 : 0));

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
      for (int i = 0; i < n; i++) {
        const int s = i % R5_NS;
        if (i >= R5_NS) mbar_wait_sleep(&empty[s], (uint32_t)(((i / R5_NS) - 1) & 1));
        mbar_arrive_expect_tx(&full[s], 16384u);
        tma_load_2d_hint(sm + s * gm.stage, &tmF, 0, (int)((t0 + i) * R5_TILE), &full[s], pol);
      }
    }
  } else if (warp == 1) {
    // the whole warp walks the tiles; one elected lane issues (tc05.cuh)
    const uint32_t id = tc::idesc_tf32(m64 ? 64 : 128, 32, true, true);
    for (int t = 0; t < n; t++) {
      const int s = t % R5_NS, w = t / R5_FT, b = w & 1;
      mbar_wait_sleep(&lo_ready[s], (uint32_t)((t / R5_NS) & 1));
      if ((t % R5_FT) == 0 && w >= 2) mbar_wait_sleep(&acc_empty[b], (uint32_t)(((w >> 1) - 1) & 1));
      tc::fence_after();
      const uint64_t d0 = tc::smem_desc(smem_u32(sm + s * gm.stage), 16384, 512, tc::kSw128B32);
      if (tc::elect_one()) {
#pragma unroll
        for (int kk = 0; kk < R5_TILE / 8; kk++) {
          const uint64_t d = d0 + (uint64_t)(kk * 64);
          tc::mma_tf32(tmem + 32 * b, d, d, id, !((t % R5_FT) == 0 && kk == 0));
        }
        tc::commit(&empty[s]);
        if ((t % R5_FT) == R5_FT - 1 || t == n - 1) tc::commit(&acc_full[b]);
      }
      __syncwarp();
    }
  } else if (warp >= 2 && warp < 6) {
    const int r = 32 * (warp & 3) + lane;
    const int sw = (r >> 2) & 1;   // rows r, r + 4 share a granule: swap chunk halves
    const int nc4 = (pf + 3) >> 2;
    for (int t = 0; t < n; t++) {
      const int s = t % R5_NS;
      char* st = sm + s * gm.stage;
      mbar_wait_sleep(&full[s], (uint32_t)((t / R5_NS) & 1));
#pragma unroll
      for (int c = 0; c < 8; c++) {
        if ((c ^ sw) >= nc4) continue;
        const uint32_t o = r5_b32(r, c ^ sw);
        const float4 v = *reinterpret_cast<const float4*>(st + o);
        *reinterpret_cast<float4*>(st + 16384 + o) =
            make_float4(r5_lo(v.x), r5_lo(v.y), r5_lo(v.z), r5_lo(v.w));
      }
      fence_proxy_async();
      tc::fence_before();
      mbar_arrive(&lo_ready[s]);
    }
  } else if (warp >= 8 && (m64 || warp < 10)) {
    const int q4 = warp & 3;
    // row of D held by this lane (-1: an unused TMEM lane)
    const int r = m64 ? (lane < 16 ? 16 * q4 + lane : -1) : 32 * q4 + lane;
    const uint32_t lane_off = (uint32_t)(32 * q4) << 16;
    double ra[32];
#pragma unroll
    for (int j = 0; j < 32; j++) ra[j] = 0.0;
    const int nw = n > 0 ? (n - 1) / R5_FT + 1 : 0;
    for (int w = 0; w < nw; w++) {
      const int b = w & 1;
      mbar_wait_sleep(&acc_full[b], (uint32_t)((w >> 1) & 1));
      tc::fence_after();
      uint32_t x0[16], x1[16];
      tc::ld16(tmem + lane_off + 32 * b, x0);
      tc::ld16(tmem + lane_off + 32 * b + 16, x1);
      tc::wait_ld();
      tc::fence_before();
      mbar_arrive(&acc_empty[b]);
#pragma unroll
      for (int j = 0; j < 16; j++) {
        ra[j] += (double)__uint_as_float(x0[j]);
        ra[16 + j] += (double)__uint_as_float(x1[j]);
      }
    }
    if (r >= 0) {
#pragma unroll
      for (int j = 0; j < 32; j++) acc[j * 64 + r] = ra[j];
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  // G[i][j] = D[i][j] + D[32 + i][j] + D[32 + j][i]  (hi hi + lo hi + (lo hi)^T)
  double* out = part + (int64_t)blockIdx.x * pf * pf;
  for (int e = tid; e < pf * pf; e += blockDim.x) {
    const int i = e / pf, j = e - i * pf;
    out[e] = acc[j * 64 + i] + acc[j * 64 + 32 + i] + acc[i * 64 + 32 + j];
  }
  __syncthreads();
  if (warp == 0) tc::dealloc(tmem, 64);
}

// out[tcol[i], tcol[j]] += sum over CTAs (CTA order) of part[.][i * pf + j]
__global__ void k_fgram_reduce(const double* __restrict__ part, int nb, int pf,
                               const int32_t* __restrict__ tcol, int c_T, double* __restrict__ out) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= (int64_t)pf * pf) return;
  const int e = (int)w, i = e / pf, j = e - i * pf;
  double s = 0.0;
  for (int b = lane; b < nb; b += 32) s += part[(int64_t)b * pf * pf + e];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const int ti = tcol[i], tj = tcol[j];
  if (lane == 0 && ti >= 0 && tj >= 0) out[(int64_t)ti * c_T + tj] += s;
}

// k_fgram_t5 with the F tile fetched as ONE 1-D bulk copy (128 rows x pf
// floats are contiguous in F) into a linear stage, and the MMA operands
// [F | F_lo] (MN-major, M = 64) written by the split warps into a small ring.
// A 2-D TMA box of 128 rows of 80 bytes moves the same bytes as 128 row
// requests; the bulk copy is one request (stream blocks with pf % 4 == 0).
constexpr int R5L_NS = 8;    // linear stages (128 x pf fp32 each)
constexpr int R5L_NO = 3;    // operand ring (F | F_lo, 32 KB)

struct R5LGeom {
  uint32_t lin;     // bytes per linear stage (1 KB aligned)
  uint32_t o_lin;   // linear stages after the operand ring
  uint32_t total;
};

__host__ __device__ inline R5LGeom r5l_geom(int pf) {
  R5LGeom g{};
  g.lin = (uint32_t)round_up(128 * pf * 4, 1024);
  g.o_lin = R5L_NO * 32768;
  g.total = g.o_lin + R5L_NS * g.lin;
  return g;
}

__global__ void __launch_bounds__(R5_THREADS, 1)
    k_fgram_t5l(const float* __restrict__ F, int pf, int64_t ntiles, R5LGeom gm,
                double* __restrict__ part) {
  extern __shared__ __align__(1024) char smem_raw[];
  char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t lin_full[R5L_NS], lin_empty[R5L_NS], op_ready[R5L_NO], op_free[R5L_NO];
  __shared__ uint64_t acc_full[2], acc_empty[2];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // operand chunks past pf are never written: zero the ring once
  for (int i = tid; i < R5L_NO * 8192; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (tid == 0) {
    for (int s = 0; s < R5L_NS; s++) {
      mbar_init(&lin_full[s], 1);
      mbar_init(&lin_empty[s], 128);   // the split threads
    }
    for (int l = 0; l < R5L_NO; l++) {
      mbar_init(&op_ready[l], 128);
      mbar_init(&op_free[l], 1);
    }
    for (int b = 0; b < 2; b++) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 128);   // the four fold warps
    }
    fence_mbar_init();
  }
  tc::fence_smem_to_async();
  if (warp == 0) tc::alloc(&tbase, 64);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tbase;
  const int64_t G = gridDim.x;
  const int64_t base = ntiles / G, rem = ntiles % G;
  const int64_t t0 = blockIdx.x * base + min64(blockIdx.x, rem);
  const int n = (int)(base + (blockIdx.x < rem ? 1 : 0));
  const uint32_t tile_bytes = 128u * pf * 4u;
  double ra[32];

  if (warp == 0) {
    const uint64_t pol = l2_policy_evict_first();
    for (int i = 0; i < n; i++) {
      const int s = i % R5L_NS;
      if (i >= R5L_NS) mbar_wait_sleep(&lin_empty[s], (uint32_t)(((i / R5L_NS) - 1) & 1));
      if (tc::elect_one()) {
        mbar_arrive_expect_tx(&lin_full[s], tile_bytes);
        bulk_g2s_hint(sm + gm.o_lin + s * gm.lin, F + (t0 + i) * 128 * pf, tile_bytes, &lin_full[s],
                      pol);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    const uint32_t id = tc::idesc_tf32(64, 32, true, true);
    for (int t = 0; t < n; t++) {
      const int l = t % R5L_NO, w = t / R5_FT, b = w & 1;
      mbar_wait_sleep(&op_ready[l], (uint32_t)((t / R5L_NO) & 1));
      if ((t % R5_FT) == 0 && w >= 2) mbar_wait_sleep(&acc_empty[b], (uint32_t)(((w >> 1) - 1) & 1));
      tc::fence_after();
      const uint64_t d0 = tc::smem_desc(smem_u32(sm + l * 32768), 16384, 512, tc::kSw128B32);
      if (tc::elect_one()) {
#pragma unroll
        for (int kk = 0; kk < R5_TILE / 8; kk++) {
          const uint64_t d = d0 + (uint64_t)(kk * 64);
          tc::mma_tf32(tmem + 32 * b, d, d, id, !((t % R5_FT) == 0 && kk == 0));
        }
        tc::commit(&op_free[l]);
        if ((t % R5_FT) == R5_FT - 1 || t == n - 1) tc::commit(&acc_full[b]);
      }
      __syncwarp();
    }
  } else if (warp >= 2 && warp < 6) {
    const int r = 32 * (warp & 3) + lane;
    const int nc4 = pf >> 2;
    for (int t = 0; t < n; t++) {
      const int s = t % R5L_NS, l = t % R5L_NO;
      const float4* src = reinterpret_cast<const float4*>(sm + gm.o_lin + s * gm.lin + r * pf * 4);
      char* op = sm + l * 32768;
      mbar_wait_sleep(&lin_full[s], (uint32_t)((t / R5L_NS) & 1));
      float4 v[7];
#pragma unroll
      for (int c = 0; c < 7; c++)
        if (c < nc4) v[c] = src[c];
      mbar_arrive(&lin_empty[s]);   // the linear stage is consumed
      if (t >= R5L_NO) mbar_wait_sleep(&op_free[l], (uint32_t)(((t / R5L_NO) - 1) & 1));
#pragma unroll
      for (int c = 0; c < 7; c++) {
        if (c < nc4) {
          const uint32_t o = r5_b32(r, c);
          *reinterpret_cast<float4*>(op + o) = v[c];
          *reinterpret_cast<float4*>(op + 16384 + o) =
              make_float4(r5_lo(v[c].x), r5_lo(v[c].y), r5_lo(v[c].z), r5_lo(v[c].w));
        }
      }
      fence_proxy_async();
      tc::fence_before();
      mbar_arrive(&op_ready[l]);
    }
  } else if (warp >= 8) {
    const uint32_t lane_off = (uint32_t)(32 * (warp & 3)) << 16;
#pragma unroll
    for (int j = 0; j < 32; j++) ra[j] = 0.0;
    const int nw = n > 0 ? (n - 1) / R5_FT + 1 : 0;
    for (int w = 0; w < nw; w++) {
      const int b = w & 1;
      mbar_wait_sleep(&acc_full[b], (uint32_t)((w >> 1) & 1));
      tc::fence_after();
      uint32_t x0[16], x1[16];
      tc::ld16(tmem + lane_off + 32 * b, x0);
      tc::ld16(tmem + lane_off + 32 * b + 16, x1);
      tc::wait_ld();
      tc::fence_before();
      mbar_arrive(&acc_empty[b]);
#pragma unroll
      for (int j = 0; j < 16; j++) {
        ra[j] += (double)__uint_as_float(x0[j]);
        ra[16 + j] += (double)__uint_as_float(x1[j]);
      }
    }
  }
  tc::fence_before();
  __syncthreads();   // everything is idle: the operand ring becomes the combine area
  tc::fence_after();
  double* acc = reinterpret_cast<double*>(sm);   // acc[col][row of D], fp64 32 x 64
  if (warp >= 8 && lane < 16) {
    const int r = 16 * (warp & 3) + lane;   // M = 64: D row i in lane 32 (i / 16) + i % 16
#pragma unroll
    for (int j = 0; j < 32; j++) acc[j * 64 + r] = ra[j];
  }
  __syncthreads();
  double* out = part + (int64_t)blockIdx.x * pf * pf;
  for (int e = tid; e < pf * pf; e += blockDim.x) {
    const int i = e / pf, j = e - i * pf;
    out[e] = acc[j * 64 + i] + acc[j * 64 + 32 + i] + acc[i * 64 + 32 + j];
  }
  __syncthreads();
  if (warp == 0) tc::dealloc(tmem, 64);
}
