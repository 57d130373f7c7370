// Stream-block part of a WIDE T^T y on the 5th-generation tensor cores
// (included inside namespace flb by ops.cu): F^T Y for stream blocks of
// <= 28 columns (pitch a multiple of 4) and 6..32 operand columns -- the
// op-level transpose_lmm (reference ops.py:237-253) and rmm = (T^T x^T)^T
// (ops.py:219-235 via the strided view), which before took one F pass per
// pair of operand columns.
//
// Y is first laid out as YD[r_pad x 32] fp32 in DEVICE row order (operand
// columns past c_y and the padding rows are zero; k_ydev32_*).  Per 128-row
// tile the F rows and the YD rows are each ONE contiguous block: a 1-D bulk
// copy apiece lands them in a linear stage (a 2-D TMA box of narrow rows is
// one request per row -- the crossprod Gram ran 1.6x faster on bulk
// copies), and the split warps write the MMA operands [F | F_lo | Y | Y_lo]
// (MN-major 128B / 32-byte-atom swizzle, descriptor layout 1, tc05.cuh) into
// a two-slot ring.  ONE M = 128, N = 64 MMA chain over the tile's rows then
// computes
//     D = [F | F_lo | Y | Y_lo]^T [Y | Y_lo]
//     F^T Y = D[F][Y] + D[F_lo][Y] + D[F][Y_lo]          (3xTF32)
// (rows 64..127 of D -- Y^T Y -- are a by-product of the M = 128 shape and
// unused).  TMEM accumulates two tiles (256 rows) in fp32; dedicated fold
// warps move them into fp64 registers; per-CTA partials are reduced in CTA
// order by k_reduce_partials.  Bytes: F (4 pf) + YD (128) per row, read once.
//
//   warp 0     producer (bulk copies of the F and Y blocks)
//   warp 1     MMA issuer (elected lane)
//   warps 2-5  split: thread = tile row, hi / lo operand rows
//   warps 8-9  fold: TMEM lanes 0..63 (the F / F_lo rows of D)
//   warps 6-7  idle
constexpr int M5_TILE = 128;
constexpr int M5_NS = 3;                     // linear stages (F block | Y block)
constexpr int M5_NO = 2;                     // operand ring slots
constexpr int M5_FT = 2;
constexpr int M5_THREADS = 320;
constexpr uint32_t M5_SLOT = 65536;          // F | F_lo | Y | Y_lo, 16 KB each
constexpr uint32_t M5_LIN = 14336 + 16384;   // F block (<= 128 x 28 fp32) | Y block
constexpr uint32_t M5_SMEM = M5_NO * M5_SLOT + M5_NS * M5_LIN + 1024;

__device__ __forceinline__ uint32_t m5_b32(int row, int c4) {
  return (uint32_t)(row * 128 + (((c4 >> 1) ^ (row & 3)) << 5) + ((c4 & 1) << 4));
}
__device__ __forceinline__ float m5_lo(float v) {
  return v - __uint_as_float(__float_as_uint(v) & 0xffffe000u);
}
__device__ __forceinline__ float4 m5_lo4(float4 v) {
  return make_float4(m5_lo(v.x), m5_lo(v.y), m5_lo(v.z), m5_lo(v.w));
}

// part[cta][i * cy + c] = sum over the CTA's rows of F[r][i] Y[r][c]
__global__ void __launch_bounds__(M5_THREADS, 1)
    k_tmm_t5(const float* __restrict__ F, const float* __restrict__ Y, int pf, int cy,
             int64_t ntiles, double* __restrict__ part, const float* __restrict__ Yg, int yp,
             const int32_t* __restrict__ perm, int64_t r_T) {
  extern __shared__ __align__(1024) char smem_raw[];
  char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t lin_full[M5_NS], lin_empty[M5_NS], op_ready[M5_NO], op_free[M5_NO];
  __shared__ uint64_t acc_full[2], acc_empty[2];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  char* lin0 = sm + M5_NO * M5_SLOT;
  // F operand chunks past pf are never written: zero the ring once
  for (int i = tid; i < M5_NO * (M5_SLOT / 16); i += blockDim.x)
    reinterpret_cast<float4*>(sm)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (tid == 0) {
    for (int s = 0; s < M5_NS; s++) {
      mbar_init(&lin_full[s], 1);
      mbar_init(&lin_empty[s], 128);   // the split threads
    }
    for (int l = 0; l < M5_NO; l++) {
      mbar_init(&op_ready[l], 128);
      mbar_init(&op_free[l], 1);
    }
    for (int b = 0; b < 2; b++) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 64);   // the two fold warps
    }
    fence_mbar_init();
  }
  tc::fence_smem_to_async();
  if (warp == 0) tc::alloc(&tbase, 128);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tbase;
  const int64_t G = gridDim.x;
  const int64_t base = ntiles / G, rem = ntiles % G;
  const int64_t t0 = blockIdx.x * base + min64(blockIdx.x, rem);
  const int n = (int)(base + (blockIdx.x < rem ? 1 : 0));
  const uint32_t fbytes = 128u * pf * 4u;
  double ra[64];   // fold warps: this lane's row of D, fp64

  if (warp == 0) {
    const uint64_t pol = l2_policy_evict_first();
    for (int i = 0; i < n; i++) {
      const int s = i % M5_NS;
      if (i >= M5_NS) mbar_wait_sleep(&lin_empty[s], (uint32_t)(((i / M5_NS) - 1) & 1));
      if (tc::elect_one()) {
        char* st = lin0 + s * M5_LIN;
        mbar_arrive_expect_tx(&lin_full[s], fbytes + (Yg ? 0u : 16384u));
        bulk_g2s_hint(st, F + (t0 + i) * M5_TILE * pf, fbytes, &lin_full[s], pol);
        if (!Yg) bulk_g2s_hint(st + 14336, Y + (t0 + i) * M5_TILE * 32, 16384u, &lin_full[s], pol);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // the whole warp walks the tiles; one elected lane issues (tc05.cuh)
    const uint32_t id = tc::idesc_tf32(128, 64, true, true);
    for (int t = 0; t < n; t++) {
      const int l = t % M5_NO, w = t / M5_FT, b = w & 1;
      mbar_wait_sleep(&op_ready[l], (uint32_t)((t / M5_NO) & 1));
      if ((t % M5_FT) == 0 && w >= 2) mbar_wait_sleep(&acc_empty[b], (uint32_t)(((w >> 1) - 1) & 1));
      tc::fence_after();
      const uint32_t op = smem_u32(sm + l * M5_SLOT);
      const uint64_t a0 = tc::smem_desc(op, 16384, 512, tc::kSw128B32);
      const uint64_t b0 = tc::smem_desc(op + 32768, 16384, 512, tc::kSw128B32);
      if (tc::elect_one()) {
#pragma unroll
        for (int kk = 0; kk < M5_TILE / 8; kk++)
          tc::mma_tf32(tmem + 64 * b, a0 + (uint64_t)(kk * 64), b0 + (uint64_t)(kk * 64), id,
                       !((t % M5_FT) == 0 && kk == 0));
        tc::commit(&op_free[l]);
        if ((t % M5_FT) == M5_FT - 1 || t == n - 1) tc::commit(&acc_full[b]);
      }
      __syncwarp();
    }
  } else if (warp >= 2 && warp < 6) {
    const int r = 32 * (warp & 3) + lane;
    const int nc4 = pf >> 2;
    const int ych = (cy + 3) >> 2;   // 16-byte chunks of a gathered y row
    // gather mode: this thread's own y row of tile t lands in the Y block of
    // linear stage t % M5_NS by async copies issued two tiles ahead (only
    // this thread reads it: no barrier, no proxy fence).  (A warp-
    // cooperative variant -- one copy instruction per 4 rows -- measured
    // 1.4-3x slower.)
    auto gather = [&](int t) {
      if (Yg && t < n) {
        char* yr = lin0 + (t % M5_NS) * M5_LIN + 14336 + r * 128;
        const int64_t p = (t0 + t) * M5_TILE + r;
        if (p < r_T) {
          const float* src = Yg + (perm ? (int64_t)perm[p] : p) * yp;
#pragma unroll
          for (int k = 0; k < 8; k++) {   // rotated chunk order: conflict-free phases
            const int c = (k + r) & 7;
            if (c < ych) cp_async16(yr + 16 * c, src + 4 * c);
            else *reinterpret_cast<float4*>(yr + 16 * c) = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        } else {
          for (int c = 0; c < 8; c++)
            *reinterpret_cast<float4*>(yr + 16 * c) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      cp_async_commit();
    };
    gather(0);
    gather(1);
    for (int t = 0; t < n; t++) {
      const int s = t % M5_NS, l = t % M5_NO;
      const char* st = lin0 + s * M5_LIN;
      char* op = sm + l * M5_SLOT;
      gather(t + 2);
      cp_async_wait_group<2>();   // tile t's row (groups t + 1, t + 2 may be in flight)
      mbar_wait_sleep(&lin_full[s], (uint32_t)((t / M5_NS) & 1));
      float4 f[7], y[8];
      const float4* fr = reinterpret_cast<const float4*>(st + r * pf * 4);
      const float4* yr = reinterpret_cast<const float4*>(st + 14336 + r * 128);
#pragma unroll
      for (int c = 0; c < 7; c++)
        if (c < nc4) f[c] = fr[c];
      // y[c] holds chunk (c + r) % 8 of the row: the rotation makes both the
      // linear reads and the swizzled writes of a store phase conflict-free
#pragma unroll
      for (int c = 0; c < 8; c++) y[c] = yr[(c + r) & 7];
      mbar_arrive(&lin_empty[s]);   // the linear stage is consumed
      if (t >= M5_NO) mbar_wait_sleep(&op_free[l], (uint32_t)(((t / M5_NO) - 1) & 1));
#pragma unroll
      for (int c = 0; c < 7; c++) {
        if (c < nc4) {
          const uint32_t o = m5_b32(r, c);
          *reinterpret_cast<float4*>(op + o) = f[c];
          *reinterpret_cast<float4*>(op + 16384 + o) = m5_lo4(f[c]);
        }
      }
#pragma unroll
      for (int c = 0; c < 8; c++) {
        const uint32_t o = m5_b32(r, (c + r) & 7);
        *reinterpret_cast<float4*>(op + 32768 + o) = y[c];
        *reinterpret_cast<float4*>(op + 49152 + o) = m5_lo4(y[c]);
      }
      fence_proxy_async();
      tc::fence_before();
      mbar_arrive(&op_ready[l]);
    }
  } else if (warp >= 8) {
    const int q4 = warp & 3;   // q4 = 0, 1: rows 0..63 of D
    const uint32_t lane_off = (uint32_t)(32 * q4) << 16;
#pragma unroll
    for (int j = 0; j < 64; j++) ra[j] = 0.0;
    const int nw = n > 0 ? (n - 1) / M5_FT + 1 : 0;
    for (int w = 0; w < nw; w++) {
      const int b = w & 1;
      mbar_wait_sleep(&acc_full[b], (uint32_t)((w >> 1) & 1));
      tc::fence_after();
#pragma unroll
      for (int u = 0; u < 4; u += 2) {
        uint32_t x0[16], x1[16];
        tc::ld16(tmem + lane_off + 64 * b + 16 * u, x0);
        tc::ld16(tmem + lane_off + 64 * b + 16 * u + 16, x1);
        tc::wait_ld();
#pragma unroll
        for (int j = 0; j < 16; j++) {
          ra[16 * u + j] += (double)__uint_as_float(x0[j]);
          ra[16 * u + 16 + j] += (double)__uint_as_float(x1[j]);
        }
      }
      tc::fence_before();
      mbar_arrive(&acc_empty[b]);
    }
  }
  tc::fence_before();
  __syncthreads();   // everything is idle: the operand ring becomes the combine area
  tc::fence_after();
  if (warp >= 8) {
    const int r = 32 * (warp & 3) + lane;
    double* acc = reinterpret_cast<double*>(sm);   // acc[col][row], fp64 64 x 64
#pragma unroll
    for (int j = 0; j < 64; j++) acc[j * 64 + r] = ra[j];
  }
  __syncthreads();
  // (F^T Y)[i][c] = D[i][c] + D[32 + i][c] + D[i][32 + c]
  const double* acc = reinterpret_cast<const double*>(sm);
  double* out = part + (int64_t)blockIdx.x * pf * cy;
  for (int e = tid; e < pf * cy; e += blockDim.x) {
    const int i = e / cy, c = e - i * cy;
    out[e] = acc[c * 64 + i] + acc[c * 64 + 32 + i] + acc[(32 + c) * 64 + i];
  }
  __syncthreads();
  if (warp == 0) tc::dealloc(tmem, 128);
}

// XT[t][c] = y(t, c) for a column-strided y view (rmm's x^T, element (t, c)
// at base[c * sc + t], sr == 1): 128 target rows x 32 columns per block
// step through shared memory, float4 reads along the columns of x and
// float4 row writes, sequential on both sides; columns past c_y are zero
__global__ void __launch_bounds__(256) k_xt32(YView yv, int cy, int64_t r_T,
                                              float* __restrict__ xt) {
  // software-pipelined: the next tile's column reads are issued before this
  // tile's row writes (twice the bytes in flight), and the tile alternates
  // between two shared buffers (one barrier per tile)
  __shared__ float tile[2][32][128 + 4];   // [buffer][column][row]
  const int tid = threadIdx.x;
  auto load = [&](int64_t t0, float4 (&v)[4]) {
    const bool full = t0 + 128 <= r_T && (((uintptr_t)(yv.base + t0) | (uintptr_t)yv.sc * 4) & 15) == 0;
#pragma unroll
    for (int k = 0; k < 4; k++) {   // 32 columns x 32 float4 = 1024 loads
      const int i = tid + 256 * k, c = i >> 5, q = i & 31;
      v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (c < cy) {
        if (full) {
          v[k] = __ldg(reinterpret_cast<const float4*>(yv.base + (int64_t)c * yv.sc + t0) + q);
        } else {
          const int64_t t = t0 + 4 * q;
          v[k].x = t < r_T ? yv.at(t, c) : 0.f;
          v[k].y = t + 1 < r_T ? yv.at(t + 1, c) : 0.f;
          v[k].z = t + 2 < r_T ? yv.at(t + 2, c) : 0.f;
          v[k].w = t + 3 < r_T ? yv.at(t + 3, c) : 0.f;
        }
      }
    }
  };
  const int64_t step = gridDim.x * 128LL;
  int64_t t0 = blockIdx.x * 128LL;
  if (t0 >= r_T) return;
  float4 v[4];
  load(t0, v);
  for (int b = 0; t0 < r_T; t0 += step, b ^= 1) {
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const int i = tid + 256 * k, c = i >> 5, q = i & 31;
      *reinterpret_cast<float4*>(&tile[b][c][4 * q]) = v[k];
    }
    __syncthreads();
    if (t0 + step < r_T) load(t0 + step, v);   // in flight during the writes below
#pragma unroll
    for (int k = 0; k < 4; k++) {   // 128 rows x 8 float4
      const int i = tid + 256 * k, row = i >> 3, c4 = i & 7;
      const int64_t t = t0 + row;
      if (t < r_T)
        reinterpret_cast<float4*>(xt + t * 32)[c4] =
            make_float4(tile[b][4 * c4][row], tile[b][4 * c4 + 1][row], tile[b][4 * c4 + 2][row],
                        tile[b][4 * c4 + 3][row]);
    }
  }
}

// bins[j][c] = sum over the members p of group j (ascending) of y's row at
// device row p -- y[(perm ? perm[p] : p) * yp + c] -- in fp64 (k_group_bins'
// order), warp per group, lane = column
__global__ void __launch_bounds__(256) k_group_bins32(const int64_t* __restrict__ grp_ptr,
                                                      const int32_t* __restrict__ grp_rows,
                                                      bool sorted, int64_t n_neg, int64_t rows,
                                                      const float* __restrict__ y, int yp,
                                                      const int32_t* __restrict__ perm, int cy,
                                                      double* __restrict__ bins) {
  const int lane = threadIdx.x & 31;
  const int ln = lane < cy ? lane : 0;
  for (int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; j < rows;
       j += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t m0 = grp_ptr[j], m1 = grp_ptr[j + 1];
    double s = 0.0;
    int64_t m = m0;
    for (; m + 8 <= m1; m += 8) {   // eight row loads in flight
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int64_t p = sorted ? n_neg + m + u : (int64_t)grp_rows[m + u];
        const int64_t row = perm ? (int64_t)perm[p] : p;
        v[u] = y[row * yp + ln];
      }
#pragma unroll
      for (int u = 0; u < 8; u++) s += (double)v[u];
    }
    for (; m < m1; m++) {
      const int64_t p = sorted ? n_neg + m : (int64_t)grp_rows[m];
      const int64_t row = perm ? (int64_t)perm[p] : p;
      s += (double)y[row * yp + ln];
    }
    if (lane < cy) bins[j * cy + lane] = s;
  }
}

// YD[p][c] = y(perm[p], c) for a row-major y view (warp per device row);
// perm == nullptr: y is in device order already
__global__ void __launch_bounds__(256) k_ydev32_rows(YView yv, int cy, int64_t r_T,
                                                     const int32_t* __restrict__ perm,
                                                     float* __restrict__ yd) {
  const int lane = threadIdx.x & 31;
  for (int64_t p = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; p < r_T;
       p += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t tr = perm ? (int64_t)perm[p] : p;
    yd[p * 32 + lane] = lane < cy ? yv.at(tr, lane) : 0.f;
  }
}

// part[cta][i * cy + c] = sum over the CTA's dimension rows r of
// S[r][i] * bins[r][c] (bins fp64, used as fp32 like k_tmm_partial) for
// <= 64 dimension columns and <= 32 operand columns: 64 rows staged with
// float4 / double2 loads, thread = 4 x 4 micro tile, fp32 over a staged
// tile, fp64 across tiles.  (k_tmm_partial's generic staging took 1.7 ms
// for C2's 1M x 50 dimension at 32 columns.)
__global__ void __launch_bounds__(128) k_sbins(const float* __restrict__ S, int pitch, int cols,
                                               const double* __restrict__ bins, int cy,
                                               int64_t rows, int64_t rows_per_cta,
                                               double* __restrict__ part) {
  __shared__ __align__(16) float Ss[64][64 + 4];
  __shared__ __align__(16) float Bs[64][32 + 4];
  const int tid = threadIdx.x;
  const int ma = (cols + 3) / 4, mb = (cy + 3) / 4;
  const bool active = tid < ma * mb;
  const int i0 = (tid / mb) * 4, k0 = (tid % mb) * 4;
  const int64_t r_begin = blockIdx.x * rows_per_cta;
  const int64_t r_end = min64(rows, r_begin + rows_per_cta);
  const bool vec = (pitch & 3) == 0;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int k = 0; k < 4; k++) acc[i][k] = 0.0;
  for (int64_t r0 = r_begin; r0 < r_end; r0 += 64) {
    const int nr = (int)min64(64, r_end - r0);
    __syncthreads();
    for (int e = tid; e < 64 * ma; e += 128) {
      const int r = e / ma, c4 = e - r * ma;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < nr) {
        const float* src = S + (r0 + r) * pitch;
        if (vec && 4 * c4 + 3 < pitch) v = __ldg(reinterpret_cast<const float4*>(src) + c4);
        else {
          v.x = 4 * c4 < cols ? src[4 * c4] : 0.f;
          v.y = 4 * c4 + 1 < cols ? src[4 * c4 + 1] : 0.f;
          v.z = 4 * c4 + 2 < cols ? src[4 * c4 + 2] : 0.f;
          v.w = 4 * c4 + 3 < cols ? src[4 * c4 + 3] : 0.f;
        }
        if (4 * c4 + 1 >= cols) v.y = 0.f;
        if (4 * c4 + 2 >= cols) v.z = 0.f;
        if (4 * c4 + 3 >= cols) v.w = 0.f;
      }
      *reinterpret_cast<float4*>(&Ss[r][4 * c4]) = v;
    }
    for (int e = tid; e < 64 * cy; e += 128) {
      const int r = e / cy, c = e - r * cy;
      Bs[r][c] = r < nr ? (float)bins[(r0 + r) * cy + c] : 0.f;
    }
    for (int e = tid; e < 64 * (4 * mb - cy); e += 128) {   // pad columns of the last quad
      const int w = 4 * mb - cy, r = e / w;
      Bs[r][cy + e - r * w] = 0.f;
    }
    __syncthreads();
    if (active) {
      float f[4][4];
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int k = 0; k < 4; k++) f[i][k] = 0.f;
      for (int r = 0; r < nr; r++) {
        const float4 a = *reinterpret_cast<const float4*>(&Ss[r][i0]);
        const float4 b = *reinterpret_cast<const float4*>(&Bs[r][k0]);
        const float av[4] = {a.x, a.y, a.z, a.w};
        const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
          for (int k = 0; k < 4; k++) f[i][k] = fmaf(av[i], bv[k], f[i][k]);
      }
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int k = 0; k < 4; k++) acc[i][k] += (double)f[i][k];
    }
  }
  if (active) {
    double* out = part + (int64_t)blockIdx.x * cols * cy;
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
      for (int k = 0; k < 4; k++)
        if (i0 + i < cols && k0 + k < cy) out[(i0 + i) * cy + k0 + k] = acc[i][k];
  }
}
