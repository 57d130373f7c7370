// T x on the 5th-generation tensor cores (included inside namespace flb by
// ops.cu): the op-level lmm (reference ops.py:219-235) for stream blocks of
// <= 28 columns and operand chunks of <= 32 columns.  The stream-block part
// F x_F is a tcgen05 MMA per 128-row tile (3xTF32: F is its own truncated hi
// part, F_lo staged by the epilogue, x_F split hi / lo once per CTA); the
// epilogue adds the gathered q_d = S_d x_d rows and writes each row's ncol
// results contiguously at its target row (perm).  Same bound as the row-
// wise kernels -- bytes: F in, T x out -- but the products no longer cost
// issue slots (k_lmm_warp_rows was issue-bound: 20 shuffles + 20 FMAs per row
// and column lane).
//
//   warp 0      producer: TMA of the F tile (128 x 32, 128B swizzle) + FKs
//   warp 1      MMA issuer (one thread): Q(t) = F x_F into TMEM buffer t & 1
//   warps 2-9   epilogue, thread = (tile row, 16-column half)
constexpr int L5_TILE = 128;
constexpr int L5_EPI = 256;
constexpr int L5_THREADS = 64 + L5_EPI;
constexpr int L5_NS = 4;

struct LmT5Args {
  int pf, c_x, col0, ncol;          // output columns [col0, col0 + ncol) of out (r_T x c_x)
  int64_t r_T, ntiles;
  int ng;
  const int32_t* fk[MAX_GATHER];
  const float* q[MAX_GATHER];       // r_d x ncol
  const float* x;                   // c_T x c_x operand
  const int32_t* f_tcol;
  const int32_t* perm;              // device row -> target row
  float* out;
  int dev_rows;                     // 1: out rows in device order
  int o_pitch, o_col0;              // out row pitch / first column
};

struct L5Geom {
  uint32_t stage, o_fk;             // stage: F (16 KB) | FKs (512 B per source)
  uint32_t o_lo;                    // 2 x F_lo (K-major SW128, 16 KB)
  uint32_t o_cst;                   // x_F hi | lo (interleave [8][32][4], 2 x 4 KB)
  uint32_t o_stg;                   // 2 x [128 rows x 33] fp32 output staging
  uint32_t total;
};

__host__ __device__ inline L5Geom l5_geom(int ng) {
  L5Geom g{};
  g.o_fk = 16384;
  g.stage = (uint32_t)round_up(16384 + 512 * (ng > 0 ? ng : 1), 1024);
  g.o_lo = L5_NS * g.stage;
  g.o_cst = g.o_lo + 2 * 16384;
  g.o_stg = g.o_cst + 8192;
  g.total = g.o_stg + 2 * L5_TILE * 33 * 4;
  return g;
}

__device__ __forceinline__ float l5_lo(float v) {
  return v - __uint_as_float(__float_as_uint(v) & 0xffffe000u);
}

__global__ void __launch_bounds__(L5_THREADS, 1)
    k_lmm_t5(const __grid_constant__ CUtensorMap tmF, LmT5Args a, L5Geom gm) {
  extern __shared__ __align__(1024) char smem_raw[];
  char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[L5_NS], empty[L5_NS], lo_ready[2], q_full[2];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int pf = a.pf, ng = a.ng;

  // B = x_F^T chunk: B[n][k] = x[f_tcol[k], col0 + n], hi (truncated) / lo
  float* cst = reinterpret_cast<float*>(sm + gm.o_cst);
  for (int i = tid; i < 8 * 32 * 4; i += blockDim.x) {
    const int ch = i >> 7, nn = (i >> 2) & 31, e = i & 3, k = ch * 4 + e;
    const int tc = k < pf ? a.f_tcol[k] : -1;
    const float v = (tc >= 0 && nn < a.ncol) ? a.x[(int64_t)tc * a.c_x + a.col0 + nn] : 0.f;
    cst[i] = v - l5_lo(v);
    cst[1024 + i] = l5_lo(v);
  }
  if (tid == 0) {
    for (int s = 0; s < L5_NS; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], L5_EPI);
    }
    for (int b = 0; b < 2; b++) {
      mbar_init(&lo_ready[b], L5_EPI);
      mbar_init(&q_full[b], 1);
    }
    fence_mbar_init();
  }
  tc::fence_smem_to_async();
  if (warp == 0) tc::alloc(&tbase, 64);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tbase;   // Q of tile parity b at column 32 b

  const int64_t G = gridDim.x;
  const int64_t base = a.ntiles / G, rem = a.ntiles % G;
  const int64_t t0 = blockIdx.x * base + min64(blockIdx.x, rem);
  const int n = (int)(base + (blockIdx.x < rem ? 1 : 0));

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
      for (int i = 0; i < n; i++) {
        const int s = i % L5_NS;
        if (i >= L5_NS) mbar_wait_sleep(&empty[s], (uint32_t)(((i / L5_NS) - 1) & 1));
        char* st = sm + s * gm.stage;
        mbar_arrive_expect_tx(&full[s], 16384u + 512u * ng);
        tma_load_2d_hint(st, &tmF, 0, (int)((t0 + i) * L5_TILE), &full[s], pol);
        for (int d = 0; d < ng; d++)
          bulk_g2s(st + gm.o_fk + 512 * d, a.fk[d] + (t0 + i) * L5_TILE, 512, &full[s]);
      }
    }
  } else if (warp == 1) {
    // the whole warp walks the tiles; one elected lane issues (tc05.cuh)
    const uint32_t idq = tc::idesc_tf32(128, 32, false, false);
    const uint32_t c0 = smem_u32(cst);
    const int kst = (pf + 7) / 8;
    for (int t = 0; t < n; t++) {
      const int b = t & 1;
      mbar_wait_sleep(&lo_ready[b], (uint32_t)((t >> 1) & 1));   // (implies the stage landed)
      tc::fence_after();
      const uint32_t st = smem_u32(sm + (t % L5_NS) * gm.stage);
      const uint32_t lo = smem_u32(sm + gm.o_lo + b * 16384);
      if (tc::elect_one()) {
        for (int ks = 0; ks < kst; ks++) {
          const uint64_t ah = tc::smem_desc(st + ks * 32, 16, 1024, tc::kSw128);
          const uint64_t al = tc::smem_desc(lo + ks * 32, 16, 1024, tc::kSw128);
          const uint64_t bh = tc::smem_desc(c0 + ks * 1024, 512, 128, tc::kInterleave);
          const uint64_t bl = tc::smem_desc(c0 + 4096 + ks * 1024, 512, 128, tc::kInterleave);
          tc::mma_tf32(tmem + 32 * b, ah, bh, idq, ks > 0);
          tc::mma_tf32(tmem + 32 * b, al, bh, idq, true);
          tc::mma_tf32(tmem + 32 * b, ah, bl, idq, true);
        }
        tc::commit(&q_full[b]);
      }
      __syncwarp();
    }
  } else {
    const int ew = warp - 2, h = ew >> 2, q4 = warp & 3;
    const int r = 32 * q4 + lane;
    const uint32_t lane_off = (uint32_t)(32 * q4) << 16;
    // F_lo of tile t into lo buffer t & 1 (this thread's four chunks)
    auto split = [&](int t) {
      const int s = t % L5_NS;
      mbar_wait_sleep(&full[s], (uint32_t)((t / L5_NS) & 1));
      const char* st = sm + s * gm.stage;
      char* lo_b = sm + gm.o_lo + (t & 1) * 16384;
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int c4 = 4 * h + u;
        const uint32_t o = (uint32_t)(r * 128 + ((c4 ^ (r & 7)) << 4));
        const float4 v = *reinterpret_cast<const float4*>(st + o);
        *reinterpret_cast<float4*>(lo_b + o) = make_float4(l5_lo(v.x), l5_lo(v.y), l5_lo(v.z), l5_lo(v.w));
      }
      fence_proxy_async();
      tc::fence_before();
      mbar_arrive(&lo_ready[t & 1]);
    };
    if (n > 0) split(0);
    for (int t = 0; t < n; t++) {
      const int s = t % L5_NS;
      const char* st = sm + s * gm.stage;
      const int64_t p = (t0 + t) * L5_TILE + r;
      const bool valid = p < a.r_T;
      // gathered q_d rows (issued before the TMEM wait)
      float acc[16];
#pragma unroll
      for (int j = 0; j < 16; j++) acc[j] = 0.f;
      const int c_lo = 16 * h;
      for (int d = 0; d < ng; d++) {
        const int f = reinterpret_cast<const int32_t*>(st + gm.o_fk)[d * L5_TILE + r];
        if (f >= 0) {
          const float* qr = a.q[d] + (int64_t)f * a.ncol + c_lo;
#pragma unroll
          for (int j = 0; j < 16; j++)
            if (c_lo + j < a.ncol) acc[j] += __ldg(qr + j);
        }
      }
      mbar_wait_sleep(&q_full[t & 1], (uint32_t)((t >> 1) & 1));
      tc::fence_after();
      uint32_t z[16];
      tc::ld16(tmem + lane_off + 32 * (t & 1) + 16 * h, z);
      tc::wait_ld();
      tc::fence_before();
      // the stage (F tile, FKs) is consumed: F_lo of the next tile, then release
      if (t + 1 < n) split(t + 1);
      mbar_arrive(&empty[s]);
      // F x_F + sum_d q_d into the staging tile (pitch 33: conflict-free),
      // then every warp writes 16 whole rows, lane = column: one coalesced
      // 128-byte store per target row instead of two scattered halves
      float* stg = reinterpret_cast<float*>(sm + gm.o_stg) + (t & 1) * (L5_TILE * 33);
#pragma unroll
      for (int j = 0; j < 16; j++) stg[r * 33 + c_lo + j] = __uint_as_float(z[j]) + acc[j];
      named_sync(1, L5_EPI);
      for (int rr = ew * 16; rr < ew * 16 + 16; rr++) {
        const int64_t pr = (t0 + t) * L5_TILE + rr;
        if (pr < a.r_T && lane < a.ncol)
          a.out[(a.dev_rows ? pr : (int64_t)a.perm[pr]) * a.o_pitch + a.o_col0 + lane] =
              stg[rr * 33 + lane];
      }
      (void)valid;
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::dealloc(tmem, 64);
}
