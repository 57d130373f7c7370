// F on the 5th-generation tensor cores: the GNMF fact-row pass with tcgen05
// MMAs from shared memory into TMEM (included inside namespace flb by
// gnmf.cu).  Same arithmetic as k_gnmf_fact (reference trainers.py:283-298:
// Q = T H^T, W <- W o Q / (W H H^T + eps), then P = W^T T and W^T W for the
// next H update), for rank tiles of R = 32 and streamed blocks of <= 32
// columns.
//
// One persistent CTA per SM walks a contiguous range of 128-row tiles.
//   warp 0     producer: TMA loads of the F and W tiles (2-D maps, 128B
//              swizzle = the canonical K-major SWIZZLE_128B operand layout)
//              and the tile's FKs into a 2-stage ring
//   warp 1     MMA issuer (one thread), every product 3xTF32:
//                Q(t)  = F H_F^T            M = 128 rows, N = 32, K = 8 QK
//                V(t)  = W HH               M = 128 rows, N = 32, K = 32
//                PG   += [W|W_lo|F|F_lo]^T [W|W_lo]   M = 128, N = 64,
//                         K = 128 rows (the row contraction: G = W^T W and
//                         P_F^T = F^T W fall out of the four hi/lo blocks)
//              Q/V double-buffered in TMEM; PG accumulates GT_FT tiles in
//              fp32, then the epilogue folds it into fp64 registers
//   warps 2-17 epilogue, thread = (tile row = TMEM lane, 8-column group): split F / W into
//              tf32 hi (in place) + exact lo, W' = W o (Q + sum_d G_d[fk]) /
//              (V + eps) into a staging tile (TMA store), the transposed PG
//              operands, Z_d[fk] += W' (segment sums, fp64 atomics), and the
//              periodic PG flush.
// Every operand is K-major (kind::tf32 takes MN-major operands only in the
// 128B_BASE32B swizzle): the TMA tiles directly, the constant H_F / HH in the
// K-major interleave layout, the PG operands in the padded interleave layout
// the K-means tcgen05 pass and fl_tc_selftest (mode 1) validate.

constexpr int GT_TILE = 128;
constexpr int GT_THREADS = 576;   // producer, MMA issuer, 16 epilogue warps
constexpr int GT_EPI = 512;       // epilogue threads
constexpr int GT_FT = 4;          // tiles per PG accumulation group (512 rows)
constexpr int GT_R = 32;
constexpr int GT_NG = 2;          // gathered sources the tcgen05 pass handles

struct GnTcArgs {
  int pf, c_T, SC, QK;            // SC = 8 QK >= pf: F columns in the MMAs
  int64_t r_T, ntiles;
  int ng, sort_g;
  const int32_t* fk[MAX_GATHER];
  const float* Gd[MAX_GATHER];
  double* Z[MAX_GATHER];
  const float* H32;               // R x c_T
  const float* HH32;              // R x R
  const int32_t* f_tcol;
  double* part;                   // gridDim.x x (R*SC + R*R), k_gnmf_fact's format
  double* scratch;                // gridDim.x x 128 x 32: folded PG rows
};

struct GtGeom {                   // byte offsets from the 1024-aligned base
  uint32_t stage, o_w, o_fk;      // stage size; W tile and FK offsets in a stage
  uint32_t o_lo, o_stg, o_apg, o_bpg, o_cst;
  uint32_t lbo_a, lbo_b;
  uint32_t total;
};

__host__ __device__ inline GtGeom gt_geom(int SC, int ng) {
  GtGeom g{};
  g.o_w = 16384;
  g.o_fk = 32768;
  g.stage = (uint32_t)round_up(32768 + 512 * (ng > 0 ? ng : 1), 1024);
  g.o_lo = 2 * g.stage;                         // F_lo | W_lo
  g.o_stg = g.o_lo + 32768;                     // W' staging (TMA store source)
  g.o_apg = g.o_stg + 16384;
  g.lbo_a = (uint32_t)((64 + 2 * SC) / 8 * 128 + 16);
  g.o_bpg = (uint32_t)round_up(g.o_apg + 32 * g.lbo_a + 256, 128);   // + M=128 over-read
  g.lbo_b = 8 * 128 + 16;
  g.o_cst = (uint32_t)round_up(g.o_bpg + 32 * g.lbo_b, 1024);         // Hh | Hl | HHh | HHl
  g.total = g.o_cst + 4 * 4096;
  return g;
}

__device__ __forceinline__ uint32_t sw128(int row, int col) {   // byte offset in a 128B-swizzled tile
  return (uint32_t)(row * 128 + ((((col >> 2) ^ (row & 7))) << 4) + (col & 3) * 4);
}
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

struct GtBars {
  uint64_t *full, *empty, *lo_ready, *qv_full, *qv_empty, *pg_ready, *pg_free, *acc_full,
      *acc_empty;
};

// the epilogue of column group h
template <bool UPDATE>
__device__ __forceinline__ void gt_epilogue(const CUtensorMap* tmW, const GnTcArgs& a,
                                            const GtGeom& gm, char* sm, uint32_t tmem,
                                            const GtBars& B, int n, int64_t t0, const int h) {
    // =================== epilogue: thread = (tile row, 8-column group) ===================
    // warp w reads TMEM lanes 32 (w % 4) ..; the 16 epilogue warps are 4
    // column groups x 4 lane quarters; group h owns W / Q / V columns
    // [8h, 8h + 8) and F chunks {2h, 2h + 1}
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int q4 = warp & 3;
    const int SC = a.SC, QK = a.QK;
    const int r = 32 * q4 + lane;
    const uint32_t lane_off = (uint32_t)(32 * q4) << 16;
    char* lo_b = sm + gm.o_lo;
    float* apg = reinterpret_cast<float*>(sm + gm.o_apg);
    float* bpg = reinterpret_cast<float*>(sm + gm.o_bpg);
    char* stg = sm + gm.o_stg;
    const int la = (int)(gm.lbo_a / 4), lb = (int)(gm.lbo_b / 4);
    const int FC = 2 * QK;                       // F chunks in the MMAs
    double acc64[8];
#pragma unroll
    for (int j = 0; j < 8; j++) acc64[j] = 0.0;

    // split this thread's chunks of tile i into tf32 hi (in place) + exact lo
    auto split = [&](int i) {
      char* st = sm + (i & 1) * gm.stage;
      mbar_wait(&B.full[i & 1], (uint32_t)((i >> 1) & 1));
#pragma unroll
      for (int u = 0; u < 2; u++) {
        const int c4 = 2 * h + u;
        const uint32_t o = sw128(r, c4 * 4);
        if (c4 < FC) {
          const float4 v = *reinterpret_cast<const float4*>(st + o);
          const float4 hv = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
          *reinterpret_cast<float4*>(st + o) = hv;
          *reinterpret_cast<float4*>(lo_b + o) =
              make_float4(v.x - hv.x, v.y - hv.y, v.z - hv.z, v.w - hv.w);
        }
        const float4 v = *reinterpret_cast<const float4*>(st + gm.o_w + o);
        const float4 hv = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
        *reinterpret_cast<float4*>(st + gm.o_w + o) = hv;
        *reinterpret_cast<float4*>(lo_b + 16384 + o) =
            make_float4(v.x - hv.x, v.y - hv.y, v.z - hv.z, v.w - hv.w);
      }
      tc::fence_smem_to_async();
      mbar_arrive(B.lo_ready);
    };
    if (UPDATE && n > 0) split(0);

    for (int t = 0; t < n; t++) {
      const int s = t & 1;
      char* st = sm + s * gm.stage;
      if (!UPDATE) mbar_wait(&B.full[s], (uint32_t)((t >> 1) & 1));
      const int32_t* fks = reinterpret_cast<const int32_t*>(st + gm.o_fk);
      int fkv[GT_NG];
#pragma unroll
      for (int d = 0; d < GT_NG; d++) fkv[d] = d < a.ng ? fks[d * GT_TILE + r] : -1;
      float w[8], f[8];
      if (UPDATE) {
        float q[8], v[8];
        // the G_d rows go out before the TMEM wait
        float4 gl[GT_NG][2];
#pragma unroll
        for (int d = 0; d < GT_NG; d++) {
          gl[d][0] = gl[d][1] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (d < a.ng && fkv[d] >= 0) {
            const float4* gr =
                reinterpret_cast<const float4*>(a.Gd[d] + (int64_t)fkv[d] * GT_R + 8 * h);
            gl[d][0] = __ldg(gr);
            gl[d][1] = __ldg(gr + 1);
          }
        }
        mbar_wait(&B.qv_full[s], (uint32_t)((t >> 1) & 1));
        tc::fence_after();
        {
          uint32_t rq[8], rv[8];
          tc::ld8(tmem + s * 64 + lane_off + 8 * h, rq);
          tc::ld8(tmem + s * 64 + lane_off + 32 + 8 * h, rv);
          tc::wait_ld();
#pragma unroll
          for (int j = 0; j < 8; j++) {
            q[j] = __uint_as_float(rq[j]);
            v[j] = __uint_as_float(rv[j]);
          }
        }
        tc::fence_before();
        mbar_arrive(&B.qv_empty[s]);
        // q += G_d[fk] in source order (as k_gnmf_fact)
#pragma unroll
        for (int d = 0; d < GT_NG; d++) {
          if (d < a.ng && fkv[d] >= 0) {
            q[0] += gl[d][0].x; q[1] += gl[d][0].y; q[2] += gl[d][0].z; q[3] += gl[d][0].w;
            q[4] += gl[d][1].x; q[5] += gl[d][1].y; q[6] += gl[d][1].z; q[7] += gl[d][1].w;
          }
        }
        // exact values: hi (in place) + lo
#pragma unroll
        for (int u = 0; u < 2; u++) {
          const int c4 = 2 * h + u;
          const uint32_t o = sw128(r, c4 * 4);
          const float4 wh = *reinterpret_cast<const float4*>(st + gm.o_w + o);
          const float4 wl = *reinterpret_cast<const float4*>(lo_b + 16384 + o);
          w[u * 4 + 0] = wh.x + wl.x;
          w[u * 4 + 1] = wh.y + wl.y;
          w[u * 4 + 2] = wh.z + wl.z;
          w[u * 4 + 3] = wh.w + wl.w;
          float4 fh = make_float4(0.f, 0.f, 0.f, 0.f), fl = fh;
          if (c4 < FC) {
            fh = *reinterpret_cast<const float4*>(st + o);
            fl = *reinterpret_cast<const float4*>(lo_b + o);
          }
          f[u * 4 + 0] = fh.x + fl.x;
          f[u * 4 + 1] = fh.y + fl.y;
          f[u * 4 + 2] = fh.z + fl.z;
          f[u * 4 + 3] = fh.w + fl.w;
        }
        mbar_arrive(&B.empty[s]);          // this thread's part of the stage is consumed
        if (t + 1 < n) split(t + 1);     // overwrites the lo buffer
        // W <- W o q / (W HH + eps)   (k_gnmf_fact's expression)
#pragma unroll
        for (int j = 0; j < 8; j++) w[j] = w[j] * __fdividef(q[j], v[j] + 1e-12f);
        // staging tile for the TMA store of W'
        if (tid == 64) bulk_wait_read<0>();
        named_sync(1, GT_EPI);
        *reinterpret_cast<float4*>(stg + sw128(r, 8 * h)) = make_float4(w[0], w[1], w[2], w[3]);
        *reinterpret_cast<float4*>(stg + sw128(r, 8 * h + 4)) = make_float4(w[4], w[5], w[6], w[7]);
        fence_proxy_async();
        named_sync(1, GT_EPI);
        if (tid == 64) {
          tma_store_2d(tmW, 0, (int)((t0 + t) * GT_TILE), stg);
          bulk_commit();
        }
      } else {
#pragma unroll
        for (int u = 0; u < 2; u++) {
          const int c4 = 2 * h + u;
          const uint32_t o = sw128(r, c4 * 4);
          const float4 wh = *reinterpret_cast<const float4*>(st + gm.o_w + o);
          w[u * 4 + 0] = wh.x;
          w[u * 4 + 1] = wh.y;
          w[u * 4 + 2] = wh.z;
          w[u * 4 + 3] = wh.w;
          float4 fh = make_float4(0.f, 0.f, 0.f, 0.f);
          if (c4 < FC) fh = *reinterpret_cast<const float4*>(st + o);
          f[u * 4 + 0] = fh.x;
          f[u * 4 + 1] = fh.y;
          f[u * 4 + 2] = fh.z;
          f[u * 4 + 3] = fh.w;
        }
        mbar_arrive(&B.empty[s]);
      }
      // ---- PG operands of this tile (transposed, padded interleave): A rows
      // [W hi | W lo | F hi | F lo], B columns [W hi | W lo]
      if (t >= 1) mbar_wait(B.pg_free, (uint32_t)((t - 1) & 1));
      const int ra = (r >> 2) * la + (r & 3), rb = (r >> 2) * lb + (r & 3);
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int j = 8 * h + u;
        const float hi = tf32_hi(w[u]), lo = w[u] - hi;
        apg[ra + (j >> 3) * 32 + (j & 7) * 4] = hi;
        apg[ra + ((32 + j) >> 3) * 32 + (j & 7) * 4] = lo;
        bpg[rb + (j >> 3) * 32 + (j & 7) * 4] = hi;
        bpg[rb + ((32 + j) >> 3) * 32 + (j & 7) * 4] = lo;
        if (j < SC) {
          const float fh = tf32_hi(f[u]), fl = f[u] - fh;
          apg[ra + ((64 + j) >> 3) * 32 + ((64 + j) & 7) * 4] = fh;
          apg[ra + ((64 + SC + j) >> 3) * 32 + ((64 + SC + j) & 7) * 4] = fl;
        }
      }
      fence_proxy_async();
      // ---- Z_d[fk] += W': warp (quarter q4, group h) takes rows 8h .. 8h+7
      // of its quarter, lane = rank column; one fp64 atomic per run of equal
      // FK (run ends found with a ballot).  The B columns are read before
      // pg_ready, so no warp can overwrite them for the next tile meanwhile.
      float v8[8];
      if (a.ng > 0) {
        named_sync(2, GT_EPI);   // a quarter's B columns come from four warps
        const int base4 = (8 * q4 + 2 * h) * lb + (lane >> 3) * 32 + (lane & 7) * 4;
        const float4 h0 = *reinterpret_cast<const float4*>(bpg + base4);
        const float4 l0 = *reinterpret_cast<const float4*>(bpg + base4 + 128);
        const float4 h1 = *reinterpret_cast<const float4*>(bpg + base4 + lb);
        const float4 l1 = *reinterpret_cast<const float4*>(bpg + base4 + lb + 128);
        v8[0] = h0.x + l0.x; v8[1] = h0.y + l0.y; v8[2] = h0.z + l0.z; v8[3] = h0.w + l0.w;
        v8[4] = h1.x + l1.x; v8[5] = h1.y + l1.y; v8[6] = h1.z + l1.z; v8[7] = h1.w + l1.w;
      }
      tc::fence_before();
      mbar_arrive(B.pg_ready);
#pragma unroll
      for (int d = 0; d < GT_NG; d++) {
        if (d >= a.ng) break;
        const int kl = fkv[d];
        const int kn = __shfl_down_sync(0xffffffffu, kl, 1);
        // bit L: row L of the quarter ends a run (forced at every 8-row group end)
        const unsigned ends = __ballot_sync(0xffffffffu, lane == 31 || kn != kl) | 0x80808080u;
        float run = 0.f;
#pragma unroll
        for (int p = 0; p < 8; p++) {
          run += v8[p];
          if ((ends >> (8 * h + p)) & 1u) {
            const int key = __shfl_sync(0xffffffffu, kl, 8 * h + p);
            if (key >= 0) atomicAdd(a.Z[d] + (int64_t)key * GT_R + lane, (double)run);
            run = 0.f;
          }
        }
      }
      // ---- fold a completed PG group into fp64 (this thread's 8 + 8 columns)
      if ((t % GT_FT) == GT_FT - 1 || t == n - 1) {
        const int g = t / GT_FT, b = g & 1;
        mbar_wait(&B.acc_full[b], (uint32_t)((g >> 1) & 1));
        tc::fence_after();
        uint32_t x0[8], x1[8];
        tc::ld8(tmem + 128 + b * 64 + lane_off + 8 * h, x0);
        tc::ld8(tmem + 128 + b * 64 + lane_off + 32 + 8 * h, x1);
        tc::wait_ld();
#pragma unroll
        for (int j = 0; j < 8; j++)
          acc64[j] += (double)__uint_as_float(x0[j]) + (double)__uint_as_float(x1[j]);
        tc::fence_before();
        mbar_arrive(&B.acc_empty[b]);
      }
    }
    if (UPDATE && tid == 64) bulk_wait<0>();
    double* sc = a.scratch + ((int64_t)blockIdx.x * GT_TILE + r) * 32 + 8 * h;
#pragma unroll
    for (int j = 0; j < 8; j++) sc[j] = acc64[j];
  }

template <bool UPDATE>
__global__ void __launch_bounds__(GT_THREADS, 1)
    k_gnmf_tc(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmF,
              GnTcArgs a, GtGeom gm) {
  extern __shared__ __align__(1024) char smem_raw[];
  char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[2], empty[2], lo_ready, qv_full[2], qv_empty[2], pg_ready, pg_free;
  __shared__ uint64_t acc_full[2], acc_empty[2];
  __shared__ uint32_t tbase;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int SC = a.SC, QK = a.QK, pf = a.pf;

  // ---- constant B operands: H_F^T (N = rank, K = F column) and HH, K-major
  // interleave [K chunk][32][4], tf32 hi / exact lo
  float* cst = reinterpret_cast<float*>(sm + gm.o_cst);
  if (UPDATE) {
    for (int i = tid; i < 8 * 32 * 4; i += blockDim.x) {
      const int ch = i >> 7, n = (i >> 2) & 31, e = i & 3, k = ch * 4 + e;
      int tcol = k < pf ? a.f_tcol[k] : -1;
      const float h = tcol >= 0 ? a.H32[(size_t)n * a.c_T + tcol] : 0.f;
      const float hh = a.HH32[k * GT_R + n];   // HH symmetric: B[k][n] = HH[k][n]
      cst[i] = tf32_hi(h);
      cst[1024 + i] = h - tf32_hi(h);
      cst[2048 + i] = tf32_hi(hh);
      cst[3072 + i] = hh - tf32_hi(hh);
    }
  }
  // A_pg rows past 64 + 2 SC (read by the M = 128 MMA into unused D rows)
  // may hold anything; zero them once so no NaN pattern ever appears
  for (uint32_t b = tid * 4; b < 32 * gm.lbo_a + 256; b += blockDim.x * 4)
    *reinterpret_cast<float*>(sm + gm.o_apg + b) = 0.f;
  if (tid == 0) {
    for (int s = 0; s < 2; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], GT_EPI);
      mbar_init(&qv_full[s], 1);
      mbar_init(&qv_empty[s], GT_EPI);
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], GT_EPI);
    }
    mbar_init(&lo_ready, GT_EPI);
    mbar_init(&pg_ready, GT_EPI);
    mbar_init(&pg_free, 1);
    fence_mbar_init();
  }
  tc::fence_smem_to_async();
  if (warp == 0) tc::alloc(&tbase, 256);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tbase;

  const int64_t G = gridDim.x;
  const int64_t base = a.ntiles / G, rem = a.ntiles % G;
  const int64_t t0 = blockIdx.x * base + min64(blockIdx.x, rem);
  const int n = (int)(base + (blockIdx.x < rem ? 1 : 0));
  const uint32_t tx = 32768u + 512u * a.ng;

  if (warp == 0) {
    // =================== producer ===================
    if (lane == 0) {
      for (int i = 0; i < n; i++) {
        const int s = i & 1;
        if (i >= 2) mbar_wait_sleep(&empty[s], (uint32_t)(((i >> 1) - 1) & 1));
        char* st = sm + s * gm.stage;
        const int row = (int)((t0 + i) * GT_TILE);
        mbar_arrive_expect_tx(&full[s], tx);
        tma_load_2d(st, &tmF, 0, row, &full[s]);
        tma_load_2d(st + gm.o_w, &tmW, 0, row, &full[s]);
        for (int d = 0; d < a.ng; d++)
          bulk_g2s(st + gm.o_fk + 512 * d, a.fk[d] + (t0 + i) * GT_TILE, 512, &full[s]);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // =================== MMA issuer ===================
    if (lane == 0 && n > 0) {
      const uint32_t idq = tc::idesc_tf32(128, 32, false, false);
      const uint32_t idp = tc::idesc_tf32(128, 64, false, false);
      const uint32_t c0 = smem_u32(cst);
      const uint32_t lo = smem_u32(sm + gm.o_lo);
      const uint32_t apg = smem_u32(sm + gm.o_apg), bpg = smem_u32(sm + gm.o_bpg);
      auto issue_qv = [&](int t) {
        const int b = t & 1;
        mbar_wait_sleep(&lo_ready, (uint32_t)(t & 1));
        if (t >= 2) mbar_wait_sleep(&qv_empty[b], (uint32_t)(((t >> 1) - 1) & 1));
        tc::fence_after();
        const uint32_t st = smem_u32(sm + (t & 1) * gm.stage);
        const uint32_t tq = tmem + b * 64, tv = tq + 32;
        for (int ks = 0; ks < QK; ks++) {
          const uint64_t ah = tc::smem_desc(st + ks * 32, 16, 1024, tc::kSw128);
          const uint64_t al = tc::smem_desc(lo + ks * 32, 16, 1024, tc::kSw128);
          const uint64_t bh = tc::smem_desc(c0 + ks * 1024, 512, 128, tc::kInterleave);
          const uint64_t bl = tc::smem_desc(c0 + 4096 + ks * 1024, 512, 128, tc::kInterleave);
          tc::mma_tf32(tq, ah, bh, idq, ks > 0);
          tc::mma_tf32(tq, al, bh, idq, true);
          tc::mma_tf32(tq, ah, bl, idq, true);
        }
        for (int ks = 0; ks < 4; ks++) {
          const uint64_t ah = tc::smem_desc(st + gm.o_w + ks * 32, 16, 1024, tc::kSw128);
          const uint64_t al = tc::smem_desc(lo + 16384 + ks * 32, 16, 1024, tc::kSw128);
          const uint64_t bh = tc::smem_desc(c0 + 8192 + ks * 1024, 512, 128, tc::kInterleave);
          const uint64_t bl = tc::smem_desc(c0 + 12288 + ks * 1024, 512, 128, tc::kInterleave);
          tc::mma_tf32(tv, ah, bh, idq, ks > 0);
          tc::mma_tf32(tv, al, bh, idq, true);
          tc::mma_tf32(tv, ah, bl, idq, true);
        }
        tc::commit(&qv_full[b]);
      };
      if (UPDATE) issue_qv(0);
      for (int t = 0; t < n; t++) {
        if (UPDATE && t + 1 < n) issue_qv(t + 1);
        const int g = t / GT_FT, b = g & 1;
        const bool first = (t % GT_FT) == 0;
        mbar_wait_sleep(&pg_ready, (uint32_t)(t & 1));
        if (first && g >= 2) mbar_wait_sleep(&acc_empty[b], (uint32_t)(((g >> 1) - 1) & 1));
        tc::fence_after();
        const uint32_t tp = tmem + 128 + b * 64;
        for (int kk = 0; kk < GT_TILE / 8; kk++) {
          const uint64_t ad = tc::smem_desc(apg + kk * 2 * gm.lbo_a, gm.lbo_a, 128, tc::kInterleave);
          const uint64_t bd = tc::smem_desc(bpg + kk * 2 * gm.lbo_b, gm.lbo_b, 128, tc::kInterleave);
          tc::mma_tf32(tp, ad, bd, idp, !(first && kk == 0));
        }
        tc::commit(&pg_free);
        if ((t % GT_FT) == GT_FT - 1 || t == n - 1) tc::commit(&acc_full[b]);
      }
    }
    __syncwarp();
  } else {
    const GtBars B{full, empty, &lo_ready, qv_full, qv_empty, &pg_ready, &pg_free, acc_full,
                   acc_empty};
    // one code copy for the four column groups: per-group template copies
    // measured slower (instruction-cache misses, "no_instruction" stalls)
    gt_epilogue<UPDATE>(&tmW, a, gm, sm, tmem, B, n, t0, (warp - 2) >> 2);
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  // CTA partial in k_gnmf_fact's format: [R x SC] P_F | [R x R] G, where
  // G[a][b] = S[a][b] + S[32+a][b] and P_F[a][c] = S[64+c][a] + S[64+SC+c][a]
  const double* S = a.scratch + (int64_t)blockIdx.x * GT_TILE * 32;
  double* out = a.part + (int64_t)blockIdx.x * (GT_R * SC + GT_R * GT_R);
  for (int i = tid; i < GT_R * SC; i += blockDim.x) {
    const int j = i / SC, c = i - j * SC;
    out[i] = S[(64 + c) * 32 + j] + S[(64 + SC + c) * 32 + j];
  }
  for (int i = tid; i < GT_R * GT_R; i += blockDim.x) {
    const int j = i / GT_R, q = i - j * GT_R;
    out[GT_R * SC + i] = S[j * 32 + q] + S[(32 + j) * 32 + q];
  }
  __syncthreads();
  if (warp == 0) tc::dealloc(tmem, 256);
}
