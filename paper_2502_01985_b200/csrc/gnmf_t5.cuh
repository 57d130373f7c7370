// F on the 5th-generation tensor cores with MN-major row-contraction
// operands (included inside namespace flb by gnmf.cu): the GNMF fact-row
// pass for rank tiles of R = 32, <= 28 streamed columns and at most one
// gathered source (the sort source).  Same arithmetic and outputs as
// k_gnmf_fact (reference trainers.py:283-298): Q = T H^T, W' = W o Q /
// (W H H^T + eps), then P_F = W'^T F, G = W'^T W' and Z = I^T W' for the next
// H update.
//
// One persistent CTA per SM walks a contiguous range of 128-row tiles:
//   warp 0      producer: TMA of the W and F tiles (128 x 32 fp32, 128B
//               swizzle = K-major SW128 operands) and the tile's FKs
//   warp 1      MMA issuer (one thread), every product 3xTF32 (kind::tf32
//               truncates, so an fp32 tile is its own hi part):
//                 Q  = F H_F^T            M = 128 rows, N = 32, K = F cols
//                 V  = W HH               M = 128 rows, N = 32, K = 32
//                 PG += [W'|W'_lo|F|F_lo]^T [W'|W'_lo]   M = 128, N = 64,
//                                         K = 128 rows of the tile
//               PG reads its four row-major [128 x 32] tiles MN-major (128B /
//               32-byte-atom swizzle, descriptor layout 1): no transposes.
//   warps 2-17  epilogue, thread = (tile row, 8-column group): lo parts of W
//               and F for Q / V, W' from Q, V and the gathered G_d row, the
//               PG operand rows, the W' TMA store, Z segment sums.
// PG accumulates in TMEM fp32 over G5_FT tiles (512 rows, k_gnmf_fact's
// window), then folds into fp64 registers.
constexpr int G5_TILE = 128;
constexpr int G5_CPT = 8;             // W / Q / V columns per epilogue thread
constexpr int G5_HG = 32 / G5_CPT;    // epilogue threads per row
constexpr int G5_EPI = 128 * G5_HG;
constexpr int G5_THREADS = 64 + G5_EPI;
constexpr int G5_NS = 3;
constexpr int G5_FT = 4;
constexpr int G5_PD = 6;              // tiles prefetched into L2 ahead of the TMA loads

struct GnT5Args {
  int pf, c_T;
  int64_t r_T, ntiles;
  int ng;                          // 0 or 1 (the sort source)
  int diag;                        // timing experiments only (FL_GN5_DIAG): 1 no Z sums, 2 no PG MMA
  int gpre;                        // G_d rows gathered one tile ahead (FL_GN5_GPRE=0: at use)
  int pd;                          // tiles prefetched into L2 ahead of the TMA loads (FL_GN5_PD)
  const int32_t* fk;
  const float* Gd;                 // r_d x 32
  double* Z;                       // r_d x 32
  const float* H32;                // 32 x c_T
  const float* HH32;               // 32 x 32
  const int32_t* f_tcol;
  double* part;                    // gridDim.x x (32 * 32 + 32 * 32): [P_F (SC = 32) | G]
  double* scratch;                 // gridDim.x x 128 x 64 fp64 PG
};

struct G5Geom {
  uint32_t stage, o_f, o_fk;       // stage: W (16 KB) | F (16 KB) | FKs (512 B)
  uint32_t o_lo;                   // W_lo | F_lo (K-major SW128, 2 x 16 KB)
  uint32_t o_ops;                  // W' | W'_lo | F | F_lo (MN-major, 4 x 16 KB)
  uint32_t o_cst;                  // H_F hi | H_F lo | HH hi | HH lo (interleave, 4 x 4 KB)
  uint32_t total;
};

__host__ __device__ inline G5Geom g5_geom() {
  G5Geom g{};
  g.o_f = 16384;
  g.o_fk = 32768;
  g.stage = 32768 + 1024;
  g.o_lo = G5_NS * g.stage;
  g.o_ops = g.o_lo + 32768;
  g.o_cst = g.o_ops + 65536;
  g.total = g.o_cst + 16384;
  return g;
}

__device__ __forceinline__ uint32_t g5_sw128(int row, int c4) {   // 16B chunk c4 of a K-major SW128 row
  return (uint32_t)(row * 128 + ((c4 ^ (row & 7)) << 4));
}
__device__ __forceinline__ uint32_t g5_b32(int row, int c4) {     // 16B chunk c4 of an MN-major B32 row
  return (uint32_t)(row * 128 + (((c4 >> 1) ^ (row & 3)) << 5) + ((c4 & 1) << 4));
}
__device__ __forceinline__ float g5_lo(float x) {
  return x - __uint_as_float(__float_as_uint(x) & 0xffffe000u);
}

template <bool UPDATE>
__global__ void __launch_bounds__(G5_THREADS, 1)
    k_gnmf_t5(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmF,
              const __grid_constant__ CUtensorMap tmWs, GnT5Args a, G5Geom gm) {
  extern __shared__ __align__(1024) char smem_raw[];
  char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[G5_NS], empty[G5_NS], lo_ready[2], qv_full[2], ops_ready, ops_free;
  __shared__ uint64_t acc_full[2], acc_empty[2];
  __shared__ uint32_t tbase;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int pf = a.pf;

  // ---- constant B operands (K-major interleave [K chunk][32 rank][4]):
  // H_F^T (K = F column) and HH, hi (truncated) / exact lo
  float* cst = reinterpret_cast<float*>(sm + gm.o_cst);
  if (UPDATE) {
    for (int i = tid; i < 8 * 32 * 4; i += blockDim.x) {
      const int ch = i >> 7, n = (i >> 2) & 31, e = i & 3, k = ch * 4 + e;
      const int tcol = k < pf ? a.f_tcol[k] : -1;
      const float h = tcol >= 0 ? a.H32[(size_t)n * a.c_T + tcol] : 0.f;
      const float hh = a.HH32[k * 32 + n];   // HH symmetric
      cst[i] = h - g5_lo(h);
      cst[1024 + i] = g5_lo(h);
      cst[2048 + i] = hh - g5_lo(hh);
      cst[3072 + i] = g5_lo(hh);
    }
  }
  if (tid == 0) {
    for (int s = 0; s < G5_NS; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; b++) {
      mbar_init(&lo_ready[b], G5_EPI);
      mbar_init(&qv_full[b], 1);
    }
    mbar_init(&ops_ready, G5_EPI);
    mbar_init(&ops_free, 1);
    for (int b = 0; b < 2; b++) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], G5_EPI);
    }
    fence_mbar_init();
  }
  tc::fence_smem_to_async();
  if (warp == 0) tc::alloc(&tbase, 256);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tbase;   // [0, 128): Q | V of tile parity b at 64 b; [128, 256): PG x 2

  const int64_t Gd = gridDim.x;
  const int64_t base = a.ntiles / Gd, rem = a.ntiles % Gd;
  const int64_t t0 = blockIdx.x * base + min64(blockIdx.x, rem);
  const int n = (int)(base + (blockIdx.x < rem ? 1 : 0));

  if (warp == 0) {
    // =================== producer ===================
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
      const int pd = a.pd;
      for (int i = 0; i < pd && i < n; i++) {
        tma_prefetch_2d(&tmW, 0, (int)((t0 + i) * G5_TILE));
        tma_prefetch_2d(&tmF, 0, (int)((t0 + i) * G5_TILE));
      }
      for (int i = 0; i < n; i++) {
        const int s = i % G5_NS;
        if (pd > 0 && i + pd < n) {
          tma_prefetch_2d(&tmW, 0, (int)((t0 + i + pd) * G5_TILE));
          tma_prefetch_2d(&tmF, 0, (int)((t0 + i + pd) * G5_TILE));
          if (a.ng) bulk_prefetch_l2(a.fk + (t0 + i + pd) * G5_TILE, 512);
        }
        if (i >= G5_NS) mbar_wait_sleep(&empty[s], (uint32_t)(((i / G5_NS) - 1) & 1));
        char* st = sm + s * gm.stage;
        const int row = (int)((t0 + i) * G5_TILE);
        mbar_arrive_expect_tx(&full[s], 32768u + (a.ng ? 512u : 0u));
        tma_load_2d_hint(st, &tmW, 0, row, &full[s], pol);
        tma_load_2d_hint(st + gm.o_f, &tmF, 0, row, &full[s], pol);
        if (a.ng) bulk_g2s(st + gm.o_fk, a.fk + (t0 + i) * G5_TILE, 512, &full[s]);
      }
    }
  } else if (warp == 1) {
    // =================== MMA issuer ===================
    // lane 0 walks the tiles and issues the MMA chains and commits.  (The
    // converged-warp form with elect.sync issues the UTC instructions back to
    // back but measured 4% slower here: 6.47 vs 6.23 ms per C4 step,
    // profiles/r02_s2_experiments.txt)
    if (lane == 0 && n > 0) {
      const uint32_t id_qv = tc::idesc_tf32(128, 32, false, false);
      const uint32_t id_pg = tc::idesc_tf32(128, 64, true, true);
      const uint32_t c0 = smem_u32(cst);
      const uint32_t ops = smem_u32(sm + gm.o_ops);
      const int kst = (pf + 7) / 8;
      // Q(t), V(t) into TMEM buffer t & 1 once the tile's lo parts are staged
      auto qv = [&](int t) {
        const int b = t & 1;
        mbar_wait_sleep(&lo_ready[b], (uint32_t)((t >> 1) & 1));   // (implies the stage landed)
        tc::fence_after();
        const uint32_t st = smem_u32(sm + (t % G5_NS) * gm.stage);
        const uint32_t lo = smem_u32(sm + gm.o_lo);
        const uint32_t tq = tmem + 64 * b;
        {
          for (int ks = 0; ks < kst; ks++) {   // Q = F H_F^T
            const uint64_t ah = tc::smem_desc(st + gm.o_f + ks * 32, 16, 1024, tc::kSw128);
            const uint64_t al = tc::smem_desc(lo + 16384 + ks * 32, 16, 1024, tc::kSw128);
            const uint64_t bh = tc::smem_desc(c0 + ks * 1024, 512, 128, tc::kInterleave);
            const uint64_t bl = tc::smem_desc(c0 + 4096 + ks * 1024, 512, 128, tc::kInterleave);
            tc::mma_tf32(tq, ah, bh, id_qv, ks > 0);
            tc::mma_tf32(tq, al, bh, id_qv, true);
            tc::mma_tf32(tq, ah, bl, id_qv, true);
          }
#pragma unroll
          for (int ks = 0; ks < 4; ks++) {     // V = W HH
            const uint64_t ah = tc::smem_desc(st + ks * 32, 16, 1024, tc::kSw128);
            const uint64_t al = tc::smem_desc(lo + ks * 32, 16, 1024, tc::kSw128);
            const uint64_t bh = tc::smem_desc(c0 + 8192 + ks * 1024, 512, 128, tc::kInterleave);
            const uint64_t bl = tc::smem_desc(c0 + 12288 + ks * 1024, 512, 128, tc::kInterleave);
            tc::mma_tf32(tq + 32, ah, bh, id_qv, ks > 0);
            tc::mma_tf32(tq + 32, al, bh, id_qv, true);
            tc::mma_tf32(tq + 32, ah, bl, id_qv, true);
          }
          tc::commit(&qv_full[b]);
        }
      };
      if (UPDATE) qv(0);
      for (int t = 0; t < n; t++) {
        const int s = t % G5_NS;
        const int w = t / G5_FT, b = w & 1;
        if (UPDATE && t + 1 < n) qv(t + 1);
        mbar_wait_sleep(&ops_ready, (uint32_t)(t & 1));
        if ((t % G5_FT) == 0 && w >= 2) mbar_wait_sleep(&acc_empty[b], (uint32_t)(((w >> 1) - 1) & 1));
        tc::fence_after();
        const uint32_t tp = tmem + 128 + 64 * b;
        // A = 4 MN groups [W' | W'_lo | F | F_lo], B = [W' | W'_lo]; a K step
        // of 8 rows advances the start address by 1024 B (64 in the 16-byte
        // address field)
        const uint64_t ad0 = tc::smem_desc(ops, 16384, 512, tc::kSw128B32);
        {
          if (!(a.diag & 2)) {
#pragma unroll
            for (int kk = 0; kk < G5_TILE / 8; kk++) {
              const uint64_t ad = ad0 + (uint64_t)(kk * 64);
              tc::mma_tf32(tp, ad, ad, id_pg, !((t % G5_FT) == 0 && kk == 0));
            }
          }
          tc::commit(&empty[s]);
          tc::commit(&ops_free);
          if ((t % G5_FT) == G5_FT - 1 || t == n - 1) tc::commit(&acc_full[b]);
        }
      }
    }
  } else {
    // =================== epilogue: thread = (tile row, G5_CPT-column group) ===================
    const int ew = warp - 2, h = ew >> 2, q4 = warp & 3;
    const int r = 32 * q4 + lane;
    const uint32_t lane_off = (uint32_t)(32 * q4) << 16;
    char* ops = sm + gm.o_ops;
    constexpr int FC = 64 / G5_HG;   // PG columns this thread folds
    double acc[FC];
#pragma unroll
    for (int j = 0; j < FC; j++) acc[j] = 0.0;
    auto fold = [&](int w) {
      const int b = w & 1;
      mbar_wait_sleep(&acc_full[b], (uint32_t)((w >> 1) & 1));
      tc::fence_after();
      uint32_t x[16];
#pragma unroll
      for (int u = 0; u < FC / 16; u++) {
        tc::ld16(tmem + lane_off + 128 + 64 * b + FC * h + 16 * u, x);
        tc::wait_ld();
#pragma unroll
        for (int j = 0; j < 16; j++) acc[16 * u + j] += (double)__uint_as_float(x[j]);
      }
      tc::fence_before();
      mbar_arrive(&acc_empty[b]);
    };
    constexpr int NU = G5_CPT / 4;   // 16-byte chunks per thread
    // this thread's G5_CPT columns of the W and F rows of tile t (exact fp32)
    auto load_row = [&](int t, float (&w)[G5_CPT], float (&x)[G5_CPT]) {
      const char* st = sm + (t % G5_NS) * gm.stage;
#pragma unroll
      for (int u = 0; u < NU; u++) {
        const int c4 = NU * h + u;
        const float4 wv = *reinterpret_cast<const float4*>(st + g5_sw128(r, c4));
        const float4 xv = *reinterpret_cast<const float4*>(st + gm.o_f + g5_sw128(r, c4));
        w[4 * u + 0] = wv.x; w[4 * u + 1] = wv.y; w[4 * u + 2] = wv.z; w[4 * u + 3] = wv.w;
        x[4 * u + 0] = xv.x; x[4 * u + 1] = xv.y; x[4 * u + 2] = xv.z; x[4 * u + 3] = xv.w;
      }
    };
    // lo parts of tile t for Q / V (K-major SW128, buffer t & 1); F_lo also
    // goes to the PG operand once the buffer is free (see below)
    float4 flo_next[NU];   // F_lo of the tile split last (reused for its PG operand)
    auto split = [&](int t) {
      mbar_wait_sleep(&full[t % G5_NS], (uint32_t)((t / G5_NS) & 1));
      float w[G5_CPT], x[G5_CPT];
      load_row(t, w, x);
      char* lo_b = sm + gm.o_lo;
#pragma unroll
      for (int u = 0; u < NU; u++) {
        const int c4 = NU * h + u;
        *reinterpret_cast<float4*>(lo_b + g5_sw128(r, c4)) =
            make_float4(g5_lo(w[4 * u]), g5_lo(w[4 * u + 1]), g5_lo(w[4 * u + 2]), g5_lo(w[4 * u + 3]));
        flo_next[u] = make_float4(g5_lo(x[4 * u]), g5_lo(x[4 * u + 1]), g5_lo(x[4 * u + 2]),
                                  g5_lo(x[4 * u + 3]));
        *reinterpret_cast<float4*>(lo_b + 16384 + g5_sw128(r, c4)) = flo_next[u];
      }
      fence_proxy_async();
      tc::fence_before();
      mbar_arrive(&lo_ready[t & 1]);
    };
    // G_d[fk] rows of tile t (L2 gathers), loaded one tile ahead: issued
    // right after the tile's stage is known to have landed (split), consumed
    // a tile later, so their latency hides behind this tile's epilogue
    float4 gl_next[NU];
    auto gload = [&](int tt) {
#pragma unroll
      for (int u = 0; u < NU; u++) gl_next[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (!a.ng) return;
      const int32_t* fk_t = reinterpret_cast<const int32_t*>(sm + (tt % G5_NS) * gm.stage + gm.o_fk);
      const int f = fk_t[r];
      if (f >= 0) {
        const float4* gr = reinterpret_cast<const float4*>(a.Gd + (int64_t)f * 32 + G5_CPT * h);
#pragma unroll
        for (int u = 0; u < NU; u++) gl_next[u] = __ldg(gr + u);
      }
    };
    if (UPDATE && n > 0) {
      split(0);
      if (a.gpre) gload(0);
    }
    for (int t = 0; t < n; t++) {
      const int s = t % G5_NS;
      char* st = sm + s * gm.stage;
      // with UPDATE the tile's split (one iteration earlier) already waited
      // for this stage
      if (!UPDATE) mbar_wait_sleep(&full[s], (uint32_t)((t / G5_NS) & 1));
      const int32_t* fks = reinterpret_cast<const int32_t*>(st + gm.o_fk);
      float w[G5_CPT], x[G5_CPT];
      float4 flo[NU];
#pragma unroll
      for (int u = 0; u < NU; u++) flo[u] = flo_next[u];
      if (UPDATE) {
        if (!a.gpre) gload(t);
        float4 gl[NU];
#pragma unroll
        for (int u = 0; u < NU; u++) gl[u] = gl_next[u];
        mbar_wait_sleep(&qv_full[t & 1], (uint32_t)((t >> 1) & 1));
        tc::fence_after();
        uint32_t qq[G5_CPT], vv[G5_CPT];
        static_assert(G5_CPT == 8, "TMEM loads are 8 columns wide");
        tc::ld8(tmem + lane_off + 64 * (t & 1) + G5_CPT * h, qq);
        tc::ld8(tmem + lane_off + 64 * (t & 1) + 32 + G5_CPT * h, vv);
        tc::wait_ld();
        tc::fence_before();
        // software pipeline: Q / V(t) are done with the lo buffer, so the
        // next tile's lo parts go out now and its MMAs overlap the rest of
        // this tile's epilogue
        if (t + 1 < n) {
          split(t + 1);
          if (a.gpre) gload(t + 1);
        }
        load_row(t, w, x);
        // W' = W o (Q + G_d[fk]) / (V + eps)   (k_gnmf_fact's expression)
#pragma unroll
        for (int u = 0; u < NU; u++) {
          const float ga[4] = {gl[u].x, gl[u].y, gl[u].z, gl[u].w};
#pragma unroll
          for (int e = 0; e < 4; e++) {
            const int j = 4 * u + e;
            const float qv = __uint_as_float(qq[j]) + ga[e];
            w[j] = w[j] * __fdividef(qv, __uint_as_float(vv[j]) + 1e-12f);
          }
        }
      } else {
        load_row(t, w, x);
      }
      // PG operand rows: W' | W'_lo | F | F_lo (MN-major B32); the previous
      // tile's PG MMAs and W' store must be done with the buffer
      if (t >= 1) mbar_wait_sleep(&ops_free, (uint32_t)((t - 1) & 1));
      if (UPDATE && tid == 64) bulk_wait_read<0>();
      if (UPDATE) named_sync(1, G5_EPI);
      static_assert(NU == 2, "the conflict-free store order below pairs two chunks");
      {
        // rows r and r + 4 share a 32-byte swizzle granule: odd row quads
        // store the thread's two 16-byte chunks in swapped order, so the
        // eight rows of a store phase hit all 32 banks once (no conflicts)
        const bool sw = (r >> 2) & 1;
        float4 wq[2], wl[2], xq[2], xl[2];
#pragma unroll
        for (int u = 0; u < 2; u++) {
          wq[u] = make_float4(w[4 * u], w[4 * u + 1], w[4 * u + 2], w[4 * u + 3]);
          wl[u] = make_float4(g5_lo(wq[u].x), g5_lo(wq[u].y), g5_lo(wq[u].z), g5_lo(wq[u].w));
          xq[u] = make_float4(x[4 * u], x[4 * u + 1], x[4 * u + 2], x[4 * u + 3]);
          xl[u] = UPDATE ? flo[u] : make_float4(g5_lo(xq[u].x), g5_lo(xq[u].y), g5_lo(xq[u].z), g5_lo(xq[u].w));
        }
#pragma unroll
        for (int u = 0; u < 2; u++) {
          const int uu = sw ? 1 - u : u;
          const uint32_t o = g5_b32(r, NU * h + uu);
          *reinterpret_cast<float4*>(ops + o) = sw ? wq[1 - u] : wq[u];
          *reinterpret_cast<float4*>(ops + 16384 + o) = sw ? wl[1 - u] : wl[u];
          *reinterpret_cast<float4*>(ops + 32768 + o) = sw ? xq[1 - u] : xq[u];
          *reinterpret_cast<float4*>(ops + 49152 + o) = sw ? xl[1 - u] : xl[u];
        }
      }
      fence_proxy_async();
      named_sync(1, G5_EPI);
      if (UPDATE && tid == 64) {
        tma_store_2d_hint(&tmWs, 0, (int)((t0 + t) * G5_TILE), ops, l2_policy_evict_first());
        bulk_commit();
      }
      // Z[fk] += W' rows: warp (q4, h) takes the ZR rows [32 q4 + ZR h, +ZR),
      // lane = rank column; a segment with one FK (the common case: keys are
      // sorted, fanout >> ZR) is one branch-free sum and one fp64 atomic
      if (a.ng && !(a.diag & 1)) {
        constexpr int ZR = 32 / G5_HG;
        const int r0 = 32 * q4 + ZR * h;
        const int c4 = lane >> 2;
        const int k0 = fks[r0], k1 = fks[r0 + ZR - 1];
        const float* zcol = reinterpret_cast<const float*>(ops + (lane & 3) * 4);
        if (k0 == k1) {
          float run = 0.f;
#pragma unroll
          for (int rr = 0; rr < ZR; rr++)
            run += *reinterpret_cast<const float*>(reinterpret_cast<const char*>(zcol) + g5_b32(r0 + rr, c4));
          if (k0 >= 0) atomicAdd(a.Z + (int64_t)k0 * 32 + lane, (double)run);
        } else {
          float run = 0.f;
          int cur = k0;
          for (int rr = r0; rr < r0 + ZR; rr++) {
            const int f = fks[rr];
            if (f != cur) {
              if (cur >= 0) atomicAdd(a.Z + (int64_t)cur * 32 + lane, (double)run);
              run = 0.f;
              cur = f;
            }
            run += *reinterpret_cast<const float*>(reinterpret_cast<const char*>(zcol) + g5_b32(rr, c4));
          }
          if (cur >= 0) atomicAdd(a.Z + (int64_t)cur * 32 + lane, (double)run);
        }
      }
      tc::fence_before();
      mbar_arrive(&ops_ready);
      // fold a finished window one tile late: its MMAs complete while the
      // next tile's epilogue runs (the PG accumulator is double-buffered)
      if ((t % G5_FT) == 0 && t >= G5_FT) fold(t / G5_FT - 1);
    }
    // the loop folded windows 0 .. wl - 1; the last one is left
    if (n > 0) fold((n - 1) / G5_FT);
    if (UPDATE && tid == 64) bulk_wait<0>();
    double* sc = a.scratch + ((int64_t)blockIdx.x * G5_TILE + r) * 64 + FC * h;
#pragma unroll
    for (int j = 0; j < FC; j++) sc[j] = acc[j];
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  // CTA partial in k_gnmf_fact's format [R x SC] P_F (SC = 32) | [R x R] G from
  // S[m][n] (m: W' | W'_lo | F | F_lo columns, n: W' | W'_lo columns)
  const double* S = a.scratch + (int64_t)blockIdx.x * G5_TILE * 64;
  double* out = a.part + (int64_t)blockIdx.x * (32 * 32 + 32 * 32);
  for (int i = tid; i < 32 * 32; i += blockDim.x) {
    const int j = i >> 5, c = i & 31;
    out[i] = c < pf ? S[(64 + c) * 64 + j] + S[(96 + c) * 64 + j] + S[(64 + c) * 64 + 32 + j] : 0.0;
  }
  for (int i = tid; i < 32 * 32; i += blockDim.x) {
    const int j = i >> 5, q = i & 31;
    out[1024 + i] = S[j * 64 + q] + S[(32 + j) * 64 + q] + S[j * 64 + 32 + q];
  }
  __syncthreads();
  if (warp == 0) tc::dealloc(tmem, 256);
}
