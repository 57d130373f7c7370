// K2 on the 5th-generation tensor cores (included inside namespace flb by
// kmeans.cu): the K-means fact-row pass with both contractions as tcgen05
// MMAs from shared memory into TMEM, and every other step thread-per-row.
// Same arithmetic and outputs as k_km_fact (reference trainers.py:225-241).
//
// One persistent CTA per SM walks a contiguous range of 128-row tiles:
//   warp 0      producer: TMA of the F tile (128 x 32 fp32, 128B swizzle =
//               the K-major SW128 operand layout) and the tile's FKs
//   warp 1      MMA issuer (one thread):
//                 screen  Z = F C_F^T        M = 128 rows, N = KP, K = F cols
//                 sums   S += [F_hi|F_lo]^T A  M = 128 (64 used), N = 32,
//                                            K = 128 rows of the tile
//               The row contraction reads its tiles MN-major (row-major
//               [rows x 32] in the 128B / 32-byte-atom swizzle, descriptor
//               layout 1), so no transposed copy exists anywhere.
//   warps 2-3   gather: the E_d rows of every tile row's FKs, copied from L2
//               into the stage by cp.async (completion on an mbarrier), so
//               the epilogue never waits on a dependent global load
//   warps 4-11  epilogue, two groups of four warps taking alternate tiles;
//               thread = tile row: distances from the screen (+ the staged
//               E_d rows), certified argmin, exact loss,
//               I_d^T A counters, then the row's one-hot, F_hi and F_lo
//               (+ the count column) into the group's MN-major operand tiles.
// The screen is one tf32 term (certified, as k_km_fact); the sums are exact
// in two terms (one-hot x (hi + lo)) and accumulate in TMEM fp32 over
// K5_FT tiles, then fold into fp64 registers (the same 512-row fp32 window
// as k_km_fact's flushes).
constexpr int K5_TILE = 128;
constexpr int K5_EPI = 256;           // epilogue threads (2 groups x 4 warps)
constexpr int K5_GAT = 64;            // gather threads
constexpr int K5_THREADS = 64 + K5_GAT + K5_EPI;
constexpr int K5_NS_MAX = 3;          // TMA stages (2 or 3: whatever fits)
constexpr int K5_FT = 4;              // tiles per fp32 sums window
constexpr int K5_SC = 32;             // F columns in the operand tiles (pf <= 28)
constexpr int K5_PD = 8;              // tiles prefetched into L2 ahead of the TMA loads

struct KmT5Args {
  int pf, c_T, k;
  int64_t r_T, ntiles;
  int ng, sort_g;
  const int32_t* fk[MAX_GATHER];
  const float* E[MAX_GATHER];        // (r_d + 1) x KP
  int32_t* cnt[MAX_GATHER];          // r_d x KP
  int64_t rows[MAX_GATHER];
  const float* C32;                  // k x c_T
  const int32_t* f_tcol;
  int32_t* assign;
  double* part;                      // gridDim.x x (KP * 32 + 1), k_km_fact's format
};

struct K5Geom {                      // byte offsets from the 1024-aligned base
  int ns;                            // stages
  uint32_t stage, o_fk, o_e;         // stage: F tile (16 KB) | FKs (512 B per source) |
                                     //        E rows [source][128][KP] fp32
  uint32_t o_ops;                    // 2 groups x [F_hi | F_lo | one-hot] (3 x 16 KB)
  uint32_t o_cb, o_cf, o_cn, o_scr;  // screen B operand, fp32 centroids, norms, fp64 scratch
  uint32_t total;
};

__host__ __device__ inline K5Geom k5_geom(int KP, int ng) {
  K5Geom g{};
  g.o_fk = 16384;
  g.o_e = (uint32_t)round_up(16384 + 512 * (ng > 0 ? ng : 1), 128);
  g.stage = (uint32_t)round_up(g.o_e + 512 * KP * ng, 1024);
  const uint32_t fixed = 2 * 49152 + (uint32_t)KP * 128 + (uint32_t)KP * 36 * 4 + KP * 4 + 1024 +
                         32 * 64 * 8;
  g.ns = (K5_NS_MAX * g.stage + fixed + 1024 <= 227 * 1024) ? K5_NS_MAX : 2;
  g.o_ops = g.ns * g.stage;
  g.o_cb = g.o_ops + 2 * 49152;
  g.o_cf = g.o_cb + (uint32_t)KP * 128;
  g.o_cn = g.o_cf + (uint32_t)KP * 36 * 4;
  g.o_scr = (uint32_t)round_up(g.o_cn + KP * 4, 1024);
  g.total = g.o_scr + 32 * 64 * 8;   // also >= 16 KB past the last ops tile (M = 128 over-read)
  return g;
}

// byte offset of fp32 element (row, col) in a [rows x 32] tile with the
// 128B swizzle (16-byte chunks XOR row % 8): the K-major SW128 layout
__device__ __forceinline__ uint32_t k5_sw128(int row, int col) {
  return (uint32_t)(row * 128 + ((((col >> 2) ^ (row & 7))) << 4) + (col & 3) * 4);
}
// byte offset of the 16-byte chunk c (columns 4c .. 4c+3) of row `row` in a
// [rows x 32] tile with the 128B swizzle of 32-byte atoms (MN-major tf32
// operand layout): 32-byte granule g of row r sits at g ^ (r % 4)
// (measured, profiles/r02_tc_probe.txt)
__device__ __forceinline__ float k5_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }
__device__ __forceinline__ uint32_t k5_b32(int row, int c) {
  return (uint32_t)(row * 128 + (((c >> 1) ^ (row & 3)) << 5) + ((c & 1) << 4));
}

template <int KP>
__global__ void __launch_bounds__(K5_THREADS, 1)
    k_km_t5(const __grid_constant__ CUtensorMap tmF, KmT5Args a, K5Geom gm) {
  extern __shared__ __align__(1024) char smem_raw[];
  char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[K5_NS_MAX], empty[K5_NS_MAX], es_ready[K5_NS_MAX];
  __shared__ uint64_t scr_full[2], ops_ready[2], ops_free[2];
  __shared__ uint64_t acc_full[2], acc_empty[2];
  __shared__ uint32_t tbase;
  __shared__ double lsum_w[K5_EPI / 32];


  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int pf = a.pf, k = a.k;
  float* cb = reinterpret_cast<float*>(sm + gm.o_cb);   // [8 K chunks][KP][4] (rounded tf32)
  float* cf = reinterpret_cast<float*>(sm + gm.o_cf);   // [KP][36] fp32 centroid F slice
  float* cn = reinterpret_cast<float*>(sm + gm.o_cn);   // [KP] ||c_F||^2 (inf past k)
  for (int i = tid; i < KP * 36; i += blockDim.x) {
    const int j = i / 36, c = i - j * 36;
    float v = 0.f;
    if (j < k && c < pf) {
      const int tc = a.f_tcol[c];
      if (tc >= 0) v = a.C32[(int64_t)j * a.c_T + tc];
    }
    cf[i] = v;
  }
  __syncthreads();
  for (int i = tid; i < 8 * KP * 4; i += blockDim.x) {
    const int ch = i / (KP * 4), n = (i / 4) % KP, e = i & 3;
    cb[i] = __uint_as_float(tf32_bits(cf[n * 36 + ch * 4 + e]));
  }
  for (int j = tid; j < KP; j += blockDim.x) {
    float s = 0.f;
    for (int c = 0; c < K5_SC; c++) s = fmaf(cf[j * 36 + c], cf[j * 36 + c], s);
    cn[j] = j < k ? s : __int_as_float(0x7f800000);
  }
  if (tid == 0) {
    for (int s = 0; s < K5_NS_MAX; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&es_ready[s], K5_GAT);
    }
    for (int g = 0; g < 2; g++) {
      mbar_init(&scr_full[g], 1);
      mbar_init(&ops_ready[g], 128);
      mbar_init(&ops_free[g], 1);
      mbar_init(&acc_full[g], 1);
      mbar_init(&acc_empty[g], 64);
    }
    fence_mbar_init();
  }
  tc::fence_smem_to_async();
  if (warp == 0) tc::alloc(&tbase, 128);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tbase;   // cols [0, 64): screen of group g at 32 g; [64, 128): sums

  const int64_t G = gridDim.x;
  const int64_t base = a.ntiles / G, rem = a.ntiles % G;
  const int64_t t0 = blockIdx.x * base + min64(blockIdx.x, rem);
  const int n = (int)(base + (blockIdx.x < rem ? 1 : 0));
  const int ng = a.ng;
  const int NS = gm.ns;

  if (warp == 0) {
    // =================== producer ===================
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
      for (int i = 0; i < K5_PD && i < n; i++) tma_prefetch_2d(&tmF, 0, (int)((t0 + i) * K5_TILE));
      for (int i = 0; i < n; i++) {
        const int s = i % NS;
        if (i + K5_PD < n) {
          tma_prefetch_2d(&tmF, 0, (int)((t0 + i + K5_PD) * K5_TILE));
          for (int d = 0; d < ng; d++) bulk_prefetch_l2(a.fk[d] + (t0 + i + K5_PD) * K5_TILE, 512);
        }
        if (i >= NS) mbar_wait_sleep(&empty[s], (uint32_t)(((i / NS) - 1) & 1));
        char* st = sm + s * gm.stage;
        mbar_arrive_expect_tx(&full[s], 16384u + 512u * ng);
        tma_load_2d_hint(st, &tmF, 0, (int)((t0 + i) * K5_TILE), &full[s], pol);
        for (int d = 0; d < ng; d++)
          bulk_g2s(st + gm.o_fk + 512 * d, a.fk[d] + (t0 + i) * K5_TILE, 512, &full[s]);
      }
    }
  } else if (warp == 1) {
    // =================== MMA issuer ===================
    if (lane == 0 && n > 0) {
      const uint32_t id_scr = tc::idesc_tf32(128, KP, false, false);
      const uint32_t id_sum = tc::idesc_tf32(128, 32, true, true);
      const uint32_t cb0 = smem_u32(cb);
      const int kst = (pf + 7) / 8;
      auto screen = [&](int t) {
        const int s = t % NS, g = t & 1;
        mbar_wait_sleep(&full[s], (uint32_t)((t / NS) & 1));
        tc::fence_after();
        const uint32_t st = smem_u32(sm + s * gm.stage);
        for (int ks = 0; ks < kst; ks++) {
          const uint64_t ad = tc::smem_desc(st + ks * 32, 16, 1024, tc::kSw128);
          const uint64_t bd = tc::smem_desc(cb0 + ks * 2 * KP * 16, KP * 16, 128, tc::kInterleave);
          tc::mma_tf32(tmem + 32 * g, ad, bd, id_scr, ks > 0);
        }
        tc::commit(&scr_full[g]);
      };
      screen(0);
      if (n > 1) screen(1);
      for (int t = 0; t < n; t++) {
        const int g = t & 1, s = t % NS;
        const int w = t / K5_FT, b = w & 1;
        mbar_wait_sleep(&ops_ready[g], (uint32_t)((t >> 1) & 1));
        if ((t % K5_FT) == 0 && w >= 2) mbar_wait_sleep(&acc_empty[b], (uint32_t)(((w >> 1) - 1) & 1));
        tc::fence_after();
        const uint32_t ops = smem_u32(sm + gm.o_ops + g * 49152);
        for (int kk = 0; kk < K5_TILE / 8; kk++) {
          // MN-major, 128B / 32B-atom swizzle: LBO = stride between 32-element
          // MN groups, SBO = stride between 4-row K groups (profiles/r02_tc_probe.txt)
          const uint64_t ad = tc::smem_desc(ops + kk * 1024, 16384, 512, tc::kSw128B32);
          const uint64_t bd = tc::smem_desc(ops + 32768 + kk * 1024, 16384, 512, tc::kSw128B32);
          tc::mma_tf32(tmem + 64 + 32 * b, ad, bd, id_sum, !((t % K5_FT) == 0 && kk == 0));
        }
        tc::commit(&empty[s]);
        tc::commit(&ops_free[g]);
        if ((t % K5_FT) == K5_FT - 1 || t == n - 1) tc::commit(&acc_full[b]);
        if (t + 2 < n) screen(t + 2);
      }
    }
  } else if (warp < 4) {
    // =================== gather: E_d rows -> the stage (cp.async) ===================
    const int gt = tid - 64;
    constexpr int Q = KP / 4;
    for (int i = 0; i < n; i++) {
      const int s = i % NS;
      char* st = sm + s * gm.stage;
      mbar_wait_sleep(&full[s], (uint32_t)((i / NS) & 1));   // the tile's FKs
      const int32_t* fks = reinterpret_cast<const int32_t*>(st + gm.o_fk);
      for (int rr = gt; rr < K5_TILE; rr += K5_GAT) {
#pragma unroll
        for (int d = 0; d < MAX_GATHER; d++) {
          if (d >= ng) break;
          const int f = fks[d * K5_TILE + rr];
          const float* src = a.E[d] + (f >= 0 ? (int64_t)f : a.rows[d]) * KP;
          char* dst = st + gm.o_e + (d * K5_TILE + rr) * KP * 4;
#pragma unroll
          for (int q = 0; q < Q; q++) cp_async16(dst + 16 * (q ^ (rr & (Q - 1))), src + 4 * q);
        }
      }
      cp_async_mbar_arrive(&es_ready[s]);
    }
  } else {
    // =================== epilogue ===================
    const int ew = warp - 4, grp = ew >> 2;
    const int q4 = warp & 3;                  // TMEM lane quarter of this warp
    const int r = 32 * q4 + lane;             // tile row
    const uint32_t lane_off = (uint32_t)(32 * q4) << 16;
    char* ops = sm + gm.o_ops + grp * 49152;
    const bool flusher = grp == 1 && q4 < 2;  // TMEM lanes 0..63 of the sums
    // fp64 sums of TMEM lane r in smem, [cluster][lane] (conflict-free)
    double* acc64 = reinterpret_cast<double*>(sm + gm.o_scr);
    if (flusher)
      for (int j = 0; j < 32; j++) acc64[j * 64 + r] = 0.0;
    double lsum = 0.0;
    const int pf4 = pf / 4;
    float cn_max = 0.f;
    for (int j = 0; j < k; j++) cn_max = fmaxf(cn_max, cn[j]);
    auto flush = [&](int w) {
      const int b = w & 1;
      mbar_wait_sleep(&acc_full[b], (uint32_t)((w >> 1) & 1));
      tc::fence_after();
      uint32_t x[16];
#pragma unroll
      for (int h = 0; h < 2; h++) {
        tc::ld16(tmem + lane_off + 64 + 32 * b + 16 * h, x);
        tc::wait_ld();
#pragma unroll
        for (int j = 0; j < 16; j++) acc64[(16 * h + j) * 64 + r] += (double)__uint_as_float(x[j]);
      }
      tc::fence_before();
      mbar_arrive(&acc_empty[b]);
    };
    for (int t = grp; t < n; t += 2) {
      const int s = t % NS;
      char* st = sm + s * gm.stage;
      mbar_wait_sleep(&full[s], (uint32_t)((t / NS) & 1));
      const int32_t* fks = reinterpret_cast<const int32_t*>(st + gm.o_fk);
      const int64_t p = (t0 + t) * K5_TILE + r;
      const bool valid = p < a.r_T;
      // E rows of every gathered source (staged by the gather warps)
      float eacc[KP];
#pragma unroll
      for (int j = 0; j < KP; j++) eacc[j] = 0.f;
      int fkv[MAX_GATHER];
      mbar_wait_sleep(&es_ready[s], (uint32_t)((t / NS) & 1));
#pragma unroll
      for (int d = 0; d < MAX_GATHER; d++) {
        if (d >= ng) break;
        fkv[d] = fks[d * K5_TILE + r];
        const char* er = st + gm.o_e + (d * K5_TILE + r) * KP * 4;
#pragma unroll
        for (int q = 0; q < KP / 4; q++) {
          const float4 v = *reinterpret_cast<const float4*>(er + 16 * (q ^ (r & (KP / 4 - 1))));
          eacc[4 * q + 0] += v.x;
          eacc[4 * q + 1] += v.y;
          eacc[4 * q + 2] += v.z;
          eacc[4 * q + 3] += v.w;
        }
      }
      // the F row (exact fp32) from the K-major tile
      float4 xr[K5_SC / 4];
#pragma unroll
      for (int c4 = 0; c4 < K5_SC / 4; c4++)
        xr[c4] = c4 < pf4 ? *reinterpret_cast<const float4*>(st + k5_sw128(r, 4 * c4))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
      // screen distances: ||c||^2 + E - 2 z
      mbar_wait_sleep(&scr_full[grp], (uint32_t)((t >> 1) & 1));
      tc::fence_after();
      float dv[KP];
      {
        uint32_t z[16];
#pragma unroll
        for (int h = 0; h < KP / 16; h++) {
          tc::ld16(tmem + lane_off + 32 * grp + 16 * h, z);
          tc::wait_ld();
#pragma unroll
          for (int j = 0; j < 16; j++)
            dv[16 * h + j] = fmaf(-2.f, __uint_as_float(z[j]), cn[16 * h + j] + eacc[16 * h + j]);
        }
      }
      // best / runner-up (ties -> lowest index)
      float v1 = dv[0], v2 = __int_as_float(0x7f800000);
      int al = 0;
#pragma unroll
      for (int j = 1; j < KP; j++) {
        const bool lt = dv[j] < v1;
        v2 = lt ? v1 : fminf(v2, dv[j]);
        al = lt ? j : al;
        v1 = lt ? dv[j] : v1;
      }
      float xn = 0.f;
#pragma unroll
      for (int c4 = 0; c4 < K5_SC / 4; c4++)
        xn = fmaf(xr[c4].x, xr[c4].x, fmaf(xr[c4].y, xr[c4].y,
             fmaf(xr[c4].z, xr[c4].z, fmaf(xr[c4].w, xr[c4].w, xn))));
      // certify (k_km_fact's bound): near-ties re-decided from exact fp32
      // differences of the F part plus the E terms
      const float tol = 4e-3f * (xn + cn_max) + 1e-5f * (fabsf(v1) + fminf(fabsf(v2), 3e38f));
      if (valid && !(v2 - v1 > tol)) {
        float bd = __int_as_float(0x7f800000);
        int bj = 0;
        for (int j = 0; j < k; j++) {
          if (!(dv[j] - v1 <= tol)) continue;
          const float4* cr = reinterpret_cast<const float4*>(cf + j * 36);
          float dj = 0.f;
#pragma unroll
          for (int c4 = 0; c4 < K5_SC / 4; c4++) {
            const float4 c = cr[c4];
            const float d0 = xr[c4].x - c.x, d1 = xr[c4].y - c.y;
            const float d2 = xr[c4].z - c.z, d3 = xr[c4].w - c.w;
            dj = fmaf(d0, d0, fmaf(d1, d1, fmaf(d2, d2, fmaf(d3, d3, dj))));
          }
          float ej = 0.f;
#pragma unroll
          for (int jj = 0; jj < KP; jj++) ej = jj == j ? eacc[jj] : ej;
          dj += ej;
          if (dj < bd) {
            bd = dj;
            bj = j;
          }
        }
        al = bj;
      }
      // exact loss: ||x - c_a||^2 + sum_d E_d[fk_d, a]
      if (valid) {
        float el = 0.f;
#pragma unroll
        for (int jj = 0; jj < KP; jj++) el = jj == al ? eacc[jj] : el;
        const float4* cr = reinterpret_cast<const float4*>(cf + al * 36);
        float l = el;
#pragma unroll
        for (int c4 = 0; c4 < K5_SC / 4; c4++) {
          const float4 c = cr[c4];
          const float d0 = xr[c4].x - c.x, d1 = xr[c4].y - c.y;
          const float d2 = xr[c4].z - c.z, d3 = xr[c4].w - c.w;
          l = fmaf(d0, d0, fmaf(d1, d1, fmaf(d2, d2, fmaf(d3, d3, l))));
        }
        lsum += (double)l;
        if (a.assign) a.assign[p] = al;
      }
      // I_d^T A counters (integer atomics; runs of the sorted source merged)
#pragma unroll
      for (int d = 0; d < MAX_GATHER; d++) {
        if (d >= ng) break;
        const int f = fkv[d];
        const int key = (valid && f >= 0) ? f * KP + al : -1 - lane;
        if (d == a.sort_g) {
          const unsigned mask = __match_any_sync(0xffffffffu, key);
          if (key >= 0 && (__ffs(mask) - 1) == lane) atomicAdd(&a.cnt[d][key], __popc(mask));
        } else if (key >= 0) {
          atomicAdd(&a.cnt[d][key], 1);
        }
      }
      // operand rows: F_hi | F_lo (+ count column 31) | one-hot
      if (t >= 2) mbar_wait_sleep(&ops_free[grp], (uint32_t)(((t >> 1) - 1) & 1));
#pragma unroll
      for (int c4 = 0; c4 < K5_SC / 4; c4++) {
        const float4 x = valid ? xr[c4] : make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 hi = make_float4(k5_hi(x.x), k5_hi(x.y), k5_hi(x.z), k5_hi(x.w));
        float4 lo = make_float4(x.x - hi.x, x.y - hi.y, x.z - hi.z, x.w - hi.w);
        if (c4 == K5_SC / 4 - 1) lo.w = valid ? 1.f : 0.f;
        *reinterpret_cast<float4*>(ops + k5_b32(r, c4)) = hi;
        *reinterpret_cast<float4*>(ops + 16384 + k5_b32(r, c4)) = lo;
        const int j0 = 4 * c4;
        const int aa = valid ? al : -1;
        *reinterpret_cast<float4*>(ops + 32768 + k5_b32(r, c4)) =
            make_float4(aa == j0 ? 1.f : 0.f, aa == j0 + 1 ? 1.f : 0.f, aa == j0 + 2 ? 1.f : 0.f,
                        aa == j0 + 3 ? 1.f : 0.f);
      }
      fence_proxy_async();
      tc::fence_before();
      mbar_arrive(&ops_ready[grp]);
      if (flusher && (t % K5_FT) == K5_FT - 1) flush(t / K5_FT);
    }
    // the last (partial) window
    if (flusher && n > 0 && ((n - 1) % K5_FT) != K5_FT - 1) flush((n - 1) / K5_FT);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
    if (lane == 0) lsum_w[ew] = lsum;
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  // CTA partial in k_km_fact's format: [KP x 32] sums (count at column pf) | loss
  const double* scr = reinterpret_cast<const double*>(sm + gm.o_scr);
  double* out = a.part + (int64_t)blockIdx.x * (KP * K5_SC + 1);
  for (int i = tid; i < KP * K5_SC; i += blockDim.x) {
    const int j = i / K5_SC, c = i - j * K5_SC;
    double v = 0.0;
    if (c < pf) v = scr[j * 64 + c] + scr[j * 64 + 32 + c];
    else if (c == pf) v = scr[j * 64 + 32 + 31];
    out[i] = v;
  }
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < K5_EPI / 32; w++) s += lsum_w[w];
    out[KP * K5_SC] = s;
  }
  __syncthreads();
  if (warp == 0) tc::dealloc(tmem, 128);
}
