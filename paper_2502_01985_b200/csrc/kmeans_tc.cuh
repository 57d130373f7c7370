// K2 on the 5th-generation tensor cores: the K-means fact-row pass with
// tcgen05 MMAs from shared memory into TMEM (included inside namespace flb
// by kmeans.cu).
//
// One persistent CTA per SM walks a contiguous range of 128-row tiles of a
// blocked copy of the stream block (per tile: [chunk][128 rows][4 floats],
// i.e. the canonical no-swizzle K-major / MN-major core-matrix layout, so a
// 1-D bulk copy lands a ready operand).  Warp roles:
//   warp 0     producer: bulk copies (F tile + every source's FKs), and the
//              periodic flush of the sums accumulator (TMEM lanes 0-31) to fp64
//   warp 1     MMA issuer (one thread):
//                Z(t)    = F C_F^T  (M = 128 rows, N = NZ clusters, 3xTF32)
//                S(t)   += F^T A    (M = 128 columns, N = NZ, K = 128 rows;
//                                    F split hi + lo, one-hot A exact)
//              every operand is K-major (kind::tf32 accepts MN-major operands
//              only in the 128B_BASE32B swizzle), so the epilogue also writes
//              F^T and A^T tiles in the K-major interleave layout
//   warps 2-5  epilogue group 0 (even tiles), warps 6-9 group 1 (odd tiles),
//              thread = tile row: split F into tf32 hi / lo in place, then
//              read its Z row from TMEM, argmin (certified exactly as in the
//              mma.sync kernel), loss, I_d^T A counters, one-hot row.
// Per tile the only SIMT work left is per-row; all products run as single-
// thread tcgen05 instructions.

constexpr int KT_TILE = 128;
constexpr int KT_NS = 3;          // stages (tiles in flight)
constexpr int KT_FT = 8;          // tiles per sums accumulation group (1024 rows)
constexpr int KT_THREADS = 320;   // 10 warps

struct KmTcArgs {
  const float* Fblk;              // tiles of [C4P chunks][128][4]
  int pf, c_T, k;
  int64_t r_T, ntiles;
  int ng, sort_g;
  const int32_t* fk[MAX_GATHER];
  const float* E[MAX_GATHER];
  int32_t* cnt[MAX_GATHER];
  int64_t rows[MAX_GATHER];
  const float* C32;
  const int32_t* f_tcol;
  int32_t* assign;
  double* part;                   // gridDim.x x (KP * SC + 1), KP = NZ rows used
  int SC;                         // partial stride (columns incl. the count column)
};

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

struct KtGeom {                   // byte offsets inside one stage / the CTA
  uint32_t stage;                 // bytes per stage
  uint32_t o_flo, o_fth, o_ftl, o_oht, o_fk;
  uint32_t lbo_ft, lbo_oh;        // K-chunk strides of the transposed tiles
  uint32_t off_cf;                // centroid data (after the stages)
};

template <int NZ>
__global__ void __launch_bounds__(KT_THREADS, 1) k_km_tc(KmTcArgs a, int C4P, KtGeom gm) {
  extern __shared__ __align__(1024) char smem_raw[];
  char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[KT_NS], lo_ready[KT_NS], oh_ready[KT_NS], empty[KT_NS];
  __shared__ uint64_t z_full[2], s_full[2], s_empty[2];
  __shared__ uint32_t tbase;
  __shared__ double lsum_w[KT_THREADS / 32];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int pf = a.pf, k = a.k;
  const int KS = (C4P + 1) / 2;                 // Z K-steps (8 columns each)
  const int SC = a.SC;
  // ---- smem carve-up
  float* cf_hi = reinterpret_cast<float*>(sm + gm.off_cf);       // [(C4P+1) chunks][NZ][4]
  float* cf_lo = cf_hi + (C4P + 1) * NZ * 4;
  float* cf = cf_lo + (C4P + 1) * NZ * 4;                        // [NZ][CFP]
  const int CFP = (C4P + 1) * 4 + 4;
  float* cn = cf + NZ * CFP;                                     // [NZ]
  double* sums64 = reinterpret_cast<double*>(cn + NZ + (NZ & 1 ? 1 : 0) + 2);   // [32][NZ]

  // ---- one-time setup: centroid slices, norms, count chunks, barriers, TMEM
  for (int i = tid; i < NZ * CFP; i += blockDim.x) {
    const int j = i / CFP, c = i - j * CFP;
    float v = 0.f;
    if (j < k && c < pf) {
      const int tc = a.f_tcol[c];
      if (tc >= 0) v = a.C32[(int64_t)j * a.c_T + tc];
    }
    cf[i] = v;
  }
  for (int i = tid; i < 32 * NZ; i += blockDim.x) sums64[i] = 0.0;
  // static parts of every stage: zero chunk C4P of F / F_lo (read by the Z
  // K-steps, multiplied by zero centroid columns) and the transposed tiles
  // (rows past pf stay zero; row pf of F^T hi is the count column of ones)
  for (int s = 0; s < KT_NS; s++) {
    char* st = sm + s * gm.stage;
    float* fs = reinterpret_cast<float*>(st);
    float* fl = reinterpret_cast<float*>(st + gm.o_flo);
    for (int r = tid; r < KT_TILE; r += blockDim.x) {
      *reinterpret_cast<float4*>(fs + C4P * 512 + r * 4) = make_float4(0.f, 0.f, 0.f, 0.f);
      *reinterpret_cast<float4*>(fl + C4P * 512 + r * 4) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (uint32_t b = tid * 4; b < gm.o_oht - gm.o_fth; b += blockDim.x * 4)
      *reinterpret_cast<float*>(st + gm.o_fth + b) = 0.f;
  }
  __syncthreads();
  for (int s = 0; s < KT_NS; s++) {
    float* fth = reinterpret_cast<float*>(sm + s * gm.stage + gm.o_fth);
    for (int r = tid; r < KT_TILE; r += blockDim.x)
      fth[((r >> 2) * gm.lbo_ft + (pf >> 3) * 128 + (pf & 7) * 16) / 4 + (r & 3)] = 1.f;
  }
  if (tid == 0) {
    for (int s = 0; s < KT_NS; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&lo_ready[s], 128);
      mbar_init(&oh_ready[s], 128);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; b++) {
      mbar_init(&z_full[b], 1);
      mbar_init(&s_full[b], 1);
      mbar_init(&s_empty[b], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  // tf32 B operands (K-major interleave [chunk][NZ][4]) and norms
  for (int i = tid; i < (C4P + 1) * NZ * 4; i += blockDim.x) {
    const int ch = i / (NZ * 4), rem = i - ch * NZ * 4, j = rem / 4, e = rem & 3;
    const int c = ch * 4 + e;
    const float v = c < CFP ? cf[j * CFP + c] : 0.f;
    const uint32_t hb = __float_as_uint(v) & 0xffffe000u;
    cf_hi[i] = __uint_as_float(hb);
    cf_lo[i] = v - __uint_as_float(hb);
  }
  for (int j = tid; j < NZ; j += blockDim.x) {
    float s = 0.f;
    for (int c = 0; c < CFP; c++) s = fmaf(cf[j * CFP + c], cf[j * CFP + c], s);
    cn[j] = j < k ? s : __int_as_float(0x7f800000);
  }
  tc::fence_smem_to_async();
  if (warp == 0) tc::alloc(&tbase, 128);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tbase;
  const uint32_t tz[2] = {tmem, tmem + NZ};                  // Z buffers
  const uint32_t ts[2] = {tmem + 2 * NZ, tmem + 3 * NZ};     // sums buffers
  float cn_max = 0.f;
  for (int j = 0; j < k; j++) cn_max = fmaxf(cn_max, cn[j]);

  // this CTA's tiles
  const int64_t G = gridDim.x;
  const int64_t base = a.ntiles / G, rem = a.ntiles % G;
  const int64_t t0 = blockIdx.x * base + min64(blockIdx.x, rem);
  const int n = (int)(base + (blockIdx.x < rem ? 1 : 0));
  const int ngrp = (n + KT_FT - 1) / KT_FT;
  const uint32_t f_bytes = (uint32_t)C4P * 2048u;
  const uint32_t fk_bytes = 512u * a.ng;

  if (warp == 0) {
    // =================== producer + sums flusher ===================
    int flushed = 0;
    auto flush_one = [&](int g) {   // whole warp; s_full(g) has completed
      const int b = g & 1;
      tc::fence_after();
      for (int c0 = 0; c0 < NZ; c0 += 16) {
        uint32_t r[16];
        tc::ld16(ts[b] + c0, r);   // lanes 0-31 = F columns 0-31
        tc::wait_ld();
#pragma unroll
        for (int j = 0; j < 16; j++) sums64[lane * NZ + c0 + j] += (double)__uint_as_float(r[j]);
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[b]);
    };
    // flush the next sums group if its accumulation is complete (warp-uniform)
    auto try_flush = [&]() -> bool {
      if (flushed >= ngrp) return false;
      int ok = 0;
      if (lane == 0) ok = mbar_try_wait(&s_full[flushed & 1], (uint32_t)((flushed >> 1) & 1));
      ok = __shfl_sync(0xffffffffu, ok, 0);
      if (ok) flush_one(flushed++);
      return ok != 0;
    };
    for (int i = 0; i < n; i++) {
      const int s = i % KT_NS;
      if (i >= KT_NS) {   // wait for the stage, flushing sums groups meanwhile
        const uint32_t par = (uint32_t)(((i / KT_NS) - 1) & 1);
        while (true) {
          int ok = 0;
          if (lane == 0) ok = mbar_try_wait(&empty[s], par);
          if (__shfl_sync(0xffffffffu, ok, 0)) break;
          try_flush();
        }
      }
      if (lane == 0) {
        char* st = sm + s * gm.stage;
        mbar_arrive_expect_tx(&full[s], f_bytes + fk_bytes);
        bulk_g2s(st, a.Fblk + (t0 + i) * (int64_t)C4P * 512, f_bytes, &full[s]);
        for (int d = 0; d < a.ng; d++)
          bulk_g2s(st + gm.o_fk + 512 * d, a.fk[d] + (t0 + i) * KT_TILE, 512, &full[s]);
      }
      __syncwarp();
      try_flush();
    }
    while (flushed < ngrp) try_flush();
  } else if (warp == 1) {
    // =================== MMA issuer ===================
    if (lane == 0 && n > 0) {
      const uint32_t idz = tc::idesc_tf32(128, NZ, false, false);
      const uint32_t ids = tc::idesc_tf32(128, NZ, false, false);
      const uint32_t chi = smem_u32(cf_hi), clo = smem_u32(cf_lo);
      auto issue_z = [&](int j) {
        const int s = j % KT_NS;
        mbar_wait(&lo_ready[s], (uint32_t)((j / KT_NS) & 1));
        tc::fence_after();
        const uint32_t fh = smem_u32(sm + s * gm.stage), fl = fh + gm.o_flo;
        for (int ks = 0; ks < KS; ks++) {
          const uint64_t ah = tc::smem_desc(fh + ks * 4096, 2048, 128, tc::kInterleave);
          const uint64_t al = tc::smem_desc(fl + ks * 4096, 2048, 128, tc::kInterleave);
          const uint64_t bh = tc::smem_desc(chi + ks * 2 * NZ * 16, NZ * 16, 128, tc::kInterleave);
          const uint64_t bl = tc::smem_desc(clo + ks * 2 * NZ * 16, NZ * 16, 128, tc::kInterleave);
          tc::mma_tf32(tz[j & 1], ah, bh, idz, ks > 0);
          tc::mma_tf32(tz[j & 1], al, bh, idz, true);
          tc::mma_tf32(tz[j & 1], ah, bl, idz, true);
        }
        tc::commit(&z_full[j & 1]);
      };
      issue_z(0);
      if (n > 1) issue_z(1);
      for (int i = 0; i < n; i++) {
        const int s = i % KT_NS, g = i / KT_FT, b = g & 1;
        mbar_wait(&oh_ready[s], (uint32_t)((i / KT_NS) & 1));
        tc::fence_after();
        if (i % KT_FT == 0 && g >= 2) {
          mbar_wait(&s_empty[b], (uint32_t)(((g >> 1) - 1) & 1));
          tc::fence_after();
        }
        const uint32_t st = smem_u32(sm + s * gm.stage);
        const uint32_t fth = st + gm.o_fth, ftl = st + gm.o_ftl, oht = st + gm.o_oht;
        for (int kk = 0; kk < KT_TILE / 8; kk++) {
          const uint64_t ah = tc::smem_desc(fth + kk * 2 * gm.lbo_ft, gm.lbo_ft, 128, tc::kInterleave);
          const uint64_t al = tc::smem_desc(ftl + kk * 2 * gm.lbo_ft, gm.lbo_ft, 128, tc::kInterleave);
          const uint64_t bo = tc::smem_desc(oht + kk * 2 * gm.lbo_oh, gm.lbo_oh, 128, tc::kInterleave);
          tc::mma_tf32(ts[b], ah, bo, ids, (i % KT_FT) != 0 || kk > 0);
          tc::mma_tf32(ts[b], al, bo, ids, true);
        }
        tc::commit(&empty[s]);
        if (i % KT_FT == KT_FT - 1 || i == n - 1) tc::commit(&s_full[b]);
        if (i + 2 < n) issue_z(i + 2);
      }
    }
    __syncwarp();
  } else {
    // =================== epilogue groups ===================
    const int grp = (warp - 2) >> 2;                 // 0: warps 2-5, 1: warps 6-9
    const int r = 32 * (warp & 3) + lane;            // tile row == TMEM lane
    const uint32_t lane_off = (uint32_t)(32 * (warp & 3)) << 16;
    float lacc = 0.f;
    double lacc64 = 0.0;
    int since = 0;
    for (int i = grp; i < n; i += 2) {
      const int s = i % KT_NS;
      const int64_t p = (t0 + i) * KT_TILE + r;
      const bool valid = p < a.r_T;
      char* st = sm + s * gm.stage;
      float* fs = reinterpret_cast<float*>(st);
      float* fl = reinterpret_cast<float*>(st + gm.o_flo);
      float* fth = reinterpret_cast<float*>(st + gm.o_fth);
      float* ftl = reinterpret_cast<float*>(st + gm.o_ftl);
      const int32_t* fks = reinterpret_cast<const int32_t*>(st + gm.o_fk);
      const uint32_t tbase_w = ((r >> 2) * gm.lbo_ft) / 4 + (r & 3);   // F^T row-r offset
      mbar_wait(&full[s], (uint32_t)((i / KT_NS) & 1));
      // split F into tf32 hi (in place) and the exact remainder lo
      float4 x[16];
#pragma unroll
      for (int c4 = 0; c4 < 16; c4++) {
        if (c4 < C4P) {
          float4 v = *reinterpret_cast<const float4*>(fs + c4 * 512 + r * 4);
          x[c4] = v;
          float4 h, l;
          h.x = __uint_as_float(__float_as_uint(v.x) & 0xffffe000u); l.x = v.x - h.x;
          h.y = __uint_as_float(__float_as_uint(v.y) & 0xffffe000u); l.y = v.y - h.y;
          h.z = __uint_as_float(__float_as_uint(v.z) & 0xffffe000u); l.z = v.z - h.z;
          h.w = __uint_as_float(__float_as_uint(v.w) & 0xffffe000u); l.w = v.w - h.w;
          *reinterpret_cast<float4*>(fs + c4 * 512 + r * 4) = h;
          *reinterpret_cast<float4*>(fl + c4 * 512 + r * 4) = l;
          // transposed (K-major over rows) copies for the sums MMA
          const float hh[4] = {h.x, h.y, h.z, h.w}, ll[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
          for (int e = 0; e < 4; e++) {
            const int c = c4 * 4 + e;
            const uint32_t o = tbase_w + (uint32_t)((c >> 3) * 32 + (c & 7) * 4);
            fth[o] = hh[e];
            ftl[o] = ll[e];
          }
        }
      }
      tc::fence_smem_to_async();
      mbar_arrive(&lo_ready[s]);
      // E terms while the tensor core runs Z
      float eacc[NZ];
#pragma unroll
      for (int j = 0; j < NZ; j++) eacc[j] = 0.f;
      int fkv[MAX_GATHER];
#pragma unroll
      for (int d = 0; d < MAX_GATHER; d++) {
        if (d >= a.ng) break;
        const int f = fks[d * KT_TILE + r];
        fkv[d] = f;
        const float4* er =
            reinterpret_cast<const float4*>(a.E[d] + (f >= 0 ? (int64_t)f : a.rows[d]) * NZ);
#pragma unroll
        for (int q = 0; q < NZ / 4; q++) {
          const float4 ev = er[q];
          eacc[q * 4 + 0] += ev.x;
          eacc[q * 4 + 1] += ev.y;
          eacc[q * 4 + 2] += ev.z;
          eacc[q * 4 + 3] += ev.w;
        }
      }
      float xn = 0.f;
#pragma unroll
      for (int c4 = 0; c4 < 16; c4++)
        if (c4 < C4P)
          xn = fmaf(x[c4].x, x[c4].x, fmaf(x[c4].y, x[c4].y,
               fmaf(x[c4].z, x[c4].z, fmaf(x[c4].w, x[c4].w, xn))));
      // ---- Z row from TMEM
      mbar_wait(&z_full[i & 1], (uint32_t)((i >> 1) & 1));
      tc::fence_after();
      float dv[NZ];
#pragma unroll
      for (int c0 = 0; c0 < NZ; c0 += 16) {
        uint32_t zr[16];
        tc::ld16(tz[i & 1] + lane_off + c0, zr);
        tc::wait_ld();
#pragma unroll
        for (int j = 0; j < 16; j++)
          dv[c0 + j] = fmaf(-2.f, __uint_as_float(zr[j]), cn[c0 + j]) + eacc[c0 + j];
      }
      float v1 = dv[0], v2 = __int_as_float(0x7f800000);
      int al = 0;
#pragma unroll
      for (int j = 1; j < NZ; j++) {
        const bool lt = dv[j] < v1;
        v2 = lt ? v1 : fminf(v2, dv[j]);
        al = lt ? j : al;
        v1 = lt ? dv[j] : v1;
      }
      float el = 0.f;
      if (valid) {
        const float tol = 1e-5f * (xn + cn_max) + 1e-5f * (fabsf(v1) + fminf(fabsf(v2), 3e38f));
        if (!(v2 - v1 > tol)) {   // near tie: decide from direct fp32 differences
          uint32_t cand = 0;
#pragma unroll
          for (int j = 0; j < NZ; j++)
            if (j < k && dv[j] - v1 <= tol) cand |= 1u << j;
          float bd = __int_as_float(0x7f800000);
          int bj = 0;
          while (cand) {
            const int j = __ffs(cand) - 1;
            cand &= cand - 1;
            const float4* cr = reinterpret_cast<const float4*>(cf + j * CFP);
            float dj = 0.f;
#pragma unroll
            for (int c4 = 0; c4 < 16; c4++)
              if (c4 < C4P) {
                const float4 c = cr[c4];
                const float d0 = x[c4].x - c.x, d1 = x[c4].y - c.y;
                const float d2 = x[c4].z - c.z, d3 = x[c4].w - c.w;
                dj = fmaf(d0, d0, fmaf(d1, d1, fmaf(d2, d2, fmaf(d3, d3, dj))));
              }
            float ej = 0.f;
#pragma unroll
            for (int jj = 0; jj < NZ; jj++) ej = jj == j ? eacc[jj] : ej;
            dj += ej;
            if (dj < bd) {
              bd = dj;
              bj = j;
            }
          }
          al = bj;
        }
#pragma unroll
        for (int jj = 0; jj < NZ; jj++) el = jj == al ? eacc[jj] : el;
        const float4* cr = reinterpret_cast<const float4*>(cf + al * CFP);
        float l = el;
#pragma unroll
        for (int c4 = 0; c4 < 16; c4++)
          if (c4 < C4P) {
            const float4 c = cr[c4];
            const float d0 = x[c4].x - c.x, d1 = x[c4].y - c.y;
            const float d2 = x[c4].z - c.z, d3 = x[c4].w - c.w;
            l = fmaf(d0, d0, fmaf(d1, d1, fmaf(d2, d2, fmaf(d3, d3, l))));
          }
        lacc += l;
      } else {
        al = -1;
      }
      // I_d^T A counters
#pragma unroll
      for (int d = 0; d < MAX_GATHER; d++) {
        if (d >= a.ng) break;
        const int f = fkv[d];
        const int key = (valid && f >= 0) ? f * NZ + al : -1 - lane;
        if (d == a.sort_g) {
          const unsigned mask = __match_any_sync(0xffffffffu, key);
          if (key >= 0 && (__ffs(mask) - 1) == lane) atomicAdd(&a.cnt[d][key], __popc(mask));
        } else if (key >= 0) {
          atomicAdd(&a.cnt[d][key], 1);
        }
      }
      if (a.assign && valid) a.assign[p] = al;
      // one-hot row, transposed (K-major over rows: [row chunk][cluster][4])
      float* oht = reinterpret_cast<float*>(st + gm.o_oht);
      const uint32_t ob = ((r >> 2) * gm.lbo_oh) / 4 + (r & 3);
#pragma unroll
      for (int j = 0; j < NZ; j++) oht[ob + (j >> 3) * 32 + (j & 7) * 4] = al == j ? 1.f : 0.f;
      tc::fence_smem_to_async();
      tc::fence_before();
      mbar_arrive(&oh_ready[s]);
      if (++since == 4) {
        lacc64 += (double)lacc;
        lacc = 0.f;
        since = 0;
      }
    }
    lacc64 += (double)lacc;
    // fixed-order warp reduction of the loss
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lacc64 += __shfl_xor_sync(0xffffffffu, lacc64, o);
    if (lane == 0) lsum_w[warp] = lacc64;
  }
  if (warp < 2 && lane == 0) lsum_w[warp] = 0.0;
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  // CTA partial: [NZ x SC] sums (rows = clusters; count at column pf) | loss
  double* out = a.part + (int64_t)blockIdx.x * ((int64_t)NZ * SC + 1);
  for (int i = tid; i < NZ * SC; i += blockDim.x) {
    const int j = i / SC, c = i - j * SC;
    out[i] = c < 32 ? sums64[c * NZ + j] : 0.0;
  }
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < KT_THREADS / 32; w++) s += lsum_w[w];
    out[NZ * SC] = s;
  }
  __syncthreads();
  if (warp == 0) tc::dealloc(tmem, 128);
}
