// K2 for SPARSE stream blocks: the GLM fact-row pass
// over a CSR copy of the stream block F (device row order).  Per nonzero
// only its value (fp32) and column (uint16) are read, so at density rho the
// pass moves ~6 rho pf + 8 bytes per row of F instead of 4 pf.
//
// One warp owns a contiguous range of 32-row units (lane = row).  Per row:
//   z = sum_nz v w_F[col] + sum_d q_d[fk_d]        (w_F in smem)
//   r = z - y | sigmoid(z) - y, loss
//   grad_F[col] += r v  into a LANE-PRIVATE smem row (deterministic: the
//                       32 lane rows are folded in a fixed order every
//                       FW_FLUSH units, fp32 -> fp64)
//   bins_sort[fk] += r  (the dense pass's warp segmented scan + carries)
// (included inside namespace flb by glm.cu)
#pragma once

struct GlmCsrArgs {
  const int64_t* rp;         // r_pad + 1 row extents (device order)
  const uint16_t* col;       // nnz stream-block columns
  const float* val;          // nnz values
  int pf;                    // gradient width (stream pitch)
  const void* y;
  int64_t r_T, nunits;       // units of 32 device rows
  int ng, sort_g;
  const int32_t* fk[MAX_GATHER];
  const float* q[MAX_GATHER];
  float* bins;
  float* resid;
  const float* wF;
  double* part;              // gridDim.x x (pf + 1)
  WarpCarry* carry;          // gridDim.x * FW_WARPS
  GlmState* state;
};

constexpr int CSR_MAXP = 128;   // stream pitch handled by the sparse pass

template <int MODEL>
__global__ void __launch_bounds__(FW_WARPS * 32) k_glm_fact_csr(GlmCsrArgs a) {
  // smem: w_F | per-warp lane-private gradient rows (32 x GP).  Measured
  // variants (profiles/r01_glm_csr.txt): this direct-load version beat a
  // register-prefetch pipeline and a per-warp TMA ring of small bulk copies.
  extern __shared__ __align__(16) float csr_sm[];
  __shared__ double gsum[FW_WARPS][CSR_MAXP];
  __shared__ double lsum[FW_WARPS];
  __shared__ int is_last;
  const int pf = a.pf, GP = pf | 1;                          // odd pitch: conflict-free
  float* w_s = csr_sm;
  float* g_s = csr_sm + round_up(pf, 4) + (threadIdx.x >> 5) * 32 * GP;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * FW_WARPS + warp;
  const int64_t NW = (int64_t)gridDim.x * FW_WARPS;
  const int64_t base = a.nunits / NW, rem = a.nunits % NW;
  const int64_t u0 = gw * base + min64(gw, rem);
  const int64_t cnt = base + (gw < rem ? 1 : 0);
  const int64_t W0 = u0 * 32;
  const int64_t W1 = min64((u0 + cnt) * 32, a.r_T);
  const bool has_sort = a.sort_g >= 0;
  const int32_t* fks = has_sort ? a.fk[a.sort_g] : nullptr;

  for (int j = threadIdx.x; j < pf; j += blockDim.x) w_s[j] = a.wF[j];
  for (int j = lane; j < CSR_MAXP; j += 32) gsum[warp][j] = 0.0;
  for (int j = lane; j < 32 * GP; j += 32) g_s[j] = 0.f;
  if (lane == 0) lsum[warp] = 0.0;
  __syncthreads();

  int head_key = -1;
  if (has_sort && cnt > 0 && W0 > 0 && W0 < a.r_T) {
    int k0 = fks[W0];
    if (k0 >= 0 && fks[W0 - 1] == k0) head_key = k0;
  }
  bool head_open = head_key >= 0;
  float head_val = 0.f;
  int ck = -1;
  float cv = 0.f;
  float lacc = 0.f;
  float* grow = g_s + lane * GP;

  auto flush = [&]() {
    __syncwarp();
    for (int c = lane; c < pf; c += 32) {       // fixed lane order per column
      float s = 0.f;
      for (int l = 0; l < 32; l++) {
        s += g_s[l * GP + c];
        g_s[l * GP + c] = 0.f;
      }
      gsum[warp][c] += (double)s;
    }
    __syncwarp();
    float v = lacc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) lsum[warp] += (double)v;
    lacc = 0.f;
  };

  for (int64_t i = 0; i < cnt; i++) {
    const int64_t p = (u0 + i) * 32 + lane;
    const bool valid = p < a.r_T;
    const int64_t e0 = a.rp[p], e1 = a.rp[p + 1];
    int key = has_sort ? fks[p] : -1;
    float gq = 0.f;
    for (int d = 0; d < a.ng; d++) {
      const int32_t fk = (d == a.sort_g) ? key : a.fk[d][p];
      if (fk >= 0) gq += __ldg(a.q[d] + fk);
    }
    float yv;
    if (MODEL == 0) yv = reinterpret_cast<const float*>(a.y)[p];
    else yv = (float)reinterpret_cast<const uint8_t*>(a.y)[p];
    float z = 0.f;
    for (int64_t e = e0; e < e1; e++) z = fmaf(__ldg(a.val + e), w_s[__ldg(a.col + e)], z);
    z += gq;
    float r, l;
    if (MODEL == 0) {
      r = z - yv;
      l = 0.5f * r * r;
    } else {
      float ex = __expf(-fabsf(z));
      float sp = log1pf(ex);
      const float inv = __frcp_rn(1.f + ex);
      float pr = z >= 0.f ? inv : ex * inv;
      r = pr - yv;
      float lp = z >= 0.f ? sp : sp - z;
      float lq = z >= 0.f ? sp + z : sp;
      l = yv != 0.f ? fminf(lp, kLogClip) : fminf(lq, kLogClip);
    }
    if (!valid) {
      r = 0.f;
      l = 0.f;
      key = -1;
    }
    lacc += l;
    for (int64_t e = e0; e < e1; e++) {
      const int c = __ldg(a.col + e);
      grow[c] = fmaf(r, __ldg(a.val + e), grow[c]);
    }
    if (a.resid && valid) a.resid[p] = r;
    if (has_sort) {   // segmented sum of r by FK (as k_glm_fact_w)
      float v = r;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        float vu = __shfl_up_sync(0xffffffffu, v, off);
        int ku = __shfl_up_sync(0xffffffffu, key, off);
        if (lane >= off && ku == key) v += vu;
      }
      if (key >= 0 && key == ck) v += cv;
      const int k0 = __shfl_sync(0xffffffffu, key, 0);
      if (ck >= 0 && k0 != ck) {
        if (head_open && ck == head_key) {
          head_val = cv;
          head_open = false;
        } else if (lane == 0) {
          a.bins[ck] = cv;
        }
      }
      const int kn = __shfl_down_sync(0xffffffffu, key, 1);
      const bool end = lane < 31 && key >= 0 && kn != key;
      const bool eh = end && head_open && key == head_key;
      const unsigned bm = __ballot_sync(0xffffffffu, eh);
      if (bm) {
        head_val = __shfl_sync(0xffffffffu, v, __ffs(bm) - 1);
        head_open = false;
      }
      if (end && !eh) a.bins[key] = v;
      ck = __shfl_sync(0xffffffffu, key, 31);
      cv = __shfl_sync(0xffffffffu, v, 31);
    }
    if ((i % FW_FLUSH) == FW_FLUSH - 1) flush();
  }
  flush();

  if (has_sort) {
    WarpCarry c;
    c.head_key = -1;
    c.tail_key = -1;
    c.through = 0;
    c.pad = 0;
    c.head_val = 0.0;
    c.tail_val = 0.0;
    if (cnt > 0) {
      if (ck >= 0) {
        const bool cont = W1 < a.r_T && fks[W1] == ck;
        if (head_open && ck == head_key) {
          head_val = cv;
          head_open = false;
          c.head_key = ck;
          c.through = cont ? 1 : 0;
        } else if (cont) {
          c.tail_key = ck;
          c.tail_val = (double)cv;
        } else if (lane == 0) {
          a.bins[ck] = cv;
        }
      }
      if (!head_open && head_key >= 0) {
        c.head_key = head_key;
        c.head_val = (double)head_val;
      }
    }
    if (lane == 0) a.carry[gw] = c;
  }
  __syncthreads();
  double* out = a.part + (int64_t)blockIdx.x * (pf + 1);
  for (int t = threadIdx.x; t <= pf; t += blockDim.x) {
    double sum = 0.0;
    if (t < pf)
      for (int w2 = 0; w2 < FW_WARPS; w2++) sum += gsum[w2][t];
    else
      for (int w2 = 0; w2 < FW_WARPS; w2++) sum += lsum[w2];
    out[t] = sum;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = atomicAdd(&a.state->done_fact, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  if (has_sort) {
    volatile WarpCarry* cr = a.carry;
    for (int64_t c = threadIdx.x; c < NW; c += blockDim.x) {
      int K = cr[c].tail_key;
      if (K < 0) continue;
      double total = cr[c].tail_val;
      for (int64_t c2 = c + 1; c2 < NW; c2++) {
        if (cr[c2].head_key != K) break;
        total += cr[c2].head_val;
        if (!cr[c2].through) break;
      }
      a.bins[K] = (float)total;
    }
  }
  if (threadIdx.x == 0) a.state->done_fact = 0;
}

// density probe: nonzeros of the whole stream block (coalesced float4 reads,
// one atomic per warp) -- decides whether the CSR copy below is built at all
__global__ void k_nnz_total(const float4* __restrict__ F4, int64_t n4,
                            unsigned long long* __restrict__ total) {
  unsigned n = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n4; i += 4 * stride) {   // 4 independent loads in flight
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; u++) v[u] = __ldcs(F4 + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; u++)
      n += (v[u].x != 0.f) + (v[u].y != 0.f) + (v[u].z != 0.f) + (v[u].w != 0.f);
  }
  for (; i < n4; i += stride) {
    const float4 v = F4[i];
    n += (v.x != 0.f) + (v.y != 0.f) + (v.z != 0.f) + (v.w != 0.f);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  if ((threadIdx.x & 31) == 0 && n) atomicAdd(total, (unsigned long long)n);
}

// CSR copy of the stream block: per-row nonzero counts, scan, compaction
__global__ void k_csr_count(const float* __restrict__ F, int64_t r_pad, int pf,
                            int64_t* __restrict__ cnt) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < r_pad;
       r += (int64_t)gridDim.x * blockDim.x) {
    int n = 0;
    for (int c = 0; c < pf; c++) n += F[r * pf + c] != 0.f;
    cnt[r] = n;
  }
}
__global__ void k_csr_fill(const float* __restrict__ F, int64_t r_pad, int pf,
                           const int64_t* __restrict__ rp, uint16_t* __restrict__ col,
                           float* __restrict__ val) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < r_pad;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t e = rp[r];
    for (int c = 0; c < pf; c++) {
      const float v = F[r * pf + c];
      if (v != 0.f) {
        col[e] = (uint16_t)c;
        val[e] = v;
        e++;
      }
    }
  }
}
