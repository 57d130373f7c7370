// Fused gradient descent for linear / logistic regression over a factorized
// table (reference trainers.py:138-195 on top of ops.py:219-271).
//
// One GD iteration = three kernels (plus one all-reduce between K3 and the
// update when the fact rows are sharded over several GPUs):
//
//  K1 k_glm_dim_q     q_d[j]   = S_d[j,:] . w_d            (S_d streamed once)
//  K2 k_glm_fact      per device row p (one pass over F, TMA-staged tiles):
//                       z  = F[p,:] . w_F + sum_d q_d[fk_d[p]]
//                       r  = z - y (linreg) | sigmoid(z) - y (logreg)
//                       loss partial, grad_F partial += r F[p,:]
//                       bins_sort[fk_sort[p]] += r  (contiguous segmented sum;
//                       rows are in FK order, so no atomics)
//                       resid[p] = r  (only if an unsorted gathered source exists)
//  K3 k_glm_dim_t     grad_d = S_d^T bins_d (S_d streamed again), then the last
//                     CTA reduces all per-CTA fp64 partials in a fixed order
//                     and (single GPU) applies w <- w - lr grad.
//
// Algorithmic HBM bytes per iteration:
//   4 r_T pf + 4 r_T n_gather + b_y r_T + sum_d 2 * 4 r_d pitch_d (+ 4 r_T if resid)
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>

#include "internal.h"
#include "reduce.cuh"
#include "tc05.cuh"

namespace flb {

struct CarryRec {
  int head_key;   // key of the CTA's first segment if it began before the CTA range
  int tail_key;   // key of the CTA's last segment if it began inside and continues
  int through;    // the whole CTA range is one segment that continues past its end
  int pad;
  double head_val;
  double tail_val;
};

struct GlmState {
  int it;          // iterations whose update has been applied
  int done_fact;   // last-block-done counters
  int done_dim;
  int pad;
};

struct GlmFactArgs {
  const float* F;
  int pf, c4;
  const void* y;
  int64_t r_T, ntiles;
  int ng, sort_g;
  const int32_t* fk[MAX_GATHER];
  const float* q[MAX_GATHER];
  float* bins;
  float* resid;
  const float* wF;
  double* part;          // gridDim.x x (pf + 1)
  CarryRec* carry;       // gridDim.x
  GlmState* state;
  uint32_t stage_bytes, off_fk, off_y;
  int nst;
};

struct DimArgs {
  int ng;
  const float* S[MAX_GATHER];
  int pitch[MAX_GATHER];
  int64_t rows[MAX_GATHER];
  int nblk[MAX_GATHER];          // CTAs used for source d (<= gridDim.x)
  const float* w[MAX_GATHER];    // fp32 w_d (pitch entries)
  float* q[MAX_GATHER];          // K1 output
  // K3 inputs
  const float* bins[MAX_GATHER]; // sorted source: bins; else null
  const int64_t* grp_ptr[MAX_GATHER];
  const int32_t* grp_rows[MAX_GATHER];
  const float* resid;
  double* part[MAX_GATHER];      // nblk x pitch
  uint32_t stage_bytes;
  int nst;
  float* bins_zero;              // K1 zeroes the sort source's bins for this iteration
  int64_t bins_n;
};

constexpr int kGlmGraphIters = 8;

struct UpdateArgs {
  int c_T, pf, ng;
  double lr;
  const int32_t* f_tcol;
  const int32_t* d_tcol[MAX_GATHER];
  int pitch[MAX_GATHER];
  float* wF;
  float* wd[MAX_GATHER];
  double* w64;
  double* red;        // c_T + 1
  double* loss_hist;
  int loss_cap;
  GlmState* state;
  // reduction inputs (K3 last block)
  const double* part_fact;
  int nblk_fact;
  double* red_fact;   // pf + 1: the fact partials, reduced early by K3's first CTAs
  const double* part_dim[MAX_GATHER];
  int nblk_dim[MAX_GATHER];
};

__device__ __forceinline__ float softplus(float x) {
  // log(1 + e^x), stable
  return x > 0.f ? x + log1pf(expf(-x)) : log1pf(expf(x));
}

// -log(clip(p, 1e-12, 1 - 1e-12)) saturates at this value (trainers.py:185-186)
__device__ __constant__ float kLogClip = 27.631021115928547f;

// ---------------------------------------------------------------------------
// K1: q_d = S_d w_d, thread per row from TMA-staged tiles
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(NTHREADS) k_glm_dim_q(DimArgs a) {
  extern __shared__ __align__(128) char smem[];
  __shared__ uint64_t bar[4];
  __shared__ float4 w4[64];
  const int d = blockIdx.y;
  const bool active = d < a.ng && (int)blockIdx.x < a.nblk[d];
  const int tid = threadIdx.x;
  const int pitch = active ? a.pitch[d] : 4, c4 = pitch / 4;
  const int64_t rows = active ? a.rows[d] : 0;
  const int64_t ntiles = ceil_div(rows, TILE);
  const int nb = active ? a.nblk[d] : 1;
  const int64_t base = ntiles / nb, rem = ntiles % nb;
  const int64_t t0 = blockIdx.x * base + min64(blockIdx.x, rem);
  const int64_t cnt = active ? base + (blockIdx.x < rem ? 1 : 0) : 0;
  const uint32_t tile_bytes = TILE * pitch * 4;
  // the CTA walks its tile range BACKWARDS: k_glm_dim_t (the previous
  // kernel) walked the same ranges forwards, so the most recently read S_d
  // tiles -- still in L2 -- come first
  auto tile_of = [&](int64_t i) { return t0 + (cnt - 1 - i); };
  // S_d is immutable: its first tiles stream in before the dependency wait
  if (tid == 0 && active) {
    for (int s = 0; s < a.nst; s++) mbar_init(&bar[s], 1);
    fence_mbar_init();
    for (int s = 0; s < a.nst && s < cnt; s++) {
      mbar_arrive_expect_tx(&bar[s], tile_bytes);
      bulk_g2s(smem + s * a.stage_bytes, a.S[d] + tile_of(s) * TILE * (int64_t)pitch, tile_bytes,
               &bar[s]);
    }
  }
  pdl_wait();      // w_d (previous update) final; previous dim_t done with bins
  pdl_trigger();
  if (a.bins_zero) {
    const int64_t nt = (int64_t)gridDim.x * gridDim.y * blockDim.x;
    for (int64_t i = ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * blockDim.x + tid;
         i < a.bins_n; i += nt)
      a.bins_zero[i] = 0.f;
  }
  if (!active) return;
  for (int j = tid; j < c4; j += NTHREADS) w4[j] = reinterpret_cast<const float4*>(a.w[d])[j];
  __syncthreads();
  for (int64_t i = 0; i < cnt; i++) {
    const int s = (int)(i % a.nst);
    mbar_wait(&bar[s], (uint32_t)((i / a.nst) & 1));
    const float4* tile = reinterpret_cast<const float4*>(smem + s * a.stage_bytes);
    float z = 0.f;
    for (int j = 0; j < c4; j++) {
      float4 v = tile[tid * c4 + j];
      float4 w = w4[j];
      z = fmaf(v.x, w.x, z);
      z = fmaf(v.y, w.y, z);
      z = fmaf(v.z, w.z, z);
      z = fmaf(v.w, w.w, z);
    }
    int64_t row = tile_of(i) * TILE + tid;
    if (row < rows) a.q[d][row] = z;
    __syncthreads();
    if (tid == 0 && i + a.nst < cnt) {
      fence_proxy_async();
      mbar_arrive_expect_tx(&bar[s], tile_bytes);
      bulk_g2s(smem + s * a.stage_bytes, a.S[d] + tile_of(i + a.nst) * TILE * (int64_t)pitch,
               tile_bytes, &bar[s]);
    }
  }
}

// ---------------------------------------------------------------------------
// K2: the fact-row pass
// ---------------------------------------------------------------------------
template <int MODEL>
__global__ void __launch_bounds__(NTHREADS, 2) k_glm_fact(GlmFactArgs a) {
  extern __shared__ __align__(128) char smem[];
  __shared__ uint64_t bar[4];
  __shared__ float4 w4[64];
  __shared__ float r_s[TILE];
  __shared__ int key_first[8], key_last[8];
  __shared__ float v_last[8];
  __shared__ int run_key[2];
  __shared__ float run_val[2];
  __shared__ int head_key_s, head_open_s, head_rec_key;
  __shared__ float head_rec_val;
  __shared__ double red_s[NTHREADS];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c4 = a.c4;
  const int64_t G = gridDim.x;
  const int64_t base = a.ntiles / G, rem = a.ntiles % G;
  const int64_t t0 = blockIdx.x * base + min64(blockIdx.x, rem);
  const int64_t cnt = base + (blockIdx.x < rem ? 1 : 0);
  const int64_t R0 = t0 * TILE, R1 = min64((t0 + cnt) * TILE, a.r_T);
  const uint32_t f_bytes = TILE * c4 * 16;
  const uint32_t y_bytes = MODEL == 1 ? TILE : TILE * 4;
  const bool has_sort = a.sort_g >= 0;
  const int32_t* fks = has_sort ? a.fk[a.sort_g] : nullptr;
  uint32_t tx_bytes = f_bytes + y_bytes + (has_sort ? TILE * 4 : 0);

  for (int j = tid; j < c4; j += NTHREADS) w4[j] = reinterpret_cast<const float4*>(a.wF)[j];
  if (tid == 0) {
    for (int s = 0; s < a.nst; s++) mbar_init(&bar[s], 1);
    fence_mbar_init();
    run_key[0] = run_key[1] = -1;
    run_val[0] = run_val[1] = 0.f;
    int hk = -1;
    if (has_sort && cnt > 0 && R0 > 0 && R0 < a.r_T) {
      int k0 = fks[R0];
      if (k0 >= 0 && fks[R0 - 1] == k0) hk = k0;
    }
    head_key_s = hk;
    head_open_s = hk >= 0;
    head_rec_key = -1;
    head_rec_val = 0.f;
  }
  __syncthreads();

  auto issue = [&](int s, int64_t tile) {
    char* st = smem + s * a.stage_bytes;
    mbar_arrive_expect_tx(&bar[s], tx_bytes);
    bulk_g2s(st, a.F + tile * TILE * (int64_t)a.pf, f_bytes, &bar[s]);
    bulk_g2s(st + a.off_y, reinterpret_cast<const char*>(a.y) + tile * (int64_t)y_bytes, y_bytes,
             &bar[s]);
    if (has_sort) bulk_g2s(st + a.off_fk, fks + tile * TILE, TILE * 4, &bar[s]);
  };
  if (tid == 0)
    for (int s = 0; s < a.nst && s < cnt; s++) issue(s, t0 + s);

  // phase-B mapping: thread -> (float4 column j, row group g)
  const int Gr = NTHREADS / c4;
  const bool pb = tid < Gr * c4;
  const int pj = tid % c4, pg = tid / c4;
  double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0, lossd = 0;
  const int head_key = head_key_s;

  for (int64_t i = 0; i < cnt; i++) {
    const int s = (int)(i % a.nst);
    const int cur = (int)(i & 1), prev = cur ^ 1;
    mbar_wait(&bar[s], (uint32_t)((i / a.nst) & 1));
    const char* st = smem + s * a.stage_bytes;
    const float4* Ft = reinterpret_cast<const float4*>(st);
    const int64_t p = (t0 + i) * TILE + tid;
    const bool valid = p < a.r_T;
    // ---- phase A: z, residual, loss
    float z = 0.f;
    for (int j = 0; j < c4; j++) {
      float4 v = Ft[tid * c4 + j];
      float4 w = w4[j];
      z = fmaf(v.x, w.x, z);
      z = fmaf(v.y, w.y, z);
      z = fmaf(v.z, w.z, z);
      z = fmaf(v.w, w.w, z);
    }
    int key = -1;
    if (has_sort) key = reinterpret_cast<const int32_t*>(st + a.off_fk)[tid];
    for (int d = 0; d < a.ng; d++) {
      int32_t fk = (d == a.sort_g) ? key : a.fk[d][p];
      if (fk >= 0) z += __ldg(a.q[d] + fk);
    }
    float r, l;
    if (MODEL == 0) {
      float yv = reinterpret_cast<const float*>(st + a.off_y)[tid];
      r = z - yv;
      l = 0.5f * r * r;
    } else {
      float yv = (float)reinterpret_cast<const uint8_t*>(st + a.off_y)[tid];
      float pr = 1.f / (1.f + expf(-z));
      r = pr - yv;
      // -(y log p + (1-y) log(1-p)) with the reference's clip
      l = yv != 0.f ? fminf(softplus(-z), kLogClip) : fminf(softplus(z), kLogClip);
    }
    if (!valid) {
      r = 0.f;
      l = 0.f;
      key = -1;
    }
    r_s[tid] = r;
    lossd += (double)l;
    if (a.resid) a.resid[p] = r;
    // ---- segmented sum of r by sorted key (warp scan)
    float v = r;
    if (has_sort) {
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        float vu = __shfl_up_sync(0xffffffffu, v, off);
        int ku = __shfl_up_sync(0xffffffffu, key, off);
        if (lane >= off && ku == key) v += vu;
      }
      if (lane == 0) key_first[warp] = key;
      if (lane == 31) {
        key_last[warp] = key;
        v_last[warp] = v;
      }
    }
    __syncthreads();
    // ---- segment ends: resolve carries and emit
    if (has_sort) {
      // the previous tile's last segment is complete unless row 0 continues it
      if (tid == 0) {
        int pk = run_key[prev];
        if (pk >= 0 && pk != key) {
          if (head_open_s && pk == head_key) {
            head_rec_key = pk;
            head_rec_val = run_val[prev];
            head_open_s = 0;
          } else {
            a.bins[pk] = run_val[prev];
          }
        }
      }
      int kn = __shfl_down_sync(0xffffffffu, key, 1);
      // a segment ends where the next ROW's key differs: for lane 31 that is
      // lane 0 of the next warp; row 255 closes the tile (running carry)
      if (lane == 31) kn = warp < NTHREADS / 32 - 1 ? key_first[warp + 1] : ~key;
      bool end = kn != key;
      if (end && key >= 0) {
        float total = v;
        if (key_first[warp] == key) {
          bool reached_start = true;
          for (int w2 = warp - 1; w2 >= 0; w2--) {
            if (key_last[w2] != key) {
              reached_start = false;
              break;
            }
            total += v_last[w2];
            if (key_first[w2] != key) {
              reached_start = false;
              break;
            }
          }
          if (reached_start && run_key[prev] == key) total += run_val[prev];
        }
        if (tid == NTHREADS - 1) {
          run_key[cur] = key;
          run_val[cur] = total;
        } else if (head_open_s && key == head_key) {
          head_rec_key = key;
          head_rec_val = total;
          head_open_s = 0;
        } else {
          a.bins[key] = total;
        }
      } else if (tid == NTHREADS - 1) {
        run_key[cur] = -1;
        run_val[cur] = 0.f;
      }
    }
    // ---- phase B: grad_F += r * F rows (column-parallel, float4)
    if (pb) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int row = pg; row < TILE; row += Gr) {
        float rr = r_s[row];
        float4 v4 = Ft[row * c4 + pj];
        acc.x = fmaf(rr, v4.x, acc.x);
        acc.y = fmaf(rr, v4.y, acc.y);
        acc.z = fmaf(rr, v4.z, acc.z);
        acc.w = fmaf(rr, v4.w, acc.w);
      }
      acc0 += acc.x;
      acc1 += acc.y;
      acc2 += acc.z;
      acc3 += acc.w;
    }
    __syncthreads();
    if (tid == 0 && i + a.nst < cnt) {
      fence_proxy_async();
      issue(s, t0 + i + a.nst);
    }
  }

  // ---- CTA end: final running segment -> carry record
  __syncthreads();
  if (tid == 0 && has_sort) {
    CarryRec c;
    c.head_key = -1;
    c.tail_key = -1;
    c.through = 0;
    c.pad = 0;
    c.head_val = 0.0;
    c.tail_val = 0.0;
    if (cnt > 0) {
      const int last = (int)((cnt - 1) & 1);
      int K = run_key[last];
      float V = run_val[last];
      if (K >= 0) {
        bool cont = R1 < a.r_T && fks[R1] == K;
        if (head_open_s && K == head_key) {
          head_rec_key = K;
          head_rec_val = V;
          head_open_s = 0;
          c.through = cont ? 1 : 0;
        } else if (cont) {
          c.tail_key = K;
          c.tail_val = (double)V;
        } else {
          a.bins[K] = V;
        }
      }
      c.head_key = head_rec_key;
      c.head_val = (double)head_rec_val;
    }
    a.carry[blockIdx.x] = c;
  }
  // ---- CTA partials (fixed-order reductions)
  double* red = red_s;
  const int pfc = c4 * 4;
  double* out = a.part + blockIdx.x * (int64_t)(pfc + 1);
  // gradient: sum over groups for each of the pfc columns
  for (int comp = 0; comp < 4; comp++) {
    double val = comp == 0 ? acc0 : comp == 1 ? acc1 : comp == 2 ? acc2 : acc3;
    __syncthreads();
    red[tid] = pb ? val : 0.0;
    __syncthreads();
    if (tid < c4) {
      double sum = 0.0;
      for (int g = 0; g < Gr; g++) sum += red[g * c4 + tid];
      out[tid * 4 + comp] = sum;
    }
  }
  // loss
  double ls = warp_sum(lossd);
  __syncthreads();
  if (lane == 0) red[warp] = ls;
  __syncthreads();
  if (tid == 0) {
    double sum = 0.0;
    for (int w2 = 0; w2 < NTHREADS / 32; w2++) sum += red[w2];
    out[pfc] = sum;
  }
  // ---- last CTA: stitch the segments that span CTAs (fixed order)
  __threadfence();
  __syncthreads();
  __shared__ int is_last;
  if (tid == 0) is_last = atomicAdd(&a.state->done_fact, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  if (has_sort) {
    volatile CarryRec* cr = a.carry;
    for (int c = tid; c < (int)gridDim.x; c += NTHREADS) {
      int K = cr[c].tail_key;
      if (K < 0) continue;
      double total = cr[c].tail_val;
      for (int c2 = c + 1; c2 < (int)gridDim.x; c2++) {
        if (cr[c2].head_key != K) break;
        total += cr[c2].head_val;
        if (!cr[c2].through) break;
      }
      a.bins[K] = (float)total;
    }
  }
  if (tid == 0) a.state->done_fact = 0;
}

__device__ void glm_apply_update(const UpdateArgs& u);
#include "glm_fact_warp.cuh"
#include "glm_fact_csr.cuh"

// solo iteration check: the widest dimension-row range one fact-pass CTA
// references (it must fit the CTA's q staging, FW_QCAP entries)
__global__ void k_glm_solo_span(const int32_t* __restrict__ fks, int64_t n_neg, int64_t r_T,
                                int64_t nunits, int rw, int nblk, int* __restrict__ out) {
  const int64_t NW = (int64_t)nblk * FW_WARPS;
  const int64_t base = nunits / NW, rem = nunits % NW;
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nblk; b += gridDim.x * blockDim.x) {
    const int64_t cw0 = (int64_t)b * FW_WARPS, cw1 = cw0 + FW_WARPS;
    const int64_t cu0 = cw0 * base + min64(cw0, rem), cu1 = cw1 * base + min64(cw1, rem);
    const int64_t rlo = max64(cu0 * rw, n_neg), rhi = min64(cu1 * rw, r_T) - 1;
    if (rlo <= rhi) atomicMax(out, fks[rhi] - fks[rlo] + 1);
  }
}
// auto-selection threshold of the CSR pass: it must beat the dense pass,
// which streams F at the HBM roofline (profiles/r01_glm_csr.txt)
constexpr double kCsrAutoDensity = 0.0;

// ---------------------------------------------------------------------------
// update: w <- w - lr * red; loss_hist[it] = red[c_T]; refresh fp32 copies
// ---------------------------------------------------------------------------
__device__ void glm_apply_update(const UpdateArgs& u) {
  const int tid = threadIdx.x;
  const int it = u.state->it;
  if (tid == 0 && it < u.loss_cap) u.loss_hist[it] = u.red[u.c_T];
  for (int c = tid; c < u.c_T; c += blockDim.x) u.w64[c] -= u.lr * u.red[c];
  __syncthreads();
  for (int j = tid; j < u.pf; j += blockDim.x) {
    int tc = u.f_tcol[j];
    u.wF[j] = tc >= 0 ? (float)u.w64[tc] : 0.f;
  }
  for (int d = 0; d < u.ng; d++)
    for (int c = tid; c < u.pitch[d]; c += blockDim.x) {
      int tc = u.d_tcol[d][c];
      u.wd[d][c] = tc >= 0 ? (float)u.w64[tc] : 0.f;
    }
  if (tid == 0) u.state->it = it + 1;
}

// the fact-pass partials are final once K3 passes its dependency wait: CTA
// b (flat index) reduces elements b, b + #CTAs, ... of the pf + 1 with its
// last warp, in parallel
// with the S_d streaming, so the serial last-CTA step is left with the
// dimension partials only
__device__ void glm_reduce_fact_early(const UpdateArgs& u) {
  if ((threadIdx.x >> 5) != (int)(blockDim.x >> 5) - 1) return;
  const int nct = gridDim.x * gridDim.y;
  for (int e = blockIdx.y * gridDim.x + blockIdx.x; e <= u.pf; e += nct) {
    const double s = warp_sum_strided(u.part_fact + e, u.pf + 1, u.nblk_fact, threadIdx.x & 31);
    if ((threadIdx.x & 31) == 0) u.red_fact[e] = s;
  }
}

__device__ void glm_reduce_all(const UpdateArgs& u) {
  // one warp per output element, two elements per step (fixed-order lane
  // sums + a fixed xor tree: deterministic); the fact elements were reduced
  // by glm_reduce_fact_early
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int c = tid; c <= u.c_T; c += blockDim.x) u.red[c] = 0.0;
  __syncthreads();
  for (int e = tid; e <= u.pf; e += blockDim.x) {
    const int dst = e == u.pf ? u.c_T : u.f_tcol[e];
    if (dst >= 0) u.red[dst] = u.red_fact[e];
  }
  int total = 0;
  for (int d = 0; d < u.ng; d++) total += u.pitch[d];
  auto locate = [&](int e, const double** base, int* stride, int* nblk, int* dst) {
    int c = e, d = 0;
    while (c >= u.pitch[d]) c -= u.pitch[d++];
    *base = u.part_dim[d] + c;
    *stride = u.pitch[d];
    *nblk = u.nblk_dim[d];
    *dst = u.d_tcol[d][c];
  };
  for (int e = 2 * warp; e < total; e += 2 * nw) {
    const double *b0, *b1 = nullptr;
    int st0, n0, dst0, st1 = 1, n1 = 0, dst1 = -1;
    locate(e, &b0, &st0, &n0, &dst0);
    if (e + 1 < total) locate(e + 1, &b1, &st1, &n1, &dst1);
    if (dst0 < 0) n0 = 0;
    if (dst1 < 0) n1 = 0;
    double s0, s1;
    warp_sum_strided2(b0, st0, n0, b1 ? b1 : b0, st1, n1, lane, &s0, &s1);
    if (lane == 0) {
      if (dst0 >= 0) u.red[dst0] = s0;
      if (dst1 >= 0) u.red[dst1] = s1;
    }
  }
  __syncthreads();
}

// K3: grad_d = S_d^T bins_d, then last CTA reduces (and optionally updates)
__global__ void __launch_bounds__(NTHREADS) k_glm_dim_t(DimArgs a, UpdateArgs u, int fuse_update) {
  extern __shared__ __align__(128) char smem[];
  __shared__ uint64_t bar[4];
  __shared__ float b_s[TILE];
  __shared__ double red[NTHREADS];
  const int d = blockIdx.y;
  const int tid = threadIdx.x;
  const bool active = d < a.ng && (int)blockIdx.x < a.nblk[d];
  if (active) {
    const int pitch = a.pitch[d], c4 = pitch / 4;
    const int64_t rows = a.rows[d];
    const int64_t ntiles = ceil_div(rows, TILE);
    const int nb = a.nblk[d];
    const int64_t base = ntiles / nb, rem = ntiles % nb;
    const int64_t t0 = blockIdx.x * base + min64(blockIdx.x, rem);
    const int64_t cnt = base + (blockIdx.x < rem ? 1 : 0);
    const uint32_t tile_bytes = TILE * pitch * 4;
    // S_d is immutable: its first tiles stream in before the dependency wait
    if (tid == 0) {
      for (int s = 0; s < a.nst; s++) mbar_init(&bar[s], 1);
      fence_mbar_init();
      for (int s = 0; s < a.nst && s < cnt; s++) {
        mbar_arrive_expect_tx(&bar[s], tile_bytes);
        bulk_g2s(smem + s * a.stage_bytes, a.S[d] + (t0 + s) * TILE * (int64_t)pitch, tile_bytes,
                 &bar[s]);
      }
    }
    pdl_wait();      // bins / residuals / partials of this iteration's fact pass are final
    pdl_trigger();
    glm_reduce_fact_early(u);
    __syncthreads();
    const int Gr = NTHREADS / c4;
    const bool pb = tid < Gr * c4;
    const int pj = tid % c4, pg = tid / c4;
    double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    // bins value of this thread's row of tile i (loaded one tile ahead, so
    // the L2 latency overlaps the previous tile instead of stalling the CTA)
    auto load_b = [&](int64_t i) -> float {
      const int64_t row = (t0 + i) * TILE + tid;
      float b = 0.f;
      if (row < rows) {
        if (a.bins[d]) {
          b = a.bins[d][row];
        } else {
          int64_t m0 = a.grp_ptr[d][row], m1 = a.grp_ptr[d][row + 1];
          for (int64_t m = m0; m < m1; m++) b += a.resid[a.grp_rows[d][m]];
        }
      }
      return b;
    };
    float b_next = cnt > 0 ? load_b(0) : 0.f;
    for (int64_t i = 0; i < cnt; i++) {
      const int s = (int)(i % a.nst);
      const float b = b_next;
      if (i + 1 < cnt) b_next = load_b(i + 1);
      b_s[tid] = b;
      mbar_wait(&bar[s], (uint32_t)((i / a.nst) & 1));
      __syncthreads();
      const float4* tile = reinterpret_cast<const float4*>(smem + s * a.stage_bytes);
      if (pb) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int r2 = pg; r2 < TILE; r2 += Gr) {
          float bb = b_s[r2];
          float4 v4 = tile[r2 * c4 + pj];
          acc.x = fmaf(bb, v4.x, acc.x);
          acc.y = fmaf(bb, v4.y, acc.y);
          acc.z = fmaf(bb, v4.z, acc.z);
          acc.w = fmaf(bb, v4.w, acc.w);
        }
        acc0 += acc.x;
        acc1 += acc.y;
        acc2 += acc.z;
        acc3 += acc.w;
      }
      __syncthreads();
      if (tid == 0 && i + a.nst < cnt) {
        fence_proxy_async();
        mbar_arrive_expect_tx(&bar[s], tile_bytes);
        bulk_g2s(smem + s * a.stage_bytes, a.S[d] + (t0 + i + a.nst) * TILE * (int64_t)pitch,
                 tile_bytes, &bar[s]);
      }
    }
    double* out = a.part[d] + blockIdx.x * (int64_t)pitch;
    for (int comp = 0; comp < 4; comp++) {
      double val = comp == 0 ? acc0 : comp == 1 ? acc1 : comp == 2 ? acc2 : acc3;
      __syncthreads();
      red[tid] = pb ? val : 0.0;
      __syncthreads();
      if (tid < c4) {
        double sum = 0.0;
        for (int g = 0; g < Gr; g++) sum += red[g * c4 + tid];
        out[tid * 4 + comp] = sum;
      }
    }
  }
  if (!active) {   // the last-CTA election below reads / writes shared state
    pdl_wait();
    glm_reduce_fact_early(u);
  }
  // last-block-done over the whole grid
  __threadfence();
  __syncthreads();
  __shared__ int is_last;
  if (tid == 0)
    is_last = atomicAdd(&u.state->done_dim, 1) == (int)(gridDim.x * gridDim.y) - 1;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  glm_reduce_all(u);
  if (fuse_update) glm_apply_update(u);
  if (tid == 0) u.state->done_dim = 0;
}

__global__ void k_glm_update(UpdateArgs u) { glm_apply_update(u); }

}  // namespace flb

namespace flb {
template <int MODEL, int C4>
static void launch_fw(const GlmFactWArgs& a, const UpdateArgs& u, int grid, size_t smem,
                      cudaStream_t st, bool pdl) {
  constexpr int RPL = C4 <= 7 ? 2 : 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(FW_WARPS * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (pdl && std::getenv("FL_NO_PDL") == nullptr) ? 1 : 0;
  (void)u;
  cudaLaunchKernelEx(&cfg, k_glm_fact_w<MODEL, C4, RPL>, a);
}
template <int MODEL, int C4>
static const void* fw_ptr() {
  constexpr int RPL = C4 <= 7 ? 2 : 1;
  return (const void*)k_glm_fact_w<MODEL, C4, RPL>;
}
#define FW_CASES(M, X) \
  X(M, 1) X(M, 3) X(M, 5) X(M, 7) X(M, 9) X(M, 11) X(M, 13) X(M, 15) X(M, 17) X(M, 19)
static bool fw_supported(int c4) { return c4 >= 1 && c4 <= 19 && (c4 & 1); }
static const void* fw_kernel(int model, int c4) {
#define FW_PTR(M, C) if (c4 == C) return fw_ptr<M, C>();
  if (model == 0) { FW_CASES(0, FW_PTR) } else { FW_CASES(1, FW_PTR) }
#undef FW_PTR
  return nullptr;
}
static void fw_launch(int model, int c4, const GlmFactWArgs& a, const UpdateArgs& u, int grid,
                      size_t smem, cudaStream_t st, bool pdl = false) {
#define FW_LAUNCH(M, C) if (c4 == C) { launch_fw<M, C>(a, u, grid, smem, st, pdl); return; }
  if (model == 0) { FW_CASES(0, FW_LAUNCH) } else { FW_CASES(1, FW_LAUNCH) }
#undef FW_LAUNCH
}
}  // namespace flb

namespace flb {
// ---- width-general GLM iteration (generic operators around two small kernels)
template <int MODEL>
__global__ void __launch_bounds__(256) k_glm_u_resid(const float* __restrict__ z,
                                                     const float* __restrict__ y, int64_t r_T,
                                                     float* __restrict__ r,
                                                     double* __restrict__ lpart) {
  __shared__ double red_s[256];
  double l64 = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r_T;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float zz = z[i], yv = y[i];
    float rv, l;
    if (MODEL == 0) {
      rv = zz - yv;
      l = 0.5f * rv * rv;
    } else {
      const float e = __expf(-fabsf(zz));
      const float sp = log1pf(e);
      const float inv = __frcp_rn(1.f + e);
      rv = (zz >= 0.f ? inv : e * inv) - yv;
      const float lp = zz >= 0.f ? sp : sp - zz, lq = zz >= 0.f ? sp + zz : sp;
      l = yv != 0.f ? fminf(lp, kLogClip) : fminf(lq, kLogClip);
    }
    r[i] = rv;
    l64 += (double)l;
  }
  red_s[threadIdx.x] = l64;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red_s[threadIdx.x] += red_s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) lpart[blockIdx.x] = red_s[0];
}

__global__ void k_glm_u_loss(const double* __restrict__ lpart, int n, double* red, int c_T) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int b = 0; b < n; b++) s += lpart[b];
    red[c_T] = s;
  }
}

__global__ void k_glm_u_update(double* w64, float* w32, const double* red, int c_T, double lr,
                               double* loss_hist, int loss_cap, GlmState* state) {
  const int it = state->it;
  if (threadIdx.x == 0 && it < loss_cap) loss_hist[it] = red[c_T];
  for (int c = threadIdx.x; c < c_T; c += blockDim.x) {
    w64[c] -= lr * red[c];
    w32[c] = (float)w64[c];
  }
  __syncthreads();
  if (threadIdx.x == 0) state->it = it + 1;
}

__global__ void k_u8_to_f32(const uint8_t* __restrict__ a, int64_t n, float* __restrict__ b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    b[i] = (float)a[i];
}
}  // namespace flb

using namespace flb;

struct fl_glm {
  fl_table* t = nullptr;
  int model = 0;
  double lr = 0;
  int nblk_fact = 0;
  int nst_fact = 0;
  uint32_t stage_fact = 0, off_fk = 0, off_y = 0;
  size_t smem_fact = 0;
  int nst_dim = 0;
  uint32_t stage_dim = 0;
  size_t smem_dim = 0;
  int dim_grid_x = 0;
  DevBuf y, wF, wd, w64, q, bins, resid, part_fact, part_dim, carry, red, loss_hist, state;
  DevBuf fw_carry, fw_part;
  // sparse stream block (CSR copy of F, f3)
  bool use_csr = false;
  GlmCsrArgs csr{};
  DevBuf csr_rp, csr_col, csr_val;
  size_t smem_csr = 0;
  double csr_density = -1.0;   // < 0: not measured yet
  GlmFactArgs fa{};
  DimArgs da{};
  UpdateArgs ua{};
  int loss_cap = 1 << 16;
  cudaGraphExec_t graph = nullptr;
  cudaGraphExec_t graph_n = nullptr;   // kGlmGraphIters iterations
  DevBuf red_fact;                     // early-reduced fact partials
  cudaStream_t cap_stream = nullptr;
  int bins_rows = 0;
  bool use_fw = false;
  bool solo = false;       // one-kernel iteration (glm_fact_warp.cuh, solo)
  DevBuf solo_part, solo_span, ua_dev, solo_gcnt, solo_gpart;
  GlmFactWArgs fw{};
  int nblk_fw = 0;
  size_t smem_fw = 0;
  // width-general path (stream blocks / dimensions too wide for the fused
  // passes): z = T w, residual, T^T r through the generic operators
  bool unfused = false;
  DevBuf y_t, z, r, w32, lpart;
  int u_blocks = 0;
  fl_comm* comm = nullptr;   // sharded run(): all-reduce of `red` between partial and update
};

namespace flb {

static int glm_u_partial(fl_glm* s, cudaStream_t st) {
  fl_table* t = s->t;
  int rc = do_lmm(t, s->w32.as<float>(), 1, s->z.as<float>(), st);
  if (rc) return rc;
  if (s->model == FL_MODEL_LINREG)
    k_glm_u_resid<0><<<s->u_blocks, 256, 0, st>>>(s->z.as<float>(), s->y_t.as<float>(), t->r_T,
                                                  s->r.as<float>(), s->lpart.as<double>());
  else
    k_glm_u_resid<1><<<s->u_blocks, 256, 0, st>>>(s->z.as<float>(), s->y_t.as<float>(), t->r_T,
                                                  s->r.as<float>(), s->lpart.as<double>());
  FL_CHECK_LAUNCH();
  FL_CUDA(cudaMemsetAsync(s->red.p, 0, (size_t)(t->c_T + 1) * 8, st));
  rc = do_tlmm(t, YView{s->r.as<float>(), 1, 0}, 1, s->red.as<double>(), 1, 0, st);
  if (rc) return rc;
  k_glm_u_loss<<<1, 32, 0, st>>>(s->lpart.as<double>(), s->u_blocks, s->red.as<double>(), t->c_T);
  FL_CHECK_LAUNCH();
  return FL_OK;
}

static int glm_u_update(fl_glm* s, cudaStream_t st) {
  k_glm_u_update<<<1, 256, 0, st>>>(s->w64.as<double>(), s->w32.as<float>(), s->red.as<double>(),
                                    s->t->c_T, s->lr, s->loss_hist.as<double>(), s->loss_cap,
                                    s->state.as<GlmState>());
  FL_CHECK_LAUNCH();
  return FL_OK;
}

// PDL launch (FL_NO_PDL=1 turns the attribute off for A/B timing).  Only
// kernels that call pdl_wait() before touching their predecessor's outputs
// may be launched with pdl = true.
static bool pdl_enabled() {
  static const bool on = std::getenv("FL_NO_PDL") == nullptr;
  return on;
}
template <typename... KArgs, typename... Args>
static cudaError_t launch_k(bool pdl, void (*k)(KArgs...), dim3 g, dim3 b, size_t smem,
                            cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (pdl && pdl_enabled()) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// nonzero fraction of the real stream-block columns (one coalesced pass)
static int glm_stream_density(fl_glm* s, cudaStream_t st) {
  const fl_table* t = s->t;
  DevBuf tot;
  int rc;
  if ((rc = tot.alloc(16))) return rc;
  FL_CUDA(cudaMemsetAsync(tot.p, 0, 8, st));
  k_nnz_total<<<(unsigned)(t->sm_count * 16), 256, 0, st>>>(
      reinterpret_cast<const float4*>(t->F->p), t->r_pad * t->pf / 4,
      reinterpret_cast<unsigned long long*>(tot.p));
  FL_CHECK_LAUNCH();
  unsigned long long nnz_all = 0;
  FL_CUDA(cudaMemcpyAsync(&nnz_all, tot.p, 8, cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  s->csr_density = (double)nnz_all / ((double)std::max<int64_t>(1, t->r_T) * std::max(1, t->nf));
  return FL_OK;
}

static int glm_launch_iteration(fl_glm* s, cudaStream_t st, bool fuse_update) {
  if (s->unfused) {
    int rc = glm_u_partial(s, st);
    if (rc) return rc;
    return fuse_update ? glm_u_update(s, st) : FL_OK;
  }
  if (s->solo) {   // one kernel: q, fact pass, gradient, reduction (+ update)
    GlmFactWArgs fw = s->fw;
    fw.fuse_update = fuse_update ? 1 : 0;
    fw_launch(s->model, s->t->pf / 4, fw, s->ua, s->nblk_fw, s->smem_fw, st, true);
    FL_CHECK_LAUNCH();
    return FL_OK;
  }
  fl_table* t = s->t;
  // the sort source's bins are zeroed by k_glm_dim_q (after its PDL wait)
  if (s->da.ng > 0) {
    dim3 grid(s->dim_grid_x, s->da.ng);
    FL_CUDA(launch_k(true, k_glm_dim_q, grid, dim3(NTHREADS), s->smem_dim, st, s->da));
  }
  if (s->use_csr) {
    if (s->model == FL_MODEL_LINREG)
      k_glm_fact_csr<0><<<s->nblk_fw, FW_WARPS * 32, s->smem_csr, st>>>(s->csr);
    else
      k_glm_fact_csr<1><<<s->nblk_fw, FW_WARPS * 32, s->smem_csr, st>>>(s->csr);
  } else if (s->use_fw)
    fw_launch(s->model, s->t->pf / 4, s->fw, s->ua, s->nblk_fw, s->smem_fw, st, true);
  else if (s->model == FL_MODEL_LINREG)
    k_glm_fact<0><<<s->nblk_fact, NTHREADS, s->smem_fact, st>>>(s->fa);
  else
    k_glm_fact<1><<<s->nblk_fact, NTHREADS, s->smem_fact, st>>>(s->fa);
  FL_CHECK_LAUNCH();
  dim3 grid3(std::max(1, s->dim_grid_x), std::max(1, s->da.ng));
  FL_CUDA(launch_k(true, k_glm_dim_t, grid3, dim3(NTHREADS), s->smem_dim, st, s->da, s->ua,
                   fuse_update ? 1 : 0));
  (void)t;
  return FL_OK;
}

}  // namespace flb

extern "C" {

int fl_glm_create(fl_table* t, int32_t model, const void* y, double learning_rate, fl_glm** out,
                  void* stream) {
  if (!t || !t->finalized || !y || !out) {
    set_error("fl_glm_create: bad arguments");
    return FL_ERR_ARG;
  }
  if (model != FL_MODEL_LINREG && model != FL_MODEL_LOGREG) {
    set_error("unknown model id %d", model);
    return FL_ERR_CONFIG;
  }
  if (!(learning_rate > 0.0)) {
    set_error("learning_rate must be > 0");
    return FL_ERR_CONFIG;
  }
  // more than MAX_GATHER gathered sources: the width-general path below
  bool wide = t->pf > 252 || (int)t->g.size() > MAX_GATHER;
  for (auto& g : t->g) wide |= (size_t)TILE * g.pitch * 4 * 2 > 200 * 1024;
  {
    const int yb0 = model == FL_MODEL_LOGREG ? 1 : 4;
    const uint32_t off_y0 = (uint32_t)(TILE * t->pf * 4);
    const uint32_t stage0 = (uint32_t)round_up(off_y0 + round_up(TILE * yb0, 128) +
                                               (t->sort_g >= 0 ? TILE * 4 : 0), 128);
    wide |= (size_t)2 * stage0 > 200 * 1024;
  }
  if (wide || getenv("FL_GLM_UNFUSED")) {
    // width-general path: generic operators (any width), same ABI and results
    FL_CUDA(cudaSetDevice(t->device));
    cudaStream_t st = (cudaStream_t)stream;
    auto* s = new fl_glm();
    std::unique_ptr<fl_glm> guard(s);
    s->t = t;
    s->model = model;
    s->lr = learning_rate;
    s->unfused = true;
    int rc;
    const int64_t r_T = t->r_T;
    if ((rc = s->y_t.alloc((size_t)r_T * 4 + 16))) return rc;
    if (model == FL_MODEL_LOGREG) {
      uint8_t* yd = nullptr;
      FL_CUDA(cudaMallocAsync((void**)&yd, (size_t)r_T + 16, st));
      FL_CUDA(cudaMemcpyAsync(yd, y, (size_t)r_T, cudaMemcpyDefault, st));
      k_u8_to_f32<<<(unsigned)std::min<int64_t>(ceil_div(r_T, 256), 4096), 256, 0, st>>>(
          yd, r_T, s->y_t.as<float>());
      FL_CHECK_LAUNCH();
      FL_CUDA(cudaFreeAsync(yd, st));
    } else {
      FL_CUDA(cudaMemcpyAsync(s->y_t.p, y, (size_t)r_T * 4, cudaMemcpyDefault, st));
    }
    if ((rc = s->z.alloc((size_t)r_T * 4 + 16))) return rc;
    if ((rc = s->r.alloc((size_t)r_T * 4 + 16))) return rc;
    if ((rc = s->w32.alloc((size_t)t->c_T * 4 + 16))) return rc;
    FL_CUDA(cudaMemsetAsync(s->w32.p, 0, (size_t)t->c_T * 4, st));
    if ((rc = s->w64.alloc((size_t)t->c_T * 8))) return rc;
    FL_CUDA(cudaMemsetAsync(s->w64.p, 0, (size_t)t->c_T * 8, st));
    s->u_blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(r_T, 256), 4 * t->sm_count));
    if ((rc = s->lpart.alloc((size_t)s->u_blocks * 8))) return rc;
    if ((rc = s->red.alloc((size_t)(t->c_T + 1) * 8))) return rc;
    FL_CUDA(cudaMemsetAsync(s->red.p, 0, (size_t)(t->c_T + 1) * 8, st));
    if ((rc = s->loss_hist.alloc((size_t)s->loss_cap * 8))) return rc;
    if ((rc = s->state.alloc(sizeof(GlmState)))) return rc;
    FL_CUDA(cudaMemsetAsync(s->state.p, 0, sizeof(GlmState), st));
    FL_CUDA(cudaStreamSynchronize(st));
    *out = guard.release();
    return FL_OK;
  }
  const PhaseTrace trace("fl_glm_create");
  FL_CUDA(cudaSetDevice(t->device));
  cudaStream_t st = (cudaStream_t)stream;
  auto* s = new fl_glm();
  std::unique_ptr<fl_glm> guard(s);
  s->t = t;
  s->model = model;
  s->lr = learning_rate;
  int rc;
  const int64_t r_pad = t->r_pad;
  const int ng = (int)t->g.size();
  // labels in device order
  const int yb = model == FL_MODEL_LOGREG ? 1 : 4;
  if ((rc = s->y.alloc((size_t)r_pad * yb + 16))) return rc;
  {
    void* ydev = nullptr;
    FL_CUDA(cudaMallocAsync(&ydev, (size_t)t->r_T * yb + 16, st));
    FL_CUDA(cudaMemcpyAsync(ydev, y, (size_t)t->r_T * yb, cudaMemcpyDefault, st));
    rc = launch_gather_rows_to_device_order(t, ydev, s->y.p, yb, st);
    if (rc) return rc;
    FL_CUDA(cudaFreeAsync(ydev, st));
  }
  trace.mark("labels issued");
  // parameters
  if ((rc = s->w64.alloc((size_t)t->c_T * 8))) return rc;
  FL_CUDA(cudaMemsetAsync(s->w64.p, 0, (size_t)t->c_T * 8, st));
  if ((rc = s->wF.alloc((size_t)t->pf * 4))) return rc;
  FL_CUDA(cudaMemsetAsync(s->wF.p, 0, (size_t)t->pf * 4, st));
  size_t wd_total = 0, q_total = 0;
  for (auto& g : t->g) {
    wd_total += g.pitch;
    q_total += round_up(g.rows, 4);
  }
  if ((rc = s->wd.alloc(wd_total * 4 + 16))) return rc;
  FL_CUDA(cudaMemsetAsync(s->wd.p, 0, wd_total * 4 + 16, st));
  if ((rc = s->q.alloc(q_total * 4 + 16))) return rc;
  bool any_unsorted = false;
  for (auto& g : t->g) any_unsorted |= !g.sorted;
  if (t->sort_g >= 0) {
    s->bins_rows = (int)t->g[t->sort_g].rows;
    if ((rc = s->bins.alloc((size_t)s->bins_rows * 4 + 16))) return rc;
  }
  if (any_unsorted) {
    if ((rc = s->resid.alloc((size_t)r_pad * 4))) return rc;
  }
  // fact-pass geometry
  const int c4 = t->pf / 4;
  s->off_y = (uint32_t)(TILE * t->pf * 4);
  s->off_fk = s->off_y + (uint32_t)round_up(TILE * yb, 128);
  s->stage_fact = (uint32_t)round_up(s->off_fk + (t->sort_g >= 0 ? TILE * 4 : 0), 128);
  s->nst_fact = s->stage_fact <= 24 * 1024 ? 4 : (s->stage_fact <= 36 * 1024 ? 3 : 2);
  s->smem_fact = (size_t)s->nst_fact * s->stage_fact;
  if (s->smem_fact > 200 * 1024) {
    set_error("fused GLM: streamed block too wide (%d columns)", t->nf);
    return FL_ERR_OP;
  }
  auto kf = model == FL_MODEL_LINREG ? (const void*)k_glm_fact<0> : (const void*)k_glm_fact<1>;
  FL_CUDA(raise_smem_limit(kf, (int)s->smem_fact));
  int occ = 1;
  FL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kf, NTHREADS, s->smem_fact));
  occ = std::max(1, std::min(occ, 2));
  const int64_t ntiles = r_pad / TILE;
  s->nblk_fact = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)t->sm_count * occ));
  if ((rc = s->part_fact.alloc((size_t)s->nblk_fact * (t->pf + 1) * 8))) return rc;
  if ((rc = s->carry.alloc((size_t)s->nblk_fact * sizeof(CarryRec)))) return rc;
  FL_CUDA(cudaMemsetAsync(s->carry.p, 0xff, (size_t)s->nblk_fact * sizeof(CarryRec), st));
  if ((rc = s->state.alloc(sizeof(GlmState)))) return rc;
  FL_CUDA(cudaMemsetAsync(s->state.p, 0, sizeof(GlmState), st));
  if ((rc = s->red.alloc((size_t)(t->c_T + 1) * 8))) return rc;
  FL_CUDA(cudaMemsetAsync(s->red.p, 0, (size_t)(t->c_T + 1) * 8, st));
  if ((rc = s->loss_hist.alloc((size_t)s->loss_cap * 8))) return rc;

  GlmFactArgs& fa = s->fa;
  fa.F = t->F->as<float>();
  fa.pf = t->pf;
  fa.c4 = c4;
  fa.y = s->y.p;
  fa.r_T = t->r_T;
  fa.ntiles = ntiles;
  fa.ng = ng;
  fa.sort_g = t->sort_g;
  {
    size_t qo = 0;
    for (int d = 0; d < ng; d++) {
      fa.fk[d] = t->g[d].fk->as<int32_t>();
      fa.q[d] = s->q.as<float>() + qo;
      qo += round_up(t->g[d].rows, 4);
    }
  }
  fa.bins = t->sort_g >= 0 ? s->bins.as<float>() : nullptr;
  fa.resid = any_unsorted ? s->resid.as<float>() : nullptr;
  fa.wF = s->wF.as<float>();
  fa.part = s->part_fact.as<double>();
  fa.carry = s->carry.as<CarryRec>();
  fa.state = s->state.as<GlmState>();
  fa.stage_bytes = s->stage_fact;
  fa.off_fk = s->off_fk;
  fa.off_y = s->off_y;
  fa.nst = s->nst_fact;

  // per-warp-pipeline fact pass (preferred when the stream width is templated)
  if (fw_supported(c4) && !getenv("FL_GLM_CTA_TILES")) {
    const int rpl = c4 <= 7 ? 2 : 1;
    const int rw = 32 * rpl;
    GlmFactWArgs& fw = s->fw;
    fw.F = fa.F;
    fw.pf = t->pf;
    fw.y = fa.y;
    fw.r_T = t->r_T;
    fw.nunits = r_pad / rw;
    fw.ng = fa.ng;
    fw.sort_g = fa.sort_g;
    for (int d = 0; d < ng; d++) {
      fw.fk[d] = fa.fk[d];
      fw.q[d] = fa.q[d];
    }
    fw.bins = fa.bins;
    fw.resid = fa.resid;
    fw.wF = fa.wF;
    fw.state = fa.state;
    fw.off_y = (uint32_t)round_up((int64_t)rw * t->pf * 4, 16);
    fw.off_fk = fw.off_y + (uint32_t)round_up((int64_t)rw * yb, 16);
    fw.stage_bytes = (uint32_t)round_up(fw.off_fk + (t->sort_g >= 0 ? rw * 4 : 0), 128);
    const size_t budget = fw_min_blocks(c4) == 2 ? 100 * 1024 : 200 * 1024;
    int nst = (int)(budget / ((size_t)FW_WARPS * fw.stage_bytes));
    if (const char* e = getenv("FL_GLM_NST")) nst = atoi(e);
    fw.nst = std::max(2, std::min(4, nst));
    s->smem_fw = (size_t)FW_WARPS * fw.nst * fw.stage_bytes;
    if (s->smem_fw <= 220 * 1024) {
      const void* kfw = fw_kernel(model, c4);
      FL_CUDA(raise_smem_limit(kfw, (int)s->smem_fw));
      int occw = 1;
      FL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occw, kfw, FW_WARPS * 32, s->smem_fw));
      occw = std::max(1, occw);
      int64_t want = ceil_div(fw.nunits, FW_WARPS);
      s->nblk_fw = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)t->sm_count * occw));
      if ((rc = s->fw_carry.alloc((size_t)s->nblk_fw * FW_WARPS * sizeof(WarpCarry)))) return rc;
      if ((rc = s->fw_part.alloc((size_t)s->nblk_fw * (t->pf + 1) * 8))) return rc;
      fw.carry = s->fw_carry.as<WarpCarry>();
      fw.part = s->fw_part.as<double>();
      s->use_fw = true;
    }
  }

  trace.mark("fact-pass geometry");
  // sparse stream block: when F is sparse, a CSR copy
  // (device order) feeds k_glm_fact_csr, which reads 6 bytes per nonzero
  // instead of 4 bytes per entry.  FL_GLM_SPARSE: unset = auto (density of
  // the real stream columns < kCsrAutoDensity), 1 = force, 0 = never.
  {
    const char* e = getenv("FL_GLM_SPARSE");
    const int mode = e ? atoi(e) : -1;
    // the density probe runs only when it can change the decision (forced
    // CSR, or an auto threshold above 0); fl_glm_path measures it on demand
    bool want_csr = false;
    if (mode != 0 && s->use_fw && t->pf <= CSR_MAXP && t->nf > 0 &&
        (mode == 1 || kCsrAutoDensity > 0.0)) {
      if ((rc = glm_stream_density(s, st))) return rc;
      want_csr = mode == 1 || s->csr_density < kCsrAutoDensity;
    }
    if (want_csr) {
      DevBuf cnt;
      if ((rc = cnt.alloc((size_t)(r_pad + 1) * 8))) return rc;
      FL_CUDA(cudaMemsetAsync(cnt.p, 0, (size_t)(r_pad + 1) * 8, st));
      const unsigned gb = (unsigned)std::min<int64_t>(ceil_div(r_pad, 256), 65535);
      k_csr_count<<<gb, 256, 0, st>>>(t->F->as<float>(), r_pad, t->pf, cnt.as<int64_t>());
      FL_CHECK_LAUNCH();
      if ((rc = s->csr_rp.alloc((size_t)(r_pad + 1) * 8))) return rc;
      size_t tb = 0;
      FL_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.as<int64_t>(), s->csr_rp.as<int64_t>(),
                                            r_pad + 1, st));
      DevBuf tmp;
      if ((rc = tmp.alloc(tb + 16))) return rc;
      FL_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt.as<int64_t>(), s->csr_rp.as<int64_t>(),
                                            r_pad + 1, st));
      int64_t nnz = 0;
      FL_CUDA(cudaMemcpyAsync(&nnz, s->csr_rp.as<int64_t>() + r_pad, 8, cudaMemcpyDeviceToHost, st));
      FL_CUDA(cudaStreamSynchronize(st));
      {
        if ((rc = s->csr_col.alloc((size_t)nnz * 2 + 16))) return rc;
        if ((rc = s->csr_val.alloc((size_t)nnz * 4 + 16))) return rc;
        k_csr_fill<<<gb, 256, 0, st>>>(t->F->as<float>(), r_pad, t->pf, s->csr_rp.as<int64_t>(),
                                       s->csr_col.as<uint16_t>(), s->csr_val.as<float>());
        FL_CHECK_LAUNCH();
        GlmCsrArgs& ca = s->csr;
        ca.rp = s->csr_rp.as<int64_t>();
        ca.col = s->csr_col.as<uint16_t>();
        ca.val = s->csr_val.as<float>();
        ca.pf = t->pf;
        ca.y = s->fw.y;
        ca.r_T = t->r_T;
        ca.nunits = r_pad / 32;
        ca.ng = s->fw.ng;
        ca.sort_g = s->fw.sort_g;
        for (int d = 0; d < ng; d++) {
          ca.fk[d] = s->fw.fk[d];
          ca.q[d] = s->fw.q[d];
        }
        ca.bins = s->fw.bins;
        ca.resid = s->fw.resid;
        ca.wF = s->fw.wF;
        ca.state = s->fw.state;
        s->smem_csr = ((size_t)round_up(t->pf, 4) + (size_t)FW_WARPS * 32 * (t->pf | 1)) * 4;
        for (int m = 0; m < 2; m++) {
          const void* kc = m == 0 ? (const void*)k_glm_fact_csr<0> : (const void*)k_glm_fact_csr<1>;
          FL_CUDA(raise_smem_limit(kc, (int)s->smem_csr));
        }
        int occc = 1;
        FL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &occc, model == 0 ? (const void*)k_glm_fact_csr<0> : (const void*)k_glm_fact_csr<1>,
            FW_WARPS * 32, s->smem_csr));
        occc = std::max(1, occc);
        const int64_t want = ceil_div(ca.nunits, FW_WARPS);
        s->nblk_fw = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)t->sm_count * occc));
        if ((rc = s->fw_carry.alloc((size_t)s->nblk_fw * FW_WARPS * sizeof(WarpCarry)))) return rc;
        if ((rc = s->fw_part.alloc((size_t)s->nblk_fw * (t->pf + 1) * 8))) return rc;
        ca.carry = s->fw_carry.as<WarpCarry>();
        ca.part = s->fw_part.as<double>();
        s->fw.carry = ca.carry;
        s->fw.part = ca.part;
        s->use_csr = true;
      }
      FL_CUDA(cudaStreamSynchronize(st));
    }
  }

  trace.mark("density probe");
  // dim geometry
  DimArgs& da = s->da;
  da.ng = ng;
  int max_pitch = 4;
  for (auto& g : t->g) max_pitch = std::max(max_pitch, g.pitch);
  s->stage_dim = (uint32_t)(TILE * max_pitch * 4);
  s->nst_dim = s->stage_dim <= 24 * 1024 ? 4 : (s->stage_dim <= 48 * 1024 ? 3 : 2);
  s->smem_dim = (size_t)s->nst_dim * s->stage_dim;
  if (s->smem_dim > 200 * 1024) {
    set_error("fused GLM: gathered source too wide");
    return FL_ERR_OP;
  }
  FL_CUDA(raise_smem_limit(k_glm_dim_q, (int)s->smem_dim));
  FL_CUDA(raise_smem_limit(k_glm_dim_t, (int)s->smem_dim));
  int occd = 1;
  FL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occd, k_glm_dim_t, NTHREADS, s->smem_dim));
  occd = std::max(1, occd);
  da.stage_bytes = s->stage_dim;
  da.nst = s->nst_dim;
  size_t part_dim_total = 0;
  s->dim_grid_x = 1;
  for (int d = 0; d < ng; d++) {
    const GatherSrc& g = t->g[d];
    int64_t tiles = ceil_div(g.rows, TILE);
    // share the SMs between sources in proportion to their bytes
    int nb = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)t->sm_count * occd));
    da.nblk[d] = nb;
    s->dim_grid_x = std::max(s->dim_grid_x, nb);
    part_dim_total += (size_t)nb * g.pitch;
  }
  if ((rc = s->part_dim.alloc(part_dim_total * 8 + 16))) return rc;
  {
    size_t wo = 0, po = 0;
    for (int d = 0; d < ng; d++) {
      const GatherSrc& g = t->g[d];
      da.S[d] = g.S->as<float>();
      da.pitch[d] = g.pitch;
      da.rows[d] = g.rows;
      da.w[d] = s->wd.as<float>() + wo;
      da.q[d] = const_cast<float*>(fa.q[d]);
      da.bins[d] = g.sorted ? fa.bins : nullptr;
      da.grp_ptr[d] = g.grp_ptr->as<int64_t>();
      da.grp_rows[d] = g.grp_rows ? g.grp_rows->as<int32_t>() : nullptr;
      da.part[d] = s->part_dim.as<double>() + po;
      wo += g.pitch;
      po += (size_t)da.nblk[d] * g.pitch;
    }
    da.resid = fa.resid;
    da.bins_zero = s->bins_rows > 0 ? s->bins.as<float>() : nullptr;
    da.bins_n = s->bins_rows;
  }
  UpdateArgs& ua = s->ua;
  ua.c_T = t->c_T;
  ua.pf = t->pf;
  ua.ng = ng;
  ua.lr = learning_rate;
  ua.f_tcol = t->d_f_tcol->as<int32_t>();
  ua.wF = s->wF.as<float>();
  ua.w64 = s->w64.as<double>();
  ua.red = s->red.as<double>();
  ua.loss_hist = s->loss_hist.as<double>();
  ua.loss_cap = s->loss_cap;
  ua.state = s->state.as<GlmState>();
  ua.part_fact = s->use_fw ? s->fw_part.as<double>() : s->part_fact.as<double>();
  ua.nblk_fact = s->use_fw ? s->nblk_fw : s->nblk_fact;
  if ((rc = s->red_fact.alloc((size_t)(t->pf + 1) * 8))) return rc;
  ua.red_fact = s->red_fact.as<double>();
  for (int d = 0; d < ng; d++) {
    ua.d_tcol[d] = t->g[d].d_tcol->as<int32_t>();
    ua.pitch[d] = t->g[d].pitch;
    ua.wd[d] = const_cast<float*>(da.w[d]);
    ua.part_dim[d] = da.part[d];
    ua.nblk_dim[d] = da.nblk[d];
  }
  trace.mark("dim geometry");
  // solo iteration (one kernel per GD step): the only gathered source is the
  // sort source, its rows are <= FW_SOLO_PITCH wide, and every fact-pass
  // CTA references <= FW_QCAP of its rows.  FL_GLM_SOLO=0 disables it.
  {
    const char* e = getenv("FL_GLM_SOLO");
    const bool off = e && atoi(e) == 0;
    if (!off && s->use_fw && !s->use_csr && ng == 1 && t->sort_g == 0 &&
        t->g[0].pitch <= FW_SOLO_PITCH) {
      const int rw = 32 * (c4 <= 7 ? 2 : 1);
      if ((rc = s->solo_span.alloc(16))) return rc;
      FL_CUDA(cudaMemsetAsync(s->solo_span.p, 0, 4, st));
      k_glm_solo_span<<<(unsigned)ceil_div(s->nblk_fw, 256), 256, 0, st>>>(
          t->g[0].fk->as<int32_t>(), t->g[0].n_neg, t->r_T, s->fw.nunits, rw, s->nblk_fw,
          s->solo_span.as<int>());
      FL_CHECK_LAUNCH();
      int span = 0;
      FL_CUDA(cudaMemcpyAsync(&span, s->solo_span.p, 4, cudaMemcpyDeviceToHost, st));
      FL_CUDA(cudaStreamSynchronize(st));
      // q staging sized to the measured span (not FW_QCAP): the solo kernel
      // must keep 2 CTAs per SM at C1 (112 KB of stages each)
      const int qcap = (int)std::min<int64_t>(FW_QCAP, round_up((int64_t)std::max(span, 1), 4));
      size_t extra = (size_t)qcap * 4 + (size_t)FW_WARPS * FW_LCAP * sizeof(SoloRec) +
                     (size_t)FW_WARPS * FW_SOLO_PITCH * 8;
      // the CTA's S_d span staged in shared memory when it is short (C1:
      // ~35 rows = 7 KB): one bulk copy before the PDL wait replaces the
      // prologue's and the gradient records' dependent L2 / HBM row reads
      const size_t s0_bytes = (size_t)span * t->g[0].pitch * 4;
      const char* e0 = getenv("FL_GLM_SOLO_S0");
      const bool s0_on = (!e0 || atoi(e0) != 0) && span > 0 && s0_bytes <= 32 * 1024;
      if (s0_on) extra += round_up((int64_t)s0_bytes, 16);
      const size_t smem_solo = s->smem_fw + extra;
      // a CTA stages its q rows before streaming: worth it while that
      // prologue is short (C1: 34 rows per CTA, one kernel instead of three);
      // at C2 (3.4K rows, 700 KB per CTA) the separate dim kernels win
      const int span_max = e ? FW_QCAP : 512;   // FL_GLM_SOLO=1 forces up to FW_QCAP
      if (span <= span_max && smem_solo <= 227 * 1024) {
        const void* kfw = fw_kernel(model, c4);
        FL_CUDA(raise_smem_limit(kfw, (int)smem_solo));
        if ((rc = s->solo_part.alloc((size_t)s->nblk_fw * t->g[0].pitch * 8))) return rc;
        GlmFactWArgs& fw = s->fw;
        fw.solo = 1;
        fw.s0_rows = s0_on ? span : 0;
        fw.qcap = qcap;
        if (const char* dg = getenv("FL_GLM_SOLO_DIAG")) fw.diag = atoi(dg);   // timing only
        fw.S0 = t->g[0].S->as<float>();
        fw.pitch0 = t->g[0].pitch;
        fw.w0d = da.w[0];
        fw.n_neg0 = t->g[0].n_neg;
        fw.part_d = s->solo_part.as<double>();
        if ((rc = s->ua_dev.alloc(sizeof(UpdateArgs)))) return rc;
        FL_CUDA(cudaMemcpy(s->ua_dev.p, &ua, sizeof(UpdateArgs), cudaMemcpyHostToDevice));
        fw.up = s->ua_dev.as<UpdateArgs>();
        const int ngroups = (int)ceil_div(s->nblk_fw, FW_GROUP);
        if ((rc = s->solo_gcnt.alloc((size_t)ngroups * 4))) return rc;
        FL_CUDA(cudaMemsetAsync(s->solo_gcnt.p, 0, (size_t)ngroups * 4, st));
        if ((rc = s->solo_gpart.alloc((size_t)ngroups * (t->pf + 1 + t->g[0].pitch) * 8))) return rc;
        fw.gcnt = s->solo_gcnt.as<int>();
        fw.gpart = s->solo_gpart.as<double>();
        s->smem_fw = smem_solo;
        s->solo = true;
      }
    }
  }
  FL_CUDA(cudaStreamSynchronize(st));
  trace.mark("done");
  *out = guard.release();
  return FL_OK;
}

int fl_glm_partial(fl_glm* s, void* stream) {
  if (!s) return FL_ERR_ARG;
  FL_CUDA(cudaSetDevice(s->t->device));
  return glm_launch_iteration(s, (cudaStream_t)stream, false);
}

int fl_glm_reduce_buffer(fl_glm* s, double** buf, int32_t* len) {
  if (!s || !buf || !len) return FL_ERR_ARG;
  *buf = s->red.as<double>();
  *len = s->t->c_T + 1;
  return FL_OK;
}

int fl_glm_update(fl_glm* s, void* stream) {
  if (!s) return FL_ERR_ARG;
  FL_CUDA(cudaSetDevice(s->t->device));
  if (s->unfused) return glm_u_update(s, (cudaStream_t)stream);
  k_glm_update<<<1, NTHREADS, 0, (cudaStream_t)stream>>>(s->ua);
  FL_CHECK_LAUNCH();
  return FL_OK;
}

// one iteration of run(): fused (single GPU), or partial -> all-reduce ->
// update when a communicator is attached
static int glm_iteration(fl_glm* s, cudaStream_t st) {
  if (!s->comm) return glm_launch_iteration(s, st, true);
  int rc = glm_launch_iteration(s, st, false);
  if (!rc) rc = comm_allreduce(s->comm, s->red.as<double>(), (size_t)s->t->c_T + 1, st);
  if (rc) return rc;
  if (s->unfused) return glm_u_update(s, st);
  k_glm_update<<<1, NTHREADS, 0, st>>>(s->ua);
  FL_CHECK_LAUNCH();
  return FL_OK;
}

int fl_glm_set_comm(fl_glm* s, fl_comm* c) {
  if (!s) return FL_ERR_ARG;
  if (s->comm != c) {   // graphs captured without / with another exchange
    if (s->graph) cudaGraphExecDestroy(s->graph);
    if (s->graph_n) cudaGraphExecDestroy(s->graph_n);
    s->graph = s->graph_n = nullptr;
  }
  s->comm = c;
  return FL_OK;
}

int fl_glm_run(fl_glm* s, int32_t iterations, void* stream) {
  if (!s || iterations < 1) {
    set_error("iterations must be >= 1");
    return FL_ERR_CONFIG;
  }
  FL_CUDA(cudaSetDevice(s->t->device));
  cudaStream_t st = (cudaStream_t)stream;
  if (s->unfused) {
    for (int i = 0; i < iterations; i++) {
      int rc = glm_iteration(s, st);
      if (rc) return rc;
    }
    return FL_OK;
  }
  // two graphs: one iteration, and kGlmGraphIters iterations back to back
  // (inside a graph the PDL edges let each kernel's prologue -- barrier
  // setup, the first TMA tiles of its immutable operands -- overlap the
  // previous kernel's tail, also across iteration boundaries)
  auto capture = [&](int n, cudaGraphExec_t* out) -> int {
    if (!s->cap_stream) FL_CUDA(cudaStreamCreateWithFlags(&s->cap_stream, cudaStreamNonBlocking));
    cudaGraph_t g;
    FL_CUDA(cudaStreamBeginCapture(s->cap_stream, cudaStreamCaptureModeThreadLocal));
    int rc = FL_OK;
    for (int i = 0; i < n && rc == FL_OK; i++) rc = glm_iteration(s, s->cap_stream);
    cudaError_t e = cudaStreamEndCapture(s->cap_stream, &g);
    if (rc) return rc;
    FL_CUDA(e);
    FL_CUDA(cudaGraphInstantiate(out, g, 0));
    FL_CUDA(cudaGraphDestroy(g));
    return FL_OK;
  };
  int rc;
  // FL_GLM_DIRECT=1: the remainder iterations as plain stream launches
  // instead of the one-iteration graph (launch-latency experiment)
  static const bool direct = [] {
    const char* e = getenv("FL_GLM_DIRECT");
    return e && atoi(e) != 0;
  }();
  if (!direct && !s->graph && (rc = capture(1, &s->graph))) return rc;
  const int nbig = iterations / kGlmGraphIters;
  if (nbig > 0 && !s->graph_n && (rc = capture(kGlmGraphIters, &s->graph_n))) return rc;
  for (int i = 0; i < nbig; i++) FL_CUDA(cudaGraphLaunch(s->graph_n, st));
  for (int i = nbig * kGlmGraphIters; i < iterations; i++) {
    if (direct) {
      if ((rc = glm_iteration(s, st))) return rc;
    } else {
      FL_CUDA(cudaGraphLaunch(s->graph, st));
    }
  }
  return FL_OK;
}

int fl_glm_path(fl_glm* s, int32_t* path, double* stream_density) {
  if (!s) {
    set_error("fl_glm_path: null session");
    return FL_ERR_ARG;
  }
  if (path) *path = s->unfused ? 3 : s->use_csr ? 2 : s->solo ? 4 : s->use_fw ? 1 : 0;
  if (stream_density) {
    if (s->csr_density < 0.0) {
      if (s->unfused || s->t->nf == 0) {
        s->csr_density = 1.0;
      } else {
        FL_CUDA(cudaSetDevice(s->t->device));
        int rc = glm_stream_density(s, nullptr);
        if (rc) return rc;
      }
    }
    *stream_density = s->csr_density;
  }
  return FL_OK;
}

int fl_glm_kernel_times(fl_glm* s, int32_t iters, float* ms_out, void* stream) {
  if (!s || iters < 1 || !ms_out) return FL_ERR_ARG;
  FL_CUDA(cudaSetDevice(s->t->device));
  cudaStream_t st = (cudaStream_t)stream;
  if (s->unfused) {   // [0, whole iteration, 0]
    cudaEvent_t e0, e1;
    FL_CUDA(cudaEventCreate(&e0));
    FL_CUDA(cudaEventCreate(&e1));
    FL_CUDA(cudaEventRecord(e0, st));
    for (int i = 0; i < iters; i++) {
      int rc = glm_launch_iteration(s, st, true);
      if (rc) return rc;
    }
    FL_CUDA(cudaEventRecord(e1, st));
    FL_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    FL_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    ms_out[0] = 0.f;
    ms_out[1] = ms / iters;
    ms_out[2] = 0.f;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return FL_OK;
  }
  if (s->solo) {   // [0, the one kernel, 0]
    cudaEvent_t e0, e1;
    FL_CUDA(cudaEventCreate(&e0));
    FL_CUDA(cudaEventCreate(&e1));
    FL_CUDA(cudaEventRecord(e0, st));
    for (int i = 0; i < iters; i++) {
      const int rc = glm_launch_iteration(s, st, true);
      if (rc) return rc;
    }
    FL_CUDA(cudaEventRecord(e1, st));
    FL_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    FL_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    ms_out[0] = ms_out[2] = 0.f;
    ms_out[1] = ms / iters;
    return FL_OK;
  }
  cudaEvent_t ev[4];
  for (auto& e : ev) FL_CUDA(cudaEventCreate(&e));
  float acc[3] = {0.f, 0.f, 0.f};
  for (int i = 0; i < iters; i++) {
    FL_CUDA(cudaEventRecord(ev[0], st));
    if (s->da.ng > 0) {   // (zeroes the bins too)
      dim3 grid(s->dim_grid_x, s->da.ng);
      k_glm_dim_q<<<grid, NTHREADS, s->smem_dim, st>>>(s->da);
      FL_CHECK_LAUNCH();
    }
    FL_CUDA(cudaEventRecord(ev[1], st));
    if (s->use_csr) {
      if (s->model == FL_MODEL_LINREG)
        k_glm_fact_csr<0><<<s->nblk_fw, FW_WARPS * 32, s->smem_csr, st>>>(s->csr);
      else
        k_glm_fact_csr<1><<<s->nblk_fw, FW_WARPS * 32, s->smem_csr, st>>>(s->csr);
    } else if (s->use_fw)
      fw_launch(s->model, s->t->pf / 4, s->fw, s->ua, s->nblk_fw, s->smem_fw, st);
    else if (s->model == FL_MODEL_LINREG)
      k_glm_fact<0><<<s->nblk_fact, NTHREADS, s->smem_fact, st>>>(s->fa);
    else
      k_glm_fact<1><<<s->nblk_fact, NTHREADS, s->smem_fact, st>>>(s->fa);
    FL_CHECK_LAUNCH();
    FL_CUDA(cudaEventRecord(ev[2], st));
    dim3 grid3(std::max(1, s->dim_grid_x), std::max(1, s->da.ng));
    k_glm_dim_t<<<grid3, NTHREADS, s->smem_dim, st>>>(s->da, s->ua, 1);
    FL_CHECK_LAUNCH();
    FL_CUDA(cudaEventRecord(ev[3], st));
    FL_CUDA(cudaEventSynchronize(ev[3]));
    for (int k = 0; k < 3; k++) {
      float ms = 0.f;
      FL_CUDA(cudaEventElapsedTime(&ms, ev[k], ev[k + 1]));
      acc[k] += ms;
    }
  }
  for (int k = 0; k < 3; k++) ms_out[k] = acc[k] / iters;
  for (auto& e : ev) cudaEventDestroy(e);
  return FL_OK;
}

int fl_glm_result(fl_glm* s, double* w, double* loss, int32_t n, int32_t* n_done, void* stream) {
  if (!s) return FL_ERR_ARG;
  FL_CUDA(cudaSetDevice(s->t->device));
  cudaStream_t st = (cudaStream_t)stream;
  GlmState h{};
  FL_CUDA(cudaMemcpyAsync(&h, s->state.p, sizeof(h), cudaMemcpyDeviceToHost, st));
  if (w) FL_CUDA(cudaMemcpyAsync(w, s->w64.p, (size_t)s->t->c_T * 8, cudaMemcpyDefault, st));
  FL_CUDA(cudaStreamSynchronize(st));
  int nd = std::min(h.it, s->loss_cap);
  if (n_done) *n_done = nd;
  if (loss && n > 0) {
    int m = std::min(n, nd);
    if (m > 0) FL_CUDA(cudaMemcpyAsync(loss, s->loss_hist.p, (size_t)m * 8, cudaMemcpyDefault, st));
    FL_CUDA(cudaStreamSynchronize(st));
  }
  return FL_OK;
}

int fl_glm_destroy(fl_glm* s) {
  if (!s) return FL_OK;
  cudaSetDevice(s->t->device);
  if (s->graph) cudaGraphExecDestroy(s->graph);
  if (s->graph_n) cudaGraphExecDestroy(s->graph_n);
  if (s->cap_stream) cudaStreamDestroy(s->cap_stream);
  delete s;
  return FL_OK;
}

}  // extern "C"
