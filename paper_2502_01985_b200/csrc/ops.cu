// Generic factorized operators behind TargetHandle (ops.py:219-328).
//
//   lmm   T x   = F x_F  +  sum_d gather(fk_d, S_d x_d)        (ops.py:227-233)
//   tlmm  T^T y = F^T y' +  sum_d S_d^T (I_d^T y')             (ops.py:264-269)
//   rmm   x T   = (T^T x^T)^T  (strided view, ops.py:243-251)
//
// y' is y read in device row order.  Per-row dot products run in fp32;
// every reduction over rows is carried in fp64 with a fixed-order final
// reduction (deterministic, independent of scheduling).  These kernels serve
// the op-level API; the trainers use the fused kernels in glm.cu / kmeans.cu.
#include <algorithm>

#include "internal.h"
#include "tc05.cuh"

namespace flb {

constexpr int CX_CHUNK = 32;   // output columns per launch chunk (lmm)

struct GatherSet {
  const float* q[MAX_GATHER];
  const int32_t* fk[MAX_GATHER];
  int n;
};

static inline unsigned gridn(int64_t n, int b = 256) { return (unsigned)ceil_div(n, b); }

// q[j, col] = sum_c S[j, c] * x[tcol[c], col0 + col]
__global__ void k_dim_q(const float* __restrict__ S, int pitch, int cols, int64_t rows,
                        const int32_t* __restrict__ tcol, const float* __restrict__ x, int c_x,
                        int col0, int ncol, float* __restrict__ q) {
  extern __shared__ float xs[];  // cols x ncol
  for (int i = threadIdx.x; i < cols * ncol; i += blockDim.x) {
    int c = i / ncol, col = i - c * ncol;
    xs[i] = x[(int64_t)tcol[c] * c_x + col0 + col];
  }
  __syncthreads();
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= rows * ncol) return;
  int64_t j = idx / ncol;
  int col = (int)(idx - j * ncol);
  const float* r = S + j * pitch;
  float acc = 0.f;
  for (int c = 0; c < cols; c++) acc = fmaf(r[c], xs[c * ncol + col], acc);
  q[j * ncol + col] = acc;
}

// out[perm[p], col0+col] = F[p,:] . xF[:, col] + sum_d q_d[fk_d[p], col]
__global__ void k_lmm_main(const float* __restrict__ F, int pf, const int32_t* __restrict__ ftcol,
                           const float* __restrict__ x, int c_x, int col0, int ncol,
                           GatherSet gs, const int32_t* __restrict__ perm, int64_t r_T,
                           float* __restrict__ out, int accum) {
  extern __shared__ float xf[];  // pf x ncol
  for (int i = threadIdx.x; i < pf * ncol; i += blockDim.x) {
    int j = i / ncol, col = i - j * ncol;
    int tc = ftcol[j];
    xf[i] = tc >= 0 ? x[(int64_t)tc * c_x + col0 + col] : 0.f;
  }
  __syncthreads();
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= r_T * ncol) return;
  int64_t p = idx / ncol;
  int col = (int)(idx - p * ncol);
  float acc = 0.f;
  if (pf > 0) {
    const float* r = F + p * pf;
    for (int j = 0; j < pf; j++) acc = fmaf(r[j], xf[j * ncol + col], acc);
  }
  for (int d = 0; d < gs.n; d++) {
    int32_t fk = gs.fk[d][p];
    if (fk >= 0) acc += gs.q[d][(int64_t)fk * ncol + col];
  }
  float* o = out + (int64_t)perm[p] * c_x + col0 + col;
  *o = accum ? *o + acc : acc;   // accum: a further group of gathered sources
}

// Narrow T x (stream block of C4 float4 per row, NC <= 2 operand columns): a
// thread per device row, the row loaded as float4s and both columns kept in
// registers; same fmaf order as k_lmm_main, so results are identical.  The
// result is written in DEVICE order (coalesced, dev[p*NC + c]) and put into
// target order by k_lmm_unperm's gathered reads: 100M scattered 4-byte
// writes (partial-sector read-modify-writes) cost more than the same number
// of scattered reads.
template <int C4, int NC>
__global__ void __launch_bounds__(256) k_lmm_narrow(const float4* __restrict__ F,
                                                    const int32_t* __restrict__ ftcol,
                                                    const float* __restrict__ x, int c_x, int col0,
                                                    GatherSet gs, int64_t r_T,
                                                    float* __restrict__ dev) {
  __shared__ float xf[C4 * 4 * NC];
  for (int i = threadIdx.x; i < C4 * 4 * NC; i += blockDim.x) {
    const int j = i / NC, col = i - j * NC;
    const int tc = ftcol[j];
    xf[i] = tc >= 0 ? x[(int64_t)tc * c_x + col0 + col] : 0.f;
  }
  __syncthreads();
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < r_T;
       p += (int64_t)gridDim.x * blockDim.x) {
    float4 v[C4];
#pragma unroll
    for (int q = 0; q < C4; q++) v[q] = F[p * C4 + q];
    float acc[NC];
#pragma unroll
    for (int c = 0; c < NC; c++) acc[c] = 0.f;
#pragma unroll
    for (int q = 0; q < C4; q++) {
      const float e4[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
#pragma unroll
      for (int e = 0; e < 4; e++)
#pragma unroll
        for (int c = 0; c < NC; c++) acc[c] = fmaf(e4[e], xf[(q * 4 + e) * NC + c], acc[c]);
    }
    for (int d = 0; d < gs.n; d++) {
      const int32_t fk = gs.fk[d][p];
      if (fk >= 0) {
#pragma unroll
        for (int c = 0; c < NC; c++) acc[c] += gs.q[d][(int64_t)fk * NC + c];
      }
    }
#pragma unroll
    for (int c = 0; c < NC; c++) dev[p * NC + c] = acc[c];
  }
}

// Wider T x (16..32 operand columns per chunk -- the dispatch gate below --
// stream block of C4 float4 per row): a
// warp per row at a time, lane = output column, grid-stride over rows.  The
// thread's x column lives in registers (loaded once), the row is one
// coalesced load broadcast by shuffle, and the target row is written as one
// contiguous run.  k_lmm_main spends a thread, a 64-bit division and a
// shared-memory refill of x per (row, column) block: ncu at C2-size k = 32
// shows it issue-bound at 35.6G warp instructions.  Same fmaf order, so
// results are identical.
template <int C4>
__global__ void __launch_bounds__(256) k_lmm_warp_rows(const float* __restrict__ F,
                                                       const int32_t* __restrict__ ftcol,
                                                       const float* __restrict__ x, int c_x,
                                                       int col0, int ncol, GatherSet gs,
                                                       const int32_t* __restrict__ perm,
                                                       int64_t r_T, float* __restrict__ out,
                                                       int o_pitch, int o_col0) {
  constexpr int PF = C4 * 4;
  const int lane = threadIdx.x & 31;
  const bool on = lane < ncol;
  float xr[PF];
#pragma unroll
  for (int j = 0; j < PF; j++) {
    const int tc = ftcol[j];
    xr[j] = (on && tc >= 0) ? x[(int64_t)tc * c_x + col0 + lane] : 0.f;
  }
  // R rows per warp iteration, all loads issued before the arithmetic
  // (one row at a time was latency-bound: ~37 ms flat in k at 100M rows)
  constexpr int R = 8;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t p0 = (blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5)) * R; p0 < r_T;
       p0 += nw * R) {
    float v[R], acc[R];
    int32_t tr[R];
#pragma unroll
    for (int r = 0; r < R; r++) {
      const int64_t p = p0 + r;
      v[r] = (lane < PF && p < r_T) ? F[p * PF + lane] : 0.f;
      tr[r] = p < r_T ? (perm ? perm[p] : (int32_t)p) : -1;   // perm null: device order out
      acc[r] = 0.f;
    }
#pragma unroll
    for (int j = 0; j < PF; j++)
#pragma unroll
      for (int r = 0; r < R; r++) acc[r] = fmaf(__shfl_sync(0xffffffffu, v[r], j), xr[j], acc[r]);
    for (int d = 0; d < gs.n; d++) {
      int32_t fk[R];
#pragma unroll
      for (int r = 0; r < R; r++) fk[r] = p0 + r < r_T ? gs.fk[d][p0 + r] : -1;
      float qv[R];
#pragma unroll
      for (int r = 0; r < R; r++) qv[r] = (fk[r] >= 0 && on) ? gs.q[d][(int64_t)fk[r] * ncol + lane] : 0.f;
#pragma unroll
      for (int r = 0; r < R; r++)
        if (fk[r] >= 0) acc[r] += qv[r];
    }
#pragma unroll
    for (int r = 0; r < R; r++)
      if (on && tr[r] >= 0) out[(int64_t)tr[r] * o_pitch + o_col0 + lane] = acc[r];
  }
}

// out[t, col0 + c] = dev[iperm[t], c] for ncol <= 32 columns: warp per
// target row, one contiguous row read (random) and one row write
// (sequential).  Scattered row WRITES cost ~2x scattered row reads on the
// B200 (tools/scatter_probe.py), so wide lmm outputs are produced in device
// order and gathered into target order here.
__global__ void __launch_bounds__(256) k_rows_unperm(const float* __restrict__ dev, int ncol,
                                                     const int32_t* __restrict__ iperm,
                                                     int64_t r_T, int c_x, int col0,
                                                     float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < r_T;
       t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t p = iperm[t];
    if (lane < ncol) out[t * c_x + col0 + lane] = dev[p * ncol + lane];
  }
}

// out[t, col0 + c] = dev[iperm[t], c]
template <int NC>
__global__ void k_lmm_unperm(const float* __restrict__ dev, const int32_t* __restrict__ iperm,
                             int64_t r_T, int c_x, int col0, float* __restrict__ out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= r_T) return;
  const int64_t p = iperm[t];
#pragma unroll
  for (int c = 0; c < NC; c++) out[t * c_x + col0 + c] = dev[p * NC + c];
}

template <int NC>
static void lmm_narrow_launch(int c4, unsigned nb, cudaStream_t s, const float* F,
                              const int32_t* ftcol, const float* x, int c_x, int col0,
                              const GatherSet& gs, const int32_t* iperm, int64_t r_T, float* dev,
                              float* out) {
  const float4* F4 = reinterpret_cast<const float4*>(F);
  switch (c4) {
#define LMN(C)                                                                         \
  case C:                                                                              \
    k_lmm_narrow<C, NC><<<nb, 256, 0, s>>>(F4, ftcol, x, c_x, col0, gs, r_T, dev); \
    break;
    LMN(1) LMN(2) LMN(3) LMN(4) LMN(5) LMN(6) LMN(7) LMN(8)
#undef LMN
    default: break;
  }
  k_lmm_unperm<NC><<<gridn(r_T), 256, 0, s>>>(dev, iperm, r_T, c_x, col0, out);
}


// Per-block partial of A^T Y over a contiguous row range, A = row-major
// (pitch) fp32 rows; Y rows either from a device-ordered fp64 buffer (bins)
// or from the strided target-order view through perm.  Rows are staged in
// 128-row chunks; each (a, y-column) pair is split over up to 8 row groups
// (fp32 within a chunk, fp64 across chunks, groups combined in a fixed
// order), so narrow outputs still use the whole CTA.  part[block][a*cy + c].
// (y columns per pass are capped so na * ny <= blockDim: with 32+ A columns
// and 9+ y columns the pairs past thread 255 were never computed.)
constexpr int TM_RC = 128;
constexpr int TM_AC = 40;    // A columns per pass
constexpr int TM_YC = 16;    // y columns per pass
template <bool BINS>
__global__ void __launch_bounds__(256) k_tmm_partial(const float* __restrict__ A, int pitch,
                                                     int acols, int64_t rows, YView yv,
                                                     const int32_t* __restrict__ perm,
                                                     const double* __restrict__ bins, int cy,
                                                     int64_t rows_per_block,
                                                     double* __restrict__ part) {
  extern __shared__ double acc[];  // acols * cy
  __shared__ float as_[TM_RC * (TM_AC + 1)];
  __shared__ float ys[TM_RC * (TM_YC + 1)];
  __shared__ float gsum[256];
  const int npair = acols * cy;
  for (int i = threadIdx.x; i < npair; i += blockDim.x) acc[i] = 0.0;
  const int64_t r0 = blockIdx.x * rows_per_block;
  const int64_t r1 = min(rows, r0 + rows_per_block);
  for (int64_t rb = r0; rb < r1; rb += TM_RC) {
    const int nr = (int)min64(TM_RC, r1 - rb);
    for (int a0 = 0; a0 < acols; a0 += TM_AC) {
      const int na = min(TM_AC, acols - a0);
      // at most one (a, y-column) pair per thread: na * ny <= blockDim
      const int ystep = min(TM_YC, max(1, (int)blockDim.x / na));
      for (int y0 = 0; y0 < cy; y0 += ystep) {
        const int ny = min(ystep, cy - y0);
        __syncthreads();
        for (int i = threadIdx.x; i < nr * na; i += blockDim.x) {
          const int r = i / na, c = i - r * na;
          as_[r * (TM_AC + 1) + c] = A[(rb + r) * pitch + a0 + c];
        }
        for (int i = threadIdx.x; i < nr * ny; i += blockDim.x) {
          const int r = i / ny, c = i - r * ny;
          float v;
          if (BINS) v = (float)bins[(rb + r) * cy + y0 + c];
          else v = yv.at(perm ? perm[rb + r] : rb + r, y0 + c);
          ys[r * (TM_YC + 1) + c] = v;
        }
        __syncthreads();
        const int np = na * ny;
        const int G = max(1, min(8, (int)blockDim.x / np));
        const int pr = threadIdx.x % np, grp = threadIdx.x / np;
        float sf = 0.f;
        if (grp < G) {
          const int a = pr / ny, c = pr - a * ny;
          for (int r = grp; r < nr; r += G)
            sf = fmaf(as_[r * (TM_AC + 1) + a], ys[r * (TM_YC + 1) + c], sf);
        }
        __syncthreads();
        if (grp < G && threadIdx.x < np * G) gsum[threadIdx.x] = sf;
        __syncthreads();
        for (int q = threadIdx.x; q < np; q += blockDim.x) {
          double t = 0.0;
          for (int g2 = 0; g2 < G; g2++) t += (double)gsum[g2 * np + q];
          const int a = q / ny, c = q - a * ny;
          acc[(a0 + a) * cy + y0 + c] += t;
        }
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < npair; i += blockDim.x)
    part[(int64_t)blockIdx.x * npair + i] = acc[i];
}

// Narrow A^T y (stream block with C4 float4 per row, CY <= 2 y columns): a
// thread per row holds the row and its y values in registers (fp32 products,
// fp64 every 64 rows), then a fixed-order block reduction -- the structure of
// the GLM fact pass without the gathers.  part[block][a*CY + c] as above.
template <int C4, int CY>
__global__ void __launch_bounds__(256) k_tmm_narrow(const float4* __restrict__ F, int64_t rows,
                                                    YView yv, const int32_t* __restrict__ perm,
                                                    int64_t rows_per_block,
                                                    double* __restrict__ part) {
  constexpr int NP = C4 * 4 * CY;
  __shared__ double wsum[8][NP];
  const int64_t r0 = blockIdx.x * rows_per_block;
  const int64_t r1 = min64(rows, r0 + rows_per_block);
  float acc[NP];
  double acc64[NP];
#pragma unroll
  for (int i = 0; i < NP; i++) {
    acc[i] = 0.f;
    acc64[i] = 0.0;
  }
  int n = 0;
  for (int64_t row = r0 + threadIdx.x; row < r1; row += blockDim.x) {
    const int64_t tr = perm ? (int64_t)perm[row] : row;
    float yc[CY];
#pragma unroll
    for (int c = 0; c < CY; c++) yc[c] = tr >= 0 ? yv.at(tr, c) : 0.f;
    float4 v[C4];
#pragma unroll
    for (int q = 0; q < C4; q++) v[q] = F[row * C4 + q];
#pragma unroll
    for (int q = 0; q < C4; q++) {
      const float e4[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
#pragma unroll
      for (int e = 0; e < 4; e++)
#pragma unroll
        for (int c = 0; c < CY; c++)
          acc[(q * 4 + e) * CY + c] = fmaf(e4[e], yc[c], acc[(q * 4 + e) * CY + c]);
    }
    if (++n == 64) {
#pragma unroll
      for (int i = 0; i < NP; i++) {
        acc64[i] += (double)acc[i];
        acc[i] = 0.f;
      }
      n = 0;
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NP; i++) {
    double v = acc64[i] + (double)acc[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) wsum[warp][i] = v;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NP; i += blockDim.x) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += wsum[w][i];
    part[(int64_t)blockIdx.x * NP + i] = t;
  }
}

template <int CY>
static void tmm_narrow_launch(int c4, unsigned nb, cudaStream_t s, const float* F, int64_t rows,
                              YView yv, const int32_t* perm, int64_t rpb, double* part) {
  const float4* F4 = reinterpret_cast<const float4*>(F);
  switch (c4) {
#define TMN(C) case C: k_tmm_narrow<C, CY><<<nb, 256, 0, s>>>(F4, rows, yv, perm, rpb, part); break;
    TMN(1) TMN(2) TMN(3) TMN(4) TMN(5) TMN(6) TMN(7) TMN(8)
#undef TMN
    default: break;
  }
}

// bins[j, col] = sum over members m of group j (ascending target row) of y'(m, col)
__global__ void k_group_bins(const int64_t* __restrict__ grp_ptr, const int32_t* __restrict__ grp_rows,
                             bool sorted, int64_t n_neg, int64_t rows, YView yv,
                             const int32_t* __restrict__ perm, int cy, double* __restrict__ bins) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= rows * cy) return;
  int64_t j = idx / cy;
  int col = (int)(idx - j * cy);
  int64_t m0 = grp_ptr[j], m1 = grp_ptr[j + 1];
  double s = 0.0;
  for (int64_t m = m0; m < m1; m++) {
    int64_t p = sorted ? n_neg + m : (int64_t)grp_rows[m];
    s += (double)yv.at(perm ? perm[p] : p, col);
  }
  bins[idx] = s;
}

// ydev[p*cy + c] = y(perm[p], c): the target-order operand read ONCE in
// device order, so the stream pass and the group bins that follow both read
// it sequentially instead of each gathering 4-byte values through perm.
__global__ void k_gather_y_dev(YView yv, const int32_t* __restrict__ perm, int64_t rows, int cy,
                               float* __restrict__ ydev) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= rows * cy) return;
  const int64_t p = idx / cy;
  const int c = (int)(idx - p * cy);
  const int32_t tr = perm[p];
  ydev[idx] = tr >= 0 ? yv.at(tr, c) : 0.f;
}

// tmp[tr*w + c] = y(tr, c0 + c) for a column-strided view (rmm's x^T):
// coalesced reads along each column, row-major chunk out.
__global__ void k_view_rows(YView yv, int64_t rows, int c0, int w, float* __restrict__ tmp) {
  const int64_t tr = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tr >= rows) return;
  for (int c = 0; c < w; c++) tmp[tr * w + c] = yv.at(tr, c0 + c);
}

// out[tcol[a] * os_t + col * os_c] += sum_b part[b][a*cy + col]  (fixed order)
__global__ void k_reduce_partials(const double* __restrict__ part, int nblocks, int acols,
                                  int cy, const int32_t* __restrict__ tcol, double* __restrict__ out,
                                  int64_t os_t, int64_t os_c) {
  // one warp per output pair: lanes stride the blocks, fixed xor tree
  const int i = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  const int npair = acols * cy;
  if (i >= npair) return;
  double s = 0.0;
  for (int b = lane; b < nblocks; b += 32) s += part[(int64_t)b * npair + i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const int a = i / cy, col = i - a * cy;
  const int tc = tcol[a];
  if (lane == 0 && tc >= 0) out[tc * os_t + col * os_c] += s;
}

__global__ void k_fill(float* p, int64_t n, float v) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

__global__ void k_gather_dev_order(const char* __restrict__ src, char* __restrict__ dst,
                                   const int32_t* __restrict__ perm, int64_t r_pad, int eb) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= r_pad) return;
  int32_t t = perm[p];
  for (int b = 0; b < eb; b++) dst[p * eb + b] = t >= 0 ? src[(int64_t)t * eb + b] : 0;
}

int launch_gather_rows_to_device_order(const fl_table* t, const void* src_target, void* dst_dev,
                                       int elem_bytes, cudaStream_t s) {
  k_gather_dev_order<<<gridn(t->r_pad), 256, 0, s>>>((const char*)src_target, (char*)dst_dev,
                                                     t->perm->as<int32_t>(), t->r_pad, elem_bytes);
  FL_CHECK_LAUNCH();
  return FL_OK;
}

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
#include "lmm_t5.cuh"

// ---------------------------------------------------------------------------
// More than MAX_GATHER gathered sources: the first group of MAX_GATHER rides
// the stream pass, every further group adds its gathered rows in another
// pass (same fp32 order per group; SURVEY.md a10 -- the reference takes any
// number of sources, ops.py:227-233)
static int do_lmm_many(fl_table* t, const float* x_dev, int c_x, float* out_dev, cudaStream_t s) {
  const int ng = (int)t->g.size();
  for (int col0 = 0; col0 < c_x; col0 += CX_CHUNK) {
    const int ncol = std::min(CX_CHUNK, c_x - col0);
    for (int d0 = 0; d0 < ng; d0 += MAX_GATHER) {
      GatherSet gs{};
      gs.n = std::min(MAX_GATHER, ng - d0);
      std::vector<float*> qs;
      for (int d = 0; d < gs.n; d++) {
        const GatherSrc& g = t->g[d0 + d];
        float* q = nullptr;
        FL_CUDA(cudaMallocAsync((void**)&q, g.rows * ncol * 4 + 16, s));
        qs.push_back(q);
        k_dim_q<<<gridn(g.rows * ncol), 256, (size_t)g.cols * ncol * 4, s>>>(
            g.S->as<float>(), g.pitch, g.cols, g.rows, g.d_tcol->as<int32_t>(), x_dev, c_x, col0,
            ncol, q);
        FL_CHECK_LAUNCH();
        gs.q[d] = q;
        gs.fk[d] = g.fk->as<int32_t>();
      }
      const bool first = d0 == 0;
      const int pf = first ? t->pf : 0;
      k_lmm_main<<<gridn(t->r_T * ncol), 256, (size_t)pf * ncol * 4, s>>>(
          pf ? t->F->as<float>() : nullptr, pf, pf ? t->d_f_tcol->as<int32_t>() : nullptr, x_dev,
          c_x, col0, ncol, gs, t->perm->as<int32_t>(), t->r_T, out_dev, first ? 0 : 1);
      FL_CHECK_LAUNCH();
      for (float* q : qs) FL_CUDA(cudaFreeAsync(q, s));
    }
  }
  return FL_OK;
}

int do_lmm(fl_table* t, const float* x_dev, int c_x, float* out_dev, cudaStream_t s) {
  if ((int)t->g.size() > MAX_GATHER) return do_lmm_many(t, x_dev, c_x, out_dev, s);
  for (int col0 = 0; col0 < c_x; col0 += CX_CHUNK) {
    int ncol = std::min(CX_CHUNK, c_x - col0);
    GatherSet gs{};
    gs.n = (int)t->g.size();
    std::vector<float*> qs;
    for (int d = 0; d < gs.n; d++) {
      const GatherSrc& g = t->g[d];
      float* q = nullptr;
      FL_CUDA(cudaMallocAsync((void**)&q, g.rows * ncol * 4 + 16, s));
      qs.push_back(q);
      size_t sm = (size_t)g.cols * ncol * 4;
      k_dim_q<<<gridn(g.rows * ncol), 256, sm, s>>>(g.S->as<float>(), g.pitch, g.cols, g.rows,
                                                    g.d_tcol->as<int32_t>(), x_dev, c_x, col0,
                                                    ncol, q);
      FL_CHECK_LAUNCH();
      gs.q[d] = q;
      gs.fk[d] = g.fk->as<int32_t>();
    }
    const float* F = t->F ? t->F->as<float>() : nullptr;
    // tcgen05 pass (lmm_t5.cuh, opt-in FL_LMM_T5=1) for >= 8 operand columns
    // over a narrow stream block past L2 (FL_LMM_T5_MIN_ROWS, default 8M
    // rows): F x_F on the tensor cores, the epilogue writes whole rows.  It
    // is bound by the scattered target-order row writes like the row-wise
    // kernels and measured slower at C2 size (k = 32: 13.3 vs 12.5 ms)
    {
      const char* mr5 = getenv("FL_LMM_T5_MIN_ROWS");
      const int64_t min5 = mr5 ? atoll(mr5) : (int64_t)1 << 23;
      const char* on5 = getenv("FL_LMM_T5");   // opt-in: measured slower
      if (on5 && atoi(on5) != 0 && F && t->pf <= 28 && ncol >= 8 && t->r_T >= min5) {
        const L5Geom g5 = l5_geom(gs.n);
        CUtensorMap tm;
        int rc = make_tmap_2d(&tm, F, (uint64_t)t->r_pad, (uint64_t)t->pf, (uint64_t)t->pf * 4,
                              L5_TILE, 32, 128);
        if (rc) return rc;
        static bool attr_set = false;
        if (!attr_set) {
          FL_CUDA(raise_smem_limit(k_lmm_t5, (int)(l5_geom(MAX_GATHER).total + 1024)));
          attr_set = true;
        }
        LmT5Args la{};
        la.pf = t->pf;
        la.c_x = c_x;
        la.col0 = col0;
        la.ncol = ncol;
        la.r_T = t->r_T;
        la.ntiles = t->r_pad / L5_TILE;
        la.ng = gs.n;
        for (int d = 0; d < gs.n; d++) {
          la.fk[d] = gs.fk[d];
          la.q[d] = gs.q[d];
        }
        la.x = x_dev;
        la.f_tcol = t->d_f_tcol->as<int32_t>();
        la.perm = t->perm->as<int32_t>();
        // FL_LMM_T5=2: device-order rows (sequential) + a row gather into
        // target order, instead of scattered row writes
        const bool devrows = atoi(on5) >= 2;
        const bool plain = atoi(on5) == 3;   // experiment: cudaMalloc'd row buffer (page size)
        float* dst = out_dev;
        la.o_pitch = c_x;
        la.o_col0 = col0;
        if (devrows) {
          if (plain) FL_CUDA(cudaMalloc((void**)&dst, (size_t)t->r_T * ncol * 4 + 16));
          else FL_CUDA(cudaMallocAsync((void**)&dst, (size_t)t->r_T * ncol * 4 + 16, s));
          la.o_pitch = ncol;
          la.o_col0 = 0;
          la.dev_rows = 1;
        }
        la.out = dst;
        const unsigned nb = (unsigned)std::max<int64_t>(1, std::min<int64_t>(la.ntiles, t->sm_count));
        k_lmm_t5<<<nb, L5_THREADS, g5.total + 1024, s>>>(tm, la, g5);
        FL_CHECK_LAUNCH();
        if (devrows) {
          const unsigned gb = (unsigned)std::min<int64_t>(ceil_div(t->r_T, 8), 16 * (int64_t)t->sm_count);
          k_rows_unperm<<<gb, 256, 0, s>>>(dst, ncol, t->iperm->as<int32_t>(), t->r_T, c_x, col0,
                                           out_dev);
          FL_CHECK_LAUNCH();
          if (plain) {
            FL_CUDA(cudaStreamSynchronize(s));
            FL_CUDA(cudaFree(dst));
          } else {
            FL_CUDA(cudaFreeAsync(dst, s));
          }
        }
        for (float* q : qs) FL_CUDA(cudaFreeAsync(q, s));
        continue;
      }
    }
    // narrow stream block: thread-per-row kernel, float4 row loads, device-
    // order output + gathered unpermute.  Only past L2 (>= 8M rows by
    // default): below that the scattered writes stay in L2 and the extra
    // launch costs more than it saves (C1, 1M rows: 46 -> 51 us).
    const char* mr = getenv("FL_LMM_NARROW_MIN_ROWS");
    const int64_t min_rows = mr ? atoll(mr) : (int64_t)1 << 23;
    if (F && t->pf % 4 == 0 && t->pf <= 32 && ncol <= 4 && t->r_T >= min_rows &&
        !getenv("FL_NO_NARROW_LMM")) {
      const unsigned nb = (unsigned)std::min<int64_t>(gridn(t->r_T), 8 * (int64_t)t->sm_count);
      float* dev = nullptr;
      FL_CUDA(cudaMallocAsync((void**)&dev, t->r_T * ncol * 4 + 16, s));
      const int32_t* ftcol = t->d_f_tcol->as<int32_t>();
      const int32_t* iperm = t->iperm->as<int32_t>();
      switch (ncol) {
#define LMC(NC)                                                                              \
  case NC:                                                                                   \
    lmm_narrow_launch<NC>(t->pf / 4, nb, s, F, ftcol, x_dev, c_x, col0, gs, iperm, t->r_T, dev, \
                          out_dev);                                                          \
    break;
        LMC(1) LMC(2) LMC(3) LMC(4)
#undef LMC
        default: break;
      }
      FL_CUDA(cudaFreeAsync(dev, s));
    } else if (F && t->pf % 4 == 0 && t->pf <= 32 && ncol >= 16 && !getenv("FL_NO_NARROW_LMM")) {
      const unsigned nb =
          (unsigned)std::min<int64_t>(ceil_div(t->r_T, 64), 8 * (int64_t)t->sm_count);
      const int32_t* ftcol = t->d_f_tcol->as<int32_t>();
      // scattered row writes straight from the pass; FL_LMM_UNPERM=1: device-
      // order rows + a row gather into target order (measured slower: the
      // pass is issue-bound either way, C2 k = 32 12.5 -> 21.0 ms)
      const char* up = getenv("FL_LMM_UNPERM");
      const bool unperm = up && atoi(up) == 1;
      const int32_t* perm = unperm ? nullptr : t->perm->as<int32_t>();
      float* dst = out_dev;
      int dc = c_x, d0 = col0;
      if (unperm) {
        FL_CUDA(cudaMallocAsync((void**)&dst, t->r_T * ncol * 4 + 16, s));
        dc = ncol;
        d0 = 0;
      }
      switch (t->pf / 4) {
#define LMW(C)                                                                                 \
  case C:                                                                                      \
    k_lmm_warp_rows<C><<<nb, 256, 0, s>>>(F, ftcol, x_dev, c_x, col0, ncol, gs, perm, t->r_T, \
                                          dst, dc, d0);                                        \
    break;
        LMW(1) LMW(2) LMW(3) LMW(4) LMW(5) LMW(6) LMW(7) LMW(8)
#undef LMW
        default: break;
      }
      if (unperm) {
        FL_CHECK_LAUNCH();
        const unsigned gb = (unsigned)std::min<int64_t>(ceil_div(t->r_T, 8), 16 * (int64_t)t->sm_count);
        k_rows_unperm<<<gb, 256, 0, s>>>(dst, ncol, t->iperm->as<int32_t>(), t->r_T, c_x, col0,
                                         out_dev);
        FL_CHECK_LAUNCH();
        FL_CUDA(cudaFreeAsync(dst, s));
      }
    } else {
      size_t sm = (size_t)t->pf * ncol * 4;
      k_lmm_main<<<gridn(t->r_T * ncol), 256, sm, s>>>(
          F, t->pf, t->pf ? t->d_f_tcol->as<int32_t>() : nullptr, x_dev, c_x, col0, ncol, gs,
          t->perm->as<int32_t>(), t->r_T, out_dev, 0);
    }
    FL_CHECK_LAUNCH();
    for (float* q : qs) FL_CUDA(cudaFreeAsync(q, s));
  }
  return FL_OK;
}

#include "tmm_t5.cuh"

static int tlmm_impl(fl_table* t, YView yv_in, int cy, double* out, int64_t os_t, int64_t os_c,
                     cudaStream_t s, bool dev_order, bool with_f);

// S_d^T bins (bins = I_d^T y, r_d x cy fp64) into out: per-CTA partials
// (k_tmm_partial) reduced in CTA order
static int tlmm_bins_product(fl_table* t, const GatherSrc& g, const double* bins, int cy,
                             double* out, int64_t os_t, int64_t os_c, cudaStream_t s) {
  if (g.rows <= 0 || g.cols <= 0) return FL_OK;
  if (g.cols <= 64 && cy <= 32) {
    int64_t nb = std::max<int64_t>(1, std::min<int64_t>(ceil_div(g.rows, 256), 16 * (int64_t)t->sm_count));
    const int64_t rpc = round_up(ceil_div(g.rows, nb), 64);
    nb = ceil_div(g.rows, rpc);
    double* part = nullptr;
    FL_CUDA(cudaMallocAsync((void**)&part, (size_t)nb * g.cols * cy * 8, s));
    k_sbins<<<(unsigned)nb, 128, 0, s>>>(g.S->as<float>(), g.pitch, g.cols, bins, cy, g.rows, rpc,
                                         part);
    FL_CHECK_LAUNCH();
    k_reduce_partials<<<gridn((int64_t)g.cols * cy * 32), 256, 0, s>>>(
        part, (int)nb, g.cols, cy, g.d_tcol->as<int32_t>(), out, os_t, os_c);
    FL_CHECK_LAUNCH();
    FL_CUDA(cudaFreeAsync(part, s));
    return FL_OK;
  }
  int64_t nb = std::min<int64_t>(std::max<int64_t>(1, ceil_div(g.rows, 2048)), 4 * t->sm_count);
  const int64_t rpb = round_up(ceil_div(g.rows, nb), 32);
  nb = ceil_div(g.rows, rpb);
  const int npair = g.cols * cy;
  const size_t sm = (size_t)npair * 8;
  double* part = nullptr;
  FL_CUDA(cudaMallocAsync((void**)&part, nb * npair * 8, s));
  FL_CUDA(raise_smem_limit(k_tmm_partial<true>, (int)sm));
  k_tmm_partial<true><<<(unsigned)nb, 256, sm, s>>>(g.S->as<float>(), g.pitch, g.cols, g.rows,
                                                    YView{nullptr, 0, 0}, nullptr, bins, cy, rpb,
                                                    part);
  FL_CHECK_LAUNCH();
  k_reduce_partials<<<gridn((int64_t)npair * 32), 256, 0, s>>>(part, (int)nb, g.cols, cy,
                                                               g.d_tcol->as<int32_t>(), out, os_t,
                                                               os_c);
  FL_CHECK_LAUNCH();
  FL_CUDA(cudaFreeAsync(part, s));
  return FL_OK;
}

// T^T y for 3..32 operand columns with the stream block on tcgen05
// (tmm_t5.cuh): y laid out once as YD (device order, 32-column rows; a
// column-strided view -- rmm's x^T -- is first transposed in target order,
// sequential on both sides, then gathered by rows), one tensor-core pass
// over F and YD, then per gathered source the group sums of YD (warp per
// group, k_group_bins' ascending fp64 order) and the S_d^T bins product
static int tlmm_wide_t5(fl_table* t, YView yv, int cy, double* out, int64_t os_t, int64_t os_c,
                        cudaStream_t s, bool dev_order) {
  const int64_t r_T = t->r_T, r_pad = t->r_pad;
  const unsigned gb = (unsigned)std::min<int64_t>(ceil_div(r_T, 32), 16 * (int64_t)t->sm_count);
  const int32_t* perm = dev_order ? nullptr : t->perm->as<int32_t>();
  // y's rows are read where they lie (target order, through perm) by the
  // pass and by the group sums: a row-major y with 16-byte rows directly,
  // any other view (rmm's column-strided x^T) after one sequential copy into
  // 32-column target-order rows.  Wider than 16 columns (or FL_TMM_YD=1): y
  // is laid out in device order first (YD) and bulk-copied per tile.
  // (measured at C2 size: gathering wins up to 16 columns -- k = 8 / 16
  // transpose_lmm 9.3 / 9.6 ms vs 11.1 / 11.2 with YD -- and loses at 32:
  // 14.7 vs 11.3 ms)
  const char* yde = getenv("FL_TMM_YD");
  const bool use_yd = yde ? atoi(yde) != 0 : cy > 16;
  float* tmp = nullptr;
  const float* yg = nullptr;
  int yp = 32;
  if (!use_yd && yv.sc == 1 && yv.sr == cy && cy % 4 == 0 && ((uintptr_t)yv.base & 15) == 0) {
    yg = yv.base;
    yp = cy;
  } else {
    FL_CUDA(cudaMallocAsync((void**)&tmp, (size_t)r_pad * 32 * 4, s));
    if (r_pad > r_T) FL_CUDA(cudaMemsetAsync(tmp + r_T * 32, 0, (size_t)(r_pad - r_T) * 32 * 4, s));
    if (yv.sc > yv.sr && yv.sr == 1) {
      // column-strided (rmm's x^T): transpose in target order, sequential both ways
      float* xt = tmp;
      if (use_yd && perm) FL_CUDA(cudaMallocAsync((void**)&xt, (size_t)r_T * 32 * 4, s));
      k_xt32<<<(unsigned)std::min<int64_t>(ceil_div(r_T, 128), 8 * (int64_t)t->sm_count), 256, 0,
               s>>>(yv, cy, r_T, xt);
      FL_CHECK_LAUNCH();
      if (use_yd && perm) {
        k_ydev32_rows<<<gb, 256, 0, s>>>(YView{xt, 32, 1}, 32, r_T, perm, tmp);
        FL_CHECK_LAUNCH();
        FL_CUDA(cudaFreeAsync(xt, s));
      }
    } else {
      k_ydev32_rows<<<gb, 256, 0, s>>>(yv, cy, r_T, use_yd ? perm : nullptr, tmp);
      FL_CHECK_LAUNCH();
    }
    yg = tmp;
  }
  // the rows of yg are in device order when YD was built (or y is already)
  const int32_t* yperm = (use_yd || dev_order) ? nullptr : perm;
  int rc = FL_OK;
  static bool attr = false;
  if (!attr) {
    FL_CUDA(raise_smem_limit(k_tmm_t5, (int)M5_SMEM));
    attr = true;
  }
  const int64_t ntiles = r_pad / M5_TILE;
  const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, t->sm_count));
  double* part = nullptr;
  FL_CUDA(cudaMallocAsync((void**)&part, (size_t)nb * t->pf * cy * 8, s));
  if (use_yd)   // YD: one bulk copy per tile
    k_tmm_t5<<<nb, M5_THREADS, M5_SMEM, s>>>(t->F->as<float>(), yg, t->pf, cy, ntiles, part,
                                             nullptr, 0, nullptr, r_T);
  else          // rows gathered in the pass
    k_tmm_t5<<<nb, M5_THREADS, M5_SMEM, s>>>(t->F->as<float>(), nullptr, t->pf, cy, ntiles, part,
                                             yg, yp, yperm, r_T);
  FL_CHECK_LAUNCH();
  k_reduce_partials<<<gridn((int64_t)t->pf * cy * 32), 256, 0, s>>>(
      part, nb, t->pf, cy, t->d_f_tcol->as<int32_t>(), out, os_t, os_c);
  FL_CHECK_LAUNCH();
  FL_CUDA(cudaFreeAsync(part, s));
  for (auto& g : t->g) {
    double* bins = nullptr;
    FL_CUDA(cudaMallocAsync((void**)&bins, g.rows * cy * 8 + 16, s));
    k_group_bins32<<<(unsigned)std::min<int64_t>(ceil_div(g.rows, 8), 32 * (int64_t)t->sm_count),
                     256, 0, s>>>(g.grp_ptr->as<int64_t>(),
                                  g.grp_rows ? g.grp_rows->as<int32_t>() : nullptr, g.sorted,
                                  g.n_neg, g.rows, yg, yp, yperm, cy, bins);
    FL_CHECK_LAUNCH();
    rc = tlmm_bins_product(t, g, bins, cy, out, os_t, os_c, s);
    if (rc) return rc;
    FL_CUDA(cudaFreeAsync(bins, s));
  }
  if (tmp) FL_CUDA(cudaFreeAsync(tmp, s));
  return FL_OK;
}

static int tmm_t5_min_cols() {
  static const int v = [] {
    const char* e = getenv("FL_TMM_T5_MIN");
    return e ? atoi(e) : 6;
  }();
  return v;
}

// generic T^T y with strided y view and strided fp64 output
int do_tlmm(fl_table* t, YView yv_in, int cy, double* out, int64_t os_t, int64_t os_c,
            cudaStream_t s, bool dev_order) {
  bool wide = t->pf > 0 && t->pf <= 28 && t->pf % 4 == 0 && cy >= tmm_t5_min_cols() && cy <= 32 &&
              t->r_T > 0 &&
              t->r_T <= (int64_t)INT32_MAX - M5_TILE && !getenv("FL_NO_TMM_T5");
  for (const auto& g : t->g)
    if ((size_t)g.cols * cy * 8 > 190 * 1024) wide = false;   // bins product smem
  if (wide) return tlmm_wide_t5(t, yv_in, cy, out, os_t, os_c, s, dev_order);
  return tlmm_impl(t, yv_in, cy, out, os_t, os_c, s, dev_order, true);
}

static int tlmm_impl(fl_table* t, YView yv_in, int cy, double* out, int64_t os_t, int64_t os_c,
                     cudaStream_t s, bool dev_order, bool with_f) {
  const int sms = t->sm_count;
  if (cy > 1 && yv_in.sc > yv_in.sr && t->r_T > 0 && !getenv("FL_NO_VIEW_ROWS")) {
    // Column-strided y (rmm: x^T of a k x r_T row-major x).  Every device-
    // order read of it would be one 32-byte sector per 4-byte value; make
    // row-major 8-column chunks first (sequential on both sides), then run
    // each chunk as an ordinary row-major T^T y.
    constexpr int VW = 8;
    float* tmp = nullptr;
    FL_CUDA(cudaMallocAsync((void**)&tmp, t->r_T * VW * 4 + 16, s));
    for (int c0 = 0; c0 < cy; c0 += VW) {
      const int w = std::min(VW, cy - c0);
      k_view_rows<<<gridn(t->r_T), 256, 0, s>>>(yv_in, t->r_T, c0, w, tmp);
      FL_CHECK_LAUNCH();
      const int rc = tlmm_impl(t, YView{tmp, w, 1}, w, out + c0 * os_c, os_t, os_c, s, dev_order, with_f);
      if (rc) return rc;
    }
    FL_CUDA(cudaFreeAsync(tmp, s));
    return FL_OK;
  }
  if (cy > 8 && !getenv("FL_NO_VIEW_ROWS")) {
    // wide y: 8-column chunks, each through the narrow passes below (C2-size
    // 32 columns: 67.8 ms in one staged pass -> 4 chunks)
    for (int c0 = 0; c0 < cy; c0 += 8) {
      const int w = std::min(8, cy - c0);
      const int rc = tlmm_impl(t, YView{yv_in.base + (int64_t)c0 * yv_in.sc, yv_in.sr, yv_in.sc},
                               w, out + c0 * os_c, os_t, os_c, s, dev_order, with_f);
      if (rc) return rc;
    }
    return FL_OK;
  }
  // With gathered sources there are two consumers of y in device order:
  // gather it once (bit-identical values; perm == nullptr means "already in
  // device order" to the kernels below).
  YView yv = yv_in;
  // dev_order: y is already in device row order (trainer-internal operands)
  const int32_t* yperm = dev_order ? nullptr : t->perm->as<int32_t>();
  float* ydev = nullptr;
  if (!dev_order && !t->g.empty() && t->r_T > 0 && !getenv("FL_NO_Y_DEVORDER")) {
    FL_CUDA(cudaMallocAsync((void**)&ydev, t->r_T * cy * 4 + 16, s));
    k_gather_y_dev<<<gridn(t->r_T * cy), 256, 0, s>>>(yv_in, yperm, t->r_T, cy, ydev);
    FL_CHECK_LAUNCH();
    yv = YView{ydev, cy, 1};
    yperm = nullptr;
  }
  auto launch_tmm = [&](const float* A, int pitch, int acols, int64_t rows, const double* bins,
                        const int32_t* tcol) -> int {
    if (rows <= 0 || acols <= 0) return FL_OK;
    int64_t nb = std::min<int64_t>(std::max<int64_t>(1, ceil_div(rows, 2048)), 4 * sms);
    int64_t rpb = round_up(ceil_div(rows, nb), 32);
    nb = ceil_div(rows, rpb);
    if (!bins && pitch == acols && acols % 4 == 0 && acols <= 32 && cy <= 8) {
      // narrow stream block: thread-per-row kernel (registers, no staging),
      // one pass per pair of y columns (C2-size 3-column T^T y: 15.4 ms
      // through k_tmm_partial's perm-staged tiles -> two streaming passes)
      double* part = nullptr;
      FL_CUDA(cudaMallocAsync((void**)&part, nb * acols * 2 * 8, s));
      for (int c0 = 0; c0 < cy; c0 += 2) {
        const int w = std::min(2, cy - c0);
        const YView sub{yv.base + (int64_t)c0 * yv.sc, yv.sr, yv.sc};
        if (w == 1)
          tmm_narrow_launch<1>(acols / 4, (unsigned)nb, s, A, rows, sub, yperm,
                               rpb, part);
        else
          tmm_narrow_launch<2>(acols / 4, (unsigned)nb, s, A, rows, sub, yperm,
                               rpb, part);
        FL_CHECK_LAUNCH();
        k_reduce_partials<<<gridn((int64_t)acols * w * 32), 256, 0, s>>>(part, (int)nb, acols, w, tcol,
                                                           out + c0 * os_c, os_t, os_c);
        FL_CHECK_LAUNCH();
      }
      FL_CUDA(cudaFreeAsync(part, s));
      return FL_OK;
    }
    int npair = acols * cy;
    size_t sm = (size_t)npair * 8;
    if (sm > 190 * 1024) {
      set_error("tlmm: %d x %d output too wide for one pass", acols, cy);
      return FL_ERR_OP;
    }
    double* part = nullptr;
    FL_CUDA(cudaMallocAsync((void**)&part, nb * npair * 8, s));
    if (bins) {
      FL_CUDA(raise_smem_limit(k_tmm_partial<true>, (int)sm));
      k_tmm_partial<true><<<(unsigned)nb, 256, sm, s>>>(A, pitch, acols, rows, yv, nullptr, bins,
                                                        cy, rpb, part);
    } else {
      FL_CUDA(raise_smem_limit(k_tmm_partial<false>, (int)sm));
      k_tmm_partial<false><<<(unsigned)nb, 256, sm, s>>>(A, pitch, acols, rows, yv,
                                                         yperm, nullptr, cy, rpb,
                                                         part);
    }
    FL_CHECK_LAUNCH();
    k_reduce_partials<<<gridn((int64_t)npair * 32), 256, 0, s>>>(part, (int)nb, acols, cy, tcol, out, os_t, os_c);
    FL_CHECK_LAUNCH();
    FL_CUDA(cudaFreeAsync(part, s));
    return FL_OK;
  };
  int rc;
  if (t->pf > 0 && with_f) {
    rc = launch_tmm(t->F->as<float>(), t->pf, t->pf, t->r_T, nullptr, t->d_f_tcol->as<int32_t>());
    if (rc) return rc;
  }
  for (auto& g : t->g) {
    double* bins = nullptr;
    FL_CUDA(cudaMallocAsync((void**)&bins, g.rows * cy * 8 + 16, s));
    k_group_bins<<<gridn(g.rows * cy), 256, 0, s>>>(
        g.grp_ptr->as<int64_t>(), g.grp_rows ? g.grp_rows->as<int32_t>() : nullptr, g.sorted,
        g.n_neg, g.rows, yv, yperm, cy, bins);
    FL_CHECK_LAUNCH();
    rc = launch_tmm(g.S->as<float>(), g.pitch, g.cols, g.rows, bins, g.d_tcol->as<int32_t>());
    if (rc) return rc;
    FL_CUDA(cudaFreeAsync(bins, s));
  }
  if (ydev) FL_CUDA(cudaFreeAsync(ydev, s));
  return FL_OK;
}

}  // namespace flb

using namespace flb;

#define FL_REQUIRE_TABLE(t)                                  \
  do {                                                       \
    if (!(t) || !(t)->finalized) {                           \
      set_error("table is null or not finalized");           \
      return FL_ERR_ARG;                                     \
    }                                                        \
    FL_CUDA(cudaSetDevice((t)->device));                     \
  } while (0)

extern "C" {

int fl_lmm(fl_table* t, const float* x, int32_t c_x, float* out, void* stream) {
  FL_REQUIRE_TABLE(t);
  if (c_x < 1 || !x || !out) {
    set_error("lmm: bad operand");
    return FL_ERR_SHAPE;
  }
  cudaStream_t s = (cudaStream_t)stream;
  float *xd, *od;
  bool xo, oo;
  int rc = to_device(x, (size_t)t->c_T * c_x, s, &xd, &xo);
  if (rc) return rc;
  rc = out_buffer(out, (size_t)t->r_T * c_x, s, &od, &oo);
  if (rc) return rc;
  rc = do_lmm(t, xd, c_x, od, s);
  if (rc) return rc;
  if (xo) FL_CUDA(cudaFreeAsync(xd, s));
  return finish_out(out, od, oo, (size_t)t->r_T * c_x, s);
}

int fl_tlmm(fl_table* t, const float* y, int32_t c_y, double* out, void* stream) {
  FL_REQUIRE_TABLE(t);
  if (c_y < 1 || !y || !out) {
    set_error("transpose_lmm: bad operand");
    return FL_ERR_SHAPE;
  }
  cudaStream_t s = (cudaStream_t)stream;
  float* yd;
  double* od;
  bool yo, oo;
  int rc = to_device(y, (size_t)t->r_T * c_y, s, &yd, &yo);
  if (rc) return rc;
  rc = out_buffer(out, (size_t)t->c_T * c_y, s, &od, &oo);
  if (rc) return rc;
  FL_CUDA(cudaMemsetAsync(od, 0, (size_t)t->c_T * c_y * 8, s));
  rc = do_tlmm(t, YView{yd, c_y, 1}, c_y, od, c_y, 1, s);
  if (rc) return rc;
  if (yo) FL_CUDA(cudaFreeAsync(yd, s));
  return finish_out(out, od, oo, (size_t)t->c_T * c_y, s);
}

int fl_rmm(fl_table* t, const float* x, int32_t r_x, double* out, void* stream) {
  FL_REQUIRE_TABLE(t);
  if (r_x < 1 || !x || !out) {
    set_error("rmm: bad operand");
    return FL_ERR_SHAPE;
  }
  cudaStream_t s = (cudaStream_t)stream;
  float* xd;
  double* od;
  bool xo, oo;
  int rc = to_device(x, (size_t)r_x * t->r_T, s, &xd, &xo);
  if (rc) return rc;
  rc = out_buffer(out, (size_t)r_x * t->c_T, s, &od, &oo);
  if (rc) return rc;
  FL_CUDA(cudaMemsetAsync(od, 0, (size_t)r_x * t->c_T * 8, s));
  // y'(target row, col) = x[col, target row]; out[col, tcol]
  rc = do_tlmm(t, YView{xd, 1, t->r_T}, r_x, od, 1, t->c_T, s);
  if (rc) return rc;
  if (xo) FL_CUDA(cudaFreeAsync(xd, s));
  return finish_out(out, od, oo, (size_t)r_x * t->c_T, s);
}

int fl_row_sum(fl_table* t, float* out, void* stream) {
  FL_REQUIRE_TABLE(t);
  cudaStream_t s = (cudaStream_t)stream;
  float* ones;
  FL_CUDA(cudaMallocAsync((void**)&ones, t->c_T * 4 + 16, s));
  k_fill<<<gridn(t->c_T), 256, 0, s>>>(ones, t->c_T, 1.0f);
  FL_CHECK_LAUNCH();
  float* od;
  bool oo;
  int rc = out_buffer(out, (size_t)t->r_T, s, &od, &oo);
  if (rc) return rc;
  rc = do_lmm(t, ones, 1, od, s);
  if (rc) return rc;
  FL_CUDA(cudaFreeAsync(ones, s));
  return finish_out(out, od, oo, (size_t)t->r_T, s);
}

int fl_col_sum(fl_table* t, double* out, void* stream) {
  FL_REQUIRE_TABLE(t);
  cudaStream_t s = (cudaStream_t)stream;
  float* ones;
  FL_CUDA(cudaMallocAsync((void**)&ones, t->r_T * 4 + 16, s));
  k_fill<<<gridn(t->r_T), 256, 0, s>>>(ones, t->r_T, 1.0f);
  FL_CHECK_LAUNCH();
  double* od;
  bool oo;
  int rc = out_buffer(out, (size_t)t->c_T, s, &od, &oo);
  if (rc) return rc;
  FL_CUDA(cudaMemsetAsync(od, 0, (size_t)t->c_T * 8, s));
  rc = do_tlmm(t, YView{ones, 1, 0}, 1, od, 1, 0, s);
  if (rc) return rc;
  FL_CUDA(cudaFreeAsync(ones, s));
  return finish_out(out, od, oo, (size_t)t->c_T, s);
}

}  // extern "C"
