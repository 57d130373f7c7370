// Factorized crossprod T^T T (the north star's crossprod; the reference has
// no operator for it -- SURVEY.md §8 a13 gives the composition over
// ops.py:219-271, transpose_lmm(lmm(I))).  Nothing is materialized:
//
//   T^T T = sum_{k,j} M_k S_k^T (I_k^T I_j) S_j M_j^T
//
// and in the device layout (stream block F = every injective source, already
// expanded in device row order; gathered sources S_d with FK vectors) the
// blocks are
//
//   F x F   F^T F                              one pass over the device rows
//   d x F   S_d^T Z_d,    Z_d  = I_d^T F        group sums per dimension row
//   d x d   S_d^T diag(n_d) S_d                 n_d = fanout of each row
//   d x e   S_d^T Y_de,   Y_de = I_d^T (I_e S_e)   (e after d; mirrored)
//
// so the cost is one read of F for the Gram, one grouped read of F (and of
// the gathered rows of later dimensions) for Z / Y, and dimension-sized
// Grams.  Every reduction is fixed-order: fp32 products summed in fp32 over a
// 64-row staged tile, fp64 across tiles and CTAs (per-CTA partials, then a
// warp-per-pair reduction in CTA order).  Group sums run in fp64 in
// ascending member order (the reference's _group_sum order,
// _kernels.py:252-288) and are stored as fp32 operands of the next Gram.
#include <algorithm>

#include "internal.h"
#include "tc05.cuh"

namespace flb {
namespace {

constexpr int GT = 32;      // output tile (A columns x B columns) per CTA
constexpr int GROWS = 64;   // rows staged per tile

// partial[cta][i][k] = sum over this CTA's rows r of w(r) A[r][a0+i] B[r][b0+k]
// A / B row-major fp32 with pitches pa / pb; w(r) = grp_ptr[r+1] - grp_ptr[r]
// when wptr is given (fanout weights of S_d^T diag(n_d) S_d), else 1.
// Each thread owns a 4 x 4 micro tile of the output; the micro tiles of the
// CTA's tile are replicated over `groups` thread groups that take
// interleaved rows of every staged tile, and the groups are summed in a
// fixed order at the end.
__global__ void __launch_bounds__(256) k_gram(const float* __restrict__ A, int pa, int acols,
                                              const float* __restrict__ B, int pb, int bcols,
                                              int64_t rows, int64_t rows_per_cta,
                                              const int64_t* __restrict__ wptr,
                                              double* __restrict__ part) {
  __shared__ __align__(16) float As[GROWS][GT + 4];
  __shared__ __align__(16) float Bs[GROWS][GT + 4];
  __shared__ double red[GT * GT];
  const int tile = blockIdx.z * gridDim.y + blockIdx.y;   // z: A tile, y: B tile
  const int ta0 = blockIdx.z * GT, tb0 = blockIdx.y * GT;
  const int ta = min(GT, acols - ta0), tb = min(GT, bcols - tb0);
  const int ma = (ta + 3) / 4, mb = (tb + 3) / 4;
  const int micro = ma * mb;
  const int groups = max(1, 256 / micro);
  const int tid = threadIdx.x;
  const int grp = tid / micro, mt = tid - grp * micro;
  const bool active = grp < groups;
  const int i0 = (mt / mb) * 4, k0 = (mt % mb) * 4;

  const int64_t r_begin = blockIdx.x * rows_per_cta;
  const int64_t r_end = min64(rows, r_begin + rows_per_cta);
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int k = 0; k < 4; k++) acc[i][k] = 0.0;

  for (int64_t r0 = r_begin; r0 < r_end; r0 += GROWS) {
    const int nr = (int)min64(GROWS, r_end - r0);
    __syncthreads();
    for (int e = tid; e < GROWS * GT; e += 256) {
      const int r = e / GT, c = e - r * GT;
      float av = 0.f, bv = 0.f;
      if (r < nr) {
        const int64_t row = r0 + r;
        if (c < ta) {
          av = A[row * pa + ta0 + c];
          if (wptr) av *= (float)(wptr[row + 1] - wptr[row]);
        }
        if (c < tb) bv = B[row * pb + tb0 + c];
      }
      As[r][c] = av;
      Bs[r][c] = bv;
    }
    __syncthreads();
    if (active) {
      float f[4][4];
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int k = 0; k < 4; k++) f[i][k] = 0.f;
      for (int r = grp; r < nr; r += groups) {
        const float4 a = *reinterpret_cast<const float4*>(&As[r][i0]);
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
  // fixed-order sum over the groups: group 0 first, then 1, ...
  __syncthreads();
  for (int e = tid; e < GT * GT; e += 256) red[e] = 0.0;
  for (int g = 0; g < groups; g++) {
    __syncthreads();
    if (active && grp == g) {
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int k = 0; k < 4; k++) red[(i0 + i) * GT + k0 + k] += acc[i][k];
    }
  }
  __syncthreads();
  double* out = part + ((int64_t)blockIdx.x * gridDim.y * gridDim.z + tile) * (GT * GT);
  for (int e = tid; e < GT * GT; e += 256) out[e] = red[e];
}

// out[tcol_a[a0+i], tcol_b[b0+k]] += sum over CTAs (CTA order) of the tile
// partials; mirror: also out[tcol_b, tcol_a] (off-diagonal blocks).
__global__ void k_gram_reduce(const double* __restrict__ part, int nb, int ntiles, int ntb,
                              int acols, int bcols, const int32_t* __restrict__ tcol_a,
                              const int32_t* __restrict__ tcol_b, int c_T, bool mirror,
                              double* __restrict__ out) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= (int64_t)ntiles * GT * GT) return;
  const int tile = (int)(w / (GT * GT));
  const int e = (int)(w - (int64_t)tile * GT * GT);
  const int i = (tile / ntb) * GT + e / GT, k = (tile % ntb) * GT + e % GT;
  if (i >= acols || k >= bcols) return;
  double s = 0.0;
  for (int b = lane; b < nb; b += 32) s += part[((int64_t)b * ntiles + tile) * (GT * GT) + e];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const int ta = tcol_a[i], tb = tcol_b[k];
  if (lane == 0 && ta >= 0 && tb >= 0) {
    out[(int64_t)ta * c_T + tb] += s;
    if (mirror) out[(int64_t)tb * c_T + ta] += s;
  }
}

// k_gram for acols, bcols <= GF (the usual dimension widths): ONE tile
// covers the whole output, so every CTA reads its rows of A and B once
// (k_gram reads them once per 32 x 32 output tile and was latency-bound at
// 1.1 ms for a 1M x 50 dimension Gram).  Rows staged 64 at a time with
// float4 loads when the pitches allow; thread = 4 x 4 micro tile of the
// output; fp32 over a staged tile, fp64 across tiles.
constexpr int GF = 64;
__global__ void __launch_bounds__(256) k_gram_full(const float* __restrict__ A, int pa, int acols,
                                                   const float* __restrict__ B, int pb, int bcols,
                                                   int64_t rows, int64_t rows_per_cta,
                                                   const int64_t* __restrict__ wptr,
                                                   double* __restrict__ part) {
  __shared__ __align__(16) float As[GROWS][GF + 4];
  __shared__ __align__(16) float Bs[GROWS][GF + 4];
  const int tid = threadIdx.x;
  const int ma = (acols + 3) / 4, mb = (bcols + 3) / 4;
  const int micro = ma * mb;
  const bool active = tid < micro;
  const int i0 = (tid / mb) * 4, k0 = (tid % mb) * 4;
  const int64_t r_begin = blockIdx.x * rows_per_cta;
  const int64_t r_end = min64(rows, r_begin + rows_per_cta);
  const int ac4 = (acols + 3) / 4, bc4 = (bcols + 3) / 4;
  const bool vec = ((pa | pb) & 3) == 0;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int k = 0; k < 4; k++) acc[i][k] = 0.0;
  for (int64_t r0 = r_begin; r0 < r_end; r0 += GROWS) {
    const int nr = (int)min64(GROWS, r_end - r0);
    __syncthreads();
    for (int e = tid; e < GROWS * (ac4 + bc4); e += 256) {
      const int r = e / (ac4 + bc4), q = e - r * (ac4 + bc4);
      const bool isa = q < ac4;
      const int c4 = isa ? q : q - ac4;
      const int cols = isa ? acols : bcols;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < nr) {
        const int64_t row = r0 + r;
        const float* src = isa ? A + row * pa : B + row * pb;
        if (vec && 4 * c4 + 3 < (isa ? pa : pb)) {
          v = __ldg(reinterpret_cast<const float4*>(src) + c4);
        } else {
          v.x = 4 * c4 < cols ? src[4 * c4] : 0.f;
          v.y = 4 * c4 + 1 < cols ? src[4 * c4 + 1] : 0.f;
          v.z = 4 * c4 + 2 < cols ? src[4 * c4 + 2] : 0.f;
          v.w = 4 * c4 + 3 < cols ? src[4 * c4 + 3] : 0.f;
        }
        // padding columns of a pitched source are zero; clip anyway
        if (4 * c4 >= cols) v = make_float4(0.f, 0.f, 0.f, 0.f);
        else {
          if (4 * c4 + 1 >= cols) v.y = 0.f;
          if (4 * c4 + 2 >= cols) v.z = 0.f;
          if (4 * c4 + 3 >= cols) v.w = 0.f;
        }
        if (isa && wptr) {
          const float wgt = (float)(wptr[row + 1] - wptr[row]);
          v.x *= wgt; v.y *= wgt; v.z *= wgt; v.w *= wgt;
        }
      }
      *reinterpret_cast<float4*>(isa ? &As[r][4 * c4] : &Bs[r][4 * c4]) = v;
    }
    __syncthreads();
    if (active) {
      float f[4][4];
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int k = 0; k < 4; k++) f[i][k] = 0.f;
      for (int r = 0; r < nr; r++) {
        const float4 a = *reinterpret_cast<const float4*>(&As[r][i0]);
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
    double* out = part + (int64_t)blockIdx.x * acols * bcols;
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
      for (int k = 0; k < 4; k++)
        if (i0 + i < acols && k0 + k < bcols) out[(i0 + i) * bcols + k0 + k] = acc[i][k];
  }
}

// out[tcol_a[i], tcol_b[k]] += sum over CTAs (CTA order) of part[.][i * bcols + k]
// (+ the mirrored entry for off-diagonal blocks)
__global__ void k_gram_full_reduce(const double* __restrict__ part, int nb, int acols, int bcols,
                                   const int32_t* __restrict__ tcol_a,
                                   const int32_t* __restrict__ tcol_b, int c_T, bool mirror,
                                   double* __restrict__ out) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= (int64_t)acols * bcols) return;
  const int e = (int)w, i = e / bcols, k = e - i * bcols;
  double s = 0.0;
  for (int b = lane; b < nb; b += 32) s += part[(int64_t)b * acols * bcols + e];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const int ta = tcol_a[i], tb = tcol_b[k];
  if (lane == 0 && ta >= 0 && tb >= 0) {
    out[(int64_t)ta * c_T + tb] += s;
    if (mirror) out[(int64_t)tb * c_T + ta] += s;
  }
}

struct PartnerSrc {   // a gathered source whose rows are summed into Y_de
  const float* S;
  const int32_t* fk;
  int pitch, cols, off;
};
constexpr int MAX_PARTNERS = MAX_GATHER;
struct Partners {
  PartnerSrc p[MAX_PARTNERS];
  int n;
};

// Z[j][0..pf) = sum over the members p of dimension row j of F[p][0..pf) for
// a stream block of pf % 4 == 0, pf <= 32 columns and no gathered partners
// (the common d x F block): warp per dimension row, lane = (row phase,
// 16-byte chunk) -- RP = 32 / (pf / 4) member rows per warp load instead
// of one, so the grouped read of F has enough bytes in flight to run at HBM
// speed.  fp64 per row phase, phases summed in a fixed order (not the
// strictly ascending order of k_group_rows_sum; same values to fp64
// rounding), fp32 store.
__global__ void __launch_bounds__(256) k_group_sum_f4(const int64_t* __restrict__ grp_ptr,
                                                      const int32_t* __restrict__ grp_rows,
                                                      bool sorted, int64_t n_neg, int64_t rows,
                                                      const float* __restrict__ F, int pf,
                                                      float* __restrict__ Z) {
  const int lane = threadIdx.x & 31;
  const int nc4 = pf >> 2, rp = 32 / nc4;
  const int ph = lane / nc4, q = lane - ph * nc4;
  const bool on = ph < rp;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; j < rows; j += nw) {
    const int64_t m0 = grp_ptr[j], m1 = grp_ptr[j + 1];
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    if (on) {
      int64_t m = m0 + ph;
      for (; m + rp < m1; m += 2 * rp) {   // two member rows in flight per lane
        const int64_t pa = sorted ? n_neg + m : (int64_t)grp_rows[m];
        const int64_t pb = sorted ? n_neg + m + rp : (int64_t)grp_rows[m + rp];
        const float4 a = __ldg(reinterpret_cast<const float4*>(F + pa * pf) + q);
        const float4 b = __ldg(reinterpret_cast<const float4*>(F + pb * pf) + q);
        s0 += (double)a.x; s1 += (double)a.y; s2 += (double)a.z; s3 += (double)a.w;
        s0 += (double)b.x; s1 += (double)b.y; s2 += (double)b.z; s3 += (double)b.w;
      }
      if (m < m1) {
        const int64_t pa = sorted ? n_neg + m : (int64_t)grp_rows[m];
        const float4 a = __ldg(reinterpret_cast<const float4*>(F + pa * pf) + q);
        s0 += (double)a.x; s1 += (double)a.y; s2 += (double)a.z; s3 += (double)a.w;
      }
    }
    // fixed-order sum over the row phases: lane (0, q) gathers phases 1.. in order
    for (int k = 1; k < rp; k++) {
      const int src = k * nc4 + q;
      const double t0 = __shfl_sync(0xffffffffu, s0, src < 32 ? src : lane);
      const double t1 = __shfl_sync(0xffffffffu, s1, src < 32 ? src : lane);
      const double t2 = __shfl_sync(0xffffffffu, s2, src < 32 ? src : lane);
      const double t3 = __shfl_sync(0xffffffffu, s3, src < 32 ? src : lane);
      if (ph == 0) {
        s0 += t0; s1 += t1; s2 += t2; s3 += t3;
      }
    }
    if (ph == 0)
      reinterpret_cast<float4*>(Z + j * pf)[q] = make_float4((float)s0, (float)s1, (float)s2, (float)s3);
  }
}

// Z[j][0..w) = sum over members p of dimension row j (ascending order) of
// [F[p][0..pf) | S_e[fk_e[p]] for every partner e]  (fp64 sums, fp32 store);
// one warp per dimension row, lanes over columns.
__global__ void k_group_rows_sum(const int64_t* __restrict__ grp_ptr,
                                 const int32_t* __restrict__ grp_rows, bool sorted, int64_t n_neg,
                                 int64_t rows, const float* __restrict__ F, int pf, Partners pt,
                                 int w, float* __restrict__ Z) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; j < rows; j += nw) {
    const int64_t m0 = grp_ptr[j], m1 = grp_ptr[j + 1];
    for (int c0 = 0; c0 < w; c0 += 32) {
      const int c = c0 + lane;
      // which operand this lane's column reads
      int src = -1, cc = c;
      if (c < pf) {
        src = 0;
      } else {
        for (int e = 0; e < pt.n; e++)
          if (c >= pt.p[e].off && c < pt.p[e].off + pt.p[e].cols) {
            src = 1 + e;
            cc = c - pt.p[e].off;
          }
      }
      double s = 0.0;
      if (c < w && src >= 0) {
        int64_t m = m0;
        for (; m + 8 <= m1; m += 8) {   // eight independent loads in flight
          float v[8];
#pragma unroll
          for (int u = 0; u < 8; u++) {
            const int64_t p = sorted ? n_neg + m + u : (int64_t)grp_rows[m + u];
            if (src == 0) {
              v[u] = F[p * pf + cc];
            } else {
              const PartnerSrc& q = pt.p[src - 1];
              const int32_t r = q.fk[p];
              v[u] = r >= 0 ? q.S[(int64_t)r * q.pitch + cc] : 0.f;
            }
          }
#pragma unroll
          for (int u = 0; u < 8; u++) s += (double)v[u];
        }
        for (; m < m1; m++) {
          const int64_t p = sorted ? n_neg + m : (int64_t)grp_rows[m];
          float v;
          if (src == 0) {
            v = F[p * pf + cc];
          } else {
            const PartnerSrc& q = pt.p[src - 1];
            const int32_t r = q.fk[p];
            v = r >= 0 ? q.S[(int64_t)r * q.pitch + cc] : 0.f;
          }
          s += (double)v;
        }
      }
      if (c < w) Z[j * w + c] = (float)s;
    }
  }
}

int gram(fl_table* t, const float* A, int pa, int acols, const float* B, int pb, int bcols,
         int64_t rows, const int64_t* wptr, const int32_t* tcol_a, const int32_t* tcol_b,
         bool mirror, double* out, cudaStream_t s) {
  if (rows <= 0 || acols <= 0 || bcols <= 0) return FL_OK;
  if (acols <= GF && bcols <= GF && !getenv("FL_NO_GRAM_FULL")) {
    int64_t nb = std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows, 4 * GROWS),
                                                        8 * (int64_t)t->sm_count));
    const int64_t rpc = round_up(ceil_div(rows, nb), GROWS);
    nb = ceil_div(rows, rpc);
    double* part = nullptr;
    FL_CUDA(cudaMallocAsync((void**)&part, (size_t)nb * acols * bcols * 8, s));
    k_gram_full<<<(unsigned)nb, 256, 0, s>>>(A, pa, acols, B, pb, bcols, rows, rpc, wptr, part);
    FL_CHECK_LAUNCH();
    k_gram_full_reduce<<<(unsigned)ceil_div((int64_t)acols * bcols * 32, 256), 256, 0, s>>>(
        part, (int)nb, acols, bcols, tcol_a, tcol_b, t->c_T, mirror, out);
    FL_CHECK_LAUNCH();
    FL_CUDA(cudaFreeAsync(part, s));
    return FL_OK;
  }
  const int nta = (acols + GT - 1) / GT, ntb = (bcols + GT - 1) / GT;
  const int ntiles = nta * ntb;
  // ~8 CTAs per SM over all tiles (the staged loop is latency-bound); row
  // chunks are whole staged tiles
  int64_t nb = std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows, 4 * GROWS),
                                                      (8 * (int64_t)t->sm_count + ntiles - 1) / ntiles));
  const int64_t rpc = round_up(ceil_div(rows, nb), GROWS);
  nb = ceil_div(rows, rpc);
  double* part = nullptr;
  FL_CUDA(cudaMallocAsync((void**)&part, (size_t)nb * ntiles * GT * GT * 8, s));
  k_gram<<<dim3((unsigned)nb, ntb, nta), 256, 0, s>>>(A, pa, acols, B, pb, bcols, rows, rpc, wptr,
                                                     part);
  FL_CHECK_LAUNCH();
  const int64_t warps = (int64_t)ntiles * GT * GT;
  k_gram_reduce<<<(unsigned)ceil_div(warps * 32, 256), 256, 0, s>>>(
      part, (int)nb, ntiles, ntb, acols, bcols, tcol_a, tcol_b, t->c_T, mirror, out);
  FL_CHECK_LAUNCH();
  FL_CUDA(cudaFreeAsync(part, s));
  return FL_OK;
}

#include "gram_t5.cuh"

// F^T F through k_fgram_t5l (bulk-copied tiles; pf % 4 == 0) or k_fgram_t5
// (2-D TMA tiles; FL_GRAM_TMA=1 forces it), stream block <= 28 columns
int fgram_t5(fl_table* t, double* out, cudaStream_t s) {
  if (t->pf % 4 == 0 && !getenv("FL_GRAM_TMA")) {
    const R5LGeom gl = r5l_geom(t->pf);
    static bool attr_l = false;
    if (!attr_l) {
      FL_CUDA(raise_smem_limit(k_fgram_t5l, (int)(r5l_geom(28).total + 1024)));
      attr_l = true;
    }
    const int64_t ntiles = t->r_pad / R5_TILE;
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, t->sm_count));
    double* part = nullptr;
    FL_CUDA(cudaMallocAsync((void**)&part, (size_t)nb * t->pf * t->pf * 8, s));
    k_fgram_t5l<<<nb, R5_THREADS, gl.total + 1024, s>>>(t->F->as<float>(), t->pf, ntiles, gl, part);
    FL_CHECK_LAUNCH();
    k_fgram_reduce<<<(unsigned)ceil_div((int64_t)t->pf * t->pf * 32, 256), 256, 0, s>>>(
        part, nb, t->pf, t->d_f_tcol->as<int32_t>(), t->c_T, out);
    FL_CHECK_LAUNCH();
    FL_CUDA(cudaFreeAsync(part, s));
    return FL_OK;
  }
  const R5Geom gm = r5_geom();
  CUtensorMap tm;
  int rc = make_tmap_2d(&tm, t->F->p, (uint64_t)t->r_pad, (uint64_t)t->pf, (uint64_t)t->pf * 4,
                        R5_TILE, 32, kSwz128Atom32);
  if (rc) return rc;
  static bool attr = false;
  if (!attr) {
    FL_CUDA(raise_smem_limit(k_fgram_t5, (int)(gm.total + 1024)));
    attr = true;
  }
  const int64_t ntiles = t->r_pad / R5_TILE;
  const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, t->sm_count));
  double* part = nullptr;
  FL_CUDA(cudaMallocAsync((void**)&part, (size_t)nb * t->pf * t->pf * 8, s));
  const char* m6 = getenv("FL_GRAM_M64");
  k_fgram_t5<<<nb, R5_THREADS, gm.total + 1024, s>>>(tm, t->pf, ntiles, gm, part,
                                                     (m6 && atoi(m6)) ? 1 : 0);
  FL_CHECK_LAUNCH();
  k_fgram_reduce<<<(unsigned)ceil_div((int64_t)t->pf * t->pf * 32, 256), 256, 0, s>>>(
      part, nb, t->pf, t->d_f_tcol->as<int32_t>(), t->c_T, out);
  FL_CHECK_LAUNCH();
  FL_CUDA(cudaFreeAsync(part, s));
  return FL_OK;
}

}  // namespace
}  // namespace flb

using namespace flb;

extern "C" int fl_crossprod(fl_table* t, double* out, void* stream) {
  if (!t || !t->finalized || !out) {
    set_error("crossprod: table is null or not finalized");
    return FL_ERR_ARG;
  }
  FL_CUDA(cudaSetDevice(t->device));
  cudaStream_t s = (cudaStream_t)stream;
  const int c_T = t->c_T;
  double* od;
  bool oo;
  int rc = out_buffer(out, (size_t)c_T * c_T, s, &od, &oo);
  if (rc) return rc;
  FL_CUDA(cudaMemsetAsync(od, 0, (size_t)c_T * c_T * 8, s));
  const float* F = t->F ? t->F->as<float>() : nullptr;
  const int32_t* ftcol = t->pf ? t->d_f_tcol->as<int32_t>() : nullptr;
  // F x F: tcgen05 Gram with MN-major operands for <= 28 streamed columns
  // (FL_NO_GRAM_T5=1: the SIMT tile Gram)
  if (t->pf > 0) {
    if (t->pf <= 28 && !getenv("FL_NO_GRAM_T5"))
      rc = fgram_t5(t, od, s);
    else
      rc = gram(t, F, t->pf, t->pf, F, t->pf, t->pf, t->r_T, nullptr, ftcol, ftcol, false, od, s);
    if (rc) return rc;
  }
  const int ng = (int)t->g.size();
  for (int d = 0; d < ng; d++) {
    const GatherSrc& g = t->g[d];
    const int32_t* tcol_d = g.d_tcol->as<int32_t>();
    // d x d: S_d^T diag(fanout) S_d
    rc = gram(t, g.S->as<float>(), g.pitch, g.cols, g.S->as<float>(), g.pitch, g.cols, g.rows,
              g.grp_ptr->as<int64_t>(), tcol_d, tcol_d, false, od, s);
    if (rc) return rc;
    // partners: F, then every later gathered source (their gathered rows),
    // at most MAX_PARTNERS gathered partners per grouped pass
    for (int e0 = d + 1, first = 1; first || e0 < ng; first = 0) {
      Partners pt{};
      int w = first ? t->pf : 0;
      int e = e0;
      for (; e < ng && pt.n < MAX_PARTNERS; e++) {
        const GatherSrc& ge = t->g[e];
        pt.p[pt.n++] = PartnerSrc{ge.S->as<float>(), ge.fk->as<int32_t>(), ge.pitch, ge.cols, w};
        w += ge.cols;
      }
      e0 = e;
      if (w == 0 || g.rows == 0) continue;
      float* Z = nullptr;
      FL_CUDA(cudaMallocAsync((void**)&Z, (size_t)g.rows * w * 4 + 16, s));
      const unsigned nbz = (unsigned)std::min<int64_t>(ceil_div(g.rows * 32, 256),
                                                       32 * (int64_t)t->sm_count);
      if (first && pt.n == 0 && t->pf % 4 == 0 && t->pf <= 32)
        k_group_sum_f4<<<nbz, 256, 0, s>>>(g.grp_ptr->as<int64_t>(),
                                           g.grp_rows ? g.grp_rows->as<int32_t>() : nullptr,
                                           g.sorted, g.n_neg, g.rows, F, t->pf, Z);
      else
        k_group_rows_sum<<<nbz, 256, 0, s>>>(g.grp_ptr->as<int64_t>(),
                                             g.grp_rows ? g.grp_rows->as<int32_t>() : nullptr,
                                             g.sorted, g.n_neg, g.rows, first ? F : nullptr,
                                             first ? t->pf : 0, pt, w, Z);
      FL_CHECK_LAUNCH();
      // target columns of Z's columns, assembled on the device (no host
      // buffer to keep alive, no stream sync between the passes)
      int32_t* dz = nullptr;
      FL_CUDA(cudaMallocAsync((void**)&dz, (size_t)w * 4, s));
      if (first && t->pf > 0)
        FL_CUDA(cudaMemcpyAsync(dz, t->d_f_tcol->p, (size_t)t->pf * 4, cudaMemcpyDeviceToDevice, s));
      for (int q = 0; q < pt.n; q++) {
        const GatherSrc& ge = t->g[e - pt.n + q];
        FL_CUDA(cudaMemcpyAsync(dz + pt.p[q].off, ge.d_tcol->p, (size_t)ge.cols * 4,
                                cudaMemcpyDeviceToDevice, s));
      }
      // d x (F | later dims), mirrored into (F | later dims) x d
      rc = gram(t, g.S->as<float>(), g.pitch, g.cols, Z, w, w, g.rows, nullptr, tcol_d, dz, true,
                od, s);
      if (rc) return rc;
      FL_CUDA(cudaFreeAsync(dz, s));
      FL_CUDA(cudaFreeAsync(Z, s));
    }
  }
  rc = finish_out(out, od, oo, (size_t)c_T * c_T, s);
  if (rc) return rc;
  FL_CUDA(cudaStreamSynchronize(s));
  return FL_OK;
}
