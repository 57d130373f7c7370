// Width-general K-means and Gaussian NMF sessions: any k / rank, any stream
// block or dimension width, any number of gathered sources.
//
// The fused passes (kmeans.cu, gnmf.cu) are specialised on k <= 32 /
// rank <= 32, streamed pitch <= 124 / 60 and <= MAX_GATHER gathered sources.
// Everything else runs here, composed like the reference's own loops from the
// generic operators (ops.cu: do_lmm, do_tlmm) plus row-local kernels -- the
// same role FL_GLM_UNFUSED plays for the GLMs.  Results follow the same
// conventions and ABI as the fused sessions (fl_kmeans_* / fl_gnmf_* dispatch
// here), including the partial / all-reduce / update split used across GPUs.
//
// K-means, one iteration (reference trainers.py:223-241):
//   E_d[r, j] = ||S_d[r,:] - C_j[cols of d]||^2  (row r_d = "no match")
//   per device row p: dist_j = ||F[p,:] - C_F,j||^2 + sum_d E_d[fk_d[p], j]
//     (direct fp32 differences), a_p = argmin (ties -> lowest j), loss += dist_a,
//     count[a_p] += 1, one-hot row written in DEVICE order
//   sums^T = T^T A through do_tlmm (deterministic fp64), then
//   C <- sums / counts for live clusters.
// Gaussian NMF (trainers.py:282-299): P = W^T T (do_tlmm), G = W^T W (fixed-
// order fp64 Gram), loss from (P, G, H), H <- H o P / (G H + eps),
// Q = T H^T (do_lmm), W <- W o Q / (W H H^T + eps).
#include <algorithm>
#include <vector>

#include "internal.h"
#include "generic.h"

namespace flb {

constexpr double GG_EPS = 1e-12;   // trainers.py:29
constexpr int KG_JC = 32;          // clusters per register chunk

struct GSrc {
  const int32_t* fk;   // r_pad, device order
  const float* E;      // (rows + 1) x k
  int64_t rows;
};

// ---------------------------------------------------------------------------
// K-means
// ---------------------------------------------------------------------------
// E_d[r * k + j] for r <= rows (r == rows: the all-zero no-match row)
__global__ void k_kg_dim_e(const float* __restrict__ S, int pitch, int cols, int64_t rows,
                           const int32_t* __restrict__ tcol, const float* __restrict__ C32,
                           int c_T, int k, float* __restrict__ E) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (rows + 1) * k;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / k;
    const int j = (int)(idx - r * k);
    const float* cj = C32 + (int64_t)j * c_T;
    float acc = 0.f;
    for (int c = 0; c < cols; c++) {
      const float sv = r < rows ? S[r * pitch + c] : 0.f;
      const float d = sv - cj[tcol[c]];
      acc = fmaf(d, d, acc);
    }
    E[idx] = acc;
  }
}

// cF[c * KPAD + j] = C[j, f_tcol[c]] (0 for padding columns / clusters)
__global__ void k_kg_cf(const float* __restrict__ C32, int c_T, int k, int pf, int KPAD,
                        const int32_t* __restrict__ ftcol, float* __restrict__ cF) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < pf * KPAD; i += gridDim.x * blockDim.x) {
    const int c = i / KPAD, j = i - c * KPAD;
    const int tc = ftcol[c];
    cF[i] = (j < k && tc >= 0) ? C32[(int64_t)j * c_T + tc] : 0.f;
  }
}

// thread per device row over the CTA's fixed row range (deterministic loss)
__global__ void __launch_bounds__(256) k_kg_fact(const float* __restrict__ F, int pf, int64_t r_T,
                                                 const float* __restrict__ cF_g, int KPAD, int k,
                                                 int stage_cf, const GSrc* __restrict__ gs,
                                                 int ng, int64_t rpb, int32_t* __restrict__ assign,
                                                 float* __restrict__ onehot,
                                                 unsigned* __restrict__ counts,
                                                 double* __restrict__ lpart) {
  extern __shared__ __align__(16) float cf_s[];
  const float* cF = cF_g;
  if (stage_cf) {
    for (int i = threadIdx.x; i < pf * KPAD; i += blockDim.x) cf_s[i] = cF_g[i];
    __syncthreads();
    cF = cf_s;
  }
  const int64_t r0 = blockIdx.x * rpb, r1 = min64(r_T, r0 + rpb);
  double lsum = 0.0;
  // uniform trip count per CTA: the whole warp reaches the counter vote
  for (int64_t base = r0; base < r1; base += blockDim.x) {
    const int64_t p = base + threadIdx.x;
    const bool valid = p < r1;
    int bi = -1 - (int)(threadIdx.x & 31);
    if (valid) {
      float best = __int_as_float(0x7f800000);
      bi = 0;
      const float* xr = F ? F + p * pf : nullptr;
      for (int jc = 0; jc < k; jc += KG_JC) {
        float acc[KG_JC];
#pragma unroll
        for (int j = 0; j < KG_JC; j++) acc[j] = 0.f;
        for (int c = 0; c < pf; c++) {
          const float x = xr[c];
          const float4* cr = reinterpret_cast<const float4*>(cF + (int64_t)c * KPAD + jc);
#pragma unroll
          for (int q = 0; q < KG_JC / 4; q++) {
            const float4 cc = cr[q];
            const float d0 = x - cc.x, d1 = x - cc.y, d2 = x - cc.z, d3 = x - cc.w;
            acc[4 * q + 0] = fmaf(d0, d0, acc[4 * q + 0]);
            acc[4 * q + 1] = fmaf(d1, d1, acc[4 * q + 1]);
            acc[4 * q + 2] = fmaf(d2, d2, acc[4 * q + 2]);
            acc[4 * q + 3] = fmaf(d3, d3, acc[4 * q + 3]);
          }
        }
        for (int d = 0; d < ng; d++) {
          const int32_t f = gs[d].fk[p];
          const float* er = gs[d].E + (f >= 0 ? (int64_t)f : gs[d].rows) * k + jc;
#pragma unroll
          for (int j = 0; j < KG_JC; j++)
            if (jc + j < k) acc[j] += er[j];
        }
#pragma unroll
        for (int j = 0; j < KG_JC; j++)
          if (jc + j < k && acc[j] < best) {   // strict: ties keep the lowest index
            best = acc[j];
            bi = jc + j;
          }
      }
      lsum += (double)best;
      assign[p] = bi;
      float* oh = onehot + p * k;
      for (int j = 0; j < k; j++) oh[j] = j == bi ? 1.f : 0.f;
    }
    // warp-aggregated integer counter (exact, order-free)
    const unsigned peers = __match_any_sync(0xffffffffu, bi);
    if (bi >= 0 && (__ffs(peers) - 1) == (int)(threadIdx.x & 31)) atomicAdd(&counts[bi], __popc(peers));
  }
  // fixed-order block reduction of the loss
  __shared__ double ws[32];
  for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = lsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) s += ws[w];
    lpart[blockIdx.x] = s;
  }
}

// red[k c_T + j] = counts[j], red[k c_T + k] = sum of the loss partials (fixed
// order); counters reset for the next pass
__global__ void k_kg_finish(unsigned* __restrict__ counts, int k, const double* __restrict__ lpart,
                            int nblk, double* __restrict__ red, int c_T) {
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    red[(int64_t)k * c_T + j] = (double)counts[j];
    counts[j] = 0u;
  }
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int b = 0; b < nblk; b++) s += lpart[b];
    red[(int64_t)k * c_T + k] = s;
  }
}

// C <- sums / counts (empty clusters keep their centroid); loss_hist[it]
__global__ void k_kg_update(const double* __restrict__ red, int k, int c_T, double* __restrict__ C64,
                            float* __restrict__ C32, double* __restrict__ loss_hist, int it,
                            int loss_cap) {
  const double* cnt = red + (int64_t)k * c_T;
  if (blockIdx.x == 0 && threadIdx.x == 0 && it < loss_cap) loss_hist[it] = red[(int64_t)k * c_T + k];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)k * c_T;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(i / c_T);
    const double n = cnt[j];
    if (n > 0.0) C64[i] = red[i] / n;
    C32[i] = (float)C64[i];
  }
}

__global__ void k_kg_c32(const double* __restrict__ C64, int64_t n, float* __restrict__ C32) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    C32[i] = (float)C64[i];
}

template <class T>
__global__ void k_kg_assign_out(const int32_t* __restrict__ a_dev, const int32_t* __restrict__ perm,
                                int64_t r_T, T* __restrict__ out) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p < r_T) out[perm[p]] = (T)a_dev[p];
}

struct KmGen {
  fl_table* t = nullptr;
  int k = 0, KPAD = 0, nblk = 0, stage_cf = 0;
  int64_t rpb = 0;
  int it = 0;
  int loss_cap = 1 << 16;
  DevBuf C64, C32, cF, E, gsrc, onehot, counts, lpart, red, loss_hist, assign;
  std::vector<int64_t> e_off;
  fl_comm* comm = nullptr;
};

void kmg_set_comm(KmGen* s, fl_comm* c) { s->comm = c; }

int kmg_create(fl_table* t, int k, const double* c0, cudaStream_t st, KmGen** out) {
  auto* s = new KmGen();
  std::unique_ptr<KmGen> guard(s);
  s->t = t;
  s->k = k;
  s->KPAD = (int)round_up(k, KG_JC);
  const int c_T = t->c_T, ng = (int)t->g.size();
  int rc;
  if ((rc = s->C64.alloc((size_t)k * c_T * 8))) return rc;
  if ((rc = s->C32.alloc((size_t)k * c_T * 4))) return rc;
  FL_CUDA(cudaMemcpyAsync(s->C64.p, c0, (size_t)k * c_T * 8, cudaMemcpyDefault, st));
  k_kg_c32<<<(unsigned)std::min<int64_t>(ceil_div((int64_t)k * c_T, 256), 1024), 256, 0, st>>>(
      s->C64.as<double>(), (int64_t)k * c_T, s->C32.as<float>());
  FL_CHECK_LAUNCH();
  if ((rc = s->cF.alloc((size_t)std::max(t->pf, 1) * s->KPAD * 4))) return rc;
  size_t e_total = 0;
  for (auto& g : t->g) {
    s->e_off.push_back((int64_t)e_total);
    e_total += (size_t)(g.rows + 1) * k;
  }
  if ((rc = s->E.alloc(e_total * 4 + 16))) return rc;
  std::vector<GSrc> hs(ng);
  for (int d = 0; d < ng; d++)
    hs[d] = GSrc{t->g[d].fk->as<int32_t>(), s->E.as<float>() + s->e_off[d], t->g[d].rows};
  if ((rc = s->gsrc.alloc(sizeof(GSrc) * std::max(ng, 1)))) return rc;
  if (ng) FL_CUDA(cudaMemcpy(s->gsrc.p, hs.data(), sizeof(GSrc) * ng, cudaMemcpyHostToDevice));
  if ((rc = s->onehot.alloc((size_t)t->r_T * k * 4 + 16))) return rc;
  if ((rc = s->counts.alloc((size_t)k * 4))) return rc;
  FL_CUDA(cudaMemsetAsync(s->counts.p, 0, (size_t)k * 4, st));
  s->nblk = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(t->r_T, 256), 8 * (int64_t)t->sm_count));
  s->rpb = ceil_div(std::max<int64_t>(t->r_T, 1), s->nblk);
  if ((rc = s->lpart.alloc((size_t)s->nblk * 8))) return rc;
  if ((rc = s->red.alloc(((size_t)k * c_T + k + 1) * 8))) return rc;
  FL_CUDA(cudaMemsetAsync(s->red.p, 0, ((size_t)k * c_T + k + 1) * 8, st));
  if ((rc = s->loss_hist.alloc((size_t)s->loss_cap * 8))) return rc;
  if ((rc = s->assign.alloc((size_t)t->r_pad * 4))) return rc;
  FL_CUDA(cudaMemsetAsync(s->assign.p, 0, (size_t)t->r_pad * 4, st));
  const size_t cf_bytes = (size_t)t->pf * s->KPAD * 4;
  s->stage_cf = cf_bytes <= 96 * 1024 ? 1 : 0;
  if (s->stage_cf)
    FL_CUDA(raise_smem_limit(k_kg_fact, (int)std::max<size_t>(cf_bytes, 16)));
  FL_CUDA(cudaStreamSynchronize(st));
  *out = guard.release();
  return FL_OK;
}

int kmg_partial(KmGen* s, cudaStream_t st) {
  fl_table* t = s->t;
  const int k = s->k, c_T = t->c_T;
  for (size_t d = 0; d < t->g.size(); d++) {
    const GatherSrc& g = t->g[d];
    k_kg_dim_e<<<(unsigned)std::min<int64_t>(ceil_div((g.rows + 1) * k, 256), 8 * (int64_t)t->sm_count),
                 256, 0, st>>>(g.S->as<float>(), g.pitch, g.cols, g.rows, g.d_tcol->as<int32_t>(),
                               s->C32.as<float>(), c_T, k, s->E.as<float>() + s->e_off[d]);
    FL_CHECK_LAUNCH();
  }
  if (t->pf > 0) {
    k_kg_cf<<<(unsigned)ceil_div((int64_t)t->pf * s->KPAD, 256), 256, 0, st>>>(
        s->C32.as<float>(), c_T, k, t->pf, s->KPAD, t->d_f_tcol->as<int32_t>(), s->cF.as<float>());
    FL_CHECK_LAUNCH();
  }
  k_kg_fact<<<s->nblk, 256, s->stage_cf ? (size_t)t->pf * s->KPAD * 4 : 0, st>>>(
      t->pf ? t->F->as<float>() : nullptr, t->pf, t->r_T, s->cF.as<float>(), s->KPAD, k,
      s->stage_cf, s->gsrc.as<GSrc>(), (int)t->g.size(), s->rpb, s->assign.as<int32_t>(),
      s->onehot.as<float>(), s->counts.as<unsigned>(), s->lpart.as<double>());
  FL_CHECK_LAUNCH();
  // sums^T = T^T A (the one-hot rows are in device order); red[j c_T + tc]
  FL_CUDA(cudaMemsetAsync(s->red.p, 0, (size_t)k * c_T * 8, st));
  int rc = do_tlmm(t, YView{s->onehot.as<float>(), k, 1}, k, s->red.as<double>(), 1, c_T, st, true);
  if (rc) return rc;
  k_kg_finish<<<1, 256, 0, st>>>(s->counts.as<unsigned>(), k, s->lpart.as<double>(), s->nblk,
                                 s->red.as<double>(), c_T);
  FL_CHECK_LAUNCH();
  return FL_OK;
}

int kmg_update(KmGen* s, cudaStream_t st) {
  const int64_t n = (int64_t)s->k * s->t->c_T;
  k_kg_update<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 1024), 256, 0, st>>>(
      s->red.as<double>(), s->k, s->t->c_T, s->C64.as<double>(), s->C32.as<float>(),
      s->loss_hist.as<double>(), s->it, s->loss_cap);
  FL_CHECK_LAUNCH();
  s->it++;
  return FL_OK;
}

int kmg_run(KmGen* s, int iterations, cudaStream_t st) {
  for (int i = 0; i < iterations; i++) {
    int rc = kmg_partial(s, st);
    if (!rc && s->comm) {
      int n = 0;
      double* red = kmg_red(s, &n);
      rc = comm_allreduce(s->comm, red, (size_t)n, st);
    }
    if (!rc) rc = kmg_update(s, st);
    if (rc) return rc;
  }
  return FL_OK;
}

double* kmg_red(KmGen* s, int* len) {
  *len = s->k * s->t->c_T + s->k + 1;
  return s->red.as<double>();
}

int kmg_result(KmGen* s, double* centroids, int32_t* assign, int64_t* assign64, double* loss,
               int n, int* n_done, cudaStream_t st) {
  fl_table* t = s->t;
  if (centroids)
    FL_CUDA(cudaMemcpyAsync(centroids, s->C64.p, (size_t)s->k * t->c_T * 8, cudaMemcpyDefault, st));
  if (assign || assign64) {
    const size_t eb = assign ? 4 : 8;
    void* tmp = nullptr;
    FL_CUDA(cudaMallocAsync(&tmp, (size_t)t->r_T * eb + 16, st));
    if (assign)
      k_kg_assign_out<int32_t><<<(unsigned)ceil_div(t->r_T, 256), 256, 0, st>>>(
          s->assign.as<int32_t>(), t->perm->as<int32_t>(), t->r_T, (int32_t*)tmp);
    else
      k_kg_assign_out<int64_t><<<(unsigned)ceil_div(t->r_T, 256), 256, 0, st>>>(
          s->assign.as<int32_t>(), t->perm->as<int32_t>(), t->r_T, (int64_t*)tmp);
    FL_CHECK_LAUNCH();
    FL_CUDA(cudaMemcpyAsync(assign ? (void*)assign : (void*)assign64, tmp, (size_t)t->r_T * eb,
                            cudaMemcpyDefault, st));
    FL_CUDA(cudaFreeAsync(tmp, st));
  }
  FL_CUDA(cudaStreamSynchronize(st));
  const int nd = std::min(s->it, s->loss_cap);
  if (n_done) *n_done = nd;
  if (loss && n > 0) {
    const int m = std::min(n, nd);
    if (m > 0) FL_CUDA(cudaMemcpy(loss, s->loss_hist.p, (size_t)m * 8, cudaMemcpyDefault));
  }
  return FL_OK;
}

void kmg_destroy(KmGen* s) { delete s; }

// ---------------------------------------------------------------------------
// Gaussian NMF
// ---------------------------------------------------------------------------
// HH[r, q] = sum_c H[r, c] H[q, c] (fp64), optional fp32 copy
__global__ void k_gg_hh(const double* __restrict__ H, int R, int c_T, double* __restrict__ HH,
                        float* __restrict__ HH32) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < R * R; i += gridDim.x * blockDim.x) {
    const int r = i / R, q = i - r * R;
    double s = 0.0;
    for (int c = 0; c < c_T; c++) s += H[(int64_t)r * c_T + c] * H[(int64_t)q * c_T + c];
    HH[i] = s;
    if (HH32) HH32[i] = (float)s;
  }
}

// loss = t_sq - 2 <P, H> + <G, HH> (fixed order: strided thread sums, then
// thread 0 in order)
__global__ void k_gg_loss(const double* __restrict__ red, const double* __restrict__ H,
                          const double* __restrict__ HH, int R, int c_T, double t_sq,
                          double* __restrict__ loss_hist, int n, int loss_cap) {
  __shared__ double part[256];
  const double* P = red;
  const double* G = red + (int64_t)R * c_T;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < (int64_t)R * c_T; i += blockDim.x) s -= 2.0 * P[i] * H[i];
  for (int i = threadIdx.x; i < R * R; i += blockDim.x) s += G[i] * HH[i];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = t_sq;
    for (int i = 0; i < (int)blockDim.x; i++) tot += part[i];
    if (n >= 0 && n < loss_cap) loss_hist[n] = tot;
  }
}

// Hn = H o P / (G H + eps)
__global__ void k_gg_hupd(const double* __restrict__ red, const double* __restrict__ H, int R,
                          int c_T, double* __restrict__ Hn) {
  const double* P = red;
  const double* G = red + (int64_t)R * c_T;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)R * c_T;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / c_T);
    const int c = (int)(i - (int64_t)r * c_T);
    double gh = 0.0;
    for (int q = 0; q < R; q++) gh += G[(int64_t)r * R + q] * H[(int64_t)q * c_T + c];
    Hn[i] = H[i] * P[i] / (gh + GG_EPS);
  }
}

// Ht32[c * R + r] = H[r, c] (the lmm operand H^T)
__global__ void k_gg_ht(const double* __restrict__ H, int R, int c_T, float* __restrict__ Ht32) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)R * c_T;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / c_T);
    const int c = (int)(i - (int64_t)r * c_T);
    Ht32[(int64_t)c * R + r] = (float)H[i];
  }
}

// W[t] <- W[t] o Q[t] / (W[t] HH + eps): a warp per row, the row in per-warp
// shared memory, lane = output column
__global__ void __launch_bounds__(256) k_gg_w(float* __restrict__ W, const float* __restrict__ Q,
                                              const float* __restrict__ HH32, int64_t r_T, int R,
                                              int stage_hh) {
  extern __shared__ float gw_s[];   // [HH (R x R) if staged] | 8 warps x R
  const float* HH = HH32;
  float* rows = gw_s;
  if (stage_hh) {
    for (int i = threadIdx.x; i < R * R; i += blockDim.x) gw_s[i] = HH32[i];
    HH = gw_s;
    rows = gw_s + R * R;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* wr = rows + warp * R;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t t = blockIdx.x * (int64_t)(blockDim.x >> 5) + warp; t < r_T; t += nw) {
    for (int j = lane; j < R; j += 32) wr[j] = W[t * R + j];
    __syncwarp();
    for (int j = lane; j < R; j += 32) {
      float den = 0.f;
      for (int q = 0; q < R; q++) den = fmaf(wr[q], HH[q * R + j], den);
      W[t * R + j] = wr[j] * Q[t * R + j] / (den + (float)GG_EPS);
    }
    __syncwarp();
  }
}

// Gram partials: CTA b owns a fixed row range; thread = up to 8 (r, q) pairs
// of the pair chunk blockIdx.y; fp32 inside 32-row tiles, fp64 across tiles
constexpr int GG_PP = 8;
__global__ void __launch_bounds__(256) k_gg_gram(const float* __restrict__ W, int64_t r_T, int R,
                                                 int64_t rpb, double* __restrict__ part) {
  extern __shared__ float tile[];   // 32 x R
  const int npair = R * R;
  const int pbase = blockIdx.y * 256 * GG_PP;
  const int64_t r0 = blockIdx.x * rpb, r1 = min64(r_T, r0 + rpb);
  double acc[GG_PP];
#pragma unroll
  for (int u = 0; u < GG_PP; u++) acc[u] = 0.0;
  for (int64_t tb = r0; tb < r1; tb += 32) {
    const int nr = (int)min64(32, r1 - tb);
    __syncthreads();
    for (int i = threadIdx.x; i < 32 * R; i += blockDim.x) {
      const int rr = i / R;
      tile[i] = rr < nr ? W[(tb + rr) * R + (i - rr * R)] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < GG_PP; u++) {
      const int pr = pbase + u * 256 + threadIdx.x;
      if (pr < npair) {
        const int a = pr / R, b = pr - a * R;
        float s = 0.f;
        for (int rr = 0; rr < 32; rr++) s = fmaf(tile[rr * R + a], tile[rr * R + b], s);
        acc[u] += (double)s;
      }
    }
  }
#pragma unroll
  for (int u = 0; u < GG_PP; u++) {
    const int pr = pbase + u * 256 + threadIdx.x;
    if (pr < npair) part[(int64_t)blockIdx.x * npair + pr] = acc[u];
  }
}

// red[off + i] = sum_b part[b * n + i] (fixed order)
__global__ void k_gg_reduce(const double* __restrict__ part, int nblk, int n,
                            double* __restrict__ dst) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nblk; b++) s += part[(int64_t)b * n + i];
    dst[i] = s;
  }
}

__global__ void k_gg_w_in(const double* __restrict__ w0, int64_t n, float* __restrict__ W) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    W[i] = (float)w0[i];
}

__global__ void k_gg_w_out(const float* __restrict__ W, int64_t n, double* __restrict__ w) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    w[i] = (double)W[i];
}

struct GnGen {
  fl_table* t = nullptr;
  int R = 0;
  double t_sq = 0.0;
  int it = 0, nloss = 0;
  bool primed = false;
  int loss_cap = 1 << 16;
  int nblk_g = 1, stage_hh = 0;
  int64_t rpb_g = 0;
  size_t smem_w = 0;
  DevBuf W, Q, H, Hn, Ht32, HH, HH32, red, gpart, loss_hist;
  fl_comm* comm = nullptr;
};

void gng_set_comm(GnGen* s, fl_comm* c) { s->comm = c; }

static unsigned gg_grid(int64_t n, int sms) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 8 * (int64_t)sms));
}

int gng_create(fl_table* t, int rank, const double* w0, const double* h0, double t_sq,
               cudaStream_t st, GnGen** out) {
  auto* s = new GnGen();
  std::unique_ptr<GnGen> guard(s);
  s->t = t;
  s->R = rank;
  s->t_sq = t_sq;
  const int R = rank, c_T = t->c_T;
  const int64_t r_T = t->r_T;
  int rc;
  if ((rc = s->W.alloc((size_t)r_T * R * 4 + 16))) return rc;
  {
    double* w0d = nullptr;
    FL_CUDA(cudaMallocAsync((void**)&w0d, (size_t)r_T * R * 8 + 16, st));
    FL_CUDA(cudaMemcpyAsync(w0d, w0, (size_t)r_T * R * 8, cudaMemcpyDefault, st));
    k_gg_w_in<<<gg_grid(r_T * R, t->sm_count), 256, 0, st>>>(w0d, r_T * R, s->W.as<float>());
    FL_CHECK_LAUNCH();
    FL_CUDA(cudaFreeAsync(w0d, st));
  }
  if ((rc = s->Q.alloc((size_t)r_T * R * 4 + 16))) return rc;
  if ((rc = s->H.alloc((size_t)R * c_T * 8))) return rc;
  FL_CUDA(cudaMemcpyAsync(s->H.p, h0, (size_t)R * c_T * 8, cudaMemcpyDefault, st));
  if ((rc = s->Hn.alloc((size_t)R * c_T * 8))) return rc;
  if ((rc = s->Ht32.alloc((size_t)R * c_T * 4))) return rc;
  if ((rc = s->HH.alloc((size_t)R * R * 8))) return rc;
  if ((rc = s->HH32.alloc((size_t)R * R * 4))) return rc;
  if ((rc = s->red.alloc(((size_t)R * c_T + (size_t)R * R) * 8))) return rc;
  FL_CUDA(cudaMemsetAsync(s->red.p, 0, ((size_t)R * c_T + (size_t)R * R) * 8, st));
  if ((rc = s->loss_hist.alloc((size_t)s->loss_cap * 8))) return rc;
  s->nblk_g = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(r_T, 1024), 2 * (int64_t)t->sm_count));
  s->rpb_g = round_up(ceil_div(std::max<int64_t>(r_T, 1), s->nblk_g), 32);
  s->nblk_g = (int)std::max<int64_t>(1, ceil_div(r_T, s->rpb_g));
  if ((rc = s->gpart.alloc((size_t)s->nblk_g * R * R * 8))) return rc;
  if ((size_t)32 * R * 4 > 200 * 1024) {
    set_error("GNMF: rank %d too large for the Gram tiles", rank);
    return FL_ERR_OP;
  }
  FL_CUDA(raise_smem_limit(k_gg_gram, (int)((size_t)32 * R * 4)));
  s->stage_hh = (size_t)R * R * 4 + (size_t)8 * R * 4 <= 160 * 1024 ? 1 : 0;
  s->smem_w = (s->stage_hh ? (size_t)R * R * 4 : 0) + (size_t)8 * R * 4;
  FL_CUDA(raise_smem_limit(k_gg_w, (int)s->smem_w));
  FL_CUDA(cudaStreamSynchronize(st));
  *out = guard.release();
  return FL_OK;
}

// loss of the products in `red` (previous iteration) and/or the H update
static int gng_h(GnGen* s, cudaStream_t st, bool update, bool loss) {
  const int R = s->R, c_T = s->t->c_T, sms = s->t->sm_count;
  k_gg_hh<<<gg_grid((int64_t)R * R, sms), 256, 0, st>>>(s->H.as<double>(), R, c_T,
                                                        s->HH.as<double>(), s->HH32.as<float>());
  FL_CHECK_LAUNCH();
  if (loss) {
    const int n = s->it - 1;
    k_gg_loss<<<1, 256, 0, st>>>(s->red.as<double>(), s->H.as<double>(), s->HH.as<double>(), R,
                                 c_T, s->t_sq, s->loss_hist.as<double>(), n, s->loss_cap);
    FL_CHECK_LAUNCH();
    s->nloss = std::max(s->nloss, n + 1);
  }
  if (update) {
    k_gg_hupd<<<gg_grid((int64_t)R * c_T, sms), 256, 0, st>>>(s->red.as<double>(),
                                                             s->H.as<double>(), R, c_T,
                                                             s->Hn.as<double>());
    FL_CHECK_LAUNCH();
    std::swap(s->H.p, s->Hn.p);   // same size: swap the storage, not the owners
    k_gg_hh<<<gg_grid((int64_t)R * R, sms), 256, 0, st>>>(s->H.as<double>(), R, c_T,
                                                          s->HH.as<double>(), s->HH32.as<float>());
    FL_CHECK_LAUNCH();
    s->it++;
  }
  k_gg_ht<<<gg_grid((int64_t)R * c_T, sms), 256, 0, st>>>(s->H.as<double>(), R, c_T,
                                                         s->Ht32.as<float>());
  FL_CHECK_LAUNCH();
  return FL_OK;
}

// (optional W update) then P = W^T T and G = W^T W into `red`
static int gng_products(GnGen* s, cudaStream_t st, bool update) {
  fl_table* t = s->t;
  const int R = s->R, c_T = t->c_T;
  int rc;
  if (update) {
    if ((rc = do_lmm(t, s->Ht32.as<float>(), R, s->Q.as<float>(), st))) return rc;
    const unsigned nb = (unsigned)std::max<int64_t>(
        1, std::min<int64_t>(ceil_div(t->r_T, 8), 4 * (int64_t)t->sm_count));
    k_gg_w<<<nb, 256, s->smem_w, st>>>(s->W.as<float>(), s->Q.as<float>(), s->HH32.as<float>(),
                                       t->r_T, R, s->stage_hh);
    FL_CHECK_LAUNCH();
  }
  FL_CUDA(cudaMemsetAsync(s->red.p, 0, (size_t)R * c_T * 8, st));
  // P[j, tc] at red[j c_T + tc]
  if ((rc = do_tlmm(t, YView{s->W.as<float>(), R, 1}, R, s->red.as<double>(), 1, c_T, st))) return rc;
  const int npair = R * R;
  dim3 gg((unsigned)s->nblk_g, (unsigned)ceil_div(npair, 256 * GG_PP));
  k_gg_gram<<<gg, 256, (size_t)32 * R * 4, st>>>(s->W.as<float>(), t->r_T, R, s->rpb_g,
                                                 s->gpart.as<double>());
  FL_CHECK_LAUNCH();
  k_gg_reduce<<<(unsigned)ceil_div(npair, 256), 256, 0, st>>>(
      s->gpart.as<double>(), s->nblk_g, npair, s->red.as<double>() + (size_t)R * c_T);
  FL_CHECK_LAUNCH();
  return FL_OK;
}

int gng_partial(GnGen* s, cudaStream_t st) {
  int rc;
  if (!s->primed) {   // products of W_0 only
    if ((rc = gng_h(s, st, false, false))) return rc;
    s->primed = true;
    return gng_products(s, st, false);
  }
  if ((rc = gng_h(s, st, true, s->it > 0))) return rc;
  return gng_products(s, st, true);
}

int gng_run(GnGen* s, int iterations, cudaStream_t st) {
  auto step = [&]() -> int {
    int rc = gng_partial(s, st);
    if (!rc && s->comm) {
      int n = 0;
      double* red = gng_red(s, &n);
      rc = comm_allreduce(s->comm, red, (size_t)n, st);
    }
    return rc;
  };
  for (int i = 0; i < iterations; i++) {
    if (!s->primed) {
      int rc = step();
      if (rc) return rc;
    }
    int rc = step();
    if (rc) return rc;
  }
  return FL_OK;
}

double* gng_red(GnGen* s, int* len) {
  *len = s->R * s->t->c_T + s->R * s->R;
  return s->red.as<double>();
}

int gng_result(GnGen* s, double* w, double* h, double* loss, int n, int* n_done, cudaStream_t st) {
  fl_table* t = s->t;
  // the last iteration's loss, from the products of the final W
  if (s->it > 0 && s->nloss < s->it) {
    int rc = gng_h(s, st, false, true);
    if (rc) return rc;
  }
  if (w) {
    double* tmp = nullptr;
    const int64_t n_w = t->r_T * s->R;
    FL_CUDA(cudaMallocAsync((void**)&tmp, (size_t)n_w * 8 + 16, st));
    k_gg_w_out<<<gg_grid(n_w, t->sm_count), 256, 0, st>>>(s->W.as<float>(), n_w, tmp);
    FL_CHECK_LAUNCH();
    FL_CUDA(cudaMemcpyAsync(w, tmp, (size_t)n_w * 8, cudaMemcpyDefault, st));
    FL_CUDA(cudaFreeAsync(tmp, st));
  }
  if (h) FL_CUDA(cudaMemcpyAsync(h, s->H.p, (size_t)s->R * t->c_T * 8, cudaMemcpyDefault, st));
  FL_CUDA(cudaStreamSynchronize(st));
  const int nd = std::min(s->nloss, s->loss_cap);
  if (n_done) *n_done = nd;
  if (loss && n > 0) {
    const int m = std::min(n, nd);
    if (m > 0) FL_CUDA(cudaMemcpy(loss, s->loss_hist.p, (size_t)m * 8, cudaMemcpyDefault));
  }
  return FL_OK;
}

void gng_destroy(GnGen* s) { delete s; }

}  // namespace flb
