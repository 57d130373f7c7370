// Gaussian NMF by multiplicative updates over a factorized table (reference
// trainers.py:256-307, built on rmm / lmm of ops.py:219-253).
//
// The reference iteration is
//     P = W^T T;  [loss of the previous iteration from P, W^T W, H]
//     H <- H o P / (W^T W H + eps);  Q = T H^T;  W <- W o Q / (W H H^T + eps)
// and a final rmm for the last loss.  Here every product with T is one fused
// pass over the fact rows, and P / W^T W of the NEXT iteration are produced
// by the same pass that writes the new W:
//
//  U  k_gnmf_h       (1 CTA) loss(it-1) from P, G = W^T W, H; H <- H o P /
//                    (G H + eps); HH = H H^T; fp32 copies (fp64 math)
//  D1 k_gnmf_dim_g   G_d = S_d H_d^T (r_d x R) for every dimension source;
//                    zero Z_d
//  F  k_gnmf_fact    per device row p (per-warp TMA pipelines, W tile in a
//                    128B-swizzled layout, 3xTF32 mma.sync):
//                      q    = F[p] H_F^T + sum_d G_d[fk_d[p]]
//                      W[p] = W[p] o q / (W[p] HH + eps)       (TMA store)
//                      P_F += W[p]^T F[p],  G += W[p]^T W[p]
//                      Z_d[fk_d[p]] += W[p]   (I_d^T W: segment one-hot MMA,
//                                             fp64 atomics of fp32 partials)
//  D2 k_gnmf_dim_p   P_d = Z_d^T S_d (fp64 per-CTA partials)
//  R  k_gnmf_reduce  fixed-order reduction of all partials into red = [P | G]
//
// A prologue (F without the update, D2, R) produces P_0, G_0 from W_0, and a
// final U (loss only) records the last loss.  With fact rows sharded over
// GPUs, `red` is all-reduced between R and the next U.
#include <algorithm>
#include <cstdlib>

#include "internal.h"
#include "generic.h"
#include "mma_tf32.cuh"
#include "reduce.cuh"
#include "tc05.cuh"

namespace flb {

constexpr int GN_WARPS = 8;
constexpr int GN_FLUSH = 16;   // stages between fp32 -> fp64 flushes (512 rows)
constexpr double GN_EPS = 1e-12;   // trainers.py:29

struct GnState {
  int it;           // iterations started (H updates applied)
  int nloss;        // losses recorded (loss_hist[0 .. nloss))
  int pad[2];
};

struct GnFactArgs {
  int pf, c_T, R;
  int64_t r_T, nunits;
  int ng, sort_g;
  const int32_t* fk[MAX_GATHER];
  const float* Gd[MAX_GATHER];     // r_d x R
  double* Z[MAX_GATHER];           // r_d x R
  const float* H32;                // R x c_T
  const float* HH32;               // R x R
  const int32_t* f_tcol;
  double* wpart;                   // per-warp fp64 partials [MR*16 x (SC + R)]
  double* part;                    // per-CTA partials
  uint32_t stage_bytes, off_f, off_fk;
  int nst;
};

struct GnDimArgs {
  int ng, R, c_T;
  const float* S[MAX_GATHER];
  int pitch[MAX_GATHER], cols[MAX_GATHER];
  int64_t rows[MAX_GATHER];
  int nblk[MAX_GATHER];
  const int32_t* tcol[MAX_GATHER];
  float* Gd[MAX_GATHER];
  double* Z[MAX_GATHER];
  double* part[MAX_GATHER];        // nblk x (R x cols)
  const float* H32;
};

struct GnHArgs {
  int c_T, R, rank;
  double* H;                       // R x c_T fp64 master
  float* H32;
  float* HH32;
  const double* red;
  double t_sq;
  double* loss_hist;
  int loss_cap;
  GnState* state;
};

// ---------------------------------------------------------------------------
// U: loss of the previous iteration, H update, HH = H H^T (one CTA, fp64)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_gnmf_h(GnHArgs a, int do_update, int do_loss,
                                                int stage) {
  extern __shared__ double sh[];
  const int R = a.R, c_T = a.c_T, tid = threadIdx.x;
  double* GH = sh;                  // R x c_T
  double* HH = GH + R * c_T;        // R x R
  __shared__ double red_s[256];
  const double* P = a.red;
  const double* G = a.red + (size_t)R * c_T;
  // H and G staged in shared memory when they fit (every product reads them
  // R times); otherwise the products read the global copies
  double* Hs = stage ? HH + R * R : a.H;            // R x c_T
  double* Gs = stage ? Hs + R * c_T : const_cast<double*>(G);   // R x R
  if (stage) {
    for (int i = tid; i < R * c_T; i += blockDim.x) Hs[i] = a.H[i];
    for (int i = tid; i < R * R; i += blockDim.x) Gs[i] = G[i];
  }
  __syncthreads();
  // HH of the current H (loss uses H of the iteration the products were made with)
  for (int i = tid; i < R * R; i += blockDim.x) {
    int r = i / R, q = i - r * R;
    double s0 = 0.0, s1 = 0.0;
    int c = 0;
    for (; c + 1 < c_T; c += 2) {
      s0 += Hs[r * c_T + c] * Hs[q * c_T + c];
      s1 += Hs[r * c_T + c + 1] * Hs[q * c_T + c + 1];
    }
    if (c < c_T) s0 += Hs[r * c_T + c] * Hs[q * c_T + c];
    HH[i] = s0 + s1;
  }
  __syncthreads();
  if (do_loss) {
    double part = 0.0;
    for (int i = tid; i < R * c_T; i += blockDim.x) part -= 2.0 * P[i] * Hs[i];
    for (int i = tid; i < R * R; i += blockDim.x) part += Gs[i] * HH[i];
    red_s[tid] = part;
    __syncthreads();
    if (tid == 0) {
      // the products in `red` were made with W of iteration it - 1's update
      double s = a.t_sq;
      for (int i = 0; i < (int)blockDim.x; i++) s += red_s[i];
      const int n = a.state->it - 1;
      if (n >= 0 && n < a.loss_cap) a.loss_hist[n] = s;
      if (n + 1 > a.state->nloss) a.state->nloss = n + 1;
    }
    __syncthreads();
  }
  if (do_update) {
    // GH = G H (R x c_T), then H <- H o P / (GH + eps)
    for (int i = tid; i < R * c_T; i += blockDim.x) {
      int r = i / c_T, c = i - r * c_T;
      double s = 0.0;
      for (int q = 0; q < R; q++) s += Gs[r * R + q] * Hs[q * c_T + c];
      GH[i] = s;
    }
    __syncthreads();
    for (int i = tid; i < R * c_T; i += blockDim.x) {
      int r = i / c_T;
      const double h = r < a.rank ? Hs[i] * P[i] / (GH[i] + GN_EPS) : 0.0;
      a.H[i] = h;
      Hs[i] = h;
    }
    __syncthreads();
    for (int i = tid; i < R * R; i += blockDim.x) {
      int r = i / R, q = i - r * R;
      double s = 0.0;
      for (int c = 0; c < c_T; c++) s += Hs[r * c_T + c] * Hs[q * c_T + c];
      a.HH32[i] = (float)s;
    }
    if (tid == 0) a.state->it += 1;
  }
  for (int i = tid; i < R * c_T; i += blockDim.x) a.H32[i] = (float)Hs[i];
}

// ---------------------------------------------------------------------------
// D1: G_d = S_d H_d^T, zero Z_d
// ---------------------------------------------------------------------------
// thread per dimension row, R accumulators; H_d sits transposed in smem
template <int R>
__global__ void __launch_bounds__(256) k_gnmf_dim_g(GnDimArgs a) {
  const int d = blockIdx.y;
  if (d >= a.ng) return;
  extern __shared__ __align__(16) float sm_g[];   // pitch x R
  const int cols = a.cols[d], pitch = a.pitch[d];
  const int64_t rows = a.rows[d];
  for (int i = threadIdx.x; i < pitch * R; i += blockDim.x) {
    const int c = i / R, j = i - c * R;
    sm_g[i] = c < cols ? a.H32[(size_t)j * a.c_T + a.tcol[d][c]] : 0.f;
  }
  __syncthreads();
  for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < rows;
       row += (int64_t)gridDim.x * blockDim.x) {
    float acc[R];
#pragma unroll
    for (int j = 0; j < R; j++) acc[j] = 0.f;
    const float4* sr = reinterpret_cast<const float4*>(a.S[d] + row * pitch);
    const int n4 = pitch / 4;
    // batches of independent float4 loads: one latency per batch (4 at R = 32,
    // where the 32 accumulators already hold most of the registers)
    constexpr int NB = R >= 32 ? 4 : 8;
    for (int c0 = 0; c0 < n4; c0 += NB) {
      float4 vb[NB];
#pragma unroll
      for (int u = 0; u < NB; u++) vb[u] = c0 + u < n4 ? sr[c0 + u] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < NB; u++) {
        if (c0 + u >= n4) break;
        const float vv[4] = {vb[u].x, vb[u].y, vb[u].z, vb[u].w};
#pragma unroll
        for (int e = 0; e < 4; e++) {
          const float4* hr = reinterpret_cast<const float4*>(sm_g + ((c0 + u) * 4 + e) * R);
#pragma unroll
          for (int q = 0; q < R / 4; q++) {
            const float4 h = hr[q];
            acc[q * 4 + 0] = fmaf(vv[e], h.x, acc[q * 4 + 0]);
            acc[q * 4 + 1] = fmaf(vv[e], h.y, acc[q * 4 + 1]);
            acc[q * 4 + 2] = fmaf(vv[e], h.z, acc[q * 4 + 2]);
            acc[q * 4 + 3] = fmaf(vv[e], h.w, acc[q * 4 + 3]);
          }
        }
      }
    }
    float4* gr = reinterpret_cast<float4*>(a.Gd[d] + row * R);
    double2* zr = reinterpret_cast<double2*>(a.Z[d] + row * R);
#pragma unroll
    for (int q = 0; q < R / 4; q++) {
      gr[q] = make_float4(acc[q * 4], acc[q * 4 + 1], acc[q * 4 + 2], acc[q * 4 + 3]);
      zr[2 * q] = make_double2(0.0, 0.0);
      zr[2 * q + 1] = make_double2(0.0, 0.0);
    }
  }
}

// ---------------------------------------------------------------------------
// F: the fact-row pass
// ---------------------------------------------------------------------------
template <int R>
__device__ __forceinline__ int widx(int row, int col) {
  // element (row, col) of a 32 x R fp32 tile written by TMA with a (4R)-byte
  // swizzle: 16-byte chunk index XOR-ed with the row's swizzle phase
  constexpr int RB = R * 4;
  constexpr int CH = RB / 16;
  const int sw = ((row * RB) >> 7) & (CH - 1);
  return row * R + ((((col >> 2) ^ sw)) << 2) + (col & 3);
}

__device__ __forceinline__ uint32_t hi_bits(float x) { return __float_as_uint(x) & 0xffffe000u; }
__device__ __forceinline__ uint32_t lo_bits(float x) {
  return __float_as_uint(x - __uint_as_float(__float_as_uint(x) & 0xffffe000u));
}

template <int NR, int KC, bool UPDATE>
__global__ void __launch_bounds__(GN_WARPS * 32, 1)
    k_gnmf_fact(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmF,
                GnFactArgs a) {
  constexpr int R = NR * 8;
  constexpr int MR = (NR + 1) / 2;     // 16-rank tiles (W^T as the A operand)
  constexpr int SC = KC * 8;
  constexpr int FP = SC + 4;
  constexpr int WP = MR * 16 * (SC + R);   // per-warp fp64 partial entries
  extern __shared__ __align__(1024) char smem[];
  __shared__ uint64_t bar[GN_WARPS][4];

  // the swizzle phase of a W tile is taken from smem address bits [7:9]:
  // place everything relative to a 1024-byte aligned base
  char* sm = smem + ((1024u - (smem_u32(smem) & 1023u)) & 1023u);
  uint4* hf = reinterpret_cast<uint4*>(sm);            // KC*NR*32: B = H_F^T
  uint4* hh = hf + KC * NR * 32;                       // NR*NR*32: B = HH
  char* stages = sm + round_up((int64_t)((KC * NR + NR * NR) * 32 * 16), 1024);

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int pf = a.pf;

  if (UPDATE) {
    for (int i = threadIdx.x; i < KC * NR * 32; i += blockDim.x) {
      int l = i & 31, kn = i >> 5;
      int kc = kn / NR, n = kn - kc * NR;
      int gg = l >> 2, tt = l & 3;
      float b[2];
      for (int h = 0; h < 2; h++) {
        int col = kc * 8 + tt + 4 * h;
        int tc = col < pf ? a.f_tcol[col] : -1;
        b[h] = tc >= 0 ? a.H32[(size_t)(n * 8 + gg) * a.c_T + tc] : 0.f;
      }
      Split s0 = split_tf32(b[0]), s1 = split_tf32(b[1]);
      hf[i] = make_uint4(s0.hi, s1.hi, s0.lo, s1.lo);
    }
    for (int i = threadIdx.x; i < NR * NR * 32; i += blockDim.x) {
      int l = i & 31, kn = i >> 5;
      int kc = kn / NR, n = kn - kc * NR;
      int gg = l >> 2, tt = l & 3;
      Split s0 = split_tf32(a.HH32[(kc * 8 + tt) * R + n * 8 + gg]);
      Split s1 = split_tf32(a.HH32[(kc * 8 + tt + 4) * R + n * 8 + gg]);
      hh[i] = make_uint4(s0.hi, s1.hi, s0.lo, s1.lo);
    }
  }
  if (lane == 0) {
    for (int s = 0; s < a.nst; s++) mbar_init(&bar[warp][s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  const int64_t gw = (int64_t)blockIdx.x * GN_WARPS + warp;
  const int64_t NW = (int64_t)gridDim.x * GN_WARPS;
  const int64_t base = a.nunits / NW, rem = a.nunits % NW;
  const int64_t u0 = gw * base + min64(gw, rem);
  const int64_t cnt = base + (gw < rem ? 1 : 0);
  const bool has_sort = a.sort_g >= 0;
  const uint32_t tx = 32u * R * 4u + 32u * FP * 4u + (has_sort ? 128u : 0u);
  char* wsm = stages + (size_t)warp * a.nst * a.stage_bytes;
  uint64_t* wbar = bar[warp];
  double* wp = a.wpart + gw * WP;
  for (int i = lane; i < WP; i += 32) wp[i] = 0.0;
  __syncwarp();
  // W and F stream through once per pass: evict_first, so the per-warp fp64
  // partials (flushed every GN_FLUSH units) and the G_d / Z_d rows stay in L2
  const uint64_t pol_stream = l2_policy_evict_first();
  auto issue = [&](int s, int64_t unit) {
    char* st = wsm + (size_t)s * a.stage_bytes;
    mbar_arrive_expect_tx(&wbar[s], tx);
    tma_load_2d_hint(st, &tmW, 0, (int)(unit * 32), &wbar[s], pol_stream);
    tma_load_2d_hint(st + a.off_f, &tmF, 0, (int)(unit * 32), &wbar[s], pol_stream);
    if (has_sort) bulk_g2s(st + a.off_fk, a.fk[a.sort_g] + unit * 32, 128, &wbar[s]);
  };
  if (lane == 0)
    for (int s = 0; s < a.nst && s < cnt; s++) issue(s, u0 + s);

  float pacc[MR][KC][4], gacc[MR][NR][4];
#pragma unroll
  for (int m = 0; m < MR; m++) {
#pragma unroll
    for (int c = 0; c < KC; c++)
#pragma unroll
      for (int e = 0; e < 4; e++) pacc[m][c][e] = 0.f;
#pragma unroll
    for (int c = 0; c < NR; c++)
#pragma unroll
      for (int e = 0; e < 4; e++) gacc[m][c][e] = 0.f;
  }
  auto flush = [&]() {
#pragma unroll
    for (int m = 0; m < MR; m++)
#pragma unroll
      for (int e = 0; e < 4; e++) {
        const int row = m * 16 + g + (e >> 1) * 8;
#pragma unroll
        for (int c = 0; c < KC; c++) {
          wp[row * (SC + R) + c * 8 + 2 * t + (e & 1)] += (double)pacc[m][c][e];
          pacc[m][c][e] = 0.f;
        }
#pragma unroll
        for (int c = 0; c < NR; c++) {
          wp[row * (SC + R) + SC + c * 8 + 2 * t + (e & 1)] += (double)gacc[m][c][e];
          gacc[m][c][e] = 0.f;
        }
      }
  };

  int s = 0;            // stage slot and its mbarrier phase
  uint32_t ph = 0;
  for (int64_t i = 0; i < cnt; i++, s = (s + 1 == a.nst) ? 0 : s + 1, ph ^= (s == 0)) {
    mbar_wait(&wbar[s], ph);
    char* st = wsm + (size_t)s * a.stage_bytes;
    float* Wt = reinterpret_cast<float*>(st);
    const float* Fs = reinterpret_cast<const float*>(st + a.off_f);
    const int32_t* fks_s = reinterpret_cast<const int32_t*>(st + a.off_fk);
    const int64_t p0 = (u0 + i) * 32;
    int fkl[MAX_GATHER];
#pragma unroll
    for (int d = 0; d < MAX_GATHER; d++) {
      if (d >= a.ng) break;
      fkl[d] = (d == a.sort_g) ? fks_s[lane] : a.fk[d][p0 + lane];
    }

    if (UPDATE) {
      // one 16-row half at a time (halves the live accumulators: 8 warps of
      // 255 registers is this kernel's occupancy limit)
#pragma unroll 1
      for (int m = 0; m < 2; m++) {
        // ---- q = F H_F^T (3xTF32), v = W HH (3xTF32)
        float q[NR][4], v[NR][4];
#pragma unroll
        for (int n = 0; n < NR; n++)
#pragma unroll
          for (int e = 0; e < 4; e++) q[n][e] = v[n][e] = 0.f;
#pragma unroll
        for (int kc = 0; kc < KC; kc++) {
          uint32_t x[4];
          ldsm_x4(x[0], x[1], x[2], x[3],
                  Fs + (m * 16 + (lane & 15)) * FP + kc * 8 + (lane >> 4) * 4);
          uint32_t xh[4], xl[4];
#pragma unroll
          for (int e = 0; e < 4; e++) {
            xh[e] = x[e] & 0xffffe000u;
            xl[e] = __float_as_uint(__uint_as_float(x[e]) - __uint_as_float(xh[e]));
          }
          uint4 b[NR];
#pragma unroll
          for (int n = 0; n < NR; n++) b[n] = hf[(kc * NR + n) * 32 + lane];
          // the three split terms as three sweeps over independent accumulators
#pragma unroll
          for (int n = 0; n < NR; n++) mma_tf32(q[n], xh[0], xh[1], xh[2], xh[3], b[n].x, b[n].y);
#pragma unroll
          for (int n = 0; n < NR; n++) mma_tf32(q[n], xl[0], xl[1], xl[2], xl[3], b[n].x, b[n].y);
#pragma unroll
          for (int n = 0; n < NR; n++) mma_tf32(q[n], xh[0], xh[1], xh[2], xh[3], b[n].z, b[n].w);
        }
#pragma unroll
        for (int kc = 0; kc < NR; kc++) {
          const int row = m * 16 + (lane & 15);
          const int col = kc * 8 + (lane >> 4) * 4;
          uint32_t x[4];
          ldsm_x4(x[0], x[1], x[2], x[3], Wt + widx<R>(row, col));
          uint32_t xh[4], xl[4];
#pragma unroll
          for (int e = 0; e < 4; e++) {
            xh[e] = x[e] & 0xffffe000u;
            xl[e] = __float_as_uint(__uint_as_float(x[e]) - __uint_as_float(xh[e]));
          }
          uint4 b[NR];
#pragma unroll
          for (int n = 0; n < NR; n++) b[n] = hh[(kc * NR + n) * 32 + lane];
#pragma unroll
          for (int n = 0; n < NR; n++) mma_tf32(v[n], xh[0], xh[1], xh[2], xh[3], b[n].x, b[n].y);
#pragma unroll
          for (int n = 0; n < NR; n++) mma_tf32(v[n], xl[0], xl[1], xl[2], xl[3], b[n].x, b[n].y);
#pragma unroll
          for (int n = 0; n < NR; n++) mma_tf32(v[n], xh[0], xh[1], xh[2], xh[3], b[n].z, b[n].w);
        }
        // ---- gathers of the dimension products G_d[fk]
#pragma unroll
        for (int d = 0; d < MAX_GATHER; d++) {
          if (d >= a.ng) break;
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int f = __shfl_sync(0xffffffffu, fkl[d], m * 16 + h * 8 + g);
            if (f >= 0) {
              const float* gr = a.Gd[d] + (int64_t)f * R + 2 * t;
#pragma unroll
              for (int n = 0; n < NR; n++) {
                const float2 gv = *reinterpret_cast<const float2*>(gr + n * 8);
                q[n][h * 2] += gv.x;
                q[n][h * 2 + 1] += gv.y;
              }
            }
          }
        }
        __syncwarp();
        // ---- W <- W o q / (W HH + eps), in place in the swizzled tile
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int row = m * 16 + h * 8 + g;
#pragma unroll
          for (int n = 0; n < NR; n++) {
            float2* wptr = reinterpret_cast<float2*>(Wt + widx<R>(row, n * 8 + 2 * t));
            float2 w = *wptr;
            w.x = w.x * __fdividef(q[n][h * 2], v[n][h * 2] + 1e-12f);
            w.y = w.y * __fdividef(q[n][h * 2 + 1], v[n][h * 2 + 1] + 1e-12f);
            *wptr = w;
          }
        }
        __syncwarp();
      }
      __syncwarp();
      if (lane == 0) {
        fence_proxy_async();
        tma_store_2d_hint(&tmW, 0, (int)p0, Wt, pol_stream);
        bulk_commit();
      }
    }
    // ---- P_F += W^T F,  G += W^T W  (3xTF32; W^T fragments from the tile)
#pragma unroll
    for (int kb = 0; kb < 4; kb++) {
      const int r0 = kb * 8 + t, r1 = r0 + 4;
      uint32_t ah[MR][4], alo[MR][4];
#pragma unroll
      for (int m = 0; m < MR; m++) {
        const float w0 = Wt[widx<R>(r0, (m * 16 + g) % R)];
        const float w1 = (m * 16 + g + 8 < R) ? Wt[widx<R>(r0, m * 16 + g + 8)] : 0.f;
        const float w2 = Wt[widx<R>(r1, (m * 16 + g) % R)];
        const float w3 = (m * 16 + g + 8 < R) ? Wt[widx<R>(r1, m * 16 + g + 8)] : 0.f;
        const float wa[4] = {m * 16 + g < R ? w0 : 0.f, w1, m * 16 + g < R ? w2 : 0.f, w3};
#pragma unroll
        for (int e = 0; e < 4; e++) {
          ah[m][e] = hi_bits(wa[e]);
          alo[m][e] = lo_bits(wa[e]);
        }
      }
#pragma unroll
      for (int c = 0; c < KC; c++) {
        const float b0 = Fs[r0 * FP + c * 8 + g], b1 = Fs[r1 * FP + c * 8 + g];
        const uint32_t bh0 = hi_bits(b0), bh1 = hi_bits(b1);
        const uint32_t bl0 = lo_bits(b0), bl1 = lo_bits(b1);
#pragma unroll
        for (int m = 0; m < MR; m++) {
          mma_tf32(pacc[m][c], ah[m][0], ah[m][1], ah[m][2], ah[m][3], bh0, bh1);
          mma_tf32(pacc[m][c], alo[m][0], alo[m][1], alo[m][2], alo[m][3], bh0, bh1);
          mma_tf32(pacc[m][c], ah[m][0], ah[m][1], ah[m][2], ah[m][3], bl0, bl1);
        }
      }
#pragma unroll
      for (int n = 0; n < NR; n++) {
        const float b0 = Wt[widx<R>(r0, n * 8 + g)], b1 = Wt[widx<R>(r1, n * 8 + g)];
        const uint32_t bh0 = hi_bits(b0), bh1 = hi_bits(b1);
        const uint32_t bl0 = lo_bits(b0), bl1 = lo_bits(b1);
#pragma unroll
        for (int m = 0; m < MR; m++) {
          // G = W^T W is symmetric: tiles strictly below the diagonal are
          // skipped (the reduction reads their transposes)
          if (n < 2 * m) continue;
          mma_tf32(gacc[m][n], ah[m][0], ah[m][1], ah[m][2], ah[m][3], bh0, bh1);
          mma_tf32(gacc[m][n], alo[m][0], alo[m][1], alo[m][2], alo[m][3], bh0, bh1);
          mma_tf32(gacc[m][n], ah[m][0], ah[m][1], ah[m][2], ah[m][3], bl0, bl1);
        }
      }
    }
    // ---- Z_d[fk] += W rows: lane = rank column, the unit's 32 rows in order,
    // one fp64 atomic per run of equal FK (run ends from one ballot).  Sums
    // of the fp32 run partials are exact in fp64 here, so the result does
    // not depend on the order the atomics land in.
#pragma unroll
    for (int d = 0; d < MAX_GATHER; d++) {
      if (d >= a.ng) break;
      const int key = fkl[d];
      const int knext = __shfl_down_sync(0xffffffffu, key, 1);
      const unsigned ends = __ballot_sync(0xffffffffu, lane == 31 || knext != key);
      if (__popc(ends) <= 2) {
        // one or two runs cover the unit (the common case for the sorted
        // source): lane = (4-column group, row group), float4 row reads into
        // one accumulator per run, then a fixed xor tree over the row groups
        constexpr int CG = R / 4, RG = 32 / CG;
        const int cg = lane % CG, rg = lane / CG;
        const int last0 = __ffs(ends) - 1;           // last row of the first run
        float4 acc[2] = {make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)};
#pragma unroll
        for (int k = 0; k < CG; k++) {
          const int p = rg * CG + k;
          const float4 v = *reinterpret_cast<const float4*>(Wt + widx<R>(p, cg * 4));
          const float m0 = p <= last0 ? 1.f : 0.f, m1 = 1.f - m0;   // exact 0 / 1 weights
          acc[0].x = fmaf(m0, v.x, acc[0].x); acc[0].y = fmaf(m0, v.y, acc[0].y);
          acc[0].z = fmaf(m0, v.z, acc[0].z); acc[0].w = fmaf(m0, v.w, acc[0].w);
          acc[1].x = fmaf(m1, v.x, acc[1].x); acc[1].y = fmaf(m1, v.y, acc[1].y);
          acc[1].z = fmaf(m1, v.z, acc[1].z); acc[1].w = fmaf(m1, v.w, acc[1].w);
        }
#pragma unroll
        for (int u = 0; u < 2; u++) {
          const int k2 = __shfl_sync(0xffffffffu, key, u == 0 ? last0 : 31);
          if (u == 1 && last0 == 31) break;
#pragma unroll
          for (int o = CG; o < 32; o <<= 1) {
            acc[u].x += __shfl_xor_sync(0xffffffffu, acc[u].x, o);
            acc[u].y += __shfl_xor_sync(0xffffffffu, acc[u].y, o);
            acc[u].z += __shfl_xor_sync(0xffffffffu, acc[u].z, o);
            acc[u].w += __shfl_xor_sync(0xffffffffu, acc[u].w, o);
          }
          if (k2 >= 0 && rg == 0) {
            double* zr = a.Z[d] + (int64_t)k2 * R + cg * 4;
            atomicAdd(zr + 0, (double)acc[u].x);
            atomicAdd(zr + 1, (double)acc[u].y);
            atomicAdd(zr + 2, (double)acc[u].z);
            atomicAdd(zr + 3, (double)acc[u].w);
          }
        }
        continue;
      }
      const int col = lane < R ? lane : 0;
      float run = 0.f;
#pragma unroll 8
      for (int p = 0; p < 32; p++) {
        run += Wt[widx<R>(p, col)];
        if ((ends >> p) & 1u) {
          const int k = __shfl_sync(0xffffffffu, key, p);
          if (k >= 0 && lane < R) atomicAdd(a.Z[d] + (int64_t)k * R + lane, (double)run);
          run = 0.f;
        }
      }
    }
    __syncwarp();
    if (lane == 0 && i + a.nst < cnt) {
      if (UPDATE) bulk_wait_read<0>();   // the W store has left this stage
      fence_proxy_async();
      issue(s, u0 + i + a.nst);
    }
    if ((i % GN_FLUSH) == GN_FLUSH - 1) flush();
  }
  flush();
  if (UPDATE && lane == 0) bulk_wait<0>();
  __syncthreads();
  // CTA partial (fixed warp order): [R x SC] P_F | [R x R] G
  double* out = a.part + (int64_t)blockIdx.x * (R * SC + R * R);
  const double* wbase = a.wpart + (int64_t)blockIdx.x * GN_WARPS * WP;
  for (int i = threadIdx.x; i < R * (SC + R); i += blockDim.x) {
    const int row = i / (SC + R), col = i - row * (SC + R);
    double s = 0.0;
    for (int w2 = 0; w2 < GN_WARPS; w2++) s += wbase[(int64_t)w2 * WP + row * (SC + R) + col];
    if (col < SC) out[row * SC + col] = s;
    else out[R * SC + row * R + (col - SC)] = s;
  }
}

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
#include "gnmf_tc.cuh"
#include "gnmf_t5.cuh"

// ---------------------------------------------------------------------------
// D2: P_d = Z_d^T S_d (fp64 per-CTA partials over row ranges)
// ---------------------------------------------------------------------------
// P_d[j, c] = sum_r Z_d[r, j] S_d[r, c]: 32-row tiles of S and Z (Z converted
// to fp32 once) in smem; thread = (column, 8 ranks); fp32 within a tile,
// fp64 across tiles.  Each thread holds its share of the NEXT tile in
// registers (loads issued before the current tile's math): one load latency
// per CTA instead of one per tile.  Pitches up to 288 floats.
constexpr int GN_P_SL = 9;
template <int R, int U, int SL>
__global__ void __launch_bounds__(256) k_gnmf_dim_p(GnDimArgs a) {
  const int d = blockIdx.y;
  if (d >= a.ng || (int)blockIdx.x >= a.nblk[d]) return;
  constexpr int JB = 8, NJB = R / JB;
  constexpr int ZL = (32 * R / 2 + 255) / 256;   // double2 slots per thread
  __shared__ float ss[32 * 257];
  __shared__ __align__(16) float zs[32 * R];
  const int cols = a.cols[d], pitch = a.pitch[d], pitch4 = pitch / 4;
  const int64_t rows = a.rows[d];
  const int nb = a.nblk[d];
  const int64_t rpb = ceil_div(ceil_div(rows, nb), 32) * 32;
  const int64_t r0 = blockIdx.x * rpb, r1 = min64(rows, r0 + rpb);
  const int nwork = cols * NJB;
  const int nS4 = 32 * pitch4;
  const int tid = threadIdx.x;
  const float4* S4 = reinterpret_cast<const float4*>(a.S[d]);
  const double2* Z2 = reinterpret_cast<const double2*>(a.Z[d]);
  float4 pv[SL];
  double2 pz[ZL];
  auto load = [&](int64_t rb) {
#pragma unroll
    for (int sl = 0; sl < SL; sl++) {
      const int i = tid + sl * 256;
      const int r = i / pitch4, c4 = i - r * pitch4;
      pv[sl] = (i < nS4 && rb + r < r1) ? S4[(rb + r) * pitch4 + c4]
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int zl = 0; zl < ZL; zl++) {
      const int i = tid + zl * 256;   // double2 index inside the tile
      const int r = (2 * i) / R;
      pz[zl] = (i < 16 * R && rb + r < r1) ? Z2[rb * (R / 2) + i] : make_double2(0.0, 0.0);
    }
  };
  double acc64[U][JB];
#pragma unroll
  for (int u = 0; u < U; u++)
#pragma unroll
    for (int j = 0; j < JB; j++) acc64[u][j] = 0.0;
  if (r0 < r1) load(r0);
  for (int64_t rb = r0; rb < r1; rb += 32) {
    __syncthreads();   // the previous tile's math is done with ss / zs
#pragma unroll
    for (int sl = 0; sl < SL; sl++) {
      const int i = tid + sl * 256;
      if (i < nS4) {   // padding columns (c >= cols) are not stored
        const int r = i / pitch4, c = 4 * (i - r * pitch4);
        if (c + 0 < cols) ss[r * 257 + c + 0] = pv[sl].x;
        if (c + 1 < cols) ss[r * 257 + c + 1] = pv[sl].y;
        if (c + 2 < cols) ss[r * 257 + c + 2] = pv[sl].z;
        if (c + 3 < cols) ss[r * 257 + c + 3] = pv[sl].w;
      }
    }
#pragma unroll
    for (int zl = 0; zl < ZL; zl++) {
      const int i = tid + zl * 256;
      if (i < 16 * R)
        *reinterpret_cast<float2*>(zs + 2 * i) = make_float2((float)pz[zl].x, (float)pz[zl].y);
    }
    __syncthreads();
    if (rb + 32 < r1) load(rb + 32);   // in flight during this tile's math
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int w = tid + u * 256;
      if (w >= nwork) break;
      const int c = w % cols, jb = w / cols;
      float acc[JB];
#pragma unroll
      for (int j = 0; j < JB; j++) acc[j] = 0.f;
#pragma unroll 8
      for (int r = 0; r < 32; r++) {
        const float v = ss[r * 257 + c];
        const float4 z0 = *reinterpret_cast<const float4*>(zs + r * R + jb * JB);
        const float4 z1 = *reinterpret_cast<const float4*>(zs + r * R + jb * JB + 4);
        acc[0] = fmaf(z0.x, v, acc[0]); acc[1] = fmaf(z0.y, v, acc[1]);
        acc[2] = fmaf(z0.z, v, acc[2]); acc[3] = fmaf(z0.w, v, acc[3]);
        acc[4] = fmaf(z1.x, v, acc[4]); acc[5] = fmaf(z1.y, v, acc[5]);
        acc[6] = fmaf(z1.z, v, acc[6]); acc[7] = fmaf(z1.w, v, acc[7]);
      }
#pragma unroll
      for (int j = 0; j < JB; j++) acc64[u][j] += (double)acc[j];
    }
  }
#pragma unroll
  for (int u = 0; u < U; u++) {
    const int w = tid + u * 256;
    if (w >= nwork) break;
    const int c = w % cols, jb = w / cols;
#pragma unroll
    for (int j = 0; j < JB; j++)
      a.part[d][(int64_t)blockIdx.x * R * cols + (jb * JB + j) * cols + c] = acc64[u][j];
  }
}

static void gn_dim_g_launch(int R, dim3 g, size_t smem, cudaStream_t st, const GnDimArgs& a) {
  if (R == 8) k_gnmf_dim_g<8><<<g, 256, smem, st>>>(a);
  else if (R == 16) k_gnmf_dim_g<16><<<g, 256, smem, st>>>(a);
  else k_gnmf_dim_g<32><<<g, 256, smem, st>>>(a);
}
// k_gnmf_dim_p<R, U, SL> for the dimension widths (few registers when narrow)
template <int R>
static const void* gn_dim_p_ptr_r(int U, int SL) {
  if (U == 1) {
    if (SL <= 3) return (const void*)k_gnmf_dim_p<R, 1, 3>;
    if (SL <= 5) return (const void*)k_gnmf_dim_p<R, 1, 5>;
    return (const void*)k_gnmf_dim_p<R, 1, 9>;
  }
  if (SL <= 3) return (const void*)k_gnmf_dim_p<R, 2, 3>;
  if (SL <= 5) return (const void*)k_gnmf_dim_p<R, 2, 5>;
  return (const void*)k_gnmf_dim_p<R, 2, 9>;
}
static const void* gn_dim_p_ptr(int R, int U, int SL) {
  return R == 8 ? gn_dim_p_ptr_r<8>(U, SL) : R == 16 ? gn_dim_p_ptr_r<16>(U, SL)
                                                     : gn_dim_p_ptr_r<32>(U, SL);
}
static cudaError_t gn_dim_p_launch(const void* fn, dim3 g, size_t smem, cudaStream_t st,
                                   const GnDimArgs& a) {
  void* args[] = {const_cast<GnDimArgs*>(&a)};
  return cudaLaunchKernel(fn, g, dim3(256), args, smem, st);
}

// ---------------------------------------------------------------------------
// R: red = [P | G], each element reduced over the partials in a fixed order
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_gnmf_reduce(const RedDesc* descs, int n, double* red) {
  reduce_descs(descs, n, red);
}

__global__ void k_gnmf_w_in(const double* __restrict__ w0, const int32_t* __restrict__ perm,
                            int64_t r_pad, int rank, int R, float* __restrict__ W) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= r_pad * R) return;
  int64_t p = idx / R;
  int j = (int)(idx - p * R);
  int32_t tr = perm[p];
  W[idx] = (tr >= 0 && j < rank) ? (float)w0[(int64_t)tr * rank + j] : 0.f;
}

__global__ void k_gnmf_w_out(const float* __restrict__ W, const int32_t* __restrict__ perm,
                             int64_t r_T, int rank, int R, double* __restrict__ out) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= r_T * rank) return;
  int64_t p = idx / rank;
  int j = (int)(idx - p * rank);
  out[(int64_t)perm[p] * rank + j] = (double)W[p * R + j];
}

#define GN_CASES(X, U) \
  X(1, 1, U) X(1, 2, U) X(1, 3, U) X(1, 4, U) X(1, 6, U) X(1, 8, U) \
  X(2, 1, U) X(2, 2, U) X(2, 3, U) X(2, 4, U) X(2, 6, U) X(2, 8, U) \
  X(4, 1, U) X(4, 2, U) X(4, 3, U) X(4, 4, U) X(4, 6, U) X(4, 8, U)
static int gn_kc_for(int pf) {
  const int need = (pf + 7) / 8;
  const int opts[] = {1, 2, 3, 4, 6, 8};
  for (int v : opts)
    if (v >= need) return v;
  return -1;
}
static const void* gn_fact_ptr(int nr, int kc, bool upd) {
#define GN_PTR(NR_, KC_, U_) \
  if (nr == NR_ && kc == KC_ && upd == U_) return (const void*)k_gnmf_fact<NR_, KC_, U_>;
  GN_CASES(GN_PTR, true) GN_CASES(GN_PTR, false)
#undef GN_PTR
  return nullptr;
}
static void gn_fact_launch(int nr, int kc, bool upd, const CUtensorMap& tw, const CUtensorMap& tf,
                           const GnFactArgs& a, int grid, size_t smem, cudaStream_t st) {
#define GN_LAUNCH(NR_, KC_, U_)                                                         \
  if (nr == NR_ && kc == KC_ && upd == U_) {                                            \
    k_gnmf_fact<NR_, KC_, U_><<<grid, GN_WARPS * 32, smem, st>>>(tw, tf, a);            \
    return;                                                                             \
  }
  GN_CASES(GN_LAUNCH, true) GN_CASES(GN_LAUNCH, false)
#undef GN_LAUNCH
}

}  // namespace flb

using namespace flb;

struct fl_gnmf {
  CUtensorMap tmW, tmF;
  // tcgen05 fact pass (R = 32, <= 32 streamed columns): 128-row tile maps
  bool tc = false;
  CUtensorMap tmWt, tmFt;
  GnTcArgs ta{};
  GtGeom gm{};
  DevBuf scratch;
  fl_table* t = nullptr;
  int rank = 0, R = 0, NR = 0, KC = 0, SC = 0;
  GnFactArgs fa{};
  GnDimArgs da{};
  GnHArgs ha{};
  int nblk_fact = 0, grid_g = 1, grid_p = 1, grid_red = 1;
  const void* fn_p = nullptr;   // k_gnmf_dim_p<R, U, SL> chosen for the dimension widths
  size_t smem_fact = 0, smem_g = 0, smem_p = 0, smem_h = 0;
  int stage_h = 0;   // k_gnmf_h stages H and G in shared memory
  DevBuf descs;
  int n_desc = 0;
  DevBuf W, H, H32, HH32, Gd, Z, wpart, part_fact, part_dim, red, loss_hist, state;
  int loss_cap = 1 << 16;
  bool primed = false;
  cudaGraphExec_t graph = nullptr;
  cudaStream_t cap_stream = nullptr;
  // tcgen05 pass with MN-major row-contraction operands (gnmf_t5.cuh)
  bool t5 = false;
  CUtensorMap tmW5, tmF5, tmWs;
  GnT5Args g5a{};
  G5Geom g5g{};
  DevBuf scratch5;
  GnGen* gen = nullptr;   // width-general session (generic.cu) when the fused pass does not apply
  fl_comm* comm = nullptr;  // sharded run(): all-reduce of `red` after every products pass
};

namespace flb {

static void gn_fact_any(fl_gnmf* s, bool update, cudaStream_t st) {
  if (s->t5) {
    const size_t smem = s->g5g.total + 1024;
    if (update)
      k_gnmf_t5<true><<<s->nblk_fact, G5_THREADS, smem, st>>>(s->tmW5, s->tmF5, s->tmWs, s->g5a,
                                                              s->g5g);
    else
      k_gnmf_t5<false><<<s->nblk_fact, G5_THREADS, smem, st>>>(s->tmW5, s->tmF5, s->tmWs, s->g5a,
                                                               s->g5g);
  } else if (s->tc) {
    const size_t smem = s->gm.total + 1024;
    if (update)
      k_gnmf_tc<true><<<s->nblk_fact, GT_THREADS, smem, st>>>(s->tmWt, s->tmFt, s->ta, s->gm);
    else
      k_gnmf_tc<false><<<s->nblk_fact, GT_THREADS, smem, st>>>(s->tmWt, s->tmFt, s->ta, s->gm);
  } else {
    gn_fact_launch(s->NR, s->KC, update, s->tmW, s->tmF, s->fa, s->nblk_fact, s->smem_fact, st);
  }
}

static int gn_products(fl_gnmf* s, cudaStream_t st, bool update) {
  if (update && s->da.ng > 0) {
    gn_dim_g_launch(s->R, dim3(s->grid_g, s->da.ng), s->smem_g, st, s->da);
    FL_CHECK_LAUNCH();
  } else {
    for (int d = 0; d < s->da.ng; d++)
      FL_CUDA(cudaMemsetAsync(s->da.Z[d], 0, (size_t)s->da.rows[d] * s->R * 8, st));
  }
  gn_fact_any(s, update, st);
  FL_CHECK_LAUNCH();
  if (s->da.ng > 0) {
    FL_CUDA(gn_dim_p_launch(s->fn_p, dim3(s->grid_p, s->da.ng), s->smem_p, st, s->da));
    FL_CHECK_LAUNCH();
  }
  k_gnmf_reduce<<<s->grid_red, 256, 0, st>>>(s->descs.as<RedDesc>(), s->n_desc,
                                             s->red.as<double>());
  FL_CHECK_LAUNCH();
  return FL_OK;
}

static int gn_h(fl_gnmf* s, cudaStream_t st, bool update, bool loss) {
  k_gnmf_h<<<1, 256, s->smem_h, st>>>(s->ha, update ? 1 : 0, loss ? 1 : 0, s->stage_h);
  FL_CHECK_LAUNCH();
  return FL_OK;
}

// products, then (sharded) the all-reduce of [W^T T | W^T W]
static int gn_products_x(fl_gnmf* s, cudaStream_t st, bool update) {
  int rc = gn_products(s, st, update);
  if (rc || !s->comm) return rc;
  return comm_allreduce(s->comm, s->red.as<double>(),
                        (size_t)s->R * s->t->c_T + (size_t)s->R * s->R, st);
}

}  // namespace flb

extern "C" {

static int gn_create_fused(fl_table* t, int32_t rank, const double* w0, const double* h0,
                           double t_sq, fl_gnmf** out, void* stream) {
  if (!t || !t->finalized || !w0 || !h0 || !out) {
    set_error("fl_gnmf_create: bad arguments");
    return FL_ERR_ARG;
  }
  if (rank < 1 || rank > std::min<int64_t>(t->r_T, t->c_T)) {
    set_error("rank = %d exceeds min(shape) = %lld", rank,
              (long long)std::min<int64_t>(t->r_T, t->c_T));
    return FL_ERR_CONFIG;
  }
  const int R = rank <= 8 ? 8 : rank <= 16 ? 16 : rank <= 32 ? 32 : -1;
  const int KC = gn_kc_for(t->pf);
  if (R < 0 || KC < 0 || (int)t->g.size() > MAX_GATHER) {
    set_error("fused GNMF supports rank <= 32, <= 60 streamed columns and <= %d gathered "
              "sources (rank=%d, streamed pitch=%d)", MAX_GATHER, rank, t->pf);
    return FL_ERR_OP;
  }
  FL_CUDA(cudaSetDevice(t->device));
  cudaStream_t st = (cudaStream_t)stream;
  auto* s = new fl_gnmf();
  std::unique_ptr<fl_gnmf> guard(s);
  s->t = t;
  s->rank = rank;
  s->R = R;
  s->NR = R / 8;
  s->KC = KC;
  s->SC = KC * 8;
  const int NR = s->NR, SC = s->SC, MR = (NR + 1) / 2, FP = SC + 4;
  const int c_T = t->c_T, ng = (int)t->g.size();
  int rc;
  // W (device order, padded rank) and H
  if ((rc = s->W.alloc((size_t)t->r_pad * R * 4))) return rc;
  {
    double* w0d = nullptr;
    FL_CUDA(cudaMallocAsync((void**)&w0d, (size_t)t->r_T * rank * 8 + 16, st));
    if (int rc = h2d_copy(w0d, w0, (size_t)t->r_T * rank * 8, st)) return rc;
    k_gnmf_w_in<<<(unsigned)ceil_div(t->r_pad * R, 256), 256, 0, st>>>(
        w0d, t->perm->as<int32_t>(), t->r_pad, rank, R, s->W.as<float>());
    FL_CHECK_LAUNCH();
    FL_CUDA(cudaFreeAsync(w0d, st));
  }
  if ((rc = s->H.alloc((size_t)R * c_T * 8))) return rc;
  FL_CUDA(cudaMemsetAsync(s->H.p, 0, (size_t)R * c_T * 8, st));
  FL_CUDA(cudaMemcpyAsync(s->H.p, h0, (size_t)rank * c_T * 8, cudaMemcpyDefault, st));
  if ((rc = s->H32.alloc((size_t)R * c_T * 4))) return rc;
  if ((rc = s->HH32.alloc((size_t)R * R * 4))) return rc;
  FL_CUDA(cudaMemsetAsync(s->HH32.p, 0, (size_t)R * R * 4, st));
  size_t gd_total = 0;
  for (auto& g : t->g) gd_total += (size_t)g.rows * R;
  if ((rc = s->Gd.alloc(gd_total * 4 + 16))) return rc;
  if ((rc = s->Z.alloc(gd_total * 8 + 16))) return rc;
  if ((rc = s->red.alloc(((size_t)R * c_T + R * R) * 8))) return rc;
  FL_CUDA(cudaMemsetAsync(s->red.p, 0, ((size_t)R * c_T + R * R) * 8, st));
  if ((rc = s->loss_hist.alloc((size_t)s->loss_cap * 8))) return rc;
  if ((rc = s->state.alloc(sizeof(GnState)))) return rc;
  FL_CUDA(cudaMemsetAsync(s->state.p, 0, sizeof(GnState), st));

  // ---- fact pass
  if ((rc = make_tmap_2d(&s->tmW, s->W.p, (uint64_t)t->r_pad, (uint64_t)R, (uint64_t)R * 4, 32,
                         (uint32_t)R, R * 4)))
    return rc;
  if ((rc = make_tmap_2d(&s->tmF, t->F->p, (uint64_t)t->r_pad, (uint64_t)t->pf,
                         (uint64_t)t->pf * 4, 32, (uint32_t)FP, 0)))
    return rc;
  GnFactArgs& fa = s->fa;
  fa.pf = t->pf;
  fa.c_T = c_T;
  fa.R = R;
  fa.r_T = t->r_T;
  fa.nunits = t->r_pad / 32;
  fa.ng = ng;
  fa.sort_g = t->sort_g;
  {
    size_t o = 0;
    for (int d = 0; d < ng; d++) {
      fa.fk[d] = t->g[d].fk->as<int32_t>();
      fa.Gd[d] = s->Gd.as<float>() + o;
      fa.Z[d] = s->Z.as<double>() + o;
      o += (size_t)t->g[d].rows * R;
    }
  }
  fa.H32 = s->H32.as<float>();
  fa.HH32 = s->HH32.as<float>();
  fa.f_tcol = t->d_f_tcol->as<int32_t>();
  fa.off_f = (uint32_t)(32 * R * 4);
  fa.off_fk = fa.off_f + (uint32_t)(32 * FP * 4);
  fa.stage_bytes = (uint32_t)round_up(fa.off_fk + 128, 1024);
  const size_t fixed = round_up((int64_t)((KC * NR + NR * NR) * 32 * 16), 1024);
  int nst = (int)((200 * 1024 - fixed) / ((size_t)GN_WARPS * fa.stage_bytes));
  if (const char* e = getenv("FL_GN_NST")) nst = atoi(e);
  fa.nst = std::max(2, std::min(4, nst));
  s->smem_fact = fixed + (size_t)GN_WARPS * fa.nst * fa.stage_bytes + 1024;  // + alignment slack
  if (s->smem_fact > 227 * 1024) {
    set_error("fused GNMF: shared memory budget exceeded (%zu bytes)", s->smem_fact);
    return FL_ERR_OP;
  }
  int occ = 1;
  for (int u = 0; u < 2; u++) {
    const void* kf = gn_fact_ptr(NR, KC, u == 0);
    FL_CUDA(raise_smem_limit(kf, (int)s->smem_fact));
    if (u == 0)
      FL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kf, GN_WARPS * 32,
                                                            s->smem_fact));
  }
  occ = std::max(1, occ);
  s->nblk_fact = (int)std::max<int64_t>(
      1, std::min<int64_t>(ceil_div(fa.nunits, GN_WARPS), (int64_t)t->sm_count * occ));
  // tcgen05 fact pass (opt-in, FL_GN_TC=1; R = 32, <= 32 streamed columns,
  // <= 2 gathered sources): parity-green but slower than the mma.sync pass at
  // C4 (profiles/r01_gnmf_tc_vs_mma.txt)
  {
    const char* e = getenv("FL_GN_TC");
    const bool want = e && atoi(e) != 0;
    const GtGeom gm = gt_geom(SC, ng);
    if (want && R == GT_R && t->pf <= 32 && ng <= GT_NG && gm.total + 1024 <= 227 * 1024) {
      s->tc = true;
      s->gm = gm;
      if ((rc = make_tmap_2d(&s->tmWt, s->W.p, (uint64_t)t->r_pad, (uint64_t)R, (uint64_t)R * 4,
                             GT_TILE, 32, 128)))
        return rc;
      if ((rc = make_tmap_2d(&s->tmFt, t->F->p, (uint64_t)t->r_pad, (uint64_t)t->pf,
                             (uint64_t)t->pf * 4, GT_TILE, 32, 128)))
        return rc;
      const int64_t ntiles = t->r_pad / GT_TILE;
      s->nblk_fact = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, t->sm_count));
      GnTcArgs& ta = s->ta;
      ta.pf = t->pf;
      ta.c_T = c_T;
      ta.SC = SC;
      ta.QK = SC / 8;
      ta.r_T = t->r_T;
      ta.ntiles = ntiles;
      ta.ng = ng;
      ta.sort_g = t->sort_g;
      for (int d = 0; d < ng; d++) {
        ta.fk[d] = fa.fk[d];
        ta.Gd[d] = fa.Gd[d];
        ta.Z[d] = fa.Z[d];
      }
      ta.H32 = fa.H32;
      ta.HH32 = fa.HH32;
      ta.f_tcol = fa.f_tcol;
      if ((rc = s->scratch.alloc((size_t)s->nblk_fact * GT_TILE * 32 * 8))) return rc;
      ta.scratch = s->scratch.as<double>();
      FL_CUDA(raise_smem_limit(k_gnmf_tc<true>, (int)(gm.total + 1024)));
      FL_CUDA(raise_smem_limit(k_gnmf_tc<false>, (int)(gm.total + 1024)));
    }
  }
  // default: the tcgen05 pass with MN-major row-contraction operands
  // (gnmf_t5.cuh) for rank tile 32, <= 28 streamed columns, <= 1 gathered
  // source (the sort source): C4 fact pass 5.56 ms vs 6.2 ms for the
  // mma.sync pass (profiles/r02_gnmf_t5.txt)
  {
    const char* e5 = getenv("FL_GN_T5");
    const bool on = !(e5 && atoi(e5) == 0);   // default; FL_GN_T5=0 selects the mma.sync pass
    const G5Geom g5 = g5_geom();
    if (on && !s->tc && R == 32 && t->pf <= 28 && ng <= 1 && (ng == 0 || t->sort_g == 0) &&
        g5.total + 1024 <= 227 * 1024) {
      s->t5 = true;
      s->g5g = g5;
      s->SC = 32;
      if ((rc = make_tmap_2d(&s->tmW5, s->W.p, (uint64_t)t->r_pad, 32, 128, G5_TILE, 32, 128)))
        return rc;
      if ((rc = make_tmap_2d(&s->tmF5, t->F->p, (uint64_t)t->r_pad, (uint64_t)t->pf,
                             (uint64_t)t->pf * 4, G5_TILE, 32, 128)))
        return rc;
      if ((rc = make_tmap_2d(&s->tmWs, s->W.p, (uint64_t)t->r_pad, 32, 128, G5_TILE, 32,
                             kSwz128Atom32)))
        return rc;
      const int64_t ntiles = t->r_pad / G5_TILE;
      s->nblk_fact = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, t->sm_count));
      if ((rc = s->scratch5.alloc((size_t)s->nblk_fact * G5_TILE * 64 * 8))) return rc;
      GnT5Args& ga = s->g5a;
      ga.pf = t->pf;
      ga.c_T = c_T;
      ga.r_T = t->r_T;
      ga.ntiles = ntiles;
      ga.ng = ng;
      ga.fk = ng ? fa.fk[0] : nullptr;
      ga.Gd = ng ? fa.Gd[0] : nullptr;
      ga.Z = ng ? fa.Z[0] : nullptr;
      ga.H32 = fa.H32;
      ga.HH32 = fa.HH32;
      ga.f_tcol = fa.f_tcol;
      ga.scratch = s->scratch5.as<double>();
      if (const char* dg = getenv("FL_GN5_DIAG")) ga.diag = atoi(dg);   // timing experiments
      {
        const char* gp = getenv("FL_GN5_GPRE");
        ga.gpre = (gp && atoi(gp) == 0) ? 0 : 1;
        const char* pd = getenv("FL_GN5_PD");
        ga.pd = pd ? atoi(pd) : G5_PD;
      }
      const size_t smem5 = g5.total + 1024;
      FL_CUDA(raise_smem_limit(k_gnmf_t5<true>, (int)smem5));
      FL_CUDA(raise_smem_limit(k_gnmf_t5<false>, (int)smem5));
    }
  }
  const size_t WP = (size_t)MR * 16 * (SC + R);
  if ((rc = s->wpart.alloc((size_t)s->nblk_fact * GN_WARPS * WP * 8))) return rc;
  const int SCP = s->SC;   // partial stride: 8 KC (mma.sync pass) or 32 (tcgen05 pass)
  if ((rc = s->part_fact.alloc((size_t)s->nblk_fact * (R * SCP + R * R) * 8))) return rc;
  fa.wpart = s->wpart.as<double>();
  fa.part = s->part_fact.as<double>();
  s->ta.part = fa.part;
  s->g5a.part = fa.part;

  // ---- dimension kernels
  GnDimArgs& da = s->da;
  da.ng = ng;
  da.R = R;
  da.c_T = c_T;
  da.H32 = s->H32.as<float>();
  int max_cols = 1;
  int64_t max_rows = 1;
  size_t part_total = 0;
  s->grid_p = 1;
  int p_u = 1, p_sl = 1;
  for (int d = 0; d < ng; d++) {
    if (t->g[d].cols * (R / 8) > 256) p_u = 2;
    p_sl = std::max(p_sl, (int)ceil_div(32 * (t->g[d].pitch / 4), 256));
  }
  s->fn_p = gn_dim_p_ptr(R, p_u, p_sl);
  int occ_p = 2;
  FL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_p, s->fn_p, 256, 0));
  occ_p = std::max(1, std::min(occ_p, 4));
  for (int d = 0; d < ng; d++) {
    const GatherSrc& g = t->g[d];
    da.S[d] = g.S->as<float>();
    da.pitch[d] = g.pitch;
    da.cols[d] = g.cols;
    da.rows[d] = g.rows;
    da.tcol[d] = g.d_tcol->as<int32_t>();
    da.Gd[d] = const_cast<float*>(fa.Gd[d]);
    da.Z[d] = fa.Z[d];
    // row ranges of >= 4 tiles, one wave of resident CTAs: the next tile is
    // prefetched in registers, and few partials keep the final reduction short
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(g.rows, 128),
                                                               (int64_t)t->sm_count * occ_p));
    da.nblk[d] = nb;
    s->grid_p = std::max(s->grid_p, nb);
    max_cols = std::max(max_cols, g.cols);
    max_rows = std::max(max_rows, g.rows);
    part_total += (size_t)nb * R * g.cols;
  }
  if ((rc = s->part_dim.alloc(part_total * 8 + 16))) return rc;
  {
    size_t po = 0;
    for (int d = 0; d < ng; d++) {
      da.part[d] = s->part_dim.as<double>() + po;
      po += (size_t)da.nblk[d] * R * t->g[d].cols;
    }
  }
  int max_pitch = 4;
  for (auto& g : t->g) max_pitch = std::max(max_pitch, g.pitch);
  s->smem_g = (size_t)max_pitch * R * 4;
  {
    const void* fg0 = R == 8 ? (const void*)k_gnmf_dim_g<8> : R == 16 ? (const void*)k_gnmf_dim_g<16>
                                                                     : (const void*)k_gnmf_dim_g<32>;
    FL_CUDA(raise_smem_limit(fg0, (int)std::max<size_t>(s->smem_g, 16)));
    int occ_g = 2;
    FL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_g, fg0, 256, s->smem_g));
    occ_g = std::max(1, std::min(occ_g, 8));
    // one wave of resident CTAs, thread per row (grid-stride)
    s->grid_g = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(max_rows, 256),
                                                            (int64_t)t->sm_count * occ_g));
  }
  s->smem_p = 0;   // static tiles
  for (auto& g : t->g)
    if (g.cols > 256 || g.cols * R / 8 > 512 || 32 * (g.pitch / 4) > GN_P_SL * 256) {
      set_error("fused GNMF: dimension source with %d columns is too wide", g.cols);
      return FL_ERR_OP;
    }
  if (s->smem_p > 200 * 1024) {
    set_error("fused GNMF: dimension source too wide");
    return FL_ERR_OP;
  }
  {
    const void* fg = R == 8 ? (const void*)k_gnmf_dim_g<8> : R == 16 ? (const void*)k_gnmf_dim_g<16>
                                                                    : (const void*)k_gnmf_dim_g<32>;
    FL_CUDA(raise_smem_limit(fg, (int)std::max<size_t>(s->smem_g, 16)));
  }
  {
    std::vector<RedDesc> dv;
    const int fst = R * SCP + R * R;
    const double* pfb = s->part_fact.as<double>();
    for (int j = 0; j < R; j++) {
      for (int c = 0; c < t->pf; c++)
        if (t->f_tcol[c] >= 0) dv.push_back(RedDesc{pfb + j * SCP + c, fst, s->nblk_fact, j * c_T + t->f_tcol[c], 0});
      for (int q = 0; q < R; q++) {
        // the fact pass skips G tiles strictly below the diagonal (rank rows
        // 16..31 x columns 0..15 when R = 32): read the transposed entry
        const bool lower = R == 32 && j >= 16 && q < 16;
        const int src = lower ? q * R + j : j * R + q;
        dv.push_back(RedDesc{pfb + R * SCP + src, fst, s->nblk_fact, R * c_T + j * R + q, 0});
      }
    }
    for (int d = 0; d < ng; d++) {
      const int cols = t->g[d].cols;
      for (int j = 0; j < R; j++)
        for (int c = 0; c < cols; c++)
          dv.push_back(RedDesc{da.part[d] + j * cols + c, R * cols, da.nblk[d], j * c_T + t->g[d].tcol[c], 0});
    }
    s->n_desc = (int)dv.size();
    if ((rc = s->descs.alloc(dv.size() * sizeof(RedDesc)))) return rc;
    FL_CUDA(cudaMemcpy(s->descs.p, dv.data(), dv.size() * sizeof(RedDesc), cudaMemcpyHostToDevice));
    s->grid_red = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(s->n_desc, 8), 4 * t->sm_count));
  }
  GnHArgs& ha = s->ha;
  ha.c_T = c_T;
  ha.R = R;
  ha.rank = rank;
  ha.H = s->H.as<double>();
  ha.H32 = s->H32.as<float>();
  ha.HH32 = s->HH32.as<float>();
  ha.red = s->red.as<double>();
  ha.t_sq = t_sq;
  ha.loss_hist = s->loss_hist.as<double>();
  ha.loss_cap = s->loss_cap;
  ha.state = s->state.as<GnState>();
  s->smem_h = ((size_t)R * c_T + (size_t)R * R) * 8;
  s->stage_h = 2 * s->smem_h <= 200 * 1024;
  if (s->stage_h) s->smem_h *= 2;
  if (s->smem_h > 200 * 1024) {
    set_error("fused GNMF: rank x columns too large for the H update");
    return FL_ERR_OP;
  }
  FL_CUDA(raise_smem_limit(k_gnmf_h, (int)s->smem_h));
  FL_CUDA(cudaStreamSynchronize(st));
  *out = guard.release();
  return FL_OK;
}

// The fused pass when it applies (rank <= 32, streamed pitch <= 60, <= 8
// gathered sources, dimension widths within its tiles); every other shape --
// or FL_GN_GENERIC=1 -- runs the width-general session of generic.cu.
int fl_gnmf_create(fl_table* t, int32_t rank, const double* w0, const double* h0, double t_sq,
                   fl_gnmf** out, void* stream) {
  const char* fg = getenv("FL_GN_GENERIC");
  const bool force = fg && atoi(fg) != 0;
  if (!force) {
    const int rc = gn_create_fused(t, rank, w0, h0, t_sq, out, stream);
    if (rc != FL_ERR_OP) return rc;
  }
  if (!t || !t->finalized || !w0 || !h0 || !out) {
    set_error("fl_gnmf_create: bad arguments");
    return FL_ERR_ARG;
  }
  if (rank < 1 || rank > std::min<int64_t>(t->r_T, t->c_T)) {
    set_error("rank = %d exceeds min(shape) = %lld", rank,
              (long long)std::min<int64_t>(t->r_T, t->c_T));
    return FL_ERR_CONFIG;
  }
  FL_CUDA(cudaSetDevice(t->device));
  auto* s = new fl_gnmf();
  std::unique_ptr<fl_gnmf> guard(s);
  s->t = t;
  s->rank = rank;
  s->R = rank;
  const int rc = gng_create(t, rank, w0, h0, t_sq, (cudaStream_t)stream, &s->gen);
  if (rc) return rc;
  *out = guard.release();
  return FL_OK;
}

int fl_gnmf_set_comm(fl_gnmf* s, fl_comm* c) {
  if (!s) return FL_ERR_ARG;
  if (s->comm != c && s->graph) {
    cudaGraphExecDestroy(s->graph);
    s->graph = nullptr;
  }
  s->comm = c;
  if (s->gen) gng_set_comm(s->gen, c);
  return FL_OK;
}

int fl_gnmf_path(fl_gnmf* s, int32_t* path) {
  if (!s || !path) return FL_ERR_ARG;
  *path = s->gen ? 2 : s->tc ? 1 : s->t5 ? 3 : 0;
  return FL_OK;
}

int fl_gnmf_run(fl_gnmf* s, int32_t iterations, void* stream) {
  if (!s || iterations < 1) {
    set_error("iterations must be >= 1");
    return FL_ERR_CONFIG;
  }
  FL_CUDA(cudaSetDevice(s->t->device));
  if (s->gen) return gng_run(s->gen, iterations, (cudaStream_t)stream);
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  if (!s->primed) {   // P_0 = W_0^T T, G_0 = W_0^T W_0
    if ((rc = gn_h(s, st, false, false))) return rc;   // fp32 copy of H_0
    if ((rc = gn_products_x(s, st, false))) return rc;
    s->primed = true;
  }
  if (!s->graph) {
    if (!s->cap_stream) FL_CUDA(cudaStreamCreateWithFlags(&s->cap_stream, cudaStreamNonBlocking));
    cudaGraph_t g;
    FL_CUDA(cudaStreamBeginCapture(s->cap_stream, cudaStreamCaptureModeThreadLocal));
    // loss of the previous iteration is recorded by U when it > 0
    rc = gn_h(s, s->cap_stream, true, true);
    if (!rc) rc = gn_products_x(s, s->cap_stream, true);
    cudaError_t e = cudaStreamEndCapture(s->cap_stream, &g);
    if (rc) return rc;
    FL_CUDA(e);
    FL_CUDA(cudaGraphInstantiate(&s->graph, g, 0));
    FL_CUDA(cudaGraphDestroy(g));
  }
  GnState h{};
  FL_CUDA(cudaMemcpyAsync(&h, s->state.p, sizeof(h), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  for (int i = 0; i < iterations; i++) {
    if (h.it + i == 0) {
      // first iteration: no previous loss
      if ((rc = gn_h(s, st, true, false))) return rc;
      if ((rc = gn_products_x(s, st, true))) return rc;
    } else {
      FL_CUDA(cudaGraphLaunch(s->graph, st));
    }
  }
  return FL_OK;
}

int fl_gnmf_kernel_times(fl_gnmf* s, int32_t iters, float* ms_out, void* stream) {
  if (!s || iters < 1 || !ms_out || (!s->primed && !s->gen)) {
    set_error("fl_gnmf_kernel_times: run at least one iteration first");
    return FL_ERR_ARG;
  }
  FL_CUDA(cudaSetDevice(s->t->device));
  cudaStream_t st = (cudaStream_t)stream;
  if (s->gen) {   // one slot: the whole width-general iteration
    cudaEvent_t e0, e1;
    FL_CUDA(cudaEventCreate(&e0));
    FL_CUDA(cudaEventCreate(&e1));
    FL_CUDA(cudaEventRecord(e0, st));
    const int rc = gng_run(s->gen, iters, st);
    if (rc) return rc;
    FL_CUDA(cudaEventRecord(e1, st));
    FL_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    FL_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    for (int j = 0; j < 5; j++) ms_out[j] = 0.f;
    ms_out[2] = ms / iters;
    return FL_OK;
  }
  cudaEvent_t ev[6];
  for (auto& e : ev) FL_CUDA(cudaEventCreate(&e));
  float acc[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
  for (int i = 0; i < iters; i++) {
    FL_CUDA(cudaEventRecord(ev[0], st));
    int rc = gn_h(s, st, true, true);
    if (rc) return rc;
    FL_CUDA(cudaEventRecord(ev[1], st));
    if (s->da.ng > 0) {
      gn_dim_g_launch(s->R, dim3(s->grid_g, s->da.ng), s->smem_g, st, s->da);
      FL_CHECK_LAUNCH();
    }
    FL_CUDA(cudaEventRecord(ev[2], st));
    gn_fact_any(s, true, st);
    FL_CHECK_LAUNCH();
    FL_CUDA(cudaEventRecord(ev[3], st));
    if (s->da.ng > 0) {
      FL_CUDA(gn_dim_p_launch(s->fn_p, dim3(s->grid_p, s->da.ng), s->smem_p, st, s->da));
      FL_CHECK_LAUNCH();
    }
    FL_CUDA(cudaEventRecord(ev[4], st));
    k_gnmf_reduce<<<s->grid_red, 256, 0, st>>>(s->descs.as<RedDesc>(), s->n_desc,
                                               s->red.as<double>());
    FL_CHECK_LAUNCH();
    FL_CUDA(cudaEventRecord(ev[5], st));
    FL_CUDA(cudaEventSynchronize(ev[5]));
    for (int j = 0; j < 5; j++) {
      float ms = 0.f;
      FL_CUDA(cudaEventElapsedTime(&ms, ev[j], ev[j + 1]));
      acc[j] += ms;
    }
  }
  for (int j = 0; j < 5; j++) ms_out[j] = acc[j] / iters;
  for (auto& e : ev) cudaEventDestroy(e);
  return FL_OK;
}

int fl_gnmf_partial(fl_gnmf* s, void* stream) {
  if (!s) return FL_ERR_ARG;
  FL_CUDA(cudaSetDevice(s->t->device));
  cudaStream_t st = (cudaStream_t)stream;
  if (s->gen) return gng_partial(s->gen, st);
  int rc;
  if (!s->primed) {   // products of W_0 only
    if ((rc = gn_h(s, st, false, false))) return rc;
    s->primed = true;
    return gn_products(s, st, false);
  }
  GnState h{};
  FL_CUDA(cudaMemcpyAsync(&h, s->state.p, sizeof(h), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  if ((rc = gn_h(s, st, true, h.it > 0))) return rc;
  return gn_products(s, st, true);
}

int fl_gnmf_reduce_buffer(fl_gnmf* s, double** buf, int32_t* len) {
  if (!s || !buf || !len) return FL_ERR_ARG;
  if (s->gen) {
    int n = 0;
    *buf = gng_red(s->gen, &n);
    *len = n;
    return FL_OK;
  }
  *buf = s->red.as<double>();
  *len = s->R * s->t->c_T + s->R * s->R;
  return FL_OK;
}

int fl_gnmf_result(fl_gnmf* s, double* w, double* h, double* loss, int32_t n, int32_t* n_done,
                   void* stream) {
  if (!s) return FL_ERR_ARG;
  FL_CUDA(cudaSetDevice(s->t->device));
  cudaStream_t st = (cudaStream_t)stream;
  if (s->gen) {
    int nd = 0;
    const int rc = gng_result(s->gen, w, h, loss, n, &nd, st);
    if (n_done) *n_done = nd;
    return rc;
  }
  GnState hs{};
  FL_CUDA(cudaMemcpyAsync(&hs, s->state.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  // the last iteration's loss (from the products of the final W) is recorded
  // on demand, once per iteration count
  if (hs.it > 0 && hs.nloss < hs.it) {
    int rc = gn_h(s, st, false, true);
    if (rc) return rc;
    FL_CUDA(cudaMemcpyAsync(&hs, s->state.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
    FL_CUDA(cudaStreamSynchronize(st));
  }
  const fl_table* t = s->t;
  if (w) {
    double* tmp = nullptr;
    FL_CUDA(cudaMallocAsync((void**)&tmp, (size_t)t->r_T * s->rank * 8 + 16, st));
    k_gnmf_w_out<<<(unsigned)ceil_div(t->r_T * s->rank, 256), 256, 0, st>>>(
        s->W.as<float>(), t->perm->as<int32_t>(), t->r_T, s->rank, s->R, tmp);
    FL_CHECK_LAUNCH();
    int rc = d2h_copy(w, tmp, (size_t)t->r_T * s->rank * 8, st);
    if (rc) return rc;
    FL_CUDA(cudaFreeAsync(tmp, st));
  }
  if (h) FL_CUDA(cudaMemcpyAsync(h, s->H.p, (size_t)s->rank * t->c_T * 8, cudaMemcpyDefault, st));
  FL_CUDA(cudaStreamSynchronize(st));
  const int nd = std::min(hs.nloss, s->loss_cap);
  if (n_done) *n_done = nd;
  if (loss && n > 0) {
    const int m = std::min(n, nd);
    if (m > 0) FL_CUDA(cudaMemcpy(loss, s->loss_hist.p, (size_t)m * 8, cudaMemcpyDefault));
  }
  return FL_OK;
}

int fl_gnmf_destroy(fl_gnmf* s) {
  if (!s) return FL_OK;
  cudaSetDevice(s->t->device);
  if (s->graph) cudaGraphExecDestroy(s->graph);
  if (s->cap_stream) cudaStreamDestroy(s->cap_stream);
  if (s->gen) gng_destroy(s->gen);
  delete s;
  return FL_OK;
}

}  // extern "C"
