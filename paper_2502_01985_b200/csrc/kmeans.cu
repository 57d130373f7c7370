// Fused Lloyd K-means over a factorized table (reference trainers.py:198-246,
// built on ops.py:219-271).
//
// The reference computes D = rowSum(T^2) 1^T - 2 T C^T + 1 ||c||^2^T with a
// full lmm, takes a row argmin (ties -> lowest index) and re-estimates
// C <- (A^T T) / (A^T 1) with a transpose_lmm of the one-hot matrix A.  Here
// one iteration is three kernels (plus the all-reduce of `red` between K3 and
// the update when fact rows are sharded across GPUs):
//
//  K1 k_km_dim_e   E_d[r, j] = ||S_d[r,:] - C_j[cols of d]||^2 for every
//                  dimension row (row r_d = the all-zero "no match" row),
//                  direct differences in fp32; zero the I_d^T A counters.
//  K2 k_km_fact    one pass over the fact rows (per-warp TMA pipelines):
//                    z    = F[p,:] C_F^T          (3xTF32 mma.sync)
//                    dist = ||c_F||^2 - 2 z + sum_d E_d[fk_d[p], :]
//                    a    = argmin_j dist (ties -> lowest j)
//                    loss += ||F[p,:] - C_F[a]||^2 + sum_d E_d[fk_d[p], a]
//                    sums_F[a,:] += F[p,:], count[a] += 1   (3xTF32 mma:
//                                    one-hot^T x [F | 1])
//                    cnt_d[fk_d[p], a] += 1      (I_d^T A: integer atomics,
//                                    warp-aggregated -- exact, order-free)
//  K3 k_km_dim_sums  sums_d = cnt_d^T S_d (fp64 per-CTA partials), then the
//                  last CTA reduces every partial in a fixed order into `red`
//                  and (single GPU) applies C <- sums / counts (empty clusters
//                  keep their centroid).
//
// Why the row term ||F||^2 never appears: it is constant per row (argmin) and
// the loss is taken from direct differences, which avoids the fp32
// cancellation of the expanded form on tight clusters.
#include <algorithm>
#include <cstdlib>

#include "internal.h"
#include "generic.h"
#include "mma_tf32.cuh"
#include "reduce.cuh"
#include "tc05.cuh"

namespace flb {

constexpr int KM_WARPS = 8;
constexpr int KM_FLUSH = 16;   // stages between fp32 -> fp64 flushes (<= 512 rows)
constexpr int KM_PF_MAX = 2;   // gathered sources whose E rows are prefetched by async copies
// per-warp scratch: the prefetched E rows, also the z transpose (32 x (KP+4))
__host__ __device__ constexpr int km_scratch_floats(int KP) {
  return KM_PF_MAX * 32 * KP > 32 * (KP + 4) ? KM_PF_MAX * 32 * KP : 32 * (KP + 4);
}
#define kInf __int_as_float(0x7f800000)

struct KmState {
  int it;
  int done_dim;
  int pad[2];
};

struct KmFactArgs {
  const float* F;
  int pf, c_T, k;
  int64_t r_T, nunits;           // units of 32 device rows
  int ng, sort_g;
  const int32_t* fk[MAX_GATHER];
  const float* E[MAX_GATHER];    // (r_d + 1) x KP
  int32_t* cnt[MAX_GATHER];      // r_d x KP
  int64_t rows[MAX_GATHER];
  const float* C32;              // k x c_T
  const int32_t* f_tcol;         // pf
  int32_t* assign;               // r_pad device order, or null
  double* part;                  // gridDim.x x (KP * SC + 1)
  double* part_w;                // gridDim.x x KM_WARPS x (MT * 16 * SC): per-warp sums
  uint32_t stage_bytes;          // 32 x FP fp32 TMA tile | 32 int32 sort-source FK
  int nst;
  int diag;                      // timing experiments only (FL_KM_DIAG): 1 no sums, 2 no loss
  int npf_max;                   // gathered sources on the async-copy E prefetch (<= KM_PF_MAX)
};

struct KmDimArgs {
  int ng, k, KP, c_T;
  const float* S[MAX_GATHER];
  int pitch[MAX_GATHER];
  int cols[MAX_GATHER];
  int64_t rows[MAX_GATHER];
  int nblk[MAX_GATHER];
  const int32_t* tcol[MAX_GATHER];
  float* E[MAX_GATHER];
  int32_t* cnt[MAX_GATHER];
  double* part[MAX_GATHER];      // nblk x (KP * cols)
  const float* C32;
};

struct KmUpdateArgs {
  int c_T, k, KP, SC, pf, ng;
  const int32_t* f_tcol;
  const int32_t* d_tcol[MAX_GATHER];
  int d_cols[MAX_GATHER];
  const double* part_fact;
  int nblk_fact;
  const double* part_dim[MAX_GATHER];
  int nblk_dim[MAX_GATHER];
  double* red;                   // k*c_T sums | k counts | loss
  double* C64;
  float* C32;
  double* loss_hist;
  int loss_cap;
  KmState* state;
};

// ---------------------------------------------------------------------------
// K1: E_d and counter reset
// ---------------------------------------------------------------------------
// thread per dimension row; the centroid slice sits transposed in smem
// ([column][cluster]) so every row step is one broadcast LDS.128 per 4 clusters
template <int KP>
__global__ void __launch_bounds__(256) k_km_dim_e(KmDimArgs a) {
  const int d = blockIdx.y;
  if (d >= a.ng) return;
  const int k = a.k;
  const int64_t rows = a.rows[d];
  const int cols = a.cols[d], pitch = a.pitch[d];
  extern __shared__ __align__(16) float sm_e[];   // pitch x KP (transposed slice)
  for (int i = threadIdx.x; i < pitch * KP; i += blockDim.x) {
    const int c = i / KP, j = i - c * KP;
    sm_e[i] = (j < k && c < cols) ? a.C32[(int64_t)j * a.c_T + a.tcol[d][c]] : 0.f;
  }
  __syncthreads();
  for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row <= rows;
       row += (int64_t)gridDim.x * blockDim.x) {   // row == rows: the "no match" row
    float acc[KP];
#pragma unroll
    for (int j = 0; j < KP; j++) acc[j] = 0.f;
    const float4* sr = reinterpret_cast<const float4*>(a.S[d] + row * pitch);
    const int n4 = pitch / 4;
    // the row is read in batches of 8 independent float4 loads (one latency
    // per batch instead of one per float4: the kernel was latency-bound)
    for (int c0 = 0; c0 < n4; c0 += 8) {
      float4 vb[8];
#pragma unroll
      for (int u = 0; u < 8; u++)
        vb[u] = (row < rows && c0 + u < n4) ? sr[c0 + u] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 8; u++) {
        if (c0 + u >= n4) break;
        const float vv[4] = {vb[u].x, vb[u].y, vb[u].z, vb[u].w};
#pragma unroll
        for (int e = 0; e < 4; e++) {
          const float4* cr = reinterpret_cast<const float4*>(sm_e + ((c0 + u) * 4 + e) * KP);
#pragma unroll
          for (int q = 0; q < KP / 4; q++) {
            const float4 cc = cr[q];
            const float d0 = vv[e] - cc.x, d1 = vv[e] - cc.y, d2 = vv[e] - cc.z, d3 = vv[e] - cc.w;
            acc[q * 4 + 0] = fmaf(d0, d0, acc[q * 4 + 0]);
            acc[q * 4 + 1] = fmaf(d1, d1, acc[q * 4 + 1]);
            acc[q * 4 + 2] = fmaf(d2, d2, acc[q * 4 + 2]);
            acc[q * 4 + 3] = fmaf(d3, d3, acc[q * 4 + 3]);
          }
        }
      }
    }
    // pitch padding columns hold S = 0 and C = 0: they add nothing; clusters
    // past k are zeroed so the screen never sees garbage
    float4* er = reinterpret_cast<float4*>(a.E[d] + row * KP);
    int4* cr = reinterpret_cast<int4*>(a.cnt[d] + row * KP);
#pragma unroll
    for (int q = 0; q < KP / 4; q++) {
      float4 o;
      o.x = q * 4 + 0 < k ? acc[q * 4 + 0] : 0.f;
      o.y = q * 4 + 1 < k ? acc[q * 4 + 1] : 0.f;
      o.z = q * 4 + 2 < k ? acc[q * 4 + 2] : 0.f;
      o.w = q * 4 + 3 < k ? acc[q * 4 + 3] : 0.f;
      er[q] = o;
      if (row < rows) cr[q] = make_int4(0, 0, 0, 0);
    }
  }
}

// v[i] for a runtime i < N (power of two) from registers: a binary select
// tree on the bits of i (log2 N levels, N - 1 selects) instead of N compare-
// and-selects
template <int N>
__device__ __forceinline__ float select_by_index(const float (&v)[N], int i) {
  float t[N];
#pragma unroll
  for (int j = 0; j < N; j++) t[j] = v[j];
#pragma unroll
  for (int w = N / 2; w >= 1; w >>= 1) {
    const bool hi = (i & w) != 0;
#pragma unroll
    for (int j = 0; j < w; j++) t[j] = hi ? t[j + w] : t[j];
  }
  return t[0];
}

// ---------------------------------------------------------------------------
// K2: the fact-row pass
// ---------------------------------------------------------------------------
template <int NT, int KC>
__global__ void __launch_bounds__(KM_WARPS * 32, (NT <= 2 && KC <= 4) ? 2 : 1)
    k_km_fact(const __grid_constant__ CUtensorMap tmF, KmFactArgs a) {
  constexpr int KP = NT * 8;          // padded cluster count
  constexpr int MT = (NT + 1) / 2;    // 16-cluster tiles of the one-hot operand
  constexpr int SC = KC * 8;          // MMA columns of F (count column = pf < SC)
  constexpr int FP = SC + 4;          // smem F row pitch (TMA box width, zero-filled)
  constexpr int CFP = SC + 4;         // fp32 centroid row pitch in smem
  constexpr int ZP = KP + 4;          // per-warp distance transpose pitch
  // E rows of the first KM_PF gathered sources are prefetched one unit ahead
  // by async copies (LDGSTS) straight into the warp's scratch; their FKs two
  // units ahead into a 2-slot ring.  Rows are copied ROW-SPLIT: QR = KP/4
  // consecutive lanes fetch the QR float4 quads of one row (one L1 tag per
  // row, not per lane); quad q of row r lands at physical quad q ^ sw(r), so
  // the lane-per-row read-back is bank-conflict free.
  constexpr int KM_PF = KM_PF_MAX;
  constexpr int QR = KP / 4, RPI = 32 / QR;
  constexpr int EW = km_scratch_floats(KP);
  // fp64 sums accumulators in registers when they fit, else per-warp global
  constexpr bool ACC_REG = MT * KC <= 4;
  extern __shared__ __align__(128) char smem[];
  __shared__ uint64_t bar[KM_WARPS][4];
  __shared__ double lsum[KM_WARPS];

  uint4* bfrag = reinterpret_cast<uint4*>(smem);                       // KC*NT*32
  float* cf = reinterpret_cast<float*>(bfrag + KC * NT * 32);          // KP x CFP
  float* cn = cf + KP * CFP;                                           // KP (+4)
  float* ebuf_all = cn + KP + 4;                                       // warps x EW
  int32_t* fkr_all = reinterpret_cast<int32_t*>(ebuf_all + KM_WARPS * EW);  // warps x 3 x KM_PF x 32
  char* stages = smem + round_up((int64_t)(reinterpret_cast<char*>(fkr_all + KM_WARPS * 3 * KM_PF * 32) -
                                           smem), 128);

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int pf = a.pf, k = a.k, pf4 = a.pf / 4;

  // centroid fact slice (zero past pf and past k), tf32 B fragments, norms
  for (int i = threadIdx.x; i < KP * CFP; i += blockDim.x) {
    int j = i / CFP, c = i - j * CFP;
    float v = 0.f;
    if (j < k && c < pf) {
      int tc = a.f_tcol[c];
      if (tc >= 0) v = a.C32[(int64_t)j * a.c_T + tc];
    }
    cf[i] = v;
  }
  // this warp's fp64 sums region (global, L2-resident)
  double* wacc = a.part_w + ((int64_t)blockIdx.x * KM_WARPS + warp) * (MT * 16 * SC);
  if (!ACC_REG)
    for (int i = lane; i < MT * 16 * SC; i += 32) wacc[i] = 0.0;
  if (lane == 0) {
    lsum[warp] = 0.0;
    for (int s = 0; s < a.nst; s++) mbar_init(&bar[warp][s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  for (int i = threadIdx.x; i < KC * NT * 32; i += blockDim.x) {
    int l = i & 31, kn = i >> 5;
    int kc = kn / NT, n = kn - kc * NT;
    int gg = l >> 2, tt = l & 3;
    // screen B fragments: one rounded tf32 term, packed (conflict-free LDS.64)
    reinterpret_cast<uint2*>(bfrag)[i] = make_uint2(tf32_bits(cf[(n * 8 + gg) * CFP + kc * 8 + tt]),
                                                    tf32_bits(cf[(n * 8 + gg) * CFP + kc * 8 + tt + 4]));
  }
  for (int j = threadIdx.x; j < KP; j += blockDim.x) {
    float s = 0.f;
    for (int c = 0; c < SC; c++) s = fmaf(cf[j * CFP + c], cf[j * CFP + c], s);
    cn[j] = j < k ? s : kInf;
  }
  __syncthreads();
  float cn_max = 0.f;
  for (int j = 0; j < k; j++) cn_max = fmaxf(cn_max, cn[j]);

  // this warp's contiguous range of 32-row units
  const int64_t gw = (int64_t)blockIdx.x * KM_WARPS + warp;
  const int64_t NW = (int64_t)gridDim.x * KM_WARPS;
  const int64_t base = a.nunits / NW, rem = a.nunits % NW;
  // row indices fit in 32 bits (fl_table_create caps r_T below INT32_MAX):
  // 32-bit unit / row arithmetic in the unit loop
  const int u0 = (int)(gw * base + min64(gw, rem));
  const int cnt = (int)(base + (gw < rem ? 1 : 0));
  const int r_T32 = (int)a.r_T;
  constexpr uint32_t F_BYTES = 32u * FP * 4u;
  // F tile + the 32 FKs of every source not in the async-copied FK ring
  const int npf = min(a.ng, a.npf_max);
  const uint32_t tx = F_BYTES + 128u * (a.ng - npf);
  char* wsm = stages + (size_t)warp * a.nst * a.stage_bytes;
  float* ebuf = ebuf_all + warp * EW;   // [KM_PF][32][KP] E rows; also the z transpose scratch
  float* zs = ebuf;
  int32_t* fkr = fkr_all + warp * 3 * KM_PF * 32;
  uint64_t* wbar = bar[warp];
  // F streams through once per pass: evict_first keeps the E_d rows and the
  // I_d^T A counters L2-resident
  const uint64_t pol_stream = l2_policy_evict_first();
  auto issue = [&](int s, int unit) {
    char* st = wsm + (size_t)s * a.stage_bytes;
    mbar_arrive_expect_tx(&wbar[s], tx);
    tma_load_2d_hint(st, &tmF, 0, (int)(unit * 32), &wbar[s], pol_stream);
#pragma unroll
    for (int d = 0; d < MAX_GATHER; d++)   // FKs of the sources without an FK ring
      if (d >= npf && d < a.ng) bulk_g2s(st + F_BYTES + 128 * d, a.fk[d] + unit * 32, 128, &wbar[s]);
  };
  if (lane == 0)
    for (int s = 0; s < a.nst && s < cnt; s++) issue(s, u0 + s);

  // the prefetched sources' loops are unrolled: compile-time source indices
  // turn a.fk[d] / a.E[d] / a.rows[d] into constant-bank operands instead
  // of indexed parameter loads per unit
  auto issue_fk = [&](int unit, int slot) {
#pragma unroll
    for (int d = 0; d < KM_PF; d++)
      if (d < npf) cp_async4(fkr + (slot * KM_PF + d) * 32 + lane, a.fk[d] + unit * 32 + lane);
  };
  auto issue_e = [&](int slot) {
#pragma unroll
    for (int d = 0; d < KM_PF; d++) {
      if (d >= npf) break;
      const int32_t* fr = fkr + (slot * KM_PF + d) * 32;
#pragma unroll
      for (int jj = 0; jj < QR; jj++) {
        const int r = jj * RPI + lane / QR, q = lane % QR;
        // FK -1 (no match) -> the all-zero row r_d: one unsigned min
        const unsigned f = min((unsigned)fr[r], (unsigned)a.rows[d]);
        cp_async16(ebuf + d * 32 * KP + r * KP + 4 * (q ^ ((r / (8 / QR)) & (QR - 1))),
                   a.E[d] + (f * KP + q * 4));
      }
    }
  };
  if (cnt > 0 && npf > 0) {
    issue_fk(u0, 0);
    if (cnt > 1) issue_fk(u0 + 1, 1);   // FK ring: unit u0 + j in slot j % 3
    cp_async_commit();
    cp_async_wait_all();
    __syncwarp();
    issue_e(0);
    cp_async_commit();
  }

  float sacc[MT][KC][4];
  double sacc64[ACC_REG ? MT : 1][ACC_REG ? KC : 1][4];
#pragma unroll
  for (int m = 0; m < MT; m++)
#pragma unroll
    for (int c = 0; c < KC; c++)
#pragma unroll
      for (int e = 0; e < 4; e++) {
        sacc[m][c][e] = 0.f;
        if (ACC_REG) sacc64[ACC_REG ? m : 0][ACC_REG ? c : 0][e] = 0.0;
      }
  float lacc = 0.f;

  auto flush = [&]() {
#pragma unroll
    for (int m = 0; m < MT; m++)
#pragma unroll
      for (int c = 0; c < KC; c++)
#pragma unroll
        for (int e = 0; e < 4; e++) {
          if (ACC_REG) {
            sacc64[ACC_REG ? m : 0][ACC_REG ? c : 0][e] += (double)sacc[m][c][e];
          } else {
            const int row = m * 16 + g + (e >> 1) * 8, col = c * 8 + 2 * t + (e & 1);
            wacc[row * SC + col] += (double)sacc[m][c][e];
          }
          sacc[m][c][e] = 0.f;
        }
    float v = lacc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) lsum[warp] += (double)v;
    lacc = 0.f;
  };

  int s = 0;            // stage slot and its mbarrier phase
  uint32_t ph = 0;
  int fslot = 0;        // FK ring slot of this unit
  for (int i = 0; i < cnt; i++, s = (s + 1 == a.nst) ? 0 : s + 1, ph ^= (s == 0),
               fslot = fslot == 2 ? 0 : fslot + 1) {
    mbar_wait(&wbar[s], ph);
    float* Fs = reinterpret_cast<float*>(wsm + (size_t)s * a.stage_bytes);
    const int32_t* fks_s = reinterpret_cast<const int32_t*>(wsm + (size_t)s * a.stage_bytes + F_BYTES);
    // the count column of [F | 1] (column pf, zero-filled by the TMA): one
    // store per row here instead of a select per B element in the sums
    Fs[lane * FP + pf] = 1.f;
    __syncwarp();
    const int p0 = (u0 + i) * 32;
    const bool valid = p0 + lane < r_T32;
    // E terms of every cluster: sum_d E_d[fk_d, j] (kept apart for the loss).
    // The first KM_PF sources were gathered into registers during the
    // previous unit; any further source is gathered here, before the screen
    float eacc[KP];
#pragma unroll
    for (int j = 0; j < KP; j++) eacc[j] = 0.f;
    if (npf > 0) {
      cp_async_wait_all();   // this unit's E rows (and the next unit's FKs)
      __syncwarp();
#pragma unroll
      for (int d = 0; d < KM_PF; d++) {
        if (d >= npf) break;
#pragma unroll
        for (int q = 0; q < QR; q++) {
          const float4 v = *reinterpret_cast<const float4*>(
              ebuf + d * 32 * KP + lane * KP + 4 * (q ^ ((lane / (8 / QR)) & (QR - 1))));
          eacc[q * 4 + 0] += v.x;
          eacc[q * 4 + 1] += v.y;
          eacc[q * 4 + 2] += v.z;
          eacc[q * 4 + 3] += v.w;
        }
      }
      __syncwarp();   // the scratch is reused for the distance transpose
    }
#pragma unroll
    for (int d = 0; d < MAX_GATHER; d++) {
      if (d >= a.ng) break;
      if (d < npf) continue;
      const int f = fks_s[d * 32 + lane];
      const float4* er = reinterpret_cast<const float4*>(a.E[d] + (f >= 0 ? (int64_t)f : a.rows[d]) * KP);
#pragma unroll
      for (int q = 0; q < KP / 4; q++) {
        const float4 ev = er[q];
        eacc[q * 4 + 0] += ev.x;
        eacc[q * 4 + 1] += ev.y;
        eacc[q * 4 + 2] += ev.z;
        eacc[q * 4 + 3] += ev.w;
      }
    }

    // ---- screen: z = F C_F^T on the tensor cores, ONE tf32 term (A
    // truncated, B rounded): the screen only proposes the winner, every row
    // whose runner-up lies inside the tf32 error bound is certified below
    float z[2][NT][4];
#pragma unroll
    for (int m = 0; m < 2; m++)
#pragma unroll
      for (int n = 0; n < NT; n++)
#pragma unroll
        for (int e = 0; e < 4; e++) z[m][n][e] = 0.f;
#pragma unroll
    for (int kc = 0; kc < KC; kc++) {
      uint2 bf[NT];
#pragma unroll
      for (int n = 0; n < NT; n++) bf[n] = reinterpret_cast<const uint2*>(bfrag)[(kc * NT + n) * 32 + lane];
#pragma unroll
      for (int m = 0; m < 2; m++) {
        // A as loaded: the tensor core truncates fp32 operand bits below the
        // tf32 mantissa (measured, profiles/r02_tc_probe.txt), which is the
        // truncated-A error the certification bound assumes
        uint32_t x[4];
        ldsm_x4(x[0], x[1], x[2], x[3], Fs + (m * 16 + (lane & 15)) * FP + kc * 8 + (lane >> 4) * 4);
#pragma unroll
        for (int n = 0; n < NT; n++) mma_tf32(z[m][n], x[0], x[1], x[2], x[3], bf[n].x, bf[n].y);
      }
    }
    // transpose to lane-per-row through the warp's smem scratch
#pragma unroll
    for (int m = 0; m < 2; m++)
#pragma unroll
      for (int n = 0; n < NT; n++) {
        *reinterpret_cast<float2*>(zs + (m * 16 + g) * ZP + n * 8 + 2 * t) =
            make_float2(z[m][n][0], z[m][n][1]);
        *reinterpret_cast<float2*>(zs + (m * 16 + g + 8) * ZP + n * 8 + 2 * t) =
            make_float2(z[m][n][2], z[m][n][3]);
      }
    __syncwarp();
    float dv[KP];
#pragma unroll
    for (int q = 0; q < KP / 4; q++) {
      const float4 zz = *reinterpret_cast<const float4*>(zs + lane * ZP + q * 4);
      dv[q * 4 + 0] = fmaf(-2.f, zz.x, cn[q * 4 + 0]) + eacc[q * 4 + 0];
      dv[q * 4 + 1] = fmaf(-2.f, zz.y, cn[q * 4 + 1]) + eacc[q * 4 + 1];
      dv[q * 4 + 2] = fmaf(-2.f, zz.z, cn[q * 4 + 2]) + eacc[q * 4 + 2];
      dv[q * 4 + 3] = fmaf(-2.f, zz.w, cn[q * 4 + 3]) + eacc[q * 4 + 3];
    }
    // best / runner-up (ties -> lowest index)
    float v1 = dv[0], v2 = kInf;
    int al = 0;
#pragma unroll
    for (int j = 1; j < KP; j++) {
      const bool lt = dv[j] < v1;
      v2 = lt ? v1 : fminf(v2, dv[j]);
      al = lt ? j : al;
      v1 = lt ? dv[j] : v1;
    }
    // F row in registers
    const float4* fr = reinterpret_cast<const float4*>(Fs + lane * FP);
    float4 xr[2 * KC];
#pragma unroll
    for (int c4 = 0; c4 < 2 * KC; c4++) xr[c4] = c4 < pf4 ? fr[c4] : make_float4(0.f, 0.f, 0.f, 0.f);
    // ---- certify: keep the screened winner unless the runner-up lies within
    // the tf32 screen's error bound; near-ties are re-decided from direct
    // fp32 differences (the reference orders them in fp64)
    float el = 0.f;
    if (valid) {
      float xn = 0.f;
#pragma unroll
      for (int c4 = 0; c4 < 2 * KC; c4++)
        xn = fmaf(xr[c4].x, xr[c4].x, fmaf(xr[c4].y, xr[c4].y,
             fmaf(xr[c4].z, xr[c4].z, fmaf(xr[c4].w, xr[c4].w, xn))));
      // v2 is +inf when k == 1: keep the bound finite
      // |screen error| per distance <= 2 sum_c |x_c (c_c - c~_c) + (x_c - x~_c) c~_c|
      // <= 1.6e-3 (xn + cn_j) for a truncated A (2^-10) and a rounded B
      // (2^-11); two distances differ by at most twice that
      const float tol = 4e-3f * (xn + cn_max) + 1e-5f * (fabsf(v1) + fminf(fabsf(v2), 3e38f));
      if (!(v2 - v1 > tol)) {
        uint32_t cand = 0;   // clusters that can still win
#pragma unroll
        for (int j = 0; j < KP; j++)
          if (j < k && dv[j] - v1 <= tol) cand |= 1u << j;
        float bd = kInf;
        int bj = 0;
        while (cand) {
          const int j = __ffs(cand) - 1;
          cand &= cand - 1;
          const float4* cr = reinterpret_cast<const float4*>(cf + j * CFP);
          float dj = 0.f;
#pragma unroll
          for (int c4 = 0; c4 < 2 * KC; c4++) {
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
#pragma unroll
      el = select_by_index<KP>(eacc, al);
    } else {
      al = -1;
    }
    // ---- prefetch the next unit's E rows (its FKs arrived a unit ago) and
    // the FKs of the unit after it: their L2 latency overlaps the rest of
    // this unit (loss, counters, sums)
    if (npf > 0 && i + 1 < cnt) {
      __syncwarp();   // every lane is done with the z scratch
      issue_e(fslot == 2 ? 0 : fslot + 1);
      if (i + 2 < cnt) issue_fk(u0 + i + 2, fslot == 0 ? 2 : fslot - 1);
      cp_async_commit();
    }
    // ---- loss (direct differences), I_d^T A counters, assignments
    if (valid && !(a.diag & 2)) {
      const float4* cr = reinterpret_cast<const float4*>(cf + al * CFP);
      float l = el;
#pragma unroll
      for (int c4 = 0; c4 < 2 * KC; c4++) {
        const float4 c = cr[c4];
        const float d0 = xr[c4].x - c.x, d1 = xr[c4].y - c.y;
        const float d2 = xr[c4].z - c.z, d3 = xr[c4].w - c.w;
        l = fmaf(d0, d0, fmaf(d1, d1, fmaf(d2, d2, fmaf(d3, d3, l))));
      }
      lacc += l;
    }
#pragma unroll
    for (int d = 0; d < MAX_GATHER; d++) {
      if (d >= a.ng) break;
      const int f = d < npf ? fkr[(fslot * KM_PF + d) * 32 + lane] : fks_s[d * 32 + lane];
      const int key = (valid && f >= 0) ? f * KP + al : -1 - lane;
      if (d == a.sort_g) {   // sorted FKs: runs of equal keys, one atomic per run
        const unsigned mask = __match_any_sync(0xffffffffu, key);
        if (key >= 0 && (__ffs(mask) - 1) == lane) atomicAdd(&a.cnt[d][key], __popc(mask));
      } else if (key >= 0) {
        atomicAdd(&a.cnt[d][key], 1);
      }
    }
    if (a.assign && valid) a.assign[p0 + lane] = al;
    // ---- sums_F | counts = one-hot^T [F | 1]: 2-term tf32 split of F (hi =
    // truncated mantissa, lo = exact remainder), one-hot exact
    if (!(a.diag & 1))
#pragma unroll
    for (int kb = 0; kb < 4; kb++) {
      // k index t <-> row kb*8 + 2t, t + 4 <-> row kb*8 + 2t + 1: with the
      // F pitch of 4 * odd words these rows hit distinct bank octets
      const int rr0 = kb * 8 + 2 * t, rr1 = rr0 + 1;
      const int ar0 = __shfl_sync(0xffffffffu, al, rr0);
      const int ar1 = __shfl_sync(0xffffffffu, al, rr1);
      uint32_t oh[MT][4];
#pragma unroll
      for (int m = 0; m < MT; m++) {
        const int j0 = m * 16 + g, j1 = j0 + 8;
        oh[m][0] = ar0 == j0 ? kTf32One : 0u;
        oh[m][1] = ar0 == j1 ? kTf32One : 0u;
        oh[m][2] = ar1 == j0 ? kTf32One : 0u;
        oh[m][3] = ar1 == j1 ? kTf32One : 0u;
      }
#pragma unroll
      for (int c = 0; c < KC; c++) {
        // column pf of [F | 1] is the count column (set to 1 after the TMA)
        const float b0 = Fs[rr0 * FP + c * 8 + g];
        const float b1 = Fs[rr1 * FP + c * 8 + g];
        const uint32_t h0 = __float_as_uint(b0) & 0xffffe000u;
        const uint32_t h1 = __float_as_uint(b1) & 0xffffe000u;
        const uint32_t l0 = __float_as_uint(b0 - __uint_as_float(h0));
        const uint32_t l1 = __float_as_uint(b1 - __uint_as_float(h1));
#pragma unroll
        for (int m = 0; m < MT; m++) {
          mma_tf32(sacc[m][c], oh[m][0], oh[m][1], oh[m][2], oh[m][3], h0, h1);
          mma_tf32(sacc[m][c], oh[m][0], oh[m][1], oh[m][2], oh[m][3], l0, l1);
        }
      }
    }
    __syncwarp();
    if (i + a.nst < cnt && tc::elect_one()) {   // converged warp: no per-instruction ELECT loop
      fence_proxy_async();
      issue(s, u0 + i + a.nst);
    }
    if ((i % KM_FLUSH) == KM_FLUSH - 1) flush();
  }
  flush();
  if (ACC_REG) {
#pragma unroll
    for (int m = 0; m < MT; m++)
#pragma unroll
      for (int c = 0; c < KC; c++)
#pragma unroll
        for (int e = 0; e < 4; e++) {
          const int row = m * 16 + g + (e >> 1) * 8, col = c * 8 + 2 * t + (e & 1);
          wacc[row * SC + col] = sacc64[ACC_REG ? m : 0][ACC_REG ? c : 0][e];
        }
  }
  __syncthreads();
  // CTA partial in fixed warp order: [KP x SC] sums (count at column pf) | loss
  double* out = a.part + (int64_t)blockIdx.x * (KP * SC + 1);
  const double* wall = a.part_w + (int64_t)blockIdx.x * KM_WARPS * (MT * 16 * SC);
  for (int i = threadIdx.x; i < KP * SC; i += blockDim.x) {
    double s = 0.0;
    for (int w2 = 0; w2 < KM_WARPS; w2++) s += wall[w2 * (MT * 16 * SC) + i];
    out[i] = s;
  }
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w2 = 0; w2 < KM_WARPS; w2++) s += lsum[w2];
    out[KP * SC] = s;
  }
}

#include "kmeans_tc.cuh"
#include "kmeans_t5.cuh"

__global__ void k_km_block(const float* __restrict__ F, int pf, int64_t r_pad, int C4P,
                           float* __restrict__ Fb) {
  // stream block -> 128-row tiles of [chunk][row][4]
  const int64_t n = r_pad * C4P * 4;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = idx / (C4P * 4);
    const int c = (int)(idx - p * C4P * 4);
    const int64_t t = p / KT_TILE;
    const int r = (int)(p - t * KT_TILE);
    Fb[((t * C4P + (c >> 2)) * KT_TILE + r) * 4 + (c & 3)] = F[p * pf + c];
  }
}

// ---------------------------------------------------------------------------
// K3: sums_d = cnt_d^T S_d, then fixed-order reduction (+ update)
// ---------------------------------------------------------------------------
__device__ void km_apply_update(const KmUpdateArgs& u) {
  const int tid = threadIdx.x;
  const int it = u.state->it;
  const double* cnt = u.red + (int64_t)u.k * u.c_T;
  if (tid == 0 && it < u.loss_cap) u.loss_hist[it] = u.red[(int64_t)u.k * u.c_T + u.k];
  for (int i = tid; i < u.k * u.c_T; i += blockDim.x) {
    int j = i / u.c_T;
    double n = cnt[j];
    if (n > 0.0) u.C64[i] = u.red[i] / n;
    u.C32[i] = (float)u.C64[i];
  }
  __syncthreads();
  if (tid == 0) u.state->it = it + 1;
}

// sums_d[j, c] = sum_r cnt_d[r, j] S_d[r, c]: 32-row tiles of S and of the
// counters (converted to fp32 once) in smem; thread = (column, 8 clusters);
// fp32 within a tile, fp64 across tiles.  Each thread holds its share of the
// NEXT tile in registers (float4 / int4 loads issued before the current
// tile's math), so a CTA pays one load latency per kernel, not per tile.
// SL float4 prefetch slots per thread (SL * 256 >= 32 * pitch / 4) and U
// work items (column x 8 clusters) per thread are template parameters, so a
// narrow dimension (the common case) needs few registers and fits 3-4 CTAs
// per SM.  Pitches up to 288 floats (SL = 9; cols <= 256 have pitch <= 260).
constexpr int KM_SUM_SL = 9;
template <int KP, int U, int SL>
__global__ void __launch_bounds__(256) k_km_dim_sums(KmDimArgs a) {
  const int d = blockIdx.y;
  if (d >= a.ng || (int)blockIdx.x >= a.nblk[d]) return;
  constexpr int JB = 8, NJB = KP / JB, Q4 = KP / 4;
  __shared__ float ss[32 * 257];
  __shared__ __align__(16) float cs[32 * KP];
  const int cols = a.cols[d], pitch = a.pitch[d], pitch4 = pitch / 4;
  const int64_t rows = a.rows[d];
  const int nb = a.nblk[d];
  const int64_t rpb = ceil_div(ceil_div(rows, nb), 32) * 32;
  const int64_t r0 = blockIdx.x * rpb, r1 = min64(rows, r0 + rpb);
  const int nwork = cols * NJB;
  const int nS4 = 32 * pitch4;
  const int tid = threadIdx.x;
  const float4* S4 = reinterpret_cast<const float4*>(a.S[d]);
  const int4* C4 = reinterpret_cast<const int4*>(a.cnt[d]);
  float4 pv[SL];
  int4 pc = make_int4(0, 0, 0, 0);
  auto load = [&](int64_t rb) {
#pragma unroll
    for (int sl = 0; sl < SL; sl++) {
      const int i = tid + sl * 256;
      const int r = i / pitch4, c4 = i - r * pitch4;
      pv[sl] = (i < nS4 && rb + r < r1) ? S4[(rb + r) * pitch4 + c4]
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (tid < 32 * Q4) {
      const int r = tid / Q4;
      pc = rb + r < r1 ? C4[rb * Q4 + tid] : make_int4(0, 0, 0, 0);
    }
  };
  double acc64[U][JB];
#pragma unroll
  for (int u = 0; u < U; u++)
#pragma unroll
    for (int j = 0; j < JB; j++) acc64[u][j] = 0.0;
  if (r0 < r1) load(r0);
  for (int64_t rb = r0; rb < r1; rb += 32) {
    __syncthreads();   // the previous tile's math is done with ss / cs
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
    if (tid < 32 * Q4)
      *reinterpret_cast<float4*>(cs + 4 * tid) =
          make_float4((float)pc.x, (float)pc.y, (float)pc.z, (float)pc.w);
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
        const float4 c0 = *reinterpret_cast<const float4*>(cs + r * KP + jb * JB);
        const float4 c1 = *reinterpret_cast<const float4*>(cs + r * KP + jb * JB + 4);
        acc[0] = fmaf(c0.x, v, acc[0]); acc[1] = fmaf(c0.y, v, acc[1]);
        acc[2] = fmaf(c0.z, v, acc[2]); acc[3] = fmaf(c0.w, v, acc[3]);
        acc[4] = fmaf(c1.x, v, acc[4]); acc[5] = fmaf(c1.y, v, acc[5]);
        acc[6] = fmaf(c1.z, v, acc[6]); acc[7] = fmaf(c1.w, v, acc[7]);
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
      a.part[d][(int64_t)blockIdx.x * KP * cols + (jb * JB + j) * cols + c] = acc64[u][j];
  }
}

// R: fixed-order reduction of every partial into `red` (+ update)
__global__ void __launch_bounds__(256) k_km_reduce(const RedDesc* descs, int n, KmUpdateArgs u,
                                                   int fuse_update, int* done) {
  reduce_descs(descs, n, u.red);
  if (last_cta_done(done) && fuse_update) km_apply_update(u);
}

__global__ void k_km_update(KmUpdateArgs u) { km_apply_update(u); }

__global__ void k_km_assign_to_target64(const int32_t* __restrict__ a_dev,
                                        const int32_t* __restrict__ perm, int64_t r_T,
                                        int64_t* __restrict__ out) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p < r_T) out[perm[p]] = (int64_t)a_dev[p];
}

__global__ void k_km_assign_to_target(const int32_t* __restrict__ a_dev,
                                      const int32_t* __restrict__ perm, int64_t r_T,
                                      int32_t* __restrict__ out) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p < r_T) out[perm[p]] = a_dev[p];
}

static void km_dim_e_launch(int KP, dim3 g, size_t smem, cudaStream_t st, const KmDimArgs& a) {
  if (KP == 8) k_km_dim_e<8><<<g, 256, smem, st>>>(a);
  else if (KP == 16) k_km_dim_e<16><<<g, 256, smem, st>>>(a);
  else k_km_dim_e<32><<<g, 256, smem, st>>>(a);
}
template <int KP>
static const void* km_dim_sums_ptr_kp(int U, int SL) {
  if (U == 1) {
    if (SL <= 3) return (const void*)k_km_dim_sums<KP, 1, 3>;
    if (SL <= 5) return (const void*)k_km_dim_sums<KP, 1, 5>;
    return (const void*)k_km_dim_sums<KP, 1, 9>;
  }
  if (SL <= 3) return (const void*)k_km_dim_sums<KP, 2, 3>;
  if (SL <= 5) return (const void*)k_km_dim_sums<KP, 2, 5>;
  return (const void*)k_km_dim_sums<KP, 2, 9>;
}
static const void* km_dim_sums_ptr(int KP, int U, int SL) {
  return KP == 8 ? km_dim_sums_ptr_kp<8>(U, SL)
                 : KP == 16 ? km_dim_sums_ptr_kp<16>(U, SL) : km_dim_sums_ptr_kp<32>(U, SL);
}
static cudaError_t km_dim_sums_launch(const void* fn, dim3 g, size_t smem, cudaStream_t st,
                                      const KmDimArgs& a) {
  void* args[] = {const_cast<KmDimArgs*>(&a)};
  return cudaLaunchKernel(fn, g, dim3(256), args, smem, st);
}

// instantiation table: NT in {1,2,4} (k <= 8/16/32), KC in {1,2,3,4,6,8,12,16}
#define KM_KC_CASES(X, NT) X(NT, 1) X(NT, 2) X(NT, 3) X(NT, 4) X(NT, 6) X(NT, 8) X(NT, 12) X(NT, 16)
static int km_kc_for(int pf) {
  const int need = pf / 8 + 1;  // pf == 4 (mod 8): KC*8 > pf leaves the count column
  const int opts[] = {1, 2, 3, 4, 6, 8, 12, 16};
  for (int v : opts)
    if (v >= need) return v;
  return -1;
}
static int km_nt_for(int k) { return k <= 8 ? 1 : k <= 16 ? 2 : k <= 32 ? 4 : -1; }
static const void* km_fact_ptr(int nt, int kc) {
#define KM_PTR(NT_, KC_) if (nt == NT_ && kc == KC_) return (const void*)k_km_fact<NT_, KC_>;
  KM_KC_CASES(KM_PTR, 1) KM_KC_CASES(KM_PTR, 2) KM_KC_CASES(KM_PTR, 4)
#undef KM_PTR
  return nullptr;
}
static void km_fact_launch(int nt, int kc, const CUtensorMap& tm, const KmFactArgs& a, int grid,
                           size_t smem, cudaStream_t st) {
#define KM_LAUNCH(NT_, KC_) \
  if (nt == NT_ && kc == KC_) { k_km_fact<NT_, KC_><<<grid, KM_WARPS * 32, smem, st>>>(tm, a); return; }
  KM_KC_CASES(KM_LAUNCH, 1) KM_KC_CASES(KM_LAUNCH, 2) KM_KC_CASES(KM_LAUNCH, 4)
#undef KM_LAUNCH
}

}  // namespace flb

using namespace flb;

struct fl_kmeans {
  CUtensorMap tmF;               // F as [r_pad x pf] fp32, box 32 x (8 KC + 4)
  fl_table* t = nullptr;
  // tcgen05 path (default): blocked copy of F and kernel geometry
  bool tc = false;
  DevBuf Fblk;
  KmTcArgs ta{};
  int C4P = 0;
  KtGeom gm{};
  size_t smem_tc = 0;
  int k = 0, KP = 0, NT = 0, KC = 0, SC = 0;
  KmFactArgs fa{};
  KmDimArgs da{};
  KmUpdateArgs ua{};
  int nblk_fact = 0;
  size_t smem_fact = 0, smem_e = 0, smem_sum = 0;
  int grid_e = 1, grid_sum = 1, grid_red = 1, n_desc = 0;
  const void* fn_sum = nullptr;   // k_km_dim_sums<KP, U, SL> chosen for the dimension widths
  DevBuf descs;
  DevBuf C64, C32, E, cnt, part_fact, part_w, part_dim, red, loss_hist, state, assign, done;
  int loss_cap = 1 << 16;
  cudaGraphExec_t graph = nullptr, graph_assign = nullptr;
  cudaStream_t cap_stream = nullptr;
  // tcgen05 pass with MN-major row-contraction operands (kmeans_t5.cuh)
  bool t5 = false;
  CUtensorMap tmF5;
  KmT5Args t5a{};
  K5Geom k5g{};
  KmGen* gen = nullptr;   // width-general session (generic.cu) when the fused pass does not apply
  fl_comm* comm = nullptr;  // sharded run(): all-reduce of `red` between partial and update
};

namespace flb {

static int km_fact_run(fl_kmeans* s, cudaStream_t st, bool write_assign) {
  if (s->t5) {
    KmT5Args ta = s->t5a;
    ta.assign = write_assign ? s->assign.as<int32_t>() : nullptr;
    const size_t smem = s->k5g.total + 1024;
    if (s->KP == 16)
      k_km_t5<16><<<s->nblk_fact, K5_THREADS, smem, st>>>(s->tmF5, ta, s->k5g);
    else
      k_km_t5<32><<<s->nblk_fact, K5_THREADS, smem, st>>>(s->tmF5, ta, s->k5g);
  } else if (s->tc) {
    KmTcArgs ta = s->ta;
    ta.assign = write_assign ? s->assign.as<int32_t>() : nullptr;
    if (s->KP == 16)
      k_km_tc<16><<<s->nblk_fact, KT_THREADS, s->smem_tc, st>>>(ta, s->C4P, s->gm);
    else
      k_km_tc<32><<<s->nblk_fact, KT_THREADS, s->smem_tc, st>>>(ta, s->C4P, s->gm);
  } else {
    KmFactArgs fa = s->fa;
    fa.assign = write_assign ? s->assign.as<int32_t>() : nullptr;
    km_fact_launch(s->NT, s->KC, s->tmF, fa, s->nblk_fact, s->smem_fact, st);
  }
  FL_CHECK_LAUNCH();
  return FL_OK;
}

static int km_launch_iteration(fl_kmeans* s, cudaStream_t st, bool fuse_update,
                               bool write_assign) {
  if (s->da.ng > 0) {
    dim3 ge(s->grid_e, s->da.ng);
    km_dim_e_launch(s->KP, ge, s->smem_e, st, s->da);
    FL_CHECK_LAUNCH();
  }
  int rc = km_fact_run(s, st, write_assign);
  if (rc) return rc;
  if (s->da.ng > 0) {
    FL_CUDA(km_dim_sums_launch(s->fn_sum, dim3(s->grid_sum, s->da.ng), s->smem_sum, st, s->da));
    FL_CHECK_LAUNCH();
  }
  k_km_reduce<<<s->grid_red, 256, 0, st>>>(s->descs.as<RedDesc>(), s->n_desc, s->ua,
                                           fuse_update ? 1 : 0, s->done.as<int>());
  FL_CHECK_LAUNCH();
  return FL_OK;
}

static int km_graph(fl_kmeans* s, bool write_assign, cudaGraphExec_t* out) {
  if (*out) return FL_OK;
  if (!s->cap_stream) FL_CUDA(cudaStreamCreateWithFlags(&s->cap_stream, cudaStreamNonBlocking));
  cudaGraph_t g;
  FL_CUDA(cudaStreamBeginCapture(s->cap_stream, cudaStreamCaptureModeThreadLocal));
  int rc;
  if (s->comm) {   // sharded: partial -> all-reduce -> update
    rc = km_launch_iteration(s, s->cap_stream, false, write_assign);
    if (!rc) rc = comm_allreduce(s->comm, s->red.as<double>(), (size_t)s->k * s->t->c_T + s->k + 1,
                                 s->cap_stream);
    if (!rc) {
      k_km_update<<<1, 256, 0, s->cap_stream>>>(s->ua);
      if (cudaGetLastError() != cudaSuccess) rc = FL_ERR_CUDA;
    }
  } else {
    rc = km_launch_iteration(s, s->cap_stream, true, write_assign);
  }
  cudaError_t e = cudaStreamEndCapture(s->cap_stream, &g);
  if (rc) return rc;
  FL_CUDA(e);
  FL_CUDA(cudaGraphInstantiate(out, g, 0));
  FL_CUDA(cudaGraphDestroy(g));
  return FL_OK;
}

}  // namespace flb

extern "C" {

static int km_create_fused(fl_table* t, int32_t k, const double* centroids0, fl_kmeans** out,
                           void* stream) {
  if (!t || !t->finalized || !centroids0 || !out) {
    set_error("fl_kmeans_create: bad arguments");
    return FL_ERR_ARG;
  }
  if (k < 1 || k > t->r_T) {
    set_error("k_clusters = %d exceeds row count %lld", k, (long long)t->r_T);
    return FL_ERR_CONFIG;
  }
  const int NT = km_nt_for(k), KC = km_kc_for(t->pf);
  if (NT < 0 || KC < 0 || (int)t->g.size() > MAX_GATHER) {
    set_error("fused K-means supports k <= 32, <= 124 streamed columns and <= %d gathered "
              "sources (k=%d, streamed pitch=%d)", MAX_GATHER, k, t->pf);
    return FL_ERR_OP;
  }
  for (auto& g : t->g)
    if ((g.rows + 1) * (int64_t)(NT * 8) >= INT32_MAX) {
      set_error("fused K-means: dimension source with %lld rows is too large", (long long)g.rows);
      return FL_ERR_OP;
    }
  FL_CUDA(cudaSetDevice(t->device));
  cudaStream_t st = (cudaStream_t)stream;
  auto* s = new fl_kmeans();
  std::unique_ptr<fl_kmeans> guard(s);
  s->t = t;
  s->k = k;
  s->NT = NT;
  s->KP = NT * 8;
  s->KC = KC;
  s->SC = KC * 8;
  // tcgen05 variant (opt-in, FL_KM_TC=1; narrow stream blocks only): parity-
  // green but 2.9x slower than the per-warp mma.sync pass at C3 (1.57 vs
  // 0.54 ms, profiles/r01_kmeans_tc_vs_mma.txt): the row-contracting sums
  // need M >= 64 tcgen05 tiles over a 24-column / 16-cluster problem and
  // transposed operand copies, so operand fetch, not math, dominates.
  s->C4P = t->pf / 4;
  s->tc = (s->C4P + 1) * 4 <= 32 && getenv("FL_KM_TC") && atoi(getenv("FL_KM_TC")) != 0;
  if (s->tc) {
    s->KP = std::max(16, NT * 8);
    s->SC = (s->C4P + 1) * 4;
  }
  // default: the tcgen05 pass with MN-major row-contraction operands
  // (kmeans_t5.cuh) for <= 28 streamed columns; FL_KM_T5=0 selects the
  // per-warp mma.sync pass
  {
    const char* e5 = getenv("FL_KM_T5");
    const bool on = e5 && atoi(e5) != 0;   // opt-in until validated on the B200
    const int kp5 = std::max(16, NT * 8);
    if (!s->tc && on && t->pf <= 28 && k <= 32 &&
        k5_geom(kp5, (int)t->g.size()).total + 1024 <= 227 * 1024) {
      s->t5 = true;
      s->KP = kp5;
      s->SC = K5_SC;
    }
  }
  const int KP = s->KP, SC = s->SC, MT = (NT + 1) / 2;
  const int ng = (int)t->g.size();
  const int c_T = t->c_T;
  int rc;
  if ((rc = s->C64.alloc((size_t)k * c_T * 8))) return rc;
  if ((rc = s->C32.alloc((size_t)k * c_T * 4))) return rc;
  FL_CUDA(cudaMemcpyAsync(s->C64.p, centroids0, (size_t)k * c_T * 8, cudaMemcpyDefault, st));
  {
    std::vector<double> h((size_t)k * c_T);
    FL_CUDA(cudaMemcpyAsync(h.data(), s->C64.p, h.size() * 8, cudaMemcpyDeviceToHost, st));
    FL_CUDA(cudaStreamSynchronize(st));
    std::vector<float> f(h.size());
    for (size_t i = 0; i < h.size(); i++) f[i] = (float)h[i];
    FL_CUDA(cudaMemcpy(s->C32.p, f.data(), f.size() * 4, cudaMemcpyHostToDevice));
  }
  size_t e_total = 0, c_total = 0;
  for (auto& g : t->g) {
    e_total += (size_t)(g.rows + 1) * KP;
    c_total += (size_t)g.rows * KP;
  }
  if ((rc = s->E.alloc(e_total * 4 + 16))) return rc;
  if ((rc = s->cnt.alloc(c_total * 4 + 16))) return rc;
  if ((rc = s->red.alloc(((size_t)k * c_T + k + 1) * 8))) return rc;
  FL_CUDA(cudaMemsetAsync(s->red.p, 0, ((size_t)k * c_T + k + 1) * 8, st));
  if ((rc = s->loss_hist.alloc((size_t)s->loss_cap * 8))) return rc;
  if ((rc = s->state.alloc(sizeof(KmState)))) return rc;
  FL_CUDA(cudaMemsetAsync(s->state.p, 0, sizeof(KmState), st));
  if ((rc = s->done.alloc(16))) return rc;
  FL_CUDA(cudaMemsetAsync(s->done.p, 0, 16, st));
  if ((rc = s->assign.alloc((size_t)t->r_pad * 4))) return rc;
  FL_CUDA(cudaMemsetAsync(s->assign.p, 0, (size_t)t->r_pad * 4, st));

  // ---- fact pass geometry
  KmFactArgs& fa = s->fa;
  fa.F = t->F->as<float>();
  fa.pf = t->pf;
  fa.c_T = c_T;
  fa.k = k;
  fa.r_T = t->r_T;
  fa.nunits = t->r_pad / 32;
  fa.ng = ng;
  fa.sort_g = t->sort_g;
  {
    size_t eo = 0, co = 0;
    for (int d = 0; d < ng; d++) {
      fa.fk[d] = t->g[d].fk->as<int32_t>();
      fa.E[d] = s->E.as<float>() + eo;
      fa.cnt[d] = s->cnt.as<int32_t>() + co;
      fa.rows[d] = t->g[d].rows;
      eo += (size_t)(t->g[d].rows + 1) * KP;
      co += (size_t)t->g[d].rows * KP;
    }
  }
  fa.C32 = s->C32.as<float>();
  fa.f_tcol = t->d_f_tcol->as<int32_t>();
  fa.assign = nullptr;
  if (const char* dg = getenv("FL_KM_DIAG")) fa.diag = atoi(dg);   // timing experiments
  fa.npf_max = KM_PF_MAX;
  if (const char* pe = getenv("FL_KM_PF")) fa.npf_max = std::max(0, std::min(KM_PF_MAX, atoi(pe)));
  const int FP = SC + 4, ZP = KP + 4;
  fa.stage_bytes = (uint32_t)round_up(32 * FP * 4 + 128 * ng, 128);
  if ((rc = make_tmap_2d(&s->tmF, t->F->p, (uint64_t)t->r_pad, (uint64_t)t->pf,
                         (uint64_t)t->pf * 4, 32, (uint32_t)FP, 0)))
    return rc;
  (void)ZP;
  const size_t fixed = (size_t)KC * NT * 32 * 16 + (size_t)KP * (SC + 4) * 4 + (KP + 4) * 4 +
                       (size_t)KM_WARPS * km_scratch_floats(KP) * 4 +
                       (size_t)KM_WARPS * 3 * KM_PF_MAX * 32 * 4;
  const size_t fixed_al = round_up((int64_t)fixed, 128);
  // two CTAs (16 warps) per SM when the tile fits in half the shared memory
  const bool two = NT <= 2 && KC <= 4 && fixed_al + (size_t)KM_WARPS * 2 * fa.stage_bytes <= 110 * 1024;
  const size_t budget = two ? 110 * 1024 : 220 * 1024;
  int nst = (int)((budget - std::min(budget, fixed_al)) / ((size_t)KM_WARPS * fa.stage_bytes));
  if (const char* e = getenv("FL_KM_NST")) nst = atoi(e);
  nst = std::max(2, std::min(4, nst));
  fa.nst = nst;
  s->smem_fact = fixed_al + (size_t)KM_WARPS * nst * fa.stage_bytes;
  if (s->smem_fact > 225 * 1024) {
    set_error("fused K-means: shared memory budget exceeded (%zu bytes)", s->smem_fact);
    return FL_ERR_OP;
  }
  // the stage area starts right after the fixed area (kernel computes the
  // same offsets); pad the fixed area so stages stay 128-byte aligned
  const void* kf = km_fact_ptr(NT, KC);
  FL_CUDA(raise_smem_limit(kf, (int)s->smem_fact));
  int occ = 1;
  FL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kf, KM_WARPS * 32, s->smem_fact));
  occ = std::max(1, occ);
  s->nblk_fact = (int)std::max<int64_t>(
      1, std::min<int64_t>(ceil_div(fa.nunits, KM_WARPS), (int64_t)t->sm_count * occ));
  if (s->tc) {
    // blocked copy of F, smem layout, one persistent CTA per SM
    const int C4P = s->C4P;
    const int64_t ntiles = t->r_pad / KT_TILE;
    if ((rc = s->Fblk.alloc((size_t)t->r_pad * C4P * 16))) return rc;
    k_km_block<<<(unsigned)std::min<int64_t>(ceil_div(t->r_pad * C4P * 4, 256), 65535 * 8), 256,
                 0, st>>>(t->F->as<float>(), t->pf, t->r_pad, C4P, s->Fblk.as<float>());
    FL_CHECK_LAUNCH();
    KtGeom& gm = s->gm;
    gm.lbo_ft = (uint32_t)(ceil_div(SC, 8) * 128 + 16);
    gm.lbo_oh = (uint32_t)((KP / 8) * 128 + 16);
    gm.o_flo = (uint32_t)(C4P + 1) * 2048u;
    gm.o_fth = gm.o_flo + (uint32_t)(C4P + 1) * 2048u;
    const uint32_t ft_bytes = (uint32_t)round_up(32 * gm.lbo_ft + 2048, 128);
    gm.o_ftl = gm.o_fth + ft_bytes;
    gm.o_oht = gm.o_ftl + ft_bytes;
    gm.o_fk = gm.o_oht + (uint32_t)round_up(32 * gm.lbo_oh, 128);
    gm.stage = (uint32_t)round_up(gm.o_fk + 512 * std::max(ng, 1), 1024);
    gm.off_cf = KT_NS * gm.stage;
    const int CFP = (C4P + 1) * 4 + 4;
    const size_t cf_bytes = (size_t)2 * (C4P + 1) * KP * 16 + (size_t)KP * CFP * 4 +
                            (size_t)(KP + 4) * 4 + (size_t)32 * KP * 8 + 64;
    s->smem_tc = gm.off_cf + cf_bytes + 1024;
    if (s->smem_tc > 227 * 1024) {
      set_error("fused K-means (tcgen05): shared memory budget exceeded (%zu bytes)", s->smem_tc);
      return FL_ERR_OP;
    }
    const void* kt = KP == 16 ? (const void*)k_km_tc<16> : (const void*)k_km_tc<32>;
    FL_CUDA(raise_smem_limit(kt, (int)s->smem_tc));
    s->nblk_fact = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, t->sm_count));
    KmTcArgs& ta = s->ta;
    ta.Fblk = s->Fblk.as<float>();
    ta.pf = t->pf;
    ta.c_T = c_T;
    ta.k = k;
    ta.r_T = t->r_T;
    ta.ntiles = ntiles;
    ta.ng = ng;
    ta.sort_g = t->sort_g;
    for (int d = 0; d < ng; d++) {
      ta.fk[d] = fa.fk[d];
      ta.E[d] = fa.E[d];
      ta.cnt[d] = fa.cnt[d];
      ta.rows[d] = fa.rows[d];
    }
    ta.C32 = s->C32.as<float>();
    ta.f_tcol = t->d_f_tcol->as<int32_t>();
    ta.assign = nullptr;
    ta.SC = SC;
  }
  if (s->t5) {
    s->k5g = k5_geom(KP, ng);
    const size_t smem5 = s->k5g.total + 1024;
    if (smem5 > 227 * 1024) {
      set_error("fused K-means (tcgen05): shared memory budget exceeded (%zu bytes)", smem5);
      return FL_ERR_OP;
    }
    if ((rc = make_tmap_2d(&s->tmF5, t->F->p, (uint64_t)t->r_pad, (uint64_t)t->pf,
                           (uint64_t)t->pf * 4, K5_TILE, 32, 128)))
      return rc;
    const void* k5 = KP == 16 ? (const void*)k_km_t5<16> : (const void*)k_km_t5<32>;
    FL_CUDA(raise_smem_limit(k5, (int)smem5));
    const int64_t ntiles = t->r_pad / K5_TILE;
    s->nblk_fact = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, t->sm_count));
    KmT5Args& ta = s->t5a;
    ta.pf = t->pf;
    ta.c_T = c_T;
    ta.k = k;
    ta.r_T = t->r_T;
    ta.ntiles = ntiles;
    ta.ng = ng;
    ta.sort_g = t->sort_g;
    for (int d = 0; d < ng; d++) {
      ta.fk[d] = fa.fk[d];
      ta.E[d] = fa.E[d];
      ta.cnt[d] = fa.cnt[d];
      ta.rows[d] = fa.rows[d];
    }
    ta.C32 = s->C32.as<float>();
    ta.f_tcol = t->d_f_tcol->as<int32_t>();
    ta.assign = nullptr;
  }
  if ((rc = s->part_fact.alloc((size_t)s->nblk_fact * (KP * SC + 1) * 8))) return rc;
  if ((rc = s->part_w.alloc((size_t)s->nblk_fact * KM_WARPS * MT * 16 * SC * 8))) return rc;
  fa.part_w = s->part_w.as<double>();
  fa.part = s->part_fact.as<double>();
  s->ta.part = fa.part;
  s->t5a.part = fa.part;

  // ---- dimension kernels
  KmDimArgs& da = s->da;
  da.ng = ng;
  da.k = k;
  da.KP = KP;
  da.c_T = c_T;
  da.C32 = s->C32.as<float>();
  int max_cols = 1;
  int64_t max_rows = 1;
  size_t part_total = 0;
  s->grid_sum = 1;
  int sum_u = 1, sum_sl = 1;
  for (int d = 0; d < ng; d++) {
    const GatherSrc& g = t->g[d];
    if (g.cols * (KP / 8) > 256) sum_u = 2;
    sum_sl = std::max(sum_sl, (int)ceil_div(32 * (g.pitch / 4), 256));
  }
  s->fn_sum = km_dim_sums_ptr(KP, sum_u, sum_sl);
  int occ_sum = 2;
  FL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_sum, s->fn_sum, 256, 0));
  occ_sum = std::max(1, std::min(occ_sum, 4));
  for (int d = 0; d < ng; d++) {
    const GatherSrc& g = t->g[d];
    da.S[d] = g.S->as<float>();
    da.pitch[d] = g.pitch;
    da.cols[d] = g.cols;
    da.rows[d] = g.rows;
    da.tcol[d] = g.d_tcol->as<int32_t>();
    da.E[d] = const_cast<float*>(fa.E[d]);
    da.cnt[d] = fa.cnt[d];
    // row ranges of >= 4 tiles, one wave of resident CTAs: the next tile is
    // prefetched in registers, and few partials keep the final reduction short
    int nb = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(g.rows, 128),
                                                         (int64_t)t->sm_count * occ_sum));
    da.nblk[d] = nb;
    s->grid_sum = std::max(s->grid_sum, nb);
    max_cols = std::max(max_cols, g.cols);
    max_rows = std::max(max_rows, g.rows + 1);
    part_total += (size_t)nb * KP * g.cols;
  }
  if ((rc = s->part_dim.alloc(part_total * 8 + 16))) return rc;
  {
    size_t po = 0;
    for (int d = 0; d < ng; d++) {
      da.part[d] = s->part_dim.as<double>() + po;
      po += (size_t)da.nblk[d] * KP * t->g[d].cols;
    }
  }
  int max_pitch = 4;
  for (auto& g : t->g) max_pitch = std::max(max_pitch, g.pitch);
  s->smem_e = (size_t)max_pitch * KP * 4;
  s->grid_e = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(max_rows + 1, 256),
                                                          (int64_t)t->sm_count * 4));
  s->smem_sum = 0;   // static tiles
  for (auto& g : t->g)
    if (g.cols > 256 || g.cols * KP / 8 > 512 || 32 * (g.pitch / 4) > KM_SUM_SL * 256) {
      set_error("fused K-means: dimension source with %d columns is too wide", g.cols);
      return FL_ERR_OP;
    }
  if (s->smem_e > 200 * 1024 || s->smem_sum > 200 * 1024) {
    set_error("fused K-means: dimension source too wide");
    return FL_ERR_OP;
  }
  {
    const void* fe = KP == 8 ? (const void*)k_km_dim_e<8> : KP == 16 ? (const void*)k_km_dim_e<16>
                                                                     : (const void*)k_km_dim_e<32>;
    FL_CUDA(raise_smem_limit(fe, (int)std::max<size_t>(s->smem_e, 16)));
  }

  KmUpdateArgs& ua = s->ua;
  ua.c_T = c_T;
  ua.k = k;
  ua.KP = KP;
  ua.SC = SC;
  ua.pf = t->pf;
  ua.ng = ng;
  ua.f_tcol = t->d_f_tcol->as<int32_t>();
  for (int d = 0; d < ng; d++) {
    ua.d_tcol[d] = t->g[d].d_tcol->as<int32_t>();
    ua.d_cols[d] = t->g[d].cols;
    ua.part_dim[d] = da.part[d];
    ua.nblk_dim[d] = da.nblk[d];
  }
  ua.part_fact = s->part_fact.as<double>();
  ua.nblk_fact = s->nblk_fact;
  ua.red = s->red.as<double>();
  ua.C64 = s->C64.as<double>();
  ua.C32 = s->C32.as<float>();
  ua.loss_hist = s->loss_hist.as<double>();
  ua.loss_cap = s->loss_cap;
  ua.state = s->state.as<KmState>();
  {
    std::vector<RedDesc> dv;
    const int fst = KP * SC + 1;
    const double* pfb = s->part_fact.as<double>();
    for (int j = 0; j < k; j++) {
      for (int c = 0; c < t->pf; c++)
        if (t->f_tcol[c] >= 0) dv.push_back(RedDesc{pfb + j * SC + c, fst, s->nblk_fact, j * c_T + t->f_tcol[c], 0});
      dv.push_back(RedDesc{pfb + j * SC + t->pf, fst, s->nblk_fact, k * c_T + j, 0});
    }
    dv.push_back(RedDesc{pfb + KP * SC, fst, s->nblk_fact, k * c_T + k, 0});
    for (int d = 0; d < ng; d++) {
      const int cols = t->g[d].cols;
      for (int j = 0; j < k; j++)
        for (int c = 0; c < cols; c++)
          dv.push_back(RedDesc{da.part[d] + j * cols + c, KP * cols, da.nblk[d], j * c_T + t->g[d].tcol[c], 0});
    }
    s->n_desc = (int)dv.size();
    if ((rc = s->descs.alloc(dv.size() * sizeof(RedDesc)))) return rc;
    FL_CUDA(cudaMemcpy(s->descs.p, dv.data(), dv.size() * sizeof(RedDesc), cudaMemcpyHostToDevice));
    s->grid_red = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(s->n_desc, 8), 4 * t->sm_count));
  }
  FL_CUDA(cudaStreamSynchronize(st));
  *out = guard.release();
  return FL_OK;
}

// The fused pass when it applies (k <= 32, streamed pitch <= 124, <= 8
// gathered sources, dimension widths within its tiles); every other shape --
// or FL_KM_GENERIC=1 -- runs the width-general session of generic.cu.
int fl_kmeans_create(fl_table* t, int32_t k, const double* centroids0, fl_kmeans** out,
                     void* stream) {
  const char* fg = getenv("FL_KM_GENERIC");
  const bool force = fg && atoi(fg) != 0;
  if (!force) {
    const int rc = km_create_fused(t, k, centroids0, out, stream);
    if (rc != FL_ERR_OP) return rc;
  }
  if (!t || !t->finalized || !centroids0 || !out) {
    set_error("fl_kmeans_create: bad arguments");
    return FL_ERR_ARG;
  }
  if (k < 1 || k > t->r_T) {
    set_error("k_clusters = %d exceeds row count %lld", k, (long long)t->r_T);
    return FL_ERR_CONFIG;
  }
  FL_CUDA(cudaSetDevice(t->device));
  auto* s = new fl_kmeans();
  std::unique_ptr<fl_kmeans> guard(s);
  s->t = t;
  s->k = k;
  const int rc = kmg_create(t, k, centroids0, (cudaStream_t)stream, &s->gen);
  if (rc) return rc;
  *out = guard.release();
  return FL_OK;
}

int fl_kmeans_set_comm(fl_kmeans* s, fl_comm* c) {
  if (!s) return FL_ERR_ARG;
  if (s->comm != c) {
    if (s->graph) cudaGraphExecDestroy(s->graph);
    if (s->graph_assign) cudaGraphExecDestroy(s->graph_assign);
    s->graph = s->graph_assign = nullptr;
  }
  s->comm = c;
  if (s->gen) kmg_set_comm(s->gen, c);
  return FL_OK;
}

int fl_kmeans_path(fl_kmeans* s, int32_t* path) {
  if (!s || !path) return FL_ERR_ARG;
  *path = s->gen ? 2 : s->tc ? 1 : s->t5 ? 3 : 0;
  return FL_OK;
}

int fl_kmeans_partial(fl_kmeans* s, int32_t write_assign, void* stream) {
  if (!s) return FL_ERR_ARG;
  FL_CUDA(cudaSetDevice(s->t->device));
  if (s->gen) return kmg_partial(s->gen, (cudaStream_t)stream);
  return km_launch_iteration(s, (cudaStream_t)stream, false, write_assign != 0);
}

int fl_kmeans_reduce_buffer(fl_kmeans* s, double** buf, int32_t* len) {
  if (!s || !buf || !len) return FL_ERR_ARG;
  if (s->gen) {
    int n = 0;
    *buf = kmg_red(s->gen, &n);
    *len = n;
    return FL_OK;
  }
  *buf = s->red.as<double>();
  *len = s->k * s->t->c_T + s->k + 1;
  return FL_OK;
}

int fl_kmeans_update(fl_kmeans* s, void* stream) {
  if (!s) return FL_ERR_ARG;
  FL_CUDA(cudaSetDevice(s->t->device));
  if (s->gen) return kmg_update(s->gen, (cudaStream_t)stream);
  k_km_update<<<1, 256, 0, (cudaStream_t)stream>>>(s->ua);
  FL_CHECK_LAUNCH();
  return FL_OK;
}

int fl_kmeans_run(fl_kmeans* s, int32_t iterations, void* stream) {
  if (!s || iterations < 1) {
    set_error("iterations must be >= 1");
    return FL_ERR_CONFIG;
  }
  FL_CUDA(cudaSetDevice(s->t->device));
  if (s->gen) return kmg_run(s->gen, iterations, (cudaStream_t)stream);
  int rc = km_graph(s, false, &s->graph);
  if (rc) return rc;
  rc = km_graph(s, true, &s->graph_assign);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  for (int i = 0; i + 1 < iterations; i++) FL_CUDA(cudaGraphLaunch(s->graph, st));
  FL_CUDA(cudaGraphLaunch(s->graph_assign, st));
  return FL_OK;
}

int fl_kmeans_kernel_times(fl_kmeans* s, int32_t iters, float* ms_out, void* stream) {
  if (!s || iters < 1 || !ms_out) return FL_ERR_ARG;
  FL_CUDA(cudaSetDevice(s->t->device));
  cudaStream_t st = (cudaStream_t)stream;
  if (s->gen) {   // one slot: the whole width-general iteration
    cudaEvent_t e0, e1;
    FL_CUDA(cudaEventCreate(&e0));
    FL_CUDA(cudaEventCreate(&e1));
    FL_CUDA(cudaEventRecord(e0, st));
    for (int i = 0; i < iters; i++) {
      const int rc = kmg_partial(s->gen, st);
      if (rc) return rc;
    }
    FL_CUDA(cudaEventRecord(e1, st));
    FL_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    FL_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    ms_out[0] = ms_out[2] = ms_out[3] = 0.f;
    ms_out[1] = ms / iters;
    return FL_OK;
  }
  cudaEvent_t ev[5];
  for (auto& e : ev) FL_CUDA(cudaEventCreate(&e));
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int i = 0; i < iters; i++) {
    FL_CUDA(cudaEventRecord(ev[0], st));
    if (s->da.ng > 0) {
      km_dim_e_launch(s->KP, dim3(s->grid_e, s->da.ng), s->smem_e, st, s->da);
      FL_CHECK_LAUNCH();
    }
    FL_CUDA(cudaEventRecord(ev[1], st));
    int rc = km_fact_run(s, st, false);
    if (rc) return rc;
    FL_CUDA(cudaEventRecord(ev[2], st));
    if (s->da.ng > 0) {
      FL_CUDA(km_dim_sums_launch(s->fn_sum, dim3(s->grid_sum, s->da.ng), s->smem_sum, st, s->da));
      FL_CHECK_LAUNCH();
    }
    FL_CUDA(cudaEventRecord(ev[3], st));
    k_km_reduce<<<s->grid_red, 256, 0, st>>>(s->descs.as<RedDesc>(), s->n_desc, s->ua, 1,
                                             s->done.as<int>());
    FL_CHECK_LAUNCH();
    FL_CUDA(cudaEventRecord(ev[4], st));
    FL_CUDA(cudaEventSynchronize(ev[4]));
    for (int j = 0; j < 4; j++) {
      float ms = 0.f;
      FL_CUDA(cudaEventElapsedTime(&ms, ev[j], ev[j + 1]));
      acc[j] += ms;
    }
  }
  for (int j = 0; j < 4; j++) ms_out[j] = acc[j] / iters;
  for (auto& e : ev) cudaEventDestroy(e);
  return FL_OK;
}

int fl_kmeans_result(fl_kmeans* s, double* centroids, int32_t* assign, double* loss, int32_t n,
                     int32_t* n_done, void* stream) {
  if (!s) return FL_ERR_ARG;
  FL_CUDA(cudaSetDevice(s->t->device));
  cudaStream_t st = (cudaStream_t)stream;
  if (s->gen) {
    int nd = 0;
    const int rc = kmg_result(s->gen, centroids, assign, nullptr, loss, n, &nd, st);
    if (n_done) *n_done = nd;
    return rc;
  }
  KmState h{};
  FL_CUDA(cudaMemcpyAsync(&h, s->state.p, sizeof(h), cudaMemcpyDeviceToHost, st));
  if (centroids)
    FL_CUDA(cudaMemcpyAsync(centroids, s->C64.p, (size_t)s->k * s->t->c_T * 8, cudaMemcpyDefault,
                            st));
  if (assign) {
    int32_t* tmp = nullptr;
    FL_CUDA(cudaMallocAsync((void**)&tmp, (size_t)s->t->r_T * 4 + 16, st));
    k_km_assign_to_target<<<(unsigned)ceil_div(s->t->r_T, 256), 256, 0, st>>>(
        s->assign.as<int32_t>(), s->t->perm->as<int32_t>(), s->t->r_T, tmp);
    FL_CHECK_LAUNCH();
    FL_CUDA(cudaMemcpyAsync(assign, tmp, (size_t)s->t->r_T * 4, cudaMemcpyDefault, st));
    FL_CUDA(cudaFreeAsync(tmp, st));
  }
  FL_CUDA(cudaStreamSynchronize(st));
  int nd = std::min(h.it, s->loss_cap);
  if (n_done) *n_done = nd;
  if (loss && n > 0) {
    int m = std::min(n, nd);
    if (m > 0) FL_CUDA(cudaMemcpy(loss, s->loss_hist.p, (size_t)m * 8, cudaMemcpyDefault));
  }
  return FL_OK;
}

int fl_kmeans_assignments64(fl_kmeans* s, int64_t* assign, void* stream) {
  if (!s || !assign) return FL_ERR_ARG;
  FL_CUDA(cudaSetDevice(s->t->device));
  cudaStream_t st = (cudaStream_t)stream;
  if (s->gen) return kmg_result(s->gen, nullptr, nullptr, assign, nullptr, 0, nullptr, st);
  int64_t* tmp = nullptr;
  FL_CUDA(cudaMallocAsync((void**)&tmp, (size_t)s->t->r_T * 8 + 16, st));
  k_km_assign_to_target64<<<(unsigned)ceil_div(s->t->r_T, 256), 256, 0, st>>>(
      s->assign.as<int32_t>(), s->t->perm->as<int32_t>(), s->t->r_T, tmp);
  FL_CHECK_LAUNCH();
  FL_CUDA(cudaMemcpyAsync(assign, tmp, (size_t)s->t->r_T * 8, cudaMemcpyDefault, st));
  FL_CUDA(cudaFreeAsync(tmp, st));
  FL_CUDA(cudaStreamSynchronize(st));
  return FL_OK;
}

int fl_kmeans_destroy(fl_kmeans* s) {
  if (!s) return FL_OK;
  cudaSetDevice(s->t->device);
  if (s->graph) cudaGraphExecDestroy(s->graph);
  if (s->graph_assign) cudaGraphExecDestroy(s->graph_assign);
  if (s->cap_stream) cudaStreamDestroy(s->cap_stream);
  if (s->gen) kmg_destroy(s->gen);
  delete s;
  return FL_OK;
}

}  // extern "C"
