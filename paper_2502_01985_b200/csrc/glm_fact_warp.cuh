// K2 v2: the fact-row pass with one independent TMA pipeline PER WARP.
//
// Why: the CTA-tile version (k_glm_fact) was latency-bound (ncu r01: 25%
// occupancy, two __syncthreads per 256-row tile, ~490 warp instructions per
// 32 rows, DRAM at 38% of peak although traffic == algorithmic bytes).
// Here each warp owns a contiguous range of device rows and streams it through
// its own NST-stage ring of TMA bulk copies (lane 0 issues, all lanes wait on
// the stage mbarrier) -- no block-level synchronisation in the main loop, so
// warps drift and hide each other's latency.  A row lives in registers
// (C4 float4, compile-time), each lane owns RPL rows per stage (ILP), and the
// I_sort^T segmented sum is a warp scan with a register-carried running
// segment; segments that cross warp ranges are stitched in a fixed order by
// the last CTA (deterministic).
#pragma once
// (included inside namespace flb by glm.cu)

constexpr int FW_WARPS = 8;        // warps per CTA
constexpr int FW_FLUSH = 16;       // stages between fp32 -> fp64 flushes
constexpr int FW_LCAP = 32;        // solo: segment records per warp before a gradient flush
constexpr int FW_QCAP = 4096;      // solo: q entries per CTA (dimension rows it references)
constexpr int FW_SOLO_PITCH = 64;  // solo: widest sort-source row
constexpr int FW_GROUP = 16;       // solo: CTAs per first-level reduction group
// narrow rows (C4 <= 7) run two CTAs (16 warps) per SM: the pass is
// latency-bound at one CTA (ncu r01: 12.5% warps active, issue 39%)
__host__ __device__ constexpr int fw_min_blocks(int c4) { return c4 <= 7 ? 2 : 1; }

struct WarpCarry {
  int head_key, tail_key, through, pad;
  double head_val, tail_val;
};

// Last CTA of a fact pass: segments that span warp ranges are stitched in a
// fixed order from a shared-memory copy of the carry records (coalesced
// 16-byte loads, all in flight together) instead of chained dependent L2
// reads; the global records are walked directly when they do not fit.
// Kept out of line so the streaming loop's register allocation is untouched.
__device__ __noinline__ void stitch_carries(const WarpCarry* carry, int64_t NW, float* bins,
                                            char* scratch, size_t scratch_bytes) {
  if ((size_t)NW * sizeof(WarpCarry) <= scratch_bytes) {
    const int4* src = reinterpret_cast<const int4*>(carry);
    int4* dst = reinterpret_cast<int4*>(scratch);
    const int64_t n16 = NW * (int64_t)(sizeof(WarpCarry) / 16);
    for (int64_t i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = __ldcg(src + i);
    __syncthreads();
    const WarpCarry* cr = reinterpret_cast<const WarpCarry*>(scratch);
    for (int64_t c = threadIdx.x; c < NW; c += blockDim.x) {
      const int K = cr[c].tail_key;
      if (K < 0) continue;
      double total = cr[c].tail_val;
      for (int64_t c2 = c + 1; c2 < NW; c2++) {
        if (cr[c2].head_key != K) break;
        total += cr[c2].head_val;
        if (!cr[c2].through) break;
      }
      bins[K] = (float)total;
    }
  } else {
    volatile const WarpCarry* cr = carry;   // records written by other CTAs
    for (int64_t c = threadIdx.x; c < NW; c += blockDim.x) {
      const int K = cr[c].tail_key;
      if (K < 0) continue;
      double total = cr[c].tail_val;
      for (int64_t c2 = c + 1; c2 < NW; c2++) {
        if (cr[c2].head_key != K) break;
        total += cr[c2].head_val;
        if (!cr[c2].through) break;
      }
      bins[K] = (float)total;
    }
  }
}

struct GlmFactWArgs {
  const float* F;
  int pf;
  const void* y;
  int64_t r_T, nunits;       // nunits = r_pad / RW
  int ng, sort_g;
  const int32_t* fk[MAX_GATHER];
  const float* q[MAX_GATHER];
  float* bins;
  float* resid;
  const float* wF;
  double* part;              // gridDim.x x (pf + 1)
  WarpCarry* carry;          // gridDim.x * FW_WARPS
  GlmState* state;
  uint32_t stage_bytes, off_y, off_fk;
  int nst;
  // solo iteration: the only gathered source is the sort source, so each CTA
  // computes the q_d entries its rows reference (a contiguous dimension-row
  // range) in its prologue, and turns its segment sums into that source's
  // gradient partial S_d^T bins (linear in the bins, so warp- and CTA-
  // boundary segments need no stitching); the last CTA reduces and updates.
  // One kernel per GD iteration (dim_q / dim_t are not launched).
  int solo, fuse_update;
  const float* S0;           // sort source values, r_0 x pitch0
  int pitch0;
  const float* w0d;          // fp32 w of the sort source's columns (pitch0)
  int64_t n_neg0;            // device rows without a match (FK -1, at the front)
  double* part_d;            // gridDim.x x pitch0
  const UpdateArgs* up;      // the session's update arguments (device copy: no param copies)
  int* gcnt;                 // per-group arrival counters (zeroed; reset by each group's last CTA)
  double* gpart;             // groups x (pf + 1 + pitch0): first-level partial sums
  int diag;                  // FL_GLM_SOLO_DIAG (timing experiments only): 1 no tail, 2 no final
                             // level, 4 no update, 16 final CTA elected but idle, 32 final sums
                             // with every group load in flight (measured slower), 64 final sums
                             // without loads, 128 __threadfence instead of acq_rel arrivals,
                             // 256 no L2 prefetch of the tail's operands
  int qcap;                  // q entries staged per CTA (a multiple of 4, <= FW_QCAP)
  int s0_rows;               // > 0: the CTA's S_d row span (<= s0_rows rows) is bulk-copied
                             // into shared memory before the PDL wait and serves both the
                             // q prologue and the gradient records (0: read through L2)
};

struct SoloRec {
  int key;
  float v;
};

// the last CTA of a solo iteration: red = the fixed-order sum of the group
// partials [grad_F | loss | grad_d], then the update.  Arguments are plain
// pointers / scalars and the update arguments live in global memory: nothing
// forces a local copy of a kernel parameter struct.  (Variants that staged
// the partials, red and w in shared memory with up-front independent loads
// measured 1.2-1.7 us slower per C1 step: profiles/r02_s2_experiments.txt.)
__device__ __noinline__ void glm_solo_final(const double* __restrict__ gpart, int ngroups, int pf,
                                            int pitch0, int sort_g, int fuse_update,
                                            const UpdateArgs* u, int batched) {
  const int tid = threadIdx.x;
  const int c_T = u->c_T, ne = pf + 1 + pitch0;
  double* red = u->red;
  for (int c = tid; c <= c_T; c += blockDim.x) red[c] = 0.0;
  __syncthreads();
  const int32_t* dt = u->d_tcol[sort_g];
  for (int e = tid; e < ne; e += blockDim.x) {
    double v = 0.0;
    if (batched == 2) {
      v = (double)ngroups;   // timing experiment only: no partial loads
    } else if (batched) {
      // A/B only: every group partial of the element in flight at once,
      // summed in the same order (measured 0.8 us slower per C1 step than
      // the loop below, profiles/r02_s2_experiments.txt)
      for (int g0 = 0; g0 < ngroups; g0 += 32) {
        double tv[32];
#pragma unroll
        for (int q = 0; q < 32; q++)
          tv[q] = g0 + q < ngroups ? __ldcg(gpart + (int64_t)(g0 + q) * ne + e) : 0.0;
#pragma unroll
        for (int q = 0; q < 32; q++)
          if (g0 + q < ngroups) v += tv[q];
      }
    } else {
      for (int g = 0; g < ngroups; g++) v += __ldcg(gpart + (int64_t)g * ne + e);
    }
    const int dst = e < pf ? u->f_tcol[e] : e == pf ? c_T : dt[e - pf - 1];
    if (dst >= 0) red[dst] = v;
  }
  __syncthreads();
  if (fuse_update) glm_apply_update(*u);
}

template <int MODEL, int C4, int RPL>
__global__ void __launch_bounds__(FW_WARPS * 32, (C4 <= 7 ? 2 : 1))
    k_glm_fact_w(GlmFactWArgs a) {
  constexpr int RW = 32 * RPL;               // rows per warp stage
  constexpr bool W_REG = C4 <= 9;            // w in registers (else smem broadcast)
  extern __shared__ __align__(128) char smem[];
  __shared__ uint64_t bar[FW_WARPS][4];
  __shared__ double gsum[FW_WARPS][C4 * 4];
  __shared__ double lsum[FW_WARPS];
  __shared__ float4 w_s[C4];
  __shared__ int is_last;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * FW_WARPS + warp;
  const int64_t NW = (int64_t)gridDim.x * FW_WARPS;
  const int64_t base = a.nunits / NW, rem = a.nunits % NW;
  const int64_t u0 = gw * base + min64(gw, rem);
  const int64_t cnt = base + (gw < rem ? 1 : 0);
  const int64_t W0 = u0 * RW;
  const int64_t W1 = min64((u0 + cnt) * RW, a.r_T);
  const bool has_sort = a.sort_g >= 0;
  const int32_t* fks = has_sort ? a.fk[a.sort_g] : nullptr;
  constexpr uint32_t F_BYTES = RW * C4 * 16;
  constexpr uint32_t Y_BYTES = MODEL == 1 ? RW : RW * 4;
  const uint32_t tx = F_BYTES + Y_BYTES + (has_sort ? RW * 4 : 0);
  char* wsm = smem + (size_t)warp * a.nst * a.stage_bytes;
  uint64_t* wbar = bar[warp];

  auto issue = [&](int s, int64_t unit) {
    char* st = wsm + (size_t)s * a.stage_bytes;
    mbar_arrive_expect_tx(&wbar[s], tx);
    bulk_g2s(st, a.F + unit * RW * (int64_t)a.pf, F_BYTES, &wbar[s]);
    bulk_g2s(st + a.off_y, reinterpret_cast<const char*>(a.y) + unit * (int64_t)Y_BYTES, Y_BYTES,
             &wbar[s]);
    if (has_sort) bulk_g2s(st + a.off_fk, fks + unit * RW, RW * 4, &wbar[s]);
  };
  // solo: this CTA's dimension-row span [k_lo, k_lo + nq) (keys are sorted)
  char* solo_sm = smem + (size_t)FW_WARPS * a.nst * a.stage_bytes;
  float* q_s = reinterpret_cast<float*>(solo_sm);
  SoloRec* rec = reinterpret_cast<SoloRec*>(q_s + a.qcap) + warp * FW_LCAP;
  double* gsd_all = reinterpret_cast<double*>(reinterpret_cast<SoloRec*>(q_s + a.qcap) +
                                              FW_WARPS * FW_LCAP);
  float* S0_s = reinterpret_cast<float*>(gsd_all + FW_WARPS * FW_SOLO_PITCH);
  __shared__ int span_s[2];
  __shared__ uint64_t s0bar;
  // F, labels, FKs and S_d are immutable: the warp's first stages (and the
  // CTA's S_d span) stream in before the dependency wait (PDL), overlapping
  // the previous kernel's tail
  if (a.solo && threadIdx.x == 0) {
    const int64_t cw0 = (int64_t)blockIdx.x * FW_WARPS, cw1 = cw0 + FW_WARPS;
    const int64_t cu0 = cw0 * base + min64(cw0, rem), cu1 = cw1 * base + min64(cw1, rem);
    const int64_t rlo = max64(cu0 * RW, a.n_neg0), rhi = min64(cu1 * RW, a.r_T) - 1;
    int klo = 0, nq = 0;
    if (rlo <= rhi) {
      klo = __ldg(fks + rlo);
      nq = __ldg(fks + rhi) - klo + 1;
    }
    span_s[0] = klo;
    span_s[1] = nq;
    if (a.s0_rows > 0 && nq > 0) {
      mbar_init(&s0bar, 1);
      fence_mbar_init();
      const uint32_t bytes = (uint32_t)nq * (uint32_t)a.pitch0 * 4u;
      mbar_arrive_expect_tx(&s0bar, bytes);
      bulk_g2s(S0_s, a.S0 + (int64_t)klo * a.pitch0, bytes, &s0bar);
    }
  }
  if (lane == 0) {
    lsum[warp] = 0.0;
    for (int s = 0; s < a.nst; s++) mbar_init(&wbar[s], 1);
    fence_mbar_init();
    for (int s = 0; s < a.nst && s < cnt; s++) issue(s, u0 + s);
  }
  // solo: the tail's small operands (update arguments, column maps, w, red,
  // the arrival counters, the fp32 w copies) are pulled into L2 while the
  // fact rows stream: after a cold L2 each of the tail's dependent accesses
  // would otherwise be an HBM round trip.  FL_GLM_SOLO_DIAG bit 256: off.
  if (a.solo && blockIdx.x == 0 && threadIdx.x == 32 && !(a.diag & 256)) {
    const UpdateArgs* u = a.up;
    auto r16 = [](int64_t b) { return (uint32_t)((b + 15) & ~(int64_t)15); };
    bulk_prefetch_l2(u, r16(sizeof(UpdateArgs)));
    const int c_T = u->c_T;
    bulk_prefetch_l2(u->f_tcol, r16((int64_t)u->pf * 4));
    bulk_prefetch_l2(u->d_tcol[0], r16((int64_t)a.pitch0 * 4));
    bulk_prefetch_l2(u->w64, r16((int64_t)c_T * 8));
    bulk_prefetch_l2(u->red, r16((int64_t)(c_T + 1) * 8));
    bulk_prefetch_l2(u->wF, r16((int64_t)u->pf * 4));
    bulk_prefetch_l2(u->wd[0], r16((int64_t)a.pitch0 * 4));
    bulk_prefetch_l2(u->state, 16);
    bulk_prefetch_l2(a.gcnt, r16(((int64_t)gridDim.x + FW_GROUP - 1) / FW_GROUP * 4));
  }
  for (int j = lane; j < C4 * 4; j += 32) gsum[warp][j] = 0.0;
  pdl_wait();      // w (previous update) and q (this iteration's dim_q) are final
  pdl_trigger();
  for (int j = threadIdx.x; j < C4; j += blockDim.x)
    w_s[j] = reinterpret_cast<const float4*>(a.wF)[j];
  // solo: q_d of the dimension rows this CTA's rows reference
  int k_lo = 0;
  const bool s0_smem = a.solo && a.s0_rows > 0;
  if (a.solo) {
    __syncthreads();   // span_s
    k_lo = span_s[0];
    const int nq = span_s[1];
    const int p4 = a.pitch0 / 4;
    const float4* w04 = reinterpret_cast<const float4*>(a.w0d);
    if (s0_smem && nq > 0) mbar_wait(&s0bar, 0);
    const float* S0b = s0_smem ? S0_s : a.S0 + (int64_t)k_lo * a.pitch0;
    for (int i = threadIdx.x; i < nq; i += blockDim.x) {
      const float4* sr = reinterpret_cast<const float4*>(S0b + (int64_t)i * a.pitch0);
      float z = 0.f;
      for (int j = 0; j < p4; j++) {
        const float4 v = sr[j], ww = w04[j];
        z = fmaf(v.x, ww.x, z);
        z = fmaf(v.y, ww.y, z);
        z = fmaf(v.z, ww.z, z);
        z = fmaf(v.w, ww.w, z);
      }
      q_s[i] = z;
    }
  }
  __syncthreads();
  // solo: this warp's share of the sort source's gradient, sum_seg v S_d[key]
  double gd[FW_SOLO_PITCH / 32] = {0.0, 0.0};
  int ln = 0;   // records pending in rec[]
  auto solo_flush = [&]() {
    __syncwarp();
    for (int e = 0; e < ln; e++) {
      const SoloRec rr = rec[e];
      if (s0_smem) {
        const float* sr = S0_s + (rr.key - k_lo) * a.pitch0;
#pragma unroll
        for (int m = 0; m < FW_SOLO_PITCH / 32; m++) {
          const int c = lane + 32 * m;
          if (c < a.pitch0) gd[m] += (double)rr.v * (double)sr[c];
        }
      } else {
        const float* sr = a.S0 + (int64_t)rr.key * a.pitch0;
#pragma unroll
        for (int m = 0; m < FW_SOLO_PITCH / 32; m++) {
          const int c = lane + 32 * m;
          if (c < a.pitch0) gd[m] += (double)rr.v * (double)__ldg(sr + c);
        }
      }
    }
    __syncwarp();
    ln = 0;
  };
  float4 w[W_REG ? C4 : 1];
  if (W_REG) {
#pragma unroll
    for (int j = 0; j < C4; j++) w[j] = w_s[j];
  }

  // the warp's first segment may have begun before W0
  int head_key = -1;
  if (has_sort && cnt > 0 && W0 > 0 && W0 < a.r_T) {
    int k0 = fks[W0];
    if (k0 >= 0 && fks[W0 - 1] == k0) head_key = k0;
  }
  if (a.solo) head_key = -1;   // linear: a partial first segment is emitted as is
  bool head_open = head_key >= 0;
  float head_val = 0.f;
  int ck = -1;          // running segment key (warp uniform)
  float cv = 0.f;       // running segment partial

  float4 acc[C4];
#pragma unroll
  for (int j = 0; j < C4; j++) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
  float lacc = 0.f;

  auto flush = [&]() {
#pragma unroll
    for (int j = 0; j < C4; j++) {
      float v4[4] = {acc[j].x, acc[j].y, acc[j].z, acc[j].w};
#pragma unroll
      for (int c = 0; c < 4; c++) {
        float v = v4[c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) gsum[warp][j * 4 + c] += (double)v;
      }
      acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float v = lacc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) lsum[warp] += (double)v;
    lacc = 0.f;
  };

  int s = 0;            // stage slot and its mbarrier phase
  uint32_t ph = 0;
  for (int64_t i = 0; i < cnt; i++, s = (s + 1 == a.nst) ? 0 : s + 1, ph ^= (s == 0)) {
    mbar_wait(&wbar[s], ph);
    const char* st = wsm + (size_t)s * a.stage_bytes;
    const float4* Ft = reinterpret_cast<const float4*>(st);
    const int64_t unit_row0 = (u0 + i) * RW;
#pragma unroll
    for (int h = 0; h < RPL; h++) {
      const int lr = h * 32 + lane;
      const int64_t p = unit_row0 + lr;
      const bool valid = p < a.r_T;
      int key = has_sort ? reinterpret_cast<const int32_t*>(st + a.off_fk)[lr] : -1;
      // issue the gathers first so their latency overlaps the dot product
      float gq = 0.f;
      for (int d = 0; d < a.ng; d++) {
        int32_t fk = (d == a.sort_g) ? key : a.fk[d][p];
        if (fk >= 0) gq += (a.solo && d == a.sort_g) ? q_s[fk - k_lo] : __ldg(a.q[d] + fk);
      }
      float4 x[C4];
#pragma unroll
      for (int j = 0; j < C4; j++) x[j] = Ft[lr * C4 + j];
      float z0 = 0.f, z1 = 0.f;
#pragma unroll
      for (int j = 0; j < C4; j++) {
        float4 wj = W_REG ? w[j] : w_s[j];
        z0 = fmaf(x[j].x, wj.x, z0);
        z1 = fmaf(x[j].y, wj.y, z1);
        z0 = fmaf(x[j].z, wj.z, z0);
        z1 = fmaf(x[j].w, wj.w, z1);
      }
      float z = z0 + z1 + gq;
      float r, l;
      if (MODEL == 0) {
        float yv = reinterpret_cast<const float*>(st + a.off_y)[lr];
        r = z - yv;
        l = 0.5f * r * r;
      } else {
        float yv = (float)reinterpret_cast<const uint8_t*>(st + a.off_y)[lr];
        float e = __expf(-fabsf(z));                 // in (0, 1]
        float sp = log1pf(e);                        // softplus(-|z|)
        const float inv = __frcp_rn(1.f + e);         // 1 + e in [1, 2]: no slow path
        float pr = z >= 0.f ? inv : e * inv;
        r = pr - yv;
        // -log(p) = softplus(-z), -log(1-p) = softplus(z); clip at 1e-12
        float lp = z >= 0.f ? sp : sp - z;           // softplus(-z)
        float lq = z >= 0.f ? sp + z : sp;           // softplus(z)
        l = yv != 0.f ? fminf(lp, kLogClip) : fminf(lq, kLogClip);
      }
      if (!valid) {
        r = 0.f;
        l = 0.f;
        key = -1;
      }
      lacc += l;
#pragma unroll
      for (int j = 0; j < C4; j++) {
        acc[j].x = fmaf(r, x[j].x, acc[j].x);
        acc[j].y = fmaf(r, x[j].y, acc[j].y);
        acc[j].z = fmaf(r, x[j].z, acc[j].z);
        acc[j].w = fmaf(r, x[j].w, acc[j].w);
      }
      if (a.resid) a.resid[p] = r;
      if (has_sort) {
        // segmented inclusive scan over the 32 rows of this sub-tile
        float v = r;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          float vu = __shfl_up_sync(0xffffffffu, v, off);
          int ku = __shfl_up_sync(0xffffffffu, key, off);
          if (lane >= off && ku == key) v += vu;
        }
        // rows continuing the running segment (keys are non-decreasing)
        if (key >= 0 && key == ck) v += cv;
        const int k0 = __shfl_sync(0xffffffffu, key, 0);
        const int kn = __shfl_down_sync(0xffffffffu, key, 1);
        const bool end = lane < 31 && key >= 0 && kn != key;
        if (a.solo) {
          // completed segments -> records (fixed order: running one first,
          // then by lane); flushed into the gradient when the list fills
          const bool run_done = ck >= 0 && k0 != ck;
          const unsigned em = __ballot_sync(0xffffffffu, end);
          const int m = __popc(em) + (run_done ? 1 : 0);
          if (ln + m > FW_LCAP) solo_flush();
          if (run_done && lane == 0) rec[ln] = SoloRec{ck, cv};
          if (end) rec[ln + (run_done ? 1 : 0) + __popc(em & ((1u << lane) - 1u))] = SoloRec{key, v};
          ln += m;
        } else {
          if (ck >= 0 && k0 != ck) {              // running segment is complete
            if (head_open && ck == head_key) {
              head_val = cv;
              head_open = false;
            } else if (lane == 0) {
              a.bins[ck] = cv;
            }
          }
          const bool eh = end && head_open && key == head_key;
          const unsigned bm = __ballot_sync(0xffffffffu, eh);
          if (bm) {
            head_val = __shfl_sync(0xffffffffu, v, __ffs(bm) - 1);
            head_open = false;
          }
          if (end && !eh) a.bins[key] = v;
        }
        ck = __shfl_sync(0xffffffffu, key, 31);
        cv = __shfl_sync(0xffffffffu, v, 31);
      }
    }
    __syncwarp();
    if (i + a.nst < cnt && tc::elect_one()) {   // converged warp: no per-instruction ELECT loop
      fence_proxy_async();
      issue(s, u0 + i + a.nst);
    }
    if ((i % FW_FLUSH) == FW_FLUSH - 1) flush();
  }
  flush();

  // solo: the running segment is emitted as is; the warp's gradient share
  // goes to shared memory for the CTA's fixed-order sum
  if (a.solo) {
    if (ck >= 0) {
      if (ln + 1 > FW_LCAP) solo_flush();
      if (lane == 0) rec[ln] = SoloRec{ck, cv};
      ln += 1;
    }
    solo_flush();
  }
  // warp range end: running segment -> carry record
  if (has_sort && !a.solo) {
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
  // CTA partials in fixed warp order
  double* out = a.part + (int64_t)blockIdx.x * (C4 * 4 + 1);
  for (int t = threadIdx.x; t <= C4 * 4; t += blockDim.x) {
    double sum = 0.0;
    if (t < C4 * 4)
      for (int w2 = 0; w2 < FW_WARPS; w2++) sum += gsum[w2][t];
    else
      for (int w2 = 0; w2 < FW_WARPS; w2++) sum += lsum[w2];
    out[t] = sum;
  }
  if (a.solo) {
    double* gsd = gsd_all;   // past all lists
#pragma unroll
    for (int m = 0; m < FW_SOLO_PITCH / 32; m++) {
      const int c = lane + 32 * m;
      if (c < a.pitch0) gsd[warp * FW_SOLO_PITCH + c] = gd[m];
    }
    __syncthreads();
    for (int c = threadIdx.x; c < a.pitch0; c += blockDim.x) {
      double sum = 0.0;
      for (int w2 = 0; w2 < FW_WARPS; w2++) sum += gsd[w2 * FW_SOLO_PITCH + c];
      a.part_d[(int64_t)blockIdx.x * a.pitch0 + c] = sum;
    }
  }
  // solo: release / acquire arrivals instead of __threadfence (MEMBAR.SC.GPU
  // + L1 invalidate, ~1 us each on the two-die B200, three of them on the
  // critical path of the tail): the CTA's partial stores are ordered before
  // thread 0's release by the barrier, the last arriver's acquire before its
  // CTA's reads by the barrier after it, and the reads go to L2 (__ldcg).
  // FL_GLM_SOLO_DIAG bit 128 restores the fences (A/B).
  const bool sc = !a.solo || (a.diag & 128);
  if (sc) __threadfence();
  __syncthreads();
  if (a.solo && (a.diag & 1)) return;   // timing experiment only: no tail (wrong results)
  if (a.solo) {
    // two-level fixed-order reduction: the last CTA of each group of
    // FW_GROUP CTAs sums the group's partials, the last group the groups'
    // (a short, parallel tail instead of one CTA reducing every partial)
    const int pf = C4 * 4, ne = pf + 1 + a.pitch0;
    const int g = blockIdx.x / FW_GROUP, g0 = g * FW_GROUP;
    const int g1 = min((int)gridDim.x, g0 + FW_GROUP);
    const int ngroups = (gridDim.x + FW_GROUP - 1) / FW_GROUP;
    if (threadIdx.x == 0) is_last = atomic_add_acq_rel_gpu(&a.gcnt[g], 1) == g1 - g0 - 1;
    __syncthreads();
    if (!is_last) return;
    if (sc) __threadfence();
    for (int e = threadIdx.x; e < ne; e += blockDim.x) {
      double sum = 0.0;
      for (int b = g0; b < g1; b++)
        sum += e <= pf ? __ldcg(a.part + (int64_t)b * (pf + 1) + e)
                       : __ldcg(a.part_d + (int64_t)b * a.pitch0 + (e - pf - 1));
      a.gpart[(int64_t)g * ne + e] = sum;
    }
    if (threadIdx.x == 0) a.gcnt[g] = 0;
    if (sc) __threadfence();
    __syncthreads();
    if (a.diag & 2) return;   // timing experiment only: no final level
    if (threadIdx.x == 0) is_last = atomic_add_acq_rel_gpu(&a.state->done_fact, 1) == ngroups - 1;
    __syncthreads();
    if (!is_last) return;
    if (sc) __threadfence();
    if (a.diag & 16) return;   // timing experiment only: the final CTA does nothing
    glm_solo_final(a.gpart, ngroups, pf, a.pitch0, a.sort_g, (a.diag & 4) ? 0 : a.fuse_update, a.up,
                   (a.diag & 64) ? 2 : (a.diag & 32) ? 1 : 0);
    if (threadIdx.x == 0) a.state->done_fact = 0;
    return;
  }
  // last CTA stitches the segments that span warp ranges (fixed order)
  if (threadIdx.x == 0) is_last = atomicAdd(&a.state->done_fact, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  if (has_sort)
    stitch_carries(a.carry, NW, a.bins, smem, (size_t)FW_WARPS * a.nst * a.stage_bytes);
  if (threadIdx.x == 0) a.state->done_fact = 0;
}
