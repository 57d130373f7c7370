// Table lifecycle, device layout derivation, selectors, materialize and
// elementwise.  Reference: metadata.py:124-225 (FactorizedTable, materialize),
// ops.py:55-74 (_build_selectors), ops.py:273-295 (elementwise).
#include <cub/cub.cuh>

#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <algorithm>

#include "internal.h"

namespace flb {

static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

cudaError_t raise_smem_limit_ptr(const void* fn, int bytes) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<int, const void*>, int>> set;   // (device, kernel) -> bytes
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  for (auto& kv : set)
    if (kv.first.first == dev && kv.first.second == fn) {
      if (bytes <= kv.second) return cudaSuccess;
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      if (e == cudaSuccess) kv.second = bytes;
      return e;
    }
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) set.push_back({{dev, fn}, bytes});
  return e;
}

// pinned two-buffer staging ring shared by d2h_copy / h2d_copy (one per
// process, serialised by g_ring_mu: concurrent callers take turns)
static constexpr size_t kChunk = (size_t)64 << 20;
static std::mutex g_ring_mu;
static int staging_ring(char*** ring_out, cudaEvent_t** ev_out) {
  static char* ring[2] = {nullptr, nullptr};
  static cudaEvent_t ev[2];
  if (!ring[0]) {
    for (int i = 0; i < 2; i++) {
      FL_CUDA(cudaHostAlloc((void**)&ring[i], kChunk, cudaHostAllocPortable));
      FL_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    }
  }
  *ring_out = ring;
  *ev_out = ev;
  return FL_OK;
}
static void host_copy(char* d, const char* from, size_t n) {   // 8-thread memcpy
  const unsigned nthr = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  const size_t per = (n + nthr - 1) / nthr;
  for (unsigned k = 0; k < nthr; k++) {
    const size_t o = k * per;
    if (o >= n) break;
    th.emplace_back([=] { std::memcpy(d + o, from + o, std::min(per, n - o)); });
  }
  for (auto& x : th) x.join();
}
static bool staged_host(const void* host, size_t bytes) {
  cudaPointerAttributes pa{};
  const bool pageable = cudaPointerGetAttributes(&pa, host) == cudaSuccess &&
                        pa.type == cudaMemoryTypeUnregistered;
  (void)cudaGetLastError();
  return pageable && bytes >= 2 * kChunk && !std::getenv("FL_NO_STAGED_COPY");
}

int h2d_copy(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (!staged_host(src, bytes)) {
    FL_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s));
    FL_CUDA(cudaStreamSynchronize(s));
    return FL_OK;
  }
  std::lock_guard<std::mutex> lk(g_ring_mu);
  char** ring;
  cudaEvent_t* ev;
  if (int rc = staging_ring(&ring, &ev)) return rc;
  const size_t nch = (bytes + kChunk - 1) / kChunk;
  const char* sp = static_cast<const char*>(src);
  char* dp = static_cast<char*>(dst);
  for (size_t i = 0; i < nch; i++) {
    const size_t n = std::min(kChunk, bytes - i * kChunk);
    if (i >= 2) FL_CUDA(cudaEventSynchronize(ev[i & 1]));   // the DMA of chunk i - 2 is done
    host_copy(ring[i & 1], sp + i * kChunk, n);
    FL_CUDA(cudaMemcpyAsync(dp + i * kChunk, ring[i & 1], n, cudaMemcpyHostToDevice, s));
    FL_CUDA(cudaEventRecord(ev[i & 1], s));
  }
  FL_CUDA(cudaStreamSynchronize(s));
  return FL_OK;
}

int d2h_copy(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (!staged_host(dst, bytes)) {
    FL_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s));
    FL_CUDA(cudaStreamSynchronize(s));
    return FL_OK;
  }
  std::lock_guard<std::mutex> lk(g_ring_mu);
  char** ring;
  cudaEvent_t* ev;
  if (int rc = staging_ring(&ring, &ev)) return rc;
  const size_t nch = (bytes + kChunk - 1) / kChunk;
  const char* sp = static_cast<const char*>(src);
  char* dp = static_cast<char*>(dst);
  for (size_t i = 0; i <= nch; i++) {
    if (i < nch) {   // issue chunk i (its buffer was drained in iteration i - 1)
      const size_t n = std::min(kChunk, bytes - i * kChunk);
      FL_CUDA(cudaMemcpyAsync(ring[i & 1], sp + i * kChunk, n, cudaMemcpyDeviceToHost, s));
      FL_CUDA(cudaEventRecord(ev[i & 1], s));
    }
    if (i > 0) {     // drain chunk i - 1 while chunk i is in flight
      const size_t j = i - 1, n = std::min(kChunk, bytes - j * kChunk);
      FL_CUDA(cudaEventSynchronize(ev[j & 1]));
      host_copy(dp + j * kChunk, ring[j & 1], n);
    }
  }
  return FL_OK;
}

int cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
  set_error("CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e), cudaGetErrorString(e),
            what, file, line);
  return FL_ERR_CUDA;
}

DevBuf::~DevBuf() {
  if (p) {
    if (pooled)
      cudaFreeAsync(p, astream);
    else
      cudaFree(p);
  }
}

// per-device pool for upload temporaries; up to 8 GB stays cached between
// tables (the C2 upload needs ~3 GB of them)
static cudaMemPool_t tmp_pool(int device) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (device < 0 || device >= 64) return nullptr;
  if (!pools[device]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    if (cudaMemPoolCreate(&pools[device], &props) != cudaSuccess) {
      cudaGetLastError();
      pools[device] = nullptr;
      return nullptr;
    }
    uint64_t thr = (uint64_t)8 << 30;
    cudaMemPoolSetAttribute(pools[device], cudaMemPoolAttrReleaseThreshold, &thr);
  }
  return pools[device];
}

// Operator temporaries come from the device's default pool
// (cudaMallocAsync).  Its default release threshold of 0 hands the memory
// back at every synchronization, so each operator call re-mapped its
// temporaries (a C2 crossprod spent ~4 ms of its 9.4 ms there); keep up to
// 32 GB cached instead.
static void keep_default_pool(int device) {
  static std::mutex mu;
  static bool done[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (device < 0 || device >= 64 || done[device]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = (uint64_t)32 << 30;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  cudaGetLastError();
  done[device] = true;
}

int DevBuf::alloc_tmp(size_t n, cudaStream_t st) {
  int dev = 0;
  FL_CUDA(cudaGetDevice(&dev));
  cudaMemPool_t pool = tmp_pool(dev);
  if (!pool) return alloc(n);
  if (p) {
    if (pooled)
      cudaFreeAsync(p, astream);
    else
      cudaFree(p);
    p = nullptr;
  }
  if (n == 0) n = 16;
  FL_CUDA(cudaMallocFromPoolAsync(&p, n, pool, st));
  bytes = n;
  astream = st;
  pooled = true;
  return FL_OK;
}

int DevBuf::alloc(size_t n) {
  if (p) {
    if (pooled)
      cudaFreeAsync(p, astream);
    else
      cudaFree(p);
    p = nullptr;
    bytes = 0;
    pooled = false;
  }
  if (n == 0) n = 16;
  FL_CUDA(cudaMalloc(&p, n));
  bytes = n;
  return FL_OK;
}

int Workspace::grow(DevBuf& buf, size_t n) {
  if (buf.bytes >= n && buf.p) return FL_OK;
  return buf.alloc(round_up((int64_t)n, 1 << 20));
}

int device_sm_count(int device) {
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 148;
  return n > 0 ? n : 148;
}

// device operands may still be in flight on the caller's streams: they are
// copied synchronously (as cudaMemcpy orders them); host buffers go async
static bool on_device_ptr(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

static std::shared_ptr<DevBuf> make_buf(size_t bytes, int* rc) {
  auto b = std::make_shared<DevBuf>();
  *rc = b->alloc(bytes);
  return b;
}

// temporary of the upload path (stream-ordered pool allocation on `st`)
static std::shared_ptr<DevBuf> make_tmp(size_t bytes, cudaStream_t st, int* rc) {
  auto b = std::make_shared<DevBuf>();
  *rc = b->alloc_tmp(bytes, st);
  return b;
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
__global__ void k_fanout(const int32_t* __restrict__ ind_sel, int64_t r_T, int32_t* cnt,
                         int64_t r_k, int32_t* bad) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= r_T) return;
  int32_t s = ind_sel[i];
  if (s >= 0) {
    if (s >= r_k) {
      atomicExch(bad, 1);
      return;
    }
    atomicAdd(&cnt[s], 1);
  }
}

__global__ void k_sort_keys(const int32_t* __restrict__ ind_sel, int64_t r_T, uint32_t* keys,
                            int32_t* vals) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= r_T) return;
  keys[i] = (uint32_t)(ind_sel[i] + 1);  // -1 sorts first
  vals[i] = (int32_t)i;
}

__global__ void k_iota_perm(int32_t* perm, int64_t r_T, int64_t r_pad) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= r_pad) return;
  perm[i] = i < r_T ? (int32_t)i : -1;
}

__global__ void k_pad_perm(int32_t* perm, int64_t r_T, int64_t r_pad) {
  int64_t i = r_T + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < r_pad) perm[i] = -1;
}

__global__ void k_inverse_perm(const int32_t* __restrict__ perm, int64_t r_T, int32_t* iperm) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= r_T) return;
  iperm[perm[p]] = (int32_t)p;
}

// F[p, off + c] = vals[ind_sel[perm[p]], c] (0 when unmatched / padding)
__global__ void k_build_stream(const float* __restrict__ vals, int cols,
                               const int32_t* __restrict__ ind_sel,
                               const int32_t* __restrict__ perm, int64_t r_pad, float* F,
                               int pf, int off) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t total = r_pad * cols;
  if (idx >= total) return;
  int64_t p = idx / cols;
  int c = (int)(idx - p * cols);
  int32_t t = perm[p];
  float v = 0.f;
  if (t >= 0) {
    int32_t s = ind_sel[t];
    if (s >= 0) v = vals[(int64_t)s * cols + c];
  }
  F[p * pf + off + c] = v;
}

// float4 form of k_build_stream (cols % 4 == 0, off % 4 == 0): thread per
// (device row, quad) -- coalesced stores, each source row read as whole
// 16-byte quads by consecutive threads
__global__ void k_build_stream4(const float4* __restrict__ vals, int c4,
                                const int32_t* __restrict__ ind_sel,
                                const int32_t* __restrict__ perm, int64_t r_pad,
                                float4* __restrict__ F, int pf4, int off4) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= r_pad * c4) return;
  const int64_t p = idx / c4;
  const int q = (int)(idx - p * c4);
  const int32_t t = perm[p];
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (t >= 0) {
    const int32_t s = ind_sel[t];
    if (s >= 0) v = vals[(int64_t)s * c4 + q];
  }
  F[p * pf4 + off4 + q] = v;
}

// host-value upload, one ring chunk: source rows [r0, r0 + nrows) of an
// injective source land at their device rows.  inv (source row -> target row,
// -1 = unreferenced) is null for the identity indicator.
__global__ void k_scatter_rows(const float* __restrict__ chunk, int cols, int64_t r0,
                               int64_t nrows, const int32_t* __restrict__ inv,
                               const int32_t* __restrict__ iperm, float* __restrict__ F, int pf,
                               int off) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= nrows * cols) return;
  int64_t row = idx / cols;
  int c = (int)(idx - row * cols);
  int64_t src = r0 + row;
  int64_t tr = inv ? (int64_t)inv[src] : src;
  if (tr < 0) return;
  F[(int64_t)iperm[tr] * pf + off + c] = chunk[idx];
}

// inv[ind_sel[t]] = t for an injective indicator (inv preset to -1)
__global__ void k_invert_sel(const int32_t* __restrict__ ind_sel, int64_t r_T, int32_t* inv) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= r_T) return;
  int32_t s = ind_sel[t];
  if (s >= 0) inv[s] = (int32_t)t;
}

__global__ void k_fk_device_order(const int32_t* __restrict__ ind_sel,
                                  const int32_t* __restrict__ perm, int64_t r_pad, int32_t* fk) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= r_pad) return;
  int32_t t = perm[p];
  fk[p] = t >= 0 ? ind_sel[t] : -1;
}

// grp_rows[m] = iperm[order[n_neg + m]]
__global__ void k_group_rows(const int32_t* __restrict__ order, int64_t n_neg, int64_t matched,
                             const int32_t* __restrict__ iperm, int32_t* grp_rows) {
  int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= matched) return;
  grp_rows[m] = iperm[order[n_neg + m]];
}

__global__ void k_cnt_to_i64(const int32_t* __restrict__ cnt, int64_t n, int64_t* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > n) return;
  out[i] = i < n ? (int64_t)cnt[i] : 0;
}

// column descriptor for materialize / crossprod: kind 0 = unmapped,
// 1 = F column (a = column), 2 = gather (a = gather idx, b = column)
struct ColDesc {
  int kind, a, b, pad;
};

struct GatherView {
  const float* S;
  const int32_t* fk;
  int pitch;
};

__global__ void k_materialize(const float* __restrict__ F, int pf, const ColDesc* __restrict__ cd,
                              const GatherView* __restrict__ gv,
                              const int32_t* __restrict__ perm, int64_t r_T, int c_T,
                              float* __restrict__ out) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= r_T * c_T) return;
  int64_t p = idx / c_T;
  int t = (int)(idx - p * c_T);
  ColDesc d = cd[t];
  float v = 0.f;
  if (d.kind == 1) {
    v = F[p * pf + d.a];
  } else if (d.kind == 2) {
    GatherView g = gv[d.a];
    int32_t fk = g.fk[p];
    if (fk >= 0) v = g.S[(int64_t)fk * g.pitch + d.b];
  }
  out[(int64_t)perm[p] * c_T + t] = v;
}

__global__ void k_elementwise(float* __restrict__ a, const float* __restrict__ src, int64_t n,
                              int func, double scalar) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = (double)src[i];
  double r;
  switch (func) {
    case FL_EW_SCALE: r = v * scalar; break;
    case FL_EW_DIVIDE: r = v / scalar; break;
    case FL_EW_SQUARE: r = v * v; break;
    case FL_EW_ABS: r = fabs(v); break;
    case FL_EW_EXPM1: r = expm1(v); break;
    default: r = 1.0 / (1.0 + exp(-v)) - 0.5; break;
  }
  a[i] = (float)r;
}

__global__ void k_ind_from_fk(const int32_t* __restrict__ fk, const int32_t* __restrict__ perm,
                              int64_t r_T, int32_t* ind_sel) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= r_T) return;
  ind_sel[perm[p]] = fk[p];
}

__global__ void k_sorted_group_rows(const int32_t* __restrict__ perm, int64_t n_neg,
                                    int64_t matched, int32_t* out) {
  int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= matched) return;
  out[m] = perm[n_neg + m];
}

__global__ void k_map_rows(const int32_t* __restrict__ grp_rows, const int32_t* __restrict__ perm,
                           int64_t matched, int32_t* out) {
  int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= matched) return;
  out[m] = perm[grp_rows[m]];
}

static inline unsigned grid_for(int64_t n, int block = 256) {
  return (unsigned)ceil_div(n, block);
}

// stable (key = ind_sel + 1, value = target row) sort over target rows
// `keep` (optional) receives the temporaries instead of freeing them here:
// cudaFree waits for the whole device, which would stall behind the upload's
// in-flight copies
static int stable_order(const int32_t* ind_sel, int64_t r_T, int64_t r_k, int32_t* order_out,
                        cudaStream_t s, std::vector<std::shared_ptr<DevBuf>>* keep = nullptr) {
  int rc;
  auto keys = make_tmp(r_T * 4, s, &rc);
  if (rc) return rc;
  auto keys2 = make_tmp(r_T * 4, s, &rc);
  if (rc) return rc;
  auto vals = make_tmp(r_T * 4, s, &rc);
  if (rc) return rc;
  k_sort_keys<<<grid_for(r_T), 256, 0, s>>>(ind_sel, r_T, keys->as<uint32_t>(),
                                            vals->as<int32_t>());
  FL_CHECK_LAUNCH();
  int end_bit = 1;
  while (end_bit < 32 && ((uint64_t)1 << end_bit) <= (uint64_t)(r_k + 1)) end_bit++;
  size_t tmp_bytes = 0;
  FL_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys->as<uint32_t>(),
                                          keys2->as<uint32_t>(), vals->as<int32_t>(), order_out,
                                          (int)r_T, 0, end_bit, s));
  auto tmp = make_tmp(tmp_bytes, s, &rc);
  if (rc) return rc;
  FL_CUDA(cub::DeviceRadixSort::SortPairs(tmp->p, tmp_bytes, keys->as<uint32_t>(),
                                          keys2->as<uint32_t>(), vals->as<int32_t>(), order_out,
                                          (int)r_T, 0, end_bit, s));
  FL_CUDA(cudaStreamSynchronize(s));
  if (keep) keep->insert(keep->end(), {keys, keys2, vals, tmp});
  return FL_OK;
}

int table_upload_tcols(fl_table* t) {
  int rc;
  if (t->pf > 0) {
    t->d_f_tcol = make_buf(t->pf * 4, &rc);
    if (rc) return rc;
    FL_CUDA(cudaMemcpy(t->d_f_tcol->p, t->f_tcol.data(), t->pf * 4, cudaMemcpyHostToDevice));
  }
  for (auto& g : t->g) {
    g.d_tcol = make_buf(g.pitch * 4, &rc);
    if (rc) return rc;
    FL_CUDA(cudaMemcpy(g.d_tcol->p, g.tcol.data(), g.pitch * 4, cudaMemcpyHostToDevice));
  }
  return FL_OK;
}

int launch_gather_rows_to_device_order(const fl_table* t, const void* src_target, void* dst_dev,
                                       int elem_bytes, cudaStream_t s);

}  // namespace flb

using namespace flb;

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

const char* fl_last_error(void) { return flb::g_last_error.c_str(); }

int fl_version(void) { return 1; }

int fl_device_info(int device, int* sm_count, int64_t* l2_bytes, int* cc_major, int* cc_minor) {
  int v = 0;
  FL_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
  if (sm_count) *sm_count = v;
  FL_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, device));
  if (l2_bytes) *l2_bytes = v;
  FL_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMajor, device));
  if (cc_major) *cc_major = v;
  FL_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMinor, device));
  if (cc_minor) *cc_minor = v;
  return FL_OK;
}

int fl_table_create(int device, int64_t r_T, int32_t c_T, fl_table** out) {
  if (!out || r_T < 1 || c_T < 1 || r_T >= (int64_t)INT32_MAX - 2 * TILE) {
    set_error("fl_table_create: invalid shape %lld x %d", (long long)r_T, c_T);
    return FL_ERR_ARG;
  }
  FL_CUDA(cudaSetDevice(device));
  keep_default_pool(device);
  auto* t = new fl_table();
  t->device = device;
  t->sm_count = device_sm_count(device);
  t->r_T = r_T;
  t->c_T = c_T;
  t->r_pad = round_up(r_T, TILE);
  *out = t;
  return FL_OK;
}

int fl_table_add_source(fl_table* t, int64_t r_k, int32_t c_k, const float* values,
                        const int32_t* ind_sel, const int32_t* col_map) {
  if (!t || t->finalized) {
    set_error("fl_table_add_source: table is finalized or null");
    return FL_ERR_ARG;
  }
  if (r_k < 1 || c_k < 1 || !values || !col_map || (!ind_sel && r_k != t->r_T)) {
    set_error("fl_table_add_source: invalid source %lld x %d", (long long)r_k, c_k);
    return FL_ERR_ARG;
  }
  const PhaseTrace tr("fl_table_add_source");
  FL_CUDA(cudaSetDevice(t->device));
  Staged st;
  st.rows = r_k;
  st.cols = c_k;
  st.col_map.assign(col_map, col_map + c_k);
  for (int c = 0; c < c_k; c++) {
    if (st.col_map[c] < 0 || st.col_map[c] >= t->c_T) {
      set_error("source %zu column %d maps to target column %d outside [0,%d)", t->staged.size(),
                c, st.col_map[c], t->c_T);
      return FL_ERR_METADATA;
    }
  }
  int rc;
  // asynchronous uploads on the table's copy streams (values and FKs on
  // separate streams, so the FKs land early and finalize's index work
  // overlaps the large value copies); the caller keeps `values` / `ind_sel`
  // valid until fl_table_finalize returns
  auto mk_stream = []() -> std::shared_ptr<void> {
    cudaStream_t cs = nullptr;
    if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    return std::shared_ptr<void>(cs, [](void* p) { cudaStreamDestroy((cudaStream_t)p); });
  };
  auto mk_event = []() -> std::shared_ptr<void> {
    cudaEvent_t e = nullptr;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    return std::shared_ptr<void>(e, [](void* p) { cudaEventDestroy((cudaEvent_t)p); });
  };
  if (!t->cp_vals) t->cp_vals = mk_stream();
  if (!t->cp_idx) t->cp_idx = mk_stream();
  st.ev_vals = mk_event();
  st.ev_idx = mk_event();
  if (!t->cp_vals || !t->cp_idx || !st.ev_vals || !st.ev_idx) {
    set_error("fl_table_add_source: stream / event creation failed");
    return FL_ERR_CUDA;
  }
  cudaStream_t cv = (cudaStream_t)t->cp_vals.get(), ci = (cudaStream_t)t->cp_idx.get();
  // the target-order indicator is an upload temporary (finalize derives the
  // device-order FKs from it); a device operand is copied synchronously, so
  // its buffer comes from the plain allocator
  st.sel_given = ind_sel != nullptr;
  if (ind_sel && on_device_ptr(ind_sel))
    st.ind_sel = make_buf((size_t)t->r_T * 4, &rc);
  else
    st.ind_sel = make_tmp((size_t)t->r_T * 4, ci, &rc);
  if (rc) return rc;
  // device operands may still be in flight on the caller's streams: copy
  // them synchronously (as cudaMemcpy orders them); host buffers go async
  if (ind_sel) {
    if (on_device_ptr(ind_sel))
      FL_CUDA(cudaMemcpy(st.ind_sel->p, ind_sel, (size_t)t->r_T * 4, cudaMemcpyDefault));
    else
      FL_CUDA(cudaMemcpyAsync(st.ind_sel->p, ind_sel, (size_t)t->r_T * 4, cudaMemcpyDefault, ci));
  } else {  // identity indicator (the fact table of a star schema)
    k_iota_perm<<<grid_for(t->r_T), 256, 0, ci>>>(st.ind_sel->as<int32_t>(), t->r_T, t->r_T);
    FL_CHECK_LAUNCH();
  }
  FL_CUDA(cudaEventRecord((cudaEvent_t)st.ev_idx.get(), ci));
  if (on_device_ptr(values)) {
    st.vals = make_buf((size_t)r_k * c_k * 4, &rc);
    if (rc) return rc;
    FL_CUDA(cudaMemcpy(st.vals->p, values, (size_t)r_k * c_k * 4, cudaMemcpyDefault));
  } else {
    // host values are not staged: finalize copies them once it knows where
    // they go (chunks through a small ring into the stream block, or straight
    // into the pitched S_d), so PCIe carries every byte exactly once and the
    // device-order scatter overlaps the copy
    st.h_vals = values;
  }
  FL_CUDA(cudaEventRecord((cudaEvent_t)st.ev_vals.get(), cv));
  t->staged.push_back(std::move(st));
  tr.mark("issued");
  return FL_OK;
}

int fl_table_finalize(fl_table* t, void* stream) {
  if (!t || t->finalized || t->staged.empty()) {
    set_error("fl_table_finalize: nothing to finalize");
    return FL_ERR_ARG;
  }
  const PhaseTrace tr("fl_table_finalize");
  auto mark = [&](const char* what) { tr.mark(what); };
  FL_CUDA(cudaSetDevice(t->device));
  // every return path (errors included) waits for the host-side copies (FKs
  // from add_source, values from here): the caller may release its host
  // arrays as soon as finalize returns
  struct CopyDrain {
    cudaStream_t a, b;
    ~CopyDrain() {
      if (a) cudaStreamSynchronize(a);
      if (b) cudaStreamSynchronize(b);
    }
  } drain{(cudaStream_t)t->cp_idx.get(), (cudaStream_t)t->cp_vals.get()};
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t r_T = t->r_T, r_pad = t->r_pad;
  int rc;
  const int n = (int)t->staged.size();
  // temporaries live until the end: no cudaFree (a device-wide wait) while
  // the value copies are in flight
  std::vector<std::shared_ptr<DevBuf>> keep;
  // the index work below needs every FK array; the values are waited for
  // just before their first use (stream block / gathered copies)
  for (auto& st : t->staged) FL_CUDA(cudaStreamWaitEvent(s, (cudaEvent_t)st.ev_idx.get(), 0));
  // column disjointness (metadata.py:196-206)
  std::vector<int> owner(t->c_T, -1);
  for (int k = 0; k < n; k++)
    for (int c : t->staged[k].col_map) {
      if (owner[c] >= 0) {
        set_error("[source %d] column claimed twice: target column %d already claimed by source %d",
                  k, c, owner[c]);
        return FL_ERR_METADATA;
      }
      owner[c] = k;
    }
  // 0. host values of stream sources travel in chunks through a small device
  // ring and are scattered to their device rows once the row order exists.
  // Identity-indicator sources are streamed for certain, so their chunks
  // start right away, overlapping the fanout analysis and the sort below.
  cudaStream_t cv = (cudaStream_t)t->cp_vals.get();
  struct Chunk {
    int k;
    int64_t r0, nrows;
  };
  std::vector<Chunk> chunks;
  size_t kChunkBytes = (size_t)64 << 20;
  if (const char* e = std::getenv("FL_UPLOAD_CHUNK_BYTES"))   // tests: force many ring wraps
    kChunkBytes = std::max<size_t>(16, (size_t)std::atoll(e));
  size_t slot_bytes = kChunkBytes;
  int64_t chunks_upper = 0;   // chunks if every host source turned out injective
  for (int k = 0; k < n; k++) {
    const Staged& st = t->staged[k];
    if (!st.h_vals) continue;
    const size_t row_bytes = (size_t)st.cols * 4;
    slot_bytes = std::max(slot_bytes, row_bytes);
    chunks_upper += ceil_div(st.rows, std::max<int64_t>(1, (int64_t)(kChunkBytes / row_bytes)));
  }
  // <= 16 slots (1 GB): covers the FK sort.  Sized for the worst case when
  // identity sources start early, else once the classification is known.
  int ring_n = 0;
  std::shared_ptr<DevBuf> ring;
  auto make_ring = [&](int64_t nchunks) -> int {
    ring_n = (int)std::min<int64_t>(nchunks, 16);
    if (ring_n <= 0) return FL_OK;
    int rc2;
    ring = make_tmp(slot_bytes * ring_n, cv, &rc2);
    return rc2;
  };
  std::vector<std::shared_ptr<void>> ev_ready, ev_free;
  auto mk_ev = []() -> std::shared_ptr<void> {
    cudaEvent_t e = nullptr;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    return std::shared_ptr<void>(e, [](void* p) { cudaEventDestroy((cudaEvent_t)p); });
  };
  auto add_chunks = [&](int k) {
    const Staged& st = t->staged[k];
    const int64_t per = std::max<int64_t>(1, (int64_t)(kChunkBytes / ((size_t)st.cols * 4)));
    for (int64_t r0 = 0; r0 < st.rows; r0 += per) {
      chunks.push_back({k, r0, std::min(per, st.rows - r0)});
      ev_ready.push_back(mk_ev());
      ev_free.push_back(mk_ev());
    }
  };
  int nissued = 0;
  // pageable host values (a drop-in caller's numpy arrays) cross through the
  // pinned staging ring: an 8-thread memcpy into pinned buffer i & 1, then
  // the DMA (the driver's own pageable path is several times slower)
  std::unique_lock<std::mutex> pin_lock(g_ring_mu, std::defer_lock);
  char** pin_ring = nullptr;
  cudaEvent_t* pin_ev = nullptr;
  int npinned = 0;
  std::vector<char> pageable(n, 0);
  for (int k = 0; k < n; k++)
    pageable[k] = t->staged[k].h_vals &&
                  staged_host(t->staged[k].h_vals, (size_t)t->staged[k].rows * t->staged[k].cols * 4);
  auto issue_chunk = [&](int c) -> int {
    const Chunk& ch = chunks[c];
    const Staged& st = t->staged[ch.k];
    if (!ev_ready[c] || !ev_free[c]) {
      set_error("fl_table_finalize: event creation failed");
      return FL_ERR_CUDA;
    }
    char* slot = ring->as<char>() + (size_t)(c % ring_n) * slot_bytes;
    if (c >= ring_n) FL_CUDA(cudaStreamWaitEvent(cv, (cudaEvent_t)ev_free[c - ring_n].get(), 0));
    const size_t nb = (size_t)ch.nrows * st.cols * 4;
    if (pageable[ch.k] && nb <= kChunk) {
      if (!pin_lock.owns_lock()) {
        pin_lock.lock();
        if (int rc2 = staging_ring(&pin_ring, &pin_ev)) return rc2;
      }
      const int b = npinned & 1;
      if (npinned >= 2) FL_CUDA(cudaEventSynchronize(pin_ev[b]));   // its previous DMA is done
      host_copy(pin_ring[b], reinterpret_cast<const char*>(st.h_vals + ch.r0 * st.cols), nb);
      FL_CUDA(cudaMemcpyAsync(slot, pin_ring[b], nb, cudaMemcpyHostToDevice, cv));
      FL_CUDA(cudaEventRecord(pin_ev[b], cv));
      npinned++;
    } else {
      FL_CUDA(cudaMemcpyAsync(slot, st.h_vals + ch.r0 * st.cols, nb, cudaMemcpyHostToDevice, cv));
    }
    FL_CUDA(cudaEventRecord((cudaEvent_t)ev_ready[c].get(), cv));
    nissued = c + 1;
    return FL_OK;
  };
  for (int k = 0; k < n; k++)
    if (t->staged[k].h_vals && !t->staged[k].sel_given) add_chunks(k);
  if (!chunks.empty() && (rc = make_ring(chunks_upper))) return rc;
  for (int c = 0; c < std::min((int)chunks.size(), ring_n); c++)
    if ((rc = issue_chunk(c))) return rc;
  mark("first chunks issued");

  // 1. fanout histograms -> classification
  std::vector<std::shared_ptr<DevBuf>> cnts(n);
  std::vector<int> maxfan(n);
  std::vector<int64_t> matched(n);
  auto bad = make_buf(4, &rc);
  if (rc) return rc;
  for (int k = 0; k < n; k++) {
    Staged& st = t->staged[k];
    cnts[k] = make_tmp((st.rows + 1) * 4, s, &rc);
    if (rc) return rc;
    FL_CUDA(cudaMemsetAsync(cnts[k]->p, 0, (st.rows + 1) * 4, s));
    FL_CUDA(cudaMemsetAsync(bad->p, 0, 4, s));
    k_fanout<<<grid_for(r_T), 256, 0, s>>>(st.ind_sel->as<int32_t>(), r_T,
                                           cnts[k]->as<int32_t>(), st.rows, bad->as<int32_t>());
    FL_CHECK_LAUNCH();
    int h_bad = 0;
    FL_CUDA(cudaMemcpyAsync(&h_bad, bad->p, 4, cudaMemcpyDeviceToHost, s));
    // max + sum of fanout
    size_t tb = 0;
    auto dmax = make_tmp(16, s, &rc);
    if (rc) return rc;
    FL_CUDA(cub::DeviceReduce::Max(nullptr, tb, cnts[k]->as<int32_t>(), dmax->as<int32_t>(),
                                   (int)st.rows, s));
    auto tmp = make_tmp(tb, s, &rc);
    if (rc) return rc;
    FL_CUDA(cub::DeviceReduce::Max(tmp->p, tb, cnts[k]->as<int32_t>(), dmax->as<int32_t>(),
                                   (int)st.rows, s));
    int h_max = 0;
    FL_CUDA(cudaMemcpyAsync(&h_max, dmax->p, 4, cudaMemcpyDeviceToHost, s));
    FL_CUDA(cudaStreamSynchronize(s));
    keep.insert(keep.end(), {dmax, tmp});
    if (h_bad) {
      set_error("[source %d] indicator shape: row index outside [0,%lld)", k, (long long)st.rows);
      return FL_ERR_METADATA;
    }
    maxfan[k] = h_max;
  }
  mark("fanout (FKs landed)");
  t->src.assign(n, SrcInfo());
  int stream_cols = 0;
  int sort_k = -1;
  for (int k = 0; k < n; k++) {
    SrcInfo& si = t->src[k];
    si.rows = t->staged[k].rows;
    si.cols = t->staged[k].cols;
    si.stream = maxfan[k] <= 1;
    if (si.stream) {
      si.f_off = stream_cols;
      stream_cols += si.cols;
    } else if (sort_k < 0 || si.rows > t->staged[sort_k].rows) {
      sort_k = k;
    }
  }
  // 1b. stream block and the rest of the host values: remaining stream-source
  // chunks join the ring queue, gathered sources land directly in their
  // pitched S_d.  Every host byte crosses PCIe once, in one stream.
  t->nf = stream_cols;
  t->pf = pitch_for(std::max(stream_cols, 1));
  t->f_tcol.assign(t->pf, -1);
  t->F = make_buf((size_t)r_pad * t->pf * 4 + 64, &rc);
  if (rc) return rc;
  FL_CUDA(cudaMemsetAsync(t->F->p, 0, (size_t)r_pad * t->pf * 4, s));
  for (int k = 0; k < n; k++)
    if (t->src[k].stream && t->staged[k].h_vals && t->staged[k].sel_given) add_chunks(k);
  if (!ring && !chunks.empty() && (rc = make_ring((int64_t)chunks.size()))) return rc;
  for (int c = nissued; c < std::min((int)chunks.size(), ring_n); c++)
    if ((rc = issue_chunk(c))) return rc;
  const int nch = (int)chunks.size();
  // (a pitched H2D copy of short rows runs far below PCIe speed: the compact
  // rows cross as one contiguous copy and are re-pitched on the device)
  std::vector<std::shared_ptr<DevBuf>> host_S(n), host_tmp(n);
  for (int k = 0; k < n; k++) {
    const Staged& st = t->staged[k];
    if (t->src[k].stream || !st.h_vals) continue;
    const int pitch = pitch_for(st.cols);
    const int64_t rows_pad = round_up(st.rows, TILE);
    host_S[k] = make_buf((size_t)rows_pad * pitch * 4 + 64, &rc);
    if (rc) return rc;
    host_tmp[k] = make_tmp((size_t)st.rows * st.cols * 4, cv, &rc);
    if (rc) return rc;
    FL_CUDA(cudaMemcpyAsync(host_tmp[k]->p, st.h_vals, (size_t)st.rows * st.cols * 4,
                            cudaMemcpyHostToDevice, cv));
    FL_CUDA(cudaMemsetAsync(host_S[k]->p, 0, (size_t)rows_pad * pitch * 4, cv));
    FL_CUDA(cudaMemcpy2DAsync(host_S[k]->p, pitch * 4, host_tmp[k]->p, st.cols * 4, st.cols * 4,
                              st.rows, cudaMemcpyDeviceToDevice, cv));
  }

  mark("value copies issued");
  // 2. device row order
  t->perm = make_buf(r_pad * 4, &rc);
  if (rc) return rc;
  t->iperm = make_buf(r_T * 4, &rc);
  if (rc) return rc;
  std::vector<std::shared_ptr<DevBuf>> orders(n);
  if (sort_k >= 0) {
    orders[sort_k] = make_tmp(r_T * 4, s, &rc);
    if (rc) return rc;
    rc = stable_order(t->staged[sort_k].ind_sel->as<int32_t>(), r_T, t->staged[sort_k].rows,
                      orders[sort_k]->as<int32_t>(), s, &keep);
    if (rc) return rc;
    FL_CUDA(cudaMemcpyAsync(t->perm->p, orders[sort_k]->p, r_T * 4, cudaMemcpyDeviceToDevice, s));
    if (r_pad > r_T) k_pad_perm<<<grid_for(r_pad - r_T), 256, 0, s>>>(t->perm->as<int32_t>(), r_T, r_pad);
  } else {
    k_iota_perm<<<grid_for(r_pad), 256, 0, s>>>(t->perm->as<int32_t>(), r_T, r_pad);
  }
  FL_CHECK_LAUNCH();
  k_inverse_perm<<<grid_for(r_T), 256, 0, s>>>(t->perm->as<int32_t>(), r_T,
                                               t->iperm->as<int32_t>());
  FL_CHECK_LAUNCH();
  mark("row order (sorted)");
  // 3. stream block F.  Every table gets one; a table with no injective
  // source keeps a 4-column all-zero block so the fused passes have one
  // code path.  Device values: gathered into device order; host values:
  // each ring chunk scattered to its device rows as it lands.
  for (auto& st : t->staged) FL_CUDA(cudaStreamWaitEvent(s, (cudaEvent_t)st.ev_vals.get(), 0));
  std::vector<std::shared_ptr<DevBuf>> invs(n);
  for (int k = 0; k < n; k++) {
    if (!t->src[k].stream) continue;
    Staged& st = t->staged[k];
    for (int c = 0; c < st.cols; c++) t->f_tcol[t->src[k].f_off + c] = st.col_map[c];
    if (st.h_vals) {
      if (st.rows == r_T && !st.sel_given) continue;   // identity indicator
      invs[k] = make_tmp((size_t)st.rows * 4, s, &rc);
      if (rc) return rc;
      FL_CUDA(cudaMemsetAsync(invs[k]->p, 0xff, (size_t)st.rows * 4, s));
      k_invert_sel<<<grid_for(r_T), 256, 0, s>>>(st.ind_sel->as<int32_t>(), r_T,
                                                 invs[k]->as<int32_t>());
      FL_CHECK_LAUNCH();
      continue;
    }
    if (st.cols % 4 == 0 && t->src[k].f_off % 4 == 0) {
      const int c4 = st.cols / 4;
      k_build_stream4<<<grid_for(r_pad * c4), 256, 0, s>>>(
          reinterpret_cast<const float4*>(st.vals->p), c4, st.ind_sel->as<int32_t>(),
          t->perm->as<int32_t>(), r_pad, reinterpret_cast<float4*>(t->F->p), t->pf / 4,
          t->src[k].f_off / 4);
    } else {
      int64_t total = r_pad * st.cols;
      k_build_stream<<<grid_for(total), 256, 0, s>>>(st.vals->as<float>(), st.cols,
                                                     st.ind_sel->as<int32_t>(),
                                                     t->perm->as<int32_t>(), r_pad,
                                                     t->F->as<float>(), t->pf, t->src[k].f_off);
    }
    FL_CHECK_LAUNCH();
  }
  for (int c = 0; c < nch; c++) {
    const Chunk& ch = chunks[c];
    const Staged& st = t->staged[ch.k];
    FL_CUDA(cudaStreamWaitEvent(s, (cudaEvent_t)ev_ready[c].get(), 0));
    const float* slot = reinterpret_cast<const float*>(ring->as<char>() +
                                                       (size_t)(c % ring_n) * slot_bytes);
    k_scatter_rows<<<grid_for(ch.nrows * st.cols), 256, 0, s>>>(
        slot, st.cols, ch.r0, ch.nrows, invs[ch.k] ? invs[ch.k]->as<int32_t>() : nullptr,
        t->iperm->as<int32_t>(), t->F->as<float>(), t->pf, t->src[ch.k].f_off);
    FL_CHECK_LAUNCH();
    FL_CUDA(cudaEventRecord((cudaEvent_t)ev_free[c].get(), s));
    if (c + ring_n < nch && (rc = issue_chunk(c + ring_n))) return rc;
  }
  if (pin_lock.owns_lock()) {   // the pinned buffers are free again before the ring is released
    for (int b = 0; b < 2 && b < npinned; b++) FL_CUDA(cudaEventSynchronize(pin_ev[b]));
    pin_lock.unlock();
  }
  mark("scatter chunks issued");
  // 4. gathered sources
  for (int k = 0; k < n; k++) {
    if (t->src[k].stream) continue;
    Staged& st = t->staged[k];
    GatherSrc g;
    g.src_index = k;
    g.rows = st.rows;
    g.cols = st.cols;
    g.pitch = pitch_for(st.cols);
    g.tcol.assign(g.pitch, -1);
    for (int c = 0; c < st.cols; c++) g.tcol[c] = st.col_map[c];
    int64_t rows_pad = round_up(st.rows, TILE);
    if (host_S[k]) {   // already in flight on the value copy stream (1b)
      g.S = host_S[k];
    } else {
      g.S = make_buf((size_t)rows_pad * g.pitch * 4 + 64, &rc);
      if (rc) return rc;
      FL_CUDA(cudaMemsetAsync(g.S->p, 0, (size_t)rows_pad * g.pitch * 4, s));
      FL_CUDA(cudaMemcpy2DAsync(g.S->p, g.pitch * 4, st.vals->p, st.cols * 4, st.cols * 4,
                                st.rows, cudaMemcpyDeviceToDevice, s));
    }
    g.fk = make_buf(r_pad * 4, &rc);
    if (rc) return rc;
    k_fk_device_order<<<grid_for(r_pad), 256, 0, s>>>(st.ind_sel->as<int32_t>(),
                                                      t->perm->as<int32_t>(), r_pad,
                                                      g.fk->as<int32_t>());
    FL_CHECK_LAUNCH();
    // group_indptr = exclusive scan of fanout (ops.py:63-65)
    g.grp_ptr = make_buf((st.rows + 1) * 8, &rc);
    if (rc) return rc;
    auto c64 = make_tmp((st.rows + 1) * 8, s, &rc);
    if (rc) return rc;
    k_cnt_to_i64<<<grid_for(st.rows + 1), 256, 0, s>>>(cnts[k]->as<int32_t>(), st.rows,
                                                       c64->as<int64_t>());
    FL_CHECK_LAUNCH();
    size_t tb = 0;
    FL_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, c64->as<int64_t>(), g.grp_ptr->as<int64_t>(),
                                          (int)(st.rows + 1), s));
    auto tmp = make_tmp(tb, s, &rc);
    if (rc) return rc;
    FL_CUDA(cub::DeviceScan::ExclusiveSum(tmp->p, tb, c64->as<int64_t>(), g.grp_ptr->as<int64_t>(),
                                          (int)(st.rows + 1), s));
    int64_t h_matched = 0;
    FL_CUDA(cudaMemcpyAsync(&h_matched, g.grp_ptr->as<int64_t>() + st.rows, 8,
                            cudaMemcpyDeviceToHost, s));
    FL_CUDA(cudaStreamSynchronize(s));
    keep.insert(keep.end(), {c64, tmp});
    g.matched = h_matched;
    g.n_neg = r_T - h_matched;
    g.sorted = (k == sort_k);
    if (!g.sorted) {
      auto order = make_tmp(r_T * 4, s, &rc);
      if (rc) return rc;
      rc = stable_order(st.ind_sel->as<int32_t>(), r_T, st.rows, order->as<int32_t>(), s, &keep);
      if (rc) return rc;
      keep.push_back(order);
      g.grp_rows = make_buf(std::max<int64_t>(g.matched, 1) * 4, &rc);
      if (rc) return rc;
      if (g.matched > 0) {
        k_group_rows<<<grid_for(g.matched), 256, 0, s>>>(order->as<int32_t>(), g.n_neg, g.matched,
                                                         t->iperm->as<int32_t>(),
                                                         g.grp_rows->as<int32_t>());
        FL_CHECK_LAUNCH();
      }
    }
    t->src[k].gidx = (int)t->g.size();
    t->g.push_back(std::move(g));
  }
  t->sort_g = sort_k >= 0 ? t->src[sort_k].gidx : -1;
  rc = table_upload_tcols(t);
  if (rc) return rc;
  mark("gathered sources issued");
  FL_CUDA(cudaStreamSynchronize(cv));
  mark("value copies done");
  FL_CUDA(cudaStreamSynchronize(s));
  mark("layout done");
  t->staged.clear();
  t->finalized = true;
  return FL_OK;
}

int fl_table_destroy(fl_table* t) {
  if (!t) return FL_OK;
  cudaSetDevice(t->device);
  // a table destroyed between add_source and finalize may still be copying
  if (t->cp_idx) cudaStreamSynchronize((cudaStream_t)t->cp_idx.get());
  if (t->cp_vals) cudaStreamSynchronize((cudaStream_t)t->cp_vals.get());
  delete t;
  return FL_OK;
}

int fl_table_shape(const fl_table* t, int64_t* r_T, int32_t* c_T, int32_t* n_sources) {
  if (!t) return FL_ERR_ARG;
  if (r_T) *r_T = t->r_T;
  if (c_T) *c_T = t->c_T;
  if (n_sources) *n_sources = (int32_t)(t->finalized ? t->src.size() : t->staged.size());
  return FL_OK;
}

int fl_table_layout(const fl_table* t, int32_t* stream_cols, int32_t* stream_pitch,
                    int32_t* n_gather, int32_t* sort_source, int64_t* device_bytes) {
  if (!t || !t->finalized) {
    set_error("fl_table_layout: table not finalized");
    return FL_ERR_ARG;
  }
  if (stream_cols) *stream_cols = t->nf;
  if (stream_pitch) *stream_pitch = t->pf;
  if (n_gather) *n_gather = (int32_t)t->g.size();
  if (sort_source) *sort_source = t->sort_g >= 0 ? t->g[t->sort_g].src_index : -1;
  if (device_bytes) {
    int64_t b = 0;
    if (t->F) b += t->F->bytes;
    if (t->perm) b += t->perm->bytes;
    if (t->iperm) b += t->iperm->bytes;
    for (auto& g : t->g) {
      b += g.S->bytes + g.fk->bytes + g.grp_ptr->bytes;
      if (g.grp_rows) b += g.grp_rows->bytes;
    }
    *device_bytes = b;
  }
  return FL_OK;
}

int fl_table_gather_info(const fl_table* t, int32_t i, int32_t* src_index, int64_t* rows,
                         int32_t* cols, int32_t* pitch, int64_t* matched) {
  if (!t || !t->finalized || i < 0 || i >= (int)t->g.size()) {
    set_error("fl_table_gather_info: bad table or gather index");
    return FL_ERR_ARG;
  }
  const flb::GatherSrc& g = t->g[i];
  if (src_index) *src_index = g.src_index;
  if (rows) *rows = g.rows;
  if (cols) *cols = g.cols;
  if (pitch) *pitch = g.pitch;
  if (matched) *matched = g.matched;
  return FL_OK;
}

int fl_table_selectors(fl_table* t, int32_t k, int32_t* ind_sel, int64_t* group_indptr,
                       int32_t* group_rows, void* stream) {
  if (!t || !t->finalized || k < 0 || k >= (int)t->src.size()) {
    set_error("fl_table_selectors: bad table or source index");
    return FL_ERR_ARG;
  }
  FL_CUDA(cudaSetDevice(t->device));
  cudaStream_t s = (cudaStream_t)stream;
  const SrcInfo& si = t->src[k];
  if (si.stream) {
    set_error("fl_table_selectors: source %d is streamed (injective); its rows live in the "
              "expanded block", k);
    return FL_ERR_OP;
  }
  const GatherSrc& g = t->g[si.gidx];
  int rc;
  if (ind_sel) {
    auto tmp = make_buf(t->r_T * 4, &rc);
    if (rc) return rc;
    k_ind_from_fk<<<grid_for(t->r_T), 256, 0, s>>>(g.fk->as<int32_t>(), t->perm->as<int32_t>(),
                                                   t->r_T, tmp->as<int32_t>());
    FL_CHECK_LAUNCH();
    FL_CUDA(cudaMemcpyAsync(ind_sel, tmp->p, t->r_T * 4, cudaMemcpyDefault, s));
    FL_CUDA(cudaStreamSynchronize(s));
  }
  if (group_indptr) {
    FL_CUDA(cudaMemcpyAsync(group_indptr, g.grp_ptr->p, (g.rows + 1) * 8, cudaMemcpyDefault, s));
  }
  if (group_rows && g.matched > 0) {
    auto tmp = make_buf(g.matched * 4, &rc);
    if (rc) return rc;
    if (g.sorted)
      k_sorted_group_rows<<<grid_for(g.matched), 256, 0, s>>>(t->perm->as<int32_t>(), g.n_neg,
                                                              g.matched, tmp->as<int32_t>());
    else
      k_map_rows<<<grid_for(g.matched), 256, 0, s>>>(g.grp_rows->as<int32_t>(),
                                                     t->perm->as<int32_t>(), g.matched,
                                                     tmp->as<int32_t>());
    FL_CHECK_LAUNCH();
    FL_CUDA(cudaMemcpyAsync(group_rows, tmp->p, g.matched * 4, cudaMemcpyDefault, s));
  }
  FL_CUDA(cudaStreamSynchronize(s));
  return FL_OK;
}

int fl_table_perm(fl_table* t, int32_t* perm, void* stream) {
  if (!t || !t->finalized || !perm) return FL_ERR_ARG;
  FL_CUDA(cudaSetDevice(t->device));
  FL_CUDA(cudaMemcpyAsync(perm, t->perm->p, t->r_T * 4, cudaMemcpyDefault, (cudaStream_t)stream));
  FL_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return FL_OK;
}

int fl_materialize(fl_table* t, float* out, void* stream) {
  if (!t || !t->finalized || !out) {
    set_error("fl_materialize: bad arguments");
    return FL_ERR_ARG;
  }
  FL_CUDA(cudaSetDevice(t->device));
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<ColDesc> cd(t->c_T, ColDesc{0, 0, 0, 0});
  for (int j = 0; j < t->pf; j++)
    if (t->f_tcol[j] >= 0) cd[t->f_tcol[j]] = ColDesc{1, j, 0, 0};
  std::vector<GatherView> gv;
  for (size_t d = 0; d < t->g.size(); d++) {
    const GatherSrc& g = t->g[d];
    for (int c = 0; c < g.cols; c++) cd[g.tcol[c]] = ColDesc{2, (int)d, c, 0};
    gv.push_back(GatherView{g.S->as<float>(), g.fk->as<int32_t>(), g.pitch});
  }
  int rc;
  auto dcd = make_buf(cd.size() * sizeof(ColDesc), &rc);
  if (rc) return rc;
  auto dgv = make_buf(std::max<size_t>(gv.size(), 1) * sizeof(GatherView), &rc);
  if (rc) return rc;
  FL_CUDA(cudaMemcpyAsync(dcd->p, cd.data(), cd.size() * sizeof(ColDesc), cudaMemcpyHostToDevice, s));
  if (!gv.empty())
    FL_CUDA(cudaMemcpyAsync(dgv->p, gv.data(), gv.size() * sizeof(GatherView),
                            cudaMemcpyHostToDevice, s));
  int64_t total = t->r_T * (int64_t)t->c_T;
  float* od;
  bool oo;
  rc = out_buffer(out, (size_t)total, s, &od, &oo);
  if (rc) return rc;
  k_materialize<<<grid_for(total), 256, 0, s>>>(t->F ? t->F->as<float>() : nullptr, t->pf,
                                                dcd->as<ColDesc>(), dgv->as<GatherView>(),
                                                t->perm->as<int32_t>(), t->r_T, t->c_T, od);
  FL_CHECK_LAUNCH();
  rc = finish_out(out, od, oo, (size_t)total, s);
  if (rc) return rc;
  FL_CUDA(cudaStreamSynchronize(s));
  return FL_OK;
}

int fl_elementwise(fl_table* t, int32_t func, double scalar, fl_table** out, void* stream) {
  if (!t || !t->finalized || !out) {
    set_error("fl_elementwise: bad arguments");
    return FL_ERR_ARG;
  }
  if (func < FL_EW_SCALE || func > FL_EW_LOGISTIC_CENTERED) {
    set_error("elementwise map %d is not registered (or does not preserve zero): requires "
              "materialization fallback", func);
    return FL_ERR_OP;
  }
  FL_CUDA(cudaSetDevice(t->device));
  cudaStream_t s = (cudaStream_t)stream;
  auto* nt = new fl_table();
  nt->device = t->device;
  nt->sm_count = t->sm_count;
  nt->r_T = t->r_T;
  nt->c_T = t->c_T;
  nt->r_pad = t->r_pad;
  nt->finalized = true;
  nt->src = t->src;
  nt->pf = t->pf;
  nt->nf = t->nf;
  nt->f_tcol = t->f_tcol;
  nt->d_f_tcol = t->d_f_tcol;
  nt->g = t->g;          // shares fk / grp / tcol buffers (metadata reuse, ops.py:285-293)
  nt->sort_g = t->sort_g;
  nt->perm = t->perm;
  nt->iperm = t->iperm;
  int rc;
  if (t->F) {
    int64_t n = (int64_t)t->r_pad * t->pf;
    nt->F = make_buf(t->F->bytes, &rc);
    if (rc) { delete nt; return rc; }
    k_elementwise<<<grid_for(n), 256, 0, s>>>(nt->F->as<float>(), t->F->as<float>(), n, func,
                                              scalar);
    FL_CHECK_LAUNCH();
  }
  for (size_t d = 0; d < t->g.size(); d++) {
    const GatherSrc& g = t->g[d];
    int64_t n = round_up(g.rows, TILE) * g.pitch;
    auto S = make_buf(g.S->bytes, &rc);
    if (rc) { delete nt; return rc; }
    k_elementwise<<<grid_for(n), 256, 0, s>>>(S->as<float>(), g.S->as<float>(), n, func, scalar);
    FL_CHECK_LAUNCH();
    nt->g[d].S = S;
  }
  FL_CUDA(cudaStreamSynchronize(s));
  *out = nt;
  return FL_OK;
}

}  // extern "C"

namespace flb {
__global__ void k_target_rows(const float* __restrict__ F, int pf, const ColDesc* __restrict__ cd,
                              const GatherView* __restrict__ gv, const int32_t* __restrict__ iperm,
                              const int64_t* __restrict__ rows, int n, int c_T,
                              float* __restrict__ out) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n * c_T) return;
  int i = (int)(idx / c_T);
  int t = (int)(idx - (int64_t)i * c_T);
  int64_t p = iperm[rows[i]];
  ColDesc d = cd[t];
  float v = 0.f;
  if (d.kind == 1) {
    v = F[p * pf + d.a];
  } else if (d.kind == 2) {
    GatherView g = gv[d.a];
    int32_t fk = g.fk[p];
    if (fk >= 0) v = g.S[(int64_t)fk * g.pitch + d.b];
  }
  out[idx] = v;
}
}  // namespace flb

extern "C" int fl_target_rows(fl_table* t, const int64_t* rows, int32_t n, float* out,
                              void* stream) {
  if (!t || !t->finalized || !rows || !out || n < 1) {
    set_error("fl_target_rows: bad arguments");
    return FL_ERR_ARG;
  }
  FL_CUDA(cudaSetDevice(t->device));
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<int64_t> h(n);
  FL_CUDA(cudaMemcpy(h.data(), rows, n * 8, cudaMemcpyDefault));
  for (int i = 0; i < n; i++)
    if (h[i] < 0 || h[i] >= t->r_T) {
      set_error("fl_target_rows: row %lld out of range", (long long)h[i]);
      return FL_ERR_SHAPE;
    }
  std::vector<ColDesc> cd(t->c_T, ColDesc{0, 0, 0, 0});
  for (int j = 0; j < t->pf; j++)
    if (t->f_tcol[j] >= 0) cd[t->f_tcol[j]] = ColDesc{1, j, 0, 0};
  std::vector<GatherView> gv;
  for (size_t d = 0; d < t->g.size(); d++) {
    const GatherSrc& g = t->g[d];
    for (int c = 0; c < g.cols; c++) cd[g.tcol[c]] = ColDesc{2, (int)d, c, 0};
    gv.push_back(GatherView{g.S->as<float>(), g.fk->as<int32_t>(), g.pitch});
  }
  int rc;
  auto dcd = make_buf(cd.size() * sizeof(ColDesc), &rc);
  if (rc) return rc;
  auto dgv = make_buf(std::max<size_t>(gv.size(), 1) * sizeof(GatherView), &rc);
  if (rc) return rc;
  auto drows = make_buf((size_t)n * 8, &rc);
  if (rc) return rc;
  auto dout = make_buf((size_t)n * t->c_T * 4, &rc);
  if (rc) return rc;
  FL_CUDA(cudaMemcpy(dcd->p, cd.data(), cd.size() * sizeof(ColDesc), cudaMemcpyHostToDevice));
  if (!gv.empty())
    FL_CUDA(cudaMemcpy(dgv->p, gv.data(), gv.size() * sizeof(GatherView), cudaMemcpyHostToDevice));
  FL_CUDA(cudaMemcpy(drows->p, h.data(), (size_t)n * 8, cudaMemcpyHostToDevice));
  int64_t total = (int64_t)n * t->c_T;
  k_target_rows<<<grid_for(total), 256, 0, s>>>(t->F ? t->F->as<float>() : nullptr, t->pf,
                                                dcd->as<ColDesc>(), dgv->as<GatherView>(),
                                                t->iperm->as<int32_t>(), drows->as<int64_t>(), n,
                                                t->c_T, dout->as<float>());
  FL_CHECK_LAUNCH();
  FL_CUDA(cudaMemcpyAsync(out, dout->p, (size_t)total * 4, cudaMemcpyDefault, s));
  FL_CUDA(cudaStreamSynchronize(s));
  return FL_OK;
}
