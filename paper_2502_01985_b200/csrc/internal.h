// Internal types shared by the fl_b200 translation units.
//
// Device layout of a factorized table T = sum_k I_k S_k M_k^T (see DESIGN.md
// "Data layout in HBM"):
//
//  * Target rows live on the device in a permuted "device order" p -> perm[p]
//    chosen so that the foreign key of the largest gathered source (the "sort
//    source") is non-decreasing.  I_sort^T then becomes a contiguous segmented
//    reduction inside the streaming pass.  Only summation order changes.
//  * Every source whose indicator is injective (fanout <= 1; the fact table,
//    union blocks) is expanded into ONE dense row-major fp32 "stream block"
//    F[r_pad x pf] in device order (zero rows where the source has no match).
//    Its columns carry their target column (f_tcol); M_k is column addressing.
//  * Every other source ("gathered", the dimension tables) stays compact:
//    S_d[r_d x pitch] fp32, plus fk_d[r_pad] int32 in device order (-1 = no
//    match) and, for unsorted sources, the inverse CSR of I_d (grp_ptr,
//    grp_rows in device rows, members in ascending TARGET row = the
//    reference's group order, ops.py:62-66).
//  * Row pitches are padded to an odd number of float4 so a thread-per-row
//    read of a TMA-staged tile from shared memory is bank-conflict free.
//  * All row arrays are padded to a multiple of TILE rows so every TMA bulk
//    copy moves whole, 16-byte aligned tiles.
#pragma once

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <string>
#include <vector>

#include "../../include/fl_b200.h"

namespace flb {

constexpr int TILE = 256;          // rows per streamed tile (= threads per CTA)
constexpr int NTHREADS = 256;
constexpr int MAX_GATHER = 8;      // gathered sources handled by the fused kernels

void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what, const char* file, int line);

// cudaFuncAttributeMaxDynamicSharedMemorySize is process-wide per kernel and
// device: sessions only ever RAISE it (a later session with a smaller plan
// must not invalidate the launches of one still alive)
cudaError_t raise_smem_limit_ptr(const void* fn, int bytes);
template <typename F>
inline cudaError_t raise_smem_limit(F* fn, int bytes) {
  return raise_smem_limit_ptr(reinterpret_cast<const void*>(fn), bytes);
}

#define FL_CUDA(call)                                                        \
  do {                                                                       \
    cudaError_t e__ = (call);                                                \
    if (e__ != cudaSuccess) return ::flb::cuda_fail(e__, #call, __FILE__, __LINE__); \
  } while (0)

#define FL_CHECK_LAUNCH() FL_CUDA(cudaGetLastError())

__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }
__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ inline int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

// pitch (floats) for c columns: multiple of 4, odd number of float4
inline int pitch_for(int c) {
  int c4 = (c + 3) / 4;
  if (c4 < 1) c4 = 1;
  if ((c4 & 1) == 0) c4 += 1;
  return 4 * c4;
}

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t astream = nullptr;   // pooled buffers: freed stream-ordered on this stream
  bool pooled = false;
  ~DevBuf();
  int alloc(size_t n);
  // stream-ordered allocation from the library's temporary pool (released
  // memory stays cached in the pool, so repeated uploads neither cudaMalloc
  // nor pay cudaFree's device-wide wait)
  int alloc_tmp(size_t n, cudaStream_t st);
  template <class T> T* as() const { return static_cast<T*>(p); }
};

struct GatherSrc {
  int src_index = -1;        // position among the user's sources
  int64_t rows = 0;          // r_d
  int cols = 0;              // c_d
  int pitch = 0;             // floats
  std::shared_ptr<DevBuf> S; // rows_pad x pitch fp32 (values; replaced by elementwise)
  std::vector<int32_t> tcol; // pitch entries (host), -1 = padding column
  std::shared_ptr<DevBuf> d_tcol;
  std::shared_ptr<DevBuf> fk;        // r_pad int32 device order
  bool sorted = false;
  int64_t n_neg = 0;                 // rows with fk = -1 (sorted source: at the front)
  std::shared_ptr<DevBuf> grp_ptr;   // (rows+1) int64
  std::shared_ptr<DevBuf> grp_rows;  // matched int32 device rows (unsorted only)
  int64_t matched = 0;
};

struct SrcInfo {
  bool stream = false;
  int gidx = -1;       // index into gathers (if gathered)
  int f_off = 0;       // column offset inside F (if stream)
  int64_t rows = 0;
  int cols = 0;
};

struct Staged {            // source data between add_source and finalize
  int64_t rows = 0;
  int cols = 0;
  std::shared_ptr<DevBuf> vals;     // rows x cols fp32 (compact); null for host values
  const float* h_vals = nullptr;    // host values: copied by finalize straight to their
                                    // final place (chunked ring -> stream block, or S_d)
  std::shared_ptr<DevBuf> ind_sel;  // r_T int32 (target order)
  bool sel_given = false;           // false: identity indicator (built on the device)
  std::vector<int32_t> col_map;     // cols target columns
  // the uploads run on the table's copy streams; finalize waits on these
  std::shared_ptr<void> ev_vals, ev_idx;   // cudaEvent_t (owned)
};

// FL_TRACE_UPLOAD=1: host-side phase timestamps of table / session setup
struct PhaseTrace {
  const char* scope;
  bool on;
  std::chrono::steady_clock::time_point t0;
  explicit PhaseTrace(const char* sc)
      : scope(sc), on(std::getenv("FL_TRACE_UPLOAD") != nullptr),
        t0(std::chrono::steady_clock::now()) {}
  void mark(const char* what) const {
    if (on)
      std::fprintf(stderr, "[%s] %-28s %8.3f ms\n", scope, what,
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                       .count());
  }
};

struct Workspace {
  DevBuf a, b, c, d, e;      // generic scratch, grown on demand
  DevBuf counter;            // last-block-done counters (zeroed)
  int grow(DevBuf& buf, size_t bytes);
};

}  // namespace flb

struct fl_table {
  int device = 0;
  int sm_count = 148;
  int64_t r_T = 0;
  int c_T = 0;
  int64_t r_pad = 0;
  bool finalized = false;
  std::vector<flb::Staged> staged;
  // copy streams of the staged uploads (values / FKs): the FK-only part of
  // finalize (sorts, fanout, device order) overlaps the value copies
  std::shared_ptr<void> cp_vals, cp_idx;   // cudaStream_t (owned)
  std::vector<flb::SrcInfo> src;
  // stream block
  int pf = 0;                        // pitch of F in floats (0 = no stream source)
  int nf = 0;                        // real F columns
  std::shared_ptr<flb::DevBuf> F;    // r_pad x pf
  std::vector<int32_t> f_tcol;       // pf entries
  std::shared_ptr<flb::DevBuf> d_f_tcol;
  std::vector<flb::GatherSrc> g;
  int sort_g = -1;                   // gather index of the sort source
  std::shared_ptr<flb::DevBuf> perm;   // r_pad int32 device row -> target row (-1 pad)
  std::shared_ptr<flb::DevBuf> iperm;  // r_T int32 target row -> device row
  flb::Workspace ws;
};

struct fl_comm;
namespace flb {
// comm.cu: in-place fp64 sum over the communicator's ranks (ncclAllReduce)
int comm_allreduce(fl_comm* c, double* buf, size_t n, cudaStream_t st);
// swizzle code for make_tmap_2d: 128B swizzle with 32-byte atoms (the smem
// layout of MN-major tf32 tcgen05 operands, descriptor layout 1)
constexpr int kSwz128Atom32 = 1032;
// tma.cu: 2-D fp32 TMA tensor map over a row-major [rows x cols] array with
// `row_bytes` pitch; box = box_rows x box_cols (columns past `cols` are
// zero-filled by the TMA unit).  swizzle_bytes in {0, 32, 64, 128}.
int make_tmap_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                 uint64_t row_bytes, uint32_t box_rows, uint32_t box_cols, int swizzle_bytes);
// table.cu
int table_upload_tcols(fl_table* t);
// ops.cu helpers used by trainers
// Strided fp32 operand view: element (target row t, col) at base[t*sr + col*sc]
struct YView {
  const float* base;
  int64_t sr, sc;
#ifdef __CUDACC__
  __device__ float at(int64_t t, int col) const { return base[t * sr + (int64_t)col * sc]; }
#endif
};
// generic operators (ops.cu), device operands, stream-ordered:
//   out (r_T x c_x, target order) = T x;   out[tcol*os_t + col*os_c] += (T^T y)
int do_lmm(fl_table* t, const float* x_dev, int c_x, float* out_dev, cudaStream_t s);
//   dev_order: y rows are in device order already (no perm gather)
int do_tlmm(fl_table* t, YView yv, int cy, double* out, int64_t os_t, int64_t os_c,
            cudaStream_t s, bool dev_order = false);
int launch_gather_rows_to_device_order(const fl_table* t, const void* src_target,
                                       void* dst_dev, int elem_bytes, cudaStream_t s);
int device_sm_count(int device);
}  // namespace flb

namespace flb {
// host-or-device operand / output staging (UVA)
template <class T>
inline int to_device(const T* p, size_t n, cudaStream_t s, T** dev, bool* owned) {
  cudaPointerAttributes a{};
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e == cudaSuccess && (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged)) {
    *dev = const_cast<T*>(p);
    *owned = false;
    return FL_OK;
  }
  cudaGetLastError();
  FL_CUDA(cudaMallocAsync((void**)dev, n * sizeof(T) + 16, s));
  FL_CUDA(cudaMemcpyAsync(*dev, p, n * sizeof(T), cudaMemcpyDefault, s));
  *owned = true;
  return FL_OK;
}

template <class T>
inline int out_buffer(T* p, size_t n, cudaStream_t s, T** dev, bool* owned) {
  cudaPointerAttributes a{};
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e == cudaSuccess && (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged)) {
    *dev = p;
    *owned = false;
    return FL_OK;
  }
  cudaGetLastError();
  FL_CUDA(cudaMallocAsync((void**)dev, n * sizeof(T) + 16, s));
  *owned = true;
  return FL_OK;
}

// device -> host copy that returns once `dst` holds the data.  Large copies
// into pageable host memory go through a pinned two-buffer ring (DMA of
// chunk i overlaps a multi-threaded host memcpy of chunk i - 1): the
// driver's pageable path measured ~4.5 GB/s for the 12.8 GB GNMF W readback.
int d2h_copy(void* dst, const void* src, size_t bytes, cudaStream_t s);
// host -> device counterpart (multi-threaded memcpy into the pinned ring,
// DMA of chunk i overlapping the memcpy of chunk i + 1); returns once `src`
// may be reused
int h2d_copy(void* dst, const void* src, size_t bytes, cudaStream_t s);

template <class T>
inline int finish_out(T* user, T* dev, bool owned, size_t n, cudaStream_t s) {
  if (owned) {
    int rc = d2h_copy(user, dev, n * sizeof(T), s);
    if (rc) return rc;
    FL_CUDA(cudaFreeAsync(dev, s));
    FL_CUDA(cudaStreamSynchronize(s));
  }
  return FL_OK;
}

}  // namespace flb

// ---------------------------------------------------------------------------
// Device helpers (PTX wrappers for TMA bulk copies and mbarriers).
// ---------------------------------------------------------------------------
#ifdef __CUDACC__
namespace flb {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Programmatic dependent launch (PDL): a kernel launched with the
// programmatic-serialization attribute may start while its predecessor
// drains; everything before pdl_wait() must touch only data the predecessor
// does not write (immutable inputs, own shared memory).  pdl_wait() returns
// once the predecessor grid has completed and its writes are visible (a
// no-op for a normal launch); pdl_trigger() lets the successor be scheduled.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// mbarrier wait that suspends the warp (hint ~1 ms per try) instead of
// spinning: waiting producer / MMA / epilogue warps give their issue slots
// to the warps that have work
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
        : "memory");
}

// arrive on an mbarrier once every prior cp.async of this thread has landed
// (the arrival is counted in the barrier's expected count: .noinc)
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// L2 eviction-priority policies (createpolicy): streamed operands that are
// touched once are loaded / stored evict_first so they do not push out the
// small, repeatedly updated working set (per-warp partials, gathered rows)
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// TMA 1-D bulk copy global -> shared, completion signalled on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// the same with an L2 cache-eviction policy (see l2_policy_evict_first)
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// TMA 2-D tile load (tensor map in param / const space), coordinates
// {column, row}; out-of-range elements are zero-filled.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int col, int row,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(col), "r"(row), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, int col,
                                                 int row, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(col), "r"(row), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d_hint(const CUtensorMap* map, int col, int row,
                                                  const void* src, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group.L2::cache_hint [%0, {%1, %2}], "
      "[%3], %4;" ::"l"(reinterpret_cast<uint64_t>(map)), "r"(col), "r"(row), "r"(smem_u32(src)),
      "l"(policy)
      : "memory");
}

// L2 prefetch of a 2-D TMA box / a 1-D bulk range (no shared memory, no
// completion): a producer runs these PD tiles ahead of its loads so the
// loads hit L2 and more HBM traffic is in flight than the stages hold
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int col, int row) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(col), "r"(row)
               : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// TMA 2-D tile store shared -> global (bulk-group completion)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int col, int row,
                                             const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::
                   "l"(reinterpret_cast<uint64_t>(map)), "r"(col), "r"(row), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until at most N committed bulk groups still READ their shared source
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// 4 fp32 8x4 matrices -> the m16n8k8 tf32 A fragment (rows 0-7 / 8-15,
// cols 0-3 / 4-7); lane l supplies the address of row (l & 15) at column
// offset (l >> 4) * 4.  Rows must be 16-byte aligned.
// Ampere-style async copies (LDGSTS): 4 / 16 bytes per thread, grouped.
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Pinned read-only loads: volatile so the compiler cannot sink a prefetch
// down to its first use (it otherwise does, which defeats the prefetch).
__device__ __forceinline__ float4 ld_nc_pinned_f4(const void* p) {
  float4 v;
  asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ int ld_nc_pinned_s32(const void* p) {
  int v;
  asm volatile("ld.global.nc.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ void ldsm_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3,
                                        const void* row_ptr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(smem_u32(row_ptr)));
}

// atomicAdd with acquire-release semantics at GPU scope: the arrival counter
// of a last-block-reduces pattern without a full __threadfence (MEMBAR.SC)
__device__ __forceinline__ int atomic_add_acq_rel_gpu(int* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace flb
#endif
