/*
 * fl_b200.h -- C ABI of the B200-native factorized-learning hot path.
 *
 * This is the drop-in boundary that replaces the reference's operator surface
 * (`pkg/src/factorlearn/ops.py:147-328`, class TargetHandle) and its trainers
 * (`pkg/src/factorlearn/trainers.py:138-331`).  The host side
 * (`paper_2502_01985_b200/ops.py`, `trainers.py`) binds these entry points
 * with ctypes; INTEGRATION.md shows the binding a reference maintainer would
 * add to `factorlearn`.
 *
 * Conventions
 *  - Every function returns an int status: FL_OK (0) or one of FL_ERR_*,
 *    which the host maps to the reference's exception classes.  The message
 *    of the last failure on the calling thread is `fl_last_error()`.
 *  - Table buffers are library-owned device memory.  Operand / output
 *    pointers are caller-owned; a pointer may be host or device memory
 *    (UVA, copied with cudaMemcpyDefault) unless it says "device".
 *  - All work is ordered on the caller's stream (`void* stream` is a
 *    cudaStream_t; NULL = legacy default stream).  Functions that return
 *    host scalars synchronise that stream.
 *  - Values are stored as fp32; every reduction over target rows is carried
 *    in fp64 (SURVEY.md §7 "fp32 parity at 1e-4").
 */
#ifndef FL_B200_H
#define FL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FL_OK 0
#define FL_ERR_SHAPE 1      /* reference sparse.py:39 ShapeError        */
#define FL_ERR_OP 2         /* reference ops.py:33 OpError              */
#define FL_ERR_METADATA 3   /* reference metadata.py:53 MetadataError   */
#define FL_ERR_CONFIG 4     /* reference trainers.py:32 ConfigError     */
#define FL_ERR_DIVERGENCE 5 /* reference trainers.py:36 DivergenceError */
#define FL_ERR_CUDA 6       /* CUDA runtime failure                     */
#define FL_ERR_ARG 7        /* invalid argument / state                 */

/* elementwise function ids (reference sparse.py:300-307 ELEMENTWISE_FUNCS) */
#define FL_EW_SCALE 0
#define FL_EW_DIVIDE 1
#define FL_EW_SQUARE 2
#define FL_EW_ABS 3
#define FL_EW_EXPM1 4
#define FL_EW_LOGISTIC_CENTERED 5

/* models (reference trainers.py:310-315 TRAINER_FUNCS) */
#define FL_MODEL_LINREG 0
#define FL_MODEL_LOGREG 1

typedef struct fl_table fl_table;
typedef struct fl_glm fl_glm;
typedef struct fl_kmeans fl_kmeans;
typedef struct fl_gnmf fl_gnmf;
typedef struct fl_comm fl_comm;

const char* fl_last_error(void);
int fl_version(void);
/* device properties used by the host for grid sizing and reporting */
int fl_device_info(int device, int* sm_count, int64_t* l2_bytes, int* cc_major, int* cc_minor);

/* ---- table lifecycle: replaces TargetHandle.factorized (ops.py:164-169) and
 *      _build_selectors (ops.py:55-74) ---------------------------------- */
int fl_table_create(int device, int64_t r_T, int32_t c_T, fl_table** out);
/* Add source k (in order).  values: r_k x c_k row-major fp32 (host or device).
 * ind_sel: r_T int32 source row per target row, -1 = no match (ops.py:58-61);
 * NULL = identity indicator (requires r_k == r_T: the fact table of a star).
 * col_map: c_k int32 target column of each source column (map_sel_t,
 * ops.py:67-72), host memory.  Host FKs are uploaded asynchronously here;
 * host VALUES are read by fl_table_finalize (64 MB chunks through a device
 * ring, scattered to device order as they land, so every byte crosses PCIe
 * once; pinned memory runs at the link rate): `values` and `ind_sel` must
 * stay valid until fl_table_finalize returns.  Device operands are copied
 * synchronously (ordered after the caller's work, as cudaMemcpy is). */
int fl_table_add_source(fl_table* t, int64_t r_k, int32_t c_k, const float* values,
                        const int32_t* ind_sel, const int32_t* col_map);
/* Build the device layout: classify sources, derive the device row order
 * (stable sort by the largest gathered source's FK) and inverse CSRs, and
 * move the host values into place (identity-indicator sources start moving
 * before the classification).  FL_TRACE_UPLOAD=1 prints the phases. */
int fl_table_finalize(fl_table* t, void* stream);
int fl_table_destroy(fl_table* t);
int fl_table_shape(const fl_table* t, int64_t* r_T, int32_t* c_T, int32_t* n_sources);
/* stream_cols = real columns in the streamed block; n_gather = gathered
 * sources; sort_source = user index of the sort source (-1 = none) */
int fl_table_layout(const fl_table* t, int32_t* stream_cols, int32_t* stream_pitch,
                    int32_t* n_gather, int32_t* sort_source, int64_t* device_bytes);
/* gathered source i (0 <= i < n_gather): user source index, r_d, c_d, row
 * pitch (floats) and the number of target rows it matches (nnz of I_d) */
int fl_table_gather_info(const fl_table* t, int32_t i, int32_t* src_index, int64_t* rows,
                         int32_t* cols, int32_t* pitch, int64_t* matched);
/* Device-derived selectors of source k in TARGET-row terms, for bit-exact
 * comparison with the reference's _build_selectors (ops.py:55-74).
 * ind_sel: r_T; group_indptr: r_k+1; group_rows: nnz(I_k).  Host or device
 * outputs.  Stream (injective) sources report ind_sel only (group_* NULL ok). */
int fl_table_selectors(fl_table* t, int32_t k, int32_t* ind_sel, int64_t* group_indptr,
                       int32_t* group_rows, void* stream);
/* device row order: perm[p] = target row of device row p (r_T entries) */
int fl_table_perm(fl_table* t, int32_t* perm, void* stream);

/* ---- operators: TargetHandle.{lmm,transpose_lmm,rmm,row_sum,col_sum,
 *      elementwise,materialize_target} (ops.py:206-328) ---------------- */
/* out (r_T x c_x fp32) = T x, x: c_T x c_x fp32 row-major (ops.py:219-235) */
int fl_lmm(fl_table* t, const float* x, int32_t c_x, float* out, void* stream);
/* out (c_T x c_y fp64) = T^T y, y: r_T x c_y fp32 (ops.py:255-271) */
int fl_tlmm(fl_table* t, const float* y, int32_t c_y, double* out, void* stream);
/* out (r_x x c_T fp64) = x T, x: r_x x r_T fp32 (ops.py:237-253) */
int fl_rmm(fl_table* t, const float* x, int32_t r_x, double* out, void* stream);
/* out (r_T fp32) = row sums (ops.py:297-311) */
int fl_row_sum(fl_table* t, float* out, void* stream);
/* out (c_T fp64) = column sums (ops.py:313-328) */
int fl_col_sum(fl_table* t, double* out, void* stream);
/* new table with f applied to every stored source value, sharing the
 * metadata (ops.py:273-295; f(0) = 0 for every registered f) */
int fl_elementwise(fl_table* t, int32_t func, double scalar, fl_table** out, void* stream);
/* dense target (r_T x c_T fp32, target row order): the join
 * (metadata.py:215-225, ops.py:206-217); values are copies (bit-exact) */
int fl_materialize(fl_table* t, float* out, void* stream);
/* rows[n] target rows of T gathered into out (n x c_T fp32, exact copies);
 * the K-means seeding step (trainers.py:213-218 fetches them via rmm) */
int fl_target_rows(fl_table* t, const int64_t* rows, int32_t n, float* out, void* stream);
/* crossprod T^T T (c_T x c_T fp64) -- named in the north star; the reference
 * has no operator for it (its composition is transpose_lmm(lmm(I))) */
int fl_crossprod(fl_table* t, double* out, void* stream);

/* ---- fused GD for linear / logistic regression (trainers.py:138-195) -----
 * One session = device-resident w (fp64 master), labels in device order and
 * a per-iteration pipeline of three kernels: [update + dim q = S_d w_d] ->
 * [fact-row pass: gather + residual/sigmoid + S^T r partials + I_sort^T
 * segmented sums] -> [dim S_d^T bins + final fixed-order reduction].
 * y: r_T values in TARGET order: fp32 for linreg, uint8 0/1 for logreg. */
int fl_glm_create(fl_table* t, int32_t model, const void* y, double learning_rate,
                  fl_glm** out, void* stream);
/* one iteration's partial (local) gradient + loss into the reduce buffer */
int fl_glm_partial(fl_glm* s, void* stream);
/* device pointer + length (c_T + 1 doubles: gradient then loss) of the buffer
 * a multi-GPU caller all-reduces between fl_glm_partial and the next step */
int fl_glm_reduce_buffer(fl_glm* s, double** buf, int32_t* len);
/* apply the pending update (w -= lr * grad; loss_history[it] = loss) */
int fl_glm_update(fl_glm* s, void* stream);
/* single-GPU convenience: iterations x (partial, update), CUDA-graph replayed */
int fl_glm_run(fl_glm* s, int32_t iterations, void* stream);
/* measurement hook: run `iters` iterations launching K1 / K2 / K3 separately
 * with CUDA events between them on `stream`; ms_out[3] = mean ms per kernel
 * (K1 includes the bins memset).  Advances the model like fl_glm_run. */
/* Which fact pass the session runs: 0 CTA tiles, 1 per-warp TMA pipelines
 * (dense stream block), 2 CSR stream block (sparse F),
 * 3 generic operators, 4 solo (the dense per-warp pass with the sort source's
 * q and gradient folded in: one kernel per iteration).  stream_density: measured nonzero density of the
 * real stream columns (1.0 when not measured). */
int fl_glm_path(fl_glm* s, int32_t* path, double* stream_density);
int fl_glm_kernel_times(fl_glm* s, int32_t iters, float* ms_out, void* stream);
/* copy out w (c_T fp64) and the first n losses (fp64); host or device */
int fl_glm_result(fl_glm* s, double* w, double* loss, int32_t n, int32_t* n_done, void* stream);
int fl_glm_destroy(fl_glm* s);

/* ---- fused K-means (trainers.py:198-246) ---------------------------------
 * centroids0: k x c_T fp64 initial centroids (host or device). */
int fl_kmeans_create(fl_table* t, int32_t k, const double* centroids0, fl_kmeans** out,
                     void* stream);
int fl_kmeans_partial(fl_kmeans* s, int32_t write_assign, void* stream);
int fl_kmeans_reduce_buffer(fl_kmeans* s, double** buf, int32_t* len);
int fl_kmeans_update(fl_kmeans* s, void* stream);
int fl_kmeans_run(fl_kmeans* s, int32_t iterations, void* stream);
/* measurement hook: `iters` iterations with CUDA events between the kernels;
 * ms_out[4] = mean ms of [dim E, fact pass, dim sums, reduce + update] */
int fl_kmeans_kernel_times(fl_kmeans* s, int32_t iters, float* ms_out, void* stream);
/* centroids k x c_T fp64, assignments r_T int32 (target order), losses */
int fl_kmeans_result(fl_kmeans* s, double* centroids, int32_t* assign, double* loss,
                     int32_t n, int32_t* n_done, void* stream);
/* assignments r_T int64 (target order) -- the reference's argmin dtype
 * (trainers.py:232-236), widened on the device so the host receives them
 * without a conversion pass */
int fl_kmeans_assignments64(fl_kmeans* s, int64_t* assign, void* stream);
int fl_kmeans_destroy(fl_kmeans* s);
/* which pass the session runs: 0 fused mma.sync, 1 fused tcgen05 (K-major,
 * opt-in), 2 width-general (any k, width or number of sources; generic
 * operators plus row kernels -- the composition of reference
 * trainers.py:223-241), 3 fused tcgen05 with MN-major row-contraction
 * operands (the default for <= 28 streamed columns) */
int fl_kmeans_path(fl_kmeans* s, int32_t* path);

/* ---- Gaussian NMF, multiplicative updates (trainers.py:256-307) ----------
 * w0: r_T x rank fp64 (target order), h0: rank x c_T fp64. */
int fl_gnmf_create(fl_table* t, int32_t rank, const double* w0, const double* h0,
                   double t_sq, fl_gnmf** out, void* stream);
int fl_gnmf_run(fl_gnmf* s, int32_t iterations, void* stream);
/* multi-GPU stepping: the first call computes the products of W_0, every
 * later call applies one H update (recording the previous loss) and computes
 * the products of the new W; all-reduce the buffer (R*c_T + R*R doubles,
 * [W^T T | W^T W], R = rank padded to 8/16/32) after every call. */
int fl_gnmf_partial(fl_gnmf* s, void* stream);
/* measurement hook (after >= 1 iteration): ms_out[5] = mean ms of
 * [H update, dim G, fact pass, dim P, reduce] per iteration */
int fl_gnmf_kernel_times(fl_gnmf* s, int32_t iters, float* ms_out, void* stream);
int fl_gnmf_reduce_buffer(fl_gnmf* s, double** buf, int32_t* len);
int fl_gnmf_result(fl_gnmf* s, double* w, double* h, double* loss, int32_t n,
                   int32_t* n_done, void* stream);
int fl_gnmf_destroy(fl_gnmf* s);
/* 0 fused mma.sync, 1 fused tcgen05 (K-major, opt-in), 2 width-general
 * (any rank / width / number of sources; reference trainers.py:282-299 over
 * the generic operators), 3 fused tcgen05 with MN-major row-contraction
 * operands (rank tile 32, <= 28 streamed columns, <= 1 gathered source) */
int fl_gnmf_path(fl_gnmf* s, int32_t* path);

/* ---- sharded sessions over NCCL (no reference counterpart:
 * the reference is single-process) -----------------------------------------
 * Rank 0 draws the id (fl_comm_unique_id), every rank receives it over the
 * host-side process group and calls fl_comm_init.  NCCL is loaded at run
 * time (the copy torch loaded, else libnccl.so.2; FL_NCCL_LIB overrides).
 * With a communicator attached, fl_{glm,kmeans,gnmf}_run() executes
 * partial -> in-place ncclAllReduce(sum) of the reduce buffer -> update per
 * iteration, captured in CUDA graphs on the session's stream. */
int fl_comm_unique_id(uint8_t* out, int32_t len);   /* len >= 128 */
int fl_comm_init(const uint8_t* id, int32_t len, int32_t nranks, int32_t rank, int32_t device,
                 fl_comm** out);
int fl_comm_allreduce(fl_comm* c, double* buf, int64_t n, void* stream);
int fl_comm_destroy(fl_comm* c);
int fl_glm_set_comm(fl_glm* s, fl_comm* c);      /* c = NULL: back to single-GPU */
int fl_kmeans_set_comm(fl_kmeans* s, fl_comm* c);
int fl_gnmf_set_comm(fl_gnmf* s, fl_comm* c);

/* ---- diagnostics ---------------------------------------------------------
 * Known-answer test of the tcgen05 (5th-gen tensor core) operand layouts:
 * D[128 x N] = A[128 x K] B[K x N] (row-major host or device buffers) through
 * kind::tf32 MMAs from shared memory into TMEM.  mode 0: K-major interleave;
 * 1: K-major interleave with padded K-chunk strides and 32 stored A rows;
 * 2: K-major SWIZZLE_128B A (K = 32).  lbo_sbo: NULL, or 4 byte offsets
 * {A LBO, A SBO, B LBO, B SBO} overriding mode 1 (-1 keeps the default). */
int fl_tc_selftest(int32_t mode, const float* A, const float* B, float* D, int32_t K, int32_t N,
                   const int32_t* lbo_sbo);
/* MN-major tf32 operand probe (csrc/tc_probe.cu): mode 0 dumps a 32 x 32
 * fp32 tile as TMA lays it out with the 128B / 32-byte-atom swizzle; modes
 * 1 / 2 compute D[128 x N] = A[128 x K] B[K x N] with A / B read MN-major in
 * that layout.  params = {LBO, SBO, descriptor layout} (NULL: 16, 1024, 1). */
int fl_tc_probe(int32_t mode, const float* A, const float* B, float* D, float* dump, int32_t K,
                int32_t N, const int32_t* params);
// diagnostics: cycles per kind::tf32 tcgen05.mma (M x N x 8; a_mn / b_mn:
// MN-major operands) issued back to back by one thread per CTA, round-robin
// over `nacc` accumulators (nacc | 256: kind::f16 with bf16 operands, K = 16),
// mean over `ctas` concurrent CTAs
int fl_tc_timing(int32_t M, int32_t N, int32_t a_mn, int32_t b_mn, int32_t reps, int32_t ctas,
                 int32_t nacc, double* cycles);

#ifdef __cplusplus
}
#endif
#endif /* FL_B200_H */
