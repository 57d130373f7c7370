// Width-general K-means / GNMF sessions (generic.cu), dispatched from the
// fl_kmeans_* / fl_gnmf_* entry points when the fused passes do not apply.
#pragma once
#include "internal.h"

namespace flb {

struct KmGen;
int kmg_create(fl_table* t, int k, const double* c0, cudaStream_t st, KmGen** out);
int kmg_partial(KmGen* s, cudaStream_t st);   // red = [sums | counts | loss] of this rank
int kmg_update(KmGen* s, cudaStream_t st);    // centroids from red, loss_hist[it++]
int kmg_run(KmGen* s, int iterations, cudaStream_t st);
double* kmg_red(KmGen* s, int* len);
void kmg_set_comm(KmGen* s, fl_comm* c);   // run(): all-reduce between partial and update
int kmg_result(KmGen* s, double* centroids, int32_t* assign, int64_t* assign64, double* loss,
               int n, int* n_done, cudaStream_t st);
void kmg_destroy(KmGen* s);

struct GnGen;
int gng_create(fl_table* t, int rank, const double* w0, const double* h0, double t_sq,
               cudaStream_t st, GnGen** out);
int gng_partial(GnGen* s, cudaStream_t st);
int gng_run(GnGen* s, int iterations, cudaStream_t st);
double* gng_red(GnGen* s, int* len);
void gng_set_comm(GnGen* s, fl_comm* c);
int gng_result(GnGen* s, double* w, double* h, double* loss, int n, int* n_done, cudaStream_t st);
void gng_destroy(GnGen* s);

}  // namespace flb
