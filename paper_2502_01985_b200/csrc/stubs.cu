// Temporary entry points for the K-means / GNMF sessions (replaced by
// kmeans.cu / gnmf.cu).
#include "internal.h"
using namespace flb;
extern "C" {
#define STUB(name, ...) int name(__VA_ARGS__) { set_error(#name " not implemented yet"); return FL_ERR_OP; }
STUB(fl_kmeans_create, fl_table*, int32_t, const double*, fl_kmeans**, void*)
STUB(fl_kmeans_partial, fl_kmeans*, int32_t, void*)
STUB(fl_kmeans_reduce_buffer, fl_kmeans*, double**, int32_t*)
STUB(fl_kmeans_update, fl_kmeans*, void*)
STUB(fl_kmeans_run, fl_kmeans*, int32_t, void*)
STUB(fl_kmeans_result, fl_kmeans*, double*, int32_t*, double*, int32_t, int32_t*, void*)
STUB(fl_kmeans_destroy, fl_kmeans*)
STUB(fl_gnmf_create, fl_table*, int32_t, const double*, const double*, double, fl_gnmf**, void*)
STUB(fl_gnmf_run, fl_gnmf*, int32_t, void*)
STUB(fl_gnmf_result, fl_gnmf*, double*, double*, double*, int32_t, int32_t*, void*)
STUB(fl_gnmf_destroy, fl_gnmf*)
}
