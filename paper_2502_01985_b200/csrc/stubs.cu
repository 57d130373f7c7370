// Temporary entry points for the K-means / GNMF sessions (replaced by
#include "internal.h"
using namespace flb;
extern "C" {
#define STUB(name, ...) int name(__VA_ARGS__) { set_error(#name " not implemented yet"); return FL_ERR_OP; }
STUB(fl_gnmf_create, fl_table*, int32_t, const double*, const double*, double, fl_gnmf**, void*)
STUB(fl_gnmf_run, fl_gnmf*, int32_t, void*)
STUB(fl_gnmf_result, fl_gnmf*, double*, double*, double*, int32_t, int32_t*, void*)
STUB(fl_gnmf_destroy, fl_gnmf*)
}
