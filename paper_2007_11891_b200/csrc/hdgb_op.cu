// Dispatch of the element-operator launchers over the polynomial degree; the template
// bodies live in hdgb_op_impl.cuh and are instantiated one degree per translation unit
// (hdgb_op_n*.cu) so the build parallelises.
#include "hdgb_internal.cuh"

namespace hdgb {

template <int N>
cudaError_t launch_n(hdgb_ctx* c, int variant, int mode, const double* u, double* r, cudaStream_t s);

cudaError_t launch_op(hdgb_ctx* c, int variant, int mode, const double* u, double* r, cudaStream_t s) {
  switch (c->N) {
#define HDGB_CASE(n) \
  case n:            \
    return launch_n<n>(c, variant, mode, u, r, s);
    HDGB_CASE(2) HDGB_CASE(3) HDGB_CASE(4) HDGB_CASE(5) HDGB_CASE(6) HDGB_CASE(7) HDGB_CASE(8) HDGB_CASE(9)
    HDGB_CASE(10) HDGB_CASE(11) HDGB_CASE(12) HDGB_CASE(13) HDGB_CASE(14) HDGB_CASE(15) HDGB_CASE(16)
    HDGB_CASE(17)
#undef HDGB_CASE
    default:
      return cudaErrorInvalidValue;
  }
}
}  // namespace hdgb
