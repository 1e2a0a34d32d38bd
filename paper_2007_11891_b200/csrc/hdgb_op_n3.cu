// Element-operator kernels for N = p + 1 = 3 (see hdgb_op_impl.cuh).
#include "hdgb_op_impl.cuh"

namespace hdgb {
template cudaError_t launch_n<3>(hdgb_ctx* c, int variant, int mode, const double* u, double* r, cudaStream_t s);
}  // namespace hdgb
