// Element records of the colour passes (hdgb_ctx::d_erec), built once per context.  Kept out of
// hdgb_op.cu: the launch_n<N> bodies must be instantiated only in their hdgb_op_n*.cu units.
#include "hdgb_op_impl.cuh"

namespace hdgb {
// Element records of the two colour passes: record (colour, t) describes the element of colour
// `colour` in element pair t (pair_elem), as 8 words: the six face offsets fid * N^2, a flag
// word (bit 0 valid, bits 1-6 shared faces, bits 8 + 3 s kind of face s) and a spare word;
// non-uniform grids add alpha0..alpha3 (ElementGeometry, mesh.py:46-56).
__global__ void build_erec_kernel(Geo g, int NQ, int64_t npairs, const double* widths, uint32_t* rec, double* al) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= 2 * npairs) return;
  const int col = (int)(idx / npairs);
  const int64_t t = idx - col * npairs;
  Elem E;
  uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  double a4[4] = {0.0, 0.0, 0.0, 0.0};
  if (pair_elem(g, t, col, E)) {
    uint32_t flags = 1u | (E.shared << 1);
    for (int s = 0; s < 6; ++s) {
      w[s] = (uint32_t)E.fid[s] * (uint32_t)NQ;
      flags |= (uint32_t)face_kind(g, s >> 1, E.c[s >> 1] + (s & 1)) << (8 + 3 * s);
    }
    w[6] = flags;
    if (al) {
      const double h1 = widths[E.c[0]], h2 = widths[g.n1 + E.c[1]], h3 = widths[g.n1 + g.n2 + E.c[2]];
      const double a0 = h1 * h2 * h3 / 8.0, t1 = 2.0 / h1, t2 = 2.0 / h2, t3 = 2.0 / h3;
      a4[0] = a0;
      a4[1] = a0 * (t1 * t1);
      a4[2] = a0 * (t2 * t2);
      a4[3] = a0 * (t3 * t3);
    }
  }
  for (int q = 0; q < 8; ++q) rec[8 * idx + q] = w[q];
  if (al)
    for (int q = 0; q < 4; ++q) al[4 * idx + q] = a4[q];
}

cudaError_t launch_build_erec(hdgb_ctx* c, cudaStream_t s) {
  if (c->npairs <= 0) return cudaSuccess;
  const int64_t n = 2 * c->npairs;
  build_erec_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(c->g, c->N * c->N, c->npairs, c->d_widths, c->d_erec,
                                                                c->uniform ? nullptr : c->d_eal);
  return cudaGetLastError();
}

}  // namespace hdgb
