// Deformation kernel tables generated on the device (paqif/ehl/kernels.py:
// 55-100): cell integrals of the half-space Green function on a uniform
// grid, one thread per offset.  The operation order is the reference's
// (products and sums rounded separately -- no contraction into FMAs), so
// the tables differ from numpy's only through the last-bit accuracy of the
// library log / asinh (CUDA's and the host libm's are both faithfully but
// not identically rounded).  At 2049^2 the host setup takes ~0.5 s, the
// device ~ms.
#include <cuda_runtime.h>

#include <cstdint>

#include "capi_util.cuh"

extern "C" {
#include "../../include/paqif_ehl.h"
}

namespace paqif {

// t (log|t| - 1), 0 at t = 0 (kernels.py:55-61)
__device__ __forceinline__ double log_antideriv(double t) {
  return t != 0.0 ? __dmul_rn(t, __dsub_rn(log(fabs(t)), 1.0)) : 0.0;
}

__global__ void kernel_line_table(int64_t nx, double h, double* table) {
  const double hh = __dmul_rn(h, 0.5);  // h / 2.0, exact
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d <= nx;
       d += (int64_t)gridDim.x * blockDim.x) {
    const double dh = __dmul_rn((double)d, h);
    table[d] = __dsub_rn(log_antideriv(__dadd_rn(dh, hh)), log_antideriv(__dsub_rn(dh, hh)));
  }
}

// |a| asinh(b / a) (kernels.py:88-91)
__device__ __forceinline__ double asinh_term(double a, double b) {
  return __dmul_rn(fabs(a), asinh(__ddiv_rn(b, a)));
}

__global__ void kernel_point_table(int64_t nx, int64_t ny, double h, double scale,
                                   double* table) {
  const double hh = __dmul_rn(h, 0.5);
  const int64_t cols = ny + 1, total = (nx + 1) * cols;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = k / cols, j = k - i * cols;
    const double dx = __dmul_rn((double)i, h), dy = __dmul_rn((double)j, h);
    const double xp = __dadd_rn(dx, hh), xm = __dsub_rn(dx, hh);
    const double yp = __dadd_rn(dy, hh), ym = __dsub_rn(dy, hh);
    double v = __dadd_rn(asinh_term(xp, yp), asinh_term(yp, xp));
    v = __dsub_rn(v, asinh_term(xm, yp));
    v = __dsub_rn(v, asinh_term(yp, xm));
    v = __dsub_rn(v, asinh_term(xp, ym));
    v = __dsub_rn(v, asinh_term(ym, xp));
    v = __dadd_rn(v, asinh_term(xm, ym));
    v = __dadd_rn(v, asinh_term(ym, xm));
    table[k] = __dmul_rn(v, scale);
  }
}

}  // namespace paqif

using namespace paqif;

extern "C" int paqif_ehl_kernel_line(int64_t nx, double h, double* table, void* stream) {
  if (nx < 0 || !(h > 0.0) || !table) return set_arg_error("ehl_kernel_line: nx / h / table");
  const int64_t cnt = nx + 1;
  const unsigned grid = (unsigned)(cnt < 148 * 256 ? (cnt + 255) / 256 : 148 * 8);
  kernel_line_table<<<grid, 256, 0, (cudaStream_t)stream>>>(nx, h, table);
  return check_launch("paqif_ehl_kernel_line");
}

extern "C" int paqif_ehl_kernel_point(int64_t nx, int64_t ny, double h, double scale,
                                      double* table, void* stream) {
  if (nx < 0 || ny < 0 || !(h > 0.0) || !table)
    return set_arg_error("ehl_kernel_point: nx / ny / h / table");
  const int64_t cnt = (nx + 1) * (ny + 1);
  const unsigned grid = (unsigned)(cnt < 148 * 256 ? (cnt + 255) / 256 : 148 * 16);
  kernel_point_table<<<grid, 256, 0, (cudaStream_t)stream>>>(nx, ny, h, scale, table);
  return check_launch("paqif_ehl_kernel_point");
}
