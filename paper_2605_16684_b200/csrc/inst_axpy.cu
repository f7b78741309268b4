// K3 launcher (precision only; no NQ dependence).
#include "esdg_kernels.cuh"
#include "esdg_launch.hpp"

namespace esdg_b200 {

template <class Real>
cudaError_t launch_axpy(Real* q, const Real* k, Real b, long long n,
                        cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  constexpr int VEC = 16 / sizeof(Real);
  long long blocks = (n / VEC + 255) / 256;
  // 148 SMs x 8 resident CTAs of 256 threads; grid-stride beyond that
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  dev::axpy_kernel<Real><<<unsigned(blocks), 256, 0, stream>>>(q, k, b, n);
  return cudaGetLastError();
}

template cudaError_t launch_axpy<double>(double*, const double*, double,
                                         long long, cudaStream_t);
template cudaError_t launch_axpy<float>(float*, const float*, float, long long,
                                        cudaStream_t);

} // namespace esdg_b200
