// esdg_inst.cuh -- body shared by inst_nq*.cu; define ESDG_NQ before including.
#include <atomic>
#include <type_traits>

#include "esdg_kernels.cuh"
#include "esdg_launch.hpp"

namespace esdg_b200 {

namespace {
constexpr int kMaxDevices = 64;
template <class Real, int NQ, bool VOL, bool SURF, int RUNG = dev::kRungProduct>
cudaError_t launch_one(const dev::RhsParams<Real, NQ>& P, long long n_groups,
                       cudaStream_t stream) {
  // the one-pass kernels (group lists, shared faces) and the split kernels may
  // use different tiles (dev::TileSplit)
  using TileT = std::conditional_t<VOL && SURF, dev::Tile<NQ, sizeof(Real)>,
                                   dev::TileSplit<NQ, sizeof(Real)>>;
  constexpr int EPB = TileT::EPB;
  constexpr int MINB = TileT::MINB;
  constexpr int T = EPB * NQ * NQ;
#ifndef ESDG_TUNE_EXTRA_SMEM
#define ESDG_TUNE_EXTRA_SMEM 0
#endif
  constexpr size_t smem = dev::SmemMap<Real, NQ, EPB>::kBytes + ESDG_TUNE_EXTRA_SMEM;
  auto kern = dev::rhs_kernel<Real, NQ, EPB, MINB, VOL, SURF, RUNG>;
  // the opt-in is a property of the (kernel, device) pair: once per device
  static std::atomic<bool> opted[kMaxDevices];
  int device = 0;
  cudaError_t err = cudaGetDevice(&device);
  if (err != cudaSuccess) return err;
  if (device < 0 || device >= kMaxDevices || !opted[device].load(std::memory_order_acquire)) {
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (err != cudaSuccess) return err;
    if (device >= 0 && device < kMaxDevices) opted[device].store(true, std::memory_order_release);
  }
  if (P.ne <= 0) return cudaSuccess;
  // n_groups > 0 without a list: the run of groups starting at P.group_base
  const long long blocks = (P.groups || n_groups > 0) ? n_groups : (P.ne + EPB - 1) / EPB;
  if (blocks <= 0) return cudaSuccess;
  kern<<<dim3(unsigned(blocks)), dim3(T), smem, stream>>>(P);
  return cudaGetLastError();
}
} // namespace

#ifdef ESDG_INST_LADDER
template <class Real, int NQ>
cudaError_t launch_ladder(int rung, const dev::RhsParams<Real, NQ>& P, cudaStream_t stream) {
  switch (rung) {
    case dev::kRungRecompute:
      return launch_one<Real, NQ, true, false, dev::kRungRecompute>(P, 0, stream);
    case dev::kRungPrecompute:
      return launch_one<Real, NQ, true, false, dev::kRungPrecompute>(P, 0, stream);
    case dev::kRungLogMean:
      return launch_one<Real, NQ, true, false, dev::kRungLogMean>(P, 0, stream);
  }
  return cudaErrorInvalidValue;
}
#define ESDG_INSTANTIATE(REAL, NQ)                                             \
  template cudaError_t launch_ladder<REAL, NQ>(int, const dev::RhsParams<REAL, NQ>&, cudaStream_t);
#else
template <class Real, int NQ>
cudaError_t launch_rhs(int mode, const dev::RhsParams<Real, NQ>& P,
                       long long n_groups, cudaStream_t stream) {
  switch (mode) {
    case kModeVolume: return launch_one<Real, NQ, true, false>(P, n_groups, stream);
    case kModeSurface: return launch_one<Real, NQ, false, true>(P, n_groups, stream);
    case kModeFused: return launch_one<Real, NQ, true, true>(P, n_groups, stream);
  }
  return cudaErrorInvalidValue;
}

template <class Real, int NQ>
cudaError_t launch_pack(const Real* q, const int32_t* send_elem,
                        const int32_t* send_face, Real* send, long long n_send,
                        cudaStream_t stream) {
  if (n_send <= 0) return cudaSuccess;
  const long long total = n_send * 5 * NQ * NQ;
  long long blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  dev::pack_kernel<Real, NQ><<<unsigned(blocks), 256, 0, stream>>>(
      q, send_elem, send_face, send, n_send);
  return cudaGetLastError();
}

template <class Real, int NQ>
void rhs_launch_shape(int mode, int* threads, int* epb, size_t* smem_bytes) {
  constexpr int E1 = dev::Tile<NQ, sizeof(Real)>::EPB;
  constexpr int E2 = dev::TileSplit<NQ, sizeof(Real)>::EPB;
  const bool one_pass = mode == kModeFused;
  *threads = (one_pass ? E1 : E2) * NQ * NQ;
  *epb = one_pass ? E1 : E2;
  *smem_bytes = one_pass ? dev::SmemMap<Real, NQ, E1>::kBytes : dev::SmemMap<Real, NQ, E2>::kBytes;
}

#define ESDG_INSTANTIATE(REAL, NQ)                                             \
  template cudaError_t launch_rhs<REAL, NQ>(                                   \
      int, const dev::RhsParams<REAL, NQ>&, long long, cudaStream_t);          \
  template cudaError_t launch_pack<REAL, NQ>(const REAL*, const int32_t*,      \
                                             const int32_t*, REAL*, long long, \
                                             cudaStream_t);                    \
  template void rhs_launch_shape<REAL, NQ>(int, int*, int*, size_t*);

#endif // ESDG_INST_LADDER

ESDG_INSTANTIATE(double, ESDG_NQ)
ESDG_INSTANTIATE(float, ESDG_NQ)

} // namespace esdg_b200
