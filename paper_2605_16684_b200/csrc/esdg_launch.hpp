// esdg_launch.hpp -- host-callable launchers of the kernels in
// esdg_kernels.cuh. One translation unit per NQ instantiates them
// (inst_nq*.cu) so the heavy, fully unrolled kernels compile in parallel.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "esdg_device.cuh"

namespace esdg_b200 {
namespace dev {
template <class Real, int NQ>
struct RhsParams;
}

enum RhsMode { kModeVolume = 0, kModeSurface = 1, kModeFused = 2 };

// P.groups == null: one CTA per EPB consecutive elements of [0, P.ne);
// otherwise n_groups CTAs, CTA i working on group P.groups[i].
template <class Real, int NQ>
cudaError_t launch_rhs(int mode, const dev::RhsParams<Real, NQ>& P,
                       long long n_groups, cudaStream_t stream);

// Volume kernel of a ladder rung below the product (dev::kRungRecompute,
// kRungPrecompute, kRungLogMean; inst_ladder_nq*.cu), all elements.
template <class Real, int NQ>
cudaError_t launch_ladder(int rung, const dev::RhsParams<Real, NQ>& P, cudaStream_t stream);

template <class Real, int NQ>
cudaError_t launch_pack(const Real* q, const int32_t* send_elem,
                        const int32_t* send_face, Real* send, long long n_send,
                        cudaStream_t stream);

template <class Real>
cudaError_t launch_axpy(Real* q, const Real* k, Real b, long long n,
                        cudaStream_t stream);

// Dynamic shared memory one CTA of rhs_kernel needs (bytes), its CTA size and
// elements per CTA, for the kernel of `mode` (RhsMode).
template <class Real, int NQ>
void rhs_launch_shape(int mode, int* threads, int* epb, size_t* smem_bytes);

} // namespace esdg_b200
