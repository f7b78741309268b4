// esdg/solver.hpp -- TYPE-SWAP header. Put this directory in front of the
// reference's own include directory:
//
//   g++ -std=c++20 -I<repo>/include/esdg_b200/swap -I<repo>/include \
//       -I<reference>/proj/core/include  caller.cpp ...  -lesdg_b200
//
// and every `#include "esdg/solver.hpp"` of the reference's own callers
// (tests/acceptance.cpp, core/src/runner.cpp, ladder.hpp, test_helpers.hpp)
// resolves here: esdg::Solver<Real> then names esdg_b200::GpuSolver<Real>,
// the B200 implementation behind the same members
// (core/include/esdg/solver.hpp:26-158). Nothing else of the reference is
// replaced -- its mesh, reference element, cases, diagnostics, time
// integration, config and runner sources compile as they are.
#pragma once

#ifndef ESDG_B200_WITH_REFERENCE
#define ESDG_B200_WITH_REFERENCE 1
#endif

// what the reference's solver.hpp makes visible to its includers
#include <algorithm>
#include <chrono>
#include <memory>

#include "esdg/diagnostics.hpp"
#include "esdg/exchange.hpp"
#include "esdg/kernels.hpp"
#include "esdg/partition.hpp"
#include "esdg/time_integration.hpp"

#include "esdg_b200/gpu_solver.hpp"

namespace esdg {

template <class Real>
using Solver = esdg_b200::GpuSolver<Real>;

} // namespace esdg
