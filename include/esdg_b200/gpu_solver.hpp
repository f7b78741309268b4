// gpu_solver.hpp -- header-only C++ mirror of the reference's solver interface
// on top of the C ABI (esdg_b200.h). This is the binding a maintainer of the
// reference adds: esdg_b200::GpuSolver<Real> presents the public members of
// esdg::Solver<Real> (core/include/esdg/solver.hpp:26-158) with the same
// names, argument meaning and error behaviour, so call sites such as the
// reference's tests (tests/test_kernels.cpp) or its runner
// (core/src/runner.cpp:135-269) switch by changing the type name.
//
//   esdg::Solver<double>      solver(mesh, 4, gc, settings, ranks);   // CPU
//   esdg_b200::GpuSolver<double> solver(mesh_config, 4, gc, settings, ranks); // B200
//
// Differences a caller sees (all forced by the device boundary):
//   - the constructor takes the MeshConfig values (the GPU library builds its
//     own Morton mesh; it is checked bitwise against the reference's);
//   - state() returns a host mirror: a non-const access downloads the device
//     registers first and marks the mirror as possibly modified, so the next
//     device operation re-uploads it. Use state_view() for read-only access;
//   - `ranks` is the number of partitions (GPUs when several are visible).
//
// When this header is compiled together with the reference's headers, define
// ESDG_B200_WITH_REFERENCE to make it throw esdg::NonPhysicalState and accept
// esdg::MeshConfig / GasConstants / KernelSettings directly.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "esdg_b200.h"

#ifdef ESDG_B200_WITH_REFERENCE
#include "esdg/error.hpp"
#include "esdg/kernels.hpp"
#include "esdg/mesh.hpp"
#endif

namespace esdg_b200 {

inline constexpr int kNumVars = 5;

// StateField<Real> (state.hpp:13-38): element-major SoA, data[e][var][node]
template <class Real>
struct StateField {
  StateField() = default;
  StateField(std::int64_t n_elements_, int nodes_per_element_)
      : n_elements(n_elements_), nodes_per_element(nodes_per_element_),
        data(size_t(n_elements_) * kNumVars * size_t(nodes_per_element_), Real(0)) {}
  std::int64_t n_elements = 0;
  int nodes_per_element = 0;
  std::vector<Real> data;
  Real* element(std::int64_t e) { return data.data() + size_t(e) * kNumVars * nodes_per_element; }
  const Real* element(std::int64_t e) const { return data.data() + size_t(e) * kNumVars * nodes_per_element; }
  Real& at(std::int64_t e, int var, int node) { return element(e)[size_t(var) * nodes_per_element + node]; }
  Real at(std::int64_t e, int var, int node) const { return element(e)[size_t(var) * nodes_per_element + node]; }
  size_t size() const { return data.size(); }
};

#ifdef ESDG_B200_WITH_REFERENCE
using NonPhysicalState = esdg::NonPhysicalState;
#else
// NonPhysicalState (error.hpp:10-42)
class NonPhysicalState : public std::runtime_error {
public:
  NonPhysicalState(double rho, double pressure, int element, int node, int stage = -1)
      : std::runtime_error("non-physical state (rho=" + std::to_string(rho) +
                           ", p=" + std::to_string(pressure) + ") at element=" +
                           std::to_string(element) + " node=" + std::to_string(node) +
                           (stage >= 0 ? " stage=" + std::to_string(stage) : "")),
        rho_(rho), pressure_(pressure), element_(element), node_(node), stage_(stage) {}
  double rho() const { return rho_; }
  double pressure() const { return pressure_; }
  int element() const { return element_; }
  int node() const { return node_; }
  int stage() const { return stage_; }
  NonPhysicalState with_stage(int stage) const {
    return NonPhysicalState(rho_, pressure_, element_, node_, stage);
  }

private:
  double rho_, pressure_;
  int element_, node_, stage_;
};
#endif

class DeviceError : public std::runtime_error {
public:
  explicit DeviceError(const std::string& m) : std::runtime_error(m) {}
};

// GasConstants<double> (constants.hpp:7-24)
struct GasConstants {
  double gamma = 1.4, R = 287.0, p0 = 1e5, gravity = 9.81;
};

// KernelSettings<Real> (kernels.hpp:59-65); variant is fixed to balanced and
// contravariant_direct to true on the GPU
struct KernelSettings {
  bool dissipation = true;
  int coriolis_mode = 0; // 0 none, 1 f-plane, 2 beta-plane
  double f0 = 0.0, beta = 0.0, y0 = 0.0;
};

// LsrkScheme / lsrk_step (time_integration.hpp:17-49), unchanged contract
template <class Real, class RhsAccum, class Axpy>
void lsrk_step(RhsAccum&& rhs_accum, Axpy&& axpy, Real dt) {
  double a[5], b[5], c[5];
  esdg_b200_lsrk_coefficients(a, b, c);
  for (int s = 0; s < 5; ++s) {
    rhs_accum(Real(a[s]), dt, Real(c[s]), s);
    axpy(Real(b[s]));
  }
}

template <class Real>
class GpuSolver {
  static_assert(sizeof(Real) == 8 || sizeof(Real) == 4, "Real is double or float");

public:
  GpuSolver(const esdg_b200_mesh_config& mesh_config, int order,
            const GasConstants& constants, const KernelSettings& settings,
            int ranks = 1, const std::vector<int>& devices = {})
      : order_(order), constants_(constants), settings_(settings), ranks_(ranks) {
    check(esdg_b200_mesh_create(&mesh_config, &mesh_));
    const esdg_b200_gas gas{constants.gamma, constants.R, constants.p0, constants.gravity};
    const esdg_b200_settings st{settings.dissipation ? 1 : 0, settings.coriolis_mode,
                                settings.f0, settings.beta, settings.y0};
    std::vector<int32_t> dev(devices.begin(), devices.end());
    if (dev.empty()) {
      const int n = esdg_b200_device_count();
      for (int r = 0; r < ranks; ++r) dev.push_back(n > 0 ? r % n : 0);
    }
    const int rc = esdg_b200_solver_create(mesh_, order, &gas, &st, int(sizeof(Real)), ranks,
                                           dev.data(), int(dev.size()), &solver_);
    if (rc != ESDG_B200_OK) {
      esdg_b200_mesh_destroy(mesh_);
      mesh_ = nullptr;
      check(rc);
    }
    nq_ = order + 1;
    n3_ = nq_ * nq_ * nq_;
    ne_ = esdg_b200_mesh_num_elements(mesh_);
    nodes_.resize(size_t(nq_));
    weights_.resize(size_t(nq_));
    diff_.resize(size_t(nq_) * size_t(nq_));
    check(esdg_b200_reference_element(order, nodes_.data(), weights_.data(), diff_.data()));
    for (int d = 0; d < 3; ++d) {
      lo_[d] = mesh_config.lo[d];
      const int64_t n = int64_t(mesh_config.base[d]) << mesh_config.refinement;
      delta_[d] = (mesh_config.hi[d] - mesh_config.lo[d]) / double(n);
    }
  }

#ifdef ESDG_B200_WITH_REFERENCE
  template <class R2>
  GpuSolver(std::shared_ptr<const esdg::MeshGeometry> mesh, int order,
            const esdg::GasConstants<double>& gc, const esdg::KernelSettings<R2>& ks,
            int ranks = 1)
      : GpuSolver(to_config(mesh->config()), order,
                  GasConstants{gc.gamma, gc.R, gc.p0, gc.gravity},
                  KernelSettings{ks.dissipation, int(ks.coriolis.mode), double(ks.coriolis.f0),
                                 double(ks.coriolis.beta), double(ks.coriolis.y0)},
                  ranks) {}
#endif

  ~GpuSolver() {
    if (solver_) esdg_b200_solver_destroy(solver_);
    if (mesh_) esdg_b200_mesh_destroy(mesh_);
  }
  GpuSolver(const GpuSolver&) = delete;
  GpuSolver& operator=(const GpuSolver&) = delete;

  int ranks() const { return ranks_; }
  int order() const { return order_; }
  int nq() const { return nq_; }
  int n3() const { return n3_; }
  std::int64_t num_elements() const { return ne_; }
  const GasConstants& constants() const { return constants_; }
  const KernelSettings& settings() const { return settings_; }
  const std::vector<double>& nodes() const { return nodes_; }
  const std::vector<double>& weights() const { return weights_; }
  const std::vector<double>& diff_matrix() const { return diff_; }
  void set_fused(bool on) {
    check(esdg_b200_solver_set_path(solver_, on ? ESDG_B200_PATH_FUSED : ESDG_B200_PATH_SPLIT));
  }
  // ESDG_B200_PATH_STAGE (default: one kernel per LSRK stage in step(), the
  // fastest; assemble_rhs as _FUSED), _FUSED, or _SPLIT (the reference's
  // volume -> surface -> axpy structure)
  void set_path(int path) { check(esdg_b200_solver_set_path(solver_, path)); }
  void set_dissipation(bool on) {
    settings_.dissipation = on;
    const esdg_b200_settings st{on ? 1 : 0, settings_.coriolis_mode, settings_.f0,
                                settings_.beta, settings_.y0};
    check(esdg_b200_solver_set_settings(solver_, &st));
  }

  // mesh.hpp:73-77
  double node_coordinate(std::int64_t e, int dir, double ref_node) const {
    const int32_t* lat = esdg_b200_mesh_lattice(mesh_) + 3 * e;
    return lo_[dir] + (double(lat[dir]) + 0.5 * (ref_node + 1.0)) * delta_[dir];
  }

  // phi() (solver.hpp:79, 166-176)
  const std::vector<Real>& phi() {
    if (phi_.empty()) {
      phi_.resize(size_t(ne_) * size_t(n3_));
      check(esdg_b200_solver_get_phi(solver_, phi_.data()));
    }
    return phi_;
  }

  // init_state(f), f(x, y, z, phi, double q[5]) (solver.hpp:92-108)
  template <class F>
  void init_state(F&& f) {
    const std::vector<Real>& ph = phi();
    host_.n_elements = ne_;
    host_.nodes_per_element = n3_;
    host_.data.assign(size_t(ne_) * kNumVars * size_t(n3_), Real(0));
    for (std::int64_t e = 0; e < ne_; ++e) {
      Real* qe = host_.element(e);
      for (int n = 0; n < n3_; ++n) {
        const int a = n % nq_, b = (n / nq_) % nq_, c = n / (nq_ * nq_);
        double qv[5];
        f(node_coordinate(e, 0, nodes_[size_t(a)]), node_coordinate(e, 1, nodes_[size_t(b)]),
          node_coordinate(e, 2, nodes_[size_t(c)]), double(ph[size_t(e) * n3_ + n]), qv);
        for (int v = 0; v < 5; ++v) qe[size_t(v) * n3_ + n] = Real(qv[v]);
      }
    }
    host_valid_ = true;
    host_dirty_ = true;
  }

  // state() (solver.hpp:80-81): host mirror, see the header comment
  StateField<Real>& state() {
    pull();
    host_dirty_ = true;
    return host_;
  }
  const StateField<Real>& state_view() {
    pull();
    return host_;
  }

  // assemble_rhs(q, out, a_old, a_new) (solver.hpp:112-119). Field is any
  // StateField-like type (ours or the reference's esdg::StateField<Real>).
  template <class Field>
  void assemble_rhs(const Field& q, Field& out, Real a_old, Real a_new) {
    push_if_needed(); // keep the internal q register as the caller left it
    stash_internal();
    guard(esdg_b200_solver_assemble_rhs(solver_, q.data.data(), out.data.data(), double(a_old),
                                        double(a_new)), -1);
  }

  // volume_rhs(q, out) (solver.hpp:122-129)
  template <class Field>
  void volume_rhs(const Field& q, Field& out) {
    push_if_needed();
    stash_internal();
    guard(esdg_b200_solver_volume_rhs(solver_, q.data.data(), out.data.data()), -1);
  }

  // step(dt) (solver.hpp:132-146): five (rhs, axpy) stages on the device
  // registers; a NonPhysicalState carries the stage like with_stage() does
  void step(Real dt) {
    restore_internal();
    push_if_needed();
    guard(esdg_b200_solver_step(solver_, double(dt), 1), 0);
    host_valid_ = false;
  }

  // compute_dt(courant) (solver.hpp:148-150)
  double compute_dt(double courant) {
    restore_internal();
    push_if_needed();
    double dt = 0.0;
    guard(esdg_b200_solver_compute_dt(solver_, courant, &dt), -1);
    return dt;
  }

  // node_mass(n) (solver.hpp:153-158): J w_a w_b w_c in 64-bit
  double node_mass(int node) const {
    const int a = node % nq_, b = (node / nq_) % nq_, c = node / (nq_ * nq_);
    return 0.125 * delta_[0] * delta_[1] * delta_[2] * weights_[size_t(a)] * weights_[size_t(b)] *
           weights_[size_t(c)];
  }

  // Where the diagnostics and compute_dt are reduced: on the device (default;
  // one double per element crosses PCIe) or on the host in the reference's
  // summation order (bitwise the reference's sums, moves the state).
  void set_reduction_on_host(bool on) {
    guard(esdg_b200_solver_set_reduction(
              solver_, on ? ESDG_B200_REDUCE_ON_HOST : ESDG_B200_REDUCE_ON_DEVICE), -1);
  }

  // diagnostics of the internal registers (diagnostics.hpp:30-106)
  double quadrature_total(int var) {
    restore_internal();
    push_if_needed();
    double v = 0.0;
    guard(esdg_b200_solver_quadrature_total(solver_, ESDG_B200_REG_Q, var, &v), -1);
    return v;
  }
  double total_entropy() {
    restore_internal();
    push_if_needed();
    double v = 0.0;
    guard(esdg_b200_solver_total_entropy(solver_, &v), -1);
    return v;
  }

  esdg_b200_solver* handle() { return solver_; }

private:
#ifdef ESDG_B200_WITH_REFERENCE
  static esdg_b200_mesh_config to_config(const esdg::MeshConfig& c) {
    esdg_b200_mesh_config m{};
    for (int d = 0; d < 3; ++d) {
      m.base[d] = c.base[size_t(d)];
      m.lo[d] = c.lo[size_t(d)];
      m.hi[d] = c.hi[size_t(d)];
      m.bc[d] = c.bc[size_t(d)] == esdg::BoundaryCondition::Reflecting ? 1 : 0;
    }
    m.refinement = c.refinement;
    return m;
  }
#endif

  static void check(int rc) {
    if (rc == ESDG_B200_OK) return;
    const char* msg = esdg_b200_last_message();
    if (rc == ESDG_B200_BADARG) throw std::invalid_argument(msg ? msg : "esdg_b200: bad argument");
    throw DeviceError(msg ? msg : "esdg_b200: device error");
  }

  // status 1 -> NonPhysicalState exactly as solver.hpp:141-143 rethrows it
  void guard(int rc, int /*default_stage*/) {
    if (rc == ESDG_B200_NONPHYSICAL) {
      esdg_b200_error e{};
      esdg_b200_solver_last_error(solver_, &e);
      throw NonPhysicalState(e.rho, e.pressure, int(e.element), e.node, e.stage);
    }
    check(rc);
  }

  void pull() {
    restore_internal();
    if (host_valid_) return;
    host_.n_elements = ne_;
    host_.nodes_per_element = n3_;
    host_.data.resize(size_t(ne_) * kNumVars * size_t(n3_));
    check(esdg_b200_solver_get_state(solver_, ESDG_B200_REG_Q, host_.data.data()));
    host_valid_ = true;
  }
  void push_if_needed() {
    if (host_valid_ && host_dirty_) {
      check(esdg_b200_solver_set_state(solver_, ESDG_B200_REG_Q, host_.data.data()));
      host_dirty_ = false;
    }
  }
  // assemble_rhs with caller-owned host fields borrows the two device
  // registers; the internal q register is parked in the host mirror meanwhile
  void stash_internal() {
    if (stashed_) return;
    if (!host_valid_) {
      host_.n_elements = ne_;
      host_.nodes_per_element = n3_;
      host_.data.resize(size_t(ne_) * kNumVars * size_t(n3_));
      check(esdg_b200_solver_get_state(solver_, ESDG_B200_REG_Q, host_.data.data()));
      host_valid_ = true;
    }
    stashed_ = true;
  }
  void restore_internal() {
    if (!stashed_) return;
    check(esdg_b200_solver_set_state(solver_, ESDG_B200_REG_Q, host_.data.data()));
    host_dirty_ = false;
    stashed_ = false;
  }

  int order_, nq_ = 0, n3_ = 0, ranks_;
  std::int64_t ne_ = 0;
  GasConstants constants_;
  KernelSettings settings_;
  esdg_b200_mesh* mesh_ = nullptr;
  esdg_b200_solver* solver_ = nullptr;
  std::vector<double> nodes_, weights_, diff_;
  double lo_[3] = {0, 0, 0}, delta_[3] = {0, 0, 0};
  std::vector<Real> phi_;
  StateField<Real> host_;
  bool host_valid_ = false, host_dirty_ = false, stashed_ = false;
};

} // namespace esdg_b200
