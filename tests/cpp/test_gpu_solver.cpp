// C++ parity tests of esdg_b200::GpuSolver<Real> (include/esdg_b200/gpu_solver.hpp)
// written the way the reference's own tests drive esdg::Solver<Real>
// (proj/tests/test_kernels.cpp, test_partition.cpp, test_time_integration.cpp),
// with the CPU oracle (oracle/esdg_oracle.h) supplying the expected values.
// Built and run by tests/test_cpp_mirror.py on a GPU box.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "esdg_b200/gpu_solver.hpp"
#include "esdg_oracle.h"

using esdg_b200::GasConstants;
using esdg_b200::GpuSolver;
using esdg_b200::KernelSettings;
using esdg_b200::StateField;

static int g_failed = 0;
#define CHECK(cond)                                                            \
  do {                                                                         \
    if (!(cond)) {                                                             \
      std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);              \
      ++g_failed;                                                              \
    }                                                                          \
  } while (0)

static esdg_b200_mesh_config bubble_mesh(int refinement, bool periodic_z) {
  esdg_b200_mesh_config c{};   // tests/test_helpers.hpp:10-21
  for (int d = 0; d < 3; ++d) c.base[d] = 1;
  c.refinement = refinement;
  c.lo[0] = c.lo[1] = -1000.0; c.lo[2] = 0.0;
  c.hi[0] = c.hi[1] = 1000.0;  c.hi[2] = 2000.0;
  c.bc[2] = periodic_z ? 0 : 1;
  return c;
}
static orc_mesh_config to_orc(const esdg_b200_mesh_config& c) {
  orc_mesh_config o{};
  std::memcpy(&o, &c, sizeof o);   // identical POD layout (checked below)
  return o;
}
static_assert(sizeof(orc_mesh_config) == sizeof(esdg_b200_mesh_config), "layout");

static double max_abs(const StateField<double>& f, int var) {
  double m = 0.0;
  for (std::int64_t e = 0; e < f.n_elements; ++e)
    for (int n = 0; n < f.nodes_per_element; ++n) m = std::fmax(m, std::fabs(f.at(e, var, n)));
  return m;
}

// test_kernels.cpp:254-265
static void hydrostatic_rest_exact_zero() {
  const auto mc = bubble_mesh(1, false);
  GpuSolver<double> solver(mc, 4, GasConstants{}, KernelSettings{});
  const GasConstants gc;
  const double cv = gc.R / (gc.gamma - 1.0), cp = gc.gamma * cv;
  solver.init_state([&](double, double, double z, double phi, double q[5]) {
    const double pi = 1.0 - gc.gravity * z / (cp * 300.0);
    const double T = 300.0 * pi, p = gc.p0 * std::pow(pi, cp / gc.R), rho = p / (gc.R * T);
    q[0] = rho; q[1] = q[2] = q[3] = 0.0; q[4] = rho * (cv * T + phi);
  });
  StateField<double> rhs(solver.num_elements(), solver.n3());
  solver.assemble_rhs(solver.state(), rhs, 0.0, 1.0);
  CHECK(max_abs(rhs, 0) == 0.0);
  CHECK(max_abs(rhs, 4) == 0.0);
  CHECK(max_abs(rhs, 3) > 0.0);
}

// test_kernels.cpp:30-44
static void free_stream() {
  esdg_b200_mesh_config mc{};
  for (int d = 0; d < 3; ++d) { mc.base[d] = 1; mc.hi[d] = 1.0; }
  mc.refinement = 1;
  GasConstants gc; gc.gravity = 0.0;
  for (int order : {2, 3, 4}) {
    GpuSolver<double> solver(mc, order, gc, KernelSettings{});
    solver.init_state([&](double, double, double, double phi, double q[5]) {
      const double rho = 1.2, u1 = 20, u2 = 10, u3 = 5, p = 1e5;
      q[0] = rho; q[1] = rho * u1; q[2] = rho * u2; q[3] = rho * u3;
      q[4] = p / 0.4 + 0.5 * rho * (u1 * u1 + u2 * u2 + u3 * u3) + rho * phi;
    });
    StateField<double> rhs(solver.num_elements(), solver.n3());
    solver.assemble_rhs(solver.state(), rhs, 0.0, 1.0);
    double m = 0.0;
    for (double v : rhs.data) m = std::fmax(m, std::fabs(v));
    CHECK(m <= 1e-13 * (2.0 * 4.0 * 10.0 * 1e5));
  }
}

// rhs and 3 steps against the oracle on identical inputs; partitions bitwise
static void parity_and_partitions() {
  const auto mc = bubble_mesh(1, true);
  const orc_mesh_config oc = to_orc(mc);
  orc_mesh* om = orc_mesh_create(&oc);
  const orc_gas og{1.4, 287.0, 1e5, 9.81};
  const orc_settings os{1, 0, 0.0, 0.0, 0.0};
  orc_solver_f64* o = orc_solver_create_f64(om, 3, &og, &os);
  orc_solver_init_case_f64(o, ORC_CASE_ENTROPY_TEST, 31, nullptr);
  const int n3 = orc_solver_n3_f64(o);
  const std::int64_t ne = orc_mesh_num_elements(om);
  const size_t total = size_t(ne) * 5 * size_t(n3);
  StateField<double> q(ne, n3), want(ne, n3), got1(ne, n3), got4(ne, n3);
  std::memcpy(q.data.data(), orc_solver_state_f64(o), sizeof(double) * total);
  orc_assemble_rhs_f64(o, q.data.data(), want.data.data(), 0.0, 1.0);
  double scale[5];
  orc_flux_scale_f64(o, q.data.data(), scale);

  GpuSolver<double> s1(mc, 3, GasConstants{}, KernelSettings{}, 1);
  GpuSolver<double> s4(mc, 3, GasConstants{}, KernelSettings{}, 4);
  s1.assemble_rhs(q, got1, 0.0, 1.0);
  s4.assemble_rhs(q, got4, 0.0, 1.0);
  CHECK(got1.data == got4.data);                       // test_partition.cpp:102-114
  double worst = 0.0;
  for (std::int64_t e = 0; e < ne; ++e)
    for (int v = 0; v < 5; ++v)
      for (int n = 0; n < n3; ++n)
        worst = std::fmax(worst, std::fabs(got1.at(e, v, n) - want.at(e, v, n)) / scale[v]);
  std::printf("  scaled RHS error %.3e\n", worst);
  CHECK(worst <= 2e-12);

  // trajectory: the internal state must survive an interleaved assemble_rhs
  s1.state().data = q.data;
  s4.state().data = q.data;
  const double dt = 1e-3;
  for (int i = 0; i < 3; ++i) {
    orc_step_f64(o, dt);
    s1.step(dt);
    s4.step(dt);
    if (i == 1) s1.assemble_rhs(q, got1, 0.0, 1.0);
  }
  const double* ref = orc_solver_state_f64(o);
  const auto& a = s1.state_view();
  const auto& b = s4.state_view();
  CHECK(a.data == b.data);                             // test_partition.cpp:94-100
  double qmax = 0.0, dmax = 0.0;
  for (size_t i = 0; i < total; ++i) {
    qmax = std::fmax(qmax, std::fabs(ref[i]));
    dmax = std::fmax(dmax, std::fabs(ref[i] - a.data[i]));
  }
  std::printf("  3-step state error %.3e of max|q|\n", dmax / qmax);
  {
    // set_path: one kernel per LSRK stage, four partitions (interior element
    // groups hide the exchange) -- the same three steps, bitwise the fused path
    GpuSolver<double> sf(mc, 3, GasConstants{}, KernelSettings{}, 1);
    GpuSolver<double> ss(mc, 3, GasConstants{}, KernelSettings{}, 4);
    sf.set_path(ESDG_B200_PATH_FUSED);
    ss.set_path(ESDG_B200_PATH_STAGE);
    sf.state().data = q.data;
    ss.state().data = q.data;
    for (int i = 0; i < 3; ++i) {
      sf.step(dt);
      ss.step(dt);
    }
    CHECK(sf.state_view().data == ss.state_view().data);
  }
  {
    // step_stream: three members advanced round-robin (the next member's state
    // arrives and the previous member's result leaves while one is stepped),
    // bitwise the plain step() of each member
    GpuSolver<double> plain(mc, 3, GasConstants{}, KernelSettings{}, 1);
    GpuSolver<double> stream(mc, 3, GasConstants{}, KernelSettings{}, 1);
    plain.set_path(ESDG_B200_PATH_STAGE);
    stream.set_path(ESDG_B200_PATH_STAGE);
    std::vector<esdg_b200::StateField<double>> member(3, q), want(3, q);
    for (int m = 0; m < 3; ++m) {
      for (auto& x : member[m].data) x *= 1.0 + 0.001 * m;
      plain.state().data = member[m].data;
      plain.step(dt);
      plain.step(dt);
      want[m].data = plain.state_view().data;
    }
    stream.state().data = member[0].data;
    for (int i = 0; i < 6; ++i)
      stream.step_stream(dt, i == 5 ? nullptr : &member[(i + 1) % 3], i ? &member[(i + 2) % 3] : nullptr);
    CHECK(member[0].data == want[0].data);
    CHECK(member[1].data == want[1].data);
    CHECK(stream.state_view().data == want[2].data);
  }
  CHECK(dmax <= 1e-12 * qmax);
  CHECK(std::fabs(s1.compute_dt(0.5) - orc_compute_dt_f64(o, 0.5)) <= 1e-12 * orc_compute_dt_f64(o, 0.5));
  {
    // device reduction (default): per-element partial sums, 1e-14 relative;
    // host reduction: the reference's serial Neumaier chain, bitwise
    const double want = orc_quadrature_total_f64(o, a.data.data(), 0);
    CHECK(std::fabs(s1.quadrature_total(0) - want) <= 1e-14 * std::fabs(want));
    s1.set_reduction_on_host(true);
    CHECK(s1.quadrature_total(0) == want);
    s1.set_reduction_on_host(false);
  }
  orc_solver_destroy_f64(o);
  orc_mesh_destroy(om);
}

// test_kernels.cpp:279-288 and solver.hpp:141-143
static void nonphysical_state() {
  esdg_b200_mesh_config mc{};
  for (int d = 0; d < 3; ++d) { mc.base[d] = 1; mc.hi[d] = 1.0; }
  mc.refinement = 1;
  GasConstants gc; gc.gravity = 0.0;
  GpuSolver<double> solver(mc, 2, gc, KernelSettings{});
  solver.init_state([&](double, double, double, double, double q[5]) {
    q[0] = 1.0; q[1] = q[2] = q[3] = 0.0; q[4] = 1e5 / 0.4;
  });
  solver.state().at(3, 0, 5) = -1.0;
  StateField<double> rhs(solver.num_elements(), solver.n3());
  bool thrown = false;
  try {
    solver.assemble_rhs(solver.state(), rhs, 0.0, 1.0);
  } catch (const esdg_b200::NonPhysicalState& e) {
    thrown = e.element() == 3 && e.node() == 5 && e.rho() == -1.0;
  }
  CHECK(thrown);
  thrown = false;
  try {
    solver.step(1e-3);
  } catch (const esdg_b200::NonPhysicalState& e) {
    thrown = e.stage() == 0 && e.element() == 3;
  }
  CHECK(thrown);
}

// test_time_integration.cpp:62-76: zero RHS leaves the registers untouched
static void lsrk_driver_contract() {
  int rhs_calls = 0, axpy_calls = 0;
  double bsum = 0.0;
  esdg_b200::lsrk_step<double>([&](double a, double, double, int s) { rhs_calls += (s == rhs_calls); CHECK(s > 0 || a == 0.0); },
                               [&](double b) { ++axpy_calls; bsum += b; }, 0.1);
  CHECK(rhs_calls == 5 && axpy_calls == 5);
  CHECK(bsum > 0.0);
}

int main() {
  if (esdg_b200_device_count() < 1) {
    std::printf("no CUDA device\n");
    return 2;
  }
  hydrostatic_rest_exact_zero();
  free_stream();
  parity_and_partitions();
  nonphysical_state();
  lsrk_driver_contract();
  std::printf(g_failed ? "FAILED (%d)\n" : "ALL PASSED\n", g_failed);
  return g_failed ? 1 : 0;
}
