// ref_shim.cpp -- C-ABI shim around the UNMODIFIED reference implementation.
//
// TEST INFRASTRUCTURE ONLY. Compiled by oracle/Makefile together with the
// reference's own sources, taken where they lie under /root/reference
// (proj/core/src/*.cpp, headers via -I), into oracle/_ref/libesdg_ref.so.
// No reference source is copied into this repository; this file only calls
// the reference's public interface (esdg::Solver<Real> & friends) and gives
// it the same C entry points the oracle restatement has, so tests can run
// both side by side and bench.py can time the reference's CPU path.
#include <cstdint>
#include <cstring>
#include <memory>
#include <thread>
#include <vector>

#include "esdg/cases.hpp"
#include "esdg/diagnostics.hpp"
#include "esdg/partition.hpp"
#include "esdg/schedule.hpp"
#include "esdg/solver.hpp"

#include "esdg_oracle.h" // shared POD types (orc_mesh_config, orc_gas, ...)

using namespace esdg;

namespace {

struct RefMesh {
  std::shared_ptr<MeshGeometry> mesh;
  std::vector<std::int32_t> lattice;
  std::vector<orc_face> faces;
  std::vector<std::int32_t> face_of;
};

template <class Real>
struct RefSolver {
  std::unique_ptr<Solver<Real>> solver;
  StateField<Real> k_view; // scratch for host-buffer calls
  orc_error err{};
};

template <class Real>
KernelSettings<Real> make_settings(const orc_settings* s) {
  KernelSettings<Real> ks;
  ks.variant = KernelVariant::Balanced;
  ks.contravariant_direct = true;
  ks.dissipation = s->dissipation != 0;
  ks.coriolis.mode = s->coriolis_mode == 0   ? CoriolisMode::None
                     : s->coriolis_mode == 1 ? CoriolisMode::FPlane
                                             : CoriolisMode::BetaPlane;
  ks.coriolis.f0 = Real(s->f0);
  ks.coriolis.beta = Real(s->beta);
  ks.coriolis.y0 = Real(s->y0);
  return ks;
}

template <class Real>
void record_error(RefSolver<Real>* h, const NonPhysicalState& e) {
  h->err.set = 1;
  h->err.rho = e.rho();
  h->err.pressure = e.pressure();
  h->err.element = e.element();
  h->err.node = e.node();
  h->err.stage = e.stage();
}

template <class Real>
StateField<Real> wrap(const Solver<Real>& s, const Real* data) {
  StateField<Real> f(s.mesh().num_elements(), s.ops().n3);
  std::memcpy(f.data.data(), data, sizeof(Real) * f.data.size());
  return f;
}

template <class Real>
int init_case(RefSolver<Real>* h, int case_id, std::uint64_t iparam,
              const double* dparam) {
  Solver<Real>& s = *h->solver;
  try {
    switch (case_id) {
      case ORC_CASE_BUBBLE_SHARP:
      case ORC_CASE_BUBBLE_SMOOTH: {
        HydrostaticBackground bg{s.constants(), 300.0};
        const bool sharp = case_id == ORC_CASE_BUBBLE_SHARP;
        s.init_state([&](double x, double y, double z, double phi, double q[5]) {
          bubble_state(bg, bubble_delta_theta(x, y, z, sharp), z, phi, q);
        });
        return 0;
      }
      case ORC_CASE_HYDROSTATIC: {
        HydrostaticBackground bg{s.constants(), 300.0};
        s.init_state([&](double, double, double z, double phi, double q[5]) {
          bg.state(z, phi, q);
        });
        return 0;
      }
      case ORC_CASE_ENTROPY_TEST: {
        const auto& mc = s.mesh().config();
        EntropyTestState gen(mc.lo, mc.hi, s.constants(), iparam);
        s.init_state([&](double x, double y, double z, double phi, double q[5]) {
          gen.state(x, y, z, phi, q);
        });
        return 0;
      }
      case ORC_CASE_CONSTANT: {
        const double gamma = s.constants().gamma;
        const double rho = dparam[0], u1 = dparam[1], u2 = dparam[2],
                     u3 = dparam[3], p = dparam[4];
        s.init_state([&](double, double, double, double phi, double q[5]) {
          q[0] = rho;
          q[1] = rho * u1;
          q[2] = rho * u2;
          q[3] = rho * u3;
          q[4] = p / (gamma - 1.0) +
                 0.5 * rho * (u1 * u1 + u2 * u2 + u3 * u3) + rho * phi;
        });
        return 0;
      }
    }
  } catch (const std::exception&) {
    return -1;
  }
  return -1;
}

} // namespace

extern "C" {

// ---- mesh -----------------------------------------------------------------

void* ref_mesh_create(const orc_mesh_config* cfg) {
  try {
    MeshConfig c;
    for (int d = 0; d < 3; ++d) {
      c.base[size_t(d)] = cfg->base[d];
      c.lo[size_t(d)] = cfg->lo[d];
      c.hi[size_t(d)] = cfg->hi[d];
      c.bc[size_t(d)] = cfg->bc[d] ? BoundaryCondition::Reflecting
                                   : BoundaryCondition::Periodic;
    }
    c.refinement = cfg->refinement;
    auto* m = new RefMesh;
    m->mesh = std::make_shared<MeshGeometry>(c);
    const std::int64_t ne = m->mesh->num_elements();
    m->lattice.resize(size_t(ne) * 3);
    m->face_of.resize(size_t(ne) * 6);
    for (std::int64_t e = 0; e < ne; ++e) {
      for (int d = 0; d < 3; ++d)
        m->lattice[size_t(e) * 3 + d] = m->mesh->lattice_of(e)[size_t(d)];
      for (int lf = 0; lf < 6; ++lf)
        m->face_of[size_t(e) * 6 + lf] = m->mesh->face_of(e, lf);
    }
    for (const Face& f : m->mesh->faces())
      m->faces.push_back(orc_face{f.minus_elem, f.plus_elem, f.dir,
                                  f.minus_side, std::uint8_t(f.reflecting), 0});
    return m;
  } catch (const std::exception&) {
    return nullptr;
  }
}
void ref_mesh_destroy(void* m) { delete static_cast<RefMesh*>(m); }
std::int64_t ref_mesh_num_elements(const void* m) {
  return static_cast<const RefMesh*>(m)->mesh->num_elements();
}
std::int32_t ref_mesh_num_faces(const void* m) {
  return std::int32_t(static_cast<const RefMesh*>(m)->faces.size());
}
const std::int32_t* ref_mesh_lattice(const void* m) {
  return static_cast<const RefMesh*>(m)->lattice.data();
}
const orc_face* ref_mesh_faces(const void* m) {
  return static_cast<const RefMesh*>(m)->faces.data();
}
const std::int32_t* ref_mesh_face_of(const void* m) {
  return static_cast<const RefMesh*>(m)->face_of.data();
}
double ref_mesh_jacobian(const void* m) {
  return static_cast<const RefMesh*>(m)->mesh->jacobian();
}

int ref_reference_element(int order, double* nodes, double* weights,
                          double* diff) {
  try {
    ReferenceElement r(order);
    std::memcpy(nodes, r.nodes().data(), sizeof(double) * r.nodes().size());
    std::memcpy(weights, r.weights().data(),
                sizeof(double) * r.weights().size());
    std::memcpy(diff, r.diff_matrix().data(),
                sizeof(double) * r.diff_matrix().size());
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

int ref_schedule(int nq, int variant, std::int16_t* partner_index,
                 std::int16_t* half_weight, std::int32_t* offsets) {
  try {
    FluxSchedule s = build_schedule(
        nq, variant == 0 ? ScheduleVariant::Indexing : ScheduleVariant::Weighted);
    for (size_t i = 0; i < s.partners.size(); ++i) {
      partner_index[i] = s.partners[i].index;
      half_weight[i] = s.partners[i].half_weight;
    }
    for (size_t i = 0; i < s.offsets.size(); ++i) offsets[i] = s.offsets[i];
    return int(s.partners.size());
  } catch (const std::exception&) {
    return -1;
  }
}

int ref_partition(std::int64_t n_elements, int ranks,
                  std::int64_t* range_begin) {
  try {
    Partition p = make_partition(n_elements, ranks);
    for (size_t i = 0; i < p.range_begin.size(); ++i)
      range_begin[i] = p.range_begin[i];
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

int ref_exchange_plan(const void* mesh, int ranks, std::int32_t* ghost_count,
                      std::int32_t* interior_count, orc_ghost_face* ghosts,
                      std::int32_t* interior) {
  try {
    const MeshGeometry& m = *static_cast<const RefMesh*>(mesh)->mesh;
    Partition part = make_partition(m.num_elements(), ranks);
    ExchangePlan plan = build_exchange_plan(m, part);
    size_t g_at = 0, i_at = 0;
    for (int r = 0; r < ranks; ++r) {
      ghost_count[r] = std::int32_t(plan.ghosts[size_t(r)].size());
      interior_count[r] = std::int32_t(plan.interior[size_t(r)].size());
      if (ghosts)
        for (const auto& g : plan.ghosts[size_t(r)])
          ghosts[g_at++] = orc_ghost_face{g.face,  g.peer,     g.my_side,
                                          g.slot,  g.my_inbox, g.peer_inbox};
      if (interior)
        for (std::int32_t f : plan.interior[size_t(r)]) interior[i_at++] = f;
    }
    return plan.n_mailboxes;
  } catch (const std::exception&) {
    return -1;
  }
}

int ref_hardware_threads() { return int(std::thread::hardware_concurrency()); }

void ref_lsrk_coefficients(double a[5], double b[5], double c[5]) {
  for (int s = 0; s < 5; ++s) {
    a[s] = LsrkScheme::a[size_t(s)];
    b[s] = LsrkScheme::b[size_t(s)];
    c[s] = LsrkScheme::c[size_t(s)];
  }
}

} // extern "C"

// ---- solver, both precisions ----------------------------------------------

#define REF_DEFINE_SOLVER(SUF, REAL)                                           \
  extern "C" {                                                                 \
  void* ref_solver_create_##SUF(const void* mesh, int order,                   \
                                const orc_gas* gas,                            \
                                const orc_settings* settings, int ranks) {    \
    try {                                                                      \
      GasConstants<double> gc;                                                 \
      gc.gamma = gas->gamma;                                                   \
      gc.R = gas->R;                                                           \
      gc.p0 = gas->p0;                                                         \
      gc.gravity = gas->gravity;                                               \
      auto* h = new RefSolver<REAL>;                                           \
      h->solver = std::make_unique<Solver<REAL>>(                              \
          static_cast<const RefMesh*>(mesh)->mesh, order, gc,                  \
          make_settings<REAL>(settings), ranks);                               \
      return h;                                                                \
    } catch (const std::exception&) {                                          \
      return nullptr;                                                          \
    }                                                                          \
  }                                                                            \
  void ref_solver_destroy_##SUF(void* h) {                                     \
    delete static_cast<RefSolver<REAL>*>(h);                                   \
  }                                                                            \
  int ref_solver_n3_##SUF(const void* h) {                                     \
    return static_cast<const RefSolver<REAL>*>(h)->solver->ops().n3;           \
  }                                                                            \
  REAL* ref_solver_state_##SUF(void* h) {                                      \
    return static_cast<RefSolver<REAL>*>(h)->solver->state().data.data();      \
  }                                                                            \
  const REAL* ref_solver_phi_##SUF(const void* h) {                            \
    return static_cast<const RefSolver<REAL>*>(h)->solver->phi().data();       \
  }                                                                            \
  void ref_solver_ops_##SUF(const void* h, REAL* d, REAL* w, REAL* metric,     \
                            REAL* face_coef, REAL* jacobian) {                 \
    const auto& o = static_cast<const RefSolver<REAL>*>(h)->solver->ops();     \
    std::memcpy(d, o.d.data(), sizeof(REAL) * o.d.size());                     \
    std::memcpy(w, o.weights.data(), sizeof(REAL) * o.weights.size());         \
    for (int k = 0; k < 3; ++k) {                                              \
      metric[k] = o.metric[size_t(k)];                                         \
      face_coef[k] = o.face_coef[size_t(k)];                                   \
    }                                                                          \
    *jacobian = o.jacobian;                                                    \
  }                                                                            \
  void ref_solver_set_settings_##SUF(void* h, const orc_settings* settings) {  \
    static_cast<RefSolver<REAL>*>(h)->solver->settings() =                     \
        make_settings<REAL>(settings);                                         \
  }                                                                            \
  int ref_solver_init_case_##SUF(void* h, int case_id, std::uint64_t iparam,   \
                                 const double* dparam) {                       \
    return init_case(static_cast<RefSolver<REAL>*>(h), case_id, iparam,        \
                     dparam);                                                  \
  }                                                                            \
  int ref_assemble_rhs_##SUF(void* hv, const REAL* q, REAL* out, REAL a_old,   \
                             REAL a_new) {                                     \
    auto* h = static_cast<RefSolver<REAL>*>(hv);                               \
    Solver<REAL>& s = *h->solver;                                              \
    h->err = orc_error{};                                                      \
    StateField<REAL> qf = wrap(s, q), of = wrap(s, out);                       \
    try {                                                                      \
      s.assemble_rhs(qf, of, a_old, a_new);                                    \
    } catch (const NonPhysicalState& e) {                                      \
      record_error(h, e);                                                      \
      return 1;                                                                \
    }                                                                          \
    std::memcpy(out, of.data.data(), sizeof(REAL) * of.data.size());           \
    return 0;                                                                  \
  }                                                                            \
  int ref_volume_rhs_##SUF(void* hv, const REAL* q, REAL* out) {               \
    auto* h = static_cast<RefSolver<REAL>*>(hv);                               \
    Solver<REAL>& s = *h->solver;                                              \
    h->err = orc_error{};                                                      \
    StateField<REAL> qf = wrap(s, q), of = wrap(s, out);                       \
    try {                                                                      \
      s.volume_rhs(qf, of);                                                    \
    } catch (const NonPhysicalState& e) {                                      \
      record_error(h, e);                                                      \
      return 1;                                                                \
    }                                                                          \
    std::memcpy(out, of.data.data(), sizeof(REAL) * of.data.size());           \
    return 0;                                                                  \
  }                                                                            \
  int ref_step_##SUF(void* hv, REAL dt) {                                      \
    auto* h = static_cast<RefSolver<REAL>*>(hv);                               \
    h->err = orc_error{};                                                      \
    try {                                                                      \
      h->solver->step(dt);                                                     \
    } catch (const NonPhysicalState& e) {                                      \
      record_error(h, e);                                                      \
      return 1;                                                                \
    }                                                                          \
    return 0;                                                                  \
  }                                                                            \
  double ref_compute_dt_##SUF(void* h, double courant) {                       \
    try {                                                                      \
      return static_cast<RefSolver<REAL>*>(h)->solver->compute_dt(courant);    \
    } catch (const std::exception&) {                                          \
      return std::nan("");                                                     \
    }                                                                          \
  }                                                                            \
  void ref_last_error_##SUF(const void* h, orc_error* e) {                     \
    *e = static_cast<const RefSolver<REAL>*>(h)->err;                          \
  }                                                                            \
  double ref_quadrature_total_##SUF(const void* hv, const REAL* q, int var) {  \
    const Solver<REAL>& s = *static_cast<const RefSolver<REAL>*>(hv)->solver;  \
    return quadrature_total(wrap(s, q), var, s.mesh(), s.ref());               \
  }                                                                            \
  double ref_total_entropy_##SUF(const void* hv, const REAL* q) {              \
    const Solver<REAL>& s = *static_cast<const RefSolver<REAL>*>(hv)->solver;  \
    return total_entropy(wrap(s, q), s.phi(), s.mesh(), s.ref(),               \
                         s.constants().gamma);                                 \
  }                                                                            \
  double ref_entropy_production_##SUF(const void* hv, const REAL* q,           \
                                      const REAL* rhs) {                       \
    const Solver<REAL>& s = *static_cast<const RefSolver<REAL>*>(hv)->solver;  \
    return entropy_production(wrap(s, q), wrap(s, rhs), s.phi(), s.mesh(),     \
                              s.ref(), s.constants().gamma);                   \
  }                                                                            \
  /* perf[0..3] = wall, volume, surface, update seconds; perf[4] = steps;     \
   * counters[0..5] = volume {flux,log,div}, surface {flux,log,div};          \
   * counters[6] = rhs_calls */                                                \
  void ref_perf_##SUF(void* hv, double* perf, std::uint64_t* counters,         \
                      int reset) {                                             \
    Solver<REAL>& s = *static_cast<RefSolver<REAL>*>(hv)->solver;              \
    PerfRecord& p = s.perf();                                                  \
    perf[0] = p.wall_seconds;                                                  \
    perf[1] = p.volume_seconds;                                                \
    perf[2] = p.surface_seconds;                                               \
    perf[3] = p.update_seconds;                                                \
    perf[4] = double(p.steps);                                                 \
    counters[0] = p.counters.volume.flux_evals;                                \
    counters[1] = p.counters.volume.log_evals;                                 \
    counters[2] = p.counters.volume.div_evals;                                 \
    counters[3] = p.counters.surface.flux_evals;                               \
    counters[4] = p.counters.surface.log_evals;                                \
    counters[5] = p.counters.surface.div_evals;                                \
    counters[6] = p.counters.rhs_calls;                                        \
    if (reset) {                                                               \
      p.wall_seconds = p.volume_seconds = p.surface_seconds =                  \
          p.update_seconds = 0.0;                                              \
      p.steps = 0;                                                             \
      p.counters.reset();                                                      \
    }                                                                          \
  }                                                                            \
  REAL ref_log_mean_##SUF(REAL am, REAL ap, REAL lam, REAL lap) {              \
    KernelCounters c;                                                          \
    return log_mean<REAL>(am, ap, lam, lap, c);                                \
  }                                                                            \
  int ref_node_vals_##SUF(const REAL* q5, REAL phi, REAL gamma, REAL* out8) {  \
    KernelCounters c;                                                          \
    try {                                                                      \
      NodeVals<REAL> v = compute_node_vals<REAL>(q5, phi, gamma, c);           \
      out8[0] = v.rho;                                                         \
      out8[1] = v.u[0];                                                        \
      out8[2] = v.u[1];                                                        \
      out8[3] = v.u[2];                                                        \
      out8[4] = v.b;                                                           \
      out8[5] = v.log_rho;                                                     \
      out8[6] = v.log_b;                                                       \
      out8[7] = v.phi;                                                         \
      return 0;                                                                \
    } catch (const NonPhysicalState&) {                                        \
      return 1;                                                                \
    }                                                                          \
  }                                                                            \
  void ref_ec_flux_##SUF(const REAL* m8, const REAL* p8, int dir, REAL gamma,  \
                         REAL* out7) {                                         \
    KernelCounters c;                                                          \
    NodeVals<REAL> m{m8[0], {m8[1], m8[2], m8[3]}, m8[4], m8[5], m8[6], m8[7]}; \
    NodeVals<REAL> p{p8[0], {p8[1], p8[2], p8[3]}, p8[4], p8[5], p8[6], p8[7]}; \
    TwoPointFlux<REAL> f = ec_flux<REAL, true, true>(m, p, dir, gamma, c);     \
    for (int v = 0; v < 5; ++v) out7[v] = f.sym[v];                            \
    out7[5] = f.gravity;                                                       \
    out7[6] = f.b_ratio;                                                       \
  }                                                                            \
  void ref_matrix_dissipation_##SUF(const REAL* m8, const REAL* p8, int dir,   \
                                    REAL gamma, REAL Rgas, REAL* out5) {       \
    KernelCounters c;                                                          \
    NodeVals<REAL> m{m8[0], {m8[1], m8[2], m8[3]}, m8[4], m8[5], m8[6], m8[7]}; \
    NodeVals<REAL> p{p8[0], {p8[1], p8[2], p8[3]}, p8[4], p8[5], p8[6], p8[7]}; \
    GasConstants<REAL> gc;                                                     \
    gc.gamma = gamma;                                                          \
    gc.R = Rgas;                                                               \
    matrix_dissipation<REAL>(m, p, dir, gc, out5, c);                          \
  }                                                                            \
  }

REF_DEFINE_SOLVER(f64, double)
REF_DEFINE_SOLVER(f32, float)
