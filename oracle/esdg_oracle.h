/* esdg_oracle.h -- CPU restatement of the reference's ESDG right-hand side
 * and LSRK(5,4) update.
 *
 * THIS IS TEST INFRASTRUCTURE. It is the checker the CUDA path is compared
 * against; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it. The product (libesdg_b200.so) never links
 * or calls anything in oracle/.
 *
 * Parity status: PINNED. The restatement is checked bitwise against the
 * reference's own implementation compiled from /root/reference into
 * oracle/_ref/libesdg_ref.so (tests/test_oracle_vs_ref.py) and against the
 * known-answer values and golden vectors in tests/golden/.
 *
 * Plain C99, one translation unit; the precision-generic part lives in
 * esdg_oracle_impl.inc and is included twice (double, float). Every function
 * cites the reference file:line it restates (paths relative to
 * /root/reference/proj/core).
 */
#ifndef ESDG_ORACLE_H
#define ESDG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- mesh (include/esdg/mesh.hpp:12-98, src/mesh.cpp:11-132) ------------ */

typedef struct {
  int32_t base[3];
  int32_t refinement;
  double lo[3];
  double hi[3];
  int32_t bc[3]; /* 0 = periodic, 1 = reflecting */
} orc_mesh_config;

typedef struct {
  int32_t minus_elem;
  int32_t plus_elem; /* -1 on reflecting faces */
  uint8_t dir;
  uint8_t minus_side;
  uint8_t reflecting;
  uint8_t pad_;
} orc_face;

typedef struct orc_mesh orc_mesh;

orc_mesh* orc_mesh_create(const orc_mesh_config* cfg);
void orc_mesh_destroy(orc_mesh* m);
int64_t orc_mesh_num_elements(const orc_mesh* m);
int32_t orc_mesh_num_faces(const orc_mesh* m);
void orc_mesh_dims(const orc_mesh* m, int32_t dims[3]);
void orc_mesh_delta(const orc_mesh* m, double delta[3]);
double orc_mesh_jacobian(const orc_mesh* m);
/* lattice[e*3 + d] */
const int32_t* orc_mesh_lattice(const orc_mesh* m);
const orc_face* orc_mesh_faces(const orc_mesh* m);
/* face_of[e*6 + dir*2 + side] */
const int32_t* orc_mesh_face_of(const orc_mesh* m);
double orc_mesh_node_coordinate(const orc_mesh* m, int64_t elem, int dir,
                                double ref_node);
uint64_t orc_morton_key(uint32_t i, uint32_t j, uint32_t k);

/* ---- reference element (src/reference_element.cpp:11-138) --------------- */
/* nodes[nq], weights[nq], diff[nq*nq] row-major; returns 0 or -1 (bad order) */
int orc_reference_element(int order, double* nodes, double* weights,
                          double* diff);

/* ---- flux schedule (src/schedule.cpp:8-43) ------------------------------ */
/* variant 0 = Indexing, 1 = Weighted. partner_index/half_weight sized
 * nq*(nq/2) at most, offsets sized nq+1. Returns number of slots or -1. */
int orc_schedule(int nq, int variant, int16_t* partner_index,
                 int16_t* half_weight, int32_t* offsets);

/* ---- partition / exchange plan (src/partition.cpp:13-66) ---------------- */
/* range_begin sized ranks+1; returns 0 or -1 */
int orc_partition(int64_t n_elements, int ranks, int64_t* range_begin);

typedef struct {
  int32_t face;
  int32_t peer;
  int32_t my_side;
  int32_t slot;
  int32_t my_inbox;
  int32_t peer_inbox;
} orc_ghost_face;

/* Counts first (ghosts == NULL), then fills. ghost_count/interior_count sized
 * ranks. ghosts is the concatenation over ranks (face-id order within a rank),
 * interior likewise. Returns n_mailboxes. */
int orc_exchange_plan(const orc_mesh* m, int ranks, int32_t* ghost_count,
                      int32_t* interior_count, orc_ghost_face* ghosts,
                      int32_t* interior);

/* ---- cases (include/esdg/cases.hpp:15-156, tests/test_helpers.hpp) ------ */

typedef struct {
  double gamma, R, p0, gravity;
} orc_gas;

enum {
  ORC_CASE_BUBBLE_SHARP = 0,
  ORC_CASE_BUBBLE_SMOOTH = 1,
  ORC_CASE_HYDROSTATIC = 2,
  ORC_CASE_ENTROPY_TEST = 3, /* iparam = seed */
  ORC_CASE_CONSTANT = 4      /* dparam = {rho,u1,u2,u3,p} */
};

/* ---- solver, both precisions -------------------------------------------- */

typedef struct {
  int32_t dissipation;   /* KernelSettings::dissipation */
  int32_t coriolis_mode; /* 0 none, 1 f-plane, 2 beta-plane */
  double f0, beta, y0;
} orc_settings;

typedef struct {
  int32_t set;
  double rho, pressure;
  int32_t element, node, stage;
} orc_error;

typedef struct orc_solver_f64 orc_solver_f64;
typedef struct orc_solver_f32 orc_solver_f32;

#define ORC_DECLARE_SOLVER(SUF, REAL)                                          \
  orc_solver_##SUF* orc_solver_create_##SUF(const orc_mesh* m, int order,     \
                                            const orc_gas* gas,               \
                                            const orc_settings* settings);    \
  void orc_solver_destroy_##SUF(orc_solver_##SUF* s);                          \
  int orc_solver_n3_##SUF(const orc_solver_##SUF* s);                          \
  REAL* orc_solver_state_##SUF(orc_solver_##SUF* s);                           \
  REAL* orc_solver_kreg_##SUF(orc_solver_##SUF* s);                            \
  const REAL* orc_solver_phi_##SUF(const orc_solver_##SUF* s);                 \
  /* ops: d[nq*nq], w[nq], metric[3], face_coef[3], jacobian rounded */       \
  void orc_solver_ops_##SUF(const orc_solver_##SUF* s, REAL* d, REAL* w,      \
                            REAL* metric, REAL* face_coef, REAL* jacobian);   \
  void orc_solver_set_settings_##SUF(orc_solver_##SUF* s,                      \
                                     const orc_settings* settings);           \
  /* init_state from a named case (solver.hpp:92-108) */                      \
  int orc_solver_init_case_##SUF(orc_solver_##SUF* s, int case_id,            \
                                 uint64_t iparam, const double* dparam);      \
  /* out <- a_old out + a_new RHS(q)  (solver.hpp:112-119, 240-340).          \
   * Returns 0, or 1 with the error payload retrievable below. */             \
  int orc_assemble_rhs_##SUF(orc_solver_##SUF* s, const REAL* q, REAL* out,   \
                             REAL a_old, REAL a_new);                         \
  /* volume term only, no Coriolis (solver.hpp:122-129) */                    \
  int orc_volume_rhs_##SUF(orc_solver_##SUF* s, const REAL* q, REAL* out);    \
  /* rank-restricted assemble (solver.hpp:240-340 for one rank):              \
   * elements [elem_begin, elem_end); ghost_slot_of_face[f] >= 0 marks a      \
   * ghost face whose REMOTE trace is ghost_traces[slot*5*n2 ...]. */         \
  int orc_assemble_rhs_rank_##SUF(orc_solver_##SUF* s, const REAL* q,         \
                                  REAL* out, REAL a_old, REAL a_new,          \
                                  int64_t elem_begin, int64_t elem_end,       \
                                  const int32_t* ghost_slot_of_face,          \
                                  const REAL* ghost_traces);                  \
  /* trace of one element side, var-major 5*n2 (kernels.hpp:331-338) */       \
  void orc_extract_trace_##SUF(const orc_solver_##SUF* s, const REAL* q,      \
                               int64_t elem, int dir, int side, REAL* out);   \
  /* q += b k on the internal registers (solver.hpp:342-353) */               \
  void orc_axpy_##SUF(orc_solver_##SUF* s, REAL b);                            \
  /* one LSRK(5,4) step on the internal registers (solver.hpp:132-146) */     \
  int orc_step_##SUF(orc_solver_##SUF* s, REAL dt);                            \
  double orc_compute_dt_##SUF(orc_solver_##SUF* s, double courant);           \
  void orc_last_error_##SUF(const orc_solver_##SUF* s, orc_error* e);         \
  /* diagnostics (diagnostics.hpp:30-106), always 64-bit */                   \
  double orc_quadrature_total_##SUF(const orc_solver_##SUF* s, const REAL* q, \
                                    int var);                                 \
  double orc_total_entropy_##SUF(const orc_solver_##SUF* s, const REAL* q);   \
  double orc_entropy_production_##SUF(const orc_solver_##SUF* s,              \
                                      const REAL* q, const REAL* rhs);        \
  /* abs-sum flux scale S_v: max over nodes of the sum of    \
   * absolute values of every term the RHS adds into that node. scale[5]. */  \
  int orc_flux_scale_##SUF(orc_solver_##SUF* s, const REAL* q, double* scale);\
  /* the same over [elem_begin, elem_end) with supplied neighbour traces */    \
  int orc_flux_scale_rank_##SUF(orc_solver_##SUF* s, const REAL* q,           \
                                int64_t elem_begin, int64_t elem_end,         \
                                const int32_t* ghost_slot_of_face,            \
                                const REAL* ghost_traces, double* scale);     \
  /* pointwise physics for known-answer tests (physics.hpp, log_mean.hpp) */  \
  REAL orc_log_mean_##SUF(REAL am, REAL ap, REAL lam, REAL lap);              \
  int orc_node_vals_##SUF(const REAL* q5, REAL phi, REAL gamma, REAL* out8);  \
  void orc_ec_flux_##SUF(const REAL* m8, const REAL* p8, int dir, REAL gamma, \
                         REAL* out7);                                         \
  void orc_matrix_dissipation_##SUF(const REAL* m8, const REAL* p8, int dir,  \
                                    REAL gamma, REAL Rgas, REAL* out5);

ORC_DECLARE_SOLVER(f64, double)
ORC_DECLARE_SOLVER(f32, float)

/* LSRK(5,4) coefficients (time_integration.hpp:17-37) */
void orc_lsrk_coefficients(double a[5], double b[5], double c[5]);

/* FNV-1a-64 over raw bytes (BASELINE.md section 4 fingerprints) */
uint64_t orc_fnv1a64(const void* data, uint64_t nbytes);

#ifdef __cplusplus
}
#endif
#endif
