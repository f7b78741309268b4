/* esdg_b200.h -- C ABI of the B200-native ESDG right-hand side.
 *
 * The reference (/root/reference/proj) has no plugin/FFI layer: its boundary
 * for this path is the C++ class esdg::Solver<Real>
 * (core/include/esdg/solver.hpp:26-158) plus lsrk_step
 * (core/include/esdg/time_integration.hpp:43-49). This header is what an FFI
 * for that path binds. Two levels:
 *
 *   1. "shard" entry points: one element partition resident on one GPU.
 *      Plain pointers and sizes; the caller keeps its own mesh / operators /
 *      partition (the reference's proj/core types) and hands over flattened
 *      arrays. Each entry point names the reference routine it replaces.
 *   2. "solver" entry points: the host-side mirror of esdg::Solver<Real>
 *      (esdg_b200::GpuSolver<Real>, include/esdg_b200/gpu_solver.hpp) behind
 *      a C handle, for bindings that do not want to rebuild the mesh logic.
 *
 * Conventions
 *   - status codes: ESDG_B200_OK, _NONPHYSICAL (payload via *_last_error),
 *     _CUDA (message via esdg_b200_last_message), _BADARG. Nothing throws
 *     across this boundary.
 *   - host arrays are borrowed for the duration of the call; device memory is
 *     owned by the handle. One caller thread per handle (the reference's
 *     coordinator is single threaded).
 *   - `precision` is sizeof(Real): 8 (FP64) or 4 (FP32). `void*` state
 *     buffers hold Real in the reference's StateField layout
 *     data[e][var][node], node = a + nq (b + nq c)  (state.hpp:13-38).
 *   - `stream` is a cudaStream_t passed as void*; NULL selects the handle's
 *     own stream. All kernel launches are asynchronous on that stream.
 *   - there is NO CPU fallback: every compute entry point fails with
 *     ESDG_B200_CUDA when no sm_100 device is usable.
 */
#ifndef ESDG_B200_H
#define ESDG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ESDG_B200_ABI_VERSION 1

enum {
  ESDG_B200_OK = 0,
  ESDG_B200_NONPHYSICAL = 1, /* NonPhysicalState, error.hpp:10-42 */
  ESDG_B200_CUDA = 2,
  ESDG_B200_BADARG = 3
};

enum { ESDG_B200_REG_Q = 0, ESDG_B200_REG_K = 1 };

/* NonPhysicalState payload (error.hpp:10-42); element is the GLOBAL Morton id */
typedef struct {
  int32_t set;
  double rho, pressure;
  int64_t element;
  int32_t node;
  int32_t stage;
} esdg_b200_error;

int esdg_b200_abi_version(void);
/* message of the last ESDG_B200_CUDA / _BADARG failure on this thread */
const char* esdg_b200_last_message(void);
/* number of usable CUDA devices (0 when none; never fails) */
int esdg_b200_device_count(void);

/* ======================================================================= */
/* Level 1: shard                                                           */
/* ======================================================================= */

typedef struct esdg_b200_shard esdg_b200_shard;

/* Flattened inputs of one partition. Replaces what Solver's constructor
 * derives (solver.hpp:26-72): Operators<Real> (kernels.hpp:70-92), phi
 * (solver.hpp:166-176), ghost phi traces (solver.hpp:178-191), the face
 * connectivity of MeshGeometry (mesh.cpp:78-132) and the rank's slice of the
 * ExchangePlan (partition.cpp:32-66). */
typedef struct {
  int32_t precision;   /* 8 or 4 */
  int32_t nq;          /* nodes per direction, 2..8 */
  int32_t device;      /* CUDA device ordinal */
  int32_t dissipation; /* KernelSettings::dissipation */
  int64_t n_elements;  /* elements in this partition */
  int64_t elem_offset; /* global id of local element 0 (error reporting) */
  const double* diff;    /* nq*nq 64-bit D, row-major (rounded to Real inside) */
  const double* weights; /* nq 64-bit LGL weights */
  double metric[3];      /* 2 / delta_d, 64-bit */
  double gamma, gas_R;
  /* Coriolis (physics.hpp:276-306): mode 0 none, else f per (y level, b) */
  int32_t coriolis_mode;
  int32_t n_ylevels;
  const int32_t* elem_ylevel; /* n_elements, may be NULL when mode == 0 */
  const void* coriolis_f;     /* Real[n_ylevels*nq]: f at node row b */
  /* connectivity: nbr[e*6 + dir*2 + side] =
   *   >= 0  local element across that face
   *   -1    reflecting wall (mirror_state, physics.hpp:309-313)
   *   <= -2 ghost face: with v = -2 - value, the receive slot is v >> 1 and
   *         bit 0 of v is set when THIS element is the face's minus side
   *         (lower global Morton id; Face::minus_elem, mesh.hpp:27-33) */
  const int32_t* nbr;
  const void* phi; /* Real[n_elements*n3] */
  /* halo: slot s of the send buffer carries the trace of local element
   * send_elem[s], local face send_face[s] (dir*2+side), var-major 5*nq^2
   * exactly like extract_trace (kernels.hpp:331-338). */
  int32_t n_ghost;       /* receive slots */
  const void* ghost_phi; /* Real[n_ghost*nq^2], remote phi traces (static) */
  int32_t n_send;
  const int32_t* send_elem;
  const int32_t* send_face;
} esdg_b200_shard_desc;

int esdg_b200_shard_create(const esdg_b200_shard_desc* desc,
                           esdg_b200_shard** out);
void esdg_b200_shard_destroy(esdg_b200_shard* s);

/* StateField upload/download of `count` elements starting at local element
 * `first` (synchronous; replaces direct access to Solver::state()). */
int esdg_b200_shard_upload(esdg_b200_shard* s, int reg, const void* host,
                           int64_t first, int64_t count);
int esdg_b200_shard_download(esdg_b200_shard* s, int reg, void* host,
                             int64_t first, int64_t count);
/* asynchronous variants on `stream` (host memory should be pinned) */
int esdg_b200_shard_upload_async(esdg_b200_shard* s, int reg, const void* host,
                                 int64_t first, int64_t count, void* stream);
int esdg_b200_shard_download_async(esdg_b200_shard* s, int reg, void* host,
                                   int64_t first, int64_t count, void* stream);
/* raw device pointers (zero-copy integration, e.g. wrapping in a tensor) */
void* esdg_b200_shard_register_ptr(esdg_b200_shard* s, int reg);
void* esdg_b200_shard_send_ptr(esdg_b200_shard* s);
void* esdg_b200_shard_recv_ptr(esdg_b200_shard* s);
void* esdg_b200_shard_stream(esdg_b200_shard* s);

/* K4: gathers the ghost-face traces of register `src` into the send buffer.
 * Replaces extract_trace + Transport::send (solver.hpp:249-257). */
int esdg_b200_shard_pack(esdg_b200_shard* s, int src, void* stream);

/* K1: dst <- a_old dst + a_new (volume(src) [+ Coriolis]).
 * Replaces Solver::volume_phase = volume_element + commit_volume
 * (solver.hpp:199-238, kernels.hpp:279-316). a_old == 0 never reads dst. */
int esdg_b200_shard_volume(esdg_b200_shard* s, int src, int dst, double a_old,
                           double a_new, int with_source, int stage,
                           void* stream);

/* K2: dst <- dst - a_new lift (F* - n F(q_own)) on every face node.
 * Replaces compute_face_record + commit_face_side (kernels.hpp:350-430) for
 * interior, reflecting and ghost faces (ghost traces are read from the
 * receive buffer, which the caller must have filled). */
int esdg_b200_shard_surface(esdg_b200_shard* s, int src, int dst, double a_new,
                            int stage, void* stream);

/* K1+K2 in one pass over the element (beyond the reference's structure):
 * dst <- a_old dst + a_new RHS(src). Same result contract as the pair. */
int esdg_b200_shard_rhs_fused(esdg_b200_shard* s, int src, int dst,
                              double a_old, double a_new, int stage,
                              void* stream);

/* K1+K2+K3, one whole LSRK stage in one kernel (lsrk_step's loop body,
 * time_integration.hpp:43-49): k <- a_old k + a_new RHS(q); q <- q + b k.
 * q is double buffered inside the shard (neighbouring elements still read
 * the old faces while an element commits), so REG_Q always names the current
 * buffer and the shard holds three state registers once this is used. */
int esdg_b200_shard_stage_fused(esdg_b200_shard* s, double a_old, double a_new,
                                double b, int stage, void* stream);

/* The one-pass kernels restricted to a part of the partition, so that they
 * overlap the halo exchange the way the reference's volume phase does
 * (rhs_job, solver.hpp:259-294: volume -> wait -> ghost faces). An element
 * group is the run of consecutive elements one CTA owns; PART_INTERIOR are
 * the groups without a ghost face (they never read the receive buffer),
 * PART_BOUNDARY the rest. Order per RHS: pack -> start the transfer ->
 * PART_INTERIOR -> traces have landed -> PART_BOUNDARY. INTERIOR followed by
 * BOUNDARY is bitwise the PART_ALL result; stage_fused_part swaps the state
 * buffers after PART_BOUNDARY (or PART_ALL), so both parts read the old q.
 * PART_BOUNDARY belongs to the PART_INTERIOR launch before it, on the same
 * stream: its groups take the lift terms of shared faces the interior groups
 * left for them. (The shard tags those terms with the parity of the
 * evaluation; a sequence that abandons an evaluation half way -- INTERIOR
 * without its BOUNDARY -- is allowed, the next evaluation starts from
 * re-initialised slots.) */
enum {
  ESDG_B200_PART_ALL = 0,
  ESDG_B200_PART_INTERIOR = 1,
  ESDG_B200_PART_BOUNDARY = 2
};
int esdg_b200_shard_rhs_fused_part(esdg_b200_shard* s, int src, int dst,
                                   double a_old, double a_new, int stage,
                                   int part, void* stream);
int esdg_b200_shard_stage_fused_part(esdg_b200_shard* s, double a_old,
                                     double a_new, double b, int stage,
                                     int part, void* stream);
/* number of elements in a part (diagnostic: how much work hides the halo) */
int esdg_b200_shard_part_elements(esdg_b200_shard* s, int part, int64_t* count);

/* K3: q <- q + b k. Replaces Solver::axpy (solver.hpp:342-353). */
int esdg_b200_shard_axpy(esdg_b200_shard* s, double b, void* stream);

/* K5: synchronises `stream`, reads the non-physical-state flag raised by
 * K1/K2 (compute_node_vals, physics.hpp:63-64,72-73) and clears it. */
int esdg_b200_shard_check(esdg_b200_shard* s, void* stream,
                          esdg_b200_error* err);

/* K6: per-element reductions on the device; the state never leaves HBM.
 * kind 0: sum_n node_weight[n] q_var            (quadrature_total, diagnostics.hpp:30-47)
 *      1: sum_n node_weight[n] eta(q)           (total_entropy, diagnostics.hpp:49-71)
 *      2: sum_n node_weight[n] v(q) . k         (entropy_production, diagnostics.hpp:73-106)
 *      3: min_n,d dx[d][i_d] / (|u_d| + c)      (compute_stable_dt, time_integration.hpp:55-92)
 * evaluated per node in 64-bit as the reference writes them, Neumaier
 * compensated within the element; partials[e] receives one double per local
 * element (host memory, n_elements entries). node_weight = J w_a w_b w_c
 * (n3 doubles), dx = half element width times LGL node gap (3*nq doubles).
 * kind 0 reads register `reg`, the others the state register (and k).
 * *nonphysical is set when a node with rho <= 0 or p <= 0 was met. */
enum { ESDG_B200_REDUCE_QUADRATURE = 0, ESDG_B200_REDUCE_ENTROPY = 1,
       ESDG_B200_REDUCE_ENTROPY_PRODUCTION = 2, ESDG_B200_REDUCE_DT = 3 };
int esdg_b200_shard_reduce(esdg_b200_shard* s, int kind, int reg, int var,
                           const double* node_weight, const double* dx, double gamma,
                           double* partials, int32_t* nonphysical);

/* number of kernels this shard has launched since creation */
int64_t esdg_b200_shard_launch_count(const esdg_b200_shard* s);

/* ======================================================================= */
/* Level 2: host-side mirror of the reference interface                     */
/* ======================================================================= */

/* MeshConfig (mesh.hpp:12-22) */
typedef struct {
  int32_t base[3];
  int32_t refinement;
  double lo[3], hi[3];
  int32_t bc[3]; /* 0 periodic, 1 reflecting */
} esdg_b200_mesh_config;

/* Face (mesh.hpp:27-33) */
typedef struct {
  int32_t minus_elem, plus_elem;
  uint8_t dir, minus_side, reflecting, pad_;
} esdg_b200_face;

/* ExchangePlan::GhostFace (partition.hpp:28-35) */
typedef struct {
  int32_t face, peer, my_side, slot, my_inbox, peer_inbox;
} esdg_b200_ghost_face;

typedef struct esdg_b200_mesh esdg_b200_mesh;

/* MeshGeometry (mesh.cpp:11-132): Morton order + face connectivity */
int esdg_b200_mesh_create(const esdg_b200_mesh_config* cfg,
                          esdg_b200_mesh** out);
void esdg_b200_mesh_destroy(esdg_b200_mesh* m);
int64_t esdg_b200_mesh_num_elements(const esdg_b200_mesh* m);
int64_t esdg_b200_mesh_num_faces(const esdg_b200_mesh* m);
const int32_t* esdg_b200_mesh_lattice(const esdg_b200_mesh* m); /* ne*3 */
/* The face list is materialised on demand (it is not needed by the GPU
 * path, which uses the neighbour table). */
const esdg_b200_face* esdg_b200_mesh_faces(esdg_b200_mesh* m);
const int32_t* esdg_b200_mesh_face_of(esdg_b200_mesh* m); /* ne*6 */
/* neighbour table in GLOBAL element ids: >=0 element, -1 reflecting */
const int32_t* esdg_b200_mesh_neighbors(const esdg_b200_mesh* m); /* ne*6 */

/* ReferenceElement (reference_element.cpp:73-138) */
int esdg_b200_reference_element(int order, double* nodes, double* weights,
                                double* diff);
/* make_partition (partition.cpp:13-30); range_begin has ranks+1 entries */
int esdg_b200_partition(int64_t n_elements, int ranks, int64_t* range_begin);
/* build_exchange_plan (partition.cpp:32-66). Call with ghosts == NULL to get
 * the per-rank counts, then again with storage. Returns n_mailboxes or <0. */
int esdg_b200_exchange_plan(esdg_b200_mesh* m, int ranks, int32_t* ghost_count,
                            int32_t* interior_count,
                            esdg_b200_ghost_face* ghosts, int32_t* interior);
/* Host-only: the face roles of the one-pass kernels for a shard with the
 * neighbour codes nbr_local [n_elements][6] (as in esdg_b200_shard_desc) and
 * elements_per_group consecutive elements per CTA (esdg_b200_rhs_launch_shape).
 * roles[e]: bit f (0..2) = the lift term of face lf = 2f of e is pushed by the
 * element across it, bit 3+d = e pushes the term of its face lf = 2d+1. split
 * != 0: the table for the interior / boundary list launches (the interior
 * list runs first, so its elements may push to the boundary list's, never the
 * other way round). A face is shared only if the element that evaluates it
 * comes no later in the launch order than the one that takes the result; the
 * others, like walls and ghost faces, are evaluated by both sides -- to
 * bitwise the same number (the reference keeps one record per face for this,
 * compute_face_record, kernels.hpp:350-384). */
int esdg_b200_face_roles(const int32_t* nbr_local, int64_t n_elements,
                         int elements_per_group, int split, uint8_t* roles);
/* Host-only: the GPU-side slice of the exchange for partition `rank` of
 * `world_size`, i.e. exactly what esdg_b200_shard_create consumes. Ghost
 * faces are ordered by (peer, face) so that one contiguous block of traces
 * moves per peer and both ends enumerate a block identically. Call with the
 * array arguments NULL to obtain *n_peers and *n_ghost first.
 *   peer/offset/count [n_peers]: block of peer p is traces
 *                                [offset, offset+count) of BOTH the send and
 *                                the receive buffer of this rank
 *   send_elem/send_face [n_ghost]: local element and local face of slot g
 *   nbr_local [(end-begin)*6]: neighbour codes as in esdg_b200_shard_desc */
int esdg_b200_rank_halo(esdg_b200_mesh* m, int world_size, int rank,
                        int32_t* n_peers, int64_t* n_ghost, int32_t* peer,
                        int64_t* offset, int64_t* count, int32_t* send_elem,
                        int32_t* send_face, int32_t* nbr_local);
/* LsrkScheme (time_integration.hpp:17-37) */
void esdg_b200_lsrk_coefficients(double a[5], double b[5], double c[5]);

/* GasConstants<double> (constants.hpp:7-24) */
typedef struct {
  double gamma, R, p0, gravity;
} esdg_b200_gas;

/* KernelSettings<Real> (kernels.hpp:59-65). variant is fixed to balanced and
 * contravariant_direct to true on the GPU. */
typedef struct {
  int32_t dissipation;
  int32_t coriolis_mode; /* 0 none, 1 f-plane, 2 beta-plane */
  double f0, beta, y0;
} esdg_b200_settings;

enum {
  ESDG_B200_CASE_BUBBLE_SHARP = 0,  /* cases.hpp:43-69 */
  ESDG_B200_CASE_BUBBLE_SMOOTH = 1,
  ESDG_B200_CASE_HYDROSTATIC = 2,   /* cases.hpp:18-38 */
  ESDG_B200_CASE_ENTROPY_TEST = 3,  /* cases.hpp:120-156, iparam = seed */
  ESDG_B200_CASE_CONSTANT = 4,      /* test_helpers.hpp:41-52 */
  ESDG_B200_CASE_BAROCLINIC = 5,    /* ours; the reference ships none */
  /* Balanced zonal jet in a beta-plane channel after Ullrich, Reed and
   * Jablonowski (2015), the test PAPER.md:465-472 runs: geostrophic and
   * hydrostatic balance in pressure coordinates against the Coriolis
   * parameter of the solver's own settings (f0, beta, y0), plus a Gaussian
   * zonal-wind perturbation. dparam = {u0, u_pert, T0, lapse rate, b}; zeros
   * select 35 m/s, 1 m/s, 288 K, 0.005 K/m, 2; u_pert < 0: none. Ours as well (runner.cpp:70-74
   * has no channel state); the balance is what the tests check. */
  ESDG_B200_CASE_BAROCLINIC_JET = 6
};

enum {
  ESDG_B200_PATH_SPLIT = 0, /* K1 then K2, as the reference structures it */
  ESDG_B200_PATH_FUSED = 1, /* K1+K2 in one kernel */
  ESDG_B200_PATH_STAGE = 2  /* default. step(): K1+K2+K3 in one kernel per stage;
                               rhs()/assemble_rhs() behave like PATH_FUSED */
};

typedef struct esdg_b200_solver esdg_b200_solver;

/* Called by a distributed solver around the volume kernel of every RHS:
 * phase 0 after the pack kernel was enqueued (start moving send -> peers'
 * recv), phase 1 before the surface kernel (make `stream` wait for the
 * receives). Return 0 on success. */
typedef int (*esdg_b200_exchange_fn)(void* user, int phase, void* stream);

/* Solver(mesh, order, constants, settings, ranks) (solver.hpp:26-72).
 * `ranks` partitions live in this process; partition r runs on
 * devices[r % n_devices] (devices == NULL: device 0). */
int esdg_b200_solver_create(esdg_b200_mesh* mesh, int order,
                            const esdg_b200_gas* gas,
                            const esdg_b200_settings* settings, int precision,
                            int ranks, const int32_t* devices, int n_devices,
                            esdg_b200_solver** out);
/* One process per GPU: this process owns partition `rank` of `world_size`
 * and delegates the trace exchange to `exchange`. */
int esdg_b200_solver_create_distributed(
    esdg_b200_mesh* mesh, int order, const esdg_b200_gas* gas,
    const esdg_b200_settings* settings, int precision, int world_size,
    int rank, int device, esdg_b200_exchange_fn exchange, void* user,
    esdg_b200_solver** out);
/* One process per GPU with the trace exchange in the library itself: per RHS
 * one ncclSend/ncclRecv pair per peer inside one ncclGroup on the partition's
 * copy stream, behind the pack kernel, overlapped with the kernels of the
 * element groups that have no ghost face (replaces Transport<Real>::send /
 * wait, exchange.hpp:32-57, call sites solver.hpp:255,294). NCCL is bound at
 * run time (dlopen of libnccl.so.2). Rank 0 obtains a 128-byte unique id with
 * esdg_b200_nccl_unique_id, the host distributes it (MPI, torch.distributed,
 * a file ...) and every rank calls esdg_b200_solver_create_nccl -- a
 * collective -- with its own device current. */
int esdg_b200_nccl_unique_id(void* id128);
int esdg_b200_solver_create_nccl(esdg_b200_mesh* mesh, int order,
                                 const esdg_b200_gas* gas,
                                 const esdg_b200_settings* settings,
                                 int precision, int world_size, int rank,
                                 int device, const void* id128,
                                 esdg_b200_solver** out);
/* The exchange routine of the process-per-GPU path (one ncclRecv / ncclSend
 * pair per peer in one group on a stream, nccl_transport.cpp) run against
 * ITSELF: a one-rank communicator on `device`, `count` values of `precision`
 * (4 or 8) bytes sent to and received from rank 0 in one group, in two peer
 * blocks. *mismatches = values that did not arrive intact. All a one-GPU box
 * can show of the NCCL data plane. */
int esdg_b200_nccl_selftest(int device, int precision, int64_t count,
                            int64_t* mismatches);
/* NCCL_VERSION_CODE of the library bound by create_nccl (0: none) */
int esdg_b200_solver_nccl_version(const esdg_b200_solver* s);
void esdg_b200_solver_destroy(esdg_b200_solver* s);

int esdg_b200_solver_set_path(esdg_b200_solver* s, int path);
/* KernelSettings::variant (kernels.hpp:27-34, 59-65): the rung of the volume
 * kernel's optimisation ladder, 0 baseline .. 5 balanced (default). Rungs
 * below 4 select a ladder instance of K1 in volume_rhs / assemble_rhs (split
 * structure); step() on PATH_STAGE always runs the product kernel. */
int esdg_b200_solver_set_variant(esdg_b200_solver* s, int variant);
/* RankEvents (exchange.hpp:83-89, filled at solver.hpp:257-262,318-319): with
 * recording on, every RHS leaves a CUDA-event timeline per local partition;
 * rank_events returns, in ns since that partition's RHS was enqueued,
 * {sends_posted, volume_start, volume_end, wait_end, last_arrival} of the
 * last one (volume = the first kernel launch of the RHS: the volume kernel,
 * or the element groups without a ghost face on the one-pass paths). The
 * overlap property tests/test_partition.cpp:116-134 checks with a delayed
 * transport reads volume_start < last_arrival. */
int esdg_b200_solver_record_events(esdg_b200_solver* s, int on);
int esdg_b200_solver_rank_events(esdg_b200_solver* s, int rank, int64_t ns[5]);
/* Test hook, the analogue of Transport::send_hook (exchange.hpp:30): every
 * partition's trace transfer is held back by `microseconds` on its copy
 * stream (in-process copies and NCCL). Results must not change
 * (tests/test_partition.cpp:136-152); with recording on, the timeline shows
 * the kernels that do not need the traces running meanwhile. 0 = off. */
int esdg_b200_solver_set_exchange_delay(esdg_b200_solver* s, int microseconds);
/* bytes of face traces this process sends (and receives) per RHS */
int64_t esdg_b200_solver_halo_bytes(const esdg_b200_solver* s);
/* PATH_FUSED / PATH_STAGE with several partitions: on (default) runs the
 * element groups without a ghost face while the traces travel and the rest
 * after they have landed (rhs_job's order, solver.hpp:259-294); off waits for
 * the traces first and launches one kernel. Results are bitwise the same.
 * interior / total (may be null): elements of this process' partitions that
 * hide the exchange / all of them. */
int esdg_b200_solver_set_overlap(esdg_b200_solver* s, int on);
int esdg_b200_solver_overlap_elements(esdg_b200_solver* s, int64_t* interior,
                                      int64_t* total);
/* PATH_FUSED / PATH_STAGE: on (default) evaluates every interior face once --
 * by the element on its minus side, which hands the other element its share
 * through device memory -- the way the reference keeps one record per face
 * (compute_face_record, kernels.hpp:350-384; commit_face_side reads it for
 * both sides). Off: every element evaluates all six of its faces. Results are
 * bitwise the same either way and for every partition count. */
int esdg_b200_solver_set_face_sharing(esdg_b200_solver* s, int on);
int esdg_b200_solver_set_settings(esdg_b200_solver* s,
                                  const esdg_b200_settings* settings);
int64_t esdg_b200_solver_local_begin(const esdg_b200_solver* s);
int64_t esdg_b200_solver_local_end(const esdg_b200_solver* s);
int esdg_b200_solver_n3(const esdg_b200_solver* s);

/* distributed halo description: for peer p (0..n_peers-1) elements
 * [offset[p], offset[p]+count[p]) of the send/recv buffers (in traces of
 * 5*nq^2 Reals) belong to rank peer[p]. Returns n_peers. */
int esdg_b200_solver_halo(const esdg_b200_solver* s, int32_t* peer,
                          int64_t* offset, int64_t* count, int capacity);
/* compute stream of the (single) local partition, as cudaStream_t */
void* esdg_b200_solver_stream(esdg_b200_solver* s);
void* esdg_b200_solver_send_ptr(esdg_b200_solver* s);
void* esdg_b200_solver_recv_ptr(esdg_b200_solver* s);
int64_t esdg_b200_solver_n_ghost(const esdg_b200_solver* s);

/* init_state (solver.hpp:92-108) from a named case, evaluated in 64-bit on
 * the host exactly like the reference and uploaded; the host copy is kept
 * only when keep_host != 0. dparam: case parameters (may be NULL). */
int esdg_b200_solver_init_case(esdg_b200_solver* s, int case_id,
                               uint64_t iparam, const double* dparam);
/* The same generators at one point, host only (no device needed): q[5] at
 * (x, y, z) with phi = gravity * z. settings may be NULL (no Coriolis).
 * Returns ESDG_B200_BADARG when the generator leaves its domain. */
int esdg_b200_case_point(int case_id, const esdg_b200_mesh_config* mesh,
                         const esdg_b200_gas* gas,
                         const esdg_b200_settings* settings, uint64_t iparam,
                         const double* dparam, double x, double y, double z,
                         double q[5]);
/* state()/k register as host StateField arrays of the LOCAL element range */
int esdg_b200_solver_set_state(esdg_b200_solver* s, int reg, const void* host);
int esdg_b200_solver_get_state(esdg_b200_solver* s, int reg, void* host);
/* get_state into host_out and set_state from host_in in one full-duplex,
 * chunk-pipelined pass (the upload of a chunk waits for its own download
 * only): what a coupled driver does between two steps when it hands state()
 * to host code and takes it back. host_in may alias host_out. Pinned host
 * memory is needed for the two directions to overlap. */
int esdg_b200_solver_swap_state(esdg_b200_solver* s, int reg, const void* host_in,
                                void* host_out);
/* esdg_b200_solver_step followed by esdg_b200_solver_swap_state(REG_Q, ...),
 * with the last LSRK stage cut into runs of elements so that finished runs
 * leave for host_out while the rest of the stage is still computing; the same
 * result bitwise. check != 0: report a non-physical state like
 * esdg_b200_solver_step does (after the transfers). */
int esdg_b200_solver_step_swap(esdg_b200_solver* s, double dt,
                               const void* host_in, void* host_out, int check);
/* Streaming of INDEPENDENT states (ensemble members, the samples of a batch)
 * through one solver: one LSRK step of the state on the device (as
 * esdg_b200_solver_step, solver.hpp:132-146) while host_in_next -- the state
 * of the next call -- is uploaded and the previous call's result is
 * downloaded to host_out_prev, each transfer on its own stream and copy
 * engine. step_swap's coupled contract (the next input is this output) can
 * not overlap LSRK stages 1-4 with a transfer; independent states can, and a
 * call costs max(step, transfer).
 *   host_in_next  != NULL: is REG_Q when the call returns, and this step's
 *                          result stays parked on the device until the next
 *                          call (or esdg_b200_solver_stream_collect) takes it;
 *   host_in_next  == NULL: REG_Q is this step's result, as after solver_step;
 *   host_out_prev          must be non-NULL exactly when a result is parked.
 * Results are bitwise those of esdg_b200_solver_step on the same state. Any
 * path and partition count; the host arrays cover the LOCAL element range as
 * for set_state / get_state. ESDG_B200_BADARG when the parked-result protocol
 * is broken. Pinned host memory is needed for the transfers to overlap. check as in esdg_b200_solver_step
 * (refers to the state this call stepped). */
int esdg_b200_solver_step_stream(esdg_b200_solver* s, double dt,
                                 const void* host_in_next, void* host_out_prev,
                                 int check);
/* delivers the parked result of the last esdg_b200_solver_step_stream call */
int esdg_b200_solver_stream_collect(esdg_b200_solver* s, void* host_out);
/* phi() (solver.hpp:79), local range */
int esdg_b200_solver_get_phi(esdg_b200_solver* s, void* host);

/* assemble_rhs(q, out, a_old, a_new) with HOST fields (solver.hpp:112-119):
 * uploads q (and out when a_old != 0), runs the RHS, downloads out. */
int esdg_b200_solver_assemble_rhs(esdg_b200_solver* s, const void* q_host,
                                  void* out_host, double a_old, double a_new);
/* volume_rhs(q, out) (solver.hpp:122-129) */
int esdg_b200_solver_volume_rhs(esdg_b200_solver* s, const void* q_host,
                                void* out_host);
/* device-resident: k <- a_old k + a_new RHS(q) on the internal registers */
int esdg_b200_solver_rhs(esdg_b200_solver* s, double a_old, double a_new,
                         int stage);
/* axpy(b) (solver.hpp:342-353) */
int esdg_b200_solver_axpy(esdg_b200_solver* s, double b);
/* step(dt) (solver.hpp:132-146): 5 x (rhs, axpy), device resident. With
 * check != 0 the non-physical flag is read after the step (one sync). */
int esdg_b200_solver_step(esdg_b200_solver* s, double dt, int check);
/* blocks until all queued work of this solver has finished */
int esdg_b200_solver_sync(esdg_b200_solver* s);
/* compute_dt(courant) (solver.hpp:148-150, time_integration.hpp:55-92);
 * local minimum for a distributed solver */
int esdg_b200_solver_compute_dt(esdg_b200_solver* s, double courant,
                                double* dt);
int esdg_b200_solver_last_error(const esdg_b200_solver* s,
                                esdg_b200_error* err);

/* diagnostics on the local range (diagnostics.hpp:30-106) and compute_dt.
 * ESDG_B200_REDUCE_ON_DEVICE (default): K6 evaluates the per-node terms on
 * the GPU and sums them per element with Neumaier compensation; one double
 * per element crosses PCIe and the host finishes with a compensated sum in
 * Morton order. compute_dt is then bitwise the reference's value (a minimum
 * is order independent), the sums agree to rounding of the result.
 * ESDG_B200_REDUCE_ON_HOST: the registers are streamed back chunk by chunk
 * and reduced on the host cores with the reference's Neumaier sum in the
 * reference's order (bitwise the reference's values, at the price of moving
 * the state). entropy_production pairs v(q register) with the k register. */
enum { ESDG_B200_REDUCE_ON_DEVICE = 0, ESDG_B200_REDUCE_ON_HOST = 1 };
int esdg_b200_solver_set_reduction(esdg_b200_solver* s, int mode);
int esdg_b200_solver_quadrature_total(esdg_b200_solver* s, int reg, int var,
                                      double* out);
int esdg_b200_solver_total_entropy(esdg_b200_solver* s, double* out);
int esdg_b200_solver_entropy_production(esdg_b200_solver* s, double* out);

/* PerfRecord-like device timings (diagnostics.hpp:125-139) accumulated by
 * CUDA events when enabled: seconds[0..3] = volume, surface, update, pack;
 * launches = kernels launched by this solver so far. */
int esdg_b200_solver_enable_timing(esdg_b200_solver* s, int on);
int esdg_b200_solver_timers(esdg_b200_solver* s, double seconds[4],
                            int64_t* launches, int reset);

/* Device self-test of the arithmetic the kernels rely on (esdg_device.cuh):
 * out5 = {max error of the fast reciprocal in ulps, samples violating
 * rcp(2x) == rcp(x)/2, 1 if rcp(1) == 1 exactly, samples tested, max
 * difference of the kernels' logarithm to the CUDA library's in ulps}. */
int esdg_b200_selftest(int device, int precision, double out5[5]);

/* DFMA / FFMA peak micro-benchmark on `device` (the roofline denominator of
 * K1; MEASURED_PEAKS.json has no CUDA-core figure). Returns TFLOP/s. */
int esdg_b200_measure_fma_peak(int device, int precision, double* tflops);

/* The same with three distinct vector-register operands per FMA. On sm_100 an
 * FP64 instruction of that shape holds the pipe for three cycles instead of
 * two, so this (about 2/3 of the figure above for FP64) is what general FP64
 * code can reach; reported next to the nominal peak, never instead of it. */
int esdg_b200_measure_fma3_peak(int device, int precision, double* tflops);

#ifdef __cplusplus
}
#endif
#endif
