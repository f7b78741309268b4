// capi.cpp -- level-2 C ABI (include/esdg_b200.h): the host-side mirror of
// the reference's mesh / partition / Solver interface behind C handles.
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "esdg_b200.h"
#include "host_types.hpp"
#include "solver_core.hpp"

using esdg_b200::host::Mesh;
using esdg_b200::host::SolverCore;

struct esdg_b200_mesh {
  std::unique_ptr<Mesh> m;
};
struct esdg_b200_solver {
  SolverCore* core;
};

extern "C" {

int esdg_b200_mesh_create(const esdg_b200_mesh_config* cfg, esdg_b200_mesh** out) {
  if (!cfg || !out) return ESDG_B200_BADARG;
  auto m = Mesh::create(*cfg);
  if (!m) {
    esdg_b200::set_message("mesh_create: invalid configuration");
    return ESDG_B200_BADARG;
  }
  *out = new esdg_b200_mesh{std::move(m)};
  return ESDG_B200_OK;
}
void esdg_b200_mesh_destroy(esdg_b200_mesh* m) { delete m; }
int64_t esdg_b200_mesh_num_elements(const esdg_b200_mesh* m) { return m ? m->m->ne : 0; }
int64_t esdg_b200_mesh_num_faces(const esdg_b200_mesh* m) {
  if (!m) return 0;
  const_cast<Mesh*>(m->m.get())->build_faces();
  return int64_t(m->m->faces.size());
}
const int32_t* esdg_b200_mesh_lattice(const esdg_b200_mesh* m) {
  return m ? m->m->lattice.data() : nullptr;
}
const esdg_b200_face* esdg_b200_mesh_faces(esdg_b200_mesh* m) {
  if (!m) return nullptr;
  m->m->build_faces();
  return m->m->faces.data();
}
const int32_t* esdg_b200_mesh_face_of(esdg_b200_mesh* m) {
  if (!m) return nullptr;
  m->m->build_faces();
  return m->m->face_of.data();
}
const int32_t* esdg_b200_mesh_neighbors(const esdg_b200_mesh* m) {
  return m ? m->m->nbr.data() : nullptr;
}

int esdg_b200_reference_element(int order, double* nodes, double* weights, double* diff) {
  esdg_b200::host::RefElement r;
  if (!nodes || !weights || !diff || !esdg_b200::host::RefElement::build(order, r))
    return ESDG_B200_BADARG;
  std::memcpy(nodes, r.nodes.data(), sizeof(double) * r.nodes.size());
  std::memcpy(weights, r.weights.data(), sizeof(double) * r.weights.size());
  std::memcpy(diff, r.diff.data(), sizeof(double) * r.diff.size());
  return ESDG_B200_OK;
}

int esdg_b200_partition(int64_t n_elements, int ranks, int64_t* range_begin) {
  std::vector<int64_t> rb;
  if (!range_begin || !esdg_b200::host::make_partition(n_elements, ranks, rb))
    return ESDG_B200_BADARG;
  std::memcpy(range_begin, rb.data(), sizeof(int64_t) * rb.size());
  return ESDG_B200_OK;
}

// build_exchange_plan (partition.cpp:32-66): faces in id order; a face whose
// two elements sit on different ranks becomes a ghost face of both, with a
// crossed pair of mailboxes.
int esdg_b200_exchange_plan(esdg_b200_mesh* m, int ranks, int32_t* ghost_count,
                            int32_t* interior_count, esdg_b200_ghost_face* ghosts,
                            int32_t* interior) {
  if (!m) return -1;
  Mesh& mesh = *m->m;
  std::vector<int64_t> rb;
  if (!esdg_b200::host::make_partition(mesh.ne, ranks, rb)) return -1;
  mesh.build_faces();
  std::vector<int32_t> gc(size_t(ranks), 0), ic(size_t(ranks), 0);
  auto classify = [&](const esdg_b200_face& f, int& rm, int& rp) {
    rm = esdg_b200::host::rank_of(rb, f.minus_elem);
    rp = (f.reflecting || f.plus_elem < 0) ? rm : esdg_b200::host::rank_of(rb, f.plus_elem);
    return rp != rm;
  };
  for (const auto& f : mesh.faces) {
    int rm, rp;
    if (classify(f, rm, rp)) {
      ++gc[size_t(rm)];
      ++gc[size_t(rp)];
    } else {
      ++ic[size_t(rm)];
    }
  }
  int n_pairs = 0;
  for (int r = 0; r < ranks; ++r) n_pairs += gc[size_t(r)];
  n_pairs /= 2;
  if (ghosts && interior) {
    std::vector<int32_t> goff(size_t(ranks) + 1, 0), ioff(size_t(ranks) + 1, 0);
    for (int r = 0; r < ranks; ++r) {
      goff[size_t(r) + 1] = goff[size_t(r)] + gc[size_t(r)];
      ioff[size_t(r) + 1] = ioff[size_t(r)] + ic[size_t(r)];
    }
    std::vector<int32_t> gn(size_t(ranks), 0), in(size_t(ranks), 0);
    int pair = 0;
    for (int32_t id = 0; id < int32_t(mesh.faces.size()); ++id) {
      int rm, rp;
      if (!classify(mesh.faces[size_t(id)], rm, rp)) {
        interior[ioff[size_t(rm)] + in[size_t(rm)]++] = id;
        continue;
      }
      const int32_t box_m = 2 * pair, box_p = 2 * pair + 1;
      ghosts[goff[size_t(rm)] + gn[size_t(rm)]] = {id, rp, 0, gn[size_t(rm)], box_m, box_p};
      ++gn[size_t(rm)];
      ghosts[goff[size_t(rp)] + gn[size_t(rp)]] = {id, rm, 1, gn[size_t(rp)], box_p, box_m};
      ++gn[size_t(rp)];
      ++pair;
    }
  }
  for (int r = 0; r < ranks; ++r) {
    if (ghost_count) ghost_count[r] = gc[size_t(r)];
    if (interior_count) interior_count[r] = ic[size_t(r)];
  }
  return 2 * n_pairs;
}

int esdg_b200_rank_halo(esdg_b200_mesh* m, int world_size, int rank, int32_t* n_peers,
                        int64_t* n_ghost, int32_t* peer, int64_t* offset, int64_t* count,
                        int32_t* send_elem, int32_t* send_face, int32_t* nbr_local) {
  if (!m || !n_peers || !n_ghost || rank < 0 || rank >= world_size) return ESDG_B200_BADARG;
  std::vector<int64_t> rb;
  if (!esdg_b200::host::make_partition(m->m->ne, world_size, rb)) return ESDG_B200_BADARG;
  esdg_b200::host::RankHalo h;
  esdg_b200::host::build_rank_halo(*m->m, rb, rank, h);
  *n_peers = int32_t(h.peers.size());
  *n_ghost = int64_t(h.send_elem.size());
  for (size_t i = 0; i < h.peers.size(); ++i) {
    if (peer) peer[i] = h.peers[i].rank;
    if (offset) offset[i] = h.peers[i].offset;
    if (count) count[i] = h.peers[i].count;
  }
  if (send_elem) std::memcpy(send_elem, h.send_elem.data(), sizeof(int32_t) * h.send_elem.size());
  if (send_face) std::memcpy(send_face, h.send_face.data(), sizeof(int32_t) * h.send_face.size());
  if (nbr_local) std::memcpy(nbr_local, h.nbr_local.data(), sizeof(int32_t) * h.nbr_local.size());
  return ESDG_B200_OK;
}

void esdg_b200_lsrk_coefficients(double a[5], double b[5], double c[5]) {
  esdg_b200::host::lsrk_coefficients(a, b, c);
}

// ---- solver ---------------------------------------------------------------

static int make_solver(esdg_b200_mesh* mesh, SolverCore::Options& opt,
                       esdg_b200_solver** out) {
  if (!mesh || !out) return ESDG_B200_BADARG;
  SolverCore* core = nullptr;
  const int rc = SolverCore::create(mesh->m.get(), opt, &core);
  if (rc != ESDG_B200_OK) return rc;
  *out = new esdg_b200_solver{core};
  return ESDG_B200_OK;
}

int esdg_b200_solver_create(esdg_b200_mesh* mesh, int order, const esdg_b200_gas* gas,
                            const esdg_b200_settings* settings, int precision, int ranks,
                            const int32_t* devices, int n_devices, esdg_b200_solver** out) {
  if (!gas || !settings || ranks < 1) return ESDG_B200_BADARG;
  SolverCore::Options opt;
  opt.order = order;
  opt.precision = precision;
  opt.gas = *gas;
  opt.settings = *settings;
  opt.world_size = ranks;
  for (int r = 0; r < ranks; ++r) {
    opt.local_ranks.push_back(r);
    opt.devices.push_back((devices && n_devices > 0) ? devices[r % n_devices] : 0);
  }
  return make_solver(mesh, opt, out);
}

int esdg_b200_solver_create_distributed(esdg_b200_mesh* mesh, int order,
                                        const esdg_b200_gas* gas,
                                        const esdg_b200_settings* settings, int precision,
                                        int world_size, int rank, int device,
                                        esdg_b200_exchange_fn exchange, void* user,
                                        esdg_b200_solver** out) {
  if (!gas || !settings || world_size < 1 || rank < 0 || rank >= world_size)
    return ESDG_B200_BADARG;
  if (world_size > 1 && !exchange) {
    esdg_b200::set_message("create_distributed: world_size > 1 needs an exchange callback");
    return ESDG_B200_BADARG;
  }
  SolverCore::Options opt;
  opt.order = order;
  opt.precision = precision;
  opt.gas = *gas;
  opt.settings = *settings;
  opt.world_size = world_size;
  opt.local_ranks = {rank};
  opt.devices = {device};
  opt.exchange = exchange;
  opt.exchange_user = user;
  return make_solver(mesh, opt, out);
}

int esdg_b200_nccl_unique_id(void* id128) {
  if (!id128) return ESDG_B200_BADARG;
  std::string why;
  if (!esdg_b200::host::NcclTransport::unique_id(id128, &why)) {
    esdg_b200::set_message("nccl_unique_id: " + why);
    return ESDG_B200_CUDA;
  }
  return ESDG_B200_OK;
}

int esdg_b200_nccl_selftest(int device, int precision, int64_t count, int64_t* mismatches) {
  if ((precision != 4 && precision != 8) || count < 2 || !mismatches) {
    esdg_b200::set_message("nccl_selftest: bad argument");
    return ESDG_B200_BADARG;
  }
  *mismatches = -1;
  std::string why;
  char id[esdg_b200::host::kNcclUniqueIdBytes];
  if (cudaSetDevice(device) != cudaSuccess) {
    esdg_b200::set_message("nccl_selftest: cudaSetDevice failed");
    return ESDG_B200_CUDA;
  }
  esdg_b200::host::NcclTransport t;
  if (!esdg_b200::host::NcclTransport::unique_id(id, &why) || !t.init(1, 0, id, &why)) {
    esdg_b200::set_message("nccl_selftest: " + why);
    return ESDG_B200_CUDA;
  }
  const size_t bytes = size_t(count) * size_t(precision);
  std::vector<unsigned char> h_send(bytes), h_recv(bytes, 0);
  for (size_t i = 0; i < bytes; ++i) h_send[i] = static_cast<unsigned char>(i * 131u + 7u);
  void *d_send = nullptr, *d_recv = nullptr;
  cudaStream_t st = nullptr;
  bool ok = cudaMalloc(&d_send, bytes) == cudaSuccess && cudaMalloc(&d_recv, bytes) == cudaSuccess &&
            cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) == cudaSuccess &&
            cudaMemcpy(d_send, h_send.data(), bytes, cudaMemcpyHostToDevice) == cudaSuccess &&
            cudaMemset(d_recv, 0, bytes) == cudaSuccess &&
            cudaDeviceSynchronize() == cudaSuccess; // the exchange runs on a non-blocking stream
  if (ok) {
    // two peer blocks, both "peers" being this rank: what a partition with
    // two neighbours issues per RHS
    const long long half = count / 2;
    const long long off[2] = {0, half}, cnt[2] = {half, count - half};
    const int peer[2] = {0, 0};
    ok = t.exchange(d_send, d_recv, off, cnt, peer, 2, precision, st, &why) &&
         cudaStreamSynchronize(st) == cudaSuccess &&
         cudaMemcpy(h_recv.data(), d_recv, bytes, cudaMemcpyDeviceToHost) == cudaSuccess;
  }
  if (st) cudaStreamDestroy(st);
  cudaFree(d_send);
  cudaFree(d_recv);
  if (!ok) {
    esdg_b200::set_message("nccl_selftest: " + (why.empty() ? std::string("CUDA error") : why));
    return ESDG_B200_CUDA;
  }
  int64_t bad = 0;
  for (int64_t i = 0; i < count; ++i)
    if (std::memcmp(&h_send[size_t(i) * precision], &h_recv[size_t(i) * precision], size_t(precision)) != 0) ++bad;
  *mismatches = bad;
  return ESDG_B200_OK;
}

int esdg_b200_solver_create_nccl(esdg_b200_mesh* mesh, int order, const esdg_b200_gas* gas,
                                 const esdg_b200_settings* settings, int precision,
                                 int world_size, int rank, int device, const void* id128,
                                 esdg_b200_solver** out) {
  if (!gas || !settings || !id128 || world_size < 1 || rank < 0 || rank >= world_size)
    return ESDG_B200_BADARG;
  SolverCore::Options opt;
  opt.order = order;
  opt.precision = precision;
  opt.gas = *gas;
  opt.settings = *settings;
  opt.world_size = world_size;
  opt.local_ranks = {rank};
  opt.devices = {device};
  opt.nccl = true;
  std::memcpy(opt.nccl_id, id128, sizeof opt.nccl_id);
  return make_solver(mesh, opt, out);
}

void esdg_b200_solver_destroy(esdg_b200_solver* s) {
  if (!s) return;
  delete s->core;
  delete s;
}

#define CORE(s) if (!(s)) return ESDG_B200_BADARG; SolverCore& c = *(s)->core

int esdg_b200_face_roles(const int32_t* nbr_local, int64_t n_elements, int elements_per_group,
                         int split, uint8_t* roles) {
  if (!nbr_local || !roles || n_elements < 0 || elements_per_group < 1) {
    esdg_b200::set_message("face_roles: bad argument");
    return ESDG_B200_BADARG;
  }
  esdg_b200::host::build_face_roles(nbr_local, n_elements, elements_per_group, split != 0, roles);
  return ESDG_B200_OK;
}

int esdg_b200_solver_set_path(esdg_b200_solver* s, int path) { CORE(s); return c.set_path(path); }
int esdg_b200_solver_set_variant(esdg_b200_solver* s, int variant) { CORE(s); return c.set_variant(variant); }
int esdg_b200_solver_record_events(esdg_b200_solver* s, int on) { CORE(s); return c.record_events(on != 0); }
int esdg_b200_solver_rank_events(esdg_b200_solver* s, int rank, int64_t ns[5]) {
  CORE(s);
  return c.rank_events(rank, ns);
}
int esdg_b200_solver_set_exchange_delay(esdg_b200_solver* s, int microseconds) {
  CORE(s);
  c.set_exchange_delay(microseconds);
  return ESDG_B200_OK;
}
int64_t esdg_b200_solver_halo_bytes(const esdg_b200_solver* s) {
  return s ? s->core->halo_bytes_per_rhs() : 0;
}
int esdg_b200_solver_nccl_version(const esdg_b200_solver* s) { return s ? s->core->nccl_version() : 0; }
int esdg_b200_solver_set_overlap(esdg_b200_solver* s, int on) {
  CORE(s);
  c.set_overlap(on != 0);
  return ESDG_B200_OK;
}
int esdg_b200_solver_set_face_sharing(esdg_b200_solver* s, int on) {
  CORE(s);
  c.set_face_sharing(on != 0);
  return ESDG_B200_OK;
}
int esdg_b200_solver_overlap_elements(esdg_b200_solver* s, int64_t* interior, int64_t* total) {
  CORE(s);
  c.overlap_elements(interior, total);
  return ESDG_B200_OK;
}
int esdg_b200_solver_set_settings(esdg_b200_solver* s, const esdg_b200_settings* st) {
  CORE(s);
  return st ? c.set_settings(*st) : ESDG_B200_BADARG;
}
int64_t esdg_b200_solver_local_begin(const esdg_b200_solver* s) { return s ? s->core->local_begin() : 0; }
int64_t esdg_b200_solver_local_end(const esdg_b200_solver* s) { return s ? s->core->local_end() : 0; }
int esdg_b200_solver_n3(const esdg_b200_solver* s) { return s ? s->core->n3() : 0; }
int esdg_b200_solver_halo(const esdg_b200_solver* s, int32_t* peer, int64_t* offset,
                          int64_t* count, int capacity) {
  return s ? s->core->halo(peer, offset, count, capacity) : 0;
}
void* esdg_b200_solver_stream(esdg_b200_solver* s) {
  return (s && s->core->n_shards() >= 1) ? s->core->shard(0)->stream() : nullptr;
}
void* esdg_b200_solver_send_ptr(esdg_b200_solver* s) {
  return (s && s->core->n_shards() == 1) ? s->core->shard(0)->send_ptr() : nullptr;
}
void* esdg_b200_solver_recv_ptr(esdg_b200_solver* s) {
  return (s && s->core->n_shards() == 1) ? s->core->shard(0)->recv_ptr() : nullptr;
}
int64_t esdg_b200_solver_n_ghost(const esdg_b200_solver* s) {
  return (s && s->core->n_shards() == 1) ? s->core->shard(0)->n_ghost() : 0;
}

int esdg_b200_case_point(int case_id, const esdg_b200_mesh_config* mesh,
                         const esdg_b200_gas* gas, const esdg_b200_settings* settings,
                         uint64_t iparam, const double* dparam, double x, double y, double z,
                         double q[5]) {
  if (!mesh || !gas || !q) return ESDG_B200_BADARG;
  esdg_b200::host::CaseEval ce;
  ce.case_id = case_id;
  ce.gas = *gas;
  ce.mesh = *mesh;
  if (settings) ce.settings = *settings;
  ce.iparam = iparam;
  if (dparam)
    for (int i = 0; i < 5; ++i) ce.dparam[i] = dparam[i];
  if (!ce.prepare()) {
    esdg_b200::set_message("case_point: unknown case");
    return ESDG_B200_BADARG;
  }
  if (!ce.point(x, y, z, gas->gravity * z, q)) {
    esdg_b200::set_message("case_point: state generator left its domain");
    return ESDG_B200_BADARG;
  }
  return ESDG_B200_OK;
}

int esdg_b200_solver_init_case(esdg_b200_solver* s, int case_id, uint64_t iparam,
                               const double* dparam) {
  CORE(s);
  return c.init_case(case_id, iparam, dparam);
}
int esdg_b200_solver_set_state(esdg_b200_solver* s, int reg, const void* host) {
  CORE(s);
  return c.set_state(reg, host);
}
int esdg_b200_solver_swap_state(esdg_b200_solver* s, int reg, const void* host_in, void* host_out) {
  CORE(s);
  return c.swap_state(reg, host_in, host_out);
}
int esdg_b200_solver_get_state(esdg_b200_solver* s, int reg, void* host) {
  CORE(s);
  return c.get_state(reg, host);
}
int esdg_b200_solver_get_phi(esdg_b200_solver* s, void* host) { CORE(s); return c.get_phi(host); }

int esdg_b200_solver_assemble_rhs(esdg_b200_solver* s, const void* q_host, void* out_host,
                                  double a_old, double a_new) {
  CORE(s);
  return c.assemble_rhs_host(q_host, out_host, a_old, a_new, false);
}
int esdg_b200_solver_volume_rhs(esdg_b200_solver* s, const void* q_host, void* out_host) {
  CORE(s);
  return c.assemble_rhs_host(q_host, out_host, 0.0, 1.0, true);
}
int esdg_b200_solver_rhs(esdg_b200_solver* s, double a_old, double a_new, int stage) {
  CORE(s);
  return c.rhs(ESDG_B200_REG_Q, ESDG_B200_REG_K, a_old, a_new, true, false, stage);
}
int esdg_b200_solver_axpy(esdg_b200_solver* s, double b) { CORE(s); return c.axpy(b); }
int esdg_b200_solver_step(esdg_b200_solver* s, double dt, int check) {
  CORE(s);
  return c.step(dt, check != 0);
}
int esdg_b200_solver_step_swap(esdg_b200_solver* s, double dt, const void* host_in, void* host_out,
                               int check) {
  CORE(s);
  return c.step_swap(dt, host_in, host_out, check != 0);
}
int esdg_b200_solver_step_stream(esdg_b200_solver* s, double dt, const void* host_in_next,
                                 void* host_out_prev, int check) {
  CORE(s);
  return c.step_stream(dt, host_in_next, host_out_prev, check != 0);
}
int esdg_b200_solver_stream_collect(esdg_b200_solver* s, void* host_out) {
  CORE(s);
  return c.stream_collect(host_out);
}
int esdg_b200_solver_sync(esdg_b200_solver* s) { CORE(s); return c.sync(); }
int esdg_b200_solver_compute_dt(esdg_b200_solver* s, double courant, double* dt) {
  CORE(s);
  return dt ? c.compute_dt(courant, dt) : ESDG_B200_BADARG;
}
int esdg_b200_solver_last_error(const esdg_b200_solver* s, esdg_b200_error* err) {
  if (!s || !err) return ESDG_B200_BADARG;
  *err = s->core->last_error();
  return ESDG_B200_OK;
}
int esdg_b200_solver_quadrature_total(esdg_b200_solver* s, int reg, int var, double* out) {
  CORE(s);
  return out ? c.quadrature_total(reg, var, out) : ESDG_B200_BADARG;
}
int esdg_b200_solver_total_entropy(esdg_b200_solver* s, double* out) {
  CORE(s);
  return out ? c.total_entropy(out) : ESDG_B200_BADARG;
}
int esdg_b200_solver_entropy_production(esdg_b200_solver* s, double* out) {
  CORE(s);
  return out ? c.entropy_production(out) : ESDG_B200_BADARG;
}
int esdg_b200_solver_set_reduction(esdg_b200_solver* s, int mode) {
  CORE(s);
  return c.set_reduction(mode);
}
int esdg_b200_solver_enable_timing(esdg_b200_solver* s, int on) {
  CORE(s);
  return c.enable_timing(on != 0);
}
int esdg_b200_solver_timers(esdg_b200_solver* s, double seconds[4], int64_t* launches, int reset) {
  CORE(s);
  return c.timers(seconds, launches, reset != 0);
}

} // extern "C"
