// host_types.hpp -- host-side mirror of the reference's mesh / operator /
// partition types for the level-2 entry points (include/esdg_b200.h).
//
// Same semantics as the reference's
//   MeshGeometry      core/include/esdg/mesh.hpp:38-98, core/src/mesh.cpp
//   ReferenceElement  core/include/esdg/reference_element.hpp, .cpp
//   Partition, ExchangePlan  core/include/esdg/partition.hpp, partition.cpp
// but laid out for feeding GPUs: the primary connectivity product is a flat
// neighbour table (6 int32 per element); the reference's Face list is only
// materialised when a caller asks for it.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <vector>

#include "esdg_b200.h"

namespace esdg_b200 {
namespace host {

struct Mesh {
  esdg_b200_mesh_config cfg{};
  std::array<int32_t, 3> dims{};
  std::array<double, 3> delta{};
  double jacobian = 0.0;
  int64_t ne = 0;
  std::vector<int32_t> lattice; // ne*3
  std::vector<int32_t> elem_at; // lattice index -> element
  std::vector<int32_t> nbr;     // ne*6, global ids, -1 reflecting
  // reference-compatible face list, built on demand
  std::vector<esdg_b200_face> faces;
  std::vector<int32_t> face_of;
  bool faces_built = false;

  static std::unique_ptr<Mesh> create(const esdg_b200_mesh_config& cfg);
  void build_faces();
  double metric(int d) const { return 2.0 / delta[size_t(d)]; }
  // mesh.hpp:73-77
  double node_coordinate(int64_t e, int d, double ref_node) const {
    return cfg.lo[d] +
           (double(lattice[size_t(e) * 3 + size_t(d)]) + 0.5 * (ref_node + 1.0)) *
               delta[size_t(d)];
  }
};

struct RefElement {
  int order = 0, nq = 0;
  std::vector<double> nodes, weights, diff;
  static bool build(int order, RefElement& out);
};

// make_partition (partition.cpp:13-30)
bool make_partition(int64_t ne, int ranks, std::vector<int64_t>& range_begin);
inline int rank_of(const std::vector<int64_t>& rb, int64_t e) {
  int lo = 0, hi = int(rb.size()) - 1; // rb[lo] <= e < rb[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) / 2;
    if (e >= rb[size_t(mid)]) lo = mid; else hi = mid;
  }
  return lo;
}

// One rank's slice of the exchange, in the order the GPU path uses it:
// ghost faces sorted by (peer, global face order), so that the send buffer of
// rank A toward B and the receive buffer of B from A enumerate the shared
// faces identically and one contiguous block moves per peer.
struct RankHalo {
  struct Peer {
    int rank;
    int64_t offset, count; // in traces, identical on the send and recv side
  };
  std::vector<Peer> peers;
  std::vector<int32_t> send_elem, send_face; // local element, local face
  std::vector<int32_t> ghost_remote_elem;    // global id of the remote element
  std::vector<int32_t> ghost_remote_face;    // its local face (dir*2+side)
  std::vector<int32_t> nbr_local;            // (end-begin)*6 shard codes
};

// Builds the per-rank neighbour codes and halo lists for rank `r`.
void build_rank_halo(const Mesh& m, const std::vector<int64_t>& rb, int r,
                     RankHalo& out);

// Face roles of the one-pass kernels (dev::RhsParams::face_roles). nbr: the
// shard's neighbour codes [ne][6] (>= 0 local element, < 0 wall or ghost);
// epb: elements per group (CTA). The face between A (its + face, lf odd) and
// B (its - face, lf - 1) is always evaluated by A; B takes A's result instead
// of evaluating the face a second time (bit f of roles[B], f = lf / 2; bit
// 3 + f of roles[A] tells A to push it) when A's group is dispatched no later
// than B's: A < B for a launch over all groups or over consecutive runs of
// them (split == false); for the interior / boundary launches (split == true)
// A < B inside a list, and between the lists A in the interior list (which
// is launched, and has finished, before the boundary list). Everything else
// -- walls, ghost faces, periodic wrap-around (A has the higher index there),
// a boundary-list A next to an interior-list B -- B evaluates itself.
void build_face_roles(const int32_t* nbr, int64_t ne, int epb, bool split, uint8_t* roles);

// Named initial conditions (cases.hpp of the reference + our baroclinic one).
struct CaseEval {
  int case_id = 0;
  esdg_b200_gas gas{};
  esdg_b200_mesh_config mesh{};
  esdg_b200_settings settings{}; // the balanced jet reads the Coriolis parameter
  uint64_t iparam = 0;
  double dparam[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  // entropy-test Fourier fields
  int k[5][3][3];
  double amp[5][3], phase[5][3];
  bool prepare();
  bool point(double x, double y, double z, double phi, double q[5]) const;
};

void lsrk_coefficients(double a[5], double b[5], double c[5]);

} // namespace host
} // namespace esdg_b200
