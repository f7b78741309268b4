// mesh.cpp -- uniform brick mesh in global Morton order; neighbour table for
// the GPU path, reference-compatible face list on demand.
// Semantics follow core/src/mesh.cpp:11-132 and core/include/esdg/morton.hpp
// of the reference (validated against it in tests/test_host_mirror.py).
#include <algorithm>
#include <numeric>

#include "host_types.hpp"

namespace esdg_b200 {
namespace host {

namespace {

// x-fastest bit interleave of three 21-bit coordinates (morton.hpp:9-26)
uint64_t dilate3(uint64_t v) {
  v &= (1ull << 21) - 1;
  v = (v | (v << 32)) & 0x001f00000000ffffull;
  v = (v | (v << 16)) & 0x001f0000ff0000ffull;
  v = (v | (v << 8)) & 0x100f00f00f00f00full;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}

} // namespace

std::unique_ptr<Mesh> Mesh::create(const esdg_b200_mesh_config& cfg) {
  for (int d = 0; d < 3; ++d)
    if (cfg.base[d] < 1 || !(cfg.hi[d] > cfg.lo[d]) ||
        (cfg.bc[d] != 0 && cfg.bc[d] != 1))
      return nullptr;
  if (cfg.refinement < 0 || cfg.refinement > 20) return nullptr;

  auto m = std::make_unique<Mesh>();
  m->cfg = cfg;
  int64_t ne = 1;
  for (int d = 0; d < 3; ++d) {
    const int64_t n = int64_t(cfg.base[d]) << cfg.refinement;
    if (n > (int64_t(1) << 21)) return nullptr;
    m->dims[size_t(d)] = int32_t(n);
    m->delta[size_t(d)] = (cfg.hi[d] - cfg.lo[d]) / double(n);
    ne *= n;
  }
  // the GPU path indexes elements with int32
  if (ne >= (int64_t(1) << 31)) return nullptr;
  m->ne = ne;
  m->jacobian = 0.125 * m->delta[0] * m->delta[1] * m->delta[2];

  const int nx = m->dims[0], ny = m->dims[1], nz = m->dims[2];
  // sort raw lattice indices by Morton key (keys are injective)
  std::vector<uint64_t> key(static_cast<size_t>(ne));
  {
    size_t raw = 0;
    for (int k = 0; k < nz; ++k)
      for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i)
          key[raw++] = dilate3(uint64_t(i)) | (dilate3(uint64_t(j)) << 1) |
                       (dilate3(uint64_t(k)) << 2);
  }
  std::vector<int32_t> order(static_cast<size_t>(ne));
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
    return key[size_t(a)] != key[size_t(b)] ? key[size_t(a)] < key[size_t(b)] : a < b;
  });
  m->lattice.resize(size_t(ne) * 3);
  m->elem_at.resize(size_t(ne));
  for (int64_t e = 0; e < ne; ++e) {
    const int32_t raw = order[size_t(e)];
    m->lattice[size_t(e) * 3 + 0] = raw % nx;
    m->lattice[size_t(e) * 3 + 1] = (raw / nx) % ny;
    m->lattice[size_t(e) * 3 + 2] = raw / (nx * ny);
    m->elem_at[size_t(raw)] = int32_t(e);
  }

  // neighbour table: lo/hi neighbour per direction, -1 at reflecting walls
  m->nbr.resize(size_t(ne) * 6);
  for (int64_t e = 0; e < ne; ++e) {
    const int32_t* lat = &m->lattice[size_t(e) * 3];
    for (int d = 0; d < 3; ++d)
      for (int side = 0; side < 2; ++side) {
        int c[3] = {lat[0], lat[1], lat[2]};
        c[d] += side ? 1 : -1;
        int32_t code;
        if (c[d] < 0 || c[d] == m->dims[size_t(d)]) {
          if (cfg.bc[d] == 1) {
            code = -1;
          } else {
            c[d] = c[d] < 0 ? m->dims[size_t(d)] - 1 : 0;
            code = m->elem_at[size_t(c[0]) + size_t(nx) * (size_t(c[1]) + size_t(ny) * size_t(c[2]))];
          }
        } else {
          code = m->elem_at[size_t(c[0]) + size_t(nx) * (size_t(c[1]) + size_t(ny) * size_t(c[2]))];
        }
        m->nbr[size_t(e) * 6 + size_t(d * 2 + side)] = code;
      }
  }
  return m;
}

// Face list in the reference's enumeration (mesh.cpp:78-132): elements in
// Morton order; per direction the hi face, then the lo wall face of
// first-layer elements; the lower-index element is the minus side.
void Mesh::build_faces() {
  if (faces_built) return;
  faces.clear();
  face_of.assign(size_t(ne) * 6, -1);
  for (int64_t e = 0; e < ne; ++e)
    for (int d = 0; d < 3; ++d) {
      const int32_t hi = nbr[size_t(e) * 6 + size_t(d * 2 + 1)];
      esdg_b200_face f{};
      f.dir = uint8_t(d);
      const int32_t id = int32_t(faces.size());
      if (hi < 0) {
        f.minus_elem = int32_t(e);
        f.plus_elem = -1;
        f.minus_side = 1;
        f.reflecting = 1;
        face_of[size_t(e) * 6 + size_t(d * 2 + 1)] = id;
      } else {
        const bool e_is_minus = hi >= e;
        f.minus_elem = e_is_minus ? int32_t(e) : hi;
        f.plus_elem = e_is_minus ? hi : int32_t(e);
        f.minus_side = e_is_minus ? 1 : 0;
        face_of[size_t(e) * 6 + size_t(d * 2 + 1)] = id;
        face_of[size_t(hi) * 6 + size_t(d * 2 + 0)] = id;
      }
      faces.push_back(f);
      if (nbr[size_t(e) * 6 + size_t(d * 2)] < 0) {
        esdg_b200_face w{};
        w.minus_elem = int32_t(e);
        w.plus_elem = -1;
        w.dir = uint8_t(d);
        w.minus_side = 0;
        w.reflecting = 1;
        face_of[size_t(e) * 6 + size_t(d * 2)] = int32_t(faces.size());
        faces.push_back(w);
      }
    }
  faces_built = true;
}

bool make_partition(int64_t ne, int ranks, std::vector<int64_t>& rb) {
  if (ranks < 1 || ranks > ne) return false;
  rb.assign(size_t(ranks) + 1, 0);
  const int64_t q = ne / ranks, r = ne % ranks;
  for (int k = 0; k < ranks; ++k)
    rb[size_t(k) + 1] = rb[size_t(k)] + q + (k < r ? 1 : 0);
  return true;
}

void build_rank_halo(const Mesh& m, const std::vector<int64_t>& rb, int r,
                     RankHalo& out) {
  const int64_t b = rb[size_t(r)], e = rb[size_t(r) + 1];
  struct Ghost {
    int peer;
    int64_t owner_key; // (element whose hi side the face is) * 3 + dir
    int32_t local_elem, local_face, remote_elem;
    bool am_minus;
  };
  std::vector<Ghost> ghosts;
  out.nbr_local.assign(size_t(e - b) * 6, -1);
  for (int64_t el = b; el < e; ++el)
    for (int lf = 0; lf < 6; ++lf) {
      const int32_t n = m.nbr[size_t(el) * 6 + size_t(lf)];
      int32_t& code = out.nbr_local[size_t(el - b) * 6 + size_t(lf)];
      if (n < 0) {
        code = -1;
      } else if (n >= b && n < e) {
        code = int32_t(n - b);
      } else {
        const int d = lf / 2, side = lf % 2;
        const int64_t hi_owner = side ? el : n;
        ghosts.push_back({rank_of(rb, n), hi_owner * 3 + d, int32_t(el - b), lf,
                          n, el < n});
        code = -2; // patched below once the slot is known
      }
    }
  std::sort(ghosts.begin(), ghosts.end(), [](const Ghost& x, const Ghost& y) {
    return x.peer != y.peer ? x.peer < y.peer : x.owner_key < y.owner_key;
  });
  out.peers.clear();
  out.send_elem.clear();
  out.send_face.clear();
  out.ghost_remote_elem.clear();
  out.ghost_remote_face.clear();
  for (size_t g = 0; g < ghosts.size(); ++g) {
    const Ghost& gh = ghosts[g];
    if (out.peers.empty() || out.peers.back().rank != gh.peer)
      out.peers.push_back({gh.peer, int64_t(g), 0});
    ++out.peers.back().count;
    out.send_elem.push_back(gh.local_elem);
    out.send_face.push_back(gh.local_face);
    out.ghost_remote_elem.push_back(gh.remote_elem);
    out.ghost_remote_face.push_back(gh.local_face ^ 1);
    out.nbr_local[size_t(gh.local_elem) * 6 + size_t(gh.local_face)] =
        -2 - int32_t(2 * g + (gh.am_minus ? 1 : 0));
  }
}

void build_face_roles(const int32_t* nbr, int64_t ne, int epb, bool split, uint8_t* roles) {
  const int64_t ng = (ne + epb - 1) / epb;
  std::vector<uint8_t> boundary(size_t(ng), 0); // group has a ghost face
  if (split)
    for (int64_t e = 0; e < ne; ++e)
      for (int lf = 0; lf < 6; ++lf)
        if (nbr[e * 6 + lf] <= -2) boundary[size_t(e / epb)] = 1;
  for (int64_t e = 0; e < ne; ++e) roles[e] = 0;
  for (int64_t b = 0; b < ne; ++b)
    for (int f = 0; f < 3; ++f) {
      const int32_t a = nbr[b * 6 + 2 * f];
      if (a < 0 || a == b || nbr[int64_t(a) * 6 + 2 * f + 1] != int32_t(b)) continue;
      if (split) {
        // the interior list is launched (and finished) before the boundary
        // list: inside a list the index decides, between the lists the launch
        const int la = boundary[size_t(a / epb)], lb = boundary[size_t(b / epb)];
        if (la > lb || (la == lb && a > b)) continue;
      } else if (a > b) {
        continue;
      }
      roles[b] |= uint8_t(1u << f);
      roles[a] |= uint8_t(8u << f);
    }
}

} // namespace host
} // namespace esdg_b200
