// esdg_kernels.cuh -- the hot-path kernels.
//
//   rhs_kernel<Real,NQ,EPB,VOL,SURF>
//     VOL  && !SURF  K1  volume term + commit   (kernels.hpp:154-316,
//                                                solver.hpp:199-238)
//     !VOL && SURF   K2  surface term           (kernels.hpp:350-430,
//                                                solver.hpp:266-337)
//     VOL  && SURF   K1+K2 fused, one pass over the element
//   axpy_kernel      K3  q += b k               (solver.hpp:342-353)
//   pack_kernel      K4  ghost-face traces      (kernels.hpp:331-338,
//                                                solver.hpp:249-257)
//
// Execution model of rhs_kernel (B200: 148 SMs, 64 FP64 lanes/SM, 227 KB smem)
//   - one CTA owns EPB consecutive (Morton) elements; EPB*NQ^2 threads.
//   - phase A, thread per node: coalesced loads of q and phi straight from
//     HBM, primitives + both logarithms once per node (precompute/logmean
//     rungs of the reference's ladder) into shared memory, SoA per quantity.
//   - phase B, thread per node LINE: the thread pulls its line's NQ nodes
//     into registers and evaluates every unordered pair (i,j) exactly once,
//     adding c_ij (S + G e_n) to node i and c_ji (S - G b_i/b_j e_n) to node
//     j in registers (the paper's pair symmetry incl. the -G b-/b+ rule for
//     the non-symmetric gravity term). No partner exchange is needed, so the
//     shared-memory pipe only sees the line load and the tendency update,
//     and the FP64 FMA pipe is the bound. Directions run one after another
//     in a rotated frame so the flux code is direction independent.
//   - phase C, thread per face node: each element side evaluates the
//     canonical (minus,plus) flux of its own face -- the flux is a pure
//     function of the two traces, so both sides obtain bitwise identical
//     values and conservation is exact without storing face records.
//   - phase D, thread per node: commit, coalesced.
#pragma once

#include "esdg_device.cuh"

namespace esdg_b200 {
namespace dev {

struct FlagRecord;

template <class Real, int NQ>
struct RhsParams {
  const Real* q;
  Real* out;
  const Real* phi;
  const int32_t* nbr;
  const Real* ghost_q;
  const Real* ghost_phi;
  const int32_t* ylevel;
  const Real* cor_f;
  unsigned long long* flag;
  FlagRecord* flag_records;
  long long ne;
  long long elem_offset;
  Real a_old, a_new;
  GasParams<Real> gas;
  Real negc[3][NQ * NQ]; // -(2 g_d D_ij), kernels.hpp:187, 224-225
  Real lift[3];          // Operators::face_coef, kernels.hpp:86-88
  int with_source;       // Coriolis on (commit_volume, solver.hpp:205-216)
  int dissipation;
  int stage;
};

// Non-physical-state record. The smallest key wins:
//   [stage:8][phase:1][element:45][node:10]
// phase 0 = the per-node sweep of phase A (the reference's volume phase,
// which runs first and throws first, solver.hpp:259-262), phase 1 = a
// neighbour state met while evaluating a face. Within a phase the smallest
// (element, node) is what the reference's serial sweep would have hit first.
// The payload (rho, p) goes to a small hashed side table so the host can
// report the values seen at detection time even after later stages ran.
struct FlagRecord {
  unsigned long long key;
  double rho, p;
};
constexpr int kFlagSlots = 61;

__device__ __forceinline__ void raise_flag(unsigned long long* flag,
                                           FlagRecord* records, int stage,
                                           int phase, long long elem, int node,
                                           double rho, double p) {
  const unsigned long long key =
      (static_cast<unsigned long long>(stage < 0 ? 0 : stage) << 56) |
      (static_cast<unsigned long long>(phase) << 55) |
      (static_cast<unsigned long long>(elem) << 10) |
      static_cast<unsigned long long>(node);
  const unsigned long long old = atomicMin(flag, key);
  if (key < old) {
    FlagRecord* r = records + (key % kFlagSlots);
    r->rho = rho;
    // compute_node_vals reports p = 0 when the density check trips first
    r->p = (rho > 0.0) ? p : 0.0;
    __threadfence();
    r->key = key;
  }
}

template <int NQ>
struct Geo {
  static constexpr int N2 = NQ * NQ;
  static constexpr int N3 = N2 * NQ;
  static constexpr int PX = NQ | 1; // odd x pitch: x-lines hit distinct banks
  static constexpr int N3P = PX * NQ * NQ;
  __device__ static __forceinline__ int sidx(int n) {
    const int bc = n / NQ;
    return (n - bc * NQ) + PX * bc;
  }
};

template <class Real>
__device__ __forceinline__ Node<Real> load_node(const Real* vals, int VS, int s,
                                                int dir) {
  Node<Real> n;
  const int d1 = dir == 2 ? 0 : dir + 1;
  const int d2 = d1 == 2 ? 0 : d1 + 1;
  n.hr = vals[V_HR * VS + s];
  n.hun = vals[(V_HU0 + dir) * VS + s];
  n.hut1 = vals[(V_HU0 + d1) * VS + s];
  n.hut2 = vals[(V_HU0 + d2) * VS + s];
  n.b = vals[V_B * VS + s];
  n.hlr = vals[V_HLR * VS + s];
  n.lb = vals[V_LB * VS + s];
  n.hphi = vals[V_HPHI * VS + s];
  n.hib = vals[V_HIB * VS + s];
  return n;
}

template <class Real>
__device__ __forceinline__ Node<Real> rotate_node(const Real nv[V_COUNT],
                                                  int dir) {
  Node<Real> n;
  const int d1 = dir == 2 ? 0 : dir + 1;
  const int d2 = d1 == 2 ? 0 : d1 + 1;
  n.hr = nv[V_HR];
  n.hun = dir == 0 ? nv[V_HU0] : (dir == 1 ? nv[V_HU1] : nv[V_HU2]);
  n.hut1 = d1 == 0 ? nv[V_HU0] : (d1 == 1 ? nv[V_HU1] : nv[V_HU2]);
  n.hut2 = d2 == 0 ? nv[V_HU0] : (d2 == 1 ? nv[V_HU1] : nv[V_HU2]);
  n.b = nv[V_B];
  n.hlr = nv[V_HLR];
  n.lb = nv[V_LB];
  n.hphi = nv[V_HPHI];
  n.hib = nv[V_HIB];
  return n;
}

template <class Real, int NQ, int EPB, int MINB, bool VOL, bool SURF>
__global__ void __launch_bounds__(EPB* NQ* NQ, MINB)
    rhs_kernel(const __grid_constant__ RhsParams<Real, NQ> P) {
  using G = Geo<NQ>;
  constexpr int N2 = G::N2, N3 = G::N3, PX = G::PX, N3P = G::N3P;
  constexpr int T = EPB * N2;
  constexpr int VS = EPB * N3P; // stride between quantity arrays

  extern __shared__ __align__(16) unsigned char smem_raw[];
  Real* vals = reinterpret_cast<Real*>(smem_raw); // [V_COUNT][VS]
  Real* tend = vals + V_COUNT * VS;               // [5][VS]

  const int tid = threadIdx.x;
  const long long e0 = static_cast<long long>(blockIdx.x) * EPB;
  const long long left = P.ne - e0;
  const int ne_blk = left < EPB ? static_cast<int>(left) : EPB;

  // ---- phase A: primitives and logarithms, once per node ------------------
  for (int idx = tid; idx < ne_blk * N3; idx += T) {
    const int e = idx / N3, n = idx - e * N3;
    const Real* qe = P.q + (e0 + e) * (5 * N3);
    Real qv[5];
#pragma unroll
    for (int v = 0; v < 5; ++v) qv[v] = qe[v * N3 + n];
    const Real ph = P.phi[(e0 + e) * N3 + n];
    Real nv[V_COUNT], pr;
    if (!node_vals(qv, ph, P.gas.gm1, nv, pr))
      raise_flag(P.flag, P.flag_records, P.stage, 0, P.elem_offset + e0 + e, n,
                 double(qv[0]), double(pr));
    const int s = e * N3P + G::sidx(n);
#pragma unroll
    for (int k = 0; k < V_COUNT; ++k) vals[k * VS + s] = nv[k];
    if (!VOL) {
#pragma unroll
      for (int v = 0; v < 5; ++v) tend[v * VS + s] = Real(0);
    }
  }
  __syncthreads();

  // pitches of the three axes in shared (padded) and global node numbering
  auto spitch = [](int ax) { return ax == 0 ? 1 : (ax == 1 ? PX : PX * NQ); };
  auto gpitch = [](int ax) { return ax == 0 ? 1 : (ax == 1 ? NQ : NQ * NQ); };
  const int e = tid / N2, l = tid - e * N2;
  const bool active = e < ne_blk;
  const int l0 = l % NQ, l1 = l / NQ;

  // ---- phase B: flux differencing, every pair of a line once --------------
  if (VOL) {
#pragma unroll 1
    for (int dir = 0; dir < 3; ++dir) {
      if (active) {
        int base, stride;
        if (dir == 0) {
          base = PX * l;
          stride = 1;
        } else if (dir == 1) {
          base = l0 + PX * NQ * l1;
          stride = PX;
        } else {
          base = l0 + PX * l1;
          stride = PX * NQ;
        }
        base += e * N3P;
        Node<Real> nd[NQ];
#pragma unroll
        for (int i = 0; i < NQ; ++i)
          nd[i] = load_node(vals, VS, base + i * stride, dir);

        Real acc[NQ][5];
        // diagonal: t_i -= 2 g_d D_ii F(q_i, q_i)  (kernels.hpp:170-188)
#pragma unroll
        for (int i = 0; i < NQ; ++i) {
          const Real cii = P.negc[dir][i * NQ + i];
#pragma unroll
          for (int v = 0; v < 5; ++v) acc[i][v] = Real(0);
          // D_ii vanishes analytically at interior LGL nodes; the host
          // flushes its O(1e-16) round-off residue to zero (shard.cu), so
          // only the two end nodes pay for a point flux here
          if (cii != Real(0)) {
            Real f[5];
            point_flux(nd[i], P.gas.cg, f);
#pragma unroll
            for (int v = 0; v < 5; ++v) acc[i][v] = cii * f[v];
          }
        }
        // off-diagonal pairs, each once (kernels.hpp:190-231)
#pragma unroll
        for (int i = 0; i < NQ; ++i) {
#pragma unroll
          for (int j = 0; j < NQ; ++j) {
            if (j <= i) continue; // constant bounds keep the unroll total
            const PairFlux<Real> pf = pair_flux(nd[i], nd[j], P.gas.cg);
            const Real cij = P.negc[dir][i * NQ + j];
            const Real cji = P.negc[dir][j * NQ + i];
            const Real fni = fma_(pf.tg, nd[i].hib, pf.f[1]);
            const Real fnj = fma_(-pf.tg, nd[j].hib, pf.f[1]);
            acc[i][0] = fma_(cij, pf.f[0], acc[i][0]);
            acc[i][1] = fma_(cij, fni, acc[i][1]);
            acc[i][2] = fma_(cij, pf.f[2], acc[i][2]);
            acc[i][3] = fma_(cij, pf.f[3], acc[i][3]);
            acc[i][4] = fma_(cij, pf.f[4], acc[i][4]);
            acc[j][0] = fma_(cji, pf.f[0], acc[j][0]);
            acc[j][1] = fma_(cji, fnj, acc[j][1]);
            acc[j][2] = fma_(cji, pf.f[2], acc[j][2]);
            acc[j][3] = fma_(cji, pf.f[3], acc[j][3]);
            acc[j][4] = fma_(cji, pf.f[4], acc[j][4]);
          }
        }
        // un-rotate into the tendency slab
        const int d1 = dir == 2 ? 0 : dir + 1;
        const int d2 = d1 == 2 ? 0 : d1 + 1;
        Real* t0 = tend;
        Real* tn = tend + (1 + dir) * VS;
        Real* tt1 = tend + (1 + d1) * VS;
        Real* tt2 = tend + (1 + d2) * VS;
        Real* t4 = tend + 4 * VS;
#pragma unroll
        for (int i = 0; i < NQ; ++i) {
          const int s = base + i * stride;
          if (dir == 0) {
            t0[s] = acc[i][0];
            tn[s] = acc[i][1];
            tt1[s] = acc[i][2];
            tt2[s] = acc[i][3];
            t4[s] = acc[i][4];
          } else {
            t0[s] += acc[i][0];
            tn[s] += acc[i][1];
            tt1[s] += acc[i][2];
            tt2[s] += acc[i][3];
            t4[s] += acc[i][4];
          }
        }
      }
      __syncthreads();
    }
  }

  // ---- phase C: surface term, each side evaluates its own face ------------
  if (SURF) {
#pragma unroll 1
    for (int dir = 0; dir < 3; ++dir) {
      if (active) {
        const int d1 = dir == 2 ? 0 : dir + 1;
        const int d2 = d1 == 2 ? 0 : d1 + 1;
        const long long eg = e0 + e;
#pragma unroll 1
        for (int side = 0; side < 2; ++side) {
          // FaceIndexer::node (mesh.hpp:107-114): tangential axes d1, d2
          // node = sum_k c_k * pitch_k with c[dir] = end, c[d1] = l0, c[d2] = l1
          const int cn = side ? NQ - 1 : 0;
          const int s_own = e * N3P + cn * spitch(dir) + l0 * spitch(d1) +
                            l1 * spitch(d2);
          const Node<Real> own = load_node(vals, VS, s_own, dir);

          const int code = P.nbr[eg * 6 + dir * 2 + side];
          Node<Real> nb;
          bool am_minus;
          if (code == -1) {
            // reflecting wall: mirror state, phi+ = phi- (kernels.hpp:364-367)
            nb = own;
            nb.hun = -own.hun;
            am_minus = true;
          } else {
            Real qv[5], ph;
            if (code >= 0) {
              const int n_nb = (NQ - 1 - cn) * gpitch(dir) + l0 * gpitch(d1) +
                               l1 * gpitch(d2);
              const Real* qn = P.q + static_cast<long long>(code) * (5 * N3);
#pragma unroll
              for (int v = 0; v < 5; ++v) qv[v] = qn[v * N3 + n_nb];
              ph = P.phi[static_cast<long long>(code) * N3 + n_nb];
              am_minus = side ? (code >= eg) : (eg < code);
            } else {
              const int gv = -2 - code;
              const long long g = gv >> 1;
              am_minus = (gv & 1) != 0;
#pragma unroll
              for (int v = 0; v < 5; ++v)
                qv[v] = P.ghost_q[(g * 5 + v) * N2 + l];
              ph = P.ghost_phi[g * N2 + l];
            }
            Real nv[V_COUNT], pr;
            if (!node_vals(qv, ph, P.gas.gm1, nv, pr))
              raise_flag(P.flag, P.flag_records, P.stage, 1, P.elem_offset + eg, l,
                         double(qv[0]), double(pr));
            nb = rotate_node(nv, dir);
          }
          // canonical orientation: lower Morton id is the minus side
          const Node<Real> m = am_minus ? own : nb;
          const Node<Real> p = am_minus ? nb : own;
          const PairFlux<Real> pf = pair_flux(m, p, P.gas.cg);
          Real dd[5] = {Real(0), Real(0), Real(0), Real(0), Real(0)};
          if (P.dissipation)
            matrix_dissipation(m, p, pf.rho_log, pf.inv_blog, P.gas, dd);
          Real fo[5];
          point_flux(own, P.gas.cg, fo);
          // commit_face_side (kernels.hpp:391-430)
          const Real n_own = side ? Real(1) : Real(-1);
          const Real dsign = am_minus ? Real(-0.5) : Real(0.5);
          const Real g_own = (am_minus ? pf.tg : -pf.tg) * own.hib;
          const Real lift = P.lift[dir];
          const Real phi_own = own.hphi + own.hphi;
          Real fl[5];
          fl[0] = n_own * pf.f[0] + dsign * dd[0];
          fl[1] = n_own * pf.f[1] + n_own * g_own + dsign * dd[1];
          fl[2] = n_own * pf.f[2] + dsign * dd[2];
          fl[3] = n_own * pf.f[3] + dsign * dd[3];
          fl[4] = n_own * pf.f[4] + dsign * fma_(phi_own, dd[0], dd[4]);
          tend[s_own] -= lift * (fl[0] - n_own * fo[0]);
          tend[(1 + dir) * VS + s_own] -= lift * (fl[1] - n_own * fo[1]);
          tend[(1 + d1) * VS + s_own] -= lift * (fl[2] - n_own * fo[2]);
          tend[(1 + d2) * VS + s_own] -= lift * (fl[3] - n_own * fo[3]);
          tend[4 * VS + s_own] -= lift * (fl[4] - n_own * fo[4]);
        }
      }
      __syncthreads();
    }
  }

  // ---- phase D: commit (solver.hpp:199-223) --------------------------------
  for (int idx = tid; idx < ne_blk * N3; idx += T) {
    const int ee = idx / N3, n = idx - ee * N3;
    const int s = ee * N3P + G::sidx(n);
    Real* oe = P.out + (e0 + ee) * (5 * N3);
    Real val[5];
#pragma unroll
    for (int v = 0; v < 5; ++v) val[v] = tend[v * VS + s];
    if (VOL) {
      if (P.with_source) {
        // coriolis_source (physics.hpp:297-306): h = (0, f q2, -f q1, 0, 0)
        const Real* qe = P.q + (e0 + ee) * (5 * N3);
        const int b = (n / NQ) % NQ;
        const Real f = P.cor_f[P.ylevel[e0 + ee] * NQ + b];
        val[1] = val[1] + f * qe[2 * N3 + n];
        val[2] = val[2] + (-f) * qe[1 * N3 + n];
      }
      if (P.a_old == Real(0)) {
#pragma unroll
        for (int v = 0; v < 5; ++v) oe[v * N3 + n] = P.a_new * val[v];
      } else {
#pragma unroll
        for (int v = 0; v < 5; ++v)
          oe[v * N3 + n] = P.a_old * oe[v * N3 + n] + P.a_new * val[v];
      }
    } else {
#pragma unroll
      for (int v = 0; v < 5; ++v)
        oe[v * N3 + n] = oe[v * N3 + n] + P.a_new * val[v];
    }
  }
}

// K3: q += b k (solver.hpp:342-353). Pure stream: 2 reads + 1 write per
// value, 16-byte vector accesses, grid-stride.
template <class Real>
__global__ void __launch_bounds__(256)
    axpy_kernel(Real* __restrict__ q, const Real* __restrict__ k, Real b,
                long long n) {
  constexpr int VEC = 16 / sizeof(Real);
  struct alignas(16) Vec {
    Real v[VEC];
  };
  const long long nvec = n / VEC;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  Vec* qv = reinterpret_cast<Vec*>(q);
  const Vec* kv = reinterpret_cast<const Vec*>(k);
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
       i < nvec; i += stride) {
    Vec a = qv[i];
    const Vec c = kv[i];
#pragma unroll
    for (int j = 0; j < VEC; ++j) a.v[j] = a.v[j] + b * c.v[j];
    qv[i] = a;
  }
  for (long long i = nvec * VEC + static_cast<long long>(blockIdx.x) * blockDim.x +
                     threadIdx.x;
       i < n; i += stride)
    q[i] = q[i] + b * k[i];
}

// K4: ghost-face traces into the send buffer, var-major 5*NQ^2 per slot,
// face nodes in FaceIndexer order (kernels.hpp:331-338, mesh.hpp:107-114).
template <class Real, int NQ>
__global__ void __launch_bounds__(256)
    pack_kernel(const Real* __restrict__ q, const int32_t* __restrict__ send_elem,
                const int32_t* __restrict__ send_face, Real* __restrict__ send,
                long long n_send) {
  constexpr int N2 = NQ * NQ, N3 = N2 * NQ;
  const long long total = n_send * 5 * N2;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
       i < total; i += stride) {
    const long long slot = i / (5 * N2);
    const int r = static_cast<int>(i - slot * (5 * N2));
    const int v = r / N2, fn = r - v * N2;
    const int lf = send_face[slot];
    const int dir = lf >> 1, side = lf & 1;
    const int d1 = dir == 2 ? 0 : dir + 1;
    const int d2 = d1 == 2 ? 0 : d1 + 1;
    const int p0 = dir == 0 ? 1 : (dir == 1 ? NQ : N2);
    const int p1 = d1 == 0 ? 1 : (d1 == 1 ? NQ : N2);
    const int p2 = d2 == 0 ? 1 : (d2 == 1 ? NQ : N2);
    const int node = (side ? NQ - 1 : 0) * p0 + (fn % NQ) * p1 + (fn / NQ) * p2;
    send[i] = q[(static_cast<long long>(send_elem[slot]) * 5 + v) * N3 + node];
  }
}

// Elements per CTA (EPB) and the resident-CTA target handed to
// __launch_bounds__ (MINB): EPB*NQ^2 threads should fill whole warps, MINB
// CTAs must fit an SM's 227 KB of shared memory at 14 quantity arrays per
// node, and the register cap 65536/(MINB*threads) must not spill the line
// state (ptxas -v is checked in DESIGN.md).
template <int NQ, int BYTES>
struct Tile;
template <> struct Tile<2, 8> { static constexpr int EPB = 32, MINB = 4; };
template <> struct Tile<3, 8> { static constexpr int EPB = 14, MINB = 4; };
template <> struct Tile<4, 8> { static constexpr int EPB = 8, MINB = 3; };
template <> struct Tile<5, 8> { static constexpr int EPB = 5, MINB = 3; };
template <> struct Tile<6, 8> { static constexpr int EPB = 3, MINB = 2; };
template <> struct Tile<7, 8> { static constexpr int EPB = 2, MINB = 2; };
template <> struct Tile<8, 8> { static constexpr int EPB = 2, MINB = 1; };
template <> struct Tile<2, 4> { static constexpr int EPB = 32, MINB = 4; };
template <> struct Tile<3, 4> { static constexpr int EPB = 14, MINB = 4; };
template <> struct Tile<4, 4> { static constexpr int EPB = 8, MINB = 4; };
template <> struct Tile<5, 4> { static constexpr int EPB = 5, MINB = 4; };
template <> struct Tile<6, 4> { static constexpr int EPB = 3, MINB = 4; };
template <> struct Tile<7, 4> { static constexpr int EPB = 2, MINB = 4; };
template <> struct Tile<8, 4> { static constexpr int EPB = 2, MINB = 2; };

} // namespace dev
} // namespace esdg_b200
