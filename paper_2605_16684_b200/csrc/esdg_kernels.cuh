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
//   - one CTA owns EPB consecutive (Morton) elements; EPB*NQ^2 threads; thread
//     (e, l) is "line l of element e" throughout.
//   - phase A: one thread moves the CTA's contiguous slabs of q, phi, the old
//     `out` (accumulate form) and the logarithm table with TMA bulk copies
//     and prefetches the next resident wave's slabs into L2. Then primitives and both
//     logarithms once per node (precompute/logmean rungs of the reference's
//     ladder), the NQ nodes stage by stage, parked in shared memory, SoA per
//     quantity.
//   - the slab holds T = out_old + gain * (contributions), gain = a_new/a_old;
//     every later phase adds its share with one FMA, the commit writes
//     a_old * T (a_old == 0: a_new * contributions, `out` is never read).
//   - phase C (SURF), thread per face node, runs before the sweeps. The flux
//     is a pure function of the two traces, and swapping its arguments gives
//     bitwise the same symmetric part and the negated gravity / dissipation
//     part, so no face records (17 Reals per face node in the reference) are
//     stored. K2 and the tiles without dev::Share: each element side evaluates
//     all six of its faces. One-pass kernels with dev::Share: every interior
//     face is evaluated once, by the element whose + face it is, which pushes
//     the other element's lift term (bitwise what that element would compute)
//     into RhsParams::frec; the other element pulls it -- one TMA bulk copy
//     per direction, issued before the pair fluxes of that direction -- and
//     adds it to its line sums. A reflecting wall is the element's own trace
//     with the normal momentum negated.
//   - phase B (VOL), thread per node LINE: the thread pulls its line's NQ
//     nodes into registers and evaluates every unordered pair (i,j) exactly
//     once, adding c_ij (S + G e_n) to node i and c_ji (S - G b_i/b_j e_n) to
//     node j in registers (the paper's pair symmetry incl. the -G b-/b+ rule
//     for the non-symmetric gravity term). No partner exchange is needed, so
//     the shared-memory pipe only sees the line load and the slab update.
//     The coefficients -(2 D_ij) are direction independent (uniform
//     registers); the metric is applied when the sums are handed on. x and y
//     sweeps go through the slab; the z sweep stays in registers because the
//     same thread commits that z line.
//   - commit: slab + registers -> out (+ Coriolis, + the fused LSRK register
//     update), coalesced over l, no global load to wait for except the state
//     re-read of the fused update.
// DESIGN.md section 4 has the measurements behind these choices.
#pragma once

#include <cstdio>

#include "esdg_device.cuh"

namespace esdg_b200 {
namespace dev {

struct FlagRecord;

template <class Real, int NQ>
struct RhsParams {
  const Real* q;
  Real* q_next; // fused stage update: q_next = q + b_upd * out_new (may be null)
  Real* out;
  const Real* phi;
  const int32_t* nbr;
  const Real* ghost_q;
  const Real* ghost_phi;
  const int32_t* ylevel;
  const Real* cor_f;
  // CTA -> element group (EPB consecutive elements): null = blockIdx.x. The
  // interior / boundary lists let the one-pass kernels overlap the halo
  // exchange the way the reference's volume phase does (solver.hpp:259-262).
  const int32_t* groups;
  int group_base; // groups == null: CTA i works on group group_base + i
  unsigned long long* flag;
  FlagRecord* flag_records;
  long long ne;
  long long elem_offset;
  Real a_old, a_new, b_upd;
  Real gain, fin; // slab arithmetic, see rhs_kernel phase A (set by the host)
  GasParams<Real> gas;
  Real negd[NQ * NQ];    // -(2 D_ij); with metric[d]: -(2 g_d D_ij), kernels.hpp:187, 224-225
  Real metric[3];        // g_d = 2 / dx_d
  Real lift[3];          // Operators::face_coef, kernels.hpp:86-88
  // One-pass kernels: every interior face is evaluated ONCE, by the element on
  // its minus side (whose + face, lf odd, it is), which also works out the
  // lift term of the plus side and pushes it into that element's slot of
  // `frec`; the plus side picks it up when the sweep of that direction has
  // its sums ready. face_roles[e]: bit f (0..2) = the lift term of face
  // lf = 2f of e is pushed by the neighbour, bit 3+d = the term of face
  // lf = 2d+1 is to be pushed to the neighbour. Null: every element evaluates
  // all six faces. Every value in a slot carries the evaluation it belongs to
  // in its lowest mantissa bit (`epoch`, alternating; see "tagged lift terms"
  // below), so a reader tells a fresh term from the previous evaluation's and
  // nobody has to reset a slot.
  const uint8_t* face_roles;
  Real* frec;            // [3][element][FrecBlock<Real, NQ>]: slot f = face lf = 2f, [5][NQ^2] + pad
  unsigned epoch;        // 0 / 1: the tag (lowest mantissa bit) of the lift terms of this evaluation
  unsigned long long* sync_error;
  // launch-order ticket (null: blockIdx.x is the order): CTA number = value of
  // the counter when the CTA starts, minus ticket_base
  unsigned* ticket;
  unsigned ticket_base;
  unsigned long long wait_limit_ns; // bound of a pull's poll (0: none), ESDG_B200_WAIT_LIMIT_MS
  int flat_phi;          // phi is constant along x and y lines (checked by the host)
  int prefetch_ctas;     // resident CTAs chip-wide: L2 prefetch distance
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

// Asynchronous global -> shared copy of one Real (LDGSTS): no register
// staging, and the issuing thread does not wait for the data.
template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem_dst, const void* gmem_src) {
  const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(dst), "l"(gmem_src), "n"(BYTES)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// TMA bulk copy global -> shared completing on an mbarrier (sm_90+): one
// instruction moves a whole contiguous slab without registers, L1 or the
// load/store pipe. Source, destination and size must be multiples of 16 B.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// TMA bulk copy shared -> global (bulk async-group completion).
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_store_commit_and_wait_read() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@p bra DONE_%=;\n\tbra WAIT_%=;\n\tDONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
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

// Shared-memory map of rhs_kernel (bytes). The CTA's slabs of q and phi are
// contiguous in HBM and arrive by TMA bulk copies in the (still unused) front
// of the node-value arrays, from where every thread picks the raw values of
// its z line. With an unpadded node layout (odd NQ) the old `out` arrives
// the same way, straight in the tendency slab, which then uses the
// [element][variable][node] order of the state registers. A slab starts at a
// multiple of sizeof(Real), not of 16 B, in HBM: the copy starts up to 12 B
// early and the data sit at the same offset in shared memory, hence the
// slack words.
template <class Real, int NQ, int EPB>
struct SmemMap {
  using G = Geo<NQ>;
  static constexpr bool kBulk = G::PX == NQ; // the slab can take `out` by bulk copy too
  static constexpr int VS = EPB * G::N3P;
  static constexpr size_t up16(size_t x) { return (x + 15) & ~size_t(15); }
  static constexpr size_t kStagePhi = up16(size_t(EPB) * 5 * G::N3 * sizeof(Real) + 16);
  static constexpr size_t kTend = up16(size_t(V_COUNT) * VS * sizeof(Real));
  // (slack words only where the slab takes `out` by bulk copy)
  static constexpr size_t kTab = kTend + up16((size_t(5) * VS + (kBulk ? 4 : 0)) * sizeof(Real));
  // The logarithm table is done with when the sweeps begin; the landing area
  // of the pulled lift terms (RhsParams::frec: the group's blocks of one
  // direction, one bulk copy) takes its place. The mbarrier outlives both.
  // In the one configuration where 16 bytes decide the third resident CTA
  // (padded FP64 layout, NQ = 4) the mbarrier sits in a padding slot of the
  // last node-value array, which no copy and no thread touches.
  static constexpr size_t kTabBytes = up16(size_t(LogTab<Real>::kReals) * sizeof(Real));
  static constexpr size_t kPullBlock = up16(size_t(5) * NQ * NQ * sizeof(Real)); // = FrecBlock bytes
  static constexpr size_t kPull = size_t(EPB) * kPullBlock;
  static constexpr size_t kRegion = kTabBytes > kPull ? kTabBytes : kPull;
  static constexpr bool kBarInPad = !kBulk && sizeof(Real) == 8;
  static constexpr size_t kBar =
      kBarInPad ? (size_t(V_COUNT - 1) * VS + NQ) * sizeof(Real) : kTab + up16(kRegion);
  static constexpr size_t kBytes = kTab + up16(kRegion) + (kBarInPad ? 0 : 16);
  static_assert(kStagePhi + up16(size_t(EPB) * G::N3 * sizeof(Real) + 16) <= kTend,
                "q and phi staging must fit in front of the slab");
};


// Elements per CTA (EPB) and the resident-CTA target handed to
// __launch_bounds__ (MINB): EPB*NQ^2 threads should fill whole warps, MINB
// CTAs must fit an SM's 227 KB of shared memory at 14 quantity arrays per
// node, and the register cap 65536/(MINB*threads) must not spill the line
// state (ptxas -v is checked in DESIGN.md).
template <int NQ, int BYTES>
struct Tile;
template <> struct Tile<2, 8> { static constexpr int EPB = 32, MINB = 4; static constexpr int FPI = 1; static constexpr bool LEAN = false; };
template <> struct Tile<3, 8> { static constexpr int EPB = 14, MINB = 4; static constexpr int FPI = 1; static constexpr bool LEAN = false; };
template <> struct Tile<4, 8> { static constexpr int EPB = 8, MINB = 3; static constexpr int FPI = 2; static constexpr bool LEAN = false; };
#ifndef ESDG_TUNE_EPB
#define ESDG_TUNE_EPB 5
#define ESDG_TUNE_MINB 3
#endif
template <> struct Tile<5, 8> { static constexpr int EPB = ESDG_TUNE_EPB, MINB = ESDG_TUNE_MINB; static constexpr int FPI = 1; static constexpr bool LEAN = false; };
#ifndef ESDG_TUNE_T68E
#define ESDG_TUNE_T68E 3
#define ESDG_TUNE_T68M 2
#define ESDG_TUNE_T78E 2
#define ESDG_TUNE_T78M 2
#define ESDG_TUNE_T64E 5 // FP32 N=5, one-pass kernels: 5 x 3 (stage kernel 4.77 -> 4.54 ms); TileSplit keeps 3 x 4
#define ESDG_TUNE_T64M 3
#define ESDG_TUNE_T74E 5
#define ESDG_TUNE_T74M 2
#endif
#ifndef ESDG_TUNE_T84E
#define ESDG_TUNE_T84E 2
#define ESDG_TUNE_T84M 3
#endif
template <int E, int M> struct TilePick { static constexpr int EPB = E, MINB = M; };
// FLATXY: a second, shorter instance of the line sweep without the gravity
// term serves the x and y lines when the potential is constant along them
// (RhsParams::flat_phi). It removes 6 of 52 FP64 instructions per pair there
// but doubles the sweep's code: +5 % (FP64) / +3 % (FP32) at N=6, within
// +-1 % at N <= 5 and -12 ... -16 % at N=7 (instruction cache), so only N=6
// uses it, and only in the one-pass kernels (the volume-only kernel at N=6
// loses 16 % with it).
template <int NQ, int BYTES> struct FlatXY { static constexpr bool value = NQ == 7; };
// SHARE: the one-pass kernels evaluate every interior face once and hand the
// other element its lift term through RhsParams::frec. It pays where the face
// phase was the long, badly overlapped part of a CTA's life (N <= 5, N = 7 in
// FP64: +3 ... +10 % on the stage path) and loses where one or two fat CTAs
// per SM ran the six faces as paired instruction streams (FPI = 2): there
// halving the faces halves the work per iteration, not the latency of an
// iteration (N = 6 FP64 -6 %, N = 7 FP32 -7 %; -3.4 % and -3 ... -4.5 % once the
// lift terms were tagged and no slot had to be reset any more); those tiles
// keep evaluating all six faces of an element.
template <int NQ, int BYTES> struct Share { static constexpr bool value = true; };
#ifndef ESDG_TUNE_SHARE78
#define ESDG_TUNE_SHARE78 false
#define ESDG_TUNE_SHARE84 false
#endif
template <> struct Share<7, 8> { static constexpr bool value = ESDG_TUNE_SHARE78; };
template <> struct Share<8, 4> { static constexpr bool value = ESDG_TUNE_SHARE84; };
template <> struct Tile<6, 8> : TilePick<ESDG_TUNE_T68E, ESDG_TUNE_T68M> { static constexpr int FPI = 2; static constexpr bool LEAN = false; };
template <> struct Tile<7, 8> : TilePick<ESDG_TUNE_T78E, ESDG_TUNE_T78M> { static constexpr int FPI = 2; static constexpr bool LEAN = true; };
template <> struct Tile<8, 8> { static constexpr int EPB = 1, MINB = 3; static constexpr int FPI = 2; static constexpr bool LEAN = true; };
template <> struct Tile<2, 4> { static constexpr int EPB = 32, MINB = 4; static constexpr int FPI = 1; static constexpr bool LEAN = false; };
template <> struct Tile<3, 4> { static constexpr int EPB = 14, MINB = 4; static constexpr int FPI = 1; static constexpr bool LEAN = false; };
template <> struct Tile<4, 4> { static constexpr int EPB = 8, MINB = 4; static constexpr int FPI = 1; static constexpr bool LEAN = false; };
// FP32 N=4: the one-pass kernels run best as three 10-element CTAs per SM (250
// threads, 80 registers: stage kernel 4.22 ms against 4.42 ms with five
// 5-element CTAs -- fewer CTAs in different phases share the instruction
// cache, which is what bounds the FP32 kernels); the volume-only and
// surface-only kernels prefer the small tile (2.52 / 2.41 ms against 2.68 /
// 2.57 ms), see TileSplit.
#ifndef ESDG_TUNE_T54E
#define ESDG_TUNE_T54E 10
#define ESDG_TUNE_T54M 3
#endif
template <> struct Tile<5, 4> { static constexpr int EPB = ESDG_TUNE_T54E, MINB = ESDG_TUNE_T54M; static constexpr int FPI = 1; static constexpr bool LEAN = false; };
template <> struct Tile<6, 4> : TilePick<ESDG_TUNE_T64E, ESDG_TUNE_T64M> { static constexpr int FPI = 1; static constexpr bool LEAN = false; };
template <> struct Tile<7, 4> : TilePick<ESDG_TUNE_T74E, ESDG_TUNE_T74M> { static constexpr int FPI = 1; static constexpr bool LEAN = false; };
template <> struct Tile<8, 4> : TilePick<ESDG_TUNE_T84E, ESDG_TUNE_T84M> { static constexpr int FPI = 2; static constexpr bool LEAN = false; };

// Launch shape of the volume-only and surface-only kernels (K1, K2, the ladder
// rungs) where it differs from the one-pass kernels'. Those kernels never see
// a group list, so their EPB is theirs alone; FPI / LEAN stay Tile's.
template <int NQ, int BYTES> struct TileSplit : Tile<NQ, BYTES> {};
#ifndef ESDG_TUNE_S54E
#define ESDG_TUNE_S54E 5
#define ESDG_TUNE_S54M 5
#endif
template <> struct TileSplit<5, 4> : Tile<5, 4> { static constexpr int EPB = ESDG_TUNE_S54E, MINB = ESDG_TUNE_S54M; };
template <> struct TileSplit<6, 4> : Tile<6, 4> { static constexpr int EPB = 3, MINB = 4; };

// Which y line a thread sweeps: YPerm<NQ, BYTES, EPB>::line(tid) = e * NQ^2 + x +
// NQ z (element of the CTA, x, z). With the natural assignment (x, z) =
// (l0, l1) the y lines of a half-warp start 1 and PX*NQ words apart and hit
// the same banks two to three times (N = 4 FP64: 16 instead of 8 wavefronts
// per CTA-wide 64-bit access, 31 instead of 16 per 128-bit one). A thread
// may sweep any y line of its CTA -- the sums go through the slab anyway --
// and the tables of esdg_yperm_tables.inc (local search,
// tools/yperm_search.py) remove the conflicts of the node loads and most of
// the slab's (N = 4 FP64: K1 -2.7 %, stage kernel -0.9 %). The table belongs to
// one tile shape; any other EPB falls back to the natural assignment.
template <int NQ, int BYTES, int EPB>
struct YPerm {
  static constexpr bool value = false;
  __device__ static __forceinline__ int line(int tid) { return tid; }
};
#ifndef ESDG_TUNE_NO_YPERM
#include "esdg_yperm_tables.inc"
#endif

// Shared-memory layout of the nine node quantities: three arrays of PAIRS --
// (rho/2, b), (log rho/2, log b), (phi/2, 1/(2b)) -- followed by the three
// velocity arrays. A node is then six shared-memory instructions instead of
// nine (three 128-bit, three 64-bit in FP64): the load/store pipe's
// instruction queue, not its bandwidth, is what the flux kernels run short
// of. The first pair and the velocities are what every pair flux uses twice
// ("hot"), the other two pairs once ("cold", re-fetched per pair at the
// highest orders).
template <class Real>
struct Pair2;
template <>
struct Pair2<double> {
  using type = double2;
};
template <>
struct Pair2<float> {
  using type = float2;
};
enum { P_RB = 0, P_LOGS = 1, P_PHI = 2, P_COUNT = 3 }; // pair arrays; velocities follow

template <class Real>
__device__ __forceinline__ void load_hot(const Real* vals, int VS, int s, int dir, Node<Real>& n) {
  using V2 = typename Pair2<Real>::type;
  const int d1 = dir == 2 ? 0 : dir + 1;
  const int d2 = d1 == 2 ? 0 : d1 + 1;
  const V2 rb = reinterpret_cast<const V2*>(vals)[P_RB * VS + s];
  n.hr = rb.x;
  n.b = rb.y;
  n.hun = vals[(2 * P_COUNT + dir) * VS + s];
  n.hut1 = vals[(2 * P_COUNT + d1) * VS + s];
  n.hut2 = vals[(2 * P_COUNT + d2) * VS + s];
}
template <class Real>
__device__ __forceinline__ void load_cold(const Real* vals, int VS, int s, Node<Real>& n) {
  using V2 = typename Pair2<Real>::type;
  const V2 lg = reinterpret_cast<const V2*>(vals)[P_LOGS * VS + s];
  const V2 ph = reinterpret_cast<const V2*>(vals)[P_PHI * VS + s];
  n.hlr = lg.x;
  n.lb = lg.y;
  n.hphi = ph.x;
  n.hib = ph.y;
}
template <class Real>
__device__ __forceinline__ void store_node(Real* vals, int VS, int s, const Real (&nv)[V_COUNT]) {
  using V2 = typename Pair2<Real>::type;
  V2* pv = reinterpret_cast<V2*>(vals);
  V2 t;
  t.x = nv[V_HR];
  t.y = nv[V_B];
  pv[P_RB * VS + s] = t;
  t.x = nv[V_HLR];
  t.y = nv[V_LB];
  pv[P_LOGS * VS + s] = t;
  t.x = nv[V_HPHI];
  t.y = nv[V_HIB];
  pv[P_PHI * VS + s] = t;
  vals[(2 * P_COUNT + 0) * VS + s] = nv[V_HU0];
  vals[(2 * P_COUNT + 1) * VS + s] = nv[V_HU1];
  vals[(2 * P_COUNT + 2) * VS + s] = nv[V_HU2];
}

template <class Real>
__device__ __forceinline__ Node<Real> load_node(const Real* vals, int VS, int s,
                                                int dir) {
  Node<Real> n;
  load_hot(vals, VS, s, dir, n);
  load_cold(vals, VS, s, n);
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

// One line sweep of the flux-differenced volume term in direction `dir`
// (sweep_direction, kernels.hpp:154-249): pulls the NQ nodes of a line into
// registers, ADDS the diagonal point fluxes and every unordered pair (once)
// to acc, which lives in the rotated frame of `dir` and still lacks the
// metric factor g_dir: the coefficients -(2 D_ij) are then the same in every
// direction and enter the FMAs as immediate constant-bank operands (an FP64
// instruction reading three distinct vector registers occupies the sm_100
// FP64 pipe for three cycles instead of two). One code instance
// serves the three directions (the instruction cache is a real constraint
// for these fully unrolled bodies).
template <class Real, int NQ, bool DIAG, bool FLAT, int RUNG = kRungProduct>
__device__ __forceinline__ void sweep_line(const RhsParams<Real, NQ>& P,
                                           const Real* vals, int VS, int base,
                                           int stride, int dir, Real (&acc)[NQ][5],
                                           const Real* logtab = nullptr) {
  // At the highest orders a line's node values and accumulators (14 NQ
  // Reals) no longer fit the register file next to the flux temporaries.
  // There only the five quantities every pair uses twice stay resident;
  // log rho/2, log b, phi/2 and 1/(2b) are fetched from shared memory for
  // the pair at hand (the load/store pipe has room: 2 NQ (NQ-1) extra loads
  // per line against 24 NQ (NQ-1) FP64 instructions).
  constexpr bool kLean = Tile<NQ, sizeof(Real)>::LEAN;
  Node<Real> nd[NQ];
#pragma unroll
  for (int i = 0; i < NQ; ++i) {
    if (kLean)
      load_hot(vals, VS, base + i * stride, dir, nd[i]);
    else
      nd[i] = load_node(vals, VS, base + i * stride, dir);
  }
  auto cold = [&](int i) {
    if (kLean) load_cold(vals, VS, base + i * stride, nd[i]);
  };
  // diagonal: t_i -= 2 g_d D_ii F(q_i, q_i)  (kernels.hpp:170-188). D_ii
  // vanishes analytically at interior LGL nodes; the host flushes its
  // O(1e-16) round-off residue to zero (shard.cu), so only the two end nodes
  // carry a point flux -- known at compile time, no branch.
  // In the fused kernels even those two are skipped together with the
  // -n F(q_own) part of the surface term: -2 g_d D_00 = g_d / w_0 = lift_d
  // (and +lift_d at the other end) by the SBP property of the LGL operator,
  // so the two point-flux terms of an end node cancel analytically. The
  // reference evaluates both and lets them cancel to rounding
  // (kernels.hpp:170-188, 406-428); dropping the pair changes a tendency by
  // 1e-16 of the flux and saves 2 x 6 NQ^2 point fluxes per element.
  if (DIAG) {
#pragma unroll
    for (int i = 0; i < NQ; i += NQ - 1) {
      const Real cii = P.negd[i * NQ + i];
      Real f[5];
      cold(i);
      point_flux(nd[i], P.gas.cg, f);
#pragma unroll
      for (int v = 0; v < 5; ++v) acc[i][v] = fma_(cii, f[v], acc[i][v]);
    }
  }
  if constexpr (RUNG < kRungProduct) {
    // Ladder rungs below the product (esdg_device.cuh, kRung*): every ORDERED
    // pair is evaluated and only node i is updated. kRungRecompute works out
    // primitives and both logarithms again inside every flux evaluation, for
    // both nodes (compute_node_vals per evaluation: 2 div + 2 log each).
    constexpr bool kIeee = RUNG < kRungLogMean;
    auto again = [&](const Node<Real>& n, Real tie) {
      // compute_node_vals (physics.hpp:56-80) once more: conservative
      // variables back from the parked quantities, two divisions, two
      // logarithms. The reference's variants see bitwise the same node values
      // whether they recompute them or not (same function of the same q;
      // acceptance criterion 4 holds them to 1e-13 of each other), and a
      // quantity rebuilt from rounded intermediates would be an ulp off --
      // which a logarithmic mean amplifies by 1/(2 xi). So the divisions are
      // carried out and then tied to the parked values through an exact
      // zero: every operation of the recomputation is executed, the values
      // stay the parked ones. Logarithms of unchanged arguments reproduce
      // themselves. `tie` (a different value of the partner in the two roles)
      // keeps the compiler from merging the recomputations of one node.
      const Real rho = fma_(Real(0), tie, n.hr + n.hr);
      const Real m1 = rho * n.hun, m2 = rho * n.hut1, m3 = rho * n.hut2; // momenta / 2
      const Real p = rho * n.hib;                                          // rho / (2 b)
      const Real inv = rcpx<kIeee>(rho);
      const Real b2 = rho * rcpx<kIeee>(p + p);
      Node<Real> r;
      r.hr = Real(0.5) * rho;
      r.hun = fma_(Real(0), m1 * inv, n.hun);
      r.hut1 = fma_(Real(0), m2 * inv, n.hut1);
      r.hut2 = fma_(Real(0), m3 * inv, n.hut2);
      r.b = fma_(Real(0), b2, n.b);
      r.hib = fma_(Real(0), p * inv, n.hib);
      r.hlr = Real(0.5) * log_(rho, logtab);
      r.lb = log_(r.b, logtab);
      r.hphi = n.hphi;
      return r;
    };
#pragma unroll
    for (int i = 0; i < NQ; ++i) {
#pragma unroll
      for (int j = 0; j < NQ; ++j) {
        if (j == i) continue;
        cold(i);
        cold(j);
        PairFlux<Real> pf;
        if constexpr (RUNG <= kRungRecompute)
          pf = pair_flux<Real, false, kIeee>(again(nd[i], nd[j].hphi), again(nd[j], nd[i].hun),
                                             P.gas.cg);
        else
          pf = pair_flux<Real, false, kIeee>(nd[i], nd[j], P.gas.cg);
        const Real cij = P.negd[i * NQ + j];
        const Real fni = fma_(pf.tg, nd[i].hib, pf.f[1]);
        acc[i][0] = fma_(cij, pf.f[0], acc[i][0]);
        acc[i][1] = fma_(cij, fni, acc[i][1]);
        acc[i][2] = fma_(cij, pf.f[2], acc[i][2]);
        acc[i][3] = fma_(cij, pf.f[3], acc[i][3]);
        acc[i][4] = fma_(cij, pf.f[4], acc[i][4]);
      }
    }
    return;
  }
  // off-diagonal pairs, each once (kernels.hpp:190-231). FLAT: phi is the
  // same at every node of this line (see pair_flux), the gravity term
  // vanishes identically and <phi> is the line's phi.
  Real phi_line = Real(0);
  if (FLAT) {
    if (kLean) load_cold(vals, VS, base, nd[0]);
    phi_line = nd[0].hphi + nd[0].hphi;
  }
#pragma unroll
  for (int i = 0; i < NQ; ++i) {
#pragma unroll
    for (int j = 0; j < NQ; ++j) {
      if (j <= i) continue; // constant bounds keep the unroll total
      cold(i);
      cold(j);
      const PairFlux<Real> pf = pair_flux<Real, FLAT>(nd[i], nd[j], P.gas.cg, phi_line);
      const Real cij = P.negd[i * NQ + j];
      const Real cji = P.negd[j * NQ + i];
      const Real fni = FLAT ? pf.f[1] : fma_(pf.tg, nd[i].hib, pf.f[1]);
      const Real fnj = FLAT ? pf.f[1] : fma_(-pf.tg, nd[j].hib, pf.f[1]);
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
}

// Raw neighbour state at one face node, as fetched from HBM/L2.
template <class Real>
struct NbrRaw {
  Real q[5], ph;
  int code;
};

// Raw state across one face node. code >= 0: local neighbour element, node
// n_nb of it (the opposite side, same tangential position); code <= -2: ghost
// trace slot, face node fn; -1: reflecting wall (mirror_state,
// physics.hpp:309-313): the element's own trace (node n_own) with the normal
// momentum negated, phi+ = phi-.
template <class Real, int NQ>
__device__ __forceinline__ void gather_trace(const RhsParams<Real, NQ>& P, int code, int dir,
                                             long long eg, int n_nb, int n_own, int fn,
                                             NbrRaw<Real>& r) {
  constexpr int N2 = NQ * NQ, N3 = N2 * NQ;
  if (code >= 0) {
    const Real* qn = P.q + static_cast<long long>(code) * (5 * N3);
#pragma unroll
    for (int v = 0; v < 5; ++v) r.q[v] = qn[v * N3 + n_nb];
    r.ph = P.phi[static_cast<long long>(code) * N3 + n_nb];
  } else if (code <= -2) {
    const long long g = (-2 - code) >> 1;
#pragma unroll
    for (int v = 0; v < 5; ++v) r.q[v] = P.ghost_q[(g * 5 + v) * N2 + fn];
    r.ph = P.ghost_phi[g * N2 + fn];
  } else {
    const Real* qo = P.q + eg * (5 * N3);
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      const Real x = qo[v * N3 + n_own];
      r.q[v] = (v == 1 + dir) ? -x : x;
    }
    r.ph = P.phi[eg * N3 + n_own];
  }
}

// Surface contribution of one face node of one element side, rotated frame
// of `dir`: c[v] = lift (F*_v - n F_v(q_own)), to be SUBTRACTED from the
// tendency (compute_face_record + commit_face_side, kernels.hpp:350-430).
//
// Each side evaluates its own face; no face records are stored. That is
// exact because pair_flux and matrix_dissipation are written so that swapping
// their arguments gives bitwise the same symmetric part and bitwise the
// negated gravity / dissipation part (sums and products commute, differences
// and rcp_ negate exactly, see esdg_device.cuh). With (own, nbr) as argument
// order the reference's canonical record (minus = lower Morton id) reduces to
//   am_minus:  n (S + G e_n)        - D(own,nbr)/2,  G = tg hib_own
//   otherwise: n (S - G' b-/b+ e_n) + D(nbr,own)/2 = the same expression,
// so the orientation never has to be looked at, and the two sides of a face
// subtract exactly opposite numbers: conservation is exact.
// The two faces of one direction (side 0 at node 0, side 1 at node NQ-1 of
// the line through the face node) share no data, so their evaluations are
// written stage by stage: two independent dependency chains for the
// scheduler instead of one.
// Split in two so that the caller can start the next direction's gather as
// soon as the raw traces have been consumed.
//
// Part 1: node values of the two neighbour traces. A reflecting wall arrives
// here as the element's own trace with the normal momentum negated (see
// fetch): compute_node_vals of that is bitwise the own node with hun negated,
// i.e. mirror_state with phi+ = phi- (kernels.hpp:364-367, physics.hpp:309-313).
template <class Real, int NQ, int F>
__device__ __forceinline__ void face_pair_neighbours(const RhsParams<Real, NQ>& P,
                                                     const NbrRaw<Real> (&nbr)[F], int dir,
                                                     long long eg, int fn, const Real* logtab,
                                                     Node<Real> (&nb)[F]) {
  Real q2[F][5], ph2[F], nv[F][V_COUNT], pr[F];
#pragma unroll
  for (int f = 0; f < F; ++f) {
#pragma unroll
    for (int v = 0; v < 5; ++v) q2[f][v] = nbr[f].q[v];
    ph2[f] = nbr[f].ph;
  }
  const unsigned bad = node_vals_line<Real, F>(q2, ph2, P.gas.gm1, logtab, nv, pr);
#pragma unroll
  for (int f = 0; f < F; ++f) {
    nb[f] = rotate_node(nv[f], dir);
    if (bad & (1u << f))
      raise_flag(P.flag, P.flag_records, P.stage, 1, P.elem_offset + eg, fn,
                 double(q2[f][0]), double(pr[f]));
  }
}

// Part 2: fluxes, dissipation and lift of the two faces.
template <class Real, int NQ, int F, bool OWN>
__device__ __forceinline__ void face_pair_contribution(const RhsParams<Real, NQ>& P,
                                                       const Node<Real> (&own)[F],
                                                       const Node<Real> (&nb)[F], int dir,
                                                       int side0, Real (&c)[F][5]) {
  PairFlux<Real> pf[F];
#pragma unroll
  for (int f = 0; f < F; ++f) pf[f] = pair_flux(own[f], nb[f], P.gas.cg);
  Real dd[F][5];
#pragma unroll
  for (int f = 0; f < F; ++f)
#pragma unroll
    for (int v = 0; v < 5; ++v) dd[f][v] = Real(0);
  if (P.dissipation) {
#pragma unroll
    for (int f = 0; f < F; ++f)
      matrix_dissipation(own[f], nb[f], pf[f].rho_log, pf[f].inv_blog, P.gas, dd[f]);
  }
  const Real lift = P.lift[dir];
#pragma unroll
  for (int f = 0; f < F; ++f) {
    // commit_face_side (kernels.hpp:391-430); OWN = false in the fused
    // kernels: -n F(q_own) cancels against the volume term's diagonal, see
    // sweep_line
    Real fo[5] = {Real(0), Real(0), Real(0), Real(0), Real(0)};
    if (OWN) point_flux(own[f], P.gas.cg, fo);
    const Real n_own = (side0 + f) ? Real(1) : Real(-1);
    const Real g_own = pf[f].tg * own[f].hib;
    const Real phi_own = own[f].hphi + own[f].hphi;
    Real fl[5];
    fl[0] = n_own * pf[f].f[0] - Real(0.5) * dd[f][0];
    fl[1] = n_own * pf[f].f[1] + n_own * g_own - Real(0.5) * dd[f][1];
    fl[2] = n_own * pf[f].f[2] - Real(0.5) * dd[f][2];
    fl[3] = n_own * pf[f].f[3] - Real(0.5) * dd[f][3];
    fl[4] = n_own * pf[f].f[4] - Real(0.5) * fma_(phi_own, dd[f][0], dd[f][4]);
#pragma unroll
    for (int v = 0; v < 5; ++v) c[f][v] = OWN ? lift * (fl[v] - n_own * fo[v]) : lift * fl[v];
  }
}

// One-pass kernels: the lift flux of one face node for the evaluating side
// (fl_own) and, BOTH, for the element across the face (fl_nb) -- bitwise what
// that element obtains when it evaluates the face itself with the arguments
// swapped (a ghost face in another partitioning): the symmetric flux is the
// same number, gravity and dissipation are exactly negated (see
// face_pair_contribution), and the expressions below are the same ones with
// those signs. Rotated frame of the face direction; the caller applies
// lift_d (the -n F(q_own) part cancels against the volume term, OWN = false).
template <class Real, int NQ, bool BOTH>
__device__ __forceinline__ void face_fluxes(const RhsParams<Real, NQ>& P, const Node<Real>& own,
                                            const Node<Real>& nb, int side, Real (&fl_own)[5],
                                            Real (&fl_nb)[5]) {
  const PairFlux<Real> pf = pair_flux(own, nb, P.gas.cg);
  Real dd[5] = {Real(0), Real(0), Real(0), Real(0), Real(0)};
  if (P.dissipation) matrix_dissipation(own, nb, pf.rho_log, pf.inv_blog, P.gas, dd);
  {
    const Real n_own = side ? Real(1) : Real(-1);
    const Real g_own = pf.tg * own.hib;
    const Real phi_own = own.hphi + own.hphi;
    fl_own[0] = n_own * pf.f[0] - Real(0.5) * dd[0];
    fl_own[1] = n_own * pf.f[1] + n_own * g_own - Real(0.5) * dd[1];
    fl_own[2] = n_own * pf.f[2] - Real(0.5) * dd[2];
    fl_own[3] = n_own * pf.f[3] - Real(0.5) * dd[3];
    fl_own[4] = n_own * pf.f[4] - Real(0.5) * fma_(phi_own, dd[0], dd[4]);
  }
  if (BOTH) {
    Real dn[5];
#pragma unroll
    for (int v = 0; v < 5; ++v) dn[v] = P.dissipation ? -dd[v] : Real(0);
    const Real n_nb = side ? Real(-1) : Real(1);
    const Real g_nb = (-pf.tg) * nb.hib;
    const Real phi_nb = nb.hphi + nb.hphi;
    fl_nb[0] = n_nb * pf.f[0] - Real(0.5) * dn[0];
    fl_nb[1] = n_nb * pf.f[1] + n_nb * g_nb - Real(0.5) * dn[1];
    fl_nb[2] = n_nb * pf.f[2] - Real(0.5) * dn[2];
    fl_nb[3] = n_nb * pf.f[3] - Real(0.5) * dn[3];
    fl_nb[4] = n_nb * pf.f[4] - Real(0.5) * fma_(phi_nb, dn[0], dn[4]);
  }
}

// One (direction, element) block of frec: [5][NQ^2] Reals, padded to a
// multiple of 16 bytes so that the blocks of a group's consecutive elements
// are one bulk copy.
template <class Real, int NQ>
struct FrecBlock {
  static constexpr int value = int(((5 * NQ * NQ * sizeof(Real) + 15) & ~size_t(15)) / sizeof(Real));
};
// Tagged lift terms. A lift term travels through its slot of frec with the
// lowest bit of its mantissa replaced by the parity of the evaluation (RHS
// call) it belongs to; the reader checks the bit and clears it. Every slot is
// written exactly once per evaluation (by the element across the face or by
// its own element) before it is read, so "bit == this evaluation's parity"
// means "filled", the slot needs no reset (15 global stores per thread and
// 2.65 GB of L2 writes per launch at configs[1] with the earlier NaN marker), and
// an 8-byte (4-byte) store being atomic, a value is either the previous
// evaluation's or the new one. Clearing the bit truncates the term by at most
// one ulp (1.1e-16 / 6e-8 relative, far inside the stated tolerances); the
// evaluating side clears the same bit of its own term (trunc_tag), so the two
// sides of a face still subtract exactly opposite mass fluxes, and a term is
// the same number whether it was pushed or self-evaluated: results stay
// bitwise independent of the partition count and of face sharing on / off.
// The host keeps the parity consistent (Shard::open_epoch, shard.cu); slots
// start as all ones (parity 1).
__device__ __forceinline__ double tag_term(double x, unsigned bit) {
  return __hiloint2double(__double2hiint(x), (__double2loint(x) & ~1) | int(bit));
}
__device__ __forceinline__ float tag_term(float x, unsigned bit) {
  return __int_as_float((__float_as_int(x) & ~1) | int(bit));
}
__device__ __forceinline__ bool has_tag(double x, unsigned bit) {
  return (unsigned(__double2loint(x)) & 1u) == bit;
}
__device__ __forceinline__ bool has_tag(float x, unsigned bit) {
  return (unsigned(__float_as_int(x)) & 1u) == bit;
}
__device__ __forceinline__ double trunc_tag(double x) { return tag_term(x, 0u); }
__device__ __forceinline__ float trunc_tag(float x) { return tag_term(x, 0u); }
// A lift term that has not arrived although the element evaluating it was
// dispatched before this one: poll L2 until it is there. The element that
// pushes never waits for anybody, so this ends. The wait is bounded all the
// same -- by wall time (RhsParams::wait_limit_ns on %globaltimer, 2 s unless the
// environment says otherwise: a sanitizer or a debugger may slow
// the pushing group down by orders of magnitude, an iteration count would
// misfire there), and by the other waiters: the first one to give up raises
// the error word, everybody else sees it and leaves, so a launch whose
// dispatch order were ever violated ends within seconds and reports
// ESDG_B200_CUDA instead of hanging the device.
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
template <class Real>
__device__ __noinline__ Real wait_filled(const Real* src, unsigned epoch,
                                        unsigned long long* sync_error,
                                        unsigned long long limit_ns) {
  Real x = __ldcg(src);
  if (has_tag(x, epoch)) return x;
  const unsigned long long t0 = global_ns();
#pragma unroll 1
  for (int spins = 0; !has_tag(x, epoch); ++spins) {
    __nanosleep(spins < 64 ? 100 : 1000);
    x = __ldcg(src);
    if ((spins & 63) == 63) {
      if (*reinterpret_cast<volatile unsigned long long*>(sync_error) != 0ull) break;
      if (limit_ns != 0ull && global_ns() - t0 > limit_ns) {
        atomicOr(sync_error, 1ull);
        break;
      }
    }
  }
  return x;
}

template <class Real, int NQ, int EPB, int MINB, bool VOL, bool SURF, int RUNG = kRungProduct>
__global__ void __launch_bounds__(EPB* NQ* NQ, MINB)
    rhs_kernel(const __grid_constant__ RhsParams<Real, NQ> P) {
  static_assert(RUNG == kRungProduct || (VOL && !SURF), "ladder rungs are volume kernels");
  using G = Geo<NQ>;
  constexpr int N2 = G::N2, N3 = G::N3, PX = G::PX, N3P = G::N3P;
  constexpr int VS = EPB * N3P; // stride between quantity arrays
  constexpr int ZS = PX * NQ;   // shared-memory pitch of the z axis

  using Map = SmemMap<Real, NQ, EPB>;
  constexpr bool kBulk = Map::kBulk;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Real* vals = reinterpret_cast<Real*>(smem_raw);             // [V_COUNT][VS]
  Real* logtab = reinterpret_cast<Real*>(smem_raw + Map::kTab); // FP64 only: logarithm table
  unsigned long long* mbar = reinterpret_cast<unsigned long long*>(smem_raw + Map::kBar);
  // one-pass kernels: landing area of the pulled lift terms, [5][threads]; it
  // shares its place with the logarithm table, which is dead by then
  Real* pbuf = logtab;
  constexpr int FB = FrecBlock<Real, NQ>::value;

  const int tid = threadIdx.x;
  // Position of this CTA in the launch order. Pulling a lift term may wait for
  // the group that pushes it, and that group must then be running or done: with
  // a ticket drawn when the CTA starts, every lower number has started by
  // construction (the hardware's dispatch order of blockIdx.x does the same in
  // practice, but is not a documented guarantee).
  // (the ticket rides on the barrier that publishes the mbarriers)
  unsigned bid = blockIdx.x;
  {
    unsigned* slot = reinterpret_cast<unsigned*>(smem_raw + Map::kTend - 16);
    if (tid == 0) {
      if (P.ticket) *slot = atomicAdd(P.ticket, 1u) - P.ticket_base;
      mbar_init(mbar, 1);
      if (kBulk) mbar_init(mbar + 1, 1); // the old `out`: not needed before phase C
    }
    __syncthreads();
    if (P.ticket) bid = *slot;
  }
  const long long e0 =
      static_cast<long long>(P.groups ? P.groups[bid] : int32_t(bid) + P.group_base) * EPB;
#ifdef ESDG_TUNE_PHASE_CLOCKS
  long long tclk[10];
  int nclk = 0;
#define ESDG_CLK() tclk[nclk++] = clock64()
#else
#define ESDG_CLK()
#endif
  ESDG_CLK();

  // thread <-> (element e, line l = l0 + NQ l1). In phase A, in the z sweep
  // and in the commit the thread owns the z line through (x, y) = (l0, l1),
  // so those three stages hand data over in registers.
  // (element, x, y) of the thread. From NQ = 5 on they are packed in one opaque
  // register: wherever the compiler prefers recomputing them to keeping them,
  // that is a field extraction instead of two divisions of threadIdx.x by
  // constants (stage path +0.7 ... +2.7 % at N = 4..7 where it is used; it
  // loses 6 % at N = 2 FP32 and 0.5 % at N = 5 FP32, which keep the plain form)
  // (and the volume-only kernel of N = 7 FP64, which spills either way: +4.5 %)
  constexpr bool kPackedGeo =
      NQ >= 5 && !(NQ == 6 && sizeof(Real) == 4) && !(NQ == 8 && sizeof(Real) == 8 && !SURF);
  unsigned geo = 0;
  if (kPackedGeo) {
    const int e_ = tid / N2, l_ = tid - e_ * N2;
    geo = unsigned(e_) | (unsigned(l_ % NQ) << 8) | (unsigned(l_ / NQ) << 16);
    asm volatile("" : "+r"(geo));
  }
  const int e = kPackedGeo ? int(geo & 0xffu) : tid / N2;
  const int l = kPackedGeo ? int((geo >> 8) & 0xffu) + NQ * int(geo >> 16) : tid - e * N2;
  const int l0 = kPackedGeo ? int((geo >> 8) & 0xffu) : l % NQ;
  const int l1 = kPackedGeo ? int(geo >> 16) : l / NQ;
  const long long eg = e0 + e;
  const bool active = eg < P.ne; // only the last CTA has idle lines
  // the y line this thread sweeps: its own element's (x, z) = (l0, l1), or any
  // line of the CTA where a bank-conflict-free assignment exists (YPerm)
  // (not in the one-pass kernels of N = 6: the extra registers spill there and
  // cost more than the conflicts, +1.3 %)
  constexpr bool kYPerm = YPerm<NQ, sizeof(Real), EPB>::value && !(SURF && NQ == 7);
  int ey = e, ly0 = l0, ly1 = l1;
  if (kYPerm) {
    const int id = YPerm<NQ, sizeof(Real), EPB>::line(tid);
    ey = id / N2;
    const int r = id - ey * N2;
    ly0 = r % NQ;
    ly1 = r / NQ;
  }
  const int zbase = e * N3P + l0 + PX * l1;
  const bool read_out = !VOL || P.a_old != Real(0);
  // The tendency slab as this thread addresses it: variable v of shared index
  // s (which includes the element offset e * N3P) is tslab[v * TV + s]. TMA
  // layout: [element][variable][node] shifted by the source's misalignment;
  // otherwise [variable][element][node].
  const long long slab0 = e0 * (5 * N3);
  const unsigned off_q = unsigned(reinterpret_cast<unsigned long long>(P.q + slab0) & 15u);
  const unsigned off_p = unsigned(reinterpret_cast<unsigned long long>(P.phi + e0 * N3) & 15u);
  const unsigned off_o = unsigned(reinterpret_cast<unsigned long long>(P.out + slab0) & 15u);
  constexpr int TV = kBulk ? N3P : VS;
  Real* const tslab_own = kBulk ? reinterpret_cast<Real*>(smem_raw + Map::kTend + off_o) + 4 * e * N3P
                                : reinterpret_cast<Real*>(smem_raw + Map::kTend);
  Real* const tslab = tslab_own;

  // pitches of the three axes in shared (padded) and global node numbering
  auto spitch = [](int ax) { return ax == 0 ? 1 : (ax == 1 ? PX : PX * NQ); };
  auto gpitch = [](int ax) { return ax == 0 ? 1 : (ax == 1 ? NQ : NQ * NQ); };

  // the one-pass kernels keep the codes of the + faces only (the sweeps
  // evaluate those); the - faces are looked at once, right before the commit
  constexpr bool kShare = VOL && SURF && Share<NQ, sizeof(Real)>::value;
  int codes[6] = {-1, -1, -1, -1, -1, -1};
  unsigned roles = 0;
  if (SURF && active) {
#pragma unroll
    for (int lf = 0; lf < 6; ++lf)
      if (!kShare || (lf & 1)) codes[lf] = P.nbr[eg * 6 + lf];
    if (kShare && P.face_roles) roles = P.face_roles[eg];
  }

  // Neighbour state of face lf, fetched one face ahead of its use so the
  // (mostly L2-resident) gather hides behind arithmetic. The six neighbour
  // codes were read at kernel start, so a fetch is one round trip, not two.
  constexpr int FPI = Tile<NQ, sizeof(Real)>::FPI;
  NbrRaw<Real> cur[FPI]; // the gathered neighbour trace(s) of the next face iteration
  auto fetch = [&](int lf, NbrRaw<Real>& r) {
    const int dir = lf >> 1, side = lf & 1;
    const int d1 = dir == 2 ? 0 : dir + 1;
    const int d2 = d1 == 2 ? 0 : d1 + 1;
    r.code = lf == 0 ? codes[0] : lf == 1 ? codes[1] : lf == 2 ? codes[2]
             : lf == 3 ? codes[3] : lf == 4 ? codes[4] : codes[5];
    // thread (l0, l1) is face node (s, t) = (l0, l1): FaceIndexer::node
    const int tang = l0 * gpitch(d1) + l1 * gpitch(d2);
    gather_trace<Real, NQ>(P, r.code, dir, eg, (side ? 0 : NQ - 1) * gpitch(dir) + tang,
                           (side ? NQ - 1 : 0) * gpitch(dir) + tang, l, r);
  };
  // ---- phase A: primitives and logarithms, once per node ------------------
  // All global loads are issued before the first logarithm, so the CTA pays
  // for one HBM round trip. In the accumulate form the old contents of `out`
  // go straight into the slab (asynchronous copies, nobody waits for them
  // before the barrier that ends phase A). The slab then holds
  //   T = out_old + gain * (contributions),  gain = a_new / a_old,
  // and the commit writes out = a_old * T; with a_old == 0 it holds
  // a_new * (contributions) and `out` is never read.
  const Real* qe = P.q + eg * (5 * N3) + l;
  const Real* pe = P.phi + eg * N3 + l;
  Real qv[NQ][5], ph[NQ];
  {
    // One thread moves the CTA's slabs of q, phi and (accumulate form, odd
    // NQ) out with TMA bulk copies; everybody else only waits on the
    // mbarrier.
    if (tid == 0) {
      const long long left = P.ne - e0;
      const unsigned nel = left < EPB ? unsigned(left) : unsigned(EPB);
      const unsigned bq = (off_q + nel * 5 * N3 * unsigned(sizeof(Real)) + 15u) & ~15u;
      const unsigned bp = (off_p + nel * N3 * unsigned(sizeof(Real)) + 15u) & ~15u;
      const unsigned bo = (kBulk && read_out)
                              ? (off_o + nel * 5 * N3 * unsigned(sizeof(Real)) + 15u) & ~15u
                              : 0u;
      // the logarithm's table (FP64) comes the same way
      constexpr unsigned bt = unsigned(LogTab<Real>::kReals * sizeof(Real));
      mbar_expect_tx(mbar, bq + bp + bt);
      if (bo) mbar_expect_tx(mbar + 1, bo);
      if (bt) bulk_g2s(logtab, log_table_address(Real(0)), bt, mbar);
      bulk_g2s(smem_raw, reinterpret_cast<const char*>(P.q + slab0) - off_q, bq, mbar);
      bulk_g2s(smem_raw + Map::kStagePhi, reinterpret_cast<const char*>(P.phi + e0 * N3) - off_p, bp,
               mbar);
      if (kBulk && read_out)
        bulk_g2s(smem_raw + Map::kTend, reinterpret_cast<const char*>(P.out + slab0) - off_o, bo,
                 mbar + 1);
    }
    if (active) {
      if (!kBulk && read_out) {
        // padded slab (even NQ): element-wise asynchronous copies
        const Real* oe = P.out + eg * (5 * N3) + l;
#pragma unroll
        for (int k = 0; k < NQ; ++k)
#pragma unroll
          for (int v = 0; v < 5; ++v)
            cp_async<sizeof(Real)>(&tslab[v * TV + zbase + k * ZS], oe + v * N3 + k * N2);
      } else if (!read_out && SURF) {
        // the faces are the slab's first writers and touch surface nodes only
#pragma unroll
        for (int k = 0; k < NQ; ++k)
#pragma unroll
          for (int v = 0; v < 5; ++v) tslab[v * TV + zbase + k * ZS] = Real(0);
      }
    }
  }
  // the q / phi / out slabs of the CTA that will follow this one on the SM
  // (one resident wave ahead), so its phase A starts from L2, not HBM: three
  // bulk prefetches (TMA engine, no registers, no load/store-pipe traffic)
  // instead of one prefetch instruction per 128 bytes -- those brought in
  // single sectors, and a quarter of the demand loads still missed L2
  {
    long long en = e0 + static_cast<long long>(P.prefetch_ctas) * EPB;
    if (P.groups) {
      const unsigned nb = bid + unsigned(P.prefetch_ctas);
      en = nb < gridDim.x ? static_cast<long long>(P.groups[nb]) * EPB : P.ne;
    }
    if (tid < 3 && en + EPB <= P.ne && (tid < 2 || read_out)) {
      const char* base = tid == 0   ? reinterpret_cast<const char*>(P.q + en * (5 * N3))
                         : tid == 1 ? reinterpret_cast<const char*>(P.phi + en * N3)
                                    : reinterpret_cast<const char*>(P.out + en * (5 * N3));
      const unsigned bytes = (tid == 1 ? EPB * N3 : EPB * 5 * N3) * unsigned(sizeof(Real));
      // 16-byte aligned start and size that cover [base, base + bytes)
      const unsigned long long lo = reinterpret_cast<unsigned long long>(base) & ~15ull;
      const unsigned long long hi = (reinterpret_cast<unsigned long long>(base) + bytes + 15ull) & ~15ull;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"(unsigned(hi - lo))
                   : "memory");
    }
  }
  {
    // the slabs have landed: every thread takes the raw values of its z line
    // out of the staging area, which the node values are about to overwrite
    mbar_wait(mbar, 0);
    if (active) {
      const Real* sq = reinterpret_cast<const Real*>(smem_raw + off_q) + e * (5 * N3) + l;
      const Real* sp = reinterpret_cast<const Real*>(smem_raw + Map::kStagePhi + off_p) + e * N3 + l;
#pragma unroll
      for (int k = 0; k < NQ; ++k) {
#pragma unroll
        for (int v = 0; v < 5; ++v) qv[k][v] = sq[v * N3 + k * N2];
        ph[k] = sp[k * N2];
      }
    }
  }
  ESDG_CLK();
  __syncthreads();
  ESDG_CLK();
  if (active) {
    if (SURF && !VOL) { // surface-only kernel: registers to spare, fetch early
      fetch(0, cur[0]);
      if (FPI == 2) fetch(1, cur[FPI - 1]);
    }
    // The NQ nodes are independent and computed stage by stage so that their
    // reciprocal and logarithm chains interleave (a rolled one-node-per-
    // iteration loop has a fifth of the code but measured 3-6 % slower). A
    // non-physical node is only remembered here and reported after the loop.
    Real nvs[NQ][V_COUNT], prs[NQ];
    const unsigned badmask =
        node_vals_line<Real, NQ>(qv, ph, P.gas.gm1, logtab, nvs, prs);
#pragma unroll
    for (int k = 0; k < NQ; ++k) {
      const int s = zbase + k * ZS;
      store_node(vals, VS, s, nvs[k]);
    }
    const int bad = badmask ? __ffs(badmask) - 1 : -1;
    if (SURF && VOL) {
      // the trace(s) across the first face(s) phase C will evaluate: issued
      // here, not before the logarithms (registers the fused kernel's node
      // loop cannot spare); they land while the CTA gathers at the barrier
      if (kShare) {
        fetch(1, cur[0]);
      } else {
        fetch(0, cur[0]);
        if (FPI == 2) fetch(1, cur[FPI - 1]);
      }
    }
    if (bad >= 0) {
      const Real* qb = qe + bad * N2;
      Real qq[5], nv[V_COUNT], pr;
#pragma unroll
      for (int v = 0; v < 5; ++v) qq[v] = qb[v * N3];
      node_vals(qq, pe[bad * N2], P.gas.gm1, logtab, nv, pr);
      raise_flag(P.flag, P.flag_records, P.stage, 0, P.elem_offset + eg, l + bad * N2,
                 double(qq[0]), double(pr));
    }
  }
  ESDG_CLK();
  cp_async_wait_all(); // this thread's share of out_old is in the slab
  if (kShare) {
    // One-pass kernels: - faces (lf even) that no other element evaluates for
    // this one -- walls, ghost faces, neighbours that come later in the launch
    // order. Thread (l0, l1) is face node (s, t) = (l0, l1); the lift term
    // goes to this element's own slot of frec, from where the z-line owners
    // pick it up before the commit exactly like a pushed one. Only groups on
    // the rim of a partition or of the mesh come through here.
    if (__syncthreads_or(active && (roles & 7u) != 7u)) {
      if (active) {
#pragma unroll 1
        for (int f = 0; f < 3; ++f) {
          if (roles & (1u << f)) continue;
          const int dir = f;
          const int d1 = dir == 2 ? 0 : dir + 1;
          const int d2 = d1 == 2 ? 0 : d1 + 1;
          const int tang = l0 * gpitch(d1) + l1 * gpitch(d2);
          NbrRaw<Real> raw[1];
          raw[0].code = P.nbr[eg * 6 + 2 * f];
          gather_trace<Real, NQ>(P, raw[0].code, dir, eg, (NQ - 1) * gpitch(dir) + tang, tang, l,
                                 raw[0]);
          Node<Real> nb[1];
          face_pair_neighbours<Real, NQ, 1>(P, raw, dir, eg, l, logtab, nb);
          const Node<Real> own =
              load_node(vals, VS, e * N3P + l0 * spitch(d1) + l1 * spitch(d2), dir);
          Real fl[5], unused[5];
          face_fluxes<Real, NQ, false>(P, own, nb[0], 0, fl, unused);
          const Real lift = P.lift[dir];
          Real* rec = P.frec + (f * P.ne + eg) * FB + l;
#pragma unroll
          for (int v = 0; v < 5; ++v) rec[v * N2] = tag_term(lift * fl[v], P.epoch);
        }
      }
      // these slots are read back by a bulk copy (async proxy) one thread issues
      __threadfence();
      __syncthreads();
      if (tid == 0) asm volatile("fence.proxy.async;" ::: "memory");
    }
  } else {
    __syncthreads();
  }
  ESDG_CLK();

  // the old `out` has had phase A to arrive in the slab
  if (kBulk && read_out) mbar_wait(mbar + 1, 0);
  // ---- phase C: the six faces, thread per face node -----------------------
  // Every face subtracts its lift term from the shared tendency slab (zeroed
  // by the z-line owners in phase A). Faces of one direction share no node,
  // faces of different directions do (edges), hence the two barriers.
  if (kShare) {
    // One-pass kernels: only the three + faces (lf = 1, 3, 5) are evaluated
    // here, for both elements they separate: this element's lift term goes to
    // the slab, the other element's -- bitwise what it would compute itself,
    // see face_fluxes -- to its slot of frec if it expects it (roles). Once
    // every push of the group is out its flag goes up; that is long before
    // any group dispatched later gets to its commit, where it needs them.
#pragma unroll 1
    for (int dir = 0; dir < 3; ++dir) {
      if (active) {
        const int d1 = dir == 2 ? 0 : dir + 1;
        const int d2 = d1 == 2 ? 0 : d1 + 1;
        Node<Real> nb[1];
        const NbrRaw<Real>(&raw)[1] = reinterpret_cast<const NbrRaw<Real>(&)[1]>(cur[0]);
        face_pair_neighbours<Real, NQ, 1>(P, raw, dir, eg, l, logtab, nb);
        const int code = cur[0].code;
        if (dir < 2) fetch(2 * dir + 3, cur[0]);
        const int s_own = e * N3P + l0 * spitch(d1) + l1 * spitch(d2) + (NQ - 1) * spitch(dir);
        const Node<Real> own = load_node(vals, VS, s_own, dir);
        Real flo[5], fln[5];
        face_fluxes<Real, NQ, true>(P, own, nb[0], 1, flo, fln);
        const Real lift = P.lift[dir];
        if (roles & (8u << dir)) {
          Real* rec = P.frec + (dir * P.ne + code) * FB + l;
#pragma unroll
          for (int v = 0; v < 5; ++v) rec[v * N2] = tag_term(lift * fln[v], P.epoch);
        }
        Real* tn = tslab + (1 + dir) * TV;
        Real* tt1 = tslab + (1 + d1) * TV;
        Real* tt2 = tslab + (1 + d2) * TV;
        Real* t4 = tslab + 4 * TV;
        Real o[5];
        o[0] = tslab[s_own];
        o[1] = tn[s_own];
        o[2] = tt1[s_own];
        o[3] = tt2[s_own];
        o[4] = t4[s_own];
        // (the same truncation the other side's term goes through in its slot)
        tslab[s_own] = fma_(-P.gain, trunc_tag(lift * flo[0]), o[0]);
        tn[s_own] = fma_(-P.gain, trunc_tag(lift * flo[1]), o[1]);
        tt1[s_own] = fma_(-P.gain, trunc_tag(lift * flo[2]), o[2]);
        tt2[s_own] = fma_(-P.gain, trunc_tag(lift * flo[3]), o[3]);
        t4[s_own] = fma_(-P.gain, trunc_tag(lift * flo[4]), o[4]);
      }
      __syncthreads();
    }
  }
  if (SURF && !kShare) {
    // FPI faces per iteration (Tile<>::FPI). 2 = both faces of a direction as
    // two interleaved instruction streams: more ILP, but twice the loop
    // body. Where three or more CTAs in different phases share an SM the
    // instruction cache decides (N <= 4 in FP64: with FPI = 2, 10 % of the
    // stall samples were `no_instruction`, 85 % of them on the first
    // instruction of a 128-byte code line; 2 % with FPI = 1); the one or two
    // fat CTAs per SM of the high orders prefer the ILP.
#pragma unroll 1
    for (int lf = 0; lf < 6; lf += FPI) {
      const int dir = lf >> 1, side0 = lf & 1;
      if (active) {
        const int d1 = dir == 2 ? 0 : dir + 1;
        const int d2 = d1 == 2 ? 0 : d1 + 1;
        // node values of the neighbour traces, then -- the raw traces are
        // dead -- the next gather into the same registers; it lands while
        // this iteration's fluxes are evaluated
        Node<Real> nb[FPI];
        face_pair_neighbours<Real, NQ, FPI>(P, cur, dir, eg, l, logtab, nb);
        if (lf + FPI < 6) {
#pragma unroll
          for (int f = 0; f < FPI; ++f) fetch(lf + FPI + f, cur[f]);
        }
        // FaceIndexer::node (mesh.hpp:107-114): tangential axes d1, d2
        const int s0 = e * N3P + l0 * spitch(d1) + l1 * spitch(d2);
        int s_own[FPI];
        Node<Real> own[FPI];
#pragma unroll
        for (int f = 0; f < FPI; ++f) {
          s_own[f] = s0 + ((side0 + f) ? (NQ - 1) * spitch(dir) : 0);
          own[f] = load_node(vals, VS, s_own[f], dir);
        }
        Real c[FPI][5], o[FPI][5];
        face_pair_contribution<Real, NQ, FPI, !(VOL && SURF)>(P, own, nb, dir, side0, c);
        Real* tn = tslab + (1 + dir) * TV;
        Real* tt1 = tslab + (1 + d1) * TV;
        Real* tt2 = tslab + (1 + d2) * TV;
        Real* t4 = tslab + 4 * TV;
#pragma unroll
        for (int f = 0; f < FPI; ++f) {
          o[f][0] = tslab[s_own[f]];
          o[f][1] = tn[s_own[f]];
          o[f][2] = tt1[s_own[f]];
          o[f][3] = tt2[s_own[f]];
          o[f][4] = t4[s_own[f]];
        }
#pragma unroll
        for (int f = 0; f < FPI; ++f) {
          tslab[s_own[f]] = fma_(-P.gain, c[f][0], o[f][0]);
          tn[s_own[f]] = fma_(-P.gain, c[f][1], o[f][1]);
          tt1[s_own[f]] = fma_(-P.gain, c[f][2], o[f][2]);
          tt2[s_own[f]] = fma_(-P.gain, c[f][3], o[f][3]);
          t4[s_own[f]] = fma_(-P.gain, c[f][4], o[f][4]);
        }
      }
      // faces of one direction share no node, faces of different directions do
      if (((lf + FPI) & 1) == 0) __syncthreads();
    }
  }

  ESDG_CLK();
  // ---- phase B: the three line sweeps, one code instance -------------------
  // x and y results are handed to the z-line owners through the shared slab;
  // the z sweep stays in registers because the same thread commits that line.
  Real acc[NQ][5];
  Real pull_z[5] = {Real(0), Real(0), Real(0), Real(0), Real(0)}; // lift term of the - z face
#pragma unroll
  for (int i = 0; i < NQ; ++i)
#pragma unroll
    for (int v = 0; v < 5; ++v) acc[i][v] = Real(0);
  if (VOL) {
#ifdef ESDG_TUNE_UNROLL_DIR
#pragma unroll
#else
#pragma unroll 1
#endif
    for (int dir = 0; dir < 3; ++dir) {
      if (kShare && tid == 0) {
        // the landing area is free: a barrier ended phase C / the previous
        // direction, whose pulled values every thread has taken out by then
        const long long left = P.ne - e0;
        const unsigned nel = left < EPB ? unsigned(left) : unsigned(EPB);
        const unsigned bytes = nel * FB * unsigned(sizeof(Real));
        fence_proxy_async_smem(); // generic-proxy reads of the area -> the copy's writes
        mbar_expect_tx(mbar, bytes);
        bulk_g2s(pbuf, P.frec + (dir * P.ne + e0) * FB, bytes, mbar);
      }
      // the line of this direction: element, and the slab as addressed for it
      const int ed = (kYPerm && dir == 1) ? ey : e;
      Real* const tslab = (kYPerm && kBulk && dir == 1) ? tslab_own + 4 * (ey - e) * N3P : tslab_own;
      if (kYPerm ? (e0 + ed < P.ne) : active) {
        const int base = dir == 0 ? e * N3P + PX * l
                                  : (dir == 1 ? ed * N3P + ly0 + ZS * ly1 : zbase);
        const int stride = dir == 0 ? 1 : (dir == 1 ? PX : ZS);
#pragma unroll
        for (int i = 0; i < NQ; ++i)
#pragma unroll
          for (int v = 0; v < 5; ++v) acc[i][v] = Real(0);
        // One-pass kernels, "pulls": the lift term of the - face this line
        // starts on (lf = 2 dir) lies in the element's block of frec -- pushed
        // by the element across the face during its phase C, or put there by
        // this group after phase A. One bulk copy (issued below, before the
        // line loads of all threads) brings the group's blocks of this
        // direction into shared memory while the pair fluxes are evaluated:
        // no register, no load/store-pipe instruction, nobody waits for L2.
        // x and y lines of a Cartesian mesh see a constant potential: no
        // gravity term there (a second, shorter code instance of the sweep)
        if (FlatXY<NQ, sizeof(Real)>::value && SURF && P.flat_phi && dir < 2)
          sweep_line<Real, NQ, !(VOL && SURF), true>(P, vals, VS, base, stride, dir, acc);
        else
          sweep_line<Real, NQ, !(VOL && SURF), false, RUNG>(P, vals, VS, base, stride, dir, acc,
                                                            logtab);
        Real pull[5];
        if (kShare) {
          // The thread that sweeps a line is the face node (s, t) of the
          // line's two faces: (l0, l1), for y lines (l1, l0).
          const int fn = dir == 1 ? ly1 + NQ * ly0 : l;
          mbar_wait(mbar, (dir + 1) & 1);
          bool filled = true;
#pragma unroll
          for (int v = 0; v < 5; ++v) {
            pull[v] = pbuf[ed * FB + v * N2 + fn];
            filled = filled && has_tag(pull[v], P.epoch);
          }
          if (!filled) {
            const Real* slot = P.frec + (dir * P.ne + e0 + ed) * FB + fn;
#pragma unroll 1
            for (int v = 0; v < 5; ++v) {
              const Real x = wait_filled(slot + v * N2, P.epoch, P.sync_error, P.wait_limit_ns);
              pull[0] = v == 0 ? x : pull[0];
              pull[1] = v == 1 ? x : pull[1];
              pull[2] = v == 2 ? x : pull[2];
              pull[3] = v == 3 ? x : pull[3];
              pull[4] = v == 4 ? x : pull[4];
            }
          }
#pragma unroll
          for (int v = 0; v < 5; ++v) pull[v] = trunc_tag(pull[v]);
          if (dir == 2) {
#pragma unroll
            for (int v = 0; v < 5; ++v) pull_z[v] = pull[v];
          }
        }
        if (dir < 2) {
          // un-rotate into the slab: normal -> 1+dir, then cyclic. Without
          // faces the x sweep is the slab's first writer and simply stores;
          // otherwise all old values are fetched before the first store
          // (one shared-memory round trip instead of 5 NQ dependent ones:
          // the compiler cannot prove that the five arrays do not alias).
          const int d1 = dir + 1, d2 = dir == 0 ? 2 : 0;
          Real* tn = tslab + (1 + dir) * TV;
          Real* tt1 = tslab + (1 + d1) * TV;
          Real* tt2 = tslab + (1 + d2) * TV;
          Real* t4 = tslab + 4 * TV;
          const Real scale = P.gain * P.metric[dir];
          if (SURF || dir != 0 || read_out) {
            Real old[NQ][5];
#pragma unroll
            for (int i = 0; i < NQ; ++i) {
              const int s = base + i * stride;
              old[i][0] = tslab[s];
              old[i][1] = tn[s];
              old[i][2] = tt1[s];
              old[i][3] = tt2[s];
              old[i][4] = t4[s];
            }
#pragma unroll
            for (int i = 0; i < NQ; ++i)
#pragma unroll
              for (int v = 0; v < 5; ++v) acc[i][v] = fma_(scale, acc[i][v], old[i][v]);
            if (kShare) {
              // the - face at the line's first node, same rotated frame
#pragma unroll
              for (int v = 0; v < 5; ++v) acc[0][v] = fma_(-P.gain, pull[v], acc[0][v]);
            }
          } else {
#pragma unroll
            for (int i = 0; i < NQ; ++i)
#pragma unroll
              for (int v = 0; v < 5; ++v) acc[i][v] = scale * acc[i][v];
          }
#pragma unroll
          for (int i = 0; i < NQ; ++i) {
            const int s = base + i * stride;
            tslab[s] = acc[i][0];
            tn[s] = acc[i][1];
            tt1[s] = acc[i][2];
            tt2[s] = acc[i][3];
            t4[s] = acc[i][4];
          }
        }
      }
      if (dir < 2) __syncthreads();
    }
  }

  ESDG_CLK();
  // ---- commit: slab (old out, faces, x, y) + registers (z) on the z line ----
  // acc: rotated frame of z: normal -> var 3, t1 = x -> 1, t2 = y -> 2
  // commit (solver.hpp:199-223), one z line per thread. With the TMA slab
  // layout (odd NQ) the results go back into shared memory -- k in place in
  // the slab, q_next into the dead front of the node-value arrays, both in
  // the state registers' [element][variable][node] order -- and one thread
  // ships each slab with a bulk store: the 16-byte-aligned interior by TMA,
  // the at most three Reals in front of / behind it by ordinary stores.
  // Otherwise every thread stores its z line, coalesced over l. Global loads
  // (only the fused stage update and the Coriolis source need any) are issued
  // before the first store: the compiler cannot prove that out / q / q_next
  // do not alias.
  const bool update = VOL && P.q_next != nullptr;
  const bool source = VOL && P.with_source != 0;
  const unsigned off_n =
      update ? unsigned(reinterpret_cast<unsigned long long>(P.q_next + slab0) & 15u) : 0u;
  Real knew[NQ][5], qc[NQ][5];
  if (active) {
    const Real* __restrict__ qe = P.q + eg * (5 * N3) + l;
    Real cf = Real(0);
    if (update) {
#pragma unroll
      for (int k = 0; k < NQ; ++k)
#pragma unroll
        for (int v = 0; v < 5; ++v) qc[k][v] = qe[v * N3 + k * N2];
    } else if (source) {
      // coriolis_source (physics.hpp:297-306) only needs the momenta
#pragma unroll
      for (int k = 0; k < NQ; ++k) {
        qc[k][1] = qe[1 * N3 + k * N2];
        qc[k][2] = qe[2 * N3 + k * N2];
      }
    }
    if (source) cf = P.cor_f[P.ylevel[eg] * NQ + l1];
    if (VOL || !kBulk) {
#pragma unroll
      for (int k = 0; k < NQ; ++k) {
        const int s = zbase + k * ZS;
#pragma unroll
        for (int v = 0; v < 5; ++v) knew[k][v] = tslab[v * TV + s];
      }
    }
    if (VOL) {
      // acc still lacks the z metric
      const Real zscale = P.gain * P.metric[2];
#pragma unroll
      for (int k = 0; k < NQ; ++k) {
        knew[k][0] = fma_(zscale, acc[k][0], knew[k][0]);
        knew[k][1] = fma_(zscale, acc[k][2], knew[k][1]);
        knew[k][2] = fma_(zscale, acc[k][3], knew[k][2]);
        knew[k][3] = fma_(zscale, acc[k][1], knew[k][3]);
        knew[k][4] = fma_(zscale, acc[k][4], knew[k][4]);
      }
      if (kShare) {
        // the - z face at the line's first node (normal -> var 3, x, y)
        knew[0][0] = fma_(-P.gain, pull_z[0], knew[0][0]);
        knew[0][3] = fma_(-P.gain, pull_z[1], knew[0][3]);
        knew[0][1] = fma_(-P.gain, pull_z[2], knew[0][1]);
        knew[0][2] = fma_(-P.gain, pull_z[3], knew[0][2]);
        knew[0][4] = fma_(-P.gain, pull_z[4], knew[0][4]);
      }
      if (source) {
        // h = (0, f q2, -f q1, 0, 0)
        const Real gcf = P.gain * cf;
#pragma unroll
        for (int k = 0; k < NQ; ++k) {
          knew[k][1] = fma_(gcf, qc[k][2], knew[k][1]);
          knew[k][2] = fma_(-gcf, qc[k][1], knew[k][2]);
        }
      }
#pragma unroll
      for (int k = 0; k < NQ; ++k)
#pragma unroll
        for (int v = 0; v < 5; ++v) knew[k][v] = P.fin * knew[k][v];
    }
    if (!kBulk) {
      Real* __restrict__ oe = P.out + eg * (5 * N3) + l;
#pragma unroll
      for (int k = 0; k < NQ; ++k)
#pragma unroll
        for (int v = 0; v < 5; ++v) oe[v * N3 + k * N2] = knew[k][v];
      if (update) {
        // LSRK register update folded into the same pass (Solver::axpy,
        // solver.hpp:342-353): q_next = q + b k. q is double buffered
        // because neighbouring CTAs still read this element's faces.
        Real* __restrict__ qn = P.q_next + eg * (5 * N3) + l;
#pragma unroll
        for (int k = 0; k < NQ; ++k)
#pragma unroll
          for (int v = 0; v < 5; ++v)
            qn[v * N3 + k * N2] = qc[k][v] + P.b_upd * knew[k][v];
      }
    }
  }
  if (kBulk) {
    // q_next goes where other threads may still be reading node values for
    // their z sweep: wait for them
    if (update) __syncthreads();
    Real* stage_n = reinterpret_cast<Real*>(smem_raw + off_n);
    if (active) {
      if (VOL) {
#pragma unroll
        for (int k = 0; k < NQ; ++k)
#pragma unroll
          for (int v = 0; v < 5; ++v) tslab[v * TV + zbase + k * ZS] = knew[k][v];
      }
      if (update) {
#pragma unroll
        for (int k = 0; k < NQ; ++k)
#pragma unroll
          for (int v = 0; v < 5; ++v)
            stage_n[(e * 5 + v) * N3 + l + k * N2] = qc[k][v] + P.b_upd * knew[k][v];
      }
    }
    fence_proxy_async_smem(); // generic-proxy writes -> visible to the TMA engine
    __syncthreads();
    const long long left = P.ne - e0;
    const unsigned nel = left < EPB ? unsigned(left) : unsigned(EPB);
    const unsigned bytes = nel * 5 * N3 * unsigned(sizeof(Real));
    // slab `which`: 0 = out from the tendency slab, 1 = q_next from the staging area
    auto ship = [&](int which, bool interior) {
      char* g = reinterpret_cast<char*>(which == 0 ? P.out + slab0 : P.q_next + slab0);
      const char* sm = reinterpret_cast<const char*>(smem_raw) +
                       (which == 0 ? Map::kTend + off_o : size_t(off_n));
      const unsigned head = (16u - unsigned(reinterpret_cast<unsigned long long>(g) & 15u)) & 15u;
      const unsigned body = (bytes - head) & ~15u;
      if (interior) {
        bulk_s2g(g + head, sm + head, body);
      } else {
        for (unsigned o = 0; o < head; o += sizeof(Real))
          *reinterpret_cast<Real*>(g + o) = *reinterpret_cast<const Real*>(sm + o);
        for (unsigned o = head + body; o < bytes; o += sizeof(Real))
          *reinterpret_cast<Real*>(g + o) = *reinterpret_cast<const Real*>(sm + o);
      }
    };
    if (tid == 0) {
      ship(0, true);
      if (update) ship(1, true);
      bulk_store_commit_and_wait_read();
    } else if (tid == 32) {
      ship(0, false);
    } else if (tid == 64 && update) {
      ship(1, false);
    }
  }
#ifdef ESDG_TUNE_PHASE_CLOCKS
  ESDG_CLK();
  if (tid == 0 && blockIdx.x == 40000)
    printf("phase clocks VOL=%d SURF=%d: loads %lld | table barrier %lld | nodes %lld | barrier %lld | faces %lld | sweeps %lld | commit %lld | total %lld\n",
           int(VOL), int(SURF), tclk[1] - tclk[0], tclk[2] - tclk[1], tclk[3] - tclk[2], tclk[4] - tclk[3],
           tclk[5] - tclk[4], tclk[6] - tclk[5], tclk[7] - tclk[6], tclk[7] - tclk[0]);
#endif
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

} // namespace dev
} // namespace esdg_b200
