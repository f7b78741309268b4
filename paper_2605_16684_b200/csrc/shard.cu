// shard.cu -- level-1 C ABI: one element partition resident on one GPU
// (include/esdg_b200.h, "shard" entry points). Owns device memory, derives
// the kernel constants exactly like the reference's Operators<Real>
// (core/include/esdg/kernels.hpp:70-92) and launches K1-K5.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "esdg_b200.h"
#include "esdg_kernels.cuh"
#include "esdg_launch.hpp"
#include "host/host_types.hpp"
#include "shard_internal.hpp"

namespace esdg_b200 {

thread_local std::string g_last_message;

void set_message(const std::string& m) { g_last_message = m; }

int cuda_fail(cudaError_t e, const char* what) {
  g_last_message = std::string(what) + ": " + cudaGetErrorString(e);
  return ESDG_B200_CUDA;
}

#define CU(call)                                                               \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);                        \
  } while (0)

namespace {

constexpr unsigned long long kNoFlag = ~0ull;

// ---- K6: per-element reductions ---------------------
// quadrature_total / total_entropy / entropy_production
// (diagnostics.hpp:30-106) and compute_stable_dt (time_integration.hpp:55-92)
// without moving the state to the host: one warp per element evaluates the
// per-node terms in 64-bit exactly as the reference writes them, sums them
// with Neumaier compensation (lanes over nodes, then lane 0 over lanes, a
// fixed order) and stores ONE double per element; the host finishes with a
// compensated sum over elements in Morton order. The dt term is a minimum and
// therefore bitwise the reference's value.
struct ReduceParams {
  const void* q;
  const void* k;
  const void* phi;
  const double* node_weight; // [n3]  J w_a w_b w_c
  const double* dx;          // [3][nq] half width * LGL gap
  double* out;               // [ne]
  unsigned* bad;
  double gamma;
  long long ne;
  int nq, n3, var;
};

__device__ __forceinline__ void neumaier_add(double& s, double& c, double x) {
  const double t = s + x;
  c += (fabs(s) >= fabs(x)) ? (s - t) + x : (x - t) + s;
  s = t;
}

template <class Real, int KIND>
__global__ void __launch_bounds__(256) reduce_kernel(const ReduceParams P) {
  const int lane = threadIdx.x & 31;
  const long long e = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (e >= P.ne) return;
  const Real* q = static_cast<const Real*>(P.q) + e * 5 * P.n3;
  const Real* k = static_cast<const Real*>(P.k) + e * 5 * P.n3;
  const Real* ph = static_cast<const Real*>(P.phi) + e * P.n3;
  const int n2 = P.nq * P.nq;
  const double gamma = P.gamma;
  double s = 0.0, c = 0.0, mn = __longlong_as_double(0x7ff0000000000000LL);
  bool bad = false;
  for (int n = lane; n < P.n3; n += 32) {
    if constexpr (KIND == 0) {
      neumaier_add(s, c, P.node_weight[n] * double(q[P.var * P.n3 + n]));
    } else {
    double u[5];
#pragma unroll
    for (int v = 0; v < 5; ++v) u[v] = double(q[v * P.n3 + n]);
    const double phi = double(ph[n]);
    if (KIND == 3) {
      if (!(u[0] > 0.0)) { bad = true; continue; }
      const double ke = 0.5 * (u[1] * u[1] + u[2] * u[2] + u[3] * u[3]) / u[0];
      const double p = (gamma - 1.0) * (u[4] - ke - u[0] * phi);
      if (!(p > 0.0)) { bad = true; continue; }
      const double cs = sqrt(gamma * p / u[0]);
      const int idx[3] = {n % P.nq, (n / P.nq) % P.nq, n / n2};
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double vel = fabs(u[1 + d] / u[0]);
        mn = fmin(mn, P.dx[d * P.nq + idx[d]] / (vel + cs));
      }
      continue;
    }
    const double rho = u[0];
    const double ke = 0.5 * (u[1] * u[1] + u[2] * u[2] + u[3] * u[3]) / rho;
    const double p = (gamma - 1.0) * (u[4] - ke - rho * phi);
    if (!(rho > 0.0) || !(p > 0.0)) bad = true;
    const double ent = log(p) - gamma * log(rho);
    if (KIND == 1) {
      neumaier_add(s, c, P.node_weight[n] * (-rho * ent / (gamma - 1.0)));
    } else {
      double r[5];
#pragma unroll
      for (int v = 0; v < 5; ++v) r[v] = double(k[v * P.n3 + n]);
      const double bq = rho / (2.0 * p);
      const double w[3] = {u[1] / rho, u[2] / rho, u[3] / rho};
      const double w2 = w[0] * w[0] + w[1] * w[1] + w[2] * w[2];
      const double vv[5] = {(gamma - ent) / (gamma - 1.0) - bq * (w2 - 2.0 * phi),
                            2.0 * bq * w[0], 2.0 * bq * w[1], 2.0 * bq * w[2], -2.0 * bq};
      neumaier_add(s, c, P.node_weight[n] * (vv[0] * r[0] + vv[1] * r[1] + vv[2] * r[2] +
                                             vv[3] * r[3] + vv[4] * r[4]));
    }
    }
  }
  if (KIND == 3) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  } else {
    for (int src = 1; src < 32; ++src) {
      const double so = __shfl_sync(0xffffffffu, s, src);
      const double co = __shfl_sync(0xffffffffu, c, src);
      if (lane == 0) {
        neumaier_add(s, c, so);
        c += co;
      }
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(P.bad, 1u);
  if (lane == 0) P.out[e] = KIND == 3 ? mn : s + c;
}

template <class Real>
class Shard final : public ShardBase {
public:
  ~Shard() override { release(); }

  int init(const esdg_b200_shard_desc& d) {
    nq_ = d.nq;
    n2_ = nq_ * nq_;
    n3_ = n2_ * nq_;
    ne_ = d.n_elements;
    elem_offset_ = d.elem_offset;
    device_ = d.device;
    n_ghost_ = d.n_ghost;
    n_send_ = d.n_send;
    dissipation_ = d.dissipation;
    coriolis_mode_ = d.coriolis_mode;
    CU(cudaSetDevice(device_));
    cudaDeviceProp prop;
    CU(cudaGetDeviceProperties(&prop, device_));
    if (prop.major < 10) {
      set_message("esdg_b200 needs an sm_100 class GPU (found sm_" +
                  std::to_string(prop.major) + std::to_string(prop.minor) + ")");
      return ESDG_B200_CUDA;
    }
    CU(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    // how long a pull may poll for a pushed lift term before the launch is
    // declared stuck (rhs_kernel, wait_filled); 0 = no limit (under a debugger)
    if (const char* ms = std::getenv("ESDG_B200_WAIT_LIMIT_MS"))
      wait_limit_ns_ = 1000000ull * std::strtoull(ms, nullptr, 10);
    sm_count_ = prop.multiProcessorCount;
    smem_per_sm_ = prop.sharedMemPerMultiprocessor;

    // Operators<Real> (kernels.hpp:79-91): 64-bit operators rounded to Real
    std::vector<Real> D(static_cast<size_t>(n2_)), w(static_cast<size_t>(nq_));
    for (int i = 0; i < n2_; ++i) D[size_t(i)] = Real(d.diff[i]);
    for (int i = 0; i < nq_; ++i) w[size_t(i)] = Real(d.weights[i]);
    for (int k = 0; k < 3; ++k) {
      metric_[k] = Real(d.metric[k]);
      lift_[k] = metric_[k] / w[0];
    }
    // The flux-differencing coefficient -(2 g_d D_ij) (kernels.hpp:187,
    // 224-225) is applied in two factors: -(2 D_ij) inside the line sweep --
    // the same for all three directions, so the kernel reads it as an
    // immediate constant-bank operand -- and the metric g_d once per node
    // when the sweep's sums are handed on.
    negd_.assign(size_t(n2_), Real(0));
    for (int i = 0; i < n2_; ++i) negd_[size_t(i)] = -(Real(2) * D[size_t(i)]);
    // D_ii is analytically zero at interior LGL nodes; the negative-row-sum
    // construction (reference_element.cpp:135) leaves an O(1e-16) residue.
    // Flush it so the kernel can skip those point fluxes: the dropped term is
    // below 1e-15 of the neighbouring off-diagonal terms.
    for (int i = 1; i + 1 < nq_; ++i) {
      const double dii = std::abs(d.diff[i * nq_ + i]);
      if (dii <= 1e-13 * std::abs(d.diff[0]))
        negd_[size_t(i * nq_ + i)] = Real(0);
    }
    const Real gamma = Real(d.gamma), R = Real(d.gas_R);
    gas_.gamma = gamma;
    gas_.gm1 = gamma - Real(1);
    gas_.cg = Real(1) / (Real(2) * (gamma - Real(1)));
    gas_.igm1 = Real(1) / (gamma - Real(1));
    gas_.Rgas = R;
    gas_.half_over_gamma = Real(1) / (Real(2) * gamma);
    gas_.gm1_over_gamma = (gamma - Real(1)) / gamma;
    gas_.half_over_R = Real(1) / (Real(2) * R);

    const size_t state_bytes = sizeof(Real) * size_t(ne_) * 5 * size_t(n3_);
    // + 64: slack for the kernels' 16-byte rounded TMA bulk reads
    CU(cudaMalloc(&q_, state_bytes + 64));
    CU(cudaMalloc(&k_, state_bytes + 64));
    CU(cudaMemset(q_, 0, state_bytes));
    CU(cudaMemset(k_, 0, state_bytes));
    CU(alloc_copy(&phi_, d.phi, sizeof(Real) * size_t(ne_) * size_t(n3_)));
    {
      // Is the potential constant along every x and y line (phi = g z on the
      // reference's Cartesian lattice, solver.hpp:166-176)? Then the volume
      // sweeps in x and y skip the gravity term, which is exactly zero there.
      const Real* ph = static_cast<const Real*>(d.phi);
      bool flat = true;
      for (int64_t e = 0; e < ne_ && flat; ++e)
        for (int c = 0; c < nq_ && flat; ++c) {
          const Real* row = ph + size_t(e) * size_t(n3_) + size_t(c) * size_t(n2_);
          for (int n = 1; n < n2_; ++n)
            if (!(row[n] == row[0])) {
              flat = false;
              break;
            }
        }
      flat_phi_ = flat ? 1 : 0;
    }
    CU(alloc_copy(&nbr_, d.nbr, sizeof(int32_t) * size_t(ne_) * 6));
    {
      const int rc = build_groups(d.nbr);
      if (rc != ESDG_B200_OK) return rc;
    }
    CU(alloc_copy(&ghost_phi_, d.ghost_phi,
                  sizeof(Real) * size_t(n_ghost_) * size_t(n2_)));
    CU(alloc_copy(&send_elem_, d.send_elem, sizeof(int32_t) * size_t(n_send_)));
    CU(alloc_copy(&send_face_, d.send_face, sizeof(int32_t) * size_t(n_send_)));
    const size_t halo = sizeof(Real) * 5 * size_t(n2_);
    CU(cudaMalloc(&recv_, n_ghost_ ? halo * size_t(n_ghost_) : 16));
    CU(cudaMalloc(&send_, n_send_ ? halo * size_t(n_send_) : 16));
    CU(cudaMemset(recv_, 0, n_ghost_ ? halo * size_t(n_ghost_) : 16));
    if (coriolis_mode_ != 0) {
      if (!d.elem_ylevel || !d.coriolis_f || d.n_ylevels < 1) {
        set_message("coriolis_mode != 0 needs elem_ylevel and coriolis_f");
        return ESDG_B200_BADARG;
      }
      CU(alloc_copy(&ylevel_, d.elem_ylevel, sizeof(int32_t) * size_t(ne_)));
      CU(alloc_copy(&cor_f_, d.coriolis_f,
                    sizeof(Real) * size_t(d.n_ylevels) * size_t(nq_)));
    }
    // [0] non-physical-state key, [1] a face-contribution wait timed out
    CU(cudaMalloc(&flag_, 2 * sizeof(unsigned long long)));
    CU(cudaMemset(flag_, 0, 2 * sizeof(unsigned long long)));
    CU(cudaMemcpy(flag_, &kNoFlag, sizeof kNoFlag, cudaMemcpyHostToDevice));
    CU(cudaMallocHost(&flag_host_, 2 * sizeof(unsigned long long)));
    CU(cudaMalloc(&flag_records_, sizeof(dev::FlagRecord) * dev::kFlagSlots));
    CU(cudaMemset(flag_records_, 0xff, sizeof(dev::FlagRecord) * dev::kFlagSlots));
    // The copies and fills above went through the legacy stream, and a copy
    // from pageable host memory returns once the data are STAGED, not once they
    // are on the device; the kernels run on a non-blocking stream that the
    // legacy stream does not order against.
    CU(cudaDeviceSynchronize());
    return ESDG_B200_OK;
  }

  int upload(int reg, const void* host, int64_t first, int64_t count,
             cudaStream_t st, bool async) override {
    if (!range_ok(reg, first, count) || !host) return bad("upload: bad range");
    CU(cudaSetDevice(device_));
    const size_t per = sizeof(Real) * 5 * size_t(n3_);
    Real* dst = reg_ptr(reg) + size_t(first) * 5 * size_t(n3_);
    if (async) {
      CU(cudaMemcpyAsync(dst, host, per * size_t(count), cudaMemcpyHostToDevice, pick(st)));
    } else {
      // On the compute stream itself, then wait: behind whatever still reads or
      // writes the register, in front of every later kernel. (A blocking
      // cudaMemcpy from pageable memory returns when the data are staged -- the
      // DMA runs on the legacy stream, which the non-blocking compute stream
      // does not wait for: a kernel launched right after could read a register
      // that had not arrived yet. Seen as a rare gross mismatch of the
      // accumulate form in tests/test_gpu_face_sharing.py.)
      CU(cudaMemcpyAsync(dst, host, per * size_t(count), cudaMemcpyHostToDevice, stream_));
      CU(cudaStreamSynchronize(stream_));
    }
    return ESDG_B200_OK;
  }

  int download(int reg, void* host, int64_t first, int64_t count,
               cudaStream_t st, bool async) override {
    if (!range_ok(reg, first, count) || !host) return bad("download: bad range");
    CU(cudaSetDevice(device_));
    const size_t per = sizeof(Real) * 5 * size_t(n3_);
    const Real* src = reg_ptr(reg) + size_t(first) * 5 * size_t(n3_);
    if (async) {
      CU(cudaMemcpyAsync(host, src, per * size_t(count), cudaMemcpyDeviceToHost, pick(st)));
    } else {
      CU(cudaMemcpyAsync(host, src, per * size_t(count), cudaMemcpyDeviceToHost, stream_));
      CU(cudaStreamSynchronize(stream_));
    }
    return ESDG_B200_OK;
  }

  void* register_ptr(int reg) override {
    return (reg == 0 || reg == 1) ? reg_ptr(reg) : nullptr;
  }
  void* send_ptr() override { return send_; }
  void* recv_ptr() override { return recv_; }
  cudaStream_t stream() override { return stream_; }
  int device() const override { return device_; }
  int64_t n_elements() const override { return ne_; }
  int64_t n_ghost() const override { return n_ghost_; }
  int64_t n_send() const override { return n_send_; }
  size_t trace_bytes() const override { return sizeof(Real) * 5 * size_t(n2_); }
  int64_t launch_count() const override { return launches_; }
  void set_dissipation(int on) override { dissipation_ = on; }
  void set_face_sharing(int on) override { share_faces_ = on; }
  void set_variant(int variant) override { variant_ = variant; }

  int pack(int src, cudaStream_t st) override {
    if (src != 0 && src != 1) return bad("pack: bad register");
    if (n_send_ == 0) return ESDG_B200_OK;
    CU(cudaSetDevice(device_));
    cudaError_t e = cudaErrorInvalidValue;
    switch (nq_) {
#define ESDG_CASE(NQ)                                                          \
  case NQ:                                                                     \
    e = launch_pack<Real, NQ>(reg_ptr(src), send_elem_, send_face_, send_,     \
                              n_send_, pick(st));                              \
    break;
      ESDG_CASE(2) ESDG_CASE(3) ESDG_CASE(4) ESDG_CASE(5) ESDG_CASE(6)
      ESDG_CASE(7) ESDG_CASE(8)
#undef ESDG_CASE
    }
    if (e != cudaSuccess) return cuda_fail(e, "pack_kernel");
    ++launches_;
    return ESDG_B200_OK;
  }

  int rhs(int mode, int src, int dst, double a_old, double a_new,
          int with_source, int stage, int part, cudaStream_t st) override {
    if ((src != 0 && src != 1) || (dst != 0 && dst != 1) || src == dst)
      return bad("rhs: src and dst must be distinct registers 0/1");
    if (part < ESDG_B200_PART_ALL || part > ESDG_B200_PART_BOUNDARY) return bad("rhs: bad part");
    return launch(mode, src, dst, a_old, a_new, 0.0, nullptr, with_source, stage, part, st);
  }

  int stage_fused(double a_old, double a_new, double b, int with_source, int stage,
                  int part, cudaStream_t st) override {
    if (part < ESDG_B200_PART_ALL || part > ESDG_B200_PART_BOUNDARY)
      return bad("stage_fused: bad part");
    CU(cudaSetDevice(device_));
    if (!q_alt_) {
      const size_t state_bytes = sizeof(Real) * size_t(ne_) * 5 * size_t(n3_);
      CU(cudaMalloc(&q_alt_, state_bytes + 64));
    }
    const int rc = launch(kModeFused, 0, 1, a_old, a_new, b, q_alt_, with_source, stage, part, st);
    // the new state is current once every element has been through the stage
    if (rc == ESDG_B200_OK && part != ESDG_B200_PART_INTERIOR) std::swap(q_, q_alt_);
    return rc;
  }

  int stage_fused_range(double a_old, double a_new, double b, int with_source, int stage,
                        int64_t first_group, int64_t n_groups, bool last,
                        cudaStream_t st) override {
    const int64_t total = (ne_ + epb_ - 1) / epb_;
    if (first_group < 0 || n_groups < 0 || first_group + n_groups > total)
      return bad("stage_fused_range: bad group range");
    CU(cudaSetDevice(device_));
    if (!q_alt_) {
      const size_t state_bytes = sizeof(Real) * size_t(ne_) * 5 * size_t(n3_);
      CU(cudaMalloc(&q_alt_, state_bytes + 64));
    }
    int rc = ESDG_B200_OK;
    // the runs of one stage must come in ascending order, starting at group 0
    // (an element pulls face contributions from elements before it)
    if (first_group == 0) range_next_ = 0;
    if (first_group != range_next_) return bad("stage_fused_range: runs must be consecutive from group 0");
    range_next_ = first_group + n_groups;
    if (n_groups > 0) {
      range_first_ = first_group;
      range_count_ = n_groups;
      rc = launch(kModeFused, 0, 1, a_old, a_new, b, q_alt_, with_source, stage, ESDG_B200_PART_ALL, st);
      range_first_ = range_count_ = 0;
    }
    if (rc == ESDG_B200_OK && last) std::swap(q_, q_alt_);
    return rc;
  }
  int elements_per_group() const override { return epb_; }

  int stream_buffers(void** in, void** out) override {
    CU(cudaSetDevice(device_));
    const size_t state_bytes = sizeof(Real) * size_t(ne_) * 5 * size_t(n3_);
    if (!q_in_) CU(cudaMalloc(&q_in_, state_bytes + 64));
    if (!q_out_) CU(cudaMalloc(&q_out_, state_bytes + 64));
    if (in) *in = q_in_;
    if (out) *out = q_out_;
    return ESDG_B200_OK;
  }
  void stream_rotate() override {
    Real* const freed = q_out_;
    q_out_ = q_;
    q_ = q_in_;
    q_in_ = freed;
  }

  int64_t part_elements(int part) const override {
    return part == ESDG_B200_PART_ALL        ? ne_
           : part == ESDG_B200_PART_INTERIOR ? n_part_elems_[0]
           : part == ESDG_B200_PART_BOUNDARY ? n_part_elems_[1]
                                             : -1;
  }

  int launch(int mode, int src, int dst, double a_old, double a_new, double b,
             Real* q_next, int with_source, int stage, int part, cudaStream_t st) {
    CU(cudaSetDevice(device_));
    const int32_t* groups = part == ESDG_B200_PART_ALL ? nullptr : groups_ + (part == ESDG_B200_PART_BOUNDARY ? n_groups_[0] : 0);
    const long long n_groups = part == ESDG_B200_PART_ALL ? range_count_ : n_groups_[part - 1];
    if (mode == kModeFused) {
      const int rc = open_epoch(part, pick(st));
      if (rc != ESDG_B200_OK) return rc;
    }
    if (part != ESDG_B200_PART_ALL && n_groups == 0) {
      if (mode == kModeFused) close_epoch(part);
      return ESDG_B200_OK;
    }
    cudaError_t e = cudaErrorInvalidValue;
    switch (nq_) {
#define ESDG_CASE(NQ)                                                          \
  case NQ:                                                                     \
    e = run_rhs<NQ>(mode, src, dst, a_old, a_new, b, q_next, with_source,      \
                    stage, groups, n_groups, pick(st));                        \
    break;
      ESDG_CASE(2) ESDG_CASE(3) ESDG_CASE(4) ESDG_CASE(5) ESDG_CASE(6)
      ESDG_CASE(7) ESDG_CASE(8)
#undef ESDG_CASE
    }
    if (e != cudaSuccess) {
      frec_parity_ = -1;
      epoch_state_ = kEpochClosed;
      return cuda_fail(e, "rhs_kernel");
    }
    if (mode == kModeFused) close_epoch(part);
    if (ne_ > 0) ++launches_;
    return ESDG_B200_OK;
  }

  // Tagged lift terms (esdg_kernels.cuh): the one-pass kernels of one RHS
  // evaluation -- a launch over all groups, the interior and the boundary
  // list, or the consecutive runs of stage_fused_range -- write every slot of
  // frec once, with the evaluation's parity in the lowest mantissa bit, and
  // read it expecting that parity. Between evaluations every slot therefore
  // holds the parity of the last one (frec_parity_), and the next evaluation
  // takes the other. Any call sequence that breaks the pattern (a boundary
  // launch without its interior launch, an abandoned series of runs, a failed
  // launch, a pull that timed out) leaves the parities mixed; the next
  // evaluation then starts from freshly initialised slots (all ones).
  enum { kEpochClosed = 0, kEpochInteriorDone = 1, kEpochRunsOpen = 2, kEpochSingle = 3, kEpochOrphan = 4 };
  int open_epoch(int part, cudaStream_t st) {
    const bool run = part == ESDG_B200_PART_ALL && range_count_ > 0;
    if ((part == ESDG_B200_PART_BOUNDARY && epoch_state_ == kEpochInteriorDone) ||
        (run && range_first_ > 0 && epoch_state_ == kEpochRunsOpen))
      return ESDG_B200_OK; // the evaluation at hand goes on
    if (epoch_state_ != kEpochClosed || frec_parity_ < 0) {
      CU(cudaMemsetAsync(frec_, 0xff, frec_bytes_, st));
      frec_parity_ = 1;
      ++frec_resets_;
    }
    epoch_ = unsigned(1 - frec_parity_);
    frec_parity_ = -1; // mixed while the evaluation is under way
    epoch_state_ = part == ESDG_B200_PART_INTERIOR   ? kEpochInteriorDone
                   : part == ESDG_B200_PART_BOUNDARY ? kEpochOrphan
                   : (run && range_first_ == 0)      ? kEpochRunsOpen
                   : run                             ? kEpochOrphan
                                                     : kEpochSingle;
    return ESDG_B200_OK;
  }
  void close_epoch(int part) {
    const int64_t total = (ne_ + epb_ - 1) / epb_;
    bool complete = false;
    switch (epoch_state_) {
      case kEpochSingle: complete = true; break;
      case kEpochInteriorDone:
        // the boundary list follows, unless it is empty
        complete = part == ESDG_B200_PART_BOUNDARY || n_groups_[1] == 0;
        if (!complete) return;
        break;
      case kEpochRunsOpen:
        complete = range_first_ + range_count_ >= total;
        if (!complete) return;
        break;
      default: break; // orphan: the slots stay mixed
    }
    frec_parity_ = complete ? int(epoch_) : -1;
    epoch_state_ = kEpochClosed;
  }

  int axpy(double b, cudaStream_t st) override {
    CU(cudaSetDevice(device_));
    const cudaError_t e = launch_axpy<Real>(
        q_, k_, Real(b), static_cast<long long>(ne_) * 5 * n3_, pick(st));
    if (e != cudaSuccess) return cuda_fail(e, "axpy_kernel");
    if (ne_ > 0) ++launches_;
    return ESDG_B200_OK;
  }

  int reduce(int kind, int reg, int var, const double* node_weight, const double* dx,
             double gamma, double* partials, int* nonphysical) override {
    if (kind < 0 || kind > 3 || (reg != 0 && reg != 1) || var < 0 || var > 4 ||
        !node_weight || !dx || !partials || !nonphysical)
      return bad("reduce: bad argument");
    *nonphysical = 0;
    if (ne_ == 0) return ESDG_B200_OK;
    CU(cudaSetDevice(device_));
    if (!red_out_) {
      CU(cudaMalloc(&red_out_, sizeof(double) * size_t(ne_)));
      CU(cudaMalloc(&red_tab_, sizeof(double) * size_t(n3_ + 3 * nq_)));
      CU(cudaMalloc(&red_bad_, sizeof(unsigned)));
    }
    CU(cudaMemcpyAsync(red_tab_, node_weight, sizeof(double) * size_t(n3_),
                       cudaMemcpyHostToDevice, stream_));
    CU(cudaMemcpyAsync(red_tab_ + n3_, dx, sizeof(double) * size_t(3 * nq_),
                       cudaMemcpyHostToDevice, stream_));
    CU(cudaMemsetAsync(red_bad_, 0, sizeof(unsigned), stream_));
    ReduceParams P;
    P.q = reg_ptr(kind == 0 ? reg : 0);
    P.k = k_;
    P.phi = phi_;
    P.node_weight = red_tab_;
    P.dx = red_tab_ + n3_;
    P.out = red_out_;
    P.bad = red_bad_;
    P.gamma = gamma;
    P.ne = ne_;
    P.nq = nq_;
    P.n3 = n3_;
    P.var = var;
    const unsigned blocks = unsigned((ne_ * 32 + 255) / 256);
    switch (kind) {
      case 0: reduce_kernel<Real, 0><<<blocks, 256, 0, stream_>>>(P); break;
      case 1: reduce_kernel<Real, 1><<<blocks, 256, 0, stream_>>>(P); break;
      case 2: reduce_kernel<Real, 2><<<blocks, 256, 0, stream_>>>(P); break;
      default: reduce_kernel<Real, 3><<<blocks, 256, 0, stream_>>>(P); break;
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "reduce_kernel");
    ++launches_;
    unsigned flag = 0;
    CU(cudaMemcpyAsync(partials, red_out_, sizeof(double) * size_t(ne_),
                       cudaMemcpyDeviceToHost, stream_));
    CU(cudaMemcpyAsync(&flag, red_bad_, sizeof(unsigned), cudaMemcpyDeviceToHost, stream_));
    CU(cudaStreamSynchronize(stream_));
    *nonphysical = flag ? 1 : 0;
    return ESDG_B200_OK;
  }

  int check(cudaStream_t st, int src, esdg_b200_error* err) override {
    CU(cudaSetDevice(device_));
    cudaStream_t s = pick(st);
    CU(cudaMemcpyAsync(flag_host_, flag_, 2 * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    const unsigned long long key = flag_host_[0];
    if (err) std::memset(err, 0, sizeof *err);
    if (flag_host_[1] != 0) {
      CU(cudaMemsetAsync(flag_ + 1, 0, sizeof(unsigned long long), s));
      CU(cudaStreamSynchronize(s));
      frec_parity_ = -1; // the slots are re-initialised before the next evaluation
      epoch_state_ = kEpochClosed;
      set_message("rhs_kernel: an element group waited in vain for the face contributions of an "
                  "earlier group (launch order violated?)");
      return ESDG_B200_CUDA;
    }
    if (key == kNoFlag) return ESDG_B200_OK;
    CU(cudaMemcpyAsync(flag_, &kNoFlag, sizeof kNoFlag, cudaMemcpyHostToDevice, s));
    CU(cudaStreamSynchronize(s));
    const int stage = int(key >> 56);
    const int phase = int((key >> 55) & 1ull);
    const int64_t elem = int64_t((key >> 10) & ((1ull << 45) - 1));
    const int node = int(key & 1023ull);
    if (err) {
      err->set = 1;
      err->element = elem;
      err->node = node;
      err->stage = stage;
      // payload captured at detection time (hashed side table)
      dev::FlagRecord rec[dev::kFlagSlots];
      CU(cudaMemcpy(rec, flag_records_, sizeof rec, cudaMemcpyDeviceToHost));
      const dev::FlagRecord& r = rec[key % dev::kFlagSlots];
      if (r.key == key) {
        err->rho = r.rho;
        err->pressure = r.p;
      } else if (phase == 0) {
        // slot overwritten by a colliding key: re-evaluate compute_node_vals'
        // checks (physics.hpp:56-74) on the flagged node of the source register
        const int64_t le = elem - elem_offset_;
        Real qv[5] = {0, 0, 0, 0, 0}, ph = 0;
        if (le >= 0 && le < ne_) {
          for (int v = 0; v < 5; ++v)
            CU(cudaMemcpy(&qv[v],
                          reg_ptr(src) + (size_t(le) * 5 + size_t(v)) * size_t(n3_) + node,
                          sizeof(Real), cudaMemcpyDeviceToHost));
          CU(cudaMemcpy(&ph, phi_ + size_t(le) * size_t(n3_) + node, sizeof(Real),
                        cudaMemcpyDeviceToHost));
        }
        err->rho = double(qv[0]);
        err->pressure = 0.0;
        if (qv[0] > Real(0)) {
          const Real inv = Real(1) / qv[0];
          const Real u0 = qv[1] * inv, u1 = qv[2] * inv, u2 = qv[3] * inv;
          const Real ke = Real(0.5) * (qv[1] * u0 + qv[2] * u1 + qv[3] * u2);
          err->pressure = double(gas_.gm1 * (qv[4] - ke - qv[0] * ph));
        }
      }
    }
    CU(cudaMemset(flag_records_, 0xff, sizeof(dev::FlagRecord) * dev::kFlagSlots));
    CU(cudaDeviceSynchronize()); // (legacy-stream fill: in place before the next kernel of the compute stream)
    return ESDG_B200_NONPHYSICAL;
  }

private:
  template <int NQ>
  cudaError_t run_rhs(int mode, int src, int dst, double a_old, double a_new,
                      double b, Real* q_next, int with_source, int stage,
                      const int32_t* groups, long long n_groups, cudaStream_t st) {
    dev::RhsParams<Real, NQ> P;
    P.groups = groups;
    P.group_base = groups ? 0 : int(range_first_);
    P.q = reg_ptr(src);
    P.q_next = q_next;
    P.b_upd = Real(b);
    P.out = reg_ptr(dst);
    P.phi = phi_;
    P.nbr = nbr_;
    P.ghost_q = recv_;
    P.ghost_phi = ghost_phi_;
    P.ylevel = ylevel_;
    P.cor_f = cor_f_;
    P.flag = flag_;
    P.flag_records = flag_records_;
    P.ne = ne_;
    P.elem_offset = elem_offset_;
    P.a_old = Real(a_old);
    P.a_new = Real(a_new);
    // slab arithmetic of rhs_kernel: T = out_old + gain * rhs, out = fin * T
    P.gain = P.a_old != Real(0) ? P.a_new / P.a_old : P.a_new;
    P.fin = P.a_old != Real(0) ? P.a_old : Real(1);
    if (!std::isfinite(double(P.gain))) {
      set_message("rhs: a_new / a_old is not finite (pass a_old = 0 to overwrite out)");
      return cudaErrorInvalidValue;
    }
    P.gas = gas_;
    for (int i = 0; i < NQ * NQ; ++i) P.negd[i] = negd_[size_t(i)];
    for (int k = 0; k < 3; ++k) {
      P.metric[k] = metric_[k];
      P.lift[k] = lift_[k];
    }
    P.with_source = (with_source && coriolis_mode_ != 0) ? 1 : 0;
    int epb_mode = epb_; // elements per CTA of THIS kernel (the split kernels may use another tile)
    {
      int threads = 0, epb = 0;
      size_t smem = 0;
      rhs_launch_shape<Real, NQ>(mode, &threads, &epb, &smem);
      epb_mode = epb;
      const int per_sm = std::max(1, std::min(int(smem_per_sm_ / std::max<size_t>(smem, 1)), 2048 / std::max(threads, 1)));
      P.prefetch_ctas = sm_count_ * per_sm;
    }
    P.dissipation = dissipation_;
    P.flat_phi = flat_phi_;
    P.stage = stage;
    // faces evaluated once and shared between the two elements (one-pass
    // kernels only): the role table fits the order the groups of this launch
    // are dispatched in
    const bool share = mode == kModeFused && share_faces_ && frec_ != nullptr;
    P.face_roles = share ? (groups ? roles_split_ : roles_all_) : nullptr;
    P.frec = frec_;
    P.epoch = epoch_;
    P.sync_error = flag_ + 1;
    P.ticket = (share && use_ticket_) ? ticket_ : nullptr;
    P.ticket_base = ticket_base_;
    if (P.ticket) ticket_base_ += unsigned((groups || n_groups > 0) ? n_groups : (ne_ + epb_mode - 1) / epb_mode);
    P.wait_limit_ns = wait_limit_ns_;
    if (mode == kModeVolume && variant_ < 4 && !groups && n_groups == 0) {
      // a rung of the reference's ladder below "symmetric" (kernels.hpp:20-34)
      const int rung = variant_ <= 1 ? dev::kRungRecompute
                                     : (variant_ == 2 ? dev::kRungPrecompute : dev::kRungLogMean);
      return launch_ladder<Real, NQ>(rung, P, st);
    }
    return launch_rhs<Real, NQ>(mode, P, n_groups, st);
  }

  // Element groups (the EPB consecutive elements one CTA of rhs_kernel owns)
  // sorted into "no ghost face" and "at least one ghost face": the one-pass
  // kernels run the first list while the traces travel and the second after
  // they have landed -- the reference's order volume -> wait -> ghost faces
  // (solver.hpp:259-294) at group granularity.
  int build_groups(const int32_t* nbr) {
    int threads = 0, epb = 1;
    size_t smem = 0;
    switch (nq_) {
#define ESDG_CASE(NQ) \
  case NQ: rhs_launch_shape<Real, NQ>(kModeFused, &threads, &epb, &smem); break;
      ESDG_CASE(2) ESDG_CASE(3) ESDG_CASE(4) ESDG_CASE(5) ESDG_CASE(6)
      ESDG_CASE(7) ESDG_CASE(8)
#undef ESDG_CASE
      default: return bad("unsupported nq");
    }
    epb_ = epb;
    const int64_t ng = (ne_ + epb - 1) / epb;
    std::vector<int32_t> interior, boundary;
    n_part_elems_[0] = n_part_elems_[1] = 0;
    for (int64_t g = 0; g < ng; ++g) {
      const int64_t lo = g * epb, hi = std::min<int64_t>(ne_, lo + epb);
      bool ghost = false;
      for (int64_t i = lo * 6; i < hi * 6 && !ghost; ++i) ghost = nbr[i] <= -2;
      (ghost ? boundary : interior).push_back(int32_t(g));
      n_part_elems_[ghost ? 1 : 0] += hi - lo;
    }
    n_groups_[0] = int64_t(interior.size());
    n_groups_[1] = int64_t(boundary.size());
    // face roles of the one-pass kernels (host/mesh.cpp)
    std::vector<uint8_t> roles[2];
    for (int t = 0; t < 2; ++t) {
      roles[t].assign(size_t(std::max<int64_t>(ne_, 1)), 0);
      host::build_face_roles(nbr, ne_, epb, t == 1, roles[t].data());
    }
    CU(alloc_copy(&roles_all_, roles[0].data(), size_t(ne_)));
    CU(alloc_copy(&roles_split_, roles[1].data(), size_t(ne_)));
    // blocks of the pushed lift terms, [3][element][5 n2 Reals padded to 16
    // bytes] (dev::FrecBlock), all ones = tagged with parity 1 (open_epoch); + 64: the
    // bulk copy of a group's blocks may be issued for the last, partial group
    const size_t frec_bytes =
        size_t(std::max<int64_t>(ne_, 1)) * 3 * ((sizeof(Real) * 5 * size_t(n2_) + 15) & ~size_t(15)) + 64;
    CU(cudaMalloc(&frec_, frec_bytes));
    CU(cudaMemset(frec_, 0xff, frec_bytes));
    frec_bytes_ = frec_bytes;
    frec_parity_ = 1; // all ones
    epoch_state_ = kEpochClosed;
    CU(cudaMalloc(&ticket_, sizeof(unsigned)));
    CU(cudaMemset(ticket_, 0, sizeof(unsigned)));
    if (const char* t = std::getenv("ESDG_B200_TICKET")) use_ticket_ = std::atoi(t);
    interior.insert(interior.end(), boundary.begin(), boundary.end());
    CU(alloc_copy(&groups_, interior.data(), sizeof(int32_t) * interior.size()));
    return ESDG_B200_OK;
  }

  static cudaError_t alloc_copy_impl(void** dst, const void* src, size_t bytes) {
    // 64 bytes of slack: the kernels' TMA bulk copies round their source
    // range outwards to multiples of 16 bytes
    cudaError_t e = cudaMalloc(dst, bytes + 64);
    if (e != cudaSuccess) return e;
    if (bytes && src) e = cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
    return e;
  }
  template <class T>
  static cudaError_t alloc_copy(T** dst, const void* src, size_t bytes) {
    return alloc_copy_impl(reinterpret_cast<void**>(dst), src, bytes);
  }

  Real* reg_ptr(int reg) { return reg == 0 ? q_ : k_; }
  cudaStream_t pick(cudaStream_t st) { return st ? st : stream_; }
  bool range_ok(int reg, int64_t first, int64_t count) const {
    return (reg == 0 || reg == 1) && first >= 0 && count >= 0 &&
           first + count <= ne_;
  }
  int bad(const char* m) {
    set_message(m);
    return ESDG_B200_BADARG;
  }

  void release() {
    if (device_ >= 0) cudaSetDevice(device_);
    cudaFree(q_);
    cudaFree(q_alt_);
    cudaFree(q_in_);
    cudaFree(q_out_);
    cudaFree(k_);
    cudaFree(phi_);
    cudaFree(nbr_);
    cudaFree(groups_);
    cudaFree(roles_all_);
    cudaFree(roles_split_);
    cudaFree(frec_);
    cudaFree(ticket_);
    cudaFree(ghost_phi_);
    cudaFree(send_elem_);
    cudaFree(send_face_);
    cudaFree(recv_);
    cudaFree(send_);
    cudaFree(ylevel_);
    cudaFree(cor_f_);
    cudaFree(flag_);
    cudaFree(red_out_);
    cudaFree(red_tab_);
    cudaFree(red_bad_);
    cudaFree(flag_records_);
    if (flag_host_) cudaFreeHost(flag_host_);
    if (stream_) cudaStreamDestroy(stream_);
  }

  int nq_ = 0, n2_ = 0, n3_ = 0, device_ = -1, sm_count_ = 148;
  size_t smem_per_sm_ = 233472;
  int64_t ne_ = 0, elem_offset_ = 0, n_ghost_ = 0, n_send_ = 0;
  int dissipation_ = 1, coriolis_mode_ = 0, flat_phi_ = 0;
  Real metric_[3] = {0, 0, 0}, lift_[3] = {0, 0, 0};
  std::vector<Real> negd_;
  dev::GasParams<Real> gas_{};
  Real *q_in_ = nullptr, *q_out_ = nullptr; // step_stream's landing and parking buffers
  Real *q_ = nullptr, *q_alt_ = nullptr, *k_ = nullptr, *phi_ = nullptr, *ghost_phi_ = nullptr;
  Real *recv_ = nullptr, *send_ = nullptr, *cor_f_ = nullptr;
  int32_t *nbr_ = nullptr, *send_elem_ = nullptr, *send_face_ = nullptr,
          *ylevel_ = nullptr, *groups_ = nullptr;
  int64_t n_groups_[2] = {0, 0}, n_part_elems_[2] = {0, 0};
  int64_t range_first_ = 0, range_count_ = 0; // stage_fused_range: groups of this launch
  int64_t range_next_ = 0;
  // shared face evaluation of the one-pass kernels (RhsParams::face_roles)
  uint8_t *roles_all_ = nullptr, *roles_split_ = nullptr;
  Real* frec_ = nullptr;
  size_t frec_bytes_ = 0;
  int frec_parity_ = 1;   // tag every slot of frec holds (0 / 1), -1: mixed
  unsigned epoch_ = 0;    // tag of the evaluation under way / last started
  int epoch_state_ = 0;   // kEpoch*
  int64_t frec_resets_ = 0;
  int share_faces_ = 1;
  unsigned* ticket_ = nullptr; // launch-order counter of the one-pass kernels
  unsigned ticket_base_ = 0;
  int use_ticket_ = 1;
  unsigned long long wait_limit_ns_ = 2000000000ull;
  int variant_ = 5; // KernelVariant::Balanced
  int epb_ = 1;
  unsigned long long *flag_ = nullptr, *flag_host_ = nullptr;
  double *red_out_ = nullptr, *red_tab_ = nullptr;
  unsigned* red_bad_ = nullptr;
  dev::FlagRecord* flag_records_ = nullptr;
  cudaStream_t stream_ = nullptr;
  int64_t launches_ = 0;
};

// ---- FMA peak micro-benchmark (roofline denominator of K1) ----------------

template <class Real>
__global__ void __launch_bounds__(256) fma_peak_kernel(Real* out, int iters) {
  Real a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = Real(threadIdx.x + i) * Real(1e-3);
  // m and c are the same in every thread, so the compiler keeps them in
  // uniform registers: each FMA reads ONE vector register. This is the pipe's
  // nominal rate (one warp instruction per two cycles per sub-partition).
  const Real m = Real(1) - Real(1e-6) * Real(1 + (iters & 1));
  const Real c = Real(1e-6) * Real(1 + (iters & 2));
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = dev::fma_(a[i], m, c);
    }
  }
  Real s = Real(0);
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == Real(123.456)) out[0] = s; // keeps the chain alive
}

// The same with three DISTINCT, thread-varying vector-register operands per
// FMA (x = fma(y, z, x)): on sm_100 such an FP64 instruction occupies the
// pipe for three cycles instead of two, so general FP64 code cannot reach
// the nominal figure (tools/ubench/fp64_operands_ubench.cu).
template <class Real>
__global__ void __launch_bounds__(256) fma3_peak_kernel(Real* out, const Real* in, int iters) {
  Real x[8], y[8], z[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    x[i] = in[(threadIdx.x + 7 * i) & 255];
    y[i] = Real(1) - Real(1e-6) * in[(threadIdx.x + 11 * i + 1) & 255];
    z[i] = Real(1e-6) * in[(threadIdx.x + 13 * i + 2) & 255];
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = dev::fma_(y[(i + r) & 7], z[(i + 3 * r + 1) & 7], x[i]);
    }
  }
  Real s = Real(0);
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == Real(123.456)) out[0] = s;
}

// Device self-test of the arithmetic identities the kernels rely on.
// out[0] = max error of rcp_ in ulps against the correctly rounded 1/x,
// out[1] = number of samples where rcp_(2x) != rcp_(x)/2,
// out[2] = 1 when rcp_(1) == 1 exactly, out[3] = samples tested,
// out[4] = max |log_ - CUDA log| in ulps over positive samples (FP64: the
// lean log_pos of esdg_log.cuh against the library routine).
template <class Real>
__global__ void selftest_kernel(double* out, int n) {
  __shared__ double s_err[256], s_log[256];
  __shared__ int s_bad[256];
  __shared__ __align__(16) Real s_tab[dev::LogTab<Real>::kReals + 1];
  dev::fill_log_table(s_tab, threadIdx.x, blockDim.x);
  __syncthreads();
  double worst = 0.0, worst_log = 0.0;
  int bad = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    // deterministic samples over ~12 decades, both signs
    unsigned long long z = 0x9e3779b97f4a7c15ull * (unsigned long long)(i + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    const double u = double(z >> 11) * (1.0 / 9007199254740992.0);
    const double mag = exp2(40.0 * u - 20.0) * (1.0 + u);
    const Real x = Real((i & 1) ? -mag : mag);
    const Real r = dev::rcp_(x);
    const Real exact = Real(1) / x; // IEEE division (-prec-div default)
    const Real ulp = sizeof(Real) == 8 ? Real(fabs(double(exact)) * 2.220446049250313e-16)
                                       : Real(fabsf(float(exact)) * 1.1920929e-7f);
    const double e = fabs(double(r) - double(exact)) / double(ulp);
    if (e > worst) worst = e;
    if (dev::rcp_(x + x) != Real(0.5) * r) ++bad;
    const Real ax = x < Real(0) ? -x : x;
    const double lref = sizeof(Real) == 8 ? log(double(ax)) : double(logf(float(ax)));
    const double lulp = fabs(lref) * (sizeof(Real) == 8 ? 2.220446049250313e-16 : 1.1920929e-7);
    const double le = fabs(double(dev::log_(ax, s_tab)) - lref) / (lulp > 0.0 ? lulp : 1.0);
    if (le > worst_log) worst_log = le;
  }
  s_err[threadIdx.x] = worst;
  s_log[threadIdx.x] = worst_log;
  s_bad[threadIdx.x] = bad;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int t = 1; t < blockDim.x; ++t) {
      if (s_err[t] > worst) worst = s_err[t];
      if (s_log[t] > worst_log) worst_log = s_log[t];
      bad += s_bad[t];
    }
    // one block: plain stores
    out[0] = worst;
    out[1] = double(bad);
    out[2] = dev::rcp_(Real(1)) == Real(1) ? 1.0 : 0.0;
    out[3] = double(n);
    out[4] = worst_log;
  }
}

template <class Real>
int run_selftest(int device, double* out5) {
  CU(cudaSetDevice(device));
  double* d = nullptr;
  CU(cudaMalloc(&d, 5 * sizeof(double)));
  selftest_kernel<Real><<<1, 256>>>(d, 1 << 20);
  CU(cudaGetLastError());
  CU(cudaMemcpy(out5, d, 5 * sizeof(double), cudaMemcpyDeviceToHost));
  cudaFree(d);
  return ESDG_B200_OK;
}

template <class Real>
int measure_peak(int device, int vector_operands, double* tflops) {
  CU(cudaSetDevice(device));
  cudaDeviceProp prop;
  CU(cudaGetDeviceProperties(&prop, device));
  Real* out = nullptr;
  CU(cudaMalloc(&out, sizeof(Real) * 257));
  {
    Real h[256];
    for (int i = 0; i < 256; ++i) h[i] = Real(1) + Real(i) * Real(1e-3);
    CU(cudaMemcpy(out + 1, h, sizeof h, cudaMemcpyHostToDevice));
  }
  const int blocks = prop.multiProcessorCount * 8, threads = 256, iters = 4096;
  cudaEvent_t t0, t1;
  CU(cudaEventCreate(&t0));
  CU(cudaEventCreate(&t1));
  double best = 0.0;
  for (int rep = 0; rep < 5; ++rep) {
    CU(cudaEventRecord(t0));
    if (vector_operands >= 3)
      fma3_peak_kernel<Real><<<blocks, threads>>>(out, out + 1, iters);
    else
      fma_peak_kernel<Real><<<blocks, threads>>>(out, iters);
    CU(cudaEventRecord(t1));
    CU(cudaEventSynchronize(t1));
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, t0, t1));
    const double flops = 2.0 * 64.0 * double(iters) * double(blocks) * threads;
    const double tf = flops / (double(ms) * 1e-3) / 1e12;
    if (rep > 0 && tf > best) best = tf;
  }
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  cudaFree(out);
  *tflops = best;
  return ESDG_B200_OK;
}

} // namespace

int create_shard(const esdg_b200_shard_desc& d, ShardBase** out) {
  if (d.nq < 2 || d.nq > 8 || d.n_elements < 0 || !d.diff || !d.weights ||
      (d.n_elements > 0 && (!d.nbr || !d.phi)) ||
      (d.n_ghost > 0 && !d.ghost_phi) ||
      (d.n_send > 0 && (!d.send_elem || !d.send_face))) {
    set_message("shard_create: bad descriptor");
    return ESDG_B200_BADARG;
  }
  if (d.n_elements >= (int64_t(1) << 31)) {
    set_message("shard_create: more than 2^31 elements in one partition");
    return ESDG_B200_BADARG;
  }
  int rc;
  if (d.precision == 8) {
    auto* s = new Shard<double>();
    rc = s->init(d);
    if (rc != ESDG_B200_OK) {
      delete s;
      return rc;
    }
    *out = s;
  } else if (d.precision == 4) {
    auto* s = new Shard<float>();
    rc = s->init(d);
    if (rc != ESDG_B200_OK) {
      delete s;
      return rc;
    }
    *out = s;
  } else {
    set_message("shard_create: precision must be 8 or 4");
    return ESDG_B200_BADARG;
  }
  return ESDG_B200_OK;
}

} // namespace esdg_b200

using esdg_b200::ShardBase;

struct esdg_b200_shard {
  ShardBase* impl;
  int last_src;
};

extern "C" {

int esdg_b200_abi_version(void) { return ESDG_B200_ABI_VERSION; }

const char* esdg_b200_last_message(void) {
  return esdg_b200::g_last_message.c_str();
}

int esdg_b200_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int esdg_b200_shard_create(const esdg_b200_shard_desc* desc,
                           esdg_b200_shard** out) {
  if (!desc || !out) return ESDG_B200_BADARG;
  ShardBase* impl = nullptr;
  const int rc = esdg_b200::create_shard(*desc, &impl);
  if (rc != ESDG_B200_OK) return rc;
  *out = new esdg_b200_shard{impl, 0};
  return ESDG_B200_OK;
}

void esdg_b200_shard_destroy(esdg_b200_shard* s) {
  if (!s) return;
  delete s->impl;
  delete s;
}

int esdg_b200_shard_upload(esdg_b200_shard* s, int reg, const void* host,
                           int64_t first, int64_t count) {
  return s ? s->impl->upload(reg, host, first, count, nullptr, false)
           : ESDG_B200_BADARG;
}
int esdg_b200_shard_download(esdg_b200_shard* s, int reg, void* host,
                             int64_t first, int64_t count) {
  return s ? s->impl->download(reg, host, first, count, nullptr, false)
           : ESDG_B200_BADARG;
}
int esdg_b200_shard_upload_async(esdg_b200_shard* s, int reg, const void* host,
                                 int64_t first, int64_t count, void* stream) {
  return s ? s->impl->upload(reg, host, first, count, cudaStream_t(stream), true)
           : ESDG_B200_BADARG;
}
int esdg_b200_shard_download_async(esdg_b200_shard* s, int reg, void* host,
                                   int64_t first, int64_t count, void* stream) {
  return s ? s->impl->download(reg, host, first, count, cudaStream_t(stream), true)
           : ESDG_B200_BADARG;
}
void* esdg_b200_shard_register_ptr(esdg_b200_shard* s, int reg) {
  return s ? s->impl->register_ptr(reg) : nullptr;
}
void* esdg_b200_shard_send_ptr(esdg_b200_shard* s) {
  return s ? s->impl->send_ptr() : nullptr;
}
void* esdg_b200_shard_recv_ptr(esdg_b200_shard* s) {
  return s ? s->impl->recv_ptr() : nullptr;
}
void* esdg_b200_shard_stream(esdg_b200_shard* s) {
  return s ? s->impl->stream() : nullptr;
}

int esdg_b200_shard_pack(esdg_b200_shard* s, int src, void* stream) {
  return s ? s->impl->pack(src, cudaStream_t(stream)) : ESDG_B200_BADARG;
}

int esdg_b200_shard_volume(esdg_b200_shard* s, int src, int dst, double a_old,
                           double a_new, int with_source, int stage,
                           void* stream) {
  if (!s) return ESDG_B200_BADARG;
  s->last_src = src;
  return s->impl->rhs(esdg_b200::kModeVolume, src, dst, a_old, a_new,
                      with_source, stage, ESDG_B200_PART_ALL, cudaStream_t(stream));
}

int esdg_b200_shard_surface(esdg_b200_shard* s, int src, int dst, double a_new,
                            int stage, void* stream) {
  if (!s) return ESDG_B200_BADARG;
  s->last_src = src;
  return s->impl->rhs(esdg_b200::kModeSurface, src, dst, 1.0, a_new, 0, stage,
                      ESDG_B200_PART_ALL, cudaStream_t(stream));
}

int esdg_b200_shard_rhs_fused(esdg_b200_shard* s, int src, int dst,
                              double a_old, double a_new, int stage,
                              void* stream) {
  if (!s) return ESDG_B200_BADARG;
  s->last_src = src;
  return s->impl->rhs(esdg_b200::kModeFused, src, dst, a_old, a_new, 1, stage,
                      ESDG_B200_PART_ALL, cudaStream_t(stream));
}

int esdg_b200_shard_rhs_fused_part(esdg_b200_shard* s, int src, int dst,
                                   double a_old, double a_new, int stage,
                                   int part, void* stream) {
  if (!s) return ESDG_B200_BADARG;
  s->last_src = src;
  return s->impl->rhs(esdg_b200::kModeFused, src, dst, a_old, a_new, 1, stage,
                      part, cudaStream_t(stream));
}

int esdg_b200_shard_stage_fused_part(esdg_b200_shard* s, double a_old,
                                     double a_new, double b, int stage,
                                     int part, void* stream) {
  if (!s) return ESDG_B200_BADARG;
  s->last_src = ESDG_B200_REG_Q;
  return s->impl->stage_fused(a_old, a_new, b, 1, stage, part, cudaStream_t(stream));
}

int esdg_b200_shard_part_elements(esdg_b200_shard* s, int part, int64_t* count) {
  if (!s || !count) return ESDG_B200_BADARG;
  *count = s->impl->part_elements(part);
  return *count < 0 ? ESDG_B200_BADARG : ESDG_B200_OK;
}

int esdg_b200_shard_stage_fused(esdg_b200_shard* s, double a_old, double a_new,
                                double b, int stage, void* stream) {
  if (!s) return ESDG_B200_BADARG;
  s->last_src = ESDG_B200_REG_Q;
  return s->impl->stage_fused(a_old, a_new, b, 1, stage, ESDG_B200_PART_ALL,
                              cudaStream_t(stream));
}

int esdg_b200_shard_axpy(esdg_b200_shard* s, double b, void* stream) {
  return s ? s->impl->axpy(b, cudaStream_t(stream)) : ESDG_B200_BADARG;
}

int esdg_b200_shard_check(esdg_b200_shard* s, void* stream,
                          esdg_b200_error* err) {
  return s ? s->impl->check(cudaStream_t(stream), s->last_src, err)
           : ESDG_B200_BADARG;
}

int esdg_b200_shard_reduce(esdg_b200_shard* s, int kind, int reg, int var,
                           const double* node_weight, const double* dx, double gamma,
                           double* partials, int32_t* nonphysical) {
  if (!s) return ESDG_B200_BADARG;
  int np = 0;
  const int rc = s->impl->reduce(kind, reg, var, node_weight, dx, gamma, partials, &np);
  if (nonphysical) *nonphysical = np;
  return rc;
}

int64_t esdg_b200_shard_launch_count(const esdg_b200_shard* s) {
  return s ? s->impl->launch_count() : 0;
}

int esdg_b200_selftest(int device, int precision, double out5[5]) {
  if (!out5) return ESDG_B200_BADARG;
  if (precision == 8) return esdg_b200::run_selftest<double>(device, out5);
  if (precision == 4) return esdg_b200::run_selftest<float>(device, out5);
  return ESDG_B200_BADARG;
}

int esdg_b200_measure_fma_peak(int device, int precision, double* tflops) {
  if (!tflops) return ESDG_B200_BADARG;
  if (precision == 8) return esdg_b200::measure_peak<double>(device, 1, tflops);
  if (precision == 4) return esdg_b200::measure_peak<float>(device, 1, tflops);
  return ESDG_B200_BADARG;
}

int esdg_b200_measure_fma3_peak(int device, int precision, double* tflops) {
  if (!tflops) return ESDG_B200_BADARG;
  if (precision == 8) return esdg_b200::measure_peak<double>(device, 3, tflops);
  if (precision == 4) return esdg_b200::measure_peak<float>(device, 3, tflops);
  return ESDG_B200_BADARG;
}

} // extern "C"
