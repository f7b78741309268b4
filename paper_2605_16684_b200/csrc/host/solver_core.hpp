// solver_core.hpp -- host driver behind the level-2 C ABI: the GPU
// counterpart of esdg::Solver<Real> (core/include/esdg/solver.hpp:26-158).
// Owns one shard per locally held partition and runs the reference's RHS
// phase order on CUDA streams:
//   post ghost traces -> volume (overlaps the exchange) -> faces -> update
// (rhs_job, solver.hpp:240-340).
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "esdg_b200.h"
#include "host_types.hpp"
#include "../shard_internal.hpp"
#include "nccl_transport.hpp"

namespace esdg_b200 {
namespace host {

class SolverCore {
public:
  struct Options {
    int order = 4;
    int precision = 8;
    esdg_b200_gas gas{};
    esdg_b200_settings settings{};
    int world_size = 1;          // number of partitions of the mesh
    std::vector<int> local_ranks; // partitions held by this process
    std::vector<int> devices;     // device of each local partition
    esdg_b200_exchange_fn exchange = nullptr; // set => peers are remote
    void* exchange_user = nullptr;
    // set => peers are remote and reached by ncclSend/ncclRecv (one rank per
    // process, communicator built from this unique id)
    bool nccl = false;
    unsigned char nccl_id[kNcclUniqueIdBytes] = {};
  };

  static int create(Mesh* mesh, const Options& opt, SolverCore** out);
  ~SolverCore();

  int n3() const { return n3_; }
  int nq() const { return nq_; }
  int precision() const { return opt_.precision; }
  int64_t local_begin() const { return local_begin_; }
  int64_t local_end() const { return local_end_; }
  int64_t local_elements() const { return local_end_ - local_begin_; }
  const RefElement& ref() const { return ref_; }
  const Mesh& mesh() const { return *mesh_; }

  int set_path(int path);
  // KernelVariant (kernels.hpp:27-34): the ladder rung of the volume kernel
  int set_variant(int variant);
  int variant() const { return variant_; }
  // RankEvents (exchange.hpp:83-89): CUDA-event timeline of the next RHS
  // evaluations of every local partition
  int record_events(bool on);
  int rank_events(int rank, int64_t ns[5]);
  int64_t halo_bytes_per_rhs() const;
  // test hook, the analogue of Transport::send_hook (exchange.hpp:30): every
  // partition's trace transfer is held back by `us` microseconds
  void set_exchange_delay(int us) { exchange_delay_us_ = us < 0 ? 0 : us; }
  int nccl_version() const { return nccl_.version(); }
  int step_swap(double dt, const void* host_in, void* host_out, bool do_check);
  int step_stream(double dt, const void* host_in_next, void* host_out_prev, bool do_check);
  int stream_collect(void* host_out);
  void set_overlap(bool on) { overlap_ = on; }
  void set_face_sharing(bool on) {
    for (auto& ls : shards_) ls.dev->set_face_sharing(on ? 1 : 0);
  }
  void overlap_elements(int64_t* interior, int64_t* total);
  int set_settings(const esdg_b200_settings& s);
  int halo(int32_t* peer, int64_t* offset, int64_t* count, int capacity) const;
  ShardBase* shard(size_t i) { return shards_[i].dev.get(); }
  size_t n_shards() const { return shards_.size(); }

  int init_case(int case_id, uint64_t iparam, const double* dparam);
  int set_state(int reg, const void* host);
  int get_state(int reg, void* host);
  int swap_state(int reg, const void* host_in, void* host_out);
  int get_phi(void* host) const;

  int assemble_rhs_host(const void* q, void* out, double a_old, double a_new,
                        bool volume_only);
  int rhs(int src, int dst, double a_old, double a_new, bool with_source,
          bool volume_only, int stage);
  int stage_fused(double a_old, double a_new, double b, int stage);
  int axpy(double b);
  int step(double dt, bool check);
  int sync();
  int check();
  int compute_dt(double courant, double* dt);
  const esdg_b200_error& last_error() const { return err_; }

  int quadrature_total(int reg, int var, double* out);
  int total_entropy(double* out);
  int entropy_production(double* out);
  // ESDG_B200_REDUCE_ON_DEVICE (default) or ESDG_B200_REDUCE_ON_HOST
  int set_reduction(int mode);

  int enable_timing(bool on);
  int timers(double seconds[4], int64_t* launches, bool reset);

private:
  struct LocalShard {
    int rank = 0;
    int64_t begin = 0, end = 0;
    RankHalo halo;
    std::unique_ptr<ShardBase> dev;
    cudaStream_t comm = nullptr, down = nullptr, up = nullptr; // copy streams (down: D2H of step_swap / step_stream, up: step_stream's H2D)
    cudaEvent_t ev_pack = nullptr, ev_recv = nullptr, ev_surf = nullptr;
    // timeline of the last recorded RHS (timing enabled): start, traces
    // packed and posted, first kernel start / end, last trace arrived,
    // compute stream past its wait
    cudaEvent_t tl[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    bool tl_valid = false;
  };
  struct TimedLaunch {
    cudaEvent_t a, b;
    int cls;
    int device;
  };

  SolverCore() = default;
  int build_shard(LocalShard& ls);
  int local_index_of_rank(int rank) const;
  int exchange_begin(int src);
  int exchange_end();
  template <class F>
  int timed(LocalShard& ls, int cls, F&& launch);
  int collect_timers();
  // downloads register `reg` chunk by chunk and calls f(global_elem, ptr)
  template <class F>
  int for_each_element_chunk(int reg, int reg2, F&& f);
  // K6 on every local shard: one partial per local element, Morton order
  int device_partials(int kind, int reg, int var, std::vector<double>& partials, bool& bad);
  int compute_dt_host(double courant, double* dt);
  int quadrature_total_host(int reg, int var, double* out);
  int total_entropy_host(double* out);
  int entropy_production_host(double* out);

  Mesh* mesh_ = nullptr;
  Options opt_;
  RefElement ref_;
  int nq_ = 0, n2_ = 0, n3_ = 0;
  std::vector<int64_t> range_begin_;
  int64_t local_begin_ = 0, local_end_ = 0;
  std::vector<LocalShard> shards_;
  int path_ = ESDG_B200_PATH_STAGE; // the fastest; SPLIT keeps the reference's kernel structure
  int reduction_ = ESDG_B200_REDUCE_ON_DEVICE;
  bool any_halo_ = false;
  bool parked_ = false; // step_stream: a result waits in the shards' `out` buffers
  bool remote_peers() const { return opt_.exchange != nullptr || opt_.nccl; }
  int mark(LocalShard& ls, int which, cudaStream_t st);
  NcclTransport nccl_;
  int variant_ = 5; // balanced
  bool record_events_ = false;
  int exchange_delay_us_ = 0;
  int delay(LocalShard& ls);
  bool overlap_ = true; // one-pass paths: interior groups hide the exchange
  esdg_b200_error err_{};
  bool timing_ = false;
  std::vector<TimedLaunch> pending_;
  std::map<int, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>> event_pool_; // per device
  double seconds_[4] = {0, 0, 0, 0};
};

} // namespace host
} // namespace esdg_b200
