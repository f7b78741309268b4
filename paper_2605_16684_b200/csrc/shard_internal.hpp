// shard_internal.hpp -- precision-erased interface of one device partition,
// shared by shard.cu (implementation) and gpu_solver.cpp (host driver).
#pragma once

#include <cstdint>
#include <string>

#include <cuda_runtime.h>

#include "esdg_b200.h"

namespace esdg_b200 {

class ShardBase {
public:
  virtual ~ShardBase() = default;
  virtual int upload(int reg, const void* host, int64_t first, int64_t count,
                     cudaStream_t st, bool async) = 0;
  virtual int download(int reg, void* host, int64_t first, int64_t count,
                       cudaStream_t st, bool async) = 0;
  virtual void* register_ptr(int reg) = 0;
  virtual void* send_ptr() = 0;
  virtual void* recv_ptr() = 0;
  virtual cudaStream_t stream() = 0;
  virtual int device() const = 0;
  virtual int64_t n_elements() const = 0;
  virtual int64_t n_ghost() const = 0;
  virtual int64_t n_send() const = 0;
  virtual size_t trace_bytes() const = 0;
  virtual int64_t launch_count() const = 0;
  virtual void set_dissipation(int on) = 0;
  virtual void set_face_sharing(int on) = 0;
  // KernelVariant 0..5 (kernels.hpp:27-34): rungs below 4 run a ladder instance
  // of the volume kernel
  virtual void set_variant(int variant) = 0;
  virtual int pack(int src, cudaStream_t st) = 0;
  // mode: RhsMode (esdg_launch.hpp); part: ESDG_B200_PART_* -- all elements,
  // or only the element groups without / with a ghost face
  virtual int rhs(int mode, int src, int dst, double a_old, double a_new,
                  int with_source, int stage, int part, cudaStream_t st) = 0;
  // k <- a_old k + a_new RHS(q); q <- q + b k in one kernel (q double buffered;
  // the buffers swap after PART_ALL or PART_BOUNDARY)
  virtual int stage_fused(double a_old, double a_new, double b, int with_source,
                          int stage, int part, cudaStream_t st) = 0;
  virtual int64_t part_elements(int part) const = 0;
  // the same stage on the run of element groups [first_group, first_group +
  // n_groups) only (a group = elements_per_group() consecutive elements);
  // the q buffers swap when `last` is set. Lets a driver start moving
  // finished elements while the rest of the stage is still running.
  virtual int stage_fused_range(double a_old, double a_new, double b, int with_source,
                                int stage, int64_t first_group, int64_t n_groups, bool last,
                                cudaStream_t st) = 0;
  virtual int elements_per_group() const = 0;
  // Streaming of independent states (SolverCore::step_stream): two more state
  // buffers beside the q pair -- `in` receives the next state while a step
  // runs, `out` holds the previous step's result while it leaves.
  // stream_rotate(): out <- q (the result), q <- in, in <- the old out.
  virtual int stream_buffers(void** in, void** out) = 0;
  virtual void stream_rotate() = 0;
  virtual int axpy(double b, cudaStream_t st) = 0;
  virtual int check(cudaStream_t st, int src, esdg_b200_error* err) = 0;
  // K6: one partial per element, see esdg_b200_shard_reduce
  virtual int reduce(int kind, int reg, int var, const double* node_weight, const double* dx,
                     double gamma, double* partials, int* nonphysical) = 0;
};

int create_shard(const esdg_b200_shard_desc& d, ShardBase** out);
void set_message(const std::string& m);
int cuda_fail(cudaError_t e, const char* what);

} // namespace esdg_b200
