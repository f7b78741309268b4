// nccl_transport.hpp -- the process-per-GPU face-trace exchange in C++: one
// ncclSend / ncclRecv pair per peer inside one ncclGroup per RHS, issued on
// the partition's copy stream (replaces the reference's Transport<Real>::send
// / wait, core/include/esdg/exchange.hpp:32-57, call sites solver.hpp:255,294).
// No Python runs inside a step.
//
// NCCL is bound at run time (dlopen of libnccl.so.2, the copy torch already
// mapped when the host is a torchrun rank, the system's otherwise): the
// product library carries no link-time dependency on it and single-GPU users
// never load it.
#pragma once

#include <cstddef>
#include <string>

#include <cuda_runtime.h>

namespace esdg_b200 {
namespace host {

constexpr int kNcclUniqueIdBytes = 128; // NCCL_UNIQUE_ID_BYTES (nccl.h:37)

class NcclTransport {
public:
  // fills id[128] (rank 0 calls this; the host distributes it to all ranks)
  static bool unique_id(void* id128, std::string* err);

  NcclTransport() = default;
  ~NcclTransport();
  NcclTransport(const NcclTransport&) = delete;
  NcclTransport& operator=(const NcclTransport&) = delete;

  // ncclCommInitRank on the current device; collective over all ranks
  bool init(int world_size, int rank, const void* id128, std::string* err);
  bool ready() const { return comm_ != nullptr; }
  int version() const { return version_; }

  // one group: receive `count[p]` values into recv + offset[p] from peer[p]
  // and send the same range of `send` to it, for all peers, on `stream`
  bool exchange(const void* send, void* recv, const long long* offset, const long long* count,
                const int* peer, int n_peers, int real_bytes, cudaStream_t stream,
                std::string* err);

private:
  void* comm_ = nullptr; // ncclComm_t
  int version_ = 0;
};

} // namespace host
} // namespace esdg_b200
