// nccl_transport.cpp -- see nccl_transport.hpp.
#include "nccl_transport.hpp"

#include <dlfcn.h>

#include <cstring>
#include <mutex>

namespace esdg_b200 {
namespace host {

namespace {

// The few NCCL entry points the exchange needs, with the types of nccl.h
// restated (ncclResult_t is an int enum with ncclSuccess = 0; ncclDataType_t
// numbers ncclFloat32 = 7, ncclFloat64 = 8, nccl.h:285-286; ncclUniqueId is
// 128 opaque bytes passed by value).
struct UniqueId {
  char internal[kNcclUniqueIdBytes];
};
using Comm = void*;
struct Api {
  int (*GetVersion)(int*) = nullptr;
  int (*GetUniqueId)(UniqueId*) = nullptr;
  int (*CommInitRank)(Comm*, int, UniqueId, int) = nullptr;
  int (*CommDestroy)(Comm) = nullptr;
  int (*Send)(const void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  bool ok = false;
  std::string why;
};

Api& api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    // RTLD_NOLOAD first: the copy the host process already mapped (torch's)
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      h = dlopen(name, RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h)
      for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
        h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
        if (h) break;
      }
    if (!h) {
      a.why = std::string("cannot load libnccl.so.2: ") + (dlerror() ? dlerror() : "?");
      return;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    a.GetVersion = reinterpret_cast<decltype(a.GetVersion)>(sym("ncclGetVersion"));
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    a.ok = a.GetVersion && a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.Send && a.Recv &&
           a.GroupStart && a.GroupEnd && a.GetErrorString;
    if (!a.ok) a.why = "libnccl.so.2 lacks an entry point the exchange needs";
  });
  return a;
}

bool fail(std::string* err, const std::string& m) {
  if (err) *err = m;
  return false;
}
bool nccl_ok(int rc, const char* what, std::string* err) {
  if (rc == 0) return true;
  return fail(err, std::string(what) + ": " + api().GetErrorString(rc));
}

} // namespace

bool NcclTransport::unique_id(void* id128, std::string* err) {
  Api& a = api();
  if (!a.ok) return fail(err, a.why);
  UniqueId id;
  if (!nccl_ok(a.GetUniqueId(&id), "ncclGetUniqueId", err)) return false;
  std::memcpy(id128, id.internal, kNcclUniqueIdBytes);
  return true;
}

NcclTransport::~NcclTransport() {
  if (comm_) api().CommDestroy(comm_);
}

bool NcclTransport::init(int world_size, int rank, const void* id128, std::string* err) {
  Api& a = api();
  if (!a.ok) return fail(err, a.why);
  if (!id128 || world_size < 1 || rank < 0 || rank >= world_size)
    return fail(err, "NcclTransport::init: bad arguments");
  a.GetVersion(&version_);
  UniqueId id;
  std::memcpy(id.internal, id128, kNcclUniqueIdBytes);
  return nccl_ok(a.CommInitRank(&comm_, world_size, id, rank), "ncclCommInitRank", err);
}

bool NcclTransport::exchange(const void* send, void* recv, const long long* offset,
                             const long long* count, const int* peer, int n_peers,
                             int real_bytes, cudaStream_t stream, std::string* err) {
  Api& a = api();
  if (!comm_) return fail(err, "NcclTransport::exchange before init");
  const int dtype = real_bytes == 8 ? 8 /* ncclFloat64 */ : 7 /* ncclFloat32 */;
  if (!nccl_ok(a.GroupStart(), "ncclGroupStart", err)) return false;
  bool ok = true;
  for (int p = 0; p < n_peers && ok; ++p) {
    const size_t off = size_t(offset[p]) * size_t(real_bytes);
    ok = nccl_ok(a.Recv(static_cast<char*>(recv) + off, size_t(count[p]), dtype, peer[p], comm_, stream),
                 "ncclRecv", err) &&
         nccl_ok(a.Send(static_cast<const char*>(send) + off, size_t(count[p]), dtype, peer[p], comm_, stream),
                 "ncclSend", err);
  }
  // the group is closed even after a failure so that NCCL's state stays sane
  const bool closed = nccl_ok(a.GroupEnd(), "ncclGroupEnd", ok ? err : nullptr);
  return ok && closed;
}

} // namespace host
} // namespace esdg_b200
