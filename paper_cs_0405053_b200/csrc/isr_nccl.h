// isr_nccl.h -- the strip exchange of the relaxation loop over NCCL, issued by
// the library on its own stream (C1 = neighbour send/recv of
// the strip-edge boundary histories, C2 = all-reduce(max) of the iteration's
// {changed, overflow} flags; "UNTIL all PEs detect no difference",
// P:584-591 the neighbours' single layer of boundary atoms, P:804-811 the
// message cost "a constant times x + log N").
//
// NCCL is loaded at run time (dlopen) so that the library uses the same
// libnccl.so.2 as the process's torch.distributed when it is already loaded
// (RTLD_NOLOAD first), else the venv's nvidia-nccl wheel, else the system
// copy.  Only the handful of entry points below are used; their ABI (an
// opaque communicator, a 128-byte unique id, int enums) is stable across
// NCCL 2.x.
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

namespace isr_nccl {

typedef struct ncclComm* Comm;
typedef int Result;  // ncclSuccess = 0
struct UniqueId {
  char internal[128];
};
enum : int { kInt8 = 0, kInt32 = 2 };  // ncclDataType_t
enum : int { kMax = 2 };              // ncclRedOp_t

struct Api {
  void* handle = nullptr;
  Result (*GetUniqueId)(UniqueId*) = nullptr;
  Result (*CommInitRank)(Comm*, int, UniqueId, int) = nullptr;
  Result (*CommDestroy)(Comm) = nullptr;
  Result (*GroupStart)() = nullptr;
  Result (*GroupEnd)() = nullptr;
  Result (*Send)(const void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  Result (*Recv)(void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  Result (*AllReduce)(const void*, void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(Result) = nullptr;
  // NCCL >= 2.28 symmetric memory and device API (isr_peer.cuh); null if absent
  void* MemAlloc = nullptr;             // ncclMemAlloc(void**, size_t)
  void* MemFree = nullptr;              // ncclMemFree(void*)
  void* CommWindowRegister = nullptr;   // ncclCommWindowRegister(comm, buf, size, ncclWindow_t*, flags)
  void* CommWindowDeregister = nullptr; // ncclCommWindowDeregister(comm, ncclWindow_t)
  void* DevCommCreate = nullptr;        // ncclDevCommCreate(comm, const ncclDevCommRequirements*, ncclDevComm*)
  void* DevCommDestroy = nullptr;       // ncclDevCommDestroy(comm, const ncclDevComm*)
  void* TeamLsa = nullptr;              // ncclTeam ncclTeamLsa(comm)
  bool ok = false;
};

inline void* try_open(const char* path, int extra) { return dlopen(path, RTLD_NOW | RTLD_GLOBAL | extra); }

// the first libnccl.so.2 that loads: already in the process, $ISING_SR_NCCL,
// the venv's nvidia/nccl/lib (found relative to python's site-packages via
// $VIRTUAL_ENV or the usual image path), then the dynamic linker's search
inline const Api& api() {
  static Api A = [] {
    Api a;
    void* h = try_open("libnccl.so.2", RTLD_NOLOAD);
    if (!h) {
      if (const char* e = std::getenv("ISING_SR_NCCL")) h = try_open(e, 0);
    }
    if (!h) {
      std::string cands[] = {
          std::string(std::getenv("VIRTUAL_ENV") ? std::getenv("VIRTUAL_ENV") : "") +
              "/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2",
          "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2", "libnccl.so.2"};
      for (const auto& p : cands)
        if (!h) h = try_open(p.c_str(), 0);
    }
    if (!h) return a;
    a.handle = h;
    auto sym = [&](const char* n) { return dlsym(h, n); };
    a.GetUniqueId = (Result(*)(UniqueId*))sym("ncclGetUniqueId");
    a.CommInitRank = (Result(*)(Comm*, int, UniqueId, int))sym("ncclCommInitRank");
    a.CommDestroy = (Result(*)(Comm))sym("ncclCommDestroy");
    a.GroupStart = (Result(*)())sym("ncclGroupStart");
    a.GroupEnd = (Result(*)())sym("ncclGroupEnd");
    a.Send = (Result(*)(const void*, size_t, int, int, Comm, cudaStream_t))sym("ncclSend");
    a.Recv = (Result(*)(void*, size_t, int, int, Comm, cudaStream_t))sym("ncclRecv");
    a.AllReduce = (Result(*)(const void*, void*, size_t, int, int, Comm, cudaStream_t))sym("ncclAllReduce");
    a.GetErrorString = (const char* (*)(Result))sym("ncclGetErrorString");
    a.MemAlloc = sym("ncclMemAlloc");
    a.MemFree = sym("ncclMemFree");
    a.CommWindowRegister = sym("ncclCommWindowRegister");
    a.CommWindowDeregister = sym("ncclCommWindowDeregister");
    a.DevCommCreate = sym("ncclDevCommCreate");
    a.DevCommDestroy = sym("ncclDevCommDestroy");
    a.TeamLsa = sym("ncclTeamLsa");
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.GroupStart && a.GroupEnd && a.Send && a.Recv &&
           a.AllReduce;
    return a;
  }();
  return A;
}

inline bool report(Result r, const char* where) {
  if (r == 0) return true;
  const Api& a = api();
  std::fprintf(stderr, "ising_sr: NCCL error at %s: %s\n", where,
               a.GetErrorString ? a.GetErrorString(r) : "(unknown)");
  return false;
}

}  // namespace isr_nccl
