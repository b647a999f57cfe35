// Probe: does the NCCL 2.28 device API (symmetric window, LSA pointers, LSA
// barrier) work on this box with a one-rank communicator (the loopback
// configuration the library's tests use on one GPU)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I$NCCL/include \
//        nccl_dev_probe.cu -L$NCCL/lib -l:libnccl.so.2 -o probe
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#define CK(x) do { auto r_ = (x); if (r_ != 0) { printf("FAIL %s -> %d (%s)\n", #x, (int)r_, ncclGetErrorString((ncclResult_t)r_)); return 1; } } while (0)
#define CKC(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("FAIL %s -> %s\n", #x, cudaGetErrorString(r_)); return 1; } } while (0)

__global__ void k(ncclDevComm dc, ncclWindow_t win, int peer, int it) {
  ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamLsa(dc), dc.lsaBarrier, 0);
  int* p = (int*)ncclGetLsaPointer(win, 0, peer);
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) p[i] = i * 7 + it;
  bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
  int* q = (int*)ncclGetLocalPointer(win, 0);
  if (threadIdx.x == 0) printf("it %d: local[5] = %d (expect %d), lsaRank %d lsaSize %d\n", it, q[5], 35 + it, dc.lsaRank, dc.lsaSize);
}

int main() {
  CKC(cudaSetDevice(0));
  ncclUniqueId id;
  CK(ncclGetUniqueId(&id));
  ncclComm_t comm;
  CK(ncclCommInitRank(&comm, 1, id, 0));
  void* buf = nullptr;
  CK(ncclMemAlloc(&buf, 1 << 21));
  ncclWindow_t win;
  CK(ncclCommWindowRegister(comm, buf, 1 << 21, &win, NCCL_WIN_COLL_SYMMETRIC));
  ncclDevCommRequirements reqs = {};
  reqs.lsaBarrierCount = 1;
  ncclDevComm dc;
  CK(ncclDevCommCreate(comm, &reqs, &dc));
  for (int it = 0; it < 3; ++it) k<<<1, 128>>>(dc, win, 0, it);
  CKC(cudaDeviceSynchronize());
  // a captured launch (the graph window loop)
  cudaStream_t s;
  CKC(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CKC(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  k<<<1, 128, 0, s>>>(dc, win, 0, 10);
  CKC(cudaStreamEndCapture(s, &g));
  CKC(cudaGraphInstantiate(&ge, g, 0));
  CKC(cudaGraphLaunch(ge, s));
  CKC(cudaStreamSynchronize(s));
  CK(ncclDevCommDestroy(comm, &dc));
  CK(ncclCommWindowDeregister(comm, win));
  CK(ncclMemFree(buf));
  CK(ncclCommDestroy(comm));
  printf("PROBE OK\n");
  return 0;
}
