// isr_peer.cuh -- the strip exchange fused into one kernel over NVLink peer
// memory (SURVEY §8(e) mitigation 3; P:584-591 the neighbours' single layer
// of boundary atoms, "UNTIL all PEs detect no difference").
//
// With the library's NCCL communicator, the receive ghost rows and a small
// flag inbox of every rank live in one NCCL symmetric window (ncclMemAlloc +
// ncclCommWindowRegister), so each rank can store into its neighbours' ghost
// rows directly (ncclGetLsaPointer: load/store-accessible peer memory over
// NVLink / NVSwitch).  One kernel per iteration then replaces pack ->
// ncclSend/ncclRecv -> ncclAllReduce(max) -> mark:
//   block b, thread column c:  my first row's north-edge history -> rank up's
//     "from below" ghost row, my last row's south-edge history -> rank down's
//     "from above" ghost row (column c, written straight into peer memory);
//   block 0, thread q < world:  my {changed, overflow} -> rank q's inbox slot;
//   LSA barrier b (one per block; block b of every rank writes and reads the
//     same columns, so a block waits only for its counterparts);
//   column c of my two ghost rows (written by the neighbours' block b):
//     regions next to a ghost that changed in this iteration are marked dirty;
//   block 0: the max over the inbox = the all-reduced flags, in place.
// Ghost rows are double-buffered by the parity of the iteration stamp: a rank
// can only write parity K & 1 again (at stamp K + 2) after passing barrier
// K + 1, i.e. after every neighbour finished iteration K + 1's K1, which is
// the last reader of the rows written at K.  No host call, no NCCL kernel:
// the launch can also be captured in a CUDA graph.
//
// One GPU: FLAG_HALO_LOOPBACK with a one-rank communicator runs exactly this
// path (the strip's neighbours are itself), which is how it is tested.
#pragma once
#if __has_include(<nccl_device.h>)
#include <nccl.h>
#include <nccl_device.h>
#define ISR_HAVE_NCCL_DEVICE 1
#else
#define ISR_HAVE_NCCL_DEVICE 0
#endif

#include "isr_big.cuh"

namespace isr {

constexpr int kPeerMaxWorld = 64;  // inbox slots per parity
constexpr int kPeerThreads = 128;  // columns per block (one LSA barrier per block)

struct PeerArgs {
  const unsigned long long* peer;  // [world] base address of every rank's window (LSA pointers)
  char* mine;                      // my window (local pointer)
  int rank, world;
  unsigned long long row;          // bytes of one ghost row (4 chunks, 256-byte aligned)
  unsigned long long o_stamp, o_t, o_pos;  // chunk offsets inside a row (cnt at 0)
  unsigned long long o_inbox;      // flag inbox: int [2 parities][kPeerMaxWorld][2]
  int* flags;                      // this iteration's {changed, overflow}: read, then all-reduced in place
};

// ghost row (parity par, dir 0 = from the rank above, 1 = from the rank below) at window base b
__host__ __device__ __forceinline__ GhostView peer_row(const PeerArgs& p, char* b, int par, int dir) {
  char* r = b + (size_t)(2 * par + dir) * p.row;
  GhostView g;
  g.cnt = (uint16_t*)r;
  g.stamp = (uint32_t*)(r + p.o_stamp);
  g.t = (double*)(r + p.o_t);
  g.pos = (uint8_t*)(r + p.o_pos);
  return g;
}

#if ISR_HAVE_NCCL_DEVICE
// W: the per-edge selector layout of the warp / big-region forms
template <bool W>
__global__ void __launch_bounds__(kPeerThreads) xchg_kernel(const KArgs a, const PeerArgs p, ncclDevComm dc) {
  const unsigned K = stamp_of(a);
  const int par = (int)(K & 1u);
  const int c = blockIdx.x * kPeerThreads + threadIdx.x;
  const int up = (p.rank + p.world - 1) % p.world, down = (p.rank + 1) % p.world;
  if (c < a.RX) {
    const GhostView to_up = peer_row(p, (char*)p.peer[up], par, 1);      // I am below rank up
    const GhostView to_down = peer_row(p, (char*)p.peer[down], par, 0);  // I am above rank down
    if (W) {
      pack_col_w(a, true, c, to_up);
      pack_col_w(a, false, c, to_down);
    } else {
      pack_col(a, true, c, to_up);
      pack_col(a, false, c, to_down);
    }
  }
  if (blockIdx.x == 0 && (int)threadIdx.x < p.world) {
    int* box = (int*)((char*)p.peer[threadIdx.x] + p.o_inbox) + 2 * (par * kPeerMaxWorld + p.rank);
    box[0] = p.flags[0];
    box[1] = p.flags[1];
  }
  {
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamLsa(dc), dc.lsaBarrier, blockIdx.x);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
  }
  if (c < a.RX) {  // mark_kernel's rule on my two rows (this block's columns)
    const GhostView gu = peer_row(p, p.mine, par, 0), gd = peer_row(p, p.mine, par, 1);
    if (__ldcv(gu.stamp + c) == K) mark_dirty(a, c, K + 1);
    if (__ldcv(gd.stamp + c) == K) mark_dirty(a, (a.RYl - 1) * a.RX + c, K + 1);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const int* box = (const int*)(p.mine + p.o_inbox) + 2 * (par * kPeerMaxWorld);
    int m0 = 0, m1 = 0;
    for (int q = 0; q < p.world; ++q) {
      m0 = max(m0, __ldcv(box + 2 * q));
      m1 = max(m1, __ldcv(box + 2 * q + 1));
    }
    p.flags[0] = m0;
    p.flags[1] = m1;
  }
}

// every rank's window base as seen from this rank (once per window registration)
__global__ void peer_bases_kernel(ncclWindow_t win, int world, unsigned long long* out) {
  const int q = threadIdx.x;
  if (q < world) out[q] = (unsigned long long)ncclGetLsaPointer(win, 0, q);
  if (q == 0) out[world] = (unsigned long long)ncclGetLocalPointer(win, 0);
}
#endif

}  // namespace isr
