// isr_runtime.cu -- host runtime and C ABI of libising_sr.so (include/ising_sr.h).
//
// Drives the synchronous-relaxation loop of the paper: for each
// window ("step") it launches the region-trajectory kernel once per
// relaxation iteration, exchanges strip halos (world > 1: NCCL send/recv on
// its own stream, or the caller's transport), all-reduces the global
// {changed, overflow} flag, and on convergence commits the window by
// swapping the committed and tentative state buffers and compacting the
// event log.  Device memory layout: DESIGN.md §5.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges for nsys / ncu --nvtx

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/ising_sr.h"
#include "isr_region.cuh"
#include "isr_warp.cuh"
#include "isr_big.cuh"
#include "isr_nccl.h"
#include "isr_peer.cuh"

namespace {

// NVTX range for the lifetime of a scope (window / iteration / commit)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

using isr::EdgeView;
using isr::GhostView;
using isr::KArgs;
using isr::StateView;

constexpr int kThreads = isr::NT;  // K1 block (and the small kernels')

// ---------------------------------------------------------------------------
// per-shape kernel table (lane-per-region forms)
// ---------------------------------------------------------------------------
struct ShapeOps {
  int bx, by;
  bool warp;         // warp-per-region form (regions > 64 sites)
  bool single_edge;  // 1x1 regions: one stored edge history (the four are identical)
  size_t spin_bytes, halo_bytes;
  int sel_words;     // selector words per region (2: packed per region; 8: pair per edge)
  int cnt_max;       // largest history length the selector can record
  double sel_read_bytes;  // selector bytes read per recomputation (own + neighbours)
  void (*region)(const KArgs&, int nreg, cudaStream_t);
  void (*replay)(const KArgs&, int nreg, cudaStream_t);  // LOG = true: writes the compact log of the listed regions
  void (*init)(const uint8_t*, int, int, int, int, unsigned long long, double, StateView, cudaStream_t);
  void (*unpack)(StateView, int, int, int, uint8_t*, cudaStream_t);
  void (*pack)(const KArgs&, GhostView, GhostView, int RX, cudaStream_t);
  void (*snap)(StateView, int n, int RX, int RYg, unsigned long long* out, cudaStream_t);  // M, B of a state
};

template <int BX, int BY>
ShapeOps make_ops() {
  using G = isr::Geo<BX, BY>;
  constexpr bool kMB = BX * BY > 32;  // 64-bit site masks: launch bounds for 5 blocks (isr_region.cuh)
  ShapeOps o;
  o.bx = BX;
  o.by = BY;
  o.warp = false;
  o.single_edge = G::SE;
  o.spin_bytes = sizeof(typename G::ST);
  o.halo_bytes = sizeof(typename G::HT);
  o.sel_words = 2;
  o.cnt_max = isr::CNT_MAX;
  o.sel_read_bytes = 5 * 16.0;
  o.region = [](const KArgs& a, int n, cudaStream_t s) {
    int grid = (n + a.tile - 1) / a.tile;
    {  // a small worklist: blocks for one region per 2^k lanes within one wave (the kernel derives k from the grid)
      int k = 0;
      while (k < a.lane_spread && ((long long)n << (k + 1)) <= (long long)isr::kSpreadBlocks * kThreads) ++k;
      if (k > 0) grid = std::max(grid, (int)((((long long)n << k) + kThreads - 1) / kThreads));
    }
    // instantiations: FLAG_OBSERVABLES (integrate M and B) x the window's first
    // iteration (no incoming histories: break-point and staging code compiled out)
    if (a.obs) {
      if (a.first) {
        if constexpr (kMB) isr::region_kernel_mb<BX, BY, false, true, true><<<grid, kThreads, 0, s>>>(a);
        else isr::region_kernel_first<BX, BY, true><<<grid, kThreads, 0, s>>>(a);
      } else {
        if constexpr (kMB) isr::region_kernel_mb<BX, BY, false, true><<<grid, kThreads, 0, s>>>(a);
        else isr::region_kernel<BX, BY, false, true><<<grid, kThreads, 0, s>>>(a);
      }
    } else if (a.plain && !a.fresh_w && a.RX > 1 && a.RYg > 1 && (a.first || a.desc)) {
      // the common case: axis-wrap and fresh-window code compiled out (ghost rows: the descriptors)
      if (a.first) {
        if constexpr (kMB) isr::region_kernel_mb<BX, BY, false, false, true, true><<<grid, kThreads, 0, s>>>(a);
        else isr::region_kernel_first<BX, BY, false, true><<<grid, kThreads, 0, s>>>(a);
      } else {
        if constexpr (kMB) isr::region_kernel_mb<BX, BY, false, false, false, true><<<grid, kThreads, 0, s>>>(a);
        else isr::region_kernel<BX, BY, false, false, false, true><<<grid, kThreads, 0, s>>>(a);
      }
    } else if (a.first) {
      if constexpr (kMB) isr::region_kernel_mb<BX, BY, false, false, true><<<grid, kThreads, 0, s>>>(a);
      else isr::region_kernel_first<BX, BY><<<grid, kThreads, 0, s>>>(a);
    } else {
      if constexpr (kMB) isr::region_kernel_mb<BX, BY, false><<<grid, kThreads, 0, s>>>(a);
      else isr::region_kernel<BX, BY, false><<<grid, kThreads, 0, s>>>(a);
    }
  };
  o.replay = [](const KArgs& a, int n, cudaStream_t s) {
    const int grid = (n + a.tile - 1) / a.tile;
    if constexpr (kMB) isr::region_kernel_mb<BX, BY, true><<<grid, kThreads, 0, s>>>(a);
    else isr::region_kernel<BX, BY, true><<<grid, kThreads, 0, s>>>(a);
  };
  o.init = [](const uint8_t* buf, int Lx, int RX, int RYl, int row0, unsigned long long seed, double eq_q,
              StateView st, cudaStream_t s) {
    const int n = RX * RYl;
    isr::init_kernel<BX, BY><<<(n + kThreads - 1) / kThreads, kThreads, 0, s>>>(buf, Lx, RX, RYl, row0, seed, eq_q,
                                                                                st);
  };
  o.unpack = [](StateView st, int Lx, int RX, int RYl, uint8_t* out, cudaStream_t s) {
    const long long n = (long long)RYl * BY * Lx;
    isr::unpack_kernel<BX, BY><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(st, Lx, RX, RYl, out);
  };
  o.pack = [](const KArgs& a, GhostView up, GhostView down, int RX, cudaStream_t s) {
    isr::pack_kernel<<<(2 * RX + 127) / 128, 128, 0, s>>>(a, up, down);
  };
  o.snap = [](StateView st, int n, int RX, int RYg, unsigned long long* out, cudaStream_t s) {
    isr::snap_kernel<BX, BY><<<(n + 255) / 256, 256, 0, s>>>(st, n, RX, RYg, out);
  };
  return o;
}

bool big_enabled() {
  static const int v = [] {
    const char* e = std::getenv("ISING_SR_BIG");
    return e ? std::atoi(e) : 1;
  }();
  return v != 0;
}

template <int BX, int BY>
ShapeOps make_ops_w() {
  ShapeOps o;
  o.bx = BX;
  o.by = BY;
  o.warp = true;
  o.single_edge = false;
  o.spin_bytes = (size_t)BY * 4;
  o.halo_bytes = 16;
  o.sel_words = 8;
  o.cnt_max = 65535;
  o.sel_read_bytes = 8 * 16.0;
  // lane-per-region K1 for big regions (isr_big.cuh); ISING_SR_BIG=0: warp form
  o.region = [](const KArgs& a, int n, cudaStream_t s) {
    if (big_enabled()) {
      // small worklists: spread to one region per 2^sl lanes while the grid stays within ~one wave
      static const int smax = [] {
        const char* e = std::getenv("ISING_SR_BIG_SPREAD");
        return e ? std::max(0, std::min(5, std::atoi(e))) : 5;
      }();
      static const long long cap = [] {  // threads the spread may fill: 148 SMs x BNT x this
        const char* e = std::getenv("ISING_SR_BIG_SPREAD_CAP");
        return 148LL * isr::BNT * (e ? std::max(1, std::atoi(e)) : 7);  // 7 = one wave (ISR_BIG_MINB): best of 2, 4, 7, 14, 28
      }();
      KArgs b = a;
      b.spread_log2 = 0;
      while (b.spread_log2 < smax && (long long)n << (b.spread_log2 + 1) <= cap) ++b.spread_log2;
      const long long threads = (long long)n << b.spread_log2;
      const int grid = (int)std::max(1LL, std::min((threads + isr::BNT - 1) / isr::BNT, 148LL * 32));
      if (a.obs) isr::region_kernel_big<BX, BY, false, true><<<grid, isr::BNT, 0, s>>>(b);
      else isr::region_kernel_big<BX, BY, false><<<grid, isr::BNT, 0, s>>>(b);
    } else {
      const int grid = std::max(1, std::min((n + 3) / 4, 148 * 16));
      isr::region_kernel_w<BX, BY, false><<<grid, kThreads, 0, s>>>(a);
    }
  };
  o.replay = [](const KArgs& a, int n, cudaStream_t s) {
    if (big_enabled()) {
      const int grid = std::max(1, std::min((n + isr::BNT - 1) / isr::BNT, 148 * 32));
      isr::region_kernel_big<BX, BY, true><<<grid, isr::BNT, 0, s>>>(a);
    } else {
      const int grid = std::max(1, std::min((n + 3) / 4, 148 * 16));
      isr::region_kernel_w<BX, BY, true><<<grid, kThreads, 0, s>>>(a);
    }
  };
  o.init = [](const uint8_t* buf, int Lx, int RX, int RYl, int row0, unsigned long long seed, double eq_q,
              StateView st, cudaStream_t s) {
    const int n = RX * RYl;
    isr::init_kernel_w<BX, BY><<<(n + kThreads - 1) / kThreads, kThreads, 0, s>>>(buf, Lx, RX, RYl, row0, seed,
                                                                                  eq_q, st);
  };
  o.unpack = [](StateView st, int Lx, int RX, int RYl, uint8_t* out, cudaStream_t s) {
    const long long n = (long long)RYl * BY * Lx;
    isr::unpack_kernel_w<BX, BY><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(st, Lx, RX, RYl, out);
  };
  o.pack = [](const KArgs& a, GhostView up, GhostView down, int RX, cudaStream_t s) {
    isr::pack_kernel_w<<<(2 * RX + 127) / 128, 128, 0, s>>>(a, up, down);
  };
  o.snap = [](StateView st, int n, int RX, int RYg, unsigned long long* out, cudaStream_t s) {
    isr::snap_kernel_w<BX, BY><<<(n + 255) / 256, 256, 0, s>>>(st, n, RX, RYg, out);
  };
  return o;
}

const ShapeOps* find_ops(int bx, int by) {
  static const ShapeOps table[] = {make_ops<1, 1>(),    make_ops<2, 2>(),    make_ops<4, 4>(),    make_ops<8, 8>(),
                                   make_ops<4, 2>(),    make_ops<2, 4>(),    make_ops<8, 4>(),    make_ops<4, 8>(),
                                   make_ops_w<16, 16>(), make_ops_w<32, 32>(), make_ops_w<16, 32>(), make_ops_w<32, 16>(),
                                   make_ops_w<16, 8>(),  make_ops_w<8, 16>()};
  for (const auto& o : table)
    if (o.bx == bx && o.by == by) return &o;
  return nullptr;
}

// ---------------------------------------------------------------------------
// exclusive scan of e_i = n_next[i] - n_comm[i] (the commit's log offsets):
// 16 consecutive regions per thread (two 64-byte vector loads), 4096 per
// block, then one block over the block sums
// ---------------------------------------------------------------------------
constexpr int kScanPer = 16, kScanThreads = 256, kScanBlock = kScanPer * kScanThreads;

__device__ __forceinline__ unsigned scan_items(const uint32_t* n1, const uint32_t* n0, int N, int i0, unsigned* e) {
  unsigned s = 0;
  if (i0 + kScanPer <= N) {  // 16-byte aligned: i0 is a multiple of 16
    const uint4* a = reinterpret_cast<const uint4*>(n1 + i0);
    const uint4* b = reinterpret_cast<const uint4*>(n0 + i0);
#pragma unroll
    for (int v = 0; v < kScanPer / 4; ++v) {
      const uint4 x = a[v], y = b[v];
      e[4 * v] = x.x - y.x;
      e[4 * v + 1] = x.y - y.y;
      e[4 * v + 2] = x.z - y.z;
      e[4 * v + 3] = x.w - y.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < kScanPer; ++q) e[q] = i0 + q < N ? n1[i0 + q] - n0[i0 + q] : 0u;
  }
#pragma unroll
  for (int q = 0; q < kScanPer; ++q) s += e[q];
  return s;
}

// block-wide exclusive scan of one value per thread; returns the prefix, *total = the block's sum
__device__ __forceinline__ unsigned long long block_excl_scan(unsigned long long v, unsigned long long* total) {
  __shared__ unsigned long long sh[kScanThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += t;
  }
  if (lane == 31) sh[w] = x;
  __syncthreads();
  unsigned long long pre = 0, tot = 0;
#pragma unroll
  for (int q = 0; q < kScanThreads / 32; ++q) {
    pre += q < w ? sh[q] : 0ull;
    tot += sh[q];
  }
  *total = tot;
  return pre + x - v;
}

__global__ void __launch_bounds__(kScanThreads) scan_block_sums(const uint32_t* n1, const uint32_t* n0, int N,
                                                                unsigned long long* bsum) {
  unsigned e[kScanPer];
  const unsigned s = scan_items(n1, n0, N, (blockIdx.x * kScanThreads + threadIdx.x) * kScanPer, e);
  unsigned long long tot;
  block_excl_scan(s, &tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

// sum of e_i = n1[i] - n0[i] (the window's committed events) without offsets
__global__ void __launch_bounds__(256) count_events(const uint32_t* n1, const uint32_t* n0, int N,
                                                    unsigned long long* total) {
  unsigned long long v = 0;
  for (int i = blockIdx.x * 256 + threadIdx.x; i < N; i += gridDim.x * 256) v += (unsigned long long)(n1[i] - n0[i]);
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(total, v);
}

// FLAG_OBSERVABLES: sums of the per-region integrals in a fixed order (a fixed
// grid of blocks over contiguous chunks, fixed per-thread strides, fixed trees),
// so the window's totals do not depend on the schedule
constexpr int kObsBlocks = 256;
__global__ void __launch_bounds__(256) obs_partial(const double* a, const double* b, int n, double* part) {
  __shared__ double sa[256], sb[256];
  const int chunk = (n + kObsBlocks - 1) / kObsBlocks;
  const int beg = blockIdx.x * chunk, end = min(n, beg + chunk);
  double x = 0.0, y = 0.0;
  for (int i = beg + (int)threadIdx.x; i < end; i += 256) {
    x += a[i];
    y += b[i];
  }
  sa[threadIdx.x] = x;
  sb[threadIdx.x] = y;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      sa[threadIdx.x] += sa[threadIdx.x + o];
      sb[threadIdx.x] += sb[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = sa[0];
    part[2 * blockIdx.x + 1] = sb[0];
  }
}
__global__ void __launch_bounds__(256) obs_final(const double* part, double* out) {
  __shared__ double sa[256], sb[256];
  sa[threadIdx.x] = part[2 * threadIdx.x];
  sb[threadIdx.x] = part[2 * threadIdx.x + 1];
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      sa[threadIdx.x] += sa[threadIdx.x + o];
      sb[threadIdx.x] += sb[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = sa[0];
    out[1] = sb[0];
  }
}

__global__ void scan_top(unsigned long long* bsum, int nb, unsigned long long* total) {
  // single block, sequential chunks of 1024 with a carried prefix
  __shared__ unsigned long long sh[1024];
  unsigned long long carry = 0;
  for (int base = 0; base < nb; base += 1024) {
    const int i = base + threadIdx.x;
    const unsigned long long v = i < nb ? bsum[i] : 0ull;
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      const unsigned long long t = threadIdx.x >= (unsigned)o ? sh[threadIdx.x - o] : 0ull;
      __syncthreads();
      sh[threadIdx.x] += t;
      __syncthreads();
    }
    if (i < nb) bsum[i] = carry + sh[threadIdx.x] - v;  // exclusive
    const unsigned long long chunk = sh[1023];
    __syncthreads();
    carry += chunk;
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void __launch_bounds__(kScanThreads) scan_apply(const uint32_t* n1, const uint32_t* n0, int N,
                                                           const unsigned long long* bsum, unsigned long long* off) {
  unsigned e[kScanPer];
  const int i0 = (blockIdx.x * kScanThreads + threadIdx.x) * kScanPer;
  const unsigned s = scan_items(n1, n0, N, i0, e);
  unsigned long long tot;
  unsigned long long o = bsum[blockIdx.x] + block_excl_scan(s, &tot);
#pragma unroll
  for (int q = 0; q < kScanPer; ++q) {
    if (i0 + q < N) off[i0 + q] = o;
    o += e[q];
  }
}


// K3 (commit, FLAG_LOG_EVENTS): compact the window's event log -- time,
// global region id, local site, ordered by region then time -- from the
// scratch log K1 wrote in each region's final recomputation (event q of
// region i at ev[q * stride + i], q < C).  A warp takes 32 consecutive
// regions and writes their events with consecutive lanes on consecutive log
// entries (each lane finds its region by a shuffle binary search over the
// warp's prefix of event counts).  A region with more than C events is
// appended to `replay` (its log is rewritten there by a K1 replay).  Also
// counts h of SURVEY §8(d.3): one entry per region edge (not along an axis
// the region wraps) that each event's site lies on.
__device__ __forceinline__ unsigned edges_of_site(unsigned site, int lbx, int bx, int by, int wrapX, int wrapY) {
  const int sr = (int)(site >> lbx), sc = (int)(site & (unsigned)(bx - 1));
  return (unsigned)((!wrapY && sr == 0) + (!wrapY && sr == by - 1) + (!wrapX && sc == 0) + (!wrapX && sc == bx - 1));
}

__global__ void __launch_bounds__(256) compact_log_kernel(const uint32_t* n1, const uint32_t* n0, int N,
                                                          const unsigned long long* off, const double* ev_t,
                                                          const uint16_t* ev_s, long long stride, int C, int RX,
                                                          int row0, int lbx, int bx, int by, int wrapX, int wrapY,
                                                          double* log_t, uint32_t* log_region, uint16_t* log_site,
                                                          int8_t* log_dm, uint32_t* replay, unsigned* n_replay,
                                                          unsigned long long* edges) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * 256 + threadIdx.x;
  const unsigned e = i < N ? n1[i] - n0[i] : 0u;
  const bool over = (int)e > C;
  if (over) replay[atomicAdd(n_replay, 1u)] = (uint32_t)i;
  const unsigned ec = over ? 0u : e;  // events compacted here
  unsigned pre = ec;                 // inclusive warp scan
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned t = __shfl_up_sync(full, pre, o);
    if (lane >= o) pre += t;
  }
  const unsigned T = __shfl_sync(full, pre, 31);
  pre -= ec;  // exclusive
  const unsigned long long my_off = i < N ? off[i] : 0ull;
  const int i_w = i - lane;  // the warp's first region
  unsigned long long ne = 0;
  for (unsigned base = 0; base < T; base += 32) {
    const unsigned k = base + lane;
    // the lane j whose range [pre_j, pre_j + ec_j) holds k: the largest j with pre_j <= k
    int j = 0;
#pragma unroll
    for (int step = 16; step >= 1; step >>= 1) {
      const unsigned pc = __shfl_sync(full, pre, (j + step) & 31);
      if (j + step < 32 && pc <= k) j += step;
    }
    const unsigned pj = __shfl_sync(full, pre, j);
    const unsigned long long oj = __shfl_sync(full, my_off, j);
    if (k < T) {
      const unsigned q = k - pj;
      const int r = i_w + j;
      const long long src = (long long)q * stride + r;
      const unsigned sv = ev_s[src];  // bit 15: the flipped site's new spin
      const unsigned site = sv & 0x7FFFu;
      const unsigned long long o = oj + q;
      const int rr = r / RX;
      log_t[o] = ev_t[src];
      log_region[o] = (uint32_t)((row0 + rr) * RX + (r - rr * RX));
      log_site[o] = (uint16_t)site;
      if (log_dm) log_dm[o] = (sv >> 15) ? 2 : -2;
      ne += edges_of_site(site, lbx, bx, by, wrapX, wrapY);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ne += __shfl_xor_sync(full, ne, o);
  if (lane == 0 && ne) atomicAdd(edges, ne);
}

// the edge entries of the replayed regions' events (after the replay wrote them)
__global__ void __launch_bounds__(256) replay_edge_entries(const uint32_t* replay, const unsigned* n_replay,
                                                           const uint32_t* n1, const uint32_t* n0,
                                                           const unsigned long long* off, const uint16_t* log_site,
                                                           int lbx, int bx, int by, int wrapX, int wrapY,
                                                           unsigned long long* edges) {
  const unsigned n = *n_replay;
  unsigned long long ne = 0;
  for (unsigned t = blockIdx.x * 256 + threadIdx.x; t < n; t += gridDim.x * 256) {
    const uint32_t i = replay[t];
    const unsigned e = n1[i] - n0[i];
    for (unsigned q = 0; q < e; ++q) ne += edges_of_site(log_site[off[i] + q], lbx, bx, by, wrapX, wrapY);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ne += __shfl_xor_sync(0xffffffffu, ne, o);
  if ((threadIdx.x & 31) == 0 && ne) atomicAdd(edges, ne);
}

// ---------------------------------------------------------------------------
// FLAG_MAG_MOMENTS: time integrals of |M| and M^2 over the window [t_c, t_w)
// (the magnetisation is the model's observable).  M(t) is piecewise
// constant and jumps by dM = +-2 at each committed event, so the integrals
// need the window's events in global time order: a bucket sort by time
// (monotone bucket index, then an insertion sort of each bucket by exact
// time; events at equal times may come in any order, they bound intervals
// of length 0), a prefix sum of dM from M(t_c), and fixed-order reductions
// (the result does not depend on the schedule).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int mm_bucket(double t, double t0, double scale, int B) {
  const int b = (int)__dmul_rn(__dsub_rn(t, t0), scale);
  return b < 0 ? 0 : b >= B ? B - 1 : b;
}

__global__ void __launch_bounds__(256) mm_count(const double* t, const unsigned long long* n_total, double t0,
                                                double scale, int B, unsigned* cnt) {
  const unsigned long long n = *n_total;
  for (unsigned long long i = (unsigned long long)blockIdx.x * 256 + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * 256)
    atomicAdd(&cnt[mm_bucket(t[i], t0, scale, B)], 1u);
}

// exclusive scan of cnt[0..B) into off[0..B] in one block (B <= 2^22)
__global__ void __launch_bounds__(1024) mm_scan_buckets(const unsigned* cnt, int B, unsigned* off) {
  __shared__ unsigned sh[1024];
  const int per = (B + 1023) / 1024;
  const int b0 = threadIdx.x * per, b1 = min(B, b0 + per);
  unsigned sum = 0;
  for (int b = b0; b < b1; ++b) sum += cnt[b];
  sh[threadIdx.x] = sum;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const unsigned v = threadIdx.x >= (unsigned)o ? sh[threadIdx.x - o] : 0u;
    __syncthreads();
    sh[threadIdx.x] += v;
    __syncthreads();
  }
  unsigned run = sh[threadIdx.x] - sum;
  for (int b = b0; b < b1; ++b) {
    off[b] = run;
    run += cnt[b];
  }
  if (threadIdx.x == 1023) off[B] = sh[1023];
}

__global__ void __launch_bounds__(256) mm_scatter(const double* t, const int8_t* dm, const unsigned long long* n_total,
                                                  double t0, double scale, int B, const unsigned* off, unsigned* fill,
                                                  double* ts, int8_t* dms) {
  const unsigned long long n = *n_total;
  for (unsigned long long i = (unsigned long long)blockIdx.x * 256 + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * 256) {
    const int b = mm_bucket(t[i], t0, scale, B);
    const unsigned p = off[b] + atomicAdd(&fill[b], 1u);
    ts[p] = t[i];
    dms[p] = dm[i];
  }
}

// each bucket sorted by exact time (insertion sort; a bucket holds ~16 events)
__global__ void __launch_bounds__(256) mm_sort_buckets(const unsigned* off, int B, double* ts, int8_t* dms) {
  const int b = blockIdx.x * 256 + threadIdx.x;
  if (b >= B) return;
  const unsigned lo = off[b], hi = off[b + 1];
  for (unsigned i = lo + 1; i < hi; ++i) {
    const double x = ts[i];
    const int8_t d = dms[i];
    unsigned j = i;
    while (j > lo && ts[j - 1] > x) {
      ts[j] = ts[j - 1];
      dms[j] = dms[j - 1];
      --j;
    }
    ts[j] = x;
    dms[j] = d;
  }
}

constexpr int kMmBlocks = 1024;
// pass 1: sum of dM over each block's fixed chunk of the sorted events
__global__ void __launch_bounds__(256) mm_chunk_sums(const int8_t* dms, const unsigned long long* n_total,
                                                     long long* csum) {
  const long long n = (long long)*n_total;
  const long long chunk = (n + kMmBlocks - 1) / kMmBlocks;
  const long long beg = blockIdx.x * chunk, end = min(n, beg + chunk);
  long long v = 0;
  for (long long i = beg + threadIdx.x; i < end; i += 256) v += dms[i];
  __shared__ long long sh[256];
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) csum[blockIdx.x] = sh[0];
}

// pass 2: each block walks its chunk in tiles of 256 events with a running M
// (M(t_c) + the dM of all earlier chunks + a block scan), adding
// |M_k| (t_{k+1} - t_k) and M_k^2 (t_{k+1} - t_k) for the interval after
// event k (t_n = t_w); fixed per-thread order and a fixed tree per block
__global__ void __launch_bounds__(256) mm_integrate(const double* ts, const int8_t* dms,
                                                    const unsigned long long* n_total, const long long* csum,
                                                    const unsigned long long* M0p, double t_w, double* part) {
  const long long n = (long long)*n_total;
  const long long chunk = (n + kMmBlocks - 1) / kMmBlocks;
  const long long beg = blockIdx.x * chunk, end = min(n, beg + chunk);
  __shared__ long long carry;
  __shared__ int wsum[8];
  if (threadIdx.x == 0) {
    long long c = (long long)*M0p;
    for (int j = 0; j < (int)blockIdx.x; ++j) c += csum[j];
    carry = c;
  }
  __syncthreads();
  double a1 = 0.0, a2 = 0.0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (long long base = beg; base < end; base += 256) {
    const long long i = base + threadIdx.x;
    const int d = i < end ? dms[i] : 0;
    int x = d;  // inclusive block scan of dM
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    int wpre = 0, tile = 0;
    for (int q = 0; q < 8; ++q) {
      wpre += q < wid ? wsum[q] : 0;
      tile += wsum[q];
    }
    if (i < end) {
      const long long M = carry + wpre + x;  // M after event i
      const double tn = i + 1 < n ? ts[i + 1] : t_w;
      const double dt = __dsub_rn(tn, ts[i]);
      const double Md = (double)M;
      a1 = __dadd_rn(a1, __dmul_rn(fabs(Md), dt));
      a2 = __dadd_rn(a2, __dmul_rn(__dmul_rn(Md, Md), dt));
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += tile;
    __syncthreads();
  }
  __shared__ double s1[256], s2[256];
  s1[threadIdx.x] = a1;
  s2[threadIdx.x] = a2;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      s1[threadIdx.x] = __dadd_rn(s1[threadIdx.x], s1[threadIdx.x + o]);
      s2[threadIdx.x] = __dadd_rn(s2[threadIdx.x], s2[threadIdx.x + o]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s1[0];
    part[2 * blockIdx.x + 1] = s2[0];
  }
}

// pass 3: the interval before the first event, |M(t_c)| (t_0 - t_c), plus the
// blocks' partial sums in a fixed tree -> out[0] = int |M| dt, out[1] = int M^2 dt
__global__ void __launch_bounds__(1024) mm_final(const double* part, const double* ts,
                                                 const unsigned long long* n_total, const unsigned long long* M0p,
                                                 double t_c, double t_w, double* out) {
  __shared__ double s1[1024], s2[1024];
  s1[threadIdx.x] = part[2 * threadIdx.x];
  s2[threadIdx.x] = part[2 * threadIdx.x + 1];
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      s1[threadIdx.x] = __dadd_rn(s1[threadIdx.x], s1[threadIdx.x + o]);
      s2[threadIdx.x] = __dadd_rn(s2[threadIdx.x], s2[threadIdx.x + o]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double M0 = (double)(long long)*M0p;
    const double t0 = *n_total ? ts[0] : t_w;
    const double dt = __dsub_rn(t0, t_c);
    out[0] = __dadd_rn(__dmul_rn(fabs(M0), dt), s1[0]);
    out[1] = __dadd_rn(__dmul_rn(__dmul_rn(M0, M0), dt), s2[0]);
  }
}

// Initial spins from the Philox init stream for the rows
// the init kernel reads: row q of buf is lattice row (y_first + q) mod Ly;
// site v is up iff bit (v & 31) of word ((v >> 5) & 3) of Philox4x32-10 with
// key (0xFFFFFFFF, seed_lo) and counter (v >> 7, 0, 1, seed_hi) is set.
__global__ void __launch_bounds__(256) philox_spins_kernel(uint8_t* buf, int rows, int y_first, int Lx, int Ly,
                                                           unsigned long long seed) {
  const long long i = (long long)blockIdx.x * 256 + threadIdx.x;
  if (i >= (long long)rows * Lx) return;
  const int q = (int)(i / Lx), x = (int)(i - (long long)q * Lx);
  const int y = ((y_first + q) % Ly + Ly) % Ly;
  const unsigned long long v = (unsigned long long)y * (unsigned long long)Lx + (unsigned long long)x;
  const isr::U4 c{(uint32_t)(v >> 7), 0u, 1u, (uint32_t)(seed >> 32)};
  const isr::U4 w = isr::philox4x32_10(c, 0xFFFFFFFFu, (uint32_t)seed);
  const int k = (int)((v >> 5) & 3);
  const uint32_t word = k == 0 ? w.x : k == 1 ? w.y : k == 2 ? w.z : w.w;
  buf[i] = (uint8_t)((word >> (v & 31)) & 1u);
}

}  // namespace

// ---------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------
// pipelined loop: everything one iteration reports, in one block (zeroed by
// one memset, read back by one copy).  Slot K & 1 holds iteration K's flags
// and counters and the length of iteration K+1's worklist.
struct IterSlot {
  int flags[4];
  unsigned long long stats[8];
  unsigned wl_next;
  unsigned pad[3];
  unsigned long long ktime[2];  // graph loop: K1's first block start / last block end (ns)
};

// device-side window loop (ISING_SR_GRAPH): what the loop's advance kernels
// accumulate over the iterations of a window, read back once per window
struct WinDev {
  unsigned trip;   // completed loop trips (two iterations each)
  int it;          // iterations up to and including the converged one
  int g;           // the iteration at which no history changed (0: not yet)
  int overflow;
  unsigned long long active[64];
  unsigned long long ev, s1, s2, s3, s5, fmax;
  unsigned long long k1_ns;
};

__global__ void slot_reset(IterSlot* sl) {
  if (threadIdx.x == 0) {
    for (int k = 0; k < 4; ++k) sl->flags[k] = 0;
    for (int k = 0; k < 8; ++k) sl->stats[k] = 0;
    sl->wl_next = 0;
    sl->ktime[0] = ~0ull;
    sl->ktime[1] = 0;
  }
}

// after each iteration of the device-side loop: account the iteration (until
// the window has converged or overflowed), reset the slot of the iteration
// after next, count the loop trip, and set the while-condition: continue
// while histories change, no capacity overflowed and fewer than max
// iterations ran ("UNTIL all PEs detect no difference")
__global__ void advance_kernel(WinDev* w, const IterSlot* cur, IterSlot* next, int max_it,
                               cudaGraphConditionalHandle h, int set_cond, int end_of_trip) {
  if (threadIdx.x != 0) return;
  if (w->g == 0 && !w->overflow) {
    const int it = ++w->it;
    w->active[min(it, 64) - 1] += cur->stats[5];
    w->ev += cur->stats[0];
    w->s1 += cur->stats[1];
    w->s2 += cur->stats[2];
    w->s3 += cur->stats[3];
    w->s5 += cur->stats[5];
    w->fmax = max(w->fmax, cur->stats[4]);
    if (cur->ktime[1] > cur->ktime[0]) w->k1_ns += cur->ktime[1] - cur->ktime[0];
    if (cur->flags[1]) w->overflow = 1;
    else if (!cur->flags[0]) w->g = it;
  }
  for (int k = 0; k < 4; ++k) next->flags[k] = 0;
  for (int k = 0; k < 8; ++k) next->stats[k] = 0;
  next->wl_next = 0;
  next->ktime[0] = ~0ull;
  next->ktime[1] = 0;
  if (end_of_trip) w->trip += 1;
  if (set_cond) cudaGraphSetConditional(h, (w->g || w->overflow || w->it >= max_it) ? 0u : 1u);
}
struct ising_sr_ctx {
  ising_sr_config cfg;
  const ShapeOps* ops = nullptr;
  int RX = 0, RYg = 0, RYl = 0, row0 = 0, nreg = 0;
  int K = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  ising_sr_status sticky = ISING_SR_OK;

  // device buffers
  StateView st[2] = {};
  int comm = 0;  // index of the committed state
  EdgeView ed[2] = {};
  long long sstride = 0;                  // elements from ed[0] to ed[1] (one allocation)
  unsigned long long* sel = nullptr;  // per region selector word
  // big-region step logs (resume; isr_big.cuh)
  double2* lg_tR = nullptr;
  uint16_t* lg_c = nullptr;
  uint2* lg_meta = nullptr;
  int LC = 0;
  bool resume = true;  // env ISING_SR_RESUME=0 disables
  double2* pcache = nullptr;  // big-region kernel: the window's pairs per region (env ISING_SR_PCACHE=0 disables)
  uint2* pmeta = nullptr;
  int PC = 0;
  uint32_t* dirty = nullptr;          // dirty-region bitmaps [2][dwords] (iteration parity)
  int dwords = 0;
  uint32_t* wl[2] = {nullptr, nullptr};
  unsigned* d_wlc = nullptr;          // [2] worklist counts
  GhostView gsend[2] = {}, grecv[2] = {};  // [0] = up, [1] = down  (world > 1)
  void* gbuf = nullptr;
  size_t gchunk[4] = {0, 0, 0, 0};
  int* d_flags = nullptr;                 // [4] flags of the step-level loop
  unsigned long long* d_stats = nullptr;  // [8]
  int* h_flags = nullptr;                 // pinned mirror
  unsigned long long* h_stats = nullptr;  // pinned mirror
  unsigned* h_wlc = nullptr;              // pinned mirror [2]
  // strip exchange (world > 1 or FLAG_HALO_LOOPBACK)
  bool ghost = false;
  size_t grow = 0;                        // bytes of one ghost row (4 chunks, contiguous)
  isr_nccl::Comm nccl = nullptr;          // the library's communicator (cfg.nccl_id)
  // peer-memory exchange (isr_peer.cuh): ghost rows + flag inbox in an NCCL
  // symmetric window, one fused kernel per iteration (env ISING_SR_EXCHANGE=
  // sendrecv: the ncclSend/ncclRecv + ncclAllReduce path instead)
  bool peer = false;
  int peer_blocks = 0;
  void* pbuf = nullptr;                   // ncclMemAlloc'ed window memory
  size_t pbytes = 0;
  void* pwin = nullptr;                   // ncclWindow_t
  unsigned long long* d_peer = nullptr;   // [world + 1] window bases (LSA pointers; [world] = local)
  unsigned long long h_peer[isr::kPeerMaxWorld + 1] = {};
  isr::PeerArgs pargs{};
#if ISR_HAVE_NCCL_DEVICE
  ncclDevComm dcomm{};
  bool dcomm_ok = false;
#endif
  // scratch event log of K1 (FLAG_LOG_EVENTS) and the commit's replay list
  double* ev_t = nullptr;
  uint16_t* ev_s = nullptr;
  int evC = 0;
  uint32_t* d_replay = nullptr;
  unsigned* d_nrep = nullptr;             // [0] replayed regions, [2..3] edge entries (u64)
  unsigned h_nrep = 0;
  unsigned long long* d_edges = nullptr;
  unsigned long long h_edges = 0;
  cudaEvent_t cev0 = nullptr, cev1 = nullptr;  // around the commit's compaction
  // FLAG_MAG_MOMENTS: dM per logged event, the time-sorted copy, buckets, partial sums
  int8_t* log_dm = nullptr;
  double* mm_ts = nullptr;
  int8_t* mm_dm = nullptr;
  unsigned* mm_cnt = nullptr;  // [2 * mm_B + 1]: counts / fill, then offsets
  unsigned* mm_off = nullptr;
  int mm_B = 0;
  long long* mm_csum = nullptr;
  double* mm_part = nullptr;   // [2 * kMmBlocks + 2]
  double h_mm[2] = {0.0, 0.0};
  // log
  double* log_t = nullptr;
  uint32_t* log_region = nullptr;
  uint16_t* log_site = nullptr;
  long long log_cap = 0, log_n = 0;
  unsigned long long* d_off = nullptr;
  unsigned long long* d_bsum = nullptr;
  unsigned long long* d_total = nullptr;
  double* d_obs = nullptr;   // [2 * kObsBlocks] partial sums, then [2] window totals
  double h_obs[2] = {0.0, 0.0};
  unsigned long long* d_snap = nullptr;  // FLAG_OBSERVABLES: {M, B} of the committed configuration
  unsigned long long h_snap[2] = {0ull, 0ull};
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t kev0 = nullptr, kev1 = nullptr;  // around each region-kernel launch
  cudaEvent_t bev[4] = {};                     // pipelined iterations: around launch j (2j, 2j+1)

  // window state
  long long w = 0;
  double t_c = 0.0, t_w = 0.0;
  unsigned Kglob = 0;  // global iteration stamp (monotone across windows)
  unsigned K0 = 1;     // stamp of the current window's first iteration
  int it = 0;
  int n_work = 0;      // regions to recompute in the next iteration
  bool in_window = false, converged = false;
  int g = 0;
  // per-window accumulators
  unsigned long long win_events = 0;
  long long win_active[64] = {};  // regions recomputed per iteration of the window in progress
  double win_bytes = 0.0;
  int win_f = 0;
  long long launches = 0;
  int pipeline = 1;  // one iteration enqueued ahead of the flag check (env ISING_SR_PIPELINE=0: off)
  cudaEvent_t pev[2] = {};  // pipelined: results of the iteration with stamp parity j copied to the host
  IterSlot* d_slot = nullptr;  // [2]
  IterSlot* h_slot = nullptr;  // pinned mirror [2]
  int graph = 0;               // device-side window loop (env ISING_SR_GRAPH=1)
  WinDev* d_win = nullptr;
  WinDev* h_win = nullptr;     // pinned
  unsigned delay_ns = 0;  // test knob (env ISING_SR_K1_DELAY_NS): K1 publishes late
  bool plain = true;           // K1's PLAIN instantiation where it applies (env ISING_SR_PLAIN=0: never)
  uint4* desc = nullptr;       // worklist descriptors of PLAIN iterations (describe_kernel)
  int lane_spread = 5;  // lane K1: small worklists spread to one region per 2^k lanes, k <= this (env ISING_SR_LANE_SPREAD; 0 = off)
  int refill = 28;  // K1 batched-refill threshold (env ISING_SR_REFILL; 28 measured best after the shared fresh-load step)
  ising_sr_stats stats;
};

namespace {

ising_sr_status fail_cuda(ising_sr_ctx* c, cudaError_t e, const char* where) {
  if (e == cudaSuccess) return ISING_SR_OK;
  std::fprintf(stderr, "ising_sr: CUDA error at %s: %s\n", where, cudaGetErrorString(e));
  if (c) c->sticky = ISING_SR_E_CUDA;
  return ISING_SR_E_CUDA;
}

#define CK(ctx, expr)                                          \
  do {                                                         \
    cudaError_t _e = (expr);                                   \
    if (_e != cudaSuccess) return fail_cuda((ctx), _e, #expr); \
  } while (0)

// device memory: the caller's allocator hooks when given (e.g. torch's
// caching allocator, stream-ordered on the ctx stream), else cudaMalloc/cudaFree
cudaError_t dmalloc_bytes(ising_sr_ctx* c, void** p, size_t bytes) {
  if (c->cfg.dev_alloc) {
    *p = c->cfg.dev_alloc(std::max<size_t>(bytes, 1), c->cfg.alloc_user);
    return *p ? cudaSuccess : cudaErrorMemoryAllocation;
  }
  return cudaMalloc(p, std::max<size_t>(bytes, 1));
}
template <class T>
cudaError_t dmalloc(ising_sr_ctx* c, T** p, size_t count) {
  return dmalloc_bytes(c, (void**)p, std::max<size_t>(count, 1) * sizeof(T));
}
void dfree(ising_sr_ctx* c, void* p) {
  if (!p) return;
  if (c->cfg.dev_free) c->cfg.dev_free(p, c->cfg.alloc_user);
  else cudaFree(p);
}

void free_edges(ising_sr_ctx* c) {
  dfree(c, c->ed[0].t);  // one allocation holds both slots
  dfree(c, c->ed[0].pos);
  for (auto& e : c->ed) e = EdgeView{};
  dfree(c, c->gbuf);
  c->gbuf = nullptr;
  for (int i = 0; i < 2; ++i) {
    c->gsend[i] = GhostView{};
    c->grecv[i] = GhostView{};
  }
}

// Boundary-history slots sized for K entries per region edge, plus (world > 1
// or halo loopback) four ghost rows: send up/down and receive from up/down,
// each laid out as cnt[RX] | stamp[RX] | t[K][RX] | pos[K][RX] (the exchange
// chunks, 256-byte aligned, one contiguous row of c->grow bytes).
ising_sr_status alloc_edges(ising_sr_ctx* c, int K) {
  free_edges(c);
  c->K = K;
  const size_t cn = (size_t)(c->ops->single_edge ? 1 : 4) * c->RYl * c->RX;
  const size_t tn = cn * (size_t)K;
  if ((size_t)c->RYl * c->RX * (size_t)K >= (1ull << 32)) return ISING_SR_E_CAPACITY;  // 32-bit offsets within one edge array
  // both slots in one allocation (slot 1 at + tn): the kernels address a slot arithmetically
  if (dmalloc(c, &c->ed[0].t, 2 * tn) != cudaSuccess || dmalloc(c, &c->ed[0].pos, 2 * tn) != cudaSuccess) {
    cudaGetLastError();
    free_edges(c);
    return ISING_SR_E_OOM;
  }
  c->ed[1].t = c->ed[0].t + tn;
  c->ed[1].pos = c->ed[0].pos + tn;
  c->sstride = (long long)tn;
  if (c->ghost) {
    const size_t RX = (size_t)c->RX;
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    c->gchunk[0] = RX * 2;
    c->gchunk[1] = RX * 4;
    c->gchunk[2] = RX * (size_t)K * 8;
    c->gchunk[3] = RX * (size_t)K;
    const size_t one = al(c->gchunk[0]) + al(c->gchunk[1]) + al(c->gchunk[2]) + al(c->gchunk[3]);
    c->grow = one;
    if (dmalloc_bytes(c, (void**)&c->gbuf, 4 * one) != cudaSuccess) {
      cudaGetLastError();
      free_edges(c);
      return ISING_SR_E_OOM;
    }
    CK(c, cudaMemsetAsync(c->gbuf, 0, 4 * one, c->stream));
    GhostView* views[4] = {&c->gsend[0], &c->gsend[1], &c->grecv[0], &c->grecv[1]};
    for (int i = 0; i < 4; ++i) {
      char* b = (char*)c->gbuf + i * one;
      views[i]->cnt = (uint16_t*)b;
      b += al(c->gchunk[0]);
      views[i]->stamp = (uint32_t*)b;
      b += al(c->gchunk[1]);
      views[i]->t = (double*)b;
      b += al(c->gchunk[2]);
      views[i]->pos = (uint8_t*)b;
    }
  }
  return ISING_SR_OK;
}

int auto_capacity(const ising_sr_config& cfg, int cnt_max) {
  // expected boundary events per edge per window at the largest rate, with a
  // generous Poisson tail margin; overflow is detected and retried anyway
  double rmax = 0.0;
  for (double r : cfg.rate) rmax = std::max(rmax, r);
  const double mu = std::max(cfg.bx, cfg.by) * rmax * cfg.W;
  const int K = (int)std::ceil(mu + 6.0 * std::sqrt(mu) + 8.0);
  return std::min(std::max(K, 8), cnt_max);
}

ising_sr_status check(const ising_sr_ctx* c) {
  if (!c) return ISING_SR_E_INVALID_ARG;
  return c->sticky;
}

// work items per block: enough blocks for >= 4 per SM, at most 8 items per
// lane (env ISING_SR_TILE_PER overrides the cap)
int tile_for(int n) {
  static const int cap = [] {
    const char* e = std::getenv("ISING_SR_TILE_PER");
    return e ? std::max(1, std::atoi(e)) : 8;  // c4: 8 > 16 (+1 %) > 4, 32, 64
  }();
  const int per = std::max(1, std::min(cap, n / (kThreads * 148 * 4)));
  return kThreads * per;
}

KArgs base_args(ising_sr_ctx* c, unsigned K, bool first) {
  KArgs a;
  std::memset(&a, 0, sizeof a);
  a.in = c->st[c->comm];
  a.out = c->st[c->comm ^ 1];
  a.ed[0] = c->ed[0];
  a.ed[1] = c->ed[1];
  a.sel = c->sel;
  a.gh_up = c->grecv[0];
  a.gh_down = c->grecv[1];
  if (c->peer) {  // the rows the neighbours stored at the previous iteration (stamp K - 1)
    a.gh_up = isr::peer_row(c->pargs, c->pargs.mine, (int)((K - 1u) & 1u), 0);
    a.gh_down = isr::peer_row(c->pargs, c->pargs.mine, (int)((K - 1u) & 1u), 1);
  }
  a.RX = c->RX;
  a.RYl = c->RYl;
  a.RYg = c->RYg;
  a.row0 = c->row0;
  a.world = c->cfg.world;
  a.ghost = c->ghost ? 1 : 0;
  a.single_edge = c->ops->single_edge ? 1 : 0;
  a.eq_q = c->cfg.eq_quantum;
  a.ev_t = c->ev_t;
  a.ev_s = c->ev_s;
  a.evC = c->evC;
  a.ev_stride = c->nreg;
  a.K = c->K;
  a.tstride = (long long)c->RYl * c->K * c->RX;
  a.sstride = c->sstride;
  a.it_K = K;
  a.it_K0 = c->K0;
  a.first = first ? 1 : 0;
  a.digest = (c->cfg.flags & ISING_SR_FLAG_DIGEST) ? 1 : 0;
  a.t_w = c->t_w;
  a.t_c = c->t_c;
  a.fresh_w = (c->cfg.flags & ISING_SR_FLAG_FRESH_WINDOW) ? 1 : 0;
  a.obs = (c->cfg.flags & ISING_SR_FLAG_OBSERVABLES) ? 1 : 0;
  a.gen = a.fresh_w ? (unsigned)c->w : 0u;
  a.seed = c->cfg.seed;
  for (int k = 0; k < 10; ++k) a.rate[k] = c->cfg.rate[k];
  a.dirty = c->dirty;
  a.dwords = c->dwords;
  a.lg_tR = c->lg_tR;
  a.lg_c = c->lg_c;
  a.lg_meta = c->lg_meta;
  a.LC = c->LC;
  a.resume = (c->resume && c->lg_meta) ? 1 : 0;
  a.pcache = c->pcache;
  a.pmeta = c->pmeta;
  a.PC = c->PC;
  a.refill = c->refill;
  a.lane_spread = c->lane_spread;
  a.plain = c->plain ? 1 : 0;
  a.delay_ns = c->delay_ns;
  {
    // magic division by RX: k = 31 + ceil(log2 RX), M = ceil(2^k / RX) < 2^32;
    // exact for every index below 2^31 (M * RX - 2^k < RX <= 2^(k - 31))
    int l = 0;
    while ((1ll << l) < c->RX) ++l;
    a.rx_k = 31 + l;
    a.rx_M = (unsigned)(((1ull << a.rx_k) + (unsigned long long)c->RX - 1) / (unsigned long long)c->RX);
  }
  a.flags = c->d_flags;
  a.stats = c->d_stats;
  return a;
}

// algorithmic bytes of one iteration: per recomputed region
// the committed state read + tentative state written, the selector word
// pairs read (own + 4 neighbours, 16 B each) and one selector word written;
// 9 bytes per history entry written, read as a break point, and compared.
double iteration_bytes(const ising_sr_ctx* c, const unsigned long long* s) {
  const double S = (double)c->ops->spin_bytes + (double)c->ops->halo_bytes + 8 + 8 + 4 +
                   ((c->cfg.flags & ISING_SR_FLAG_DIGEST) ? 8 : 0);
  const double regions = (double)s[5];
  return regions * (2.0 * S + c->ops->sel_read_bytes + 8.0) + 9.0 * ((double)s[1] + (double)s[2] + (double)s[3]);
}

int compact_grid(const ising_sr_ctx* c) {
  const int per = isr::kCompactThreads * isr::kCompactWords;
  return std::max(1, (c->dwords + per - 1) / per);
}

// iterations after the first run K1's PLAIN instantiation from worklist
// descriptors when the strip has no ghost rows, no region spans an axis and
// windows do not restart afresh (the general kernel reads the selectors itself)
bool plain_desc(const ising_sr_ctx* c) {
  return c->plain && c->desc && !(c->cfg.flags & (ISING_SR_FLAG_FRESH_WINDOW | ISING_SR_FLAG_JACOBI_ALL)) &&
         c->RX > 1 && c->RYg > 1 && !(c->cfg.flags & ISING_SR_FLAG_OBSERVABLES);
}

// descriptors of the worklist iteration K will read (its length read on the
// device; `bound` sizes the grid -- worklists shrink as the relaxation
// converges, and a longer one is covered by the grid-stride loop)
void describe(ising_sr_ctx* c, unsigned K, const unsigned* count, int bound) {
  KArgs a = base_args(c, K, false);
  const int grid = std::max(1, std::min((bound + 255) / 256, 148 * 16));
  isr::describe_kernel<<<grid, 256, 0, c->stream>>>(a, K, c->wl[K & 1], count, c->desc);
  ++c->launches;
}

ising_sr_status peer_exchange(ising_sr_ctx* c, const KArgs& a, int* flags);  // (below)

ising_sr_status compact_worklist(ising_sr_ctx* c) {
  const unsigned K = c->Kglob;
  isr::compact_kernel<<<compact_grid(c), isr::kCompactThreads, 0, c->stream>>>(c->dirty + (size_t)((K + 1) & 1) * c->dwords,
                                                                       c->dwords, c->nreg, c->wl[(K + 1) & 1],
                                                                     c->d_wlc + ((K + 1) & 1));
  ++c->launches;
  CK(c, cudaGetLastError());
  if (plain_desc(c)) {
    describe(c, K + 1, c->d_wlc + ((K + 1) & 1), std::max(c->n_work, 1));
    CK(c, cudaGetLastError());
  }
  return ISING_SR_OK;
}

ising_sr_status launch_iteration(ising_sr_ctx* c) {
  NvtxRange nv("isr iteration");
  ++c->it;
  const unsigned K = ++c->Kglob;
  const bool first = c->it == 1;
  const bool all = first || (c->cfg.flags & ISING_SR_FLAG_JACOBI_ALL);  // Jacobi: every region, every iteration
  const int nw = all ? c->nreg : c->n_work;
  CK(c, cudaMemsetAsync(c->d_flags, 0, 4 * sizeof(int), c->stream));
  CK(c, cudaMemsetAsync(c->d_stats, 0, 8 * sizeof(unsigned long long), c->stream));
  CK(c, cudaMemsetAsync(c->d_wlc + ((K + 1) & 1), 0, sizeof(unsigned), c->stream));
  KArgs a = base_args(c, K, first);
  a.wl_in = all ? nullptr : c->wl[K & 1];
  a.desc = (!all && plain_desc(c)) ? c->desc : nullptr;
  a.n_work = nw;
  a.tile = tile_for(nw);
  a.wl_out = c->wl[(K + 1) & 1];
  a.wl_out_count = c->d_wlc + ((K + 1) & 1);
  CK(c, cudaEventRecord(c->kev0, c->stream));
  if (nw > 0) {
    c->ops->region(a, nw, c->stream);
    ++c->launches;
    CK(c, cudaGetLastError());
  }
  CK(c, cudaEventRecord(c->kev1, c->stream));
  if (c->ghost && c->peer) {
    return peer_exchange(c, a, c->d_flags);
  } else if (c->ghost) {
    c->ops->pack(a, c->gsend[0], c->gsend[1], c->RX, c->stream);
    ++c->launches;
    CK(c, cudaGetLastError());
  } else {
    return compact_worklist(c);
  }
  return ISING_SR_OK;
}

ising_sr_status mark_ghosts(ising_sr_ctx* c) {
  if (!c->ghost) return ISING_SR_OK;
  if (c->peer) return compact_worklist(c);  // the fused launch marked already
  const unsigned K = c->Kglob;
  KArgs a = base_args(c, K, c->it == 1);
  a.wl_out = c->wl[(K + 1) & 1];
  a.wl_out_count = c->d_wlc + ((K + 1) & 1);
  isr::mark_kernel<<<(2 * c->RX + 127) / 128, 128, 0, c->stream>>>(a, c->grecv[0], c->grecv[1]);
  ++c->launches;
  CK(c, cudaGetLastError());
  return compact_worklist(c);
}

// iteration `it` (1-based) of the window in progress
void account_iteration(ising_sr_ctx* c, float kms, const unsigned long long* s, int it) {
  const double ib = iteration_bytes(c, s);
  c->win_active[std::min(std::max(it, 1), 64) - 1] += (long long)s[5];
  c->stats.region_launches++;
  c->stats.region_ms += kms;
  c->stats.region_bytes += ib;
  c->stats.iterations_total++;
  c->stats.recomputations_total += (long long)s[5];
  c->win_bytes += ib;
  c->win_events += s[0];  // events of the recomputed regions (see commit)
  c->win_f = std::max(c->win_f, (int)s[4]);
}

ising_sr_status read_flags(ising_sr_ctx* c) {
  const unsigned K = c->Kglob;
  CK(c, cudaMemcpyAsync(c->h_flags, c->d_flags, 4 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaMemcpyAsync(c->h_stats, c->d_stats, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                        c->stream));
  CK(c, cudaMemcpyAsync(c->h_wlc, c->d_wlc + ((K + 1) & 1), sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  float kms = 0.f;
  CK(c, cudaEventElapsedTime(&kms, c->kev0, c->kev1));
  account_iteration(c, kms, c->h_stats, c->it);
  c->n_work = (int)c->h_wlc[0];
  return ISING_SR_OK;
}


void fill_halo(ising_sr_ctx* c, ising_sr_halo* h) {
  std::memset(h, 0, sizeof *h);
  h->nchunks = 4;
  for (int k = 0; k < 4; ++k) h->chunk_bytes[k] = c->gchunk[k];
  const GhostView* v[4] = {&c->gsend[0], &c->gsend[1], &c->grecv[0], &c->grecv[1]};
  void** dst[4] = {h->send_up, h->send_down, h->recv_from_up, h->recv_from_down};
  for (int i = 0; i < 4; ++i) {
    dst[i][0] = v[i]->cnt;
    dst[i][1] = v[i]->stamp;
    dst[i][2] = v[i]->t;
    dst[i][3] = v[i]->pos;
  }
  h->flags = c->d_flags;
  h->stream = (void*)c->stream;
  h->row_bytes = c->grow;
}

// C1 + C2 of one iteration on the ctx stream: my first row's
// north-edge histories to rank - 1 and my last row's south-edge histories to
// rank + 1 (periodic), the neighbours' into my ghost rows, in one NCCL group;
// then all-reduce(max) of the iteration's {changed, overflow}.  Per peer the
// sends and receives are matched in issue order (send up, send down; receive
// from down, receive from up), which pairs them correctly for world 1 (the
// loopback to itself), 2 (both neighbours are the other rank) and more.
ising_sr_status nccl_exchange(ising_sr_ctx* c, int* flags) {
  const isr_nccl::Api& A = isr_nccl::api();
  const int W = c->cfg.world, q = c->cfg.rank;
  const int up = (q + W - 1) % W, down = (q + 1) % W;
  bool ok = isr_nccl::report(A.GroupStart(), "ncclGroupStart");
  ok = ok && isr_nccl::report(A.Send(c->gsend[0].cnt, c->grow, isr_nccl::kInt8, up, c->nccl, c->stream), "ncclSend");
  ok = ok && isr_nccl::report(A.Send(c->gsend[1].cnt, c->grow, isr_nccl::kInt8, down, c->nccl, c->stream), "ncclSend");
  ok = ok && isr_nccl::report(A.Recv(c->grecv[1].cnt, c->grow, isr_nccl::kInt8, down, c->nccl, c->stream), "ncclRecv");
  ok = ok && isr_nccl::report(A.Recv(c->grecv[0].cnt, c->grow, isr_nccl::kInt8, up, c->nccl, c->stream), "ncclRecv");
  ok = isr_nccl::report(A.GroupEnd(), "ncclGroupEnd") && ok;
  ok = ok && isr_nccl::report(A.AllReduce(flags, flags, 2, isr_nccl::kInt32, isr_nccl::kMax, c->nccl, c->stream),
                              "ncclAllReduce");
  return ok ? ISING_SR_OK : ISING_SR_E_NCCL;
}

// ---------------------------------------------------------------------------
// Peer-memory exchange (isr_peer.cuh): the window of ghost rows + flag inbox
// (collective over the ranks: every rank allocates, registers and frees it at
// the same points -- init, capacity growth, destroy) and the fused launch.
// ---------------------------------------------------------------------------
#if ISR_HAVE_NCCL_DEVICE
void peer_free_rows(ising_sr_ctx* c) {
  const isr_nccl::Api& A = isr_nccl::api();
  if (c->pwin)
    ((ncclResult_t(*)(ncclComm_t, ncclWindow_t))A.CommWindowDeregister)((ncclComm_t)c->nccl, (ncclWindow_t)c->pwin);
  if (c->pbuf) ((ncclResult_t(*)(void*))A.MemFree)(c->pbuf);
  c->pwin = nullptr;
  c->pbuf = nullptr;
  c->pbytes = 0;
}

ising_sr_status peer_alloc_rows(ising_sr_ctx* c) {
  const isr_nccl::Api& A = isr_nccl::api();
  peer_free_rows(c);
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  isr::PeerArgs& p = c->pargs;
  p.row = c->grow;
  p.o_stamp = al(c->gchunk[0]);
  p.o_t = p.o_stamp + al(c->gchunk[1]);
  p.o_pos = p.o_t + al(c->gchunk[2]);
  p.o_inbox = 4 * c->grow;
  const size_t inbox = 2 * (size_t)isr::kPeerMaxWorld * 2 * sizeof(int);
  c->pbytes = (4 * c->grow + inbox + NCCL_WIN_REQUIRED_ALIGNMENT - 1) / NCCL_WIN_REQUIRED_ALIGNMENT *
              NCCL_WIN_REQUIRED_ALIGNMENT;
  if (!isr_nccl::report(((ncclResult_t(*)(void**, size_t))A.MemAlloc)(&c->pbuf, c->pbytes), "ncclMemAlloc")) {
    c->pbuf = nullptr;
    return ISING_SR_E_OOM;
  }
  // zeroed before the (collective) registration: no peer can store into it earlier
  CK(c, cudaMemsetAsync(c->pbuf, 0, c->pbytes, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  ncclWindow_t win = nullptr;
  if (!isr_nccl::report(((ncclResult_t(*)(ncclComm_t, void*, size_t, ncclWindow_t*, int))A.CommWindowRegister)(
                            (ncclComm_t)c->nccl, c->pbuf, c->pbytes, &win, NCCL_WIN_COLL_SYMMETRIC),
                        "ncclCommWindowRegister"))
    return ISING_SR_E_NCCL;
  c->pwin = win;
  isr::peer_bases_kernel<<<1, isr::kPeerMaxWorld + 1, 0, c->stream>>>(win, c->cfg.world, c->d_peer);
  CK(c, cudaGetLastError());
  CK(c, cudaMemcpyAsync(c->h_peer, c->d_peer, sizeof(unsigned long long) * (c->cfg.world + 1), cudaMemcpyDeviceToHost,
                        c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  p.peer = c->d_peer;
  p.mine = (char*)c->h_peer[c->cfg.world];
  p.rank = c->cfg.rank;
  p.world = c->cfg.world;
  return ISING_SR_OK;
}

void peer_teardown(ising_sr_ctx* c);

// after ncclCommInitRank: the peer path if this NCCL has the device API, every
// rank is load/store-reachable (one NVLink domain) and it was not switched off
ising_sr_status peer_setup(ising_sr_ctx* c) {
  const isr_nccl::Api& A = isr_nccl::api();
  const char* e = std::getenv("ISING_SR_EXCHANGE");  // sendrecv: never; peer: required (else E_NCCL)
  if (e && std::strcmp(e, "sendrecv") == 0) return ISING_SR_OK;
  const ising_sr_status unavailable = (e && std::strcmp(e, "peer") == 0) ? ISING_SR_E_NCCL : ISING_SR_OK;
  if (!A.MemAlloc || !A.MemFree || !A.CommWindowRegister || !A.CommWindowDeregister || !A.DevCommCreate ||
      !A.DevCommDestroy || !A.TeamLsa || c->cfg.world > isr::kPeerMaxWorld)
    return unavailable;
  const ncclTeam lsa = ((ncclTeam(*)(ncclComm_t))A.TeamLsa)((ncclComm_t)c->nccl);
  if (lsa.nRanks != c->cfg.world || lsa.rank != c->cfg.rank) return unavailable;  // not one NVLink domain
  c->peer_blocks = (c->RX + isr::kPeerThreads - 1) / isr::kPeerThreads;
  ncclDevCommRequirements req = {};
  req.lsaBarrierCount = c->peer_blocks;  // one barrier per block of the fused kernel
  // a failure from here on (no symmetric memory on this machine, ...) is the
  // same on every rank of one node: fall back to the send/recv transport
  // unless the peer one was asked for by name
  auto fallback = [&](const char* what) {
    std::fprintf(stderr, "ising_sr: peer-memory exchange unavailable (%s); using ncclSend/ncclRecv\n", what);
    peer_teardown(c);
    return unavailable;
  };
  if (!isr_nccl::report(((ncclResult_t(*)(ncclComm_t, const ncclDevCommRequirements*, ncclDevComm*))A.DevCommCreate)(
                            (ncclComm_t)c->nccl, &req, &c->dcomm),
                        "ncclDevCommCreate"))
    return fallback("ncclDevCommCreate");
  c->dcomm_ok = true;
  if (dmalloc(c, &c->d_peer, isr::kPeerMaxWorld + 1) != cudaSuccess) return ISING_SR_E_OOM;
  c->peer = true;
  const ising_sr_status s = peer_alloc_rows(c);
  if (s == ISING_SR_E_NCCL || s == ISING_SR_E_OOM) return fallback("symmetric window");
  return s;
}

void peer_teardown(ising_sr_ctx* c) {
  if (!c->nccl) return;
  peer_free_rows(c);
  if (c->dcomm_ok)
    ((ncclResult_t(*)(ncclComm_t, const ncclDevComm*))isr_nccl::api().DevCommDestroy)((ncclComm_t)c->nccl, &c->dcomm);
  c->dcomm_ok = false;
  c->peer = false;
}

// pack into the neighbours' rows + flags + barrier + mark, one launch
ising_sr_status peer_exchange(ising_sr_ctx* c, const KArgs& a, int* flags) {
  const auto x0 = std::chrono::steady_clock::now();
  isr::PeerArgs p = c->pargs;
  p.flags = flags;
  if (c->ops->warp)
    isr::xchg_kernel<true><<<c->peer_blocks, isr::kPeerThreads, 0, c->stream>>>(a, p, c->dcomm);
  else
    isr::xchg_kernel<false><<<c->peer_blocks, isr::kPeerThreads, 0, c->stream>>>(a, p, c->dcomm);
  ++c->launches;
  CK(c, cudaGetLastError());
  c->stats.ms_exchange_total +=
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - x0).count();
  return ISING_SR_OK;
}
#else
ising_sr_status peer_setup(ising_sr_ctx*) {
  const char* e = std::getenv("ISING_SR_EXCHANGE");
  return (e && std::strcmp(e, "peer") == 0) ? ISING_SR_E_NCCL : ISING_SR_OK;
}
void peer_teardown(ising_sr_ctx*) {}
ising_sr_status peer_alloc_rows(ising_sr_ctx*) { return ISING_SR_E_NCCL; }
ising_sr_status peer_exchange(ising_sr_ctx*, const KArgs&, int*) { return ISING_SR_E_NCCL; }
#endif

// the exchange of one iteration (after K1 and pack): the library's NCCL
// communicator, or the caller's callback (which must order its work on the
// ctx stream); `flags` = the iteration's device {changed, overflow}
ising_sr_status exchange(ising_sr_ctx* c, int* flags) {
  if (!c->ghost || c->peer) return ISING_SR_OK;  // (peer: done by the fused launch)
  const auto x0 = std::chrono::steady_clock::now();
  ising_sr_status s = ISING_SR_OK;
  if (c->nccl) {
    s = nccl_exchange(c, flags);
  } else if (c->cfg.exchange) {
    ising_sr_halo h;
    fill_halo(c, &h);
    h.flags = flags;
    if (c->cfg.exchange(c->cfg.exchange_user, &h) != 0) s = ISING_SR_E_NCCL;
  } else {
    s = ISING_SR_E_INVALID_ARG;
  }
  c->stats.ms_exchange_total +=
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - x0).count();
  return s;
}

// {M, B} of committed state st into c->h_snap (enqueued; read after the next sync)
ising_sr_status enqueue_snapshot(ising_sr_ctx* c, const StateView& st) {
  CK(c, cudaMemsetAsync(c->d_snap, 0, 2 * sizeof(unsigned long long), c->stream));
  c->ops->snap(st, c->nreg, c->RX, c->RYg, c->d_snap, c->stream);
  ++c->launches;
  CK(c, cudaGetLastError());
  CK(c, cudaMemcpyAsync(c->h_snap, c->d_snap, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
  return ISING_SR_OK;
}

ising_sr_status grow_capacity(ising_sr_ctx* c) {
  if (c->K >= c->ops->cnt_max) return ISING_SR_E_CAPACITY;
  const int K = std::min(c->ops->cnt_max, c->K * 2);
  ising_sr_status s = alloc_edges(c, K);
  if (s != ISING_SR_OK) return s;
  if (c->peer && (s = peer_alloc_rows(c)) != ISING_SR_OK) return s;
  c->stats.overflow_retries++;
  c->stats.hist_capacity = K;
  return ISING_SR_OK;
}

void start_window(ising_sr_ctx* c) {
  c->t_c = (double)c->w * c->cfg.W;
  const double next = (double)(c->w + 1) * c->cfg.W;
  c->t_w = next < c->cfg.t_end ? next : c->cfg.t_end;
  c->it = 0;
  c->K0 = c->Kglob + 1;  // every selector stamp < K0 now reads as "empty"
  c->n_work = c->nreg;
  c->in_window = true;
  c->converged = false;
  c->g = 0;
  c->win_events = 0;
  c->win_bytes = 0.0;
  c->win_f = 0;
  std::memset(c->win_active, 0, sizeof c->win_active);
}

// ---------------------------------------------------------------------------
// Pipelined relaxation (worklist schedule, any world size): iteration k+1
// is enqueued before the host reads iteration k's flags, so the host round
// trip overlaps the GPU's work.  K1 reads the length of its worklist on the
// device (n_work_dev); its grid is sized from an upper bound -- the length of
// iteration k+1's worklist is known once iteration k's results are back, and
// worklists shrink as the relaxation converges (a longer one only enlarges
// each block's tile).  When iteration k changed nothing, the iteration
// enqueued after it finds an empty worklist and does nothing, so g and every
// result are those of the one-iteration-per-sync loop.  Per-iteration flags,
// counters and kernel events use slot K & 1.  With strips, every rank
// enqueues the same iterations (its decisions use all-reduced flags), so the
// speculative iteration's exchange is matched on every rank.
// ---------------------------------------------------------------------------
ising_sr_status enqueue_pipelined(ising_sr_ctx* c, int bound) {
  NvtxRange nv("isr iteration (pipelined)");
  ++c->it;
  const unsigned K = ++c->Kglob;
  const int j = (int)(K & 1u);
  const bool first = c->it == 1;
  const int nb = first ? c->nreg : bound;
  IterSlot* sl = c->d_slot + j;             // this iteration's flags, counters, next worklist length
  const IterSlot* prev = c->d_slot + (j ^ 1);  // ... the previous one's: this worklist's length
  CK(c, cudaMemsetAsync(sl, 0, sizeof(IterSlot), c->stream));
  KArgs a = base_args(c, K, first);
  a.flags = sl->flags;
  a.stats = sl->stats;
  a.wl_in = first ? nullptr : c->wl[K & 1];
  a.desc = (!first && plain_desc(c)) ? c->desc : nullptr;
  a.n_work = nb;
  a.n_work_dev = first ? nullptr : &prev->wl_next;
  a.tile = tile_for(std::max(nb, 1));
  a.wl_out = c->wl[(K + 1) & 1];
  a.wl_out_count = &sl->wl_next;
  CK(c, cudaEventRecord(c->bev[2 * j], c->stream));
  if (nb > 0) {
    c->ops->region(a, nb, c->stream);
    ++c->launches;
    CK(c, cudaGetLastError());
  }
  CK(c, cudaEventRecord(c->bev[2 * j + 1], c->stream));
  if (c->ghost && c->peer) {  // strip edges: one fused launch over peer memory
    ising_sr_status s = peer_exchange(c, a, sl->flags);
    if (s) return s;
  } else if (c->ghost) {  // strip edges: pack, C1 + C2, mark the regions next to changed ghosts
    c->ops->pack(a, c->gsend[0], c->gsend[1], c->RX, c->stream);
    ++c->launches;
    CK(c, cudaGetLastError());
    ising_sr_status s = exchange(c, sl->flags);
    if (s) return s;
    isr::mark_kernel<<<(2 * c->RX + 127) / 128, 128, 0, c->stream>>>(a, c->grecv[0], c->grecv[1]);
    ++c->launches;
    CK(c, cudaGetLastError());
  }
  isr::compact_kernel<<<compact_grid(c), isr::kCompactThreads, 0, c->stream>>>(c->dirty + (size_t)((K + 1) & 1) * c->dwords,
                                                                       c->dwords, c->nreg, c->wl[(K + 1) & 1],
                                                                       &sl->wl_next);
  ++c->launches;
  CK(c, cudaGetLastError());
  if (plain_desc(c)) {  // descriptors of iteration K + 1's worklist
    describe(c, K + 1, &sl->wl_next, nb);
    CK(c, cudaGetLastError());
  }
  CK(c, cudaMemcpyAsync(c->h_slot + j, sl, sizeof(IterSlot), cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaEventRecord(c->pev[j], c->stream));
  return ISING_SR_OK;
}

ising_sr_status run_window_pipelined(ising_sr_ctx* c) {
  ising_sr_status s;
  int bound = c->nreg;
  if ((s = enqueue_pipelined(c, bound))) return s;  // iteration 1: every region
  for (;;) {
    const int k = c->it;                 // the iteration whose results are read next
    const unsigned Kk = c->Kglob;
    const int j = (int)(Kk & 1u);
    const bool ahead = k < c->cfg.max_iterations;
    if (ahead && (s = enqueue_pipelined(c, bound))) return s;  // iteration k+1, speculative
    CK(c, cudaEventSynchronize(c->pev[j]));
    float kms = 0.f;
    CK(c, cudaEventElapsedTime(&kms, c->bev[2 * j], c->bev[2 * j + 1]));
    account_iteration(c, kms, c->h_slot[j].stats, k);
    const int* f = c->h_slot[j].flags;
    if (f[1]) {  // history capacity overflow: drain, forget the speculative iteration, grow, restart
      CK(c, cudaStreamSynchronize(c->stream));
      CK(c, cudaMemsetAsync(c->dirty, 0, 2 * (size_t)c->dwords * sizeof(uint32_t), c->stream));
      if ((s = grow_capacity(c))) return s;
      start_window(c);
      bound = c->nreg;
      if ((s = enqueue_pipelined(c, bound))) return s;
      continue;
    }
    if (!f[0]) {  // converged at k; the iteration enqueued after it is a no-op
      c->converged = true;
      c->g = k;
      c->it = k;
      return ISING_SR_OK;
    }
    if (!ahead) {
      CK(c, cudaStreamSynchronize(c->stream));
      c->in_window = false;
      return ISING_SR_E_DIVERGED;
    }
    bound = (int)c->h_slot[j].wl_next;  // length of iteration k+1's worklist: the bound for k+2
    c->n_work = bound;
  }
}

// ---------------------------------------------------------------------------
// Device-side window loop (ISING_SR_GRAPH=1; world 1): the whole relaxation of a window
// is one CUDA graph -- iteration 1 (the canonical assumption) followed by a
// conditional while node whose body runs two iterations, each K1 [+ pack,
// NCCL send/recv, all-reduce, mark] + worklist compaction + an advance kernel
// that accounts the iteration and decides whether to go on.  The body's two
// iterations have fixed parities, so every pointer is fixed at capture; a
// kernel's iteration stamp is it_K + 2 * trip with trip counted on the
// device.  No host round trip per iteration; one synchronisation per window.
// An iteration after the converged one (the body's second half) finds an
// empty worklist and changes nothing, so g and every result are those of the
// host loops.
// ---------------------------------------------------------------------------
ising_sr_status capture_iteration(ising_sr_ctx* c, unsigned K, bool first, const unsigned* trip,
                                  cudaGraphConditionalHandle h, int set_cond, int end_of_trip) {
  const int j = (int)(K & 1u);
  IterSlot* sl = c->d_slot + j;
  IterSlot* prev = c->d_slot + (j ^ 1);
  KArgs a = base_args(c, K, first);
  a.trip = trip;
  a.ktime = sl->ktime;
  a.flags = sl->flags;
  a.stats = sl->stats;
  a.wl_in = first ? nullptr : c->wl[K & 1];
  a.n_work = c->nreg;
  a.n_work_dev = first ? nullptr : &prev->wl_next;
  a.tile = tile_for(c->nreg);
  a.wl_out = c->wl[(K + 1) & 1];
  a.wl_out_count = &sl->wl_next;
  c->ops->region(a, c->nreg, c->stream);
  CK(c, cudaGetLastError());
  if (c->ghost && c->peer) {
    ising_sr_status s = peer_exchange(c, a, sl->flags);
    if (s) return s;
  } else if (c->ghost) {
    c->ops->pack(a, c->gsend[0], c->gsend[1], c->RX, c->stream);
    CK(c, cudaGetLastError());
    ising_sr_status s = nccl_exchange(c, sl->flags);
    if (s) return s;
    isr::mark_kernel<<<(2 * c->RX + 127) / 128, 128, 0, c->stream>>>(a, c->grecv[0], c->grecv[1]);
    CK(c, cudaGetLastError());
  }
  isr::compact_kernel<<<compact_grid(c), isr::kCompactThreads, 0, c->stream>>>(
      c->dirty + (size_t)((K + 1) & 1) * c->dwords, c->dwords, c->nreg, c->wl[(K + 1) & 1], &sl->wl_next);
  CK(c, cudaGetLastError());
  advance_kernel<<<1, 32, 0, c->stream>>>(c->d_win, sl, prev, c->cfg.max_iterations, h, set_cond, end_of_trip);
  CK(c, cudaGetLastError());
  return ISING_SR_OK;
}

ising_sr_status build_window_graph(ising_sr_ctx* c, cudaGraphExec_t* exec) {
  const unsigned K0 = c->Kglob + 1;  // iteration 1's stamp (== c->K0)
  cudaGraph_t g = nullptr;
  CK(c, cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  cudaError_t e = cudaGraphConditionalHandleCreate(&h, g, 1u, cudaGraphCondAssignDefault);
  const cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  std::vector<cudaGraphNode_t> leaf;
  ising_sr_status st = ISING_SR_OK;
  // prefix: reset the window's accumulators and iteration 1's slot, iteration 1
  if (e == cudaSuccess) e = cudaStreamBeginCaptureToGraph(c->stream, g, nullptr, nullptr, 0, mode);
  if (e == cudaSuccess) {
    cudaMemsetAsync(c->d_win, 0, sizeof(WinDev), c->stream);
    slot_reset<<<1, 32, 0, c->stream>>>(c->d_slot + (K0 & 1u));
    st = capture_iteration(c, K0, true, nullptr, h, 1, 0);
    cudaStreamCaptureStatus cs;
    if (cudaStreamGetCaptureInfo(c->stream, &cs, nullptr, nullptr, &deps, &ndeps) == cudaSuccess)
      leaf.assign(deps, deps + ndeps);
    cudaGraph_t gg = nullptr;
    e = cudaStreamEndCapture(c->stream, &gg);
  }
  // the loop: while (changed) { iteration K0 + 1 + 2 trip; iteration K0 + 2 + 2 trip }
  cudaGraph_t body = nullptr;
  if (e == cudaSuccess && st == ISING_SR_OK) {
    alignas(cudaGraphNodeParams) unsigned char pbuf[sizeof(cudaGraphNodeParams)];
    std::memset(pbuf, 0, sizeof pbuf);  // (the struct's union has no default constructor)
    cudaGraphNodeParams& p = *reinterpret_cast<cudaGraphNodeParams*>(pbuf);
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t cn;
    e = cudaGraphAddNode(&cn, g, leaf.data(), leaf.size(), &p);
    if (e == cudaSuccess) body = p.conditional.phGraph_out[0];
  }
  if (e == cudaSuccess && st == ISING_SR_OK) {
    e = cudaStreamBeginCaptureToGraph(c->stream, body, nullptr, nullptr, 0, mode);
    if (e == cudaSuccess) {
      st = capture_iteration(c, K0 + 1, false, &c->d_win->trip, h, 0, 0);
      if (st == ISING_SR_OK) st = capture_iteration(c, K0 + 2, false, &c->d_win->trip, h, 1, 1);
      cudaGraph_t bb = nullptr;
      const cudaError_t e2 = cudaStreamEndCapture(c->stream, &bb);
      if (e == cudaSuccess) e = e2;
    }
  }
  if (e == cudaSuccess && st == ISING_SR_OK) e = cudaGraphInstantiate(exec, g, 0);
  cudaGraphDestroy(g);
  if (st != ISING_SR_OK) return st;
  return fail_cuda(c, e, "build_window_graph");
}

ising_sr_status run_window_graph(ising_sr_ctx* c) {
  for (;;) {
    const unsigned K0 = c->Kglob + 1;
    cudaGraphExec_t exec = nullptr;
    ising_sr_status s = build_window_graph(c, &exec);
    if (s) return s;
    cudaError_t e = cudaGraphLaunch(exec, c->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(c->h_win, c->d_win, sizeof(WinDev), cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    cudaGraphExecDestroy(exec);
    CK(c, e);
    const WinDev& w = *c->h_win;
    // every launch of the graph: iteration 1 and two per loop trip
    const int launched = 1 + 2 * (int)w.trip;
    c->Kglob = K0 + 2 * w.trip;
    c->launches += (long long)launched * (c->ghost ? (c->peer ? 3 : 4) : 2) + launched + 2;
    const double S = (double)c->ops->spin_bytes + (double)c->ops->halo_bytes + 8 + 8 + 4 +
                     ((c->cfg.flags & ISING_SR_FLAG_DIGEST) ? 8 : 0);
    const double ib = (double)w.s5 * (2.0 * S + c->ops->sel_read_bytes + 8.0) + 9.0 * ((double)w.s1 + (double)w.s2 + (double)w.s3);
    for (int k = 0; k < 64; ++k) c->win_active[k] += (long long)w.active[k];
    c->stats.region_launches += launched;
    c->stats.region_ms += (double)w.k1_ns * 1e-6;
    c->stats.region_bytes += ib;
    c->stats.iterations_total += w.it;
    c->stats.recomputations_total += (long long)w.s5;
    c->win_bytes += ib;
    c->win_events += w.ev;
    c->win_f = std::max(c->win_f, (int)w.fmax);
    if (w.overflow) {  // history capacity overflow: grow and restart the window
      CK(c, cudaMemsetAsync(c->dirty, 0, 2 * (size_t)c->dwords * sizeof(uint32_t), c->stream));
      if ((s = grow_capacity(c))) return s;
      start_window(c);
      continue;
    }
    if (!w.g) {
      c->in_window = false;
      return ISING_SR_E_DIVERGED;
    }
    c->converged = true;
    c->g = w.g;
    c->it = w.g;
    return ISING_SR_OK;
  }
}

// FLAG_MAG_MOMENTS: the window's int |M| dt and int M^2 dt into c->h_mm
// (enqueued; read after the commit's synchronisation).  n = events of the
// window (the log is complete on the stream).
ising_sr_status mag_moments(ising_sr_ctx* c, long long n) {
  int B = 1024;
  while (B < (1 << 22) && (long long)B * 16 < n) B <<= 1;
  if (B > c->mm_B) {
    dfree(c, c->mm_cnt);
    c->mm_cnt = nullptr;
    if (dmalloc(c, &c->mm_cnt, 3 * (size_t)B + 1) != cudaSuccess) return ISING_SR_E_OOM;
    c->mm_B = B;
  }
  if (!c->mm_csum && (dmalloc(c, &c->mm_csum, kMmBlocks) != cudaSuccess ||
                      dmalloc(c, &c->mm_part, 2 * kMmBlocks + 2) != cudaSuccess))
    return ISING_SR_E_OOM;
  unsigned* cnt = c->mm_cnt;
  unsigned* fill = cnt + B;
  unsigned* off = cnt + 2 * B;
  CK(c, cudaMemsetAsync(cnt, 0, 2 * (size_t)B * sizeof(unsigned), c->stream));
  const double scale = (double)B / (c->t_w - c->t_c);
  mm_count<<<148 * 4, 256, 0, c->stream>>>(c->log_t, c->d_total, c->t_c, scale, B, cnt);
  mm_scan_buckets<<<1, 1024, 0, c->stream>>>(cnt, B, off);
  mm_scatter<<<148 * 4, 256, 0, c->stream>>>(c->log_t, c->log_dm, c->d_total, c->t_c, scale, B, off, fill, c->mm_ts,
                                             c->mm_dm);
  mm_sort_buckets<<<(B + 255) / 256, 256, 0, c->stream>>>(off, B, c->mm_ts, c->mm_dm);
  mm_chunk_sums<<<kMmBlocks, 256, 0, c->stream>>>(c->mm_dm, c->d_total, c->mm_csum);
  mm_integrate<<<kMmBlocks, 256, 0, c->stream>>>(c->mm_ts, c->mm_dm, c->d_total, c->mm_csum, c->d_snap, c->t_w,
                                                 c->mm_part);
  mm_final<<<1, 1024, 0, c->stream>>>(c->mm_part, c->mm_ts, c->d_total, c->d_snap, c->t_c, c->t_w,
                                      c->mm_part + 2 * kMmBlocks);
  c->launches += 7;
  CK(c, cudaGetLastError());
  CK(c, cudaMemcpyAsync(c->h_mm, c->mm_part + 2 * kMmBlocks, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  (void)n;
  return ISING_SR_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

const char* ising_sr_strerror(ising_sr_status s) {
  switch (s) {
    case ISING_SR_OK: return "ok";
    case ISING_SR_E_INVALID_ARG: return "invalid argument";
    case ISING_SR_E_DIMENSION: return "invalid dimension (Lx, Ly >= 3 required)";
    case ISING_SR_E_PARTITION: return "partition error (region size / strips must divide the lattice)";
    case ISING_SR_E_DIVERGED: return "relaxation did not converge within max_iterations";
    case ISING_SR_E_CAPACITY: return "boundary-history capacity exhausted";
    case ISING_SR_E_CUDA: return "CUDA error";
    case ISING_SR_E_NCCL: return "halo exchange failed (NCCL or the exchange callback)";
    case ISING_SR_E_OOM: return "device out of memory";
    case ISING_SR_E_STATE: return "call out of order";
  }
  return "unknown status";
}

void ising_sr_destroy(ising_sr_ctx* c) {
  if (!c) return;
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& s : c->st) {
    dfree(c, s.spins);
    dfree(c, s.halo);
    dfree(c, s.ts);
    dfree(c, s.R);
    dfree(c, s.n);
    dfree(c, s.dig);
    dfree(c, s.oM);
    dfree(c, s.oB);
  }
  free_edges(c);
  dfree(c, c->sel);
  dfree(c, c->dirty);
  dfree(c, c->lg_tR);
  dfree(c, c->lg_c);
  dfree(c, c->lg_meta);
  dfree(c, c->pcache);
  dfree(c, c->pmeta);
  dfree(c, c->wl[0]);
  dfree(c, c->wl[1]);
  dfree(c, c->d_wlc);
  dfree(c, c->d_flags);
  dfree(c, c->d_stats);
  dfree(c, c->ev_t);
  dfree(c, c->ev_s);
  dfree(c, c->desc);
  dfree(c, c->log_dm);
  dfree(c, c->mm_ts);
  dfree(c, c->mm_dm);
  dfree(c, c->mm_cnt);
  dfree(c, c->mm_csum);
  dfree(c, c->mm_part);
  dfree(c, c->d_replay);
  dfree(c, c->d_nrep);
  dfree(c, c->d_edges);
  if (c->cev0) cudaEventDestroy(c->cev0);
  if (c->cev1) cudaEventDestroy(c->cev1);
  peer_teardown(c);
  dfree(c, c->d_peer);
  if (c->nccl) isr_nccl::api().CommDestroy(c->nccl);
  for (auto& e : c->bev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->pev)
    if (e) cudaEventDestroy(e);
  cudaFreeHost(c->h_flags);
  cudaFreeHost(c->h_stats);
  cudaFreeHost(c->h_wlc);
  dfree(c, c->d_slot);
  dfree(c, c->d_win);
  if (c->h_win) cudaFreeHost(c->h_win);
  dfree(c, c->d_snap);
  cudaFreeHost(c->h_slot);
  dfree(c, c->log_t);
  dfree(c, c->log_region);
  dfree(c, c->log_site);
  dfree(c, c->d_off);
  dfree(c, c->d_bsum);
  dfree(c, c->d_total);
  dfree(c, c->d_obs);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->kev0) cudaEventDestroy(c->kev0);
  if (c->kev1) cudaEventDestroy(c->kev1);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

ising_sr_status ising_sr_nccl_unique_id(void* out) {
  if (!out) return ISING_SR_E_INVALID_ARG;
  const isr_nccl::Api& A = isr_nccl::api();
  if (!A.ok) return ISING_SR_E_NCCL;
  isr_nccl::UniqueId id;
  if (!isr_nccl::report(A.GetUniqueId(&id), "ncclGetUniqueId")) return ISING_SR_E_NCCL;
  std::memcpy(out, &id, sizeof id);
  return ISING_SR_OK;
}

ising_sr_status ising_sr_init(const ising_sr_config* cfg, const uint8_t* spins, ising_sr_ctx** out) {
  if (!cfg || !out) return ISING_SR_E_INVALID_ARG;
  *out = nullptr;
  if (cfg->Lx < 3 || cfg->Ly < 3) return ISING_SR_E_DIMENSION;
  if (cfg->bx < 1 || cfg->by < 1 || cfg->Lx % cfg->bx || cfg->Ly % cfg->by) return ISING_SR_E_PARTITION;
  if (std::isnan(cfg->W) || std::isinf(cfg->W) || !(cfg->t_end >= 0.0)) return ISING_SR_E_INVALID_ARG;
  for (double r : cfg->rate)
    if (!(r >= 0.0) || std::isinf(r)) return ISING_SR_E_INVALID_ARG;
  const int world = cfg->world < 1 ? 1 : cfg->world;
  if (cfg->rank < 0 || cfg->rank >= world) return ISING_SR_E_INVALID_ARG;
  const ShapeOps* ops = find_ops(cfg->bx, cfg->by);
  if (!ops) return ISING_SR_E_INVALID_ARG;
  const int RX = cfg->Lx / cfg->bx, RY = cfg->Ly / cfg->by;
  if (RY % world) return ISING_SR_E_PARTITION;
  if ((long long)RX * RY > 0x7fffffffLL) return ISING_SR_E_INVALID_ARG;
  const bool loopback = (cfg->flags & ISING_SR_FLAG_HALO_LOOPBACK) != 0;
  if ((cfg->flags & ISING_SR_FLAG_MAG_MOMENTS) && world != 1) return ISING_SR_E_INVALID_ARG;  // needs the global order
  if (loopback && (world != 1 || !cfg->nccl_id)) return ISING_SR_E_INVALID_ARG;
  if (world > 1 && !cfg->nccl_id && !cfg->exchange) {
    // only the step-level API can drive such a ctx (the caller moves the ghost rows)
  }
  if (!(cfg->eq_quantum >= 0.0) || std::isinf(cfg->eq_quantum)) return ISING_SR_E_INVALID_ARG;

  ising_sr_ctx* c = new (std::nothrow) ising_sr_ctx();
  if (!c) return ISING_SR_E_OOM;
  c->cfg = *cfg;
  c->cfg.world = world;
  if (c->cfg.flags & ISING_SR_FLAG_MAG_MOMENTS) c->cfg.flags |= ISING_SR_FLAG_LOG_EVENTS | ISING_SR_FLAG_OBSERVABLES;
  if (!(cfg->W > 0.0)) {  // the paper's T_max = ln N / (lambda |dG_i|)
    double lam = 0.0;
    for (double r : cfg->rate) lam = std::max(lam, r);
    const double N = (double)RX * (double)RY;
    const double dG = (cfg->bx == 1 || cfg->by == 1) ? (double)cfg->bx * cfg->by : 2.0 * (cfg->bx + cfg->by) - 4.0;
    c->cfg.W = (N > 1.0 && lam > 0.0) ? std::log(N) / (lam * dG) : 1.0;
  }
  c->cfg.nccl_id = nullptr;  // copied into the communicator below, never kept
  c->ghost = world > 1 || loopback;
  if (c->cfg.max_iterations <= 0) c->cfg.max_iterations = 1000;
  c->ops = ops;
  c->RX = RX;
  c->RYg = RY;
  c->RYl = RY / world;
  c->row0 = cfg->rank * c->RYl;
  c->nreg = c->RX * c->RYl;
  c->dwords = ((c->nreg + 31) / 32 + 7) / 8 * 8;  // a multiple of 8 words: 32-byte aligned bitmaps (compact_kernel)
  std::memset(&c->stats, 0, sizeof c->stats);
  if (const char* e = std::getenv("ISING_SR_PIPELINE")) c->pipeline = std::atoi(e) != 0;
  if (const char* e = std::getenv("ISING_SR_PLAIN")) c->plain = std::atoi(e) != 0;
  if (const char* e = std::getenv("ISING_SR_LANE_SPREAD")) c->lane_spread = std::max(0, std::min(5, std::atoi(e)));
  if (const char* e = std::getenv("ISING_SR_REFILL")) c->refill = std::max(1, std::min(32, std::atoi(e)));
  if (const char* e = std::getenv("ISING_SR_K1_DELAY_NS")) c->delay_ns = (unsigned)std::max(0, std::atoi(e));
  if (const char* e = std::getenv("ISING_SR_GRAPH")) c->graph = std::atoi(e) != 0;
  if ((c->cfg.flags & ISING_SR_FLAG_OBSERVABLES) && ops->warp && !big_enabled()) {
    delete c;
    return ISING_SR_E_INVALID_ARG;  // observables are accumulated by the lane-per-region K1 forms only
  }

  auto bail = [&](ising_sr_status s) {
    ising_sr_destroy(c);
    return s;
  };
  if (cudaSetDevice(cfg->device) != cudaSuccess) return bail(ISING_SR_E_CUDA);
  if (cfg->stream) {
    c->stream = (cudaStream_t)cfg->stream;
  } else {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) return bail(ISING_SR_E_CUDA);
    c->own_stream = true;
  }
  const size_t n = (size_t)c->nreg;
  for (auto& s : c->st) {
    if (dmalloc_bytes(c, (void**)&s.spins, n * ops->spin_bytes) != cudaSuccess ||
        dmalloc_bytes(c, (void**)&s.halo, n * ops->halo_bytes) != cudaSuccess || dmalloc(c, &s.ts, n) != cudaSuccess ||
        dmalloc(c, &s.R, n) != cudaSuccess || dmalloc(c, &s.n, n) != cudaSuccess || dmalloc(c, &s.dig, n) != cudaSuccess)
      return bail(ISING_SR_E_OOM);
    if ((c->cfg.flags & ISING_SR_FLAG_OBSERVABLES) &&
        (dmalloc(c, &s.oM, n) != cudaSuccess || dmalloc(c, &s.oB, n) != cudaSuccess))
      return bail(ISING_SR_E_OOM);
  }
  if (dmalloc(c, &c->sel, (size_t)ops->sel_words * n) != cudaSuccess || dmalloc(c, &c->dirty, 2 * (size_t)c->dwords) != cudaSuccess ||
      dmalloc(c, &c->wl[0], n) != cudaSuccess || dmalloc(c, &c->wl[1], n) != cudaSuccess ||
      dmalloc(c, &c->d_wlc, 2) != cudaSuccess || dmalloc(c, &c->d_flags, 4) != cudaSuccess ||
      dmalloc(c, &c->d_stats, 8) != cudaSuccess || dmalloc(c, &c->d_nrep, 4) != cudaSuccess ||
      dmalloc(c, &c->d_edges, 1) != cudaSuccess ||
      cudaMallocHost((void**)&c->h_flags, 4 * sizeof(int)) != cudaSuccess ||
      cudaMallocHost((void**)&c->h_stats, 8 * sizeof(unsigned long long)) != cudaSuccess ||
      cudaMallocHost((void**)&c->h_wlc, 2 * sizeof(unsigned)) != cudaSuccess ||
      dmalloc(c, &c->d_off, n) != cudaSuccess || dmalloc(c, &c->d_bsum, (n + kThreads - 1) / kThreads) != cudaSuccess ||
      dmalloc(c, &c->d_total, 1) != cudaSuccess || dmalloc(c, &c->d_obs, 2 * kObsBlocks + 2) != cudaSuccess ||
      dmalloc(c, &c->d_slot, 2) != cudaSuccess || dmalloc(c, &c->d_snap, 2) != cudaSuccess ||
      dmalloc(c, &c->d_win, 1) != cudaSuccess || cudaMallocHost((void**)&c->h_win, sizeof(WinDev)) != cudaSuccess ||
      cudaMallocHost((void**)&c->h_slot, 2 * sizeof(IterSlot)) != cudaSuccess)
    return bail(ISING_SR_E_OOM);
  if (!ops->warp && dmalloc(c, &c->desc, n) != cudaSuccess) return bail(ISING_SR_E_OOM);
  if (cudaMemsetAsync(c->sel, 0, n * 8 * (size_t)ops->sel_words, c->stream) != cudaSuccess ||
      cudaMemsetAsync(c->dirty, 0, 2 * (size_t)c->dwords * 4, c->stream) != cudaSuccess)
    return bail(ISING_SR_E_CUDA);
  if (cudaEventCreate(&c->ev0) != cudaSuccess || cudaEventCreate(&c->ev1) != cudaSuccess ||
      cudaEventCreate(&c->kev0) != cudaSuccess || cudaEventCreate(&c->kev1) != cudaSuccess ||
      cudaEventCreate(&c->cev0) != cudaSuccess || cudaEventCreate(&c->cev1) != cudaSuccess)
    return bail(ISING_SR_E_CUDA);
  for (auto& e : c->bev)
    if (cudaEventCreate(&e) != cudaSuccess) return bail(ISING_SR_E_CUDA);
  for (auto& e : c->pev)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return bail(ISING_SR_E_CUDA);
  if (c->cfg.flags & ISING_SR_FLAG_LOG_EVENTS) {
    // scratch event log: 1.5 x the expected events per region per window at
    // the largest rate + 8, within 8 GB in all (a region with more events is
    // replayed at commit -- a latency-bound K1 pass, so it should be rare)
    double rmax = 0.0;
    for (double r : cfg->rate) rmax = std::max(rmax, r);
    const double mu = (double)cfg->bx * cfg->by * rmax * std::min(c->cfg.W, std::max(cfg->t_end, 1e-9));
    long long C = cfg->log_capacity > 0 ? cfg->log_capacity : (long long)std::ceil(1.5 * mu) + 8;
    C = std::min<long long>(C, 65535);
    if (cfg->log_capacity <= 0) C = std::max<long long>(2, std::min<long long>(C, (8LL << 30) / (10LL * std::max(1, c->nreg))));
    c->evC = (int)C;
    if (dmalloc(c, &c->ev_t, n * (size_t)C) != cudaSuccess || dmalloc(c, &c->ev_s, n * (size_t)C) != cudaSuccess ||
        dmalloc(c, &c->d_replay, n) != cudaSuccess)
      return bail(ISING_SR_E_OOM);
  }
  int K0 = cfg->hist_capacity > 0 ? std::min(cfg->hist_capacity, ops->cnt_max) : auto_capacity(c->cfg, ops->cnt_max);
  if (cfg->hist_capacity <= 0) {
    // the automatic capacity never takes more than 60 % of the free device
    // memory for the two history slots (4 edges x K entries x 9 bytes per
    // region each); a longer history is caught by the overflow retry
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) == cudaSuccess && fr > 0) {
      const double per_k = 2.0 * (ops->single_edge ? 1.0 : 4.0) * (double)c->nreg * 9.0;
      const int kmax = (int)std::max(2.0, 0.6 * (double)fr / per_k);
      K0 = std::min(K0, kmax);
    }
  }
  ising_sr_status s = alloc_edges(c, K0);
  if (s != ISING_SR_OK) return bail(s);
  if (const char* e = std::getenv("ISING_SR_RESUME")) c->resume = std::atoi(e) != 0;
  if (ops->warp && big_enabled() && c->resume) {
    // step log per region: incoming break points (<= 4 K) + events (twice the
    // expectation at the largest rate) + slack; capped at 48 GB in all (a
    // region whose log overflows is simply recomputed in full)
    double rmax = 0.0;
    for (double r : cfg->rate) rmax = std::max(rmax, r);
    long long LC = 4LL * K0 + 2LL * (long long)std::ceil((double)cfg->bx * cfg->by * cfg->W * rmax) + 64;
    LC = std::min<long long>(LC, 32768);
    const long long cap = (48LL << 30) / (18LL * std::max(1, c->nreg));
    LC = std::min(LC, cap);
    if (LC >= 16) {
      c->LC = (int)LC;
      const size_t nl = (size_t)c->nreg * (size_t)LC;
      if (dmalloc(c, &c->lg_tR, nl) != cudaSuccess || dmalloc(c, &c->lg_c, nl) != cudaSuccess ||
          dmalloc(c, &c->lg_meta, n) != cudaSuccess) {
        cudaGetLastError();
        dfree(c, c->lg_tR); dfree(c, c->lg_c); dfree(c, c->lg_meta);
        c->lg_tR = nullptr; c->lg_c = nullptr; c->lg_meta = nullptr;
        c->LC = 0;
      } else if (cudaMemsetAsync(c->lg_meta, 0, n * sizeof(uint2), c->stream) != cudaSuccess) {
        return bail(ISING_SR_E_CUDA);
      }
    }
  }
  bool pcache_on = true;
  if (const char* e = std::getenv("ISING_SR_PCACHE")) pcache_on = std::atoi(e) != 0;
  if (ops->warp && big_enabled() && pcache_on) {
    // the window's pairs per region: 1.25 x the expected events at the
    // largest rate + slack, capped at 8192 and at 24 GB in all (a region
    // with more events draws the rest)
    double rmax = 0.0;
    for (double r : cfg->rate) rmax = std::max(rmax, r);
    const double Wd = std::min(c->cfg.W, std::max(cfg->t_end, 1e-9));
    long long PC = (long long)std::ceil(1.25 * cfg->bx * cfg->by * rmax * Wd) + 32;
    PC = std::min<long long>(PC, 8192);
    PC = std::min<long long>(PC, (24LL << 30) / (16LL * std::max(1, c->nreg)));
    if (PC >= 8) {
      c->PC = (int)PC;
      if (dmalloc(c, &c->pcache, (size_t)c->nreg * (size_t)PC) != cudaSuccess || dmalloc(c, &c->pmeta, n) != cudaSuccess) {
        cudaGetLastError();
        dfree(c, c->pcache); dfree(c, c->pmeta);
        c->pcache = nullptr; c->pmeta = nullptr;
        c->PC = 0;
      } else if (cudaMemsetAsync(c->pmeta, 0, n * sizeof(uint2), c->stream) != cudaSuccess) {
        return bail(ISING_SR_E_CUDA);
      }
    }
  }
  c->stats.hist_capacity = c->K;

  // strip + one halo row above and below (periodic), packed by K0 (any
  // nonzero byte is an up spin).  Copied straight from the caller's buffer in
  // at most three row runs (DMA at full speed when it is pinned).
  const int Lx = cfg->Lx, Ly = cfg->Ly, by = cfg->by;
  const int rows = c->RYl * by + 2;
  const int y_first = c->row0 * by - 1;
  uint8_t* dbuf = nullptr;
  if (dmalloc_bytes(c, (void**)&dbuf, (size_t)rows * Lx) != cudaSuccess) return bail(ISING_SR_E_OOM);
  if (!spins) {  // the Philox init stream, generated on the device
    const long long ns = (long long)rows * Lx;
    philox_spins_kernel<<<(unsigned)((ns + 255) / 256), 256, 0, c->stream>>>(dbuf, rows, y_first, Lx, Ly, cfg->seed);
    c->launches++;
  }
  for (int q = 0; spins && q < rows;) {
    const int y = ((y_first + q) % Ly + Ly) % Ly;
    const int run = std::min(rows - q, Ly - y);  // contiguous up to the lattice's last row
    if (cudaMemcpyAsync(dbuf + (size_t)q * Lx, spins + (size_t)y * Lx, (size_t)run * Lx, cudaMemcpyHostToDevice,
                        c->stream) != cudaSuccess) {
      dfree(c, dbuf);
      return bail(ISING_SR_E_CUDA);
    }
    q += run;
  }
  ops->init(dbuf, Lx, RX, c->RYl, c->row0, cfg->seed, cfg->eq_quantum, c->st[0], c->stream);
  c->launches++;
  if ((c->cfg.flags & ISING_SR_FLAG_OBSERVABLES) && enqueue_snapshot(c, c->st[0]) != ISING_SR_OK)
    return bail(ISING_SR_E_CUDA);
  cudaError_t e = cudaStreamSynchronize(c->stream);
  dfree(c, dbuf);
  if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) return bail(ISING_SR_E_CUDA);
  c->stats.obs_M_now = (int64_t)c->h_snap[0];
  c->stats.obs_B_now = (int64_t)c->h_snap[1];
  c->stats.edge_entries_last_window = -1;
  c->stats.log_replayed_last_window = -1;
  c->comm = 0;
  if (cfg->nccl_id) {  // the library's communicator for C1/C2 (collective over the ranks)
    const isr_nccl::Api& A = isr_nccl::api();
    if (!A.ok) return bail(ISING_SR_E_NCCL);
    isr_nccl::UniqueId id;
    std::memcpy(&id, cfg->nccl_id, sizeof id);
    if (!isr_nccl::report(A.CommInitRank(&c->nccl, world, id, cfg->rank), "ncclCommInitRank")) {
      c->nccl = nullptr;
      return bail(ISING_SR_E_NCCL);
    }
    if (ising_sr_status ps = peer_setup(c)) return bail(ps);
  }
  *out = c;
  return ISING_SR_OK;
}

ising_sr_status ising_sr_begin_window(ising_sr_ctx* c) {
  ising_sr_status s = check(c);
  if (s) return s;
  if (!(((double)c->w * c->cfg.W) < c->cfg.t_end)) return ISING_SR_E_STATE;
  start_window(c);
  CK(c, cudaEventRecord(c->ev0, c->stream));
  return ISING_SR_OK;
}

ising_sr_status ising_sr_iterate(ising_sr_ctx* c, int32_t flags_out[2]) {
  ising_sr_status s = check(c);
  if (s) return s;
  if (!c->in_window || c->converged) return ISING_SR_E_STATE;
  if ((s = launch_iteration(c))) return s;
  if ((s = read_flags(c))) return s;
  if (flags_out) {
    flags_out[0] = c->h_flags[0];
    flags_out[1] = c->h_flags[1];
  }
  return ISING_SR_OK;
}

ising_sr_status ising_sr_halo_get(ising_sr_ctx* c, ising_sr_halo* out) {
  ising_sr_status s = check(c);
  if (s) return s;
  if (!out || !c->in_window || c->it < 1 || !c->ghost || c->peer) return ISING_SR_E_STATE;
  fill_halo(c, out);
  return ISING_SR_OK;
}

ising_sr_status ising_sr_exchange_done(ising_sr_ctx* c) {
  ising_sr_status s = check(c);
  if (s) return s;
  if (!c->in_window || c->it < 1) return ISING_SR_E_STATE;
  if ((s = mark_ghosts(c))) return s;
  const unsigned K = c->Kglob;
  CK(c, cudaMemcpyAsync(c->h_wlc, c->d_wlc + ((K + 1) & 1), sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  c->n_work = (int)c->h_wlc[0];
  return ISING_SR_OK;
}

ising_sr_status ising_sr_end_iterations(ising_sr_ctx* c, int32_t g) {
  ising_sr_status s = check(c);
  if (s) return s;
  if (!c->in_window) return ISING_SR_E_STATE;
  if (g == -1) {
    if ((s = grow_capacity(c))) return s;
    c->in_window = false;
    return ISING_SR_OK;
  }
  if (g != c->it || g < 1) return ISING_SR_E_INVALID_ARG;
  c->converged = true;
  c->g = g;
  return ISING_SR_OK;
}

ising_sr_status ising_sr_run_window(ising_sr_ctx* c, int32_t* g_out) {
  NvtxRange nv("isr window");
  ising_sr_status s = check(c);
  if (s) return s;
  if (c->ghost && !c->nccl && !c->cfg.exchange) return ISING_SR_E_INVALID_ARG;  // step-level API only
  if ((s = ising_sr_begin_window(c))) return s;
  // (strips keep the host loop: NCCL's captured work is not allowed inside a
  // conditional node's body -- cudaGraphAddNode/EndCapture reject it)
  if (c->graph && c->pipeline && !(c->cfg.flags & ISING_SR_FLAG_JACOBI_ALL) && (!c->ghost || c->peer)) {
    if ((s = run_window_graph(c))) return s;
    if (g_out) *g_out = c->g;
    return ISING_SR_OK;
  }
  if (c->pipeline && !(c->cfg.flags & ISING_SR_FLAG_JACOBI_ALL)) {
    if ((s = run_window_pipelined(c))) return s;
    if (g_out) *g_out = c->g;
    return ISING_SR_OK;
  }
  // one iteration per host synchronisation (ISING_SR_PIPELINE=0, or the
  // Jacobi schedule over all regions)
  for (;;) {
    if ((s = launch_iteration(c))) return s;
    if (c->ghost) {
      if ((s = exchange(c, c->d_flags))) return s;
      if ((s = mark_ghosts(c))) return s;
    }
    if ((s = read_flags(c))) return s;
    if (c->h_flags[1]) {  // history capacity overflow: grow and restart the window
      if ((s = grow_capacity(c))) return s;
      start_window(c);
      continue;
    }
    if (!c->h_flags[0]) {
      c->converged = true;
      c->g = c->it;
      break;
    }
    if (c->it >= c->cfg.max_iterations) {
      c->in_window = false;
      return ISING_SR_E_DIVERGED;
    }
  }
  if (g_out) *g_out = c->g;
  return ISING_SR_OK;
}

static ising_sr_status commit_impl(ising_sr_ctx* c, int64_t* events_out) {
  NvtxRange nv("isr commit");
  ising_sr_status s = check(c);
  if (s) return s;
  if (!c->in_window || !c->converged) return ISING_SR_E_STATE;
  const StateView& s0 = c->st[c->comm];
  const StateView& s1 = c->st[c->comm ^ 1];
  const int nbs = (c->nreg + kScanBlock - 1) / kScanBlock;
  // e_i = n_next - n_comm: the window's total, and (event log) the scan for the log offsets
  const bool log = (c->cfg.flags & ISING_SR_FLAG_LOG_EVENTS) != 0;
  if (!log) {
    CK(c, cudaMemsetAsync(c->d_total, 0, sizeof(unsigned long long), c->stream));
    count_events<<<std::max(1, std::min((c->nreg + 255) / 256, 148 * 8)), 256, 0, c->stream>>>(s1.n, s0.n, c->nreg,
                                                                                             c->d_total);
    c->launches++;
  } else {
    scan_block_sums<<<nbs, kScanThreads, 0, c->stream>>>(s1.n, s0.n, c->nreg, c->d_bsum);
    scan_top<<<1, 1024, 0, c->stream>>>(c->d_bsum, nbs, c->d_total);
    c->launches += 2;
  }
  if (log) {
    scan_apply<<<nbs, kScanThreads, 0, c->stream>>>(s1.n, s0.n, c->nreg, c->d_bsum, c->d_off);
    c->launches++;
  }
  CK(c, cudaGetLastError());
  const bool obs = (c->cfg.flags & ISING_SR_FLAG_OBSERVABLES) != 0;
  const bool mag = (c->cfg.flags & ISING_SR_FLAG_MAG_MOMENTS) != 0;
  if (obs) {  // the window's int M dt, int B dt: fixed-order sums of the regions' integrals
    obs_partial<<<kObsBlocks, 256, 0, c->stream>>>(s1.oM, s1.oB, c->nreg, c->d_obs);
    obs_final<<<1, 256, 0, c->stream>>>(c->d_obs, c->d_obs + 2 * kObsBlocks);
    c->launches += 2;
    CK(c, cudaGetLastError());
    CK(c, cudaMemcpyAsync(c->h_obs, c->d_obs + 2 * kObsBlocks, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                          c->stream));
    if (!mag) {  // (with MAG_MOMENTS after the moments, which start from M(t_c))
      ising_sr_status ss = enqueue_snapshot(c, s1);  // the configuration at the new committed time
      if (ss) return ss;
    }
  }
  unsigned long long total = 0;
  CK(c, cudaMemcpyAsync(&total, c->d_total, sizeof total, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  c->win_events = total;
  if (log) {
    if ((long long)total > c->log_cap) {
      for (void* q : {(void*)c->log_t, (void*)c->log_region, (void*)c->log_site, (void*)c->log_dm,
                      (void*)c->mm_ts, (void*)c->mm_dm})
        dfree(c, q);
      c->log_t = nullptr;
      c->log_region = nullptr;
      c->log_site = nullptr;
      c->log_dm = nullptr;
      c->mm_ts = nullptr;
      c->mm_dm = nullptr;
      const long long cap = std::max<long long>((long long)total * 5 / 4 + 1024, c->log_cap * 2);
      if (dmalloc(c, &c->log_t, cap) != cudaSuccess || dmalloc(c, &c->log_region, cap) != cudaSuccess ||
          dmalloc(c, &c->log_site, cap) != cudaSuccess ||
          (mag && (dmalloc(c, &c->log_dm, cap) != cudaSuccess || dmalloc(c, &c->mm_ts, cap) != cudaSuccess ||
                   dmalloc(c, &c->mm_dm, cap) != cudaSuccess))) {
        cudaGetLastError();
        c->log_cap = 0;
        return ISING_SR_E_OOM;
      }
      c->log_cap = cap;
    }
    // K3: compact the scratch log of every region's final recomputation;
    // regions with more than evC events are listed and replayed against the
    // final (latest) histories
    CK(c, cudaEventRecord(c->cev0, c->stream));
    CK(c, cudaMemsetAsync(c->d_nrep, 0, 4 * sizeof(unsigned), c->stream));
    CK(c, cudaMemsetAsync(c->d_edges, 0, sizeof(unsigned long long), c->stream));
    int lbx = 0;
    while ((1 << lbx) < c->cfg.bx) ++lbx;  // region widths are powers of two
    const int wx = c->RX == 1 ? 1 : 0, wy = c->RYg == 1 ? 1 : 0;
    compact_log_kernel<<<(c->nreg + 255) / 256, 256, 0, c->stream>>>(
        s1.n, s0.n, c->nreg, c->d_off, c->ev_t, c->ev_s, (long long)c->nreg, c->evC, c->RX, c->row0, lbx, c->cfg.bx,
        c->cfg.by, wx, wy, c->log_t, c->log_region, c->log_site, mag ? c->log_dm : nullptr, c->d_replay, c->d_nrep,
        c->d_edges);
    c->launches++;
    CK(c, cudaGetLastError());
    KArgs a = base_args(c, c->Kglob + 1, false);
    a.wl_in = c->d_replay;
    a.n_work = 0;
    a.n_work_dev = c->d_nrep;  // the list's length, read on the device
    a.tile = kThreads;
    a.log_t = c->log_t;
    a.log_region = c->log_region;
    a.log_site = c->log_site;
    a.log_dm = mag ? c->log_dm : nullptr;
    a.log_off = c->d_off;
    a.log_cap = c->log_cap;
    c->ops->replay(a, 148 * 4 * kThreads, c->stream);  // a fixed grid; tiles sized on the device
    c->launches++;
    CK(c, cudaGetLastError());
    replay_edge_entries<<<148, 256, 0, c->stream>>>(c->d_replay, c->d_nrep, s1.n, s0.n, c->d_off, c->log_site, lbx,
                                                    c->cfg.bx, c->cfg.by, wx, wy, c->d_edges);
    c->launches++;
    CK(c, cudaGetLastError());
    CK(c, cudaEventRecord(c->cev1, c->stream));
    CK(c, cudaMemcpyAsync(&c->h_nrep, c->d_nrep, sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaMemcpyAsync(&c->h_edges, c->d_edges, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
    c->log_n = (long long)total;
    c->win_bytes += (double)total * 14.0 + (double)c->nreg * 8.0;
    if (mag) {  // int |M| dt, int M^2 dt over [t_c, t_w): the log in time order
      ising_sr_status ms_ = mag_moments(c, (long long)total);
      if (ms_) return ms_;
      if ((ms_ = enqueue_snapshot(c, s1))) return ms_;
    }
  }
  CK(c, cudaEventRecord(c->ev1, c->stream));
  CK(c, cudaEventSynchronize(c->ev1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, c->ev0, c->ev1);
  c->comm ^= 1;  // committed <- fixed point
  c->w += 1;
  c->t_c = (double)c->w * c->cfg.W;
  c->in_window = false;
  c->stats.t_c = c->t_c < c->cfg.t_end ? c->t_c : c->cfg.t_end;
  c->stats.windows++;
  c->stats.events_total += (long long)c->win_events;
  c->stats.events_last_window = (long long)c->win_events;
  c->stats.g_last = c->g;
  c->stats.g_max = std::max(c->stats.g_max, c->g);
  c->stats.g_hist[std::min(c->g, 63)]++;
  c->stats.f_last = c->win_f;
  c->stats.f_max = std::max(c->stats.f_max, c->win_f);
  c->stats.bytes_alg_last_window = c->win_bytes;
  std::memcpy(c->stats.active_last, c->win_active, sizeof c->win_active);
  c->stats.ms_last_window = ms;
  if (log) {
    float cms = 0.f;
    cudaEventElapsedTime(&cms, c->cev0, c->cev1);
    c->stats.ms_compact_total += cms;
    c->stats.edge_entries_last_window = (int64_t)c->h_edges;
    c->stats.log_replayed_last_window = (int64_t)c->h_nrep;
  }
  if (mag) {
    c->stats.obs_absM_last = c->h_mm[0];
    c->stats.obs_M2_last = c->h_mm[1];
    c->stats.obs_absM_total += c->h_mm[0];
    c->stats.obs_M2_total += c->h_mm[1];
  }
  if (obs) {
    c->stats.obs_M_last = c->h_obs[0];
    c->stats.obs_B_last = c->h_obs[1];
    c->stats.obs_M_total += c->h_obs[0];
    c->stats.obs_B_total += c->h_obs[1];
    c->stats.obs_time_total += c->t_w - (double)(c->w - 1) * c->cfg.W;  // t_w - t_c of this window
    c->stats.obs_M_now = (int64_t)c->h_snap[0];
    c->stats.obs_B_now = (int64_t)c->h_snap[1];
  }
  if (events_out) *events_out = (long long)c->win_events;
  return ISING_SR_OK;
}

ising_sr_status ising_sr_commit(ising_sr_ctx* c, int64_t* events_out) {
  const auto t0 = std::chrono::steady_clock::now();
  const ising_sr_status s = commit_impl(c, events_out);
  if (c) c->stats.ms_commit_total += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return s;
}

ising_sr_status ising_sr_run(ising_sr_ctx* c, int64_t* events_out) {
  ising_sr_status s = check(c);
  if (s) return s;
  long long tot = 0;
  while (((double)c->w * c->cfg.W) < c->cfg.t_end) {
    int32_t g = 0;
    int64_t ev = 0;
    if ((s = ising_sr_run_window(c, &g))) return s;
    if ((s = ising_sr_commit(c, &ev))) return s;
    tot += ev;
  }
  if (events_out) *events_out = tot;
  return ISING_SR_OK;
}

ising_sr_status ising_sr_stats_get(const ising_sr_ctx* c, ising_sr_stats* out) {
  if (!c || !out) return ISING_SR_E_INVALID_ARG;
  *out = c->stats;
  return c->sticky;
}

ising_sr_status ising_sr_get_spins(ising_sr_ctx* c, uint8_t* out) {
  ising_sr_status s = check(c);
  if (s) return s;
  if (!out) return ISING_SR_E_INVALID_ARG;
  const size_t n = (size_t)c->RYl * c->cfg.by * c->cfg.Lx;
  uint8_t* d = nullptr;
  CK(c, dmalloc_bytes(c, (void**)&d, n));
  c->ops->unpack(c->st[c->comm], c->cfg.Lx, c->RX, c->RYl, d, c->stream);
  c->launches++;
  cudaError_t e = cudaMemcpyAsync(out, d, n, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  dfree(c, d);
  CK(c, e);
  return ISING_SR_OK;
}

ising_sr_status ising_sr_get_events(ising_sr_ctx* c, double* t, uint32_t* region, uint16_t* site, int64_t cap,
                                    int64_t* n) {
  ising_sr_status s = check(c);
  if (s) return s;
  if (!(c->cfg.flags & ISING_SR_FLAG_LOG_EVENTS)) return ISING_SR_E_STATE;
  if (n) *n = c->log_n;
  const long long m = std::min<long long>(cap, c->log_n);
  if (m > 0) {
    if (t) CK(c, cudaMemcpyAsync(t, c->log_t, m * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (region)
      CK(c, cudaMemcpyAsync(region, c->log_region, m * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
    if (site) CK(c, cudaMemcpyAsync(site, c->log_site, m * sizeof(uint16_t), cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
  }
  return ISING_SR_OK;
}

ising_sr_status ising_sr_get_digests(ising_sr_ctx* c, uint64_t* digest, uint64_t* count) {
  ising_sr_status s = check(c);
  if (s) return s;
  const StateView& st = c->st[c->comm];
  if (digest) {
    if (!(c->cfg.flags & ISING_SR_FLAG_DIGEST)) return ISING_SR_E_STATE;
    CK(c, cudaMemcpyAsync(digest, st.dig, (size_t)c->nreg * 8, cudaMemcpyDeviceToHost, c->stream));
  }
  if (count) {
    std::vector<uint32_t> tmp((size_t)c->nreg);
    CK(c, cudaMemcpyAsync(tmp.data(), st.n, (size_t)c->nreg * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    for (size_t i = 0; i < tmp.size(); ++i) count[i] = tmp[i];
  }
  CK(c, cudaStreamSynchronize(c->stream));
  return ISING_SR_OK;
}

// ---------------------------------------------------------------------------
// checkpoint / resume: header + the committed state arrays of this rank
// ---------------------------------------------------------------------------
namespace {
struct CkptHeader {
  char magic[8];  // "ISRCKPT1"
  int32_t Lx, Ly, bx, by, rank, world;
  uint32_t flags, pad;
  uint64_t seed;
  double W, t_end, rate[10];
  int64_t w;  // committed windows: t_c = fl(w W)
  int64_t windows, events_total;
  double obs_M_total, obs_B_total, obs_time_total;
  int64_t nreg;
  int64_t bytes[6];  // spins, halo, ts, R, n, dig
  uint64_t checksum;  // FNV-1a over the arrays
};

void state_bytes(const ising_sr_ctx* c, int64_t b[6]) {
  const int64_t n = c->nreg;
  b[0] = n * (int64_t)c->ops->spin_bytes;
  b[1] = n * (int64_t)c->ops->halo_bytes;
  b[2] = n * 8;
  b[3] = n * 8;
  b[4] = n * 4;
  b[5] = n * 8;
}

uint64_t fnv1a(const unsigned char* p, int64_t n, uint64_t h) {
  for (int64_t i = 0; i < n; ++i) h = (h ^ p[i]) * 0x100000001b3ULL;
  return h;
}
}  // namespace

ising_sr_status ising_sr_checkpoint_size(const ising_sr_ctx* c, int64_t* bytes) {
  if (!c || !bytes) return ISING_SR_E_INVALID_ARG;
  int64_t b[6];
  state_bytes(c, b);
  *bytes = (int64_t)sizeof(CkptHeader) + b[0] + b[1] + b[2] + b[3] + b[4] + b[5];
  return c->sticky;
}

ising_sr_status ising_sr_checkpoint_save(ising_sr_ctx* c, void* buf, int64_t cap) {
  ising_sr_status s = check(c);
  if (s) return s;
  if (!buf) return ISING_SR_E_INVALID_ARG;
  if (c->in_window) return ISING_SR_E_STATE;
  int64_t need = 0;
  ising_sr_checkpoint_size(c, &need);
  if (cap < need) return ISING_SR_E_INVALID_ARG;
  CkptHeader h;
  std::memset(&h, 0, sizeof h);
  std::memcpy(h.magic, "ISRCKPT1", 8);
  h.Lx = c->cfg.Lx; h.Ly = c->cfg.Ly; h.bx = c->cfg.bx; h.by = c->cfg.by;
  h.rank = c->cfg.rank; h.world = c->cfg.world;
  h.flags = c->cfg.flags;
  h.seed = c->cfg.seed;
  h.W = c->cfg.W; h.t_end = c->cfg.t_end;
  for (int k = 0; k < 10; ++k) h.rate[k] = c->cfg.rate[k];
  h.w = c->w;
  h.windows = c->stats.windows;
  h.events_total = c->stats.events_total;
  h.obs_M_total = c->stats.obs_M_total;
  h.obs_B_total = c->stats.obs_B_total;
  h.obs_time_total = c->stats.obs_time_total;
  h.nreg = c->nreg;
  state_bytes(c, h.bytes);
  unsigned char* p = (unsigned char*)buf + sizeof(CkptHeader);
  const StateView& st = c->st[c->comm];
  void* src[6] = {st.spins, st.halo, st.ts, st.R, st.n, st.dig};
  unsigned char* q = p;
  for (int i = 0; i < 6; ++i) {
    CK(c, cudaMemcpyAsync(q, src[i], (size_t)h.bytes[i], cudaMemcpyDeviceToHost, c->stream));
    q += h.bytes[i];
  }
  CK(c, cudaStreamSynchronize(c->stream));
  h.checksum = fnv1a(p, need - (int64_t)sizeof(CkptHeader), 0xcbf29ce484222325ULL);
  std::memcpy(buf, &h, sizeof h);
  return ISING_SR_OK;
}

ising_sr_status ising_sr_checkpoint_load(ising_sr_ctx* c, const void* buf, int64_t len) {
  ising_sr_status s = check(c);
  if (s) return s;
  if (!buf || len < (int64_t)sizeof(CkptHeader)) return ISING_SR_E_INVALID_ARG;
  if (c->in_window) return ISING_SR_E_STATE;
  CkptHeader h;
  std::memcpy(&h, buf, sizeof h);
  int64_t b[6], need = 0;
  state_bytes(c, b);
  ising_sr_checkpoint_size(c, &need);
  bool ok = std::memcmp(h.magic, "ISRCKPT1", 8) == 0 && len >= need && h.Lx == c->cfg.Lx && h.Ly == c->cfg.Ly &&
            h.bx == c->cfg.bx && h.by == c->cfg.by && h.rank == c->cfg.rank && h.world == c->cfg.world &&
            h.flags == c->cfg.flags && h.seed == c->cfg.seed && h.W == c->cfg.W && h.nreg == c->nreg &&
            h.w >= 0;
  for (int k = 0; k < 10 && ok; ++k) ok = h.rate[k] == c->cfg.rate[k];
  for (int i = 0; i < 6 && ok; ++i) ok = h.bytes[i] == b[i];
  const unsigned char* p = (const unsigned char*)buf + sizeof(CkptHeader);
  if (ok) ok = fnv1a(p, need - (int64_t)sizeof(CkptHeader), 0xcbf29ce484222325ULL) == h.checksum;
  if (!ok) return ISING_SR_E_INVALID_ARG;
  const StateView& st = c->st[c->comm];
  void* dst[6] = {st.spins, st.halo, st.ts, st.R, st.n, st.dig};
  for (int i = 0; i < 6; ++i) {
    CK(c, cudaMemcpyAsync(dst[i], p, (size_t)b[i], cudaMemcpyHostToDevice, c->stream));
    p += b[i];
  }
  CK(c, cudaStreamSynchronize(c->stream));
  c->w = h.w;
  c->t_c = (double)c->w * c->cfg.W;
  c->in_window = false;
  c->converged = false;
  c->stats.windows = h.windows;
  c->stats.events_total = h.events_total;
  c->stats.obs_M_total = h.obs_M_total;
  c->stats.obs_B_total = h.obs_B_total;
  c->stats.obs_time_total = h.obs_time_total;
  if (c->cfg.flags & ISING_SR_FLAG_OBSERVABLES) {
    ising_sr_status ss = enqueue_snapshot(c, st);
    if (ss) return ss;
    CK(c, cudaStreamSynchronize(c->stream));
    c->stats.obs_M_now = (int64_t)c->h_snap[0];
    c->stats.obs_B_now = (int64_t)c->h_snap[1];
  }
  c->stats.t_c = c->t_c < c->cfg.t_end ? c->t_c : c->cfg.t_end;
  return ISING_SR_OK;
}

int64_t ising_sr_launch_count(const ising_sr_ctx* c) { return c ? c->launches : 0; }

size_t ising_sr_struct_size(int32_t which) {
  return which == 0 ? sizeof(ising_sr_config) : which == 1 ? sizeof(ising_sr_stats) : which == 2 ? sizeof(ising_sr_halo) : 0;
}

}  // extern "C"
