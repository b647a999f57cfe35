// isr_runtime.cu -- host runtime and C ABI of libising_sr.so (include/ising_sr.h).
//
// Drives the synchronous-relaxation loop of the paper: for each
// window ("step") it launches the region-trajectory kernel once per
// relaxation iteration, exchanges strip halos through the caller's
// transport (world > 1), reads the global {changed, overflow} flag, and on
// convergence commits the window by swapping the committed and tentative
// state buffers.  Device memory layout: DESIGN.md §5.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/ising_sr.h"
#include "isr_region.cuh"

namespace {

using isr::EdgeView;
using isr::KArgs;
using isr::StateView;

constexpr int kThreads = 128;

// ---------------------------------------------------------------------------
// per-shape kernel table (lane-per-region forms)
// ---------------------------------------------------------------------------
struct ShapeOps {
  int bx, by;
  size_t spin_bytes, halo_bytes;
  void (*region)(const KArgs&, int nreg, cudaStream_t);
  void (*replay)(const KArgs&, int nreg, cudaStream_t);
  void (*init)(const uint8_t*, int, int, int, int, unsigned long long, StateView, cudaStream_t);
  void (*unpack)(StateView, int, int, int, uint8_t*, cudaStream_t);
};

template <int BX, int BY>
ShapeOps make_ops() {
  using G = isr::Geo<BX, BY>;
  ShapeOps o;
  o.bx = BX;
  o.by = BY;
  o.spin_bytes = sizeof(typename G::ST);
  o.halo_bytes = sizeof(typename G::HT);
  o.region = [](const KArgs& a, int nreg, cudaStream_t s) {
    const int grid = (nreg + kThreads - 1) / kThreads;
    isr::region_kernel<BX, BY, false><<<grid, kThreads, 0, s>>>(a);
  };
  o.replay = [](const KArgs& a, int nreg, cudaStream_t s) {
    const int grid = (nreg + kThreads - 1) / kThreads;
    isr::region_kernel<BX, BY, true><<<grid, kThreads, 0, s>>>(a);
  };
  o.init = [](const uint8_t* buf, int Lx, int RX, int RYl, int row0, unsigned long long seed, StateView st,
              cudaStream_t s) {
    const int n = RX * RYl;
    isr::init_kernel<BX, BY><<<(n + kThreads - 1) / kThreads, kThreads, 0, s>>>(buf, Lx, RX, RYl, row0, seed, st);
  };
  o.unpack = [](StateView st, int Lx, int RX, int RYl, uint8_t* out, cudaStream_t s) {
    const long long n = (long long)RYl * BY * Lx;
    isr::unpack_kernel<BX, BY><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(st, Lx, RX, RYl, out);
  };
  return o;
}

const ShapeOps* find_ops(int bx, int by) {
  static const ShapeOps table[] = {make_ops<1, 1>(), make_ops<2, 2>(), make_ops<4, 4>(), make_ops<8, 8>(),
                                   make_ops<4, 2>(), make_ops<2, 4>(), make_ops<8, 4>(), make_ops<4, 8>()};
  for (const auto& o : table)
    if (o.bx == bx && o.by == by) return &o;
  return nullptr;
}

// ---------------------------------------------------------------------------
// exclusive scan of e_i = n_next[i] - n_comm[i] (log offsets for the replay)
// ---------------------------------------------------------------------------
__global__ void scan_block_sums(const uint32_t* n1, const uint32_t* n0, int N, unsigned long long* bsum) {
  __shared__ unsigned long long sh[32];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long v = i < N ? (unsigned long long)(n1[i] - n0[i]) : 0ull;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
    bsum[blockIdx.x] = s;
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

__global__ void scan_apply(const uint32_t* n1, const uint32_t* n0, int N, const unsigned long long* bsum,
                           unsigned long long* off) {
  __shared__ unsigned long long sh[32];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long v = i < N ? (unsigned long long)(n1[i] - n0[i]) : 0ull;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long x = v;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += t;
  }
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long s = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
      const unsigned long long t = sh[q];
      sh[q] = s;
      s += t;
    }
  }
  __syncthreads();
  if (i < N) off[i] = bsum[blockIdx.x] + sh[w] + x - v;
}

}  // namespace

// ---------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------
struct ising_sr_ctx {
  ising_sr_config cfg;
  const ShapeOps* ops = nullptr;
  int RX = 0, RYg = 0, RYl = 0, row0 = 0, nreg = 0, rows_s = 0;
  int K = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  ising_sr_status sticky = ISING_SR_OK;

  // device buffers
  StateView st[2] = {};
  int comm = 0;  // index of the committed state
  EdgeView ed[2] = {};
  int* d_flags = nullptr;               // [4]
  unsigned long long* d_stats = nullptr;  // [8]
  int* h_flags = nullptr;               // pinned mirror [4]
  unsigned long long* h_stats = nullptr;  // pinned mirror [8]
  // log
  double* log_t = nullptr;
  uint32_t* log_region = nullptr;
  uint16_t* log_site = nullptr;
  long long log_cap = 0, log_n = 0;
  unsigned long long* d_off = nullptr;
  unsigned long long* d_bsum = nullptr;
  unsigned long long* d_total = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t kev0 = nullptr, kev1 = nullptr;  // around each region-kernel launch

  // window state
  long long w = 0;
  double t_c = 0.0, t_w = 0.0;
  int it = 0;
  bool in_window = false, converged = false;
  int g = 0;
  // per-window accumulators
  unsigned long long win_events = 0;
  double win_bytes = 0.0;
  int win_f = 0;
  long long launches = 0;
  ising_sr_stats stats;
};

namespace {

ising_sr_status fail_cuda(ising_sr_ctx* c, cudaError_t e, const char* where) {
  if (e == cudaSuccess) return ISING_SR_OK;
  std::fprintf(stderr, "ising_sr: CUDA error at %s: %s\n", where, cudaGetErrorString(e));
  if (c) c->sticky = ISING_SR_E_CUDA;
  return ISING_SR_E_CUDA;
}

#define CK(ctx, expr)                                                     \
  do {                                                                    \
    cudaError_t _e = (expr);                                              \
    if (_e != cudaSuccess) return fail_cuda((ctx), _e, #expr);            \
  } while (0)

template <class T>
cudaError_t dmalloc(T** p, size_t count) {
  return cudaMalloc((void**)p, std::max<size_t>(count, 1) * sizeof(T));
}

void free_edges(ising_sr_ctx* c) {
  for (auto& e : c->ed) {
    cudaFree(e.cnt);
    cudaFree(e.t);
    cudaFree(e.pos);
    e = EdgeView{};
  }
}

ising_sr_status alloc_edges(ising_sr_ctx* c, int K) {
  free_edges(c);
  c->K = K;
  const size_t cn = (size_t)4 * c->rows_s * c->RX;
  const size_t tn = cn * (size_t)K;
  for (auto& e : c->ed) {
    if (dmalloc(&e.cnt, cn) != cudaSuccess || dmalloc(&e.t, tn) != cudaSuccess ||
        dmalloc(&e.pos, tn) != cudaSuccess) {
      cudaGetLastError();
      free_edges(c);
      return ISING_SR_E_OOM;
    }
    // ghost rows must read as "no events" before the first exchange
    CK(c, cudaMemsetAsync(e.cnt, 0, cn, c->stream));
  }
  return ISING_SR_OK;
}

int auto_capacity(const ising_sr_config& cfg) {
  // expected boundary events per edge per window at the largest rate, with a
  // generous Poisson tail margin; overflow is detected and retried anyway
  double rmax = 0.0;
  for (double r : cfg.rate) rmax = std::max(rmax, r);
  const double mu = std::max(cfg.bx, cfg.by) * rmax * cfg.W;
  const int K = (int)std::ceil(mu + 6.0 * std::sqrt(mu) + 8.0);
  return std::min(std::max(K, 8), 255);
}

ising_sr_status check(const ising_sr_ctx* c) {
  if (!c) return ISING_SR_E_INVALID_ARG;
  return c->sticky;
}

KArgs base_args(ising_sr_ctx* c, int it_parity_prev, int it_parity_cur, bool first) {
  KArgs a;
  std::memset(&a, 0, sizeof a);
  a.in = c->st[c->comm];
  a.out = c->st[c->comm ^ 1];
  a.prev = c->ed[it_parity_prev];
  a.cur = c->ed[it_parity_cur];
  a.RX = c->RX;
  a.RYl = c->RYl;
  a.RYg = c->RYg;
  a.row0 = c->row0;
  a.world = c->cfg.world;
  a.K = c->K;
  a.cstride = (long long)c->rows_s * c->RX;
  a.tstride = (long long)c->rows_s * c->K * c->RX;
  a.first = first ? 1 : 0;
  a.digest = (c->cfg.flags & ISING_SR_FLAG_DIGEST) ? 1 : 0;
  a.t_w = c->t_w;
  a.seed = c->cfg.seed;
  for (int k = 0; k < 10; ++k) a.rate[k] = c->cfg.rate[k];
  a.flags = c->d_flags;
  a.stats = c->d_stats;
  return a;
}

// algorithmic bytes of one iteration: state in + out per
// recomputed region, 3 count bytes x 4 edges, 9 bytes per history entry
// written, read by the neighbour, and compared.
double iteration_bytes(const ising_sr_ctx* c, const unsigned long long* s) {
  const double S = (double)c->ops->spin_bytes + (double)c->ops->halo_bytes + 8 + 8 + 4 +
                   ((c->cfg.flags & ISING_SR_FLAG_DIGEST) ? 8 : 0);
  const double regions = (double)s[5];
  return regions * (2.0 * S + 12.0) + 9.0 * ((double)s[1] + (double)s[2] + (double)s[3]);
}

ising_sr_status launch_iteration(ising_sr_ctx* c) {
  ++c->it;
  const int cur = c->it & 1, prev = cur ^ 1;
  CK(c, cudaMemsetAsync(c->d_flags, 0, 4 * sizeof(int), c->stream));
  CK(c, cudaMemsetAsync(c->d_stats, 0, 8 * sizeof(unsigned long long), c->stream));
  KArgs a = base_args(c, prev, cur, c->it == 1);
  CK(c, cudaEventRecord(c->kev0, c->stream));
  c->ops->region(a, c->nreg, c->stream);
  ++c->launches;
  CK(c, cudaGetLastError());
  CK(c, cudaEventRecord(c->kev1, c->stream));
  return ISING_SR_OK;
}

ising_sr_status read_flags(ising_sr_ctx* c) {
  CK(c, cudaMemcpyAsync(c->h_flags, c->d_flags, 4 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaMemcpyAsync(c->h_stats, c->d_stats, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                        c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  float kms = 0.f;
  CK(c, cudaEventElapsedTime(&kms, c->kev0, c->kev1));
  const double ib = iteration_bytes(c, c->h_stats);
  c->stats.region_launches++;
  c->stats.region_ms += kms;
  c->stats.region_bytes += ib;
  c->stats.iterations_total++;
  c->stats.recomputations_total += (long long)c->h_stats[5];
  c->win_bytes += ib;
  c->win_events = c->h_stats[0];
  c->win_f = std::max(c->win_f, (int)c->h_stats[4]);
  return ISING_SR_OK;
}

void fill_halo(ising_sr_ctx* c, ising_sr_halo* h) {
  std::memset(h, 0, sizeof *h);
  const EdgeView& e = c->ed[c->it & 1];
  const size_t RX = (size_t)c->RX, K = (size_t)c->K;
  const size_t cst = (size_t)c->rows_s * RX, tst = cst * K;
  const size_t rowN = 1, rowS = (size_t)c->RYl;  // storage rows of my first / last region row
  const size_t gUp = 0, gDown = (size_t)c->RYl + 1;
  h->nchunks = 3;
  h->chunk_bytes[0] = RX;
  h->chunk_bytes[1] = K * RX * sizeof(double);
  h->chunk_bytes[2] = K * RX;
  const size_t N = isr::EDGE_N, S = isr::EDGE_S;
  h->send_up[0] = e.cnt + N * cst + rowN * RX;
  h->send_up[1] = e.t + N * tst + rowN * K * RX;
  h->send_up[2] = e.pos + N * tst + rowN * K * RX;
  h->send_down[0] = e.cnt + S * cst + rowS * RX;
  h->send_down[1] = e.t + S * tst + rowS * K * RX;
  h->send_down[2] = e.pos + S * tst + rowS * K * RX;
  h->recv_from_up[0] = e.cnt + S * cst + gUp * RX;
  h->recv_from_up[1] = e.t + S * tst + gUp * K * RX;
  h->recv_from_up[2] = e.pos + S * tst + gUp * K * RX;
  h->recv_from_down[0] = e.cnt + N * cst + gDown * RX;
  h->recv_from_down[1] = e.t + N * tst + gDown * K * RX;
  h->recv_from_down[2] = e.pos + N * tst + gDown * K * RX;
  h->flags = c->d_flags;
  h->stream = (void*)c->stream;
}

ising_sr_status grow_capacity(ising_sr_ctx* c) {
  if (c->K >= 255) return ISING_SR_E_CAPACITY;
  const int K = std::min(255, c->K * 2);
  ising_sr_status s = alloc_edges(c, K);
  if (s != ISING_SR_OK) return s;
  c->stats.overflow_retries++;
  c->stats.hist_capacity = K;
  return ISING_SR_OK;
}

void start_window(ising_sr_ctx* c) {
  c->t_c = (double)c->w * c->cfg.W;
  const double next = (double)(c->w + 1) * c->cfg.W;
  c->t_w = next < c->cfg.t_end ? next : c->cfg.t_end;
  c->it = 0;
  c->in_window = true;
  c->converged = false;
  c->g = 0;
  c->win_events = 0;
  c->win_bytes = 0.0;
  c->win_f = 0;
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
    case ISING_SR_E_NCCL: return "halo exchange failed";
    case ISING_SR_E_OOM: return "device out of memory";
    case ISING_SR_E_STATE: return "call out of order";
  }
  return "unknown status";
}

void ising_sr_destroy(ising_sr_ctx* c) {
  if (!c) return;
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& s : c->st) {
    cudaFree(s.spins);
    cudaFree(s.halo);
    cudaFree(s.ts);
    cudaFree(s.R);
    cudaFree(s.n);
    cudaFree(s.dig);
  }
  free_edges(c);
  cudaFree(c->d_flags);
  cudaFree(c->d_stats);
  cudaFreeHost(c->h_flags);
  cudaFreeHost(c->h_stats);
  cudaFree(c->log_t);
  cudaFree(c->log_region);
  cudaFree(c->log_site);
  cudaFree(c->d_off);
  cudaFree(c->d_bsum);
  cudaFree(c->d_total);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->kev0) cudaEventDestroy(c->kev0);
  if (c->kev1) cudaEventDestroy(c->kev1);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

ising_sr_status ising_sr_init(const ising_sr_config* cfg, const uint8_t* spins, ising_sr_ctx** out) {
  if (!cfg || !spins || !out) return ISING_SR_E_INVALID_ARG;
  *out = nullptr;
  if (cfg->Lx < 3 || cfg->Ly < 3) return ISING_SR_E_DIMENSION;
  if (cfg->bx < 1 || cfg->by < 1 || cfg->Lx % cfg->bx || cfg->Ly % cfg->by) return ISING_SR_E_PARTITION;
  if (!(cfg->W > 0.0) || !(cfg->t_end >= 0.0)) return ISING_SR_E_INVALID_ARG;
  for (double r : cfg->rate)
    if (!(r >= 0.0) || std::isinf(r)) return ISING_SR_E_INVALID_ARG;
  const int world = cfg->world < 1 ? 1 : cfg->world;
  if (cfg->rank < 0 || cfg->rank >= world) return ISING_SR_E_INVALID_ARG;
  if (world > 1 && !cfg->exchange) return ISING_SR_E_INVALID_ARG;
  const ShapeOps* ops = find_ops(cfg->bx, cfg->by);
  if (!ops) return ISING_SR_E_INVALID_ARG;
  const int RX = cfg->Lx / cfg->bx, RY = cfg->Ly / cfg->by;
  if (RY % world) return ISING_SR_E_PARTITION;
  if ((long long)RX * RY > 0xffffffffLL) return ISING_SR_E_INVALID_ARG;
  if (world > 1 && RY / world < 1) return ISING_SR_E_PARTITION;

  ising_sr_ctx* c = new (std::nothrow) ising_sr_ctx();
  if (!c) return ISING_SR_E_OOM;
  c->cfg = *cfg;
  c->cfg.world = world;
  if (c->cfg.max_iterations <= 0) c->cfg.max_iterations = 1000;
  c->ops = ops;
  c->RX = RX;
  c->RYg = RY;
  c->RYl = RY / world;
  c->row0 = cfg->rank * c->RYl;
  c->nreg = c->RX * c->RYl;
  c->rows_s = c->RYl + 2;
  std::memset(&c->stats, 0, sizeof c->stats);

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
    if (cudaMalloc(&s.spins, n * ops->spin_bytes) != cudaSuccess || cudaMalloc(&s.halo, n * ops->halo_bytes) != cudaSuccess ||
        dmalloc(&s.ts, n) != cudaSuccess || dmalloc(&s.R, n) != cudaSuccess || dmalloc(&s.n, n) != cudaSuccess ||
        dmalloc(&s.dig, n) != cudaSuccess)
      return bail(ISING_SR_E_OOM);
  }
  if (dmalloc(&c->d_flags, 4) != cudaSuccess || dmalloc(&c->d_stats, 8) != cudaSuccess ||
      cudaMallocHost((void**)&c->h_flags, 4 * sizeof(int)) != cudaSuccess ||
      cudaMallocHost((void**)&c->h_stats, 8 * sizeof(unsigned long long)) != cudaSuccess ||
      dmalloc(&c->d_off, n) != cudaSuccess || dmalloc(&c->d_bsum, (n + kThreads - 1) / kThreads) != cudaSuccess ||
      dmalloc(&c->d_total, 1) != cudaSuccess)
    return bail(ISING_SR_E_OOM);
  if (cudaEventCreate(&c->ev0) != cudaSuccess || cudaEventCreate(&c->ev1) != cudaSuccess ||
      cudaEventCreate(&c->kev0) != cudaSuccess || cudaEventCreate(&c->kev1) != cudaSuccess)
    return bail(ISING_SR_E_CUDA);
  const int K0 = cfg->hist_capacity > 0 ? std::min(cfg->hist_capacity, 255) : auto_capacity(*cfg);
  ising_sr_status s = alloc_edges(c, K0);
  if (s != ISING_SR_OK) return bail(s);
  c->stats.hist_capacity = c->K;

  // strip + one halo row above and below (periodic), packed by K0
  const int Lx = cfg->Lx, Ly = cfg->Ly, by = cfg->by;
  const int rows = c->RYl * by + 2;
  std::vector<uint8_t> buf((size_t)rows * Lx);
  const int y_first = c->row0 * by - 1;
  for (int q = 0; q < rows; ++q) {
    const int y = ((y_first + q) % Ly + Ly) % Ly;
    for (int x = 0; x < Lx; ++x) buf[(size_t)q * Lx + x] = spins[(size_t)y * Lx + x] ? 1 : 0;
  }
  uint8_t* dbuf = nullptr;
  if (cudaMalloc(&dbuf, buf.size()) != cudaSuccess) return bail(ISING_SR_E_OOM);
  if (cudaMemcpyAsync(dbuf, buf.data(), buf.size(), cudaMemcpyHostToDevice, c->stream) != cudaSuccess) {
    cudaFree(dbuf);
    return bail(ISING_SR_E_CUDA);
  }
  ops->init(dbuf, Lx, RX, c->RYl, c->row0, cfg->seed, c->st[0], c->stream);
  c->launches++;
  cudaError_t e = cudaStreamSynchronize(c->stream);
  cudaFree(dbuf);
  if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) return bail(ISING_SR_E_CUDA);
  c->comm = 0;
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
  if (!out || !c->in_window || c->it < 1) return ISING_SR_E_STATE;
  fill_halo(c, out);
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
  ising_sr_status s = check(c);
  if (s) return s;
  if ((s = ising_sr_begin_window(c))) return s;
  for (;;) {
    if ((s = launch_iteration(c))) return s;
    if (c->cfg.world > 1) {
      ising_sr_halo h;
      fill_halo(c, &h);
      if (c->cfg.exchange(c->cfg.exchange_user, &h) != 0) return ISING_SR_E_NCCL;
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

ising_sr_status ising_sr_commit(ising_sr_ctx* c, int64_t* events_out) {
  ising_sr_status s = check(c);
  if (s) return s;
  if (!c->in_window || !c->converged) return ISING_SR_E_STATE;
  const int fin = c->g & 1;
  if (c->cfg.flags & ISING_SR_FLAG_LOG_EVENTS) {
    const StateView& s0 = c->st[c->comm];
    const StateView& s1 = c->st[c->comm ^ 1];
    const int nb = (c->nreg + kThreads - 1) / kThreads;
    scan_block_sums<<<nb, kThreads, 0, c->stream>>>(s1.n, s0.n, c->nreg, c->d_bsum);
    scan_top<<<1, 1024, 0, c->stream>>>(c->d_bsum, nb, c->d_total);
    scan_apply<<<nb, kThreads, 0, c->stream>>>(s1.n, s0.n, c->nreg, c->d_bsum, c->d_off);
    c->launches += 3;
    CK(c, cudaGetLastError());
    unsigned long long total = 0;
    CK(c, cudaMemcpyAsync(&total, c->d_total, sizeof total, cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    if ((long long)total > c->log_cap) {
      cudaFree(c->log_t);
      cudaFree(c->log_region);
      cudaFree(c->log_site);
      c->log_t = nullptr;
      c->log_region = nullptr;
      c->log_site = nullptr;
      const long long cap = std::max<long long>((long long)total * 5 / 4 + 1024, c->log_cap * 2);
      if (dmalloc(&c->log_t, cap) != cudaSuccess || dmalloc(&c->log_region, cap) != cudaSuccess ||
          dmalloc(&c->log_site, cap) != cudaSuccess) {
        cudaGetLastError();
        c->log_cap = 0;
        return ISING_SR_E_OOM;
      }
      c->log_cap = cap;
    }
    KArgs a = base_args(c, fin, fin, false);
    a.log_t = c->log_t;
    a.log_region = c->log_region;
    a.log_site = c->log_site;
    a.log_off = c->d_off;
    c->ops->replay(a, c->nreg, c->stream);
    c->launches++;
    CK(c, cudaGetLastError());
    c->log_n = (long long)total;
    c->win_bytes += (double)total * 14.0 + (double)c->nreg * 8.0;
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
  c->stats.ms_last_window = ms;
  if (events_out) *events_out = (long long)c->win_events;
  return ISING_SR_OK;
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
  CK(c, cudaMalloc(&d, n));
  c->ops->unpack(c->st[c->comm], c->cfg.Lx, c->RX, c->RYl, d, c->stream);
  c->launches++;
  cudaError_t e = cudaMemcpyAsync(out, d, n, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(d);
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
    if (region) CK(c, cudaMemcpyAsync(region, c->log_region, m * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
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

int64_t ising_sr_launch_count(const ising_sr_ctx* c) { return c ? c->launches : 0; }

}  // extern "C"
