// Second workload: checkerboard Metropolis sweeps -- the
// discrete-time dynamics of the paper's §2: a visited atom v
// flips with probability p(v) = p_k of its class k = 5(s+1)/2 + u (eq. p,
// P:166-181), else keeps its spin.  Visiting order: the two-colour sweep,
// first every site with (x + y) even, then every site with (x + y) odd;
// sites of one colour share no bond, so one colour is one data-parallel pass.
// Random numbers (R29): in row y the sites of colour c are
// numbered j = 0, 1, ... in increasing x; sites 2m and 2m+1 share one
// Philox4x32-10 draw, key = (0xFFFFFFFE, seed_lo), counter = (q, s_lo,
// s_hi | c << 31, seed_hi), q = y ceil(Lx/4) + m; site 2m takes U from words
// (x0, x1), site 2m+1 from (x2, x3), mapped exactly as the n-fold way's pairs
// (isr_device.cuh); a site flips iff U < p_k.  include/ising_sr.h documents
// the C ABI.
//
// The pass is bound by integer issue (one Philox-10 per two visited sites),
// not by HBM: a thread owns one aligned 4-byte word of a row (the 2 sites of
// the colour that share a draw), reads it and the words above and below (coalesced), the two
// bytes left and right of it (L1 hits: the neighbouring lanes' words), and
// writes the word back only when a site flipped.  Grid-stride over the
// lattice's words, one flip-count atomic per block.
#include <cstdint>
#include <cuda_runtime.h>

#include "isr_device.cuh"
#include "../../include/ising_sr.h"

namespace isr {
namespace cb {

struct Probs {
  double p[10];
};

constexpr int kThreads = 256;

// i / d == (i * M) >> k for every i < 2^31 (k = 31 + ceil(log2 d), M = ceil(2^k / d))
struct Div {
  unsigned M;
  int k;
  __device__ __forceinline__ unsigned operator()(unsigned i) const {
    return (unsigned)(((unsigned long long)i * M) >> k);
  }
};
Div make_div(unsigned d) {
  int l = 0;
  while ((1ull << l) < d) ++l;
  Div v;
  v.k = 31 + l;
  v.M = (unsigned)(((1ull << v.k) + d - 1) / d);
  return v;
}

// 0x01 in every nonzero byte of w
__device__ __forceinline__ uint32_t nz_bytes(uint32_t w) {
  return (((w & 0x7f7f7f7fu) + 0x7f7f7f7fu) | w) >> 7 & 0x01010101u;
}

// the flip probabilities in shared memory (indexed by class at run time);
// a macro so that the kernel parameter is read in place (no local copy)
#define ISR_CB_STAGE_PROBS(P, sp)                                                          \
  __shared__ double sp[10];                                                                \
  if (threadIdx.x == 0) {                                                                  \
    sp[0] = P.p[0]; sp[1] = P.p[1]; sp[2] = P.p[2]; sp[3] = P.p[3]; sp[4] = P.p[4];        \
    sp[5] = P.p[5]; sp[6] = P.p[6]; sp[7] = P.p[7]; sp[8] = P.p[8]; sp[9] = P.p[9];        \
  }                                                                                        \
  __syncthreads();

// the draw shared by sites 2m and 2m+1 of colour `colour` in a row (q = y ceil(Lx/4) + m)
__device__ __forceinline__ U4 draw_cb(unsigned long long seed, uint32_t q, unsigned long long sweep, int colour) {
  U4 c{q, (uint32_t)sweep, (uint32_t)(sweep >> 32) | ((uint32_t)colour << 31), (uint32_t)(seed >> 32)};
  return philox4x32_10(c, 0xFFFFFFFEu, (uint32_t)seed);
}

__device__ __forceinline__ void block_count(unsigned n32, unsigned long long* flips) {
  unsigned long long n = n32;
  __shared__ unsigned long long part[kThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = n;
  __syncthreads();
  if (threadIdx.x == 0 && flips) {
    unsigned long long t = 0;
    for (int w = 0; w < kThreads / 32; ++w) t += part[w];
    if (t) atomicAdd(flips, t);
  }
}

// word form (Lx % 4 == 0): thread = one aligned word of 4 sites
__global__ void __launch_bounds__(kThreads) half_sweep_w(uint8_t* spins, int Lx, int Ly, Probs P,
                                                          unsigned long long seed, unsigned long long sweep, int colour,
                                                          unsigned long long* flips, Div dw) {
  const int wpr = Lx >> 2;  // words per row
  const unsigned nw = (unsigned)wpr * (unsigned)Ly;  // < 2^30
  uint32_t* W = reinterpret_cast<uint32_t*>(spins);
  ISR_CB_STAGE_PROBS(P, p)
  unsigned n = 0;
  for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < nw; t += gridDim.x * blockDim.x) {
    const int y = (int)dw(t), j = (int)(t - (unsigned)y * wpr);
    const int yu = y == 0 ? Ly - 1 : y - 1, yd = y == Ly - 1 ? 0 : y + 1;
    const uint32_t w = nz_bytes(__ldcg(W + t));
    const uint32_t wu = nz_bytes(__ldcg(W + ((unsigned)yu * wpr + j)));
    const uint32_t wd = nz_bytes(__ldcg(W + ((unsigned)yd * wpr + j)));
    const int x0 = j << 2;
    const uint8_t* row = spins + (unsigned)y * Lx;
    const uint32_t bl = row[x0 == 0 ? Lx - 1 : x0 - 1] != 0;
    const uint32_t br = row[x0 + 4 == Lx ? 0 : x0 + 4] != 0;
    // horizontal neighbours of each byte: (w << 8 | bl) and (w >> 8 | br << 24)
    const uint32_t left = (w << 8) | bl, right = (w >> 8) | (br << 24);
    const uint32_t ups = wu + wd + left + right;  // per byte: up neighbours, 0..4 (no carries)
    const int o = (y + colour) & 1;               // first byte of the colour in this word
    const U4 r = draw_cb(seed, (uint32_t)t, sweep, colour);  // q = y (Lx/4) + j = t: sites 2t', 2t'+1 of the row
    uint32_t out = w;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int b = o + 2 * h;
      const int s = (int)((w >> (8 * b)) & 1u);
      const int k = 5 * s + (int)((ups >> (8 * b)) & 0xFFu);
      const double U = h ? unit52(r.z, r.w) : unit52(r.x, r.y);
      if (U < p[k]) {
        out ^= 1u << (8 * b);
        ++n;
      }
    }
    if (out != __ldcg(W + t)) W[t] = out;
  }
  block_count(n, flips);
}

// site form (any even Lx): thread = the (one or two) sites of the colour
// that share a draw
__global__ void __launch_bounds__(kThreads) half_sweep_s(uint8_t* spins, int Lx, int Ly, Probs P,
                                                          unsigned long long seed, unsigned long long sweep, int colour,
                                                          unsigned long long* flips, Div dq) {
  const int hx = Lx >> 1, ppr = (Lx + 2) >> 2;  // sites of the colour per row, draws per row
  const unsigned nq = (unsigned)ppr * (unsigned)Ly;  // < 2^31
  ISR_CB_STAGE_PROBS(P, p)
  unsigned n = 0;
  for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < nq; t += gridDim.x * blockDim.x) {
    const int y = (int)dq(t), m = (int)(t - (unsigned)y * ppr);
    const int yu = y == 0 ? Ly - 1 : y - 1, yd = y == Ly - 1 ? 0 : y + 1;
    const U4 r = draw_cb(seed, (uint32_t)t, sweep, colour);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = 2 * m + h;
      if (j >= hx) break;
      const int x = 2 * j + ((y + colour) & 1);
      const int xl = x == 0 ? Lx - 1 : x - 1, xr = x == Lx - 1 ? 0 : x + 1;
      const unsigned i = (unsigned)y * Lx + x;  // < 2^32
      const uint8_t v = spins[i];
      const int up = (spins[(unsigned)yu * Lx + x] != 0) + (spins[(unsigned)yd * Lx + x] != 0) +
                     (spins[(unsigned)y * Lx + xl] != 0) + (spins[(unsigned)y * Lx + xr] != 0);
      const int s = v != 0;
      const double U = h ? unit52(r.z, r.w) : unit52(r.x, r.y);
      const bool f = U < p[5 * s + up];
      n += f;
      const uint8_t nv = (uint8_t)(f ? 1 - s : s);
      if (nv != v) spins[i] = nv;
    }
  }
  block_count(n, flips);
}

int grid_for(long long items) {
  const long long g = (items + kThreads - 1) / kThreads;
  return (int)(g < 148LL * 16 ? (g < 1 ? 1 : g) : 148LL * 16);
}

ising_sr_status check_args(const uint8_t* spins, int32_t Lx, int32_t Ly, const double* p, int64_t sweep0,
                           int32_t nsweeps) {
  if (!spins || !p || nsweeps < 0 || sweep0 < 0) return ISING_SR_E_INVALID_ARG;
  if (Lx < 4 || Ly < 4 || (Lx & 1) || (Ly & 1)) return ISING_SR_E_DIMENSION;
  if ((long long)Lx * Ly > 0xffffffffLL) return ISING_SR_E_INVALID_ARG;  // draw ids are 32-bit counters
  if (sweep0 + (long long)nsweeps > 0x3fffffffffffffffLL) return ISING_SR_E_INVALID_ARG;  // the colour bit of s_hi
  for (int k = 0; k < 10; ++k)
    if (!(p[k] >= 0.0 && p[k] <= 1.0)) return ISING_SR_E_INVALID_ARG;
  return ISING_SR_OK;
}

}  // namespace cb
}  // namespace isr

extern "C" {

ising_sr_status ising_cb_sweeps(uint8_t* d_spins, int32_t Lx, int32_t Ly, const double p[10], uint64_t seed,
                                int64_t sweep0, int32_t nsweeps, uint64_t* d_flips, void* stream) {
  using namespace isr::cb;
  ising_sr_status st = check_args(d_spins, Lx, Ly, p, sweep0, nsweeps);
  if (st) return st;
  Probs P;
  for (int k = 0; k < 10; ++k) P.p[k] = p[k];
  cudaStream_t s = (cudaStream_t)stream;
  const bool word = (Lx & 3) == 0 && ((uintptr_t)d_spins & 3) == 0;
  const long long items = word ? (long long)(Lx >> 2) * Ly : (long long)((Lx + 2) >> 2) * Ly;
  const int grid = grid_for(items);
  const Div dv = make_div(word ? (unsigned)(Lx >> 2) : (unsigned)((Lx + 2) >> 2));
  for (int64_t q = 0; q < nsweeps; ++q) {
    const unsigned long long sw = (unsigned long long)(sweep0 + q);
    for (int colour = 0; colour < 2; ++colour) {
      if (word)
        half_sweep_w<<<grid, kThreads, 0, s>>>(d_spins, Lx, Ly, P, seed, sw, colour, (unsigned long long*)d_flips,
                                                dv);
      else
        half_sweep_s<<<grid, kThreads, 0, s>>>(d_spins, Lx, Ly, P, seed, sw, colour, (unsigned long long*)d_flips,
                                                dv);
    }
  }
  return cudaGetLastError() == cudaSuccess ? ISING_SR_OK : ISING_SR_E_CUDA;
}

ising_sr_status ising_cb_run(const uint8_t* spins_in, uint8_t* spins_out, int32_t Lx, int32_t Ly,
                             const double p[10], uint64_t seed, int64_t sweep0, int32_t nsweeps, int64_t* flips_out,
                             int32_t device) {
  using namespace isr::cb;
  if (!spins_in || !spins_out) return ISING_SR_E_INVALID_ARG;
  ising_sr_status st = check_args(spins_in, Lx, Ly, p, sweep0, nsweeps);
  if (st) return st;
  if (cudaSetDevice(device) != cudaSuccess) return ISING_SR_E_CUDA;
  const size_t n = (size_t)Lx * Ly;
  uint8_t* d = nullptr;
  unsigned long long* df = nullptr;
  if (cudaMalloc(&d, n) != cudaSuccess) return ISING_SR_E_OOM;
  if (cudaMalloc(&df, sizeof *df) != cudaSuccess) {
    cudaFree(d);
    return ISING_SR_E_OOM;
  }
  cudaError_t e = cudaMemcpy(d, spins_in, n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(df, 0, sizeof *df);
  if (e == cudaSuccess) st = ising_cb_sweeps(d, Lx, Ly, p, seed, sweep0, nsweeps, (uint64_t*)df, nullptr);
  unsigned long long f = 0;
  if (e == cudaSuccess && st == ISING_SR_OK) e = cudaMemcpy(spins_out, d, n, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && st == ISING_SR_OK) e = cudaMemcpy(&f, df, sizeof f, cudaMemcpyDeviceToHost);
  cudaFree(d);
  cudaFree(df);
  if (e != cudaSuccess) return ISING_SR_E_CUDA;
  if (st) return st;
  if (flips_out) *flips_out = (int64_t)f;
  return ISING_SR_OK;
}

}  // extern "C"
