// Second workload: checkerboard Metropolis sweeps -- the
// discrete-time dynamics of the paper's §2: a visited atom v
// flips with probability p(v) = p_k of its class k = 5(s+1)/2 + u (eq. p,
// P:166-181), else keeps its spin.  Visiting order: the two-colour sweep,
// first every site with (x + y) even, then every site with (x + y) odd;
// sites of one colour share no bond, so one colour is one data-parallel pass.
// Site i = y Lx + x in global sweep s decides with Philox4x32-10, key =
// (0xFFFFFFFE, seed_lo), counter = (i, s_lo, s_hi, seed_hi), U from words
// (x0, x1) exactly as the n-fold way's pairs (isr_device.cuh): flip iff
// U < p_k.  include/ising_sr.h documents the C ABI.
//
// The pass is bound by integer issue (one Philox-10 per visited site), not
// by HBM: a thread owns one aligned 4-byte word of a row (2 sites of the
// colour), reads it and the words above and below (coalesced), the two
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

__device__ __forceinline__ bool decide(const double* p, unsigned long long seed, uint32_t site,
                                       unsigned long long sweep, int k) {
  U4 c{site, (uint32_t)sweep, (uint32_t)(sweep >> 32), (uint32_t)(seed >> 32)};
  const U4 x = philox4x32_10(c, 0xFFFFFFFEu, (uint32_t)seed);
  return unit52(x.x, x.y) < p[k];
}

__device__ __forceinline__ void block_count(unsigned long long n, unsigned long long* flips) {
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
                                                          unsigned long long* flips) {
  const int wpr = Lx >> 2;  // words per row
  const long long nw = (long long)wpr * Ly;
  uint32_t* W = reinterpret_cast<uint32_t*>(spins);
  ISR_CB_STAGE_PROBS(P, p)
  unsigned long long n = 0;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < nw; t += (long long)gridDim.x * blockDim.x) {
    const int y = (int)(t / wpr), j = (int)(t - (long long)y * wpr);
    const int yu = y == 0 ? Ly - 1 : y - 1, yd = y == Ly - 1 ? 0 : y + 1;
    const uint32_t w = nz_bytes(__ldcg(W + t));
    const uint32_t wu = nz_bytes(__ldcg(W + (long long)yu * wpr + j));
    const uint32_t wd = nz_bytes(__ldcg(W + (long long)yd * wpr + j));
    const int x0 = j << 2;
    const uint8_t* row = spins + (long long)y * Lx;
    const uint32_t bl = row[x0 == 0 ? Lx - 1 : x0 - 1] != 0;
    const uint32_t br = row[x0 + 4 == Lx ? 0 : x0 + 4] != 0;
    // horizontal neighbours of each byte: (w << 8 | bl) and (w >> 8 | br << 24)
    const uint32_t left = (w << 8) | bl, right = (w >> 8) | (br << 24);
    const uint32_t ups = wu + wd + left + right;  // per byte: up neighbours, 0..4 (no carries)
    const int o = (y + colour) & 1;               // first byte of the colour in this word
    uint32_t out = w;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int b = o + 2 * h;
      const int s = (int)((w >> (8 * b)) & 1u);
      const int k = 5 * s + (int)((ups >> (8 * b)) & 0xFFu);
      if (decide(p, seed, (uint32_t)((long long)y * Lx + x0 + b), sweep, k)) {
        out ^= 1u << (8 * b);
        ++n;
      }
    }
    if (out != __ldcg(W + t)) W[t] = out;
  }
  block_count(n, flips);
}

// site form (any even Lx): thread = one site of the colour
__global__ void __launch_bounds__(kThreads) half_sweep_s(uint8_t* spins, int Lx, int Ly, Probs P,
                                                          unsigned long long seed, unsigned long long sweep, int colour,
                                                          unsigned long long* flips) {
  const int hx = Lx >> 1;
  const long long ns = (long long)hx * Ly;
  ISR_CB_STAGE_PROBS(P, p)
  unsigned long long n = 0;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < ns; t += (long long)gridDim.x * blockDim.x) {
    const int y = (int)(t / hx);
    const int x = 2 * (int)(t - (long long)y * hx) + ((y + colour) & 1);
    const int yu = y == 0 ? Ly - 1 : y - 1, yd = y == Ly - 1 ? 0 : y + 1;
    const int xl = x == 0 ? Lx - 1 : x - 1, xr = x == Lx - 1 ? 0 : x + 1;
    const long long i = (long long)y * Lx + x;
    const uint8_t v = spins[i];
    const int up = (spins[(long long)yu * Lx + x] != 0) + (spins[(long long)yd * Lx + x] != 0) +
                   (spins[(long long)y * Lx + xl] != 0) + (spins[(long long)y * Lx + xr] != 0);
    const int s = v != 0;
    const bool f = decide(p, seed, (uint32_t)i, sweep, 5 * s + up);
    n += f;
    const uint8_t nv = (uint8_t)(f ? 1 - s : s);
    if (nv != v) spins[i] = nv;
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
  if ((long long)Lx * Ly > 0xffffffffLL) return ISING_SR_E_INVALID_ARG;  // site ids are 32-bit counters
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
  const long long items = word ? (long long)(Lx >> 2) * Ly : (long long)(Lx >> 1) * Ly;
  const int grid = grid_for(items);
  for (int64_t q = 0; q < nsweeps; ++q) {
    const unsigned long long sw = (unsigned long long)(sweep0 + q);
    for (int colour = 0; colour < 2; ++colour) {
      if (word)
        half_sweep_w<<<grid, kThreads, 0, s>>>(d_spins, Lx, Ly, P, seed, sw, colour, (unsigned long long*)d_flips);
      else
        half_sweep_s<<<grid, kThreads, 0, s>>>(d_spins, Lx, Ly, P, seed, sw, colour, (unsigned long long*)d_flips);
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
