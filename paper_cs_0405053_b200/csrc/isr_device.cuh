// isr_device.cuh -- device arithmetic of the synchronous-relaxation n-fold way
// (arXiv cs/0405053) for sm_100a.  Independent of oracle/ (no shared code).
//
// Every floating-point operation on the dynamics path is an explicit IEEE
// round-to-nearest intrinsic (__dadd_rn, __dmul_rn, __ddiv_rn, ...) so that
// no FMA contraction or reassociation can change a result bit; the library is
// additionally compiled with -fmad=false.  The operation order is frozen in
// DESIGN.md §3 and matches the paper's formulas as cited below.
#pragma once
#include <cstdint>
#include <cstdio>

// ISR_CHECK=1 (a debugging build, tools/build_variants.py checked=-DISR_CHECK=1):
// bounds checks on the kernels' computed indices; a violation prints its
// location and traps, so the launch fails with a CUDA error
#ifndef ISR_CHECK
#define ISR_CHECK 0
#endif
#if ISR_CHECK
#define ISR_ASSERT(cond)                                                                              \
  do {                                                                                                \
    if (!(cond)) {                                                                                    \
      printf("ISR_ASSERT failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__, __LINE__,     \
             (int)blockIdx.x, (int)threadIdx.x);                                                      \
      __trap();                                                                                       \
    }                                                                                                 \
  } while (0)
#else
#define ISR_ASSERT(cond) \
  do {                   \
  } while (0)
#endif

namespace isr {

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al. 2011): the paper's "presimulated list" of
// random numbers, indexed rather than stored.
// Pair n of region i: key = (i, seed_lo), counter = (n_lo, n_hi, 0, seed_hi).
// ---------------------------------------------------------------------------
struct U4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    U4 n;
    n.x = __umulhi(0xCD9E8D57u, c.z) ^ c.y ^ k0;
    n.y = 0xCD9E8D57u * c.z;
    n.z = __umulhi(0xD2511F53u, c.x) ^ c.w ^ k1;
    n.w = 0xD2511F53u * c.x;
    c = n;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// 52 random bits -> (a + 0.5) * 2^-52 in [2^-53, 1 - 2^-53]; exact.
__device__ __forceinline__ double unit52(uint32_t hi, uint32_t lo) {
  const unsigned long long a = ((((unsigned long long)hi) << 32) | (unsigned long long)lo) >> 12;
  return __dmul_rn(__dadd_rn(__ull2double_rn(a), 0.5), 0x1p-52);
}

// gen: generation of the random numbers (counter word 2), 0 except in the
// alternate approach to subsequent steps, where window w uses w
__device__ __forceinline__ void draw_pair(unsigned long long seed, uint32_t region, uint32_t n,
                                          double& U, double& V, uint32_t gen = 0u) {
  U4 c{n, 0u, gen, (uint32_t)(seed >> 32)};
  const U4 x = philox4x32_10(c, region, (uint32_t)seed);
  U = unit52(x.x, x.y);
  V = unit52(x.z, x.w);
}

// ---------------------------------------------------------------------------
// E(U) = -log U with IEEE +,-,*,/ only: eq. nextau's exponential variate
// (P:247-252).  U = m 2^e, m in (sqrt2/2, sqrt2]; log m = 2 atanh(s),
// s = (m-1)/(m+1), series in z = s^2 to z^10.
// ---------------------------------------------------------------------------
// The series coefficients 1/(2j+3), j = 9 .. 0, then ln2 split hi/lo and the
// sqrt2 threshold, in constant memory: DMUL/DADD take them as c[bank][offset]
// operands (a 64-bit immediate costs two UMOVs per use on the draw path)
static __constant__ double kExpC[13] = {0x1.8618618618618p-5, 0x1.af286bca1af28p-5, 0x1.e1e1e1e1e1e1ep-5,
                                        0x1.1111111111111p-4, 0x1.3b13b13b13b14p-4, 0x1.745d1745d1746p-4,
                                        0x1.c71c71c71c71cp-4, 0x1.2492492492492p-3, 0x1.999999999999ap-3,
                                        0x1.5555555555555p-2, 0x1.62e42feep-1,      0x1.a39ef35793c76p-33,
                                        0x1.6a09e667f3bcdp+0};
__device__ __forceinline__ double expvar(double U) {
  const long long bits = __double_as_longlong(U);
  int e = (int)((bits >> 52) & 0x7ff) - 1023;
  double m = __longlong_as_double((bits & 0x000fffffffffffffLL) | 0x3ff0000000000000LL);
  if (m > kExpC[12]) {
    m = __dmul_rn(m, 0.5);
    e += 1;
  }
  const double f = __dsub_rn(m, 1.0);
  const double s = __ddiv_rn(f, __dadd_rn(2.0, f));
  const double z = __dmul_rn(s, s);
  double P = kExpC[0];
#pragma unroll
  for (int j = 1; j < 10; ++j) P = __dadd_rn(__dmul_rn(P, z), kExpC[j]);
  const double u = __dadd_rn(s, s);
  const double logm = __dadd_rn(u, __dmul_rn(u, __dmul_rn(z, P)));
  const double de = (double)e;
  const double logU = __dadd_rn(__dmul_rn(de, kExpC[10]), __dadd_rn(__dmul_rn(de, kExpC[11]), logm));
  return -logU;
}

// Candidate event time from budget R at rate lam starting at t (eq. nextau,
// and eq. newtau in remaining-budget form); +inf when lam == 0; a result that
// rounds onto t is bumped to the next double (reading R11).
__device__ __forceinline__ double cand_time(double t, double R, double lam) {
  if (lam == 0.0) return __longlong_as_double(0x7ff0000000000000LL);
  const double tau = __dadd_rn(t, __ddiv_rn(R, lam));
  return tau == t ? __longlong_as_double(__double_as_longlong(t) + 1) : tau;
}

// Per-region event digest step (R27): h <- (h ^ tau_bits) * K + site + 1,
// a bijection of h for fixed (tau, site), so a difference in any event of a
// sequence survives to the final digest.
__device__ __forceinline__ unsigned long long digest_step(unsigned long long h, double tau, int site) {
  return (h ^ (unsigned long long)__double_as_longlong(tau)) * 0x9E3779B97F4A7C15ULL + (unsigned long long)(site + 1);
}

}  // namespace isr
