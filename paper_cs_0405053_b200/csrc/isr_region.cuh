// isr_region.cuh -- the region-trajectory kernel (K1) and its commit-time
// log replay, lane-per-region form for regions of <= 64 sites.
//
// One CUDA thread owns one region G_i for one relaxation
// iteration: it regenerates the region's n-fold-way history over the window
// [t_c, t_w) (statement (a) of the relaxation loop) from the
// committed state, treating every boundary flip of a neighbour from the
// previous iteration as a break point, writes its own four edge
// histories (the "single layer of atoms that border its region")
// and, fused, compares them with its previous ones (statement (c)).
//
// Spins, ghost spins and the ten n-fold-way classes live in registers as bit
// masks over the region's sites (bit = local_row * BX + local_col); class
// counts N_k (eq. nidef) are popcounts of bit-sliced "number of up
// neighbours" planes, the j-th site of a class in local row-major order is a
// rank-select on the class mask (the linear order of P:280, R6).
#pragma once
#include <cstdint>
#include <type_traits>

#include "isr_device.cuh"

namespace isr {

enum : int { EDGE_N = 0, EDGE_S = 1, EDGE_W = 2, EDGE_E = 3 };

template <int BITS>
using uint_for = typename std::conditional<
    (BITS <= 8), uint8_t,
    typename std::conditional<(BITS <= 16), uint16_t,
                              typename std::conditional<(BITS <= 32), uint32_t, unsigned long long>::type>::type>::type;

template <int BX_, int BY_>
struct Geo {
  static constexpr int BX = BX_, BY = BY_, NS = BX * BY;
  static_assert(NS <= 64, "lane-per-region form holds <= 64 sites");
  using M = typename std::conditional<(NS <= 32), uint32_t, unsigned long long>::type;  // site mask
  using ST = uint_for<NS>;                   // stored spins
  using HT = uint_for<2 * BX + 2 * BY>;      // stored ghost bits: N[BX] S[BX] W[BY] E[BY]
  static constexpr M ONE = 1;
  __host__ __device__ static constexpr M full() {
    return NS >= (int)(8 * sizeof(M)) ? ~M(0) : (M)((M(1) << (NS % (8 * sizeof(M)))) - 1);
  }
  __host__ __device__ static constexpr M row0() { return (M(1) << BX) - 1; }
  __host__ __device__ static constexpr M col0() {
    M m = 0;
    for (int r = 0; r < BY; ++r) m |= M(1) << (r * BX);
    return m;
  }
  __host__ __device__ static constexpr M coll() { return col0() << (BX - 1); }
};

struct StateView {
  void* spins;
  void* halo;
  double* ts;
  double* R;
  uint32_t* n;
  unsigned long long* dig;
};

struct EdgeView {
  uint8_t* cnt;  // [4][rows_s][RX]
  double* t;     // [4][rows_s][K][RX]
  uint8_t* pos;  // [4][rows_s][K][RX]
};

struct KArgs {
  StateView in, out;
  EdgeView prev, cur;
  int RX, RYl, RYg, row0, world;
  int K;
  long long cstride;  // elements per edge in cnt  (rows_s * RX)
  long long tstride;  // elements per edge in t/pos (rows_s * K * RX)
  int first;          // iteration 1: canonical assumption
  int digest;
  double t_w;         // window end
  unsigned long long seed;
  double rate[10];
  int* flags;                   // [0] changed, [1] overflow
  unsigned long long* stats;    // [0] events [1] entries out [2] entries in [3] entries cmp [4] f max [5] regions
  // log replay
  double* log_t;
  uint32_t* log_region;
  uint16_t* log_site;
  const unsigned long long* log_off;
};

// bit-sliced per-site count of up neighbours: m[u] = sites with exactly u.
template <class G>
struct Classes {
  using M = typename G::M;
  M up, dn, m0, m1, m2, m3, m4;

  __device__ __forceinline__ void build(M spins, M gN, M gS, M gW, M gE, bool wrapX, bool wrapY) {
    constexpr M FULL = G::full();
    // neighbour-is-up masks for every site (periodic stencil)
    M nN = (M)((spins << G::BX) & FULL);
    M nS = (M)(spins >> G::BX);
    M nW = (M)((spins << 1) & FULL & ~G::col0());
    M nE = (M)((spins >> 1) & ~G::coll());
    if (wrapY) {  // region spans the lattice height: wrap inside the region
      nN |= (M)(spins >> ((G::BY - 1) * G::BX)) & G::row0();
      nS |= (M)((spins & G::row0()) << ((G::BY - 1) * G::BX));
    } else {
      nN |= gN;
      nS |= gS;
    }
    if (wrapX) {
      nW |= (M)(spins >> (G::BX - 1)) & G::col0();
      nE |= (M)((spins & G::col0()) << (G::BX - 1));
    } else {
      nW |= gW;
      nE |= gE;
    }
    // 4-input bit-sliced adder
    const M s1 = nN ^ nS, c1 = nN & nS;
    const M s2 = nW ^ nE, c2 = nW & nE;
    const M p0 = s1 ^ s2, k = s1 & s2;
    const M p1 = c1 ^ c2 ^ k;
    const M p2 = (c1 & c2) | (k & (c1 ^ c2));
    up = spins;
    dn = (M)(~spins) & FULL;
    m0 = (M)(~(p0 | p1 | p2)) & FULL;
    m1 = p0 & ~p1;
    m2 = ~p0 & p1;
    m3 = p0 & p1;
    m4 = p2;
  }
  __device__ __forceinline__ M mask(int k) const {
    const M s = k >= 5 ? up : dn;
    const int u = k >= 5 ? k - 5 : k;
    const M mu = u == 0 ? m0 : u == 1 ? m1 : u == 2 ? m2 : u == 3 ? m3 : m4;
    return s & mu;
  }
};

template <class M>
__device__ __forceinline__ int popc_m(M x) {
  if constexpr (sizeof(M) == 8) return __popcll(x);
  else return __popc(x);
}

// j-th (0-based) set bit of x, LSB first (local row-major order)
template <class M>
__device__ __forceinline__ int nth_bit(M x, int j) {
  if constexpr (sizeof(M) == 8) {
    const uint32_t lo = (uint32_t)x;
    const int pl = __popc(lo);
    if (j < pl) return (int)__fns(lo, 0, j + 1);
    return 32 + (int)__fns((uint32_t)(x >> 32), 0, j - pl + 1);
  } else {
    return (int)__fns((uint32_t)x, 0, j + 1);
  }
}

// eq. biglambda, fixed fold order (R3): c_k = c_{k-1} + N_k r_k
template <class G>
__device__ __forceinline__ double fold_lambda(const Classes<G>& C, const double* rate) {
  double c = 0.0;
#pragma unroll
  for (int k = 0; k < 10; ++k) c = __dadd_rn(c, __dmul_rn((double)popc_m(C.mask(k)), rate[k]));
  return c;
}

// Phases 2-3 of atom selection (eqs. Wsum, Wstop, nores, vindex)
// in x = V*Lambda space: k* = first k with x <= c_k,
// j = min(floor((x - c_{k*-1}) / r_k*), N_k* - 1); returns the local site.
template <class G>
__device__ __forceinline__ int select_site(const Classes<G>& C, const double* rate, double V, double lam) {
  const double x = __dmul_rn(V, lam);
  double c = 0.0, cprev = 0.0;
  int ks = -1;
#pragma unroll
  for (int k = 0; k < 10; ++k) {
    const double cn = __dadd_rn(c, __dmul_rn((double)popc_m(C.mask(k)), rate[k]));
    if (ks < 0 && x <= cn) {
      ks = k;
      cprev = c;
    }
    c = cn;
  }
  if (ks < 0) {  // unreachable for V < 1 (x <= Lambda = c_9)
    ks = 9;
    while (ks > 0 && popc_m(C.mask(ks)) == 0) --ks;
    cprev = 0.0;
  }
  const typename G::M mk = C.mask(ks);
  const int nk = popc_m(mk);
  long long j = (long long)floor(__ddiv_rn(__dsub_rn(x, cprev), rate[ks]));
  if (j > nk - 1) j = nk - 1;
  if (j < 0) j = 0;
  return nth_bit(mk, (int)j);
}

// Expand/compress the stored ghost bits (N[BX] S[BX] W[BY] E[BY]) to/from
// site-position masks (bit of the in-region site adjacent to the ghost).
template <class G>
__device__ __forceinline__ void expand_halo(unsigned long long h, typename G::M& gN, typename G::M& gS,
                                            typename G::M& gW, typename G::M& gE) {
  using M = typename G::M;
  constexpr int BX = G::BX, BY = G::BY;
  const M lowx = (M)((1ull << BX) - 1);
  gN = (M)h & lowx;
  gS = (M)(((M)(h >> BX) & lowx) << ((BY - 1) * BX));
  gW = 0;
  gE = 0;
#pragma unroll
  for (int r = 0; r < BY; ++r) {
    gW |= (M)((h >> (2 * BX + r)) & 1ull) << (r * BX);
    gE |= (M)((h >> (2 * BX + BY + r)) & 1ull) << (r * BX + BX - 1);
  }
}

template <class G>
__device__ __forceinline__ unsigned long long compress_halo(typename G::M gN, typename G::M gS, typename G::M gW,
                                                            typename G::M gE) {
  constexpr int BX = G::BX, BY = G::BY;
  const unsigned long long lowx = (1ull << BX) - 1;
  unsigned long long h = (unsigned long long)gN & lowx;
  h |= ((unsigned long long)(gS >> ((BY - 1) * BX)) & lowx) << BX;
#pragma unroll
  for (int r = 0; r < BY; ++r) {
    h |= (unsigned long long)((gW >> (r * BX)) & 1) << (2 * BX + r);
    h |= (unsigned long long)((gE >> (r * BX + BX - 1)) & 1) << (2 * BX + BY + r);
  }
  return h;
}

__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7ff0000000000000LL); }

// ---------------------------------------------------------------------------
// K1: one relaxation iteration for every region of the shard (LOG = false),
// or the commit-time replay that writes the compact event log (LOG = true).
// ---------------------------------------------------------------------------
template <int BX, int BY, bool LOG>
__global__ void __launch_bounds__(128) region_kernel(const KArgs a) {
  using G = Geo<BX, BY>;
  using M = typename G::M;
  using ST = typename G::ST;
  using HT = typename G::HT;

  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int nreg = a.RX * a.RYl;
  const bool live = idx < nreg;
  const int r = live ? idx / a.RX : 0;
  const int c = live ? idx - r * a.RX : 0;
  const bool wrapX = a.RX == 1, wrapY = a.RYg == 1;
  const uint32_t gid = (uint32_t)((a.row0 + r) * a.RX + c);

  unsigned long long n_ev = 0, n_out = 0, n_in = 0, n_cmp = 0, n_bev = 0;
  bool changed = false, overflow = false;

  if (live) {
    // ---- committed state (the old tau_m becomes tau_0) ----
    M spins = (M)((const ST*)a.in.spins)[idx];
    M gN, gS, gW, gE;
    expand_halo<G>((unsigned long long)((const HT*)a.in.halo)[idx], gN, gS, gW, gE);
    double ts = a.in.ts[idx];
    double R = a.in.R[idx];
    uint32_t n = a.in.n[idx];
    unsigned long long dig = a.digest ? a.in.dig[idx] : 0ull;

    // ---- incoming boundary histories of the previous iteration ----
    // direction d's neighbour wrote them as its opposite edge (d ^ 1).
    const int srow = r + 1;  // storage row of my region row
    int nrow[4], ncol[4];
    uint32_t nid[4];
    {
      const int rn = a.world == 1 ? ((r - 1 + a.RYl) % a.RYl) + 1 : r;      // north neighbour row
      const int rs = a.world == 1 ? ((r + 1) % a.RYl) + 1 : r + 2;          // south neighbour row
      const int gr = a.row0 + r;
      nrow[EDGE_N] = rn; ncol[EDGE_N] = c; nid[EDGE_N] = (uint32_t)(((gr - 1 + a.RYg) % a.RYg) * a.RX + c);
      nrow[EDGE_S] = rs; ncol[EDGE_S] = c; nid[EDGE_S] = (uint32_t)(((gr + 1) % a.RYg) * a.RX + c);
      const int cw = (c - 1 + a.RX) % a.RX, ce = (c + 1) % a.RX;
      nrow[EDGE_W] = srow; ncol[EDGE_W] = cw; nid[EDGE_W] = (uint32_t)(gr * a.RX + cw);
      nrow[EDGE_E] = srow; ncol[EDGE_E] = ce; nid[EDGE_E] = (uint32_t)(gr * a.RX + ce);
    }
    int hcnt[4], hidx[4], hpos[4];
    double ht[4];
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      const bool axis_off = (d < 2) ? wrapY : wrapX;
      hcnt[d] = (a.first || axis_off) ? 0
                : (int)a.prev.cnt[(long long)(d ^ 1) * a.cstride + (long long)nrow[d] * a.RX + ncol[d]];
      hidx[d] = 0;
      ht[d] = dinf();
      hpos[d] = 0;
      if (hcnt[d] > 0) {
        const long long off = (long long)(d ^ 1) * a.tstride + ((long long)nrow[d] * a.K) * a.RX + ncol[d];
        ht[d] = a.prev.t[off];
        hpos[d] = a.prev.pos[off];
      }
      n_in += hcnt[d];
    }
    // own previous histories (for the fused diff)
    int oc[4], pc[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      oc[e] = 0;
      pc[e] = (LOG || a.first) ? 0 : (int)a.prev.cnt[(long long)e * a.cstride + (long long)srow * a.RX + c];
    }
    const unsigned long long log_base = LOG ? a.log_off[idx] : 0ull;

    // pair n: U already spent into R (carried), V selects the next atom
    double U, V;
    draw_pair(a.seed, gid, n, U, V);
    Classes<G> C;
    C.build(spins, gN, gS, gW, gE, wrapX, wrapY);
    double lam = fold_lambda<G>(C, a.rate);
    double tc = cand_time(ts, R, lam);

    for (;;) {
      // earliest pending break point, (time, neighbour id) order (R10)
      int dstar = -1;
      double tb = dinf();
      uint32_t nb = 0xffffffffu;
#pragma unroll
      for (int d = 0; d < 4; ++d) {
        if (hidx[d] < hcnt[d] && (ht[d] < tb || (ht[d] == tb && nid[d] < nb))) {
          dstar = d;
          tb = ht[d];
          nb = nid[d];
        }
      }
      const bool bp = dstar >= 0 && (tb < tc || (tb == tc && nb < gid));
      const bool ev = !bp && tc < a.t_w;
      if (!bp && !ev) break;
      double tnew;
      if (ev) {
        // ---- own event at tc ----
        const int site = select_site<G>(C, a.rate, V, lam);
        spins ^= G::ONE << site;
        tnew = tc;
        const int sr = site / BX, sc = site - sr * BX;
        if (a.digest) {
          dig = mix64(mix64(dig ^ (unsigned long long)__double_as_longlong(tc)) ^ (unsigned long long)site);
        }
        if (LOG) {
          const unsigned long long o = log_base + n_ev;
          a.log_t[o] = tc;
          a.log_region[o] = gid;
          a.log_site[o] = (uint16_t)site;
        } else {
          // own boundary history
          bool bev = false;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const bool on = e == EDGE_N ? (!wrapY && sr == 0)
                          : e == EDGE_S ? (!wrapY && sr == BY - 1)
                          : e == EDGE_W ? (!wrapX && sc == 0)
                                        : (!wrapX && sc == BX - 1);
            if (on) {
              bev = true;
              const int k = oc[e];
              const uint8_t p = (uint8_t)(e < 2 ? sc : sr);
              if (k < a.K) {
                const long long off = (long long)e * a.tstride + ((long long)srow * a.K + k) * a.RX + c;
                a.cur.t[off] = tc;
                a.cur.pos[off] = p;
                if (k >= pc[e]) {
                  changed = true;
                } else {
                  ++n_cmp;
                  const double pt = a.prev.t[off];
                  const uint8_t pp = a.prev.pos[off];
                  if (__double_as_longlong(pt) != __double_as_longlong(tc) || pp != p) changed = true;
                }
              } else {
                overflow = true;
              }
              oc[e] = k + 1;
            }
          }
          n_bev += bev ? 1 : 0;
        }
        ++n_ev;
      } else {
        // ---- break point at tb (eqs. lambdataua..newtau) ----
        double Rn = __dsub_rn(R, __dmul_rn(lam, __dsub_rn(tb, ts)));
        R = Rn < 0.0 ? 0.0 : Rn;
        tnew = tb;
        // toggle the ghost spin and advance that history's cursor; unrolled
        // over the four directions so the cursor state stays in registers
#pragma unroll
        for (int d = 0; d < 4; ++d) {
          if (d == dstar) {
            const int p = hpos[d];
            if (d == EDGE_N) gN ^= G::ONE << p;
            else if (d == EDGE_S) gS ^= G::ONE << ((BY - 1) * BX + p);
            else if (d == EDGE_W) gW ^= G::ONE << (p * BX);
            else gE ^= G::ONE << (p * BX + BX - 1);
            const int nx = ++hidx[d];
            if (nx < hcnt[d]) {
              const long long off =
                  (long long)(d ^ 1) * a.tstride + ((long long)nrow[d] * a.K + nx) * a.RX + ncol[d];
              ht[d] = a.prev.t[off];
              hpos[d] = a.prev.pos[off];
            }
          }
        }
      }
      ts = tnew;
      C.build(spins, gN, gS, gW, gE, wrapX, wrapY);
      lam = fold_lambda<G>(C, a.rate);
      if (ev) {
        // next pair of the list; the unused remainder carries over
        ++n;
        draw_pair(a.seed, gid, n, U, V);
        R = expvar(U);
      }
      tc = cand_time(ts, R, lam);
    }

    if (!LOG) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (oc[e] != pc[e]) changed = true;
        a.cur.cnt[(long long)e * a.cstride + (long long)srow * a.RX + c] = (uint8_t)(oc[e] < a.K ? oc[e] : a.K);
        n_out += oc[e];
      }
      // tentative end-of-window state (committed by pointer swap at commit)
      ((ST*)a.out.spins)[idx] = (ST)spins;
      ((HT*)a.out.halo)[idx] = (HT)compress_halo<G>(gN, gS, gW, gE);
      a.out.ts[idx] = ts;
      a.out.R[idx] = R;
      a.out.n[idx] = n;
      if (a.digest) a.out.dig[idx] = dig;
    }
  }

  if (!LOG) {
    // warp-aggregated flags and counters (one atomic per warp)
    const unsigned full = 0xffffffffu;
    const unsigned anych = __ballot_sync(full, changed);
    const unsigned anyov = __ballot_sync(full, overflow);
    unsigned long long v0 = n_ev, v1 = n_out, v2 = n_in, v3 = n_cmp;
    unsigned fmax = (unsigned)n_bev;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      v0 += __shfl_xor_sync(full, v0, o);
      v1 += __shfl_xor_sync(full, v1, o);
      v2 += __shfl_xor_sync(full, v2, o);
      v3 += __shfl_xor_sync(full, v3, o);
      fmax = max(fmax, __shfl_xor_sync(full, fmax, o));
    }
    const unsigned nlive = __popc(__ballot_sync(full, live));
    if ((threadIdx.x & 31) == 0) {
      if (anych) atomicOr(&a.flags[0], 1);
      if (anyov) atomicOr(&a.flags[1], 1);
      if (nlive) {
        atomicAdd(&a.stats[0], v0);
        atomicAdd(&a.stats[1], v1);
        atomicAdd(&a.stats[2], v2);
        atomicAdd(&a.stats[3], v3);
        atomicMax(&a.stats[4], (unsigned long long)fmax);
        atomicAdd(&a.stats[5], (unsigned long long)nlive);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K0: pack the strip's spins (+1 halo row above and below, periodic) into
// region bit masks and ghost bits; tau_0 = 0 and R = E(U_0).
// buf: (RYl*BY + 2) rows x Lx, row 0 = lattice row above the strip.
// ---------------------------------------------------------------------------
template <int BX, int BY>
__global__ void init_kernel(const uint8_t* buf, int Lx, int RX, int RYl, int row0, unsigned long long seed,
                            StateView st) {
  using G = Geo<BX, BY>;
  using M = typename G::M;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= RX * RYl) return;
  const int r = idx / RX, c = idx - r * RX;
  const int y0 = 1 + r * BY, x0 = c * BX;
  M s = 0;
  unsigned long long h = 0;
  for (int ly = 0; ly < BY; ++ly)
    for (int lx = 0; lx < BX; ++lx)
      if (buf[(long long)(y0 + ly) * Lx + x0 + lx]) s |= G::ONE << (ly * BX + lx);
  for (int lx = 0; lx < BX; ++lx) {
    if (buf[(long long)(y0 - 1) * Lx + x0 + lx]) h |= 1ull << lx;
    if (buf[(long long)(y0 + BY) * Lx + x0 + lx]) h |= 1ull << (BX + lx);
  }
  for (int ly = 0; ly < BY; ++ly) {
    if (buf[(long long)(y0 + ly) * Lx + (x0 - 1 + Lx) % Lx]) h |= 1ull << (2 * BX + ly);
    if (buf[(long long)(y0 + ly) * Lx + (x0 + BX) % Lx]) h |= 1ull << (2 * BX + BY + ly);
  }
  ((typename G::ST*)st.spins)[idx] = (typename G::ST)s;
  ((typename G::HT*)st.halo)[idx] = (typename G::HT)h;
  double U, V;
  draw_pair(seed, (uint32_t)((row0 + r) * RX + c), 0u, U, V);
  st.ts[idx] = 0.0;
  st.R[idx] = expvar(U);
  st.n[idx] = 0;
  st.dig[idx] = 0ull;
}

// unpack committed region spins to a row-major uint8 strip
template <int BX, int BY>
__global__ void unpack_kernel(StateView st, int Lx, int RX, int RYl, uint8_t* out) {
  using G = Geo<BX, BY>;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nsite = (long long)RYl * BY * Lx;
  if (i >= nsite) return;
  const int y = (int)(i / Lx), x = (int)(i - (long long)y * Lx);
  const int r = y / BY, c = x / BX;
  const typename G::M s = (typename G::M)((const typename G::ST*)st.spins)[r * RX + c];
  out[i] = (uint8_t)((s >> ((y - r * BY) * BX + (x - c * BX))) & 1);
}

}  // namespace isr
