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

// Boundary histories of one slot: cnt[4][RYl][RX], t/pos[4][RYl][K][RX].
// Every region edge has two slots; which one holds its latest history is
// recorded in the region's selector word (see latest_of).
struct EdgeView {
  uint8_t* cnt;
  double* t;
  uint8_t* pos;
};

// A ghost row received from a neighbouring strip (world > 1):
// cnt[RX], stamp[RX] (global iteration of the last change), t/pos[K][RX].
struct GhostView {
  uint8_t* cnt;
  uint32_t* stamp;
  double* t;
  uint8_t* pos;
};

struct KArgs {
  StateView in, out;
  EdgeView ed[2];
  unsigned long long* sel;      // per region selector word
  GhostView gh_up, gh_down;     // world > 1: rows above / below the strip
  int RX, RYl, RYg, row0, world;
  int K;
  long long cstride;  // elements per edge in cnt  (RYl * RX)
  long long tstride;  // elements per edge in t/pos (RYl * K * RX)
  unsigned it_K;      // global iteration stamp of this launch (>= 1)
  unsigned it_K0;     // stamp of the window's first iteration
  int first;          // window's first iteration: canonical assumption
  int digest;
  double t_w;         // window end
  unsigned long long seed;
  double rate[10];
  const uint32_t* wl_in;   // regions to recompute (nullptr: all regions)
  int n_work;              // number of regions to recompute
  uint32_t* wl_out;        // worklist of the next iteration
  unsigned* wl_out_count;
  uint32_t* dirty;         // per region: last stamp it was queued for
  int* flags;                   // [0] changed, [1] overflow
  unsigned long long* stats;    // [0] events [1] entries out [2] entries in [3] entries cmp [4] f max [5] regions
  // log replay
  double* log_t;
  uint32_t* log_region;
  uint16_t* log_site;
  const unsigned long long* log_off;
};

// Selector word of a region (64 bits, written only by its own thread, read
// racily by neighbours -- a 64-bit aligned store/load is single-copy atomic
// and both the old and the new value decode to the same answer):
//   bits 0-3  slot of the latest history of edge e
//   bits 4-7  edges changed at K_last
//   bits 8-11 edges holding a history written in this window (as of K_last)
//   bits 12-15 the same before the K_last change
//   bits 32-63 K_last, global iteration of the last change
// latest_of(): the edge's latest history as of the end of iteration K-1.
struct Latest {
  int slot;
  bool valid;  // false: canonical empty history
};

__device__ __forceinline__ Latest latest_of(unsigned long long v, int e, unsigned K, unsigned K0) {
  const unsigned Kl = (unsigned)(v >> 32);
  const unsigned slots = (unsigned)v & 0xF, ch = ((unsigned)v >> 4) & 0xF;
  const unsigned ne = ((unsigned)v >> 8) & 0xF, nep = ((unsigned)v >> 12) & 0xF;
  if (Kl < K0) return {0, false};
  if (Kl < K) return {(int)((slots >> e) & 1u), ((ne >> e) & 1u) != 0};
  return {(int)(((slots ^ ch) >> e) & 1u), ((nep >> e) & 1u) != 0};  // changed concurrently in K
}

__device__ __forceinline__ unsigned long long sel_after_change(unsigned long long v, unsigned chmask, unsigned K,
                                                               unsigned K0) {
  const unsigned Kl = (unsigned)(v >> 32);
  const unsigned slots = (unsigned)v & 0xF;
  const unsigned ne_old = Kl >= K0 ? (((unsigned)v >> 8) & 0xF) : 0u;
  const unsigned lo = (slots ^ chmask) | (chmask << 4) | ((ne_old | chmask) << 8) | (ne_old << 12);
  return ((unsigned long long)K << 32) | lo;
}

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
// K1: one relaxation iteration for the regions of the worklist (all regions
// in the window's first iteration), or the commit-time replay that writes
// the compact event log (LOG = true; all regions, latest histories).
//
// Only regions with a changed incoming history are recomputed: a region
// whose inputs did not change would regenerate exactly its previous history
// (the same presimulated random list), so skipping it does not
// change the iteration count g or any result.
// ---------------------------------------------------------------------------
template <int BX, int BY, bool LOG>
__global__ void __launch_bounds__(128) region_kernel(const KArgs a) {
  using G = Geo<BX, BY>;
  using M = typename G::M;
  using ST = typename G::ST;
  using HT = typename G::HT;

  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = tid < a.n_work;
  const int idx = live ? (a.wl_in ? (int)a.wl_in[tid] : tid) : 0;
  const int r = idx / a.RX;
  const int c = idx - r * a.RX;
  const bool wrapX = a.RX == 1, wrapY = a.RYg == 1;
  const uint32_t gid = (uint32_t)((a.row0 + r) * a.RX + c);
  const unsigned K = a.it_K, K0 = a.it_K0;

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

    // ---- incoming boundary histories (latest as of the previous iteration) ----
    // direction d's neighbour wrote them as its opposite edge (d ^ 1).
    const int gr = a.row0 + r;
    uint32_t nid[4];
    nid[EDGE_N] = (uint32_t)(((gr - 1 + a.RYg) % a.RYg) * a.RX + c);
    nid[EDGE_S] = (uint32_t)(((gr + 1) % a.RYg) * a.RX + c);
    nid[EDGE_W] = (uint32_t)(gr * a.RX + (c - 1 + a.RX) % a.RX);
    nid[EDGE_E] = (uint32_t)(gr * a.RX + (c + 1) % a.RX);
    // cursor of each incoming history, packed: cnt | idx << 8 | pos << 16 |
    // source << 24 (source 0/1 = slot, 2 = ghost row above, 3 = below);
    // hoff = element offset of entry 0, entry q at hoff + q * RX
    unsigned hm[4], hoff[4];
    double ht[4];
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      hm[d] = 0; hoff[d] = 0; ht[d] = dinf();
      const bool axis_off = (d < 2) ? wrapY : wrapX;
      if (a.first || axis_off) continue;
      const bool ghost = a.world > 1 && ((d == EDGE_N && r == 0) || (d == EDGE_S && r == a.RYl - 1));
      unsigned cnt = 0, src = 0;
      if (ghost) {
        const GhostView& g = d == EDGE_N ? a.gh_up : a.gh_down;
        cnt = g.cnt[c];
        src = d == EDGE_N ? 2u : 3u;
        hoff[d] = (unsigned)c;
      } else {
        const int nr = d == EDGE_N ? (r - 1 + a.RYl) % a.RYl : d == EDGE_S ? (r + 1) % a.RYl : r;
        const int nc = d == EDGE_W ? (c - 1 + a.RX) % a.RX : d == EDGE_E ? (c + 1) % a.RX : c;
        const unsigned long long v = __ldcg(&a.sel[(long long)nr * a.RX + nc]);
        const Latest L = latest_of(v, d ^ 1, K, K0);
        if (L.valid) {
          const EdgeView& E = L.slot ? a.ed[1] : a.ed[0];
          cnt = E.cnt[(long long)(d ^ 1) * a.cstride + (long long)nr * a.RX + nc];
          src = (unsigned)L.slot;
          hoff[d] = (unsigned)((long long)(d ^ 1) * a.tstride + ((long long)nr * a.K) * a.RX + nc);
        }
      }
      unsigned pos = 0;
      if (cnt > 0) {
        const double* T = src == 0 ? a.ed[0].t : src == 1 ? a.ed[1].t : src == 2 ? a.gh_up.t : a.gh_down.t;
        const uint8_t* P = src == 0 ? a.ed[0].pos : src == 1 ? a.ed[1].pos : src == 2 ? a.gh_up.pos : a.gh_down.pos;
        ht[d] = T[hoff[d]];
        pos = P[hoff[d]];
      }
      hm[d] = cnt | (pos << 16) | (src << 24);
      n_in += cnt;
    }

    // ---- own latest histories (fused diff, statement (c)) ----
    // packed per edge: new count | latest count << 8 | latest slot << 16 | diverged << 17
    const unsigned long long vown = LOG ? 0ull : a.sel[idx];
    unsigned om[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const unsigned ps = (unsigned)((vown >> e) & 1ull);
      unsigned pc = 0;
      if (!LOG) {
        const Latest L = latest_of(vown, e, K, K0);
        if (L.valid) pc = (ps ? a.ed[1] : a.ed[0]).cnt[(long long)e * a.cstride + (long long)r * a.RX + c];
      }
      om[e] = (pc << 8) | (ps << 16);
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
        const bool pend = ((hm[d] >> 8) & 0xFFu) < (hm[d] & 0xFFu);
        if (pend && (ht[d] < tb || (ht[d] == tb && nid[d] < nb))) {
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
          // own boundary history; an edge history is
          // written only once it diverges from its latest version
          bool bev = false;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const bool on = e == EDGE_N ? (!wrapY && sr == 0)
                          : e == EDGE_S ? (!wrapY && sr == BY - 1)
                          : e == EDGE_W ? (!wrapX && sc == 0)
                                        : (!wrapX && sc == BX - 1);
            if (on) {
              bev = true;
              const unsigned k = om[e] & 0xFFu;
              const unsigned pc = (om[e] >> 8) & 0xFFu;
              const unsigned ps = (om[e] >> 16) & 1u;
              bool dve = (om[e] >> 17) & 1u;
              const uint8_t p = (uint8_t)(e < 2 ? sc : sr);
              if ((int)k < a.K) {
                const long long base = (long long)e * a.tstride + ((long long)r * a.K) * a.RX + c;
                const EdgeView& Pold = ps ? a.ed[1] : a.ed[0];
                const EdgeView& Pnew = ps ? a.ed[0] : a.ed[1];
                bool same = false;
                if (!dve && k < pc) {
                  ++n_cmp;
                  same = __double_as_longlong(Pold.t[base + (long long)k * a.RX]) == __double_as_longlong(tc) &&
                         Pold.pos[base + (long long)k * a.RX] == p;
                }
                if (!same) {
                  if (!dve) {  // copy the agreeing prefix into the new slot
                    for (unsigned q = 0; q < k; ++q) {
                      Pnew.t[base + (long long)q * a.RX] = Pold.t[base + (long long)q * a.RX];
                      Pnew.pos[base + (long long)q * a.RX] = Pold.pos[base + (long long)q * a.RX];
                    }
                    dve = true;
                  }
                  Pnew.t[base + (long long)k * a.RX] = tc;
                  Pnew.pos[base + (long long)k * a.RX] = p;
                  ++n_out;
                }
              } else {
                overflow = true;
              }
              const unsigned kk = k < 255u ? k + 1 : 255u;
              om[e] = kk | (pc << 8) | (ps << 16) | ((unsigned)dve << 17);
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
            const int p = (int)((hm[d] >> 16) & 0xFFu);
            if (d == EDGE_N) gN ^= G::ONE << p;
            else if (d == EDGE_S) gS ^= G::ONE << ((BY - 1) * BX + p);
            else if (d == EDGE_W) gW ^= G::ONE << (p * BX);
            else gE ^= G::ONE << (p * BX + BX - 1);
            const unsigned nx = ((hm[d] >> 8) & 0xFFu) + 1;
            const unsigned src = hm[d] >> 24;
            unsigned pos = 0;
            if (nx < (hm[d] & 0xFFu)) {
              const double* T = src == 0 ? a.ed[0].t : src == 1 ? a.ed[1].t : src == 2 ? a.gh_up.t : a.gh_down.t;
              const uint8_t* P =
                  src == 0 ? a.ed[0].pos : src == 1 ? a.ed[1].pos : src == 2 ? a.gh_up.pos : a.gh_down.pos;
              const unsigned long long off = (unsigned long long)hoff[d] + (unsigned long long)nx * a.RX;
              ht[d] = T[off];
              pos = P[off];
            }
            hm[d] = (hm[d] & 0xFF0000FFu) | (nx << 8) | (pos << 16);
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
      unsigned chmask = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const unsigned oc = om[e] & 0xFFu, pc = (om[e] >> 8) & 0xFFu, ps = (om[e] >> 16) & 1u;
        bool dve = (om[e] >> 17) & 1u;
        if ((int)oc > a.K) overflow = true;
        const EdgeView& Pold = ps ? a.ed[1] : a.ed[0];
        const EdgeView& Pnew = ps ? a.ed[0] : a.ed[1];
        if (!dve && oc != pc) {
          // new history is a strict prefix of the latest one: copy it over
          const long long base = (long long)e * a.tstride + ((long long)r * a.K) * a.RX + c;
          for (unsigned q = 0; q < oc && (int)q < a.K; ++q) {
            Pnew.t[base + (long long)q * a.RX] = Pold.t[base + (long long)q * a.RX];
            Pnew.pos[base + (long long)q * a.RX] = Pold.pos[base + (long long)q * a.RX];
          }
          dve = true;
        }
        if (dve) {
          chmask |= 1u << e;
          Pnew.cnt[(long long)e * a.cstride + (long long)r * a.RX + c] = (uint8_t)((int)oc < a.K ? oc : a.K);
        }
      }
      if (chmask) {
        changed = true;
        a.sel[idx] = sel_after_change(vown, chmask, K, K0);
        // neighbours across changed edges must be recomputed next iteration
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (!((chmask >> e) & 1u)) continue;
          if (a.world > 1 && ((e == EDGE_N && r == 0) || (e == EDGE_S && r == a.RYl - 1))) continue;
          const int nr = e == EDGE_N ? (r - 1 + a.RYl) % a.RYl : e == EDGE_S ? (r + 1) % a.RYl : r;
          const int nc = e == EDGE_W ? (c - 1 + a.RX) % a.RX : e == EDGE_E ? (c + 1) % a.RX : c;
          const int nidx = nr * a.RX + nc;
          if (atomicMax(&a.dirty[nidx], K + 1) < K + 1) a.wl_out[atomicAdd(a.wl_out_count, 1u)] = (uint32_t)nidx;
        }
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
// K4 (world > 1): pack the latest north-edge histories of the strip's first
// region row and south-edge histories of its last row into the send rows,
// with the stamp of their last change (the neighbour marks its adjacent
// regions dirty when the stamp equals the current iteration).
// ---------------------------------------------------------------------------
__global__ void pack_kernel(const KArgs a, GhostView send_up, GhostView send_down) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 2 * a.RX) return;
  const bool up = i < a.RX;
  const int c = up ? i : i - a.RX;
  const int r = up ? 0 : a.RYl - 1;
  const int e = up ? EDGE_N : EDGE_S;
  const GhostView& g = up ? send_up : send_down;
  const unsigned long long v = a.sel[(long long)r * a.RX + c];
  // latest as of the end of this iteration
  const Latest L = latest_of(v, e, a.it_K + 1, a.it_K0);
  int cnt = 0;
  if (L.valid) {
    const EdgeView& E = a.ed[L.slot];
    cnt = E.cnt[(long long)e * a.cstride + (long long)r * a.RX + c];
    const long long base = (long long)e * a.tstride + ((long long)r * a.K) * a.RX + c;
    for (int q = 0; q < cnt; ++q) {
      g.t[(long long)q * a.RX + c] = E.t[base + (long long)q * a.RX];
      g.pos[(long long)q * a.RX + c] = E.pos[base + (long long)q * a.RX];
    }
  }
  g.cnt[c] = (uint8_t)cnt;
  const unsigned Kl = (unsigned)(v >> 32);
  const bool ch_now = Kl == a.it_K && ((v >> (4 + e)) & 1ull);
  g.stamp[c] = ch_now ? a.it_K : 0u;
}

// after the exchange: regions next to a ghost row that changed in this
// iteration are recomputed in the next one
__global__ void mark_kernel(const KArgs a, GhostView up, GhostView down) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 2 * a.RX) return;
  const bool isup = i < a.RX;
  const int c = isup ? i : i - a.RX;
  const GhostView& g = isup ? up : down;
  if (g.stamp[c] != a.it_K) return;
  const int r = isup ? 0 : a.RYl - 1;
  const int nidx = r * a.RX + c;
  if (atomicMax(&a.dirty[nidx], a.it_K + 1) < a.it_K + 1) a.wl_out[atomicAdd(a.wl_out_count, 1u)] = (uint32_t)nidx;
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
