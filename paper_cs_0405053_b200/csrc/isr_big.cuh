// isr_big.cuh -- region-trajectory kernel (K1), lane-per-region form for
// regions of more than 64 sites (8x16 .. 32x32: BASELINE c3 16x16, c5 32x32).
//
// One thread owns one region for one relaxation iteration, exactly like the
// small-region lane kernel (isr_region.cuh), so a warp advances 32 regions
// per step instead of one (the warp form, isr_warp.cuh, spends a whole warp
// on one region).  What changes with the region size:
//   * the spins live in shared memory, one 32-bit row mask per region row;
//   * the n-fold-way class counts N_k (eq. nidef) are exact
//     integers updated incrementally: a flip changes the class of the
//     flipped site (spin) and of its in-region neighbours (up-neighbour
//     count +-1); a break point changes the class of the one site next to
//     the flipped halo spin.  Lambda (eq. biglambda) is still re-folded from
//     the counts in the fixed order after every change (R3);
//   * per-row class counts (4 rows per 32-bit word, one byte each) let the
//     atom selection (eqs. Wsum..vindex; j-th site of class k* in
//     local row-major order, R6) skip to the right row and build
//     only that row's class mask;
//   * incoming history entries are read from global memory one ahead (the
//     entry after the head is always in flight), own entries are diffed
//     against the latest history at write time with the old entry read one
//     ahead as well.
// State, selector and history layouts are those of the warp form, so the two
// are interchangeable (ISING_SR_BIG=0 selects the warp form) and bit-identical.
#pragma once
#include "isr_warp.cuh"

namespace isr {

constexpr int BNT = 64;  // threads per block of the big-region lane kernel

template <int BX, int BY>
struct BigSmem {
  static constexpr int RQ = (BY + 3) / 4;  // row-count words per class
  uint32_t rows[BY][BNT];                  // spins, bit c of rows[r] = site (r, c)
  uint32_t rc[10][RQ][BNT];                // per-row class counts, byte (r & 3) of word r >> 2
};

template <int BX, int BY>
struct BigRegion {
  static constexpr uint32_t ROWM = BX == 32 ? 0xffffffffu : ((1u << BX) - 1u);
  BigSmem<BX, BY>& S;
  int t;                 // column (thread index)
  bool wrapX, wrapY;
  uint32_t gN, gS, gW, gE;  // ghost row above / below (bit = column), ghost columns (bit = row)
  unsigned long long Nq[2];  // class counts: N_k in the 12-bit field k % 5 of Nq[k / 5] (N_k <= 1024)

  __device__ __forceinline__ uint32_t row(int r) const { return S.rows[r][t]; }
  __device__ __forceinline__ uint32_t above(int r) const {
    return r > 0 ? row(r - 1) : (wrapY ? row(BY - 1) : gN);
  }
  __device__ __forceinline__ uint32_t below(int r) const {
    return r < BY - 1 ? row(r + 1) : (wrapY ? row(0) : gS);
  }
  // neighbour-is-up bit of the column to the west / east of the row's ends
  __device__ __forceinline__ uint32_t wbit(int r, uint32_t rw) const {
    return wrapX ? (rw >> (BX - 1)) & 1u : (gW >> r) & 1u;
  }
  __device__ __forceinline__ uint32_t ebit(int r, uint32_t rw) const { return wrapX ? rw & 1u : (gE >> r) & 1u; }

  // class mask of class k in row r (sites of the row whose class is k)
  __device__ __forceinline__ uint32_t class_mask(int r, int k) const {
    const uint32_t rw = row(r);
    const uint32_t nN = above(r), nS = below(r);
    const uint32_t nW = ((rw << 1) | wbit(r, rw)) & ROWM;
    const uint32_t nE = (rw >> 1) | (ebit(r, rw) << (BX - 1));
    const uint32_t s1 = nN ^ nS, c1 = nN & nS, s2 = nW ^ nE, c2 = nW & nE;
    const uint32_t p0 = s1 ^ s2, kk = s1 & s2, p1 = c1 ^ c2 ^ kk, p2 = (c1 & c2) | (kk & (c1 ^ c2));
    const int u = k >= 5 ? k - 5 : k;
    const uint32_t mu = u == 0 ? ~(p0 | p1 | p2) : u == 1 ? (p0 & ~p1) : u == 2 ? (~p0 & p1) : u == 3 ? (p0 & p1) : p2;
    return (k >= 5 ? rw : ~rw) & mu & ROWM;
  }
  // all ten class masks of row r
  __device__ __forceinline__ void class_masks(int r, uint32_t* m) const {
    const uint32_t rw = row(r);
    const uint32_t nN = above(r), nS = below(r);
    const uint32_t nW = ((rw << 1) | wbit(r, rw)) & ROWM;
    const uint32_t nE = (rw >> 1) | (ebit(r, rw) << (BX - 1));
    const uint32_t s1 = nN ^ nS, c1 = nN & nS, s2 = nW ^ nE, c2 = nW & nE;
    const uint32_t p0 = s1 ^ s2, kk = s1 & s2, p1 = c1 ^ c2 ^ kk, p2 = (c1 & c2) | (kk & (c1 ^ c2));
    const uint32_t mu[5] = {~(p0 | p1 | p2), p0 & ~p1, ~p0 & p1, p0 & p1, p2};
#pragma unroll
    for (int k = 0; k < 10; ++k) m[k] = (k >= 5 ? rw : ~rw) & mu[k >= 5 ? k - 5 : k] & ROWM;
  }
  // class of site (r, c) = 5 * s + u (u = number of up neighbours)
  __device__ __forceinline__ int site_class(int r, int c) const {
    const uint32_t rw = row(r);
    const uint32_t s = (rw >> c) & 1u;
    const uint32_t un = (above(r) >> c) & 1u, us = (below(r) >> c) & 1u;
    const uint32_t uw = c > 0 ? (rw >> (c - 1)) & 1u : wbit(r, rw);
    const uint32_t ue = c < BX - 1 ? (rw >> (c + 1)) & 1u : ebit(r, rw);
    return (int)(5u * s + un + us + uw + ue);
  }
  __device__ __forceinline__ int N(int k) const {
    return (int)((Nq[k >= 5 ? 1 : 0] >> (12 * (k >= 5 ? k - 5 : k))) & 0xFFFull);
  }
  // FLAG_OBSERVABLES: spins of the owned-bond partners of site (r, c) -- north
  // and west always (in-region, wrapped, or the ghost), south and east only
  // inside the region or wrapped (the bonds across the south/east border
  // belong to the neighbouring regions) -- as the sum of +-1 values
  __device__ __forceinline__ int owned_partner_sum(int r, int c) const {
    const uint32_t rw = row(r);
    int s = 0;
    s += (int)((above(r) >> c) & 1u);
    s += (int)(c > 0 ? (rw >> (c - 1)) & 1u : wbit(r, rw));
    int n = 2;
    if (r < BY - 1 || wrapY) {
      s += (int)((below(r) >> c) & 1u);
      ++n;
    }
    if (c < BX - 1 || wrapX) {
      s += (int)(c < BX - 1 ? (rw >> (c + 1)) & 1u : ebit(r, rw));
      ++n;
    }
    return 2 * s - n;
  }
  // magnetisation and owned bond sum of the whole region
  __device__ __forceinline__ void obs_counts(int& Mi, int& Bi) const {
    int m = 0, b = 0;
    for (int r = 0; r < BY; ++r) {
      const uint32_t rw = row(r);
      m += 2 * __popc(rw) - BX;
      b += 2 * __popc(~(rw ^ (rw >> 1)) & (ROWM >> 1)) - (BX - 1);  // (c, c + 1) inside the row
      b += 2 * __popc(~(rw ^ above(r)) & ROWM) - BX;                 // north bonds
      const uint32_t w = (rw & 1u) ^ wbit(r, rw);                     // west bond of column 0
      b += w ? -1 : 1;
    }
    Mi = m;
    Bi = b;
  }
  // N_k += d and the row count of class k in row r += d (d = +-1)
  __device__ __forceinline__ void add(int k, int r, int d) {
    const bool hi = k >= 5;
    const unsigned long long inc = (unsigned long long)(long long)d << (12 * (hi ? k - 5 : k));
    Nq[0] += hi ? 0ull : inc;  // two's complement: a -1 borrows only inside the (nonzero) field
    Nq[1] += hi ? inc : 0ull;
    S.rc[k][r >> 2][t] += (uint32_t)d << (8 * (r & 3));
  }
  // a site whose up-neighbour count changes by du (spin unchanged)
  __device__ __forceinline__ void neighbour_changed(int r, int c, int du_after_flip) {
    const int k = site_class(r, c);  // class after the flip
    add(k, r, 1);
    add(k - du_after_flip, r, -1);
  }
};

// eq. biglambda, fixed fold order: c_k = c_{k-1} + fl(N_k r_k)
template <class BR>
__device__ __forceinline__ double big_fold(const BR& B, const double* rate) {
  double c = 0.0;
#pragma unroll
  for (int k = 0; k < 10; ++k) c = __dadd_rn(c, __dmul_rn((double)B.N(k), rate[k]));
  return c;
}

// atom selection: returns the local site index r * BX + c
template <int BX, int BY>
__device__ __forceinline__ int big_select(const BigRegion<BX, BY>& B, const double* rate, double V, double lam) {
  const double x = __dmul_rn(V, lam);
  double c = 0.0, cprev = 0.0;
  int ks = -1, nk = 0, lastnz = 0, nlast = B.N(0);
#pragma unroll
  for (int k = 0; k < 10; ++k) {
    const int n = B.N(k);
    const double cn = __dadd_rn(c, __dmul_rn((double)n, rate[k]));
    const bool hit = ks < 0 && x <= cn;
    ks = hit ? k : ks;
    cprev = hit ? c : cprev;
    nk = hit ? n : nk;
    lastnz = n > 0 ? k : lastnz;
    nlast = n > 0 ? n : nlast;
    c = cn;
  }
  if (ks < 0) {  // unreachable for V < 1 (x <= Lambda = c_9)
    ks = lastnz;
    nk = nlast;
    cprev = 0.0;
  }
  const double aq = __dsub_rn(x, cprev);
  const double rk = rate[ks];
  long long j = __double2ll_rd(rk == 1.0 ? aq : __ddiv_rn(aq, rk));
  if (j > nk - 1) j = nk - 1;
  if (j < 0) j = 0;
  int jj = (int)j;
  // skip whole groups of 4 rows, then rows, using the per-row counts: the
  // class's RQ count words are read at once (independent loads), then the
  // group holding the j-th site is found with a branch-free scan
  constexpr int RQ = BigSmem<BX, BY>::RQ;
  uint32_t wq[RQ];
#pragma unroll
  for (int q = 0; q < RQ; ++q) wq[q] = B.S.rc[ks][q][B.t];
  int qs = RQ - 1;
  uint32_t w = wq[RQ - 1];
  bool found = false;
#pragma unroll
  for (int q = 0; q < RQ; ++q) {
    const int s = (int)((wq[q] * 0x01010101u) >> 24);  // sum of the 4 byte counts (<= 128)
    const bool here = !found && jj < s;
    qs = here ? q : qs;
    w = here ? wq[q] : w;
    jj -= (!found && !here) ? s : 0;
    found = found || here;
  }
  int r = 4 * qs;
  int c0 = (int)(w & 0xFFu);
  if (jj >= c0) {
    jj -= c0;
    ++r;
    c0 = (int)((w >> 8) & 0xFFu);
    if (jj >= c0) {
      jj -= c0;
      ++r;
      c0 = (int)((w >> 16) & 0xFFu);
      if (jj >= c0) {
        jj -= c0;
        ++r;
      }
    }
  }
  return r * BX + nth_bit<uint32_t, 32>(B.class_mask(r, ks), jj);
}

#ifndef ISR_BIG_MINB
#define ISR_BIG_MINB 7  // resident 64-thread blocks per SM asked of ptxas (128 registers, 8 fit): c3 +14 %, c5 32x32 +20-27 % over 221 unbounded
#endif
#if ISR_BIG_MINB > 0
#define ISR_BIG_BOUNDS __launch_bounds__(BNT, ISR_BIG_MINB)
#else
#define ISR_BIG_BOUNDS __launch_bounds__(BNT)
#endif
template <int BX, int BY, bool LOG, bool OBS = false>
__global__ void ISR_BIG_BOUNDS region_kernel_big(const KArgs a) {
  using BR = BigRegion<BX, BY>;
  static_assert(BX <= 32 && BY <= 32 && BX >= 3 && BY >= 3, "rows of up to 32 sites");
  __shared__ BigSmem<BX, BY> SM;
  const int t = threadIdx.x;
  const bool wrapX = a.RX == 1, wrapY = a.RYg == 1;
  const unsigned K = stamp_of(a), K0 = a.it_K0;
  ktime_begin(a);
  unsigned long long n_ev = 0, n_out = 0, n_in = 0, n_cmp = 0, n_reg = 0;
  unsigned fmax = 0;
  bool changed = false, overflow = false;
  // a small worklist (late iterations, bounded by the slowest region's serial
  // chain) is spread to one region per 2^spread_log2 lanes, so no region's
  // chain waits on other lanes' divergent steps in its warp
  const int sl = a.spread_log2;
  const int stride = (gridDim.x * BNT) >> sl;
  const int n_all = a.n_work_dev ? (int)__ldcg(a.n_work_dev) : a.n_work;
  const int first_item = (t & ((1 << sl) - 1)) ? n_all : (blockIdx.x * BNT + t) >> sl;  // idle lanes skip

  for (int item = first_item; item < n_all; item += stride) {
    const int idx = a.wl_in ? (int)a.wl_in[item] : item;
    const int r = idx / a.RX, c = idx - r * a.RX;
    const uint32_t gid = (uint32_t)((a.row0 + r) * a.RX + c);
    ++n_reg;
    BR B{SM, t, wrapX, wrapY, 0u, 0u, 0u, 0u, {0ull, 0ull}};
    // ---- committed state ----
    {
      const uint32_t* src = (const uint32_t*)a.in.spins + (long long)idx * BY;
#pragma unroll
      for (int q = 0; q < BY; ++q) SM.rows[q][t] = src[q];
      const uint4 h = ((const uint4*)a.in.halo)[idx];
      B.gN = h.x;
      B.gS = h.y;
      B.gW = h.z;
      B.gE = h.w;
    }
    double ts = a.fresh_w ? a.t_c : a.in.ts[idx], R = a.in.R[idx];
    uint32_t n = a.in.n[idx];
    // the paper's presimulated list ("reuse the random numbers"):
    // the window's pairs of this region, (E(U_m), V_m) for m = n0, n0 + 1, ...,
    // are kept from the recomputation that first drew them, so that the
    // following recomputations of the window read them instead of drawing
    const uint32_t n0 = n;
    unsigned pfill = 0;
    if (a.pcache) {
      const uint2 pm = a.pmeta[idx];
      pfill = pm.x == K0 ? pm.y : 0u;
    }
    const long long pbase = (long long)idx * a.PC;
    auto get_pair = [&](uint32_t m, double& E, double& Vm) {
      const unsigned q = m - n0;
      ISR_ASSERT(!a.pcache || pfill <= (unsigned)a.PC);
      if (a.pcache && q < pfill) {
        const double2 c = a.pcache[pbase + q];
        E = c.x;
        Vm = c.y;
      } else {
        double Um;
        draw_pair(a.seed, gid, m, Um, Vm, a.gen);
        E = budget(a, Um);
        if (a.pcache && q == pfill && q < (unsigned)a.PC) {
          a.pcache[pbase + q] = make_double2(E, Vm);
          ++pfill;
        }
      }
    };
    unsigned long long dig = a.digest ? a.in.dig[idx] : 0ull;
    unsigned n_ev_r = 0, bev = 0;
    // FLAG_OBSERVABLES: M and the owned bond sum B now, their integrals since t_c
    int Mi = 0, Bi = 0;
    double iM = 0.0, iB = 0.0, tpv = a.t_c;
    if (OBS && !LOG) B.obs_counts(Mi, Bi);
    auto obs_adv = [&](double tt) {
      const double dt = __dsub_rn(tt, tpv);
      iM = __dadd_rn(iM, __dmul_rn((double)Mi, dt));
      iB = __dadd_rn(iB, __dmul_rn((double)Bi, dt));
      tpv = tt;
    };
    // ---- incoming histories: head entry + the next one in flight ----
    unsigned hcnt[4], hidx[4], hsrc[4], hoff[4];
    double ht[4], hn[4];
    unsigned hp = 0, hq = 0;  // byte d: position of the head / next entry of direction d
    unsigned chg = 0;         // bit d: incoming history d changed in the previous iteration
    unsigned qd[4];           // ... its first changed entry
    // the four neighbours' edge selector pairs, all in flight before any is
    // used (a direction without one re-reads the region's own pair)
    ulonglong2 wpn[4];
    bool use[4];
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      const bool axis_off = (d < 2) ? wrapY : wrapX;
      const bool ghost = a.ghost && ((d == EDGE_N && r == 0) || (d == EDGE_S && r == a.RYl - 1));
      use[d] = !a.first && !axis_off && !ghost;
      const int nr = d == EDGE_N ? wdec(r, a.RYl) : d == EDGE_S ? winc(r, a.RYl) : r;
      const int nc = d == EDGE_W ? wdec(c, a.RX) : d == EDGE_E ? winc(c, a.RX) : c;
      wpn[d] = __ldcg(reinterpret_cast<const ulonglong2*>(a.sel) +
                      (use[d] ? ((long long)nr * a.RX + nc) * 4 + (d ^ 1) : (long long)idx * 4));
    }
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      hcnt[d] = 0; hidx[d] = 0; hsrc[d] = 0; hoff[d] = 0; ht[d] = dinf(); hn[d] = dinf(); qd[d] = 0;
      const bool axis_off = (d < 2) ? wrapY : wrapX;
      if (a.first || axis_off) continue;
      const bool ghost = !use[d];
      if (ghost) {
        const GhostView& gv = d == EDGE_N ? a.gh_up : a.gh_down;
        hcnt[d] = gv.cnt[c];
        hsrc[d] = d == EDGE_N ? 2u : 3u;
        hoff[d] = (unsigned)c;
        if (gv.stamp[c] == K - 1) chg |= 1u << d;  // first changed entry unknown: 0
      } else {
        const int nr = d == EDGE_N ? wdec(r, a.RYl) : d == EDGE_S ? winc(r, a.RYl) : r;
        const int nc = d == EDGE_W ? wdec(c, a.RX) : d == EDGE_E ? winc(c, a.RX) : c;
        const unsigned long long v = latest_word(wpn[d], K);
        if (word_valid(v, K0)) {
          hcnt[d] = ew_count(v);
          hsrc[d] = ew_slot(v);
          hoff[d] = ((unsigned)nr * (unsigned)a.K) * (unsigned)a.RX + (unsigned)nc;
          if ((unsigned)(v >> 32) == K - 1) {
            chg |= 1u << d;
            qd[d] = ew_fd(v);
          }
        }
      }
      n_in += hcnt[d];
    }

    // ---- own latest histories ----
    unsigned oc[4], pc[4], ps[4], dv[4], wh[4], k0[4], fdk[4];
    double ot[4];
    unsigned op = 0;  // byte e: position of the old entry at index oc[e]
    const unsigned obase = (unsigned)(((long long)r * a.K) * a.RX + c);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      oc[e] = 0; pc[e] = 0; ps[e] = 0; dv[e] = 0; wh[e] = 0; ot[e] = 0.0; k0[e] = 0; fdk[e] = 0;
      if (LOG) continue;
      const ulonglong2 wp = reinterpret_cast<const ulonglong2*>(a.sel)[(long long)idx * 4 + e];
      const int li = latest_index(wp, K);
      const unsigned long long v = li ? wp.y : wp.x;
      ps[e] = ew_slot(v);
      pc[e] = word_valid(v, K0) ? ew_count(v) : 0u;
      wh[e] = (unsigned)(li ^ 1);
      n_cmp += pc[e];
    }

    // ---- resume: the trajectory of the region's last recomputation in this
    // window (its step log) is unchanged up to the first changed incoming
    // entry; replay that prefix instead of re-simulating it ----
    const long long lb = (long long)idx * a.LC;
    unsigned lpos = 0;  // steps of this recomputation (log length)
    if (!LOG && a.resume && !a.first && chg) {
      const uint2 meta = a.lg_meta[idx];
      if (meta.x >= K0 && meta.y != 0xffffffffu) {
        const unsigned len = meta.y;
        // earliest time at which an input differs: the new entry q_d ...
        double tst = dinf();
#pragma unroll
        for (int d = 0; d < 4; ++d)
          if (((chg >> d) & 1u) && qd[d] < hcnt[d])
            tst = fmin(tst, src_t(a, hsrc[d], d ^ 1)[hoff[d] + qd[d] * (unsigned)a.RX]);
        // ... or the old entry q_d, consumed as that direction's q_d-th break point
        unsigned cntd = 0;  // byte d: break points of direction d so far
        unsigned i = 0;
        bool stop = false;
        // 4 log entries in flight per round (all inside the region's log)
        for (unsigned i0 = 0; i0 < len && !stop; i0 += 4) {
          double tq[4];
          unsigned cq[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const unsigned iu = min(i0 + (unsigned)u, (unsigned)a.LC - 1u);
            tq[u] = a.lg_tR[lb + iu].x;
            cq[u] = a.lg_c[lb + iu];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (stop || i0 + u >= len) continue;
            i = i0 + u;
            if (!(tq[u] < tst)) {
              stop = true;
              continue;
            }
            const unsigned code = cq[u];
            if (code & 0x8000u) {
              const int d = (int)((code >> 12) & 3u);
              const unsigned kd = (cntd >> (8 * d)) & 0xFFu;
              if (((chg >> d) & 1u) && kd == qd[d]) {
                tst = tq[u];
                stop = true;
                continue;
              }
              if (kd < 255u) cntd += 1u << (8 * d);
            }
          }
        }
        if (!stop) i = len;
        while (i > 0 && !(a.lg_tR[lb + i - 1].x < tst)) --i;  // steps at time tst are re-simulated
        // replay steps [0, i): flips, cursors, own-history counts, digest
        for (unsigned j = 0; j < i; ++j) {
          const unsigned code = a.lg_c[lb + j];
          if (OBS && !LOG) obs_adv(a.lg_tR[lb + j].x);
          if (code & 0x8000u) {
            const int d = (int)((code >> 12) & 3u);
            const int p = (int)(code & 0xFFu);
            if (OBS && !LOG) {  // owned bonds: the north and west ghosts
              if (d == EDGE_N) Bi += ((B.gN >> p) & 1u) == ((B.row(0) >> p) & 1u) ? -2 : 2;
              else if (d == EDGE_W) Bi += ((B.gW >> p) & 1u) == (B.row(p) & 1u) ? -2 : 2;
            }
            if (d == EDGE_N) B.gN ^= 1u << p;
            else if (d == EDGE_S) B.gS ^= 1u << p;
            else if (d == EDGE_W) B.gW ^= 1u << p;
            else B.gE ^= 1u << p;
#pragma unroll
            for (int q = 0; q < 4; ++q) hidx[q] += q == d ? 1u : 0u;
          } else {
            const int site = (int)code;
            const int sr = site / BX, sc = site - sr * BX;
            if (OBS && !LOG) {
              const int sg = ((B.row(sr) >> sc) & 1u) ? 1 : -1;
              Mi -= 2 * sg;
              Bi -= 2 * sg * B.owned_partner_sum(sr, sc);
            }
            SM.rows[sr][t] ^= 1u << sc;
            if (a.digest) dig = digest_step(dig, a.lg_tR[lb + j].x, site);
            ++n_ev_r;
            bool on_edge = false;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const bool on = e == EDGE_N ? (!wrapY && sr == 0)
                            : e == EDGE_S ? (!wrapY && sr == BY - 1)
                            : e == EDGE_W ? (!wrapX && sc == 0)
                                          : (!wrapX && sc == BX - 1);
              oc[e] += on ? 1u : 0u;
              on_edge |= on;
            }
            bev += on_edge ? 1u : 0u;
          }
        }
        if (i > 0) {
          const double2 e = a.lg_tR[lb + i - 1];
          ts = e.x;
          R = e.y;
        }
        n += n_ev_r;
        lpos = i;
#pragma unroll
        for (int e = 0; e < 4; ++e) k0[e] = oc[e];  // own-history prefix == the latest history's
      }
    }

    // class counts and per-row class counts of the committed state
    for (int q = 0; q < BigSmem<BX, BY>::RQ; ++q) {
      uint32_t w[10];
#pragma unroll
      for (int k = 0; k < 10; ++k) w[k] = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int rr = 4 * q + i;
        if (rr < BY) {
          uint32_t m[10];
          B.class_masks(rr, m);
#pragma unroll
          for (int k = 0; k < 10; ++k) w[k] |= (uint32_t)__popc(m[k]) << (8 * i);
        }
      }
#pragma unroll
      for (int k = 0; k < 10; ++k) {
        SM.rc[k][q][t] = w[k];
        B.Nq[k >= 5 ? 1 : 0] += (unsigned long long)((w[k] * 0x01010101u) >> 24) << (12 * (k >= 5 ? k - 5 : k));
      }
    }

    // incoming heads at the cursors: the head entry and the next one in flight
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      const unsigned x = hidx[d];
      if (x < hcnt[d]) {
        const double* T = src_t(a, hsrc[d], d ^ 1);
        const uint8_t* P = src_p(a, hsrc[d], d ^ 1);
        ht[d] = T[hoff[d] + x * (unsigned)a.RX];
        hp |= (unsigned)P[hoff[d] + x * (unsigned)a.RX] << (8 * d);
        if (x + 1 < hcnt[d]) {
          hn[d] = T[hoff[d] + (x + 1) * (unsigned)a.RX];
          hq |= (unsigned)P[hoff[d] + (x + 1) * (unsigned)a.RX] << (8 * d);
        }
      }
    }
    // the old own entry at each edge's write position, read ahead for the diff
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (!LOG && oc[e] < pc[e]) {
        ot[e] = src_t(a, ps[e], e)[obase + oc[e] * (unsigned)a.RX];
        op |= (unsigned)src_p(a, ps[e], e)[obase + oc[e] * (unsigned)a.RX] << (8 * e);
      }
    }

    double E0, V;
    get_pair(n, E0, V);
    if (a.fresh_w && lpos == 0) R = E0;  // the slate is wiped at t_c; a replay restored R
    // pair n+1 drawn one event ahead: an event takes its new budget and atom
    // variate from here and draws the following pair off the step's critical
    // path (the region's serial step chain bounds every iteration, §6)
    double Rn, Vn;
    get_pair(n + 1, Rn, Vn);
    double lam = big_fold(B, a.rate);
    double tc = cand_time(ts, R, lam);

    for (;;) {
      int dstar = -1;
      double tb = dinf();
#pragma unroll
      for (int d = 0; d < 4; ++d) {
        if (ht[d] < tb) {
          tb = ht[d];
          dstar = d;
        }
      }
      bool bp = false;
      if (dstar >= 0) {
        if (tb < tc) {
          bp = true;
          // exactly equal head times in two directions: smallest neighbour id first
          uint32_t nb = 0xffffffffu;
#pragma unroll
          for (int d = 0; d < 4; ++d) {
            if (ht[d] == tb) {
              const uint32_t nid = neighbour_id(a, gid, d);
              if (nid < nb) {
                nb = nid;
                dstar = d;
              }
            }
          }
        } else if (tb == tc) {
          uint32_t nb = 0xffffffffu;
#pragma unroll
          for (int d = 0; d < 4; ++d) {
            if (ht[d] == tb) {
              const uint32_t nid = neighbour_id(a, gid, d);
              if (nid < nb) {
                nb = nid;
                dstar = d;
              }
            }
          }
          bp = nb < gid;
        }
      }
      if (!bp && !(tc < a.t_w)) break;
      unsigned code = 0;  // step log code: site, or 0x8000 | direction << 12 | position
      if (bp) {
        // break point (eqs. lambdataua..newtau): budget at the old rate
        const double Rn = __dsub_rn(R, __dmul_rn(lam, __dsub_rn(tb, ts)));
        R = Rn < 0.0 ? 0.0 : Rn;
        ts = tb;
        const int p = (int)((hp >> (8 * dstar)) & 0xFFu);
        code = 0x8000u | ((unsigned)dstar << 12) | (unsigned)p;
        if (OBS && !LOG) {
          obs_adv(tb);
          if (dstar == EDGE_N) Bi += ((B.gN >> p) & 1u) == ((B.row(0) >> p) & 1u) ? -2 : 2;
          else if (dstar == EDGE_W) Bi += ((B.gW >> p) & 1u) == (B.row(p) & 1u) ? -2 : 2;
        }
        // the in-region site next to the flipped halo spin and its change of
        // up-neighbour count
        int sr, sc;
        uint32_t was;
        if (dstar == EDGE_N) { sr = 0; sc = p; was = (B.gN >> p) & 1u; B.gN ^= 1u << p; }
        else if (dstar == EDGE_S) { sr = BY - 1; sc = p; was = (B.gS >> p) & 1u; B.gS ^= 1u << p; }
        else if (dstar == EDGE_W) { sr = p; sc = 0; was = (B.gW >> p) & 1u; B.gW ^= 1u << p; }
        else { sr = p; sc = BX - 1; was = (B.gE >> p) & 1u; B.gE ^= 1u << p; }
        B.neighbour_changed(sr, sc, was ? -1 : 1);
        // advance the cursor: the next entry becomes the head, read the one after
#pragma unroll
        for (int d = 0; d < 4; ++d) {
          if (d != dstar) continue;
          const unsigned nx = ++hidx[d];
          double h1 = dinf();
          unsigned p1 = 0;
          if (nx + 1 < hcnt[d]) {
            const unsigned off = hoff[d] + (nx + 1) * (unsigned)a.RX;
            h1 = src_t(a, hsrc[d], d ^ 1)[off];
            p1 = src_p(a, hsrc[d], d ^ 1)[off];
          }
          ht[d] = nx < hcnt[d] ? hn[d] : dinf();
          hp = (hp & ~(0xFFu << (8 * d))) | (((hq >> (8 * d)) & 0xFFu) << (8 * d));
          hn[d] = h1;
          hq = (hq & ~(0xFFu << (8 * d))) | (p1 << (8 * d));
        }
      } else {
        // own event at tc
        const int site = big_select<BX, BY>(B, a.rate, V, lam);
        // pair n+1 (drawn ahead) becomes current; pair n+2 is drawn here, where
        // its instructions interleave with the flip's bookkeeping below
        R = Rn;
        V = Vn;
        get_pair(n + 2, Rn, Vn);
        const int sr = site / BX, sc = site - sr * BX;
        code = (unsigned)site;
        if (OBS && !LOG) {
          obs_adv(tc);
          const int sg = ((B.row(sr) >> sc) & 1u) ? 1 : -1;
          Mi -= 2 * sg;
          Bi -= 2 * sg * B.owned_partner_sum(sr, sc);
        }
        {
          const int k0 = B.site_class(sr, sc);
          const uint32_t s = (uint32_t)(k0 >= 5);
          // flip: the site changes spin, its in-region neighbours' up-count moves by du
          const int du = s ? -1 : 1;
          B.add(k0, sr, -1);
          SM.rows[sr][t] ^= 1u << sc;
          B.add(s ? k0 - 5 : k0 + 5, sr, 1);
          if (sr > 0) B.neighbour_changed(sr - 1, sc, du);
          else if (wrapY) B.neighbour_changed(BY - 1, sc, du);
          if (sr < BY - 1) B.neighbour_changed(sr + 1, sc, du);
          else if (wrapY) B.neighbour_changed(0, sc, du);
          if (sc > 0) B.neighbour_changed(sr, sc - 1, du);
          else if (wrapX) B.neighbour_changed(sr, BX - 1, du);
          if (sc < BX - 1) B.neighbour_changed(sr, sc + 1, du);
          else if (wrapX) B.neighbour_changed(sr, 0, du);
        }
        if (a.digest) dig = digest_step(dig, tc, site);
        const unsigned up_new = (SM.rows[sr][t] >> sc) & 1u;  // the flipped site's new spin (for dM)
        if (LOG) {
          const unsigned long long o = a.log_off[idx] + n_ev_r;
          ISR_ASSERT(a.log_cap == 0 || (long long)o < a.log_cap);
          a.log_t[o] = tc;
          a.log_region[o] = gid;
          a.log_site[o] = (uint16_t)site;
          if (a.log_dm) a.log_dm[o] = up_new ? 2 : -2;
        } else {
          if (a.ev_t && (int)n_ev_r < a.evC) {  // scratch event log (a resumed prefix is already there)
            const long long o = (long long)n_ev_r * a.ev_stride + idx;
            a.ev_t[o] = tc;
            a.ev_s[o] = (uint16_t)(site | (up_new << 15));
          }
          bool on_edge = false;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const bool on = e == EDGE_N ? (!wrapY && sr == 0)
                          : e == EDGE_S ? (!wrapY && sr == BY - 1)
                          : e == EDGE_W ? (!wrapX && sc == 0)
                                        : (!wrapX && sc == BX - 1);
            if (!on) continue;
            on_edge = true;
            const unsigned k = oc[e];
            const uint8_t p = (uint8_t)(e < 2 ? sc : sr);
            if ((int)k < a.K) {
              const unsigned o = obase + k * (unsigned)a.RX;
              slot_t(a, ps[e] ^ 1u, e)[o] = tc;  // the other slot
              slot_p(a, ps[e] ^ 1u, e)[o] = p;
              ++n_out;
              if (!dv[e]) {
                fdk[e] = k;  // first differing entry, if it differs here
                if (k >= pc[e]) {
                  dv[e] = 1;
                } else {
                  dv[e] = (__double_as_longlong(ot[e]) != __double_as_longlong(tc) ||
                           ((op >> (8 * e)) & 0xFFu) != p) ? 1u : 0u;
                  if (!dv[e] && k + 1 < pc[e]) {  // read the next old entry ahead
                    const unsigned o1 = o + (unsigned)a.RX;
                    ot[e] = src_t(a, ps[e], e)[o1];
                    op = (op & ~(0xFFu << (8 * e))) | ((unsigned)src_p(a, ps[e], e)[o1] << (8 * e));
                  }
                }
              }
            } else {
              overflow = true;
            }
            oc[e] = k + 1;
          }
          bev += on_edge ? 1u : 0u;
        }
        ++n_ev_r;
        ts = tc;
        ++n;
      }
      if (!LOG && a.resume) {  // step log: time, budget after the step, code
        if (lpos < (unsigned)a.LC) {
          a.lg_tR[lb + lpos] = make_double2(ts, R);
          a.lg_c[lb + lpos] = (uint16_t)code;
        }
        ++lpos;
      }
      lam = big_fold(B, a.rate);
      tc = cand_time(ts, R, lam);
    }
    n_ev += n_ev_r;
    fmax = max(fmax, bev);
    if (!LOG && a.resume) a.lg_meta[idx] = make_uint2(K, lpos <= (unsigned)a.LC ? lpos : 0xffffffffu);
    if (!LOG && a.pcache) a.pmeta[idx] = make_uint2(K0, pfill);

    if (!LOG && a.delay_ns) k1_delay(a.delay_ns);  // test knob: publish late
    if (!LOG) {
      unsigned chmask = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if ((int)oc[e] > a.K) overflow = true;
        const bool diff = dv[e] || oc[e] != pc[e];
        if (diff) {
          chmask |= 1u << e;
          const unsigned cnt = (int)oc[e] < a.K ? oc[e] : (unsigned)a.K;
          // a resumed recomputation wrote only the entries after its replayed
          // prefix: complete the new history with the (identical) prefix
          if (k0[e] > 0 && (int)k0[e] <= a.K) {
            const double* To = src_t(a, ps[e], e);
            const uint8_t* Po = src_p(a, ps[e], e);
            double* Tn = const_cast<double*>(src_t(a, ps[e] ^ 1u, e));
            uint8_t* Pn = const_cast<uint8_t*>(src_p(a, ps[e] ^ 1u, e));
            // 8 entries per round, all loads issued before the stores (the two
            // slots may alias as far as the compiler knows, so a plain loop
            // serialises one memory latency per entry)
            unsigned q = 0;
            for (; q + 8 <= k0[e]; q += 8) {
              double tv[8];
              uint8_t pv[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const unsigned o = obase + (q + u) * (unsigned)a.RX;
                tv[u] = __ldcg(To + o);
                pv[u] = __ldcg(Po + o);
              }
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const unsigned o = obase + (q + u) * (unsigned)a.RX;
                Tn[o] = tv[u];
                Pn[o] = pv[u];
              }
            }
            if (q < k0[e]) {  // the last < 8 entries, also with their loads issued together
              double tv[8];
              uint8_t pv[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const unsigned o = obase + (q + u) * (unsigned)a.RX;
                if (q + u < k0[e]) {
                  tv[u] = __ldcg(To + o);
                  pv[u] = __ldcg(Po + o);
                }
              }
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const unsigned o = obase + (q + u) * (unsigned)a.RX;
                if (q + u < k0[e]) {
                  Tn[o] = tv[u];
                  Pn[o] = pv[u];
                }
              }
            }
          }
          const unsigned fd = min(dv[e] ? fdk[e] : min(oc[e], pc[e]), 0x7FFFu);
          a.sel[((long long)idx * 4 + e) * 2 + wh[e]] = ((unsigned long long)K << 32) |
                                                       ((unsigned long long)fd << 17) |
                                                       ((unsigned long long)cnt << 1) | (ps[e] ^ 1u);
        }
      }
      if (chmask) {
        changed = true;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (!((chmask >> e) & 1u)) continue;
          if (a.ghost && ((e == EDGE_N && r == 0) || (e == EDGE_S && r == a.RYl - 1))) continue;
          const int nr = e == EDGE_N ? wdec(r, a.RYl) : e == EDGE_S ? winc(r, a.RYl) : r;
          const int nc = e == EDGE_W ? wdec(c, a.RX) : e == EDGE_E ? winc(c, a.RX) : c;
          mark_dirty(a, nr * a.RX + nc, K + 1);
        }
      }
      if (OBS) {  // integrals up to the window end
        obs_adv(a.t_w);
        a.out.oM[idx] = iM;
        a.out.oB[idx] = iB;
      }
      uint32_t* dst = (uint32_t*)a.out.spins + (long long)idx * BY;
#pragma unroll
      for (int q = 0; q < BY; ++q) dst[q] = SM.rows[q][t];
      ((uint4*)a.out.halo)[idx] = make_uint4(B.gN, B.gS, B.gW, B.gE);
      a.out.ts[idx] = ts;
      a.out.R[idx] = R;
      a.out.n[idx] = n;
      if (a.digest) a.out.dig[idx] = dig;
    }
  }

  ktime_end(a);
  if (!LOG) {
    const unsigned full = 0xffffffffu;
    const unsigned anych = __ballot_sync(full, changed);
    const unsigned anyov = __ballot_sync(full, overflow);
    unsigned long long v0 = n_ev, v1 = n_out, v2 = n_in, v3 = n_cmp, v5 = n_reg;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      v0 += __shfl_xor_sync(full, v0, o);
      v1 += __shfl_xor_sync(full, v1, o);
      v2 += __shfl_xor_sync(full, v2, o);
      v3 += __shfl_xor_sync(full, v3, o);
      v5 += __shfl_xor_sync(full, v5, o);
      fmax = max(fmax, __shfl_xor_sync(full, fmax, o));
    }
    if ((t & 31) == 0) {
      if (anych) atomicOr(&a.flags[0], 1);
      if (anyov) atomicOr(&a.flags[1], 1);
      if (v5) {
        atomicAdd(&a.stats[0], v0);
        atomicAdd(&a.stats[1], v1);
        atomicAdd(&a.stats[2], v2);
        atomicAdd(&a.stats[3], v3);
        atomicMax(&a.stats[4], (unsigned long long)fmax);
        atomicAdd(&a.stats[5], v5);
      }
    }
  }
}

}  // namespace isr
