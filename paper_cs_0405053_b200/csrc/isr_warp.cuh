// isr_warp.cuh -- region-trajectory kernel, warp-per-region form for regions
// of up to 32 x 32 sites (BASELINE configs c3 16x16 and c5 32x32).
//
// One warp owns one region for one relaxation iteration: lane r holds row r
// of the region's spins as a bit mask; the ten n-fold-way class counts N_k
// (eq. nidef) are warp reductions (redux.sync) of per-row
// popcounts of bit-sliced "up neighbours" planes; the atom of class k* with
// index j (eqs. Wsum..vindex; linear order = local row-major,
// DESIGN.md R6) is found by a warp prefix scan of the per-row class counts
// and a ballot.  Scalars (times, budget, rates, cursors) are uniform across
// the warp and computed redundantly by every lane.  Same semantics, bit for
// bit, as the lane-per-region kernel (isr_region.cuh).
//
// Boundary histories use the same slot layout as the lane kernel; the
// selector is a pair of 64-bit words per region EDGE (stamp << 32 | count
// << 1 | slot), so edge histories may hold up to 65535 entries.
#pragma once
#include "isr_region.cuh"

namespace isr {

__device__ __forceinline__ unsigned long long latest_edge_word(const unsigned long long* sel, long long i, unsigned K) {
  const ulonglong2 w = __ldcg(reinterpret_cast<const ulonglong2*>(sel) + i);
  return latest_word(w, K);
}
__device__ __forceinline__ unsigned ew_count(unsigned long long v) { return (unsigned)((v >> 1) & 0xFFFFu); }
__device__ __forceinline__ unsigned ew_slot(unsigned long long v) { return (unsigned)(v & 1ull); }
// first entry in which this history differs from the edge's previous one (bits 17-31, capped at 32767)
__device__ __forceinline__ unsigned ew_fd(unsigned long long v) { return (unsigned)((v >> 17) & 0x7FFFu); }

template <int BX, int BY>
struct WGeo {
  static_assert(BX <= 32 && BY <= 32, "warp form holds up to 32 x 32 sites");
  static constexpr int NS = BX * BY;
  static constexpr uint32_t ROW = BX == 32 ? 0xffffffffu : ((1u << BX) - 1u);
};

// per-lane class planes of row `lane`
struct WClasses {
  uint32_t up, dn, m0, m1, m2, m3, m4;
  __device__ __forceinline__ uint32_t mask(int k) const {
    const uint32_t s = k >= 5 ? up : dn;
    const int u = k >= 5 ? k - 5 : k;
    const uint32_t mu = u == 0 ? m0 : u == 1 ? m1 : u == 2 ? m2 : u == 3 ? m3 : m4;
    return s & mu;
  }
};

template <int BX, int BY>
__device__ __forceinline__ WClasses wbuild(uint32_t row, uint32_t gN, uint32_t gS, uint32_t gWb, uint32_t gEb,
                                           bool wrapX, bool wrapY) {
  using G = WGeo<BX, BY>;
  const int lane = threadIdx.x & 31;
  const bool live = lane < BY;
  const uint32_t above = __shfl_sync(0xffffffffu, row, (lane - 1 + BY) % BY);
  const uint32_t below = __shfl_sync(0xffffffffu, row, (lane + 1) % BY);
  uint32_t nN = lane == 0 ? (wrapY ? above : gN) : above;
  uint32_t nS = lane == BY - 1 ? (wrapY ? below : gS) : below;
  uint32_t nW = (row << 1) & G::ROW;
  uint32_t nE = row >> 1;
  nW |= wrapX ? ((row >> (BX - 1)) & 1u) : gWb;
  nE |= (wrapX ? (row & 1u) : gEb) << (BX - 1);
  const uint32_t s1 = nN ^ nS, c1 = nN & nS, s2 = nW ^ nE, c2 = nW & nE;
  const uint32_t p0 = s1 ^ s2, k = s1 & s2, p1 = c1 ^ c2 ^ k, p2 = (c1 & c2) | (k & (c1 ^ c2));
  WClasses C;
  C.up = live ? row : 0u;
  C.dn = live ? (~row & G::ROW) : 0u;
  C.m0 = ~(p0 | p1 | p2) & G::ROW;
  C.m1 = p0 & ~p1;
  C.m2 = ~p0 & p1;
  C.m3 = p0 & p1;
  C.m4 = p2;
  return C;
}

__device__ __forceinline__ void wcounts(const WClasses& C, int N[10]) {
#pragma unroll
  for (int k = 0; k < 10; ++k) N[k] = (int)__reduce_add_sync(0xffffffffu, (unsigned)__popc(C.mask(k)));
}

__device__ __forceinline__ double wfold(const int N[10], const double* rate) {
  double c = 0.0;
#pragma unroll
  for (int k = 0; k < 10; ++k) c = __dadd_rn(c, __dmul_rn((double)N[k], rate[k]));
  return c;
}

// returns the local site index (row * BX + col) chosen by V (uniform)
template <int BX, int BY>
__device__ __forceinline__ int wselect(const WClasses& C, const int N[10], const double* rate, double V, double lam) {
  const int lane = threadIdx.x & 31;
  const double x = __dmul_rn(V, lam);
  double c = 0.0, cprev = 0.0;
  int ks = -1, nk = 0, lastnz = 0, nlast = N[0];
#pragma unroll
  for (int k = 0; k < 10; ++k) {
    const double cn = __dadd_rn(c, __dmul_rn((double)N[k], rate[k]));
    const bool hit = ks < 0 && x <= cn;
    ks = hit ? k : ks;
    cprev = hit ? c : cprev;
    nk = hit ? N[k] : nk;
    lastnz = N[k] > 0 ? k : lastnz;
    nlast = N[k] > 0 ? N[k] : nlast;
    c = cn;
  }
  if (ks < 0) {  // unreachable for V < 1
    ks = lastnz;
    nk = nlast;
    cprev = 0.0;
  }
  const double aq = __dsub_rn(x, cprev);
  const double rk = rate[ks];
  long long j = __double2ll_rd(rk == 1.0 ? aq : __ddiv_rn(aq, rk));
  if (j > nk - 1) j = nk - 1;
  if (j < 0) j = 0;
  // rank-select across rows: exclusive prefix of per-row counts
  const uint32_t mk = C.mask(ks);
  const int cnt = __popc(mk);
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const int excl = incl - cnt;
  const unsigned b = __ballot_sync(0xffffffffu, excl <= (int)j && (int)j < incl);
  const int rs = __ffs(b) - 1;
  const int jj = __shfl_sync(0xffffffffu, (int)j - excl, rs);
  const uint32_t rowmask = __shfl_sync(0xffffffffu, mk, rs);
  return rs * BX + nth_bit<uint32_t, 32>(rowmask, jj);
}

// ---------------------------------------------------------------------------
// K1 (warp form).  Grid-stride over the work items, one warp per region.
// ---------------------------------------------------------------------------
template <int BX, int BY, bool LOG>
__global__ void __launch_bounds__(128) region_kernel_w(const KArgs a) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const bool wrapX = a.RX == 1, wrapY = a.RYg == 1;
  const unsigned K = stamp_of(a), K0 = a.it_K0;
  ktime_begin(a);
  unsigned long long n_ev = 0, n_out = 0, n_in = 0, n_cmp = 0, n_reg = 0;
  unsigned fmax = 0;
  bool changed = false, overflow = false;

  const int n_all = a.n_work_dev ? (int)__ldcg(a.n_work_dev) : a.n_work;
  for (int item = warp; item < n_all; item += nwarps) {
    const int idx = a.wl_in ? (int)a.wl_in[item] : item;
    const int r = idx / a.RX, c = idx - r * a.RX;
    const uint32_t gid = (uint32_t)((a.row0 + r) * a.RX + c);
    ++n_reg;
    // ---- committed state ----
    uint32_t row = lane < BY ? ((const uint32_t*)a.in.spins)[(long long)idx * BY + lane] : 0u;
    const uint4 h = ((const uint4*)a.in.halo)[idx];  // gN, gS, gW (bit per row), gE
    uint32_t gN = h.x, gS = h.y;
    uint32_t gWb = lane < BY ? (h.z >> lane) & 1u : 0u, gEb = lane < BY ? (h.w >> lane) & 1u : 0u;
    double ts = a.fresh_w ? a.t_c : a.in.ts[idx], R = a.in.R[idx];
    uint32_t n = a.in.n[idx];
    unsigned long long dig = a.digest ? a.in.dig[idx] : 0ull;
    unsigned n_ev_r = 0, bev = 0;

    // ---- incoming histories (uniform cursors) ----
    // lane q caches entry 32 * floor(hidx / 32) + q of each incoming history
    // (lt, lp), so a break point reads its successor with a shuffle
    unsigned hcnt[4], hidx[4], hsrc[4], hoff[4];
    double ht[4], lt[4];
    int hpos[4];
    unsigned lp = 0;  // byte d: cached position of direction d
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      hcnt[d] = 0; hidx[d] = 0; hsrc[d] = 0; hoff[d] = 0; ht[d] = dinf(); hpos[d] = 0;
      const bool axis_off = (d < 2) ? wrapY : wrapX;
      if (a.first || axis_off) continue;
      const bool ghost = a.ghost && ((d == EDGE_N && r == 0) || (d == EDGE_S && r == a.RYl - 1));
      if (ghost) {
        hcnt[d] = (d == EDGE_N ? a.gh_up : a.gh_down).cnt[c];
        hsrc[d] = d == EDGE_N ? 2u : 3u;
        hoff[d] = (unsigned)c;
      } else {
        const int nr = d == EDGE_N ? wdec(r, a.RYl) : d == EDGE_S ? winc(r, a.RYl) : r;
        const int nc = d == EDGE_W ? wdec(c, a.RX) : d == EDGE_E ? winc(c, a.RX) : c;
        const unsigned long long v = latest_edge_word(a.sel, ((long long)nr * a.RX + nc) * 4 + (d ^ 1), K);
        if (word_valid(v, K0)) {
          hcnt[d] = ew_count(v);
          hsrc[d] = ew_slot(v);
          hoff[d] = ((unsigned)nr * (unsigned)a.K) * (unsigned)a.RX + (unsigned)nc;
        }
      }
      lt[d] = dinf();
      if (hcnt[d] > 0) {
        if ((unsigned)lane < hcnt[d]) {
          const unsigned off = hoff[d] + (unsigned)lane * (unsigned)a.RX;
          lt[d] = src_t(a, hsrc[d], d ^ 1)[off];
          lp |= (unsigned)src_p(a, hsrc[d], d ^ 1)[off] << (8 * d);
        }
        ht[d] = __shfl_sync(0xffffffffu, lt[d], 0);
        hpos[d] = (int)((__shfl_sync(0xffffffffu, lp, 0) >> (8 * d)) & 0xFFu);
      }
      n_in += hcnt[d];
    }
    // ---- own latest histories ----
    unsigned oc[4], pc[4], ps[4], dv[4], wh[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      oc[e] = 0; pc[e] = 0; ps[e] = 0; dv[e] = 0; wh[e] = 0;
      if (LOG) continue;
      const ulonglong2 wp = reinterpret_cast<const ulonglong2*>(a.sel)[(long long)idx * 4 + e];
      const int li = latest_index(wp, K);
      const unsigned long long v = li ? wp.y : wp.x;
      ps[e] = ew_slot(v);
      pc[e] = word_valid(v, K0) ? ew_count(v) : 0u;
      wh[e] = (unsigned)(li ^ 1);
      n_cmp += pc[e];
    }
    const unsigned obase = (unsigned)(((long long)r * a.K) * a.RX + c);

    double U, V;
    draw_pair(a.seed, gid, n, U, V, a.gen);
    if (a.fresh_w) R = budget(a, U);  // the slate is wiped at t_c
    WClasses C = wbuild<BX, BY>(row, gN, gS, gWb, gEb, wrapX, wrapY);
    int N[10];
    wcounts(C, N);
    double lam = wfold(N, a.rate);
    double tc = cand_time(ts, R, lam);

    for (;;) {
      int dstar = -1;
      double tb = dinf();
      uint32_t nb = 0xffffffffu;
#pragma unroll
      for (int d = 0; d < 4; ++d) {
        if (hidx[d] < hcnt[d]) {
          const uint32_t nid = neighbour_id(a, gid, d);
          if (ht[d] < tb || (ht[d] == tb && nid < nb)) {
            dstar = d;
            tb = ht[d];
            nb = nid;
          }
        }
      }
      const bool bp = dstar >= 0 && (tb < tc || (tb == tc && nb < gid));
      const bool ev = !bp && tc < a.t_w;
      if (!bp && !ev) break;
      if (ev) {
        const int site = wselect<BX, BY>(C, N, a.rate, V, lam);
        const int sr = site / BX, sc = site - sr * BX;
        if (lane == sr) row ^= 1u << sc;
        if (a.digest)
          dig = digest_step(dig, tc, site);
        const unsigned up_new = (__shfl_sync(0xffffffffu, row, sr) >> sc) & 1u;  // the new spin (for dM)
        if (LOG) {
          if (lane == 0) {
            const unsigned long long o = a.log_off[idx] + n_ev_r;
            a.log_t[o] = tc;
            a.log_region[o] = gid;
            a.log_site[o] = (uint16_t)site;
            if (a.log_dm) a.log_dm[o] = up_new ? 2 : -2;
          }
        } else {
          if (lane == 0 && a.ev_t && (int)n_ev_r < a.evC) {  // scratch event log
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
              const long long o = e * a.tstride + (long long)(obase + k * (unsigned)a.RX);
              if (lane == 0) {
                const EdgeView& Pnew = ps[e] ? a.ed[0] : a.ed[1];
                Pnew.t[o] = tc;
                Pnew.pos[o] = p;
              }
              ++n_out;
            } else {
              overflow = true;
            }
            oc[e] = k + 1;
          }
          bev += on_edge ? 1u : 0u;
        }
        ++n_ev_r;
        ts = tc;
      } else {
        const double Rn = __dsub_rn(R, __dmul_rn(lam, __dsub_rn(tb, ts)));
        R = Rn < 0.0 ? 0.0 : Rn;
        ts = tb;
#pragma unroll
        for (int d = 0; d < 4; ++d) {
          if (d != dstar) continue;
          const int p = hpos[d];
          if (d == EDGE_N) gN ^= 1u << p;
          else if (d == EDGE_S) gS ^= 1u << p;
          else if (d == EDGE_W) { if (lane == p) gWb ^= 1u; }
          else { if (lane == p) gEb ^= 1u; }
          const unsigned nx = ++hidx[d];
          if (nx < hcnt[d]) {
            if ((nx & 31u) == 0) {  // next chunk of 32 entries
              lp &= ~(0xFFu << (8 * d));
              if (nx + (unsigned)lane < hcnt[d]) {
                const unsigned off = hoff[d] + (nx + (unsigned)lane) * (unsigned)a.RX;
                lt[d] = src_t(a, hsrc[d], d ^ 1)[off];
                lp |= (unsigned)src_p(a, hsrc[d], d ^ 1)[off] << (8 * d);
              }
            }
            ht[d] = __shfl_sync(0xffffffffu, lt[d], (int)(nx & 31u));
            hpos[d] = (int)((__shfl_sync(0xffffffffu, lp, (int)(nx & 31u)) >> (8 * d)) & 0xFFu);
          }
        }
      }
      C = wbuild<BX, BY>(row, gN, gS, gWb, gEb, wrapX, wrapY);
      wcounts(C, N);
      lam = wfold(N, a.rate);
      if (ev) {
        ++n;
        draw_pair(a.seed, gid, n, U, V, a.gen);
        R = budget(a, U);
      }
      tc = cand_time(ts, R, lam);
    }
    n_ev += n_ev_r;
    fmax = max(fmax, bev);

    if (!LOG) {
      // statement (c): compare each new edge history with the latest one,
      // 32 entries per warp step (the new entries were stored by lane 0)
      __syncwarp();
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (oc[e] != pc[e] || oc[e] == 0 || (int)oc[e] > a.K) continue;
        const double* Tn = src_t(a, ps[e] ^ 1u, e);
        const double* To = src_t(a, ps[e], e);
        const uint8_t* Pn = src_p(a, ps[e] ^ 1u, e);
        const uint8_t* Po = src_p(a, ps[e], e);
        for (unsigned q0 = 0; q0 < oc[e] && !dv[e]; q0 += 32) {
          bool df = false;
          const unsigned q = q0 + (unsigned)lane;
          if (q < oc[e]) {
            const unsigned o = obase + q * (unsigned)a.RX;
            df = __double_as_longlong(__ldcg(Tn + o)) != __double_as_longlong(__ldcg(To + o)) ||
                 __ldcg(Pn + o) != __ldcg(Po + o);
          }
          dv[e] = __any_sync(0xffffffffu, df) ? 1u : 0u;
        }
      }
      unsigned chmask = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if ((int)oc[e] > a.K) overflow = true;
        const bool diff = dv[e] || oc[e] != pc[e];
        if (diff) {
          chmask |= 1u << e;
          if (lane == 0) {
            const unsigned cnt = (int)oc[e] < a.K ? oc[e] : (unsigned)a.K;
            a.sel[((long long)idx * 4 + e) * 2 + wh[e]] =
                ((unsigned long long)K << 32) | ((unsigned long long)cnt << 1) | (ps[e] ^ 1u);
          }
        }
      }
      if (chmask) {
        changed = true;
        if (lane == 0) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (!((chmask >> e) & 1u)) continue;
            if (a.ghost && ((e == EDGE_N && r == 0) || (e == EDGE_S && r == a.RYl - 1))) continue;
            const int nr = e == EDGE_N ? wdec(r, a.RYl) : e == EDGE_S ? winc(r, a.RYl) : r;
            const int nc = e == EDGE_W ? wdec(c, a.RX) : e == EDGE_E ? winc(c, a.RX) : c;
            mark_dirty(a, nr * a.RX + nc, K + 1);
          }
        }
      }
      if (lane < BY) ((uint32_t*)a.out.spins)[(long long)idx * BY + lane] = row;
      const uint32_t gw = __ballot_sync(0xffffffffu, gWb != 0u), ge = __ballot_sync(0xffffffffu, gEb != 0u);
      if (lane == 0) {
        ((uint4*)a.out.halo)[idx] = make_uint4(gN, gS, gw, ge);
        a.out.ts[idx] = ts;
        a.out.R[idx] = R;
        a.out.n[idx] = n;
        if (a.digest) a.out.dig[idx] = dig;
      }
    }
  }

  ktime_end(a);
  if (!LOG && lane == 0) {
    if (changed) atomicOr(&a.flags[0], 1);
    if (overflow) atomicOr(&a.flags[1], 1);
    if (n_reg) {
      atomicAdd(&a.stats[0], n_ev);
      atomicAdd(&a.stats[1], n_out);
      atomicAdd(&a.stats[2], n_in);
      atomicAdd(&a.stats[3], n_cmp);
      atomicMax(&a.stats[4], (unsigned long long)fmax);
      atomicAdd(&a.stats[5], n_reg);
    }
  }
}

// FLAG_OBSERVABLES snapshot for the row layout (see snap_kernel): M and the
// owned bonds (internal, north, west) of every region, exact integers
template <int BX, int BY>
__global__ void __launch_bounds__(256) snap_kernel_w(StateView st, int n, int RX, int RYg, unsigned long long* out) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  long long m = 0, b = 0;
  if (idx < n) {
    constexpr uint32_t FULL = BX == 32 ? 0xffffffffu : ((1u << BX) - 1u);
    const uint32_t* rows = (const uint32_t*)st.spins + (long long)idx * BY;
    const uint4 h = ((const uint4*)st.halo)[idx];
    const bool wrapX = RX == 1, wrapY = RYg == 1;
    for (int ly = 0; ly < BY; ++ly) {
      const uint32_t r = rows[ly];
      m += 2 * __popc(r) - BX;
      if (BX > 1) b += 2 * __popc(~(r ^ (r >> 1)) & (FULL >> 1)) - (BX - 1);  // (x, x+1) in the row
      const uint32_t up = ly > 0 ? rows[ly - 1] : (wrapY ? rows[BY - 1] : h.x);  // north neighbour row
      b += 2 * __popc(~(r ^ up) & FULL) - BX;
      const uint32_t wb = wrapX ? (r >> (BX - 1)) & 1u : (h.z >> ly) & 1u;        // west neighbour bit
      b += ((r & 1u) == wb) ? 1 : -1;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    m += __shfl_xor_sync(0xffffffffu, m, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(out, (unsigned long long)m);
    atomicAdd(out + 1, (unsigned long long)b);
  }
}

// K0 for the warp form: rows as u32 masks, halo as {N row, S row, W bits, E bits}
template <int BX, int BY>
__global__ void init_kernel_w(const uint8_t* buf, int Lx, int RX, int RYl, int row0, unsigned long long seed, double eq_q,
                              StateView st) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= RX * RYl) return;
  const int r = idx / RX, c = idx - r * RX;
  const int y0 = 1 + r * BY, x0 = c * BX;
  uint32_t gN = 0, gS = 0, gW = 0, gE = 0;
  for (int ly = 0; ly < BY; ++ly) {
    uint32_t row = 0;
    for (int lx = 0; lx < BX; ++lx)
      if (buf[(long long)(y0 + ly) * Lx + x0 + lx]) row |= 1u << lx;
    ((uint32_t*)st.spins)[(long long)idx * BY + ly] = row;
    if (buf[(long long)(y0 + ly) * Lx + (x0 - 1 + Lx) % Lx]) gW |= 1u << ly;
    if (buf[(long long)(y0 + ly) * Lx + (x0 + BX) % Lx]) gE |= 1u << ly;
  }
  for (int lx = 0; lx < BX; ++lx) {
    if (buf[(long long)(y0 - 1) * Lx + x0 + lx]) gN |= 1u << lx;
    if (buf[(long long)(y0 + BY) * Lx + x0 + lx]) gS |= 1u << lx;
  }
  ((uint4*)st.halo)[idx] = make_uint4(gN, gS, gW, gE);
  double U, V;
  draw_pair(seed, (uint32_t)((row0 + r) * RX + c), 0u, U, V);
  st.ts[idx] = 0.0;
  st.R[idx] = quantize_budget(expvar(U), eq_q);
  st.n[idx] = 0;
  st.dig[idx] = 0ull;
}

template <int BX, int BY>
__global__ void unpack_kernel_w(StateView st, int Lx, int RX, int RYl, uint8_t* out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nsite = (long long)RYl * BY * Lx;
  if (i >= nsite) return;
  const int y = (int)(i / Lx), x = (int)(i - (long long)y * Lx);
  const int r = y / BY, c = x / BX;
  const uint32_t row = ((const uint32_t*)st.spins)[(long long)(r * RX + c) * BY + (y - r * BY)];
  out[i] = (uint8_t)((row >> (x - c * BX)) & 1u);
}

// K4 for the per-edge selector layout: column c of one direction
__device__ __forceinline__ void pack_col_w(const KArgs& a, bool up, int c, const GhostView& g) {
  const int r = up ? 0 : a.RYl - 1;
  const int e = up ? EDGE_N : EDGE_S;
  const ulonglong2 wp = reinterpret_cast<const ulonglong2*>(a.sel)[((long long)r * a.RX + c) * 4 + e];
  const unsigned K = stamp_of(a);
  const unsigned long long v = latest_word(wp, K + 1);
  int cnt = 0;
  if (word_valid(v, a.it_K0)) {
    const EdgeView& E = ew_slot(v) ? a.ed[1] : a.ed[0];
    cnt = (int)ew_count(v);
    const long long base = (long long)e * a.tstride + ((long long)r * a.K) * a.RX + c;
    for (int q = 0; q < cnt; ++q) {
      g.t[(long long)q * a.RX + c] = E.t[base + (long long)q * a.RX];
      g.pos[(long long)q * a.RX + c] = E.pos[base + (long long)q * a.RX];
    }
  }
  g.cnt[c] = (uint16_t)cnt;
  g.stamp[c] = (unsigned)(v >> 32) == K ? K : 0u;
}

__global__ void pack_kernel_w(const KArgs a, GhostView send_up, GhostView send_down) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 2 * a.RX) return;
  const bool up = i < a.RX;
  pack_col_w(a, up, up ? i : i - a.RX, up ? send_up : send_down);
}

}  // namespace isr
