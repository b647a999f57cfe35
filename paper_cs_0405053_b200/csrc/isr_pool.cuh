// isr_pool.cuh -- region-trajectory kernel (K1), slot-pool form for regions
// of <= 64 sites: the same relaxation iteration as region_kernel
// (isr_region.cuh), scheduled for SIMT efficiency.
//
// Each warp keeps a pool of S regions ("slots") resident in shared memory.
// One round of the warp:
//   decide  every occupied slot finds its next step -- the earliest of its
//           next break point and its own event (next_bp2), or "done" when
//           both lie beyond the window end;
//   events  the slots whose next step is an own event are dealt densely to
//           the 32 lanes (slot = q-th set bit of the event mask), so every
//           lane runs the same event code (select, flip, history, next pair
//           of the list, refold);
//   breaks  likewise for the slots whose next step is a break point;
//   refill  when enough slots are done, they are published (lane_finish,
//           with the history diff of statement (c)) and reloaded
//           with the next regions of the block's work tile.
// Per region the steps run in exactly the order of the lane kernel, so the
// results are bit-identical; only the assignment of regions to lanes moves.
#pragma once
#include "isr_region.cuh"

namespace isr {

#ifndef ISR_POOL_S
#define ISR_POOL_S 64   // slots per warp (<= 64: slot masks are 64-bit)
#endif
#ifndef ISR_POOL_CI
#define ISR_POOL_CI 2   // staged incoming entries per history
#endif
constexpr int PW = 4;   // warps per block of the pool kernel

template <class G, int S>
struct PoolSlots {
  using M = typename G::M;
  uint32_t idx[S];
  M sp[S], gn[S], gs[S], gw[S], ge[S];
  double ts[S], R[S], V[S], lam[S], tc[S];
  uint32_t n[S], nev[S], bev[S];
  int site[S];     // atom of the next event (ISR_SELAHEAD)
  uint32_t fl[S];  // bit 0: selector word to overwrite; bits 4-5: direction of the next break point
  unsigned long long dig[S];
  uint32_t hm[4][S];
  double ht[4][S];
  uint32_t hoff[4][S];
  uint32_t om[4][S];
};

template <class G, int S>
struct PoolSmem {
  ProdTable<G> PT;
  StageT<PW * S, false, ISR_POOL_CI> St;  // column = warp * S + slot
  PoolSlots<G, S> W[PW];
  unsigned q_next;
};

template <class G, int S>
constexpr size_t pool_smem_bytes() {
  return sizeof(PoolSmem<G, S>);
}

__device__ __forceinline__ int nth_bit64(unsigned long long m, int q) {
  const unsigned lo = (unsigned)m;
  const int c = __popc(lo);
  if (q < c) return nth_bit<uint32_t, 32>(lo, q);
  return 32 + nth_bit<uint32_t, 32>((unsigned)(m >> 32), q - c);
}

template <class G, int S>
__device__ __forceinline__ void slot_get(const KArgs& a, const PoolSlots<G, S>& P, int s, Lane<G>& L) {
  L.idx = (int)P.idx[s];
  L.gid = (uint32_t)(a.row0 * a.RX) + (uint32_t)L.idx;
  const int r = div_rx(a, L.idx), c = L.idx - r * a.RX;
  L.obase = (unsigned)(((long long)r * a.K) * a.RX + c);
  L.spins = P.sp[s];
  L.gN = P.gn[s];
  L.gS = P.gs[s];
  L.gW = P.gw[s];
  L.gE = P.ge[s];
  L.ts = P.ts[s];
  L.R = P.R[s];
  L.V = P.V[s];
  L.lam = P.lam[s];
  L.tc = P.tc[s];
  L.n = P.n[s];
  L.n_ev = P.nev[s];
  L.bev = P.bev[s];
  L.whalf = (int)(P.fl[s] & 1u);
  L.site = P.site[s];
  L.dig = P.dig[s];
#pragma unroll
  for (int d = 0; d < 4; ++d) {
    L.hm[d] = P.hm[d][s];
    L.ht[d] = P.ht[d][s];
    L.hoff[d] = P.hoff[d][s];
    L.om[d] = P.om[d][s];
  }
}

// the fields a step (event or break point) and its refold change
template <class G, int S>
__device__ __forceinline__ void slot_put_step(PoolSlots<G, S>& P, int s, const Lane<G>& L) {
  P.lam[s] = L.lam;
  P.tc[s] = L.tc;
  P.site[s] = L.site;
}

template <class G, int S>
__device__ __forceinline__ void slot_put_all(PoolSlots<G, S>& P, int s, const Lane<G>& L) {
  P.idx[s] = (uint32_t)L.idx;
  P.sp[s] = L.spins;
  P.gn[s] = L.gN;
  P.gs[s] = L.gS;
  P.gw[s] = L.gW;
  P.ge[s] = L.gE;
  P.ts[s] = L.ts;
  P.R[s] = L.R;
  P.V[s] = L.V;
  P.lam[s] = L.lam;
  P.tc[s] = L.tc;
  P.n[s] = L.n;
  P.nev[s] = L.n_ev;
  P.bev[s] = L.bev;
  P.fl[s] = (unsigned)L.whalf;
  P.dig[s] = L.dig;
#pragma unroll
  for (int d = 0; d < 4; ++d) {
    P.hm[d][s] = L.hm[d];
    P.ht[d][s] = L.ht[d];
    P.hoff[d][s] = L.hoff[d];
    P.om[d][s] = L.om[d];
  }
  slot_put_step<G, S>(P, s, L);
}

template <int BX, int BY, int S>
__global__ void __launch_bounds__(PW * 32) region_kernel_pool(const KArgs a) {
  using G = Geo<BX, BY>;
  static_assert(S >= 32 && S <= 64, "32 <= S <= 64");
  extern __shared__ __align__(16) unsigned char pool_smem_raw[];
  PoolSmem<G, S>& SM = *reinterpret_cast<PoolSmem<G, S>*>(pool_smem_raw);
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  PoolSlots<G, S>& P = SM.W[wid];
  const int col0 = wid * S;
  // work: a static tile per block, or (work_ctr set) the whole worklist as
  // one global queue shared by a persistent grid, its length read on device
  const bool global_q = a.work_ctr != nullptr;
  const int n_all = a.n_work_dev ? (int)__ldcg(a.n_work_dev) : a.n_work;
  const int tile_begin = global_q ? 0 : blockIdx.x * a.tile;
  const int tile_n = global_q ? n_all : min(a.tile, n_all - tile_begin);
  if (threadIdx.x == 0) SM.q_next = 0;
  fill_prod<G>(SM.PT, a.rate);
  __syncthreads();
  const ProdTable<G>& PT = SM.PT;
  constexpr unsigned long long ALL = S == 64 ? ~0ull : ((1ull << S) - 1ull);
  const int REFILL = a.refill;

  unsigned n_ev = 0, n_out = 0, n_in = 0, n_cmp = 0, n_bev = 0, n_reg = 0;
  bool changed = false, overflow = false;
  unsigned long long occ = 0;  // slots holding a region (warp-uniform)
  bool exhausted = tile_n <= 0;

  for (;;) {
    // ---- decide: next step of every occupied slot ----
    unsigned long long evm = 0, bpm = 0;
#pragma unroll
    for (int h = 0; h < (S + 31) / 32; ++h) {
      const int s = h * 32 + lane;
      int typ = 0;
      if (s < S && ((occ >> s) & 1ull)) {
        Lane<G> L;
        L.gid = (uint32_t)(a.row0 * a.RX) + P.idx[s];
        L.tc = P.tc[s];
#pragma unroll
        for (int d = 0; d < 4; ++d) L.ht[d] = P.ht[d][s];
        double tb;
        const int d = next_bp2<G>(a, L, tb);
        if (d >= 0) {
          typ = 2;
          P.fl[s] = (P.fl[s] & 1u) | ((unsigned)d << 4);
        } else if (L.tc < a.t_w) {
          typ = 1;
        }
      }
      evm |= (unsigned long long)__ballot_sync(FULL, typ == 1) << (32 * h);
      bpm |= (unsigned long long)__ballot_sync(FULL, typ == 2) << (32 * h);
    }
    __syncwarp();  // the break-point directions written above are read by other lanes
    const unsigned long long done = occ & ~(evm | bpm);
    const unsigned long long freem = ~occ & ALL;

    // ---- refill: publish finished regions, load the next ones ----
    if ((evm | bpm) == 0 || (!exhausted && __popcll(done | freem) >= REFILL)) {
      if ((evm | bpm) == 0 && done == 0 && exhausted) break;
      const unsigned long long cand = done | (exhausted ? 0ull : freem);
      const int ncand = __popcll(cand);
      int base = 0, nnew = 0;
      if (!exhausted) {
        unsigned b = 0;
        if (lane == 0) b = atomicAdd(global_q ? a.work_ctr : &SM.q_next, (unsigned)ncand);
        base = (int)__shfl_sync(FULL, b, 0);
        nnew = max(0, min(ncand, tile_n - base));
        if (base + ncand >= tile_n) exhausted = true;
      }
      // publish the finished regions
      const int ndone = __popcll(done);
      for (int p = 0; p * 32 < ndone; ++p) {
        const int q = p * 32 + lane;
        if (q < ndone) {
          const int s = nth_bit64(done, q);
          Lane<G> L;
          slot_get<G, S>(a, P, s, L);
          lane_finish<G, true>(a, L, changed, overflow, &n_cmp);
          n_ev += L.n_ev;
          n_bev = max(n_bev, L.bev);
        }
      }
      // load the next regions into the first nnew candidate slots
      unsigned long long loaded = 0;
      for (int p = 0; p * 32 < nnew; ++p) {
        const int q = p * 32 + lane;
        int s = 0;
        if (q < nnew) {
          s = nth_bit64(cand, q);
          const int item = base + q;
          const int idx = a.wl_in ? (int)a.wl_in[tile_begin + item] : tile_begin + item;
          Lane<G> L;
          lane_load<G, false>(a, L, idx, SM.St, PT, col0 + s);
          n_in += (L.hm[0] & 0xFFu) + (L.hm[1] & 0xFFu) + (L.hm[2] & 0xFFu) + (L.hm[3] & 0xFFu);
          ++n_reg;
          slot_put_all<G, S>(P, s, L);
        }
        const bool ld = q < nnew;
        const unsigned lo = __reduce_or_sync(FULL, (ld && s < 32) ? (1u << s) : 0u);
        const unsigned hi = __reduce_or_sync(FULL, (ld && s >= 32) ? (1u << (s - 32)) : 0u);
        loaded |= (unsigned long long)lo | ((unsigned long long)hi << 32);
      }
      occ = (occ & ~done) | loaded;
      __syncwarp();
      continue;
    }

    // ---- own events, dealt densely to the lanes ----
    const int nev = __popcll(evm);
    for (int p = 0; p * 32 < nev; ++p) {
      const int q = p * 32 + lane;
      if (q < nev) {
        const int s = nth_bit64(evm, q);
        Lane<G> L;
        slot_get<G, S>(a, P, s, L);
        ev_pre2<G, false, true>(a, L, SM.St, PT, col0 + s, n_out, overflow);
        refold<G>(a, L, PT);
        P.sp[s] = L.spins;
        P.ts[s] = L.ts;
        P.R[s] = L.R;
        P.V[s] = L.V;
        slot_put_step<G, S>(P, s, L);
        P.n[s] = L.n;
        P.nev[s] = L.n_ev;
        P.bev[s] = L.bev;
        P.dig[s] = L.dig;
#pragma unroll
        for (int e = 0; e < 4; ++e) P.om[e][s] = L.om[e];
      }
    }
    // ---- break points, dealt densely to the lanes ----
    const int nbp = __popcll(bpm);
    for (int p = 0; p * 32 < nbp; ++p) {
      const int q = p * 32 + lane;
      if (q < nbp) {
        const int s = nth_bit64(bpm, q);
        const int d = (int)((P.fl[s] >> 4) & 3u);
        Lane<G> L;
        slot_get<G, S>(a, P, s, L);
        const double tb = d == 0 ? L.ht[0] : d == 1 ? L.ht[1] : d == 2 ? L.ht[2] : L.ht[3];
        bp_pre2<G>(a, L, SM.St, col0 + s, d, tb);
        refold<G>(a, L, PT);
        P.gn[s] = L.gN;
        P.gs[s] = L.gS;
        P.gw[s] = L.gW;
        P.ge[s] = L.gE;
        P.ts[s] = L.ts;
        P.R[s] = L.R;
        slot_put_step<G, S>(P, s, L);
        P.hm[d][s] = d == 0 ? L.hm[0] : d == 1 ? L.hm[1] : d == 2 ? L.hm[2] : L.hm[3];
        P.ht[d][s] = d == 0 ? L.ht[0] : d == 1 ? L.ht[1] : d == 2 ? L.ht[2] : L.ht[3];
      }
    }
    __syncwarp();
  }

  // warp-aggregated flags and counters (one atomic per warp)
  const unsigned anych = __ballot_sync(FULL, changed);
  const unsigned anyov = __ballot_sync(FULL, overflow);
  unsigned long long v0 = n_ev, v1 = n_out, v2 = n_in, v3 = n_cmp, v5 = n_reg;
  unsigned fmax = n_bev;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v0 += __shfl_xor_sync(FULL, v0, o);
    v1 += __shfl_xor_sync(FULL, v1, o);
    v2 += __shfl_xor_sync(FULL, v2, o);
    v3 += __shfl_xor_sync(FULL, v3, o);
    v5 += __shfl_xor_sync(FULL, v5, o);
    fmax = max(fmax, __shfl_xor_sync(FULL, fmax, o));
  }
  if (lane == 0) {
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

}  // namespace isr
