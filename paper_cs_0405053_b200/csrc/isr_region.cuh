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
  // 1x1 regions: the single site is on all four edges, so the four edge
  // histories are identical; only edge 0's is stored (and read for every
  // direction), the selector word repeats its slot and count for all edges
  static constexpr bool SE = NS == 1;
  __host__ __device__ static constexpr int arr(int e) { return SE ? 0 : e; }
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
  double* oM;  // FLAG_OBSERVABLES: int M dt, int B dt of the region over the window
  double* oB;
};

// Boundary histories of one slot: t/pos[4][RYl][K][RX] (entry q of edge e of
// region (r, c) at ((e * RYl + r) * K + q) * RX + c).  Every region edge has
// two slots; which one holds its latest history, and how many entries it
// has, is recorded in the region's selector words (see latest_word).
struct EdgeView {
  double* t;
  uint8_t* pos;
};

// A ghost row received from a neighbouring strip (world > 1):
// cnt[RX], stamp[RX] (global iteration of the last change), t/pos[K][RX].
struct GhostView {
  uint16_t* cnt;
  uint32_t* stamp;
  double* t;
  uint8_t* pos;
};

struct KArgs {
  StateView in, out;
  EdgeView ed[2];
  unsigned long long* sel;      // per region: 2 selector words (parity K & 1)
  GhostView gh_up, gh_down;     // world > 1: rows above / below the strip
  int RX, RYl, RYg, row0, world;
  int ghost;          // the strip's first/last region rows read ghost rows (world > 1, or halo loopback)
  int single_edge;    // 1x1 regions: one stored edge history per region (Geo::SE)
  int K;
  long long tstride;  // elements per edge in t/pos (RYl * K * RX)
  long long sstride;  // elements from slot 0's arrays to slot 1's (ed[1].t == ed[0].t + sstride: one allocation)
  unsigned it_K;      // global iteration stamp of this launch (>= 1); with `trip`: the stamp of loop trip 0
  // device-side window loop (a CUDA graph with a conditional while node): the
  // loop body holds two iterations, so this launch's stamp is it_K + 2 * (*trip)
  const unsigned* trip;
  // the launch's device time: min start / max end of its blocks (%globaltimer, ns)
  unsigned long long* ktime;
  unsigned it_K0;     // stamp of the window's first iteration
  int first;          // window's first iteration: canonical assumption
  int digest;
  double t_w;         // window end
  double t_c;         // window start (committed time)
  int fresh_w;        // alternate approach: every region restarts at t_c with fresh numbers
  int obs;            // FLAG_OBSERVABLES: accumulate int M dt, int B dt per region
  unsigned gen;       // generation of the random numbers in use (window index if fresh_w, else 0)
  unsigned long long seed;
  double rate[10];
  // big-region kernel: step log of each region's last recomputation in this
  // window (time, budget after the step, step code), so a recomputation can
  // resume just before the first changed incoming entry (isr_big.cuh)
  double2* lg_tR;          // {time, budget after the step}
  uint16_t* lg_c;
  uint2* lg_meta;          // per region: {stamp of the recomputation that wrote the log, length}
  int LC;                  // log capacity (steps) per region
  int resume;
  // big-region kernel: the window's pairs (E(U_m), V_m) per region, m = n0 ..
  // n0 + fill - 1 (the paper's presimulated list); pmeta = {stamp
  // of the window's first iteration, fill}
  double2* pcache;
  uint2* pmeta;
  int PC;
  const uint32_t* wl_in;   // regions to recompute (nullptr: all regions)
  int n_work;              // number of regions to recompute
  const unsigned* n_work_dev;  // if set: the number is read here on the device (pipelined / graph loop, replay)
  int tile;                // work items per block (lane-persistent scheduling)
  unsigned rx_M;           // idx / RX == (idx * rx_M) >> rx_k for idx < 2^31 (host-computed)
  int rx_k;
  int refill;              // idle lanes per warp that trigger a batched refill
  int plain;               // launch the PLAIN instantiation where it applies (host dispatch only)
  int spread_log2;         // big-region K1: one region per 2^spread_log2 threads (small worklists)
  int lane_spread;         // lane K1: the largest k of its spread (one region per 2^k lanes; 0 = off)
  // PLAIN iterations after the first: per worklist item {region, incoming
  // counts (byte d), own latest counts (byte e), incoming slots (2 bits per d)
  // | own latest slots << 8 | word to overwrite << 12}, written by
  // describe_kernel from the selector words after the compaction
  const uint4* desc;
  uint32_t* wl_out;        // worklist of the next iteration
  unsigned* wl_out_count;
  uint32_t* dirty;         // dirty-region bitmaps [2][dwords], parity of the iteration they are for
  int dwords;              // 32-bit words per bitmap
  int* flags;                   // [0] changed, [1] overflow
  unsigned long long* stats;    // [0] events [1] entries out [2] entries in [3] entries cmp [4] f max [5] regions
  // scratch event log (FLAG_LOG_EVENTS): event q of a region's latest
  // recomputation at ev_t/ev_s[q * ev_stride + idx] for q < evC; commit
  // compacts it (regions with more events are replayed)
  double* ev_t;
  uint16_t* ev_s;
  long long ev_stride;
  int evC;
  double eq_q;        // > 0: quantized budgets E <- (floor(E q) + 1) / q (exact time ties; test mode)
  unsigned delay_ns;  // test knob (env ISING_SR_K1_DELAY_NS): K1 blocks sleep before publishing their flags
  // log replay
  int8_t* log_dm;     // dM of each logged event (+2 / -2), may be null
  double* log_t;
  uint32_t* log_region;
  uint16_t* log_site;
  const unsigned long long* log_off;
  long long log_cap;  // entries allocated for the log (ISR_CHECK bounds)
};

__device__ __forceinline__ unsigned stamp_of(const KArgs& a) { return a.trip ? a.it_K + 2u * __ldcg(a.trip) : a.it_K; }
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// block-level start / end stamps of a launch (the graph loop's K1 timing)
__device__ __forceinline__ void ktime_begin(const KArgs& a) {
  if (a.ktime && threadIdx.x == 0) atomicMin(a.ktime, globaltimer_ns());
}
__device__ __forceinline__ void ktime_end(const KArgs& a) {
  if (a.ktime && threadIdx.x == 0) atomicMax(a.ktime + 1, globaltimer_ns());
}

// The budget drawn from U: E(U) (R25), or with eq_q > 0 (tie test
// mode, R30) the quantized (floor(E(U) eq_q) + 1) / eq_q, exact
// for a power-of-two eq_q, so that equal event times across regions are common.
__device__ __forceinline__ double quantize_budget(double E, double q) {
  return q > 0.0 ? __ddiv_rn(__dadd_rn(floor(__dmul_rn(E, q)), 1.0), q) : E;
}
__device__ __forceinline__ double budget(const KArgs& a, double U) { return quantize_budget(expvar(U), a.eq_q); }

// test knob: a K1 made artificially slow (exposes any work that is not
// ordered after K1 on the stream, e.g. an exchange on another stream)
__device__ __noinline__ void k1_delay(unsigned ns) {
  for (unsigned t = 0; t < ns; t += 1000) __nanosleep(1000);
}

// Selector words of a region: two 64-bit words.  When its histories change
// in iteration K the region's thread overwrites the OLDER of its two words
// with stamp K; readers take the word with the largest stamp below K, which
// therefore is never the one being written (a 64-bit aligned store is
// single-copy atomic, so the word being written reads either as its old,
// older-stamped value or with stamp K, and is ignored either way).  Layout:
//   bits 0-3   slot holding the history of edge e
//   bits 4-31  4 x 7-bit entry counts (edge e at bit 4 + 7e)
//   bits 32-63 stamp: global iteration of the change
// A stamp below K0 (before this window) means "canonical empty history".
constexpr int CNT_BITS = 7;
constexpr int CNT_MAX = (1 << CNT_BITS) - 1;

// index (0/1) of the word with the largest stamp below K
__device__ __forceinline__ int latest_index(ulonglong2 w, unsigned K) {
  const unsigned s0 = (unsigned)(w.x >> 32), s1 = (unsigned)(w.y >> 32);
  const bool v0 = s0 < K, v1 = s1 < K;
  return (v0 && (!v1 || s0 >= s1)) ? 0 : 1;
}

__device__ __forceinline__ unsigned long long latest_word(ulonglong2 w, unsigned K) {
  const int i = latest_index(w, K);
  const unsigned long long v = i ? w.y : w.x;
  return (unsigned)(v >> 32) < K ? v : 0ull;
}

__device__ __forceinline__ bool word_valid(unsigned long long v, unsigned K0) { return (unsigned)(v >> 32) >= K0; }
__device__ __forceinline__ int word_slot(unsigned long long v, int e) { return (int)((v >> e) & 1ull); }
__device__ __forceinline__ unsigned word_count(unsigned long long v, int e) {
  return (unsigned)((v >> (4 + CNT_BITS * e)) & CNT_MAX);
}

// bit-sliced per-site count of up neighbours u = p2 p1 p0 (binary, u <= 4);
// the sites of class k = 5 s + u are those with spin s and count u.
template <class G>
struct Classes {
  using M = typename G::M;
  M up, p0, p1, p2;

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
    const M k = s1 & s2;
    up = spins;
    p0 = s1 ^ s2;
    p1 = c1 ^ c2 ^ k;
    p2 = (c1 & c2) | (k & (c1 ^ c2));
  }
  // sites of class k (k may be a run-time value: selects, no branches)
  __device__ __forceinline__ M mask(int k) const {
    constexpr M FULL = G::full();
    const bool hi = k >= 5;
    const int u = hi ? k - 5 : k;
    const M a0 = (u & 1) ? p0 : (M)~p0, a1 = (u & 2) ? p1 : (M)~p1, a2 = (u & 4) ? p2 : (M)~p2;
    return (M)((hi ? up : (M)~up) & a0 & a1 & a2 & FULL);
  }
};

template <class M>
__device__ __forceinline__ int popc_m(M x) {
  if constexpr (sizeof(M) == 8) return __popcll(x);
  else return __popc(x);
}

// j-th (0-based) set bit of x, LSB first (local row-major order): binary
// search on popcounts of halves
template <class M, int NBITS>
__device__ __forceinline__ int nth_bit(M x, int j) {
  int pos = 0;
  if constexpr (NBITS > 32) {
    const int c = __popc((uint32_t)x);
    if (j >= c) { j -= c; x >>= 32; pos += 32; }
  }
  uint32_t y = (uint32_t)x;
  if constexpr (NBITS > 16) {
    const int c = __popc(y & 0xFFFFu);
    if (j >= c) { j -= c; y >>= 16; pos += 16; }
  }
  if constexpr (NBITS > 8) {
    const int c = __popc(y & 0xFFu);
    if (j >= c) { j -= c; y >>= 8; pos += 8; }
  }
  if constexpr (NBITS > 4) {
    const int c = __popc(y & 0xFu);
    if (j >= c) { j -= c; y >>= 4; pos += 4; }
  }
  if constexpr (NBITS > 2) {
    const int c = __popc(y & 0x3u);
    if (j >= c) { j -= c; y >>= 2; pos += 2; }
  }
  if constexpr (NBITS > 1) {
    const int c = (int)(y & 1u);
    if (j >= c) pos += 1;
  }
  return pos;
}


// Products fl(N * r_k) for N = 0..NS, one table per block in shared memory:
// the fold below adds exactly the values __dmul_rn((double)N_k, r_k) would
// give, so the result is bit-identical to multiplying in place.
template <class G>
struct ProdTable {
  double v[10][G::NS + 1];
  double rinv[10];  // fl(1 / r_k): screens floor((x - c_{k-1}) / r_k) (exact fallback near integers)
  __device__ __forceinline__ double at(int k, int n) const { return v[k][n]; }
};

template <class G>
__device__ __forceinline__ void fill_prod(ProdTable<G>& T, const double* rate) {
  for (int i = threadIdx.x; i < 10 * (G::NS + 1); i += blockDim.x) {
    const int k = i / (G::NS + 1), n = i - k * (G::NS + 1);
    T.v[k][n] = __dmul_rn((double)n, rate[k]);
  }
  if (threadIdx.x < 10) T.rinv[threadIdx.x] = __ddiv_rn(1.0, rate[threadIdx.x]);
}

// j = floor(fl(aq / rk)) for aq > 0, q = aq / rk <= 64: a product with the
// rounded reciprocal is within 1e-13 of the correctly rounded quotient, so it
// decides the floor unless the quotient is that close to an integer; then
// the IEEE division decides (bit-identical to always dividing)
static __constant__ double kFloorEps = 1e-12;  // a c[] operand, not two UMOVs per use
__device__ __forceinline__ long long floor_div(double aq, double rk, double rinv) {
  if (rk == 1.0) return __double2ll_rd(aq);  // aq / 1.0 == aq exactly
  const double qa = __dmul_rn(aq, rinv);
  const long long jl = __double2ll_rd(__dsub_rn(qa, kFloorEps)), jh = __double2ll_rd(__dadd_rn(qa, kFloorEps));
  return jl == jh ? jl : __double2ll_rd(__ddiv_rn(aq, rk));
}

// eq. biglambda followed at once by the atom selection for the next event
// (eqs. Wsum..vindex) on the same state: the partial sums c_k are still in
// registers, so the selection needs no second fold.  The decisions of eqs.
// Wstop/vindex with readings R8/R9 (first k with x <= c_k; j clamped);
// returns the site (any value when Lambda = 0, then no event can happen: the
// candidate time is +inf).
template <class G>
__device__ __forceinline__ int fold_select(const Classes<G>& C, const ProdTable<G>& T, const double* rate, double V,
                                           double& lam) {
  using M = typename G::M;
  double cs[10];
  double c = 0.0;
#pragma unroll
  for (int k = 0; k < 10; ++k) {
    c = __dadd_rn(c, T.at(k, popc_m(C.mask(k))));
    cs[k] = c;
  }
  lam = c;
  const double x = __dmul_rn(V, lam);
  // k* = the first k with x <= c_k = the number of k with c_k < x (the
  // partial sums never decrease: every term is >= 0); x = fl(V lam) <= lam for
  // V < 1, so k* <= 9, and the class k* has N_k* > 0 (x > 0)
  int ks = 0;
  double cprev = 0.0;
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const bool below = cs[k] < x;
    ks += below ? 1 : 0;
    cprev = below ? cs[k] : cprev;  // the last partial sum below x: c_{k*-1}
  }
  const M mk = C.mask(ks);
  const int nk = popc_m(mk);
  long long j = floor_div(__dsub_rn(x, cprev), rate[ks], T.rinv[ks]);
  j = j > nk - 1 ? nk - 1 : j;
  j = j < 0 ? 0 : j;
  return nth_bit<M, G::NS>(mk, (int)j);
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

// periodic neighbour row/column index without an integer division
__device__ __forceinline__ int wdec(int v, int n) { return v == 0 ? n - 1 : v - 1; }
__device__ __forceinline__ int winc(int v, int n) { return v == n - 1 ? 0 : v + 1; }

// FLAG_OBSERVABLES: magnetisation of the region and the sum of s(v) s(u) over
// its owned bonds (internal bonds, bonds to the north row and the west
// column: every lattice bond is owned by exactly one region), from the masks
template <class G>
__device__ __forceinline__ void obs_counts(typename G::M sp, typename G::M gN, typename G::M gW, bool wrapX,
                                           bool wrapY, int& Mi, int& Bi) {
  using M = typename G::M;
  constexpr int BX = G::BX, BY = G::BY;
  constexpr M FULL = G::full();
  Mi = 2 * popc_m(sp) - G::NS;
  int B = 0;
  if (BX > 1) {  // horizontal internal bonds (c, c + 1)
    const M h = FULL & ~G::coll();
    B += 2 * popc_m((M)(~(sp ^ (sp >> 1)) & h)) - (BX - 1) * BY;
  }
  if (BY > 1) {  // vertical internal bonds (r, r + 1)
    const M v = (M)(FULL >> BX);
    B += 2 * popc_m((M)(~(sp ^ (sp >> BX)) & v)) - BX * (BY - 1);
  }
  // north row: the ghost row, or (region spanning the height) the last row
  const M nrow = wrapY ? (M)((sp >> ((BY - 1) * BX)) & G::row0()) : gN;
  B += 2 * popc_m((M)(~(sp ^ nrow) & G::row0())) - BX;
  // west column: the ghost column, or (spanning the width) the last column
  const M wcol = wrapX ? (M)((sp >> (BX - 1)) & G::col0()) : gW;
  B += 2 * popc_m((M)(~(sp ^ wcol) & G::col0())) - BY;
  Bi = B;
}

__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7ff0000000000000LL); }

// region row of a shard-local index without an integer division
__device__ __forceinline__ int div_rx(const KArgs& a, int idx) {
  return (int)(((unsigned long long)(unsigned)idx * a.rx_M) >> a.rx_k);
}

// ---------------------------------------------------------------------------
// K1: one relaxation iteration for the regions of the worklist (all regions
// in the window's first iteration), or the commit-time replay that writes
// the compact event log (LOG = true; all regions, latest histories).
//
// Only regions with a changed incoming history are recomputed: a region
// whose inputs did not change would regenerate exactly its previous history
// (the same presimulated random list), so skipping it does not
// change the iteration count g or any result.
//
// Lane-persistent scheduling: each block owns a tile of `tile` consecutive
// work items; a lane whose region reached the window end waits until
// `refill` lanes of its warp are idle, then they publish their regions and
// pull the next ones from the block's shared queue together, so a warp does
// not idle while its slowest region finishes (region histories have
// Poisson-distributed lengths) and the memory-heavy load/publish code runs
// with many lanes at once.  Each round, every active lane performs exactly one
// step -- its next break point or its own event -- and both kinds then share
// the draw of the next pair and the refold/selection/candidate code.
// ---------------------------------------------------------------------------
// Per-lane shared-memory stage of the histories a region reads: up to CI
// entries of each incoming direction and of each of its own latest edge
// histories are copied global -> shared with cp.async when the region is
// loaded (one memory latency per refill batch, many loads in flight).  The
// break-point merge and the diff against the latest own history then read
// shared memory only.
#ifndef ISR_CI
#define ISR_CI 3
#endif
#ifndef ISR_MINB
#define ISR_MINB 6   // resident blocks asked of ptxas for <= 32-site regions (0: ptxas' choice, 96 registers)
#endif
// Launch bounds of K1: 8x8 regions (64-bit site masks) otherwise take 112
// registers and 4 resident blocks; asking for 5 (region_kernel_mb) is 31 %
// faster on the c5 8x8 points.  Smaller regions: 6 blocks (80 registers, no
// spills since the staged positions are packed, 31 KB of shared memory per
// block): +3.8 % on c4 over ptxas' own 96 registers / 5 blocks; 7 blocks (72
// registers) spill and lose 1.5 %.
#ifndef ISR_SPREAD
#define ISR_SPREAD 1  // small worklists spread to one region per 2^k lanes (KArgs.lane_spread = max k)
#endif
#ifndef ISR_NT
#define ISR_NT 128
#endif
constexpr int NT = ISR_NT;   // threads per block of K1
constexpr int kSpreadBlocks = 148 * 6;  // the spread's room: one wave of K1 blocks
constexpr int CI = ISR_CI;   // staged entries per history

// Staged history entries, column si per region in flight: incoming
// histories (and, with OWN, the region's own latest ones for the diff).
template <int NC, bool OWN, int NCI = CI, int NCO = NCI>
struct StageT {
  static constexpr bool HAS_OWN = OWN;
  static constexpr int CIN = NCI;  // staged entries per incoming history
  static constexpr int CIO = NCO;  // ... per own latest history
  static_assert(NCI <= 4 && NCO <= 4, "positions of a history are staged as the bytes of one word");
  double in_t[4][NCI][NC];
  uint32_t in_p[4][NC];        // positions of the staged entries of direction d, entry q in byte q
  double own_t[4][OWN ? NCO : 1][OWN ? NC : 1];
  uint32_t own_p[4][OWN ? NC : 1];
};
#ifndef ISR_CO
#define ISR_CO ISR_CI  // staged own latest entries per edge
#endif
using Stage = StageT<NT, true, CI, ISR_CO>;

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_all;\n" ::: "memory");
}

template <class G>
struct Lane {
  using M = typename G::M;
  int idx;
  uint32_t gid;    // global region id (Philox key, tie order)
  unsigned obase;  // (r * K) * RX + c: own-edge history offset without the edge term
  M spins, gN, gS, gW, gE;
  double ts, R, V, lam, tc;
  int site;       // atom of the next event on the current state (selected at the last refold)
  uint32_t n;
  unsigned long long dig;
  // incoming history cursors: cnt | idx << 8 | pos << 16 | source << 24
  // (source 0/1 = slot, 2/3 = ghost row above/below; bit 28 = staged in smem)
  unsigned hm[4];
  double ht[4];
  unsigned hoff[4];  // element offset of entry 0 of each incoming history
  // own edges: new count | latest count << 8 | latest slot << 16 |
  // diverged << 17 | latest staged in smem << 18
  unsigned om[4];
  int whalf;      // selector word to overwrite on change
  unsigned n_ev;  // events of this region (log offset)
  int Mi, Bi;     // FLAG_OBSERVABLES: magnetisation and owned bond sum now
  double iM, iB;  // ... their integrals since t_c
  double tpv;     // ... up to this time
  unsigned bev;   // own boundary events of this region
};

// element offset of entry 0 of the history that direction d reads, within
// its edge array (edge d ^ 1 of the neighbour; < 2^32, checked at allocation)
__device__ __forceinline__ unsigned in_off(const KArgs& a, int r, int c, int d, unsigned src) {
  if (src >= 2) return (unsigned)c;
  const int nr = d == EDGE_N ? wdec(r, a.RYl) : d == EDGE_S ? winc(r, a.RYl) : r;
  const int nc = d == EDGE_W ? wdec(c, a.RX) : d == EDGE_E ? winc(c, a.RX) : c;
  return ((unsigned)nr * (unsigned)a.K) * (unsigned)a.RX + (unsigned)nc;
}

// base of edge e's array in slot `src` (0/1), or of a ghost row (2 = above, 3 = below)
// (the two slots are one allocation: slot s of edge e starts s * sstride + e * tstride elements in)
__device__ __forceinline__ double* slot_t(const KArgs& a, unsigned s, int e) {
  return a.ed[0].t + ((long long)s * a.sstride + (long long)e * a.tstride);
}
__device__ __forceinline__ uint8_t* slot_p(const KArgs& a, unsigned s, int e) {
  return a.ed[0].pos + ((long long)s * a.sstride + (long long)e * a.tstride);
}
__device__ __forceinline__ const double* src_t(const KArgs& a, unsigned src, int e) {
  return src < 2 ? slot_t(a, src, e) : src == 2 ? a.gh_up.t : a.gh_down.t;
}
__device__ __forceinline__ const uint8_t* src_p(const KArgs& a, unsigned src, int e) {
  return src < 2 ? slot_p(a, src, e) : src == 2 ? a.gh_up.pos : a.gh_down.pos;
}

// advance the integrals of M and B to time t (before a step at t)
template <class G>
__device__ __forceinline__ void obs_advance(Lane<G>& L, double t) {
  const double dt = __dsub_rn(t, L.tpv);
  L.iM = __dadd_rn(L.iM, __dmul_rn((double)L.Mi, dt));
  L.iB = __dadd_rn(L.iB, __dmul_rn((double)L.Bi, dt));
  L.tpv = t;
}

// FULL = false: stop after the state and histories are in; the caller draws
// the pair and refolds (sharing that code with the step)
// FIRST: the window's first iteration (canonical assumption): no
// incoming histories to read or stage.  The own selector pair is still read:
// the new word must flip the slot bit of every changed edge relative to the
// other word (pack_kernel's change test for the strip exchange).
template <class G, bool LOG, class SG, bool FULL = true, bool OBS = false, bool FIRST = false, bool PLAIN = false,
          bool DESC = false>
__device__ __forceinline__ void lane_load(const KArgs& a, Lane<G>& L, int idx, SG& S, const ProdTable<G>& PT,
                                          int si, uint4 dsc = make_uint4(0u, 0u, 0u, 0u)) {
  using M = typename G::M;
  const bool wrapX = !PLAIN && a.RX == 1, wrapY = !PLAIN && a.RYg == 1;
  const unsigned K = stamp_of(a), K0 = a.it_K0;
  const int lane = si;
  const int r = div_rx(a, idx), c = idx - r * a.RX;
  L.idx = idx;
  L.gid = (uint32_t)((a.row0 + r) * a.RX + c);
  L.obase = (unsigned)(((long long)r * a.K) * a.RX + c);
  L.n_ev = 0;
  L.bev = 0;
  // selector words first: they gate the history loads (DESC: resolved by describe_kernel)
  ulonglong2 wp_own = make_ulonglong2(0ull, 0ull);
  if (!LOG && !DESC) wp_own = reinterpret_cast<const ulonglong2*>(a.sel)[idx];
  unsigned cnt[4], src[4];
#pragma unroll
  for (int d = 0; d < 4; ++d) {
    cnt[d] = 0;
    src[d] = 0;
    if (DESC) {
      cnt[d] = (dsc.y >> (8 * d)) & 0xFFu;
      src[d] = (dsc.w >> (2 * d)) & 3u;
      continue;
    }
    const bool axis_off = (d < 2) ? wrapY : wrapX;
    if (FIRST || a.first || axis_off) continue;
    const bool ghost = a.ghost && ((d == EDGE_N && r == 0) || (d == EDGE_S && r == a.RYl - 1));
    if (ghost) {
      cnt[d] = (d == EDGE_N ? a.gh_up : a.gh_down).cnt[c];
      src[d] = d == EDGE_N ? 2u : 3u;
    } else {
      const int nr = d == EDGE_N ? wdec(r, a.RYl) : d == EDGE_S ? winc(r, a.RYl) : r;
      const int nc = d == EDGE_W ? wdec(c, a.RX) : d == EDGE_E ? winc(c, a.RX) : c;
      const ulonglong2 wp = __ldcg(reinterpret_cast<const ulonglong2*>(a.sel) + ((long long)nr * a.RX + nc));
      const unsigned long long v = latest_word(wp, K);
      if (word_valid(v, K0)) {
        cnt[d] = word_count(v, d ^ 1);
        src[d] = (unsigned)word_slot(v, d ^ 1);
      }
    }
  }
  // own latest histories: slot and count per edge
  unsigned long long vown = 0ull;
  L.whalf = 0;
  if (DESC) {  // the same fields, from the descriptor
#pragma unroll
    for (int e = 0; e < 4; ++e)
      vown |= ((unsigned long long)((dsc.w >> (8 + e)) & 1u) << e) |
              ((unsigned long long)((dsc.z >> (8 * e)) & 0xFFu) << (4 + CNT_BITS * e));
    L.whalf = (int)((dsc.w >> 12) & 1u);
  } else if (!LOG) {
    const int li = latest_index(wp_own, K);
    const unsigned long long v = li ? wp_own.y : wp_own.x;
    vown = word_valid(v, K0) ? v : (v & 0xFull);  // outside the window: slots only, counts 0
    L.whalf = li ^ 1;                             // overwrite the older word
  }
  // committed state (the old tau_m becomes tau_0)
  L.spins = (M)((const typename G::ST*)a.in.spins)[idx];
  expand_halo<G>((unsigned long long)((const typename G::HT*)a.in.halo)[idx], L.gN, L.gS, L.gW, L.gE);
  L.ts = (!PLAIN && a.fresh_w) ? a.t_c : a.in.ts[idx];  // fresh_w: every region starts afresh at t_c
  L.R = a.in.R[idx];
  L.n = a.in.n[idx];
  L.dig = a.digest ? a.in.dig[idx] : 0ull;
  if (OBS && !LOG) {  // integrals over [t_c, t_w) start at the window start
    obs_counts<G>(L.spins, L.gN, L.gW, wrapX, wrapY, L.Mi, L.Bi);
    L.iM = 0.0;
    L.iB = 0.0;
    L.tpv = a.t_c;
  }
  // stage incoming histories (above CI entries: read lazily from global): the
  // times global -> shared with cp.async, the position bytes loaded as they are
  // and packed into one word per history after the wait
  bool staged_any = false;
  unsigned ipos[4], opos[4];
#pragma unroll
  for (int d = 0; d < 4; ++d) {
    L.ht[d] = dinf();
    L.hoff[d] = 0;
    ipos[d] = 0;
    unsigned flags = 0;
    if (cnt[d] > 0) {
      const unsigned off = in_off(a, r, c, d, src[d]);
      L.hoff[d] = off;
      const double* T = src_t(a, src[d], G::arr(d ^ 1));
      const uint8_t* P = src_p(a, src[d], G::arr(d ^ 1));
      if (cnt[d] <= (unsigned)SG::CIN) {
        flags = 1u << 28;
        staged_any = true;
#pragma unroll
        for (int q = 0; q < SG::CIN; ++q) {
          if (q < (int)cnt[d]) {
            const unsigned o = off + (unsigned)q * (unsigned)a.RX;
            ISR_ASSERT(src[d] >= 2 ? (int)(o / (unsigned)a.RX) < a.K : (long long)o < a.tstride);
            cp_async8(&S.in_t[d][q][lane], T + o);
            ipos[d] |= (unsigned)P[o] << (8 * q);
          }
        }
      } else {
        L.ht[d] = T[off];
        flags |= (unsigned)P[off] << 16;
      }
    }
    L.hm[d] = cnt[d] | (src[d] << 24) | flags;
  }
  // stage own latest histories for the diff
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    if (G::SE && e > 0) {  // the same history as edge 0's
      L.om[e] = L.om[0];
      continue;
    }
    const unsigned pc = word_count(vown, e), ps = (unsigned)word_slot(vown, e);
    unsigned st = 0;
    opos[e] = 0;
    if (SG::HAS_OWN && !LOG && pc > 0 && pc <= (unsigned)SG::CIO) {
      st = 1;
      staged_any = true;
      const double* Et = src_t(a, ps, e);
      const uint8_t* Ep = src_p(a, ps, e);
#pragma unroll
      for (int q = 0; q < SG::CIO; ++q) {
        if (q < (int)pc) {
          const unsigned o = L.obase + (unsigned)q * (unsigned)a.RX;
          cp_async8(&S.own_t[e][q][lane], Et + o);
          opos[e] |= (unsigned)Ep[o] << (8 * q);
        }
      }
    }
    L.om[e] = (pc << 8) | (ps << 16) | (st << 18);
  }
  if (staged_any) {
    cp_async_wait_all();
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      if (!(L.hm[d] & (1u << 28))) continue;
      S.in_p[d][lane] = ipos[d];
      L.hm[d] |= (ipos[d] & 0xFFu) << 16;
      L.ht[d] = S.in_t[d][0][lane];
    }
    if (SG::HAS_OWN) {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if ((L.om[e] >> 18) & 1u) S.own_p[e][lane] = opos[e];
    }
  }
  if (!FULL) return;
  // pair n: U already spent into R (carried), V selects the next atom
  double U;
  draw_pair(a.seed, L.gid, L.n, U, L.V, a.gen);
  if (a.fresh_w) L.R = budget(a, U);  // the slate is wiped at t_c: the budget restarts from pair n
  Classes<G> C;
  C.build(L.spins, L.gN, L.gS, L.gW, L.gE, wrapX, wrapY);
  L.site = fold_select<G>(C, PT, a.rate, L.V, L.lam);
  L.tc = cand_time(L.ts, L.R, L.lam);
}

// queue region i for the iteration with stamp `stamp` (bitmap of its parity)
__device__ __forceinline__ void mark_dirty(const KArgs& a, int i, unsigned stamp) {
  ISR_ASSERT(i >= 0 && (i >> 5) < a.dwords);
  atomicOr(a.dirty + (size_t)(stamp & 1u) * (size_t)a.dwords + (i >> 5), 1u << (i & 31));
}

// neighbour id in direction d (only needed to order exactly equal times)
__device__ __forceinline__ uint32_t neighbour_id(const KArgs& a, uint32_t gid, int d) {
  const int c = (int)(gid % (uint32_t)a.RX);
  const int gr = (int)(gid / (uint32_t)a.RX);
  return d == EDGE_N ? (uint32_t)(((gr - 1 + a.RYg) % a.RYg) * a.RX + c)
       : d == EDGE_S ? (uint32_t)(((gr + 1) % a.RYg) * a.RX + c)
       : d == EDGE_W ? (uint32_t)(gr * a.RX + wdec(c, a.RX))
                     : (uint32_t)(gr * a.RX + winc(c, a.RX));
}

// publish: selector word of the changed edges (the entry-by-entry diff was
// taken while writing, hist_put), dirty bits of the neighbours across them,
// and the tentative end-of-window state
template <class G, bool OBS = false, bool PLAIN = false>
__device__ __forceinline__ void lane_finish(const KArgs& a, Lane<G>& L, bool& changed, bool& overflow) {
  const int idx = L.idx;
  const int r = div_rx(a, idx), c = idx - r * a.RX;
  const unsigned K = stamp_of(a);
  unsigned chmask = 0;
  unsigned long long word = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const unsigned oc = L.om[e] & 0xFFu, pc = (L.om[e] >> 8) & 0xFFu, ps = (L.om[e] >> 16) & 1u;
    if ((int)oc > a.K) overflow = true;
    const bool diff = ((L.om[e] >> 17) & 1u) || oc != pc;
    const unsigned slot = diff ? ps ^ 1u : ps;
    const unsigned cnt = diff ? ((int)oc < a.K ? oc : (unsigned)a.K) : pc;
    chmask |= (diff ? 1u : 0u) << e;
    word |= ((unsigned long long)slot << e) | ((unsigned long long)cnt << (4 + CNT_BITS * e));
  }
  if (chmask) {
    changed = true;
    a.sel[2 * (long long)idx + L.whalf] = ((unsigned long long)K << 32) | word;
    // neighbours across changed edges must be recomputed next iteration
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (!((chmask >> e) & 1u)) continue;
      if (a.ghost && ((e == EDGE_N && r == 0) || (e == EDGE_S && r == a.RYl - 1))) continue;  // another strip's
      const int nr = e == EDGE_N ? wdec(r, a.RYl) : e == EDGE_S ? winc(r, a.RYl) : r;
      const int nc = e == EDGE_W ? wdec(c, a.RX) : e == EDGE_E ? winc(c, a.RX) : c;
      mark_dirty(a, nr * a.RX + nc, K + 1);
    }
  }
  if (OBS) {  // integrals up to the window end
    obs_advance<G>(L, a.t_w);
    a.out.oM[idx] = L.iM;
    a.out.oB[idx] = L.iB;
  }
  // tentative end-of-window state (committed by pointer swap at commit)
  ((typename G::ST*)a.out.spins)[idx] = (typename G::ST)L.spins;
  ((typename G::HT*)a.out.halo)[idx] = (typename G::HT)compress_halo<G>(L.gN, L.gS, L.gW, L.gE);
  a.out.ts[idx] = L.ts;
  a.out.R[idx] = L.R;
  a.out.n[idx] = L.n;
  if (a.digest) a.out.dig[idx] = L.dig;
}


// ---------------------------------------------------------------------------
// One step of a region: the earliest of its next break point and its own
// event.  Both kinds share the refold/candidate code (refold), so lanes on
// different kinds of step share those instructions.  An incoming head whose
// history is exhausted reads as +inf.
// ---------------------------------------------------------------------------
// minimum of two times (never NaN): a compare and a select, where fmin also
// handles NaN operands (~8 instructions for doubles)
__device__ __forceinline__ double tmin(double x, double y) { return x < y ? x : y; }

template <class G>
__device__ __forceinline__ int next_bp2(const KArgs& a, const Lane<G>& L, double& tb) {
  const double m01 = tmin(L.ht[0], L.ht[1]), m23 = tmin(L.ht[2], L.ht[3]);
  tb = tmin(m01, m23);
  if (!(tb <= L.tc) || tb == dinf()) return -1;
  const int neq = (L.ht[0] == tb) + (L.ht[1] == tb) + (L.ht[2] == tb) + (L.ht[3] == tb);
  const int dstar = L.ht[0] == tb ? 0 : L.ht[1] == tb ? 1 : L.ht[2] == tb ? 2 : 3;
  if (tb < L.tc && neq == 1) return dstar;
  // rare: equal times, resolve by region id (R10)
  uint32_t nb = 0xffffffffu;
  int dm = -1;
#pragma unroll
  for (int d = 0; d < 4; ++d) {
    if (L.ht[d] == tb) {
      const uint32_t nid = neighbour_id(a, L.gid, d);
      if (nid < nb) {
        dm = d;
        nb = nid;
      }
    }
  }
  return (tb < L.tc || nb < L.gid) ? dm : -1;
}

// break point at tb from direction dstar, up to (not including) the refold
template <class G, class SG>
__device__ __forceinline__ void bp_pre2(const KArgs& a, Lane<G>& L, SG& S, int si, int dstar, double tb) {
  constexpr int BX = G::BX, BY = G::BY;
  using M = typename G::M;
  const int lane = si;
  const double Rn = __dsub_rn(L.R, __dmul_rn(L.lam, __dsub_rn(tb, L.ts)));
  L.R = Rn < 0.0 ? 0.0 : Rn;
  L.ts = tb;
  const unsigned hmd = dstar == 0 ? L.hm[0] : dstar == 1 ? L.hm[1] : dstar == 2 ? L.hm[2] : L.hm[3];
  const int p = (int)((hmd >> 16) & 0xFFu);
  L.gN ^= dstar == EDGE_N ? (M)(G::ONE << p) : (M)0;
  L.gS ^= dstar == EDGE_S ? (M)(G::ONE << ((BY - 1) * BX + p)) : (M)0;
  L.gW ^= dstar == EDGE_W ? (M)(G::ONE << (p * BX)) : (M)0;
  L.gE ^= dstar == EDGE_E ? (M)(G::ONE << (p * BX + BX - 1)) : (M)0;
  const unsigned nx = ((hmd >> 8) & 0xFFu) + 1;
  double tn = dinf();
  unsigned pos = 0;
  if (nx < (hmd & 0xFFu)) {
    if (hmd & (1u << 28)) {
      tn = S.in_t[dstar][nx][lane];
      pos = (S.in_p[dstar][lane] >> (8 * nx)) & 0xFFu;
    } else {
      const unsigned src = (hmd >> 24) & 3u;
      const unsigned hoff = dstar == 0 ? L.hoff[0] : dstar == 1 ? L.hoff[1] : dstar == 2 ? L.hoff[2] : L.hoff[3];
      const unsigned off = hoff + nx * (unsigned)a.RX;
      tn = src_t(a, src, G::arr(dstar ^ 1))[off];
      pos = src_p(a, src, G::arr(dstar ^ 1))[off];
    }
  }
  const unsigned hn = (hmd & 0xFF0000FFu) | (nx << 8) | (pos << 16);
#pragma unroll
  for (int d = 0; d < 4; ++d) {
    L.hm[d] = d == dstar ? hn : L.hm[d];
    L.ht[d] = d == dstar ? tn : L.ht[d];
  }
}

// one own-history entry on edge e (EDGE_*), diffed against the latest one
template <class SG>
__device__ __forceinline__ unsigned hist_put(const KArgs& a, unsigned om, int e, unsigned obase, double tc, uint8_t p,
                                             const SG& S, int si, unsigned& n_out, bool& overflow) {
  const int lane = si;
  const unsigned k = om & 0xFFu, pc = (om >> 8) & 0xFFu;
  const unsigned ps = (om >> 16) & 1u;
  unsigned dv = (om >> 17) & 1u;
  if ((int)k < a.K) {
    const unsigned o = obase + k * (unsigned)a.RX;
    ISR_ASSERT((long long)o < a.tstride);
    double* Tn = slot_t(a, ps ^ 1u, e);  // the other slot
    uint8_t* Pn = slot_p(a, ps ^ 1u, e);
    Tn[o] = tc;
    Pn[o] = p;
    ++n_out;
    if (!dv) {
      if (k >= pc) {
        dv = 1;
      } else if (SG::HAS_OWN && ((om >> 18) & 1u)) {
        const unsigned pw = (S.own_p[e][lane] >> (8 * k)) & 0xFFu;
        dv = (__double_as_longlong(S.own_t[e][k][lane]) != __double_as_longlong(tc) || pw != p)
                 ? 1u : 0u;
      } else {
        const double* To = slot_t(a, ps, e);
        const uint8_t* Po = slot_p(a, ps, e);
        dv = (__double_as_longlong(To[o]) != __double_as_longlong(tc) || Po[o] != p) ? 1u : 0u;
      }
    }
  } else {
    overflow = true;
  }
  return (om & ~((1u << 17) | 0xFFu)) | (dv << 17) | (k < 255u ? k + 1 : 255u);
}

// own event at tc, up to (not including) the refold; draws the next pair
// DRAW = false: leave drawing the next pair to the caller (shared code)
template <class G, bool LOG, class SG, bool DRAW = true, bool PLAIN = false>
__device__ __forceinline__ void ev_pre2(const KArgs& a, Lane<G>& L, SG& S, const ProdTable<G>& PT, int si,
                                        unsigned& n_out, bool& overflow) {
  constexpr int BX = G::BX, BY = G::BY;
  const bool wrapX = !PLAIN && a.RX == 1, wrapY = !PLAIN && a.RYg == 1;
  const int site = L.site;
  L.spins ^= G::ONE << site;
  const int sr = site / BX, sc = site - sr * BX;
  if (a.digest) L.dig = digest_step(L.dig, L.tc, site);
  if (LOG) {
    const unsigned long long o = a.log_off[L.idx] + L.n_ev;
    ISR_ASSERT(a.log_cap == 0 || (long long)o < a.log_cap);
    a.log_t[o] = L.tc;
    a.log_region[o] = L.gid;
    a.log_site[o] = (uint16_t)site;
    if (a.log_dm) a.log_dm[o] = ((L.spins >> site) & 1) ? 2 : -2;
  } else if (a.ev_t && (int)L.n_ev < a.evC) {  // scratch event log of this recomputation
    const long long o = (long long)L.n_ev * a.ev_stride + L.idx;
    a.ev_t[o] = L.tc;
    a.ev_s[o] = (uint16_t)(site | (((unsigned)(L.spins >> site) & 1u) << 15));  // bit 15: the new spin
  }
  if (LOG) {
  } else if (BX > 1 && BY > 1) {
    // a site lies on at most one vertical (N/S) and one horizontal (W/E) edge
    const bool onV = !wrapY && (sr == 0 || sr == BY - 1);
    const bool onH = !wrapX && (sc == 0 || sc == BX - 1);
    if (onV) {
      const bool n = sr == 0;
      const unsigned om = hist_put(a, n ? L.om[EDGE_N] : L.om[EDGE_S], n ? EDGE_N : EDGE_S, L.obase, L.tc,
                                   (uint8_t)sc, S, si, n_out, overflow);
      L.om[EDGE_N] = n ? om : L.om[EDGE_N];
      L.om[EDGE_S] = n ? L.om[EDGE_S] : om;
    }
    if (onH) {
      const bool w = sc == 0;
      const unsigned om = hist_put(a, w ? L.om[EDGE_W] : L.om[EDGE_E], w ? EDGE_W : EDGE_E, L.obase, L.tc,
                                   (uint8_t)sr, S, si, n_out, overflow);
      L.om[EDGE_W] = w ? om : L.om[EDGE_W];
      L.om[EDGE_E] = w ? L.om[EDGE_E] : om;
    }
    L.bev += (onV || onH) ? 1u : 0u;
  } else if (G::SE) {  // 1x1: one stored history for the four edges
    L.om[0] = hist_put(a, L.om[0], 0, L.obase, L.tc, (uint8_t)0, S, si, n_out, overflow);
    L.om[1] = L.om[0];
    L.om[2] = L.om[0];
    L.om[3] = L.om[0];
    L.bev += 1u;
  } else {
    bool on_edge = false;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const bool on = e == EDGE_N ? (!wrapY && sr == 0)
                    : e == EDGE_S ? (!wrapY && sr == BY - 1)
                    : e == EDGE_W ? (!wrapX && sc == 0)
                                  : (!wrapX && sc == BX - 1);
      if (!on) continue;
      on_edge = true;
      L.om[e] = hist_put(a, L.om[e], e, L.obase, L.tc, (uint8_t)(e < 2 ? sc : sr), S, si, n_out, overflow);
    }
    L.bev += on_edge ? 1u : 0u;
  }
  ++L.n_ev;
  L.ts = L.tc;
  ++L.n;
  if (!DRAW) return;
  double U;
  draw_pair(a.seed, L.gid, L.n, U, L.V, a.gen);
  L.R = budget(a, U);
}

template <class G, bool PLAIN = false>
__device__ __forceinline__ void refold(const KArgs& a, Lane<G>& L, const ProdTable<G>& PT) {
  Classes<G> C;
  C.build(L.spins, L.gN, L.gS, L.gW, L.gE, !PLAIN && a.RX == 1, !PLAIN && a.RYg == 1);
  L.site = fold_select<G>(C, PT, a.rate, L.V, L.lam);
  L.tc = cand_time(L.ts, L.R, L.lam);
}

// Lane-persistent scheduling over a static tile of the worklist per block.
// n_work_dev (pipelined launch): the worklist length is read on the device;
// the grid was sized for an upper bound, and the tile grows if the bound was
// short.
// PLAIN: no region spanning a lattice axis, no fresh-window restart (the
// common case, chosen at launch; strip ghost rows come with the descriptors)
template <int BX, int BY, bool LOG, bool OBS, bool FIRST, bool PLAIN = false>
__device__ __forceinline__ void region_body(const KArgs& a) {
  using G = Geo<BX, BY>;
  __shared__ unsigned q_next;
  // the first iteration stages nothing (no incoming histories, no latest own
  // history in this window): a minimal stage frees shared memory for more
  // resident blocks
  using SG = typename std::conditional<FIRST, StageT<NT, false, 1>, Stage>::type;
  __shared__ SG S;
  __shared__ ProdTable<G> PT;
  // the block's tile (block-uniform, kept in shared memory)
  __shared__ int s_tile_begin, s_tile_n, s_spread;
  if (threadIdx.x == 0) {
    int tile = a.tile, n = a.n_work;
    if (a.n_work_dev) {  // the host's tile rule (tile_for) on the actual length, >= n / grid
      n = (int)__ldcg(a.n_work_dev);
      const int per = max(1, min(8, n / (NT * 148 * 4)));
      const int need = (n + (int)gridDim.x - 1) / (int)gridDim.x;
      tile = max(NT * per, (need + NT - 1) / NT * NT);
    }
    // a small worklist (late iterations: a handful of regions, each a serial chain of steps) is
    // spread to one region per 2^k lanes, the largest k <= 5 the launched grid (at most one wave)
    // covers, so a region's chain does not wait on the divergent steps of other regions in its warp
    int k = 0;
#if ISR_SPREAD
    const long long room = (long long)min((int)gridDim.x, kSpreadBlocks) * NT;
    while (k < a.lane_spread && ((long long)n << (k + 1)) <= room) ++k;
    if (k > 0) tile = NT >> k;
#endif
    s_spread = k;
    s_tile_begin = blockIdx.x * tile;
    s_tile_n = min(tile, n - (int)(blockIdx.x * tile));
    q_next = blockDim.x;  // the first blockDim items are taken statically
  }
  __syncthreads();
  if (s_tile_n <= 0) return;  // block-uniform: a grid sized for a longer worklist
  ktime_begin(a);
  fill_prod<G>(PT, a.rate);
  __syncthreads();

  unsigned n_ev = 0, n_out = 0, n_in = 0, n_cmp = 0, n_bev = 0, n_reg = 0;
  bool changed = false, overflow = false;
  Lane<G> L;
  // Refill in batches: lanes whose region reached the window end wait until
  // at least REFILL lanes of the warp are idle, then publish and reload
  // together, so the (memory-heavy) load/publish path runs converged.
  const int REFILL = a.refill;
  bool active = false, pending = false, exhausted = false, fresh = false;
  int item = (int)threadIdx.x;
  if (s_spread > 0)  // one region per 2^k lanes: the other lanes find the tile exhausted
    item = (threadIdx.x & ((1u << s_spread) - 1u)) ? s_tile_n : (int)(threadIdx.x >> s_spread);
  for (;;) {
    const unsigned idle = __ballot_sync(0xffffffffu, !active);
    if (__popc(idle) >= REFILL || idle == 0xffffffffu) {
      if (!active) {
        if (pending) {
          if (!LOG) lane_finish<G, OBS, PLAIN>(a, L, changed, overflow);
          n_ev += L.n_ev;
          n_bev = max(n_bev, L.bev);
          pending = false;
        }
        if (!exhausted) {
          if (item < 0) item = (int)atomicAdd(&q_next, 1u);
          if (item < s_tile_n) {
            constexpr bool DESC = PLAIN && !FIRST && !LOG && !OBS;  // (the host passes a.desc for these)
            uint4 dsc = make_uint4(0u, 0u, 0u, 0u);
            if (DESC) dsc = __ldcs(a.desc + s_tile_begin + item);
            const int idx = DESC ? (int)dsc.x : a.wl_in ? (int)a.wl_in[s_tile_begin + item] : s_tile_begin + item;
            ISR_ASSERT(idx >= 0 && idx < a.RX * a.RYl);
            lane_load<G, LOG, SG, false, OBS, FIRST, PLAIN, DESC>(a, L, idx, S, PT, threadIdx.x, dsc);
            fresh = true;
            n_in += (L.hm[0] & 0xFFu) + (L.hm[1] & 0xFFu) + (L.hm[2] & 0xFFu) + (L.hm[3] & 0xFFu);
            n_cmp += ((L.om[0] >> 8) & 0xFFu) + ((L.om[1] >> 8) & 0xFFu) + ((L.om[2] >> 8) & 0xFFu) +
                     ((L.om[3] >> 8) & 0xFFu);  // latest own entries read for the diff
            ++n_reg;
            active = pending = true;
          } else {
            exhausted = true;
          }
          item = -1;
        }
      }
      if (__all_sync(0xffffffffu, exhausted && !active)) break;
    }
    if (active) {
      // one step per round: the earliest of (next break point, own event);
      // a region loaded in this round only draws its pair and refolds
      bool go = true, ev = false;
      if (!fresh) {
        double tb = 0.0;
        const int d = FIRST ? -1 : next_bp2<G>(a, L, tb);  // no break points in the first iteration
        if (d < 0 && !(L.tc < a.t_w)) {
          active = false;
          go = false;
        } else if (d >= 0) {
          if (OBS && !LOG) obs_advance<G>(L, tb);
          bp_pre2<G>(a, L, S, threadIdx.x, d, tb);
        } else {
          if (OBS && !LOG) obs_advance<G>(L, L.tc);
          ev_pre2<G, LOG, SG, false, PLAIN>(a, L, S, PT, threadIdx.x, n_out, overflow);
          ev = true;
        }
      }
      if (go) {
        if (OBS && !LOG && !fresh)  // M and B after the step
          obs_counts<G>(L.spins, L.gN, L.gW, a.RX == 1, a.RYg == 1, L.Mi, L.Bi);
        {  // pair n: V picks the next atom, E(U) its budget.  Drawn by every lane in one
           // straight-line block with the refold (the Philox/E(U) and fold chains interleave); after a
           // break point pair n is the pair already in use (the same V), so only an event (or a fresh_w
           // load, whose budget restarts at t_c) takes its budget
          double U;
          draw_pair(a.seed, L.gid, L.n, U, L.V, a.gen);
          const double Eu = budget(a, U);
          if (ev || (fresh && !PLAIN && a.fresh_w)) L.R = Eu;
        }
        refold<G, PLAIN>(a, L, PT);  // shared by both kinds of step
        // finished now: the candidate lies beyond the window and no break point is left (every incoming
        // entry lies inside the window, so one left would come first) -- the decision the next round's
        // next_bp2 would take, without spending that round
        if (!(L.tc < a.t_w) && L.ht[0] == dinf() && L.ht[1] == dinf() && L.ht[2] == dinf() && L.ht[3] == dinf())
          active = false;
      }
      fresh = false;
    }
  }

  ktime_end(a);
  if (!LOG) {
    if (a.delay_ns) k1_delay(a.delay_ns);
    // warp-aggregated flags and counters (one atomic per warp)
    const unsigned full = 0xffffffffu;
    const unsigned anych = __ballot_sync(full, changed);
    const unsigned anyov = __ballot_sync(full, overflow);
    unsigned long long v0 = n_ev, v1 = n_out, v2 = n_in, v3 = n_cmp, v5 = n_reg;
    unsigned fmax = n_bev;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      v0 += __shfl_xor_sync(full, v0, o);
      v1 += __shfl_xor_sync(full, v1, o);
      v2 += __shfl_xor_sync(full, v2, o);
      v3 += __shfl_xor_sync(full, v3, o);
      v5 += __shfl_xor_sync(full, v5, o);
      fmax = max(fmax, __shfl_xor_sync(full, fmax, o));
    }
    if ((threadIdx.x & 31) == 0) {
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

#if ISR_MINB > 0
#define ISR_K1_BOUNDS __launch_bounds__(NT, ISR_MINB)
#else
#define ISR_K1_BOUNDS __launch_bounds__(NT)
#endif
template <int BX, int BY, bool LOG, bool OBS = false, bool FIRST = false, bool PLAIN = false>
__global__ void ISR_K1_BOUNDS region_kernel(const KArgs a) {
  region_body<BX, BY, LOG, OBS, FIRST, PLAIN>(a);
}
#ifndef ISR_MB_MINB
#define ISR_MB_MINB 5
#endif
template <int BX, int BY, bool LOG, bool OBS = false, bool FIRST = false, bool PLAIN = false>
__global__ void __launch_bounds__(NT, ISR_MB_MINB) region_kernel_mb(const KArgs a) {
  region_body<BX, BY, LOG, OBS, FIRST, PLAIN>(a);
}
// the window's first iteration (≤ 32-site regions): no staging, so shared
// memory no longer caps the resident blocks; ISR_FIRST_MINB asks ptxas for
// that many (0: its own choice; 8 = 64 registers spills)
#ifndef ISR_FIRST_MINB
#define ISR_FIRST_MINB 7  // 72 registers, 7 blocks: +0.7 % on c4 over 6 blocks (80 registers)
#endif
#if ISR_FIRST_MINB > 0
#define ISR_FIRST_BOUNDS __launch_bounds__(NT, ISR_FIRST_MINB)
#else
#define ISR_FIRST_BOUNDS __launch_bounds__(NT)
#endif
template <int BX, int BY, bool OBS = false, bool PLAIN = false>
__global__ void ISR_FIRST_BOUNDS region_kernel_first(const KArgs a) {
  region_body<BX, BY, false, OBS, true, PLAIN>(a);
}

// ---------------------------------------------------------------------------
// K4 (world > 1): pack the latest north-edge histories of the strip's first
// region row and south-edge histories of its last row into the send rows,
// with the stamp of their last change (the neighbour marks its adjacent
// regions dirty when the stamp equals the current iteration).
// ---------------------------------------------------------------------------
// the latest history of column c's strip-edge region (up: first row, north
// edge; else: last row, south edge) into ghost-row view g at column c
__device__ __forceinline__ void pack_col(const KArgs& a, bool up, int c, const GhostView& g) {
  const int r = up ? 0 : a.RYl - 1;
  const int e = up ? EDGE_N : EDGE_S;
  const ulonglong2 wp = reinterpret_cast<const ulonglong2*>(a.sel)[(long long)r * a.RX + c];
  // latest as of the end of this iteration
  const unsigned K = stamp_of(a);
  const unsigned long long v = latest_word(wp, K + 1);
  int cnt = 0;
  if (word_valid(v, a.it_K0)) {
    const EdgeView& E = word_slot(v, e) ? a.ed[1] : a.ed[0];
    cnt = (int)word_count(v, e);
    const long long base = (long long)(a.single_edge ? 0 : e) * a.tstride + ((long long)r * a.K) * a.RX + c;
    for (int q = 0; q < cnt; ++q) {
      g.t[(long long)q * a.RX + c] = E.t[base + (long long)q * a.RX];
      g.pos[(long long)q * a.RX + c] = E.pos[base + (long long)q * a.RX];
    }
  }
  g.cnt[c] = (uint16_t)cnt;
  // changed in this iteration: the word was rewritten now and edge e moved
  // slot relative to the previous latest word (the other one)
  const unsigned long long other = latest_index(wp, K + 1) ? wp.x : wp.y;
  const bool ch_now = (unsigned)(v >> 32) == K && (((v ^ other) >> e) & 1ull);
  g.stamp[c] = ch_now ? K : 0u;
}

__global__ void pack_kernel(const KArgs a, GhostView send_up, GhostView send_down) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 2 * a.RX) return;
  const bool up = i < a.RX;
  pack_col(a, up, up ? i : i - a.RX, up ? send_up : send_down);
}

// after the exchange: regions next to a ghost row that changed in this
// iteration are recomputed in the next one
__global__ void mark_kernel(const KArgs a, GhostView up, GhostView down) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 2 * a.RX) return;
  const bool isup = i < a.RX;
  const int c = isup ? i : i - a.RX;
  const GhostView& g = isup ? up : down;
  const unsigned K = stamp_of(a);
  if (g.stamp[c] != K) return;
  const int r = isup ? 0 : a.RYl - 1;
  const int nidx = r * a.RX + c;
  mark_dirty(a, nidx, K + 1);
}

// Ordered worklist of the next iteration from its dirty bitmap: 8
// consecutive 32-bit words (256 regions) per thread, 2048 words per block,
// compacted in region order within each block (one atomic per block); the
// bitmap is cleared for reuse two iterations later.
constexpr int kCompactWords = 8, kCompactThreads = 256;
__global__ void __launch_bounds__(kCompactThreads) compact_kernel(uint32_t* bm, int nwords, int n, uint32_t* wl,
                                                                  unsigned* count) {
  __shared__ unsigned wsum[kCompactThreads / 32];
  __shared__ unsigned base;
  const int w0 = (blockIdx.x * kCompactThreads + threadIdx.x) * kCompactWords;
  uint32_t w[kCompactWords];
  if (w0 + kCompactWords <= nwords) {  // 32-byte aligned: two 16-byte loads
    const uint4 x = reinterpret_cast<const uint4*>(bm + w0)[0], y = reinterpret_cast<const uint4*>(bm + w0)[1];
    w[0] = x.x; w[1] = x.y; w[2] = x.z; w[3] = x.w; w[4] = y.x; w[5] = y.y; w[6] = y.z; w[7] = y.w;
  } else {
#pragma unroll
    for (int q = 0; q < kCompactWords; ++q) w[q] = w0 + q < nwords ? bm[w0 + q] : 0u;
  }
  int c = 0;
#pragma unroll
  for (int q = 0; q < kCompactWords; ++q) c += __popc(w[q]);
  if (c) {
#pragma unroll
    for (int q = 0; q < kCompactWords; ++q)
      if (w[q]) bm[w0 + q] = 0u;
  }
  const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = c;  // inclusive warp scan of the counts
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, x, o);
    if ((int)lane >= o) x += t;
  }
  if (lane == 31) wsum[wid] = (unsigned)x;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned s = 0;
    for (int q = 0; q < kCompactThreads / 32; ++q) {
      const unsigned t = wsum[q];
      wsum[q] = s;
      s += t;
    }
    base = s ? atomicAdd(count, s) : 0u;
  }
  __syncthreads();
  unsigned o = base + wsum[wid] + (unsigned)(x - c);
#pragma unroll
  for (int q = 0; q < kCompactWords; ++q) {
    uint32_t v = w[q];
    while (v) {
      const int b = __ffs(v) - 1;
      v &= v - 1u;
      const int r = (w0 + q) * 32 + b;
      if (r < n) wl[o++] = (uint32_t)r;
    }
  }
}

// The worklist's descriptors for a PLAIN iteration with stamp K (no wrapped
// axis): each item's incoming (slot, count) pairs from the neighbours' latest
// selector words with stamp < K (strip edges: the ghost row's count, source
// 2 = the row above, 3 = below) and its own latest word -- what lane_load
// would read itself, resolved here with whole warps so that a K1 refill
// starts with one coalesced 16-byte read.
__global__ void __launch_bounds__(256) describe_kernel(const KArgs a, unsigned K, const uint32_t* wl,
                                                       const unsigned* count, uint4* desc) {
  const unsigned n = __ldcg(count), K0 = a.it_K0;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int idx = (int)wl[i];
    const int r = div_rx(a, idx), c = idx - r * a.RX;
    const ulonglong2* sel = reinterpret_cast<const ulonglong2*>(a.sel);
    const ulonglong2 wp_own = __ldcg(sel + idx);
    ulonglong2 wn[4];
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      const int nr = d == EDGE_N ? wdec(r, a.RYl) : d == EDGE_S ? winc(r, a.RYl) : r;
      const int nc = d == EDGE_W ? wdec(c, a.RX) : d == EDGE_E ? winc(c, a.RX) : c;
      wn[d] = __ldcg(sel + ((long long)nr * a.RX + nc));
    }
    uint32_t cnt4 = 0, pc4 = 0, bits = 0;
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      if (a.ghost && ((d == EDGE_N && r == 0) || (d == EDGE_S && r == a.RYl - 1))) {
        cnt4 |= (uint32_t)__ldcg((d == EDGE_N ? a.gh_up : a.gh_down).cnt + c) << (8 * d);
        bits |= (d == EDGE_N ? 2u : 3u) << (2 * d);
        continue;
      }
      const unsigned long long v = latest_word(wn[d], K);
      if (word_valid(v, K0)) {
        cnt4 |= word_count(v, d ^ 1) << (8 * d);
        bits |= (unsigned)word_slot(v, d ^ 1) << (2 * d);
      }
    }
    const int li = latest_index(wp_own, K);
    const unsigned long long vv = li ? wp_own.y : wp_own.x;
    const unsigned long long vown = word_valid(vv, K0) ? vv : (vv & 0xFull);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      pc4 |= word_count(vown, e) << (8 * e);
      bits |= (unsigned)word_slot(vown, e) << (8 + e);
    }
    bits |= (unsigned)(li ^ 1) << 12;
    desc[i] = make_uint4((uint32_t)idx, cnt4, pc4, bits);
  }
}

// ---------------------------------------------------------------------------
// K0: pack the strip's spins (+1 halo row above and below, periodic) into
// region bit masks and ghost bits; tau_0 = 0 and R = E(U_0).
// buf: (RYl*BY + 2) rows x Lx, row 0 = lattice row above the strip.
// ---------------------------------------------------------------------------
template <int BX, int BY>
__global__ void init_kernel(const uint8_t* buf, int Lx, int RX, int RYl, int row0, unsigned long long seed,
                            double eq_q, StateView st) {
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
  st.R[idx] = quantize_budget(expvar(U), eq_q);
  st.n[idx] = 0;
  st.dig[idx] = 0ull;
}

// FLAG_OBSERVABLES snapshot: M = sum s and the bond sum B of a committed
// configuration, each region contributing its own sites and the bonds it owns
// (internal, to its north and west neighbours: every bond exactly once; the
// ghost bits are the neighbours' committed spins).  Integers: exact in any order.
template <int BX, int BY>
__global__ void __launch_bounds__(256) snap_kernel(StateView st, int n, int RX, int RYg, unsigned long long* out) {
  using G = Geo<BX, BY>;
  using M = typename G::M;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  long long m = 0, b = 0;
  if (idx < n) {
    M gN, gS, gW, gE;
    expand_halo<G>((unsigned long long)((const typename G::HT*)st.halo)[idx], gN, gS, gW, gE);
    int Mi, Bi;
    obs_counts<G>((M)((const typename G::ST*)st.spins)[idx], gN, gW, RX == 1, RYg == 1, Mi, Bi);
    m = Mi;
    b = Bi;
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
