/*
 * include/ising_sr.h -- C ABI of libising_sr.so, the B200 (sm_100a) engine for
 * the synchronous-relaxation parallel n-fold way Ising simulation of
 * Lubachevsky & Weiss, arXiv cs/0405053 ("the paper"; P:n = line n of its
 * text).
 *
 * What the library computes.  The periodic Lx x Ly lattice G is
 * cut into bx x by regions G_i, one per virtual processing element
 * (P:494-500); region id = region_row * (Lx/bx) + region_col.  Simulated time
 * advances in windows [t_c, t_c + W) (committed time and step size T_max,
 * P:320-335, 400-402).  Within a window every region repeatedly regenerates its
 * continuous-time n-fold-way history from its own
 * counter-based random list, integrating its total rate
 * over break points caused by the neighbours' boundary flips of the previous
 * iteration (eqs. lambdataua..newtau); the boundary histories are
 * compared with the previous iteration's and the iteration repeats until no
 * history changes.  The fixed point is the unique
 * trajectory of the per-region-stream dynamics; it is
 * independent of W (except with ISING_SR_FLAG_FRESH_WINDOW) and of the number
 * of shards.
 *
 * Bit-level semantics (Philox layout, E(U), Lambda fold order, selection,
 * candidate bump, tie order) are frozen in DESIGN.md §3; results are
 * bit-reproducible across runs, W and shard counts.
 *
 * Conventions (all entry points):
 *  - every call returns ising_sr_status (0 = OK, < 0 = error) unless noted;
 *  - host buffers are owned by the caller; `init` copies `spins`;
 *  - device state is owned by the library (cudaMalloc on cfg.device);
 *  - one ctx per rank / shard; a ctx is not thread-safe;
 *  - all device work is issued on cfg.stream (a cudaStream_t; NULL = the
 *    library creates its own stream); calls that return host data
 *    synchronize that stream;
 *  - after a CUDA error every later call returns ISING_SR_E_CUDA (sticky).
 */
#ifndef ISING_SR_H
#define ISING_SR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ising_sr_ctx ising_sr_ctx; /* opaque; owned by the library */

typedef enum {
  ISING_SR_OK = 0,
  ISING_SR_E_INVALID_ARG = -1, /* NULL pointer, bad rate/W/t_end, unsupported region shape */
  ISING_SR_E_DIMENSION = -2,   /* Lx or Ly < 3 (neighbours must be distinct) */
  ISING_SR_E_PARTITION = -3,   /* bx, by do not divide Lx, Ly; strips do not divide region rows */
  ISING_SR_E_DIVERGED = -4,    /* max_iterations reached without a fixed point */
  ISING_SR_E_CAPACITY = -5,    /* boundary-history capacity cannot be grown further */
  ISING_SR_E_CUDA = -6,        /* CUDA runtime error (sticky) */
  ISING_SR_E_NCCL = -7,        /* NCCL (or the exchange callback) failed, or NCCL cannot be loaded */
  ISING_SR_E_OOM = -8,         /* device allocation failed */
  ISING_SR_E_STATE = -9        /* call out of order (commit without a converged window, run past t_end) */
} ising_sr_status;

/* cfg.flags */
#define ISING_SR_FLAG_LOG_EVENTS 0x1u /* commit writes the window's compact event log (get_events) */
#define ISING_SR_FLAG_DIGEST 0x2u     /* maintain per-region event digests (get_digests) */
/* The paper's alternate approach to subsequent steps: at every
 * committed time t_c = fl(w W), w >= 1, each region discards its pending
 * budget and restarts at t_c with pair n of random-number generation w
 * (Philox counter word 2 = w).  Unbiased (memorylessness), but the
 * trajectory then depends on W.  Default off (the carried budget of P:726-742). */
#define ISING_SR_FLAG_FRESH_WINDOW 0x4u
/* Time integrals of the magnetisation M = sum_v s(v) and of the bond sum
 * B = sum_<vu> s(v) s(u) (energy E = -J B - H M, eq. hamil) over every
 * committed window, accumulated per region inside K1 (each region owns its
 * internal bonds and the bonds to its north and west neighbours) and reduced
 * in a fixed order at commit (ising_sr_stats.obs_*).  Lane-per-region K1 forms
 * only (E_INVALID_ARG with ISING_SR_BIG=0, the warp form). */
#define ISING_SR_FLAG_OBSERVABLES 0x8u
/* Paper-faithful Jacobi schedule: every relaxation iteration
 * recomputes every region, not only those whose incoming histories changed.
 * Same fixed point, same g, same bits; only slower (the default worklist skips
 * regions that would regenerate their previous trajectory). */
#define ISING_SR_FLAG_JACOBI_ALL 0x10u
/* Halo loopback (world == 1 with nccl_id): the strip's first and last region
 * rows read their wrap-around neighbours' histories from ghost rows filled
 * by the library's NCCL exchange with itself (ncclSend/ncclRecv to rank 0 of
 * a one-rank communicator), exactly as a strip of a multi-GPU run reads its
 * neighbours'.  Same results as without the flag; it exercises the in-library
 * exchange on one GPU. */
#define ISING_SR_FLAG_HALO_LOOPBACK 0x20u
/* Time integrals of |M| and M^2 over every committed window (the model's
 * observable; stats.obs_absM_* / obs_M2_*): the commit sorts the
 * window's events by time on the device (bucket sort + per-bucket insertion
 * sort), prefix-sums dM = +-2 from M(t_c) and reduces |M| dt and M^2 dt in a
 * fixed order.  Implies FLAG_LOG_EVENTS and FLAG_OBSERVABLES; world == 1
 * only (E_INVALID_ARG otherwise: it needs the global time order). */
#define ISING_SR_FLAG_MAG_MOMENTS 0x40u

/* Halo exchange between strips (world > 1).  Rank q owns a band of region
 * rows; "up" is toward region row 0 (rank q-1, periodic), "down" toward rank
 * q+1.  With cfg.nccl_id the library performs the exchange itself on its
 * stream (ncclSend/ncclRecv of the ghost rows + ncclAllReduce(max) of the
 * flags).  Otherwise, after each relaxation iteration
 * the library calls the exchange callback with device pointers into the
 * current iteration's boundary-history buffers; the callee must
 *   (a) copy my send_up chunks into rank (q-1)'s recv_from_down chunks and my
 *       send_down chunks into rank (q+1)'s recv_from_up chunks (periodic in
 *       q; with world == 2 both go to the other rank), chunk k being
 *       chunk_bytes[k] long, and
 *   (b) replace flags[0..1] (device int32 {changed, overflow}) by their
 *       maximum over all ranks (the "UNTIL all PEs detect no difference" of
 *       P:427-429).
 * send_up = my first region row's north-edge histories, send_down = my last
 * row's south-edge histories, each in 4 chunks (all four must be moved):
 *   chunk 0: u16 count[RX]     entries of each region's edge history
 *   chunk 1: u32 stamp[RX]     global iteration of the edge's last change (the
 *                              receiver marks its adjacent region dirty when
 *                              stamp == the current iteration)
 *   chunk 2: f64 t[K][RX]      entry times (entry q of column c at q*RX + c)
 *   chunk 3: u8  pos[K][RX]    entry positions along the edge
 * The chunks of one row are contiguous in that order (each start 256-byte
 * aligned), so one copy of row_bytes from send_up[0] moves a whole row.
 * Work may be enqueued on `stream` (the ctx stream) and must be ordered on it
 * on return (NCCL: issue it on that stream).  Return 0 on success (anything
 * else -> ISING_SR_E_NCCL). */
typedef struct {
  int32_t nchunks;          /* 4: count (u16), stamp (u32), times (f64), positions (u8) */
  void* send_up[4];
  void* send_down[4];
  void* recv_from_up[4];    /* ghost row above my strip: up neighbour's south edges */
  void* recv_from_down[4];  /* ghost row below my strip: down neighbour's north edges */
  size_t chunk_bytes[4];
  int32_t* flags;           /* device int32[2]: {changed, overflow}; all-reduce(max) */
  void* stream;             /* cudaStream_t of the ctx */
  size_t row_bytes;         /* bytes from send_up[0] through the end of send_up[3] (one contiguous row) */
} ising_sr_halo;

typedef int (*ising_sr_exchange_fn)(void* user, const ising_sr_halo* halo);

typedef struct {
  int32_t Lx, Ly;           /* lattice, periodic both ways; >= 3                 */
  int32_t bx, by;           /* region size; divides Lx, Ly; supported: 1x1, 2x2, 4x4, 8x8,   *
                             * 4x2, 2x4, 8x4, 4x8 (lane form), 16x16, 32x32, 16x32, 32x16,   *
                             * 16x8, 8x16 (big-region form); else E_INVALID_ARG             */
  double J, H, T;           /* recorded for observables; the dynamics use `rate` only        */
  double rate[10];          /* r_k = lambda p_k, class k = 5(s+1)/2 + u          */
  double W;                 /* window length = the paper's T_max, > 0; <= 0:     *
                             * the paper's rule W = ln N / (lambda |dG_i|), N = Lx Ly/(bx by)*
                             * regions, |dG_i| = 2bx + 2by - 4 boundary sites (bx by if a   *
                             * side is 1), lambda = max_k rate[k]                           */
  double t_end;             /* simulate events with tau < t_end                              */
  uint64_t seed;            /* Philox key/counter seed                         */
  int32_t max_iterations;   /* relaxation iterations per window before E_DIVERGED; 0 = 1000  */
  int32_t hist_capacity;    /* initial boundary-history slots per region edge; 0 = auto      */
  uint32_t flags;           /* ISING_SR_FLAG_*                                               */
  int32_t rank, world;      /* this ctx owns region rows [rank*RY/world, (rank+1)*RY/world)  */
  int32_t device;           /* CUDA ordinal                                                  */
  void* stream;             /* cudaStream_t; NULL = library-owned stream                     */
  ising_sr_exchange_fn exchange; /* world > 1: used by run_window (step API: unused)       */
  void* exchange_user;
  /* Optional device allocator for every device buffer of the ctx (e.g. torch's
   * caching allocator).  dev_alloc(bytes, user) returns a device pointer or
   * NULL (-> E_OOM); dev_free(ptr, user) releases it.  Allocations are used on
   * `stream` only, so a stream-ordered allocator needs no extra
   * synchronisation.  Both NULL = cudaMalloc / cudaFree. */
  void* (*dev_alloc)(size_t bytes, void* user);
  void (*dev_free)(void* ptr, void* user);
  void* alloc_user;
  /* world > 1 (or FLAG_HALO_LOOPBACK): the 128-byte ncclUniqueId shared by
   * all ranks (rank 0 gets one from ising_sr_nccl_unique_id and broadcasts
   * it, e.g. with torch.distributed); the library creates its communicator
   * (ncclCommInitRank(world, id, rank)) and runs the exchange on `stream`:
   * by default one fused kernel per iteration that stores the strip-edge
   * histories straight into the neighbours' ghost rows in an NCCL symmetric
   * window (NCCL >= 2.28 device API, all ranks in one NVLink team)
   * and combines the flags through an inbox + LSA barrier; env
   * ISING_SR_EXCHANGE=sendrecv uses ncclSend/ncclRecv + ncclAllReduce instead
   * (=peer: the fused kernel or E_NCCL; unset: send/recv also where the
   * device API, one NVLink team or the symmetric window is unavailable, with
   * a note on stderr).  init, capacity growth and destroy
   * are then collective over the ranks.  With the fused kernel the step-level
   * halo_get returns E_STATE (there are no host-visible send rows).
   * NULL: the exchange callback (or the step-level API) moves the ghost rows.
   * Copied at init. */
  const void* nccl_id;
  /* > 0 (a power of two): test mode forcing exact time ties -- every budget
   * E(U) is replaced by (floor(E(U) q) + 1) / q (R30); 0 = off */
  double eq_quantum;
  /* FLAG_LOG_EVENTS: events per region per window kept by K1 for the commit
   * compaction (a region with more is replayed at commit); 0 = auto */
  int32_t log_capacity;
} ising_sr_config;

typedef struct {
  double t_c;               /* committed time                                                */
  int64_t windows;          /* committed windows                                             */
  int64_t events_total;     /* committed events (this rank)                                  */
  int64_t events_last_window;
  int32_t g_last, g_max;    /* relaxation iterations of the last window / max    */
  int64_t g_hist[64];       /* histogram of g over committed windows (g >= 63 -> bin 63)     */
  int32_t f_last, f_max;    /* max own-boundary events of a region in an iteration */
  int64_t iterations_total; /* relaxation iterations run (all windows, incl. retries)        */
  int32_t overflow_retries; /* windows restarted after history-capacity overflow             */
  int32_t hist_capacity;    /* current slots per region edge                                 */
  int64_t recomputations_total; /* region trajectories computed (sum over iterations)        */
  double bytes_alg_last_window; /* algorithmic HBM bytes of the last window   */
  double ms_last_window;    /* device time of run_window + commit of the last window          */
  /* cumulative instrumentation of the region-trajectory kernel (all windows):
   * launches, device time (CUDA events on the ctx stream around each launch)
   * and algorithmic bytes */
  int64_t region_launches;
  double region_ms;
  double region_bytes;
  /* FLAG_OBSERVABLES: integrals over the last committed window and over all
   * committed windows (this rank's regions): int M dt, int B dt, and the time */
  double obs_M_last, obs_B_last, obs_M_total, obs_B_total, obs_time_total;
  /* regions recomputed in relaxation iteration k+1 of the last committed
   * window (the worklist length; bin 63 collects iterations >= 64) */
  int64_t active_last[64];
  /* host wall time (ms, all windows) inside the world > 1 exchange callback
   * (halo exchange + flag all-reduce) and inside ising_sr_commit */
  double ms_exchange_total, ms_commit_total;
  /* FLAG_OBSERVABLES: M = sum s and the bond sum B (E = -J B - H M) of the
   * configuration at the committed time t_c (this rank's regions, each owning
   * its internal bonds and those to its north and west neighbours), exact */
  int64_t obs_M_now, obs_B_now;
  /* FLAG_LOG_EVENTS: boundary-history entries of the last committed window's
   * fixed point (h of SURVEY §8(d.3): each event counted once per region edge
   * its site lies on), and its regions replayed at commit because their event
   * count exceeded log_capacity; -1 without the flag */
  int64_t edge_entries_last_window;
  int64_t log_replayed_last_window;
  /* device time (ms, all windows) of the commit's compaction kernels */
  double ms_compact_total;
  /* FLAG_MAG_MOMENTS: int |M| dt and int M^2 dt over the last committed
   * window and over all committed windows */
  double obs_absM_last, obs_M2_last, obs_absM_total, obs_M2_total;
} ising_sr_stats;

/* Validate cfg, allocate device state, copy the full Ly*Lx row-major spin
 * configuration (nonzero = up, 0 = down; caller-owned, copied) and set
 * committed time 0.  Each rank passes the whole lattice and keeps
 * its strip; only its rows (+1 halo row each side) are read, by host-to-device
 * copies straight from `spins` (full DMA speed when it is page-locked).
 * spins == NULL: the iid +-1 (p = 1/2) configuration of the Philox init
 * stream is generated on the device (Philox4x32-10 with key
 * (0xFFFFFFFF, seed_lo), counter (v >> 7, 0, 1, seed_hi); site v is up iff
 * bit (v & 31) of output word ((v >> 5) & 3) is set).  With nccl_id this
 * call is collective (every rank must call it). */
ising_sr_status ising_sr_init(const ising_sr_config* cfg, const uint8_t* spins, ising_sr_ctx** out);

/* A fresh 128-byte ncclUniqueId into `out` (for cfg.nccl_id; rank 0 calls it
 * and broadcasts the bytes).  E_NCCL if NCCL cannot be loaded. */
ising_sr_status ising_sr_nccl_unique_id(void* out);

/* Relax the window [t_c, min(t_c + W, t_end)) to the fixed point.
 * Deterministic and idempotent until commit.  *g_out = iterations run,
 * including the final no-change iteration.  E_DIVERGED leaves the committed
 * state untouched.  E_STATE if t_c >= t_end. */
ising_sr_status ising_sr_run_window(ising_sr_ctx* ctx, int32_t* g_out);

/* Commit the converged window: committed state <- fixed point, t_c += W
 * (P:430).  *events_out = events committed in the window on this rank.
 * E_STATE without a converged run_window. */
ising_sr_status ising_sr_commit(ising_sr_ctx* ctx, int64_t* events_out);

/* Convenience: run_window + commit until t_c >= t_end. */
ising_sr_status ising_sr_run(ising_sr_ctx* ctx, int64_t* events_out);

ising_sr_status ising_sr_stats_get(const ising_sr_ctx* ctx, ising_sr_stats* out);

/* Own strip's committed spins, (Ly/world) x Lx row-major, 1 = up, into the
 * caller's buffer (page-locked memory gives a full-speed copy). */
ising_sr_status ising_sr_get_spins(ising_sr_ctx* ctx, uint8_t* out);

/* Last committed window's event log (requires FLAG_LOG_EVENTS), ordered by
 * region id then time: time, global region id, local site (row*bx + col).
 * Built at commit by compacting the events K1 recorded in its final
 * recomputation of each region (K3; regions with more than
 * log_capacity events are replayed).
 * Copies min(cap, n) entries; *n = number of events in the window. */
ising_sr_status ising_sr_get_events(ising_sr_ctx* ctx, double* t, uint32_t* region, uint16_t* site,
                                    int64_t cap, int64_t* n);

/* Per own region (region-id order): digest chain over all committed events,
 * h <- (h ^ tau_bits) * 0x9E3779B97F4A7C15 + site + 1 mod 2^64 (requires
 * FLAG_DIGEST; R27), and the
 * committed event count n.  Either pointer may be NULL. */
ising_sr_status ising_sr_get_digests(ising_sr_ctx* ctx, uint64_t* digest, uint64_t* count);

/* Step-level API used by multi-rank drivers (the loop of run_window, one
 * iteration at a time).  begin_window starts a window; iterate runs one
 * relaxation iteration (the regions whose incoming histories changed; all
 * regions in the window's first iteration) and returns this rank's local
 * {changed, overflow} in flags_out; for world > 1, halo_get then describes
 * the send/receive ghost rows of that iteration (same contract as the
 * exchange callback, flags excluded), and after the caller has moved them
 * exchange_done marks the regions next to changed ghosts for the next
 * iteration.  end_iterations declares the window converged after `g`
 * iterations (the caller's global decision: no rank changed).
 * g == -1 in end_iterations: some rank overflowed its history capacity; the
 * library doubles the capacity (the same on every rank) and the caller
 * restarts the window with begin_window. */
ising_sr_status ising_sr_begin_window(ising_sr_ctx* ctx);
ising_sr_status ising_sr_iterate(ising_sr_ctx* ctx, int32_t flags_out[2]);
ising_sr_status ising_sr_halo_get(ising_sr_ctx* ctx, ising_sr_halo* out);
ising_sr_status ising_sr_exchange_done(ising_sr_ctx* ctx);
ising_sr_status ising_sr_end_iterations(ising_sr_ctx* ctx, int32_t g);

/* Checkpoint / resume at a committed time (the committed state is
 * the whole state of the simulation; the next window starts from the
 * canonical assumption, so no boundary history is saved).  checkpoint_size
 * gives the bytes of this rank's checkpoint; checkpoint_save writes them to a
 * caller-owned host buffer of `cap` bytes (E_INVALID_ARG if too small);
 * checkpoint_load restores a checkpoint into a ctx created with the same
 * configuration (lattice, regions, rates, seed, W, flags, rank/world;
 * E_INVALID_ARG on any mismatch or a corrupted buffer).  Both are allowed
 * only between windows (E_STATE inside one).  A resumed run is bit-identical
 * to the uninterrupted one. */
ising_sr_status ising_sr_checkpoint_size(const ising_sr_ctx* ctx, int64_t* bytes);
ising_sr_status ising_sr_checkpoint_save(ising_sr_ctx* ctx, void* buf, int64_t cap);
ising_sr_status ising_sr_checkpoint_load(ising_sr_ctx* ctx, const void* buf, int64_t len);

/* sizeof of the ABI structs as compiled into the library (binding checks:
 * 0 = ising_sr_config, 1 = ising_sr_stats, 2 = ising_sr_halo; else 0). */
size_t ising_sr_struct_size(int32_t which);

/* Number of kernel launches issued by this ctx so far (instrumentation). */
int64_t ising_sr_launch_count(const ising_sr_ctx* ctx);

void ising_sr_destroy(ising_sr_ctx* ctx); /* NULL-safe */
const char* ising_sr_strerror(ising_sr_status s);

/* ------------------------------------------------------------------------
 * Second workload: checkerboard Metropolis sweeps, the
 * discrete-time dynamics of §2 -- a visited atom flips with
 * probability p_k of its class k = 5(s+1)/2 + u (eq. p; the rate
 * table with lambda = 1), else keeps its spin -- with the two-colour
 * visiting order: a sweep visits every site with (x + y) even, then every
 * site with (x + y) odd.  Random numbers (R29): in row y the
 * sites of colour c are numbered j = 0, 1, ... in increasing x; sites 2m and
 * 2m+1 share the Philox4x32-10 draw with key = (0xFFFFFFFE, seed_lo),
 * counter = (y*ceil(Lx/4) + m, s_lo, s_hi | c << 31, seed_hi), s the global
 * sweep; site 2m takes U = the 52-bit unit of words (x0, x1), site 2m+1 of
 * (x2, x3), as for the event pairs; a site flips iff U < p[k].  A statistical cross-check and conventional baseline for
 * the n-fold way (same equilibrium, a different dynamics).
 *
 * spins: Ly*Lx row-major bytes, 0 = down, 1 = up (any nonzero byte reads as
 * up; every byte of a visited word is rewritten as 0/1).  Lx, Ly even and
 * >= 4 (a bipartite periodic lattice; else E_DIMENSION), Lx*Ly < 2^32;
 * p[k] in [0, 1], nsweeps >= 0, 0 <= sweep0, sweep0 + nsweeps < 2^62
 * (else E_INVALID_ARG).
 * Sweeps sweep0 .. sweep0+nsweeps-1 are run, so a run split at any sweep is
 * bit-identical to the run in one piece.
 * ------------------------------------------------------------------------ */

/* Device-resident lattice: d_spins is a device pointer (caller-owned,
 * updated in place); *d_flips (device, may be NULL) is incremented by the
 * number of accepted flips; the work is enqueued on `stream` (cudaStream_t,
 * NULL = legacy default stream) and not synchronised.  E_CUDA if a launch
 * fails. */
ising_sr_status ising_cb_sweeps(uint8_t* d_spins, int32_t Lx, int32_t Ly, const double p[10], uint64_t seed,
                                int64_t sweep0, int32_t nsweeps, uint64_t* d_flips, void* stream);

/* Host buffers: copies spins_in (host, caller-owned) to `device`, runs the
 * sweeps, copies the lattice back to spins_out (host, caller-owned; may
 * equal spins_in) and stores the accepted flips in *flips_out (may be NULL).
 * Synchronous.  E_OOM / E_CUDA on device failures. */
ising_sr_status ising_cb_run(const uint8_t* spins_in, uint8_t* spins_out, int32_t Lx, int32_t Ly,
                             const double p[10], uint64_t seed, int64_t sweep0, int32_t nsweeps,
                             int64_t* flips_out, int32_t device);

#ifdef __cplusplus
}
#endif
#endif /* ISING_SR_H */
