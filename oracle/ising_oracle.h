/*
 * oracle/ising_oracle.h -- CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load or call anything under oracle/.  The
 * product (paper_cs_0405053_b200/, include/ising_sr.h) shares no code, no
 * header, no table and no constant with this file and never calls it.
 *
 * What it computes: the unique trajectory of the
 * per-region-stream continuous-time n-fold-way Ising dynamics of
 * arXiv cs/0405053 -- region i draws its n-th (U,V) pair from its own
 * counter-based stream, its n-th event time solves
 *      integral_{tau_{n-1}}^{tau} Lambda_i(t) dt = -log U_n   (eq. lambdataua)
 * under the true evolving global state, and the site is chosen by V_n via
 * eqs. Wsum / Wstop / nores / vindex.  Synchronous relaxation
 * reaches exactly this trajectory, so the oracle is
 * the plain definition, computed serially by always processing the
 * globally earliest region event.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math (no FMA contraction:
 * every double operation is one IEEE-754 operation in program order).
 */
#ifndef ISING_ORACLE_H
#define ISING_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Philox4x32-10 (Salmon et al., Random123), standard constants. */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* The n-th (U,V) pair of stream `stream` (SURVEY §8c.3 "Philox", "U, V"):
 * key = (stream, seed_lo), counter = (n_lo, n_hi, 0, seed_hi);
 * U from (x0,x1), V from (x2,x3): a = ((x_hi<<32)|x_lo)>>12,
 * value = ((double)a + 0.5) * 2^-52, in [2^-53, 1-2^-53]. */
void orc_pair(uint64_t seed, uint32_t stream, uint64_t n, double* U, double* V);
/* pair n of generation g (counter word 2 = g): the "fresh" random numbers of
 * the alternate approach to subsequent steps; g = 0 is orc_pair */
void orc_pair_g(uint64_t seed, uint32_t stream, uint64_t n, uint32_t g, double* U, double* V);

/* E(U) = -log U evaluated with IEEE +,-,*,/ only (SURVEY §8c.3 "E(U)"),
 * the exponential variate of eq. nextau. */
double orc_expvar(double U);

/* splitmix64 finalizer (kept for tests; the per-region digest chain is
 * h <- (h ^ tau_bits) * 0x9E3779B97F4A7C15 + site + 1, R27). */
uint64_t orc_mix64(uint64_t z);

typedef struct {
  int32_t  Lx, Ly;         /* periodic lattice, >= 3 each                       */
  int32_t  bx, by;         /* region size; divides Lx, Ly                        */
  double   rate[10];       /* r_k = lambda p_k, class k = 5(s+1)/2 + u          */
  uint64_t seed;
  double   t_end;          /* process events with tau < t_end                    */
  double   t_obs0;         /* time averages accumulate over [t_obs0, t_end)      */
  int32_t  check;          /* 1: verify incremental (B, M, N_k) after every event */
  double   fresh_W;        /* > 0: alternate approach to subsequent steps: at
                              every t_c = fl(w fresh_W), w >= 1, each region discards its
                              pending budget and restarts at t_c with pair (n, generation w) */
  double   eq_quantum;     /* > 0: tie test mode, budgets (floor(E(U) q) + 1) / q (R30) */
} orc_cfg;

typedef struct {
  /* per-region outputs (n_regions entries), may be NULL */
  uint64_t* digest;
  uint64_t* count;
  /* global event log in processing order, may be NULL */
  double*   log_t;
  uint32_t* log_region;
  uint16_t* log_site;      /* local site index = local_row*bx + local_col */
  int64_t   log_cap;
  /* magnetisation M = sum s and bond sum B = sum_bonds s s' sampled at
   * sorted times (state after every event with tau <= t), may be NULL */
  const double* sample_t;
  int32_t   n_samples;
  int64_t*  sample_M;
  int64_t*  sample_B;
  /* results */
  int64_t   n_events;      /* total events processed (tau < t_end)               */
  int64_t   log_n;         /* min(n_events, log_cap)                              */
  double    obs[5];        /* integrals over [t_obs0,t_end): dt, B dt, M dt, |M| dt, M^2 dt */
  int32_t   check_failures;
  int64_t   n_bumps;       /* O1: candidates bumped to nextafter(t_s) (reading #11), for tests */
} orc_out;

/* Per-region-stream DES (O1). spins: Ly*Lx row-major, 1 = up (+1), 0 = down.
 * Returns 0 on success, <0 on invalid input. */
int orc_des_run(const orc_cfg* cfg, const uint8_t* spins0, uint8_t* spins_out, orc_out* out);

/* Single-stream global n-fold way (O2), stream id `stream`:
 * the textbook algorithm with no regions.  Same outputs (digest/count have
 * one entry, region field of the log is 0). */
int orc_bkl_run(const orc_cfg* cfg, uint32_t stream, const uint8_t* spins0,
                uint8_t* spins_out, orc_out* out);

/* single-step forms: cand(t,R,Lambda); break-point budget update
 * max(R - Lambda_old (t_b - t_s), 0); Lambda fold; class/index selection */
double orc_cand(double t, double R, double lam);
double orc_breakpoint_budget(double R, double lam_old, double t_b, double t_s);
double orc_fold(const int32_t* N, const double* rate);
void orc_select(const int32_t* N, const double* rate, double V, double lam, int32_t* kstar,
                int64_t* j);

/* per-region class counts N[region*10 + k] of a configuration */
int orc_class_counts(int32_t Lx, int32_t Ly, int32_t bx, int32_t by, const uint8_t* spins,
                     int32_t* N);

/* Second workload: the discrete-time Metropolis dynamics
 * of §2: a visited atom v flips with probability p(v) = p_k of
 * its class k = 5(s+1)/2 + u (eq. p and the table of; p_k is the
 * rate table with lambda = 1), else stays.  Visiting order: the conventional
 * two-colour (checkerboard) sweep -- first every site with (x + y) even,
 * then every site with (x + y) odd, each colour in row-major order.  (Sites
 * of one colour share no bond, so any order within a colour gives the same
 * result.)  Random numbers (R29): in row y the sites of colour c
 * in increasing x are numbered j = 0, 1, ...; sites 2m and 2m+1 share the
 * Philox4x32-10 draw with key = (0xFFFFFFFE, seed_lo), counter = (q, s_lo,
 * s_hi | c << 31, seed_hi), q = y * ceil(Lx/4) + m, s the global sweep; site
 * 2m takes U from words (x0, x1), site 2m+1 from (x2, x3), mapped as in
 * orc_pair; the site flips iff U < p_k.
 * Lx, Ly even and >= 4 (a bipartite periodic lattice); spins in/out,
 * row-major, nonzero = up on input, 0/1 on output; *flips = accepted flips.
 * Returns 0, or -1 on invalid arguments. */
int orc_cb_run(int32_t Lx, int32_t Ly, const double* p, uint64_t seed, int64_t sweep0, int32_t nsweeps,
               uint8_t* spins, int64_t* flips);

/* batch forms of the scalar functions above (for tests) */
void orc_expvar_n(const double* U, double* E, int64_t n);
void orc_pair_n(uint64_t seed, const uint32_t* stream, const uint64_t* idx, double* U, double* V,
                int64_t n);
void orc_philox_n(const uint32_t* ctr, const uint32_t* key, uint32_t* out, int64_t n);

#ifdef __cplusplus
}
#endif
#endif
