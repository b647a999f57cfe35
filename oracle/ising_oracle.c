/*
 * oracle/ising_oracle.c -- CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 * (see ising_oracle.h for the contract; only tests/, smoke() and bench.py's
 * CPU-baseline leg may use it.  Shares no code with the CUDA path.)
 *
 * Citations: P:n = line n of the paper text; SURVEY §8c.x are the
 * bit-level readings frozen in DESIGN.md §3 ("Readings of the paper").
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC.
 */
#include "ising_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Random123).  Round:                                        */
/*   (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2                                    */
/*   c' = (hi1^c1^k0, lo1, hi0^c3^k1, lo0); key bumped by (W0,W1) between     */
/*   rounds.  Used as the paper's "presimulated list" of random numbers,      */
/*   P:454-472 ("reuse the (pseudo)random numbers").              */
/* ------------------------------------------------------------------------ */
void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* 52 random bits -> uniform double strictly inside (0,1): ((a + 0.5) * 2^-52).
 * P:251-252 "U_i is the ith independent sample of a random (0,1) uniformly
 * distributed variable" -- never 0 (so -log U is finite) and never 1. */
static double unit_from_words(uint32_t hi, uint32_t lo) {
  uint64_t a = ((((uint64_t)hi) << 32) | (uint64_t)lo) >> 12;
  return ((double)a + 0.5) * 0x1p-52;
}

void orc_pair(uint64_t seed, uint32_t stream, uint64_t n, double* U, double* V) {
  orc_pair_g(seed, stream, n, 0u, U, V);
}

void orc_pair_g(uint64_t seed, uint32_t stream, uint64_t n, uint32_t g, double* U, double* V) {
  uint32_t ctr[4] = {(uint32_t)n, (uint32_t)(n >> 32), g, (uint32_t)(seed >> 32)};
  uint32_t key[2] = {stream, (uint32_t)seed};
  uint32_t x[4];
  orc_philox4x32_10(ctr, key, x);
  *U = unit_from_words(x[0], x[1]);
  *V = unit_from_words(x[2], x[3]);
}

/* ------------------------------------------------------------------------ */
/* E(U) = -log U, the exponential variate of eq. nextau,          */
/* computed with IEEE +,-,*,/ and exact bit operations only:   */
/*   U = m 2^e, m in [1,2); if m > sqrt2: m /= 2, e += 1                      */
/*   f = m-1, s = f/(2+f), z = s^2, P = sum_{j=0..9} z^j/(2j+3) (Horner)      */
/*   log m = 2s + 2s z P   (2 atanh s series),  log U = e ln2 + log m         */
/* ------------------------------------------------------------------------ */
double orc_expvar(double U) {
  uint64_t bits;
  memcpy(&bits, &U, 8);
  int e = (int)((bits >> 52) & 0x7ff) - 1023;
  uint64_t mb = (bits & 0x000fffffffffffffULL) | 0x3ff0000000000000ULL;
  double m;
  memcpy(&m, &mb, 8);
  if (m > 0x1.6a09e667f3bcdp+0) {
    m = m * 0.5;
    e = e + 1;
  }
  double f = m - 1.0;
  double s = f / (2.0 + f);
  double z = s * s;
  double P = 0x1.8618618618618p-5;      /* 1/21 */
  P = P * z + 0x1.af286bca1af28p-5;     /* 1/19 */
  P = P * z + 0x1.e1e1e1e1e1e1ep-5;     /* 1/17 */
  P = P * z + 0x1.1111111111111p-4;     /* 1/15 */
  P = P * z + 0x1.3b13b13b13b14p-4;     /* 1/13 */
  P = P * z + 0x1.745d1745d1746p-4;     /* 1/11 */
  P = P * z + 0x1.c71c71c71c71cp-4;     /* 1/9  */
  P = P * z + 0x1.2492492492492p-3;     /* 1/7  */
  P = P * z + 0x1.999999999999ap-3;     /* 1/5  */
  P = P * z + 0x1.5555555555555p-2;     /* 1/3  */
  double u = s + s;
  double logm = u + u * (z * P);
  double de = (double)e;
  double logU = de * 0x1.62e42feep-1 + (de * 0x1.a39ef35793c76p-33 + logm);
  return -logU;
}

uint64_t orc_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* per-region digest chain (R27): h <- (h ^ tau_bits) * K + site + 1
 * mod 2^64, K = 0x9E3779B97F4A7C15 (odd: a bijection of h) */
static uint64_t digest_step(uint64_t h, double tau, uint32_t site) {
  uint64_t tb;
  memcpy(&tb, &tau, 8);
  return (h ^ tb) * 0x9E3779B97F4A7C15ULL + (uint64_t)site + 1u;
}

/* The budget a region draws from U: E(U), or in the tie test mode
 * (cfg->eq_quantum = q > 0, R30) (floor(E(U) q) + 1) / q -- exact
 * for a power-of-two q -- so that equal event times in different regions
 * are common and the (time, region id) order (reading #10) and the
 * candidate bump (reading #11) are exercised. */
static double budget_of(const orc_cfg* cfg, double U) {
  double E = orc_expvar(U);
  if (cfg->eq_quantum > 0.0) E = (floor(E * cfg->eq_quantum) + 1.0) / cfg->eq_quantum;
  return E;
}

/* ------------------------------------------------------------------------ */
/* Lattice helpers.  Spins stored 1 = up (+1), 0 = down (-1).    */
/* ------------------------------------------------------------------------ */
typedef struct {
  int Lx, Ly;
  uint8_t* s;    /* spins 0/1 */
  uint8_t* cls;  /* class k = 5 s + u  (reading #7) */
} lat_t;

static int site_nb(const lat_t* L, int v, int d) {
  int y = v / L->Lx, x = v % L->Lx;
  switch (d) {
    case 0: y = (y + L->Ly - 1) % L->Ly; break;  /* north (row-1) */
    case 1: y = (y + 1) % L->Ly; break;          /* south (row+1) */
    case 2: x = (x + L->Lx - 1) % L->Lx; break;  /* west  (col-1) */
    default: x = (x + 1) % L->Lx; break;         /* east  (col+1) */
  }
  return y * L->Lx + x;
}

static int site_class(const lat_t* L, int v) {
  int u = 0;
  for (int d = 0; d < 4; ++d) u += L->s[site_nb(L, v, d)];
  return 5 * L->s[v] + u;
}

static int64_t spin_pm(const lat_t* L, int v) { return L->s[v] ? 1 : -1; }

/* M = sum_v s(v); B = sum over bonds (each once: east and south) of s s'
 * (eq. hamil P:160-163 with reading #16). */
static void scratch_MB(const lat_t* L, int64_t* M, int64_t* B) {
  int64_t m = 0, b = 0;
  int n = L->Lx * L->Ly;
  for (int v = 0; v < n; ++v) {
    m += spin_pm(L, v);
    b += spin_pm(L, v) * spin_pm(L, site_nb(L, v, 1));
    b += spin_pm(L, v) * spin_pm(L, site_nb(L, v, 3));
  }
  *M = m;
  *B = b;
}

/* ------------------------------------------------------------------------ */
/* n-fold way quantities.                                        */
/* Lambda fold, eq. biglambda with lambda folded into r_k (reading #14):      */
/*   c_{-1} = 0, c_k = c_{k-1} + N_k r_k, Lambda = c_9   (fixed order 0..9)   */
/* ------------------------------------------------------------------------ */
static double fold_lambda(const int32_t* N, const double* rate) {
  double c = 0.0;
  for (int k = 0; k < 10; ++k) c = c + (double)N[k] * rate[k];
  return c;
}

/* candidate time: eq. nextau / eq. newtau in remaining-budget form,
 * cand(t, R, Lambda) = t + R/Lambda (readings #1, #2, #11); +inf if
 * Lambda = 0; bumped to nextafter(t, +inf) if it rounds onto t. */
/* candidates that rounded onto their start and were bumped (reading #11), per run */
static int64_t n_bumps;

static double cand_time(double t, double R, double lam) {
  if (lam == 0.0) return INFINITY;
  double tau = t + R / lam;
  if (tau == t) {
    tau = nextafter(t, INFINITY);
    n_bumps++;
  }
  return tau;
}

/* Phase 2 (eqs. Wsum/Wstop) in x = V*Lambda space (reading #9):
 * k* = first k with x <= c_k.  Phase 3 (eqs. nores/vindex):
 * j = min(floor((x - c_{k*-1}) / r_{k*}), N_{k*} - 1)   (0-based, reading #8). */
static void select_class_index(const int32_t* N, const double* rate, double V, double lam,
                               int* kstar, int64_t* jidx) {
  double x = V * lam;
  double c = 0.0, cprev = 0.0;
  int ks = -1;
  for (int k = 0; k < 10; ++k) {
    cprev = c;
    c = c + (double)N[k] * rate[k];
    if (x <= c) {
      ks = k;
      break;
    }
  }
  if (ks < 0) { /* unreachable for V < 1 (x <= Lambda = c_9); keep defined */
    ks = 9;
    while (ks > 0 && N[ks] == 0) --ks;
  }
  double q = (x - cprev) / rate[ks];
  int64_t j = (int64_t)floor(q);
  if (j > (int64_t)N[ks] - 1) j = (int64_t)N[ks] - 1;
  if (j < 0) j = 0;
  *kstar = ks;
  *jidx = j;
}

/* ------------------------------------------------------------------------ */
/* Indexed binary min-heap of regions keyed by (tau_c, region id),          */
/* lexicographic (reading #10).                                              */
/* ------------------------------------------------------------------------ */
typedef struct {
  int32_t n;
  int32_t* h;    /* heap slots -> region */
  int32_t* pos;  /* region -> slot */
  const double* key;
} heap_t;

static int heap_less(const heap_t* H, int32_t a, int32_t b) {
  double ka = H->key[a], kb = H->key[b];
  return ka < kb || (ka == kb && a < b);
}

static void heap_swap(heap_t* H, int i, int j) {
  int32_t a = H->h[i], b = H->h[j];
  H->h[i] = b; H->h[j] = a;
  H->pos[b] = i; H->pos[a] = j;
}

static void heap_up(heap_t* H, int i) {
  while (i > 0) {
    int p = (i - 1) / 2;
    if (heap_less(H, H->h[i], H->h[p])) { heap_swap(H, i, p); i = p; }
    else break;
  }
}

static void heap_down(heap_t* H, int i) {
  for (;;) {
    int l = 2 * i + 1, r = l + 1, m = i;
    if (l < H->n && heap_less(H, H->h[l], H->h[m])) m = l;
    if (r < H->n && heap_less(H, H->h[r], H->h[m])) m = r;
    if (m == i) break;
    heap_swap(H, i, m);
    i = m;
  }
}

static void heap_fix(heap_t* H, int32_t region) {
  int i = H->pos[region];
  heap_up(H, i);
  heap_down(H, H->pos[region]);
}

/* ------------------------------------------------------------------------ */
/* Observables: samples at fixed times and time integrals.                   */
/* ------------------------------------------------------------------------ */
typedef struct {
  int64_t M, B;
  double t_last;  /* time up to which integrals have been accumulated */
  int32_t next_sample;
} obs_t;

static void obs_advance(obs_t* O, const orc_cfg* cfg, orc_out* out, double t_next) {
  /* samples strictly before t_next see the current state (state after all
   * events with tau <= t_sample) */
  if (out->sample_t) {
    while (O->next_sample < out->n_samples && out->sample_t[O->next_sample] < t_next) {
      if (out->sample_M) out->sample_M[O->next_sample] = O->M;
      if (out->sample_B) out->sample_B[O->next_sample] = O->B;
      O->next_sample++;
    }
  }
  double a = O->t_last > cfg->t_obs0 ? O->t_last : cfg->t_obs0;
  double b = t_next < cfg->t_end ? t_next : cfg->t_end;
  if (b > a) {
    double dt = b - a;
    double M = (double)O->M, B = (double)O->B;
    out->obs[0] += dt;
    out->obs[1] += dt * B;
    out->obs[2] += dt * M;
    out->obs[3] += dt * fabs(M);
    out->obs[4] += dt * M * M;
  }
  if (t_next > O->t_last) O->t_last = t_next;
}

/* Flip site v: spin, classes of v and its 4 neighbours, per-region class
 * counts, and the integer (M, B) invariant (O(1) class update). */
static void flip_site(lat_t* L, int v, int32_t* Ncnt, const int32_t* region_of, obs_t* O) {
  int nb[4];
  for (int d = 0; d < 4; ++d) nb[d] = site_nb(L, v, d);
  int64_t sn = L->s[v] ? -1 : 1; /* new spin */
  int64_t nbsum = 0;
  for (int d = 0; d < 4; ++d) nbsum += spin_pm(L, nb[d]);
  O->M += 2 * sn;
  O->B += 2 * sn * nbsum;
  L->s[v] ^= 1;
  /* v's class and neighbours' classes */
  int touched[5] = {v, nb[0], nb[1], nb[2], nb[3]};
  for (int t = 0; t < 5; ++t) {
    int w = touched[t];
    int dup = 0;
    for (int q = 0; q < t; ++q) dup |= (touched[q] == w);
    if (dup) continue;
    int oldk = L->cls[w], newk = site_class(L, w);
    if (oldk != newk) {
      int32_t* N = Ncnt + (size_t)region_of[w] * 10;
      N[oldk]--;
      N[newk]++;
      L->cls[w] = (uint8_t)newk;
    }
  }
}

static int validate(const orc_cfg* c) {
  if (c->Lx < 3 || c->Ly < 3) return -2;
  if (c->bx < 1 || c->by < 1 || c->Lx % c->bx || c->Ly % c->by) return -3;
  return 0;
}

static void record_event(orc_out* out, int64_t idx, double tau, uint32_t region, uint32_t site) {
  if (out->log_t && idx < out->log_cap) {
    out->log_t[idx] = tau;
    if (out->log_region) out->log_region[idx] = region;
    if (out->log_site) out->log_site[idx] = (uint16_t)site;
  }
}

/* ------------------------------------------------------------------------ */
/* O1: per-region-stream DES.                                 */
/*  regions G_i, region id = region_row*(Lx/bx)+region_col;      */
/*  each region's n-th event uses pair(i, n);  */
/*  a flip of a neighbour in another region is a break point for that region */
/*  (P:617-674): R <- max(R - Lambda_old (tau - t_s), 0), t_s <- tau, refold. */
/* ------------------------------------------------------------------------ */
int orc_des_run(const orc_cfg* cfg, const uint8_t* spins0, uint8_t* spins_out, orc_out* out) {
  int rc = validate(cfg);
  if (rc) return rc;
  const int Lx = cfg->Lx, Ly = cfg->Ly, bx = cfg->bx, by = cfg->by;
  const int RX = Lx / bx, RY = Ly / by;
  const int64_t NS = (int64_t)Lx * Ly;
  const int32_t NR = RX * RY;

  lat_t L = {Lx, Ly, (uint8_t*)malloc(NS), (uint8_t*)malloc(NS)};
  int32_t* region_of = (int32_t*)malloc(sizeof(int32_t) * NS);
  int32_t* Ncnt = (int32_t*)calloc((size_t)NR * 10, sizeof(int32_t));
  double* ts = (double*)malloc(sizeof(double) * NR);
  double* Rb = (double*)malloc(sizeof(double) * NR);
  double* lam = (double*)malloc(sizeof(double) * NR);
  double* Vv = (double*)malloc(sizeof(double) * NR);
  double* tc = (double*)malloc(sizeof(double) * NR);
  uint64_t* nev = (uint64_t*)calloc(NR, sizeof(uint64_t));
  uint64_t* dig = (uint64_t*)calloc(NR, sizeof(uint64_t));
  heap_t H = {NR, (int32_t*)malloc(sizeof(int32_t) * NR), (int32_t*)malloc(sizeof(int32_t) * NR), tc};
  if (!L.s || !L.cls || !region_of || !Ncnt || !ts || !Rb || !lam || !Vv || !tc || !nev || !dig || !H.h || !H.pos) {
    rc = -8;
    goto done;
  }
  for (int64_t v = 0; v < NS; ++v) L.s[v] = spins0[v] ? 1 : 0;
  for (int64_t v = 0; v < NS; ++v) {
    int y = (int)(v / Lx), x = (int)(v % Lx);
    region_of[v] = (y / by) * RX + (x / bx);
  }
  for (int64_t v = 0; v < NS; ++v) {
    L.cls[v] = (uint8_t)site_class(&L, (int)v);
    Ncnt[(size_t)region_of[v] * 10 + L.cls[v]]++;
  }
  obs_t O = {0, 0, 0.0, 0};
  scratch_MB(&L, &O.M, &O.B);
  out->n_events = 0;
  out->log_n = 0;
  out->check_failures = 0;
  n_bumps = 0;
  for (int q = 0; q < 5; ++q) out->obs[q] = 0.0;

  /* initial state of every region: tau_0 = 0 */
  for (int32_t r = 0; r < NR; ++r) {
    double U, V;
    orc_pair(cfg->seed, (uint32_t)r, 0, &U, &V);
    Rb[r] = budget_of(cfg, U);
    Vv[r] = V;
    ts[r] = 0.0;
    lam[r] = fold_lambda(Ncnt + (size_t)r * 10, cfg->rate);
    tc[r] = cand_time(0.0, Rb[r], lam[r]);
  }
  for (int32_t i = 0; i < NR; ++i) { H.h[i] = i; H.pos[i] = i; }
  for (int i = NR / 2 - 1; i >= 0; --i) heap_down(&H, i);

  /* alternate approach to subsequent steps: generation of the
   * random numbers in use and the next committed time at which every region
   * starts afresh */
  uint32_t gen = 0;
  int64_t w_next = 1;
  double t_next = cfg->fresh_W > 0.0 ? (double)w_next * cfg->fresh_W : INFINITY;

  for (;;) {
    int32_t r = H.h[0];
    double tau = tc[r];
    if (t_next < cfg->t_end && !(tau < t_next)) {
      /* wipe the slate at t_c = t_next: pending budgets are discarded, each
       * region draws pair n of generation w (taken later than any so far) */
      gen = (uint32_t)w_next;
      for (int32_t q = 0; q < NR; ++q) {
        double U, V;
        orc_pair_g(cfg->seed, (uint32_t)q, nev[q], gen, &U, &V);
        Rb[q] = budget_of(cfg, U);
        Vv[q] = V;
        ts[q] = t_next;
        tc[q] = cand_time(t_next, Rb[q], lam[q]);
      }
      for (int i = NR / 2 - 1; i >= 0; --i) heap_down(&H, i);
      w_next++;
      t_next = (double)w_next * cfg->fresh_W;
      continue;
    }
    if (!(tau < cfg->t_end)) break;
    obs_advance(&O, cfg, out, tau);

    /* select the atom (Phases 1-3) */
    int32_t* N = Ncnt + (size_t)r * 10;
    int kstar;
    int64_t j;
    select_class_index(N, cfg->rate, Vv[r], lam[r], &kstar, &j);
    int ry = r / RX, rx = r % RX;
    int v = -1;
    uint32_t local = 0;
    int64_t seen = 0;
    for (int ly = 0; ly < by && v < 0; ++ly)
      for (int lx = 0; lx < bx; ++lx) {
        int g = (ry * by + ly) * Lx + (rx * bx + lx);
        if (L.cls[g] == kstar) {
          if (seen == j) { v = g; local = (uint32_t)(ly * bx + lx); break; }
          seen++;
        }
      }
    if (v < 0) { rc = -10; goto done; } /* class count / class array disagree */

    /* apply the flip */
    flip_site(&L, v, Ncnt, region_of, &O);
    record_event(out, out->n_events, tau, (uint32_t)r, local);
    out->n_events++;
    dig[r] = digest_step(dig[r], tau, local);
    nev[r]++;

    /* renew region r: next pair of its list */
    {
      double U, V;
      orc_pair_g(cfg->seed, (uint32_t)r, nev[r], gen, &U, &V);
      Rb[r] = budget_of(cfg, U);
      Vv[r] = V;
      ts[r] = tau;
      lam[r] = fold_lambda(N, cfg->rate);
      tc[r] = cand_time(tau, Rb[r], lam[r]);
      heap_fix(&H, r);
    }

    /* break points in the other regions adjacent to v */
    int32_t done_q[4];
    int nd = 0;
    for (int d = 0; d < 4; ++d) {
      int32_t q = region_of[site_nb(&L, v, d)];
      if (q == r) continue;
      int dup = 0;
      for (int t = 0; t < nd; ++t) dup |= (done_q[t] == q);
      if (dup) continue;
      done_q[nd++] = q;
      double Rq = Rb[q] - lam[q] * (tau - ts[q]);
      if (Rq < 0.0) Rq = 0.0;
      Rb[q] = Rq;
      ts[q] = tau;
      lam[q] = fold_lambda(Ncnt + (size_t)q * 10, cfg->rate);
      tc[q] = cand_time(tau, Rb[q], lam[q]);
      heap_fix(&H, q);
    }

    if (cfg->check) {
      int64_t M2, B2;
      scratch_MB(&L, &M2, &B2);
      if (M2 != O.M || B2 != O.B) out->check_failures++;
      int32_t* chk = (int32_t*)calloc((size_t)NR * 10, sizeof(int32_t));
      for (int64_t w = 0; w < NS; ++w) {
        int k = site_class(&L, (int)w);
        if (k != L.cls[w]) out->check_failures++;
        chk[(size_t)region_of[w] * 10 + k]++;
      }
      if (memcmp(chk, Ncnt, sizeof(int32_t) * (size_t)NR * 10)) out->check_failures++;
      free(chk);
    }
  }
  obs_advance(&O, cfg, out, cfg->t_end);
  if (out->sample_t) { /* samples at/after t_end see the final state */
    while (O.next_sample < out->n_samples) {
      if (out->sample_M) out->sample_M[O.next_sample] = O.M;
      if (out->sample_B) out->sample_B[O.next_sample] = O.B;
      O.next_sample++;
    }
  }
  out->log_n = out->n_events < out->log_cap ? out->n_events : out->log_cap;
  out->n_bumps = n_bumps;
  if (spins_out) memcpy(spins_out, L.s, NS);
  if (out->digest) memcpy(out->digest, dig, sizeof(uint64_t) * NR);
  if (out->count) memcpy(out->count, nev, sizeof(uint64_t) * NR);
  rc = 0;
done:
  free(L.s); free(L.cls); free(region_of); free(Ncnt); free(ts); free(Rb); free(lam);
  free(Vv); free(tc); free(nev); free(dig); free(H.h); free(H.pos);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* O2: textbook single-stream n-fold way over the whole lattice             */
/* (P:191-309): Lambda from global class counts (eq. biglambda), next time  */
/* tau_i = tau_{i-1} + (-log U_i)/Lambda(tau_{i-1}) (eq. nextau) with the   */
/* same rounding-onto-itself bump, atom chosen by V_i (eqs. Wsum..vindex)    */
/* scanning the whole lattice in row-major order.  Written independently of  */
/* O1: no heap, no regions, no break points.                                 */
/* ------------------------------------------------------------------------ */
int orc_bkl_run(const orc_cfg* cfg, uint32_t stream, const uint8_t* spins0,
                uint8_t* spins_out, orc_out* out) {
  if (cfg->Lx < 3 || cfg->Ly < 3) return -2;
  const int Lx = cfg->Lx, Ly = cfg->Ly;
  const int NS = Lx * Ly;
  lat_t L = {Lx, Ly, (uint8_t*)malloc(NS), (uint8_t*)malloc(NS)};
  int32_t* zero_region = (int32_t*)calloc(NS, sizeof(int32_t));
  int32_t N[10] = {0};
  if (!L.s || !L.cls || !zero_region) {
    free(L.s); free(L.cls); free(zero_region);
    return -8;
  }
  for (int v = 0; v < NS; ++v) L.s[v] = spins0[v] ? 1 : 0;
  for (int v = 0; v < NS; ++v) { L.cls[v] = (uint8_t)site_class(&L, v); N[L.cls[v]]++; }
  obs_t O = {0, 0, 0.0, 0};
  scratch_MB(&L, &O.M, &O.B);
  out->n_events = 0;
  out->check_failures = 0;
  for (int q = 0; q < 5; ++q) out->obs[q] = 0.0;
  uint64_t h = 0;
  double t = 0.0; /* tau_0 = 0 */
  for (uint64_t i = 0;; ++i) {
    double U, V;
    orc_pair(cfg->seed, stream, i, &U, &V);
    /* W(k) partial sums times Lambda: cum[k] = sum_{j<=k} N_j r_j, in order */
    double cum[10];
    double acc = 0.0;
    for (int k = 0; k < 10; ++k) {
      acc = acc + (double)N[k] * cfg->rate[k];
      cum[k] = acc;
    }
    double lam = cum[9];
    double tau = cand_time(t, budget_of(cfg, U), lam);
    if (!(tau < cfg->t_end)) break;
    obs_advance(&O, cfg, out, tau);
    /* W(k-1) < V <= W(k)  <=>  cum[k-1] < V*Lambda <= cum[k] */
    double x = V * lam;
    int kstar = 0;
    while (kstar < 9 && !(x <= cum[kstar])) kstar++;
    double below = kstar > 0 ? cum[kstar - 1] : 0.0;
    int64_t j = (int64_t)floor((x - below) / cfg->rate[kstar]);
    if (j >= N[kstar]) j = N[kstar] - 1;
    int v = -1;
    int64_t seen = 0;
    for (int g = 0; g < NS; ++g)
      if (L.cls[g] == kstar) {
        if (seen == j) { v = g; break; }
        seen++;
      }
    if (v < 0) break;
    flip_site(&L, v, N, zero_region, &O);
    record_event(out, out->n_events, tau, 0u, (uint32_t)v);
    out->n_events++;
    h = digest_step(h, tau, (uint32_t)v);
    t = tau;
  }
  obs_advance(&O, cfg, out, cfg->t_end);
  if (out->sample_t)
    while (O.next_sample < out->n_samples) {
      if (out->sample_M) out->sample_M[O.next_sample] = O.M;
      if (out->sample_B) out->sample_B[O.next_sample] = O.B;
      O.next_sample++;
    }
  out->log_n = out->n_events < out->log_cap ? out->n_events : out->log_cap;
  if (spins_out) memcpy(spins_out, L.s, NS);
  if (out->digest) out->digest[0] = h;
  if (out->count) out->count[0] = (uint64_t)out->n_events;
  free(L.s); free(L.cls); free(zero_region);
  return 0;
}

/* batch helpers for the tests (loops over the scalar definitions above) */
void orc_expvar_n(const double* U, double* E, int64_t n) {
  for (int64_t i = 0; i < n; ++i) E[i] = orc_expvar(U[i]);
}

void orc_pair_n(uint64_t seed, const uint32_t* stream, const uint64_t* idx, double* U, double* V,
                int64_t n) {
  for (int64_t i = 0; i < n; ++i) orc_pair(seed, stream[i], idx[i], &U[i], &V[i]);
}

void orc_philox_n(const uint32_t* ctr, const uint32_t* key, uint32_t* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) orc_philox4x32_10(ctr + 4 * i, key + 2 * i, out + 4 * i);
}

/* exported single-step forms of the static definitions (unit tests pin them
 * against the paper's closed forms: eq. nextau, eqs. lambdataua..newtau,
 * eqs. Wsum..vindex) */
double orc_cand(double t, double R, double lam) { return cand_time(t, R, lam); }

double orc_breakpoint_budget(double R, double lam_old, double t_b, double t_s) {
  double r = R - lam_old * (t_b - t_s);
  if (r < 0.0) r = 0.0;
  return r;
}

double orc_fold(const int32_t* N, const double* rate) { return fold_lambda(N, rate); }

void orc_select(const int32_t* N, const double* rate, double V, double lam, int32_t* kstar,
                int64_t* j) {
  int k;
  select_class_index(N, rate, V, lam, &k, j);
  *kstar = k;
}

/* per-region class counts N_k (eq. nidef) of a configuration,
 * using the same site classification as orc_des_run */
int orc_class_counts(int32_t Lx, int32_t Ly, int32_t bx, int32_t by, const uint8_t* spins,
                     int32_t* N) {
  orc_cfg c;
  memset(&c, 0, sizeof c);
  c.Lx = Lx; c.Ly = Ly; c.bx = bx; c.by = by;
  int rc = validate(&c);
  if (rc) return rc;
  lat_t L = {Lx, Ly, (uint8_t*)spins, NULL};
  int RX = Lx / bx, RY = Ly / by;
  memset(N, 0, sizeof(int32_t) * 10 * (size_t)RX * RY);
  for (int v = 0; v < Lx * Ly; ++v) {
    int y = v / Lx, x = v % Lx;
    N[((y / by) * RX + x / bx) * 10 + site_class(&L, v)]++;
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Checkerboard Metropolis (§2 dynamics; see ising_oracle.h):      */
/* the plain definition, one site at a time.                                  */
/* ------------------------------------------------------------------------ */
int orc_cb_run(int32_t Lx, int32_t Ly, const double* p, uint64_t seed, int64_t sweep0, int32_t nsweeps,
               uint8_t* spins, int64_t* flips) {
  if (Lx < 4 || Ly < 4 || (Lx & 1) || (Ly & 1) || nsweeps < 0 || sweep0 < 0 || !spins || !p) return -1;
  if ((int64_t)Lx * Ly > 0xFFFFFFFFLL || sweep0 + (int64_t)nsweeps > 0x7FFFFFFFFFFFFFFFLL / 2) return -1;
  for (int k = 0; k < 10; ++k)
    if (!(p[k] >= 0.0 && p[k] <= 1.0)) return -1;
  const int64_t N = (int64_t)Lx * Ly;
  for (int64_t i = 0; i < N; ++i) spins[i] = spins[i] ? 1 : 0;
  const int32_t ppr = (Lx + 2) / 4;  /* draws per row and colour: ceil((Lx/2) / 2) */
  int64_t nflip = 0;
  for (int64_t s = sweep0; s < sweep0 + nsweeps; ++s) {
    for (int colour = 0; colour < 2; ++colour) {
      for (int32_t y = 0; y < Ly; ++y) {
        for (int32_t x = 0; x < Lx; ++x) {
          if (((x + y) & 1) != colour) continue;
          const int64_t i = (int64_t)y * Lx + x;
          /* periodic 4-neighbourhood */
          const int up = spins[(int64_t)((y + Ly - 1) % Ly) * Lx + x] + spins[(int64_t)((y + 1) % Ly) * Lx + x] +
                         spins[(int64_t)y * Lx + (x + Lx - 1) % Lx] + spins[(int64_t)y * Lx + (x + 1) % Lx];
          const int k = (spins[i] ? 5 : 0) + up;
          /* this site is the j-th of its colour in row y; sites 2m and 2m+1
             share draw q = y * ppr + m: U from words (x0,x1), resp. (x2,x3) */
          const int32_t j = x >> 1, m = j >> 1;
          const uint32_t q = (uint32_t)((int64_t)y * ppr + m);
          uint32_t ctr[4] = {q, (uint32_t)s, (uint32_t)((uint64_t)s >> 32) | ((uint32_t)colour << 31),
                             (uint32_t)(seed >> 32)};
          uint32_t key[2] = {0xFFFFFFFEu, (uint32_t)seed};
          uint32_t xw[4];
          orc_philox4x32_10(ctr, key, xw);
          const double U = (j & 1) ? unit_from_words(xw[2], xw[3]) : unit_from_words(xw[0], xw[1]);
          if (U < p[k]) {
            spins[i] ^= 1;
            ++nflip;
          }
        }
      }
    }
  }
  if (flips) *flips = nflip;
  return 0;
}
