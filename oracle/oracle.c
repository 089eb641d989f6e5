/*
 * oracle.c — CPU restatement of the InfMoE MoE-layer hot path.
 * TEST INFRASTRUCTURE ONLY (see oracle.h header): the product never uses it.
 *
 * Each function cites the reference file:line it restates
 * (paths relative to /root/reference/proj/include/moesim/).
 * Compiled with -ffp-contract=off so a*b+c stays two roundings, as in the
 * reference build (SURVEY.md §8c FP-contract caveat).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ======================= prng.hpp ======================================= */

/* prng.hpp:18-23 */
uint64_t or_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

/* prng.hpp:27-29 */
uint64_t or_derive_seed(uint64_t seed, uint64_t tag) {
  return or_splitmix64(seed ^ or_splitmix64(tag));
}

/* std::mt19937_64 (the standardised engine behind prng.hpp:68) */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ull * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}

static uint64_t mt64_next(mt64* s) {
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ull) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFull);
      uint64_t xa = x >> 1;
      if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
      s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
    }
    s->idx = 0;
  }
  uint64_t y = s->mt[s->idx++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

uint64_t or_mt64_first(uint64_t seed) {
  mt64 s;
  mt64_seed(&s, seed);
  return mt64_next(&s);
}

/* prng.hpp:32-34 */
static double uniform01(mt64* s) { return (double)(mt64_next(s) >> 11) * 0x1.0p-53; }
/* prng.hpp:37-39 */
static double uniform01_open0(mt64* s) {
  return ((double)(mt64_next(s) >> 11) + 1.0) * 0x1.0p-53;
}
/* prng.hpp:44-46 */
static uint64_t uniform_below(mt64* s, uint64_t n) {
  return (uint64_t)(uniform01(s) * (double)n) % n;
}

/* prng.hpp:49-71 — Box-Muller, cos first, sin cached as the spare */
void or_gaussian_fill(uint64_t seed, double* out, uint64_t n) {
  mt64 s;
  mt64_seed(&s, seed);
  const double pi = 3.141592653589793238462643383279502884;
  uint64_t i = 0;
  while (i < n) {
    const double u1 = uniform01_open0(&s);
    const double u2 = uniform01(&s);
    const double r = sqrt(-2.0 * log(u1));
    const double theta = 2.0 * pi * u2;
    out[i++] = r * cos(theta);
    if (i < n) out[i++] = r * sin(theta);
  }
}

/* --- counter-hash fill (builder-defined synthetic-input contract shared with
 * the product's fill kernels, csrc/kernels/fill.cu).  element i:
 *   h = splitmix64(seed ^ splitmix64(i)); u = (h >> 40) * 2^-24 (exact fp32)
 *   v = (2u - 1) * scale  (one fp32 rounding)  -> uniform, variance scale^2/3 */
static float hash_uniform(uint64_t seed, uint64_t i, float scale) {
  uint64_t h = or_splitmix64(seed ^ or_splitmix64(i));
  float u = (float)(h >> 40) * 5.9604644775390625e-8f;
  float c = 2.0f * u - 1.0f;
  return c * scale;
}

uint16_t or_f32_to_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40u); /* NaN */
  uint32_t lsb = (u >> 16) & 1u;
  u += 0x7fffu + lsb;
  return (uint16_t)(u >> 16);
}

float or_bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

void or_fill_uniform_f32(uint64_t seed, uint64_t n, float scale, float* out) {
  for (uint64_t i = 0; i < n; ++i) out[i] = hash_uniform(seed, i, scale);
}

void or_fill_uniform_bf16(uint64_t seed, uint64_t n, float scale, uint16_t* out) {
  for (uint64_t i = 0; i < n; ++i) out[i] = or_f32_to_bf16(hash_uniform(seed, i, scale));
}

/* ======================= gating.hpp ===================================== */

/* gating.hpp:47-56 — bit-major projection drawn from GaussianStream(seed) */
int or_gating_projection(uint64_t seed, int bits, int hidden, double* out) {
  if (bits < 1 || bits > 31 || hidden < 1) return 2;
  or_gaussian_fill(seed, out, (uint64_t)bits * (uint64_t)hidden);
  return 0;
}

/* gating.hpp:61-82 — sequential d-order fp64 dot, bit j set when dot >= 0 */
int or_lsh_codes(uint64_t seed, int bits, int hidden, const double* x, uint64_t n,
                 uint32_t* codes) {
  double* proj = (double*)malloc(sizeof(double) * (size_t)bits * (size_t)hidden);
  if (!proj) return 5;
  int rc = or_gating_projection(seed, bits, hidden, proj);
  if (rc) {
    free(proj);
    return rc;
  }
  for (uint64_t t = 0; t < n; ++t) {
    const double* row = x + t * (uint64_t)hidden;
    uint32_t code = 0;
    for (int j = 0; j < bits; ++j) {
      const double* hp = proj + (size_t)j * hidden;
      double dot = 0.0;
      for (int c = 0; c < hidden; ++c) dot += row[c] * hp[c];
      if (dot >= 0.0) code |= (1u << j);
    }
    codes[t] = code;
  }
  free(proj);
  return 0;
}

/* gating.hpp:87-104 */
int or_route_tokens(uint64_t seed, int bits, int hidden, const double* x, uint64_t n,
                    int n_experts, uint64_t* counts) {
  if (n_experts < 1) return 2;
  int b = bits < 31 ? bits : 31;
  if ((1u << b) < (uint32_t)n_experts) return 2;
  uint32_t* codes = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  int rc = or_lsh_codes(seed, bits, hidden, x, n, codes);
  if (rc == 0) {
    memset(counts, 0, sizeof(uint64_t) * (size_t)n_experts);
    for (uint64_t t = 0; t < n; ++t) counts[codes[t] % (uint32_t)n_experts]++;
  }
  free(codes);
  return rc;
}

/* gating.hpp:122-165 */
int or_synthetic_workload(int kind, uint64_t total, int n_experts, uint64_t seed,
                          double zipf_s, uint64_t* counts) {
  if (n_experts < 1) return 2;
  memset(counts, 0, sizeof(uint64_t) * (size_t)n_experts);
  if (kind == 2) { /* balanced */
    uint64_t base = total / (uint64_t)n_experts, rem = total % (uint64_t)n_experts;
    for (int e = 0; e < n_experts; ++e) counts[e] = base + ((uint64_t)e < rem ? 1 : 0);
    return 0;
  }
  mt64 s;
  mt64_seed(&s, seed);
  if (kind == 0) { /* uniform */
    for (uint64_t t = 0; t < total; ++t) counts[uniform_below(&s, (uint64_t)n_experts)]++;
    return 0;
  }
  if (kind == 1) { /* zipf */
    if (!(zipf_s > 0.0)) return 2;
    double* cum = (double*)malloc(sizeof(double) * (size_t)n_experts);
    double acc = 0.0;
    for (int e = 0; e < n_experts; ++e) {
      acc += pow((double)(e + 1), -zipf_s);
      cum[e] = acc;
    }
    for (uint64_t t = 0; t < total; ++t) {
      const double u = uniform01(&s) * acc;
      /* std::lower_bound: first cum[i] >= u */
      int lo = 0, hi = n_experts;
      while (lo < hi) {
        int mid = (lo + hi) / 2;
        if (cum[mid] < u) lo = mid + 1; else hi = mid;
      }
      int e = lo < n_experts - 1 ? lo : n_experts - 1;
      counts[e]++;
    }
    free(cum);
    return 0;
  }
  return 2;
}

/* ======================= model_config / cost_model ====================== */

/* model_config.hpp:69-73 */
uint64_t or_expert_param_bytes(int d_model, int d_ff, int bpp) {
  return 2ull * (uint64_t)d_model * (uint64_t)d_ff * (uint64_t)bpp;
}
/* model_config.hpp:77-80 */
uint64_t or_expert_flops(int d_model, int d_ff, uint64_t n) {
  return 4ull * n * (uint64_t)d_model * (uint64_t)d_ff;
}

/* cost_model.hpp:43-62 */
int or_compute_costs(int d_model, int d_ff, int bpp, double peak_flops, double h2d_bw,
                     const uint64_t* counts, int T, double* alphas, double* beta) {
  if (!(peak_flops > 0.0) || !(h2d_bw > 0.0)) return 2;
  for (int i = 0; i < T; ++i)
    alphas[i] = (double)or_expert_flops(d_model, d_ff, counts[i]) / peak_flops;
  *beta = (double)or_expert_param_bytes(d_model, d_ff, bpp) / h2d_bw;
  return 0;
}

/* cost_model.hpp:65-78 */
int or_resident_capacity(int d_model, int d_ff, int bpp, uint64_t device_memory,
                         uint64_t reserved, int* K) {
  if (device_memory <= reserved) return 2;
  uint64_t k = (device_memory - reserved) / or_expert_param_bytes(d_model, d_ff, bpp);
  if (k < 1) return 3;
  *K = (int)k;
  return 0;
}

/* ======================= tolerance.hpp ================================== */
static double cmp_tol(double a, double b) {
  double m = fmax(fabs(a), fabs(b));
  double r = 1e-9 * m;
  return r > 1e-15 ? r : 1e-15;
}
static int approx_geq(double a, double b) { return a >= b - cmp_tol(a, b); }
static int approx_leq(double a, double b) { return a <= b + cmp_tol(a, b); }
static int approx_eq(double a, double b) { return fabs(a - b) <= cmp_tol(a, b); }
static int definitely_lt(double a, double b) { return !approx_geq(a, b); }

/* ======================= scheduler.hpp ================================== */

static int is_perm(const int* order, int T) {
  char* seen = (char*)calloc((size_t)T + 1, 1);
  int ok = 1;
  for (int i = 0; i < T; ++i) {
    int e = order[i];
    if (e < 0 || e >= T || seen[e]) { ok = 0; break; }
    seen[e] = 1;
  }
  free(seen);
  return ok;
}

/* scheduler.hpp:70-95 */
int or_check_constraints(const int* order, const double* alphas, int T, double beta,
                         int K, double* slack, int* feasible, int* viol_pos,
                         int* viol_side) {
  if (!is_perm(order, T) || K < 1) return 2;
  int feas = 1, vp = -1, vs = -1;
  double prefix = 0.0;
  for (int m = 0; m < T; ++m) {
    const double lo = m * beta;
    const double hi = (m + K) * beta;
    if (slack) slack[m] = prefix - lo;
    if (feas && !approx_geq(prefix, lo)) { feas = 0; vp = m; vs = 0; }
    if (feas && !approx_leq(prefix, hi)) { feas = 0; vp = m; vs = 1; }
    prefix += alphas[order[m]];
  }
  *feasible = feas;
  if (viol_pos) *viol_pos = vp;
  if (viol_side) *viol_side = vs;
  return 0;
}

static double total_alpha(const double* a, int T) {
  double s = 0.0; /* std::accumulate order, cost_model.hpp:28-30 */
  for (int i = 0; i < T; ++i) s += a[i];
  return s;
}

/* scheduler.hpp:102-109 */
static int classify_infeasible(const double* alphas, int T, double beta) {
  double mn = alphas[0];
  for (int i = 1; i < T; ++i) if (alphas[i] < mn) mn = alphas[i];
  const double best = total_alpha(alphas, T) - mn;
  const double need = (T - 1) * beta;
  return definitely_lt(best, need) ? 1 : 2;
}

static int validate_costs(const double* alphas, int T, double beta) {
  if (T < 1) return 2;
  if (!(beta > 0.0)) return 2;
  for (int i = 0; i < T; ++i) if (!(alphas[i] >= 0.0)) return 2;
  return 0;
}

/* scheduler.hpp:143-180 */
int or_greedy_order(const double* alphas, int T, double beta, int K, int* order,
                    int* feasible, int* diagnosis) {
  if (validate_costs(alphas, T, beta) || K < 1) return 2;
  int* rem = (int*)malloc(sizeof(int) * (size_t)T);
  int nrem = T;
  for (int i = 0; i < T; ++i) rem[i] = i;
  double prefix = 0.0;
  int pos = 0;
  for (int m = 1; m < T; ++m) {
    const double lo = m * beta;
    const double hi = (m + K) * beta;
    int bib = -1, buh = -1, bs = -1;
    for (int r = 0; r < nrem; ++r) {
      int e = rem[r];
      const double p = prefix + alphas[e];
      const int under_hi = approx_leq(p, hi);
      const int in_band = under_hi && approx_geq(p, lo);
      if (in_band && (bib < 0 || alphas[e] < alphas[bib])) bib = e;
      if (under_hi && (buh < 0 || alphas[e] > alphas[buh])) buh = e;
      if (bs < 0 || alphas[e] < alphas[bs]) bs = e;
    }
    int pick = bib >= 0 ? bib : (buh >= 0 ? buh : bs);
    order[pos++] = pick;
    prefix += alphas[pick];
    for (int r = 0; r < nrem; ++r)
      if (rem[r] == pick) {
        memmove(rem + r, rem + r + 1, sizeof(int) * (size_t)(nrem - r - 1));
        --nrem;
        break;
      }
  }
  order[pos++] = rem[0];
  free(rem);
  int feas = 0;
  or_check_constraints(order, alphas, T, beta, K, NULL, &feas, NULL, NULL);
  *feasible = feas;
  *diagnosis = feas ? -1 : classify_infeasible(alphas, T, beta);
  return 0;
}

/* scheduler.hpp:187-237 */
typedef struct {
  const double* a;
  int T, K;
  double beta;
  char* dead;
  int* order;
  int n;
} dfs_ctx;

static int dfs(dfs_ctx* c, uint32_t mask, int m, double prefix) {
  if (m == c->T) return 1;
  if (c->dead[mask]) return 0;
  for (int e = 0; e < c->T; ++e) {
    if (mask & (1u << e)) continue;
    const double p = prefix + c->a[e];
    if (m + 1 <= c->T - 1) {
      const double lo = (m + 1) * c->beta;
      const double hi = (m + 1 + c->K) * c->beta;
      if (!approx_geq(p, lo) || !approx_leq(p, hi)) continue;
    }
    c->order[c->n++] = e;
    if (dfs(c, mask | (1u << e), m + 1, p)) return 1;
    c->n--;
  }
  c->dead[mask] = 1;
  return 0;
}

int or_exact_order(const double* alphas, int T, double beta, int K, int max_T,
                   int* order, int* feasible, int* diagnosis) {
  if (validate_costs(alphas, T, beta) || K < 1) return 2;
  if (max_T > 24) max_T = 24;
  if (T > max_T) return 2;
  dfs_ctx c = {alphas, T, K, beta, (char*)calloc((size_t)1 << T, 1), order, 0};
  int ok = dfs(&c, 0u, 0, 0.0);
  free(c.dead);
  if (ok) {
    int feas = 0;
    or_check_constraints(order, alphas, T, beta, K, NULL, &feas, NULL, NULL);
    *feasible = feas;
    *diagnosis = -1; /* set_diagnosis=false, scheduler.hpp:224-226 */
    return 0;
  }
  for (int i = 0; i < T; ++i) order[i] = i;
  *feasible = 0;
  *diagnosis = classify_infeasible(alphas, T, beta);
  return 0;
}

/* scheduler.hpp:243-248 */
int or_auto_order(const double* alphas, int T, double beta, int K, int max_T,
                  int* order, int* feasible, int* diagnosis, int* method) {
  int rc = or_greedy_order(alphas, T, beta, K, order, feasible, diagnosis);
  if (rc) return rc;
  *method = 0;
  if (*feasible || T > max_T) return 0;
  *method = 1;
  return or_exact_order(alphas, T, beta, K, max_T, order, feasible, diagnosis);
}

/* scheduler.hpp:253-258 */
int or_diagnose(const double* alphas, int T, double beta, int K, int max_T) {
  int* order = (int*)malloc(sizeof(int) * (size_t)T);
  int feas = 0, diag = -1, method = 0;
  int rc = or_auto_order(alphas, T, beta, K, max_T, order, &feas, &diag, &method);
  free(order);
  if (rc) return -2;
  if (feas) return 0;
  return classify_infeasible(alphas, T, beta);
}

/* verification.hpp:33-48 (FNV-1a over bytes) */
uint64_t or_instance_digest(const double* alphas, int T, double beta, int K) {
  uint64_t h = 0xcbf29ce484222325ull;
#define MIX(v)                                  \
  do {                                          \
    uint64_t vv = (v);                          \
    for (int i = 0; i < 8; ++i) {               \
      h ^= (vv >> (8 * i)) & 0xff;              \
      h *= 0x100000001b3ull;                    \
    }                                           \
  } while (0)
  MIX((uint64_t)T);
  MIX((uint64_t)(int64_t)K);
  uint64_t b;
  memcpy(&b, &beta, 8);
  MIX(b);
  for (int i = 0; i < T; ++i) {
    memcpy(&b, &alphas[i], 8);
    MIX(b);
  }
#undef MIX
  return h;
}

static int next_perm(int* a, int n) {
  int i = n - 2;
  while (i >= 0 && a[i] >= a[i + 1]) --i;
  if (i < 0) return 0;
  int j = n - 1;
  while (a[j] <= a[i]) --j;
  int t = a[i]; a[i] = a[j]; a[j] = t;
  for (int l = i + 1, r = n - 1; l < r; ++l, --r) { t = a[l]; a[l] = a[r]; a[r] = t; }
  return 1;
}

/* verification.hpp:50-72 */
int or_enumerate_feasibility(const double* alphas, int T, double beta, int K,
                             int* witness) {
  if (T > 9) return -2;
  int perm[16];
  for (int i = 0; i < T; ++i) perm[i] = i;
  do {
    int feas = 0;
    or_check_constraints(perm, alphas, T, beta, K, NULL, &feas, NULL, NULL);
    if (feas) {
      if (witness) memcpy(witness, perm, sizeof(int) * (size_t)T);
      return 1;
    }
  } while (next_perm(perm, T));
  return 0;
}

/* ======================= simulator.hpp ================================== */

typedef struct {
  double t;
  int d;
} edge;
static int edge_cmp(const void* a, const void* b) {
  const edge* x = (const edge*)a;
  const edge* y = (const edge*)b;
  if (x->t != y->t) return x->t < y->t ? -1 : 1;
  return x->d - y->d; /* -1 before +1 */
}

/* simulator.hpp:63-80 */
static int peak_residency(const double* arrive, const double* evict, int n) {
  edge* e = (edge*)malloc(sizeof(edge) * (size_t)(2 * n + 1));
  for (int i = 0; i < n; ++i) {
    e[2 * i] = (edge){arrive[i], +1};
    e[2 * i + 1] = (edge){evict[i], -1};
  }
  qsort(e, (size_t)(2 * n), sizeof(edge), edge_cmp);
  int cur = 0, peak = 0;
  for (int i = 0; i < 2 * n; ++i) {
    cur += e[i].d;
    if (cur > peak) peak = cur;
  }
  free(e);
  return peak;
}

/* simulator.hpp:53-56 */
double or_lower_bound(const double* alphas, int T, double beta) {
  double a = beta + total_alpha(alphas, T);
  double b = (double)T * beta;
  return a > b ? a : b;
}

/* simulator.hpp:102-194 */
int or_run_layers(int n_layers, const int* Ts, const int* orders, const double* alphas,
                  const double* betas, int K, int mode, int continuous, or_event* ev,
                  or_report* rep, double* layer_stall, int* layer_peak) {
  if (K < 1) return 2;
  double load_free = 0.0, compute_free = 0.0, prev_ce = -1.0;
  memset(rep, 0, sizeof(*rep));
  int ne = 0, off = 0;
  for (int l = 0; l < n_layers; ++l) {
    const int T = Ts[l];
    const int* ord = orders + off;
    const double* a = alphas + off;
    const double beta = betas[l];
    if (!is_perm(ord, T)) return 2;
    double* ce_at = (double*)malloc(sizeof(double) * (size_t)T);
    double* arr = (double*)malloc(sizeof(double) * (size_t)T);
    double* evc = (double*)malloc(sizeof(double) * (size_t)T);
    double lprev = -1.0, lstall = 0.0, lload = 0.0, lcomp = 0.0, layer_end = 0.0;
    if (mode == 0 && !continuous && l > 0) load_free = fmax(load_free, compute_free);
    for (int j = 0; j < T; ++j) {
      const int e = ord[j];
      const double alpha = a[e];
      double ls, le, cs, ce;
      if (mode == 1) {
        ls = fmax(load_free, compute_free);
        le = ls + beta;
        cs = le;
        ce = cs + alpha;
        load_free = le;
        compute_free = ce;
      } else {
        const double gate = j >= K ? ce_at[j - K] : 0.0;
        const double natural = load_free + beta;
        if (gate > natural) {
          le = gate;
          ls = gate - beta;
        } else {
          ls = load_free;
          le = natural;
        }
        load_free = le;
        cs = fmax(le, compute_free);
        ce = cs + alpha;
        compute_free = ce;
      }
      ce_at[j] = ce;
      arr[j] = le;
      evc[j] = ce;
      if (ev) {
        ev[ne++] = (or_event){0, l, e, ls, le};
        ev[ne++] = (or_event){1, l, e, cs, ce};
      }
      lload += le - ls;
      lcomp += ce - cs;
      if (lprev >= 0.0 && cs > lprev) lstall += cs - lprev;
      lprev = ce;
      if (prev_ce >= 0.0 && cs > prev_ce) rep->compute_stall += cs - prev_ce;
      prev_ce = ce;
      if (ce > layer_end) layer_end = ce;
    }
    int pk = peak_residency(arr, evc, T);
    if (layer_stall) layer_stall[l] = lstall;
    if (layer_peak) layer_peak[l] = pk;
    rep->load_busy += lload;
    rep->compute_busy += lcomp;
    if (pk > rep->peak_resident) rep->peak_resident = pk;
    if (layer_end > rep->makespan) rep->makespan = layer_end;
    free(ce_at);
    free(arr);
    free(evc);
    off += T;
  }
  rep->overlap_efficiency = rep->makespan > 0.0 ? rep->compute_busy / rep->makespan : 0.0;
  return 0;
}

/* verification.hpp:108-198 (kinds: 0 overlap, 1 causality, 2 residency,
 * 3 duration, 4 makespan, 5 malformed) */
int or_replay_check(const or_event* ev, int n_ev, int n_layers, const int* Ts,
                    const double* alphas, const double* betas, int K,
                    int check_durations, int* kinds6) {
  int nv = 0;
  int* aoff = (int*)malloc(sizeof(int) * (size_t)(n_layers + 1));
  aoff[0] = 0;
  for (int l = 0; l < n_layers; ++l) aoff[l + 1] = aoff[l] + Ts[l];
  memset(kinds6, 0, sizeof(int) * 6);
#define ADD(k) do { kinds6[k]++; nv++; } while (0)
  for (int i = 0; i < n_ev; ++i) {
    const or_event* e = &ev[i];
    if (e->end < e->start) { ADD(5); continue; }
    if (e->layer_id < 0 || e->layer_id >= n_layers) { ADD(5); continue; }
    if (e->expert_id < 0 || e->expert_id >= Ts[e->layer_id]) { ADD(5); continue; }
    if (check_durations) {
      double want = e->stream == 0 ? betas[e->layer_id] : alphas[aoff[e->layer_id] + e->expert_id];
      if (!approx_eq(e->end - e->start, want)) ADD(3);
    }
  }
  /* stream exclusivity: stable sort by start */
  for (int s = 0; s < 2; ++s) {
    int n = 0;
    int* idx = (int*)malloc(sizeof(int) * (size_t)(n_ev + 1));
    for (int i = 0; i < n_ev; ++i) if (ev[i].stream == s) idx[n++] = i;
    for (int i = 1; i < n; ++i) { /* insertion sort = stable */
      int v = idx[i], j = i - 1;
      while (j >= 0 && ev[idx[j]].start > ev[v].start) { idx[j + 1] = idx[j]; --j; }
      idx[j + 1] = v;
    }
    for (int i = 1; i < n; ++i)
      if (!approx_leq(ev[idx[i - 1]].end, ev[idx[i]].start)) ADD(0);
    free(idx);
  }
  /* causality + residency per layer */
  for (int l = 0; l < n_layers; ++l) {
    int T = Ts[l];
    int* li = (int*)malloc(sizeof(int) * (size_t)T);
    int* ci = (int*)malloc(sizeof(int) * (size_t)T);
    for (int e = 0; e < T; ++e) li[e] = ci[e] = -1;
    for (int i = 0; i < n_ev; ++i)
      if (ev[i].layer_id == l && ev[i].expert_id >= 0 && ev[i].expert_id < T) {
        if (ev[i].stream == 0) li[ev[i].expert_id] = i; else ci[ev[i].expert_id] = i;
      }
    double* arr = (double*)malloc(sizeof(double) * (size_t)T);
    double* evc = (double*)malloc(sizeof(double) * (size_t)T);
    int n = 0;
    for (int e = 0; e < T; ++e) {
      if (li[e] < 0 && ci[e] < 0) continue;
      if (li[e] < 0 || ci[e] < 0) { ADD(1); continue; }
      if (!approx_geq(ev[ci[e]].start, ev[li[e]].end)) ADD(1);
      arr[n] = ev[li[e]].end;
      evc[n] = ev[ci[e]].end;
      ++n;
    }
    if (n && peak_residency(arr, evc, n) > K) ADD(2);
    free(li); free(ci); free(arr); free(evc);
  }
#undef ADD
  free(aoff);
  return nv;
}

/* ======================= MoE layer forward (unpinned) =================== */

/* GeLU, erf form (builder-defined; the reference never names the activation) */
double or_gelu(double v) { return 0.5 * v * (1.0 + erf(v * 0.70710678118654752440)); }

void or_gate_softmax(const float* x, uint64_t N, int d, const float* wg,
                     const float* bias, int E, int k, int32_t* topk_idx,
                     float* topk_w, int32_t* counts) {
  /* tokens are independent: OpenMP over tokens, counts tallied afterwards */
#pragma omp parallel
  {
    float* lg = (float*)malloc(sizeof(float) * (size_t)E);
#pragma omp for schedule(static)
    for (int64_t ti = 0; ti < (int64_t)N; ++ti) {
      const uint64_t t = (uint64_t)ti;
      const float* xr = x + t * (uint64_t)d;
      for (int e = 0; e < E; ++e) {
        const float* wr = wg + (uint64_t)e * (uint64_t)d;
        /* the gate's reduction order (gate.cu N1a): d is walked in chunks of
         * 256 columns; lane l (of 32) owns columns 8l..8l+7 of every chunk
         * and keeps one fmaf chain over them in ascending order (columns past
         * d, up to the chunk end, contribute fmaf(0, 0, acc)); the 32 partial
         * sums are then combined by a butterfly (offsets 16, 8, 4, 2, 1:
         * p[l] = p[l] + p[l ^ off]) and the bias is added last */
        float part[32];
        const int dpad = (d + 255) / 256 * 256;
        for (int l = 0; l < 32; ++l) {
          float acc = 0.0f;
          for (int c0 = 0; c0 < dpad; c0 += 256)
            for (int i = 0; i < 8; ++i) {
              const int c = c0 + 8 * l + i;
              const float xv = c < d ? xr[c] : 0.0f, wv = c < d ? wr[c] : 0.0f;
              acc = fmaf(xv, wv, acc);
            }
          part[l] = acc;
        }
        for (int off = 16; off > 0; off >>= 1) {
          float nxt[32];
          for (int l = 0; l < 32; ++l) nxt[l] = part[l] + part[l ^ off];
          for (int l = 0; l < 32; ++l) part[l] = nxt[l];
        }
        float acc = part[0];
        if (bias) acc = acc + bias[e];
        lg[e] = acc;
      }
      int picked[8];
      for (int j = 0; j < k; ++j) {
        int best = -1;
        for (int e = 0; e < E; ++e) {
          int used = 0;
          for (int q = 0; q < j; ++q) used |= (picked[q] == e);
          if (used) continue;
          if (best < 0) { best = e; continue; }
          if (lg[e] > lg[best] || (lg[best] != lg[best] && lg[e] == lg[e])) best = e;
        }
        picked[j] = best;
        topk_idx[t * k + j] = best;
      }
      /* softmax over all E in fp64 */
      double mx = -INFINITY;
      for (int e = 0; e < E; ++e) if (lg[e] > mx) mx = lg[e];
      double s = 0.0;
      for (int e = 0; e < E; ++e) s += exp((double)lg[e] - mx);
      double p[8], ps = 0.0;
      for (int j = 0; j < k; ++j) {
        p[j] = exp((double)lg[picked[j]] - mx) / s;
        ps += p[j];
      }
      for (int j = 0; j < k; ++j) topk_w[t * k + j] = (float)(k > 1 ? p[j] / ps : p[j]);
    }
    free(lg);
  }
  memset(counts, 0, sizeof(int32_t) * (size_t)E);
  for (uint64_t a = 0; a < N * (uint64_t)k; ++a) counts[topk_idx[a]]++;
}

void or_gate_lsh(const float* x, uint64_t N, int d, const double* proj, int bits,
                 int E, int32_t* topk_idx, float* topk_w, int32_t* counts) {
  memset(counts, 0, sizeof(int32_t) * (size_t)E);
  for (uint64_t t = 0; t < N; ++t) {
    const float* xr = x + t * (uint64_t)d;
    uint32_t code = 0;
    for (int j = 0; j < bits; ++j) {
      const double* hp = proj + (size_t)j * (size_t)d;
      double dot = 0.0;
      for (int c = 0; c < d; ++c) dot += (double)xr[c] * hp[c];
      if (dot >= 0.0) code |= (1u << j);
    }
    int e = (int)(code % (uint32_t)E);
    topk_idx[t] = e;
    topk_w[t] = 1.0f;
    counts[e]++;
  }
}

void or_dispatch(const int32_t* topk_idx, uint64_t N, int k, int E, int32_t* offsets,
                 int32_t* perm, int32_t* inv) {
  int32_t* cur = (int32_t*)calloc((size_t)E + 1, sizeof(int32_t));
  uint64_t A = N * (uint64_t)k;
  for (uint64_t a = 0; a < A; ++a) cur[topk_idx[a]]++;
  offsets[0] = 0;
  for (int e = 0; e < E; ++e) offsets[e + 1] = offsets[e] + cur[e];
  for (int e = 0; e < E; ++e) cur[e] = offsets[e];
  for (uint64_t a = 0; a < A; ++a) {
    int32_t p = cur[topk_idx[a]]++;
    perm[p] = (int32_t)a;
    inv[a] = p;
  }
  free(cur);
}

/* or_expert_ffn lives in oracle_ffn.c (vectorised, OpenMP over rows x columns) */

void or_combine(const float* y_perm, const int32_t* inv, const float* topk_w,
                uint64_t N, int k, int d, float* y) {
  for (uint64_t t = 0; t < N; ++t) {
    float* out = y + t * (uint64_t)d;
    for (int c = 0; c < d; ++c) {
      float acc = 0.0f;
      for (int j = 0; j < k; ++j) {
        int32_t p = inv[t * k + j];
        acc = fmaf(topk_w[t * k + j], y_perm[(uint64_t)p * (uint64_t)d + c], acc);
      }
      out[c] = acc;
    }
  }
}
