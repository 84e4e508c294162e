/* SPDX-License-Identifier: Apache-2.0
 *
 * TEST INFRASTRUCTURE ONLY — never linked into or called by the product
 * (paper_2211_16270_b200/). Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / reference arm may use it, as the checker.
 *
 * Plain-C restatement of the sequential parts of the reference's
 * sample-wise transducer path, in float64. The dense linear algebra of the
 * same path is restated in numpy in swt_oracle.py. Pinned against the
 * reference (oracle/_ref) and its known-answer tests by
 * tests/test_oracle_cpu.py and the committed fixtures in tests/golden/.
 *
 * Restated reference items (paths relative to /root/reference/proj):
 *   mt64_*                std::mt19937_64 as used by core/include/swt/rng.hpp:14-37
 *   orc_padded_lengths    core/src/bench.cpp:48-64
 *   orc_synth_inputs      core/src/bench.cpp:66-115 (draw order, mapping)
 *   orc_parallel_iter     core/src/engine.cpp:31-50 (Eq. 9)
 *   orc_log_add_exp       core/include/swt/loss.hpp:56-64
 *   orc_lattice           core/src/loss.cpp:41-81 (alpha/beta recursions)
 *   orc_count_paths       core/src/oracle.cpp:10-22
 *   orc_enumerate_loss    core/src/oracle.cpp:24-85 (pairwise log-sum)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- mt19937_64 (ISO C++ [rand.predef]: w=64 n=312 m=156 r=31) ---- */
typedef struct {
  uint64_t s[312];
  int i;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->s[0] = seed;
  for (int k = 1; k < 312; ++k)
    g->s[k] = 6364136223846793005ULL * (g->s[k - 1] ^ (g->s[k - 1] >> 62)) +
              (uint64_t)k;
  g->i = 312;
}

static uint64_t mt64_next(mt64* g) {
  if (g->i >= 312) {
    for (int k = 0; k < 312; ++k) {
      const uint64_t y = (g->s[k] & 0xFFFFFFFF80000000ULL) |
                         (g->s[(k + 1) % 312] & 0x7FFFFFFFULL);
      g->s[k] = g->s[(k + 156) % 312] ^ (y >> 1) ^
                ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
    }
    g->i = 0;
  }
  uint64_t x = g->s[g->i++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

uint64_t orc_mt64_first(uint64_t seed, int64_t n, uint64_t* out) {
  mt64 g;
  mt64_seed(&g, seed);
  for (int64_t k = 0; k < n; ++k) out[k] = mt64_next(&g);
  return n > 0 ? out[n - 1] : 0;
}

void orc_padded_lengths(int64_t B, int64_t T, int64_t U, int64_t* t_len,
                        int64_t* u_len) {
  for (int64_t b = 0; b < B; ++b) {
    const double ramp = B == 1 ? 0.0 : (double)b / (double)(B - 1);
    const int64_t t = llround((double)T * (1.0 - 0.093 * ramp));
    const int64_t u = llround((double)U * (1.0 - 0.458 * ramp));
    t_len[b] = t < 1 ? 1 : t;
    u_len[b] = u < 1 ? 1 : u;
  }
}

/* value = lo + (hi - lo) * unit(), unit() = (x >> 11) * 2^-53 */
static void fill_u(mt64* g, float* p, int64_t n) {
  const double lo = -0.1, hi = 0.1;
  for (int64_t k = 0; k < n; ++k) {
    const double unit = (double)(mt64_next(g) >> 11) * 0x1.0p-53;
    volatile double span = hi - lo; /* keep the reference's op order */
    p[k] = (float)(lo + span * unit);
  }
}

int orc_synth_inputs(int64_t B, int64_t T, int64_t U, int64_t H, int64_t HA,
                     int64_t HL, int64_t V, uint64_t seed, float* acoustic,
                     float* label, int32_t* labels, int64_t* t_len,
                     int64_t* u_len, float* wa, float* wl, float* bz,
                     float* wo, float* bo) {
  if (B < 1 || T < 1 || U < 1 || H < 1 || HA < 1 || HL < 1 || V < 2) return 2;
  orc_padded_lengths(B, T, U, t_len, u_len);
  mt64 g;
  mt64_seed(&g, seed);
  fill_u(&g, acoustic, B * T * HA);
  for (int64_t b = 0; b < B; ++b)
    for (int64_t k = (b * T + t_len[b]) * HA; k < (b + 1) * T * HA; ++k)
      acoustic[k] = 0.f;
  fill_u(&g, label, B * (U + 1) * HL);
  for (int64_t b = 0; b < B; ++b)
    for (int64_t k = (b * (U + 1) + u_len[b] + 1) * HL;
         k < (b + 1) * (U + 1) * HL; ++k)
      label[k] = 0.f;
  fill_u(&g, wa, H * HA);
  fill_u(&g, wl, H * HL);
  fill_u(&g, bz, H);
  fill_u(&g, wo, V * H);
  fill_u(&g, bo, V);
  memset(labels, 0, (size_t)(B * U) * sizeof(int32_t));
  for (int64_t b = 0; b < B; ++b)
    for (int64_t k = 0; k < u_len[b]; ++k)
      labels[b * U + k] = (int32_t)(1 + (int64_t)(mt64_next(&g) % (uint64_t)(V - 1)));
  return 0;
}

int orc_parallel_iter(int64_t frames, int64_t labels, int64_t vocab,
                      int64_t budget) {
  if (frames < 1 || labels < 1 || vocab < 1) return -1;
  const unsigned __int128 base =
      (unsigned __int128)4 * (unsigned __int128)frames *
      (unsigned __int128)labels * (unsigned __int128)vocab;
  if (budget <= 0 || base > (unsigned __int128)budget) return 1;
  int e = 0;
  unsigned __int128 cur = base;
  while (e < 4 && cur * 2 <= (unsigned __int128)budget) {
    cur *= 2;
    ++e;
  }
  return 1 << e;
}

double orc_log_add_exp(double a, double b) {
  if (a == -INFINITY) return b;
  if (b == -INFINITY) return a;
  const double hi = a > b ? a : b, lo = a > b ? b : a;
  return hi + log1p(exp(lo - hi));
}

/* lpb[t*U1+u] = lp(blank | t,u); lpy[t*U1+u] = lp(y_{u+1} | t,u) for
 * u < U1-1. alpha/beta row-major [T][U1]. Returns beta[0] (log Z). */
double orc_lattice(const double* lpb, const double* lpy, int64_t T,
                   int64_t U1, double* alpha, double* beta) {
  alpha[0] = 0.0;
  for (int64_t t = 0; t < T; ++t)
    for (int64_t u = 0; u < U1; ++u) {
      if (t == 0 && u == 0) continue;
      const double fb = t > 0 ? alpha[(t - 1) * U1 + u] + lpb[(t - 1) * U1 + u]
                              : -INFINITY;
      const double fl = u > 0 ? alpha[t * U1 + u - 1] + lpy[t * U1 + u - 1]
                              : -INFINITY;
      alpha[t * U1 + u] = orc_log_add_exp(fb, fl);
    }
  beta[(T - 1) * U1 + U1 - 1] = lpb[(T - 1) * U1 + U1 - 1];
  for (int64_t t = T - 1; t >= 0; --t)
    for (int64_t u = U1 - 1; u >= 0; --u) {
      if (t == T - 1 && u == U1 - 1) continue;
      const double vb = t < T - 1 ? lpb[t * U1 + u] + beta[(t + 1) * U1 + u]
                                  : -INFINITY;
      const double vl = u < U1 - 1 ? lpy[t * U1 + u] + beta[t * U1 + u + 1]
                                   : -INFINITY;
      beta[t * U1 + u] = orc_log_add_exp(vb, vl);
    }
  return beta[0];
}

int64_t orc_count_paths(int64_t frames, int64_t labels) {
  if (frames < 1 || labels < 0) return -1;
  const int64_t n = frames + labels - 1;
  const int64_t k = labels < n - labels ? labels : n - labels;
  int64_t c = 1;
  for (int64_t i = 1; i <= k; ++i) c = c * (n - k + i) / i;
  return c;
}

static double log_sum_pairwise(const double* x, int64_t n) {
  if (n == 0) return -INFINITY;
  if (n == 1) return x[0];
  const int64_t h = n / 2;
  return orc_log_add_exp(log_sum_pairwise(x, h), log_sum_pairwise(x + h, n - h));
}

typedef struct {
  const double* lpb;
  const double* lpy;
  int64_t T, U1, n;
  double* out;
} walker;

static void walk(walker* w, int64_t t, int64_t u, double acc) {
  const int last_t = t == w->T - 1, last_u = u == w->U1 - 1;
  if (last_t && last_u) {
    w->out[w->n++] = acc + w->lpb[t * w->U1 + u];
    return;
  }
  if (!last_t) walk(w, t + 1, u, acc + w->lpb[t * w->U1 + u]);
  if (!last_u) walk(w, t, u + 1, acc + w->lpy[t * w->U1 + u]);
}

/* -log sum over every monotone alignment path; -1e300 if over the guard. */
double orc_enumerate_loss(const double* lpb, const double* lpy, int64_t T,
                          int64_t U1, int64_t max_paths) {
  const int64_t total = orc_count_paths(T, U1 - 1);
  if (total < 0 || total > max_paths) return -1e300;
  walker w = {lpb, lpy, T, U1, 0, (double*)malloc(sizeof(double) * (size_t)total)};
  walk(&w, 0, 0, 0.0);
  const double r = -log_sum_pairwise(w.out, w.n);
  free(w.out);
  return r;
}
