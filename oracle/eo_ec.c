/* eo_ec.c -- TEST INFRASTRUCTURE (parity oracle, see evorl_oracle.h).
 * EC algorithms: centred ranks, OpenES, ARS, VanillaES, CMA-ES, CEM.
 * Restates proj/src/ec.cpp and proj/include/evorl/ec.hpp. */
#define _GNU_SOURCE
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "evorl_oracle.h"

int eo_set_error(int code, const char* fmt, ...);

/* ------------------------------------------------ stable sort (merge sort)
 * std::stable_sort with a strict weak order; ties keep index order. */
typedef int (*eo_less_fn)(const double* f, int32_t a, int32_t b);
static int less_asc(const double* f, int32_t a, int32_t b) { return f[a] < f[b]; }
static int less_desc(const double* f, int32_t a, int32_t b) { return f[a] > f[b]; }

static void merge_sort(int32_t* idx, int32_t* tmp, int64_t n, const double* f, eo_less_fn less) {
  for (int64_t w = 1; w < n; w *= 2) {
    for (int64_t lo = 0; lo < n; lo += 2 * w) {
      int64_t mid = lo + w < n ? lo + w : n;
      int64_t hi = lo + 2 * w < n ? lo + 2 * w : n;
      int64_t i = lo, j = mid, k = lo;
      while (i < mid && j < hi) {
        /* take right only if strictly less: stability */
        if (less(f, idx[j], idx[i]))
          tmp[k++] = idx[j++];
        else
          tmp[k++] = idx[i++];
      }
      while (i < mid) tmp[k++] = idx[i++];
      while (j < hi) tmp[k++] = idx[j++];
    }
    memcpy(idx, tmp, sizeof(int32_t) * (size_t)n);
  }
}

static void stable_order(const double* f, int64_t n, int32_t* idx, eo_less_fn less) {
  for (int64_t i = 0; i < n; ++i) idx[i] = (int32_t)i;
  int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  merge_sort(idx, tmp, n, f, less);
  free(tmp);
}

/* proj/src/ec.cpp:14-20 */
void eo_rank_desc(const double* f, int64_t n, int32_t* idx) { stable_order(f, n, idx, less_desc); }
void eo_rank_asc(const double* f, int64_t n, int32_t* idx) { stable_order(f, n, idx, less_asc); }

/* proj/src/ec.cpp:32-46 */
void eo_centered_ranks(const double* f, int64_t n, double* shaped) {
  if (n <= 0) return;
  if (n == 1) {
    shaped[0] = 0.0;
    return;
  }
  int32_t* idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  eo_rank_asc(f, n, idx);
  for (int64_t rank = 0; rank < n; ++rank)
    shaped[idx[rank]] = (double)rank / (double)(n - 1) - 0.5;
  free(idx);
}

/* ============================================================= OpenES */
/* proj/include/evorl/ec.hpp:21-29, defaults of proj/src/config.cpp:45-50 */
eo_openes_cfg eo_openes_default(void) {
  eo_openes_cfg c;
  c.pop = 128;
  c.sigma = 0.02;
  c.lr = 0.01;
  c.weight_decay = 0.005;
  c.mirrored = 1;
  c.noise_table = 0;
  c.noise_table_size = (int64_t)1 << 22;
  return c;
}

/* proj/src/ec.cpp:50-61 */
int eo_openes_init(eo_openes_state* s, const eo_openes_cfg* cfg, const double* mean0, int64_t d,
                   eo_key key) {
  memset(s, 0, sizeof *s);
  s->cfg = *cfg;
  s->d = d;
  s->mean = (double*)malloc(sizeof(double) * (size_t)d);
  s->m = (double*)calloc((size_t)d, sizeof(double));
  s->v = (double*)calloc((size_t)d, sizeof(double));
  if (!s->mean || !s->m || !s->v) return eo_set_error(EO_E_NOMEM, "out of memory");
  memcpy(s->mean, mean0, sizeof(double) * (size_t)d);
  s->sigma = cfg->sigma;
  s->t = 0;
  if (cfg->noise_table) {
    s->table_seed = eo_fold_in(key, 0x7ab1e).lo;
    eo_openes_rebuild_table(s);
  }
  return EO_OK;
}

void eo_openes_free(eo_openes_state* s) {
  free(s->mean);
  free(s->m);
  free(s->v);
  free(s->table);
  memset(s, 0, sizeof *s);
}

/* proj/src/ec.cpp:63-69 */
void eo_openes_rebuild_table(eo_openes_state* s) {
  if (!s->cfg.noise_table) return;
  free(s->table);
  s->table = (double*)malloc(sizeof(double) * (size_t)s->cfg.noise_table_size);
  eo_stream st;
  eo_stream_init(&st, eo_key_from_seed(s->table_seed));
  for (int64_t i = 0; i < s->cfg.noise_table_size; ++i) s->table[i] = eo_normal(&st);
}

/* proj/src/ec.cpp:71-97 */
int eo_openes_ask(const eo_openes_state* s, eo_key key, int n, double* candidates, double* eps) {
  if (n < 2) return eo_set_error(EO_E_INVALID_ARGUMENT, "openes_ask: population must be at least 2");
  if (s->cfg.mirrored && n % 2 != 0)
    return eo_set_error(EO_E_INVALID_ARGUMENT,
                        "openes_ask: mirrored sampling needs an even population");
  const int64_t d = s->d;
  const int base = s->cfg.mirrored ? n / 2 : n;
  if (s->cfg.noise_table) {
    eo_stream st;
    eo_stream_init(&st, key);
    const uint64_t span = (uint64_t)(s->cfg.noise_table_size - d);
    for (int i = 0; i < base; ++i) {
      const int64_t off = (int64_t)eo_randint(&st, span + 1);
      memcpy(eps + (int64_t)i * d, s->table + off, sizeof(double) * (size_t)d);
    }
  } else {
    eo_gaussian_matrix(key, base, d, eps);
  }
  if (s->cfg.mirrored)
    for (int i = 0; i < base; ++i)
      for (int64_t p = 0; p < d; ++p) eps[(int64_t)(base + i) * d + p] = -eps[(int64_t)i * d + p];
  if (candidates)
    for (int i = 0; i < n; ++i)
      for (int64_t p = 0; p < d; ++p)
        candidates[(int64_t)i * d + p] = s->sigma * eps[(int64_t)i * d + p] + s->mean[p];
  return EO_OK;
}

/* proj/src/ec.cpp:99-109 */
int eo_openes_tell(eo_openes_state* s, const double* eps, const double* fitness, int n) {
  const int64_t d = s->d;
  double* shaped = (double*)malloc(sizeof(double) * (size_t)n);
  double* g = (double*)malloc(sizeof(double) * (size_t)d);
  eo_centered_ranks(fitness, n, shaped);
  const double denom = (double)n * s->sigma;
  for (int64_t p = 0; p < d; ++p) {
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc += eps[(int64_t)i * d + p] * shaped[i];
    g[p] = -(acc / denom); /* Adam descends; ascent direction negated */
  }
  eo_adam_cfg cfg = eo_adam_default();
  cfg.lr = s->cfg.lr;
  cfg.weight_decay = s->cfg.weight_decay;
  eo_adam_step(s->mean, g, s->m, s->v, &s->t, d, &cfg);
  free(shaped);
  free(g);
  return EO_OK;
}

/* ================================================================ ARS */
eo_ars_cfg eo_ars_default(void) {
  eo_ars_cfg c = {128, 16, 0.03, 0.02};
  return c;
}

/* proj/src/ec.cpp:113-125 */
int eo_ars_ask(const double* mean, int64_t d, double sigma, eo_key key, int n, double* deltas,
               double* candidates) {
  if (n < 2 || n % 2 != 0) return eo_set_error(EO_E_INVALID_ARGUMENT, "ars_ask: population must be even");
  const int half = n / 2;
  eo_gaussian_matrix(key, half, d, deltas);
  if (candidates)
    for (int k = 0; k < half; ++k)
      for (int64_t p = 0; p < d; ++p) {
        const double sd = sigma * deltas[(int64_t)k * d + p];
        candidates[(int64_t)(2 * k) * d + p] = mean[p] + sd;
        candidates[(int64_t)(2 * k + 1) * d + p] = mean[p] - sd;
      }
  return EO_OK;
}

/* proj/src/ec.cpp:127-154 */
int eo_ars_tell(double* mean, int64_t d, const eo_ars_cfg* cfg, const double* deltas,
                const double* r_plus, const double* r_minus, int half) {
  const int b = cfg->elites < half ? cfg->elites : half;
  double* scores = (double*)calloc((size_t)(half > 0 ? half : 1), sizeof(double));
  int32_t* idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)(half > 0 ? half : 1));
  /* r_plus.cwiseMax(r_minus): std::max(a, b) = (a < b) ? b : a */
  for (int i = 0; i < half; ++i) scores[i] = r_plus[i] < r_minus[i] ? r_minus[i] : r_plus[i];
  eo_rank_desc(scores, half, idx);
  double* elite = (double*)malloc(sizeof(double) * (size_t)(2 * b > 0 ? 2 * b : 1));
  for (int k = 0; k < b; ++k) {
    elite[2 * k] = r_plus[idx[k]];
    elite[2 * k + 1] = r_minus[idx[k]];
  }
  double sum = 0.0;
  for (int k = 0; k < 2 * b; ++k) sum += elite[k];
  const double emean = sum / (double)(2 * b);
  double sq = 0.0;
  for (int k = 0; k < 2 * b; ++k) sq += (elite[k] - emean) * (elite[k] - emean);
  const double sigma_r = sqrt(sq / (double)(2 * b));
  if (sigma_r == 0.0) {
    free(scores);
    free(idx);
    free(elite);
    return 0;
  }
  double* step = (double*)calloc((size_t)d, sizeof(double));
  for (int k = 0; k < b; ++k) {
    const double diff = r_plus[idx[k]] - r_minus[idx[k]];
    const double* dl = deltas + (int64_t)idx[k] * d;
    for (int64_t p = 0; p < d; ++p) step[p] += diff * dl[p];
  }
  const double scale = cfg->lr / ((double)b * sigma_r);
  for (int64_t p = 0; p < d; ++p) mean[p] += scale * step[p];
  free(step);
  free(scores);
  free(idx);
  free(elite);
  return 1;
}

/* ========================================================== VanillaES */
eo_ves_cfg eo_ves_default(void) {
  eo_ves_cfg c = {128, 16, 0.02, 1};
  return c;
}

/* proj/src/ec.cpp:158-162 */
void eo_canonical_es_weights(int mu, double* w) {
  double s = 0.0;
  for (int i = 0; i < mu; ++i) {
    w[i] = log(mu + 0.5) - log(i + 1.0);
    s += w[i];
  }
  for (int i = 0; i < mu; ++i) w[i] /= s;
}

/* proj/src/ec.cpp:164-175 */
int eo_ves_ask(const double* mean, int64_t d, const eo_ves_cfg* cfg, eo_key key, int n,
               double* candidates) {
  if (n < 2) return eo_set_error(EO_E_INVALID_ARGUMENT, "ves_ask: population must be at least 2");
  if (cfg->mirrored && n % 2 != 0)
    return eo_set_error(EO_E_INVALID_ARGUMENT, "ves_ask: mirrored sampling needs an even population");
  const int base = cfg->mirrored ? n / 2 : n;
  eo_gaussian_matrix(key, base, d, candidates);
  if (cfg->mirrored)
    for (int i = 0; i < base; ++i)
      for (int64_t p = 0; p < d; ++p)
        candidates[(int64_t)(base + i) * d + p] = -candidates[(int64_t)i * d + p];
  for (int i = 0; i < n; ++i)
    for (int64_t p = 0; p < d; ++p)
      candidates[(int64_t)i * d + p] = cfg->sigma * candidates[(int64_t)i * d + p] + mean[p];
  return EO_OK;
}

/* proj/src/ec.cpp:177-187 */
int eo_ves_tell(double* mean, int64_t d, const eo_ves_cfg* cfg, const double* candidates,
                const double* fitness, int n) {
  const int mu = cfg->elites < n ? cfg->elites : n;
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  double* w = (double*)malloc(sizeof(double) * (size_t)mu);
  eo_rank_desc(fitness, n, order);
  eo_canonical_es_weights(mu, w);
  for (int64_t p = 0; p < d; ++p) {
    double acc = 0.0;
    for (int i = 0; i < mu; ++i) acc += w[i] * candidates[(int64_t)order[i] * d + p];
    mean[p] = acc;
  }
  free(order);
  free(w);
  return EO_OK;
}

/* ============================================================== CMA-ES */
eo_cma_cfg eo_cma_default(void) {
  eo_cma_cfg c = {128, 64, 0.1, 4096};
  return c;
}

/* proj/src/ec.cpp:191-224 */
int eo_cma_init(eo_cma_state* s, const eo_cma_cfg* cfg, const double* mean0, int64_t d) {
  memset(s, 0, sizeof *s);
  if (d > cfg->max_dim)
    return eo_set_error(EO_E_LENGTH,
                        "cmaes: genotype dimension %lld exceeds the full-covariance capacity cap %d",
                        (long long)d, cfg->max_dim);
  s->cfg = *cfg;
  s->dim = (int)d;
  s->mean = (double*)malloc(sizeof(double) * (size_t)d);
  memcpy(s->mean, mean0, sizeof(double) * (size_t)d);
  s->sigma = cfg->sigma0;
  s->C = (double*)calloc((size_t)(d * d), sizeof(double));
  s->B = (double*)calloc((size_t)(d * d), sizeof(double));
  s->D = (double*)malloc(sizeof(double) * (size_t)d);
  s->ps = (double*)calloc((size_t)d, sizeof(double));
  s->pc = (double*)calloc((size_t)d, sizeof(double));
  if (!s->C || !s->B) return eo_set_error(EO_E_NOMEM, "out of memory");
  for (int64_t i = 0; i < d; ++i) {
    s->C[i * d + i] = 1.0;
    s->B[i * d + i] = 1.0;
    s->D[i] = 1.0;
  }
  const int mu = cfg->elites;
  s->mu = mu;
  s->weights = (double*)malloc(sizeof(double) * (size_t)mu);
  double sum = 0.0;
  for (int i = 0; i < mu; ++i) {
    double w = log((cfg->pop + 1) / 2.0) - log(i + 1.0);
    if (w < 0) w = 0.0;
    s->weights[i] = w;
    sum += w;
  }
  double sq = 0.0;
  for (int i = 0; i < mu; ++i) {
    s->weights[i] /= sum;
    sq += s->weights[i] * s->weights[i];
  }
  s->mueff = 1.0 / sq;
  const double dd = (double)d;
  s->cs = (s->mueff + 2.0) / (dd + s->mueff + 5.0);
  const double t = sqrt((s->mueff - 1.0) / (dd + 1.0)) - 1.0;
  s->ds = 1.0 + 2.0 * (t > 0.0 ? t : 0.0) + s->cs;
  s->cc = (4.0 + s->mueff / dd) / (dd + 4.0 + 2.0 * s->mueff / dd);
  s->c1 = 2.0 / ((dd + 1.3) * (dd + 1.3) + s->mueff);
  const double cmu = 2.0 * (s->mueff - 2.0 + 1.0 / s->mueff) / ((dd + 2.0) * (dd + 2.0) + s->mueff);
  s->cmu = (1.0 - s->c1) < cmu ? (1.0 - s->c1) : cmu;
  s->chi_n = sqrt(dd) * (1.0 - 1.0 / (4.0 * dd) + 1.0 / (21.0 * dd * dd));
  return EO_OK;
}

void eo_cma_free(eo_cma_state* s) {
  free(s->mean);
  free(s->C);
  free(s->B);
  free(s->D);
  free(s->ps);
  free(s->pc);
  free(s->weights);
  memset(s, 0, sizeof *s);
}

/* proj/src/ec.cpp:226-234: y = ((z .* D^T) B^T) sigma + mean */
int eo_cma_ask(const eo_cma_state* s, eo_key key, int n, double* cand) {
  const int64_t d = s->dim;
  double* z = (double*)malloc(sizeof(double) * (size_t)(n * d));
  double* zd = (double*)malloc(sizeof(double) * (size_t)d);
  eo_gaussian_matrix(key, n, d, z);
  for (int i = 0; i < n; ++i) {
    for (int64_t j = 0; j < d; ++j) zd[j] = z[(int64_t)i * d + j] * s->D[j];
    for (int64_t p = 0; p < d; ++p) {
      double acc = 0.0;
      /* (zD B^T)_p = sum_j zD_j B(p, j); B column-major: B(p,j) = B[j*d + p] */
      for (int64_t j = 0; j < d; ++j) acc += zd[j] * s->B[j * d + p];
      cand[(int64_t)i * d + p] = acc * s->sigma + s->mean[p];
    }
  }
  free(z);
  free(zd);
  return EO_OK;
}

/* Cyclic Jacobi eigensolver (fp64).  Returns ascending eigenvalues and the
 * matching eigenvectors (column-major), each normalised so that its largest
 * |component| is positive. */
int eo_sym_eig(const double* Ain, int n, double* evals, double* V) {
  double* A = (double*)malloc(sizeof(double) * (size_t)n * n);
  memcpy(A, Ain, sizeof(double) * (size_t)n * n);
  for (int i = 0; i < n * n; ++i) V[i] = 0.0;
  for (int i = 0; i < n; ++i) V[(int64_t)i * n + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        const double a = A[(int64_t)i * n + j];
        tot += a * a;
        if (i != j) off += a * a;
      }
    if (off <= 1e-30 * tot || off == 0.0) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = A[(int64_t)p * n + q];
        if (apq == 0.0) continue;
        const double app = A[(int64_t)p * n + p], aqq = A[(int64_t)q * n + q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) { /* rows p, q */
          const double akp = A[(int64_t)k * n + p], akq = A[(int64_t)k * n + q];
          A[(int64_t)k * n + p] = c * akp - s * akq;
          A[(int64_t)k * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = A[(int64_t)p * n + k], aqk = A[(int64_t)q * n + k];
          A[(int64_t)p * n + k] = c * apk - s * aqk;
          A[(int64_t)q * n + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) { /* V columns p,q (col-major: V[col*n + row]) */
          const double vkp = V[(int64_t)p * n + k], vkq = V[(int64_t)q * n + k];
          V[(int64_t)p * n + k] = c * vkp - s * vkq;
          V[(int64_t)q * n + k] = s * vkp + c * vkq;
        }
      }
  }
  /* sort ascending (selection; stable for ties by original index) */
  int* order = (int*)malloc(sizeof(int) * (size_t)n);
  for (int i = 0; i < n; ++i) order[i] = i;
  for (int i = 0; i < n; ++i) {
    int best = i;
    for (int j = i + 1; j < n; ++j) {
      const double a = A[(int64_t)order[j] * n + order[j]], b = A[(int64_t)order[best] * n + order[best]];
      if (a < b) best = j;
    }
    const int tmp = order[i];
    order[i] = order[best];
    order[best] = tmp;
  }
  double* W = (double*)malloc(sizeof(double) * (size_t)n * n);
  for (int i = 0; i < n; ++i) {
    const int o = order[i];
    evals[i] = A[(int64_t)o * n + o];
    int am = 0;
    for (int k = 1; k < n; ++k)
      if (fabs(V[(int64_t)o * n + k]) > fabs(V[(int64_t)o * n + am])) am = k;
    const double sg = V[(int64_t)o * n + am] < 0 ? -1.0 : 1.0;
    for (int k = 0; k < n; ++k) W[(int64_t)i * n + k] = sg * V[(int64_t)o * n + k];
  }
  memcpy(V, W, sizeof(double) * (size_t)n * n);
  free(W);
  free(order);
  free(A);
  return EO_OK;
}

/* proj/src/ec.cpp:236-288 */
int eo_cma_tell(eo_cma_state* s, const double* cand, const double* fitness, int n) {
  const int64_t d = s->dim;
  const int mu = s->mu;
  /* The reference indexes order[i] for i < mu without a check (undefined
   * behaviour when elites > pop, proj/src/ec.cpp:243-245); refuse instead. */
  if (mu > n)
    return eo_set_error(EO_E_INVALID_ARGUMENT, "cmaes_tell: elites (%d) exceed population (%d)", mu, n);
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  eo_rank_desc(fitness, n, order);
  double* ytop = (double*)malloc(sizeof(double) * (size_t)(mu * d));
  for (int i = 0; i < mu; ++i)
    for (int64_t p = 0; p < d; ++p)
      ytop[(int64_t)i * d + p] = (cand[(int64_t)order[i] * d + p] - s->mean[p]) / s->sigma;
  double* yw = (double*)malloc(sizeof(double) * (size_t)d);
  for (int64_t p = 0; p < d; ++p) {
    double acc = 0.0;
    for (int i = 0; i < mu; ++i) acc += ytop[(int64_t)i * d + p] * s->weights[i];
    yw[p] = acc;
  }
  for (int64_t p = 0; p < d; ++p) s->mean[p] += s->sigma * yw[p];

  /* c_inv_half_yw = B ((B^T yw) ./ max(D, 1e-300)) */
  double* tmp = (double*)malloc(sizeof(double) * (size_t)d);
  double* cih = (double*)malloc(sizeof(double) * (size_t)d);
  for (int64_t j = 0; j < d; ++j) {
    double acc = 0.0;
    for (int64_t p = 0; p < d; ++p) acc += s->B[j * d + p] * yw[p];
    const double dj = s->D[j] > 1e-300 ? s->D[j] : 1e-300;
    tmp[j] = acc / dj;
  }
  for (int64_t p = 0; p < d; ++p) {
    double acc = 0.0;
    for (int64_t j = 0; j < d; ++j) acc += s->B[j * d + p] * tmp[j];
    cih[p] = acc;
  }
  const double cps = sqrt(s->cs * (2.0 - s->cs) * s->mueff);
  for (int64_t p = 0; p < d; ++p) s->ps[p] = (1.0 - s->cs) * s->ps[p] + cps * cih[p];

  const double gen1 = (double)(s->generation + 1);
  double nrm = 0.0;
  for (int64_t p = 0; p < d; ++p) nrm += s->ps[p] * s->ps[p];
  const double ps_norm = sqrt(nrm);
  const int hsig = ps_norm / sqrt(1.0 - pow(1.0 - s->cs, 2.0 * gen1)) <
                   (1.4 + 2.0 / ((double)d + 1.0)) * s->chi_n;
  const double cpc = hsig ? sqrt(s->cc * (2.0 - s->cc) * s->mueff) : 0.0;
  for (int64_t p = 0; p < d; ++p) s->pc[p] = (1.0 - s->cc) * s->pc[p] + cpc * yw[p];

  const double dhsig = (hsig ? 0.0 : 1.0) * s->cc * (2.0 - s->cc);
  const double a = 1.0 - s->c1 - s->cmu;
  for (int64_t r = 0; r < d; ++r)
    for (int64_t c = 0; c < d; ++c) {
      double rmu = 0.0;
      for (int i = 0; i < mu; ++i) rmu += s->weights[i] * ytop[(int64_t)i * d + r] * ytop[(int64_t)i * d + c];
      const double Crc = s->C[r * d + c];
      s->C[r * d + c] = a * Crc + s->c1 * (s->pc[r] * s->pc[c] + dhsig * Crc) + s->cmu * rmu;
    }
  s->sigma *= exp((s->cs / s->ds) * (ps_norm / s->chi_n - 1.0));
  s->generation += 1;

  for (int64_t r = 0; r < d; ++r)
    for (int64_t c = r + 1; c < d; ++c) {
      const double v = 0.5 * (s->C[r * d + c] + s->C[c * d + r]);
      s->C[r * d + c] = v;
      s->C[c * d + r] = v;
    }
  double* ev = (double*)malloc(sizeof(double) * (size_t)d);
  eo_sym_eig(s->C, (int)d, ev, s->B);
  double mn = ev[0];
  for (int64_t i = 1; i < d; ++i)
    if (ev[i] < mn) mn = ev[i];
  if (mn <= 0.0) {
    for (int64_t i = 0; i < d; ++i) s->C[i * d + i] += (1e-10 - mn);
    eo_sym_eig(s->C, (int)d, ev, s->B);
    s->recondition_count += 1;
  }
  for (int64_t i = 0; i < d; ++i) s->D[i] = sqrt(ev[i] > 0.0 ? ev[i] : 0.0);
  free(ev);
  free(order);
  free(ytop);
  free(yw);
  free(tmp);
  free(cih);
  return EO_OK;
}

/* ================================================================ CEM */
eo_cem_cfg eo_cem_default(void) {
  eo_cem_cfg c = {10, 5, 1e-3, 1e-3, 1e-5, 2000};
  return c;
}
