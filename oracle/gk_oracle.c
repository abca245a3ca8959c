/*
 * gk_oracle.c -- CPU restatement of the gktab reference (arXiv 1901.04162).
 *
 * TEST INFRASTRUCTURE ONLY (see gk_oracle.h).  Compiled with
 * -O2 -ffp-contract=off so every expression rounds exactly like the
 * reference's x86-64 build (no FMA contraction).  Each function cites the
 * reference file:line it restates; paths are relative to
 * /root/reference/proj/include/gktab/.
 */
#define _GNU_SOURCE
#include "gk_oracle.h"

#include <float.h>
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ------------------------------------------------------------------ kernel */

/* kernel.hpp:30-44 */
static int medium_validate(const go_medium* m) {
  if (!(isfinite(m->lambda0) && m->lambda0 > 0.0)) return GO_INVALID;
  if (!(isfinite(m->eps_r) && m->eps_r > 0.0)) return GO_INVALID;
  if (!(isfinite(m->mu_r) && m->mu_r > 0.0)) return GO_INVALID;
  return GO_OK;
}

int go_wavenumber(const go_medium* m, double* k) {
  int s = medium_validate(m);
  if (s) return s;
  *k = 2.0 * M_PI * sqrt(m->eps_r * m->mu_r) / m->lambda0;
  return GO_OK;
}

/* kernel.hpp:48-61 */
int go_eval_analytic(int kind, double k, double r, go_c128* out) {
  if (!(k >= 0.0)) return GO_INVALID;
  if (kind == GO_GREEN) {
    if (r == 0.0) return GO_DOMAIN;
    if (!(r > 0.0)) return GO_INVALID;
    const double kr = k * r;
    out->re = cos(kr) / r;
    out->im = -sin(kr) / r;
    return GO_OK;
  }
  if (!(r >= 0.0)) return GO_INVALID;
  const double kr = k * r;
  out->re = cos(kr);
  out->im = -sin(kr);
  return GO_OK;
}

/* Extension for lossy media: exp(-jkr) with k = k_re + j k_im,
   i.e. exp(k_im r) (cos(k_re r) - j sin(k_re r)); reduces bitwise to
   kernel.hpp:48-61 when k_im == 0. */
int go_eval_analytic_ck(int kind, double k_re, double k_im, double r, go_c128* out) {
  if (k_im == 0.0) return go_eval_analytic(kind, k_re, r, out);
  if (!(k_re >= 0.0)) return GO_INVALID;
  if (kind == GO_GREEN) {
    if (r == 0.0) return GO_DOMAIN;
    if (!(r > 0.0)) return GO_INVALID;
  } else if (!(r >= 0.0)) {
    return GO_INVALID;
  }
  const double kr = k_re * r;
  const double att = exp(k_im * r);
  double re = cos(kr) * att;
  double im = -sin(kr) * att;
  if (kind == GO_GREEN) {
    re = re / r;
    im = im / r;
  }
  out->re = re;
  out->im = im;
  return GO_OK;
}

int go_eval_analytic_batch(int kind, double k, double k_im, const double* r, size_t n,
                           go_c128* out) {
  for (size_t i = 0; i < n; ++i) {
    int s = go_eval_analytic_ck(kind, k, k_im, r[i], &out[i]);
    if (s) return s;
  }
  return GO_OK;
}

/* ---------------------------------------------------------------- sampling */

/* sampling.hpp:18-45 */
void go_sampling_cfg_default(go_sampling_cfg* c) {
  c->r_min = 1e-4;
  c->r_max = 1.0;
  c->samples_per_wavelength = 1000;
  c->refine_interval_divisor = 2;
  c->refine_halfwidth_in_t = 2.0;
  c->dedup_fraction = 0.5;
  c->refine = 1;
}

int go_sampling_cfg_validate(const go_sampling_cfg* c) {
  if (!(isfinite(c->r_min) && isfinite(c->r_max) && 0.0 < c->r_min && c->r_min < c->r_max))
    return GO_INVALID;
  if (c->samples_per_wavelength < 2) return GO_INVALID;
  if (c->refine_interval_divisor < (c->refine ? 2 : 1)) return GO_INVALID;
  if (!(c->refine_halfwidth_in_t > 0.0)) return GO_INVALID;
  if (!(c->dedup_fraction > 0.0 && c->dedup_fraction <= 1.0)) return GO_INVALID;
  if (c->refine && c->refine_halfwidth_in_t * c->refine_interval_divisor < 1.0) return GO_INVALID;
  return GO_OK;
}

/* sampling.hpp:112-122 */
int go_base_interval(const go_medium* m, int S, double* t) {
  int s = medium_validate(m);
  if (s) return s;
  if (S < 2) return GO_INVALID;
  *t = m->lambda0 / ((double)S * sqrt(m->eps_r * m->mu_r));
  return GO_OK;
}

/* sampling.hpp:127-141 */
int go_zero_crossings(double k, double r_min, double r_max, double* out, size_t cap,
                      size_t* count) {
  if (!(k > 0.0)) return GO_INVALID;
  if (!(0.0 < r_min && r_min < r_max)) return GO_INVALID;
  const double quarter_period = M_PI / (2.0 * k);
  int64_t n = (int64_t)floor(r_min / quarter_period);
  if (n < 1) n = 1;
  size_t c = 0;
  for (;; ++n) {
    const double z = (double)n * quarter_period;
    if (z > r_max) break;
    if (z >= r_min) {
      if (out && c < cap) out[c] = z;
      ++c;
    }
  }
  *count = c;
  return GO_OK;
}

/* SamplingPlan::validate (sampling.hpp:59-88) */
static int plan_validate(const go_plan* p) {
  if (p->n < 2) return GO_INVALID;
  double lo = 0.0, hi = 0.0;
  for (size_t i = 0; i < p->n; ++i) {
    if (!isfinite(p->absc[i])) return GO_INVALID;
    if (i == 0) continue;
    const double gap = p->absc[i] - p->absc[i - 1];
    if (!(gap > 0.0)) return GO_INVALID;
    if (i == 1) {
      lo = hi = gap;
    } else {
      lo = gap < lo ? gap : lo;
      hi = gap > hi ? gap : hi;
    }
  }
  if (lo != p->dr_min) return GO_INVALID;
  if (hi != p->t) return GO_INVALID;
  for (size_t i = 0; i < p->nz; ++i) {
    if (i > 0 && !(p->zeros[i] > p->zeros[i - 1])) return GO_INVALID;
    /* binary_search */
    size_t lo_i = 0, hi_i = p->n;
    while (lo_i < hi_i) {
      size_t mid = lo_i + (hi_i - lo_i) / 2;
      if (p->absc[mid] < p->zeros[i]) lo_i = mid + 1; else hi_i = mid;
    }
    if (!(lo_i < p->n && !(p->zeros[i] < p->absc[lo_i]))) return GO_INVALID;
  }
  return GO_OK;
}

static void plan_gaps(go_plan* p) {
  p->dr_min = p->t = p->absc[1] - p->absc[0];
  for (size_t i = 2; i < p->n; ++i) {
    const double gap = p->absc[i] - p->absc[i - 1];
    p->dr_min = gap < p->dr_min ? gap : p->dr_min; /* std::min(a,b): b<a?b:a */
    p->t = p->t < gap ? gap : p->t;                /* std::max(a,b): a<b?b:a */
  }
}

void go_plan_free(go_plan* p) {
  free(p->absc);
  free(p->zeros);
  memset(p, 0, sizeof(*p));
}

/* make_plan (sampling.hpp:92-105) */
int go_make_plan(const double* absc, size_t n, const double* zeros, size_t nz, go_plan* out) {
  memset(out, 0, sizeof(*out));
  if (n < 2) return GO_INVALID;
  out->absc = (double*)malloc(n * sizeof(double));
  out->zeros = (double*)malloc((nz ? nz : 1) * sizeof(double));
  memcpy(out->absc, absc, n * sizeof(double));
  if (nz) memcpy(out->zeros, zeros, nz * sizeof(double));
  out->n = n;
  out->nz = nz;
  plan_gaps(out);
  int s = plan_validate(out);
  if (s) go_plan_free(out);
  return s;
}

int go_plan_copy_out(const go_plan* p, double* absc, double* zeros) {
  if (absc) memcpy(absc, p->absc, p->n * sizeof(double));
  if (zeros && p->nz) memcpy(zeros, p->zeros, p->nz * sizeof(double));
  return GO_OK;
}

/* std::map<double,bool> kept (sampling.hpp:194) as a sorted array. */
typedef struct {
  double* r;
  unsigned char* z;
  size_t n, cap;
} kept_set;

static size_t kept_lower_bound(const kept_set* s, double r) {
  size_t lo = 0, hi = s->n;
  while (lo < hi) {
    size_t mid = lo + (hi - lo) / 2;
    if (s->r[mid] < r) lo = mid + 1; else hi = mid;
  }
  return lo;
}

static void kept_insert_at(kept_set* s, size_t at, double r, unsigned char z) {
  if (s->n == s->cap) {
    s->cap = s->cap ? 2 * s->cap : 1024;
    s->r = (double*)realloc(s->r, s->cap * sizeof(double));
    s->z = (unsigned char*)realloc(s->z, s->cap);
  }
  memmove(s->r + at + 1, s->r + at, (s->n - at) * sizeof(double));
  memmove(s->z + at + 1, s->z + at, s->n - at);
  s->r[at] = r;
  s->z[at] = z;
  s->n++;
}

/* sampling.hpp:195-206 try_insert */
static void kept_try_insert(kept_set* s, double r, unsigned char is_zero, double keep_gap) {
  size_t it = kept_lower_bound(s, r);
  if (it != s->n) {
    if (s->r[it] == r) {
      s->z[it] = s->z[it] || is_zero;
      return;
    }
    if (s->r[it] - r < keep_gap) return;
  }
  if (it != 0 && r - s->r[it - 1] < keep_gap) return;
  kept_insert_at(s, it, r, is_zero);
}

/* sampling.hpp:149-236 with the medium-derived scalars passed in. */
int go_build_plan_core(const go_sampling_cfg* cfg, double k, double t_nominal, go_plan* out) {
  memset(out, 0, sizeof(*out));
  int s = go_sampling_cfg_validate(cfg);
  if (s) return s;
  const double span = cfg->r_max - cfg->r_min;
  if (!(span >= 2.0 * t_nominal)) return GO_INVALID;
  const size_t steps = (size_t)ceil(span / t_nominal);
  const double t_eff = span / (double)steps;

  if (!cfg->refine) {
    out->n = steps + 1;
    out->absc = (double*)malloc(out->n * sizeof(double));
    out->zeros = (double*)malloc(sizeof(double));
    out->absc[0] = cfg->r_min;
    for (size_t i = 1; i < steps; ++i) out->absc[i] = cfg->r_min + (double)i * t_eff;
    out->absc[steps] = cfg->r_max;
    plan_gaps(out);
    s = plan_validate(out);
    if (s) go_plan_free(out);
    return s;
  }

  const double refined = t_eff / (double)cfg->refine_interval_divisor;
  const double min_gap = cfg->dedup_fraction * refined;
  const int side_steps =
      (int)floor(cfg->refine_halfwidth_in_t * cfg->refine_interval_divisor + 1e-9);
  const double keep_gap = min_gap - 8.0 * DBL_EPSILON * cfg->r_max;

  kept_set ks = {0};
  kept_insert_at(&ks, 0, cfg->r_min, 0);
  kept_insert_at(&ks, 1, cfg->r_max, 0);
  size_t nzc = 0;
  s = go_zero_crossings(k, cfg->r_min, cfg->r_max, NULL, 0, &nzc);
  if (s) {
    free(ks.r);
    free(ks.z);
    return s;
  }
  double* zeros = (double*)malloc((nzc ? nzc : 1) * sizeof(double));
  go_zero_crossings(k, cfg->r_min, cfg->r_max, zeros, nzc, &nzc);
  for (size_t i = 0; i < nzc; ++i) kept_try_insert(&ks, zeros[i], 1, keep_gap);
  for (size_t i = 1; i < steps; ++i)
    kept_try_insert(&ks, cfg->r_min + (double)i * t_eff, 0, keep_gap);
  for (size_t zi = 0; zi < nzc; ++zi) {
    const double z = zeros[zi];
    for (int st = 1; st <= side_steps; ++st) {
      const double off = (double)st * refined;
      if (z - off > cfg->r_min) kept_try_insert(&ks, z - off, 0, keep_gap);
      if (z + off < cfg->r_max) kept_try_insert(&ks, z + off, 0, keep_gap);
    }
  }
  free(zeros);

  out->n = ks.n;
  out->absc = ks.r;
  out->zeros = (double*)malloc((ks.n ? ks.n : 1) * sizeof(double));
  out->nz = 0;
  for (size_t i = 0; i < ks.n; ++i)
    if (ks.z[i]) out->zeros[out->nz++] = ks.r[i];
  free(ks.z);
  plan_gaps(out);
  s = plan_validate(out);
  if (s) go_plan_free(out);
  return s;
}

/* build_plan (sampling.hpp:149-236) */
int go_build_plan(const go_sampling_cfg* cfg, const go_medium* m, go_plan* out) {
  memset(out, 0, sizeof(*out));
  int s = go_sampling_cfg_validate(cfg);
  if (s) return s;
  double k, t;
  if ((s = go_wavenumber(m, &k))) return s;
  if ((s = go_base_interval(m, cfg->samples_per_wavelength, &t))) return s;
  return go_build_plan_core(cfg, k, t, out);
}

/* ------------------------------------------------------------------- table */

/* table.hpp:54-82 */
int go_build_hash(const go_plan* p, go_hash* h) {
  memset(h, 0, sizeof(*h));
  if (p->n < 2) return GO_INVALID;
  if (p->n > 0xffffffffull) return GO_INVALID;
  h->r_min = p->absc[0];
  h->r_max = p->absc[p->n - 1];
  h->dr_min = p->dr_min;
  h->inv_dr_min = 1.0 / p->dr_min;
  const size_t nb = (size_t)ceil((h->r_max - h->r_min) / h->dr_min) + 1;
  h->nb = nb;
  h->buckets = (uint32_t*)calloc(nb, sizeof(uint32_t));
  for (size_t j = 1; j < p->n; ++j) {
    size_t b = (size_t)((p->absc[j] - h->r_min) * h->inv_dr_min);
    if (h->r_min + (double)b * h->dr_min < p->absc[j]) ++b;
    if (b < nb) h->buckets[b] = (uint32_t)j;
  }
  for (size_t b = 1; b < nb; ++b)
    h->buckets[b] = h->buckets[b] < h->buckets[b - 1] ? h->buckets[b - 1] : h->buckets[b];
  return GO_OK;
}

void go_hash_free(go_hash* h) {
  free(h->buckets);
  memset(h, 0, sizeof(*h));
}

/* table.hpp:48-51 */
static size_t bucket_of(const go_hash* h, double r) {
  const size_t b = (size_t)((r - h->r_min) * h->inv_dr_min);
  return b < h->nb ? b : h->nb - 1;
}

/* table.hpp:87-102 */
int go_locate(const go_hash* h, const go_plan* p, double r, size_t* out) {
  if (!(r >= h->r_min && r <= h->r_max)) return GO_RANGE;
  const double* a = p->absc;
  const size_t count = p->n;
  const size_t j = h->buckets[bucket_of(h, r)];
  const size_t back = (size_t)(j > 0 && r < a[j]);
  const size_t fwd1 = (size_t)(j + 1 < count && a[j + 1] <= r);
  const size_t fwd2 = (size_t)(j + 2 < count && a[j + 2] <= r);
  const size_t jc = j - back + fwd1 + fwd2;
  const size_t last_pair = count - 2;
  *out = jc < last_pair ? jc : last_pair;
  return GO_OK;
}

/* --------------------------------------------------------------- evaluator */

struct go_evaluator {
  go_plan plan;
  go_hash hash;
  go_c128* exp_vals;
  go_c128* green_vals;
  double k, k_im;
  int degree;
  double* packed;  /* (n+2) x {r, re, im} */
  double* inv_den; /* 4 (n-3) */
  uint64_t fallbacks;
};

static int analytic(const go_evaluator* ev, int kind, double r, go_c128* out) {
  return go_eval_analytic_ck(kind, ev->k, ev->k_im, r, out);
}

/* table.hpp:24-34 */
static int build_table(const go_plan* p, int kind, double k, double k_im, go_c128* vals) {
  if (p->n < 2) return GO_INVALID;
  if (!(k >= 0.0)) return GO_INVALID;
  if (kind == GO_GREEN && !(p->absc[0] > 0.0)) return GO_DOMAIN;
  for (size_t i = 0; i < p->n; ++i) {
    int s = go_eval_analytic_ck(kind, k, k_im, p->absc[i], &vals[i]);
    if (s) return s;
  }
  return GO_OK;
}

/* evaluator.hpp:274-298 */
static void pack_green_stencils(go_evaluator* ev) {
  const size_t n = ev->plan.n;
  ev->packed = (double*)malloc(3 * (n + 2) * sizeof(double));
  for (size_t i = 0; i < n; ++i) {
    ev->packed[3 * i + 0] = ev->plan.absc[i];
    ev->packed[3 * i + 1] = ev->green_vals[i].re;
    ev->packed[3 * i + 2] = ev->green_vals[i].im;
  }
  for (size_t i = n; i < n + 2; ++i) {
    ev->packed[3 * i + 0] = INFINITY;
    ev->packed[3 * i + 1] = 0.0;
    ev->packed[3 * i + 2] = 0.0;
  }
  ev->inv_den = (double*)malloc(4 * (n - 3) * sizeof(double));
  const double* a = ev->plan.absc;
  for (size_t start = 0; start + 4 <= n; ++start) {
    const double e01 = a[start] - a[start + 1];
    const double e02 = a[start] - a[start + 2];
    const double e03 = a[start] - a[start + 3];
    const double e12 = a[start + 1] - a[start + 2];
    const double e13 = a[start + 1] - a[start + 3];
    const double e23 = a[start + 2] - a[start + 3];
    double* inv = ev->inv_den + 4 * start;
    inv[0] = 1.0 / ((e01 * e02) * e03);
    inv[1] = 1.0 / -((e01 * e12) * e13);
    inv[2] = 1.0 / ((e02 * e12) * e23);
    inv[3] = 1.0 / -((e03 * e13) * e23);
  }
}

void go_evaluator_free(go_evaluator* ev) {
  if (!ev) return;
  go_plan_free(&ev->plan);
  go_hash_free(&ev->hash);
  free(ev->exp_vals);
  free(ev->green_vals);
  free(ev->packed);
  free(ev->inv_den);
  free(ev);
}

/* evaluator.hpp:104-114 */
go_evaluator* go_evaluator_create(const double* absc, size_t n, const double* zeros, size_t nz,
                                  double k, double k_im, int degree, int* status) {
  go_evaluator* ev = (go_evaluator*)calloc(1, sizeof(go_evaluator));
  int s = go_make_plan(absc, n, zeros, nz, &ev->plan);
  if (s) goto fail;
  ev->k = k;
  ev->k_im = k_im;
  ev->degree = degree;
  if (degree < 1) { s = GO_INVALID; goto fail; }
  if ((size_t)degree + 1 > n) { s = GO_INVALID; goto fail; }
  ev->exp_vals = (go_c128*)malloc(n * sizeof(go_c128));
  ev->green_vals = (go_c128*)malloc(n * sizeof(go_c128));
  if ((s = build_table(&ev->plan, GO_EXP, k, k_im, ev->exp_vals))) goto fail;
  if ((s = build_table(&ev->plan, GO_GREEN, k, k_im, ev->green_vals))) goto fail;
  if ((s = go_build_hash(&ev->plan, &ev->hash))) goto fail;
  if (degree == 3) pack_green_stencils(ev);
  *status = GO_OK;
  return ev;
fail:
  *status = s;
  go_evaluator_free(ev);
  return NULL;
}

size_t go_evaluator_size(const go_evaluator* ev) { return ev->plan.n; }
const go_plan* go_evaluator_plan(const go_evaluator* ev) { return &ev->plan; }
const go_hash* go_evaluator_hash(const go_evaluator* ev) { return &ev->hash; }
uint64_t go_evaluator_fallbacks(const go_evaluator* ev) {
  return __atomic_load_n(&ev->fallbacks, __ATOMIC_RELAXED);
}
int go_evaluator_tables(const go_evaluator* ev, go_c128* e, go_c128* g) {
  if (e) memcpy(e, ev->exp_vals, ev->plan.n * sizeof(go_c128));
  if (g) memcpy(g, ev->green_vals, ev->plan.n * sizeof(go_c128));
  return GO_OK;
}

/* evaluator.hpp:22-30 */
static int interp_linear(const go_c128* vals, const go_plan* p, const go_hash* h, double r,
                         go_c128* out) {
  size_t j;
  int s = go_locate(h, p, r, &j);
  if (s) return s;
  const double r0 = p->absc[j];
  const double r1 = p->absc[j + 1];
  const double w0 = (r - r1) / (r0 - r1);
  const double w1 = (r - r0) / (r1 - r0);
  out->re = vals[j].re * w0 + vals[j + 1].re * w1;
  out->im = vals[j].im * w0 + vals[j + 1].im * w1;
  return GO_OK;
}

/* evaluator.hpp:40-95 */
static int interp_lagrange(const go_c128* table, const go_plan* p, const go_hash* h, int degree,
                           double r, go_c128* out) {
  if (degree < 1) return GO_INVALID;
  const size_t width = (size_t)degree + 1;
  const size_t count = p->n;
  if (width > count) return GO_INVALID;
  size_t j;
  int s = go_locate(h, p, r, &j);
  if (s) return s;
  const size_t back_shift = (size_t)((degree - 1) / 2);
  size_t start = j > back_shift ? j - back_shift : 0;
  if (start + width > count) start = count - width;
  const double* nodes = p->absc + start;
  const go_c128* vals = table + start;
  if (degree == 3) {
    const double d0 = r - nodes[0];
    const double d1 = r - nodes[1];
    const double d2 = r - nodes[2];
    const double d3 = r - nodes[3];
    if (d0 == 0.0) { *out = vals[0]; return GO_OK; }
    if (d1 == 0.0) { *out = vals[1]; return GO_OK; }
    if (d2 == 0.0) { *out = vals[2]; return GO_OK; }
    if (d3 == 0.0) { *out = vals[3]; return GO_OK; }
    const double e01 = nodes[0] - nodes[1];
    const double e02 = nodes[0] - nodes[2];
    const double e03 = nodes[0] - nodes[3];
    const double e12 = nodes[1] - nodes[2];
    const double e13 = nodes[1] - nodes[3];
    const double e23 = nodes[2] - nodes[3];
    const double s01 = d0 * d1;
    const double s23 = d2 * d3;
    const double w0 = (d1 * s23) / ((e01 * e02) * e03);
    const double w1 = (d0 * s23) / (-((e01 * e12) * e13));
    const double w2 = (s01 * d3) / ((e02 * e12) * e23);
    const double w3 = (s01 * d2) / (-((e03 * e13) * e23));
    out->re = vals[0].re * w0 + vals[1].re * w1 + vals[2].re * w2 + vals[3].re * w3;
    out->im = vals[0].im * w0 + vals[1].im * w1 + vals[2].im * w2 + vals[3].im * w3;
    return GO_OK;
  }
  double are = 0.0, aim = 0.0;
  for (size_t a = 0; a < width; ++a) {
    double num = 1.0, den = 1.0;
    for (size_t m = 0; m < width; ++m) {
      if (m == a) continue;
      num *= r - nodes[m];
      den *= nodes[a] - nodes[m];
    }
    const double c = num / den;
    are += vals[a].re * c;
    aim += vals[a].im * c;
  }
  out->re = are;
  out->im = aim;
  return GO_OK;
}

int go_interp_linear(const go_evaluator* ev, int kind, double r, go_c128* out) {
  return interp_linear(kind == GO_EXP ? ev->exp_vals : ev->green_vals, &ev->plan, &ev->hash, r,
                       out);
}

int go_interp_lagrange(const go_evaluator* ev, int kind, int degree, double r, go_c128* out) {
  return interp_lagrange(kind == GO_EXP ? ev->exp_vals : ev->green_vals, &ev->plan, &ev->hash,
                         degree, r, out);
}

/* evaluator.hpp:237-272 */
static void green_from_bucket(const go_evaluator* ev, size_t bucket_value, double r,
                              go_c128* out) {
  const double* nodes = ev->packed;
  const size_t n = ev->plan.n;
  const size_t j = bucket_value;
  const size_t back = (size_t)(j > 0 && r < nodes[3 * j]);
  const size_t fwd1 = (size_t)(nodes[3 * (j + 1)] <= r);
  const size_t fwd2 = (size_t)(nodes[3 * (j + 2)] <= r);
  size_t jc = j - back + fwd1 + fwd2;
  const size_t last_pair = n - 2;
  if (jc > last_pair) jc = last_pair;
  size_t start = jc > 0 ? jc - 1 : 0;
  if (start + 4 > n) start = n - 4;
  const double* s = nodes + 3 * start;
  const double d0 = r - s[0];
  const double d1 = r - s[3];
  const double d2 = r - s[6];
  const double d3 = r - s[9];
  if (d0 == 0.0) { out->re = s[1]; out->im = s[2]; return; }
  if (d1 == 0.0) { out->re = s[4]; out->im = s[5]; return; }
  if (d2 == 0.0) { out->re = s[7]; out->im = s[8]; return; }
  if (d3 == 0.0) { out->re = s[10]; out->im = s[11]; return; }
  const double* inv = ev->inv_den + 4 * start;
  const double s01 = d0 * d1;
  const double s23 = d2 * d3;
  const double w0 = (d1 * s23) * inv[0];
  const double w1 = (d0 * s23) * inv[1];
  const double w2 = (s01 * d3) * inv[2];
  const double w3 = (s01 * d2) * inv[3];
  out->re = s[1] * w0 + s[4] * w1 + s[7] * w2 + s[10] * w3;
  out->im = s[2] * w0 + s[5] * w1 + s[8] * w2 + s[11] * w3;
}

/* evaluator.hpp:131 */
int go_eval_exp(const go_evaluator* ev, double r, go_c128* out) {
  return interp_linear(ev->exp_vals, &ev->plan, &ev->hash, r, out);
}

/* evaluator.hpp:138-143 */
int go_eval_green(const go_evaluator* ev, double r, go_c128* out) {
  if (ev->degree != 3) return interp_lagrange(ev->green_vals, &ev->plan, &ev->hash, ev->degree, r, out);
  if (!(r >= ev->hash.r_min && r <= ev->hash.r_max)) return GO_RANGE;
  green_from_bucket(ev, ev->hash.buckets[bucket_of(&ev->hash, r)], r, out);
  return GO_OK;
}

/* evaluator.hpp:199-205 */
int go_eval_kernel(go_evaluator* ev, int kind, double r, go_c128* out) {
  if (r >= ev->plan.absc[0]) return kind == GO_EXP ? go_eval_exp(ev, r, out) : go_eval_green(ev, r, out);
  int s = analytic(ev, kind, r, out);
  if (s) return s;
  __atomic_fetch_add(&ev->fallbacks, 1, __ATOMIC_RELAXED);
  return GO_OK;
}

/* evaluator.hpp:209-221 (every failure is rethrown as invalid_argument) */
int go_eval_batch(go_evaluator* ev, int kind, const double* r, size_t n, go_c128* out,
                  size_t* fail_index) {
  for (size_t i = 0; i < n; ++i) {
    int s = go_eval_kernel(ev, kind, r[i], &out[i]);
    if (s) {
      if (fail_index) *fail_index = i;
      return GO_INVALID;
    }
  }
  return GO_OK;
}

/* evaluator.hpp:150-194 */
int go_accumulate_green(go_evaluator* ev, const double* radii, const double* weights, size_t count,
                        go_c128* out) {
  enum { kMaxBlock = 4096 };
  const uint32_t kScalar = 0xffffffffu;
  if (ev->degree != 3 || count > kMaxBlock) {
    double are = 0.0, aim = 0.0;
    for (size_t i = 0; i < count; ++i) {
      go_c128 v;
      int s = go_eval_kernel(ev, GO_GREEN, radii[i], &v);
      if (s) return s;
      are += v.re * weights[i];
      aim += v.im * weights[i];
    }
    out->re = are;
    out->im = aim;
    return GO_OK;
  }
  uint32_t staged[kMaxBlock];
  for (size_t i = 0; i < count; ++i) {
    const double r = radii[i];
    if (r >= ev->hash.r_min && r <= ev->hash.r_max)
      staged[i] = ev->hash.buckets[bucket_of(&ev->hash, r)];
    else
      staged[i] = kScalar;
  }
  double re0 = 0.0, im0 = 0.0, re1 = 0.0, im1 = 0.0;
  for (size_t i = 0; i < count; ++i) {
    go_c128 v;
    if (staged[i] == kScalar) {
      int s = go_eval_kernel(ev, GO_GREEN, radii[i], &v);
      if (s) return s;
    } else {
      green_from_bucket(ev, staged[i], radii[i], &v);
    }
    if (i & 1) {
      re1 += v.re * weights[i];
      im1 += v.im * weights[i];
    } else {
      re0 += v.re * weights[i];
      im0 += v.im * weights[i];
    }
  }
  out->re = re0 + re1;
  out->im = im0 + im1;
  return GO_OK;
}

/* -------------------------------------------------------------- quadrature */

/* quadrature.hpp:35-76 */
int go_triangle_rule(int m, double* b0, double* b1, double* b2, double* w) {
  static const double r1[1][4] = {{1.0 / 3.0, 1.0 / 3.0, 1.0 / 3.0, 1.0}};
  static const double r3[3][4] = {{2.0 / 3.0, 1.0 / 6.0, 1.0 / 6.0, 1.0 / 3.0},
                                  {1.0 / 6.0, 2.0 / 3.0, 1.0 / 6.0, 1.0 / 3.0},
                                  {1.0 / 6.0, 1.0 / 6.0, 2.0 / 3.0, 1.0 / 3.0}};
  static const double r4[4][4] = {{1.0 / 3.0, 1.0 / 3.0, 1.0 / 3.0, -27.0 / 48.0},
                                  {0.6, 0.2, 0.2, 25.0 / 48.0},
                                  {0.2, 0.6, 0.2, 25.0 / 48.0},
                                  {0.2, 0.2, 0.6, 25.0 / 48.0}};
  static const double r6[6][4] = {
      {0.108103018168070, 0.445948490915965, 0.445948490915965, 0.223381589678011},
      {0.445948490915965, 0.108103018168070, 0.445948490915965, 0.223381589678011},
      {0.445948490915965, 0.445948490915965, 0.108103018168070, 0.223381589678011},
      {0.816847572980459, 0.091576213509771, 0.091576213509771, 0.109951743655322},
      {0.091576213509771, 0.816847572980459, 0.091576213509771, 0.109951743655322},
      {0.091576213509771, 0.091576213509771, 0.816847572980459, 0.109951743655322}};
  static const double r7[7][4] = {
      {1.0 / 3.0, 1.0 / 3.0, 1.0 / 3.0, 0.225},
      {0.059715871789770, 0.470142064105115, 0.470142064105115, 0.132394152788506},
      {0.470142064105115, 0.059715871789770, 0.470142064105115, 0.132394152788506},
      {0.470142064105115, 0.470142064105115, 0.059715871789770, 0.132394152788506},
      {0.797426985353087, 0.101286507323456, 0.101286507323456, 0.125939180544827},
      {0.101286507323456, 0.797426985353087, 0.101286507323456, 0.125939180544827},
      {0.101286507323456, 0.101286507323456, 0.797426985353087, 0.125939180544827}};
  const double(*rule)[4];
  switch (m) {
    case 1: rule = r1; break;
    case 3: rule = r3; break;
    case 4: rule = r4; break;
    case 6: rule = r6; break;
    case 7: rule = r7; break;
    default: return GO_INVALID;
  }
  for (int i = 0; i < m; ++i) {
    b0[i] = rule[i][0];
    b1[i] = rule[i][1];
    b2[i] = rule[i][2];
    w[i] = rule[i][3];
  }
  return GO_OK;
}

/* quadrature.hpp:85-110 */
int go_gauss_legendre_unit(int n, double* xs, double* ws) {
  if (n < 1) return GO_INVALID;
  const int half = (n + 1) / 2;
  for (int i = 0; i < half; ++i) {
    double x = cos(M_PI * ((double)i + 0.75) / ((double)n + 0.5));
    double dp = 0.0;
    for (int iter = 0; iter < 100; ++iter) {
      double p0 = 1.0, p1 = x;
      for (int j = 2; j <= n; ++j) {
        const double p2 = ((2.0 * j - 1.0) * x * p1 - (j - 1.0) * p0) / (double)j;
        p0 = p1;
        p1 = p2;
      }
      dp = n == 1 ? 1.0 : (double)n * (x * p1 - p0) / (x * x - 1.0);
      const double dx = p1 / dp;
      x -= dx;
      if (fabs(dx) < 1e-15) break;
    }
    const double w = 2.0 / ((1.0 - x * x) * dp * dp);
    xs[i] = (1.0 - x) / 2.0;
    ws[i] = w / 2.0;
    xs[n - 1 - i] = (1.0 + x) / 2.0;
    ws[n - 1 - i] = w / 2.0;
  }
  return GO_OK;
}

/* -------------------------------------------------------------------- mesh */

typedef struct { double x, y, z; } v3;
static v3 v3_add(v3 a, v3 b) { v3 r = {a.x + b.x, a.y + b.y, a.z + b.z}; return r; }
static v3 v3_sub(v3 a, v3 b) { v3 r = {a.x - b.x, a.y - b.y, a.z - b.z}; return r; }
static v3 v3_mul(v3 a, double s) { v3 r = {a.x * s, a.y * s, a.z * s}; return r; }
static double v3_dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static v3 v3_cross(v3 a, v3 b) {
  v3 r = {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
  return r;
}
static double v3_norm(v3 a) { return sqrt(v3_dot(a, a)); }
static v3 vert(const double* v, uint32_t i) { v3 r = {v[3 * i], v[3 * i + 1], v[3 * i + 2]}; return r; }

/* mesh.hpp:39-44 */
double go_triangle_area(const double* verts, const uint32_t* tri) {
  const v3 e1 = v3_sub(vert(verts, tri[1]), vert(verts, tri[0]));
  const v3 e2 = v3_sub(vert(verts, tri[2]), vert(verts, tri[0]));
  return 0.5 * v3_norm(v3_cross(e1, e2));
}

/* mesh.hpp:46-57 */
int go_mesh_validate(const double* verts, size_t nv, const uint32_t* tris, size_t nt) {
  for (size_t i = 0; i < nt; ++i) {
    for (int c = 0; c < 3; ++c)
      if (tris[3 * i + c] >= nv) return GO_INVALID;
    if (!(go_triangle_area(verts, tris + 3 * i) > 1e-12)) return GO_INVALID;
  }
  return GO_OK;
}

/* mesh.hpp:62-68 */
double go_max_vertex_distance(const double* verts, size_t nv) {
  double best = 0.0;
  for (size_t i = 0; i < nv; ++i)
    for (size_t j = i + 1; j < nv; ++j) {
      const double d = v3_norm(v3_sub(vert(verts, (uint32_t)i), vert(verts, (uint32_t)j)));
      best = best < d ? d : best;
    }
  return best;
}

void go_mesh_free(double* verts, uint32_t* tris) {
  free(verts);
  free(tris);
}

/* open-addressed edge -> midpoint map (mesh.hpp:286-296 uses std::map; only
   creation order matters for the output and both create on first sight) */
typedef struct { uint64_t* keys; uint32_t* vals; size_t cap; } edge_map;
static uint64_t mix64(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return x;
}

/* mesh.hpp:154-202 */
int go_sphere_mesh(double radius, int subdivisions, double** verts_out, size_t* nv_out,
                   uint32_t** tris_out, size_t* nt_out) {
  if (!(radius > 0.0)) return GO_INVALID;
  if (subdivisions < 0 || subdivisions > 6) return GO_INVALID;
  const double phi = (1.0 + sqrt(5.0)) / 2.0;
  const double base_v[12][3] = {{-1, phi, 0}, {1, phi, 0},   {-1, -phi, 0}, {1, -phi, 0},
                                {0, -1, phi}, {0, 1, phi},   {0, -1, -phi}, {0, 1, -phi},
                                {phi, 0, -1}, {phi, 0, 1},   {-phi, 0, -1}, {-phi, 0, 1}};
  const uint32_t base_t[20][3] = {{0, 11, 5}, {0, 5, 1},  {0, 1, 7},   {0, 7, 10}, {0, 10, 11},
                                  {1, 5, 9},  {5, 11, 4}, {11, 10, 2}, {10, 7, 6}, {7, 1, 8},
                                  {3, 9, 4},  {3, 4, 2},  {3, 2, 6},   {3, 6, 8},  {3, 8, 9},
                                  {4, 9, 5},  {2, 4, 11}, {6, 2, 10},  {8, 6, 7},  {9, 8, 1}};
  size_t nt = 20;
  for (int l = 0; l < subdivisions; ++l) nt *= 4;
  const size_t vcap = 10 * nt / 20 * 1 + 12 + nt; /* V = 10*4^L + 2 */
  double* v = (double*)malloc(3 * vcap * sizeof(double));
  uint32_t* t = (uint32_t*)malloc(3 * nt * sizeof(uint32_t));
  uint32_t* nxt = (uint32_t*)malloc(3 * nt * sizeof(uint32_t));
  memcpy(v, base_v, sizeof(base_v));
  memcpy(t, base_t, sizeof(base_t));
  size_t nv = 12, cur = 20;
  for (int level = 0; level < subdivisions; ++level) {
    edge_map em;
    em.cap = 1;
    while (em.cap < 4 * cur) em.cap <<= 1;
    em.keys = (uint64_t*)malloc(em.cap * sizeof(uint64_t));
    em.vals = (uint32_t*)malloc(em.cap * sizeof(uint32_t));
    memset(em.keys, 0xff, em.cap * sizeof(uint64_t));
    size_t nn = 0;
    for (size_t ti = 0; ti < cur; ++ti) {
      uint32_t mids[3];
      for (int e = 0; e < 3; ++e) {
        const uint32_t a = t[3 * ti + e], b = t[3 * ti + (e + 1) % 3];
        const uint64_t key = a < b ? ((uint64_t)a << 32) | b : ((uint64_t)b << 32) | a;
        size_t h = mix64(key) & (em.cap - 1);
        while (em.keys[h] != ~0ull && em.keys[h] != key) h = (h + 1) & (em.cap - 1);
        if (em.keys[h] == key) {
          mids[e] = em.vals[h];
        } else {
          const v3 m = v3_mul(v3_add(vert(v, a), vert(v, b)), 0.5);
          v[3 * nv] = m.x;
          v[3 * nv + 1] = m.y;
          v[3 * nv + 2] = m.z;
          em.keys[h] = key;
          em.vals[h] = (uint32_t)nv;
          mids[e] = (uint32_t)nv++;
        }
      }
      const uint32_t t0 = t[3 * ti], t1 = t[3 * ti + 1], t2 = t[3 * ti + 2];
      const uint32_t ab = mids[0], bc = mids[1], ca = mids[2];
      const uint32_t quad[4][3] = {{t0, ab, ca}, {t1, bc, ab}, {t2, ca, bc}, {ab, bc, ca}};
      memcpy(nxt + 3 * nn, quad, sizeof(quad));
      nn += 4;
    }
    free(em.keys);
    free(em.vals);
    uint32_t* sw = t; t = nxt; nxt = sw;
    cur = nn;
  }
  free(nxt);
  for (size_t i = 0; i < nv; ++i) {
    const v3 p = vert(v, (uint32_t)i);
    const v3 q = v3_mul(p, radius / v3_norm(p));
    v[3 * i] = q.x;
    v[3 * i + 1] = q.y;
    v[3 * i + 2] = q.z;
  }
  int s = go_mesh_validate(v, nv, t, cur);
  if (s) {
    free(v);
    free(t);
    return s;
  }
  *verts_out = v;
  *nv_out = nv;
  *tris_out = t;
  *nt_out = cur;
  return GO_OK;
}

/* workload jitter (not in the reference): splitmix64, per coordinate */
static uint64_t splitmix64(uint64_t* s) {
  uint64_t z = (*s += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

void go_jitter(double* verts, size_t nv, uint64_t seed, double amp) {
  uint64_t st = seed;
  for (size_t i = 0; i < 3 * nv; ++i) {
    const double u = (double)(splitmix64(&st) >> 11) * 0x1.0p-53;
    verts[i] += amp * (2.0 * u - 1.0);
  }
}

/* flat side x side plate on a cells x cells grid, two right triangles per cell */
int go_plate_mesh(double side, int cells, double** verts_out, size_t* nv_out, uint32_t** tris_out,
                  size_t* nt_out) {
  if (!(side > 0.0) || cells < 1) return GO_INVALID;
  const size_t c1 = (size_t)cells + 1;
  double* v = (double*)malloc(3 * c1 * c1 * sizeof(double));
  uint32_t* t = (uint32_t*)malloc(3 * 2 * (size_t)cells * cells * sizeof(uint32_t));
  for (size_t j = 0; j < c1; ++j)
    for (size_t i = 0; i < c1; ++i) {
      double* p = v + 3 * (j * c1 + i);
      p[0] = side * (double)i / (double)cells;
      p[1] = side * (double)j / (double)cells;
      p[2] = 0.0;
    }
  size_t nt = 0;
  for (size_t j = 0; j < (size_t)cells; ++j)
    for (size_t i = 0; i < (size_t)cells; ++i) {
      const uint32_t v00 = (uint32_t)(j * c1 + i), v10 = v00 + 1;
      const uint32_t v01 = (uint32_t)(v00 + c1), v11 = v01 + 1;
      uint32_t* a = t + 3 * nt++;
      a[0] = v00; a[1] = v10; a[2] = v11;
      uint32_t* b = t + 3 * nt++;
      b[0] = v00; b[1] = v11; b[2] = v01;
    }
  *verts_out = v;
  *nv_out = c1 * c1;
  *tris_out = t;
  *nt_out = nt;
  return go_mesh_validate(v, c1 * c1, t, nt);
}

/* ----------------------------------------------------------------- matfill */

/* matfill.hpp:116-128 */
int go_outer_points(const double* verts, size_t nv, const uint32_t* tris, size_t nt, int m,
                    double* x, double* y, double* z, double* w) {
  (void)nv;
  double b0[7], b1[7], b2[7], rw[7];
  int s = go_triangle_rule(m, b0, b1, b2, rw);
  if (s) return s;
  for (size_t i = 0; i < nt; ++i) {
    const uint32_t* tri = tris + 3 * i;
    const v3 a = vert(verts, tri[0]), b = vert(verts, tri[1]), c = vert(verts, tri[2]);
    const double area = go_triangle_area(verts, tri);
    for (int q = 0; q < m; ++q) {
      const v3 p = v3_add(v3_add(v3_mul(a, b0[q]), v3_mul(b, b1[q])), v3_mul(c, b2[q]));
      const size_t o = i * (size_t)m + (size_t)q;
      x[o] = p.x; y[o] = p.y; z[o] = p.z;
      w[o] = rw[q] * area;
    }
  }
  return GO_OK;
}

/* matfill.hpp:132-144 */
int go_inner_points(const double* verts, size_t nv, const uint32_t* tris, size_t nt, int n,
                    double* x, double* y, double* z, double* w) {
  (void)nv;
  if (n < 1) return GO_INVALID;
  double* gx = (double*)malloc((size_t)n * sizeof(double));
  double* gw = (double*)malloc((size_t)n * sizeof(double));
  go_gauss_legendre_unit(n, gx, gw);
  size_t o = 0;
  for (size_t i = 0; i < nt; ++i) {
    const uint32_t* tri = tris + 3 * i;
    for (int e = 0; e < 3; ++e) {
      const v3 a = vert(verts, tri[e]);
      const v3 b = vert(verts, tri[(e + 1) % 3]);
      const double len = v3_norm(v3_sub(a, b));
      for (int g = 0; g < n; ++g) {
        const v3 p = v3_add(a, v3_mul(v3_sub(b, a), gx[g]));
        x[o] = p.x; y[o] = p.y; z[o] = p.z;
        w[o] = gw[g] * len;
        ++o;
      }
    }
  }
  free(gx);
  free(gw);
  return GO_OK;
}

/* matfill.hpp:50-56 */
int go_predicted_calls(uint64_t N, uint64_t m, uint64_t n, uint64_t* out) {
  const unsigned __int128 wide = (unsigned __int128)3 * m * n * ((unsigned __int128)N * N);
  if (wide > (unsigned __int128)UINT64_MAX) return GO_OVERFLOW;
  *out = (uint64_t)wide;
  return GO_OK;
}

static int spec_validate(int m, int n) {
  if (m != 1 && m != 3 && m != 4 && m != 6 && m != 7) return GO_INVALID;
  if (n < 1) return GO_INVALID;
  return GO_OK;
}

typedef struct {
  const double *ox, *oy, *oz, *ow, *ix, *iy, *iz, *iw;
  size_t N, m, inner_per_tri;
  int mode, kind;
  double k, k_im;
  go_evaluator* ev;
  size_t p_begin, p_end, row_begin;
  go_c128* z;
  size_t ldz;
  uint64_t calls;
  int status;
} fill_job;

/* matfill.hpp:62-68 (AnalyticKernel::accumulate) */
static int analytic_accumulate(int kind, double k, double k_im, const double* r, const double* w,
                               size_t count, go_c128* out) {
  double are = 0.0, aim = 0.0;
  for (size_t i = 0; i < count; ++i) {
    go_c128 v;
    int s = go_eval_analytic_ck(kind, k, k_im, r[i], &v);
    if (s) return s;
    are += v.re * w[i];
    aim += v.im * w[i];
  }
  out->re = are;
  out->im = aim;
  return GO_OK;
}

/* matfill.hpp:78-86 (TableKernel::accumulate) */
static int table_accumulate(go_evaluator* ev, int kind, const double* r, const double* w,
                            size_t count, go_c128* out) {
  if (kind == GO_GREEN) return go_accumulate_green(ev, r, w, count, out);
  double are = 0.0, aim = 0.0;
  for (size_t i = 0; i < count; ++i) {
    go_c128 v;
    int s = go_eval_kernel(ev, kind, r[i], &v);
    if (s) return s;
    are += v.re * w[i];
    aim += v.im * w[i];
  }
  out->re = are;
  out->im = aim;
  return GO_OK;
}

/* matfill.hpp:169-203 (fill_rows) */
static void* fill_worker(void* arg) {
  fill_job* jb = (fill_job*)arg;
  const size_t block = jb->m * jb->inner_per_tri;
  double* br = (double*)malloc(block * sizeof(double));
  double* bw = (double*)malloc(block * sizeof(double));
  for (size_t p = jb->p_begin; p < jb->p_end && !jb->status; ++p) {
    const size_t ob = p * jb->m;
    for (size_t q = 0; q < jb->N; ++q) {
      if (p == q) continue;
      const size_t ib = q * jb->inner_per_tri;
      const double* ix = jb->ix + ib;
      const double* iy = jb->iy + ib;
      const double* iz = jb->iz + ib;
      const double* iw = jb->iw + ib;
      size_t idx = 0;
      for (size_t o = 0; o < jb->m; ++o) {
        const double ox = jb->ox[ob + o], oy = jb->oy[ob + o], oz = jb->oz[ob + o];
        const double ow = jb->ow[ob + o];
        for (size_t i = 0; i < jb->inner_per_tri; ++i) {
          const double dx = ox - ix[i];
          const double dy = oy - iy[i];
          const double dz = oz - iz[i];
          br[idx] = sqrt(dx * dx + dy * dy + dz * dz);
          bw[idx] = ow * iw[i];
          ++idx;
        }
      }
      go_c128* dst = jb->z + (p - jb->row_begin) * jb->ldz + q;
      int s = jb->mode == GO_MODE_DIRECT
                  ? analytic_accumulate(jb->kind, jb->k, jb->k_im, br, bw, block, dst)
                  : table_accumulate(jb->ev, jb->kind, br, bw, block, dst);
      if (s) {
        jb->status = s;
        break;
      }
      jb->calls += block;
    }
  }
  free(br);
  free(bw);
  return NULL;
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* matfill.hpp:144-228 */
int go_fill_rows(const double* verts, size_t nv, const uint32_t* tris, size_t nt, int m, int n,
                 int mode, double k, double k_im, go_evaluator* ev, int kind, int threads,
                 size_t row_begin, size_t row_end, go_c128* z, size_t ldz, go_fill_report* rep) {
  int s = spec_validate(m, n);
  if (s) return s;
  if ((s = go_mesh_validate(verts, nv, tris, nt))) return s;
  if (threads < 1) return GO_INVALID;
  if (mode == GO_MODE_TABLE && !ev) return GO_INVALID;
  if (row_end > nt || row_begin > row_end) return GO_INVALID;
  const size_t N = nt;
  const size_t inner_per_tri = (size_t)(3 * n);
  double* o4 = (double*)malloc(4 * N * (size_t)m * sizeof(double));
  double* i4 = (double*)malloc(4 * N * inner_per_tri * sizeof(double));
  const size_t no = N * (size_t)m, ni = N * inner_per_tri;
  go_outer_points(verts, nv, tris, nt, m, o4, o4 + no, o4 + 2 * no, o4 + 3 * no);
  go_inner_points(verts, nv, tris, nt, n, i4, i4 + ni, i4 + 2 * ni, i4 + 3 * ni);

  go_fill_report report;
  memset(&report, 0, sizeof(report));
  report.N = N;
  report.m = m;
  report.n = n;
  if ((s = go_predicted_calls(N, (uint64_t)m, (uint64_t)n, &report.predicted_calls))) {
    free(o4);
    free(i4);
    return s;
  }
  for (size_t p = row_begin; p < row_end; ++p) {
    go_c128* row = z + (p - row_begin) * ldz;
    row[p].re = 0.0; /* self-pairs stay zero (matfill.hpp:178) */
    row[p].im = 0.0;
  }
  const uint64_t fb_before = ev ? go_evaluator_fallbacks(ev) : 0;
  const size_t rows = row_end - row_begin;
  fill_job* jobs = (fill_job*)calloc((size_t)threads, sizeof(fill_job));
  pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  const size_t chunk = (rows + (size_t)threads - 1) / (size_t)threads;
  int launched = 0;
  const double t0 = now_s();
  for (int wi = 0; wi < threads; ++wi) {
    const size_t b = row_begin + (size_t)wi * chunk;
    const size_t e = b + chunk < row_end ? b + chunk : row_end;
    if (b >= e) break;
    fill_job* jb = &jobs[wi];
    jb->ox = o4; jb->oy = o4 + no; jb->oz = o4 + 2 * no; jb->ow = o4 + 3 * no;
    jb->ix = i4; jb->iy = i4 + ni; jb->iz = i4 + 2 * ni; jb->iw = i4 + 3 * ni;
    jb->N = N; jb->m = (size_t)m; jb->inner_per_tri = inner_per_tri;
    jb->mode = mode; jb->kind = kind; jb->k = k; jb->k_im = k_im; jb->ev = ev;
    jb->p_begin = b; jb->p_end = e; jb->row_begin = row_begin; jb->z = z; jb->ldz = ldz;
    if (threads == 1) {
      fill_worker(jb);
    } else {
      pthread_create(&tids[wi], NULL, fill_worker, jb);
    }
    ++launched;
  }
  if (threads > 1)
    for (int wi = 0; wi < launched; ++wi) pthread_join(tids[wi], NULL);
  const double t1 = now_s();
  report.wall_time_s = t1 - t0;
  for (int wi = 0; wi < launched; ++wi) {
    report.actual_calls += jobs[wi].calls;
    if (jobs[wi].status && !s) s = jobs[wi].status;
  }
  report.fallback_calls = ev ? go_evaluator_fallbacks(ev) - fb_before : 0;
  if (rep) *rep = report;
  free(jobs);
  free(tids);
  free(o4);
  free(i4);
  return s;
}

/* matfill.hpp:237-254 */
int go_compare_fills(const go_c128* test, const go_c128* ref, size_t n, double* max_rel_re,
                     double* max_rel_im) {
  double mre = 0.0, mim = 0.0;
  for (size_t p = 0; p < n; ++p)
    for (size_t q = 0; q < n; ++q) {
      if (p == q) continue;
      const go_c128 a = ref[p * n + q], b = test[p * n + q];
      if (a.re != 0.0) {
        const double e = fabs(b.re - a.re) / fabs(a.re);
        mre = mre < e ? e : mre;
      }
      if (a.im != 0.0) {
        const double e = fabs(b.im - a.im) / fabs(a.im);
        mim = mim < e ? e : mim;
      }
    }
  *max_rel_re = mre;
  *max_rel_im = mim;
  return GO_OK;
}

/* ------------------------------------------------------------------ bounds */

static double factorial(int n) {
  double f = 1.0;
  for (int i = 2; i <= n; ++i) f *= (double)i;
  return f;
}

/* bounds.hpp:37-51 */
int go_derivative_bound(int kind, double k, double r_low, int order, double* out) {
  if (order < 1) return GO_INVALID;
  if (!(k >= 0.0)) return GO_INVALID;
  if (kind == GO_EXP) {
    *out = pow(k, order);
    return GO_OK;
  }
  if (!(r_low > 0.0)) return GO_DOMAIN;
  double sum = 0.0, binom = 1.0;
  for (int p = 0; p <= order; ++p) {
    sum += binom * pow(k, p) * factorial(order - p) / pow(r_low, order - p + 1);
    binom = binom * (double)(order - p) / (double)(p + 1);
  }
  *out = sum;
  return GO_OK;
}

/* bounds.hpp:55-58 */
int go_linear_bound(double h, int kind, double k, double r_low, double* out) {
  if (!(h > 0.0)) return GO_INVALID;
  double d;
  int s = go_derivative_bound(kind, k, r_low, 2, &d);
  if (s) return s;
  *out = h * h * d / 8.0;
  return GO_OK;
}

/* bounds.hpp:63-77 */
int go_lagrange_bound(const double* stencil, size_t n, double r, int kind, double k, double* out) {
  if (n < 2) return GO_INVALID;
  for (size_t i = 1; i < n; ++i)
    if (!(stencil[i] > stencil[i - 1])) return GO_INVALID;
  if (!(r >= stencil[0] && r <= stencil[n - 1])) return GO_DOMAIN;
  double prod = 1.0;
  for (size_t i = 0; i < n; ++i) prod *= fabs(r - stencil[i]);
  double d;
  int s = go_derivative_bound(kind, k, stencil[0], (int)n, &d);
  if (s) return s;
  *out = prod * d / factorial((int)n);
  return GO_OK;
}

/* bounds.hpp:97-111.  For complex k the bound uses |k|. */
int go_pointwise_bound(const go_evaluator* ev, int kind, int method, double r, double* out) {
  const go_plan* plan = &ev->plan;
  size_t j;
  int s = go_locate(&ev->hash, plan, r, &j);
  if (s) return s;
  const double kb = ev->k_im == 0.0 ? ev->k : hypot(ev->k, ev->k_im);
  if (method == 0) {
    const double h = plan->absc[j + 1] - plan->absc[j];
    return go_linear_bound(h, kind, kb, plan->absc[j], out);
  }
  const int degree = ev->degree;
  const size_t width = (size_t)degree + 1;
  const size_t back_shift = (size_t)((degree - 1) / 2);
  size_t start = j > back_shift ? j - back_shift : 0;
  if (start + width > plan->n) start = plan->n - width;
  return go_lagrange_bound(plan->absc + start, width, r, kind, kb, out);
}

/* one observation row of the parity tolerance */
static int entry_bound_row(const double* o4, const double* i4, size_t N, size_t m, size_t ipt,
                           const go_evaluator* ev, double k_abs, double rnd, size_t p,
                           double* row) {
  const size_t no = N * m, ni = N * ipt;
  int s = 0;
  row[p] = 0.0;
  for (size_t q = 0; q < N && !s; ++q) {
    if (q == p) continue;
    double acc = 0.0;
    for (size_t o = 0; o < m; ++o) {
      const size_t oi = p * m + o;
      for (size_t i = 0; i < ipt; ++i) {
        const size_t ii = q * ipt + i;
        const double dx = o4[oi] - i4[ii];
        const double dy = o4[no + oi] - i4[ni + ii];
        const double dz = o4[2 * no + oi] - i4[2 * ni + ii];
        const double r = sqrt(dx * dx + dy * dy + dz * dz);
        double pw = 0.0;
        if (ev && r >= ev->hash.r_min && r <= ev->hash.r_max) {
          s = go_pointwise_bound(ev, GO_GREEN, 1, r, &pw);
          if (s) break;
        }
        acc += fabs(o4[3 * no + oi] * i4[3 * ni + ii]) * (pw + rnd * (1.0 + k_abs * r) / r);
      }
    }
    row[q] = acc;
  }
  return s;
}

typedef struct {
  const double *o4, *i4;
  size_t N, m, ipt;
  const go_evaluator* ev;
  double k_abs, rnd;
  const uint64_t* rows;
  size_t rb, re;
  double* bound;
  size_t ldb;
  int status;
} bound_job;

static void* bound_worker(void* arg) {
  bound_job* j = (bound_job*)arg;
  for (size_t r = j->rb; r < j->re && !j->status; ++r)
    j->status = entry_bound_row(j->o4, j->i4, j->N, j->m, j->ipt, j->ev, j->k_abs, j->rnd,
                                (size_t)j->rows[r], j->bound + r * j->ldb);
  return NULL;
}

int go_entry_bounds_rows(const double* verts, size_t nv, const uint32_t* tris, size_t nt, int m,
                         int n, const go_evaluator* ev, double k_abs, double ulps,
                         const uint64_t* rows, size_t nrows, int threads, double* bound,
                         size_t ldb) {
  int s = spec_validate(m, n);
  if (s) return s;
  if (threads < 1) return GO_INVALID;
  for (size_t r = 0; r < nrows; ++r)
    if (rows[r] >= nt) return GO_INVALID;
  const size_t N = nt, ipt = (size_t)(3 * n);
  const size_t no = N * (size_t)m, ni = N * ipt;
  double* o4 = (double*)malloc(4 * no * sizeof(double));
  double* i4 = (double*)malloc(4 * ni * sizeof(double));
  go_outer_points(verts, nv, tris, nt, m, o4, o4 + no, o4 + 2 * no, o4 + 3 * no);
  go_inner_points(verts, nv, tris, nt, n, i4, i4 + ni, i4 + 2 * ni, i4 + 3 * ni);
  bound_job* jobs = (bound_job*)calloc((size_t)threads, sizeof(bound_job));
  pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  const size_t chunk = (nrows + (size_t)threads - 1) / (size_t)threads;
  int launched = 0;
  for (int w = 0; w < threads; ++w) {
    const size_t b = (size_t)w * chunk, e = b + chunk < nrows ? b + chunk : nrows;
    if (b >= e) break;
    bound_job* j = &jobs[w];
    j->o4 = o4; j->i4 = i4; j->N = N; j->m = (size_t)m; j->ipt = ipt; j->ev = ev;
    j->k_abs = k_abs; j->rnd = ulps * 0x1.0p-53; j->rows = rows; j->rb = b; j->re = e;
    j->bound = bound; j->ldb = ldb;
    if (threads == 1) bound_worker(j);
    else pthread_create(&tids[w], NULL, bound_worker, j);
    ++launched;
  }
  if (threads > 1)
    for (int w = 0; w < launched; ++w) pthread_join(tids[w], NULL);
  for (int w = 0; w < launched; ++w)
    if (jobs[w].status && !s) s = jobs[w].status;
  free(jobs);
  free(tids);
  free(o4);
  free(i4);
  return s;
}

int go_entry_bounds(const double* verts, size_t nv, const uint32_t* tris, size_t nt, int m, int n,
                    const go_evaluator* ev, double k_abs, double ulps, size_t row_begin,
                    size_t row_end, double* bound, size_t ldb) {
  if (row_end > nt || row_begin > row_end) return GO_INVALID;
  const size_t nrows = row_end - row_begin;
  uint64_t* rows = (uint64_t*)malloc((nrows ? nrows : 1) * sizeof(uint64_t));
  for (size_t r = 0; r < nrows; ++r) rows[r] = row_begin + r;
  const int s = go_entry_bounds_rows(verts, nv, tris, nt, m, n, ev, k_abs, ulps, rows, nrows, 1,
                                     bound, ldb);
  free(rows);
  return s;
}

int go_distance_range(const double* verts, size_t nv, const uint32_t* tris, size_t nt, int m,
                      int n, size_t row_begin, size_t row_end, double* r_min, double* r_max) {
  int s = spec_validate(m, n);
  if (s) return s;
  if (nt < 2 || row_end > nt || row_begin >= row_end) return GO_INVALID;
  const size_t N = nt, ipt = (size_t)(3 * n);
  const size_t no = N * (size_t)m, ni = N * ipt;
  double* o4 = (double*)malloc(4 * no * sizeof(double));
  double* i4 = (double*)malloc(4 * ni * sizeof(double));
  go_outer_points(verts, nv, tris, nt, m, o4, o4 + no, o4 + 2 * no, o4 + 3 * no);
  go_inner_points(verts, nv, tris, nt, n, i4, i4 + ni, i4 + 2 * ni, i4 + 3 * ni);
  double lo = INFINITY, hi = 0.0;
  for (size_t p = row_begin; p < row_end; ++p)
    for (size_t q = 0; q < N; ++q) {
      if (q == p) continue;
      for (size_t o = 0; o < (size_t)m; ++o) {
        const size_t oi = p * (size_t)m + o;
        for (size_t i = 0; i < ipt; ++i) {
          const size_t ii = q * ipt + i;
          const double dx = o4[oi] - i4[ii];
          const double dy = o4[no + oi] - i4[ni + ii];
          const double dz = o4[2 * no + oi] - i4[2 * ni + ii];
          const double r = sqrt(dx * dx + dy * dy + dz * dz);
          lo = r < lo ? r : lo;
          hi = r > hi ? r : hi;
        }
      }
    }
  free(o4);
  free(i4);
  *r_min = lo;
  *r_max = hi;
  return GO_OK;
}
