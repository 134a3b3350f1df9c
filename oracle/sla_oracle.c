/*
 * sla_oracle.c -- CPU restatement of the SLA reference algorithm.
 *
 * TEST INFRASTRUCTURE ONLY: the checker for the CUDA path (see sla_oracle.h).
 * Citations are relative to /root/reference/proj/core.  Compile with
 * -ffp-contract=off so every a*b+c rounds twice, as in the reference build.
 */
#include "sla_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define ORC_LSE_SENTINEL (-1e300) /* forward.hpp:18-24 (f64) */

/* ----------------------------------------------------------------------------------- */
/* rng.hpp:22-64 SplitMix64                                                            */
/* ----------------------------------------------------------------------------------- */
uint64_t orc_rng_next(uint64_t* state) {
  *state += 0x9E3779B97F4A7C15ULL;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

double orc_rng_uniform(uint64_t* state) {
  return (double)((orc_rng_next(state) >> 11) + 1) * 0x1.0p-53;
}

static double rng_gauss1(uint64_t* state) {
  const double u1 = orc_rng_uniform(state);
  const double u2 = orc_rng_uniform(state);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793238462643383279502884 * u2);
}

void orc_rng_gaussian(uint64_t* state, double* out, size_t count, double stddev) {
  for (size_t i = 0; i < count; ++i) out[i] = stddev * rng_gauss1(state);
}

void orc_rng_uniform_range(uint64_t* state, double* out, size_t count, double lo, double hi) {
  for (size_t i = 0; i < count; ++i) out[i] = lo + (hi - lo) * (orc_rng_uniform(state) - 0x1.0p-53);
}

/* tests/test_support.hpp:99-116 */
void orc_random_mask(uint64_t* state, size_t t_m, size_t t_n, double p_critical,
                     double p_marginal, int allow_empty_critical, int8_t* labels) {
  for (size_t i = 0; i < t_m; ++i) {
    int has_critical = 0;
    for (size_t j = 0; j < t_n; ++j) {
      const double u = orc_rng_uniform(state);
      int8_t lab = u < p_critical ? 1 : (u < p_critical + p_marginal ? 0 : -1);
      labels[i * t_n + j] = lab;
      has_critical |= lab == 1;
    }
    if (!has_critical && !allow_empty_critical) labels[i * t_n + orc_rng_next(state) % t_n] = 1;
  }
}

/* ----------------------------------------------------------------------------------- */
/* layout.cpp:8-26, config.cpp:7-19                                                    */
/* ----------------------------------------------------------------------------------- */
int orc_validate(size_t n, size_t d, size_t b_q, size_t b_kv, double k_h, double k_l, char* err,
                 size_t err_len) {
  char buf[160];
  buf[0] = 0;
  if (n == 0 || d == 0 || b_q == 0 || b_kv == 0)
    snprintf(buf, sizeof buf, "make_block_layout: all sizes must be positive");
  else if (n % b_q != 0)
    snprintf(buf, sizeof buf, "make_block_layout: b_q=%zu does not divide N=%zu", b_q, n);
  else if (n % b_kv != 0)
    snprintf(buf, sizeof buf, "make_block_layout: b_kv=%zu does not divide N=%zu", b_kv, n);
  else if (!(k_h > 0.0 && k_h <= 100.0))
    snprintf(buf, sizeof buf, "config: k_h must be in (0, 100]");
  else if (!(k_l >= 0.0 && k_l < 100.0))
    snprintf(buf, sizeof buf, "config: k_l must be in [0, 100)");
  else if (k_h + k_l > 100.0)
    snprintf(buf, sizeof buf, "config: k_h + k_l must be <= 100");
  if (buf[0]) {
    if (err && err_len) {
      strncpy(err, buf, err_len - 1);
      err[err_len - 1] = 0;
    }
    return 2;
  }
  return 0;
}

/* ----------------------------------------------------------------------------------- */
/* mask.cpp:40-55 pool_mean: ascending row sum, then one division                        */
/* ----------------------------------------------------------------------------------- */
int orc_pool_mean(const double* x, size_t rows, size_t cols, size_t b, double* out) {
  if (b == 0 || rows % b != 0) return 2;
  const size_t groups = rows / b;
  memset(out, 0, sizeof(double) * groups * cols);
  for (size_t g = 0; g < groups; ++g) {
    double* dst = out + g * cols;
    for (size_t r = 0; r < b; ++r) {
      const double* src = x + (g * b + r) * cols;
      for (size_t c = 0; c < cols; ++c) dst[c] += src[c];
    }
    for (size_t c = 0; c < cols; ++c) dst[c] /= (double)b;
  }
  return 0;
}

/* mask.cpp:57-64 + mat.hpp:83-97 (matmul_nt, ascending-k dot) + scale */
int orc_scores(const double* q, const double* k, size_t n, size_t d, size_t b_q, size_t b_kv,
               double* s) {
  if (b_q == 0 || b_kv == 0 || n % b_q || n % b_kv) return 2;
  const size_t t_m = n / b_q, t_n = n / b_kv;
  double* pq = (double*)malloc(sizeof(double) * t_m * d);
  double* pk = (double*)malloc(sizeof(double) * t_n * d);
  orc_pool_mean(q, n, d, b_q, pq);
  orc_pool_mean(k, n, d, b_kv, pk);
  const double inv_sqrt_d = 1.0 / sqrt((double)d);
  for (size_t i = 0; i < t_m; ++i)
    for (size_t j = 0; j < t_n; ++j) {
      double acc = 0;
      for (size_t c = 0; c < d; ++c) acc += pq[i * d + c] * pk[j * d + c];
      s[i * t_n + j] = acc * inv_sqrt_d;
    }
  free(pq);
  free(pk);
  return 0;
}

/* mask.cpp:57-81: max-shifted row softmax of the pooled scores, all in f64 */
int orc_predict(const double* q, const double* k, size_t n, size_t d, size_t b_q, size_t b_kv,
                double* p_c) {
  int rc = orc_scores(q, k, n, d, b_q, b_kv, p_c);
  if (rc) return rc;
  const size_t t_m = n / b_q, t_n = n / b_kv;
  for (size_t i = 0; i < t_m; ++i) {
    double* row = p_c + i * t_n;
    double m = row[0];
    for (size_t j = 1; j < t_n; ++j) m = row[j] > m ? row[j] : m;
    double sum = 0;
    for (size_t j = 0; j < t_n; ++j) {
      row[j] = exp(row[j] - m);
      sum += row[j];
    }
    for (size_t j = 0; j < t_n; ++j) row[j] /= sum;
  }
  return 0;
}

/* Ragged-N extension (SLA_B200_FLAG_RAGGED; the reference has no counterpart -- it rejects
 * N % b != 0, layout.cpp:12-17): T = ceil(n / b) blocks, the last one averaging its r valid
 * rows; otherwise mask.cpp:40-81 operation for operation (ascending row sums, ascending-k dot,
 * max-shifted softmax with the ascending normaliser). */
int orc_predict_ragged(const double* q, const double* k, size_t n, size_t d, size_t b, double* p_c) {
  if (b == 0 || n == 0) return 2;
  const size_t t = (n + b - 1) / b;
  double* pq = (double*)calloc(t * d, sizeof(double));
  double* pk = (double*)calloc(t * d, sizeof(double));
  for (size_t g = 0; g < t; ++g) {
    const size_t rows = (g + 1) * b <= n ? b : n - g * b;
    for (size_t r = 0; r < rows; ++r)
      for (size_t c = 0; c < d; ++c) {
        pq[g * d + c] += q[(g * b + r) * d + c];
        pk[g * d + c] += k[(g * b + r) * d + c];
      }
    for (size_t c = 0; c < d; ++c) {
      pq[g * d + c] /= (double)rows;
      pk[g * d + c] /= (double)rows;
    }
  }
  const double inv_sqrt_d = 1.0 / sqrt((double)d);
  for (size_t i = 0; i < t; ++i) {
    double* row = p_c + i * t;
    for (size_t j = 0; j < t; ++j) {
      double acc = 0;
      for (size_t c = 0; c < d; ++c) acc += pq[i * d + c] * pk[j * d + c];
      row[j] = acc * inv_sqrt_d;
    }
    double m = row[0];
    for (size_t j = 1; j < t; ++j) m = row[j] > m ? row[j] : m;
    double sum = 0;
    for (size_t j = 0; j < t; ++j) {
      row[j] = exp(row[j] - m);
      sum += row[j];
    }
    for (size_t j = 0; j < t; ++j) row[j] /= sum;
  }
  free(pq);
  free(pk);
  return 0;
}

/* mask.cpp:85-101 */
static size_t round_half_up(double x) { return (size_t)floor(x + 0.5); }

void orc_counts(size_t t_n, double k_h, double k_l, size_t* n1, size_t* n_neg) {
  size_t a = round_half_up(k_h * (double)t_n / 100.0);
  if (a < 1) a = 1;
  if (a > t_n) a = t_n;
  size_t b = round_half_up(k_l * (double)t_n / 100.0);
  if (b > t_n - a) b = t_n - a;
  *n1 = a;
  *n_neg = b;
}

/* order = (value descending, column ascending): the total order std::stable_sort with
 * `row[a] > row[b]` produces from the iota start (mask.cpp:105-113). */
static const double* g_sort_row;
static int cmp_desc_stable(const void* pa, const void* pb) {
  const uint32_t a = *(const uint32_t*)pa, b = *(const uint32_t*)pb;
  const double va = g_sort_row[a], vb = g_sort_row[b];
  if (va > vb) return -1;
  if (vb > va) return 1;
  return a < b ? -1 : (a > b ? 1 : 0);
}

/* mask.cpp:91-119 */
int orc_classify(const double* p_c, size_t t_m, size_t t_n, double k_h, double k_l,
                 int8_t* labels) {
  if (k_h + k_l > 100.0) return 2;
  size_t n1, n_neg;
  orc_counts(t_n, k_h, k_l, &n1, &n_neg);
  uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * t_n);
  memset(labels, 0, t_m * t_n);
  for (size_t i = 0; i < t_m; ++i) {
    for (size_t j = 0; j < t_n; ++j) order[j] = (uint32_t)j;
    g_sort_row = p_c + i * t_n;
    qsort(order, t_n, sizeof(uint32_t), cmp_desc_stable);
    for (size_t r = 0; r < n1; ++r) labels[i * t_n + order[r]] = 1;
    for (size_t r = 0; r < n_neg; ++r) labels[i * t_n + order[t_n - 1 - r]] = -1;
  }
  free(order);
  return 0;
}

/* ----------------------------------------------------------------------------------- */
/* feature_map.cpp:10-73                                                                 */
/* ----------------------------------------------------------------------------------- */
static void softmax_row(double* row, size_t d) {
  double m = row[0];
  for (size_t c = 1; c < d; ++c) m = row[c] > m ? row[c] : m;
  double sum = 0;
  for (size_t c = 0; c < d; ++c) {
    row[c] = exp(row[c] - m);
    sum += row[c];
  }
  for (size_t c = 0; c < d; ++c) row[c] /= sum;
}

void orc_phi(const double* x, size_t rows, size_t d, int phi, double* out) {
  const size_t total = rows * d;
  if (out != x) memcpy(out, x, sizeof(double) * total);
  switch (phi) {
    case 0:
      for (size_t i = 0; i < total; ++i) out[i] = out[i] >= 0.0 ? out[i] + 1.0 : exp(out[i]);
      break;
    case 1:
      for (size_t i = 0; i < total; ++i) out[i] = out[i] > 0.0 ? out[i] : 0.0;
      break;
    default:
      for (size_t r = 0; r < rows; ++r) softmax_row(out + r * d, d);
      break;
  }
}

void orc_phi_vjp(const double* x, size_t rows, size_t d, int phi, const double* d_phi,
                 double* out) {
  const size_t total = rows * d;
  switch (phi) {
    case 0:
      for (size_t i = 0; i < total; ++i) out[i] = (x[i] >= 0.0 ? 1.0 : exp(x[i])) * d_phi[i];
      break;
    case 1:
      for (size_t i = 0; i < total; ++i) out[i] = x[i] > 0.0 ? d_phi[i] : 0.0;
      break;
    default: {
      double* s = (double*)malloc(sizeof(double) * d);
      for (size_t r = 0; r < rows; ++r) {
        memcpy(s, x + r * d, sizeof(double) * d);
        softmax_row(s, d);
        double dot = 0;
        for (size_t c = 0; c < d; ++c) dot += s[c] * d_phi[r * d + c];
        for (size_t c = 0; c < d; ++c) out[r * d + c] = s[c] * (d_phi[r * d + c] - dot);
      }
      free(s);
    }
  }
}

/* ----------------------------------------------------------------------------------- */
/* summaries.cpp:17-42 and aggregation.cpp:40-56                                          */
/* ----------------------------------------------------------------------------------- */
void orc_summaries(const double* k_feat, const double* v, size_t n, size_t d, size_t b_kv,
                   double* h, double* z) {
  const size_t t_n = n / b_kv;
  memset(h, 0, sizeof(double) * t_n * d * d);
  memset(z, 0, sizeof(double) * t_n * d);
  for (size_t j = 0; j < t_n; ++j) {
    double* hj = h + j * d * d;
    double* zj = z + j * d;
    for (size_t t = j * b_kv; t < (j + 1) * b_kv; ++t) {
      const double* kf = k_feat + t * d;
      const double* vt = v + t * d;
      for (size_t a = 0; a < d; ++a) {
        zj[a] += kf[a];
        const double ka = kf[a];
        if (ka == 0.0) continue;
        double* ha = hj + a * d;
        for (size_t b = 0; b < d; ++b) ha[b] += ka * vt[b];
      }
    }
  }
}

void orc_aggregate_direct(const double* h, const double* z, size_t d, const uint32_t* idx,
                          size_t count, double* h_out, double* z_out) {
  memset(h_out, 0, sizeof(double) * d * d);
  memset(z_out, 0, sizeof(double) * d);
  for (size_t p = 0; p < count; ++p) {
    const double* hj = h + (size_t)idx[p] * d * d;
    const double* zj = z + (size_t)idx[p] * d;
    if (p == 0) {
      memcpy(h_out, hj, sizeof(double) * d * d);
      memcpy(z_out, zj, sizeof(double) * d);
    } else {
      for (size_t e = 0; e < d * d; ++e) h_out[e] += hj[e];
      for (size_t c = 0; c < d; ++c) z_out[c] += zj[c];
    }
  }
}

/* ----------------------------------------------------------------------------------- */
/* block_ops.hpp:12-26 score tile                                                         */
/* ----------------------------------------------------------------------------------- */
static void score_block(const double* q, const double* k, size_t d, size_t b_q, size_t b_kv,
                        size_t bi, size_t bj, double* out) {
  const double inv_sqrt_d = 1.0 / sqrt((double)d);
  for (size_t r = 0; r < b_q; ++r) {
    const double* qr = q + (bi * b_q + r) * d;
    for (size_t c = 0; c < b_kv; ++c) {
      const double* kc = k + (bj * b_kv + c) * d;
      double acc = 0;
      for (size_t e = 0; e < d; ++e) acc += qr[e] * kc[e];
      out[r * b_kv + c] = acc * inv_sqrt_d;
    }
  }
}

static int find_non_finite(const double* a, size_t rows, size_t cols, size_t* r, size_t* c) {
  for (size_t i = 0; i < rows; ++i)
    for (size_t j = 0; j < cols; ++j)
      if (!isfinite(a[i * cols + j])) {
        *r = i;
        *c = j;
        return 1;
      }
  return 0;
}

/* forward.cpp:29-79: streaming restricted softmax over an (ascending) column list */
static void sparse_block_row_forward(const double* q, const double* k, const double* v,
                                     size_t d, size_t b_q, size_t b_kv, size_t block_row,
                                     const uint32_t* cols, size_t n_cols, double* out,
                                     double* lse) {
  const size_t r0 = block_row * b_q;
  double* m_run = (double*)malloc(sizeof(double) * b_q);
  double* l_run = (double*)calloc(b_q, sizeof(double));
  double* acc = (double*)calloc(b_q * d, sizeof(double));
  double* s = (double*)malloc(sizeof(double) * b_q * b_kv);
  for (size_t r = 0; r < b_q; ++r) m_run[r] = -INFINITY;
  for (size_t p = 0; p < n_cols; ++p) {
    const size_t j = cols[p];
    score_block(q, k, d, b_q, b_kv, block_row, j, s);
    const size_t c0 = j * b_kv;
    for (size_t r = 0; r < b_q; ++r) {
      const double* sr = s + r * b_kv;
      double row_max = sr[0];
      for (size_t c = 1; c < b_kv; ++c) row_max = sr[c] > row_max ? sr[c] : row_max;
      const double m_new = m_run[r] > row_max ? m_run[r] : row_max;
      const double alpha = exp(m_run[r] - m_new);
      double p_sum = 0;
      double* ar = acc + r * d;
      for (size_t e = 0; e < d; ++e) ar[e] *= alpha;
      for (size_t c = 0; c < b_kv; ++c) {
        const double pv = exp(sr[c] - m_new);
        p_sum += pv;
        const double* vc = v + (c0 + c) * d;
        for (size_t e = 0; e < d; ++e) ar[e] += pv * vc[e];
      }
      l_run[r] = alpha * l_run[r] + p_sum;
      m_run[r] = m_new;
    }
  }
  for (size_t r = 0; r < b_q; ++r) {
    double* orow = out + (r0 + r) * d;
    if (l_run[r] == 0.0) {
      for (size_t e = 0; e < d; ++e) orow[e] = 0.0;
      lse[r0 + r] = ORC_LSE_SENTINEL;
    } else {
      const double* ar = acc + r * d;
      for (size_t e = 0; e < d; ++e) orow[e] = ar[e] / l_run[r];
      lse[r0 + r] = m_run[r] + log(l_run[r]);
    }
  }
  free(m_run);
  free(l_run);
  free(acc);
  free(s);
}

/* list of columns with the given label in row i, ascending (mask.cpp:121-153) */
static size_t row_list(const int8_t* labels, size_t t_n, size_t i, int lab, uint32_t* out) {
  size_t c = 0;
  for (size_t j = 0; j < t_n; ++j)
    if (labels[i * t_n + j] == lab) out[c++] = (uint32_t)j;
  return c;
}

/* forward.cpp:81-172 (sla_forward_with_mask) */
int orc_forward(const double* q, const double* k, const double* v, const int8_t* labels,
                size_t n, size_t d, size_t b_q, size_t b_kv, int phi,
                const int32_t* block_rows, size_t n_block_rows, double* o_s, double* o_l,
                double* lse, double* row_h, double* row_z) {
  if (!b_q || !b_kv || n % b_q || n % b_kv) return 2;
  size_t br, bc;
  if (find_non_finite(q, n, d, &br, &bc) || find_non_finite(k, n, d, &br, &bc) ||
      find_non_finite(v, n, d, &br, &bc))
    return 2;
  const size_t t_m = n / b_q, t_n = n / b_kv;
  for (size_t e = 0; e < t_m * t_n; ++e)
    if (labels[e] < -1 || labels[e] > 1) return 2;

  double* q_feat = (double*)malloc(sizeof(double) * n * d);
  double* k_feat = (double*)malloc(sizeof(double) * n * d);
  orc_phi(q, n, d, phi, q_feat);
  orc_phi(k, n, d, phi, k_feat);
  double* h = (double*)malloc(sizeof(double) * t_n * d * d);
  double* z = (double*)malloc(sizeof(double) * t_n * d);
  orc_summaries(k_feat, v, n, d, b_kv, h, z);

  uint32_t* crit = (uint32_t*)malloc(sizeof(uint32_t) * t_n);
  uint32_t* marg = (uint32_t*)malloc(sizeof(uint32_t) * t_n);
  double* hi = (double*)malloc(sizeof(double) * d * d);
  double* zi = (double*)malloc(sizeof(double) * d);
  const size_t rows = block_rows ? n_block_rows : t_m;
  int rc = 0;
  for (size_t ri = 0; ri < rows; ++ri) {
    const size_t i = block_rows ? (size_t)block_rows[ri] : ri;
    const size_t nc = row_list(labels, t_n, i, 1, crit);
    const size_t nm = row_list(labels, t_n, i, 0, marg);
    sparse_block_row_forward(q, k, v, d, b_q, b_kv, i, crit, nc, o_s, lse);
    orc_aggregate_direct(h, z, d, marg, nm, hi, zi);
    if (row_h) memcpy(row_h + i * d * d, hi, sizeof(double) * d * d);
    if (row_z) memcpy(row_z + i * d, zi, sizeof(double) * d);
    for (size_t r = i * b_q; r < (i + 1) * b_q; ++r) {
      double* orow = o_l + r * d;
      for (size_t b = 0; b < d; ++b) orow[b] = 0.0;
    }
    if (nm) {
      for (size_t r = i * b_q; r < (i + 1) * b_q; ++r) {
        const double* qf = q_feat + r * d;
        double den = 0;
        for (size_t a = 0; a < d; ++a) den += qf[a] * zi[a];
        if (den == 0.0) continue;
        double* orow = o_l + r * d;
        for (size_t a = 0; a < d; ++a) {
          const double qa = qf[a];
          if (qa == 0.0) continue;
          const double* ha = hi + a * d;
          for (size_t b = 0; b < d; ++b) orow[b] += qa * ha[b];
        }
        for (size_t b = 0; b < d; ++b) orow[b] /= den;
      }
    }
    for (size_t r = i * b_q; r < (i + 1) * b_q; ++r)
      for (size_t b = 0; b < d; ++b)
        if (!isfinite(o_s[r * d + b]) || !isfinite(o_l[r * d + b])) rc = 1;
  }
  free(q_feat);
  free(k_feat);
  free(h);
  free(z);
  free(crit);
  free(marg);
  free(hi);
  free(zi);
  return rc;
}

/* forward.cpp:187-195: O = O^l W + O^s (mat.hpp:65-81 matmul order) */
void orc_combine(const double* o_s, const double* o_l, const double* w, size_t n, size_t d,
                 double* o) {
  for (size_t i = 0; i < n; ++i) {
    double* oi = o + i * d;
    for (size_t j = 0; j < d; ++j) oi[j] = 0.0;
    for (size_t a = 0; a < d; ++a) {
      const double x = o_l[i * d + a];
      if (x == 0.0) continue;
      for (size_t j = 0; j < d; ++j) oi[j] += x * w[a * d + j];
    }
    for (size_t j = 0; j < d; ++j) oi[j] += o_s[i * d + j];
  }
}

/* ----------------------------------------------------------------------------------- */
/* backward.cpp:12-22                                                                      */
/* ----------------------------------------------------------------------------------- */
static void matmul_tn_acc(const double* a, const double* b, size_t rows, size_t d, double* c) {
  memset(c, 0, sizeof(double) * d * d);
  for (size_t r = 0; r < rows; ++r) {
    const double* ak = a + r * d;
    const double* bk = b + r * d;
    for (size_t i = 0; i < d; ++i) {
      const double aki = ak[i];
      if (aki == 0.0) continue;
      for (size_t j = 0; j < d; ++j) c[i * d + j] += aki * bk[j];
    }
  }
}

void orc_proj_backward(const double* d_out, const double* o_l, const double* w, size_t n,
                       size_t d, double* d_out_s, double* d_out_l, double* dw) {
  memcpy(d_out_s, d_out, sizeof(double) * n * d);
  for (size_t i = 0; i < n; ++i)
    for (size_t j = 0; j < d; ++j) {
      double acc = 0;
      for (size_t e = 0; e < d; ++e) acc += d_out[i * d + e] * w[j * d + e];
      d_out_l[i * d + j] = acc;
    }
  matmul_tn_acc(o_l, d_out, n, d, dw);
}

/* backward.cpp:24-216 */
int orc_backward(const double* q, const double* k, const double* v, const int8_t* labels,
                 const double* o_s, const double* o_l, const double* lse,
                 const double* row_h, const double* row_z, const double* d_out_s,
                 const double* d_out_l, size_t n, size_t d, size_t b_q, size_t b_kv, int phi,
                 double* dq, double* dk, double* dv, double* dq_feat, double* dk_feat,
                 double* dproj, double* dq_total, double* dk_total) {
  if (!b_q || !b_kv || n % b_q || n % b_kv) return 2;
  const size_t t_m = n / b_q, t_n = n / b_kv;
  memset(dq, 0, sizeof(double) * n * d);
  memset(dk, 0, sizeof(double) * n * d);
  memset(dv, 0, sizeof(double) * n * d);
  memset(dq_feat, 0, sizeof(double) * n * d);
  memset(dk_feat, 0, sizeof(double) * n * d);
  matmul_tn_acc(o_l, d_out_s, n, d, dproj);

  double* q_feat = (double*)malloc(sizeof(double) * n * d);
  double* k_feat = (double*)malloc(sizeof(double) * n * d);
  orc_phi(q, n, d, phi, q_feat);
  orc_phi(k, n, d, phi, k_feat);

  double* ds_row = (double*)malloc(sizeof(double) * n);
  double* dl_row = (double*)malloc(sizeof(double) * n);
  for (size_t r = 0; r < n; ++r) {
    double a = 0, b = 0;
    for (size_t c = 0; c < d; ++c) {
      a += d_out_s[r * d + c] * o_s[r * d + c];
      b += d_out_l[r * d + c] * o_l[r * d + c];
    }
    ds_row[r] = a;
    dl_row[r] = b;
  }
  const double inv_sqrt_d = 1.0 / sqrt((double)d);
  double* gh = (double*)calloc(t_m * d * d, sizeof(double));
  double* gz = (double*)calloc(t_m * d, sizeof(double));
  uint32_t* list = (uint32_t*)malloc(sizeof(uint32_t) * (t_m > t_n ? t_m : t_n));
  double* s = (double*)malloc(sizeof(double) * b_q * b_kv);

  /* block-row phase (backward.cpp:68-120) */
  for (size_t i = 0; i < t_m; ++i) {
    const size_t nm = row_list(labels, t_n, i, 0, list);
    if (nm) {
      double* dh_i = gh + i * d * d;
      double* dz_i = gz + i * d;
      const double* h_i = row_h + i * d * d;
      const double* z_i = row_z + i * d;
      for (size_t r = i * b_q; r < (i + 1) * b_q; ++r) {
        const double* qf = q_feat + r * d;
        double den = 0;
        for (size_t a = 0; a < d; ++a) den += qf[a] * z_i[a];
        if (den == 0.0) continue;
        const double* go = d_out_l + r * d;
        const double dl = dl_row[r];
        for (size_t a = 0; a < d; ++a) {
          const double qa = qf[a] / den;
          if (qa != 0.0) {
            double* dha = dh_i + a * d;
            for (size_t b = 0; b < d; ++b) dha[b] += qa * go[b];
            dz_i[a] -= qa * dl;
          }
          const double* ha = h_i + a * d;
          double acc = 0;
          for (size_t b = 0; b < d; ++b) acc += go[b] * ha[b];
          dq_feat[r * d + a] = (acc - dl * z_i[a]) / den;
        }
      }
    }
    const size_t nc = row_list(labels, t_n, i, 1, list);
    for (size_t p = 0; p < nc; ++p) {
      const size_t j = list[p];
      score_block(q, k, d, b_q, b_kv, i, j, s);
      const size_t c0 = j * b_kv;
      for (size_t r = 0; r < b_q; ++r) {
        const size_t row = i * b_q + r;
        const double* go = d_out_s + row * d;
        const double ds_base = ds_row[row];
        double* dq_row = dq + row * d;
        for (size_t c = 0; c < b_kv; ++c) {
          const double pv = exp(s[r * b_kv + c] - lse[row]);
          const double* vc = v + (c0 + c) * d;
          double dp = 0;
          for (size_t e = 0; e < d; ++e) dp += go[e] * vc[e];
          const double ds = pv * (dp - ds_base) * inv_sqrt_d;
          const double* kc = k + (c0 + c) * d;
          for (size_t e = 0; e < d; ++e) dq_row[e] += ds * kc[e];
        }
      }
    }
  }

  /* block-column phase (backward.cpp:142-199) */
  double* dh_agg = (double*)malloc(sizeof(double) * d * d);
  double* dz_agg = (double*)malloc(sizeof(double) * d);
  double* dv_lin = (double*)malloc(sizeof(double) * d);
  for (size_t j = 0; j < t_n; ++j) {
    const size_t c0 = j * b_kv;
    for (size_t i = 0; i < t_m; ++i) {
      if (labels[i * t_n + j] != 1) continue;
      score_block(q, k, d, b_q, b_kv, i, j, s);
      for (size_t r = 0; r < b_q; ++r) {
        const size_t row = i * b_q + r;
        const double* go = d_out_s + row * d;
        const double ds_base = ds_row[row];
        const double* qr = q + row * d;
        for (size_t c = 0; c < b_kv; ++c) {
          const double pv = exp(s[r * b_kv + c] - lse[row]);
          double* dv_row = dv + (c0 + c) * d;
          for (size_t e = 0; e < d; ++e) dv_row[e] += pv * go[e];
          const double* vc = v + (c0 + c) * d;
          double dp = 0;
          for (size_t e = 0; e < d; ++e) dp += go[e] * vc[e];
          const double ds = pv * (dp - ds_base) * inv_sqrt_d;
          double* dk_row = dk + (c0 + c) * d;
          for (size_t e = 0; e < d; ++e) dk_row[e] += ds * qr[e];
        }
      }
    }
    size_t nr = 0;
    for (size_t i = 0; i < t_m; ++i)
      if (labels[i * t_n + j] == 0) list[nr++] = (uint32_t)i;
    if (nr) {
      orc_aggregate_direct(gh, gz, d, list, nr, dh_agg, dz_agg);
      for (size_t t = j * b_kv; t < (j + 1) * b_kv; ++t) {
        const double* vt = v + t * d;
        const double* kf = k_feat + t * d;
        double* dkf = dk_feat + t * d;
        for (size_t b = 0; b < d; ++b) dv_lin[b] = 0.0;
        for (size_t a = 0; a < d; ++a) {
          const double* dha = dh_agg + a * d;
          double acc = 0;
          for (size_t b = 0; b < d; ++b) acc += vt[b] * dha[b];
          dkf[a] += acc + dz_agg[a];
          const double ka = kf[a];
          if (ka != 0.0)
            for (size_t b = 0; b < d; ++b) dv_lin[b] += ka * dha[b];
        }
        double* dvt = dv + t * d;
        for (size_t b = 0; b < d; ++b) dvt[b] += dv_lin[b];
      }
    }
  }

  /* backward.cpp:211-214 */
  orc_phi_vjp(q, n, d, phi, dq_feat, dq_total);
  for (size_t e = 0; e < n * d; ++e) dq_total[e] += dq[e];
  orc_phi_vjp(k, n, d, phi, dk_feat, dk_total);
  for (size_t e = 0; e < n * d; ++e) dk_total[e] += dk[e];

  free(q_feat);
  free(k_feat);
  free(ds_row);
  free(dl_row);
  free(gh);
  free(gz);
  free(list);
  free(s);
  free(dh_agg);
  free(dz_agg);
  free(dv_lin);
  return 0;
}

/* flops.cpp:7-33 */
void orc_flops(size_t n, size_t d, size_t b_q, size_t b_kv, const int8_t* labels,
               uint64_t out[6]) {
  const size_t t_m = n / b_q, t_n = n / b_kv;
  uint64_t crit = 0, marg_total = 0, covered = 0;
  for (size_t i = 0; i < t_m; ++i) {
    uint64_t m = 0;
    for (size_t j = 0; j < t_n; ++j) {
      crit += labels[i * t_n + j] == 1;
      m += labels[i * t_n + j] == 0;
    }
    marg_total += m;
    if (m) covered += b_q;
  }
  out[0] = 4ull * n * n * d;
  out[1] = 4ull * b_q * b_kv * d * crit;
  out[2] = 2ull * covered * d * d + (marg_total ? (uint64_t)n * d : 0);
  out[3] = 2ull * n * d * d;
  out[4] = 2ull * n * d + 2ull * t_m * t_n * d;
  out[5] = out[1] + out[2] + out[3] + out[4];
}
