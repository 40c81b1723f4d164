/* CPU oracle for the logistic-regression potential and gradient.
 *
 * TEST INFRASTRUCTURE ONLY (tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py): never linked into the product.
 *
 * Restates turnstile/kernels.py:90-123 (numba path): row loop in order,
 * eta accumulated left to right, stable log1p(exp) and sigmoid by sign
 * branch, gradient updated row by row.  Compiled with -ffp-contract=off so
 * the sequential entry points round exactly like the numba loops.
 *
 * ts_oracle_logistic_seq  - bit-for-bit restatement (one thread)
 * ts_oracle_logistic_omp  - same per-row math, rows split over OpenMP
 *                           threads (partials combined in thread order);
 *                           the multi-core CPU baseline of bench.py
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline double row_eta(const double* xr, const double* theta, int p) {
  double eta = theta[p];
  for (int j = 0; j < p; ++j) eta += xr[j] * theta[j];
  return eta;
}

/* kernels.py:90-104 */
double ts_oracle_logistic_potential_seq(const double* x, const double* y, int64_t n, int p, const double* theta) {
  double acc = 0.5 * theta[p] * theta[p];
  for (int j = 0; j < p; ++j) acc += 0.5 * theta[j] * theta[j];
  for (int64_t i = 0; i < n; ++i) {
    const double eta = row_eta(x + i * p, theta, p);
    const double m = eta > 0.0 ? eta : 0.0;
    const double l = m + log1p(exp(-fabs(eta)));
    acc -= y[i] * eta - l;
  }
  return acc;
}

/* kernels.py:106-123 */
void ts_oracle_logistic_gradient_seq(const double* x, const double* y, int64_t n, int p, const double* theta,
                                     double* out) {
  for (int j = 0; j <= p; ++j) out[j] = theta[j];
  for (int64_t i = 0; i < n; ++i) {
    const double* xr = x + i * p;
    const double eta = row_eta(xr, theta, p);
    double sig;
    if (eta >= 0.0) {
      sig = 1.0 / (1.0 + exp(-eta));
    } else {
      const double e = exp(eta);
      sig = e / (1.0 + e);
    }
    const double resid = y[i] - sig;
    for (int j = 0; j < p; ++j) out[j] -= resid * xr[j];
    out[p] -= resid;
  }
}

/* Fused one-pass variant over fp32 rows, OpenMP over row blocks.
 * out[0] = U, out[1..p+1] = gradient.  Returns threads used. */
int ts_oracle_logistic_omp(const float* x, const uint8_t* y, int64_t n, int p, const double* theta, double* out) {
  int nt = 1;
#ifdef _OPENMP
  nt = omp_get_max_threads();
#endif
  double* part = (double*)calloc((size_t)nt * (p + 2), sizeof(double));
#pragma omp parallel num_threads(nt)
  {
    int t = 0;
#ifdef _OPENMP
    t = omp_get_thread_num();
#endif
    double* acc = part + (size_t)t * (p + 2);
    const int64_t lo = n * t / nt, hi = n * (t + 1) / nt;
    for (int64_t i = lo; i < hi; ++i) {
      const float* xr = x + i * p;
      double eta = theta[p];
      for (int j = 0; j < p; ++j) eta += (double)xr[j] * theta[j];
      const double e = exp(-fabs(eta));
      const double l = (eta > 0.0 ? eta : 0.0) + log1p(e);
      const double sig = (eta >= 0.0 ? 1.0 : e) / (1.0 + e);
      const double yi = (double)y[i];
      const double resid = yi - sig;
      acc[p + 1] += yi * eta - l;
      for (int j = 0; j < p; ++j) acc[j] += resid * (double)xr[j];
      acc[p] += resid;
    }
  }
  double prior = 0.5 * theta[p] * theta[p];
  for (int j = 0; j < p; ++j) prior += 0.5 * theta[j] * theta[j];
  double ll = 0.0;
  for (int j = 0; j <= p; ++j) out[1 + j] = theta[j];
  for (int t = 0; t < nt; ++t) {
    const double* acc = part + (size_t)t * (p + 2);
    ll += acc[p + 1];
    for (int j = 0; j <= p; ++j) out[1 + j] -= acc[j];
  }
  out[0] = prior - ll;
  free(part);
  return nt;
}
