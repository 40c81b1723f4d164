// Device target models: potential U(q) and gradient dU/dq.
//
// Small models (evaluated inside one team, no communication beyond the team
// sum) restate turnstile/kernels.py with the numba loop order:
//   std_normal  kernels.py:44-53    U = sum 0.5 q_i q_i,             g = q
//   gaussian    kernels.py:55-67    U = sum 0.5 q_i q_i inv_var_i,   g = q inv_var
//   funnel      kernels.py:69-88    Neal funnel, q[0] = log scale
//   eight_schools (new built-in, SURVEY.md 8(d) cfg 3; no reference kernel)
// The data-parallel model, logistic regression (kernels.py:90-123), lives in
// ts_logistic.cuh: one fused pass over X computes U and the gradient.
#pragma once
#include "ts_team.cuh"
#include "ts_libm.cuh"

namespace ts {

enum ModelKind : int {
  kStdNormal = 0,
  kGaussian = 1,
  kLogistic = 2,
  kFunnel = 3,
  kEightSchools = 4,
};

struct SmallModel {
  int kind;
  int dim;
  const double* params;  // gaussian: inv_var[dim]; eight_schools: y[J], sigma[J]
};

// Evaluate U at vector qid of `S`, writing the gradient into vector gid.
// Callers sync the team before (q visible) and after (g visible).
template <class Team>
__device__ double small_model_eval(const Team& T, const SmallModel& m, const VecStore& S, int qid, int gid) {
  const int D = m.dim;
  const double* q = S.v(qid);
  double* g = S.v(gid);
  const int64_t ds = S.dstride;
  switch (m.kind) {
    case kStdNormal: {
      double acc = 0.0;
      for (int d = T.rank(); d < D; d += T.size()) {
        double x = q[d * ds];
        acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(0.5, x), x));
        g[d * ds] = x;
      }
      return T.sum(acc);
    }
    case kGaussian: {
      const double* iv = m.params;
      double acc = 0.0;
      for (int d = T.rank(); d < D; d += T.size()) {
        double x = q[d * ds];
        acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(__dmul_rn(0.5, x), x), iv[d]));
        g[d * ds] = __dmul_rn(x, iv[d]);
      }
      return T.sum(acc);
    }
    case kFunnel: {
      // U = v*v/18 + 0.5*(D-1)*v + 0.5*exp(-v)*ssq ; ssq = sum_{i>=1} q_i^2
      const double v = q[0];
      const double inv_scale = x_exp<Team::kExactMath>(-v);
      double ssq = 0.0;
      for (int d = T.rank(); d < D; d += T.size()) {
        if (d == 0) continue;
        double x = q[d * ds];
        ssq = __dadd_rn(ssq, __dmul_rn(x, x));
        g[d * ds] = __dmul_rn(inv_scale, x);
      }
      ssq = T.sum(ssq);
      const double half_n1 = __dmul_rn(0.5, (double)(D - 1));
      if (T.rank() == 0)
        g[0] = __dsub_rn(__dadd_rn(__ddiv_rn(v, 9.0), half_n1), __dmul_rn(__dmul_rn(0.5, inv_scale), ssq));
      return __dadd_rn(__dadd_rn(__ddiv_rn(__dmul_rn(v, v), 18.0), __dmul_rn(half_n1, v)),
                       __dmul_rn(__dmul_rn(0.5, inv_scale), ssq));
    }
    case kEightSchools: {
      // q = (mu, log tau, theta_1..J) non-centred; y, sigma in params.
      // U = mu^2/50 + log1p((tau/5)^2) - log tau + sum_j [0.5 th_j^2 + 0.5 z_j^2],
      // z_j = (y_j - mu - tau th_j) / sigma_j.   Oracle: oracle/turnstile_oracle.py
      const int J = D - 2;
      const double* y = m.params;
      const double* sg = m.params + J;
      const double mu = q[0], lt = q[ds];
      const double tau = x_exp<Team::kExactMath>(lt);
      const double s = __ddiv_rn(tau, 5.0);
      const double s2 = __dmul_rn(s, s);
      double ulik = 0.0, smu = 0.0, slt = 0.0;
      for (int d = T.rank(); d < D; d += T.size()) {
        if (d < 2) continue;
        const int j = d - 2;
        const double th = q[d * ds];
        const double z = __ddiv_rn(__dsub_rn(__dsub_rn(y[j], mu), __dmul_rn(tau, th)), sg[j]);
        const double zs = __ddiv_rn(z, sg[j]);
        ulik = __dadd_rn(ulik, __dmul_rn(__dmul_rn(0.5, th), th));
        ulik = __dadd_rn(ulik, __dmul_rn(__dmul_rn(0.5, z), z));
        smu = __dadd_rn(smu, zs);
        slt = __dadd_rn(slt, __dmul_rn(__dmul_rn(zs, tau), th));
        g[d * ds] = __dsub_rn(th, __dmul_rn(zs, tau));
      }
      ulik = T.sum(ulik);
      smu = T.sum(smu);
      slt = T.sum(slt);
      if (T.rank() == 0) {
        g[0] = __dsub_rn(__ddiv_rn(mu, 25.0), smu);
        g[ds] = __dsub_rn(__dsub_rn(__ddiv_rn(__dmul_rn(2.0, s2), __dadd_rn(1.0, s2)), 1.0), slt);
      }
      const double prior = __dsub_rn(__dadd_rn(__ddiv_rn(__dmul_rn(mu, mu), 50.0), x_log1p<Team::kExactMath>(s2)), lt);
      return __dadd_rn(prior, ulik);
    }
    default:
      return __longlong_as_double(0x7ff8000000000000LL);
  }
}

}  // namespace ts
