// Host build of csrc/ts_libm.cuh for tests/test_libm.py (g++ -ffp-contract=off):
// evaluates the restated glibc functions over arrays.
#include "../paper_1912_11554_b200/csrc/ts_libm.cuh"
extern "C" void probe_exp(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = ts::lm_exp(x[i]); }
extern "C" void probe_log1p(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = ts::lm_log1p(x[i]); }
extern "C" void probe_log(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = ts::lm_log(x[i]); }
