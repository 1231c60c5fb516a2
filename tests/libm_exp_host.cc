// Host build of csrc/pnms_libm.cuh for tests/test_libm_exp.py: y[i] = glibc_exp(x[i]).
#include "../paper_2502_00535_b200/csrc/pnms_libm.cuh"

extern "C" void libm_exp_restated(const double* x, double* y, long long n) {
  for (long long i = 0; i < n; ++i) y[i] = pnms::glibc_exp(x[i]);
}
