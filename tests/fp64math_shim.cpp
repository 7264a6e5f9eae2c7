// Host build of csrc/nx_fp64math.h for tests/test_fp64math.py (same code the
// composite kernel runs on the device).
#include "../paper_2512_13796_b200/csrc/nx_fp64math.h"

extern "C" void fm_exp(const double* x, double* y, long n) {
    for (long i = 0; i < n; ++i) y[i] = nx::fm::exp64(x[i]);
}
extern "C" void fm_log(const double* x, double* y, long n) {
    for (long i = 0; i < n; ++i) y[i] = nx::fm::log64(x[i]);
}
extern "C" void fm_eval_kernel(const double* u, const double* v, const double* o, const double* gx,
                               const double* gy, double* y, long n) {
    for (long i = 0; i < n; ++i) y[i] = nx::fm::eval_kernel(u[i], v[i], o[i], gx[i], gy[i]);
}
