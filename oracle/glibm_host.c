/* glibm_host.c — TEST INFRASTRUCTURE ONLY. The glibc libm restatement of
 * include/odegpu/device/glibm.h compiled for the host (-ffp-contract=off),
 * next to the live glibc functions, so tests/test_glibm_cpu.py can check
 * the restatement bit for bit against the libm the reference links. */
#define _GNU_SOURCE
#include <math.h>

#include "odegpu/device/glibm.h"

#define BATCH1(name, expr)                                                   \
    void name(long n, const double* x, double* out) {                        \
        for (long i = 0; i < n; ++i) out[i] = (expr);                        \
    }
BATCH1(glm_cos_batch, glm_cos(x[i]))
BATCH1(libm_cos_batch, cos(x[i]))

void glm_sincos_batch(long n, const double* x, double* s, double* c) {
    for (long i = 0; i < n; ++i) glm_sincos(x[i], s + i, c + i);
}
void libm_sincos_batch(long n, const double* x, double* s, double* c) {
    for (long i = 0; i < n; ++i) sincos(x[i], s + i, c + i);
}
void glm_pow_batch(long n, const double* x, const double* y, double* out) {
    for (long i = 0; i < n; ++i) out[i] = glm_pow(x[i], y[i]);
}
void libm_pow_batch(long n, const double* x, const double* y, double* out) {
    for (long i = 0; i < n; ++i) out[i] = pow(x[i], y[i]);
}
int glm_trig_in_range_host(double x) { return glm_trig_in_range(x); }
