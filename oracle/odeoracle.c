#define _POSIX_C_SOURCE 200809L
/*
 * odeoracle.c — TEST INFRASTRUCTURE ONLY (the CPU checker; never shipped,
 * never on the product path). Plain-C single-threaded restatement of the
 * reference's hot path. Every function cites the reference lines it follows
 * (paths relative to /root/reference/proj/include/odensemble/).
 *
 * Built with -O2 -ffp-contract=off so every expression rounds exactly like
 * the reference's -O3 / no -march build; with the same glibc libm the
 * results are bitwise identical to oracle/_ref/libodref.so — that is the pin
 * (tests/test_oracle_pinning.py) together with tests/golden/.
 */
#include "odeoracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define MAXN 4
#define MAXE 2
#define MAXA 4
#define MAXP 13

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* odo_last_error(void) { return g_err; }

/* std::max / std::min / std::clamp semantics (NaN behaviour included). */
static double smax(double a, double b) { return (a < b) ? b : a; }
static double smin(double a, double b) { return (b < a) ? b : a; }
static double sclamp(double v, double lo, double hi) { return (v < lo) ? lo : (hi < v) ? hi : v; }

/* ------------------------------------------------------------------ models */

typedef struct {
    int id;
    const double* k;
    int n, np, ne, na;
    int dir[MAXE];
    double tol[MAXE];
    int64_t stop[MAXE];
    int64_t max_zone;
} Model;

static const double kTwoPi = 2.0 * 3.14159265358979323846; /* 2*std::numbers::pi_v<double> */

static int model_init(Model* md, const odegpu_model* m) {
    memset(md, 0, sizeof *md);
    md->id = m->id;
    md->k = m->consts;
    md->max_zone = 50; /* system.hpp:42 default */
    switch (m->id) {
    case ODEGPU_MODEL_DUFFING: md->n = 2; md->np = 4; break;
    case ODEGPU_MODEL_DUFFING_MAX_ACCESSORY: md->n = 2; md->np = 4; md->na = 2; break;
    case ODEGPU_MODEL_DUFFING_MAX_EVENT: /* duffing.hpp:128-132 */
        md->n = 2; md->np = 4; md->ne = 1; md->na = 2;
        md->dir[0] = -1; md->tol[0] = m->consts[0]; md->stop[0] = (int64_t)m->consts[1];
        break;
    case ODEGPU_MODEL_DUFFING_MAXMIN: md->n = 2; md->np = 4; md->na = 4; break;
    case ODEGPU_MODEL_KELLER_MIKSIS: md->n = 2; md->np = 13; break;
    case ODEGPU_MODEL_BUBBLE_COLLAPSE: /* keller_miksis.hpp:316-320 */
        md->n = 2; md->np = 13; md->ne = 1; md->na = 4;
        md->dir[0] = -1; md->tol[0] = m->consts[0]; md->stop[0] = 1;
        break;
    case ODEGPU_MODEL_VALVE: /* valve.hpp:423-430 */
        md->n = 3; md->np = 5; md->ne = 2; md->na = 2;
        md->dir[0] = -1; md->dir[1] = -1; md->tol[0] = md->tol[1] = m->consts[0];
        md->stop[0] = 1; md->stop[1] = 0; md->max_zone = 50;
        break;
    case ODEGPU_MODEL_DUFFING_LYAPUNOV: md->n = 4; md->np = 4; md->na = 1; break;
    case ODEGPU_MODEL_CONSTANT:
    case ODEGPU_MODEL_CUBIC_TIME:
    case ODEGPU_MODEL_EXPONENTIAL:
    case ODEGPU_MODEL_UNIT_SLOPE:
    case ODEGPU_MODEL_BLOWUP: md->n = 1; break;
    case ODEGPU_MODEL_COUNTING: md->n = 2; md->np = 4; md->na = 3; break;
    case ODEGPU_MODEL_RAMP:
        md->n = 1; md->ne = 1;
        md->dir[0] = (int)m->consts[2]; md->stop[0] = (int64_t)m->consts[3];
        md->tol[0] = m->consts[4]; md->max_zone = (int64_t)m->consts[5];
        break;
    case ODEGPU_MODEL_DECAY:
        md->n = 1; md->ne = 1; md->dir[0] = 0; md->tol[0] = 1e-6; md->stop[0] = 0;
        break;
    case ODEGPU_MODEL_SEAT_CONTACT:
        md->n = 3; md->np = 5; md->ne = 1; md->dir[0] = -1; md->tol[0] = 1e-6; md->stop[0] = 1;
        break;
    case ODEGPU_MODEL_HARMONIC: md->n = 2; break;
    default: return fail(ODEGPU_ERR_UNSUPPORTED, "odo: unknown model");
    }
    return 0;
}

/* duffing.hpp:37-42 */
static void duffing_rhs(double t, const double* y, const double* p, double* dy) {
    const double k = p[0], B = p[1], delta = p[2], omega = p[3];
    dy[0] = y[1];
    dy[1] = delta * y[0] - y[0] * y[0] * y[0] - k * y[1] + B * cos(omega * t);
}

/* duffing.hpp:47-57 */
static void duffing_lyapunov_rhs(double t, const double* y, const double* p, double* dy) {
    duffing_rhs(t, y, p, dy);
    const double k = p[0], delta = p[2];
    const double g1 = delta - 3.0 * y[0] * y[0];
    const double g2 = -k;
    const double s = sin(y[3]);
    const double c = cos(y[3]);
    dy[2] = y[2] * ((1.0 + g1) * s * c + g2 * s * s);
    dy[3] = -s * s + (g1 * c + g2 * s) * c;
}

/* keller_miksis.hpp:82-103 */
static void keller_miksis_rhs(double tau, const double* y, const double* c, double* dy) {
    const double y1 = y[0], y2 = y[1];
    if (!(y1 > 0)) {
        dy[0] = NAN;
        dy[1] = NAN;
        return;
    }
    const double arg1 = kTwoPi * tau;
    const double arg2 = kTwoPi * c[11] * tau + c[12];
    const double numerator =
        (c[0] + c[1] * y2) * pow(1.0 / y1, c[10]) - c[2] * (1.0 + c[9] * y2) - c[3] / y1 -
        c[4] * y2 / y1 - (1.0 - c[9] * y2 / 3.0) * 1.5 * y2 * y2 -
        (c[5] * sin(arg1) + c[6] * sin(arg2)) * (1.0 + c[9] * y2) -
        y1 * (c[7] * cos(arg1) + c[8] * cos(arg2));
    const double denominator = y1 - c[9] * y1 * y2 + c[4] * c[9];
    dy[0] = y2;
    dy[1] = numerator / denominator;
}

/* valve.hpp:41-46 */
static void valve_rhs(const double* y, const double* p, double* dy) {
    const double kappa = p[0], delta = p[1], beta = p[2], q = p[3];
    dy[0] = y[1];
    dy[1] = -kappa * y[1] - (y[0] + delta) + y[2];
    dy[2] = beta * (q - y[0] * sqrt(y[2]));
}

static void ode_rhs(const Model* m, double t, const double* y, const double* p, double* dy) {
    switch (m->id) {
    case ODEGPU_MODEL_DUFFING:
    case ODEGPU_MODEL_DUFFING_MAX_ACCESSORY:
    case ODEGPU_MODEL_DUFFING_MAX_EVENT:
    case ODEGPU_MODEL_DUFFING_MAXMIN:
    case ODEGPU_MODEL_COUNTING: duffing_rhs(t, y, p, dy); break;
    case ODEGPU_MODEL_DUFFING_LYAPUNOV: duffing_lyapunov_rhs(t, y, p, dy); break;
    case ODEGPU_MODEL_KELLER_MIKSIS:
    case ODEGPU_MODEL_BUBBLE_COLLAPSE: keller_miksis_rhs(t, y, p, dy); break;
    case ODEGPU_MODEL_VALVE:
    case ODEGPU_MODEL_SEAT_CONTACT: valve_rhs(y, p, dy); break;
    case ODEGPU_MODEL_CONSTANT: dy[0] = m->k[0]; break;
    case ODEGPU_MODEL_CUBIC_TIME: dy[0] = t * t * t; break;
    case ODEGPU_MODEL_EXPONENTIAL: dy[0] = y[0]; break;
    case ODEGPU_MODEL_UNIT_SLOPE: dy[0] = 1.0; break;
    case ODEGPU_MODEL_RAMP: dy[0] = m->k[0]; break;
    case ODEGPU_MODEL_DECAY: dy[0] = -y[0]; break;
    case ODEGPU_MODEL_HARMONIC: dy[0] = y[1]; dy[1] = -y[0]; break;
    case ODEGPU_MODEL_BLOWUP: dy[0] = NAN; break;
    default: break;
    }
}

static void event_values(const Model* m, double t, const double* y, const double* p, double* f) {
    (void)t;
    (void)p;
    switch (m->id) {
    case ODEGPU_MODEL_DUFFING_MAX_EVENT: /* duffing.hpp:136-138 */
    case ODEGPU_MODEL_BUBBLE_COLLAPSE: f[0] = y[1]; break; /* keller_miksis.hpp:324-326 */
    case ODEGPU_MODEL_VALVE: f[0] = y[1]; f[1] = y[0]; break; /* valve.hpp:434-437 */
    case ODEGPU_MODEL_RAMP: f[0] = y[0] - m->k[1]; break;
    case ODEGPU_MODEL_DECAY:
    case ODEGPU_MODEL_SEAT_CONTACT: f[0] = y[0]; break;
    default: break;
    }
}

static void event_action(const Model* m, int64_t ei, int64_t ec, double t, double* y, const double* p) {
    (void)ec;
    (void)t;
    if (m->id == ODEGPU_MODEL_VALVE && ei == 1) { /* valve.hpp:52-58 */
        y[0] = 0.0;
        y[1] = -p[4] * y[1];
    }
}

static void ordinary_accessory(const Model* m, double t, const double* y, const double* p, double* acc) {
    (void)p;
    switch (m->id) {
    case ODEGPU_MODEL_DUFFING_MAX_ACCESSORY: /* duffing.hpp:107-113 */
        if (y[0] > acc[0]) { acc[0] = y[0]; acc[1] = t; }
        break;
    case ODEGPU_MODEL_DUFFING_MAXMIN:
        if (y[0] > acc[0]) { acc[0] = y[0]; acc[1] = t; }
        if (y[0] < acc[2]) { acc[2] = y[0]; acc[3] = t; }
        break;
    case ODEGPU_MODEL_BUBBLE_COLLAPSE: /* keller_miksis.hpp:334-340 */
        if (y[0] < acc[3]) { acc[3] = y[0]; acc[2] = t; }
        break;
    case ODEGPU_MODEL_VALVE: /* valve.hpp:447-451 */
        acc[0] = smax(acc[0], y[0]);
        acc[1] = smin(acc[1], y[0]);
        break;
    case ODEGPU_MODEL_COUNTING: acc[2] += 1; break;
    default: break;
    }
}

static void event_accessory(const Model* m, int64_t ei, int64_t ec, double t, const double* y, const double* p,
                            double* acc) {
    (void)ec;
    (void)p;
    if (m->id == ODEGPU_MODEL_DUFFING_MAX_EVENT) { /* duffing.hpp:144-150 */
        if (ei == 0 && y[0] > acc[0]) { acc[0] = y[0]; acc[1] = t; }
    }
}

static void initialize(const Model* m, double t, double* td, double* y, const double* p, double* acc) {
    (void)td;
    (void)p;
    switch (m->id) {
    case ODEGPU_MODEL_DUFFING_MAX_ACCESSORY:
    case ODEGPU_MODEL_DUFFING_MAX_EVENT: acc[0] = y[0]; acc[1] = t; break; /* duffing.hpp:102-106, 139-143 */
    case ODEGPU_MODEL_DUFFING_MAXMIN: acc[0] = y[0]; acc[1] = t; acc[2] = y[0]; acc[3] = t; break;
    case ODEGPU_MODEL_BUBBLE_COLLAPSE: /* keller_miksis.hpp:327-333 */
        acc[0] = t; acc[1] = y[0]; acc[2] = t; acc[3] = y[0];
        break;
    case ODEGPU_MODEL_VALVE: acc[0] = y[0]; acc[1] = y[0]; break; /* valve.hpp:442-446 */
    case ODEGPU_MODEL_COUNTING: acc[0] += 1; break;
    default: break;
    }
}

static void finalize(const Model* m, double t, double* td, double* y, const double* p, double* acc) {
    (void)p;
    switch (m->id) {
    case ODEGPU_MODEL_BUBBLE_COLLAPSE: td[0] = t; break; /* keller_miksis.hpp:341-344 */
    case ODEGPU_MODEL_DUFFING_LYAPUNOV: acc[0] = y[2]; y[2] = 1.0; break; /* duffing.hpp:172-176 */
    case ODEGPU_MODEL_COUNTING: acc[1] += 1; break;
    default: break;
    }
}

/* ---------------------------------------------------------------- steppers */

/* steppers.hpp:16-39 */
static const double c2 = 1.0 / 5.0, c3 = 3.0 / 10.0, c4 = 3.0 / 5.0, c5 = 1.0, c6 = 7.0 / 8.0;
static const double a21 = 1.0 / 5.0;
static const double a31 = 3.0 / 40.0, a32 = 9.0 / 40.0;
static const double a41 = 3.0 / 10.0, a42 = -9.0 / 10.0, a43 = 6.0 / 5.0;
static const double a51 = -11.0 / 54.0, a52 = 5.0 / 2.0, a53 = -70.0 / 27.0, a54 = 35.0 / 27.0;
static const double a61 = 1631.0 / 55296.0, a62 = 175.0 / 512.0, a63 = 575.0 / 13824.0,
                    a64 = 44275.0 / 110592.0, a65 = 253.0 / 4096.0;
static const double b1 = 37.0 / 378.0, b3 = 250.0 / 621.0, b4 = 125.0 / 594.0, b6 = 512.0 / 1771.0;
static const double e1 = 2825.0 / 27648.0, e3 = 18575.0 / 48384.0, e4 = 13525.0 / 55296.0,
                    e5 = 277.0 / 14336.0, e6 = 1.0 / 4.0;
#define D1 (b1 - e1)
#define D3 (b3 - e3)
#define D4 (b4 - e4)
#define D5 (-e5)
#define D6 (b6 - e6)

static int all_finite(int n, const double* v) {
    for (int i = 0; i < n; ++i)
        if (!isfinite(v[i])) return 0;
    return 1;
}

/* steppers.hpp:82-101 */
static void rk4_step(const Model* m, double t, double h, const double* y, const double* p, double* out,
                     double* err, int* nonfinite) {
    const int n = m->n;
    double k1[MAXN], k2[MAXN], k3[MAXN], k4[MAXN], yt[MAXN];
    ode_rhs(m, t, y, p, k1);
    for (int i = 0; i < n; ++i) yt[i] = y[i] + 0.5 * h * k1[i];
    ode_rhs(m, t + 0.5 * h, yt, p, k2);
    for (int i = 0; i < n; ++i) yt[i] = y[i] + 0.5 * h * k2[i];
    ode_rhs(m, t + 0.5 * h, yt, p, k3);
    for (int i = 0; i < n; ++i) yt[i] = y[i] + h * k3[i];
    ode_rhs(m, t + h, yt, p, k4);
    for (int i = 0; i < n; ++i) {
        out[i] = y[i] + (h / 6.0) * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);
        err[i] = 0.0;
    }
    *nonfinite = !all_finite(n, out);
}

/* steppers.hpp:105-139 */
static void rkck45_step(const Model* m, double t, double h, const double* y, const double* p, double* out,
                        double* err, int* nonfinite) {
    const int n = m->n;
    double k1[MAXN], k2[MAXN], k3[MAXN], k4[MAXN], k5[MAXN], k6[MAXN], yt[MAXN];
    ode_rhs(m, t, y, p, k1);
    for (int i = 0; i < n; ++i) yt[i] = y[i] + h * (a21 * k1[i]);
    ode_rhs(m, t + c2 * h, yt, p, k2);
    for (int i = 0; i < n; ++i) yt[i] = y[i] + h * (a31 * k1[i] + a32 * k2[i]);
    ode_rhs(m, t + c3 * h, yt, p, k3);
    for (int i = 0; i < n; ++i) yt[i] = y[i] + h * (a41 * k1[i] + a42 * k2[i] + a43 * k3[i]);
    ode_rhs(m, t + c4 * h, yt, p, k4);
    for (int i = 0; i < n; ++i) yt[i] = y[i] + h * (a51 * k1[i] + a52 * k2[i] + a53 * k3[i] + a54 * k4[i]);
    ode_rhs(m, t + c5 * h, yt, p, k5);
    for (int i = 0; i < n; ++i)
        yt[i] = y[i] + h * (a61 * k1[i] + a62 * k2[i] + a63 * k3[i] + a64 * k4[i] + a65 * k5[i]);
    ode_rhs(m, t + c6 * h, yt, p, k6);
    for (int i = 0; i < n; ++i) {
        out[i] = y[i] + h * (b1 * k1[i] + b3 * k3[i] + b4 * k4[i] + b6 * k6[i]);
        err[i] = fabs(h * (D1 * k1[i] + D3 * k3[i] + D4 * k4[i] + D5 * k5[i] + D6 * k6[i]));
    }
    *nonfinite = !all_finite(n, out) || !all_finite(n, err);
}

/* steppers.hpp:142-149 */
static void take_step(const Model* m, int alg, double t, double h, const double* y, const double* p, double* out,
                      double* err, int* nonfinite) {
    if (alg == ODEGPU_RK4)
        rk4_step(m, t, h, y, p, out, err, nonfinite);
    else
        rkck45_step(m, t, h, y, p, out, err, nonfinite);
}

/* steppers.hpp:154-163 */
double odo_error_ratio(int n, const double* err, const double* y_old, const double* y_new, const double* rel_tol,
                       const double* abs_tol) {
    double ratio = 0.0;
    for (int i = 0; i < n; ++i) {
        const double scale = abs_tol[i] + rel_tol[i] * smax(fabs(y_old[i]), fabs(y_new[i]));
        ratio = smax(ratio, err[i] / scale);
    }
    return ratio;
}

/* steppers.hpp:176-198 */
int odo_control_step(double ratio, double h, const odegpu_ode_controls* c, int nonfinite, double* next_step,
                     int* fatal) {
    *fatal = 0;
    if (nonfinite) {
        if (h <= c->min_step) {
            *fatal = 1;
            *next_step = c->min_step;
            return 0;
        }
        *next_step = smax(h * c->step_shrink_limit, c->min_step);
        return 0;
    }
    int accepted = ratio <= 1.0;
    double factor = 0.9 * pow(ratio, -0.2);
    factor = sclamp(factor, c->step_shrink_limit, c->step_grow_limit);
    *next_step = sclamp(h * factor, c->min_step, c->max_step);
    if (!accepted && h <= c->min_step) {
        accepted = 1;
        *next_step = c->min_step;
    }
    return accepted;
}

/* ------------------------------------------------------------------ events */

enum { ZONE_NONE = -1, ZONE_BELOW = 0, ZONE_INSIDE = 1, ZONE_ABOVE = 2 };
enum { KIND_NONE = -1, KIND_STEPPED_ACROSS = 0, KIND_FROM_ABOVE = 1, KIND_FROM_BELOW = 2 };
enum { PHASE_NORMAL = 0, PHASE_LEAVING = 1 };

/* events.hpp:22-26 */
static int zone_of(double v, double tol) {
    if (!isfinite(v)) return ZONE_NONE;
    if (fabs(v) <= tol) return ZONE_INSIDE;
    return v > 0 ? ZONE_ABOVE : ZONE_BELOW;
}

/* events.hpp:54-70 */
static int classify_transition(int prev, int next, int direction, int phase) {
    if (phase != PHASE_NORMAL) return KIND_NONE;
    if (prev == ZONE_ABOVE) {
        if (next == ZONE_BELOW && direction <= 0) return KIND_STEPPED_ACROSS;
        if (next == ZONE_INSIDE && direction <= 0) return KIND_FROM_ABOVE;
        return KIND_NONE;
    }
    if (prev == ZONE_BELOW) {
        if (next == ZONE_ABOVE && direction >= 0) return KIND_STEPPED_ACROSS;
        if (next == ZONE_INSIDE && direction >= 0) return KIND_FROM_BELOW;
        return KIND_NONE;
    }
    return KIND_NONE;
}

typedef struct {
    int phase[MAXE];
    double prev_value[MAXE];
    int64_t counter[MAXE];
    int64_t steps_in_zone;
} Machine;

/* events.hpp:93-101 */
static void machine_init(Machine* mc, const Model* m, const double* values) {
    for (int i = 0; i < m->ne; ++i) {
        mc->prev_value[i] = values[i];
        mc->phase[i] = zone_of(values[i], m->tol[i]) == ZONE_INSIDE ? PHASE_LEAVING : PHASE_NORMAL;
        mc->counter[i] = 0;
    }
    mc->steps_in_zone = 0;
}

/* events.hpp:111-125: returns index (or -1), writes needs_location */
static int machine_peek(const Machine* mc, const Model* m, const double* end_values, int* needs_location) {
    *needs_location = 0;
    for (int i = m->ne - 1; i >= 0; --i) {
        const int prev = zone_of(mc->prev_value[i], m->tol[i]);
        const int next = zone_of(end_values[i], m->tol[i]);
        if (prev == ZONE_NONE || next == ZONE_NONE) continue;
        const int kind = classify_transition(prev, next, m->dir[i], mc->phase[i]);
        if (kind != KIND_NONE) {
            *needs_location = kind == KIND_STEPPED_ACROSS;
            return i;
        }
    }
    return -1;
}

typedef struct {
    int index;
    int64_t counter;
    double value;
    int in_zone;
} Detection;

/* events.hpp:134-156 */
static int machine_commit(Machine* mc, const Model* m, const double* landed, int forced, Detection* out) {
    int nd = 0;
    for (int i = 0; i < m->ne; ++i) {
        const double value = landed[i];
        int kind = KIND_NONE;
        const int prev = zone_of(mc->prev_value[i], m->tol[i]);
        const int next = zone_of(value, m->tol[i]);
        if (prev != ZONE_NONE && next != ZONE_NONE) kind = classify_transition(prev, next, m->dir[i], mc->phase[i]);
        if (kind == KIND_NONE && i != forced) continue;
        ++mc->counter[i];
        out[nd].index = i;
        out[nd].counter = mc->counter[i];
        out[nd].value = value;
        out[nd].in_zone = isfinite(value) && fabs(value) <= m->tol[i];
        ++nd;
    }
    return nd;
}

/* events.hpp:160-173 */
static void machine_refresh(Machine* mc, const Model* m, const double* post) {
    int any_inside = 0;
    for (int i = 0; i < m->ne; ++i) {
        const int z = zone_of(post[i], m->tol[i]);
        if (z == ZONE_NONE) continue;
        mc->prev_value[i] = post[i];
        mc->phase[i] = z == ZONE_INSIDE ? PHASE_LEAVING : PHASE_NORMAL;
        any_inside = any_inside || z == ZONE_INSIDE;
    }
    mc->steps_in_zone = any_inside ? mc->steps_in_zone + 1 : 0;
}

/* events.hpp:190-241 */
static int locate_secant(const Model* m, int alg, double t, const double* y, const double* p, double h, int ev,
                         double f_at_start, double f_at_end, double tolerance, double* y_best, double* best_theta,
                         double* best_value, int* converged) {
    double b_theta = h, b_value = f_at_end;
    int b_iter = 0, conv = 0;
    double theta_prev = 0, f_prev = f_at_start;
    double theta_cur = h, f_cur = f_at_end;
    const double theta_min = h * 1e-12;
    double out[MAXN], err[MAXN], fs[MAXE];
    for (int it = 1; it <= 50; ++it) {
        const double denom = f_cur - f_prev;
        if (denom == 0) break;
        double theta = theta_cur - f_cur * (theta_cur - theta_prev) / denom;
        if (!isfinite(theta)) break;
        theta = sclamp(theta, theta_min, h);
        if (theta == theta_cur) break;
        int nf;
        take_step(m, alg, t, theta, y, p, out, err, &nf);
        event_values(m, t + theta, out, p, fs);
        const double f = fs[ev];
        if (!isfinite(f)) break;
        if (fabs(f) < fabs(b_value)) {
            b_theta = theta;
            b_value = f;
            b_iter = it;
            memcpy(y_best, out, sizeof(double) * (size_t)m->n);
        }
        if (fabs(f) <= tolerance) {
            conv = 1;
            break;
        }
        theta_prev = theta_cur;
        f_prev = f_cur;
        theta_cur = theta;
        f_cur = f;
    }
    *best_theta = b_theta;
    *best_value = b_value;
    *converged = conv;
    return b_iter;
}

/* ------------------------------------------------------------------ driver */

/* driver.hpp:83-234 */
static void integrate_system(const Model* m, int alg, double dt, const odegpu_ode_controls* ode, double* td,
                             double* state, const double* p, double* acc, odegpu_outcome* oc) {
    const int n = m->n, ne = m->ne;
    Machine mc;
    double f_end[MAXE], f_landed[MAXE], f_post[MAXE];
    double prop[MAXN], err[MAXN], y_landed[MAXN];
    Detection det[MAXE];

    memset(oc, 0, sizeof *oc);
    oc->reason = ODEGPU_REACHED_END_TIME;
    oc->smallest_step = INFINITY;

    initialize(m, td[0], td, state, p, acc);
    double t = td[0];
    const double t1 = td[1];
    if (ne > 0) {
        event_values(m, t, state, p, f_end);
        machine_init(&mc, m, f_end);
    } else {
        memset(&mc, 0, sizeof mc);
    }
    double h = alg == ODEGPU_RK4 ? dt : sclamp(dt, ode->min_step, ode->max_step);

    /* Debug aid only (unset = reference behaviour): abandon a system after
     * ODO_DEBUG_MAX_STEPS trial steps and report it on stderr. */
    static long long debug_cap = -2;
    if (debug_cap == -2) {
        const char* e = getenv("ODO_DEBUG_MAX_STEPS");
        debug_cap = e ? atoll(e) : -1;
    }
    while (t < t1) {
        if (debug_cap > 0 && oc->accepted_steps + oc->rejected_steps > debug_cap) {
            fprintf(stderr, "odo: step cap hit at t=%.17g h=%.17g y=(%.17g, %.17g) p0=%.17g p1=%.17g\n", t, h,
                    state[0], m->n > 1 ? state[1] : 0.0, m->np ? p[0] : 0.0, m->np > 1 ? p[1] : 0.0);
            break;
        }
        double h_try = h;
        int clipped = 0;
        if (t + h_try >= t1) {
            h_try = t1 - t;
            clipped = 1;
        }
        if (!(h_try > 0)) {
            t = t1;
            break;
        }
        int nonfinite;
        take_step(m, alg, t, h_try, state, p, prop, err, &nonfinite);

        double next_step = h;
        if (alg == ODEGPU_RK4) {
            if (nonfinite) {
                oc->reason = ODEGPU_NONFINITE_ABORT;
                break;
            }
        } else {
            const double ratio = odo_error_ratio(n, err, state, prop, ode->rel_tol, ode->abs_tol);
            int fatal;
            const int accepted = odo_control_step(ratio, h_try, ode, nonfinite, &next_step, &fatal);
            if (fatal) {
                oc->reason = ODEGPU_NONFINITE_ABORT;
                break;
            }
            if (!accepted) {
                ++oc->rejected_steps;
                h = next_step;
                continue;
            }
        }

        double t_landed = clipped ? t1 : t + h_try;
        memcpy(y_landed, prop, sizeof(double) * (size_t)n);
        int located = -1, relocated = 0;
        if (ne > 0) {
            event_values(m, t_landed, y_landed, p, f_end);
            int needs;
            const int idx = machine_peek(&mc, m, f_end, &needs);
            located = idx;
            if (idx >= 0 && needs) {
                double theta, value;
                int conv;
                locate_secant(m, alg, t, state, p, h_try, idx, mc.prev_value[idx], f_end[idx], m->tol[idx],
                              y_landed, &theta, &value, &conv);
                if (!conv) ++oc->secant_failures;
                relocated = theta < h_try;
                t_landed = (clipped && !relocated) ? t1 : t + theta;
                event_values(m, t_landed, y_landed, p, f_landed);
            } else {
                memcpy(f_landed, f_end, sizeof(double) * (size_t)ne);
            }
        }
        if (t_landed <= t) {
            oc->reason = ODEGPU_NONFINITE_ABORT;
            break;
        }
        const double advanced = t_landed - t;
        memcpy(state, y_landed, sizeof(double) * (size_t)n);
        t = t_landed;
        ++oc->accepted_steps;
        oc->smallest_step = smin(oc->smallest_step, advanced);

        int event_stop = 0;
        if (ne > 0) {
            const int nd = machine_commit(&mc, m, f_landed, located, det);
            oc->event_detections += nd;
            if (located >= 0) event_action(m, located, mc.counter[located], t, state, p);
            if (located >= 0)
                event_values(m, t, state, p, f_post);
            else
                memcpy(f_post, f_landed, sizeof(double) * (size_t)ne);
            machine_refresh(&mc, m, f_post);
            for (int d = 0; d < nd; ++d) event_accessory(m, det[d].index, det[d].counter, t, state, p, acc);
            for (int d = 0; d < nd; ++d) {
                const int i = det[d].index;
                if (m->stop[i] != 0 && det[d].counter >= m->stop[i]) event_stop = 1;
            }
        }
        ordinary_accessory(m, t, state, p, acc);
        if (event_stop) {
            oc->reason = ODEGPU_EVENT_STOP;
            break;
        }
        if (ne > 0 && mc.steps_in_zone >= m->max_zone) {
            oc->reason = ODEGPU_EQUILIBRIUM_STOP;
            break;
        }
        if (alg == ODEGPU_RKCK45 && !relocated) h = next_step;
    }
    finalize(m, t, td, state, p, acc);
    oc->final_t = t;
}

/* solve.hpp:60-128 (single worker) + solve_iteratively solve.hpp:133-142 */
int odo_solve(const odegpu_model* mdesc, odegpu_index n, double* td, double* y, const double* p, double* acc,
              odegpu_outcome* outcomes, int keep_outcomes, const odegpu_solver_config* cfg,
              const odegpu_ode_controls* ode, odegpu_index iterations, double* trace_td, double* trace_state,
              double* trace_acc, odegpu_outcome* trace_outcomes, double* seconds) {
    Model m;
    int rc = model_init(&m, mdesc);
    if (rc) return rc;
    if (iterations < 1) return fail(ODEGPU_ERR_INVALID_ARGUMENT, "solve_iteratively: iterations must be >= 1");
    if (cfg->initial_time_step <= 0) return fail(ODEGPU_ERR_INVALID_ARGUMENT, "solve: initial_time_step must be > 0");
    if (cfg->tile_size < 1) return fail(ODEGPU_ERR_INVALID_ARGUMENT, "solve: tile_size must be >= 1");
    if (cfg->algorithm != ODEGPU_RK4 && cfg->initial_time_step > ode->max_step)
        return fail(ODEGPU_ERR_INVALID_ARGUMENT, "solve: initial_time_step exceeds max_step");
    if (!keep_outcomes) /* linear_set resets outcomes, batch.cpp:102-103 */
        for (odegpu_index i = 0; i < n; ++i) {
            memset(&outcomes[i], 0, sizeof outcomes[i]);
            outcomes[i].smallest_step = INFINITY;
        }
    struct timespec a, b;
    clock_gettime(CLOCK_MONOTONIC, &a);
    double tdl[2], yl[MAXN], pl[MAXP], al[MAXA];
    for (odegpu_index it = 0; it < iterations; ++it) {
        for (odegpu_index i = 0; i < n; ++i)
            if (td[i + n] < td[i]) {
                snprintf(g_err, sizeof g_err, "solve: system %lld has t1 < t0", (long long)i);
                return ODEGPU_ERR_INVALID_ARGUMENT;
            }
        for (odegpu_index i = 0; i < n; ++i) {
            if (outcomes[i].reason == ODEGPU_NONFINITE_ABORT) continue; /* solve.hpp:98-100 */
            /* gather_system, batch.cpp:20-30 */
            for (int c = 0; c < 2; ++c) tdl[c] = td[i + c * n];
            for (int c = 0; c < m.n; ++c) yl[c] = y[i + c * n];
            for (int c = 0; c < m.np; ++c) pl[c] = p[i + c * n];
            for (int c = 0; c < m.na; ++c) al[c] = acc[i + c * n];
            integrate_system(&m, cfg->algorithm, cfg->initial_time_step, ode, tdl, yl, pl, al, &outcomes[i]);
            /* scatter_system, batch.cpp:32-40 */
            for (int c = 0; c < 2; ++c) td[i + c * n] = tdl[c];
            for (int c = 0; c < m.n; ++c) y[i + c * n] = yl[c];
            for (int c = 0; c < m.na; ++c) acc[i + c * n] = al[c];
        }
        if (trace_td) memcpy(trace_td + it * 2 * n, td, sizeof(double) * 2 * (size_t)n);
        if (trace_state) memcpy(trace_state + it * m.n * n, y, sizeof(double) * (size_t)(m.n * n));
        if (trace_acc && m.na) memcpy(trace_acc + it * m.na * n, acc, sizeof(double) * (size_t)(m.na * n));
        if (trace_outcomes) memcpy(trace_outcomes + it * n, outcomes, sizeof(odegpu_outcome) * (size_t)n);
    }
    clock_gettime(CLOCK_MONOTONIC, &b);
    if (seconds) *seconds = (double)(b.tv_sec - a.tv_sec) + 1e-9 * (double)(b.tv_nsec - a.tv_nsec);
    return 0;
}

int odo_take_step(const odegpu_model* mdesc, int algorithm, double t, double h, const double* y, const double* p,
                  double* proposed, double* err, int* any_nonfinite) {
    Model m;
    int rc = model_init(&m, mdesc);
    if (rc) return rc;
    take_step(&m, algorithm, t, h, y, p, proposed, err, any_nonfinite);
    return 0;
}

int odo_locate_secant(const odegpu_model* mdesc, int algorithm, double t, const double* y, const double* p,
                      double h, int event_index, double f_at_start, double f_at_end, double tolerance,
                      double* y_best, double* theta, double* value, int* converged) {
    Model m;
    int rc = model_init(&m, mdesc);
    if (rc) return rc;
    return locate_secant(&m, algorithm, t, y, p, h, event_index, f_at_start, f_at_end, tolerance, y_best, theta,
                         value, converged);
}

int odo_rhs(const odegpu_model* mdesc, double t, const double* y, const double* p, double* dy) {
    Model m;
    int rc = model_init(&m, mdesc);
    if (rc) return rc;
    ode_rhs(&m, t, y, p, dy);
    return 0;
}

/* ode_rhs of n systems (SoA, stride n) at per-system times t[i]: the parity
 * checker's event slopes dF/dt at full pool sizes (tests/parity.py). */
int odo_rhs_batch(const odegpu_model* mdesc, odegpu_index n, const double* t, const double* y, const double* p,
                  odegpu_index dim, odegpu_index np, double* dy) {
    Model m;
    int rc = model_init(&m, mdesc);
    if (rc) return rc;
    double yi[8], pi[16], di[8];
    if (dim > 8 || np > 16) return fail(ODEGPU_ERR_INVALID_ARGUMENT, "rhs_batch: model too wide");
    for (odegpu_index i = 0; i < n; ++i) {
        for (odegpu_index c = 0; c < dim; ++c) yi[c] = y[i + c * n];
        for (odegpu_index c = 0; c < np; ++c) pi[c] = p[i + c * n];
        ode_rhs(&m, t[i], yi, pi, di);
        for (odegpu_index c = 0; c < dim; ++c) dy[i + c * n] = di[c];
    }
    return 0;
}

/* keller_miksis.hpp:47-77 */
int odo_bubble_coefficients(odegpu_index n, const double* phys, double* out) {
    for (odegpu_index i = 0; i < n; ++i) {
        const double* f = phys + 13 * i;
        const double pa1 = f[0], pa2 = f[1], omega1 = f[2], omega2 = f[3], theta = f[4], R_E = f[5], c_L = f[6],
                     rho_L = f[7], P_inf = f[8], p_V = f[9], sigma = f[10], mu_L = f[11], gamma = f[12];
        if (!(omega1 > 0)) return fail(ODEGPU_ERR_INVALID_ARGUMENT, "bubble_coefficients: omega1 must be > 0");
        if (!(R_E > 0)) return fail(ODEGPU_ERR_INVALID_ARGUMENT, "bubble_coefficients: R_E must be > 0");
        if (!(gamma > 1)) return fail(ODEGPU_ERR_INVALID_ARGUMENT, "bubble_coefficients: gamma must be > 1");
        if (!(rho_L > 0) || !(c_L > 0))
            return fail(ODEGPU_ERR_INVALID_ARGUMENT, "bubble_coefficients: invalid material constants");
        const double w = R_E * omega1;
        const double S = kTwoPi / w;
        const double G = S * S / rho_L;
        const double A = P_inf - p_V;
        const double B = 2.0 * sigma / R_E;
        double c[13];
        c[0] = (A + B) * G;
        c[1] = (1.0 - 3.0 * gamma) * (A + B) * S / (rho_L * c_L);
        c[2] = A * G;
        c[3] = B * G;
        c[4] = 4.0 * mu_L / (rho_L * R_E * R_E) * (kTwoPi / omega1);
        c[5] = pa1 * G;
        c[6] = pa2 * G;
        c[7] = (w / c_L) * c[5];
        c[8] = (w / c_L) * c[6];
        c[9] = w / (kTwoPi * c_L);
        c[10] = 3.0 * gamma;
        c[11] = omega2 / omega1;
        c[12] = theta;
        for (int k = 0; k < 13; ++k) out[i + k * n] = c[k];
    }
    return 0;
}
