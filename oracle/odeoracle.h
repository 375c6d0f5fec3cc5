/*
 * odeoracle.h — TEST INFRASTRUCTURE ONLY. Plain-C, single-threaded
 * restatement of the reference hot path (odensemble solve /
 * integrate_system / RK4 / RKCK45 / event engine / built-in models).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it, and only as the checker. Pinned bit-for-bit against the compiled
 * reference (oracle/_ref/libodref.so) and the golden fixtures in
 * tests/golden/ (see tests/test_oracle_pinning.py).
 */
#ifndef ODEORACLE_H
#define ODEORACLE_H

#include "odegpu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Same contract as odref_solve (oracle/ref_harness.cpp): `iterations`
 * solve() calls over n systems in SoA arrays, in place. Event controls are
 * derived from the model exactly like the reference models derive them. */
int odo_solve(const odegpu_model* m, odegpu_index n, double* td, double* y, const double* p, double* acc,
              odegpu_outcome* outcomes, int keep_outcomes, const odegpu_solver_config* cfg,
              const odegpu_ode_controls* ode, odegpu_index iterations, double* trace_td,
              double* trace_state, double* trace_acc, odegpu_outcome* trace_outcomes, double* seconds);

/* Single steps, for the stepper known-answer tests (steppers.hpp:82-139). */
int odo_take_step(const odegpu_model* m, int algorithm, double t, double h, const double* y, const double* p,
                  double* proposed, double* err, int* any_nonfinite);
/* steppers.hpp:154-163 */
double odo_error_ratio(int n, const double* err, const double* y_old, const double* y_new,
                       const double* rel_tol, const double* abs_tol);
/* steppers.hpp:176-198; returns accepted, writes next_step and fatal */
int odo_control_step(double ratio, double h, const odegpu_ode_controls* c, int nonfinite, double* next_step,
                     int* fatal);
/* events.hpp:200-241 on a single model; y_best in/out. Returns iterations,
 * writes theta, value, converged. */
int odo_locate_secant(const odegpu_model* m, int algorithm, double t, const double* y, const double* p, double h,
                      int event_index, double f_at_start, double f_at_end, double tolerance, double* y_best,
                      double* theta, double* value, int* converged);
/* models: rhs and bubble coefficients */
int odo_rhs(const odegpu_model* m, double t, const double* y, const double* p, double* dy);
int odo_rhs_batch(const odegpu_model* m, odegpu_index n, const double* t, const double* y, const double* p,
                  odegpu_index dim, odegpu_index np, double* dy);
int odo_bubble_coefficients(odegpu_index n, const double* phys, double* out);
const char* odo_last_error(void);

#ifdef __cplusplus
}
#endif

#endif
