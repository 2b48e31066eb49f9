/* Plain-C CPU restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).
 *
 * This is the parity oracle for paper_1706_06844_b200: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it, and only as the checker.  The product never links it.
 *
 * Every function restates the reference algorithm it names (file:line,
 * relative to /root/reference).  Pinning: tests/test_oracle_pins.py checks it
 * against the reference's own known-answer values (verify.cpp:163-181,
 * SPEC.md:227-247,262) and against oracle/_ref (the unmodified reference
 * built by oracle/Makefile) on seeded inputs; tests/golden/ holds vectors
 * produced by oracle/_ref for the GPU box, where /root/reference is absent.
 *
 * Not in the reference (parity "unpinned" by the reference, restated from the
 * published algorithms): WSGD (p,q)=(1,-1) weights and left-preconditioned
 * BiCGSTAB (BASELINE cfg3).
 */
#ifndef FDE_ORACLE_H
#define FDE_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same layout as oracle/ref_harness.cpp's ref_spec (ctypes shares one struct). */
typedef struct {
  int cfg, n1, n2, steps, precond, restart, max_outer, cycles, coarse, coarse_sweeps, pq,
      source_kind;
  double tol, omega, alpha, beta, tau;
  unsigned long long seed;
} orc_spec;

const char* orc_last_error(void);
int orc_wsgd_weights(double gamma, int K, int pq, double* g, double* w);
int orc_fft(int n, double* interleaved, int inverse);
int orc_naive_dft(int n, const double* in, double* out, int inverse);
int orc_toeplitz_apply_both(double gamma, int n, int pq, const double* x, double* y, double* yt);
int orc_toeplitz_apply_colrow(int n, const double* col, const double* row, const double* x,
                              double* y, double* yt);
int orc_grid(const orc_spec* s, double* out);
int orc_coefficients(const orc_spec* s, double* dp, double* dm, double* ep, double* em);
int orc_op_apply(const orc_spec* s, int sign, const double* x, double* y);
int orc_op_diagonal(const orc_spec* s, double* d);
int orc_plan(const orc_spec* s, int* dims, int max_levels, double* ratio0);
int orc_plan_raw(int n1, int n2, double ratio0, double alpha, double beta, int* dims,
                 int max_levels);
int orc_transfer(int n1, int n2, int cx, int cy, int op, const double* in, double* out);
int orc_vcycle(const orc_spec* s, const double* b, double* x);
int orc_precond_apply(const orc_spec* s, const double* r, double* z);
int orc_initial(const orc_spec* s, double* u);
int orc_source(const orc_spec* s, int m, double* v);
int orc_rhs(const orc_spec* s, int m, const double* u_prev, double* b);
int orc_gmres(const orc_spec* s, const double* b, double* x, int* iterations, int* converged,
              double* history, int max_history, int* n_history);
int orc_bicgstab(const orc_spec* s, const double* b, double* x, int* iterations, int* converged,
                 double* history, int max_history, int* n_history);
/* solver: 0 = GMRES(restart), 1 = BiCGSTAB */
int orc_march(const orc_spec* s, int solver, double* u_out, int* its, double* res,
              double* u_steps, double* wall);
int orc_time_apply(const orc_spec* s, int reps, double* seconds_each);
int orc_time_vcycle(const orc_spec* s, int reps, double* seconds_each);

#ifdef __cplusplus
}
#endif
#endif
