/* fde_b200.h -- C ABI of the B200-native CN-WSGD time-step solver.
 *
 * Drop-in boundary for the reference hot path (arXiv 1706.06844 reference,
 * /root/reference/proj).  Each entry point names the reference interface it
 * replaces (file:line under proj/).  Plain pointers and sizes only; every
 * function returns an fde_status, and fde_last_error() holds the message of
 * the last failure on the calling thread.
 *
 * Memory: vectors passed to fde_op_*, fde_mg_*, fde_precond_*, fde_gmres and
 * fde_bicgstab are DEVICE pointers (cudaMalloc'd, FP64, x index fastest:
 * p = i + j*n1, proj/src/problem.cpp:59).  fde_march_* and fde_time_march
 * take HOST arrays (the reference time_march signature) and do the copies.
 * Streams are cudaStream_t passed as void* (NULL = legacy default stream).
 * Handles own their device memory; operations on one handle are ordered on
 * the stream given and are not re-entrant across streams.
 * There is no CPU fallback: without a usable CUDA device every call that
 * touches the device fails with FDE_ECUDA.
 */
#ifndef FDE_B200_H
#define FDE_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FDE_OK = 0,
  FDE_EINVAL = 1,   /* std::invalid_argument in the reference (sizes, gamma, signs, diagonal) */
  FDE_ERUNTIME = 2, /* std::runtime_error in the reference (singular factorisation) */
  FDE_ECUDA = 3,    /* CUDA runtime failure */
  FDE_ENOMEM = 4
} fde_status;

/* PrecondKind (proj/include/fde/precond.hpp:18; numbered none, p2, mgm, p2-exact, mgm-galerkin here,
 * see fde_precond_create) and mg::CoarseSolve (proj/include/fde/multigrid.hpp:95).
 * p2-exact is a single-CTA shared-memory banded solve: at most 25,600 unknowns with half bandwidth
 * <= 256 (FDE_EINVAL beyond that; the reference's Eigen SparseLU has no such limit).  mgm-galerkin
 * keeps the reference's own guard n1, n2 <= 128 (precond.cpp:121-123). */
enum { FDE_PRECOND_NONE = 0, FDE_PRECOND_P2 = 1, FDE_PRECOND_MGM = 2, FDE_PRECOND_P2_EXACT = 3,
       FDE_PRECOND_MGM_GALERKIN = 4 };
enum { FDE_COARSE_LU = 0, FDE_COARSE_SWEEPS = 1, FDE_COARSE_NONE = 2 };

const char* fde_last_error(void);
int fde_abi_version(void); /* FDE_B200_ABI_VERSION */
#define FDE_B200_ABI_VERSION 1

/* ---------------------------------------------------------------- weights
 * binom_coeffs + wsgd_weights (proj/include/fde/weights.hpp:14-25,
 * proj/src/weights.cpp:21-51).  pq = 0: WSGD (p,q) = (1,0) (the reference);
 * pq = 1: (1,-1) (BASELINE cfg3 extension, not in the reference).
 * g and w receive K+1 values. */
int fde_wsgd_weights(double gamma, size_t K, int pq, double* g, double* w);

/* ----------------------------------------------- structured operator
 * StructuredFdeOperator (proj/include/fde/structured.hpp:57-97) built from
 * ToeplitzBlock(first_col, first_row) pairs (structured.hpp:22) and the four
 * diagonal coefficient fields (host arrays, n1*n2 each). */
typedef struct fde_op_s* fde_op;
int fde_op_create(size_t n1, size_t n2, double inv_r, double s_over_r, const double* col_x,
                  const double* row_x, const double* col_y, const double* row_y,
                  const double* dp, const double* dm, const double* ep, const double* em,
                  fde_op* out);
/* Same with ToeplitzBlock::fractional blocks (structured.cpp:47-55). */
int fde_op_create_fractional(size_t n1, size_t n2, double inv_r, double s_over_r,
                             double alpha, double beta, int pq, const double* dp,
                             const double* dm, const double* ep, const double* em,
                             fde_op* out);
int fde_op_size(fde_op op, size_t* n);
/* LinOp::apply (proj/include/fde/linop.hpp:13): y = M x */
int fde_op_apply(fde_op op, const double* x, double* y, void* stream);
/* StructuredFdeOperator::apply_rhs (structured.hpp:86): structured terms negated */
int fde_op_apply_rhs(fde_op op, const double* x, double* y, void* stream);
/* LinOp::diagonal (linop.hpp:14): copies the diagonal to host array d (n values) */
int fde_op_diagonal(fde_op op, double* d);
/* StructuredFdeOperator::scale (structured.hpp:91) */
int fde_op_scale(fde_op op, double s);
int fde_op_destroy(fde_op op);

/* ---------------------------------------------------------- the problem
 * FdeProblem (proj/include/fde/problem.hpp:22-33) with C callbacks in place
 * of std::function.  ctx is passed back to every callback. */
typedef double (*fde_field_fn)(double x, double y, double t, void* ctx);
typedef double (*fde_initial_fn)(double x, double y, void* ctx);
typedef struct {
  double alpha, beta;
  double ax, bx, ay, by;
  double t_final;
  int time_dependent_coeffs; /* re-assemble operator + preconditioner every step (driver.cpp:37-41) */
  int pq;                    /* 0 = (1,0) reference weights, 1 = (1,-1) */
  fde_field_fn d_plus, d_minus, e_plus, e_minus, source;
  fde_initial_fn initial;
  void* ctx;
  /* BASELINE preset id (1..5), 100 + k for the reference's manufactured
   * example k (1..3, fde_problem_example), or 0 for a custom problem.  Presets
   * evaluate coefficients/sources natively (on the device per step). */
  int preset;
  int source_kind; /* presets: 0 U[0,1), 1 1e-2 N(0,1), 2 zero */
  unsigned long long seed;
} fde_problem;

/* The five BASELINE configurations; steps = 0 / tau <= 0 /
 * source_kind < 0 select the config defaults.  Writes n (grid size per
 * direction) and steps to *n_out / *steps_out when non-NULL. */
int fde_problem_preset(int cfg, unsigned long long seed, int source_kind, size_t steps,
                       double tau, fde_problem* out, size_t* n_out, size_t* steps_out);
/* Grid (problem.cpp:27-48): out[5] = {hx, hy, dt, inv_r, s_over_r} */
/* make_example_on / make_example (proj/include/fde/problem.hpp:73-79,
 * proj/src/problem.cpp:172-260): manufactured example which = 1..3 on
 * [ax,bx] x [ay,by] (example 2 has time-dependent coefficients; t_final = 1;
 * exact solution known).  fde_problem_example_default uses [0,len]^2, len = 2
 * for example 1 and 1 otherwise. */
int fde_problem_example(int which, double alpha, double beta, double ax, double bx, double ay,
                        double by, fde_problem* out);
int fde_problem_example_default(int which, double alpha, double beta, fde_problem* out);
/* error_inf (problem.hpp:69-70): max |u - exact(., t)| over the grid, u HOST */
int fde_error_inf(const fde_problem* p, size_t n1, size_t n2, size_t steps, double t,
                  const double* u, double* err);
int fde_grid(const fde_problem* p, size_t n1, size_t n2, size_t steps, double* out);
/* assemble_step_operator (problem.hpp:54-55) */
int fde_assemble_step_operator(const fde_problem* p, size_t n1, size_t n2, size_t steps,
                               size_t m, fde_op* out);
/* sample_initial / source samples v(x_i, y_j, t^{m-1/2}) to host arrays */
int fde_sample_initial(const fde_problem* p, size_t n1, size_t n2, size_t steps, double* u);
int fde_sample_source(const fde_problem* p, size_t n1, size_t n2, size_t steps, size_t m,
                      double* v);

/* ---------------------------------------------------------- multigrid
 * mg::plan_level_dims (proj/include/fde/multigrid.hpp:39-40): dims receives
 * n_levels (n1, n2) pairs (at most max_levels). */
int fde_plan_level_dims(size_t n1, size_t n2, double ratio0, double alpha, double beta,
                        size_t* dims, size_t max_levels, size_t* n_levels);
/* mg::anisotropy_ratio (multigrid.hpp:28-29) */
int fde_anisotropy_ratio(fde_op op, double alpha, double beta, double* ratio);
/* GridTransfer (multigrid.hpp:50-77), device arrays:
 * op 0 prolong (coarse -> fine), 1 restrict_full, 2 restrict_transpose. */
int fde_transfer(size_t n1, size_t n2, int coarsen_x, int coarsen_y, int op, const double* in,
                 double* out, void* stream);

typedef struct fde_mg_s* fde_mg;
/* CoarseSolve (multigrid.hpp:95): 0 lu, 1 sweeps, 2 none */
/* build_geometric_hierarchy (multigrid.hpp:141-144) */
int fde_mg_build_geometric(const fde_problem* p, size_t n1, size_t n2, size_t steps, size_t m,
                           double omega, int coarse, size_t coarse_sweeps, fde_mg* out);
/* MgHierarchy(levels, geometric, ...) from caller-built level operators
 * (multigrid.hpp:109-111); the handles are retained by the hierarchy. */
int fde_mg_create(const fde_op* levels, size_t n_levels, double omega, int coarse,
                  size_t coarse_sweeps, fde_mg* out);
/* Galerkin hierarchy of the banded P2 companion (P2VcyclePrecond,
 * proj/src/precond.cpp:75-83) */
int fde_mg_build_p2(fde_op fine, double omega, fde_mg* out);
int fde_mg_depth(fde_mg h, size_t* depth);
int fde_mg_level_dims(fde_mg h, size_t level, size_t* n1, size_t* n2);
/* MgHierarchy::vcycle (multigrid.hpp:119): x is the initial guess, updated.
 * zero_guess != 0 asserts x == 0 (the reference scans for it). */
int fde_mg_vcycle(fde_mg h, const double* b, double* x, int zero_guess, void* stream);
int fde_mg_destroy(fde_mg h);

/* ------------------------------------------------------ preconditioner
 * make_preconditioner (proj/include/fde/precond.hpp:94-98): kind 0 none,
 * 1 p2 (banded Galerkin V-cycle), 2 mgm (geometric V-cycle), 3 p2-exact
 * (exact banded solve with the order-2 companion, P2ExactPrecond), 4
 * mgm-galerkin (Galerkin R A P levels of the full operator, n1, n2 <= 128,
 * MgmGalerkinPrecond; p must be given).  The reference numbers its enum
 * none, p2, p2_exact, mgm, mgm_galerkin (precond.hpp:18). */
typedef struct fde_precond_s* fde_precond;
int fde_precond_create(int kind, const fde_problem* p, size_t n1, size_t n2, size_t steps,
                       size_t m, fde_op op, double omega, size_t cycles, int coarse,
                       size_t coarse_sweeps, fde_precond* out);
/* Precond::apply (krylov.hpp:11-14): z = M^-1 r */
int fde_precond_apply(fde_precond pc, const double* r, double* z, void* stream);
int fde_precond_destroy(fde_precond pc);

/* --------------------------------------------------------------- Krylov
 * SolverConfig / KrylovResult (proj/include/fde/krylov.hpp:16-30). */
typedef struct {
  double tol;
  size_t restart;
  size_t max_outer;
} fde_solver_config;
typedef struct {
  size_t total_iterations;
  int converged;
  size_t n_history;        /* entries written to history (<= history_capacity) */
  size_t history_length;   /* full length of residual_history */
  double* history;         /* caller buffer, may be NULL */
  size_t history_capacity;
} fde_krylov_result;
/* gmres (krylov.hpp:38-40), zero initial guess; x (device) receives the solution. */
int fde_gmres(fde_op a, fde_precond m, const fde_solver_config* cfg, const double* b,
              double* x, fde_krylov_result* res, void* stream);
/* Left-preconditioned BiCGSTAB with the gmres stopping rule (extension; max
 * iterations = restart * max_outer). */
int fde_bicgstab(fde_op a, fde_precond m, const fde_solver_config* cfg, const double* b,
                 double* x, fde_krylov_result* res, void* stream);

/* ----------------------------------------------------------- time march
 * DriverConfig (proj/include/fde/driver.hpp:12-21) + solver choice. */
typedef struct {
  int precond;          /* 0 none, 1 p2, 2 mgm, 3 p2-exact, 4 mgm-galerkin */
  double tol;
  size_t restart;
  size_t max_outer;
  double omega;
  size_t cycles;
  int coarse;           /* 0 lu, 1 sweeps, 2 none */
  size_t coarse_sweeps;
  int solver;           /* 0 gmres (reference), 1 bicgstab (extension) */
} fde_driver_config;
void fde_driver_config_default(fde_driver_config* cfg); /* reference defaults */

typedef struct fde_march_s* fde_march;
/* Set-up half of time_march (driver.cpp:20-33): u0, step operator and
 * preconditioner resident on the device. */
int fde_march_create(const fde_problem* p, size_t n1, size_t n2, size_t steps,
                     const fde_driver_config* cfg, fde_march* out);
/* One time step m (driver.cpp:34-52): b = apply_rhs(u) + 2 hx^alpha v, GMRES
 * from zero, u <- solution.  source: v(x_i, y_j, t^{m-1/2}) as
 *   source_mode 0: evaluated by the library (problem callback or preset),
 *   source_mode 1: HOST array (copied to the device inside the call),
 *   source_mode 2: DEVICE array,
 *   source_mode 3: the array given to fde_march_prefetch_source. */
int fde_march_step(fde_march h, const double* source, int source_mode, void* stream,
                   size_t* iterations, double* residual);
/* Current step index m (steps taken so far) */
int fde_march_steps_taken(fde_march h, size_t* m);
/* u^m to a host (to_host != 0) or device array */
int fde_march_solution(fde_march h, double* u, int to_host, void* stream);
/* Device pointer of u^m (valid until the next step) */
int fde_march_solution_ptr(fde_march h, const double** u_dev);
/* Pipelined host I/O (no reference counterpart: time_march keeps everything
 * on the host, driver.cpp:10-69).  The copies run on the march's own copy
 * stream, overlapped with the neighbouring steps' solves:
 *   fde_march_prefetch_source: H2D of a coming step's source from a host
 *     (preferably pinned) array, at most two ahead; each fde_march_step with
 *     source_mode 3 consumes the oldest one.
 *   fde_march_solution_async: D2H of u^m into a host array; the data is valid
 *     after fde_march_wait.  The step that would overwrite u^m's buffer (two
 *     steps later) waits for this copy on the device.
 *   fde_march_wait: block until every copy issued so far has completed. */
int fde_march_prefetch_source(fde_march h, const double* host_source);
int fde_march_solution_async(fde_march h, double* host_u);
int fde_march_wait(fde_march h);
int fde_march_destroy(fde_march h);

/* time_march (proj/include/fde/driver.hpp:39-40): all steps, host outputs.
 * step_iterations / step_residuals hold `steps` entries; solution n1*n2. */
int fde_time_march(const fde_problem* p, size_t n1, size_t n2, size_t steps,
                   const fde_driver_config* cfg, double* solution, size_t* step_iterations,
                   double* step_residuals, double* wall_seconds);

/* ------------------------------------------------ multi-GPU building blocks
 * y-slab decomposition.  A slab is rank r's piece of a level
 * operator (d1 x d2 grid of problem p at step m, rescaled onto the fine
 * nf1 x nf2 level like build_geometric_hierarchy): rows [r0, r1) for the row
 * pass and columns [c0, c1) for the column pass.  The caller moves data
 * between the two layouts (all-to-all); these entry points are the local
 * compute.  Device arrays. */
typedef struct fde_slab_s* fde_slab;
int fde_slab_create(const fde_problem* p, size_t nf1, size_t nf2, size_t d1, size_t d2,
                    size_t steps, size_t m, size_t r0, size_t r1, size_t c0, size_t c1,
                    fde_slab* out);
/* QT[c * d2 + j] = sign * s/r * (ep T_b x + em T_b^T x) at column c0 + c, from
 * xT[c * d2 + j] = x[(c0 + c) + j * d1] */
int fde_slab_ypass(fde_slab h, const double* xT, double* QT, double sign, void* stream);
/* rows r0..r1 (local row-major blocks of width d1): out = epilogue(inv_r x +
 * sign (dp T_a x + dm T_a^T x) + Q); epi 0 store, 1 rhs (+ src_scale src),
 * 2 residual (b - .), 3 Jacobi (x + omega dinv (b - .)) */
int fde_slab_xpass(fde_slab h, const double* x, const double* Q, double* out, double sign,
                   int epi, const double* b, const double* dinv, double omega, const double* src,
                   double src_scale, void* stream);
int fde_slab_diagonal(fde_slab h, double* d); /* host copy, (r1 - r0) * d1 values */
int fde_slab_destroy(fde_slab h);
/* out[c * rows + r] = in[r * cols + c] (row-major rows x cols -> cols x rows) */
int fde_transpose(const double* in, double* out, size_t rows, size_t cols, void* stream);
/* GridTransfer on row windows: `in` holds global rows starting at in_lo of its
 * grid, `out` receives global rows [out_lo, out_lo + out_rows) of the other
 * grid.  op 0 prolong (add != 0: out += P in), 1 restrict_full, 2 restrict_transpose. */
int fde_transfer_rows(size_t n1, size_t n2, int coarsen_x, int coarsen_y, int op, int add,
                      const double* in, size_t in_lo, double* out, size_t out_lo,
                      size_t out_rows, void* stream);
/* vector kernels: op 0 out = a * x .* y (zero-guess smoothing), 1 out += a * x
 * (axpy, y unused), 2 out += a * x .* y (Jacobi update), 3 out = x * a (scale) */
int fde_vec(int op, size_t n, double a, const double* x, const double* y, double* out,
            void* stream);
/* All-to-all layout helper.  Row ranges of the P ranks: offsets[0..P]
 * (offsets[0] = 0, offsets[P] = d2).  dir 0 (unpack): in holds P chunks, chunk
 * s = [nc][offsets[s+1]-offsets[s]] at element offset nc*offsets[s]; out is
 * [nc][d2] with out[c*d2 + j] = chunk_owner(j)[c][j - offsets[owner]].  dir 1
 * (pack) is the inverse map. */
int fde_block_permute(const double* in, double* out, size_t nc, size_t d2,
                      const long long* offsets_host, int nranks, int dir, void* stream);
/* out += sgn * (*a_dev) * x (device scalar, e.g. a projection coefficient) */
int fde_axpy_dev(size_t n, const double* a_dev, double sgn, const double* x, double* out,
                 void* stream);
/* *out_dev = <x, y> (deterministic two-level reduction; sqrt_out: sqrt of it) */
int fde_dot(size_t n, const double* x, const double* y, double* out_dev, int sqrt_out,
            void* stream);

/* Number of kernels this library has launched since load (instrumentation). */
unsigned long long fde_kernel_launches(void);
/* ------------------------------------------------ multi-GPU time step
 * The per-step loop of the y-slab decomposition in C++ (csrc/dist.cu): slab
 * levels, the distributed V-cycle with its replicated coarse tail, GMRES with
 * device-resident scalars and rank-ordered inner products, and the march
 * (reference: driver.cpp:10-69, krylov.cpp:34-166, multigrid.cpp:318-394 --
 * the reference itself is single-process).  One process per GPU; the
 * transport is NCCL, opened at run time.  fde_dist_unique_id on one rank
 * produces the 128-byte id every rank passes to fde_dist_comm_create (the
 * launcher moves it, e.g. by a torch.distributed broadcast). */
typedef struct fde_dist_comm_s* fde_dist_comm;
int fde_dist_unique_id(unsigned char* id128);
int fde_dist_comm_create(const unsigned char* id128, int rank, int world, fde_dist_comm* out);
int fde_dist_comm_destroy(fde_dist_comm c);
typedef struct fde_dist_march_s* fde_dist_march;
/* cfg: solver 0 (gmres), precond none or mgm, cycles 1.  Levels of at most
 * `agglomerate` unknowns are replicated on every rank. */
int fde_dist_march_create(fde_dist_comm c, const fde_problem* p, size_t n1, size_t n2,
                          size_t steps, const fde_driver_config* cfg, size_t agglomerate,
                          fde_dist_march* out);
/* grid rows [r0, r1) this rank owns; local vectors hold (r1 - r0) * n1 values */
int fde_dist_march_rows(fde_dist_march h, size_t* r0, size_t* r1);
/* one time step; source_local: the rank's rows of v(., t^{m-1/2}) on the
 * DEVICE, or NULL (evaluated by the library) */
int fde_dist_march_step(fde_dist_march h, const double* source_local, void* stream,
                        size_t* iterations, double* residual);
int fde_dist_march_solution(fde_dist_march h, double* u_local, int to_host, void* stream);
int fde_dist_march_solution_ptr(fde_dist_march h, const double** u_dev);
/* y_local = (A x)_local and x_local = V-cycle(b_local): device arrays */
int fde_dist_march_apply(fde_dist_march h, const double* x_local, double* y_local, void* stream);
int fde_dist_march_vcycle(fde_dist_march h, const double* b_local, double* x_local, void* stream);
/* collectives issued so far (all-to-all, all-gather, halo exchanges) */
int fde_dist_march_collectives(fde_dist_march h, unsigned long long* n);
int fde_dist_march_destroy(fde_dist_march h);
/* The partition (host only, no device needed): balanced row offsets[0..nranks]
 * of the fine level, and the offsets a coarser level inherits (coarse row b
 * goes to the rank that owns its centre fine row 2b + 1 - par). */
int fde_dist_split_rows(size_t n, int nranks, size_t* offsets);
int fde_dist_induced_rows(const size_t* fine_offsets, int nranks, size_t d2, int coarsen_y,
                          size_t* coarse_offsets);
/* The same code on `nranks` VIRTUAL ranks of the current device (one host
 * thread per rank, one shared stream, collectives as ordered device copies):
 * how the N > 1 paths are exercised on one GPU.  HOST vectors of the whole
 * grid.  what 0: march `nrun` steps, out = u^nrun, iterations / residuals
 * [nrun]; what 1: out = A in; what 2: out = V-cycle(in). */
int fde_vdist_run(const fde_problem* p, size_t n1, size_t n2, size_t steps,
                  const fde_driver_config* cfg, int nranks, size_t agglomerate, int what,
                  size_t nrun, const double* in_full, double* out_full, size_t* iterations,
                  double* residuals, unsigned long long* collectives);

/* Measured FP64 FMA throughput of the current device in TFLOP/s (a pure DFMA
 * kernel, best of three timed launches): the roofline denominator of the
 * FP64-issue-bound line kernels, taken in the reporting run. */
int fde_fp64_peak(double* tflops, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FDE_B200_H */
