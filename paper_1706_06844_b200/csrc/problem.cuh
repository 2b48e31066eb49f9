// FdeProblem / Grid mirror and the level builders (reference:
// proj/include/fde/problem.hpp:16-79, proj/src/problem.cpp:27-104,
// proj/src/multigrid.cpp:407-475, proj/src/precond.cpp:50-88).
#pragma once
#include <cstdint>
#include <functional>
#include <memory>
#include <vector>

#include "examples.cuh"
#include "mg.cuh"

namespace fde_b200 {

struct Problem {
  double alpha = 1.5, beta = 1.5;
  double ax = 0.0, bx = 1.0, ay = 0.0, by = 1.0;
  double t_final = 1.0;
  bool time_dependent_coeffs = false;
  int pq = 0;  // 0: WSGD (1,0) (reference); 1: (1,-1) (BASELINE cfg3 extension)
  std::function<double(double, double, double)> d_plus, d_minus, e_plus, e_minus, source;
  std::function<double(double, double)> initial;
  // BASELINE preset identity (0 = custom); lets the source be generated on device
  int preset = 0;
  int source_kind = 0;  // 0 U[0,1), 1 1e-2 N(0,1), 2 zero
  uint64_t seed = 0;
  // reference manufactured example (make_example_on) when example.which != 0:
  // coefficients / sources / exact solution also evaluable on the device
  ExampleSpec example;
  std::function<double(double, double, double)> exact;  // may be empty
};

struct Grid {  // problem.cpp:27-48
  size_t n1 = 0, n2 = 0, steps = 0;
  double ax = 0, bx = 0, ay = 0, by = 0, t_final = 0;
  double hx = 0, hy = 0, dt = 0;
  double r = 0, s = 0, inv_r = 0, s_over_r = 0;
  Grid() = default;
  Grid(const Problem& p, size_t n1, size_t n2, size_t steps);
  double x(size_t i) const { return ax + hx * static_cast<double>(i + 1); }
  double y(size_t j) const { return ay + hy * static_cast<double>(j + 1); }
  size_t size() const { return n1 * n2; }
};

// problem.cpp:50-71 (coefficients frozen at t^m = m dt)
std::shared_ptr<StructuredOp> assemble_step_operator(const Problem& p, const Grid& g, size_t m);
// problem.cpp:98-104
std::vector<double> sample_initial(const Problem& p, const Grid& g);
// v(x_i, y_j, t^{m-1/2}) on the host (problem.cpp:80-88 call pattern)
void sample_source(const Problem& p, const Grid& g, size_t m, double* v);
// Same values generated on the device for BASELINE presets (counter hash).
void generate_source_device(const Problem& p, const Grid& g, size_t m, double* v,
                            cudaStream_t s);

// multigrid.cpp:407-441
std::shared_ptr<Hierarchy> build_geometric_hierarchy(const Problem& p, const Grid& g, size_t m,
                                                     double omega, int coarse,
                                                     size_t coarse_sweeps);
// P2VcyclePrecond hierarchy: build_p2 (precond.cpp:50-73) + Galerkin R A P
// levels (multigrid.cpp:443-475), coarsest CoarseSolve::none.
std::shared_ptr<Hierarchy> build_p2_hierarchy(const StructuredOp& fine, double omega);
// build_p2 as CSR (5-point, precond.cpp:50-73), for the exact banded solve
Csr build_p2_csr(const StructuredOp& op);
// build_galerkin_hierarchy on the full operator (MgmGalerkinPrecond,
// precond.cpp:115-133, multigrid.cpp:443-475): CSR(M) and R A P coarse
// levels over the given plan; the reference limits it to 128 x 128 grids.
std::shared_ptr<Hierarchy> build_galerkin_csr_hierarchy(const StructuredOp& fine,
                                                        std::vector<std::pair<size_t, size_t>> plan,
                                                        double omega, int coarse,
                                                        size_t coarse_sweeps);

// make_example_on (problem.cpp:172-255): the manufactured problems 1..3
// (example 2 has time-dependent coefficients); t_final = 1.
Problem make_example_problem(int which, double alpha, double beta, double ax, double bx,
                             double ay, double by);
// make_example (problem.cpp:257-260): [0, len]^2 with len 2 for example 1, else 1
Problem make_example_default(int which, double alpha, double beta);
// error_inf (problem.cpp:106-117): max |u - exact(., t)|, exact sampled on the host
double error_inf(const std::vector<double>& u, const Problem& p, const Grid& g, double t);

// Coefficient fields of step m (t = m dt) on grid g into DEVICE arrays,
// unscaled: on the device for example problems, else host callbacks + upload.
void sample_fields_device(const Problem& p, const Grid& g, size_t m, double* dp, double* dm,
                          double* ep, double* em, cudaStream_t s);
// v(x_i, y_j, t^{m-1/2}) of an example problem on the device
void example_source_device(const Problem& p, const Grid& g, size_t m, double* v,
                           cudaStream_t s);

// Device scratch for one level's four coefficient fields.
struct FieldScratch {
  DevBuf<double> dp, dm, ep, em, partial;
  DevBuf<int> flag;
  void ensure(size_t n);
};

// anisotropy_ratio (multigrid.cpp:116-128) of a fine operator whose UNSCALED
// fields sit in `f` (deterministic device sums; the reference sums
// sequentially, so the ratio can differ in the last bits).
double anisotropy_ratio_device(FieldScratch& f, size_t n, double s_over_r, double alpha,
                               double beta, cudaStream_t s);

// Time-dependent re-assembly of a geometric hierarchy at step m in place
// (driver.cpp:37-41 rebuilds it; multigrid.cpp:407-441 is what it rebuilds):
// every level's coefficients re-sampled on its own grid and refreshed with
// its fine-level scaling, dinv and the coarsest LU updated.  Returns false
// (nothing changed) when the step-m level plan differs from the hierarchy's;
// the caller then builds a new hierarchy.
bool refresh_geometric_hierarchy(Hierarchy& h, const Problem& p, const Grid& g, size_t m,
                                 FieldScratch& f, cudaStream_t s);
// The step operator itself (assemble_step_operator at step m) in place.
void refresh_step_operator(StructuredOp& op, const Problem& p, const Grid& g, size_t m,
                           FieldScratch& f, cudaStream_t s);

// BASELINE configurations: coefficient fields,
// u0 = x^2(1-x)^2 y^2(1-y)^2, counter-hash seeded sources.
struct PresetInfo {
  size_t n;
  double alpha, beta, tau;
  size_t steps;
  int pq, source_kind;
};
PresetInfo preset_info(int cfg);
Problem make_preset(int cfg, uint64_t seed, int source_kind, size_t steps, double tau);

// counter-hash inputs
__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__host__ __device__ inline uint64_t source_key(uint64_t seed, uint64_t m, uint64_t j,
                                               uint64_t i) {
  return seed ^ (m << 42) ^ (j << 21) ^ i;
}
__host__ __device__ inline double hash_u01(uint64_t key) {
  return static_cast<double>(mix64(key) >> 11) * 0x1.0p-53;
}

}  // namespace fde_b200
