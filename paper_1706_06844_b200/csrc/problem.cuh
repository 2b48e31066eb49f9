// FdeProblem / Grid mirror and the level builders (reference:
// proj/include/fde/problem.hpp:16-79, proj/src/problem.cpp:27-104,
// proj/src/multigrid.cpp:407-475, proj/src/precond.cpp:50-88).
#pragma once
#include <cstdint>
#include <functional>
#include <memory>
#include <vector>

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
