// The reference's manufactured problems (make_example_on, proj/src/problem.cpp:
// 125-265) as plain data + __host__ __device__ formulas, so the same code
// samples coefficients, sources and exact solutions on the host (bit-identical
// to the reference's lambdas: same operations in the same order, host libm)
// and on the device (per-step re-assembly of time-dependent coefficients,
// SURVEY.md 8(f)1; CUDA pow/exp agree with libm to an ulp or two).
//
// Device code using these formulas is compiled with -fmad=false (Makefile) so
// no product-sum is contracted into an FMA the host evaluation does not have.
#pragma once
#include <cmath>

namespace fde_b200 {

constexpr int kMaxPoly = 8;

// EndPolynomial (proj/include/fde/problem.hpp:13-21) plus the per-term
// Riemann-Liouville factors of frac_deriv for one order gamma:
//   f[p] = c[p] * Gamma(p+1) / Gamma(p+1-gamma)   (0: zero / pole term)
//   e[p] = q - 1, q = p + 1 - gamma                 (the power of xi)
struct EndPoly {
  int n = 0;
  double c[kMaxPoly] = {};
  double f[kMaxPoly] = {};
  double e[kMaxPoly] = {};
  bool keep[kMaxPoly] = {};
};

struct ExampleSpec {
  int which = 0;  // 1..3; 0 = not an example problem
  double alpha = 0, beta = 0, ax = 0, bx = 0, ay = 0, by = 0, amp = 0;
  double ga = 0, gb = 0;  // example 1: tgamma(3 - alpha), tgamma(3 - beta)
  EndPoly px, py;         // px carries the alpha factors, py the beta factors
};

// EndPolynomial::value (problem.cpp:8-12): Horner from the top coefficient
__host__ __device__ inline double poly_value(const EndPoly& q, double xi) {
  double acc = 0.0;
  for (int p = q.n - 1; p >= 0; --p) acc = acc * xi + q.c[p];
  return acc;
}

// EndPolynomial::frac_deriv (problem.cpp:14-25) with the Gamma ratios folded
// into f[p] on the host: c*Gamma(p+1)/Gamma(q) * pow(xi, q-1), left to right.
__host__ __device__ inline double poly_frac_deriv(const EndPoly& q, double xi) {
  double acc = 0.0;
  for (int p = 0; p < q.n; ++p) {
    if (!q.keep[p]) continue;
    acc += q.f[p] * pow(xi, q.e[p]);
  }
  return acc;
}

// field 0 d_plus, 1 d_minus, 2 e_plus, 3 e_minus (problem.cpp:196-255)
__host__ __device__ inline double example_coeff(const ExampleSpec& s, int field, double x,
                                                double y, double t) {
  const double al = s.alpha, be = s.beta, ax = s.ax, bx = s.bx, ay = s.ay, by = s.by;
  if (s.which == 1) {
    switch (field) {
      case 0: return s.ga * pow(1.0 + x - ax, al) * (1.0 + y - ay) * (1.0 + y - ay);
      case 1: return s.ga * pow(1.0 + bx - x, al) * (1.0 + by - y) * (1.0 + by - y);
      case 2: return s.gb * (1.0 + x - ax) * (1.0 + x - ax) * pow(1.0 + y - ay, be);
      default: return s.gb * (1.0 + bx - x) * (1.0 + bx - x) * pow(1.0 + by - y, be);
    }
  }
  if (s.which == 2) {
    switch (field) {
      case 0: return 4.0 * (1.0 + t) * pow(x - ax, al) * (1.0 + y - ay);
      case 1: return 4.0 * (1.0 + t) * pow(bx - x, al) * (1.0 + y - ay);
      case 2: return 4.0 * (1.0 + t) * (1.0 + x - ax) * pow(y - ay, be);
      default: return 4.0 * (1.0 + t) * (1.0 + x - ax) * pow(by - y, be);
    }
  }
  switch (field) {
    case 0: return 6.0 * pow(x - ax, al);
    case 1: return 6.0 * pow(bx - x, al);
    case 2: return 6.0 * pow(y - ay, be);
    default: return 6.0 * pow(by - y, be);
  }
}

// attach_source (problem.cpp:150-170)
__host__ __device__ inline double example_source(const ExampleSpec& s, double x, double y,
                                                 double t) {
  const double pref = s.amp * exp(-t);
  const double vx = poly_value(s.px, x - s.ax), vy = poly_value(s.py, y - s.ay);
  const double u = pref * vx * vy;
  const double dx = example_coeff(s, 0, x, y, t) * poly_frac_deriv(s.px, x - s.ax) +
                    example_coeff(s, 1, x, y, t) * poly_frac_deriv(s.px, s.bx - x);
  const double dy = example_coeff(s, 2, x, y, t) * poly_frac_deriv(s.py, y - s.ay) +
                    example_coeff(s, 3, x, y, t) * poly_frac_deriv(s.py, s.by - y);
  return -u - pref * (dx * vy + vx * dy);
}

// make_separable (problem.cpp:128-146): exact amp e^{-t} X(x) Y(y), initial t = 0
__host__ __device__ inline double example_exact(const ExampleSpec& s, double x, double y,
                                                double t) {
  return s.amp * exp(-t) * poly_value(s.px, x - s.ax) * poly_value(s.py, y - s.ay);
}
__host__ __device__ inline double example_initial(const ExampleSpec& s, double x, double y) {
  return s.amp * poly_value(s.px, x - s.ax) * poly_value(s.py, y - s.ay);
}

// Host: validation + profiles + Gamma factors (problem.cpp:172-180,
// 113-124 quartic/sextic profiles).
ExampleSpec make_example_spec(int which, double alpha, double beta, double ax, double bx,
                              double ay, double by);

}  // namespace fde_b200
