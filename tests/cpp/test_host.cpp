// C++ host-layer check on the GPU: the reference-shaped API (eigenid::
// IdentityEngine, eigenid::eigenvalues, typed exceptions) over the C-ABI.
// Prints PASS/FAIL lines; exit code = number of failures.
#include <cmath>
#include <cstdio>
#include <vector>

#include "eigenid/errors.hpp"
#include "eigenid/identity.hpp"

using namespace eigenid;

static int failures = 0;
static void report(const char* name, bool ok) {
  std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", name);
  if (!ok) ++failures;
}

int main() {
  IdentityEngine engine;
  {  // hand case (test_identity.cpp:225-227)
    auto m = engine.all_magnitudes(SymmetricMatrix::build(2, {2, 1, 1, 2}));
    bool ok = true;
    for (double v : m) ok = ok && std::fabs(v - 0.5) <= 1e-12;
    report("hand-case", ok);
  }
  {  // diagonal -> standard basis
    auto m = engine.all_magnitudes(SymmetricMatrix::diagonal({1, 2, 3}));
    bool ok = true;
    for (int j = 0; j < 3; ++j)
      for (int i = 0; i < 3; ++i) ok = ok && std::fabs(m[j * 3 + i] - (i == j)) <= 1e-12;
    report("diagonal", ok);
  }
  {  // degenerate -> typed error with the gap
    bool ok = false;
    try {
      engine.all_magnitudes(SymmetricMatrix::identity(5));
    } catch (const DegenerateEigenvalue& e) {
      ok = e.gap() == 0.0;
    }
    report("degenerate", ok);
  }
  {  // MatrixTooSmall / ConfigError / AsymmetricInput
    bool a = false, b = false, c = false;
    try { engine.all_magnitudes(SymmetricMatrix::identity(1)); } catch (const MatrixTooSmall&) { a = true; }
    try { IdentityConfig cfg; cfg.batch_size = 0; IdentityEngine bad(cfg); } catch (const ConfigError&) { b = true; }
    try { SymmetricMatrix::build(2, {1, 2, 3, 4}); } catch (const AsymmetricInput&) { c = true; }
    report("typed-errors", a && b && c);
  }
  {  // doubly stochastic + solve count n+1 on the two-stage path
    const std::size_t n = 120;
    std::vector<double> e(n * n);
    unsigned long long x = 88172645463325252ULL;
    for (auto& v : e) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      v = (double)(x >> 11) * 0x1.0p-53 - 0.5;
    }
    auto a = SymmetricMatrix::build(n, e, SymmetryPolicy::kSymmetrize);
    engine.reset_solve_count();
    auto m = engine.all_magnitudes(a);
    double worst = 0.0;
    for (std::size_t j = 0; j < n; ++j) {
      double row = 0.0, col = 0.0;
      for (std::size_t i = 0; i < n; ++i) { row += m[j * n + i]; col += m[i * n + j]; }
      worst = std::fmax(worst, std::fmax(std::fabs(row - 1), std::fabs(col - 1)));
    }
    report("doubly-stochastic", worst <= 1e-8);
    report("solve-count", engine.eigenvalue_solve_count() == n + 1);
    auto s = eigenvalues(a);
    double tr = 0.0, sum = 0.0;
    for (std::size_t i = 0; i < n; ++i) tr += a(i, i);
    for (double v : s.values) sum += v;
    report("eigenvalues-trace", std::fabs(tr - sum) <= 1e-11 && s.n() == n);
  }
  {  // recover_signs hand cases (test_identity.cpp:313-323) and errors (:350-354)
    auto v = recover_signs(SymmetricMatrix::build(2, {2, 1, 1, 2}), 0, {0.5, 0.5}, 1.0);
    const double s = 1.0 / std::sqrt(2.0);
    bool ok = std::fabs(v[0] - s) <= 1e-12 && std::fabs(v[1] + s) <= 1e-12;
    auto vd = recover_signs(SymmetricMatrix::diagonal({1, 2}), 1, {0.0, 1.0}, 2.0);
    ok = ok && vd[0] == 0.0 && vd[1] == 1.0;
    report("recover-signs", ok);
    bool a = false, b = false;
    std::vector<double> junk(10, 0.1);
    std::vector<double> e(100);
    for (int r = 0; r < 10; ++r)
      for (int c = 0; c < 10; ++c) e[r * 10 + c] = (r == c) ? r : 0.1 * (r + c);
    auto m = SymmetricMatrix::build(10, e);
    try { recover_signs(m, 0, junk, 123.0); } catch (const SignRecoveryFailure&) { a = true; }
    try { recover_signs(m, 0, std::vector<double>(9, 0.1), 123.0); } catch (const DimensionMismatch&) { b = true; }
    report("recover-signs-errors", a && b);
  }
  return failures;
}
