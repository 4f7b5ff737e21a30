// C++ host-layer check on the GPU: the reference-shaped API (eigenid::
// IdentityEngine, eigenid::eigenvalues, typed exceptions) over the C-ABI.
// Prints PASS/FAIL lines; exit code = number of failures.
#include <cmath>
#include <cstdio>
#include <vector>

#include <cstring>

#include "eigenid/errors.hpp"
#include "eigenid/identity.hpp"
#include "eigenid/matrix_io.hpp"
#include "eigenid_b200.h"

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
  {  // the rest of the reference surface: matrix / spectrum helpers
    auto a = random_symmetric(7, 30);
    double tr = 0.0, fro = 0.0;
    for (std::size_t i = 0; i < 30; ++i) tr += a(i, i);
    for (double v : a.entries()) fro += v * v;
    auto s = eigenvalues(a);
    report("trace-frobenius-sum", a.trace() == tr && a.frobenius_norm() == std::sqrt(fro) &&
                                      std::fabs(s.sum() - tr) <= 1e-12);
    // tridiagonalize + eigenvalues(TridiagonalForm) reproduce eigenvalues(A)
    auto t = tridiagonalize(a);
    auto st = eigenvalues(t);
    double dev = 0.0;
    for (std::size_t i = 0; i < 30; ++i) dev = std::fmax(dev, std::fabs(st[i] - s[i]));
    report("tridiagonal-form", t.diag.size() == 30 && t.offdiag.size() == 29 && dev <= 1e-12);
  }
  {  // per-component entries agree with all_magnitudes (acceptance.cpp:130-174)
    auto a = random_symmetric(3000, 24);
    auto all = engine.all_magnitudes(a);
    IdentityEngine base;
    base.reset_solve_count();
    auto rb = base.component_magnitude_baseline(a, 5, 7);
    auto rc = base.component_magnitude(a, 5, 7);
    auto rl = base.log_domain_magnitude(a, 5, 7);
    const double want = all[7 * 24 + 5];
    bool ok = std::fabs(rb.value - want) <= 1e-10 * want && std::fabs(rc.value - want) <= 1e-12 &&
              std::fabs(rl.value - want) <= 1e-10 * want;
    ok = ok && rb.method == EvaluationMethod::kBaseline &&
         rl.method == EvaluationMethod::kLogDomain && rb.i == 5 && rb.j == 7 &&
         rc.condition_flag > 0.0 && base.eigenvalue_solve_count() == 6;
    report("component-variants", ok);
    auto v = base.vector_magnitudes(a, 5);
    double vdev = 0.0, vs = 0.0;
    for (std::size_t j = 0; j < 24; ++j) {
      vdev = std::fmax(vdev, std::fabs(v[j].value - all[j * 24 + 5]));
      vs += v[j].value;
    }
    report("vector-magnitudes", v.size() == 24 && vdev <= 1e-12 && std::fabs(vs - 1) <= 1e-10);
    // pairing / batches / log-domain product helpers (identity.cpp:59-122)
    auto sa = eigenvalues(a), sm = eigenvalues(a.minor_matrix(7));
    auto f = make_sorted_pairing(sa, sm, 5);
    auto plan = prepare_batches(f, 8);
    const double lp = log_domain_product(f);
    report("pairing-helpers", f.size() == 23 && plan.batch_count() == 3 &&
                                  plan.batches[2].size() == 7 &&
                                  std::fabs(lp - rl.raw_value) <= 1e-13 * lp);
    bool nf = false, deg = false;
    try {  // the naive products overflow at n = 300, x1e3 (acceptance.cpp:198-231)
      auto big = random_symmetric(1, 300).scaled(1e3);
      for (std::size_t i = 0; i < 300 && !nf; i += 37)
        for (std::size_t j = 0; j < 300 && !nf; j += 53) base.component_magnitude_baseline(big, i, j);
    } catch (const NonFiniteIntermediate&) { nf = true; }
    try { base.component_magnitude_baseline(SymmetricMatrix::identity(5), 0, 0); }
    catch (const DegenerateEigenvalue&) { deg = true; }
    report("baseline-errors", nf && deg);
  }
  {  // multi-device context over the visible GPUs: bit-identical to one GPU
    int ndev = eigenid_gpu_device_count();
    eigenid_gpu_ctx* multi = nullptr;
    eigenid_gpu_err e{};
    const int st = eigenid_gpu_create_multi(&multi, 0, ndev < 8 ? ndev : 8, &e);
    bool ok = st == EIGENID_OK;
    if (ok) {
      auto a = random_symmetric(11, 200).scaled(0.1);
      auto want = engine.all_magnitudes(a);
      std::vector<double> got(200 * 200);
      eigenid_gpu_config c{64, 1e-12, 0};
      ok = eigenid_gpu_all_magnitudes(multi, a.entries().data(), 200, &c, got.data(), nullptr,
                                      nullptr, &e) == EIGENID_OK &&
           std::memcmp(got.data(), want.data(), sizeof(double) * got.size()) == 0;
      eigenid_gpu_destroy(multi);
    } else {
      std::printf("create_multi: %s\n", e.msg);
    }
    report("multi-gpu-nccl", ok);
  }
  return failures;
}
