// eigenid_host.cpp — the reference-shaped C++ API over the C-ABI.
//
// SymmetricMatrix keeps the reference's construction contract
// (matrix.cpp:10-38); eigenvalues / IdentityEngine call the sm_100a library
// through include/eigenid_b200.h and turn its status codes back into the
// typed exceptions of eigenid/errors.hpp.  Nothing here computes on the CPU.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <string>

#include "eigenid/errors.hpp"
#include "eigenid/identity.hpp"
#include "eigenid/matrix_io.hpp"
#include "eigenid_b200.h"

namespace eigenid {

namespace {

[[noreturn]] void rethrow(const eigenid_gpu_err& e) {
  const std::string msg(e.msg);
  switch (e.code) {
    case EIGENID_E_MATRIX_TOO_SMALL: throw MatrixTooSmall(msg);
    case EIGENID_E_DEGENERATE: throw DegenerateEigenvalue(msg, e.gap);
    case EIGENID_E_CONVERGENCE: throw ConvergenceFailure(msg);
    case EIGENID_E_NONFINITE: throw NonFiniteIntermediate(msg);
    case EIGENID_E_INTERNAL: throw InternalInconsistency(msg);
    case EIGENID_E_CONFIG: throw ConfigError(msg);
    case EIGENID_E_INDEX: throw IndexOutOfRange(msg);
    case EIGENID_E_SIGN_RECOVERY: throw SignRecoveryFailure(msg);
    case EIGENID_E_DIMENSION: throw DimensionMismatch(msg);
    case EIGENID_E_NONFINITE_ENTRY: throw NonFiniteEntry(msg);
    case EIGENID_E_ASYMMETRIC: throw AsymmetricInput(msg);
    default: throw DeviceError(msg, e.cuda_error);
  }
}

void check(int st, const eigenid_gpu_err& e) {
  if (st != EIGENID_OK) rethrow(e);
}

eigenid_gpu_ctx* shared_ctx(int device) {
  // one context per device and process, created once (SPEC D5)
  static eigenid_gpu_ctx* ctxs[64] = {};
  static std::atomic<bool> lock{false};
  while (lock.exchange(true)) {
  }
  eigenid_gpu_ctx* c = ctxs[device & 63];
  if (!c) {
    eigenid_gpu_err e{};
    const int st = eigenid_gpu_create(&c, device, &e);
    if (st != EIGENID_OK) {
      lock.store(false);
      rethrow(e);
    }
    ctxs[device & 63] = c;
  }
  lock.store(false);
  return c;
}

}  // namespace

// ---- SymmetricMatrix (matrix.cpp:10-86 semantics)
SymmetricMatrix SymmetricMatrix::build(std::size_t n, std::vector<double> e,
                                       SymmetryPolicy policy) {
  if (n < 1) throw DimensionMismatch("matrix dimension must be >= 1");
  if (e.size() != n * n)
    throw DimensionMismatch("expected " + std::to_string(n * n) + " entries, got " +
                            std::to_string(e.size()));
  for (double v : e)
    if (!std::isfinite(v)) throw NonFiniteEntry("matrix entry is not finite");
  double asym = 0.0;
  for (std::size_t r = 0; r < n; ++r)
    for (std::size_t c = r + 1; c < n; ++c)
      asym = std::fmax(asym, std::fabs(e[r * n + c] - e[c * n + r]));
  if (asym > 0.0) {
    if (policy == SymmetryPolicy::kStrict)
      throw AsymmetricInput("input is not symmetric (max |a_rc - a_cr| = " +
                            std::to_string(asym) + ")");
    for (std::size_t r = 0; r < n; ++r)
      for (std::size_t c = r + 1; c < n; ++c) {
        const double m = 0.5 * (e[r * n + c] + e[c * n + r]);
        e[r * n + c] = m;
        e[c * n + r] = m;
      }
  }
  return SymmetricMatrix(n, std::move(e));
}

SymmetricMatrix SymmetricMatrix::diagonal(const std::vector<double>& d) {
  std::vector<double> e(d.size() * d.size(), 0.0);
  for (std::size_t i = 0; i < d.size(); ++i) e[i * d.size() + i] = d[i];
  return build(d.size(), std::move(e));
}

SymmetricMatrix SymmetricMatrix::identity(std::size_t n) {
  return diagonal(std::vector<double>(n, 1.0));
}

SymmetricMatrix SymmetricMatrix::minor_matrix(std::size_t j) const {
  if (n_ == 1) throw MatrixTooSmall("cannot take a minor of a 1x1 matrix");
  if (j >= n_) throw IndexOutOfRange("minor index out of range");
  const std::size_t m = n_ - 1;
  std::vector<double> e(m * m);
  for (std::size_t r = 0; r < m; ++r)
    for (std::size_t c = 0; c < m; ++c)
      e[r * m + c] = e_[(r + (r >= j)) * n_ + (c + (c >= j))];
  return SymmetricMatrix(m, std::move(e));
}

SymmetricMatrix SymmetricMatrix::scaled(double factor) const {
  std::vector<double> e(e_);
  for (double& v : e) v *= factor;
  return SymmetricMatrix(n_, std::move(e));
}

double SymmetricMatrix::trace() const {  // matrix.cpp:70-74
  double t = 0.0;
  for (std::size_t i = 0; i < n_; ++i) t += e_[i * n_ + i];
  return t;
}

double SymmetricMatrix::frobenius_norm() const {  // matrix.cpp:75-79
  double s = 0.0;
  for (double v : e_) s += v * v;
  return std::sqrt(s);
}

// ---- seeded generator (matrix_io.cpp:171-181): the C-ABI's host generator
SymmetricMatrix random_symmetric(std::uint64_t seed, std::size_t n,
                                 RandomDistribution dist) {
  if (n < 1) throw DimensionMismatch("random matrix dimension must be >= 1");
  std::vector<double> e(n * n);
  eigenid_random_symmetric(seed, n, dist == RandomDistribution::kUniform ? 1 : 0,
                           e.data());
  // already symmetrised exactly as build(kSymmetrize) does: build() keeps it
  return SymmetricMatrix::build(n, std::move(e), SymmetryPolicy::kSymmetrize);
}

double Spectrum::sum() const {  // eigensolve.cpp:13-15
  return std::accumulate(values.begin(), values.end(), 0.0);
}

// ---- eigenvalues
Spectrum eigenvalues(const SymmetricMatrix& a) {
  eigenid_gpu_ctx* c = shared_ctx(0);
  Spectrum s;
  s.values.resize(a.n());
  eigenid_gpu_err e{};
  check(eigenid_gpu_eigenvalues(c, a.entries().data(), a.n(), s.values.data(), &e), e);
  return s;
}

TridiagonalForm tridiagonalize(const SymmetricMatrix& a) {
  TridiagonalForm t;
  t.diag.resize(a.n());
  t.offdiag.resize(a.n() > 0 ? a.n() - 1 : 0);
  eigenid_gpu_err e{};
  check(eigenid_gpu_tridiagonalize(shared_ctx(0), a.entries().data(), a.n(), t.diag.data(),
                                   t.offdiag.data(), &e),
        e);
  return t;
}

Spectrum eigenvalues(TridiagonalForm t) {
  const std::size_t n = t.diag.size();
  if (n > 0 && t.offdiag.size() != n - 1)
    throw DimensionMismatch("tridiagonal form needs n-1 off-diagonal values");
  Spectrum s;
  s.values.resize(n);
  eigenid_gpu_err e{};
  check(eigenid_gpu_tridiagonal_eigenvalues(shared_ctx(0), t.diag.data(), t.offdiag.data(),
                                            n, s.values.data(), &e),
        e);
  return s;
}

// ---- identity helpers (identity.cpp:12-122)
std::string method_name(EvaluationMethod m) {
  switch (m) {
    case EvaluationMethod::kBaseline: return "baseline";
    case EvaluationMethod::kBatched: return "batched";
    case EvaluationMethod::kBatchedParallel: return "batched-parallel";
    case EvaluationMethod::kLogDomain: return "log-domain";
  }
  return "?";
}

FactorPairing make_natural_pairing(const Spectrum& spectrum_a,
                                   const Spectrum& spectrum_minor, std::size_t i) {
  const std::size_t n = spectrum_a.n();
  FactorPairing f;
  f.numerator.reserve(n ? n - 1 : 0);
  f.denominator.reserve(n ? n - 1 : 0);
  const double lambda = spectrum_a[i];
  for (std::size_t k = 0; k + 1 < n; ++k) f.numerator.push_back(lambda - spectrum_minor[k]);
  for (std::size_t k = 0; k < n; ++k)
    if (k != i) f.denominator.push_back(lambda - spectrum_a[k]);
  return f;
}

FactorPairing make_sorted_pairing(const Spectrum& spectrum_a,
                                  const Spectrum& spectrum_minor, std::size_t i) {
  FactorPairing f = make_natural_pairing(spectrum_a, spectrum_minor, i);
  std::sort(f.numerator.begin(), f.numerator.end());
  std::sort(f.denominator.begin(), f.denominator.end());
  return f;
}

BatchPlan prepare_batches(const FactorPairing& factors, std::size_t batch_size) {
  if (batch_size < 1) throw ConfigError("batch size must be >= 1");
  BatchPlan plan;
  plan.batch_size = batch_size;
  const std::size_t total = factors.size();
  for (std::size_t b = 0; b < total; b += batch_size)
    plan.batches.push_back({b, std::min(b + batch_size, total)});
  return plan;
}

double log_domain_product(const FactorPairing& factors) {
  if (factors.denominator.size() != factors.numerator.size())
    throw DimensionMismatch("factor lists differ in length");
  double out = 0.0;
  eigenid_gpu_err e{};
  check(eigenid_gpu_log_domain_product(shared_ctx(0), factors.numerator.data(),
                                       factors.denominator.data(), factors.size(), &out,
                                       &e),
        e);
  return out;
}

// ---- IdentityEngine
IdentityEngine::IdentityEngine(IdentityConfig cfg) : cfg_(cfg) {
  if (cfg_.batch_size < 1) throw ConfigError("batch size must be >= 1");
  if (!(cfg_.degeneracy_tol >= 0.0))
    throw ConfigError("degeneracy tolerance must be >= 0");
  if (cfg_.num_gpus < 1) throw ConfigError("num_gpus must be >= 1");
  if (cfg_.num_gpus == 1) {
    ctx_ = shared_ctx(cfg_.device);
  } else {  // an engine-owned multi-device context (NCCL communicator inside)
    eigenid_gpu_err e{};
    check(eigenid_gpu_create_multi(&ctx_, cfg_.device, cfg_.num_gpus, &e), e);
    owns_ctx_ = true;
  }
}

IdentityEngine::~IdentityEngine() {
  if (owns_ctx_) eigenid_gpu_destroy(ctx_);
}

static eigenid_gpu_config to_c(const IdentityConfig& cfg) {
  eigenid_gpu_config c;
  c.batch_size = cfg.batch_size;
  c.degeneracy_tol = cfg.degeneracy_tol;
  c.log_domain = cfg.evaluation == IdentityConfig::Evaluation::kLogDomain;
  return c;
}

std::vector<double> IdentityEngine::all_magnitudes(const SymmetricMatrix& a) const {
  const std::size_t n = a.n();
  if (n < 2) throw MatrixTooSmall("component magnitudes need n >= 2");
  std::vector<double> out(n * n);
  const eigenid_gpu_config c = to_c(cfg_);
  eigenid_gpu_err e{};
  const std::size_t before = eigenid_gpu_solve_count(ctx_);
  const int st = eigenid_gpu_all_magnitudes(ctx_, a.entries().data(), n, &c,
                                            out.data(), nullptr, nullptr, &e);
  solves_ += eigenid_gpu_solve_count(ctx_) - before;
  check(st, e);
  return out;
}

std::vector<double> IdentityEngine::all_magnitudes_batched(
    const std::vector<double>& a, std::size_t count, std::size_t n) const {
  if (a.size() != count * n * n) throw DimensionMismatch("batched input size");
  std::vector<double> out(count * n * n);
  const eigenid_gpu_config c = to_c(cfg_);
  eigenid_gpu_err e{};
  const std::size_t before = eigenid_gpu_solve_count(ctx_);
  const int st = eigenid_gpu_all_magnitudes_batched(ctx_, a.data(), count, n, &c,
                                                    out.data(), &e);
  solves_ += eigenid_gpu_solve_count(ctx_) - before;
  check(st, e);
  return out;
}

MagnitudeResult IdentityEngine::component(const SymmetricMatrix& a, std::size_t i,
                                          std::size_t j, const Spectrum* sa,
                                          const Spectrum* sm, int variant) const {
  if (a.n() < 2) throw MatrixTooSmall("component magnitudes need n >= 2");
  if (i >= a.n() || j >= a.n())
    throw IndexOutOfRange("component index (i=" + std::to_string(i) + ", j=" +
                          std::to_string(j) + ") out of range for n = " +
                          std::to_string(a.n()));
  const eigenid_gpu_config c = to_c(cfg_);
  eigenid_gpu_magnitude m{};
  eigenid_gpu_err e{};
  const bool cached = sa && sm;
  const std::size_t before = eigenid_gpu_solve_count(ctx_);
  const int st = eigenid_gpu_component(ctx_, a.entries().data(), a.n(), i, j,
                                       cached ? sa->values.data() : nullptr,
                                       cached ? sm->values.data() : nullptr, &c, variant,
                                       &m, &e);
  solves_ += eigenid_gpu_solve_count(ctx_) - before;
  check(st, e);
  MagnitudeResult r;
  r.value = m.value;
  r.raw_value = m.raw_value;
  r.i = i;
  r.j = j;
  r.method = static_cast<EvaluationMethod>(m.method);
  r.condition_flag = m.condition_flag;
  return r;
}

MagnitudeResult IdentityEngine::component_magnitude_baseline(const SymmetricMatrix& a,
                                                             std::size_t i,
                                                             std::size_t j) const {
  return component(a, i, j, nullptr, nullptr, 2);
}

MagnitudeResult IdentityEngine::component_magnitude(const SymmetricMatrix& a, std::size_t i,
                                                    std::size_t j, const Spectrum* sa,
                                                    const Spectrum* sm) const {
  MagnitudeResult r = component(a, i, j, sa, sm, 0);
  // the reference reports its pool dispatch (identity.cpp:215-223); the
  // device result is the same either way
  if (r.method == EvaluationMethod::kBatched && cfg_.resolved_workers() > 1 &&
      (a.n() - 1 + cfg_.batch_size - 1) / cfg_.batch_size > 1)
    r.method = EvaluationMethod::kBatchedParallel;
  return r;
}

MagnitudeResult IdentityEngine::log_domain_magnitude(const SymmetricMatrix& a, std::size_t i,
                                                     std::size_t j, const Spectrum* sa,
                                                     const Spectrum* sm) const {
  return component(a, i, j, sa, sm, 1);
}

std::vector<MagnitudeResult> IdentityEngine::vector_magnitudes(const SymmetricMatrix& a,
                                                               std::size_t i) const {
  const std::size_t n = a.n();
  if (n < 2) throw MatrixTooSmall("component magnitudes need n >= 2");
  if (i >= n)
    throw IndexOutOfRange("component index (i=" + std::to_string(i) +
                          ", j=0) out of range for n = " + std::to_string(n));
  const eigenid_gpu_config c = to_c(cfg_);
  std::vector<eigenid_gpu_magnitude> m(n);
  eigenid_gpu_err e{};
  const std::size_t before = eigenid_gpu_solve_count(ctx_);
  const int st = eigenid_gpu_vector(ctx_, a.entries().data(), n, i, &c, m.data(), &e);
  solves_ += eigenid_gpu_solve_count(ctx_) - before;
  check(st, e);
  std::vector<MagnitudeResult> out(n);
  for (std::size_t j = 0; j < n; ++j) {
    out[j].value = m[j].value;
    out[j].raw_value = m[j].raw_value;
    out[j].i = i;
    out[j].j = j;
    out[j].method = static_cast<EvaluationMethod>(m[j].method);
    out[j].condition_flag = m[j].condition_flag;
  }
  return out;
}

// ---- recover_signs
std::vector<double> recover_signs(const SymmetricMatrix& a, std::size_t i,
                                  const std::vector<double>& magnitudes,
                                  double lambda_i, double sign_tol) {
  std::vector<double> v(a.n());
  eigenid_gpu_err e{};
  check(eigenid_gpu_recover_signs(shared_ctx(0), a.entries().data(), a.n(), i,
                                  magnitudes.data(), magnitudes.size(), lambda_i,
                                  sign_tol, v.data(), &e),
        e);
  return v;
}

}  // namespace eigenid
