// eigenid_host.cpp — the reference-shaped C++ API over the C-ABI.
//
// SymmetricMatrix keeps the reference's construction contract
// (matrix.cpp:10-38); eigenvalues / IdentityEngine call the sm_100a library
// through include/eigenid_b200.h and turn its status codes back into the
// typed exceptions of eigenid/errors.hpp.  Nothing here computes on the CPU.
#include <cmath>
#include <string>

#include "eigenid/errors.hpp"
#include "eigenid/identity.hpp"
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

// ---- eigenvalues
Spectrum eigenvalues(const SymmetricMatrix& a) {
  eigenid_gpu_ctx* c = shared_ctx(0);
  Spectrum s;
  s.values.resize(a.n());
  eigenid_gpu_err e{};
  check(eigenid_gpu_eigenvalues(c, a.entries().data(), a.n(), s.values.data(), &e), e);
  return s;
}

// ---- IdentityEngine
IdentityEngine::IdentityEngine(IdentityConfig cfg) : cfg_(cfg) {
  if (cfg_.batch_size < 1) throw ConfigError("batch size must be >= 1");
  if (!(cfg_.degeneracy_tol >= 0.0))
    throw ConfigError("degeneracy tolerance must be >= 0");
  ctx_ = shared_ctx(cfg_.device);
}

IdentityEngine::~IdentityEngine() = default;

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
