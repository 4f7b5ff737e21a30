// ref_shim.cpp — C entry points over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together
// with /root/reference/proj/src/*.cpp (read in place, never copied) into
// oracle/_ref/libeigenid_ref.so, with -Deigenid=eigenid_ref so the
// reference's symbols cannot collide with the product's eigenid:: host layer.
// Used by tests/ to pin the oracle restatement and by bench.py's
// --impl reference arm to time the reference's own CPU path.
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "eigenid/errors.hpp"
#include "eigenid/identity.hpp"
#include "eigenid/matrix_io.hpp"
#include "eigenid/thread_pool.hpp"

using namespace eigenid;  // expands to eigenid_ref

namespace {

struct RefErr {
  int code;
  int64_t index;
  double gap;
  char msg[256];
};

void fill(RefErr* err, int code, double gap, const char* what) {
  if (!err) return;
  err->code = code;
  err->index = -1;
  err->gap = gap;
  std::snprintf(err->msg, sizeof(err->msg), "%s", what);
}

template <class F>
int guarded(RefErr* err, F&& f) {
  try {
    f();
    return 0;
  } catch (const MatrixTooSmall& e) {
    fill(err, 1, 0.0, e.what());
    return 1;
  } catch (const DegenerateEigenvalue& e) {
    fill(err, 2, e.gap(), e.what());
    return 2;
  } catch (const ConvergenceFailure& e) {
    fill(err, 3, 0.0, e.what());
    return 3;
  } catch (const NonFiniteIntermediate& e) {
    fill(err, 4, 0.0, e.what());
    return 4;
  } catch (const InternalInconsistency& e) {
    fill(err, 5, 0.0, e.what());
    return 5;
  } catch (const ConfigError& e) {
    fill(err, 6, 0.0, e.what());
    return 6;
  } catch (const IndexOutOfRange& e) {
    fill(err, 7, 0.0, e.what());
    return 7;
  } catch (const SignRecoveryFailure& e) {
    fill(err, 8, 0.0, e.what());
    return 8;
  } catch (const DimensionMismatch& e) {
    fill(err, 9, 0.0, e.what());
    return 9;
  } catch (const std::exception& e) {
    fill(err, 29, 0.0, e.what());
    return 29;
  }
}

SymmetricMatrix wrap(const double* a, std::size_t n) {
  return SymmetricMatrix::build(n, std::vector<double>(a, a + n * n),
                                SymmetryPolicy::kStrict);
}

IdentityEngine make_engine(std::size_t batch, std::size_t workers, double tol,
                           int log_domain) {
  IdentityConfig cfg;
  cfg.batch_size = batch;
  cfg.workers = workers;
  cfg.degeneracy_tol = tol;
  if (log_domain) cfg.evaluation = IdentityConfig::Evaluation::kLogDomain;
  return IdentityEngine(cfg);
}

}  // namespace

extern "C" {

void ref_random_symmetric(uint64_t seed, std::size_t n, int uniform,
                          double* out) {
  auto a = random_symmetric(seed, n,
                            uniform ? RandomDistribution::kUniform
                                    : RandomDistribution::kGaussian);
  std::memcpy(out, a.entries().data(), n * n * sizeof(double));
}

void ref_tridiagonalize(const double* a, std::size_t n, double* d,
                        double* off) {
  auto t = tridiagonalize(wrap(a, n));
  std::memcpy(d, t.diag.data(), n * sizeof(double));
  if (n > 1) std::memcpy(off, t.offdiag.data(), (n - 1) * sizeof(double));
}

int ref_eigenvalues(const double* a, std::size_t n, double* out,
                    RefErr* err) {
  return guarded(err, [&] {
    auto s = eigenvalues(wrap(a, n));
    std::memcpy(out, s.values.data(), n * sizeof(double));
  });
}

int ref_all_magnitudes(const double* a, std::size_t n, std::size_t batch,
                       std::size_t workers, double tol, int log_domain,
                       double* out, std::size_t* solves, RefErr* err) {
  return guarded(err, [&] {
    auto engine = make_engine(batch, workers, tol, log_domain);
    auto m = engine.all_magnitudes(wrap(a, n));
    std::memcpy(out, m.data(), n * n * sizeof(double));
    if (solves) *solves = engine.eigenvalue_solve_count();
  });
}

// component_magnitude with cached spectra (identity.cpp:240-251), the
// reference's identity-only entry.  Only a.n() of the matrix is consulted, so
// a diagonal dummy of size n is built once per n and cached.
int ref_component_magnitude_cached(std::size_t n, std::size_t i, std::size_t j,
                                   const double* lambda, const double* mu,
                                   std::size_t batch, double tol,
                                   double* value, double* raw, int* method,
                                   RefErr* err) {
  static std::mutex mu_lock;
  static std::unique_ptr<SymmetricMatrix> dummy;
  return guarded(err, [&] {
    const SymmetricMatrix* a;
    {
      std::lock_guard<std::mutex> g(mu_lock);
      if (!dummy || dummy->n() != n) {
        std::vector<double> d(n);
        for (std::size_t k = 0; k < n; ++k) d[k] = static_cast<double>(k);
        dummy = std::make_unique<SymmetricMatrix>(SymmetricMatrix::diagonal(d));
      }
      a = dummy.get();
    }
    auto engine = make_engine(batch, 1, tol, 0);
    Spectrum sa{std::vector<double>(lambda, lambda + n)};
    Spectrum sm{std::vector<double>(mu, mu + n - 1)};
    auto r = engine.component_magnitude(*a, i, j, &sa, &sm);
    *value = r.value;
    *raw = r.raw_value;
    *method = static_cast<int>(r.method);
  });
}

// Minor spectra for a list of minor indices on the reference's own
// ThreadPool, exactly the fan-out of all_magnitudes (identity.cpp:303-306).
int ref_minor_spectra(const double* a, std::size_t n, const std::size_t* js,
                      std::size_t count, std::size_t workers, double* mu,
                      RefErr* err) {
  return guarded(err, [&] {
    auto m = wrap(a, n);
    ThreadPool pool(workers);
    pool.parallel_for(count, [&](std::size_t r) {
      auto s = eigenvalues(m.minor_matrix(js[r]));
      std::memcpy(mu + r * (n - 1), s.values.data(),
                  (n - 1) * sizeof(double));
    });
  });
}

// Identity stage for whole columns j from cached spectra, one 1-worker engine
// per pool thread (avoids per-component pool dispatch).
int ref_identity_rows(const double* lambda, const double* mu, std::size_t n,
                      std::size_t rows, std::size_t batch, double tol,
                      std::size_t workers, double* out, RefErr* err) {
  return guarded(err, [&] {
    std::vector<double> dd(n);
    for (std::size_t k = 0; k < n; ++k) dd[k] = static_cast<double>(k);
    const auto a = SymmetricMatrix::diagonal(dd);
    const Spectrum sa{std::vector<double>(lambda, lambda + n)};
    ThreadPool pool(workers);
    pool.parallel_for(rows, [&](std::size_t r) {
      auto engine = make_engine(batch, 1, tol, 0);
      const Spectrum sm{std::vector<double>(mu + r * (n - 1),
                                            mu + (r + 1) * (n - 1))};
      for (std::size_t i = 0; i < n; ++i)
        out[r * n + i] = engine.component_magnitude(a, i, r % n, &sa, &sm).value;
    });
  });
}

int ref_jacobi(const double* a, std::size_t n, double* evals, double* evecs,
               RefErr* err) {
  return guarded(err, [&] {
    auto dec = jacobi_eigendecomposition(wrap(a, n));
    std::memcpy(evals, dec.spectrum.values.data(), n * sizeof(double));
    if (evecs) std::memcpy(evecs, dec.vectors.data(), n * n * sizeof(double));
  });
}

// recover_signs (signs.cpp:48-120): signed eigenvector i from magnitudes.
int ref_recover_signs(const double* a, std::size_t n, std::size_t i,
                      const double* mags, std::size_t nmags, double lambda_i,
                      double sign_tol, double* out, RefErr* err) {
  return guarded(err, [&] {
    const auto v = recover_signs(wrap(a, n), i, std::vector<double>(mags, mags + nmags),
                                 lambda_i, sign_tol);
    std::memcpy(out, v.data(), n * sizeof(double));
  });
}

}  // extern "C"
