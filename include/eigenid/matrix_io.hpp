// eigenid/matrix_io.hpp — the seeded generator of the reference
// (matrix_io.hpp:15-42, matrix_io.cpp:39-71,171-187): mt19937_64 draws,
// Box-Muller Gaussian or uniform(-1, 1), symmetrised by build(kSymmetrize);
// bit-identical to the reference for a fixed (seed, distribution, n).  The
// reference's CSV / Matrix Market file I/O is out of scope.
#pragma once

#include <cstdint>

#include "eigenid/matrix.hpp"

namespace eigenid {

enum class RandomDistribution {
  kGaussian,
  kUniform,  // uniform on (-1, 1)
};

SymmetricMatrix random_symmetric(std::uint64_t seed, std::size_t n,
                                 RandomDistribution dist =
                                     RandomDistribution::kGaussian);

}  // namespace eigenid
