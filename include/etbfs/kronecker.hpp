// Drop-in: Kronecker generator (reference: proj/include/etbfs/kronecker.hpp:12-34).
// Runs on the GPU (etb_generate_kronecker); byte-identical tuples.
#pragma once

#include <cstdint>

#include "etbfs/types.hpp"

namespace etbfs {

struct KroneckerParams {
  std::uint32_t scale = 0;
  std::uint64_t edgefactor = 16;
  double a = 0.57;
  double b = 0.19;
  double c = 0.19;
  double d = 0.05;
  std::uint64_t seed = 0;
};

// 2^scale * edgefactor tuples, tuple i seeded by seed ^ i*0x2545f4914f6cdd1d,
// no label scrambling. Throws std::invalid_argument / std::runtime_error with
// the reference's messages.
EdgeList generate_kronecker(const KroneckerParams& params);

}  // namespace etbfs
