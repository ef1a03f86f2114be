#pragma once
// fsvd drop-in: the part of the reference compressor the serving path needs.
//
// Only rank_for_ratio (reference proj/src/compress.cpp:68-80) is on the hot
// path: it sizes every factor of the synthetic benchmark checkpoints. The SVD
// compressors themselves are offline tooling and out of scope.

#include <cstddef>
#include <stdexcept>
#include <string>

namespace fsvd {

struct CalibrationError : std::runtime_error {
    explicit CalibrationError(const std::string& what) : std::runtime_error(what) {}
};

// r = clamp(round(rho * m * n / (m + n)), 1, min(m, n)); rho == 1 -> min(m, n).
size_t rank_for_ratio(double rho, size_t m, size_t n);

}  // namespace fsvd
