#pragma once
// fsvd drop-in: core value types shared by the loader and the runtime.
//
// Mirrors the public surface of the reference header proj/include/fsvd/tensor.hpp
// (typed errors :17-31, Rng64 :35-62, Tensor2D :64-92) so existing callers
// compile unchanged. The B200 runtime never computes through Tensor2D; it is
// the host-side carrier between the FSVD15 reader, the normalizer and the
// device upload.

#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace fsvd {

// Error taxonomy (1:1 with the reference; each maps to one fsvd_status code
// in fsvd_c.h so no exception ever crosses the C ABI).
#define FSVD_DECLARE_ERROR(Name)                                              \
    struct Name : std::runtime_error {                                        \
        explicit Name(const std::string& what) : std::runtime_error(what) {}  \
    }
FSVD_DECLARE_ERROR(ShapeError);
FSVD_DECLARE_ERROR(RankError);
FSVD_DECLARE_ERROR(NumericError);
FSVD_DECLARE_ERROR(CapacityError);
FSVD_DECLARE_ERROR(ConfigError);
#undef FSVD_DECLARE_ERROR

// SplitMix64 stream. The k-th output (k = 1, 2, ...) of a stream seeded with
// s is mix(s + k * golden), which is what lets the device-side synthetic
// weight generator reproduce any stream position without walking the stream.
struct Rng64 {
    static constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
    uint64_t state = 0;

    explicit Rng64(uint64_t seed) : state(seed) {}

    static constexpr uint64_t mix(uint64_t z) {
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    uint64_t next_u64() {
        state += kGolden;
        return mix(state);
    }
    // [0,1) from the top 53 bits.
    double next_unit() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    // [-a, a]
    double next_symmetric(double a) { return (2.0 * next_unit() - 1.0) * a; }
    // [0, n)
    uint64_t next_below(uint64_t n) {
        return static_cast<uint64_t>(next_unit() * static_cast<double>(n));
    }
};

// Row-major dense matrix (host side only).
template <typename T>
struct Tensor2D {
    size_t rows = 0;
    size_t cols = 0;
    std::vector<T> data;

    Tensor2D() = default;
    Tensor2D(size_t r, size_t c) : rows(r), cols(c) {
        if (r == 0 || c == 0)
            throw ShapeError("Tensor2D: zero dimension " + std::to_string(r) + "x" +
                             std::to_string(c));
        data.assign(r * c, T(0));
    }
    Tensor2D(size_t r, size_t c, std::vector<T> values)
        : rows(r), cols(c), data(std::move(values)) {
        if (r == 0 || c == 0 || data.size() != r * c)
            throw ShapeError("Tensor2D: value count does not match " +
                             std::to_string(r) + "x" + std::to_string(c));
    }

    T& at(size_t i, size_t j) { return data[i * cols + j]; }
    const T& at(size_t i, size_t j) const { return data[i * cols + j]; }
    std::span<T> row(size_t i) { return {data.data() + i * cols, cols}; }
    std::span<const T> row(size_t i) const { return {data.data() + i * cols, cols}; }
    size_t size() const { return data.size(); }
};

using Tensor2Df = Tensor2D<float>;
using Tensor2Dd = Tensor2D<double>;

}  // namespace fsvd
