#pragma once
// Loader error types of the reference API (checkpoint.hpp:21-23 FormatError,
// canonical.hpp:21-23 NormalizeError), in their own header so the runtime
// wrapper (runtime.hpp) can re-throw them without the JSON dependency.
#include <stdexcept>
#include <string>

namespace fsvd {

struct FormatError : std::runtime_error {
    explicit FormatError(const std::string& what) : std::runtime_error(what) {}
};
struct NormalizeError : std::runtime_error {
    explicit NormalizeError(const std::string& what) : std::runtime_error(what) {}
};

}  // namespace fsvd
