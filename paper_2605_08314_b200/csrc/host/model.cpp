// ModelConfig validation, presets and rank sizing.
// Follows reference proj/src/model.cpp:11-32 (validate, presets) and
// proj/src/compress.cpp:68-80 (rank_for_ratio).
#include <array>
#include <cmath>

#include "fsvd/compress.hpp"
#include "fsvd/model.hpp"

namespace fsvd {

void ModelConfig::validate() const {
    const size_t counts[] = {n_layers, d_model, n_heads, d_head, d_ff, vocab};
    for (size_t c : counts)
        if (c == 0) throw ConfigError("ModelConfig: all counts must be >= 1");
    if (n_heads * d_head != d_model)
        throw ConfigError("ModelConfig: d_model (" + std::to_string(d_model) +
                          ") != n_heads * d_head (" + std::to_string(n_heads * d_head) + ")");
    if (d_head & 1) throw ConfigError("ModelConfig: d_head must be even");
    if (!(rope_base > 0.0) || !(norm_eps > 0.0))
        throw ConfigError("ModelConfig: rope_base and norm_eps must be positive");
}

namespace {
const std::array<Preset, 5> kPresetTable = {{
    // reference presets (model.cpp:29-32)
    {"desk", {4, 256, 8, 32, 1024, 1024, 10000.0, 1e-5}, 8192},
    {"bench", {8, 512, 8, 64, 2048, 4096, 10000.0, 1e-5}, 8192},
    // BASELINE.json config 1: tiny LLaMA-style decoder, 4 heads
    {"tiny", {4, 256, 4, 64, 1024, 1024, 10000.0, 1e-5}, 8192},
    // LLaMA-7B / 13B shapes (BASELINE.json configs 2-5)
    {"llama7b", {32, 4096, 32, 128, 11008, 32000, 10000.0, 1e-5}, 8192},
    {"llama13b", {40, 5120, 40, 128, 13824, 32000, 10000.0, 1e-5}, 8192},
}};
}  // namespace

const Preset& preset(const std::string& name) {
    for (const Preset& p : kPresetTable)
        if (p.name == name) return p;
    throw ConfigError("unknown preset '" + name + "' (desk|bench|tiny|llama7b|llama13b)");
}

std::span<const Preset> presets() { return {kPresetTable.data(), kPresetTable.size()}; }

size_t rank_for_ratio(double rho, size_t m, size_t n) {
    if (!(rho > 0.0) || rho > 1.0) throw ConfigError("retained ratio must be in (0, 1]");
    const size_t cap = m < n ? m : n;
    if (rho >= 1.0) return cap;
    const long long r = std::llround(rho * static_cast<double>(m) * static_cast<double>(n) /
                                     static_cast<double>(m + n));
    if (r < 1) return 1;
    return static_cast<size_t>(r) > cap ? cap : static_cast<size_t>(r);
}

}  // namespace fsvd
