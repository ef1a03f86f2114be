#pragma once
// fsvd drop-in: decoder shape configuration.
//
// ModelConfig and its validation rules follow the reference
// proj/include/fsvd/model.hpp:18-29 and proj/src/model.cpp:11-25; the
// "desk"/"bench" presets are the reference's (model.cpp:29-32). The
// LLaMA-shaped presets are the B200 benchmark shapes named in BASELINE.json.

#include <array>
#include <cstddef>
#include <span>
#include <string>

#include "fsvd/tensor.hpp"

namespace fsvd {

struct ModelConfig {
    size_t n_layers = 0;
    size_t d_model = 0;
    size_t n_heads = 0;
    size_t d_head = 0;  // d_model / n_heads, even
    size_t d_ff = 0;
    size_t vocab = 0;
    double rope_base = 10000.0;
    double norm_eps = 1e-5;

    void validate() const;
};

struct Preset {
    std::string name;
    ModelConfig config;
    size_t capacity;
};

// desk, bench (reference presets), tiny (BASELINE config 1), llama7b, llama13b.
const Preset& preset(const std::string& name);
std::span<const Preset> presets();

inline constexpr const char* kProjNames[7] = {"q", "k", "v", "o", "up", "gate", "down"};
inline constexpr size_t kNumProj = 7;
enum ProjIndex : size_t { kQ = 0, kK, kV, kO, kUp, kGate, kDown };

// (d_in, d_out) of projection `proj` (index into kProjNames).
inline std::array<size_t, 2> proj_dims(const ModelConfig& c, size_t proj) {
    if (proj == kUp || proj == kGate) return {c.d_model, c.d_ff};
    if (proj == kDown) return {c.d_ff, c.d_model};
    return {c.d_model, c.d_model};
}

}  // namespace fsvd
