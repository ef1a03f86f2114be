#pragma once
// Synthetic random-init factorized checkpoints (benchmark + parity inputs).
//
// There are no public LLaMA SVD checkpoints in this environment, so the
// benchmark shapes are filled from one seeded SplitMix64 stream, following the
// reference's toy-model conventions (proj/src/model.cpp:34-46, :75-111):
// values uniform in [-a, a] with a = sqrt(1/fan_in), drawn in a fixed tensor
// order, rounded to f32 -- and additionally rounded to bf16 (RNE) so the fp32
// mode, the bf16 mode and the CPU oracle all see the same weights for families
// A and C. Ranks come from rank_for_ratio (proj/src/compress.cpp:68-80), with
// optional deterministic per-(layer, projection) jitter for the heterogeneous
// rank families (B: SVD-LLM v2, D: activation-truncated).
//
// Draw order (one stream, element k of the whole stream = Rng64::mix(seed +
// (k+1) * golden), so any element can be regenerated independently -- the
// device generator in csrc/cuda/synth.cu relies on this):
//   embedding [V x d] (fan_in V)
//   per layer, per projection q,k,v,o,up,gate,down:
//     A: [A d_in x r (fan_in d_in)] [B r x d_out (fan_in r)]
//     B: [Uf d_in x r] [Vt r x d_out] [scale d_in, in [0.5,1.5)]
//     C: [shared.{p}.{g}.A d_in x r, only at the first layer of group g] [B]
//     D: [U d_in x r] [S r, in [0.5,1.5)] [Vt r x d_out]
//   per layer: attn_gamma [d], mlp_gamma [d]   (fan_in d, or 1 + U(+-0.1)
//                                               when `conditioned`)
//   final_gamma [d], head [d x V] (fan_in d)

#include <array>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "fsvd/checkpoint.hpp"
#include "fsvd/model.hpp"

namespace fsvd {

struct SynthSpec {
    ModelConfig config;
    size_t capacity = 0;
    char family = 'A';        // 'A' | 'B' | 'C' | 'D'
    double rho = 0.6;         // retained parameter ratio
    size_t group_size = 2;    // family C: layers per shared basis
    uint64_t seed = 1;
    bool conditioned = false; // gammas ~ 1 + U(+-0.1) instead of U(+-sqrt(1/d))
    double rank_jitter = 0.0; // families B/D: r *= 1 + jitter * U(-1, 1)
};

struct SynthTensor {
    enum Kind : int { kUniform = 0, kOnePlus = 1, kPositive = 2 };
    std::string name;
    std::vector<size_t> shape;
    uint64_t stream_offset = 0;  // index of the tensor's first draw in the stream
    double amp = 0.0;            // a of U(-a, a)
    Kind kind = kUniform;

    size_t count() const {
        size_t n = 1;
        for (size_t d : shape) n *= d;
        return n;
    }
};

struct SynthLayout {
    std::vector<SynthTensor> tensors;   // in draw order
    std::vector<std::array<size_t, kNumProj>> ranks;  // [layer][proj]
    nlohmann::ordered_json header;      // family, config, capacity, ...
    uint64_t total_draws = 0;

    const SynthTensor* find(const std::string& name) const;
};

SynthLayout synth_layout(const SynthSpec& spec);

// Round-to-nearest-even to the closest bf16-representable float.
inline float round_bf16(float x) {
    uint32_t u;
    std::memcpy(&u, &x, 4);
    if ((u & 0x7F800000u) == 0x7F800000u) return x;  // inf / nan untouched
    u += 0x7FFFu + ((u >> 16) & 1u);
    u &= 0xFFFF0000u;
    float y;
    std::memcpy(&y, &u, 4);
    return y;
}

// Element i (row-major) of tensor t for the stream seeded with `seed`.
inline float synth_value(uint64_t seed, const SynthTensor& t, uint64_t i) {
    const uint64_t z = Rng64::mix(seed + (t.stream_offset + i + 1) * Rng64::kGolden);
    const double unit = static_cast<double>(z >> 11) * 0x1.0p-53;
    double v;
    switch (t.kind) {
        case SynthTensor::kOnePlus: v = 1.0 + (2.0 * unit - 1.0) * t.amp; break;
        case SynthTensor::kPositive: v = 0.5 + unit; break;
        default: v = (2.0 * unit - 1.0) * t.amp; break;
    }
    return round_bf16(static_cast<float>(v));
}

// Host materialization (multi-threaded over tensors; deterministic).
Checkpoint make_synthetic_checkpoint(const SynthSpec& spec);

}  // namespace fsvd
