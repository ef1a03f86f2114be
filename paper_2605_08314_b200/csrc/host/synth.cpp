// Synthetic factorized checkpoints: layout (names, shapes, ranks, stream
// offsets) and host materialization. See include/fsvd/synth.hpp for the
// stream definition shared with the device generator (csrc/cuda/synth.cu).
#include <algorithm>
#include <cmath>
#include <thread>

#include "fsvd/compress.hpp"
#include "fsvd/synth.hpp"

namespace fsvd {

const SynthTensor* SynthLayout::find(const std::string& name) const {
    for (const auto& t : tensors)
        if (t.name == name) return &t;
    return nullptr;
}

SynthLayout synth_layout(const SynthSpec& s) {
    const ModelConfig& c = s.config;
    c.validate();
    if (s.family < 'A' || s.family > 'D') throw ConfigError("synthetic family must be A, B, C or D");
    if (s.family == 'C' && (s.group_size == 0 || c.n_layers % s.group_size != 0))
        throw ConfigError("group_size must divide n_layers");

    SynthLayout out;
    // Per-(layer, projection) ranks. Families B and D get deterministic jitter
    // from a side stream so ranks are heterogeneous like SVD-LLM v2 / Dobi.
    Rng64 jitter_rng(s.seed ^ 0xD1B54A32D192ED03ull);
    out.ranks.resize(c.n_layers);
    for (size_t li = 0; li < c.n_layers; ++li)
        for (size_t p = 0; p < kNumProj; ++p) {
            const auto [d_in, d_out] = proj_dims(c, p);
            size_t r = rank_for_ratio(s.rho, d_in, d_out);
            const double u = jitter_rng.next_unit();
            if ((s.family == 'B' || s.family == 'D') && s.rank_jitter > 0.0) {
                long long rj = std::llround(static_cast<double>(r) * (1.0 + s.rank_jitter * (2.0 * u - 1.0)));
                rj = std::clamp<long long>(rj, 1, static_cast<long long>(std::min(d_in, d_out)));
                r = static_cast<size_t>(rj);
            }
            out.ranks[li][p] = r;
        }

    uint64_t cursor = 0;
    auto push = [&](std::string name, std::vector<size_t> shape, double amp,
                    SynthTensor::Kind kind = SynthTensor::kUniform) {
        SynthTensor t;
        t.name = std::move(name);
        t.shape = std::move(shape);
        t.stream_offset = cursor;
        t.amp = amp;
        t.kind = kind;
        cursor += t.count();
        out.tensors.push_back(std::move(t));
    };
    auto fan = [](size_t n) { return std::sqrt(1.0 / static_cast<double>(n)); };

    push("embedding", {c.vocab, c.d_model}, fan(c.vocab));
    for (size_t li = 0; li < c.n_layers; ++li) {
        const std::string base = "layers." + std::to_string(li) + ".";
        for (size_t p = 0; p < kNumProj; ++p) {
            const auto [d_in, d_out] = proj_dims(c, p);
            const size_t r = out.ranks[li][p];
            const std::string pb = base + kProjNames[p];
            switch (s.family) {
                case 'A':
                    push(pb + ".A", {d_in, r}, fan(d_in));
                    push(pb + ".B", {r, d_out}, fan(r));
                    break;
                case 'B':
                    push(pb + ".Uf", {d_in, r}, fan(d_in));
                    push(pb + ".Vt", {r, d_out}, fan(r));
                    push(pb + ".scale", {d_in}, 0.0, SynthTensor::kPositive);
                    break;
                case 'C':
                    if (li % s.group_size == 0)
                        push(std::string("shared.") + kProjNames[p] + "." + std::to_string(li / s.group_size) + ".A",
                             {d_in, r}, fan(d_in));
                    push(pb + ".B", {r, d_out}, fan(r));
                    break;
                default:  // 'D'
                    push(pb + ".U", {d_in, r}, fan(d_in));
                    push(pb + ".S", {r}, 0.0, SynthTensor::kPositive);
                    push(pb + ".Vt", {r, d_out}, fan(r));
                    break;
            }
        }
        if (s.conditioned) {
            push(base + "attn_gamma", {c.d_model}, 0.1, SynthTensor::kOnePlus);
            push(base + "mlp_gamma", {c.d_model}, 0.1, SynthTensor::kOnePlus);
        } else {
            push(base + "attn_gamma", {c.d_model}, fan(c.d_model));
            push(base + "mlp_gamma", {c.d_model}, fan(c.d_model));
        }
    }
    if (s.conditioned)
        push("final_gamma", {c.d_model}, 0.1, SynthTensor::kOnePlus);
    else
        push("final_gamma", {c.d_model}, fan(c.d_model));
    push("head", {c.d_model, c.vocab}, fan(c.d_model));
    out.total_draws = cursor;

    auto& h = out.header;
    h["family"] = std::string(1, s.family);
    {
        nlohmann::ordered_json cj;
        cj["n_layers"] = c.n_layers;
        cj["d_model"] = c.d_model;
        cj["n_heads"] = c.n_heads;
        cj["d_head"] = c.d_head;
        cj["d_ff"] = c.d_ff;
        cj["vocab"] = c.vocab;
        cj["rope_base"] = c.rope_base;
        cj["norm_eps"] = c.norm_eps;
        h["config"] = std::move(cj);
    }
    h["capacity"] = s.capacity;
    h["retained_ratio"] = s.rho;
    if (s.family == 'C') {
        h["group_size"] = s.group_size;
        std::vector<size_t> groups(c.n_layers);
        for (size_t li = 0; li < c.n_layers; ++li) groups[li] = li / s.group_size;
        h["layer_groups"] = groups;
    }
    nlohmann::ordered_json syn;
    syn["seed"] = s.seed;
    syn["conditioned"] = s.conditioned;
    syn["rank_jitter"] = s.rank_jitter;
    h["synthetic"] = std::move(syn);
    return out;
}

Checkpoint make_synthetic_checkpoint(const SynthSpec& spec) {
    SynthLayout lay = synth_layout(spec);
    Checkpoint ck;
    ck.header = lay.header;
    for (const auto& t : lay.tensors) ck.add(t.name, t.shape);
    // Fill every tensor; work split in fixed slices so the result does not
    // depend on the thread count (each element is a pure function of its
    // stream index anyway).
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (unsigned w = 0; w < hw; ++w)
        pool.emplace_back([&, w] {
            for (size_t ti = 0; ti < lay.tensors.size(); ++ti) {
                const SynthTensor& t = lay.tensors[ti];
                float* dst = ck.tensors[ti].data.data();
                const size_t n = t.count();
                const size_t lo = n * w / hw, hi = n * (w + 1) / hw;
                for (size_t i = lo; i < hi; ++i) dst[i] = synth_value(spec.seed, t, i);
            }
        });
    for (auto& th : pool) th.join();
    return ck;
}

}  // namespace fsvd
