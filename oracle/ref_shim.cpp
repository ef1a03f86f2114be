// C shim over the REFERENCE implementation (compiled from /root/reference by
// oracle/Makefile into oracle/_ref/libfsvd_ref.so) -- TEST INFRASTRUCTURE ONLY.
//
// Exposes the reference's own primitives, loader, toy-model generator,
// compressor and dense gold forward to the Python tests so the restated oracle
// (fsvd_oracle.cpp) and the product loader are pinned against the real thing,
// and so tests/golden/make_golden.py can freeze reference outputs as fixtures
// (the GPU box has no /root/reference). Nothing here is reference source; it
// only calls the reference API.
#include <cstring>
#include <string>
#include <vector>

#include "fsvd/canonical.hpp"
#include "fsvd/checkpoint.hpp"
#include "fsvd/compress.hpp"
#include "fsvd/kernels.hpp"
#include "fsvd/math.hpp"
#include "fsvd/model.hpp"

using namespace fsvd;

namespace {
thread_local std::string g_err;
template <typename F>
int wrap(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}
ModelConfig cfg_of(const uint64_t* c6, const double* c2) {
    ModelConfig c;
    c.n_layers = c6[0];
    c.d_model = c6[1];
    c.n_heads = c6[2];
    c.d_head = c6[3];
    c.d_ff = c6[4];
    c.vocab = c6[5];
    c.rope_base = c2[0];
    c.norm_eps = c2[1];
    return c;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
int ref_force_variant(const char* name) { return kern::force_variant(name) ? 1 : 0; }
const char* ref_active_variant() { return kern::active().name; }
void* ref_gemv_f32_ptr() { return reinterpret_cast<void*>(kern::ops<float>().gemv); }

void ref_gemv_f32(float* y, const float* x, const float* a, uint64_t m, uint64_t n) {
    kern::ops<float>().gemv(y, x, a, m, n);
}
void ref_gemv_f64(double* y, const double* x, const double* a, uint64_t m, uint64_t n) {
    kern::ops<double>().gemv(y, x, a, m, n);
}
void ref_rmsnorm_f64(double* y, const double* x, const double* g, uint64_t n, double eps) {
    const auto out = rmsnorm<double>(std::span<const double>(x, n), std::span<const double>(g, n), eps);
    std::memcpy(y, out.data(), n * 8);
}
void ref_rmsnorm_f32(float* y, const float* x, const float* g, uint64_t n, float eps) {
    const auto out = rmsnorm<float>(std::span<const float>(x, n), std::span<const float>(g, n), eps);
    std::memcpy(y, out.data(), n * 4);
}
void ref_rope_f64(double* v, uint64_t d, double pos, double base) { rope_inplace<double>(v, d, pos, base); }
void ref_rope_f32(float* v, uint64_t d, double pos, double base) { rope_inplace<float>(v, d, pos, base); }

int ref_online_attend_f64(const double* q, const double* k, const double* v, uint64_t d, double scale,
                          const uint64_t* blocks, uint64_t nblocks, double* out) {
    return wrap([&] {
        std::vector<std::pair<Tensor2Dd, Tensor2Dd>> bl;
        size_t r0 = 0;
        for (size_t b = 0; b < nblocks; ++b) {
            std::vector<double> kb(k + r0 * d, k + (r0 + blocks[b]) * d), vb(v + r0 * d, v + (r0 + blocks[b]) * d);
            bl.emplace_back(Tensor2Dd(blocks[b], d, kb), Tensor2Dd(blocks[b], d, vb));
            r0 += blocks[b];
        }
        const auto o = online_softmax_attend<double>(std::span<const double>(q, d),
                                                     std::span<const std::pair<Tensor2Dd, Tensor2Dd>>(bl), scale);
        std::memcpy(out, o.data(), d * 8);
    });
}

uint64_t ref_argmax_f64(const double* x, uint64_t n) { return argmax_greedy<double>(std::span<const double>(x, n)); }

uint64_t ref_rng_u64(uint64_t seed, uint64_t k) {
    Rng64 r(seed);
    uint64_t v = 0;
    for (uint64_t i = 0; i <= k; ++i) v = r.next_u64();
    return v;
}
uint64_t ref_rank_for_ratio(double rho, uint64_t m, uint64_t n) { return rank_for_ratio(rho, m, n); }

int ref_dense_checksum(const uint64_t* c6, const double* c2, uint64_t seed, uint32_t* out) {
    return wrap([&] { *out = dense_model_checksum(generate_toy_dense(cfg_of(c6, c2), seed)); });
}

// generate_toy_dense + compress (A plain, B whitened, C basis-shared) -> file
int ref_compress_to_file(const uint64_t* c6, const double* c2, uint64_t capacity, uint64_t seed, char family,
                         double rho, uint64_t group, const char* path) {
    return wrap([&] {
        const DenseModel dm = generate_toy_dense(cfg_of(c6, c2), seed);
        CompressionSpec spec;
        spec.retained_ratio = rho;
        spec.group_size = group;
        spec.method = family == 'A' ? CompressMethod::plain
                                    : (family == 'B' ? CompressMethod::whitened : CompressMethod::basis_shared);
        write_checkpoint_file(compress(dm, spec, capacity), path);
    });
}

int ref_dense_forward_all(const uint64_t* c6, const double* c2, uint64_t seed, const int32_t* tok, uint64_t T,
                          double* out) {
    return wrap([&] {
        const DenseModel dm = generate_toy_dense(cfg_of(c6, c2), seed);
        std::vector<int> t(tok, tok + T);
        const Tensor2Dd lg = dense_forward_all(dm, t);
        std::memcpy(out, lg.data.data(), lg.data.size() * 8);
    });
}

int ref_normalize_tensor(const char* path, const char* name, float* out, uint64_t count) {
    return wrap([&] {
        const CanonicalModel<float> m = normalize<float>(read_checkpoint_file(path));
        const std::string n(name);
        const std::vector<float>* v = nullptr;
        if (n == "embedding") v = &m.embedding.data;
        else if (n == "head") v = &m.head.data;
        else if (n == "final_gamma") v = &m.final_gamma;
        else {
            const size_t d1 = n.find('.', 7);
            const size_t l = std::stoul(n.substr(7, d1 - 7));
            const std::string rest = n.substr(d1 + 1);
            const auto& L = m.layers.at(l);
            if (rest == "attn_gamma") v = &L.attn_gamma;
            else if (rest == "mlp_gamma") v = &L.mlp_gamma;
            else if (rest == "a_ug") v = &L.a_ug.data;
            else
                for (size_t p = 0; p < 7; ++p) {
                    if (rest == std::string(kProjNames[p]) + ".A") v = &L.proj(p).a->data;
                    if (rest == std::string(kProjNames[p]) + ".B") v = &L.proj(p).b->data;
                }
        }
        if (!v || v->size() != count) throw std::runtime_error("bad tensor request " + n);
        std::memcpy(out, v->data(), count * 4);
    });
}

int ref_shared_count(const char* path, uint64_t* out) {
    return wrap([&] { *out = normalize<float>(read_checkpoint_file(path)).shared_basis_table.size(); });
}

// read -> write; returns the rewritten bytes' size and content in out (cap bytes)
int ref_roundtrip(const char* path_in, const char* path_out) {
    return wrap([&] { write_checkpoint_file(read_checkpoint_file(path_in), path_out); });
}

}  // extern "C"
