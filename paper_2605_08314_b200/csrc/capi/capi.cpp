// extern "C" boundary (include/fsvd_c.h): exception -> status mapping,
// host<->device copies for the host-pointer entry points.
#include <cstdlib>
#include <cstring>
#include <string>

#include "../host/runtime.h"
#include "fsvd/canonical.hpp"
#include "fsvd/compress.hpp"
#include "fsvd/synth.hpp"
#include "fsvd_c.h"

struct fsvd_canonical {
    fsvd::CanonicalModel<float> m;
};
struct fsvd_model {
    std::unique_ptr<fsvd::rt::DeviceModel> dm;
};
struct fsvd_session {
    std::unique_ptr<fsvd::rt::Session> s;
    fsvd_model* model;
};

namespace {

thread_local std::string g_last_error;
thread_local fsvd::rt::LoadStats g_last_load;

template <typename F>
fsvd_status guarded(F&& f) {
    try {
        f();
        g_last_error.clear();
        return FSVD_OK;
    } catch (const fsvd::ShapeError& e) {
        g_last_error = e.what();
        return FSVD_ERR_SHAPE;
    } catch (const fsvd::RankError& e) {
        g_last_error = e.what();
        return FSVD_ERR_RANK;
    } catch (const fsvd::NumericError& e) {
        g_last_error = e.what();
        return FSVD_ERR_NUMERIC;
    } catch (const fsvd::CapacityError& e) {
        g_last_error = e.what();
        return FSVD_ERR_CAPACITY;
    } catch (const fsvd::ConfigError& e) {
        g_last_error = e.what();
        return FSVD_ERR_CONFIG;
    } catch (const fsvd::FormatError& e) {
        g_last_error = e.what();
        return FSVD_ERR_FORMAT;
    } catch (const fsvd::NormalizeError& e) {
        g_last_error = e.what();
        return FSVD_ERR_NORMALIZE;
    } catch (const fsvd::CalibrationError& e) {
        g_last_error = e.what();
        return FSVD_ERR_CALIBRATION;
    } catch (const fsvd::rt::CudaError& e) {
        g_last_error = e.what();
        return FSVD_ERR_CUDA;
    } catch (const fsvd::rt::OomError& e) {
        g_last_error = e.what();
        return FSVD_ERR_OOM;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return FSVD_ERR_OOM;
    } catch (const std::invalid_argument& e) {
        g_last_error = e.what();
        return FSVD_ERR_INVALID;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return FSVD_ERR_INTERNAL;
    } catch (...) {
        g_last_error = "unknown error";
        return FSVD_ERR_INTERNAL;
    }
}

void need(const void* p, const char* what) {
    if (!p) throw std::invalid_argument(std::string(what) + " is null");
}

fsvd::ModelConfig to_cfg(const fsvd_config& c) {
    fsvd::ModelConfig m;
    m.n_layers = c.n_layers;
    m.d_model = c.d_model;
    m.n_heads = c.n_heads;
    m.d_head = c.d_head;
    m.d_ff = c.d_ff;
    m.vocab = c.vocab;
    m.rope_base = c.rope_base;
    m.norm_eps = c.norm_eps;
    return m;
}

fsvd_config from_cfg(const fsvd::ModelConfig& m) {
    return {m.n_layers, m.d_model, m.n_heads, m.d_head, m.d_ff, m.vocab, m.rope_base, m.norm_eps};
}

fsvd::SynthSpec to_spec(const fsvd_synth_spec* s) {
    fsvd::SynthSpec o;
    o.config = to_cfg(s->config);
    o.capacity = s->capacity;
    o.family = s->family;
    o.rho = s->rho;
    o.group_size = s->group_size;
    o.seed = s->seed;
    o.conditioned = s->conditioned != 0;
    o.rank_jitter = s->rank_jitter;
    return o;
}

void check_dtype(fsvd_dtype d) {
    if (d != FSVD_DTYPE_F32 && d != FSVD_DTYPE_BF16) throw std::invalid_argument("unknown dtype");
}

// Parse "layers.{i}.{rest}" -> (i, rest)
bool parse_layer(const std::string& name, size_t& layer, std::string& rest) {
    if (name.rfind("layers.", 0) != 0) return false;
    const size_t dot = name.find('.', 7);
    if (dot == std::string::npos) return false;
    layer = std::stoul(name.substr(7, dot - 7));
    rest = name.substr(dot + 1);
    return true;
}

}  // namespace

extern "C" {

const char* fsvd_last_error(void) { return g_last_error.c_str(); }
const char* fsvd_version(void) { return "fsvd-b200 0.1 (sm_100a)"; }

// ------------------------------------------------------------ host loader --
fsvd_status fsvd_canonical_load_file(const char* path, fsvd_canonical** out) {
    return guarded([&] {
        need(path, "path");
        need(out, "out");
        auto c = std::make_unique<fsvd_canonical>();
        c->m = fsvd::normalize<float>(fsvd::read_checkpoint_file(path));
        *out = c.release();
    });
}

fsvd_status fsvd_canonical_load_bytes(const uint8_t* bytes, size_t len, fsvd_canonical** out) {
    return guarded([&] {
        need(bytes, "bytes");
        need(out, "out");
        auto c = std::make_unique<fsvd_canonical>();
        c->m = fsvd::normalize<float>(fsvd::read_checkpoint(bytes, len));
        *out = c.release();
    });
}

fsvd_status fsvd_canonical_synthetic(const fsvd_synth_spec* spec, fsvd_canonical** out) {
    return guarded([&] {
        need(spec, "spec");
        need(out, "out");
        auto c = std::make_unique<fsvd_canonical>();
        c->m = fsvd::normalize<float>(fsvd::make_synthetic_checkpoint(to_spec(spec)));
        *out = c.release();
    });
}

fsvd_status fsvd_canonical_config(const fsvd_canonical* c, fsvd_config* cfg, uint64_t* capacity) {
    return guarded([&] {
        need(c, "canonical");
        if (cfg) *cfg = from_cfg(c->m.config);
        if (capacity) *capacity = c->m.capacity;
    });
}

fsvd_status fsvd_canonical_rank(const fsvd_canonical* c, uint64_t layer, uint32_t proj, uint64_t* rank) {
    return guarded([&] {
        need(c, "canonical");
        need(rank, "rank");
        if (layer >= c->m.layers.size() || proj >= fsvd::kNumProj) throw fsvd::ShapeError("rank: index out of range");
        *rank = c->m.layers[layer].proj(proj).rank;
    });
}

fsvd_status fsvd_canonical_copy(const fsvd_canonical* c, const char* name, float* out, uint64_t count) {
    return guarded([&] {
        need(c, "canonical");
        need(name, "name");
        need(out, "out");
        const auto& m = c->m;
        const std::string n(name);
        const std::vector<float>* vec = nullptr;
        const fsvd::Tensor2D<float>* mat = nullptr;
        if (n == "embedding") mat = &m.embedding;
        else if (n == "head") mat = &m.head;
        else if (n == "final_gamma") vec = &m.final_gamma;
        else {
            size_t li;
            std::string rest;
            if (!parse_layer(n, li, rest) || li >= m.layers.size())
                throw fsvd::ShapeError("unknown canonical tensor '" + n + "'");
            const auto& L = m.layers[li];
            if (rest == "attn_gamma") vec = &L.attn_gamma;
            else if (rest == "mlp_gamma") vec = &L.mlp_gamma;
            else if (rest == "a_ug") mat = &L.a_ug;
            else {
                for (size_t p = 0; p < fsvd::kNumProj; ++p) {
                    const std::string pn = fsvd::kProjNames[p];
                    if (rest == pn + ".A") mat = L.proj(p).a.get();
                    if (rest == pn + ".B") mat = L.proj(p).b.get();
                }
            }
        }
        const std::vector<float>& data = vec ? *vec : (mat ? mat->data : throw fsvd::ShapeError("unknown canonical tensor '" + n + "'"));
        if (data.size() != count)
            throw fsvd::ShapeError("tensor '" + n + "' has " + std::to_string(data.size()) + " elements, caller asked " +
                                   std::to_string(count));
        std::memcpy(out, data.data(), count * sizeof(float));
    });
}

fsvd_status fsvd_canonical_shared_count(const fsvd_canonical* c, uint64_t* n) {
    return guarded([&] {
        need(c, "canonical");
        need(n, "n");
        *n = c->m.shared_basis_table.size();
    });
}

fsvd_status fsvd_canonical_aliased(const fsvd_canonical* c, uint64_t l0, uint64_t l1, uint32_t proj, int32_t* out) {
    return guarded([&] {
        need(c, "canonical");
        need(out, "out");
        if (l0 >= c->m.layers.size() || l1 >= c->m.layers.size() || proj >= fsvd::kNumProj)
            throw fsvd::ShapeError("aliased: index out of range");
        *out = c->m.layers[l0].proj(proj).a.get() == c->m.layers[l1].proj(proj).a.get() ? 1 : 0;
    });
}

fsvd_status fsvd_canonical_destroy(fsvd_canonical* c) {
    return guarded([&] { delete c; });
}

fsvd_status fsvd_canonical_write_file(const fsvd_canonical* c, const char* path) {
    return guarded([&] {
        need(c, "canonical");
        need(path, "path");
        fsvd::write_checkpoint_file(fsvd::export_family_a(c->m), path);
    });
}

fsvd_status fsvd_synthetic_write_file(const fsvd_synth_spec* spec, const char* path) {
    return guarded([&] {
        need(spec, "spec");
        need(path, "path");
        fsvd::write_checkpoint_file(fsvd::make_synthetic_checkpoint(to_spec(spec)), path);
    });
}

// ----------------------------------------------------------- device model --
fsvd_status fsvd_model_load(const char* path, fsvd_dtype dtype, int32_t device, fsvd_model** out) {
    return guarded([&] {
        need(path, "path");
        need(out, "out");
        check_dtype(dtype);
        auto m = std::make_unique<fsvd_model>();
        // streaming loader (no host CanonicalModel); FSVD_LOADER=canonical selects the
        // read_checkpoint_file -> normalize<float> -> upload path (tests compare the two bitwise)
        const char* ld = std::getenv("FSVD_LOADER");
        if (ld && std::string(ld) == "canonical") {
            const auto canon = fsvd::normalize<float>(fsvd::read_checkpoint_file(path));
            m->dm = fsvd::rt::upload_canonical(canon, dtype, device);
        } else {
            fsvd::rt::LoadStats st;
            m->dm = fsvd::rt::load_streaming(path, dtype, device, &st);
            g_last_load = st;
        }
        *out = m.release();
    });
}

fsvd_status fsvd_last_load_stats(double* seconds, uint64_t* payload_bytes, uint64_t* pinned_bytes) {
    return guarded([&] {
        if (seconds) *seconds = g_last_load.seconds;
        if (payload_bytes) *payload_bytes = g_last_load.bytes;
        if (pinned_bytes) *pinned_bytes = g_last_load.pinned_bytes;
    });
}

fsvd_status fsvd_model_from_canonical(const fsvd_canonical* c, fsvd_dtype dtype, int32_t device, fsvd_model** out) {
    return guarded([&] {
        need(c, "canonical");
        need(out, "out");
        check_dtype(dtype);
        auto m = std::make_unique<fsvd_model>();
        m->dm = fsvd::rt::upload_canonical(c->m, dtype, device);
        *out = m.release();
    });
}

fsvd_status fsvd_model_synthetic(const fsvd_synth_spec* spec, fsvd_dtype dtype, int32_t device, fsvd_model** out) {
    return guarded([&] {
        need(spec, "spec");
        need(out, "out");
        check_dtype(dtype);
        auto m = std::make_unique<fsvd_model>();
        m->dm = fsvd::rt::generate_synthetic(to_spec(spec), dtype, device);
        *out = m.release();
    });
}

fsvd_status fsvd_model_info(const fsvd_model* m, fsvd_config* cfg, uint64_t* capacity, uint64_t* weight_bytes,
                            uint64_t* decode_weight_bytes) {
    return guarded([&] {
        need(m, "model");
        if (cfg) *cfg = from_cfg(m->dm->cfg);
        if (capacity) *capacity = m->dm->capacity;
        if (weight_bytes) *weight_bytes = m->dm->stored_weight_bytes;
        if (decode_weight_bytes) *decode_weight_bytes = m->dm->decode_weight_bytes;
    });
}

fsvd_status fsvd_model_copy_factor(const fsvd_model* m, uint64_t layer, uint32_t proj, int32_t which_b, float* out,
                                   uint64_t count) {
    return guarded([&] {
        need(m, "model");
        need(out, "out");
        fsvd::rt::copy_factor(*m->dm, layer, proj, which_b != 0, out, count);
    });
}

fsvd_status fsvd_model_destroy(fsvd_model* m) {
    return guarded([&] { delete m; });
}

// --------------------------------------------------------------- sessions --
fsvd_status fsvd_route_ffn_auto(fsvd_plan_mode plan, fsvd_ffn_backend requested, fsvd_ffn_backend* out) {
    return guarded([&] {
        need(out, "out");
        if (plan < FSVD_PLAN_EAGER || plan > FSVD_PLAN_SPLIT) throw fsvd::ConfigError("unknown plan mode");
        if (requested < FSVD_FFN_AUTO || requested > FSVD_FFN_PACKED) throw fsvd::ConfigError("unknown ffn backend");
        *out = fsvd::rt::route_ffn_auto(plan, requested);
    });
}

fsvd_status fsvd_session_create(fsvd_model* m, const fsvd_session_opts* opts, fsvd_session** out) {
    return guarded([&] {
        need(m, "model");
        need(opts, "opts");
        need(out, "out");
        auto s = std::make_unique<fsvd_session>();
        s->s = std::make_unique<fsvd::rt::Session>(m->dm.get(), *opts);
        s->model = m;
        *out = s.release();
    });
}

fsvd_status fsvd_prefill(fsvd_session* s, const int32_t* tokens, uint64_t T, float* logits_out) {
    return guarded([&] {
        need(s, "session");
        need(tokens, "tokens");
        auto& S = *s->s;
        const size_t B = S.batch(), V = S.vocab();
        if (T == 0) throw fsvd::ShapeError("prefill: empty prompt");
        const size_t tok_bytes = B * T * 4, log_bytes = B * V * 4;
        char* stage = static_cast<char*>(S.staging(tok_bytes + log_bytes + 256));
        int32_t* d_tok = reinterpret_cast<int32_t*>(stage);
        float* d_log = reinterpret_cast<float*>(stage + ((tok_bytes + 255) & ~size_t(255)));
        FSVD_CUDA(cudaMemcpyAsync(d_tok, tokens, tok_bytes, cudaMemcpyHostToDevice, S.stream()));
        S.prefill(d_tok, T, d_log);
        if (logits_out) FSVD_CUDA(cudaMemcpyAsync(logits_out, d_log, log_bytes, cudaMemcpyDeviceToHost, S.stream()));
        FSVD_CUDA(cudaStreamSynchronize(S.stream()));
        S.stats().copy_bytes += tok_bytes + (logits_out ? log_bytes : 0);
    });
}

fsvd_status fsvd_decode_step(fsvd_session* s, const int32_t* tokens, float* logits_out) {
    return guarded([&] {
        need(s, "session");
        need(tokens, "tokens");
        auto& S = *s->s;
        const size_t B = S.batch(), V = S.vocab();
        const size_t tok_bytes = B * 4, log_bytes = B * V * 4;
        int32_t* d_tok = static_cast<int32_t*>(S.staging(tok_bytes));
        FSVD_CUDA(cudaMemcpyAsync(d_tok, tokens, tok_bytes, cudaMemcpyHostToDevice, S.stream()));
        S.decode_step(d_tok, nullptr);  // logits stay in the session buffer: one D2H copy, no staging hop
        if (logits_out)
            FSVD_CUDA(cudaMemcpyAsync(logits_out, S.logits_device(), log_bytes, cudaMemcpyDeviceToHost, S.stream()));
        FSVD_CUDA(cudaStreamSynchronize(S.stream()));
        S.stats().copy_bytes += tok_bytes + (logits_out ? log_bytes : 0);
    });
}

fsvd_status fsvd_generate(fsvd_session* s, const int32_t* prompt, uint64_t T, uint64_t max_new, int32_t* out) {
    return guarded([&] {
        need(s, "session");
        need(prompt, "prompt");
        if (max_new) need(out, "out");
        auto& S = *s->s;
        const size_t B = S.batch();
        const size_t tok_bytes = B * T * 4, out_bytes = B * max_new * 4;
        char* stage = static_cast<char*>(S.staging(tok_bytes + out_bytes + 256));
        int32_t* d_tok = reinterpret_cast<int32_t*>(stage);
        int32_t* d_out = reinterpret_cast<int32_t*>(stage + ((tok_bytes + 255) & ~size_t(255)));
        FSVD_CUDA(cudaMemcpyAsync(d_tok, prompt, tok_bytes, cudaMemcpyHostToDevice, S.stream()));
        S.generate(d_tok, T, max_new, d_out);
        if (max_new) FSVD_CUDA(cudaMemcpyAsync(out, d_out, out_bytes, cudaMemcpyDeviceToHost, S.stream()));
        FSVD_CUDA(cudaStreamSynchronize(S.stream()));
        S.stats().copy_bytes += tok_bytes + out_bytes;
    });
}

fsvd_status fsvd_prefill_device(fsvd_session* s, const int32_t* d_tokens, uint64_t T, float* d_logits) {
    return guarded([&] {
        need(s, "session");
        need(d_tokens, "tokens");
        s->s->prefill(d_tokens, T, d_logits);
    });
}

fsvd_status fsvd_decode_step_device(fsvd_session* s, const int32_t* d_tokens, float* d_logits) {
    return guarded([&] {
        need(s, "session");
        s->s->decode_step(d_tokens, d_logits);
    });
}

fsvd_status fsvd_decode_steps_device(fsvd_session* s, uint64_t n, int32_t* d_out) {
    return guarded([&] {
        need(s, "session");
        s->s->decode_steps(n, d_out, static_cast<int>(n));
    });
}

fsvd_status fsvd_generate_device(fsvd_session* s, const int32_t* d_prompt, uint64_t T, uint64_t max_new,
                                 int32_t* d_out) {
    return guarded([&] {
        need(s, "session");
        need(d_prompt, "prompt");
        if (max_new) need(d_out, "out");
        s->s->generate(d_prompt, T, max_new, d_out);
    });
}

fsvd_status fsvd_session_sync(fsvd_session* s) {
    return guarded([&] {
        need(s, "session");
        FSVD_CUDA(cudaStreamSynchronize(s->s->stream()));
    });
}

fsvd_status fsvd_session_stream(fsvd_session* s, void** stream) {
    return guarded([&] {
        need(s, "session");
        need(stream, "stream");
        *stream = s->s->stream();
    });
}

fsvd_status fsvd_session_position(const fsvd_session* s, uint64_t* position) {
    return guarded([&] {
        need(s, "session");
        need(position, "position");
        *position = s->s->position();
    });
}

fsvd_status fsvd_session_reset(fsvd_session* s) {
    return guarded([&] {
        need(s, "session");
        s->s->reset();
    });
}

fsvd_status fsvd_session_stats(const fsvd_session* s, fsvd_step_stats* st) {
    return guarded([&] {
        need(s, "session");
        need(st, "stats");
        const auto& x = s->s->stats();
        *st = {x.steps, x.dispatches, x.kernel_launches, x.graph_launches, x.allocs, x.copy_bytes, x.last_dispatches,
               x.recon_flops};
    });
}

fsvd_status fsvd_session_resolved(const fsvd_session* s, fsvd_ffn_backend* ffn, fsvd_plan_mode* plan) {
    return guarded([&] {
        need(s, "session");
        if (ffn) *ffn = s->s->ffn();
        if (plan) *plan = s->s->plan();
    });
}

fsvd_status fsvd_session_engine(const fsvd_session* s, int32_t* megakernel, int32_t* stage_bytes, int32_t* nstage,
                                int32_t* attn_splits) {
    return guarded([&] {
        need(s, "session");
        const auto e = s->s->engine();
        if (megakernel) *megakernel = e[0];
        if (stage_bytes) *stage_bytes = e[1];
        if (nstage) *nstage = e[2];
        if (attn_splits) *attn_splits = e[3];
    });
}

fsvd_status fsvd_session_trace(fsvd_session* s, uint64_t* out, uint64_t count, int32_t* phases, int32_t* grid) {
    return guarded([&] {
        need(s, "session");
        need(out, "out");
        int g = 0;
        const int n = s->s->read_trace(reinterpret_cast<unsigned long long*>(out), count, &g);
        if (phases) *phases = n;
        if (grid) *grid = g;
    });
}

fsvd_status fsvd_session_read_kv(fsvd_session* s, uint64_t layer, uint64_t b, int32_t which, uint64_t pos0,
                                 uint64_t npos, float* out) {
    return guarded([&] {
        need(s, "session");
        need(out, "out");
        s->s->read_kv(layer, b, which, pos0, npos, out);
    });
}

fsvd_status fsvd_session_destroy(fsvd_session* s) {
    return guarded([&] { delete s; });
}

}  // extern "C"
