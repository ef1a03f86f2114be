#pragma once
// fsvd drop-in: the SPEC'd runtime entry points for C++
// callers of the reference API, backed by the B200 C ABI (fsvd_c.h).
//
//   fsvd::gpu::Model m = fsvd::gpu::Model::load("model.fsvd", FSVD_DTYPE_BF16);
//   fsvd::gpu::Session s(m, {.batch = 1, .capacity = 4096});
//   std::vector<float> logits = s.prefill(tokens);
//   logits = s.decode_step(next);
//   std::vector<int32_t> out = s.generate(prompt, 64);
//
// Every fsvd_status maps back to the reference's exception type (tensor.hpp
// ShapeError/RankError/NumericError/CapacityError/ConfigError,
// checkpoint.hpp FormatError, canonical.hpp NormalizeError), so existing
// `catch (fsvd::CapacityError&)` sites keep working. Header-only; link
// libfsvd_b200.so.

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../fsvd_c.h"
#include "errors.hpp"
#include "tensor.hpp"

namespace fsvd::gpu {

struct CudaError : std::runtime_error {
    explicit CudaError(const std::string& w) : std::runtime_error(w) {}
};
struct OutOfMemory : std::runtime_error {
    explicit OutOfMemory(const std::string& w) : std::runtime_error(w) {}
};

// fsvd_status -> the reference exception type (no exception crosses the C ABI)
inline void check(fsvd_status st) {
    if (st == FSVD_OK) return;
    const std::string msg = fsvd_last_error();
    switch (st) {
        case FSVD_ERR_SHAPE: throw ShapeError(msg);
        case FSVD_ERR_RANK: throw RankError(msg);
        case FSVD_ERR_NUMERIC: throw NumericError(msg);
        case FSVD_ERR_CAPACITY: throw CapacityError(msg);
        case FSVD_ERR_CONFIG: throw ConfigError(msg);
        case FSVD_ERR_FORMAT: throw FormatError(msg);
        case FSVD_ERR_NORMALIZE: throw NormalizeError(msg);
        case FSVD_ERR_CUDA: throw CudaError(msg);
        case FSVD_ERR_OOM: throw OutOfMemory(msg);
        default: throw std::runtime_error(msg);
    }
}

// Device-resident model (immutable after load; backs any number of sessions).
class Model {
  public:
    static Model load(const std::string& path, fsvd_dtype dtype = FSVD_DTYPE_BF16, int device = 0) {
        fsvd_model* m = nullptr;
        check(fsvd_model_load(path.c_str(), dtype, device, &m));
        return Model(m);
    }
    fsvd_config config() const {
        fsvd_config c{};
        uint64_t cap = 0, wb = 0, db = 0;
        check(fsvd_model_info(m_.get(), &c, &cap, &wb, &db));
        return c;
    }
    fsvd_model* get() const { return m_.get(); }

  private:
    struct Del {
        void operator()(fsvd_model* m) const { fsvd_model_destroy(m); }
    };
    explicit Model(fsvd_model* m) : m_(m, Del{}) {}
    std::shared_ptr<fsvd_model> m_;
};

// SPEC.md:293-298 Session: KV cache + workspace + plans for `batch`
// independent sequences advanced in lock step. Host-buffer API (the
// device-pointer variants are in fsvd_c.h).
class Session {
  public:
    Session(const Model& m, fsvd_session_opts o) : model_(m) {
        if (o.batch == 0) o.batch = 1;
        fsvd_session* s = nullptr;
        check(fsvd_session_create(m.get(), &o, &s));
        s_.reset(s);
        batch_ = o.batch;
        vocab_ = m.config().vocab;
    }
    // tokens: [batch][T] -> last-position logits [batch][vocab]
    std::vector<float> prefill(const std::vector<int32_t>& tokens) {
        std::vector<float> out(batch_ * vocab_);
        if (tokens.size() % batch_) throw ShapeError("prefill: tokens not a multiple of batch");
        check(fsvd_prefill(s_.get(), tokens.data(), tokens.size() / batch_, out.data()));
        return out;
    }
    // token per sequence -> logits [batch][vocab]
    std::vector<float> decode_step(const std::vector<int32_t>& tokens) {
        if (tokens.size() != batch_) throw ShapeError("decode_step: one token per sequence");
        std::vector<float> out(batch_ * vocab_);
        check(fsvd_decode_step(s_.get(), tokens.data(), out.data()));
        return out;
    }
    // prompt [batch][T] -> greedy tokens [batch][max_new] (ties -> lowest index)
    std::vector<int32_t> generate(const std::vector<int32_t>& prompt, size_t max_new) {
        if (prompt.size() % batch_) throw ShapeError("generate: prompt not a multiple of batch");
        std::vector<int32_t> out(batch_ * max_new);
        check(fsvd_generate(s_.get(), prompt.data(), prompt.size() / batch_, max_new, out.data()));
        return out;
    }
    size_t position() const {
        uint64_t p = 0;
        check(fsvd_session_position(s_.get(), &p));
        return p;
    }
    void reset() { check(fsvd_session_reset(s_.get())); }

  private:
    struct Del {
        void operator()(fsvd_session* s) const { fsvd_session_destroy(s); }
    };
    Model model_;
    std::unique_ptr<fsvd_session, Del> s_;
    size_t batch_ = 1, vocab_ = 0;
};

}  // namespace fsvd::gpu
