// Internal runtime objects behind the C ABI: device-resident model and
// decode/prefill sessions (SPEC.md:283-446 runtime + plan modules).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../cuda/kernels.h"
#include "fsvd/canonical.hpp"
#include "fsvd/synth.hpp"
#include "fsvd_c.h"

namespace fsvd::rt {

struct CudaError : std::runtime_error {
    explicit CudaError(const std::string& w) : std::runtime_error(w) {}
};
struct OomError : std::runtime_error {
    explicit OomError(const std::string& w) : std::runtime_error(w) {}
};

void cuda_check(cudaError_t e, const char* what);
#define FSVD_CUDA(call) ::fsvd::rt::cuda_check((call), #call)

inline int pad8(size_t v) { return static_cast<int>((v + 7) / 8 * 8); }

// Device weights in the output-major layout the GEMV/GEMM kernels stream:
//   A^T [r][ld_in]  (row j = column j of the reference's d_in x r factor)
//   B^T [d_out][rp] (row n = column n of the r x d_out factor), rp = pad8(r)
// Per layer the q/k/v input factors are packed row-wise into one A^T_qkv and
// up/gate into A^T_ug (packing is an exact copy). Shared
// bases (family C) are uploaded once per distinct storage instance.
struct DeviceLayer {
    int r[kNumProj];
    int rp[kNumProj];
    const void* at_qkv;  // [r_q + r_k + r_v][ldd]
    const void* at_o;    // [r_o][ldd]
    const void* at_ug;   // [r_up + r_gate][ldd]
    const void* at_down; // [r_down][ldff]
    const void* bt[kNumProj];
    const float* attn_gamma;
    const float* mlp_gamma;
};

struct DeviceModel {
    ModelConfig cfg;
    size_t capacity = 0;
    k::WType wt = k::kBF16;
    int esize = 2;
    int device = 0;
    int sm_count = 148;
    int ldd = 0, ldff = 0;
    char family = 'A';
    void* arena = nullptr;
    size_t arena_bytes = 0, used = 0;
    const void* emb = nullptr;     // [V][ldd]
    const void* head_t = nullptr;  // [V][ldd]
    const float* final_gamma = nullptr;
    std::vector<DeviceLayer> layers;
    uint64_t stored_weight_bytes = 0;   // bytes actually resident (shared bases once)
    uint64_t decode_weight_bytes = 0;   // bytes one B=1 decode step streams
    uint64_t prefill_flops_per_token = 0;  // 2 * sum of factor params (GEMM part)

    ~DeviceModel();
    void* alloc(size_t bytes);
};

std::unique_ptr<DeviceModel> upload_canonical(const CanonicalModel<float>& m, fsvd_dtype dt, int device);
std::unique_ptr<DeviceModel> generate_synthetic(const SynthSpec& spec, fsvd_dtype dt, int device);
void copy_factor(const DeviceModel& m, size_t layer, size_t proj, bool b, float* out, size_t count);

struct StepStats {
    uint64_t steps = 0, dispatches = 0, kernel_launches = 0, graph_launches = 0, allocs = 0, copy_bytes = 0,
             last_dispatches = 0;
};

fsvd_ffn_backend route_ffn_auto(fsvd_plan_mode plan, fsvd_ffn_backend requested);

class Session {
  public:
    Session(DeviceModel* m, const fsvd_session_opts& o);
    ~Session();

    void prefill(const int32_t* d_tokens, size_t T, float* d_logits);  // device pointers
    void decode_step(const int32_t* d_tokens, float* d_logits);        // d_tokens may be null: use last argmax
    void generate(const int32_t* d_prompt, size_t T, size_t max_new, int32_t* d_out);
    void reset();
    void read_kv(size_t layer, size_t b, int which, size_t pos0, size_t npos, float* out);

    size_t position() const { return position_; }
    int batch() const { return B_; }
    int vocab() const { return static_cast<int>(m_->cfg.vocab); }
    cudaStream_t stream() const { return stream_; }
    const StepStats& stats() const { return stats_; }
    StepStats& stats() { return stats_; }
    fsvd_ffn_backend ffn() const { return ffn_; }
    fsvd_plan_mode plan() const { return plan_; }
    // device staging for host-pointer API calls (grown on demand)
    void* staging(size_t bytes);

  private:
    void layer_body(size_t l);
    void step_head(float* d_logits, int32_t* d_out, int out_ld);
    void run_decode(int32_t* d_out, int out_ld, float* d_logits);
    void capture_graphs();
    void prefill_chunk(const int32_t* d_tokens, size_t T_total, size_t t0, size_t Tc);
    void ensure_prefill_workspace(size_t rows);
    void launch_gemv(const k::GemvArgs& a);
    void* dalloc(size_t bytes);

    DeviceModel* m_;
    int B_;
    size_t cap_;
    fsvd_ffn_backend ffn_;
    fsvd_plan_mode plan_;
    cudaStream_t stream_ = nullptr;
    std::vector<void*> allocations_;
    StepStats stats_;
    size_t position_ = 0;
    int splits_ = 1;
    bool pdl_ = true;

    // decode state
    void* kc_ = nullptr;
    void* vc_ = nullptr;
    long long cache_bstride_ = 0, cache_hstride_ = 0, cache_lstride_ = 0;
    float2* rope_ = nullptr;
    int* pos_ = nullptr;
    int* step_ = nullptr;
    int* tokens_ = nullptr;
    unsigned* tickets_ = nullptr;
    unsigned* counters_ = nullptr;
    float *x_ = nullptr, *p_qkv_ = nullptr, *q_ = nullptr, *attn_ = nullptr, *p_o_ = nullptr, *p_ug_ = nullptr,
          *h_ = nullptr, *p_d_ = nullptr, *logits_ = nullptr, *partial_ = nullptr;
    int ld_qkv_ = 0, ld_ug_ = 0;
    void* staging_ = nullptr;
    size_t staging_bytes_ = 0;

    // plans
    std::vector<cudaGraphExec_t> layer_graphs_;
    cudaGraphExec_t step_graph_ = nullptr;
    int32_t* graph_out_ = nullptr;  // out pointer baked into the step graph
    int graph_out_ld_ = 0;
    float* graph_logits_ = nullptr;
    bool capturing_ = false;
    uint64_t launches_this_step_ = 0;

    // prefill workspace
    size_t pf_rows_ = 0;
    float* pf_x_ = nullptr;
    void *pf_xn_ = nullptr, *pf_pqkv_ = nullptr, *pf_q_ = nullptr, *pf_att_ = nullptr, *pf_po_ = nullptr,
         *pf_pug_ = nullptr, *pf_h_ = nullptr, *pf_pd_ = nullptr;
    int32_t* pf_tok_ = nullptr;
};

}  // namespace fsvd::rt
