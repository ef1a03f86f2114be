// Internal runtime objects behind the C ABI: device-resident model and
// decode/prefill sessions (SPEC.md:283-446 runtime + plan modules).
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../cuda/decode_mk.h"
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
inline int pad64(size_t v) { return static_cast<int>((v + 63) / 64 * 64); }

// A factor matrix W^T on the device, tile layout (csrc/cuda/layout.h).
struct DeviceMatrix {
    const void* w = nullptr;
    int rows = 0, k = 0, kp = 0;
    k::WLayout layout(int esize) const { return k::WLayout{rows, k, kp, esize}; }
};

// Per layer: A^T (rows r, K d_in) and B^T (rows d_out, K r) of every
// projection q,k,v,o,up,gate,down. The q/k/v input factors are allocated
// adjacently (one packed projection) and so are up/gate;
// shared bases (family C) are uploaded once per storage instance.
struct DeviceLayer {
    int r[kNumProj];
    int rp[kNumProj];  // rank padded to 64: stride of the rank-space vectors
    DeviceMatrix at[kNumProj];
    DeviceMatrix bt[kNumProj];
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
    int ldd = 0, ldff = 0;  // activation strides (d_model, d_ff padded to 64)
    char family = 'A';
    void* arena = nullptr;
    size_t arena_bytes = 0, used = 0;
    const void* emb = nullptr;  // [V][ldd] row-major
    DeviceMatrix head_t;        // rows V, K d_model
    const float* final_gamma = nullptr;
    std::vector<DeviceLayer> layers;
    uint64_t stored_weight_bytes = 0;      // bytes resident (shared bases once, incl. padding)
    uint64_t decode_weight_bytes = 0;      // algorithmic bytes of one B=1 decode step
    uint64_t prefill_flops_per_token = 0;  // 2 * sum of factor params (GEMM part)

    ~DeviceModel();
    void* alloc(size_t bytes);
};

std::unique_ptr<DeviceModel> upload_canonical(const CanonicalModel<float>& m, fsvd_dtype dt, int device);
std::unique_ptr<DeviceModel> generate_synthetic(const SynthSpec& spec, fsvd_dtype dt, int device);
// FSVD15 file -> device model without a host CanonicalModel (load_streaming in
// runtime.cu): positioned reads into pinned staging buffers, CRC-32 checked on
// the fly, f32 -> weight dtype + family fold on the device straight into the
// tile layout. Same validation and errors as read_checkpoint_file +
// normalize<float>; device factors bitwise equal to upload_canonical's.
struct LoadStats {
    double seconds = 0;
    uint64_t bytes = 0;        // payload bytes read
    uint64_t pinned_bytes = 0; // host staging held at once
};
std::unique_ptr<DeviceModel> load_streaming(const std::string& path, fsvd_dtype dt, int device, LoadStats* st = nullptr);
void copy_factor(const DeviceModel& m, size_t layer, size_t proj, bool b, float* out, size_t count);

struct StepStats {
    uint64_t steps = 0, dispatches = 0, kernel_launches = 0, graph_launches = 0, allocs = 0, copy_bytes = 0,
             last_dispatches = 0, recon_flops = 0;
};

fsvd_ffn_backend route_ffn_auto(fsvd_plan_mode plan, fsvd_ffn_backend requested);

class Session {
  public:
    Session(DeviceModel* m, const fsvd_session_opts& o);
    ~Session();

    void prefill(const int32_t* d_tokens, size_t T, float* d_logits);  // device pointers
    void decode_step(const int32_t* d_tokens, float* d_logits);        // d_tokens may be null: use last argmax
    void generate(const int32_t* d_prompt, size_t T, size_t max_new, int32_t* d_out);
    // n greedy steps from the last argmax, on the device; d_out [B][out_ld] at columns *step.. (may be null)
    void decode_steps(size_t n, int32_t* d_out, int out_ld);
    void reset();
    void read_kv(size_t layer, size_t b, int which, size_t pos0, size_t npos, float* out);

    size_t position() const { return position_; }
    const float* logits_device() const { return logits_; }  // [B][V] of the last prefill / decode step
    int batch() const { return B_; }
    int vocab() const { return static_cast<int>(m_->cfg.vocab); }
    cudaStream_t stream() const { return stream_; }
    const StepStats& stats() const { return stats_; }
    StepStats& stats() { return stats_; }
    fsvd_ffn_backend ffn() const { return ffn_; }
    fsvd_plan_mode plan() const { return plan_; }
    fsvd_attn_route attn_route() const { return attn_route_; }
    // device staging for host-pointer API calls (grown on demand)
    void* staging(size_t bytes);
    // copies the last traced full step: [grid][phases][4] ns stamps; returns phases
    int read_trace(unsigned long long* out, size_t count, int* grid);
    // {1 megakernel | 2 batched layer engine, ring chunk bytes, ring stages, attention splits}
    std::array<int, 4> engine() const {
        return batched_ ? std::array<int, 4>{2, 0, 0, 0} : std::array<int, 4>{1, k::kChunkBytes, mk_stages_, mk_splits_};
    }
    bool batched() const { return batched_; }

  private:
    void init(const fsvd_session_opts& o);
    void release();  // frees every device resource; safe on a partly built session
    void build_program();
    void add_layer_phases(size_t l, const float* next_gamma);
    void mk_run(int p_begin, int p_end, int reps = 1);
    void mk_decode(int32_t* d_out, int out_ld);
    void mk_set_out(int32_t* d_out, int out_ld);
    void prefill_chunk(const int32_t* d_tokens, size_t T_total, size_t t0, size_t Tc);
    // every layer over M = B*T rows of pf_x_ (positions p0 + t, or *p0_dev + t)
    void layers_forward(int M, int T, int p0, const int* p0_dev);
    // batched engine (B > 2): final norm + head GEMM + argmax over rows x[B]
    void head_rows(const float* x, int32_t* d_out, int out_ld, int pos_inc);
    void batched_decode(int32_t* d_out, int out_ld);
    void decode_any(int32_t* d_out, int out_ld) { batched_ ? batched_decode(d_out, out_ld) : mk_decode(d_out, out_ld); }
    void ensure_prefill_workspace(size_t rows);
    void* dalloc(size_t bytes);
    k::GemvSeg seg(const DeviceMatrix& m, int x_off, int y_off, int epi) const;
    k::Planes planes(int len);
    k::MkGemv& add_gemv(const std::vector<k::GemvSeg>& segs, int dual, const k::Planes& in, const float* norm_src,
                        int out_kind);
    int add_vec(const void* emb, const float* src, float* xres, const float* gamma, const k::Planes& out);

    DeviceModel* m_;
    int B_;
    size_t cap_;
    fsvd_ffn_backend ffn_;
    fsvd_plan_mode plan_;
    fsvd_attn_route attn_route_ = FSVD_ATTN_DENSE_KV;
    // lowrank_history route: pre-RoPE rank-space K / V history
    // [L][B][cap][ld_hist_], rebuilt into the dense cache every decode step
    void* hist_k_ = nullptr;
    void* hist_v_ = nullptr;
    int ld_hist_ = 0;
    // split plan: first FFN phase of each layer, boundary-copy buffer
    std::vector<int> ph_ffn_begin_;
    void* split_buf_ = nullptr;
    cudaStream_t stream_ = nullptr;
    std::vector<void*> allocations_;
    StepStats stats_;
    size_t position_ = 0;

    // decode state
    void* kc_ = nullptr;
    void* vc_ = nullptr;
    long long cache_bstride_ = 0, cache_hstride_ = 0, cache_lstride_ = 0;
    float2* rope_ = nullptr;
    int* pos_ = nullptr;
    int* step_ = nullptr;
    int* tokens_ = nullptr;
    float* xres_ = nullptr;    // residual stream [B][ldd] fp32 (updated in place by the finalizers)
    float* x_ = nullptr;       // prefill: final hidden state of each sequence's last position
    float* qbuf_ = nullptr;    // RoPE'd q of the current position
    float* logits_ = nullptr;
    float* cand_v_ = nullptr;  // per head tile best logit / index
    int* cand_i_ = nullptr;
    float* attn_part_ = nullptr;
    unsigned* attn_count_ = nullptr;
    k::Planes xpl_{}, pqkv_{}, att_{}, po_{}, pug_{}, h_{}, pd_{};  // phase inputs (decode_mk.h Planes)
    int ld_qkv_ = 0, ld_o_ = 0, ld_ug_ = 0, ld_d_ = 0;
    void* staging_ = nullptr;
    size_t staging_bytes_ = 0;

    // megakernel program (decode_mk.cu)
    std::vector<k::MkPhase> h_phases_;
    int x_bytes_ = 0, rec_chunks_ = 0;
    k::MkPhase* d_phases_ = nullptr;
    k::MkChunk* d_chunks_ = nullptr;
    int* d_chunk_start_ = nullptr;
    int* d_chunk_tiles_ = nullptr;
    volatile int* mk_progress_ = nullptr;
    int* mk_progress_host_ = nullptr;
    unsigned* mk_bar_ = nullptr;
    bool mk_attn_pairs_ = false;  // decode attention: one CTA pair (cluster of 2) per (b, h) when B*H <= grid/2
    bool mk_exact_ = false;  // even unit splits for the kOutPlanes phases (FSVD_MK_EXACT=1; measured slower)
    int mk_smem_ = 0, mk_grid_ = 0, mk_splits_ = 0, mk_stages_ = 0, mk_l2_ahead_ = 16;
    int ph_head_ = 0, ph_argmax_ = 0, ph_pf_head_ = 0, ph_pf_argmax_ = 0;
    std::vector<int> ph_layer_begin_, ph_layer_end_;
    unsigned long long* trace_ = nullptr;  // FSVD_TRACE=1: per-phase globaltimer stamps of the full step
    int32_t* mk_out_ = nullptr;
    int mk_out_ld_ = 0;
    uint64_t launches_this_step_ = 0;

    // batched engine (B > 2, or FSVD_BATCHED=1): layer-by-layer tcgen05 GEMMs
    // with the batch as the M dimension, one graph per step for the graph plans
    bool batched_ = false;
    cudaGraphExec_t bstep_graph_ = nullptr;
    float* dec_part_ = nullptr;  // split-KV decode attention partials
    int dec_splits_ = 1;
    int32_t* bstep_out_ = nullptr;
    int bstep_out_ld_ = 0;

    // plans
    std::vector<cudaGraphExec_t> layer_graphs_;
    cudaGraphExec_t step_graph_ = nullptr;

    // prefill workspace
    size_t pf_rows_ = 0;
    float* pf_x_ = nullptr;
    void *pf_xn_ = nullptr, *pf_pqkv_ = nullptr, *pf_q_ = nullptr, *pf_att_ = nullptr, *pf_po_ = nullptr,
         *pf_pug_ = nullptr, *pf_h_ = nullptr, *pf_pd_ = nullptr;
    int32_t* pf_tok_ = nullptr;
    float* pf_ws_ = nullptr;
    size_t pf_ws_floats_ = 0;
    float* pf_ss_ = nullptr;  // RMSNorm fold: sums of squares per 32-column chunk [rows][ldd / 32]
};

}  // namespace fsvd::rt
