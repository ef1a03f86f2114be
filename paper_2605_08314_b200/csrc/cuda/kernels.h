// Host-side launch interface of the sm_100a kernels (plain pointers; used by
// the runtime in csrc/host/runtime.cu). No torch types.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fsvd::k {

enum WType : int { kF32 = 0, kBF16 = 1 };

// ---------------------------------------------------------------- GEMV ----
// y = epilogue(x . W^T) for a decode batch of B <= 4 rows. W^T is stored
// output-major (row n = column n of the reference's d_in x d_out factor, K
// contiguous), so every output row is one contiguous 16-byte-aligned stream.
enum GemvEpi : int {
    kEpiStore = 0,     // y[b][y_off + n] = v
    kEpiAdd = 1,       // y[b][y_off + n] += v           (residual)
    kEpiRopeQ = 2,     // interleaved-pair RoPE at *pos, then store to y
    kEpiRopeK = 3,     // RoPE, then K cache row *pos
    kEpiV = 4,         // V cache row *pos
};

struct GemvSeg {
    const void* w;   // W^T rows, [rows][ldw] elements
    int rows;
    int ldw;         // elements; multiple of 8
    int k;           // used row length (elements, multiple of 8; x segment length)
    int x_off;       // start of this segment's input inside x (elements)
    int y_off;       // output index of row 0
    int epi;         // GemvEpi
};

struct GemvArgs {
    GemvSeg seg[3];
    int nseg;
    int dual;            // 1: h = silu(seg1 . x) * (seg0 . x) row-wise (up = seg0, gate = seg1)
    const float* x;      // [B][x_ld] fp32
    int x_ld;
    int x_len;           // elements staged to smem per batch row (multiple of 8)
    const float* gamma;  // RMSNorm prologue if non-null: x * inv_rms(x[0:norm_len]) * gamma
    float eps;
    int norm_len;
    float* y;            // [B][y_ld]
    int y_ld;
    // RoPE / KV append
    const float2* rope;  // [capacity][d_head/2] (cos, sin), computed on the host in double
    const int* pos;      // device length register
    int d_head;
    void* kcache;        // layer base, [B][H][cap][d_head] in weight dtype
    void* vcache;
    long long cache_bstride, cache_hstride;  // elements
};

void gemv(WType wt, int batch, const GemvArgs& a, int grid, cudaStream_t s, bool pdl);
int gemv_smem_bytes(int batch, int x_len);

// ----------------------------------------------------------- attention ----
constexpr int kAttnMaxChunk = 4096;  // max cache rows per decode split
// Decode attention of B x H query heads against cache rows [0, *pos]
// (after the append), split-K over the sequence with a deterministic
// last-CTA combine. q, out: [B][d_model] fp32.
struct AttnDecodeArgs {
    const float* q;
    const void* kcache;  // layer base [B][H][cap][d_head]
    const void* vcache;
    long long cache_bstride, cache_hstride;
    const int* pos;      // attends positions 0 .. *pos inclusive
    float* out;
    float* partial;      // [B][H][splits][d_head + 2]
    unsigned* counters;  // [B][H], zero-initialized, self-resetting
    int batch, n_heads, d_head, splits;
    float scale;
};
void attn_decode(WType wt, const AttnDecodeArgs& a, cudaStream_t s, bool pdl);

// Prefill causal attention: queries at positions [p0, p0 + T) of each of B
// sequences against cache rows [0, p0 + T) (causal).
struct AttnPrefillArgs {
    const void* q;       // [B*T][q_ld], weight dtype
    int q_ld;
    const void* kcache;
    const void* vcache;
    long long cache_bstride, cache_hstride;
    void* out;           // [B*T][out_ld], weight dtype
    int out_ld;
    int batch, T, p0, n_heads, d_head;
    float scale;
};
void attn_prefill(WType wt, const AttnPrefillArgs& a, cudaStream_t s);

// ---------------------------------------------------------------- GEMM ----
// Prefill GEMM: Y[t][n] = epi(sum_k X[t][k] * W^T[n][k]) with X, W^T in the
// weight dtype (activations rounded to it), fp32 accumulate.
enum GemmEpi : int {
    kGemmStore = 0,   // Y (act dtype) [t][y_off + n]
    kGemmAddF32 = 1,  // Yf32[t][n] += v (residual)
    kGemmQKV = 2,     // RoPE q/k at position p0 + t%T; q -> Y, k/v -> cache
    kGemmSilu = 3,    // dual: Y[t][n] = silu(gate) * up (act dtype)
};
struct GemmArgs {
    const void* x;    // [M][x_ld]
    int x_ld;
    int M;            // rows (tokens)
    // up to 3 weight segments along N (QKV) or 2 (dual silu)
    GemvSeg seg[3];
    int nseg;
    int epi;
    void* y;          // act dtype, or fp32 for kGemmAddF32
    int y_ld;
    // QKV epilogue
    const float2* rope;
    int p0, T, d_head, n_heads;
    void* kcache;
    void* vcache;
    long long cache_bstride, cache_hstride;
};
void gemm(WType wt, const GemmArgs& a, cudaStream_t s);       // dispatch: tcgen05 (bf16) / CUDA cores (f32)
void gemm_simt(WType wt, const GemmArgs& a, cudaStream_t s);  // CUDA-core path

// ----------------------------------------------------------------- misc ----
// x[b][:] = E[tokens[b]][:]  (fp32 out)
void embed(WType wt, const void* emb, int ld_emb, const int* tokens, int n, int d, float* x, int x_ld,
           cudaStream_t s, bool pdl);
// y[r][:] = x[r] * inv_rms(x[r]) * gamma (y in weight dtype)
void rmsnorm_rows(WType wt, const float* x, int x_ld, const float* gamma, float eps, int rows, int d, void* y,
                  int y_ld, cudaStream_t s);
// Copy rows {(b*T + T-1)} of x to xl[b] (last position of each sequence).
void gather_last(const float* x, int x_ld, int batch, int T, int d, float* xl, int xl_ld, cudaStream_t s);
// tokens[b] = argmax(logits[b]) (ties -> lowest index); *pos += pos_inc;
// out_tokens[b * out_ld + *step] written when out_tokens != null.
// ticket: zero-initialized device counter (self-resetting).
void argmax_step(const float* logits, int batch, int vocab, int* tokens, int* pos, int pos_inc,
                 int* out_tokens, int out_ld, int* step, unsigned* ticket, cudaStream_t s, bool pdl);
void set_int(int* p, int v, cudaStream_t s);
void add_int(int* p, int v, cudaStream_t s, bool pdl);

// Synthetic-weight generation (include/fsvd/synth.hpp stream) into a strided
// destination: dst[(i / cols) * rs + (i % cols) * cs] for logical element i
// of a rows x cols tensor. fold: 0 none, 1 row-scale by 1/s[row] (family B),
// 2 col-scale by s[col] (family D); scale tensor is itself generated from the
// stream at scale_offset.
struct SynthFill {
    uint64_t seed;
    uint64_t offset;   // stream offset of element 0
    double amp;
    int kind;          // SynthTensor::Kind
    long long rows, cols, rs, cs;
    int fold;
    uint64_t scale_offset;
    void* dst;
    WType dt;          // destination dtype
};
void synth_fill(const SynthFill& f, cudaStream_t s);

}  // namespace fsvd::k
