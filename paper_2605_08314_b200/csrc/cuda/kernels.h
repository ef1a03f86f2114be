// Host-side launch interface of the sm_100a kernels (plain pointers; used by
// the runtime in csrc/host/runtime.cu). No torch types.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "layout.h"

namespace fsvd::k {

enum WType : int { kF32 = 0, kBF16 = 1 };

// ------------------------------------------------------ projection segment --
// One factor matrix W^T (tile layout, layout.h) of a GEMV/GEMM phase, and what
// to do with its outputs.
enum GemvEpi : int {
    kEpiStore = 0,   // y[b][y_off + n] = v
    kEpiAdd = 1,     // y[b][y_off + n] += v            (residual)
    kEpiRopeQ = 2,   // interleaved-pair RoPE at *pos, then store to y
    kEpiRopeK = 3,   // RoPE, then K cache row *pos
    kEpiV = 4,       // V cache row *pos
    kEpiLogits = 5,  // logits + per-tile argmax candidates
};

struct GemvSeg {
    const void* w;  // tile-layout matrix
    int rows;       // outputs
    int k;          // reduction length
    int kp;         // padded reduction length (layout)
    int x_off;      // start of this segment's input inside x (elements, multiple of 4)
    int y_off;      // output index of row 0
    int epi;        // GemvEpi

    FSVD_HD WLayout layout(int esize) const { return WLayout{rows, k, kp, esize}; }
};

// ----------------------------------------------------------- attention ----
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
    const int* p0_dev;   // non-null: p0 = *p0_dev (graph-replayed batched decode)
};
void attn_prefill(WType wt, const AttnPrefillArgs& a, cudaStream_t s);
// tcgen05/TMEM flash attention (attn_tc.cu, bf16, d_head 64 / 128); false if not covered
bool attn_prefill_tcgen05(const AttnPrefillArgs& a, cudaStream_t s);
// Split-KV flash decode (T = 1, bf16, d_head 128): partials [B][H][S][d_head + 2]
// fp32 then an in-order merge; false if the shape is not covered.
int attn_decode_splits(int batch, int n_heads, int capacity);
bool attn_decode(WType wt, const AttnPrefillArgs& a, float* part, int S, cudaStream_t s);

// ---------------------------------------------------------------- GEMM ----
// Prefill GEMM: Y[t][n] = epi(sum_k X[t][k] * W^T[n][k]) with X in the weight
// dtype (activations rounded to it), W^T in tile layout, fp32 accumulate.
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
    GemvSeg seg[3];
    int nseg;
    int epi;
    void* y;          // act dtype, or fp32 for kGemmAddF32
    int y_ld;
    // QKV epilogue
    const float2* rope;
    int p0, T, d_head, n_heads;
    const int* p0_dev;   // non-null: p0 = *p0_dev (graph-replayed batched decode)
    void* kcache;
    void* vcache;
    long long cache_bstride, cache_hstride;
    // split-K scratch for the plain-store / residual epilogues (few output
    // tiles): fp32 [splits][M][y_ld]; null disables split-K
    float* ws;
    size_t ws_floats;
    // RMSNorm folded into the GEMMs (tcgen05 path, prefill): a residual-add
    // epilogue with norm_xg set also writes xg = bf16(x_new * norm_gamma)
    // [M][norm_xg_ld] and the sums of squares of x_new per 32-column chunk into
    // norm_ss [M][norm_ss_ld] (forces an unsplit launch); a plain-store epilogue
    // with norm_ss_in set scales row t by 1 / sqrt(sum_j norm_ss_in[t][j] / norm_d
    // + norm_eps), j < norm_ss_n (a multiple of 4) in index order, row stride
    // norm_ss_ld -- x.A of the normalized row.
    void* norm_xg;
    int norm_xg_ld;
    const float* norm_gamma;
    float* norm_ss;
    int norm_ss_ld;
    const float* norm_ss_in;
    int norm_ss_n, norm_d;
    float norm_eps;
};
void gemm(WType wt, const GemmArgs& a, cudaStream_t s);       // dispatch: tcgen05 (bf16) / CUDA cores (f32)
void gemm_simt(WType wt, const GemmArgs& a, cudaStream_t s);  // CUDA-core path
// tcgen05/TMEM path (bf16): X is read through a TMA tensor map of x_rows rows
bool gemm_tc_supported(const GemmArgs& a);
void gemm_tc(const GemmArgs& a, int x_rows, cudaStream_t s);

// ----------------------------------------------------------------- misc ----
// x[b][:] = E[tokens[b]][:]  (fp32 out; E row-major [V][ld])
void embed(WType wt, const void* emb, int ld_emb, const int* tokens, int n, int d, float* x, int x_ld,
           cudaStream_t s);
// y[r][:] = x[r] * inv_rms(x[r]) * gamma (y in weight dtype)
void rmsnorm_rows(WType wt, const float* x, int x_ld, const float* gamma, float eps, int rows, int d, void* y,
                  int y_ld, cudaStream_t s);
// Copy rows {(b*T + T-1)} of x to xl[b] (last position of each sequence).
void gather_last(const float* x, int x_ld, int batch, int T, int d, float* xl, int xl_ld, cudaStream_t s);
void set_int(int* p, int v, cudaStream_t s);
// Greedy argmax of each logits row (ties -> lowest index, math.hpp:132-140):
// tokens[b] = argmax(logits[b][0..V)); out[b][*step] = tokens[b] if out.
void argmax_rows(const float* logits, int V, int batch, int* tokens, int* out, int out_ld, const int* step,
                 cudaStream_t s);
// *pos += pos_inc; *step += 1 (if step) -- after argmax_rows
void advance_pos(int* pos, int pos_inc, int* step, cudaStream_t s);

// Synthetic-weight generation (include/fsvd/synth.hpp stream). Logical tensor
// element i = (r, c) of a rows x cols tensor goes to
//   mode 0: dst[r * rs + c * cs]            (plain, elements)
//   mode 1: byte offset lay.offset(c, r)    (transposed into the tile layout)
// fold: 0 none, 1 row-scale by 1/s[r] (family B), 2 col-scale by s[c]
// (family D); the scale vector is itself generated from the stream.
struct SynthFill {
    uint64_t seed;
    uint64_t offset;   // stream offset of element 0
    double amp;
    int kind;          // SynthTensor::Kind
    long long rows, cols, rs, cs;
    int mode;
    WLayout lay;
    int fold;
    uint64_t scale_offset;
    void* dst;
    WType dt;          // destination dtype
};
void synth_fill(const SynthFill& f, cudaStream_t s);

// Checkpoint streaming loader (runtime.cu load_streaming): rows [r0, r0 + nrows)
// of a row-major f32 matrix with `cols` columns (already on the device) go to
//   mode 0: dst[r * ld + c]                     (embedding rows, vectors)
//   mode 1: byte offset lay.offset(c, r)        (W^T in the tile layout)
// in dtype dt, after the family fold of normalize<float> (canonical.cpp):
// fold 1: x *= 1 / scale[r] (family B), fold 2: x *= scale[c] (family D).
struct PackArgs {
    const float* src;
    long long r0, nrows, cols;
    int mode;
    long long ld;
    WLayout lay;
    const float* scale;
    int fold;
    void* dst;
    WType dt;
};
void pack_f32(const PackArgs& a, cudaStream_t s);

// lowrank_history route: rank-space rows (b, t) of a [B*T][src_ld] buffer,
// columns [col0, col0 + ncols), to dst[b * dst_bstride + (p0 + t) * dst_ld + j]
// (p0 = *p0_dev if given); esize-byte elements.
void copy_rows_at(const void* src, int src_ld, int col0, int ncols, void* dst, long long dst_bstride, int dst_ld,
                  int batch, int T, int p0, const int* p0_dev, int esize, cudaStream_t s);

}  // namespace fsvd::k
