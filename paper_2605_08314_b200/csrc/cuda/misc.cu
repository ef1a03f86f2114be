// Small kernels around the prefill chain and model setup: embedding gather,
// row RMSNorm (prefill prologue), last-position gather, the length-register
// setter and the synthetic-weight generator.
#include <math_constants.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace fsvd::k {
namespace {

using namespace fsvd::dev;

template <typename T>
__global__ void embed_kernel(const T* emb, int ld, const int* tokens, int d, float* x, int x_ld) {
    const int b = blockIdx.y;
    const T* row = emb + static_cast<long long>(tokens[b]) * ld;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d; i += gridDim.x * blockDim.x)
        x[static_cast<long long>(b) * x_ld + i] = to_f32<T>(row[i]);
}

// reference rmsnorm (kernels_scalar.cpp:55-61): y = x * (1/sqrt(sum(x^2)/n + eps)) * gamma
template <typename T>
__global__ void rmsnorm_rows_kernel(const float* x, int x_ld, const float* gamma, float eps, int d, T* y, int y_ld) {
    __shared__ float red[32];
    __shared__ float inv;
    const float* xr = x + static_cast<long long>(blockIdx.x) * x_ld;
    float ss = 0.f;
    for (int i = threadIdx.x; i < d; i += blockDim.x) ss = fmaf(xr[i], xr[i], ss);
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.f;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += red[w];
        inv = 1.0f / sqrtf(t / static_cast<float>(d) + eps);
    }
    __syncthreads();
    T* yr = y + static_cast<long long>(blockIdx.x) * y_ld;
    for (int i = threadIdx.x; i < d; i += blockDim.x) yr[i] = from_f32<T>(xr[i] * inv * gamma[i]);
}

// Same op, float4-vectorized with every load of the row in flight at once and
// the row kept in registers between the two passes (d % 4 == 0, d <= 8192).
template <typename T>
__global__ void __launch_bounds__(256) rmsnorm_rows_vec_kernel(const float* x, int x_ld, const float* gamma, float eps,
                                                               int d, T* y, int y_ld) {
    constexpr int kIt = 8;
    __shared__ float red[8];
    pdl_launch_dependents();
    pdl_wait();
    const float4* xr = reinterpret_cast<const float4*>(x + static_cast<long long>(blockIdx.x) * x_ld);
    const int n4 = d >> 2;
    float4 v[kIt];
    float ss = 0.f;
#pragma unroll
    for (int it = 0; it < kIt; ++it) {
        const int i = threadIdx.x + it * 256;
        v[it] = i < n4 ? xr[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int it = 0; it < kIt; ++it) {
        ss = fmaf(v[it].x, v[it].x, ss);
        ss = fmaf(v[it].y, v[it].y, ss);
        ss = fmaf(v[it].z, v[it].z, ss);
        ss = fmaf(v[it].w, v[it].w, ss);
    }
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w];
    const float inv = 1.0f / sqrtf(t / static_cast<float>(d) + eps);
    const float4* g4 = reinterpret_cast<const float4*>(gamma);
    T* yr = y + static_cast<long long>(blockIdx.x) * y_ld;
#pragma unroll
    for (int it = 0; it < kIt; ++it) {
        const int i = threadIdx.x + it * 256;
        if (i < n4) {
            const float4 gv = __ldg(g4 + i);
            const float o0 = v[it].x * inv * gv.x, o1 = v[it].y * inv * gv.y;
            const float o2 = v[it].z * inv * gv.z, o3 = v[it].w * inv * gv.w;
            if constexpr (sizeof(T) == 2) {
                __nv_bfloat162 a = __floats2bfloat162_rn(o0, o1), b = __floats2bfloat162_rn(o2, o3);
                uint2 u;
                u.x = *reinterpret_cast<uint32_t*>(&a);
                u.y = *reinterpret_cast<uint32_t*>(&b);
                reinterpret_cast<uint2*>(yr)[i] = u;
            } else {
                reinterpret_cast<float4*>(yr)[i] = make_float4(o0, o1, o2, o3);
            }
        }
    }
}

__global__ void gather_last_kernel(const float* x, int x_ld, int T, int d, float* xl, int xl_ld) {
    const int b = blockIdx.y;
    const float* src = x + (static_cast<long long>(b) * T + T - 1) * x_ld;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d; i += gridDim.x * blockDim.x)
        xl[static_cast<long long>(b) * xl_ld + i] = src[i];
}

__global__ void set_int_kernel(int* p, int v) { *p = v; }

// one CTA per row; ties -> lowest index (math.hpp:132-140)
__global__ void __launch_bounds__(256) argmax_rows_kernel(const float* logits, int V, int* tokens, int* out, int out_ld,
                                                          const int* step) {
    __shared__ float sv[8];
    __shared__ int si[8];
    const int b = blockIdx.x;
    const float* row = logits + static_cast<long long>(b) * V;
    float bv = -CUDART_INF_F;
    int bi = 0x7fffffff;
    for (int i = threadIdx.x; i < V; i += 256) {
        const float v = row[i];
        if (v > bv) {  // strictly greater: the first (lowest) index wins within a thread
            bv = v;
            bi = i;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
            bv = ov;
            bi = oi;
        }
    }
    if ((threadIdx.x & 31) == 0) {
        sv[threadIdx.x >> 5] = bv;
        si[threadIdx.x >> 5] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w)
            if (sv[w] > bv || (sv[w] == bv && si[w] < bi)) {
                bv = sv[w];
                bi = si[w];
            }
        if (bi == 0x7fffffff) bi = 0;
        tokens[b] = bi;
        if (out) out[static_cast<long long>(b) * out_ld + (step ? *step : 0)] = bi;
    }
}

__global__ void advance_pos_kernel(int* pos, int inc, int* step) {
    *pos += inc;
    if (step) *step += 1;
}

__device__ __forceinline__ float round_bf16_dev(float x) {
    uint32_t u = __float_as_uint(x);
    if ((u & 0x7F800000u) == 0x7F800000u) return x;
    u += 0x7FFFu + ((u >> 16) & 1u);
    return __uint_as_float(u & 0xFFFF0000u);
}

// include/fsvd/synth.hpp synth_value, bit for bit.
__device__ __forceinline__ float synth_dev(uint64_t seed, uint64_t idx, double amp, int kind) {
    uint64_t z = seed + (idx + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    const double unit = __dmul_rn(static_cast<double>(z >> 11), 0x1.0p-53);
    const double sym = __dsub_rn(__dmul_rn(2.0, unit), 1.0);
    double v;
    if (kind == 1)
        v = __dadd_rn(1.0, __dmul_rn(sym, amp));
    else if (kind == 2)
        v = __dadd_rn(0.5, unit);
    else
        v = __dmul_rn(sym, amp);
    return round_bf16_dev(__double2float_rn(v));
}

// Iteration order follows the destination (transposed targets walk r
// fastest) so the writes coalesce; the values are a pure function of the
// logical index, so the order does not change them.
__global__ void synth_fill_kernel(const SynthFill f) {
    const long long n = f.rows * f.cols;
    const bool by_col = f.mode == 1 || (f.rs == 1 && f.cs != 1);
    for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < n;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        long long r, c;
        if (by_col) {
            c = t / f.rows;
            r = t - c * f.rows;
        } else {
            r = t / f.cols;
            c = t - r * f.cols;
        }
        const long long i = r * f.cols + c;
        float v = synth_dev(f.seed, f.offset + i, f.amp, f.kind);
        if (f.fold == 1) {
            const float s = synth_dev(f.seed, f.scale_offset + r, 0.0, 2);
            v = __fmul_rn(v, __fdiv_rn(1.0f, s));
        } else if (f.fold == 2) {
            const float s = synth_dev(f.seed, f.scale_offset + c, 0.0, 2);
            v = __fmul_rn(v, s);
        }
        if (f.mode == 1) {
            char* p = static_cast<char*>(f.dst) + f.lay.offset(static_cast<int>(c), static_cast<int>(r));
            if (f.dt == kBF16)
                *reinterpret_cast<__nv_bfloat16*>(p) = __float2bfloat16_rn(v);
            else
                *reinterpret_cast<float*>(p) = v;
        } else {
            const long long o = r * f.rs + c * f.cs;
            if (f.dt == kBF16)
                static_cast<__nv_bfloat16*>(f.dst)[o] = __float2bfloat16_rn(v);
            else
                static_cast<float*>(f.dst)[o] = v;
        }
    }
}

}  // namespace

void embed(WType wt, const void* emb, int ld_emb, const int* tokens, int n, int d, float* x, int x_ld,
           cudaStream_t s) {
    const dim3 grid((d + 255) / 256 < 16 ? (d + 255) / 256 : 16, n);
    if (wt == kBF16)
        embed_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(emb), ld_emb, tokens, d, x,
                                                         x_ld);
    else
        embed_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(emb), ld_emb, tokens, d, x, x_ld);
}

void rmsnorm_rows(WType wt, const float* x, int x_ld, const float* gamma, float eps, int rows, int d, void* y,
                  int y_ld, cudaStream_t s) {
    const bool vec = d % 4 == 0 && d <= 8192 && x_ld % 4 == 0 && y_ld % 4 == 0 &&
                     (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(gamma) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(y) & 15) == 0;
    if (vec) {
        if (wt == kBF16)
            launch_pdl(rmsnorm_rows_vec_kernel<__nv_bfloat16>, dim3(rows), dim3(256), 0, s, x, x_ld, gamma, eps, d,
                       static_cast<__nv_bfloat16*>(y), y_ld);
        else
            launch_pdl(rmsnorm_rows_vec_kernel<float>, dim3(rows), dim3(256), 0, s, x, x_ld, gamma, eps, d,
                       static_cast<float*>(y), y_ld);
        return;
    }
    if (wt == kBF16)
        rmsnorm_rows_kernel<__nv_bfloat16><<<rows, 256, 0, s>>>(x, x_ld, gamma, eps, d,
                                                                  static_cast<__nv_bfloat16*>(y), y_ld);
    else
        rmsnorm_rows_kernel<float><<<rows, 256, 0, s>>>(x, x_ld, gamma, eps, d, static_cast<float*>(y), y_ld);
}

void gather_last(const float* x, int x_ld, int batch, int T, int d, float* xl, int xl_ld, cudaStream_t s) {
    gather_last_kernel<<<dim3(4, batch), 256, 0, s>>>(x, x_ld, T, d, xl, xl_ld);
}

void set_int(int* p, int v, cudaStream_t s) { set_int_kernel<<<1, 1, 0, s>>>(p, v); }

// Streaming-loader conversion (one element per thread, grid-stride): the
// f32 -> bf16 RNE of __float2bfloat16_rn equals the host path's bf16_bits for
// finite values, and the folds are the IEEE ops normalize<float> performs
// (inv = 1 / s, then x * inv; x * S), so device factors match the host
// normalize + upload path bit for bit.
__global__ void pack_f32_kernel(const PackArgs a) {
    const long long n = a.nrows * a.cols;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < n;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long lr = e / a.cols, c = e - lr * a.cols, r = a.r0 + lr;
        float v = a.src[e];
        if (a.fold == 1) v = __fmul_rn(v, __fdiv_rn(1.0f, a.scale[r]));
        else if (a.fold == 2) v = __fmul_rn(v, a.scale[c]);
        char* base = static_cast<char*>(a.dst);
        if (a.mode == 0) {
            const long long o = r * a.ld + c;
            if (a.dt == kBF16) reinterpret_cast<__nv_bfloat16*>(base)[o] = __float2bfloat16_rn(v);
            else reinterpret_cast<float*>(base)[o] = v;
        } else {
            const size_t o = a.lay.offset(static_cast<int>(c), static_cast<int>(r));
            if (a.dt == kBF16) *reinterpret_cast<__nv_bfloat16*>(base + o) = __float2bfloat16_rn(v);
            else *reinterpret_cast<float*>(base + o) = v;
        }
    }
}

template <typename E>
__global__ void copy_rows_at_kernel(const E* src, int src_ld, int col0, int ncols, E* dst, long long dst_bstride,
                                    int dst_ld, int T, int p0, const int* p0_dev) {
    const int row = blockIdx.x, b = row / T, t = row - b * T;
    const int p = (p0_dev ? *p0_dev : p0) + t;
    for (int j = threadIdx.x; j < ncols; j += blockDim.x)
        dst[b * dst_bstride + static_cast<long long>(p) * dst_ld + j] = src[static_cast<long long>(row) * src_ld + col0 + j];
}

void copy_rows_at(const void* src, int src_ld, int col0, int ncols, void* dst, long long dst_bstride, int dst_ld,
                  int batch, int T, int p0, const int* p0_dev, int esize, cudaStream_t s) {
    if (esize == 2)
        copy_rows_at_kernel<uint16_t><<<batch * T, 256, 0, s>>>(static_cast<const uint16_t*>(src), src_ld, col0, ncols,
                                                               static_cast<uint16_t*>(dst), dst_bstride, dst_ld, T, p0,
                                                               p0_dev);
    else
        copy_rows_at_kernel<float><<<batch * T, 256, 0, s>>>(static_cast<const float*>(src), src_ld, col0, ncols,
                                                            static_cast<float*>(dst), dst_bstride, dst_ld, T, p0, p0_dev);
}

void pack_f32(const PackArgs& a, cudaStream_t s) {
    const long long n = a.nrows * a.cols;
    if (n <= 0) return;
    const int blocks = static_cast<int>(std::min<long long>((n + 255) / 256, 148LL * 16));
    pack_f32_kernel<<<blocks, 256, 0, s>>>(a);
}

void argmax_rows(const float* logits, int V, int batch, int* tokens, int* out, int out_ld, const int* step,
                 cudaStream_t s) {
    argmax_rows_kernel<<<batch, 256, 0, s>>>(logits, V, tokens, out, out_ld, step);
}

void advance_pos(int* pos, int pos_inc, int* step, cudaStream_t s) { advance_pos_kernel<<<1, 1, 0, s>>>(pos, pos_inc, step); }

void synth_fill(const SynthFill& f, cudaStream_t s) {
    const long long n = f.rows * f.cols;
    long long blocks = (n + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    synth_fill_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(f);
}

}  // namespace fsvd::k
