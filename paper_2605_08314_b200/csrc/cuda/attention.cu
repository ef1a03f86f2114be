// Prefill causal attention: a T-token chunk at positions
// [p0, p0+T) attends cache rows [0, p0+T). Blockwise online softmax
// (partition-invariant; math.hpp:56-101) with 64-key tiles
// staged in shared memory. Decode attention lives in the megakernel
// (decode_mk_attn.cuh).
#include <math_constants.h>

#include "common.cuh"
#include "kernels.h"

namespace fsvd::k {
namespace {

using namespace fsvd::dev;

constexpr int kPQ = 64;        // queries per CTA
constexpr int kPK = 64;        // keys per tile
constexpr int kPThreads = 256; // 4 threads per query
template <typename T, int DH>
__global__ void __launch_bounds__(kPThreads) attn_prefill_kernel(const __grid_constant__ AttnPrefillArgs a) {
    extern __shared__ float sm[];
    constexpr int dh = DH;
    float* Ks = sm;                 // [kPK][dh + 1]
    float* Vs = Ks + kPK * (dh + 1);  // [kPK][dh]
    const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int tid = threadIdx.x, qi = tid >> 2, part = tid & 3;
    constexpr int slice = DH / 4;  // dims owned by this thread
    const int t = qt * kPQ + qi;
    const bool active = t < a.T;
    const int qpos = a.p0 + t;

    float qv[slice], acc[slice];
    const T* qrow = static_cast<const T*>(a.q) + static_cast<long long>(b * a.T + (active ? t : 0)) * a.q_ld + h * dh;
#pragma unroll
    for (int e = 0; e < slice; ++e) {
        qv[e] = to_f32<T>(qrow[part * slice + e]) * a.scale;
        acc[e] = 0.f;
    }
    float m = -CUDART_INF_F, l = 0.f;

    const T* K = static_cast<const T*>(a.kcache) + b * a.cache_bstride + h * a.cache_hstride;
    const T* V = static_cast<const T*>(a.vcache) + b * a.cache_bstride + h * a.cache_hstride;
    const int last_q = min(a.T, (qt + 1) * kPQ) - 1;
    const int kend = a.p0 + last_q + 1;  // keys needed by this CTA
    float sc[kPK];
    for (int k0 = 0; k0 < kend; k0 += kPK) {
        __syncthreads();
        for (int i = tid; i < kPK * dh; i += kPThreads) {
            const int r = i / dh, c = i % dh;
            const int j = k0 + r;
            const bool ok = j < kend;
            Ks[r * (dh + 1) + c] = ok ? to_f32<T>(K[static_cast<long long>(j) * dh + c]) : 0.f;
            Vs[r * dh + c] = ok ? to_f32<T>(V[static_cast<long long>(j) * dh + c]) : 0.f;
        }
        __syncthreads();
        float mt = -CUDART_INF_F;
#pragma unroll
        for (int r = 0; r < kPK; ++r) {
            float d = 0.f;
            const float* kr = Ks + r * (dh + 1) + part * slice;
#pragma unroll
            for (int e = 0; e < slice; ++e) d = fmaf(qv[e], kr[e], d);
            d += __shfl_xor_sync(0xffffffffu, d, 1);
            d += __shfl_xor_sync(0xffffffffu, d, 2);
            const bool ok = k0 + r <= qpos && k0 + r < kend;
            sc[r] = ok ? d : -CUDART_INF_F;
            mt = fmaxf(mt, sc[r]);
        }
        const float mn = fmaxf(m, mt);
        if (mn == -CUDART_INF_F) continue;
        const float rescale = expf(m - mn);
        l *= rescale;
#pragma unroll
        for (int e = 0; e < slice; ++e) acc[e] *= rescale;
#pragma unroll
        for (int r = 0; r < kPK; ++r) {
            const float w = expf(sc[r] - mn);
            l += w;
            const float* vr = Vs + r * dh + part * slice;
#pragma unroll
            for (int e = 0; e < slice; ++e) acc[e] = fmaf(w, vr[e], acc[e]);
        }
        m = mn;
    }
    if (!active) return;
    T* orow = static_cast<T*>(a.out) + static_cast<long long>(b * a.T + t) * a.out_ld + h * dh;
#pragma unroll
    for (int e = 0; e < slice; ++e) orow[part * slice + e] = from_f32<T>(acc[e] / l);
}

}  // namespace

void attn_prefill(WType wt, const AttnPrefillArgs& a, cudaStream_t s) {
    dim3 grid((a.T + kPQ - 1) / kPQ, a.n_heads, a.batch);
    const int smem = (kPK * (a.d_head + 1) + kPK * a.d_head) * static_cast<int>(sizeof(float));
#define FSVD_PRE(DH)                                                                                   \
    case DH:                                                                                           \
        if (wt == kBF16) {                                                                             \
            cudaFuncSetAttribute(attn_prefill_kernel<__nv_bfloat16, DH>,                               \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem);                   \
            attn_prefill_kernel<__nv_bfloat16, DH><<<grid, kPThreads, smem, s>>>(a);                   \
        } else {                                                                                       \
            cudaFuncSetAttribute(attn_prefill_kernel<float, DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
            attn_prefill_kernel<float, DH><<<grid, kPThreads, smem, s>>>(a);                           \
        }                                                                                              \
        break;
    switch (a.d_head) { FSVD_PRE(32) FSVD_PRE(64) FSVD_PRE(128) FSVD_PRE(256) default: break; }
#undef FSVD_PRE
}

}  // namespace fsvd::k
