// Dense-KV attention kernels (sm_100a).
//
// Decode: each query head attends the contiguous dense
// cache rows [0, pos]. The reference runs one OnlineAttend::update over the
// whole history (math.hpp:56-101); here the history is split over `splits`
// CTAs per (sequence, head) -- split-K flash-decode -- and the last CTA to
// finish (atomic ticket) merges the partial (m, l, acc) triples in split
// order 0..S-1, so the result is deterministic for a given length.
//
// Prefill: causal attention of a T-token chunk at positions
// [p0, p0+T) against cache rows [0, p0+T). Blockwise online softmax
// (partition-invariant) with 64-key tiles staged in shared
// memory.
#include <math_constants.h>

#include "common.cuh"
#include "kernels.h"

namespace fsvd::k {
namespace {

using namespace fsvd::dev;

constexpr int kDecThreads = 128;
constexpr int kDecWarps = kDecThreads / 32;
constexpr int kMaxDh = 256;

template <typename T, int PER>
__device__ __forceinline__ void load_row(const T* p, int lane, float* out) {
#pragma unroll
    for (int e = 0; e < PER; ++e) out[e] = to_f32<T>(p[lane * PER + e]);
}

template <typename T, int DH>
__global__ void __launch_bounds__(kDecThreads) attn_decode_kernel(const __grid_constant__ AttnDecodeArgs a) {
    constexpr int per = DH / 32;
    extern __shared__ float scores[];  // [chunk_max]
    __shared__ float wred[kDecWarps][kMaxDh + 2];
    __shared__ int is_last;

    pdl_launch_dependents();
    pdl_wait();

    const int s = blockIdx.x % a.splits;
    const int bh = blockIdx.x / a.splits;
    const int b = bh / a.n_heads, h = bh % a.n_heads;
    const int len = *a.pos + 1;
    const int chunk = (len + a.splits - 1) / a.splits;
    const int j0 = min(len, s * chunk), j1 = min(len, j0 + chunk);
    constexpr int dh = DH;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    const T* K = static_cast<const T*>(a.kcache) + b * a.cache_bstride + h * a.cache_hstride;
    const T* V = static_cast<const T*>(a.vcache) + b * a.cache_bstride + h * a.cache_hstride;
    const float* q = a.q + static_cast<long long>(b) * a.n_heads * dh + h * dh;

    float qr[per];
#pragma unroll
    for (int e = 0; e < per; ++e) qr[e] = q[lane * per + e];

    // scores for this split
    float mloc = -CUDART_INF_F;
    for (int j = j0 + warp; j < j1; j += kDecWarps) {
        float kr[per];
        load_row<T, per>(K + static_cast<long long>(j) * dh, lane, kr);
        float d = 0.f;
#pragma unroll
        for (int e = 0; e < per; ++e) d = fmaf(qr[e], kr[e], d);
        d = warp_sum(d) * a.scale;
        if (lane == 0) scores[j - j0] = d;
        mloc = fmaxf(mloc, d);
    }
    if (lane == 0) wred[warp][0] = mloc;
    __syncthreads();
    float m = -CUDART_INF_F;
    for (int w = 0; w < kDecWarps; ++w) m = fmaxf(m, wred[w][0]);
    __syncthreads();

    // weighted value sum (each warp a strided subset of keys)
    float acc[per];
#pragma unroll
    for (int e = 0; e < per; ++e) acc[e] = 0.f;
    float l = 0.f;
    for (int j = j0 + warp; j < j1; j += kDecWarps) {
        const float w = expf(scores[j - j0] - m);
        l += w;
        float vr[per];
        load_row<T, per>(V + static_cast<long long>(j) * dh, lane, vr);
#pragma unroll
        for (int e = 0; e < per; ++e) acc[e] = fmaf(w, vr[e], acc[e]);
    }
#pragma unroll
    for (int e = 0; e < per; ++e) wred[warp][lane * per + e] = acc[e];
    if (lane == 0) wred[warp][dh] = l;
    __syncthreads();

    float* part = a.partial + (static_cast<long long>(bh) * a.splits + s) * (dh + 2);
    for (int i = tid; i < dh + 1; i += kDecThreads) {
        float t = 0.f;
        for (int w = 0; w < kDecWarps; ++w) t += wred[w][i];
        part[i] = t;  // acc[0..dh), l at [dh]
    }
    if (tid == 0) part[dh + 1] = m;
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        const unsigned ticket = atomicAdd(a.counters + bh, 1u);
        is_last = ticket == static_cast<unsigned>(a.splits - 1);
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();

    // merge the splits in fixed order
    const float* pbase = a.partial + static_cast<long long>(bh) * a.splits * (dh + 2);
    float M = -CUDART_INF_F;
    for (int t = 0; t < a.splits; ++t) M = fmaxf(M, __ldcg(pbase + t * (dh + 2) + dh + 1));
    float L = 0.f;
    for (int t = 0; t < a.splits; ++t) {
        const float mt = __ldcg(pbase + t * (dh + 2) + dh + 1);
        if (mt != -CUDART_INF_F) L += __ldcg(pbase + t * (dh + 2) + dh) * expf(mt - M);
    }
    for (int i = tid; i < dh; i += kDecThreads) {
        float o = 0.f;
        for (int t = 0; t < a.splits; ++t) {
            const float mt = __ldcg(pbase + t * (dh + 2) + dh + 1);
            if (mt != -CUDART_INF_F) o += __ldcg(pbase + t * (dh + 2) + i) * expf(mt - M);
        }
        a.out[static_cast<long long>(b) * a.n_heads * dh + h * dh + i] = o / L;
    }
    if (tid == 0) a.counters[bh] = 0u;
}

// ---------------------------------------------------------------- prefill --
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

void attn_decode(WType wt, const AttnDecodeArgs& a, cudaStream_t s, bool pdl) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(a.batch * a.n_heads * a.splits);
    cfg.blockDim = dim3(kDecThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    // scores buffer: the largest split chunk (runtime guarantees splits * kMaxChunk >= capacity)
    cfg.dynamicSmemBytes = kAttnMaxChunk * sizeof(float);
#define FSVD_DEC(DH)                                                             \
    case DH:                                                                     \
        if (wt == kBF16)                                                         \
            cudaLaunchKernelEx(&cfg, attn_decode_kernel<__nv_bfloat16, DH>, a);  \
        else                                                                     \
            cudaLaunchKernelEx(&cfg, attn_decode_kernel<float, DH>, a);          \
        break;
    switch (a.d_head) { FSVD_DEC(32) FSVD_DEC(64) FSVD_DEC(128) FSVD_DEC(256) default: break; }
#undef FSVD_DEC
}

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
