// Prefill causal attention: a T-token chunk at positions
// [p0, p0+T) attends cache rows [0, p0+T). Blockwise online softmax
// (partition-invariant; math.hpp:56-101) with 64-key tiles
// staged in shared memory. Batch-1/2 decode attention runs inside the decode
// megakernel (decode_mk.cu, attn_phase); the batched engine's split-KV flash
// decode is attn_decode_kernel below.
#include <math_constants.h>

#include <algorithm>
#include <cstdlib>

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
    const int p0 = a.p0_dev ? *a.p0_dev : a.p0;
    extern __shared__ float sm[];
    constexpr int dh = DH;
    float* Ks = sm;                 // [kPK][dh + 1]
    float* Vs = Ks + kPK * (dh + 1);  // [kPK][dh]
    const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int tid = threadIdx.x, qi = tid >> 2, part = tid & 3;
    constexpr int slice = DH / 4;  // dims owned by this thread
    const int t = qt * kPQ + qi;
    const bool active = t < a.T;
    const int qpos = p0 + t;

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
    const int kend = p0 + last_q + 1;  // keys needed by this CTA
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

// ------------------------------------------------ tensor-core flash attention --
// bf16 mode: 64 queries of one (sequence, head) per CTA, 4 warps x 16 rows;
// 64-key tiles double-buffered in shared memory with cp.async; S = Q.K^T and
// O += P.V on the tensor cores (mma.sync m16n8k16, fp32 accumulate), online
// softmax in registers (the running-max recurrence of math.hpp:75-100).
constexpr int kFQ = 64, kFK = 64, kFThreads = kFQ / 16 * 32;  // 16 queries per warp

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool pred) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src), "r"(pred ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_addr(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_addr(p)));
}
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&v);
}

template <int DH>
__global__ void __launch_bounds__(kFThreads) attn_prefill_tc_kernel(const __grid_constant__ AttnPrefillArgs a) {
    pdl_launch_dependents();
    pdl_wait();
    const int p0 = a.p0_dev ? *a.p0_dev : a.p0;
    constexpr int LD = DH + 8;  // padded smem row (bf16): conflict-free ldmatrix
    extern __shared__ __align__(128) __nv_bfloat16 fsm[];
    __nv_bfloat16* Qs = fsm;                 // [kFQ][LD]
    __nv_bfloat16* Ks = Qs + kFQ * LD;       // [2][kFK][LD]
    __nv_bfloat16* Vs = Ks + 2 * kFK * LD;   // [2][kFK][LD]
    // causal work grows with the query tile: the heaviest tiles are scheduled first
    const int qt = gridDim.x - 1 - blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
    const int q0 = qt * kFQ;
    const __nv_bfloat16* Q = static_cast<const __nv_bfloat16*>(a.q) + static_cast<long long>(b) * a.T * a.q_ld + h * DH;
    const __nv_bfloat16* K = static_cast<const __nv_bfloat16*>(a.kcache) + b * a.cache_bstride + h * a.cache_hstride;
    const __nv_bfloat16* V = static_cast<const __nv_bfloat16*>(a.vcache) + b * a.cache_bstride + h * a.cache_hstride;
    const int last_q = min(a.T, q0 + kFQ) - 1;
    const int kend = p0 + last_q + 1;
    const int ntiles = (kend + kFK - 1) / kFK;
    constexpr int CPR = DH / 8;  // 16-byte chunks per row

    // Q tile + first K/V tile
    for (int i = tid; i < kFQ * CPR; i += kFThreads) {
        const int r = i / CPR, c = (i % CPR) * 8;
        const bool ok = q0 + r < a.T;
        cp_async16(Qs + r * LD + c, Q + static_cast<long long>(ok ? q0 + r : 0) * a.q_ld + c, ok);
    }
    auto load_kv = [&](int tile, int buf) {
        const int k0 = tile * kFK;
        for (int i = tid; i < kFK * CPR; i += kFThreads) {
            const int r = i / CPR, c = (i % CPR) * 8;
            const bool ok = k0 + r < kend;
            const long long off = static_cast<long long>(ok ? k0 + r : 0) * DH + c;
            cp_async16(Ks + (buf * kFK + r) * LD + c, K + off, ok);
            cp_async16(Vs + (buf * kFK + r) * LD + c, V + off, ok);
        }
    };
    load_kv(0, 0);
    cp_async_commit();

    // this thread's two query rows: g and g + 8 of the warp's 16
    const int rq0 = warp * 16 + g, rq1 = rq0 + 8;
    const int pos0 = p0 + min(q0 + rq0, a.T - 1), pos1 = p0 + min(q0 + rq1, a.T - 1);
    const float sl2 = a.scale * 1.4426950408889634f;  // scores in log2 units
    float m0 = -CUDART_INF_F, m1 = -CUDART_INF_F, l0 = 0.f, l1 = 0.f;
    float o[DH / 8][4];
#pragma unroll
    for (int n = 0; n < DH / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    uint32_t qf[DH / 16][4];

    for (int tile = 0; tile < ntiles; ++tile) {
        const int buf = tile & 1;
        if (tile + 1 < ntiles) load_kv(tile + 1, buf ^ 1);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        if (tile == 0) {
#pragma unroll
            for (int kk = 0; kk < DH / 16; ++kk)
                ldsm_x4(qf[kk], Qs + (warp * 16 + (lane & 7) + 8 * ((lane >> 3) & 1)) * LD + kk * 16 + 8 * (lane >> 4));
        }
        const __nv_bfloat16* Kb = Ks + buf * kFK * LD;
        const __nv_bfloat16* Vb = Vs + buf * kFK * LD;
        // S = Q K^T : 16 x 64 per warp (8 key n-tiles)
        float sc[kFK / 8][4];
#pragma unroll
        for (int n = 0; n < kFK / 8; ++n) sc[n][0] = sc[n][1] = sc[n][2] = sc[n][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk)
#pragma unroll
            for (int np = 0; np < kFK / 16; ++np) {
                uint32_t kb[4];
                ldsm_x4(kb, Kb + (np * 16 + (lane & 7) + 8 * (lane >> 4)) * LD + kk * 16 + 8 * ((lane >> 3) & 1));
                mma16816(sc[2 * np], qf[kk], kb[0], kb[1]);
                mma16816(sc[2 * np + 1], qf[kk], kb[2], kb[3]);
            }
        // causal mask + online softmax (per row: max over the quad)
        const int k0 = tile * kFK;
        float mx0 = -CUDART_INF_F, mx1 = -CUDART_INF_F;
#pragma unroll
        for (int n = 0; n < kFK / 8; ++n) {
            const int j = k0 + n * 8 + 2 * t4;
            sc[n][0] = j <= pos0 ? sc[n][0] * sl2 : -CUDART_INF_F;
            sc[n][1] = j + 1 <= pos0 ? sc[n][1] * sl2 : -CUDART_INF_F;
            sc[n][2] = j <= pos1 ? sc[n][2] * sl2 : -CUDART_INF_F;
            sc[n][3] = j + 1 <= pos1 ? sc[n][3] * sl2 : -CUDART_INF_F;
            mx0 = fmaxf(mx0, fmaxf(sc[n][0], sc[n][1]));
            mx1 = fmaxf(mx1, fmaxf(sc[n][2], sc[n][3]));
        }
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
        const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
        const float r0 = mn0 == -CUDART_INF_F ? 1.f : exp2f(m0 - mn0);
        const float r1 = mn1 == -CUDART_INF_F ? 1.f : exp2f(m1 - mn1);
        m0 = mn0;
        m1 = mn1;
        float s0 = 0.f, s1 = 0.f;
        uint32_t pf[kFK / 16][4];
#pragma unroll
        for (int n = 0; n < kFK / 8; ++n) {
            const float p0v = mn0 == -CUDART_INF_F ? 0.f : exp2f(sc[n][0] - mn0);
            const float p1v = mn0 == -CUDART_INF_F ? 0.f : exp2f(sc[n][1] - mn0);
            const float p2v = mn1 == -CUDART_INF_F ? 0.f : exp2f(sc[n][2] - mn1);
            const float p3v = mn1 == -CUDART_INF_F ? 0.f : exp2f(sc[n][3] - mn1);
            s0 += p0v + p1v;
            s1 += p2v + p3v;
            // P as the A operand of P.V: n-tile 2kk -> a0/a1, 2kk+1 -> a2/a3
            pf[n >> 1][(n & 1) * 2 + 0] = pack_bf16x2(p0v, p1v);
            pf[n >> 1][(n & 1) * 2 + 1] = pack_bf16x2(p2v, p3v);
        }
        l0 = l0 * r0 + s0;
        l1 = l1 * r1 + s1;
#pragma unroll
        for (int n = 0; n < DH / 8; ++n) {
            o[n][0] *= r0;
            o[n][1] *= r0;
            o[n][2] *= r1;
            o[n][3] *= r1;
        }
        // O += P V : k = 64 keys (4 steps), n = DH
#pragma unroll
        for (int kk = 0; kk < kFK / 16; ++kk)
#pragma unroll
            for (int dp = 0; dp < DH / 16; ++dp) {
                uint32_t vb[4];
                ldsm_x4_t(vb, Vb + (kk * 16 + (lane & 7) + 8 * ((lane >> 3) & 1)) * LD + dp * 16 + 8 * (lane >> 4));
                mma16816(o[2 * dp], pf[kk], vb[0], vb[1]);
                mma16816(o[2 * dp + 1], pf[kk], vb[2], vb[3]);
            }
        __syncthreads();
    }
    // row sums over the quad, normalize, store
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
    const float i0 = 1.f / l0, i1 = 1.f / l1;
    __nv_bfloat16* O = static_cast<__nv_bfloat16*>(a.out) + static_cast<long long>(b) * a.T * a.out_ld + h * DH;
    const int t0 = q0 + rq0, t1 = q0 + rq1;
#pragma unroll
    for (int n = 0; n < DH / 8; ++n) {
        const int c = n * 8 + 2 * t4;
        if (t0 < a.T)
            *reinterpret_cast<uint32_t*>(O + static_cast<long long>(t0) * a.out_ld + c) = pack_bf16x2(o[n][0] * i0, o[n][1] * i0);
        if (t1 < a.T)
            *reinterpret_cast<uint32_t*>(O + static_cast<long long>(t1) * a.out_ld + c) = pack_bf16x2(o[n][2] * i1, o[n][3] * i1);
    }
}

// ---------------------------------------------------------------- decode --
// Split-KV flash decode for one new query per sequence (batched engine, T = 1):
// grid (splits, H, B); CTA s takes keys [len*s/S, len*(s+1)/S) of (b, h), its 4
// warps stream 16-key batches (every K/V load of a batch in flight; lane = 4
// dims), online softmax per warp (math.hpp:56-101), warps merged in order into
// a partial (acc, l, m); attn_decode_combine merges the splits in split order.
constexpr int kDThreads = 128, kDKU = 16;

template <int DH>
__global__ void __launch_bounds__(kDThreads) attn_decode_kernel(const __grid_constant__ AttnPrefillArgs a, float* part,
                                                                int S) {
    constexpr int PER = DH / 32, ST = DH + 2, NW = kDThreads / 32;
    __shared__ float wst[NW][ST];
    pdl_launch_dependents();
    pdl_wait();
    const int sp = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int len = (a.p0_dev ? *a.p0_dev : a.p0) + 1;
    const int j0 = static_cast<int>(static_cast<long long>(len) * sp / S);
    const int j1 = static_cast<int>(static_cast<long long>(len) * (sp + 1) / S);
    const __nv_bfloat16* Kc = static_cast<const __nv_bfloat16*>(a.kcache) + b * a.cache_bstride + h * a.cache_hstride;
    const __nv_bfloat16* Vc = static_cast<const __nv_bfloat16*>(a.vcache) + b * a.cache_bstride + h * a.cache_hstride;
    float qr[PER];
    {
        const __nv_bfloat16* q = static_cast<const __nv_bfloat16*>(a.q) + static_cast<long long>(b) * a.q_ld + h * DH +
                                 lane * PER;
#pragma unroll
        for (int e = 0; e < PER; ++e) qr[e] = __bfloat162float(q[e]) * a.scale;
    }
    float m = -CUDART_INF_F, l = 0.f, acc[PER];
#pragma unroll
    for (int e = 0; e < PER; ++e) acc[e] = 0.f;
    for (int kb = j0 + warp * kDKU; kb < j1; kb += NW * kDKU) {
        const int k1 = min(kb + kDKU, j1);
        uint2 kq[kDKU], vq[kDKU];
#pragma unroll
        for (int u = 0; u < kDKU; ++u) {
            const int jj = min(kb + u, k1 - 1);  // clamp: duplicates are masked below
            kq[u] = __ldcs(reinterpret_cast<const uint2*>(Kc + static_cast<long long>(jj) * DH + lane * PER));
            vq[u] = __ldcs(reinterpret_cast<const uint2*>(Vc + static_cast<long long>(jj) * DH + lane * PER));
        }
        float sc[kDKU];
        float mb = -CUDART_INF_F;
#pragma unroll
        for (int u = 0; u < kDKU; ++u) {
            float d = qr[0] * bf16lo(kq[u].x);
            d = fmaf(qr[1], bf16hi(kq[u].x), d);
            d = fmaf(qr[2], bf16lo(kq[u].y), d);
            d = fmaf(qr[3], bf16hi(kq[u].y), d);
            d = warp_sum(d);
            sc[u] = kb + u < k1 ? d : -CUDART_INF_F;
            mb = fmaxf(mb, sc[u]);
        }
        const float mn = fmaxf(m, mb);
        const float r = expf(m - mn);
        l *= r;
#pragma unroll
        for (int e = 0; e < PER; ++e) acc[e] *= r;
#pragma unroll
        for (int u = 0; u < kDKU; ++u) {
            const float w = expf(sc[u] - mn);
            l += w;
            acc[0] = fmaf(w, bf16lo(vq[u].x), acc[0]);
            acc[1] = fmaf(w, bf16hi(vq[u].x), acc[1]);
            acc[2] = fmaf(w, bf16lo(vq[u].y), acc[2]);
            acc[3] = fmaf(w, bf16hi(vq[u].y), acc[3]);
        }
        m = mn;
    }
#pragma unroll
    for (int e = 0; e < PER; ++e) wst[warp][lane * PER + e] = acc[e];
    if (lane == 0) {
        wst[warp][DH] = l;
        wst[warp][DH + 1] = m;
    }
    __syncthreads();
    float M = -CUDART_INF_F;
#pragma unroll
    for (int w = 0; w < NW; ++w) M = fmaxf(M, wst[w][DH + 1]);
    float* dst = part + ((static_cast<long long>(b) * gridDim.y + h) * S + sp) * ST;
    for (int e = threadIdx.x; e < DH + 1; e += kDThreads) {
        float t = 0.f;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const float mw = wst[w][DH + 1];
            if (mw != -CUDART_INF_F) t += wst[w][e] * expf(mw - M);
        }
        dst[e] = t;
    }
    if (threadIdx.x == 0) dst[DH + 1] = M;
}

// Same split-KV decode with the K / V rows of a split streamed into shared
// memory by one producer thread (cp.async.bulk, 32 keys = 16 KiB per stage,
// kBStages deep): the bytes in flight per SM no longer depend on registers.
// Warp w reduces keys w, w + 4, ... of each stage (online softmax per warp, the
// same order as attn_decode_kernel's per-warp batches is not required: the
// warps are merged by max / rescale afterwards); same partial format.
constexpr int kBKeys = 32, kBStages = 6, kBThreads = 160;  // 4 consumer warps + 1 producer warp

__device__ __forceinline__ uint32_t sa32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int DH>
__global__ void __launch_bounds__(kBThreads) attn_decode_bulk_kernel(const __grid_constant__ AttnPrefillArgs a,
                                                                     float* part, int S) {
    constexpr int PER = DH / 32, ST = DH + 2, NW = 4;
    constexpr uint32_t kRow = DH * 2;  // bytes per key row (bf16)
    extern __shared__ __align__(128) uint8_t bsm[];
    uint8_t* ring = bsm;  // [stages][K 32 rows | V 32 rows]
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + kBStages * 2 * kBKeys * kRow);
    uint64_t* empty = full + kBStages;
    float* wst = reinterpret_cast<float*>(empty + kBStages);  // [NW][ST]
    const int sp = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kBStages; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa32(&full[i])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa32(&empty[i])), "r"(NW));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_launch_dependents();
    pdl_wait();
    const int len = (a.p0_dev ? *a.p0_dev : a.p0) + 1;
    const int j0 = static_cast<int>(static_cast<long long>(len) * sp / S);
    const int j1 = static_cast<int>(static_cast<long long>(len) * (sp + 1) / S);
    const int nchunks = (j1 - j0 + kBKeys - 1) / kBKeys;
    const __nv_bfloat16* Kc = static_cast<const __nv_bfloat16*>(a.kcache) + b * a.cache_bstride + h * a.cache_hstride;
    const __nv_bfloat16* Vc = static_cast<const __nv_bfloat16*>(a.vcache) + b * a.cache_bstride + h * a.cache_hstride;
    auto wait = [&](uint64_t* bar, uint32_t par) {
        asm volatile(
            "{\n.reg .pred p;\nBW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra BW_%=;\n}\n" ::"r"(
                sa32(bar)),
            "r"(par)
            : "memory");
    };
    if (warp == NW) {
        if (lane == 0) {
            for (int c = 0; c < nchunks; ++c) {
                const int st = c % kBStages;
                const uint32_t par = (c / kBStages) & 1;
                wait(&empty[st], par ^ 1);
                const int k0 = j0 + c * kBKeys, n = min(kBKeys, j1 - k0);
                const uint32_t bytes = static_cast<uint32_t>(n) * kRow;
                uint8_t* dk = ring + st * 2 * kBKeys * kRow;
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa32(&full[st])), "r"(2 * bytes)
                             : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        sa32(dk)),
                    "l"(Kc + static_cast<long long>(k0) * DH), "r"(bytes), "r"(sa32(&full[st]))
                    : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        sa32(dk + kBKeys * kRow)),
                    "l"(Vc + static_cast<long long>(k0) * DH), "r"(bytes), "r"(sa32(&full[st]))
                    : "memory");
            }
        }
        return;
    }
    float qr[PER];
    {
        const __nv_bfloat16* q = static_cast<const __nv_bfloat16*>(a.q) + static_cast<long long>(b) * a.q_ld + h * DH +
                                 lane * PER;
#pragma unroll
        for (int e = 0; e < PER; ++e) qr[e] = __bfloat162float(q[e]) * a.scale;
    }
    float m = -CUDART_INF_F, l = 0.f, acc[PER];
#pragma unroll
    for (int e = 0; e < PER; ++e) acc[e] = 0.f;
    constexpr int KW = kBKeys / NW;  // keys per warp per stage
    for (int c = 0; c < nchunks; ++c) {
        const int st = c % kBStages;
        wait(&full[st], (c / kBStages) & 1);
        const int n = min(kBKeys, j1 - (j0 + c * kBKeys));
        const uint8_t* kb = ring + st * 2 * kBKeys * kRow;
        const uint8_t* vb = kb + kBKeys * kRow;
        uint2 kq[KW], vq[KW];
#pragma unroll
        for (int u = 0; u < KW; ++u) {
            const int r = min(warp + NW * u, n - 1);  // clamp: masked below
            kq[u] = *reinterpret_cast<const uint2*>(kb + r * kRow + lane * PER * 2);
            vq[u] = *reinterpret_cast<const uint2*>(vb + r * kRow + lane * PER * 2);
        }
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa32(&empty[st])) : "memory");
        float sc[KW];
        float mb = -CUDART_INF_F;
#pragma unroll
        for (int u = 0; u < KW; ++u) {
            float d = qr[0] * bf16lo(kq[u].x);
            d = fmaf(qr[1], bf16hi(kq[u].x), d);
            d = fmaf(qr[2], bf16lo(kq[u].y), d);
            d = fmaf(qr[3], bf16hi(kq[u].y), d);
            d = warp_sum(d);
            sc[u] = warp + NW * u < n ? d : -CUDART_INF_F;
            mb = fmaxf(mb, sc[u]);
        }
        const float mn = fmaxf(m, mb);
        if (mn == -CUDART_INF_F) continue;
        const float r = expf(m - mn);
        l *= r;
#pragma unroll
        for (int e = 0; e < PER; ++e) acc[e] *= r;
#pragma unroll
        for (int u = 0; u < KW; ++u) {
            const float w = expf(sc[u] - mn);
            l += w;
            acc[0] = fmaf(w, bf16lo(vq[u].x), acc[0]);
            acc[1] = fmaf(w, bf16hi(vq[u].x), acc[1]);
            acc[2] = fmaf(w, bf16lo(vq[u].y), acc[2]);
            acc[3] = fmaf(w, bf16hi(vq[u].y), acc[3]);
        }
        m = mn;
    }
#pragma unroll
    for (int e = 0; e < PER; ++e) wst[warp * ST + lane * PER + e] = acc[e];
    if (lane == 0) {
        wst[warp * ST + DH] = l;
        wst[warp * ST + DH + 1] = m;
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    float M = -CUDART_INF_F;
#pragma unroll
    for (int w = 0; w < NW; ++w) M = fmaxf(M, wst[w * ST + DH + 1]);
    float* dst = part + ((static_cast<long long>(b) * gridDim.y + h) * S + sp) * ST;
    for (int e = threadIdx.x; e < DH + 1; e += NW * 32) {
        float t = 0.f;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const float mw = wst[w * ST + DH + 1];
            if (mw != -CUDART_INF_F) t += wst[w * ST + e] * expf(mw - M);
        }
        dst[e] = t;
    }
    if (threadIdx.x == 0) dst[DH + 1] = M;
}

template <int DH>
__global__ void __launch_bounds__(DH) attn_decode_combine(const __grid_constant__ AttnPrefillArgs a, const float* part,
                                                          int S) {
    constexpr int ST = DH + 2;
    pdl_launch_dependents();
    pdl_wait();
    const int h = blockIdx.x, b = blockIdx.y, e = threadIdx.x;
    const float* src = part + (static_cast<long long>(b) * gridDim.x + h) * S * ST;
    float MM = -CUDART_INF_F;
    for (int q = 0; q < S; ++q) MM = fmaxf(MM, __ldcg(src + q * ST + DH + 1));
    float L = 0.f, o = 0.f;
    for (int q = 0; q < S; ++q) {
        const float mq = __ldcg(src + q * ST + DH + 1);
        if (mq == -CUDART_INF_F) continue;  // empty split
        const float w = expf(mq - MM);
        L = fmaf(__ldcg(src + q * ST + DH), w, L);
        o = fmaf(__ldcg(src + q * ST + e), w, o);
    }
    static_cast<__nv_bfloat16*>(a.out)[static_cast<long long>(b) * a.out_ld + h * DH + e] = __float2bfloat16_rn(o / L);
}

}  // namespace

int attn_decode_splits(int batch, int n_heads, int capacity) {
    // Wave model of the bulk-copy kernel (2 CTAs per SM, ~96 KiB in flight each):
    // time ~ waves x (4 us per CTA + keys per split x 21.5 ns), fitted to the C3 / C5
    // split sweeps (C3 1 split 4.60 ms/step, 2: 4.70; C5 1: 6.40, 2: 6.50); a split
    // must win by 5 %; splits keep >= 64 keys each.
    const int n = batch * n_heads, slots = 2 * 148;
    int S = 1;
    double best = 1e30;
    for (int sp = 1; sp <= 16 && capacity / sp >= 64; ++sp) {
        const double waves = static_cast<double>((n * sp + slots - 1) / slots);
        const double t = waves * (4.0 + 0.0215 * capacity / sp);
        if (t < best * 0.95) {
            best = t;
            S = sp;
        }
    }
    if (const char* e = std::getenv("FSVD_ATTN_SPLITS")) S = std::atoi(e);  // development: forced split count
    return std::max(1, std::min(S, 64));
}

bool attn_decode(WType wt, const AttnPrefillArgs& a, float* part, int S, cudaStream_t s) {
    if (wt != kBF16 || a.T != 1 || a.d_head != 128 || a.q_ld % 4 || a.out_ld % 2) return false;
    if (!std::getenv("FSVD_ATTN_DEC_REG")) {
        constexpr int smem = kBStages * 2 * kBKeys * 256 + kBStages * 16 + 4 * (128 + 2) * 4;
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(attn_decode_bulk_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            attr = true;
        }
        launch_pdl(attn_decode_bulk_kernel<128>, dim3(S, a.n_heads, a.batch), dim3(kBThreads), smem, s, a, part, S);
    } else {
        launch_pdl(attn_decode_kernel<128>, dim3(S, a.n_heads, a.batch), dim3(kDThreads), 0, s, a, part, S);
    }
    launch_pdl(attn_decode_combine<128>, dim3(a.n_heads, a.batch), dim3(128), 0, s, a, static_cast<const float*>(part),
               S);
    return true;
}

void attn_prefill(WType wt, const AttnPrefillArgs& a, cudaStream_t s) {
    if (wt == kBF16 && attn_prefill_tcgen05(a, s)) return;
    if (wt == kBF16 && (a.d_head == 64 || a.d_head == 128) && a.q_ld % 8 == 0 && a.out_ld % 8 == 0) {
        dim3 grid((a.T + kFQ - 1) / kFQ, a.n_heads, a.batch);
        const int smem = (kFQ + 4 * kFK) * (a.d_head + 8) * 2;
        if (a.d_head == 128) {
            cudaFuncSetAttribute(attn_prefill_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            launch_pdl(attn_prefill_tc_kernel<128>, grid, dim3(kFThreads), smem, s, a);
        } else {
            cudaFuncSetAttribute(attn_prefill_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            launch_pdl(attn_prefill_tc_kernel<64>, grid, dim3(kFThreads), smem, s, a);
        }
        return;
    }
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
