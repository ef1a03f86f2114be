// Shared pieces of the decode megakernel: PTX wrappers (mbarrier, bulk copy,
// fences, mma), the shared-memory map, the unit split, and the phase-input
// staging that resolves the producer's pieces + epilogue.
#pragma once

#include <math_constants.h>

#include "common.cuh"
#include "decode_mk.h"
#include "kernels.h"

namespace fsvd::k::mk {

using namespace fsvd::dev;

constexpr int kWarpsMk = 8;
constexpr int kThreadsMk = kWarpsMk * 32;
constexpr int kSlots = 2;
constexpr int kPrefetch = 6;  // L2-prefetch distance (units) beyond the shared-memory slots

// ------------------------------------------------------------ PTX helpers --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// D(16x8, f32) += A(16x16, bf16, row) * B(16x8, bf16, col)
__device__ __forceinline__ void mma_bf16(float* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ bool better(float v, int i, float bv, int bi) { return v > bv || (v == bv && i < bi); }

// ------------------------------------------------------------ unit split --
__device__ __forceinline__ int unit_lo(int total, int c, int G) {
    return static_cast<int>(static_cast<long long>(total) * c / G);
}
// CTA owning unit U
__device__ __forceinline__ int unit_cta(int U, int total, int G) {
    int c = static_cast<int>(static_cast<long long>(U) * G / total);
    while (c + 1 < G && unit_lo(total, c + 1, G) <= U) ++c;
    while (c > 0 && unit_lo(total, c, G) > U) --c;
    return c;
}

// --------------------------------------------------------- shared memory --
struct Smem {
    char* slots;     // [warp][kSlots][kUnitBytes]
    uint64_t* full;  // [warp][kSlots]
    void* x;         // per phase: bf16 [2B][x_len] hi/lo planes, or f32 [B][x_len]
    int x_cap;       // elements per plane (this phase's x_len)
    float* part;     // [CTA-local unit][16][B] partials
    float* red;      // [kWarpsMk][d_head + 2] scratch
    float* misc;     // 256 floats
};

template <typename W>
struct XPlanes;
// bf16 weights: x is staged as two bf16 planes per batch row, x = hi + lo
// (RNE), the B operand of the tensor-core GEMV (column 2b = hi, 2b+1 = lo).
template <>
struct XPlanes<__nv_bfloat16> {
    static constexpr int kPlanes = 2;
    static __device__ __forceinline__ void put(const Smem& sm, int b, int i, float v) {
        __nv_bfloat16* p = static_cast<__nv_bfloat16*>(sm.x);
        const __nv_bfloat16 h = __float2bfloat16_rn(v);
        p[(2 * b) * sm.x_cap + i] = h;
        p[(2 * b + 1) * sm.x_cap + i] = __float2bfloat16_rn(v - __bfloat162float(h));
    }
};
template <>
struct XPlanes<float> {
    static constexpr int kPlanes = 1;
    static __device__ __forceinline__ void put(const Smem& sm, int b, int i, float v) {
        static_cast<float*>(sm.x)[b * sm.x_cap + i] = v;
    }
};

// ---------------------------------------------------------------- pieces --
__device__ __forceinline__ float4 ldcg4(const float* p) { return __ldcg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ float4 add4(float4 a, float4 b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }
__device__ __forceinline__ float comp(const float4& v, int i) { return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w)); }

// Sum of the S slot planes of pieces row r, batch b. The first four planes
// are loaded together; the summation order is fixed (((p0+p1)+p2)+p3)+...
template <int B>
__device__ __forceinline__ float piece_sum(const Pieces& pc, int r, int b) {
    const float* p = pc.base + static_cast<size_t>(r) * B + b;
    const size_t pl = static_cast<size_t>(pc.R) * B;
    const float p0 = __ldcg(p), p1 = pc.S > 1 ? __ldcg(p + pl) : 0.f;
    const float p2 = pc.S > 2 ? __ldcg(p + 2 * pl) : 0.f, p3 = pc.S > 3 ? __ldcg(p + 3 * pl) : 0.f;
    float s = ((p0 + p1) + p2) + p3;
    for (int j = 4; j < pc.S; ++j) s += __ldcg(p + j * pl);
    return s;
}
// The same for the 4 consecutive floats at row r (4/B rows x B), r aligned.
template <int B>
__device__ __forceinline__ float4 piece_sum4(const Pieces& pc, int r) {
    const float* p = pc.base + static_cast<size_t>(r) * B;
    const size_t pl = static_cast<size_t>(pc.R) * B;
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 p0 = ldcg4(p), p1 = pc.S > 1 ? ldcg4(p + pl) : z;
    const float4 p2 = pc.S > 2 ? ldcg4(p + 2 * pl) : z, p3 = pc.S > 3 ? ldcg4(p + 3 * pl) : z;
    float4 s = add4(add4(add4(p0, p1), p2), p3);
    for (int j = 4; j < pc.S; ++j) s = add4(s, ldcg4(p + j * pl));
    return s;
}

// -------------------------------------------------------- input staging --
// A "quad" = 4 consecutive floats of the [row][b] order: rows j0 .. j0+4/B-1
// of input x for every batch row b. Quads never straddle a segment boundary
// (segment offsets are multiples of 8); rows past a segment's logical rows
// inside its last tile read pieces of zero-padded weight rows, i.e. 0.
template <int B>
__device__ __forceinline__ float4 src_quad(const float* src, int ld, int j0) {
    if constexpr (B == 1) {
        return __ldcg(reinterpret_cast<const float4*>(src + j0));
    } else {
        const float2 a = __ldcg(reinterpret_cast<const float2*>(src + j0));
        const float2 b = __ldcg(reinterpret_cast<const float2*>(src + ld + j0));
        return make_float4(a.x, b.x, a.y, b.y);
    }
}
template <int B>
__device__ __forceinline__ void dst_quad(float* dst, int ld, int j0, float4 v) {
    if constexpr (B == 1) {
        *reinterpret_cast<float4*>(dst + j0) = v;
    } else {
        *reinterpret_cast<float2*>(dst + j0) = make_float2(v.x, v.z);
        *reinterpret_cast<float2*>(dst + ld + j0) = make_float2(v.y, v.w);
    }
}
template <typename W, int B>
__device__ __forceinline__ float4 emb_quad(const InputSpec& in, int j0) {
    float o[4];
#pragma unroll
    for (int b = 0; b < B; ++b) {
        const W* row = static_cast<const W*>(in.emb) + static_cast<long long>(__ldcg(in.tokens + b)) * in.emb_ld + j0;
#pragma unroll
        for (int rr = 0; rr < 4 / B; ++rr) o[rr * B + b] = to_f32<W>(row[rr]);
    }
    return make_float4(o[0], o[1], o[2], o[3]);
}

template <typename W, int B, int KIND>
__device__ __forceinline__ float4 quad_value(const InputSpec& in, int j0) {
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    if constexpr (KIND == kInPlain) {
        return j0 < in.len ? src_quad<B>(in.src + 0, in.src_ld, j0) : z;
    } else if constexpr (KIND == kInResidual) {
        if (j0 >= in.len) return z;
        const float4 x = src_quad<B>(in.src, in.src_ld, j0);
        return in.nseg ? add4(x, piece_sum4<B>(in.seg[0].pc, (in.seg[0].tbase * 16 + j0) * 1)) : x;
    } else if constexpr (KIND == kInEmbed) {
        return j0 < in.len ? emb_quad<W, B>(in, j0) : z;
    } else if constexpr (KIND == kInSilu) {
        const int r = j0 - in.seg[0].x_off;
        if (r < 0 || r >= in.seg[0].rows) return z;
        const float4 u = piece_sum4<B>(in.seg[0].pc, in.seg[0].tbase * 16 + r);
        const float4 g = piece_sum4<B>(in.seg[1].pc, in.seg[1].tbase * 16 + r);
        return make_float4(silu_mul(g.x, u.x), silu_mul(g.y, u.y), silu_mul(g.z, u.z), silu_mul(g.w, u.w));
    } else {  // kInPieces
#pragma unroll
        for (int s = 0; s < 3; ++s) {
            if (s >= in.nseg) break;
            const int r = j0 - in.seg[s].x_off;
            if (r >= 0 && r < in.seg[s].rows) return piece_sum4<B>(in.seg[s].pc, in.seg[s].tbase * 16 + r);
        }
        return z;
    }
}

// Stage quads of x into the shared planes (times gamma when the phase
// RMSNorms); residual kinds write their CTA's share of quads back to dst.
template <typename W, int B, int KIND>
__device__ void stage_loop(const MkGemv& g, const Smem& sm, int tid, int cta, int ncta, float* ss) {
    constexpr int RQ = 4 / B, QB = 4;
    const InputSpec& in = g.in;
    const int nq = g.x_len / RQ;
    const int nql = in.len / RQ;  // quads of the written-back residual
    const int w0 = unit_lo(nql, cta, ncta), w1 = unit_lo(nql, cta + 1, ncta);
    for (int q0 = tid; q0 < nq; q0 += QB * kThreadsMk) {
        float4 v[QB];
#pragma unroll
        for (int u = 0; u < QB; ++u) {
            const int q = q0 + u * kThreadsMk;
            v[u] = q < nq ? quad_value<W, B, KIND>(in, q * RQ) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < QB; ++u) {
            const int q = q0 + u * kThreadsMk;
            if (q >= nq) break;
            const int j0 = q * RQ;
            if constexpr (KIND == kInResidual || KIND == kInEmbed)
                if (in.dst && q >= w0 && q < w1) dst_quad<B>(in.dst, in.dst_ld, j0, v[u]);
#pragma unroll
            for (int rr = 0; rr < RQ; ++rr) {
                const int j = j0 + rr;
                const float gm = g.gamma ? (j < g.norm_len ? g.gamma[j] : 0.f) : 1.f;
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    const float x = comp(v[u], rr * B + b);
                    ss[b] = fmaf(x, x, ss[b]);
                    XPlanes<W>::put(sm, b, j, x * gm);
                }
            }
        }
    }
}

// Attention merge: x[b][h*dh + e] = sum_c acc_c[e] exp(m_c - M) / sum_c l_c exp(m_c - M)
// over the CTAs c whose cache-row range intersected head (b, h), in CTA
// order (slot j = j-th such CTA). sm.red: per head (M, 1/L, n).
template <typename W, int B>
__device__ void stage_attn(const InputSpec& in, const Smem& sm, int tid, int ncta) {
    const AttnMerge& am = in.am;
    const int dh = am.d_head, H = am.n_heads, st = dh + 4;
    const int len = *am.pos + 1;
    const long long N = static_cast<long long>(B) * H * len;
    float* rec = sm.red;
    for (int bh = tid; bh < B * H; bh += kThreadsMk) {
        const long long lo_bh = static_cast<long long>(bh) * len, hi_bh = lo_bh + len;
        int c = static_cast<int>(lo_bh * ncta / N);
        while (c > 0 && N * c / ncta > lo_bh) --c;
        int n = 0;
        for (; c < ncta; ++c) {
            const long long s0 = N * c / ncta, s1 = N * (c + 1) / ncta;
            if (s0 >= hi_bh) break;
            if ((s0 > lo_bh ? s0 : lo_bh) < (s1 < hi_bh ? s1 : hi_bh)) ++n;
        }
        const float* pb = am.partial + static_cast<long long>(bh) * am.splits * st;
        float M = -CUDART_INF_F;
        for (int j = 0; j < n; ++j) M = fmaxf(M, __ldcg(pb + j * st + dh + 1));
        float L = 0.f;
        for (int j = 0; j < n; ++j) L += __ldcg(pb + j * st + dh) * expf(__ldcg(pb + j * st + dh + 1) - M);
        rec[bh * 3 + 0] = M;
        rec[bh * 3 + 1] = 1.0f / L;
        rec[bh * 3 + 2] = __int_as_float(n);
    }
    __syncthreads();
    const int qph = dh / 4;
    for (int qq = tid; qq < B * H * qph; qq += kThreadsMk) {
        const int bh = qq / qph, e = (qq - bh * qph) * 4;
        const float M = rec[bh * 3], inv = rec[bh * 3 + 1];
        const int n = __float_as_int(rec[bh * 3 + 2]);
        const float* pb = am.partial + static_cast<long long>(bh) * am.splits * st;
        float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int j = 0; j < n; ++j) {
            const float w = expf(__ldcg(pb + j * st + dh + 1) - M);
            const float4 a = ldcg4(pb + j * st + e);
            o.x = fmaf(a.x, w, o.x);
            o.y = fmaf(a.y, w, o.y);
            o.z = fmaf(a.z, w, o.z);
            o.w = fmaf(a.w, w, o.w);
        }
        const int b = bh / H, hh = bh - b * H;
        XPlanes<W>::put(sm, b, hh * dh + e + 0, o.x * inv);
        XPlanes<W>::put(sm, b, hh * dh + e + 1, o.y * inv);
        XPlanes<W>::put(sm, b, hh * dh + e + 2, o.z * inv);
        XPlanes<W>::put(sm, b, hh * dh + e + 3, o.w * inv);
    }
}

// Stage this phase's input x (producer epilogue applied; times gamma when the
// phase RMSNorms) and compute inv_rms into misc[128 + b].
template <typename W, int B>
__device__ void stage_x(const MkGemv& g, const Smem& sm, int tid, int cta, int ncta) {
    const InputSpec& in = g.in;
    float ss[B];
#pragma unroll
    for (int b = 0; b < B; ++b) ss[b] = 0.f;
    switch (in.kind) {
        case kInAttn: {
            stage_attn<W, B>(in, sm, tid, ncta);
            const int H_dh = in.am.n_heads * in.am.d_head;
            for (int j = H_dh + tid; j < g.x_len; j += kThreadsMk)
#pragma unroll
                for (int b = 0; b < B; ++b) XPlanes<W>::put(sm, b, j, 0.f);
            break;
        }
        case kInPlain: stage_loop<W, B, kInPlain>(g, sm, tid, cta, ncta, ss); break;
        case kInResidual: stage_loop<W, B, kInResidual>(g, sm, tid, cta, ncta, ss); break;
        case kInEmbed: stage_loop<W, B, kInEmbed>(g, sm, tid, cta, ncta, ss); break;
        case kInSilu: stage_loop<W, B, kInSilu>(g, sm, tid, cta, ncta, ss); break;
        default: stage_loop<W, B, kInPieces>(g, sm, tid, cta, ncta, ss); break;
    }
    if (g.gamma) {
#pragma unroll
        for (int b = 0; b < B; ++b) ss[b] = warp_sum(ss[b]);
        if ((tid & 31) == 0)
#pragma unroll
            for (int b = 0; b < B; ++b) sm.misc[(tid >> 5) * 4 + b] = ss[b];
        __syncthreads();
        if (tid < B) {
            float t = 0.f;
            for (int w = 0; w < kWarpsMk; ++w) t += sm.misc[w * 4 + tid];
            sm.misc[128 + tid] = 1.0f / sqrtf(t / static_cast<float>(g.norm_len) + g.eps);
        }
    } else if (tid < B) {
        sm.misc[128 + tid] = 1.f;
    }
    __syncthreads();
}

}  // namespace fsvd::k::mk
