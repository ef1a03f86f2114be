// Decode attention phase of the megakernel (dense-KV).
//
// Prologue: q for every head this CTA touches is reduced from the QKV
// reconstruction pieces and rotated (RoPE, math.hpp:30-44); the CTA whose
// cache-row range holds the current position of a head also reduces and
// rotates k, reduces v, and appends both to the dense cache.
// Body: the B*H*len cache rows are split evenly over the CTAs; each warp
// takes a contiguous run of keys, loads K and V for 8 keys per round trip
// (history prefetched to L2 during the QKV phases) and keeps a warp-local
// online softmax (m, l, acc) -- math.hpp:56-101. Warp states merge in warp
// order into the CTA's partial for the head, stored in the head's slot =
// rank of this CTA among the head's CTAs. The o-projection's input staging
// merges the slots in CTA order (decode_mk_common.cuh stage_attn), so the
// result is deterministic for a given length and grid.
#pragma once

#include "decode_mk_common.cuh"

namespace fsvd::k::mk {

__device__ __forceinline__ long long attn_row_start(long long N, int c, int G) { return N * c / G; }

template <typename T, int PER>
__device__ __forceinline__ void load_kv_row(const T* p, float* out) {
    if constexpr (sizeof(T) == 2 && PER == 4) {
        const uint2 v = __ldcg(reinterpret_cast<const uint2*>(p));
        out[0] = bf16lo(v.x);
        out[1] = bf16hi(v.x);
        out[2] = bf16lo(v.y);
        out[3] = bf16hi(v.y);
    } else if constexpr (sizeof(T) == 4 && PER == 4) {
        const float4 v = __ldcg(reinterpret_cast<const float4*>(p));
        out[0] = v.x;
        out[1] = v.y;
        out[2] = v.z;
        out[3] = v.w;
    } else {
#pragma unroll
        for (int e = 0; e < PER; ++e) out[e] = to_f32<T>(p[e]);
    }
}

// RoPE'd value of element e of head h (segment rows h*dh + e) from pieces
template <int B>
__device__ __forceinline__ float rope_elem(const MkAttn& a, int tbase, int h, int e, int b, int pos) {
    const int r = h * a.d_head + e, rp = h * a.d_head + (e ^ 1);
    const float v = piece_sum<B>(a.pc, tbase * 16 + r, b);
    const float u = piece_sum<B>(a.pc, tbase * 16 + rp, b);
    const float2 cs = a.rope[static_cast<long long>(pos) * (a.d_head / 2) + (e >> 1)];
    const float x0 = (e & 1) ? u : v, x1 = (e & 1) ? v : u;
    return (e & 1) ? __fadd_rn(__fmul_rn(x0, cs.y), __fmul_rn(x1, cs.x)) : __fsub_rn(__fmul_rn(x0, cs.x), __fmul_rn(x1, cs.y));
}

template <typename T, int B, int DH>
__device__ void attn_phase(const MkAttn& a, const Smem& sm, int tid, int cta, int ncta) {
    constexpr int PER = DH / 32, KU = 8;
    const int warp = tid >> 5, lane = tid & 31;
    const int pos = *a.pos, len = pos + 1;
    const long long N = static_cast<long long>(B) * a.n_heads * len;
    const long long r0 = attn_row_start(N, cta, ncta), r1 = attn_row_start(N, cta + 1, ncta);
    float* wst = sm.red;                          // [warps][DH + 2]: acc, l, m
    float* qs = static_cast<float*>(sm.x);        // [DH] q of the current head
    for (int bh = static_cast<int>(r0 / len); static_cast<long long>(bh) * len < r1; ++bh) {
        const long long lo_bh = static_cast<long long>(bh) * len, hi_bh = lo_bh + len;
        const int j0 = static_cast<int>((r0 > lo_bh ? r0 : lo_bh) - lo_bh);
        const int j1 = static_cast<int>((r1 < hi_bh ? r1 : hi_bh) - lo_bh);
        if (j1 <= j0) continue;
        const int b = bh / a.n_heads, h = bh % a.n_heads;
        T* Kc = static_cast<T*>(const_cast<void*>(a.kcache)) + b * a.cache_bstride + h * a.cache_hstride;
        T* Vc = static_cast<T*>(const_cast<void*>(a.vcache)) + b * a.cache_bstride + h * a.cache_hstride;
        // ---- prologue: q (and the new k/v row if it falls in this range) ----
        for (int e = tid; e < DH; e += kThreadsMk) {
            const float qv = rope_elem<B>(a, a.tbase_q, h, e, b, pos);
            qs[e] = qv;
            if (a.q_out) a.q_out[static_cast<long long>(b) * a.n_heads * DH + h * DH + e] = qv;
            if (pos >= j0 && pos < j1) {
                Kc[static_cast<long long>(pos) * DH + e] = from_f32<T>(rope_elem<B>(a, a.tbase_k, h, e, b, pos));
                const int r = h * DH + e;
                Vc[static_cast<long long>(pos) * DH + e] =
                    from_f32<T>(piece_sum<B>(a.pc, a.tbase_v * 16 + r, b));
            }
        }
        __syncthreads();
        float qr[PER];
#pragma unroll
        for (int e = 0; e < PER; ++e) qr[e] = qs[lane * PER + e] * a.scale;
        // ---- this warp's keys ----
        const int n = j1 - j0;
        const int k0 = j0 + n * warp / kWarpsMk, k1 = j0 + n * (warp + 1) / kWarpsMk;
        float m = -CUDART_INF_F, l = 0.f, acc[PER];
#pragma unroll
        for (int e = 0; e < PER; ++e) acc[e] = 0.f;
        for (int kb = k0; kb < k1; kb += KU) {
            float kr[KU][PER], vr[KU][PER];
#pragma unroll
            for (int u = 0; u < KU; ++u) {
                const int jj = min(kb + u, k1 - 1);  // clamp: duplicate loads are masked below
                load_kv_row<T, PER>(Kc + static_cast<long long>(jj) * DH + lane * PER, kr[u]);
                load_kv_row<T, PER>(Vc + static_cast<long long>(jj) * DH + lane * PER, vr[u]);
            }
            float s[KU];
            float mb = -CUDART_INF_F;
#pragma unroll
            for (int u = 0; u < KU; ++u) {
                float d = 0.f;
#pragma unroll
                for (int e = 0; e < PER; ++e) d = fmaf(qr[e], kr[u][e], d);
                d = warp_sum(d);
                s[u] = kb + u < k1 ? d : -CUDART_INF_F;
                mb = fmaxf(mb, s[u]);
            }
            const float mn = fmaxf(m, mb);
            const float rs = expf(m - mn);  // exp(-inf) = 0 on the first round
            l *= rs;
#pragma unroll
            for (int e = 0; e < PER; ++e) acc[e] *= rs;
#pragma unroll
            for (int u = 0; u < KU; ++u) {
                const float w = expf(s[u] - mn);
                l += w;
#pragma unroll
                for (int e = 0; e < PER; ++e) acc[e] = fmaf(w, vr[u][e], acc[e]);
            }
            m = mn;
        }
#pragma unroll
        for (int e = 0; e < PER; ++e) wst[warp * (DH + 2) + lane * PER + e] = acc[e];
        if (lane == 0) {
            wst[warp * (DH + 2) + DH] = l;
            wst[warp * (DH + 2) + DH + 1] = m;
        }
        __syncthreads();
        // slot of this CTA = number of contributors of bh before it
        int slot = 0;
        {
            int c = static_cast<int>(lo_bh * ncta / N);
            while (c > 0 && attn_row_start(N, c, ncta) > lo_bh) --c;
            for (; c < cta; ++c) {
                const long long s0 = attn_row_start(N, c, ncta), s1 = attn_row_start(N, c + 1, ncta);
                if ((s0 > lo_bh ? s0 : lo_bh) < (s1 < hi_bh ? s1 : hi_bh)) ++slot;
            }
        }
        float* part = a.partial + (static_cast<long long>(bh) * a.splits + slot) * (DH + 4);
        float M = -CUDART_INF_F;
        for (int w = 0; w < kWarpsMk; ++w) M = fmaxf(M, wst[w * (DH + 2) + DH + 1]);
        for (int i = tid; i < DH + 1; i += kThreadsMk) {
            float t = 0.f;
            for (int w = 0; w < kWarpsMk; ++w) {
                const float mw = wst[w * (DH + 2) + DH + 1];
                if (mw != -CUDART_INF_F) t += wst[w * (DH + 2) + i] * expf(mw - M);
            }
            part[i] = t;  // acc[0..DH), l at [DH]
        }
        if (tid == 0) part[DH + 1] = M;
        __syncthreads();
    }
}

// Prefetch this CTA's attention key range into L2 (the history rows are
// immutable during the step).
template <typename T, int B, int DH>
__device__ void attn_prefetch(const MkAttn& a, int tid, int cta, int ncta) {
    const int len = *a.pos + 1;
    const long long N = static_cast<long long>(B) * a.n_heads * len;
    const long long r0 = attn_row_start(N, cta, ncta), r1 = attn_row_start(N, cta + 1, ncta);
    int k = 0;
    for (int bh = static_cast<int>(r0 / len); static_cast<long long>(bh) * len < r1; ++bh, ++k) {
        const long long lo_bh = static_cast<long long>(bh) * len;
        const int j0 = static_cast<int>((r0 > lo_bh ? r0 : lo_bh) - lo_bh);
        const int j1 = static_cast<int>((r1 < lo_bh + len ? r1 : lo_bh + len) - lo_bh);
        if (j1 <= j0) continue;
        const int b = bh / a.n_heads, h = bh % a.n_heads;
        const size_t off = (b * a.cache_bstride + h * a.cache_hstride + static_cast<long long>(j0) * DH) * sizeof(T);
        const size_t bytes = static_cast<size_t>(j1 - j0) * DH * sizeof(T);
        if (tid == 2 * k) prefetch_l2_range(static_cast<const char*>(a.kcache) + off, bytes, 0, 1);
        if (tid == 2 * k + 1) prefetch_l2_range(static_cast<const char*>(a.vcache) + off, bytes, 0, 1);
    }
}

}  // namespace fsvd::k::mk
