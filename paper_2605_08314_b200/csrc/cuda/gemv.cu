// Decode low-rank GEMV chain kernels (sm_100a).
//
// One launch computes y = epilogue(x . W^T) for a decode batch of B <= 4
// rows: the x.A rank projection ("rank projections x.A") and the
// .B reconstruction (with fused RoPE + KV append, residual add, or SiLU.mul),
// replacing the reference's per-op Ops::gemv (kernels_scalar.cpp:11-21,
// kernels_avx2.cpp:26-71) chain. Weights stream from HBM exactly once.
//
// Work split: grid = one CTA per SM. CTA c owns the contiguous output-row
// range [R*c/G, R*(c+1)/G) (even-aligned so RoPE pairs stay in one CTA), so
// per-SM bytes are balanced to one row. A warp handles 4 rows at a time as
// 4 groups of 8 lanes; lane s of a group streams 16-byte chunks s, s+8, ...
// of its row with U chunks in flight, so each row is read as 128-byte
// coalesced segments and the 4 rows of a warp share the broadcast x chunk in
// shared memory. Rows reduce with 3 xor-shuffles inside the 8-lane group
// (fixed order: results are bitwise reproducible and independent of which
// CTA or launch computes a row -- the packed/no_merge and replay/eager
// bitwise invariants, rely on this).
//
// PDL: before griddepcontrol.wait the CTA issues cp.async.bulk.prefetch.L2
// for its whole weight slice, so the HBM stream of this kernel starts while
// the previous kernel is still finishing; activations are only touched after
// the wait.
#include "common.cuh"
#include "kernels.h"

namespace fsvd::k {
namespace {

using namespace fsvd::dev;

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

template <typename W>
struct Chunk;
template <>
struct Chunk<__nv_bfloat16> {
    static constexpr int kElems = 8;
    static __device__ __forceinline__ float dot(const uint4 w, const float* x, float acc) {
        const float4 x0 = *reinterpret_cast<const float4*>(x);
        const float4 x1 = *reinterpret_cast<const float4*>(x + 4);
        acc = fmaf(bf16lo(w.x), x0.x, acc);
        acc = fmaf(bf16hi(w.x), x0.y, acc);
        acc = fmaf(bf16lo(w.y), x0.z, acc);
        acc = fmaf(bf16hi(w.y), x0.w, acc);
        acc = fmaf(bf16lo(w.z), x1.x, acc);
        acc = fmaf(bf16hi(w.z), x1.y, acc);
        acc = fmaf(bf16lo(w.w), x1.z, acc);
        acc = fmaf(bf16hi(w.w), x1.w, acc);
        return acc;
    }
};
template <>
struct Chunk<float> {
    static constexpr int kElems = 4;
    static __device__ __forceinline__ float dot(const uint4 w, const float* x, float acc) {
        const float4 xv = *reinterpret_cast<const float4*>(x);
        acc = fmaf(__uint_as_float(w.x), xv.x, acc);
        acc = fmaf(__uint_as_float(w.y), xv.y, acc);
        acc = fmaf(__uint_as_float(w.z), xv.z, acc);
        acc = fmaf(__uint_as_float(w.w), xv.w, acc);
        return acc;
    }
};

struct RowRef {
    const char* w;    // row base
    int nchunk;       // 16-byte chunks in the row
    int x_off;        // elements
    int seg;
    int row;          // row index inside the segment
};

__device__ __forceinline__ RowRef resolve(const GemvArgs& a, int g, int esize) {
    RowRef r;
    int s = 0, start = 0;
    while (s + 1 < a.nseg && g >= start + a.seg[s].rows) {
        start += a.seg[s].rows;
        ++s;
    }
    const GemvSeg& sg = a.seg[s];
    r.seg = s;
    r.row = g - start;
    r.w = static_cast<const char*>(sg.w) + static_cast<size_t>(r.row) * sg.ldw * esize;
    r.nchunk = sg.k * esize / 16;
    r.x_off = sg.x_off;
    return r;
}

template <typename W>
__device__ __forceinline__ void store_cache(void* base, long long bstr, long long hstr, int b, int n, int d_head,
                                            int pos, float v) {
    const int h = n / d_head, i = n - h * d_head;
    W* p = static_cast<W*>(base) + b * bstr + h * hstr + static_cast<long long>(pos) * d_head + i;
    *p = from_f32<W>(v);
}

template <typename W, int B, bool DUAL, int U>
__global__ void __launch_bounds__(kThreads, 2) gemv_kernel(const __grid_constant__ GemvArgs a) {
    extern __shared__ float4 smem_f4[];
    float* xs = reinterpret_cast<float*>(smem_f4);
    constexpr int E = Chunk<W>::kElems;
    constexpr int ES = sizeof(W);
    const int tid = threadIdx.x;

    int total = DUAL ? a.seg[0].rows : 0;
    if (!DUAL)
        for (int s = 0; s < a.nseg; ++s) total += a.seg[s].rows;
    const int lo = static_cast<int>(static_cast<long long>(total) * blockIdx.x / gridDim.x) & ~1;
    const int hi = blockIdx.x + 1 == gridDim.x
                       ? total
                       : static_cast<int>(static_cast<long long>(total) * (blockIdx.x + 1) / gridDim.x) & ~1;

    // ---- weight prefetch into L2 (independent of the previous kernel) ----
    if (tid < 32) {
        int start = 0;
        for (int s = 0; s < a.nseg; ++s) {
            const GemvSeg& sg = a.seg[s];
            const int s_lo = DUAL ? lo : max(lo - start, 0);
            const int s_hi = DUAL ? hi : min(hi - start, sg.rows);
            if (s_hi > s_lo)
                prefetch_l2_range(static_cast<const char*>(sg.w) + static_cast<size_t>(s_lo) * sg.ldw * ES,
                                  static_cast<size_t>(s_hi - s_lo) * sg.ldw * ES, tid, 32);
            if (!DUAL) start += sg.rows;
        }
    }
    pdl_launch_dependents();
    pdl_wait();

    // ---- stage x (optionally RMSNorm'ed) in shared memory ----
    __shared__ float red[kWarps][B];
    __shared__ float inv_rms[B];
    if (a.gamma) {
        float ss[B];
#pragma unroll
        for (int b = 0; b < B; ++b) ss[b] = 0.f;
        for (int i = tid; i < a.norm_len; i += kThreads)
#pragma unroll
            for (int b = 0; b < B; ++b) {
                const float v = a.x[b * a.x_ld + i];
                ss[b] = fmaf(v, v, ss[b]);
            }
#pragma unroll
        for (int b = 0; b < B; ++b) ss[b] = warp_sum(ss[b]);
        if ((tid & 31) == 0)
#pragma unroll
            for (int b = 0; b < B; ++b) red[tid >> 5][b] = ss[b];
        __syncthreads();
        if (tid < B) {
            float t = 0.f;
            for (int w = 0; w < kWarps; ++w) t += red[w][tid];
            inv_rms[tid] = 1.0f / sqrtf(t / static_cast<float>(a.norm_len) + a.eps);
        }
        __syncthreads();
    }
    for (int i = tid; i < a.x_len; i += kThreads)
#pragma unroll
        for (int b = 0; b < B; ++b) {
            float v = a.x[b * a.x_ld + i];
            if (a.gamma) v = i < a.norm_len ? v * inv_rms[b] * a.gamma[i] : 0.f;
            xs[b * a.x_len + i] = v;
        }
    __syncthreads();

    const int warp = tid >> 5, lane = tid & 31, grp = lane >> 3, sub = lane & 7;
    for (int base = lo + warp * 4; base < hi; base += kWarps * 4) {
        const int g = base + grp;
        const bool valid = g < hi;
        RowRef r0 = resolve(a, valid ? g : lo, ES);
        RowRef r1 = r0;
        if constexpr (DUAL) {
            r1.seg = 1;
            r1.row = r0.row;
            r1.w = static_cast<const char*>(a.seg[1].w) + static_cast<size_t>(r0.row) * a.seg[1].ldw * ES;
            r1.nchunk = a.seg[1].k * ES / 16;
            r1.x_off = a.seg[1].x_off;
        }
        float acc0[B], acc1[B];
#pragma unroll
        for (int b = 0; b < B; ++b) acc0[b] = acc1[b] = 0.f;

        const int n0 = valid ? r0.nchunk : 0;
        const int n1 = DUAL && valid ? r1.nchunk : 0;
        const int nmax = max(n0, n1);
        for (int c0 = 0; c0 < nmax; c0 += 8 * U) {
            uint4 w0[U], w1[DUAL ? U : 1];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int c = c0 + sub + 8 * u;
                w0[u] = c < n0 ? ld_stream(r0.w + static_cast<size_t>(c) * 16) : make_uint4(0, 0, 0, 0);
                if constexpr (DUAL)
                    w1[u] = c < n1 ? ld_stream(r1.w + static_cast<size_t>(c) * 16) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int c = c0 + sub + 8 * u;
                if (c < n0)
#pragma unroll
                    for (int b = 0; b < B; ++b)
                        acc0[b] = Chunk<W>::dot(w0[u], xs + b * a.x_len + r0.x_off + c * E, acc0[b]);
                if constexpr (DUAL)
                    if (c < n1)
#pragma unroll
                        for (int b = 0; b < B; ++b)
                            acc1[b] = Chunk<W>::dot(w1[u], xs + b * a.x_len + r1.x_off + c * E, acc1[b]);
            }
        }
        __syncwarp();
#pragma unroll
        for (int b = 0; b < B; ++b) {
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) {
                acc0[b] += __shfl_xor_sync(0xffffffffu, acc0[b], o);
                if constexpr (DUAL) acc1[b] += __shfl_xor_sync(0xffffffffu, acc1[b], o);
            }
        }
        if constexpr (DUAL) {
            if (valid && sub == 0)
#pragma unroll
                for (int b = 0; b < B; ++b) a.y[b * a.y_ld + a.seg[0].y_off + r0.row] = silu_mul(acc1[b], acc0[b]);
            continue;
        } else {
            const int epi = a.seg[r0.seg].epi;
            // partner value for RoPE pairs (rows 2i, 2i+1 live in groups grp, grp^1)
            float partner[B];
#pragma unroll
            for (int b = 0; b < B; ++b) partner[b] = __shfl_xor_sync(0xffffffffu, acc0[b], 8);
            if (!valid || sub != 0) continue;
            const int yo = a.seg[r0.seg].y_off + r0.row;
            if (epi == kEpiStore) {
#pragma unroll
                for (int b = 0; b < B; ++b) a.y[b * a.y_ld + yo] = acc0[b];
            } else if (epi == kEpiAdd) {
#pragma unroll
                for (int b = 0; b < B; ++b) a.y[b * a.y_ld + yo] += acc0[b];
            } else {
                const int pos = *a.pos;
                const int n = r0.row;
                float out[B];
                if (epi == kEpiV) {
#pragma unroll
                    for (int b = 0; b < B; ++b) out[b] = acc0[b];
                } else {
                    // reference math.hpp:30-44: pair (2i, 2i+1), x0*c - x1*s, x0*s + x1*c
                    const int i = n % a.d_head;
                    const float2 cs = a.rope[static_cast<long long>(pos) * (a.d_head / 2) + (i >> 1)];
#pragma unroll
                    for (int b = 0; b < B; ++b) {
                        const float x0 = (i & 1) ? partner[b] : acc0[b];
                        const float x1 = (i & 1) ? acc0[b] : partner[b];
                        out[b] = (i & 1) ? __fadd_rn(__fmul_rn(x0, cs.y), __fmul_rn(x1, cs.x))
                                         : __fsub_rn(__fmul_rn(x0, cs.x), __fmul_rn(x1, cs.y));
                    }
                }
                if (epi == kEpiRopeQ) {
#pragma unroll
                    for (int b = 0; b < B; ++b) a.y[b * a.y_ld + yo] = out[b];
                } else {
                    void* cache = epi == kEpiRopeK ? a.kcache : a.vcache;
#pragma unroll
                    for (int b = 0; b < B; ++b)
                        store_cache<W>(cache, a.cache_bstride, a.cache_hstride, b, n, a.d_head, pos, out[b]);
                }
            }
        }
    }
}

template <typename W, int B>
void launch(const GemvArgs& a, int grid, cudaStream_t s, bool pdl) {
    const int smem = gemv_smem_bytes(B, a.x_len);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    if (a.dual) {
        constexpr int U = sizeof(W) == 2 ? 8 : 8;
        auto fn = gemv_kernel<W, B, true, U>;
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaLaunchKernelEx(&cfg, fn, a);
    } else {
        constexpr int U = sizeof(W) == 2 ? 16 : 16;
        auto fn = gemv_kernel<W, B, false, U>;
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaLaunchKernelEx(&cfg, fn, a);
    }
}

}  // namespace

int gemv_smem_bytes(int batch, int x_len) { return batch * x_len * static_cast<int>(sizeof(float)); }

void gemv(WType wt, int batch, const GemvArgs& a, int grid, cudaStream_t s, bool pdl) {
#define FSVD_GEMV_CASE(BB)                                  \
    case BB:                                                \
        if (wt == kBF16)                                    \
            launch<__nv_bfloat16, BB>(a, grid, s, pdl);     \
        else                                                \
            launch<float, BB>(a, grid, s, pdl);             \
        break;
    switch (batch) {
        FSVD_GEMV_CASE(1)
        FSVD_GEMV_CASE(2)
        FSVD_GEMV_CASE(3)
        FSVD_GEMV_CASE(4)
        default:
            break;
    }
#undef FSVD_GEMV_CASE
}

}  // namespace fsvd::k
