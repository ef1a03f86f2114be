// Prefill GEMM, CUDA-core path: Y[t][n] = epi(sum_k X[t][k] * W^T[n][k]).
//
// Used for the fp32 parity mode (f32 runtime accumulates in
// f32), where tensor cores would change the arithmetic. The bf16 mode runs
// the tcgen05 GEMM in gemm_tc.cu. Weights are read from the tile layout
// (layout.h). Same epilogues as the tensor-core path:
// plain store, residual add, RoPE + KV append for the QKV reconstruction
// (SPEC.md:308), and the dual up/gate SiLU.mul.
#include "common.cuh"
#include "kernels.h"

namespace fsvd::k {
namespace {

using namespace fsvd::dev;

constexpr int BM = 64, BN = 128, BK = 32, TM = 4, TN = 8, NT = 256;

template <typename T, bool DUAL>
__global__ void __launch_bounds__(NT) gemm_simt_kernel(const __grid_constant__ GemmArgs a) {
    __shared__ float Xs[BK][BM + 4];
    __shared__ float Ws[1][BK][BN + 4];

    // map blockIdx.y -> (segment, feature tile)
    int tile = blockIdx.y, s = 0;
    const int nseg = DUAL ? 1 : a.nseg;
    while (s + 1 < nseg && tile >= (a.seg[s].rows + BN - 1) / BN) {
        tile -= (a.seg[s].rows + BN - 1) / BN;
        ++s;
    }
    const GemvSeg& sg = a.seg[s];
    const int n0 = tile * BN, m0 = blockIdx.x * BM;
    const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
    const T* X = static_cast<const T*>(a.x);

    float acc[DUAL ? 2 : 1][TM][TN];
#pragma unroll
    for (int d = 0; d < (DUAL ? 2 : 1); ++d)
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) acc[d][i][j] = 0.f;

#pragma unroll
    for (int d = 0; d < (DUAL ? 2 : 1); ++d) {
        const GemvSeg& sd = a.seg[DUAL ? d : s];
        const char* Wt = static_cast<const char*>(sd.w);
        const WLayout lay = sd.layout(sizeof(T));
        for (int k0 = 0; k0 < sd.k; k0 += BK) {
            __syncthreads();
            for (int i = tid; i < BM * BK; i += NT) {
                const int m = i / BK, kk = i % BK;
                const int t = m0 + m, k = k0 + kk;
                Xs[kk][m] = (t < a.M && k < sd.k) ? to_f32<T>(X[static_cast<long long>(t) * a.x_ld + sd.x_off + k]) : 0.f;
            }
            for (int i = tid; i < BN * BK; i += NT) {
                const int n = i / BK, kk = i % BK;
                const int r = n0 + n, k = k0 + kk;
                Ws[0][kk][n] = (r < sd.rows && k < sd.k) ? to_f32<T>(*reinterpret_cast<const T*>(Wt + lay.offset(r, k))) : 0.f;
            }
            __syncthreads();
#pragma unroll 8
            for (int kk = 0; kk < BK; ++kk) {
                float xa[TM], wb[TN];
#pragma unroll
                for (int i = 0; i < TM; ++i) xa[i] = Xs[kk][ty * TM + i];
#pragma unroll
                for (int j = 0; j < TN; ++j) wb[j] = Ws[0][kk][tx * TN + j];
#pragma unroll
                for (int i = 0; i < TM; ++i)
#pragma unroll
                    for (int j = 0; j < TN; ++j) acc[d][i][j] = fmaf(xa[i], wb[j], acc[d][i][j]);
            }
        }
    }

    // epilogue
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int t = m0 + ty * TM + i;
        if (t >= a.M) continue;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const int n = n0 + tx * TN + j;
            if (n >= sg.rows) continue;
            const float v = acc[0][i][j];
            if constexpr (DUAL) {
                static_cast<T*>(a.y)[static_cast<long long>(t) * a.y_ld + sg.y_off + n] =
                    from_f32<T>(silu_mul(acc[1][i][j], v));
            } else if (a.epi == kGemmStore) {
                static_cast<T*>(a.y)[static_cast<long long>(t) * a.y_ld + sg.y_off + n] = from_f32<T>(v);
            } else if (a.epi == kGemmAddF32) {
                static_cast<float*>(a.y)[static_cast<long long>(t) * a.y_ld + sg.y_off + n] += v;
            } else {  // kGemmQKV
                const int b = t / a.T, pos = (a.p0_dev ? *a.p0_dev : a.p0) + t % a.T;
                float out = v;
                if (sg.epi != kEpiV) {
                    const float other = acc[0][i][j ^ 1];
                    const int ih = n % a.d_head;
                    const float2 cs = a.rope[static_cast<long long>(pos) * (a.d_head / 2) + (ih >> 1)];
                    out = (ih & 1) ? __fadd_rn(__fmul_rn(other, cs.y), __fmul_rn(v, cs.x))
                                   : __fsub_rn(__fmul_rn(v, cs.x), __fmul_rn(other, cs.y));
                }
                if (sg.epi == kEpiRopeQ) {
                    static_cast<T*>(a.y)[static_cast<long long>(t) * a.y_ld + sg.y_off + n] = from_f32<T>(out);
                } else {
                    const int h = n / a.d_head, ih = n % a.d_head;
                    T* c = static_cast<T*>(sg.epi == kEpiRopeK ? a.kcache : a.vcache);
                    c[b * a.cache_bstride + h * a.cache_hstride + static_cast<long long>(pos) * a.d_head + ih] =
                        from_f32<T>(out);
                }
            }
        }
    }
}

}  // namespace

void gemm_simt(WType wt, const GemmArgs& a, cudaStream_t s) {
    int tiles = 0;
    const int nseg = a.epi == kGemmSilu ? 1 : a.nseg;
    for (int i = 0; i < nseg; ++i) tiles += (a.seg[i].rows + BN - 1) / BN;
    dim3 grid((a.M + BM - 1) / BM, tiles);
    const bool dual = a.epi == kGemmSilu;
    if (wt == kBF16) {
        if (dual)
            gemm_simt_kernel<__nv_bfloat16, true><<<grid, NT, 0, s>>>(a);
        else
            gemm_simt_kernel<__nv_bfloat16, false><<<grid, NT, 0, s>>>(a);
    } else {
        if (dual)
            gemm_simt_kernel<float, true><<<grid, NT, 0, s>>>(a);
        else
            gemm_simt_kernel<float, false><<<grid, NT, 0, s>>>(a);
    }
}

}  // namespace fsvd::k
