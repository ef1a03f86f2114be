// Microbenchmark for the decode GEMV streaming engine (development tool, not
// part of the product): y = W x for a large bf16 W [R x K] streamed by one
// CTA per SM. Each warp owns a contiguous range of (16-row tile, k-chunk)
// blocks; lanes 0..15 issue one cp.async.bulk per row into padded shared
// memory rows, optional L2 prefetch runs ahead, and the block is reduced with
// mma.sync.m16n8k16 (bf16 in, fp32 accumulate) using x split into hi/lo bf16
// columns. Prints GB/s and the max error vs a double-precision CPU product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/bench_stream.cu -o /tmp/bs && /tmp/bs
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e = (x);                                                                    \
        if (e != cudaSuccess) {                                                                 \
            printf("CUDA %s at %s:%d: %s\n", #x, __FILE__, __LINE__, cudaGetErrorString(e));     \
            exit(1);                                                                            \
        }                                                                                       \
    } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                     smem_u32(b)),
                 "r"(par)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void pf_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mma_bf16(float* d, const uint32_t* a, const uint32_t* b) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <int WARPS, int SLOTS, int KS, int PF>
__global__ void __launch_bounds__(WARPS * 32, 1)
    gemv_stream(const __nv_bfloat16* __restrict__ W, int R, int K, const float* __restrict__ x, float* y) {
    constexpr int RS = KS * 2 + 32;           // padded smem row stride (bytes)
    constexpr int BLK = 16 * RS;              // slot bytes
    extern __shared__ __align__(128) uint8_t sm[];
    uint8_t* slots = sm;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + WARPS * SLOTS * BLK);
    // x hi/lo planes (bf16), [2][K]
    __nv_bfloat16* xh = reinterpret_cast<__nv_bfloat16*>(full + WARPS * SLOTS);
    __nv_bfloat16* xl = xh + K + 16;
    float* part = reinterpret_cast<float*>(xl + K + 16);  // [tiles][nkc][16]

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int lo = (int)((long long)R * blockIdx.x / gridDim.x), hi = (int)((long long)R * (blockIdx.x + 1) / gridDim.x);
    const int ntile = (hi - lo + 15) / 16, nkc = (K + KS - 1) / KS, nblk = ntile * nkc;
    const int q0 = nblk * warp / WARPS, q1 = nblk * (warp + 1) / WARPS;
    if (tid < WARPS * SLOTS) mbar_init(&full[tid], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = tid; i < K; i += WARPS * 32) {
        const float v = x[i];
        const __nv_bfloat16 h = __float2bfloat16_rn(v);
        xh[i] = h;
        xl[i] = __float2bfloat16_rn(v - __bfloat162float(h));
    }
    __syncthreads();

    auto issue = [&](int q, int slot) {
        const int tile = q / nkc, kc = q - tile * nkc;
        const int r0 = lo + tile * 16, k0 = kc * KS, kb = min(KS, K - k0) * 2;
        const int nrows = min(16, hi - r0);
        uint64_t* bar = &full[warp * SLOTS + slot];
        uint8_t* dst = slots + (warp * SLOTS + slot) * BLK;
        if (lane == 0) mbar_expect_tx(bar, nrows * kb);
        __syncwarp();
        if (lane < nrows) bulk_g2s(dst + lane * RS, W + (size_t)(r0 + lane) * K + k0, kb, bar);
    };
    for (int s = 0; s < SLOTS && q0 + s < q1; ++s) issue(q0 + s, s);
    for (int s = SLOTS; s < SLOTS + PF && q0 + s < q1; ++s) {
        const int q = q0 + s, tile = q / nkc, kc = q - tile * nkc, r0 = lo + tile * 16;
        if (lane < min(16, hi - r0)) pf_l2(W + (size_t)(r0 + lane) * K + kc * KS, min(KS, K - kc * KS) * 2);
    }
    uint32_t seq = 0;
    for (int q = q0; q < q1; ++q, ++seq) {
        const int slot = seq % SLOTS;
        mbar_wait(&full[warp * SLOTS + slot], (seq / SLOTS) & 1);
        const int tile = q / nkc, kc = q - tile * nkc, k0 = kc * KS, kn = min(KS, K - k0);
        const uint8_t* buf = slots + (warp * SLOTS + slot) * BLK;
        float d[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
        for (int ks = 0; ks < kn; ks += 16) {
            uint32_t a[4], b[2];
            const uint2 r0v = *reinterpret_cast<const uint2*>(buf + g * RS + (ks + 4 * t) * 2);
            const uint2 r1v = *reinterpret_cast<const uint2*>(buf + (g + 8) * RS + (ks + 4 * t) * 2);
            a[0] = r0v.x;
            a[2] = r0v.y;
            a[1] = r1v.x;
            a[3] = r1v.y;
            uint2 xv = make_uint2(0, 0);
            if (g < 2) xv = *reinterpret_cast<const uint2*>((g == 0 ? xh : xl) + k0 + ks + 4 * t);
            b[0] = xv.x;
            b[1] = xv.y;
            mma_bf16(d, a, b);
        }
        if (t == 0) {
            part[(tile * nkc + kc) * 16 + g] = d[0] + d[1];
            part[(tile * nkc + kc) * 16 + g + 8] = d[2] + d[3];
        }
        __syncwarp();
        if (q + SLOTS < q1) issue(q + SLOTS, slot);
        if (q + SLOTS + PF < q1) {
            const int qq = q + SLOTS + PF, tl = qq / nkc, kk = qq - tl * nkc, rr = lo + tl * 16;
            if (lane < min(16, hi - rr)) pf_l2(W + (size_t)(rr + lane) * K + kk * KS, min(KS, K - kk * KS) * 2);
        }
    }
    __syncthreads();
    for (int r = lo + tid; r < hi; r += WARPS * 32) {
        const int tile = (r - lo) / 16, i = (r - lo) % 16;
        float s = 0.f;
        for (int kc = 0; kc < nkc; ++kc) s += part[(tile * nkc + kc) * 16 + i];
        y[r] = s;
    }
}


// Variant B: weights pre-arranged tile-major in HBM ([tile][kc][16 rows][KS],
// 16-byte chunks XOR-swizzled by row&7) so a block is ONE contiguous bulk copy
// that lands bank-conflict-free. CTA ranges are whole tiles.
template <int WARPS, int SLOTS, int KS>
__global__ void __launch_bounds__(WARPS * 32, 1)
    gemv_tiles(const __nv_bfloat16* __restrict__ Wt, int R, int K, const float* __restrict__ x, float* y) {
    constexpr int BLK = 16 * KS * 2;
    extern __shared__ __align__(128) uint8_t sm[];
    uint8_t* slots = sm;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + WARPS * SLOTS * BLK);
    __nv_bfloat16* xh = reinterpret_cast<__nv_bfloat16*>(full + WARPS * SLOTS);
    __nv_bfloat16* xl = xh + K + 16;
    float* part = reinterpret_cast<float*>(xl + K + 16);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int ntiles = (R + 15) / 16, nkc = K / KS;
    const int t0 = (int)((long long)ntiles * blockIdx.x / gridDim.x), t1 = (int)((long long)ntiles * (blockIdx.x + 1) / gridDim.x);
    const int nblk = (t1 - t0) * nkc;
    const int q0 = nblk * warp / WARPS, q1 = nblk * (warp + 1) / WARPS;
    if (tid < WARPS * SLOTS) mbar_init(&full[tid], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = tid; i < K; i += WARPS * 32) {
        const float v = x[i];
        const __nv_bfloat16 h = __float2bfloat16_rn(v);
        xh[i] = h;
        xl[i] = __float2bfloat16_rn(v - __bfloat162float(h));
    }
    __syncthreads();
    auto issue = [&](int q, int slot) {
        uint64_t* bar = &full[warp * SLOTS + slot];
        if (lane == 0) {
            mbar_expect_tx(bar, BLK);
            bulk_g2s(slots + (warp * SLOTS + slot) * BLK, reinterpret_cast<const uint8_t*>(Wt) + ((size_t)t0 * nkc + q) * BLK, BLK, bar);
        }
    };
    for (int s = 0; s < SLOTS && q0 + s < q1; ++s) issue(q0 + s, s);
    uint32_t seq = 0;
    for (int q = q0; q < q1; ++q, ++seq) {
        const int slot = seq % SLOTS;
        mbar_wait(&full[warp * SLOTS + slot], (seq / SLOTS) & 1);
        const int tile = q / nkc, kc = q - tile * nkc, k0 = kc * KS;
        const uint8_t* buf = slots + (warp * SLOTS + slot) * BLK;
        float d[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
        for (int ks = 0; ks < KS; ks += 16) {
            const int c = (ks + 4 * t) / 8;  // 16-byte chunk index within the row
            const int off = ((c ^ (g & 7)) << 4) + ((t & 1) << 3);
            const uint2 r0v = *reinterpret_cast<const uint2*>(buf + g * KS * 2 + off);
            const uint2 r1v = *reinterpret_cast<const uint2*>(buf + (g + 8) * KS * 2 + off);
            uint32_t a[4] = {r0v.x, r1v.x, r0v.y, r1v.y}, b[2];
            uint2 xv = make_uint2(0, 0);
            if (g < 2) xv = *reinterpret_cast<const uint2*>((g == 0 ? xh : xl) + k0 + ks + 4 * t);
            b[0] = xv.x;
            b[1] = xv.y;
            mma_bf16(d, a, b);
        }
        if (t == 0) {
            part[(tile * nkc + kc) * 16 + g] = d[0] + d[1];
            part[(tile * nkc + kc) * 16 + g + 8] = d[2] + d[3];
        }
        __syncwarp();
        if (q + SLOTS < q1) issue(q + SLOTS, slot);
    }
    __syncthreads();
    for (int r = t0 * 16 + tid; r < min(R, t1 * 16); r += WARPS * 32) {
        const int tile = r / 16 - t0, i = r % 16;
        float s = 0.f;
        for (int kc = 0; kc < nkc; ++kc) s += part[(tile * nkc + kc) * 16 + i];
        y[r] = s;
    }
}

template <int WARPS, int SLOTS, int KS>
void run_tiles(const std::vector<__nv_bfloat16>& Wb, int R, int K, const float* dx, float* dy,
               const std::vector<float>& Wh, const std::vector<float>& xh, int iters) {
    if (K % KS) return;
    const int ntiles = (R + 15) / 16, nkc = K / KS;
    std::vector<__nv_bfloat16> T((size_t)ntiles * 16 * K, __float2bfloat16_rn(0.f));
    for (int r = 0; r < R; ++r)
        for (int k = 0; k < K; ++k) {
            const int tile = r / 16, i = r % 16, kc = k / KS, kk = k % KS;
            const int c = kk / 8, e = kk % 8;
            const size_t off = ((size_t)tile * nkc + kc) * 16 * KS + i * KS + (((c ^ (i & 7)) * 8) + e);
            T[off] = Wb[(size_t)r * K + k];
        }
    __nv_bfloat16* dT;
    CK(cudaMalloc(&dT, T.size() * 2));
    CK(cudaMemcpy(dT, T.data(), T.size() * 2, cudaMemcpyHostToDevice));
    constexpr int BLK = 16 * KS * 2;
    const int tiles_cta = (ntiles + 147) / 148 + 1;
    const int smem = WARPS * SLOTS * BLK + WARPS * SLOTS * 8 + (2 * (K + 16)) * 2 + tiles_cta * nkc * 16 * 4 + 64;
    if (smem > 227 * 1024) {
        printf("tiles W%d S%d KS%d: smem %d too big\n", WARPS, SLOTS, KS, smem);
        cudaFree(dT);
        return;
    }
    auto fn = gemv_tiles<WARPS, SLOTS, KS>;
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    fn<<<148, WARPS * 32, smem>>>(dT, R, K, dx, dy);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < iters; ++i) fn<<<148, WARPS * 32, smem>>>(dT, R, K, dx, dy);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<float> y(R);
    CK(cudaMemcpy(y.data(), dy, R * 4, cudaMemcpyDeviceToHost));
    double maxerr = 0, maxref = 0;
    for (int r = 0; r < R; r += 97) {
        double s = 0;
        for (int k = 0; k < K; ++k) s += (double)Wh[(size_t)r * K + k] * xh[k];
        maxerr = fmax(maxerr, fabs(s - y[r]));
        maxref = fmax(maxref, fabs(s));
    }
    printf("TILES R=%6d K=%5d W%d S%d KS%4d: %7.3f us/iter %7.1f GB/s  relerr %.2e\n", R, K, WARPS, SLOTS, KS,
           ms * 1e3 / iters, (double)R * K * 2 * iters / (ms * 1e-3) / 1e9, maxerr / maxref);
    cudaFree(dT);
}

template <int WARPS, int SLOTS, int KS, int PF>
void run(const __nv_bfloat16* dW, int R, int K, const float* dx, float* dy, const std::vector<float>& Wh,
         const std::vector<float>& xh, int iters) {
    constexpr int RS = KS * 2 + 32, BLK = 16 * RS;
    const int rows_cta = (R + 147) / 148 + 1;
    const int smem = WARPS * SLOTS * BLK + WARPS * SLOTS * 8 + (2 * (K + 16)) * 2 + ((rows_cta + 15) / 16) * ((K + KS - 1) / KS) * 16 * 4 + 64;
    if (smem > 227 * 1024) {
        printf("W%d S%d KS%d PF%d: smem %d too big\n", WARPS, SLOTS, KS, PF, smem);
        return;
    }
    auto fn = gemv_stream<WARPS, SLOTS, KS, PF>;
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    fn<<<148, WARPS * 32, smem>>>(dW, R, K, dx, dy);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < iters; ++i) fn<<<148, WARPS * 32, smem>>>(dW, R, K, dx, dy);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<float> y(R);
    CK(cudaMemcpy(y.data(), dy, R * 4, cudaMemcpyDeviceToHost));
    double maxerr = 0, maxref = 0;
    for (int r = 0; r < R; r += 97) {
        double s = 0;
        for (int k = 0; k < K; ++k) s += (double)Wh[(size_t)r * K + k] * xh[k];
        maxerr = fmax(maxerr, fabs(s - y[r]));
        maxref = fmax(maxref, fabs(s));
    }
    const double gbs = (double)R * K * 2 * iters / (ms * 1e-3) / 1e9;
    printf("R=%6d K=%5d W%d S%d KS%4d PF%2d: %7.3f us/iter %7.1f GB/s  relerr %.2e\n", R, K, WARPS, SLOTS, KS, PF,
           ms * 1e3 / iters, gbs, maxerr / maxref);
}

int main() {
    const int shapes[][2] = {{32000, 4096}, {11008, 1792}, {12288, 1280}, {1792, 11008}, {3696, 4096}};
    for (auto& sh : shapes) {
        const int R = sh[0], K = sh[1];
        std::vector<float> Wh((size_t)R * K), xh(K);
        std::vector<__nv_bfloat16> Wb((size_t)R * K);
        uint64_t st = 12345;
        auto rnd = [&] {
            st = st * 6364136223846793005ull + 1442695040888963407ull;
            return ((st >> 33) & 0xFFFFFF) / 16777216.0f - 0.5f;
        };
        for (size_t i = 0; i < Wh.size(); ++i) {
            Wb[i] = __float2bfloat16_rn(rnd());
            Wh[i] = __bfloat162float(Wb[i]);
        }
        for (auto& v : xh) v = rnd();
        __nv_bfloat16* dW;
        float *dx, *dy;
        CK(cudaMalloc(&dW, Wb.size() * 2));
        CK(cudaMalloc(&dx, K * 4));
        CK(cudaMalloc(&dy, R * 4));
        CK(cudaMemcpy(dW, Wb.data(), Wb.size() * 2, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dx, xh.data(), K * 4, cudaMemcpyHostToDevice));
        const int iters = 20;
        run<8, 2, 256, 0>(dW, R, K, dx, dy, Wh, xh, iters);
        run_tiles<8, 2, 256>(Wb, R, K, dx, dy, Wh, xh, iters);
        run_tiles<8, 3, 256>(Wb, R, K, dx, dy, Wh, xh, iters);
        run_tiles<4, 3, 512>(Wb, R, K, dx, dy, Wh, xh, iters);
        run_tiles<8, 2, 512>(Wb, R, K, dx, dy, Wh, xh, iters);
        run_tiles<4, 4, 256>(Wb, R, K, dx, dy, Wh, xh, iters);
        run_tiles<16, 2, 128>(Wb, R, K, dx, dy, Wh, xh, iters);
        run_tiles<12, 2, 256>(Wb, R, K, dx, dy, Wh, xh, iters);
        cudaFree(dW);
        cudaFree(dx);
        cudaFree(dy);
    }
    return 0;
}
