// Development tool (not product): correctness + throughput of the prefill
// GEMM paths of libfsvd_b200.so on one shape, Y = X . W^T (bf16, fp32 acc).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++20 -I include \
//        tools/gemm_bench.cu -o /tmp/gemm_bench -L paper_2605_08314_b200 -lfsvd_b200 \
//        -Xlinker -rpath=$PWD/paper_2605_08314_b200
//   /tmp/gemm_bench M N K [reps]
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2605_08314_b200/csrc/cuda/kernels.h"

using namespace fsvd::k;

#define CK(x)                                                                            \
    do {                                                                                 \
        cudaError_t e = (x);                                                             \
        if (e != cudaSuccess) {                                                          \
            printf("CUDA %s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));         \
            exit(1);                                                                     \
        }                                                                                \
    } while (0)

static float frand(uint64_t& s) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    return ((s >> 40) / float(1 << 24)) * 2.f - 1.f;
}

int main(int argc, char** argv) {
    const int M = argc > 1 ? atoi(argv[1]) : 512, N = argc > 2 ? atoi(argv[2]) : 4096,
              K = argc > 3 ? atoi(argv[3]) : 4096, reps = argc > 4 ? atoi(argv[4]) : 20;
    const WLayout lay = make_layout(N, K, 2);
    const int ldx = (K + 63) / 64 * 64;
    std::vector<__nv_bfloat16> hx(size_t(M) * ldx), hw(lay.bytes() / 2);
    std::vector<float> fx(size_t(M) * K), fw(size_t(N) * K);
    uint64_t s = 1;
    for (int t = 0; t < M; ++t)
        for (int k = 0; k < ldx; ++k) {
            const float v = k < K ? frand(s) : 0.f;
            hx[size_t(t) * ldx + k] = __float2bfloat16_rn(v);
            if (k < K) fx[size_t(t) * K + k] = __bfloat162float(hx[size_t(t) * ldx + k]);
        }
    for (size_t i = 0; i < hw.size(); ++i) hw[i] = __float2bfloat16_rn(0.f);
    for (int n = 0; n < N; ++n)
        for (int k = 0; k < K; ++k) {
            const __nv_bfloat16 v = __float2bfloat16_rn(frand(s) * 0.05f);
            hw[lay.offset(n, k) / 2] = v;
            fw[size_t(n) * K + k] = __bfloat162float(v);
        }
    __nv_bfloat16 *dx, *dw, *dy, *dy2;
    CK(cudaMalloc(&dx, hx.size() * 2));
    CK(cudaMalloc(&dw, hw.size() * 2));
    CK(cudaMalloc(&dy, size_t(M) * N * 2));
    CK(cudaMalloc(&dy2, size_t(M) * N * 2));
    CK(cudaMemcpy(dx, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dw, hw.data(), hw.size() * 2, cudaMemcpyHostToDevice));
    GemmArgs a{};
    a.x = dx;
    a.x_ld = ldx;
    a.M = M;
    a.seg[0] = GemvSeg{dw, N, K, lay.kp, 0, 0, kEpiStore};
    a.nseg = 1;
    a.epi = kGemmStore;
    a.y = dy;
    a.y_ld = N;
    cudaStream_t st;
    CK(cudaStreamCreate(&st));
    gemm_tc(a, M, st);
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    GemmArgs b = a;
    b.y = dy2;
    gemm_simt(kBF16, b, st);
    CK(cudaStreamSynchronize(st));
    std::vector<__nv_bfloat16> hy(size_t(M) * N), hy2(size_t(M) * N);
    CK(cudaMemcpy(hy.data(), dy, hy.size() * 2, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hy2.data(), dy2, hy2.size() * 2, cudaMemcpyDeviceToHost));
    // spot-check vs fp64 host on a sample of outputs
    double maxerr = 0, maxref = 0, maxerr_simt = 0;
    for (int i = 0; i < 4096; ++i) {
        const int t = (i * 7919) % M, n = (i * 104729) % N;
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += double(fx[size_t(t) * K + k]) * fw[size_t(n) * K + k];
        maxref = fmax(maxref, fabs(ref));
        maxerr = fmax(maxerr, fabs(__bfloat162float(hy[size_t(t) * N + n]) - ref));
        maxerr_simt = fmax(maxerr_simt, fabs(__bfloat162float(hy2[size_t(t) * N + n]) - ref));
    }
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int i = 0; i < 3; ++i) gemm_tc(a, M, st);
    CK(cudaEventRecord(e0, st));
    for (int i = 0; i < reps; ++i) gemm_tc(a, M, st);
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double us = ms * 1e3 / reps;
    const double tf = 2.0 * M * N * K / (us * 1e-6) / 1e12;
    printf("gemm_tc M=%d N=%d K=%d: %.2f us  %.1f TFLOP/s  maxerr %.3e (simt %.3e) of max|ref| %.3e\n", M, N, K, us, tf,
           maxerr, maxerr_simt, maxref);
    return 0;
}
