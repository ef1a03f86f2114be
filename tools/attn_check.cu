// Development tool (not product): the tcgen05 prefill flash attention
// (attn_tc.cu) against an fp64 CPU reference and the mma.sync kernel, over
// chunk lengths / history offsets / head sizes / batch, plus timing.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++20 tools/attn_check.cu \
//        -o /tmp/attn_check -L paper_2605_08314_b200 -lfsvd_b200 -Xlinker -rpath=$PWD/paper_2605_08314_b200
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2605_08314_b200/csrc/cuda/kernels.h"

using namespace fsvd::k;

static float bf(float x) { return __bfloat162float(__float2bfloat16(x)); }

static int run(int B, int H, int DH, int T, int p0, int cap, bool timing) {
    const int ld = H * DH;
    std::vector<__nv_bfloat16> q(static_cast<size_t>(B) * T * ld), kc(static_cast<size_t>(B) * H * cap * DH),
        vc(kc.size());
    unsigned s = 12345u + T * 7 + p0;
    auto rnd = [&] {
        s = s * 1664525u + 1013904223u;
        return (static_cast<int>(s >> 9) % 2001 - 1000) / 1000.f;
    };
    for (auto& x : q) x = __float2bfloat16(rnd());
    for (size_t i = 0; i < kc.size(); ++i) {
        const size_t pos = (i / DH) % cap;
        // rows past the history hold NaN: they must never reach the output
        kc[i] = __float2bfloat16(pos < static_cast<size_t>(p0 + T) ? rnd() : NAN);
        vc[i] = __float2bfloat16(pos < static_cast<size_t>(p0 + T) ? rnd() : NAN);
    }
    void *dq, *dk, *dv, *dout;
    cudaMalloc(&dq, q.size() * 2);
    cudaMalloc(&dk, kc.size() * 2);
    cudaMalloc(&dv, vc.size() * 2);
    cudaMalloc(&dout, q.size() * 2);
    cudaMemcpy(dq, q.data(), q.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dk, kc.data(), kc.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dv, vc.data(), vc.size() * 2, cudaMemcpyHostToDevice);
    AttnPrefillArgs a{};
    a.q = dq;
    a.q_ld = ld;
    a.kcache = dk;
    a.vcache = dv;
    a.cache_hstride = static_cast<long long>(cap) * DH;
    a.cache_bstride = H * a.cache_hstride;
    a.out = dout;
    a.out_ld = ld;
    a.batch = B;
    a.T = T;
    a.p0 = p0;
    a.n_heads = H;
    a.d_head = DH;
    a.scale = 1.f / std::sqrt(static_cast<float>(DH));
    std::vector<__nv_bfloat16> o_tc(q.size()), o_mma(q.size());
    cudaStream_t st;
    cudaStreamCreate(&st);
    unsetenv("FSVD_ATTN_MMA");
    attn_prefill(kBF16, a, st);
    cudaStreamSynchronize(st);
    cudaError_t e1 = cudaGetLastError();
    cudaMemcpy(o_tc.data(), dout, q.size() * 2, cudaMemcpyDeviceToHost);
    setenv("FSVD_ATTN_MMA", "1", 1);
    attn_prefill(kBF16, a, st);
    cudaStreamSynchronize(st);
    cudaMemcpy(o_mma.data(), dout, q.size() * 2, cudaMemcpyDeviceToHost);
    unsetenv("FSVD_ATTN_MMA");
    // fp64 reference on a sample of rows
    double err_tc = 0, err_mma = 0, mx = 0;
    int nan_tc = 0;
    for (int b = 0; b < B; ++b)
        for (int h = 0; h < H; ++h)
            for (int t = 0; t < T; t += (T > 64 ? 7 : 1)) {
                const int len = p0 + t + 1;
                std::vector<double> sc(len);
                double m = -1e300;
                for (int j = 0; j < len; ++j) {
                    double d = 0;
                    for (int e = 0; e < DH; ++e)
                        d += double(__bfloat162float(q[(size_t(b) * T + t) * ld + h * DH + e])) *
                             __bfloat162float(kc[((size_t(b) * H + h) * cap + j) * DH + e]);
                    sc[j] = d * a.scale;
                    m = std::max(m, sc[j]);
                }
                double L = 0;
                for (int j = 0; j < len; ++j) L += (sc[j] = std::exp(sc[j] - m));
                for (int e = 0; e < DH; ++e) {
                    double o = 0;
                    for (int j = 0; j < len; ++j) o += sc[j] * __bfloat162float(vc[((size_t(b) * H + h) * cap + j) * DH + e]);
                    o /= L;
                    const size_t idx = (size_t(b) * T + t) * ld + h * DH + e;
                    const double g1 = __bfloat162float(o_tc[idx]), g2 = __bfloat162float(o_mma[idx]);
                    if (std::isnan(g1)) ++nan_tc;
                    err_tc = std::max(err_tc, std::abs(g1 - o));
                    err_mma = std::max(err_mma, std::abs(g2 - o));
                    mx = std::max(mx, std::abs(o));
                }
            }
    float us_tc = 0, us_mma = 0;
    if (timing) {
        cudaEvent_t e0, e2;
        cudaEventCreate(&e0);
        cudaEventCreate(&e2);
        for (int mode = 0; mode < 2; ++mode) {
            if (mode) setenv("FSVD_ATTN_MMA", "1", 1);
            for (int i = 0; i < 3; ++i) attn_prefill(kBF16, a, st);
            cudaEventRecord(e0, st);
            for (int i = 0; i < 20; ++i) attn_prefill(kBF16, a, st);
            cudaEventRecord(e2, st);
            cudaEventSynchronize(e2);
            float ms;
            cudaEventElapsedTime(&ms, e0, e2);
            (mode ? us_mma : us_tc) = ms * 1e3f / 20;
        }
        unsetenv("FSVD_ATTN_MMA");
    }
    const bool ok = e1 == cudaSuccess && nan_tc == 0 && err_tc <= 2e-2 * std::max(1.0, mx);
    std::printf("%s B=%d H=%d DH=%d T=%d p0=%d: max|err| tcgen05 %.3e  mma.sync %.3e  (max|o| %.3f, NaN %d) %s",
                ok ? "ok  " : "FAIL", B, H, DH, T, p0, err_tc, err_mma, mx, nan_tc, cudaGetErrorString(e1));
    if (timing) std::printf("  | %.2f us vs %.2f us", us_tc, us_mma);
    std::printf("\n");
    cudaFree(dq);
    cudaFree(dk);
    cudaFree(dv);
    cudaFree(dout);
    cudaStreamDestroy(st);
    return ok ? 0 : 1;
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    int bad = 0;
    bad += run(1, 2, 128, 9, 0, 64, false);
    bad += run(1, 2, 128, 128, 0, 256, false);
    bad += run(1, 2, 128, 200, 37, 512, false);
    bad += run(2, 3, 64, 150, 0, 256, false);
    bad += run(2, 2, 64, 33, 300, 512, false);
    bad += run(1, 4, 128, 512, 700, 1536, false);
    bad += run(1, 32, 128, 512, 0, 1024, true);
    bad += run(1, 32, 64, 512, 0, 1024, true);
    bad += run(4, 40, 128, 1024, 1024, 4096, true);
    std::printf(bad ? "FAILURES %d\n" : "all ok\n", bad);
    return bad;
}
