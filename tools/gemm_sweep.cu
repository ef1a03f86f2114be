// Development tool (not product): tile-shape sweep of the prefill GEMMs of one
// C2 layer (LLaMA-7B shape, rho 0.6, 512 tokens) through gemm_tc with forced
// FSVD_GEMM_{BN,BMT,SPLITS}; weights rotate over 6 copies (> L2) so they
// stream from HBM like in a real prefill.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../paper_2605_08314_b200/csrc/cuda/kernels.h"

using namespace fsvd::k;

struct Shape {
    const char* name;
    std::vector<int> rows;  // per segment
    int k;
    int epi;
};

int main(int argc, char** argv) {
    const int M = argc > 1 ? atoi(argv[1]) : 512;
    const int max_sp = argc > 2 ? atoi(argv[2]) : 4;
    const int NC = 6;
    std::vector<Shape> shapes = {
        {"qkvA", {1229, 1229, 1229}, 4096, kGemmStore}, {"qkvB", {4096, 4096, 4096}, 1229, kGemmStore},
        {"oA", {1229}, 4096, kGemmStore},               {"oB", {4096}, 1229, kGemmAddF32},
        {"ugA", {1791, 1791}, 4096, kGemmStore},        {"ugB", {11008, 11008}, 1791, kGemmSilu},
        {"dA", {1791}, 11008, kGemmStore},              {"dB", {4096}, 1791, kGemmAddF32},
    };
    cudaStream_t st;
    cudaStreamCreate(&st);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (const Shape& sh : shapes) {
        const WLayout lay = make_layout(sh.rows[0], sh.k, 2);
        const int x_ld = (sh.k + 63) / 64 * 64;
        const int nseg = static_cast<int>(sh.rows.size());
        int ytot = 0;
        for (int r : sh.rows) ytot += (sh.epi == kGemmSilu ? 0 : (r + 7) / 8 * 8);
        if (sh.epi == kGemmSilu) ytot = sh.rows[0];
        const int y_ld = (ytot + 7) / 8 * 8;
        void* x;
        cudaMalloc(&x, size_t(M) * x_ld * 2);
        cudaMemset(x, 0x3c, size_t(M) * x_ld * 2);
        std::vector<void*> w(NC * nseg);
        for (auto& p : w) {
            cudaMalloc(&p, lay.bytes());
            cudaMemset(p, 0x3c, lay.bytes());
        }
        void* y;
        cudaMalloc(&y, size_t(M) * y_ld * 4);
        cudaMemset(y, 0, size_t(M) * y_ld * 4);
        const size_t wsf = static_cast<size_t>(std::max(4, max_sp)) * M * y_ld;
        float* ws;
        cudaMalloc(&ws, wsf * 4);
        auto args = [&](int c) {
            GemmArgs a{};
            a.x = x;
            a.x_ld = x_ld;
            a.M = M;
            int off = 0;
            for (int s = 0; s < nseg; ++s) {
                a.seg[s] = GemvSeg{w[c * nseg + s], sh.rows[s], sh.k, lay.kp, 0, sh.epi == kGemmSilu ? 0 : off, kEpiStore};
                off += (sh.rows[s] + 7) / 8 * 8;
            }
            a.nseg = nseg;
            a.epi = sh.epi;
            a.y = y;
            a.y_ld = y_ld;
            a.ws = ws;
            a.ws_floats = wsf;
            return a;
        };
        struct Cf { int bn, bmt, sp; };
        std::vector<Cf> cfs;
        const int spmax = (sh.epi == kGemmStore || sh.epi == kGemmAddF32) ? max_sp : 1;
        for (int bn : {64, 96, 128, 160, 192, 224, 256})
            for (int sp = 1; sp <= spmax; sp += (sp < 4 ? 1 : 2)) cfs.push_back({bn, 1, sp});
        if (sh.epi != kGemmSilu && M > 128)
            for (int sp = 1; sp <= spmax; ++sp) cfs.push_back({256, 2, sp});
        cfs.push_back({0, 0, 0});  // the library's own choice
        for (const Cf& cf : cfs) {
            if (cf.bn) {
                setenv("FSVD_GEMM_BN", std::to_string(cf.bn).c_str(), 1);
                setenv("FSVD_GEMM_BMT", std::to_string(cf.bmt).c_str(), 1);
                setenv("FSVD_GEMM_SPLITS", std::to_string(cf.sp).c_str(), 1);
            } else {
                unsetenv("FSVD_GEMM_BN");
                unsetenv("FSVD_GEMM_BMT");
                unsetenv("FSVD_GEMM_SPLITS");
            }
            for (int i = 0; i < 3; ++i) gemm_tc(args(i % NC), M, st);
            const int reps = 12;
            cudaEventRecord(e0, st);
            for (int i = 0; i < reps; ++i) gemm_tc(args(i % NC), M, st);
            cudaEventRecord(e1, st);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            cudaError_t err = cudaGetLastError();
            printf("%-5s M=%d BN=%3d BMT=%d sp=%d : %7.2f us %s %s\n", sh.name, M, cf.bn, cf.bmt, cf.sp, ms * 1e3 / reps,
                   cf.bn ? "" : "<- auto", err == cudaSuccess ? "" : cudaGetErrorString(err));
        }
        cudaFree(x);
        cudaFree(y);
        cudaFree(ws);
        for (auto p : w) cudaFree(p);
    }
    return 0;
}
