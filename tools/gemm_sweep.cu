// Development tool (not product): tile-shape sweep of the prefill GEMMs of one
// C2 layer (LLaMA-7B shape, rho 0.6, 512 tokens) through gemm_tc with forced
// FSVD_GEMM_{BN,BMT,SPLITS,CG}; weights rotate over 6 copies (> L2) so they
// stream from HBM like in a real prefill. Inputs are random; every config's
// output is compared with the library's own choice (max |diff|, and whether
// the fp32/bf16 results are bitwise equal).
//   gemm_sweep [M] [max_splits] [mode: all | pair]
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
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
    const std::string mode = argc > 3 ? argv[3] : "all";
    const std::string only = argc > 4 ? argv[4] : "";
    setvbuf(stdout, nullptr, _IONBF, 0);
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
        if (!only.empty() && only != sh.name) continue;
        const WLayout lay = make_layout(sh.rows[0], sh.k, 2);
        const int x_ld = (sh.k + 63) / 64 * 64;
        const int nseg = static_cast<int>(sh.rows.size());
        int ytot = 0;
        for (int r : sh.rows) ytot += (sh.epi == kGemmSilu ? 0 : (r + 7) / 8 * 8);
        if (sh.epi == kGemmSilu) ytot = sh.rows[0];
        const int y_ld = (ytot + 7) / 8 * 8;
        void* x;
        cudaMalloc(&x, size_t(M) * x_ld * 2);
        auto fill = [](void* d, size_t n_el, unsigned seed) {
            std::vector<__nv_bfloat16> h(n_el);
            unsigned v = seed * 2654435761u + 1;
            for (auto& e : h) {
                v = v * 1664525u + 1013904223u;
                e = __float2bfloat16((static_cast<int>(v >> 9) % 2001 - 1000) / 1000.f);
            }
            cudaMemcpy(d, h.data(), n_el * 2, cudaMemcpyHostToDevice);
        };
        fill(x, size_t(M) * x_ld, 7);
        std::vector<void*> w(NC * nseg);
        unsigned sd = 11;
        for (auto& p : w) {
            cudaMalloc(&p, lay.bytes());
            fill(p, lay.bytes() / 2, sd++);
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
        struct Cf { int bn, bmt, sp, cg, cr = 0; };
        std::vector<Cf> cfs;
        cfs.push_back({0, 0, 0, 1});  // the library's own choice (first: the comparison reference)
        const int spmax = (sh.epi == kGemmStore || sh.epi == kGemmAddF32) ? max_sp : 1;
        if (mode == "cred") {  // decode-sized M: DSMEM cluster reduction vs the reduce kernel, same splits
            cfs.clear();
            cfs.push_back({0, 0, 0, -1});  // reference: library choice, reduce-kernel path
            cfs.push_back({-1, 0, 0, 0});  // library choice, cluster path
            for (int sp : {2, 4, 8}) { cfs.push_back({-1, 0, sp, -1}); cfs.push_back({-1, 0, sp, 0}); }
        }
        if (mode == "cred512") {  // cluster split-K (DSMEM) vs the reduce kernel, CTA pairs and single CTAs
            cfs.clear();
            cfs.push_back({0, 0, 0, 1});
            for (int cg : {1, 2})
                for (int bn : {128, 192, 256})
                    for (int sp : {2, 3, 4}) {
                        if (cg * sp > 8 || bn % (32 * sp) || sh.epi == kGemmSilu) continue;
                        cfs.push_back({bn, 1, sp, cg, 0});
                        cfs.push_back({bn, 1, sp, cg, 1});
                    }
        }
        for (int cg = (mode == "pair" ? 2 : 1); mode != "cred" && mode != "cred512" && cg <= 2; ++cg) {
            for (int bn : {64, 96, 128, 160, 192, 224, 256}) {
                if (cg == 2 && bn < 128) continue;
                for (int sp = 1; sp <= spmax; sp += (sp < 4 ? 1 : 2)) cfs.push_back({bn, 1, sp, cg});
            }
            if (sh.epi != kGemmSilu && M > 128)
                for (int sp = 1; sp <= spmax; ++sp) cfs.push_back({256, 2, sp, cg});
        }
        const size_t ybytes = size_t(M) * y_ld * (sh.epi == kGemmAddF32 ? 4 : 2);
        std::vector<unsigned char> yref(ybytes), ygot(ybytes), yprev(ybytes);
        const Cf* prev = nullptr;
        for (const Cf& cf : cfs) {
            if (cf.cg == -1) setenv("FSVD_NO_CRED", "1", 1); else unsetenv("FSVD_NO_CRED");
            if (cf.cr) setenv("FSVD_GEMM_CRED", "1", 1); else unsetenv("FSVD_GEMM_CRED");
            if (cf.bn == -1 || (cf.bn == 0 && cf.cg == -1)) {
                unsetenv("FSVD_GEMM_BN");
                unsetenv("FSVD_GEMM_BMT");
                unsetenv("FSVD_GEMM_CG");
                if (cf.sp) setenv("FSVD_GEMM_SPLITS", std::to_string(cf.sp).c_str(), 1); else unsetenv("FSVD_GEMM_SPLITS");
            } else if (cf.bn) {
                setenv("FSVD_GEMM_BN", std::to_string(cf.bn).c_str(), 1);
                setenv("FSVD_GEMM_BMT", std::to_string(cf.bmt).c_str(), 1);
                setenv("FSVD_GEMM_SPLITS", std::to_string(cf.sp).c_str(), 1);
                setenv("FSVD_GEMM_CG", std::to_string(cf.cg).c_str(), 1);
            } else {
                unsetenv("FSVD_GEMM_BN");
                unsetenv("FSVD_GEMM_BMT");
                unsetenv("FSVD_GEMM_SPLITS");
                unsetenv("FSVD_GEMM_CG");
            }
            // correctness: one call on zeroed Y vs the library choice
            cudaMemset(y, 0, size_t(M) * y_ld * 4);
            gemm_tc(args(0), M, st);
            cudaStreamSynchronize(st);
            cudaMemcpy(cf.bn ? ygot.data() : yref.data(), y, ybytes, cudaMemcpyDeviceToHost);
            double maxd = 0, maxr = 0;
            bool same = true;
            if (cf.bn) {
                same = ygot == yref;
                const size_t n = ybytes / (sh.epi == kGemmAddF32 ? 4 : 2);
                for (size_t i = 0; i < n; ++i) {
                    float r, g;
                    if (sh.epi == kGemmAddF32) {
                        r = reinterpret_cast<float*>(yref.data())[i];
                        g = reinterpret_cast<float*>(ygot.data())[i];
                    } else {
                        r = __bfloat162float(reinterpret_cast<__nv_bfloat16*>(yref.data())[i]);
                        g = __bfloat162float(reinterpret_cast<__nv_bfloat16*>(ygot.data())[i]);
                    }
                    maxd = std::max(maxd, static_cast<double>(std::abs(r - g)));
                    maxr = std::max(maxr, static_cast<double>(std::abs(r)));
                }
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
            // cluster twin of the previous config (same tile / splits, in-kernel DSMEM reduction instead of the
            // reduction kernel): must be bitwise equal
            const bool twin = prev && cf.bn != 0 && cf.sp != 0 &&
                              ((mode == "cred" && prev->cg == -1 && cf.cg == 0 && prev->sp == cf.sp) ||
                               (mode == "cred512" && prev->cr == 0 && cf.cr == 1 && prev->bn == cf.bn &&
                                prev->sp == cf.sp && prev->cg == cf.cg));
            if (twin) printf("PAIRCHECK %-5s M=%d BN=%d sp=%d CG=%d cluster vs reduction kernel: %s\n", sh.name, M, cf.bn,
                             cf.sp, cf.cg, ygot == yprev ? "bitwise" : "DIFF");
            yprev = cf.bn ? ygot : yref;
            prev = &cf;
            const double fl = 2.0 * M * sh.k * (sh.epi == kGemmSilu ? 2.0 : 1.0) *
                              [&] { double n = 0; for (int r : sh.rows) n += r; return sh.epi == kGemmSilu ? n / 2 : n; }();
            printf("%-5s M=%d BN=%3d BMT=%d CG=%d sp=%d%s : %7.2f us %6.0f TF/s  %s maxdiff %.3g (max|y| %.3g) %s %s\n",
                   sh.name, M, cf.bn, cf.bmt, cf.cg, cf.sp, cf.cr ? " cluster" : "", ms * 1e3 / reps, fl / (ms * 1e-3 / reps) / 1e12,
                   cf.bn ? (same ? "bitwise" : "DIFF") : "<- auto", maxd, maxr, "", err == cudaSuccess ? "" : cudaGetErrorString(err));
        }
        cudaFree(x);
        cudaFree(y);
        cudaFree(ws);
        for (auto p : w) cudaFree(p);
    }
    return 0;
}
