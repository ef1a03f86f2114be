// Prefill GEMM dispatch: the tcgen05/TMEM tensor-core kernel (gemm_tc.cu)
// for the bf16 mode; the fp32 parity mode (f32 accumulates in
// f32 from f32 operands) runs on the CUDA cores (gemm_simt.cu).
#include <cstdlib>

#include "kernels.h"

namespace fsvd::k {

void gemm(WType wt, const GemmArgs& a, cudaStream_t s) {
    static const bool force_simt = [] {
        const char* e = std::getenv("FSVD_PREFILL_SIMT");
        return e && e[0] == '1';
    }();
    if (wt == kBF16 && !force_simt && gemm_tc_supported(a))
        gemm_tc(a, a.M, s);
    else
        gemm_simt(wt, a, s);
}

}  // namespace fsvd::k
