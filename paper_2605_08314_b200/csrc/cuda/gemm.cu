// Prefill GEMM dispatch: tcgen05 tensor-core kernel for bf16 (gemm_tc.cu),
// CUDA cores for the fp32 parity mode (gemm_simt.cu).
#include "kernels.h"

namespace fsvd::k {

void gemm(WType wt, const GemmArgs& a, cudaStream_t s) { gemm_simt(wt, a, s); }

}  // namespace fsvd::k
