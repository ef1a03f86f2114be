// Shared device helpers for the sm_100a kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

namespace fsvd::dev {

constexpr int kWarp = 32;

// ---- programmatic dependent launch (PDL) ----
// launch_dependents: let the next kernel in the stream start its prologue
// (weight prefetch) now. wait: block until the previous grid has completed
// and its memory is visible. Both are no-ops when the kernel was launched
// without the PDL attribute.
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Host: launch `k` with the PDL attribute (it must pdl_wait() before touching
// anything the previous kernel writes).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// Bulk L2 prefetch of a contiguous byte range (no smem, no registers):
// cp.async.bulk.prefetch.L2 -- size multiple of 16, address 16-aligned.
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// Issue L2 prefetches for [p, p + bytes) in <= 64 KiB pieces, spread over the
// calling threads (tid in [0, nthreads)).
__device__ __forceinline__ void prefetch_l2_range(const void* p, size_t bytes, int tid, int nthreads) {
    const uintptr_t lo = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
    const uintptr_t hi = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
    constexpr uintptr_t kPiece = 64 * 1024;
    for (uintptr_t a = lo + uintptr_t(tid) * kPiece; a < hi; a += uintptr_t(nthreads) * kPiece) {
        const uintptr_t n = hi - a < kPiece ? hi - a : kPiece;
        prefetch_l2_bulk(reinterpret_cast<const void*>(a), static_cast<uint32_t>(n));
    }
}

// ---- streaming 128-bit loads (weights are read once per step) ----
__device__ __forceinline__ uint4 ld_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ float bf16lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }

template <typename T>
__device__ __forceinline__ float to_f32(T v);
template <>
__device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T>
__device__ __forceinline__ T from_f32(float v);
template <>
__device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// silu(g) * u with IEEE exp (the reference uses std::exp, kernels_scalar.cpp:63-69)
__device__ __forceinline__ float silu_mul(float g, float u) { return g / (1.0f + expf(-g)) * u; }

}  // namespace fsvd::dev
