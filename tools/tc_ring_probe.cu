// Development probe (not product code): throughput of the decode megakernel's
// weight ring -- one producer warp streaming 16 KiB chunks with cp.async.bulk
// into an S-slot shared-memory ring, one consumer -- for three consumers:
//   mode 0: no compute (the consumer thread frees each slot on arrival)
//   mode 1: tcgen05.mma M=128 N=16 K=16 x4 per chunk + tcgen05.commit (one chain)
//   mode 2: as 1 with 8 accumulator chains
//   mode 3: as 1, but the slot is freed by a plain mbarrier arrive after the commit wait
// One CTA per SM, each streams its own contiguous range. Prints GB/s per mode.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tc_ring_probe.cu -o /tmp/trp && /tmp/trp
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

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
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
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
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void pf_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(
            tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
    d |= static_cast<uint64_t>(1) << 16;
    d |= static_cast<uint64_t>(1024 >> 4) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}

constexpr int kChunk = 16384;

template <int S>
__global__ void __launch_bounds__(64, 1) probe(const char* w, size_t per_cta, int mode, unsigned long long* cyc,
                                                int l2res) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    char* ring = reinterpret_cast<char*>(base);
    char* xs = ring + S * kChunk;  // 2 KiB B operand
    uint64_t* full = reinterpret_cast<uint64_t*>(xs + 2048);
    uint64_t* empty = full + S;
    uint64_t* done = empty + S;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = threadIdx.x; i < (S * kChunk + 2048) / 16; i += 64)
        reinterpret_cast<uint4*>(ring)[i] = make_uint4(0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tslot;
    const char* src = w + per_cta * blockIdx.x;
    const int n = static_cast<int>(per_cta / kChunk);
    unsigned long long t0 = clock64();
    if (warp == 0) {
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        const int pfd = mode >= 4 ? (mode == 4 ? 8 : 0) : 0;  // mode 4: L2 prefetch 8 ahead + evict_first; 5: hint only
        if (lane == 0)
            for (int i = 0; i < n; ++i) {
                const int s = i % S;
                if (pfd && i + pfd < n) pf_l2(src + static_cast<size_t>(i + pfd) * kChunk, kChunk);
                mbar_wait(&empty[s], ((i / S) & 1) ^ 1);
                mbar_expect_tx(&full[s], kChunk);
                const size_t off = l2res ? static_cast<size_t>(i % 16) * kChunk : static_cast<size_t>(i) * kChunk;
                if (mode >= 4)
                    bulk_g2s_hint(ring + s * kChunk, src + off, kChunk, &full[s], pol);
                else
                    bulk_g2s(ring + s * kChunk, src + off, kChunk, &full[s]);
            }
    } else {
        if (lane == 0) {
            const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (2u << 17) | (8u << 24);  // M128 N16
            const uint32_t xsa = smem_u32(xs);
            for (int i = 0; i < n; ++i) {
                const int s = i % S;
                mbar_wait(&full[s], (i / S) & 1);
                if (mode == 0) {
                    mbar_arrive(&empty[s]);
                    continue;
                }
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint64_t da = sw128_desc(smem_u32(ring + s * kChunk)), db = sw128_desc(xsa);
                const uint32_t td = mode == 2 ? tmem + (i & 1) * 64 : tmem;
                for (int kk = 0; kk < 4; ++kk)
                    tc_mma(mode == 2 ? td + kk * 16 : td, da + 2 * kk, db + 2 * kk, idesc, (i > 1 || kk > 0) ? 1u : 0u);
                if (mode == 3) {
                    tc_commit(done);
                    mbar_wait(done, i & 1);
                    mbar_arrive(&empty[s]);
                } else {
                    tc_commit(&empty[s]);
                }
            }
            tc_commit(done);
            if (mode != 3) mbar_wait(done, 0);
            else mbar_wait(done, n & 1);
        }
    }
    __syncwarp();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

int main() {
    const int G = 148;
    const size_t per_cta = 16ull << 20;  // 16 MiB per CTA: 2.4 GB total
    char* w;
    CK(cudaMalloc(&w, per_cta * G));
    CK(cudaMemset(w, 0x3c, per_cta * G));  // bf16 0x3c3c ~ 0.0115: finite, nonzero
    unsigned long long* cyc;
    CK(cudaMalloc(&cyc, 8 * G));
    constexpr int S = 10;
    const int smem = 1024 + S * kChunk + 2048 + 1024;
    CK(cudaFuncSetAttribute(probe<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int l2res = 0; l2res < 2; ++l2res)
    for (int mode = 0; mode < 6; ++mode) {
        if (l2res) printf("(L2-resident source) ");
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            probe<S><<<G, 64, smem>>>(w, per_cta, mode, cyc, l2res);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep == 2)
                printf("mode %d: %.3f ms  %.1f GB/s  (%.1f GB/s per SM, %.3f us per chunk)\n", mode, ms,
                       per_cta * G / ms / 1e6, per_cta / ms / 1e6, ms * 1e3 / (per_cta / kChunk));
        }
    }
    CK(cudaGetLastError());
    return 0;
}
