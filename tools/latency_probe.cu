// Development probe (not product): latency of dependent L2-hit loads while
// every SM has `inflight` bytes of cp.async.bulk weight copies outstanding.
// Answers: do activation loads queue behind the HBM weight stream?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/latency_probe.cu -o /tmp/lp && /tmp/lp
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void probe(const char* __restrict__ W, size_t wbytes, const unsigned* __restrict__ chase, int inflight,
                      int hops, unsigned long long* out, int chunk) {
    extern __shared__ __align__(128) char sm[];
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const size_t base = (static_cast<size_t>(blockIdx.x) * 8 * 1024 * 1024) % (wbytes - 16 * 1024 * 1024);
    if (tid == 0 && inflight > 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(inflight)
                     : "memory");
        for (int off = 0; off < inflight; off += chunk)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(sm + off)),
                "l"(W + base + off), "r"(chunk), "r"(smem_u32(&bar))
                : "memory");
    }
    if (tid == 32) {
        unsigned long long t0;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
        unsigned idx = blockIdx.x * 64;
        for (int h = 0; h < hops; ++h) idx = __ldcg(chase + idx);
        unsigned long long t1;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
        out[blockIdx.x * 2] = t1 - t0;
        out[blockIdx.x * 2 + 1] = idx;
    }
    if (tid == 0 && inflight > 0) {
        asm volatile(
            "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(
                smem_u32(&bar))
            : "memory");
    }
    __syncthreads();
}

int main() {
    const size_t wbytes = 2ull << 30;
    char* W;
    cudaMalloc(&W, wbytes);
    cudaMemset(W, 1, wbytes);
    const int n = 1 << 20;  // 4 MB chase table (L2 resident)
    std::vector<unsigned> h(n);
    for (int i = 0; i < n; ++i) h[i] = (i * 2654435761u + 12345u) % n;
    unsigned* chase;
    cudaMalloc(&chase, n * 4);
    cudaMemcpy(chase, h.data(), n * 4, cudaMemcpyHostToDevice);
    unsigned long long* out;
    cudaMalloc(&out, 148 * 2 * 8);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int hops = 50;
    for (int rep = 0; rep < 2; ++rep)
        for (int chunk : {16384}) {
            for (int inflight : {0, 16384, 65536, 131072, 196608}) {
                // warm the chase table into L2
                probe<<<148, 64, 200 * 1024>>>(W, wbytes, chase, 0, hops, out, chunk);
                probe<<<148, 64, 200 * 1024>>>(W, wbytes, chase, inflight, hops, out, chunk);
                cudaDeviceSynchronize();
                std::vector<unsigned long long> o(148 * 2);
                cudaMemcpy(o.data(), out, o.size() * 8, cudaMemcpyDeviceToHost);
                double s = 0, mx = 0;
                for (int c = 0; c < 148; ++c) {
                    s += o[2 * c];
                    mx = o[2 * c] > mx ? o[2 * c] : mx;
                }
                if (rep)
                    printf("inflight %6d B/SM (%5.1f MB total): L2-hit dependent load %6.0f ns avg, %6.0f ns max/hop\n",
                           inflight, inflight * 148 / 1e6, s / 148 / hops, mx / hops);
            }
        }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
