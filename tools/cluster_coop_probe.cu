// Development probe (not product): can the decode megakernel's shape (1 CTA/SM,
// ~220 KiB dynamic shared memory, cooperative launch) run as clusters of 2/4/8?
// Prints cudaOccupancyMaxActiveClusters and tries the launch at a few grids.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* out) {
    extern __shared__ char sm[];
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    unsigned sid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sid));
    if (threadIdx.x == 0) { sm[0] = 1; out[blockIdx.x] = sid * 16 + r; }
}
int main() {
    int* d;
    cudaMalloc(&d, 4096);
    const int smem = 220 * 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {1, 2, 4, 8}) {
        cudaLaunchConfig_t cfg{};
        cfg.blockDim = dim3(288);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributeCooperative;
        at[1].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cfg.gridDim = dim3(cs);
        int ncl = -1;
        cudaError_t e0 = cudaOccupancyMaxActiveClusters(&ncl, k, &cfg);
        printf("cluster %d: max active clusters %d (%s) -> %d CTAs\n", cs, ncl, cudaGetErrorString(e0), ncl * cs);
        for (int grid : {148, 144, 140, 136, 128}) {
            if (grid % cs) continue;
            cfg.gridDim = dim3(grid);
            cfg.numAttrs = 2;
            cudaError_t e = cudaLaunchKernelEx(&cfg, k, d);
            cudaError_t e2 = cudaDeviceSynchronize();
            printf("   coop launch grid %d: %s / %s\n", grid, cudaGetErrorString(e), cudaGetErrorString(e2));
            cudaGetLastError();
        }
    }
}
