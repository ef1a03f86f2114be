// Development probe (not product): shared-memory address forms inside a CTA pair
// (cvta shared::cta vs mapa shared::cluster) -- what the cta_group::2 TMA's
// mbarrier operand must look like.
#include <cstdio>
#include <cstdint>
__global__ void __cluster_dims__(2, 1, 1) probe() {
    __shared__ uint64_t bar[4];
    uint32_t r, a = static_cast<uint32_t>(__cvta_generic_to_shared(&bar[1])), m0, m1;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(m0) : "r"(a));
    asm volatile("mapa.shared::cluster.u32 %0, %1, 1;" : "=r"(m1) : "r"(a));
    if (threadIdx.x == 0) printf("block %d rank %u: cta addr %#x  mapa(0) %#x  mapa(1) %#x\n", blockIdx.x, r, a, m0, m1);
}
int main() {
    probe<<<4, 32>>>();
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
