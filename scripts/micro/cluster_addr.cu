// Prints the shared-window address of one smem variable per CTA of a 4-CTA cluster,
// and its mapa.shared::cluster translation to every rank.
#include <cstdio>
#include <cstdint>
__global__ void __cluster_dims__(4, 1, 1) k(unsigned* out) {
    __shared__ unsigned x;
    unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(&x));
    unsigned rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    if (threadIdx.x == 0) {
        out[blockIdx.x * 8 + 0] = rank;
        out[blockIdx.x * 8 + 1] = a;
        for (int r = 0; r < 4; ++r) {
            unsigned m;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(m) : "r"(a), "r"(r));
            out[blockIdx.x * 8 + 2 + r] = m;
        }
    }
}
int main() {
    unsigned* d; cudaMalloc(&d, 8 * 8 * 4);
    k<<<8, 32>>>(d);
    unsigned h[64]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    for (int b = 0; b < 8; ++b)
        printf("block %d rank %u local 0x%08x mapa->0:0x%08x 1:0x%08x 2:0x%08x 3:0x%08x\n", b, h[b*8], h[b*8+1], h[b*8+2], h[b*8+3], h[b*8+4], h[b*8+5]);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
