// Tooling probe: are shared-memory atomicAdd return values of lanes that hit
// the same address within ONE warp instruction handed out in lane order?
#include <cstdio>
#include <cstdint>
__global__ void k(const uint32_t* digits, int iters, int* bad, int nb) {
    __shared__ uint32_t h[16][512];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 16 * 512; i += blockDim.x) (&h[0][0])[i] = 0;
    __syncthreads();
    for (int it = 0; it < iters; ++it) {
        const uint32_t d = digits[(blockIdx.x * iters + it) * blockDim.x + threadIdx.x] % nb;
        const uint32_t old = atomicAdd(&h[w][d], 1u);
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const uint32_t lt = peers & ((1u << lane) - 1);
        // expected: old == base + popc(lt), base = old of the lowest peer
        const int leader = __ffs(peers) - 1;
        const uint32_t base = __shfl_sync(0xffffffffu, old, leader);
        if (old != base + __popc(lt)) atomicAdd(bad, 1);
    }
}
int main() {
    const int blocks = 296, threads = 512, iters = 64;
    size_t n = (size_t)blocks * threads * iters;
    uint32_t* d; int* bad;
    cudaMalloc(&d, n * 4); cudaMalloc(&bad, 4);
    uint32_t* h = new uint32_t[n];
    uint64_t x = 88172645463325252ull;
    for (size_t i = 0; i < n; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h[i] = (uint32_t)x; }
    cudaMemcpy(d, h, n * 4, cudaMemcpyHostToDevice);
    for (int nb : {2, 8, 64, 512}) {
        cudaMemset(bad, 0, 4);
        k<<<blocks, threads>>>(d, iters, bad, nb);
        int hb; cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
        printf("bins %3d: lanes out of order = %d of %zu\n", nb, hb, n);
    }
    return 0;
}
