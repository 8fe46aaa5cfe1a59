// Microbenchmark (tooling, not product): how fast does the memory system take
// the onesweep write pattern?  Each CTA reads a contiguous tile of `tile`
// u64 (coalesced) and writes it as nbins runs of tile/nbins elements to
// nbins far-apart regions (bucket d of tile t at d*(n/nbins) + t*run), the
// pattern a radix pass produces after smem staging.  Compares with a plain
// copy.  Usage: scatter_pattern_bench n tile nbins
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void copy_k(const uint64_t* __restrict__ in, uint64_t* __restrict__ out, size_t n) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (; i < n; i += (size_t)gridDim.x * blockDim.x) out[i] = in[i];
}

template <int THREADS>
__global__ void scatter_k(const uint64_t* __restrict__ in, uint64_t* __restrict__ out, size_t n, int tile,
                          int nbins) {
    const size_t t = blockIdx.x;
    const size_t base = t * tile;
    const int run = tile / nbins;
    const size_t region = n / nbins;
    for (int i = threadIdx.x; i < tile; i += THREADS) {
        const uint64_t v = in[base + i];
        const int d = i / run, r = i % run;
        out[(size_t)d * region + t * run + r] = v;
    }
}

// segmented: G persistent CTAs, CTA g owns tiles [g*T/G, (g+1)*T/G); bucket d
// of its k-th tile goes to d*region + g*(region/G) + k*run -- the pattern of
// segsort.cu (each CTA appends to nbins private streams)
template <int THREADS>
__global__ void seg_k(const uint64_t* __restrict__ in, uint64_t* __restrict__ out, size_t n, int tile, int nbins) {
    const size_t T = n / tile, G = gridDim.x;
    const size_t t0 = blockIdx.x * T / G, t1 = (blockIdx.x + 1) * T / G;
    const int run = tile / nbins;
    const size_t region = n / nbins;
    const size_t sub = region / G;
    for (size_t t = t0; t < t1; ++t) {
        for (int i = threadIdx.x; i < tile; i += THREADS) {
            const uint64_t v = in[t * tile + i];
            const int d = i / run, r = i % run;
            out[(size_t)d * region + blockIdx.x * sub + (t - t0) * run + r] = v;
        }
    }
}


// tile in smem, then run d of the tile leaves with ONE bulk (TMA) store per
// run, issued by thread d (runs of `run` 8-B elements, 16-B aligned here)
template <int THREADS>
__global__ void bulk_k(const uint64_t* __restrict__ in, uint64_t* __restrict__ out, size_t n, int tile, int nbins) {
    extern __shared__ __align__(16) uint64_t sm[];
    const size_t t = blockIdx.x;
    const size_t base = t * tile;
    const int run = tile / nbins;
    const size_t region = n / nbins;
    for (int i = threadIdx.x; i < tile; i += THREADS) sm[i] = in[base + i];
    __syncthreads();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int d = threadIdx.x; d < nbins; d += THREADS) {
        const unsigned s = (unsigned)__cvta_generic_to_shared(sm + (size_t)d * run);
        uint64_t* g = out + (size_t)d * region + t * run;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(s), "r"(run * 8)
                     : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}


// persistent: `per_sm` CTAs per SM loop over tiles in global order from a
// dispenser; each thread reads its elements of the tile and writes them to
// the runs (no staging) -- isolates persistence + dispensing from the rest
template <int THREADS>
__global__ void persist_k(const uint64_t* __restrict__ in, uint64_t* __restrict__ out, size_t n, int tile, int nbins,
                          unsigned int* ticket) {
    __shared__ unsigned int t_sh;
    const size_t T = n / tile;
    const int run = tile / nbins;
    const size_t region = n / nbins;
    for (;;) {
        if (threadIdx.x == 0) t_sh = atomicAdd(ticket, 1u);
        __syncthreads();
        const size_t t = t_sh;
        __syncthreads();
        if (t >= T) break;
        const size_t base = t * tile;
        for (int i = threadIdx.x; i < tile; i += THREADS) {
            const uint64_t v = in[base + i];
            const int d = i / run, r = i % run;
            out[(size_t)d * region + t * run + r] = v;
        }
    }
}

int main(int argc, char** argv) {
    size_t n = argc > 1 ? strtoull(argv[1], 0, 10) : 400000000ull;
    int tile = argc > 2 ? atoi(argv[2]) : 6144;
    int nbins = argc > 3 ? atoi(argv[3]) : 512;
    n = n / tile * tile;
    uint64_t *a, *b;
    cudaMalloc(&a, n * 8);
    cudaMalloc(&b, n * 8);
    cudaMemset(a, 1, n * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int it = 0; it < 3; ++it) {
        cudaEventRecord(e0);
        copy_k<<<148 * 8, 512>>>(a, b, n);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it == 2) printf("copy     : %.3f ms  %.0f GB/s\n", ms, 16.0 * n / ms / 1e6);
    }
    for (int it = 0; it < 3; ++it) {
        cudaEventRecord(e0);
        scatter_k<512><<<(unsigned)(n / tile), 512>>>(a, b, n, tile, nbins);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it == 2) printf("scatter  : tile %d bins %d run %d: %.3f ms  %.0f GB/s\n", tile, nbins, tile / nbins, ms,
                            16.0 * n / ms / 1e6);
    }
    cudaFuncSetAttribute(bulk_k<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, tile * 8);
    for (int it = 0; it < 3; ++it) {
        cudaEventRecord(e0);
        bulk_k<512><<<(unsigned)(n / tile), 512, tile * 8>>>(a, b, n, tile, nbins);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it == 2) printf("bulk     : tile %d bins %d run %d: %.3f ms  %.0f GB/s  (%s)\n", tile, nbins, tile / nbins, ms,
                            16.0 * n / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
    unsigned int* ticket;
    cudaMalloc(&ticket, 4);
    for (int per_sm : {1, 2, 4, 8}) {
        for (int it = 0; it < 3; ++it) {
            cudaMemset(ticket, 0, 4);
            cudaEventRecord(e0);
            persist_k<256><<<148 * per_sm, 256>>>(a, b, n, tile, nbins, ticket);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (it == 2) printf("persist256: %d CTA/SM tile %d bins %d: %.3f ms  %.0f GB/s\n", per_sm, tile, nbins, ms,
                                16.0 * n / ms / 1e6);
        }
    }
    for (int G : {148, 296, 592}) {
        for (int it = 0; it < 3; ++it) {
            cudaEventRecord(e0);
            seg_k<512><<<G, 512>>>(a, b, n, tile, nbins);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (it == 2) printf("segmented: G %d tile %d bins %d run %d: %.3f ms  %.0f GB/s\n", G, tile, nbins, tile / nbins, ms,
                                16.0 * n / ms / 1e6);
        }
    }
    return 0;
}
