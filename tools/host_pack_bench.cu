// Tooling (not product): can the host pack (key, payload) u64 SoA into 8-B
// records fast enough to halve the PCIe bytes of the e2e path?
// Measures: plain pinned H2D of 16 B/tuple; threaded packing alone; packing
// pipelined with H2D of the packed chunks.
#include <cuda_runtime.h>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

static void pack(const uint64_t* k, const uint64_t* p, uint64_t* o, size_t a, size_t b, uint64_t lower, int pw) {
    for (size_t i = a; i < b; ++i) o[i] = ((k[i] - lower) << pw) | p[i];
}

int main(int argc, char** argv) {
    size_t n = argc > 1 ? strtoull(argv[1], 0, 10) : 500000000ull;
    int T = argc > 2 ? atoi(argv[2]) : 16;
    size_t chunk = argc > 3 ? strtoull(argv[3], 0, 10) : (8ull << 20);  // tuples per chunk
    uint64_t *k, *p, *o, *d;
    cudaHostAlloc(&k, n * 8, 0);
    cudaHostAlloc(&p, n * 8, 0);
    cudaHostAlloc(&o, n * 8, 0);
    cudaMalloc(&d, n * 16);
    for (size_t i = 0; i < n; ++i) { k[i] = 1 + (i * 2654435761ull) % 100000000ull; p[i] = i & 0xffffffffull; }
    cudaStream_t s;
    cudaStreamCreate(&s);
    // 1) plain H2D 16 B/tuple
    for (int it = 0; it < 2; ++it) {
        double t0 = now();
        cudaMemcpyAsync(d, k, n * 8, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(d + n, p, n * 8, cudaMemcpyHostToDevice, s);
        cudaStreamSynchronize(s);
        if (it) printf("H2D 16B/tuple: %.1f ms (%.1f GB/s)\n", (now() - t0) * 1e3, n * 16 / (now() - t0) / 1e9);
    }
    // 2) packing alone
    for (int it = 0; it < 2; ++it) {
        double t0 = now();
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t) th.emplace_back(pack, k, p, o, n * t / T, n * (t + 1) / T, 1ull, 37);
        for (auto& x : th) x.join();
        if (it) printf("pack %d threads: %.1f ms (%.1f GB/s input)\n", T, (now() - t0) * 1e3, n * 16 / (now() - t0) / 1e9);
    }
    // 3) packed H2D alone
    {
        double t0 = now();
        cudaMemcpyAsync(d, o, n * 8, cudaMemcpyHostToDevice, s);
        cudaStreamSynchronize(s);
        printf("H2D 8B/tuple: %.1f ms\n", (now() - t0) * 1e3);
    }
    // 4) pipelined: threads pack chunk c, then the chunk's H2D is queued
    for (int it = 0; it < 2; ++it) {
        double t0 = now();
        size_t nch = (n + chunk - 1) / chunk;
        std::vector<cudaEvent_t> ev(nch);
        for (size_t c = 0; c < nch; ++c) {
            size_t a = c * chunk, b = std::min(n, a + chunk);
            std::vector<std::thread> th;
            for (int t = 0; t < T; ++t) th.emplace_back(pack, k, p, o, a + (b - a) * t / T, a + (b - a) * (t + 1) / T, 1ull, 37);
            for (auto& x : th) x.join();
            cudaMemcpyAsync(d + a, o + a, (b - a) * 8, cudaMemcpyHostToDevice, s);
        }
        cudaStreamSynchronize(s);
        if (it) printf("pipelined pack+H2D (chunk %zu): %.1f ms\n", chunk, (now() - t0) * 1e3);
    }
    return 0;
}
