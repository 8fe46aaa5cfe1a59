// Yardstick only (not product code): time CUB DeviceRadixSort::SortPairs on
// n u64 (key, payload) pairs over `bits` key bits, to calibrate what a
// onesweep LSD sort reaches on this B200.  Usage: cub_yardstick n bits
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdlib>
#include <cstdint>

__global__ void fill(uint64_t* k, uint64_t* p, size_t n, uint64_t mask) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint64_t x = i * 0x9E3779B97F4A7C15ull;
        x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 29;
        k[i] = x & mask; p[i] = i;
    }
}

int main(int argc, char** argv) {
    size_t n = argc > 1 ? strtoull(argv[1], 0, 10) : 400000000ull;
    int bits = argc > 2 ? atoi(argv[2]) : 27;
    uint64_t *k0, *k1, *p0, *p1;
    cudaMalloc(&k0, n * 8); cudaMalloc(&k1, n * 8); cudaMalloc(&p0, n * 8); cudaMalloc(&p1, n * 8);
    fill<<<4096, 256>>>(k0, p0, n, (bits == 64) ? ~0ull : ((1ull << bits) - 1));
    cub::DoubleBuffer<uint64_t> dk(k0, k1), dp(p0, p1);
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, dk, dp, n, 0, bits);
    void* t; cudaMalloc(&t, tmp);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int it = 0; it < 4; ++it) {
        fill<<<4096, 256>>>(dk.Current(), dp.Current(), n, (bits == 64) ? ~0ull : ((1ull << bits) - 1));
        cudaEventRecord(a);
        cub::DeviceRadixSort::SortPairs(t, tmp, dk, dp, n, 0, bits);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("cub SortPairs n=%zu bits=%d: %.3f ms  (%.1f Gpairs/s)\n", n, bits, ms, n / ms / 1e6);
    }
    // keys only: 8-B records, the layout of our record passes
    {
        cub::DoubleBuffer<uint64_t> kk(k0, k1);
        size_t t2 = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, t2, kk, n, 0, bits);
        void* tt; cudaMalloc(&tt, t2);
        for (int it = 0; it < 4; ++it) {
            fill<<<4096, 256>>>(kk.Current(), p0, n, (bits == 64) ? ~0ull : ((1ull << bits) - 1));
            cudaEventRecord(a);
            cub::DeviceRadixSort::SortKeys(tt, t2, kk, n, 0, bits);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            printf("cub SortKeys u64 n=%zu bits=%d: %.3f ms  (%.1f Gkeys/s)\n", n, bits, ms, n / ms / 1e6);
        }
    }
    return 0;
}
