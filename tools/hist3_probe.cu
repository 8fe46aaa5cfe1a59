// Tooling (not product): can one sweep over 400M keys build the digit
// histograms of all three 9-bit LSD passes (3 shared atomics per key) at the
// speed of the single-digit count sweep (1 atomic per key)?  Usage: hist3_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int ND>
__global__ void __launch_bounds__(512, 2) k_hist(const uint64_t* __restrict__ in, int64_t n, uint32_t* __restrict__ out) {
    __shared__ uint32_t h[ND][512];
    for (int i = threadIdx.x; i < ND * 512; i += blockDim.x) (&h[0][0])[i] = 0;
    __syncthreads();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 2;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2; i < n; i += stride * 4) {
        ulonglong2 q[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) q[u] = (i + u * stride + 1 < n) ? __ldcs(reinterpret_cast<const ulonglong2*>(in + i + u * stride)) : make_ulonglong2(0, 0);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int d = 0; d < ND; ++d) {
                atomicAdd(&h[d][(q[u].x >> (37 + 9 * d)) & 511], 1u);
                atomicAdd(&h[d][(q[u].y >> (37 + 9 * d)) & 511], 1u);
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < ND * 512; i += blockDim.x) atomicAdd(&out[i], (&h[0][0])[i]);
}

__global__ void k_fill(uint64_t* d, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t z = i * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        d[i] = z ^ (z >> 31);
    }
}

int main() {
    const int64_t n = 400000000;
    uint64_t* d;
    uint32_t* o;
    cudaMalloc(&d, n * 8);
    cudaMalloc(&o, 3 * 512 * 4);
    k_fill<<<4096, 256>>>(d, n);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep) {
        float t1, t3;
        cudaEventRecord(a);
        k_hist<1><<<sms * 2, 512>>>(d, n, o);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&t1, a, b);
        cudaEventRecord(a);
        k_hist<3><<<sms * 2, 512>>>(d, n, o);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&t3, a, b);
        printf("400M keys: 1 digit %.3f ms (%.0f GB/s), 3 digits %.3f ms (%.0f GB/s)\n", t1, n * 8 / t1 / 1e6, t3,
               n * 8 / t3 / 1e6);
    }
    // random data
    return 0;
}
