// place_probe.cu -- microbenchmark for a direct-placement pass: records that
// are already grouped by the top bits of their key (2^18-key buckets, random
// order inside a bucket) are stored at out[key - min].  Measures how fast
// uncoalesced 8-B stores inside a moving L2-resident window go, with and
// without a shared-memory bitmap of the bucket (exact duplicate detection).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o place_probe place_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>

__global__ void k_place(const uint64_t* __restrict__ in, int64_t n, int pw, uint64_t* __restrict__ out) {
    // grid-stride in chunks so the CTAs sweep the input in order together
    const int64_t CH = 4096;
    for (int64_t c = (int64_t)blockIdx.x * CH; c < n; c += (int64_t)gridDim.x * CH) {
        const int64_t e = min(c + CH, n);
        for (int64_t i = c + threadIdx.x * 2; i + 1 < e; i += 2 * blockDim.x) {
            const ulonglong2 v = __ldcs(reinterpret_cast<const ulonglong2*>(in + i));
            out[v.x >> pw] = v.x;
            out[v.y >> pw] = v.y;
        }
    }
}

// one bucket per CTA-range: cluster-free, bitmap in smem
template <int SB>
__global__ void k_place_bm(const uint64_t* __restrict__ in, int64_t n, int pw, uint64_t* __restrict__ out,
                           int per_bucket_ctas, unsigned long long* pop) {
    extern __shared__ uint32_t bm[];
    const int words = (1 << SB) / 32;
    for (int i = threadIdx.x; i < words; i += blockDim.x) bm[i] = 0;
    __syncthreads();
    const int64_t bucket = blockIdx.x / per_bucket_ctas, part = blockIdx.x % per_bucket_ctas;
    const int64_t b0 = bucket << SB, b1 = min(b0 + (1 << SB), n);
    if (b0 >= n) return;
    const int64_t len = b1 - b0, per = (len + per_bucket_ctas - 1) / per_bucket_ctas;
    const int64_t s = b0 + part * per, e = min(s + per, b1);
    for (int64_t i = s + threadIdx.x * 2; i + 1 < e; i += 2 * blockDim.x) {
        const ulonglong2 v = __ldcs(reinterpret_cast<const ulonglong2*>(in + i));
        const uint32_t k0 = (uint32_t)(v.x >> pw) - (uint32_t)b0, k1 = (uint32_t)(v.y >> pw) - (uint32_t)b0;
        atomicOr(&bm[k0 >> 5], 1u << (k0 & 31));
        atomicOr(&bm[k1 >> 5], 1u << (k1 & 31));
        out[v.x >> pw] = v.x;
        out[v.y >> pw] = v.y;
    }
    __syncthreads();
    uint32_t c = 0;
    for (int i = threadIdx.x; i < words; i += blockDim.x) c += __popc(bm[i]);
    atomicAdd(pop, (unsigned long long)c);
}

int main(int argc, char** argv) {
    const int64_t n = argc > 1 ? atoll(argv[1]) : 100000000;
    const int pw = 37, SB = 18;
    std::vector<uint64_t> h(n);
    std::mt19937_64 rng(1);
    for (int64_t b = 0; b < n; b += (1 << SB)) {
        const int64_t e = std::min<int64_t>(b + (1 << SB), n);
        for (int64_t i = b; i < e; ++i) h[i] = ((uint64_t)i << pw) | (rng() & 0xffffffffu);
        std::shuffle(h.begin() + b, h.begin() + e, rng);
    }
    uint64_t *din, *dout;
    unsigned long long* dpop;
    cudaMalloc(&din, n * 8);
    cudaMalloc(&dout, n * 8);
    cudaMalloc(&dpop, 8);
    cudaMemcpy(din, h.data(), n * 8, cudaMemcpyHostToDevice);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](auto f) {
        f();
        cudaDeviceSynchronize();
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a);
            f();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = std::min(best, ms);
        }
        return best;
    };
    for (int occ : {1, 2, 4, 8}) {
        for (int th : {256, 512, 1024}) {
            if (occ * th > 2048) continue;
            float ms = timeit([&] { k_place<<<sms * occ, th>>>(din, n, pw, dout); });
            printf("plain  occ %d threads %4d: %.3f ms  %.1f GB/s (16 B/rec)\n", occ, th, ms, n * 16.0 / ms / 1e6);
        }
    }
    cudaFuncSetAttribute(k_place_bm<18>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    for (int pb : {4, 8, 16, 32, 64}) {
        for (int th : {512, 1024}) {
            const int64_t nb = (n + (1 << SB) - 1) >> SB;
            cudaMemset(dpop, 0, 8);
            float ms = timeit([&] { k_place_bm<18><<<(int)(nb * pb), th, 32768>>>(din, n, pw, dout, pb, dpop); });
            unsigned long long pop;
            cudaMemcpy(&pop, dpop, 8, cudaMemcpyDeviceToHost);
            printf("bitmap per_bucket %2d threads %4d: %.3f ms  %.1f GB/s  pop/run %.3f\n", pb, th, ms, n * 16.0 / ms / 1e6,
                   (double)pop / 6 / n);
        }
    }
    // check
    std::vector<uint64_t> o(n);
    cudaMemcpy(o.data(), dout, n * 8, cudaMemcpyDeviceToHost);
    int64_t bad = 0;
    for (int64_t i = 0; i < n; ++i) bad += (int64_t)(o[i] >> pw) != i;
    printf("bad %lld\n", (long long)bad);
    // yardstick: plain copy
    float ms = timeit([&] { cudaMemcpyAsync(dout, din, n * 8, cudaMemcpyDeviceToDevice); });
    printf("copy: %.3f ms %.1f GB/s\n", ms, n * 16.0 / ms / 1e6);
    return 0;
}
