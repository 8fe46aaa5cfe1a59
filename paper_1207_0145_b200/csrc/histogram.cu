// histogram.cu -- private-input radix histogram with fused domain check.
//
// Replaces _kernels.radix_histogram (/root/reference/pkg/src/mpsm/_kernels.py
// 247-259) behind partition.build_radix_histogram (partition.py:110-122):
// counts[(key - lower) >> shift] += 1 over 2^B buckets.  One read of 8 B per
// key.  Out-of-domain keys are reported through *d_bad and counted in the
// clamped bucket (the same clamp the partition scatter applies), so a scatter
// built on these counts never leaves its regions even for bad input.

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"

namespace mpsm {

constexpr int HIST_SMEM_MAX_BUCKETS = 1 << 14;

__global__ void __launch_bounds__(512) k_radix_hist_smem(const uint64_t* __restrict__ keys, int64_t n, uint64_t lower,
                                                         uint64_t span_m1, int shift, int nbuckets,
                                                         unsigned long long* __restrict__ counts,
                                                         unsigned long long* __restrict__ d_bad) {
    extern __shared__ uint32_t sh[];
    for (int i = threadIdx.x; i < nbuckets; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        uint64_t nk = ld_stream(keys + i) - lower;
        if (nk > span_m1 && d_bad) atomicMin(d_bad, (unsigned long long)i);
        uint64_t b = nk >> shift;
        if (b >= (uint64_t)nbuckets) b = nbuckets - 1;
        atomicAdd(&sh[b], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nbuckets; i += blockDim.x)
        if (sh[i]) atomicAdd(&counts[i], (unsigned long long)sh[i]);
}

__global__ void __launch_bounds__(512) k_radix_hist_global(const uint64_t* __restrict__ keys, int64_t n, uint64_t lower,
                                                           uint64_t span_m1, int shift, int64_t nbuckets,
                                                           unsigned long long* __restrict__ counts,
                                                           unsigned long long* __restrict__ d_bad) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        uint64_t nk = ld_stream(keys + i) - lower;
        if (nk > span_m1 && d_bad) atomicMin(d_bad, (unsigned long long)i);
        uint64_t b = nk >> shift;
        if (b >= (uint64_t)nbuckets) b = nbuckets - 1;
        atomicAdd(&counts[b], 1ull);
    }
}

}  // namespace mpsm

using namespace mpsm;

extern "C" int mpsm_radix_histogram(const uint64_t* keys, int64_t n, uint64_t lower, uint64_t span_m1, int shift,
                                    int nbuckets, int64_t* d_counts, unsigned long long* d_bad, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n < 0 || nbuckets < 1 || shift < 0 || shift > 63) return MPSM_ERR_ARG;
    if (n == 0) return MPSM_OK;
    int grid = (int)std::min<int64_t>(num_sms() * 4, (n + 511) / 512);
    ProfScope ps("radix_histogram", st);
    if (nbuckets <= HIST_SMEM_MAX_BUCKETS) {
        size_t smem = sizeof(uint32_t) * nbuckets;
        if (smem > 48 * 1024)
            MPSM_TRY(cuda_status(cudaFuncSetAttribute(k_radix_hist_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                      (int)smem),
                                 "smem attr"));
        k_radix_hist_smem<<<grid, 512, smem, st>>>(keys, n, lower, span_m1, shift, nbuckets,
                                                   (unsigned long long*)d_counts, d_bad);
    } else {
        k_radix_hist_global<<<grid, 512, 0, st>>>(keys, n, lower, span_m1, shift, nbuckets,
                                                  (unsigned long long*)d_counts, d_bad);
    }
    return check_launch("k_radix_hist");
}
