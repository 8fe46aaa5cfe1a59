// relio.cu -- device side of the relation-file input path: split interleaved
// (key, payload) records (the MPSMREL1 body, bench.py:8-11) into the SoA
// columns the join reads.  Streaming, 32 B per tuple.

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"

namespace mpsm {

__global__ void __launch_bounds__(256) k_deinterleave(const ulonglong2* __restrict__ rec, int64_t n,
                                                      uint64_t* __restrict__ keys, uint64_t* __restrict__ pays) {
    constexpr int U = 4;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n; i += U * stride) {
        ulonglong2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcs(rec + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            __stcs((unsigned long long*)keys + i + u * stride, v[u].x);
            __stcs((unsigned long long*)pays + i + u * stride, v[u].y);
        }
    }
    for (; i < n; i += stride) {
        const ulonglong2 v = __ldcs(rec + i);
        keys[i] = v.x;
        pays[i] = v.y;
    }
}

}  // namespace mpsm

using namespace mpsm;

extern "C" int mpsm_deinterleave(const uint64_t* d_records, int64_t n, uint64_t* d_keys, uint64_t* d_pays,
                                 void* stream) {
    if (n < 0 || (n && (!d_records || !d_keys || !d_pays))) return MPSM_ERR_ARG;
    if (((uintptr_t)d_records & 15) != 0) {
        set_error("mpsm_deinterleave: records must be 16-B aligned");
        return MPSM_ERR_ARG;
    }
    if (n == 0) return MPSM_OK;
    const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8);
    {
        ProfScope ps("deinterleave", (cudaStream_t)stream);
        k_deinterleave<<<grid, 256, 0, (cudaStream_t)stream>>>((const ulonglong2*)d_records, n, d_keys, d_pays);
    }
    return check_launch("k_deinterleave");
}
