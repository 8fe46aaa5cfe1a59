// abi.cu -- library-level entry points of the C ABI (include/mpsm_b200.h):
// version, error reporting, device selection, launch accounting, CUDA IPC.

#include <algorithm>
#include <cuda_runtime.h>

#include <atomic>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace mpsm {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

std::atomic<uint64_t>& launch_counter() {
    static std::atomic<uint64_t> c{0};
    return c;
}

struct ProfState {
    std::mutex mu;
    bool on = false;
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    std::map<std::string, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>> rec;
};

static ProfState& prof() {
    static ProfState p;
    return p;
}

bool profiling_enabled() { return prof().on; }

cudaEvent_t profile_event() {
    ProfState& p = prof();
    std::lock_guard<std::mutex> g(p.mu);
    if (p.used == p.pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        p.pool.push_back(e);
    }
    return p.pool[p.used++];
}

void profile_record(const char* name, cudaEvent_t a, cudaEvent_t b) {
    ProfState& p = prof();
    std::lock_guard<std::mutex> g(p.mu);
    p.rec[name].push_back({a, b});
}

}  // namespace mpsm

using namespace mpsm;

extern "C" int mpsm_profile_enable(int on) {
    ProfState& p = prof();
    std::lock_guard<std::mutex> g(p.mu);
    p.on = on != 0;
    p.used = 0;
    p.rec.clear();
    return MPSM_OK;
}

extern "C" int mpsm_profile_read(const char* name, double* total_ms, uint64_t* launches) {
    ProfState& p = prof();
    std::lock_guard<std::mutex> g(p.mu);
    double tot = 0;
    uint64_t cnt = 0;
    auto it = p.rec.find(name);
    if (it != p.rec.end()) {
        for (auto& ev : it->second) {
            MPSM_TRY(cuda_status(cudaEventSynchronize(ev.second), "cudaEventSynchronize"));
            float ms = 0;
            MPSM_TRY(cuda_status(cudaEventElapsedTime(&ms, ev.first, ev.second), "cudaEventElapsedTime"));
            tot += ms;
            ++cnt;
        }
    }
    *total_ms = tot;
    *launches = cnt;
    return MPSM_OK;
}

extern "C" int mpsm_version(void) { return 1; }

extern "C" const char* mpsm_last_error(void) { return g_last_error.c_str(); }

extern "C" uint64_t mpsm_launch_count(void) { return launch_counter().load(); }

namespace mpsm {
// a join's small results (pair records, flags) straight into pinned host
// memory: a kernel right behind the join's last kernel, where a device ->
// host copy starts ~12-14 us after it (copy-engine hand-off)
__global__ void __launch_bounds__(256) k_fetch(uint64_t* __restrict__ dst, const uint64_t* __restrict__ a, int64_t na,
                                               const uint64_t* __restrict__ b, int64_t nb) {
    const int64_t step = (int64_t)gridDim.x * blockDim.x, t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t i = t; i < na; i += step) dst[i] = a[i];
    for (int64_t i = t; i < nb; i += step) dst[na + i] = b[i];
}
}  // namespace mpsm

extern "C" int mpsm_fetch_small(void* host_dst, const void* src_a, int64_t words_a, const void* src_b, int64_t words_b,
                                void* stream) {
    if (!host_dst || words_a < 0 || words_b < 0 || (words_a && !src_a) || (words_b && !src_b)) {
        set_error("mpsm_fetch_small: null pointer or negative size");
        return MPSM_ERR_ARG;
    }
    // pinned host memory is device-accessible at its host address (unified
    // addressing); anything else is refused rather than faulting
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, host_dst) != cudaSuccess || at.type != cudaMemoryTypeHost ||
        at.devicePointer == nullptr) {
        cudaGetLastError();
        set_error("mpsm_fetch_small: destination is not pinned host memory");
        return MPSM_ERR_ARG;
    }
    if (words_a + words_b == 0) return MPSM_OK;
    const int grid = (int)std::min<int64_t>(1024, (words_a + words_b + 255) / 256);
    k_fetch<<<grid, 256, 0, (cudaStream_t)stream>>>((uint64_t*)at.devicePointer, (const uint64_t*)src_a, words_a,
                                                (const uint64_t*)src_b, words_b);
    return check_launch("k_fetch");
}

extern "C" int mpsm_device_init(int device) {
    MPSM_TRY(cuda_status(cudaSetDevice(device), "cudaSetDevice"));
    cudaDeviceProp prop;
    MPSM_TRY(cuda_status(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties"));
    if (prop.major != 10 || prop.minor != 0) {
        set_error(std::string("device is sm_") + std::to_string(prop.major) + std::to_string(prop.minor) +
                  "; this library is built for sm_100a (B200) only");
        return MPSM_ERR_CONFIG;
    }
    return prop.multiProcessorCount;
}

// base of the allocation holding d_ptr (the caching allocator sub-allocates:
// the IPC handle names the whole cudaMalloc block), through the driver's
// cuMemGetAddressRange fetched at run time (no link-time libcuda)
static int alloc_base(const void* d_ptr, uintptr_t* base) {
    typedef int (*range_fn)(unsigned long long*, size_t*, unsigned long long);
    static range_fn fn = nullptr;
    if (!fn) {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        MPSM_TRY(cuda_status(cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q),
                             "cudaGetDriverEntryPoint"));
        if (!f || q != cudaDriverEntryPointSuccess) {
            set_error("cuMemGetAddressRange unavailable");
            return MPSM_ERR_CUDA;
        }
        fn = (range_fn)f;
    }
    unsigned long long b = 0;
    size_t size = 0;
    if (fn(&b, &size, (unsigned long long)(uintptr_t)d_ptr) != 0) {
        set_error("cuMemGetAddressRange failed");
        return MPSM_ERR_CUDA;
    }
    *base = (uintptr_t)b;
    return MPSM_OK;
}

extern "C" int mpsm_ipc_get_handle(const void* d_ptr, void* handle64, int64_t* offset) {
    if (!d_ptr || !handle64 || !offset) return MPSM_ERR_ARG;
    uintptr_t base = 0;
    MPSM_TRY(alloc_base(d_ptr, &base));
    cudaIpcMemHandle_t h;
    MPSM_TRY(cuda_status(cudaIpcGetMemHandle(&h, (void*)base), "cudaIpcGetMemHandle"));
    static_assert(sizeof(h) == 64, "IPC handle size");
    std::memcpy(handle64, &h, 64);
    *offset = (int64_t)((uintptr_t)d_ptr - base);
    return MPSM_OK;
}

// maps the block into the CURRENT device's context with lazy peer access, so
// this rank's kernels read it over NVLink
extern "C" int mpsm_ipc_open_handle(const void* handle64, void** d_ptr) {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, 64);
    return cuda_status(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
}

extern "C" int mpsm_ipc_close_handle(void* d_ptr) {
    return cuda_status(cudaIpcCloseMemHandle(d_ptr), "cudaIpcCloseMemHandle");
}
