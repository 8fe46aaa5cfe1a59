// common.cuh -- shared helpers for the sm_100a MPSM kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstring>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <string>

#include "../../include/mpsm_b200.h"

namespace mpsm {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
std::atomic<uint64_t>& launch_counter();

inline int cuda_status(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return MPSM_OK;
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return MPSM_ERR_CUDA;
}

// call after every kernel launch
inline int check_launch(const char* name) {
    launch_counter().fetch_add(1, std::memory_order_relaxed);
    return cuda_status(cudaGetLastError(), name);
}

#define MPSM_TRY(expr)                 \
    do {                               \
        int _rc = (expr);              \
        if (_rc != MPSM_OK) return _rc; \
    } while (0)

// optional per-kernel CUDA-event timing (mpsm_profile_enable / _read)
bool profiling_enabled();
void profile_record(const char* name, cudaEvent_t start, cudaEvent_t stop);
cudaEvent_t profile_event();

struct ProfScope {
    const char* name;
    cudaStream_t st;
    cudaEvent_t a = nullptr, b = nullptr;
    ProfScope(const char* n, cudaStream_t s) : name(n), st(s) {
        if (profiling_enabled()) {
            a = profile_event();
            b = profile_event();
            cudaEventRecord(a, st);
        }
    }
    ~ProfScope() {
        if (a) {
            cudaEventRecord(b, st);
            profile_record(name, a, b);
        }
    }
};

inline int num_sms() {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// bump allocator over a caller-provided workspace
struct Carve {
    char* base;
    size_t cap;
    size_t off = 0;
    bool ok = true;
    template <class T>
    T* take(size_t count) {
        size_t bytes = align_up(count * sizeof(T));
        if (off + bytes > cap) {
            ok = false;
            return nullptr;
        }
        T* p = reinterpret_cast<T*>(base + off);
        off += bytes;
        return p;
    }
};

// ---------------------------------------------------------------- device
// device-side bounds checks of the hot kernels' shared- and global-memory
// indexing, compiled in only for the checked build (tools/checked_build.sh:
// -DMPSM_DEBUG_CHECKS=1); a violation prints the site and traps
#ifndef MPSM_DEBUG_CHECKS
#define MPSM_DEBUG_CHECKS 0
#endif
#if MPSM_DEBUG_CHECKS
#define MPSM_CHECK(cond)                                                                              \
    do {                                                                                              \
        if (!(cond)) {                                                                                \
            printf("MPSM_CHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__, __LINE__, \
                   (int)blockIdx.x, (int)threadIdx.x);                                                 \
            __trap();                                                                                 \
        }                                                                                             \
    } while (0)
#else
#define MPSM_CHECK(cond) \
    do {                 \
    } while (0)
#endif

__device__ __forceinline__ uint64_t rotl64(uint64_t x, unsigned r) { return (x << r) | (x >> (64 - r)); }

// splitmix64 finalizer
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t pair_hash(uint64_t r_pay, uint64_t s_pay) {
    return mix64(r_pay ^ rotl64(s_pay, 17));
}

__device__ __forceinline__ uint64_t ld_volatile_u64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_volatile_u64(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// streaming loads/stores that do not allocate in L1
__device__ __forceinline__ uint64_t ld_stream(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}

// ---- bulk async copies (TMA, 1-D) completing on a shared-memory mbarrier
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// named barrier id over nthreads threads (a multiple of 32)
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// MPSM_MBAR_SUSPEND_NS > 0: try_wait with a suspend-time hint -- a waiting
// warp sleeps until the phase completes (or the hint runs out) instead of
// spinning through issue slots its SM sub-partition's working warps need
#ifndef MPSM_MBAR_SUSPEND_NS
#define MPSM_MBAR_SUSPEND_NS 0
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    unsigned done;
    do {
        if (MPSM_MBAR_SUSPEND_NS > 0) {
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(done)
                : "r"(smem_addr(bar)), "r"(parity), "n"(MPSM_MBAR_SUSPEND_NS)
                : "memory");
        } else {
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(done)
                : "r"(smem_addr(bar)), "r"(parity)
                : "memory");
        }
    } while (!done);
}

// bytes (multiple of 16, 16-B aligned) of global memory into L2
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// generic-proxy writes to shared memory before an async-proxy write to it
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// bytes (multiple of 16; both addresses 16-B aligned) global -> shared
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    return v;
}

// ------------------------------------------------------------ small puts
// Host -> device copies of a few hundred bytes (run descriptors, plan arrays,
// flag resets) issued as the parameters of a one-CTA kernel: behind a kernel
// it starts ~1 us after it, where a copy-engine transfer or memset starts
// ~8-10 us after it (torch.profiler timeline of a cfg2 join) -- and a copy
// from pageable memory needs no staging.  Batches that do not fit fall back
// to cudaMemcpyAsync / cudaMemsetAsync.
struct PutBatch {
    static constexpr int WORDS = 640;  // 2.5 KB of data: well inside the 4 KB parameter space
    static constexpr int ITEMS = 6;
    uint32_t data[WORDS];
    uint32_t* dst[ITEMS];
    int off[ITEMS];
    int nw[ITEMS];
    int n = 0;
    int used = 0;
};

// the launch carries only the words in use: a 2.5 KB parameter block starts
// ~7 us after the kernel before it, a 100-B one ~2.5 us (same timeline)
template <int WORDS>
struct PutParams {
    uint32_t data[WORDS];
    uint32_t* dst[PutBatch::ITEMS];
    int off[PutBatch::ITEMS];
    int nw[PutBatch::ITEMS];
    int n;
};

template <int WORDS>
__global__ void __launch_bounds__(256) k_put(const PutParams<WORDS> b) {
    for (int i = 0; i < b.n; ++i)
        for (int w = threadIdx.x; w < b.nw[i]; w += blockDim.x) b.dst[i][w] = b.data[b.off[i] + w];
}

template <int WORDS>
inline void put_launch(const PutBatch& b, cudaStream_t st) {
    PutParams<WORDS> p;
    std::memcpy(p.data, b.data, sizeof(uint32_t) * b.used);
    for (int i = 0; i < b.n; ++i) {
        p.dst[i] = b.dst[i];
        p.off[i] = b.off[i];
        p.nw[i] = b.nw[i];
    }
    p.n = b.n;
    static bool carve = [] {
        // the same shared-memory carveout as the sort kernels it runs between
        // (no L1 / shared reconfiguration of the SMs around it)
        cudaFuncSetAttribute(k_put<WORDS>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        return true;
    }();
    (void)carve;
    k_put<WORDS><<<1, 256, 0, st>>>(p);
}

// queue `bytes` (a multiple of 4) from host memory for dst; src == nullptr:
// zeros; v != 0: fill every word with v.  false: no room (caller copies)
inline bool put_add(PutBatch& b, void* dst, const void* src, size_t bytes, uint32_t v = 0) {
    const int nw = (int)(bytes / 4);
    if (bytes % 4 || b.n == PutBatch::ITEMS || b.used + nw > PutBatch::WORDS) return false;
    if (src) std::memcpy(b.data + b.used, src, bytes);
    else
        for (int w = 0; w < nw; ++w) b.data[b.used + w] = v;
    b.dst[b.n] = (uint32_t*)dst;
    b.off[b.n] = b.used;
    b.nw[b.n] = nw;
    ++b.n;
    b.used += nw;
    return true;
}

inline int put_flush(PutBatch& b, cudaStream_t st) {
    if (b.n == 0) return 0;
    if (b.used <= 32) put_launch<32>(b, st);
    else if (b.used <= 160) put_launch<160>(b, st);
    else put_launch<PutBatch::WORDS>(b, st);
    b.n = b.used = 0;
    return check_launch("k_put");
}

// copy (or with src == nullptr zero / fill) through the batch, or directly
// when it is full
inline int put_or_copy(PutBatch& b, void* dst, const void* src, size_t bytes, cudaStream_t st, uint32_t v = 0) {
    if (bytes == 0 || put_add(b, dst, src, bytes, v)) return 0;
    if (src) return cuda_status(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st), "h2d");
    if (v == 0 || v == 0xffffffffu || v == 0x01010101u)
        return cuda_status(cudaMemsetAsync(dst, (int)(v & 0xff), bytes, st), "memset");
    return -1;
}

}  // namespace mpsm
