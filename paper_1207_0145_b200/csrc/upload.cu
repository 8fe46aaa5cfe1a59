// upload.cu -- host->HBM input path that halves the PCIe bytes: host worker
// threads pack (key, payload) u64 SoA into 8-B records
// (key - lower) << pw | payload (the layout every sort pass after the first
// moves anyway) in pinned staging slots, and each packed chunk goes to HBM
// with its own async copy while later chunks are being packed.  The domain
// check of the first sort pass (DomainError, sorter.py:97-98) and the
// payload-width check of the packed layout move into the packing loop.
// Measured on the GPU box (tools/host_pack_bench.cu, bench.py e2e): plain
// pinned H2D of 16 B/tuple 55.6 GB/s (144 ms for cfg2's 500M tuples);
// 1 MB staging slots, 12 packing threads: cfg2 end to end 155 -> 101 ms.
// Slots small enough to stay in the host's last-level cache matter: the copy
// then reads the packed chunk from cache, and host DRAM sees little more
// than the column reads (1M-tuple slots: 120 ms).

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"
#include "hostcpu.h"

namespace mpsm {

// raw chunks: the GPU reads the (pinned, device-mapped) host columns itself
// over PCIe and packs them -- moves 16 B per tuple, but no host CPU work, so
// mixing raw and host-packed chunks balances host memory bandwidth against
// PCIe
__global__ void __launch_bounds__(256) k_pack_mapped(const uint64_t* __restrict__ hk, const uint64_t* __restrict__ hp,
                                                     int64_t m, int64_t base, uint64_t lower, uint64_t span_m1, int pw,
                                                     uint64_t* __restrict__ out, unsigned long long* __restrict__ bad,
                                                     unsigned int* __restrict__ ovf) {
    uint64_t o = 0;
    unsigned long long first = ~0ull;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = hk[i] - lower, p = hp[i];
        if (k > span_m1 && (unsigned long long)(base + i) < first) first = (unsigned long long)(base + i);
        o |= p >> pw;
        out[i] = (k << pw) | p;
    }
    if (first != ~0ull) atomicMin(bad, first);
    if (__any_sync(0xffffffffu, o != 0) && (threadIdx.x & 31) == 0) atomicOr(ovf, 1u);
}

namespace {

// tuples per staging slot (packed: 8 B each); MPSM_UPLOAD_CHUNK overrides
int64_t chunk_default() {
    const char* e = getenv("MPSM_UPLOAD_CHUNK");
    // 1 MB packed slots: packed data is still in the host's last-level cache
    // when its copy reads it (cfg2 e2e: 1M-tuple slots 120 ms, 128K 100 ms,
    // 64K 122 ms: per-copy overhead)
    return e ? std::max<int64_t>(4096, atoll(e)) : (int64_t)1 << 17;
}
std::atomic<uint64_t> g_upload_bytes{0};  // host->device bytes moved by uploads

// every raw_every-th chunk is packed by the GPU from mapped host memory
// (0: all chunks packed by the host); MPSM_UPLOAD_RAW_EVERY overrides
int raw_every_default() {
    const char* e = getenv("MPSM_UPLOAD_RAW_EVERY");
    return e ? atoi(e) : 0;  // off: with cache-sized slots the host alone keeps up
}

struct Uploader {
    int64_t CHUNK = 0;
    int nslots = 0;
    std::vector<uint64_t*> slot;         // pinned staging
    std::vector<cudaEvent_t> slot_done;  // copy of the slot's last chunk finished
    cudaStream_t copy = nullptr;
    cudaEvent_t done = nullptr;
    std::vector<std::thread> pool;
    std::mutex mu;
    std::condition_variable cv_work, cv_idle;
    // job
    const uint64_t* keys = nullptr;
    const uint64_t* pays = nullptr;
    int64_t n = 0, nch = 0;
    uint64_t lower = 0, span_m1 = 0;
    int pw = 0;
    uint64_t gen = 0;  // job generation
    int finished = 0;  // workers done with the current generation
    std::atomic<int64_t> next{0};
    std::vector<std::atomic<int>> ready, issued;
    std::atomic<int64_t> bad{INT64_MAX};
    std::atomic<int> overflow{0};
    int raw_every = 0;  // this job
    unsigned long long* d_bad = nullptr;
    unsigned int* d_ovf = nullptr;
    bool stop = false;

    bool is_raw(int64_t c) const { return raw_every > 0 && c % raw_every == raw_every - 1; }

    ~Uploader() {  // process exit: release the workers (CUDA objects die with the context)
        {
            std::lock_guard<std::mutex> g(mu);
            stop = true;
        }
        cv_work.notify_all();
        for (auto& t : pool)
            if (t.joinable()) t.join();
    }

    int init(int threads) {
        if (copy) return MPSM_OK;
        CHUNK = chunk_default();
        if (threads <= 0) {
            const char* e = getenv("MPSM_UPLOAD_THREADS");
            // leave the issuing thread a core
            // the copy is host-memory-bandwidth bound: 3/4 of the cores pack
            // (measured best on the 16-core GPU box: 12 -> 113 ms, 16 -> 121 ms
            // for cfg2's 500M tuples); one process per GPU: a rank's share of the cores
            threads = e ? atoi(e) : std::max(1, usable_cores_per_rank() * 3 / 4);
        }
        nslots = 2 * threads;
        slot.resize(nslots);
        slot_done.resize(nslots);
        for (int i = 0; i < nslots; ++i) {
            MPSM_TRY(cuda_status(cudaHostAlloc((void**)&slot[i], CHUNK * 8, cudaHostAllocDefault), "pinned staging"));
            MPSM_TRY(cuda_status(cudaEventCreateWithFlags(&slot_done[i], cudaEventDisableTiming), "event"));
        }
        MPSM_TRY(cuda_status(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking), "copy stream"));
        MPSM_TRY(cuda_status(cudaEventCreateWithFlags(&done, cudaEventDisableTiming), "event"));
        MPSM_TRY(cuda_status(cudaMalloc(&d_bad, sizeof(unsigned long long)), "flag"));
        MPSM_TRY(cuda_status(cudaMalloc(&d_ovf, sizeof(unsigned int)), "flag"));
        for (int i = 0; i < threads; ++i) pool.emplace_back([this] { worker(); });
        return MPSM_OK;
    }

    void pack_chunk(int64_t c) {
        const int64_t a = c * CHUNK, b = std::min(n, a + CHUNK);
        uint64_t* out = slot[c % nslots];
        uint64_t ovf = 0;
        int64_t first_bad = INT64_MAX;
        for (int64_t i = a; i < b; ++i) {
            const uint64_t k = keys[i] - lower, p = pays[i];
            if (k > span_m1 && i < first_bad) first_bad = i;
            ovf |= p >> pw;
            out[i - a] = (k << pw) | p;
        }
        if (first_bad != INT64_MAX) {
            int64_t cur = bad.load();
            while (first_bad < cur && !bad.compare_exchange_weak(cur, first_bad)) {
            }
        }
        if (ovf) overflow.store(1);
    }

    void worker() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> g(mu);
                cv_work.wait(g, [&] { return stop || gen != seen; });
                if (stop) return;
                seen = gen;
            }
            for (;;) {
                const int64_t c = next.fetch_add(1);
                if (c >= nch) break;
                if (is_raw(c)) continue;  // the GPU packs it
                if (c >= nslots) {  // the slot's previous chunk must have left
                    while (!issued[c - nslots].load(std::memory_order_acquire)) std::this_thread::yield();
                    cudaEventSynchronize(slot_done[c % nslots]);
                }
                pack_chunk(c);
                ready[c].store(1, std::memory_order_release);
            }
            {
                std::lock_guard<std::mutex> g(mu);
                if (++finished == (int)pool.size()) cv_idle.notify_all();
            }
        }
    }

    int run(const uint64_t* k, const uint64_t* p, int64_t n_, uint64_t lo, uint64_t span, int pw_, uint64_t* d_rec,
            int gpu_every, cudaStream_t st, cudaEvent_t ready_ev, int64_t* bad_out, int* ovf_out) {
        // the copy stream must not overwrite a slot that a previous call's
        // copies still read: drain it first
        MPSM_TRY(cuda_status(cudaStreamSynchronize(copy), "drain"));
        n = n_;
        nch = (n + CHUNK - 1) / CHUNK;
        keys = k;
        pays = p;
        lower = lo;
        span_m1 = span;
        pw = pw_;
        bad.store(INT64_MAX);
        overflow.store(0);
        next.store(0);
        // raw chunks need host columns the GPU can read (pinned / registered)
        raw_every = 0;
        if (gpu_every < 0) gpu_every = raw_every_default();
        if (gpu_every > 0) {
            cudaPointerAttributes ak, ap;
            if (cudaPointerGetAttributes(&ak, k) == cudaSuccess && cudaPointerGetAttributes(&ap, p) == cudaSuccess &&
                ak.type == cudaMemoryTypeHost && ap.type == cudaMemoryTypeHost && ak.devicePointer == k &&
                ap.devicePointer == p)
                raw_every = gpu_every;
            cudaGetLastError();
        }
        MPSM_TRY(cuda_status(cudaMemsetAsync(d_bad, 0xff, sizeof(unsigned long long), copy), "flag"));
        MPSM_TRY(cuda_status(cudaMemsetAsync(d_ovf, 0, sizeof(unsigned int), copy), "flag"));
        ready = std::vector<std::atomic<int>>(nch);
        issued = std::vector<std::atomic<int>>(nch);
        for (int64_t c = 0; c < nch; ++c) {
            ready[c].store(0);
            issued[c].store(0);
        }
        // the compute stream's earlier work (which may still use d_rec's
        // memory) first: all of it, or what preceded the caller's `ready`
        // event (recorded when d_rec was allocated -- later work, e.g. a sort
        // queued meanwhile, then runs concurrently with the upload)
        if (ready_ev) {
            MPSM_TRY(cuda_status(cudaStreamWaitEvent(copy, ready_ev, 0), "wait"));
        } else {
            MPSM_TRY(cuda_status(cudaEventRecord(done, st), "event"));
            MPSM_TRY(cuda_status(cudaStreamWaitEvent(copy, done, 0), "wait"));
        }
        {
            std::lock_guard<std::mutex> g(mu);
            finished = 0;
            ++gen;
        }
        cv_work.notify_all();
        int rc = MPSM_OK;
        for (int64_t c = 0; c < nch; ++c) {
            const int64_t a = c * CHUNK, m = std::min(n, a + CHUNK) - a;
            g_upload_bytes += (uint64_t)m * (is_raw(c) ? 16 : 8);
            if (is_raw(c)) {
                if (rc == MPSM_OK) {
                    k_pack_mapped<<<num_sms() * 2, 256, 0, copy>>>(keys + a, pays + a, m, a, lower, span_m1, pw,
                                                                   d_rec + a, d_bad, d_ovf);
                    rc = check_launch("k_pack_mapped");
                }
                issued[c].store(1, std::memory_order_release);
                continue;
            }
            while (!ready[c].load(std::memory_order_acquire)) std::this_thread::yield();
            if (rc == MPSM_OK)
                rc = cuda_status(cudaMemcpyAsync(d_rec + a, slot[c % nslots], m * 8, cudaMemcpyHostToDevice, copy),
                                 "h2d");
            if (rc == MPSM_OK) rc = cuda_status(cudaEventRecord(slot_done[c % nslots], copy), "event");
            issued[c].store(1, std::memory_order_release);
        }
        {  // every worker has seen this job through: the next job may reset it
            std::unique_lock<std::mutex> g(mu);
            cv_idle.wait(g, [&] { return finished == (int)pool.size(); });
        }
        MPSM_TRY(rc);
        // later work on the caller's stream sees the records
        MPSM_TRY(cuda_status(cudaEventRecord(done, copy), "event"));
        MPSM_TRY(cuda_status(cudaStreamWaitEvent(st, done, 0), "wait"));
        int64_t b = bad.load();
        int o = overflow.load();
        if (raw_every > 0) {  // the GPU-packed chunks' checks
            unsigned long long db = 0;
            unsigned int dovf = 0;
            MPSM_TRY(cuda_status(cudaMemcpyAsync(&db, d_bad, sizeof(db), cudaMemcpyDeviceToHost, copy), "d2h"));
            MPSM_TRY(cuda_status(cudaMemcpyAsync(&dovf, d_ovf, sizeof(dovf), cudaMemcpyDeviceToHost, copy), "d2h"));
            MPSM_TRY(cuda_status(cudaStreamSynchronize(copy), "sync"));
            if (db != ~0ull && (int64_t)db < b) b = (int64_t)db;
            o |= dovf != 0;
        }
        *bad_out = b == INT64_MAX ? -1 : b;
        *ovf_out = o;
        return MPSM_OK;
    }
};

Uploader& uploader() {
    static Uploader u;
    return u;
}

}  // namespace
}  // namespace mpsm

using namespace mpsm;

extern "C" int mpsm_upload_records(const uint64_t* h_keys, const uint64_t* h_pays, int64_t n, uint64_t lower,
                                   uint64_t span_m1, int width_bits, uint64_t* d_rec, int threads, int gpu_pack_every,
                                   void* stream, void* ready_event, int64_t* bad_index, int* overflow) {
    if (n < 0 || width_bits < 1 || width_bits > 63 || !bad_index || !overflow) return MPSM_ERR_ARG;
    *bad_index = -1;
    *overflow = 0;
    if (n == 0) return MPSM_OK;
    if (!h_keys || !h_pays || !d_rec) return MPSM_ERR_ARG;
    Uploader& u = uploader();
    MPSM_TRY(u.init(threads));
    return u.run(h_keys, h_pays, n, lower, span_m1, 64 - width_bits, d_rec, gpu_pack_every, (cudaStream_t)stream,
                 (cudaEvent_t)ready_event, bad_index, overflow);
}

extern "C" uint64_t mpsm_upload_bytes(int reset) {
    return reset ? g_upload_bytes.exchange(0) : g_upload_bytes.load();
}

extern "C" int mpsm_pack_records(const uint64_t* d_keys, const uint64_t* d_pays, int64_t n, uint64_t lower,
                                 uint64_t span_m1, int width_bits, uint64_t* d_rec, unsigned long long* d_bad,
                                 unsigned int* d_overflow, void* stream) {
    if (n < 0 || width_bits < 1 || width_bits > 63 || !d_bad || !d_overflow) return MPSM_ERR_ARG;
    if (n == 0) return MPSM_OK;
    const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8);
    k_pack_mapped<<<grid, 256, 0, (cudaStream_t)stream>>>(d_keys, d_pays, n, 0, lower, span_m1, 64 - width_bits, d_rec,
                                                          d_bad, d_overflow);
    return check_launch("k_pack_mapped");
}
