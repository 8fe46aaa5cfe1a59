// partition_scatter.cu -- the private-input partition scatter for sm_100a:
// every tuple of a worker's chunk goes to the arena region of its partition
// (splitter-vector lookup of its radix bucket), stable, so the arena layout
// is exactly the reference's (worker regions in input order).  Replaces
// _kernels.scatter_chunk (/root/reference/pkg/src/mpsm/_kernels.py:262-284).
//
// One kernel: tiles take a ticket in launch order, rank their tuples stably
// per partition with warp ballots, publish per-partition tile counts,
// resolve their global offsets with a decoupled look-back over predecessor
// tiles (few partitions: short chains), stage the tile in shared memory in
// partition order and write it out in coalesced runs.  (This was the first
// design of the run sort too; segsort.cu replaced it there.)

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>

#include "common.cuh"

namespace mpsm {

#ifndef MPSM_SORT_THREADS
#define MPSM_SORT_THREADS 512
#endif
#ifndef MPSM_SORT_ITEMS
#define MPSM_SORT_ITEMS 12
#endif
constexpr int SORT_THREADS = MPSM_SORT_THREADS;
constexpr int SORT_ITEMS = MPSM_SORT_ITEMS;
constexpr int SORT_TILE = SORT_THREADS * SORT_ITEMS;
constexpr int SORT_WARPS = SORT_THREADS / 32;
constexpr int MAX_BITS = 9;  // at most 512 partitions
constexpr int MAX_BINS = 1 << MAX_BITS;

// look-back status word: [63:62] flag, [61:40] epoch, [39:0] count
constexpr uint64_t FLAG_AGG = 1ull << 62;
constexpr uint64_t FLAG_PREFIX = 2ull << 62;
constexpr uint64_t VALUE_MASK = (1ull << 40) - 1;
constexpr int EPOCH_SHIFT = 40;
constexpr uint64_t EPOCH_MASK = (1ull << 22) - 1;

// process-wide epoch so stale look-back words from earlier calls never match
static uint32_t next_epoch(bool* wrapped) {
    static std::atomic<uint32_t> epoch{0};
    uint32_t e = (epoch.fetch_add(1) + 1) & (uint32_t)EPOCH_MASK;
    *wrapped = (e == 0);
    if (e == 0) e = (epoch.fetch_add(1) + 1) & (uint32_t)EPOCH_MASK;
    return e;
}

struct PartitionDigit {
    uint64_t lower;
    int shift;
    const int32_t* sp;
    int nbuckets;
    __device__ __forceinline__ uint32_t operator()(uint64_t key) const {
        uint64_t b = (key - lower) >> shift;
        // out-of-domain keys were counted in the clamped bucket by the histogram
        if (b >= (uint64_t)nbuckets) b = nbuckets - 1;
        return (uint32_t)__ldg(sp + b);
    }
};

// -------------------------------------------------------------- one pass
// smem: the warp histograms alias the staging buffer (they are dead once
// every thread holds its staging positions).  Keys and payloads are staged
// one after the other through the same buffer; dig[] remembers each staged
// slot's digit for the payload write-out.
struct PassSmem {
    union {
        uint32_t whist[SORT_WARPS][MAX_BINS];
        uint64_t stage[SORT_TILE];
    } u;
    uint16_t dig[SORT_TILE];
    uint32_t tile_off[MAX_BINS];  // exclusive prefix of tile counts over digits
    int64_t gdelta[MAX_BINS];     // global slot of staged position i = gdelta[d] + i
    uint32_t ticket;
};

// peers of this lane among the lanes of vmask holding the same digit: one
// ballot per digit bit (cheaper than match.any on sm_100)
__device__ __forceinline__ unsigned ballot_match(uint32_t d, int bits, unsigned vmask) {
    unsigned peers = vmask;
#pragma unroll
    for (int b = 0; b < MAX_BITS; ++b) {
        if (b < bits) {
            const bool set = (d >> b) & 1u;
            const unsigned bal = __ballot_sync(0xffffffffu, set);
            peers &= set ? bal : ~bal;
        }
    }
    return peers;
}

template <class DigitOp>
__global__ void __launch_bounds__(SORT_THREADS, 2) k_onesweep(
    const uint64_t* __restrict__ in_k, const uint64_t* __restrict__ in_p, uint64_t* __restrict__ out_k,
    uint64_t* __restrict__ out_p, int64_t n, DigitOp digit, int bits, int nbins, const int64_t* __restrict__ bin_base,
    uint64_t* __restrict__ status, int64_t st_stride, unsigned int* __restrict__ ticket_ctr, uint32_t epoch,
    int64_t* __restrict__ written) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PassSmem& sm = *reinterpret_cast<PassSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    if (tid == 0) sm.ticket = atomicAdd(ticket_ctr, 1u);
    for (int i = tid; i < SORT_WARPS * MAX_BINS; i += SORT_THREADS) (&sm.u.whist[0][0])[i] = 0;
    __syncthreads();
    const uint32_t tile = sm.ticket;
    const int64_t tile_base = (int64_t)tile * SORT_TILE;
    const int64_t warp_base = tile_base + (int64_t)warp * (32 * SORT_ITEMS);
    const bool full = tile_base + SORT_TILE <= n;

    // ---- keys, warp-striped: item k of lane l is warp_base + 32k + l
    uint64_t key[SORT_ITEMS];
    uint32_t pos[SORT_ITEMS];  // digit << 20 | rank until offsets are known
#pragma unroll
    for (int k = 0; k < SORT_ITEMS; ++k) {
        const int64_t idx = warp_base + 32 * k + lane;
        key[k] = (full || idx < n) ? ld_stream(in_k + idx) : 0;
    }
    // ---- stable rank within the warp: ballot match + running per-warp counts
    uint32_t* wh = sm.u.whist[warp];
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int k = 0; k < SORT_ITEMS; ++k) {
        const int64_t idx = warp_base + 32 * k + lane;
        const bool valid = full || idx < n;
        const unsigned vmask = full ? 0xffffffffu : __ballot_sync(0xffffffffu, valid);
        const uint32_t d = digit(key[k]);
        unsigned peers = ballot_match(d, bits, vmask);  // every lane votes (full-mask ballots)
        if (!valid) peers = 0;
        uint32_t before = 0;
        if (peers) before = wh[d];
        __syncwarp();
        if (peers && (peers & lt) == 0) wh[d] = before + __popc(peers);
        __syncwarp();
        pos[k] = peers ? ((d << 20) | (before + __popc(peers & lt))) : 0xffffffffu;
    }
    __syncthreads();

    // ---- per digit (DPT per thread): column sum (independent loads), publish
    // the aggregate as early as possible, then the exclusive scan over warps
    constexpr int DPT = (MAX_BINS + SORT_THREADS - 1) / SORT_THREADS;
    uint32_t my_cnt[DPT];
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
        const int d = tid + j * SORT_THREADS;
        my_cnt[j] = 0;
        if (d < nbins) {
            uint32_t col[SORT_WARPS];
#pragma unroll
            for (int w = 0; w < SORT_WARPS; ++w) col[w] = sm.u.whist[w][d];
#pragma unroll
            for (int w = 0; w < SORT_WARPS; ++w) my_cnt[j] += col[w];
            const uint64_t word =
                (uint64_t)my_cnt[j] | ((uint64_t)epoch << EPOCH_SHIFT) | (tile == 0 ? FLAG_PREFIX : FLAG_AGG);
            st_volatile_u64(status + (size_t)tile * nbins + d, word);
            uint32_t run = 0;
#pragma unroll
            for (int w = 0; w < SORT_WARPS; ++w) {
                sm.u.whist[w][d] = run;
                run += col[w];
            }
        }
        if (d < MAX_BINS) sm.tile_off[d] = my_cnt[j];
    }
    (void)st_stride;
    __syncthreads();
    // ---- tile-local exclusive scan of counts over digits (warp 0)
    if (warp == 0) {
        constexpr int PER = MAX_BINS / 32;
        uint32_t loc[PER];
        uint32_t sum = 0;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            loc[q] = sm.tile_off[lane * PER + q];
            sum += loc[q];
        }
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        uint32_t run = incl - sum;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const uint32_t c = loc[q];
            sm.tile_off[lane * PER + q] = run;
            run += c;
        }
    }
    // ---- decoupled look-back for this thread's digits, two predecessors per step
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
        const int d = tid + j * SORT_THREADS;
        if (d < nbins) {
            uint64_t excl = 0;
            if (tile > 0) {
                int64_t t = (int64_t)tile - 1;
                while (true) {
                    const uint64_t w1 = ld_volatile_u64(status + (size_t)t * nbins + d);
                    const uint64_t w2 = t > 0 ? ld_volatile_u64(status + (size_t)(t - 1) * nbins + d) : 0;
                    if (((w1 >> EPOCH_SHIFT) & EPOCH_MASK) != epoch || (w1 >> 62) == 0) continue;
                    excl += w1 & VALUE_MASK;
                    if ((w1 >> 62) == 2) break;
                    --t;
                    if (((w2 >> EPOCH_SHIFT) & EPOCH_MASK) != epoch || (w2 >> 62) == 0) continue;
                    excl += w2 & VALUE_MASK;
                    if ((w2 >> 62) == 2) break;
                    --t;
                }
                st_volatile_u64(status + (size_t)tile * nbins + d,
                                (excl + my_cnt[j]) | ((uint64_t)epoch << EPOCH_SHIFT) | FLAG_PREFIX);
            }
            sm.gdelta[d] = bin_base[d] + (int64_t)excl;
            if (written && my_cnt[j])
                atomicAdd((unsigned long long*)(written + d), (unsigned long long)my_cnt[j]);
        }
    }
    __syncthreads();
    for (int d = tid; d < nbins; d += SORT_THREADS) sm.gdelta[d] -= (int64_t)sm.tile_off[d];
    // ---- staging positions (whist now holds the warp-exclusive offsets);
    // the digit stays in bits 20.. for the write-out
#pragma unroll
    for (int k = 0; k < SORT_ITEMS; ++k) {
        if (pos[k] != 0xffffffffu) {
            const uint32_t dk = pos[k] >> 20;
            pos[k] = (dk << 20) | (sm.tile_off[dk] + sm.u.whist[warp][dk] + (pos[k] & 0xfffffu));
        }
    }
    __syncthreads();  // whist dead from here; stage aliases it
#pragma unroll
    for (int k = 0; k < SORT_ITEMS; ++k) {
        if (pos[k] != 0xffffffffu) {
            const uint32_t p = pos[k] & 0xfffffu;
            sm.u.stage[p] = key[k];
            sm.dig[p] = (uint16_t)(pos[k] >> 20);
        }
    }
    __syncthreads();
    const int valid_in_tile = full ? SORT_TILE : (int)(n - tile_base);
    {
        // payload loads go out now and land while the keys are written
        uint64_t pay[SORT_ITEMS];
#pragma unroll
        for (int k = 0; k < SORT_ITEMS; ++k) {
            const int64_t idx = warp_base + 32 * k + lane;
            pay[k] = (full || idx < n) ? ld_stream(in_p + idx) : 0;
        }
#pragma unroll 4
        for (int i = tid; i < valid_in_tile; i += SORT_THREADS) out_k[sm.gdelta[sm.dig[i]] + i] = sm.u.stage[i];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < SORT_ITEMS; ++k)
            if (pos[k] != 0xffffffffu) sm.u.stage[pos[k] & 0xfffffu] = pay[k];
        __syncthreads();
#pragma unroll 4
        for (int i = tid; i < valid_in_tile; i += SORT_THREADS) out_p[sm.gdelta[sm.dig[i]] + i] = sm.u.stage[i];
    }
}

static size_t pass_smem_bytes() { return sizeof(PassSmem); }

static int64_t num_tiles(int64_t n) { return (n + SORT_TILE - 1) / SORT_TILE; }
// look-back rows are 32-B aligned
static int64_t status_stride(int64_t n) { return (std::max<int64_t>(num_tiles(n), 1) + 3) & ~(int64_t)3; }

static int set_pass_smem() {
    static bool done = false;
    if (!done) {
        MPSM_TRY(cuda_status(cudaFuncSetAttribute(k_onesweep<PartitionDigit>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pass_smem_bytes()),
                             "smem attr"));
        done = true;
    }
    return MPSM_OK;
}

}  // namespace mpsm

using namespace mpsm;

// ------------------------------------------------------------ partition scatter
extern "C" int mpsm_scatter_workspace_bytes(int64_t n, int npart, size_t* bytes) {
    if (!bytes || n < 0 || npart < 1 || npart > MAX_BINS) return MPSM_ERR_ARG;
    size_t b = 0;
    b += align_up(sizeof(unsigned int) * 1);
    b += align_up(sizeof(uint64_t) * (size_t)status_stride(n) * npart);
    *bytes = b;
    return MPSM_OK;
}

extern "C" int mpsm_scatter_chunk(const uint64_t* keys, const uint64_t* pays, int64_t n, uint64_t lower, int shift,
                                  const int32_t* d_sp, int nbuckets, int npart, const int64_t* d_cursors,
                                  uint64_t* arena_keys, uint64_t* arena_pays, int64_t* d_written, void* workspace,
                                  size_t ws_bytes, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n < 0 || npart < 1 || npart > MAX_BINS || nbuckets < 1 || shift < 0 || shift > 63) {
        set_error("scatter: bad arguments (npart must be <= 512)");
        return MPSM_ERR_ARG;
    }
    if (n == 0) return MPSM_OK;
    Carve c{(char*)workspace, ws_bytes};
    unsigned int* ticket = c.take<unsigned int>(1);
    uint64_t* status = c.take<uint64_t>((size_t)status_stride(n) * npart);
    if (!c.ok) {
        set_error("scatter workspace too small");
        return MPSM_ERR_ARG;
    }
    MPSM_TRY(set_pass_smem());
    MPSM_TRY(cuda_status(cudaMemsetAsync(ticket, 0, sizeof(unsigned int), st), "memset"));
    bool wrapped = false;
    uint32_t epoch = next_epoch(&wrapped);
    if (wrapped)
        MPSM_TRY(cuda_status(cudaMemsetAsync(status, 0, sizeof(uint64_t) * (size_t)status_stride(n) * npart, st), "memset"));
    PartitionDigit dig{lower, shift, d_sp, nbuckets};
    int pbits = 0;
    while ((1 << pbits) < npart) ++pbits;
    ProfScope ps("scatter", st);
    k_onesweep<PartitionDigit><<<(unsigned)num_tiles(n), SORT_THREADS, pass_smem_bytes(), st>>>(
        keys, pays, arena_keys, arena_pays, n, dig, pbits, npart, d_cursors, status, status_stride(n), ticket, epoch,
        d_written);
    return check_launch("k_onesweep<partition>");
}
