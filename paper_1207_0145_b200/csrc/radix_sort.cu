// radix_sort.cu -- onesweep LSD radix sort of (u64 key, u64 payload) SoA pairs
// and the stable partition scatter, for sm_100a.
//
// Replaces the reference run sort _kernels.three_phase_sort
// (/root/reference/pkg/src/mpsm/_kernels.py:217-244; MSD radix cluster +
// introsort + insertion pass on CPU) and the private-input scatter
// _kernels.scatter_chunk (_kernels.py:262-284).
//
// Sort = one upfront sweep that histograms every digit of every pass and
// checks the key domain (8 B/tuple), then one scatter pass per digit
// (16 B read + 16 B write per tuple).  Each pass is a single kernel: tiles
// take a ticket in launch order, rank their keys stably per digit with warp
// match_any, publish per-digit tile counts, resolve their global offsets with
// a decoupled look-back over predecessor tiles, stage the tile in shared
// memory in digit order and write it out with coalesced runs.
//
// The partition scatter is the same pass with digit = partition id
// (splitter-vector lookup of the radix bucket) and per-partition base
// offsets = the worker's write cursors, so the arena layout is exactly the
// reference's (worker regions in input order).

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>

#include "common.cuh"

namespace mpsm {

constexpr int SORT_THREADS = 256;
constexpr int SORT_ITEMS = 16;
constexpr int SORT_TILE = SORT_THREADS * SORT_ITEMS;
constexpr int SORT_WARPS = SORT_THREADS / 32;
constexpr int MAX_BITS = 9;
constexpr int MAX_BINS = 1 << MAX_BITS;
constexpr int MAX_PASSES = 8;

// look-back status word: [63:62] flag, [61:40] epoch, [39:0] count
constexpr uint64_t FLAG_AGG = 1ull << 62;
constexpr uint64_t FLAG_PREFIX = 2ull << 62;
constexpr uint64_t VALUE_MASK = (1ull << 40) - 1;
constexpr int EPOCH_SHIFT = 40;
constexpr uint64_t EPOCH_MASK = (1ull << 22) - 1;

struct PassPlan {
    int npasses;
    int shift[MAX_PASSES];
    int bits[MAX_PASSES];
};

static PassPlan plan_passes(int width_bits) {
    PassPlan p{};
    if (width_bits <= 0) return p;
    int np = (width_bits + MAX_BITS - 1) / MAX_BITS;
    int base = width_bits / np, rem = width_bits % np, sh = 0;
    p.npasses = np;
    for (int i = 0; i < np; ++i) {
        p.bits[i] = base + (i < rem ? 1 : 0);
        p.shift[i] = sh;
        sh += p.bits[i];
    }
    return p;
}

// process-wide epoch so stale look-back words from earlier passes never match
static uint32_t next_epoch(bool* wrapped) {
    static std::atomic<uint32_t> epoch{0};
    uint32_t e = (epoch.fetch_add(1) + 1) & (uint32_t)EPOCH_MASK;
    *wrapped = (e == 0);
    if (e == 0) e = (epoch.fetch_add(1) + 1) & (uint32_t)EPOCH_MASK;
    return e;
}

// ------------------------------------------------------------ upfront sweep
__global__ void __launch_bounds__(512) k_upfront_hist(const uint64_t* __restrict__ keys, int64_t n, uint64_t lower,
                                                      uint64_t span_m1, PassPlan plan,
                                                      unsigned long long* __restrict__ g_hist,
                                                      unsigned long long* __restrict__ d_bad) {
    __shared__ uint32_t sh[MAX_PASSES * MAX_BINS];
    const int nb = plan.npasses * MAX_BINS;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        uint64_t nk = ld_stream(keys + i) - lower;
        // out-of-domain keys are flagged but still counted, so the scatter
        // passes stay in bounds; the caller discards the result
        if (nk > span_m1 && d_bad) atomicMin(d_bad, (unsigned long long)i);
        for (int p = 0; p < plan.npasses; ++p) {
            uint32_t d = (uint32_t)(nk >> plan.shift[p]) & ((1u << plan.bits[p]) - 1u);
            atomicAdd(&sh[p * MAX_BINS + d], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nb; i += blockDim.x)
        if (sh[i]) atomicAdd(&g_hist[i], (unsigned long long)sh[i]);
}

// exclusive scan of each pass's histogram -> bucket start offsets
__global__ void __launch_bounds__(MAX_BINS) k_bucket_starts(const unsigned long long* __restrict__ g_hist,
                                                            PassPlan plan, int64_t* __restrict__ starts) {
    __shared__ int64_t s[MAX_BINS];
    const int p = blockIdx.x;
    const int nbins = 1 << plan.bits[p];
    const int t = threadIdx.x;
    int64_t v = (t < nbins) ? (int64_t)g_hist[p * MAX_BINS + t] : 0;
    s[t] = v;
    __syncthreads();
    for (int off = 1; off < MAX_BINS; off <<= 1) {
        int64_t add = (t >= off) ? s[t - off] : 0;
        __syncthreads();
        s[t] += add;
        __syncthreads();
    }
    if (t < nbins) starts[p * MAX_BINS + t] = s[t] - v;
}

// ---------------------------------------------------------------- digit ops
struct RadixDigit {
    uint64_t lower;
    int shift;
    uint32_t mask;
    __device__ __forceinline__ uint32_t operator()(uint64_t key) const {
        return (uint32_t)((key - lower) >> shift) & mask;
    }
};

struct PartitionDigit {
    uint64_t lower;
    int shift;
    const int32_t* sp;
    int nbuckets;
    __device__ __forceinline__ uint32_t operator()(uint64_t key) const {
        uint64_t b = (key - lower) >> shift;
        // out-of-domain keys were rejected by the histogram; clamp defensively
        if (b >= (uint64_t)nbuckets) b = nbuckets - 1;
        return (uint32_t)__ldg(sp + b);
    }
};

// -------------------------------------------------------------- one pass
// smem: warp histograms alias the staging buffer (they are dead once every
// thread has its staging positions)
struct PassSmem {
    union {
        uint32_t whist[SORT_WARPS][MAX_BINS];
        uint64_t stage[SORT_TILE];
    } u;
    uint16_t dig[SORT_TILE];
    uint32_t tile_off[MAX_BINS];  // exclusive prefix of tile counts over digits
    int64_t gdelta[MAX_BINS];     // global position of staged slot i = gdelta[d] + i
    uint32_t ticket;
};

template <class DigitOp>
__global__ void __launch_bounds__(SORT_THREADS) k_onesweep(const uint64_t* __restrict__ in_k,
                                                           const uint64_t* __restrict__ in_p,
                                                           uint64_t* __restrict__ out_k, uint64_t* __restrict__ out_p,
                                                           int64_t n, DigitOp digit, int nbins,
                                                           const int64_t* __restrict__ bin_base,
                                                           uint64_t* __restrict__ status,
                                                           unsigned int* __restrict__ ticket_ctr, uint32_t epoch,
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

    // ---- load keys (warp-striped: item k of lane l is warp_base + 32k + l)
    uint64_t key[SORT_ITEMS];
    uint32_t pos[SORT_ITEMS];
#pragma unroll
    for (int k = 0; k < SORT_ITEMS; ++k) {
        int64_t idx = warp_base + 32 * k + lane;
        key[k] = idx < n ? ld_stream(in_k + idx) : 0;
    }
    // ---- stable rank within the warp's sub-tile
    uint32_t* wh = sm.u.whist[warp];
#pragma unroll
    for (int k = 0; k < SORT_ITEMS; ++k) {
        int64_t idx = warp_base + 32 * k + lane;
        const bool valid = idx < n;
        const unsigned vmask = __ballot_sync(0xffffffffu, valid);
        uint32_t rank = 0;
        if (valid) {
            uint32_t d = digit(key[k]);
            unsigned peers = __match_any_sync(vmask, d);
            uint32_t before = wh[d];
            rank = before + __popc(peers & lanemask_lt());
            __syncwarp(vmask);
            if ((peers & lanemask_lt()) == 0) wh[d] = before + __popc(peers);
            __syncwarp(vmask);
            pos[k] = rank | (d << 20);  // stash digit until offsets exist
        } else {
            pos[k] = 0xffffffffu;
        }
    }
    __syncthreads();

    // ---- per digit: exclusive scan over warps, tile count, publish aggregate
    uint32_t my_cnt[MAX_BINS / SORT_THREADS > 0 ? MAX_BINS / SORT_THREADS : 1];
#pragma unroll
    for (int j = 0; j < MAX_BINS / SORT_THREADS; ++j) {
        const int d = tid + j * SORT_THREADS;
        uint32_t run = 0;
        if (d < nbins) {
#pragma unroll
            for (int w = 0; w < SORT_WARPS; ++w) {
                uint32_t c = sm.u.whist[w][d];
                sm.u.whist[w][d] = run;
                run += c;
            }
            uint64_t word = (uint64_t)run | ((uint64_t)epoch << EPOCH_SHIFT) | (tile == 0 ? FLAG_PREFIX : FLAG_AGG);
            st_volatile_u64(status + (size_t)tile * nbins + d, word);
        }
        my_cnt[j] = run;
        sm.tile_off[d] = run;
    }
    __syncthreads();
    // ---- tile-local exclusive scan of counts over digits (single warp-based scan)
    if (warp == 0) {
        // each lane owns MAX_BINS/32 consecutive digits
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
            uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        uint32_t run = incl - sum;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            uint32_t c = loc[q];
            sm.tile_off[lane * PER + q] = run;
            run += c;
        }
    }
    // ---- decoupled look-back for this tile's digits
#pragma unroll
    for (int j = 0; j < MAX_BINS / SORT_THREADS; ++j) {
        const int d = tid + j * SORT_THREADS;
        if (d < nbins) {
            uint64_t excl = 0;
            if (tile > 0) {
                int64_t t = (int64_t)tile - 1;
                while (true) {
                    uint64_t w = ld_volatile_u64(status + (size_t)t * nbins + d);
                    if (((w >> EPOCH_SHIFT) & EPOCH_MASK) != epoch || (w >> 62) == 0) continue;
                    excl += w & VALUE_MASK;
                    if ((w >> 62) == 2) break;
                    --t;
                }
                st_volatile_u64(status + (size_t)tile * nbins + d,
                                (excl + my_cnt[j]) | ((uint64_t)epoch << EPOCH_SHIFT) | FLAG_PREFIX);
            }
            sm.gdelta[d] = bin_base[d] + (int64_t)excl;  // tile_off subtracted below
            if (written && my_cnt[j]) atomicAdd((unsigned long long*)(written + d), (unsigned long long)my_cnt[j]);
        }
    }
    __syncthreads();
    for (int d = tid; d < nbins; d += SORT_THREADS) sm.gdelta[d] -= (int64_t)sm.tile_off[d];
    // ---- staging positions
#pragma unroll
    for (int k = 0; k < SORT_ITEMS; ++k) {
        if (pos[k] != 0xffffffffu) {
            uint32_t d = pos[k] >> 20;
            pos[k] = sm.tile_off[d] + sm.u.whist[warp][d] + (pos[k] & 0xfffffu);
        }
    }
    __syncthreads();  // whist dead from here; stage aliases it
#pragma unroll
    for (int k = 0; k < SORT_ITEMS; ++k) {
        if (pos[k] != 0xffffffffu) {
            sm.u.stage[pos[k]] = key[k];
            sm.dig[pos[k]] = (uint16_t)digit(key[k]);
        }
    }
    __syncthreads();
    const int valid_in_tile = (int)min((int64_t)SORT_TILE, n - tile_base);
#pragma unroll 4
    for (int i = tid; i < valid_in_tile; i += SORT_THREADS) {
        out_k[sm.gdelta[sm.dig[i]] + i] = sm.u.stage[i];
    }
    // ---- payloads follow the same permutation
    uint64_t pay[SORT_ITEMS];
#pragma unroll
    for (int k = 0; k < SORT_ITEMS; ++k) {
        int64_t idx = warp_base + 32 * k + lane;
        pay[k] = idx < n ? ld_stream(in_p + idx) : 0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < SORT_ITEMS; ++k)
        if (pos[k] != 0xffffffffu) sm.u.stage[pos[k]] = pay[k];
    __syncthreads();
#pragma unroll 4
    for (int i = tid; i < valid_in_tile; i += SORT_THREADS) {
        out_p[sm.gdelta[sm.dig[i]] + i] = sm.u.stage[i];
    }
}

static size_t pass_smem_bytes() { return sizeof(PassSmem); }

static int64_t num_tiles(int64_t n) { return (n + SORT_TILE - 1) / SORT_TILE; }

struct SortWorkspace {
    unsigned long long* hist;  // [MAX_PASSES][MAX_BINS]
    int64_t* starts;           // [MAX_PASSES][MAX_BINS]
    unsigned int* tickets;     // [MAX_PASSES]
    uint64_t* status;          // [tiles][MAX_BINS]
};

static size_t sort_ws_bytes(int64_t n) {
    size_t b = 0;
    b += align_up(sizeof(unsigned long long) * MAX_PASSES * MAX_BINS);
    b += align_up(sizeof(int64_t) * MAX_PASSES * MAX_BINS);
    b += align_up(sizeof(unsigned int) * MAX_PASSES);
    b += align_up(sizeof(uint64_t) * (size_t)std::max<int64_t>(num_tiles(n), 1) * MAX_BINS);
    return b;
}

static bool carve_sort(void* ws, size_t bytes, int64_t n, SortWorkspace* out) {
    Carve c{(char*)ws, bytes};
    out->hist = c.take<unsigned long long>(MAX_PASSES * MAX_BINS);
    out->starts = c.take<int64_t>(MAX_PASSES * MAX_BINS);
    out->tickets = c.take<unsigned int>(MAX_PASSES);
    out->status = c.take<uint64_t>((size_t)std::max<int64_t>(num_tiles(n), 1) * MAX_BINS);
    return c.ok;
}

static int set_pass_smem() {
    static bool done = false;
    if (!done) {
        MPSM_TRY(cuda_status(cudaFuncSetAttribute(k_onesweep<RadixDigit>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)pass_smem_bytes()),
                             "smem attr"));
        MPSM_TRY(cuda_status(cudaFuncSetAttribute(k_onesweep<PartitionDigit>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pass_smem_bytes()),
                             "smem attr"));
        done = true;
    }
    return MPSM_OK;
}

static int clear_status_if_wrapped(bool wrapped, uint64_t* status, int64_t n, cudaStream_t st) {
    if (!wrapped) return MPSM_OK;
    return cuda_status(
        cudaMemsetAsync(status, 0, sizeof(uint64_t) * (size_t)std::max<int64_t>(num_tiles(n), 1) * MAX_BINS, st),
        "memset status");
}

}  // namespace mpsm

using namespace mpsm;

extern "C" int mpsm_sort_pass_count(int width_bits) { return plan_passes(width_bits).npasses; }

extern "C" int mpsm_sort_workspace_bytes(int64_t n, int width_bits, size_t* bytes) {
    if (!bytes || n < 0 || width_bits < 0 || width_bits > 64) return MPSM_ERR_ARG;
    *bytes = sort_ws_bytes(n);
    return MPSM_OK;
}

extern "C" int mpsm_sort_pairs(const uint64_t* in_keys, const uint64_t* in_pays, int64_t n, uint64_t lower,
                               uint64_t span_m1, int width_bits, uint64_t* out_keys, uint64_t* out_pays,
                               uint64_t* tmp_keys, uint64_t* tmp_pays, void* workspace, size_t ws_bytes,
                               unsigned long long* d_bad, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n < 0 || width_bits < 0 || width_bits > 64) return MPSM_ERR_ARG;
    if (n == 0) return MPSM_OK;
    SortWorkspace ws;
    if (!carve_sort(workspace, ws_bytes, n, &ws)) {
        set_error("sort workspace too small");
        return MPSM_ERR_ARG;
    }
    MPSM_TRY(set_pass_smem());
    PassPlan plan = plan_passes(width_bits);
    MPSM_TRY(cuda_status(cudaMemsetAsync(ws.hist, 0, sizeof(unsigned long long) * MAX_PASSES * MAX_BINS, st), "memset"));
    MPSM_TRY(cuda_status(cudaMemsetAsync(ws.tickets, 0, sizeof(unsigned int) * MAX_PASSES, st), "memset"));
    {
        int grid = std::min<int64_t>(num_sms() * 4, (n + 511) / 512);
        ProfScope ps("upfront_hist", st);
        k_upfront_hist<<<grid, 512, 0, st>>>(in_keys, n, lower, span_m1, plan, ws.hist, d_bad);
        MPSM_TRY(check_launch("k_upfront_hist"));
    }
    if (plan.npasses == 0) {  // one-value domain: already sorted
        if (out_keys != in_keys) {
            MPSM_TRY(cuda_status(cudaMemcpyAsync(out_keys, in_keys, 8 * n, cudaMemcpyDeviceToDevice, st), "copy"));
            MPSM_TRY(cuda_status(cudaMemcpyAsync(out_pays, in_pays, 8 * n, cudaMemcpyDeviceToDevice, st), "copy"));
        }
        return MPSM_OK;
    }
    k_bucket_starts<<<plan.npasses, MAX_BINS, 0, st>>>(ws.hist, plan, ws.starts);
    MPSM_TRY(check_launch("k_bucket_starts"));

    // buffer schedule: the last pass must land in out; never write in place
    int P = plan.npasses;
    const uint64_t *src_k = in_keys, *src_p = in_pays;
    bool in_is_out = (in_keys == out_keys);
    // choose dst of pass 0 so that after P passes we end in out
    // sequence alternates dst between A and B; last = out.
    uint64_t *A_k = out_keys, *A_p = out_pays, *B_k = tmp_keys, *B_p = tmp_pays;
    // pass i writes to (P-1-i) even ? A : B
    if (in_is_out && (P % 2 == 1)) {
        // first pass would write into its own input; copy input to tmp first
        MPSM_TRY(cuda_status(cudaMemcpyAsync(tmp_keys, in_keys, 8 * n, cudaMemcpyDeviceToDevice, st), "copy"));
        MPSM_TRY(cuda_status(cudaMemcpyAsync(tmp_pays, in_pays, 8 * n, cudaMemcpyDeviceToDevice, st), "copy"));
        src_k = tmp_keys;
        src_p = tmp_pays;
        // now passes: tmp -> out -> tmp -> ... -> out (P odd): pass 0 writes A(out) fine
    }
    const int64_t tiles = num_tiles(n);
    for (int i = 0; i < P; ++i) {
        bool to_a = ((P - 1 - i) % 2) == 0;
        uint64_t* dk = to_a ? A_k : B_k;
        uint64_t* dp = to_a ? A_p : B_p;
        bool wrapped = false;
        uint32_t epoch = next_epoch(&wrapped);
        MPSM_TRY(clear_status_if_wrapped(wrapped, ws.status, n, st));
        RadixDigit dig{lower, plan.shift[i], (1u << plan.bits[i]) - 1u};
        ProfScope ps("onesweep", st);
        k_onesweep<RadixDigit><<<(unsigned)tiles, SORT_THREADS, pass_smem_bytes(), st>>>(
            src_k, src_p, dk, dp, n, dig, 1 << plan.bits[i], ws.starts + i * MAX_BINS, ws.status, ws.tickets + i,
            epoch, nullptr);
        MPSM_TRY(check_launch("k_onesweep"));
        src_k = dk;
        src_p = dp;
    }
    return MPSM_OK;
}

// ------------------------------------------------------------ partition scatter
extern "C" int mpsm_scatter_workspace_bytes(int64_t n, int npart, size_t* bytes) {
    if (!bytes || n < 0 || npart < 1 || npart > MAX_BINS) return MPSM_ERR_ARG;
    size_t b = 0;
    b += align_up(sizeof(unsigned int) * 1);
    b += align_up(sizeof(uint64_t) * (size_t)std::max<int64_t>(num_tiles(n), 1) * npart);
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
    uint64_t* status = c.take<uint64_t>((size_t)std::max<int64_t>(num_tiles(n), 1) * npart);
    if (!c.ok) {
        set_error("scatter workspace too small");
        return MPSM_ERR_ARG;
    }
    MPSM_TRY(set_pass_smem());
    MPSM_TRY(cuda_status(cudaMemsetAsync(ticket, 0, sizeof(unsigned int), st), "memset"));
    bool wrapped = false;
    uint32_t epoch = next_epoch(&wrapped);
    if (wrapped)
        MPSM_TRY(cuda_status(cudaMemsetAsync(status, 0, sizeof(uint64_t) * (size_t)num_tiles(n) * npart, st), "memset"));
    PartitionDigit dig{lower, shift, d_sp, nbuckets};
    ProfScope ps("scatter", st);
    k_onesweep<PartitionDigit><<<(unsigned)num_tiles(n), SORT_THREADS, pass_smem_bytes(), st>>>(
        keys, pays, arena_keys, arena_pays, n, dig, npart, d_cursors, status, ticket, epoch, d_written);
    return check_launch("k_onesweep<partition>");
}
