// segsort.cu -- segmented reduce-then-scan LSD radix sort for sm_100a.
//
// The run sort of the join (replaces _kernels.three_phase_sort,
// /root/reference/pkg/src/mpsm/_kernels.py:217-244).  Per digit pass:
//
//   count    one CTA per contiguous input segment counts the segment's digits
//            (8 B read per tuple; for the first pass this sweep also checks
//            the key domain)
//   scan     per (segment, digit) base offsets: digit start + counts of the
//            same digit in earlier segments
//   scatter  the same CTA/segment pairing streams its segment tile by tile:
//            cp.async double buffering brings tile i+1 into shared memory
//            while tile i is ranked (stable, warp ballots), staged in digit
//            order and written out as coalesced runs at running per-digit
//            cursors.  No CTA waits for another: this replaces the decoupled
//            look-back of radix_sort.cu, whose latency chain held that kernel
//            to ~35 % of HBM bandwidth although the scatter write pattern
//            itself runs at 6 TB/s (tools/scatter_pattern_bench.cu).
//
// Layouts: (key, payload) pairs throughout (SS); pairs in -> packed 8-B
// records (key - lower) << pw | payload out (SP, first pass of a packed sort);
// records in and out (PP).  Packed records halve the bytes of every later
// pass and of the merge join.

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>

#include "common.cuh"

namespace mpsm {
namespace seg {

#ifndef MPSM_SEG_THREADS
#define MPSM_SEG_THREADS 512
#endif
#ifndef MPSM_SEG_ITEMS
#define MPSM_SEG_ITEMS 8
#endif
#ifndef MPSM_SEG_PP_BLOCKS
#define MPSM_SEG_PP_BLOCKS 2
#endif
constexpr int THREADS = MPSM_SEG_THREADS;
constexpr int ITEMS = MPSM_SEG_ITEMS;
constexpr int TILE = THREADS * ITEMS;  // 4096 tuples
constexpr int WARPS = THREADS / 32;
constexpr int MAX_BITS = 9;
constexpr int MAX_BINS = 1 << MAX_BITS;
constexpr int MAX_PASSES = 8;
constexpr int COUNT_UNROLL = 8;
static_assert(WARPS * MAX_BINS * 4 <= TILE * 8, "warp histograms alias one tile buffer");

enum Layout { SS = 0, SP = 1, PP = 2 };

struct Plan {
    int npasses;
    int shift[MAX_PASSES];
    int bits[MAX_PASSES];
};

static Plan make_plan(int width_bits) {
    Plan p{};
    if (width_bits <= 0) return p;
    const int np = (width_bits + MAX_BITS - 1) / MAX_BITS;
    int base = width_bits / np, rem = width_bits % np, sh = 0;
    p.npasses = np;
    for (int i = 0; i < np; ++i) {
        p.bits[i] = base + (i < rem ? 1 : 0);
        p.shift[i] = sh;
        sh += p.bits[i];
    }
    return p;
}

// digit of a key (SS/SP input) or of a record (PP input: lower = 0 and the
// shift includes the payload bits)
struct Digit {
    uint64_t lower;
    int shift;
    uint32_t mask;
    __device__ __forceinline__ uint32_t operator()(uint64_t v) const { return (uint32_t)((v - lower) >> shift) & mask; }
};

struct Segs {
    int64_t n;
    int64_t seg_len;  // multiple of TILE
    __device__ __forceinline__ int64_t begin(int g) const { return min((int64_t)g * seg_len, n); }
    __device__ __forceinline__ int64_t end(int g) const { return min((int64_t)(g + 1) * seg_len, n); }
};

// ------------------------------------------------------------------ count
// counts[g][d] for segment g; optional domain check (first pass)
__global__ void __launch_bounds__(THREADS) k_count(const uint64_t* __restrict__ in, Segs sg, Digit dig, int nbins,
                                                   uint32_t* __restrict__ counts, uint64_t span_m1,
                                                   unsigned long long* __restrict__ d_bad) {
    __shared__ uint32_t h[MAX_BINS];
    for (int i = threadIdx.x; i < MAX_BINS; i += THREADS) h[i] = 0;
    __syncthreads();
    const int64_t b = sg.begin(blockIdx.x), e = sg.end(blockIdx.x);
    constexpr int CHUNK = THREADS * COUNT_UNROLL;
    for (int64_t base = b; base < e; base += CHUNK) {
        uint64_t v[COUNT_UNROLL];
#pragma unroll
        for (int u = 0; u < COUNT_UNROLL; ++u) {
            const int64_t i = base + u * THREADS + threadIdx.x;
            v[u] = i < e ? ld_stream(in + i) : 0;
        }
#pragma unroll
        for (int u = 0; u < COUNT_UNROLL; ++u) {
            const int64_t i = base + u * THREADS + threadIdx.x;
            if (i < e) {
                if (d_bad && v[u] - dig.lower > span_m1) atomicMin(d_bad, (unsigned long long)i);
                atomicAdd(&h[dig(v[u])], 1u);
            }
        }
    }
    __syncthreads();
    for (int d = threadIdx.x; d < nbins; d += THREADS) counts[(size_t)blockIdx.x * nbins + d] = h[d];
}

// ------------------------------------------------------------------- scan
// base[g][d] = start(d) + sum_{g' < g} counts[g'][d]  (single CTA)
__global__ void __launch_bounds__(MAX_BINS) k_scan(const uint32_t* __restrict__ counts, int G, int nbins,
                                                   int64_t* __restrict__ base) {
    __shared__ int64_t tot[MAX_BINS];
    const int d = threadIdx.x;
    int64_t run = 0;
    if (d < nbins) {
        for (int g = 0; g < G; ++g) {
            const uint32_t c = counts[(size_t)g * nbins + d];
            base[(size_t)g * nbins + d] = run;
            run += c;
        }
    }
    tot[d] = run;
    __syncthreads();
    for (int off = 1; off < MAX_BINS; off <<= 1) {
        const int64_t a = d >= off ? tot[d - off] : 0;
        __syncthreads();
        tot[d] += a;
        __syncthreads();
    }
    const int64_t start = tot[d] - run;  // exclusive
    if (d < nbins)
        for (int g = 0; g < G; ++g) base[(size_t)g * nbins + d] += start;
}

// ---------------------------------------------------------------- scatter
template <int LAYOUT>
struct Smem {
    static constexpr int NARR = (LAYOUT == PP) ? 1 : 2;
    uint64_t buf[2][NARR][TILE];  // double-buffered tile data; staging in place
    uint32_t tile_off[MAX_BINS];
    int64_t gdelta[MAX_BINS];
    int64_t cur[MAX_BINS];  // running output cursor per digit of this segment
};

__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp8(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}

// async copy of cnt elements from g[0..cnt) into s[0..cnt)
__device__ __forceinline__ void tile_copy(uint64_t* s, const uint64_t* g, int cnt, bool vec) {
    if (vec) {  // g and s 16-B aligned; cnt may be odd only on the last tile
        const int pairs = cnt >> 1;
        for (int i = threadIdx.x; i < pairs; i += THREADS) cp16(s + 2 * i, g + 2 * i);
        if ((cnt & 1) && threadIdx.x == 0) cp8(s + cnt - 1, g + cnt - 1);
    } else {
        for (int i = threadIdx.x; i < cnt; i += THREADS) cp8(s + i, g + i);
    }
}

__device__ __forceinline__ unsigned ballot_peers(uint32_t d, int bits, unsigned vmask) {
#ifdef MPSM_SEG_MATCH_ANY
    return __match_any_sync(0xffffffffu, d) & vmask;
#endif
    // lanes whose digit differs from mine in some bit; bits above `bits` are
    // zero in every lane, so all MAX_BITS ballots can run unconditionally.
    // Per bit: predicate, ballot, select-complement, or -- 4 SASS ops.
    unsigned diff = ~vmask;
#pragma unroll
    for (int b = 0; b < MAX_BITS; ++b) {
        asm("{\n\t.reg .pred p;\n\t.reg .b32 t, u;\n\t"
            "and.b32 u, %1, %2;\n\t"
            "setp.ne.u32 p, u, 0;\n\t"
            "vote.sync.ballot.b32 t, p, 0xffffffff;\n\t"
            "not.b32 u, t;\n\t"
            "selp.b32 t, u, t, p;\n\t"
            "or.b32 %0, %0, t;\n\t}"
            : "+r"(diff)
            : "r"(d), "r"(1u << b));
    }
    (void)bits;
    return ~diff;
}

#ifdef MPSM_DBG_TIMING
__device__ long long g_seg_ts[1 << 22][8];
#define SEG_TS(i) \
    if (tid == 0) g_seg_ts[(t0 / TILE) & ((1 << 22) - 1)][i] = clock64();
#else
#define SEG_TS(i)
#endif

// STABLE = false ranks with one shared atomicAdd per tuple (order within a
// digit arbitrary) -- allowed for the first LSD pass only, whose input order
// carries no information.  STABLE = true ranks with warp ballots so equal
// digits keep their input order (every later pass).
template <int LAYOUT, bool STABLE>
__global__ void __launch_bounds__(THREADS, LAYOUT == PP ? MPSM_SEG_PP_BLOCKS : 1) k_scatter(
    const uint64_t* __restrict__ in_k, const uint64_t* __restrict__ in_p, uint64_t* __restrict__ out_k,
    uint64_t* __restrict__ out_p, Segs sg, Digit dig, Digit odig, int bits, int nbins,
    const int64_t* __restrict__ base, uint64_t pk_lower, int pk_pw, unsigned int* __restrict__ overflow) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem<LAYOUT>& sm = *reinterpret_cast<Smem<LAYOUT>*>(smem_raw);
    constexpr int NARR = Smem<LAYOUT>::NARR;
    constexpr int HW = STABLE ? WARPS : 1;  // histogram rows: per warp, or one per tile
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned lt = lanemask_lt();
    const int g = blockIdx.x;
    const int64_t sb = sg.begin(g), se = sg.end(g);
    if (sb >= se) return;
    const bool vec = ((((uintptr_t)in_k) | (NARR == 2 ? (uintptr_t)in_p : 0)) & 15) == 0;  // sb is a TILE multiple
    for (int d = tid; d < nbins; d += THREADS) sm.cur[d] = base[(size_t)g * nbins + d];

    auto issue = [&](int b, int64_t t0) {
        const int cnt = (int)min((int64_t)TILE, se - t0);
        tile_copy(sm.buf[b][0], in_k + t0, cnt, vec);
        if (NARR == 2) tile_copy(sm.buf[b][1], in_p + t0, cnt, vec);
    };
    issue(0, sb);
    asm volatile("cp.async.commit_group;" ::: "memory");
    int b = 0;
    for (int64_t t0 = sb; t0 < se; t0 += TILE) {
        if (t0 + TILE < se) issue(b ^ 1, t0 + TILE);
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        SEG_TS(0)
        __syncthreads();  // tile t0 is in buf[b]
        SEG_TS(1)
        const int cnt = (int)min((int64_t)TILE, se - t0);
        const bool full = cnt == TILE;

        // ---- items into registers (warp-striped)
        uint64_t key[ITEMS];
        uint32_t pos[ITEMS];
        const int wb = warp * (32 * ITEMS);
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            const int li = wb + 32 * k + lane;
            key[k] = (full || li < cnt) ? sm.buf[b][0][li] : 0;
        }
        __syncthreads();  // buf[b][0] now hosts the digit histograms [HW][MAX_BINS]
        uint32_t* hist = reinterpret_cast<uint32_t*>(sm.buf[b][0]);
        for (int i = tid; i < HW * MAX_BINS / 4; i += THREADS)
            reinterpret_cast<uint4*>(hist)[i] = make_uint4(0, 0, 0, 0);
        __syncthreads();
        if (STABLE) {
            uint32_t* wh = hist + warp * MAX_BINS;
            unsigned peers[ITEMS];
#pragma unroll
            for (int k = 0; k < ITEMS; ++k) {  // independent: the ballots pipeline
                const int li = wb + 32 * k + lane;
                const bool valid = full || li < cnt;
                const unsigned vmask = full ? 0xffffffffu : __ballot_sync(0xffffffffu, valid);
                const uint32_t d = dig(key[k]);
                peers[k] = ballot_peers(d, bits, vmask);
                if (!valid) peers[k] = 0;
                pos[k] = d << 20;
            }
#pragma unroll
            for (int k = 0; k < ITEMS; ++k) {  // running per-warp digit counts
                const uint32_t d = pos[k] >> 20;
                uint32_t before = 0;
                if (peers[k]) before = wh[d];
                __syncwarp();
                if (peers[k] && (peers[k] & lt) == 0) wh[d] = before + __popc(peers[k]);
                __syncwarp();
                pos[k] = peers[k] ? ((d << 20) | (before + __popc(peers[k] & lt))) : 0xffffffffu;
            }
        } else {
#pragma unroll
            for (int k = 0; k < ITEMS; ++k) {
                const int li = wb + 32 * k + lane;
                const uint32_t d = dig(key[k]);
                pos[k] = (full || li < cnt) ? ((d << 20) | atomicAdd(&hist[d], 1u)) : 0xffffffffu;
            }
        }
        __syncthreads();
        SEG_TS(2)
        // ---- per digit: tile count; after the digit scan the histogram rows
        // become absolute staging offsets tile_off[d] + (earlier rows' d's)
        constexpr int DPT = (MAX_BINS + THREADS - 1) / THREADS;  // digits per thread
        uint32_t mycnt[DPT];
        uint32_t col[DPT][HW];
#pragma unroll
        for (int j = 0; j < DPT; ++j) {
            const int dd = tid + j * THREADS;
            mycnt[j] = 0;
            if (dd < nbins) {
#pragma unroll
                for (int w = 0; w < HW; ++w) {
                    col[j][w] = hist[w * MAX_BINS + dd];
                    mycnt[j] += col[j][w];
                }
            }
            if (dd < MAX_BINS) sm.tile_off[dd] = mycnt[j];
        }
        __syncthreads();
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
        __syncthreads();
#pragma unroll
        for (int j = 0; j < DPT; ++j) {
            const int dd = tid + j * THREADS;
            if (dd < nbins) {
                const uint32_t toff = sm.tile_off[dd];
                uint32_t run = toff;
#pragma unroll
                for (int w = 0; w < HW; ++w) {
                    hist[w * MAX_BINS + dd] = run;
                    run += col[j][w];
                }
                sm.gdelta[dd] = sm.cur[dd] - (int64_t)toff;
                sm.cur[dd] += mycnt[j];
            }
        }
        __syncthreads();
        SEG_TS(3)
        // ---- final staging positions
#pragma unroll
        for (int k = 0; k < ITEMS; ++k)
            if (pos[k] != 0xffffffffu)
                pos[k] = hist[(STABLE ? warp : 0) * MAX_BINS + (pos[k] >> 20)] + (pos[k] & 0xfffffu);
        uint64_t pay[ITEMS];
        if (LAYOUT != PP) {
#pragma unroll
            for (int k = 0; k < ITEMS; ++k) {
                const int li = wb + 32 * k + lane;
                pay[k] = (full || li < cnt) ? sm.buf[b][1][li] : 0;
            }
        }
        if (LAYOUT == SP) {
            uint64_t ovf = 0;
            const uint64_t pmask = (1ull << pk_pw) - 1ull;
#pragma unroll
            for (int k = 0; k < ITEMS; ++k) {
                ovf |= pay[k] >> pk_pw;
                // a wider payload is masked so the key bits stay exact; the
                // caller sees *overflow and redoes the join on pairs
                key[k] = ((key[k] - pk_lower) << pk_pw) | (pay[k] & pmask);
            }
            if (__any_sync(0xffffffffu, ovf != 0) && lane == 0) atomicOr(overflow, 1u);
        }
        __syncthreads();  // histograms and tile reads done: stage in place
        SEG_TS(4)
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            if (pos[k] != 0xffffffffu) {
                sm.buf[b][0][pos[k]] = key[k];
                if (LAYOUT == SS) sm.buf[b][1][pos[k]] = pay[k];
            }
        }
        __syncthreads();
        SEG_TS(5)
#pragma unroll 4
        for (int i = tid; i < cnt; i += THREADS) {
            const uint64_t v = sm.buf[b][0][i];
            const int64_t o = sm.gdelta[odig(v)] + i;
            out_k[o] = v;
            if (LAYOUT == SS) out_p[o] = sm.buf[b][1][i];
        }
        __syncthreads();  // buf[b] free for the tile after next
        SEG_TS(6)
        b ^= 1;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// ------------------------------------------------------------------- host
struct Ws {
    uint32_t* counts;  // [G][MAX_BINS]
    int64_t* base;     // [G][MAX_BINS]
};

// one CTA per resident slot: the pair layouts (146 KB of shared memory) fit
// one CTA per SM, the record layout (82 KB) two
template <int LAYOUT>
static int grid_size() {
    static int per_sm = 0;
    if (per_sm == 0) {
        cudaFuncSetAttribute(k_scatter<LAYOUT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(Smem<LAYOUT>));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_scatter<LAYOUT, true>, THREADS, sizeof(Smem<LAYOUT>));
        if (per_sm < 1) per_sm = 1;
    }
    return num_sms() * per_sm;
}

static int max_grid() { return num_sms() * 4; }

static Segs make_segs(int64_t n, int G) {
    int64_t seg = (n + G - 1) / G;
    seg = (seg + TILE - 1) / TILE * TILE;
    if (seg == 0) seg = TILE;
    return Segs{n, seg};
}

static size_t ws_bytes() {
    const int G = max_grid();
    return align_up(sizeof(uint32_t) * (size_t)G * MAX_BINS) + align_up(sizeof(int64_t) * (size_t)G * MAX_BINS);
}

static bool carve(void* ws, size_t bytes, Ws* o) {
    Carve c{(char*)ws, bytes};
    const int G = max_grid();
    o->counts = c.take<uint32_t>((size_t)G * MAX_BINS);
    o->base = c.take<int64_t>((size_t)G * MAX_BINS);
    return c.ok;
}

template <int LAYOUT, bool STABLE>
static int set_attr() {
    static bool done = false;
    if (!done) {
        MPSM_TRY(cuda_status(cudaFuncSetAttribute(k_scatter<LAYOUT, STABLE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)sizeof(Smem<LAYOUT>)),
                             "smem attr"));
        done = true;
    }
    return MPSM_OK;
}

// one digit pass: count, scan, scatter
template <int LAYOUT, bool STABLE>
static int pass(const uint64_t* in_k, const uint64_t* in_p, uint64_t* out_k, uint64_t* out_p, int64_t n,
                Digit count_dig, Digit dig, int bits, const Ws& ws, uint64_t span_m1, unsigned long long* d_bad,
                uint64_t pk_lower, int pk_pw, unsigned int* overflow, cudaStream_t st) {
    const int G = std::min(grid_size<LAYOUT>(), max_grid());
    const Segs sg = make_segs(n, G);
    const int nbins = 1 << bits;
    {
        ProfScope ps("seg_count", st);
        k_count<<<G, THREADS, 0, st>>>(in_k, sg, count_dig, nbins, ws.counts, span_m1, d_bad);
    }
    MPSM_TRY(check_launch("k_count"));
    k_scan<<<1, MAX_BINS, 0, st>>>(ws.counts, G, nbins, ws.base);
    MPSM_TRY(check_launch("k_scan"));
    MPSM_TRY((set_attr<LAYOUT, STABLE>()));
    {
        ProfScope ps("seg_scatter", st);
        ProfScope ps2(LAYOUT == SS ? "seg_scatter_ss" : (LAYOUT == SP ? "seg_scatter_sp" : "seg_scatter_pp"), st);
        // digit of a staged value: records staged by the SP pass carry the key
        // above the payload bits
        const Digit odig = (LAYOUT == SP) ? Digit{0, pk_pw + dig.shift, dig.mask} : dig;
        k_scatter<LAYOUT, STABLE><<<G, THREADS, sizeof(Smem<LAYOUT>), st>>>(in_k, in_p, out_k, out_p, sg, dig, odig, bits,
                                                                    nbins, ws.base, pk_lower, pk_pw, overflow);
    }
    return check_launch("k_scatter");
}

}  // namespace seg
}  // namespace mpsm

using namespace mpsm;

#ifdef MPSM_DBG_TIMING
extern "C" int mpsm_dbg_seg_ts(long long* host, int ntiles) {
    return cuda_status(cudaMemcpyFromSymbol(host, seg::g_seg_ts, sizeof(long long) * 8 * (size_t)ntiles), "dbg");
}
#endif

extern "C" int mpsm_sort_pass_count(int width_bits) { return seg::make_plan(width_bits).npasses; }

extern "C" int mpsm_sort_workspace_bytes(int64_t n, int width_bits, size_t* bytes) {
    if (!bytes || n < 0 || width_bits < 0 || width_bits > 64) return MPSM_ERR_ARG;
    *bytes = seg::ws_bytes();
    return MPSM_OK;
}

extern "C" int mpsm_sort_pairs(const uint64_t* in_keys, const uint64_t* in_pays, int64_t n, uint64_t lower,
                               uint64_t span_m1, int width_bits, uint64_t* out_keys, uint64_t* out_pays,
                               uint64_t* tmp_keys, uint64_t* tmp_pays, void* workspace, size_t ws_bytes,
                               unsigned long long* d_bad, void* stream) {
    using namespace seg;
    cudaStream_t st = (cudaStream_t)stream;
    if (n < 0 || width_bits < 0 || width_bits > 64) return MPSM_ERR_ARG;
    if (n == 0) return MPSM_OK;
    Ws ws;
    if (!carve(workspace, ws_bytes, &ws)) {
        set_error("sort workspace too small");
        return MPSM_ERR_ARG;
    }
    const Plan plan = make_plan(width_bits);
    if (plan.npasses == 0) {  // one-value domain: check it and copy
        const int G = max_grid();
        k_count<<<G, THREADS, 0, st>>>(in_keys, make_segs(n, G), Digit{lower, 0, 0}, 1, ws.counts, span_m1, d_bad);
        MPSM_TRY(check_launch("k_count"));
        if (out_keys != in_keys) {
            MPSM_TRY(cuda_status(cudaMemcpyAsync(out_keys, in_keys, 8 * n, cudaMemcpyDeviceToDevice, st), "copy"));
            MPSM_TRY(cuda_status(cudaMemcpyAsync(out_pays, in_pays, 8 * n, cudaMemcpyDeviceToDevice, st), "copy"));
        }
        return MPSM_OK;
    }
    const int P = plan.npasses;
    const uint64_t *sk = in_keys, *sp = in_pays;
    if (in_keys == out_keys && (P % 2 == 1)) {
        // the first pass may not write its own input: start from a copy
        MPSM_TRY(cuda_status(cudaMemcpyAsync(tmp_keys, in_keys, 8 * n, cudaMemcpyDeviceToDevice, st), "copy"));
        MPSM_TRY(cuda_status(cudaMemcpyAsync(tmp_pays, in_pays, 8 * n, cudaMemcpyDeviceToDevice, st), "copy"));
        sk = tmp_keys;
        sp = tmp_pays;
    }
    for (int i = 0; i < P; ++i) {
        const bool to_out = ((P - 1 - i) % 2) == 0;
        uint64_t* dk = to_out ? out_keys : tmp_keys;
        uint64_t* dp = to_out ? out_pays : tmp_pays;
        const Digit dg{lower, plan.shift[i], (1u << plan.bits[i]) - 1u};
        // the first LSD pass may reorder equal digits; later passes must not
        if (i == 0)
            MPSM_TRY((pass<SS, false>(sk, sp, dk, dp, n, dg, dg, plan.bits[i], ws, span_m1, d_bad, 0, 0, nullptr, st)));
        else
            MPSM_TRY((pass<SS, true>(sk, sp, dk, dp, n, dg, dg, plan.bits[i], ws, ~0ull, nullptr, 0, 0, nullptr, st)));
        sk = dk;
        sp = dp;
    }
    return MPSM_OK;
}

extern "C" int mpsm_sort_packed(const uint64_t* in_keys, const uint64_t* in_pays, int64_t n, uint64_t lower,
                                uint64_t span_m1, int width_bits, uint64_t* out_rec, uint64_t* tmp_rec, void* workspace,
                                size_t ws_bytes, unsigned long long* d_bad, unsigned int* d_overflow, void* stream) {
    using namespace seg;
    cudaStream_t st = (cudaStream_t)stream;
    if (n < 0 || width_bits < 1 || width_bits > 63 || !d_overflow) return MPSM_ERR_ARG;
    if (n == 0) return MPSM_OK;
    Ws ws;
    if (!carve(workspace, ws_bytes, &ws)) {
        set_error("sort workspace too small");
        return MPSM_ERR_ARG;
    }
    const Plan plan = make_plan(width_bits);
    const int pw = 64 - width_bits;
    const int P = plan.npasses;
    const uint64_t* src = nullptr;
    for (int i = 0; i < P; ++i) {
        uint64_t* dst = ((P - 1 - i) % 2 == 0) ? out_rec : tmp_rec;
        if (i == 0) {
            const Digit dg{lower, plan.shift[0], (1u << plan.bits[0]) - 1u};
            MPSM_TRY((pass<SP, false>(in_keys, in_pays, dst, nullptr, n, dg, dg, plan.bits[0], ws, span_m1, d_bad,
                                      lower, pw, d_overflow, st)));
        } else {
            const Digit dg{0, pw + plan.shift[i], (1u << plan.bits[i]) - 1u};
            MPSM_TRY((pass<PP, true>(src, nullptr, dst, nullptr, n, dg, dg, plan.bits[i], ws, ~0ull, nullptr, 0, pw,
                                     nullptr, st)));
        }
        src = dst;
    }
    return MPSM_OK;
}
