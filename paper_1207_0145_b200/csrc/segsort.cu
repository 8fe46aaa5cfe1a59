// segsort.cu -- reduce-then-scan LSD radix sort for sm_100a.
//
// The run sort of the join (replaces _kernels.three_phase_sort,
// /root/reference/pkg/src/mpsm/_kernels.py:217-244).  Digits of <= 9 bits;
// per digit pass:
//
//   count    one CTA per contiguous input segment (4 per SM) counts the
//            digits of every scatter tile of its segment and writes each
//            tile's segment-local digit prefixes (8 B read per tuple; the
//            first pass also checks the key domain)
//   scan     per (segment, digit) base offsets and digit totals
//   scatter  persistent CTAs take tiles IN GLOBAL ORDER from an atomic tile
//            dispenser, so tiles in flight are neighbours and their runs of
//            one digit land next to each other (per-CTA segments halved the
//            write bandwidth, tools/scatter_pattern_bench.cu).  Thread 0
//            brings tile i+1 (tuples + digit prefixes) into shared memory with
//            TMA bulk copies while tile i is ranked -- one shared atomicAdd
//            per tuple into per-warp 16-bit histogram rows gives a stable
//            rank (lane-ordered atomics, probed at start-up per device;
//            warp-ballot fallback) -- scanned, staged in digit order in place
//            and written out in coalesced runs.  No CTA waits for another
//            (the decoupled look-back of the first design held its kernel to
//            ~35 % of HBM; the partition scatter of the reference's arena,
//            mpsm_scatter_chunk, is now this pass with the partition as digit
//            and the worker's cursors as digit starts).
//
// One call sorts one array, or (multi-segment, Segs::nseg > 0) up to 1024
// independent segments of it in the same launches -- the T runs of a join.
//
// Layouts: (key, payload) pairs throughout (SS); pairs in -> packed 8-B
// records (key - lower) << pw | payload out (SP, first pass of a packed sort);
// records in and out (PP, 8192-tuple tiles).  Packed records halve the bytes
// of every later pass and of the merge join.

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <string>

#include "common.cuh"

namespace mpsm {
namespace seg {

#ifndef MPSM_SEG_THREADS
#define MPSM_SEG_THREADS 512
#endif
#ifndef MPSM_SEG_ITEMS
#define MPSM_SEG_ITEMS 8
#endif
#ifndef MPSM_SEG_COUNT_PER_SM  // count CTAs (segments) per SM
#define MPSM_SEG_COUNT_PER_SM 4
#endif
#ifndef MPSM_SEG_PP_BLOCKS  // record-pass scatter CTAs per SM
#define MPSM_SEG_PP_BLOCKS 1
#endif
#ifndef MPSM_SEG_PP_ITEMS  // record-pass tuples per thread per tile
#define MPSM_SEG_PP_ITEMS 16
#endif
#ifndef MPSM_SEG_PP_STAGES  // record-pass tile buffers in shared memory
#define MPSM_SEG_PP_STAGES 2
#endif
#ifndef MPSM_SEG_STAGES  // pair-input (SS / SP) tile buffers in shared memory
#define MPSM_SEG_STAGES 2
#endif
constexpr int THREADS = MPSM_SEG_THREADS;
constexpr int ITEMS = MPSM_SEG_ITEMS;
constexpr int TILE = THREADS * ITEMS;  // 4096 tuples: the count chunk and the smallest scatter tile
constexpr int WARPS = THREADS / 32;
constexpr int MAX_BITS = 9;
constexpr int MAX_BINS = 1 << MAX_BITS;
constexpr int MAX_PASSES = 8;

enum Layout { SS = 0, SP = 1, PP = 2 };

// per-layout scatter shape: tuples per thread, tile, tile buffers, CTAs/SM
template <int LAYOUT>
struct LCfg {
    static constexpr int ITEMS_L = LAYOUT == PP ? MPSM_SEG_PP_ITEMS : ITEMS;
    static constexpr int TILE_L = THREADS * ITEMS_L;
    static constexpr int NST = LAYOUT == PP ? MPSM_SEG_PP_STAGES : MPSM_SEG_STAGES;
    static constexpr int BLOCKS = LAYOUT == PP ? MPSM_SEG_PP_BLOCKS : 1;
    static_assert(TILE_L % TILE == 0, "scatter tiles are whole count chunks");
};

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
    // partition passes (TABLE kernels): digit = table[min(bucket, nbuckets - 1)]
    // with bucket = (v - lower) >> shift -- the splitter vector of P-MPSM
    const int32_t* table = nullptr;
    int nbuckets = 0;
    __device__ __forceinline__ uint32_t operator()(uint64_t v) const { return (uint32_t)((v - lower) >> shift) & mask; }
    __device__ __forceinline__ uint32_t lookup(uint64_t v) const {
        uint64_t b = (v - lower) >> shift;
        if (b >= (uint64_t)nbuckets) b = (uint64_t)nbuckets - 1;
        return (uint32_t)__ldg(table + b);
    }
};

// Tile geometry of one pass.  Single mode (nseg == 0): one sort over n
// elements, count CTA g covers [g * seg_len, (g + 1) * seg_len), scatter tile
// t starts at t * TL.  Multi mode (nseg > 0): nseg independent sorts of the
// element ranges [off[s], off[s+1]) in one launch sequence (the T public
// chunks of a join); scatter tiles never straddle a segment (tile t of
// segment s starts at off[s] + (t - tb[s]) * TL), count CTA g covers the
// tiles [tb[s] + (g - gb[s]) * tpc, ...) of its segment s.
struct Segs {
    int64_t n;
    int64_t seg_len;  // single mode: multiple of the scatter tile
    int nseg = 0;
    const int64_t* off = nullptr;  // [nseg + 1] element offsets
    const int64_t* tb = nullptr;   // [nseg + 1] first scatter tile of each segment
    const int64_t* gb = nullptr;   // [nseg + 1] first count CTA of each segment
    int64_t tpc = 0;               // scatter tiles per count CTA
    // single mode: explicit output start of each digit (the partition
    // scatter's cursors) instead of the exclusive scan of the digit totals
    const int64_t* dbase = nullptr;
    __device__ __forceinline__ int seg_of(const int64_t* starts, int64_t x) const {  // last s with starts[s] <= x
        int lo = 0, hi = nseg - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (starts[mid] <= x) lo = mid;
            else hi = mid - 1;
        }
        return lo;
    }
    // count CTA g -> its element range [b, e) and first scatter tile
    __device__ __forceinline__ void cta(int g, int64_t TL, int64_t& b, int64_t& e, int64_t& t0) const {
        if (nseg == 0) {
            b = min((int64_t)g * seg_len, n);
            e = min((int64_t)(g + 1) * seg_len, n);
            t0 = b / TL;
            return;
        }
        if (g >= gb[nseg]) {  // launched for the bound, not needed
            b = e = t0 = 0;
            return;
        }
        const int s = seg_of(gb, g);
        t0 = tb[s] + (int64_t)(g - gb[s]) * tpc;
        const int64_t t1 = min(t0 + tpc, tb[s + 1]);
        b = off[s] + (t0 - tb[s]) * TL;
        e = min(off[s] + (t1 - tb[s]) * TL, off[s + 1]);
        if (t0 >= t1) e = b;
    }
    // scatter tile t -> element start, count, count CTA
    __device__ __forceinline__ void tile(int64_t t, int64_t TL, int64_t& start, int& cnt, int64_t& g) const {
        if (nseg == 0) {
            start = t * TL;
            cnt = (int)min(TL, n - start);
            g = t / (seg_len / TL);
            return;
        }
        const int s = seg_of(tb, t);
        start = off[s] + (t - tb[s]) * TL;
        cnt = (int)min(TL, off[s + 1] - start);
        g = gb[s] + (t - tb[s]) / tpc;
    }
    __device__ __forceinline__ int64_t ntiles(int64_t TL) const { return nseg == 0 ? (n + TL - 1) / TL : tb[nseg]; }
};

// Segs::tile for one thread that asks for increasing tiles (the tile
// fetcher of a scatter CTA): the current segment's geometry stays in
// registers, so a fetch costs no dependent loads unless the segment changes
struct SegCursor {
    int s = -1;
    int64_t tb0 = 0, tb1 = 0, off0 = 0, off1 = 0, gb0 = 0;
    __device__ __forceinline__ void tile(const Segs& sg, int64_t t, int64_t TL, int64_t& start, int& cnt, int64_t& g) {
        if (sg.nseg == 0) {
            sg.tile(t, TL, start, cnt, g);
            return;
        }
        if (s < 0 || t < tb0 || t >= tb1) {
            s = (s >= 0 && t >= tb1 && t < sg.tb[s + 2 <= sg.nseg ? s + 2 : sg.nseg]) ? s + 1 : sg.seg_of(sg.tb, t);
            tb0 = sg.tb[s];
            tb1 = sg.tb[s + 1];
            off0 = sg.off[s];
            off1 = sg.off[s + 1];
            gb0 = sg.gb[s];
        }
        start = off0 + (t - tb0) * TL;
        cnt = (int)min(TL, off1 - start);
        g = gb0 + (t - tb0) / sg.tpc;
    }
};

// ------------------------------------------------------------------ count
// counts[g][d] for segment g, and for every tile t of the segment the
// segment-local exclusive prefix toffs[t][d] (digit d's tuples in earlier
// tiles of the segment); optional domain check (first pass)
#ifndef MPSM_SEG_COUNT_TPS  // one-chunk scatter tiles (SP / SS passes) whose prefixes one barrier flushes
#define MPSM_SEG_COUNT_TPS 1
#endif
template <int CPT, bool TABLE = false, bool MSEG = false>  // count chunks (TILE tuples) per scatter tile
__global__ void __launch_bounds__(THREADS, 2) k_count(const uint64_t* __restrict__ in, Segs sg, Digit dig, int nbins,
                                                   uint32_t* __restrict__ counts, uint32_t* __restrict__ toffs,
                                                   unsigned int* __restrict__ ticket, uint64_t span_m1,
                                                   unsigned long long* __restrict__ d_bad) {
    constexpr int STILE = CPT * TILE;
    // TPS scatter tiles are counted per barrier (each into its own row);
    // flush group g counts into h[g & 1], so one barrier per group suffices
    constexpr int TPS = CPT == 1 ? MPSM_SEG_COUNT_TPS : 1;
    __shared__ uint32_t h[2][TPS][MAX_BINS];
    const int tid = threadIdx.x;
#pragma unroll
    for (int j = 0; j < TPS; ++j) h[0][j][tid] = h[1][j][tid] = 0;
    if (blockIdx.x == 0 && tid == 0 && ticket) *ticket = 0;  // the scatter's tile dispenser
    __syncthreads();
    int64_t b, e, tfirst;
    if (MSEG) {
        sg.cta(blockIdx.x, STILE, b, e, tfirst);
    } else {
        b = min((int64_t)blockIdx.x * sg.seg_len, sg.n);
        e = min((int64_t)(blockIdx.x + 1) * sg.seg_len, sg.n);
        tfirst = b / STILE;
    }
    uint32_t run = 0;  // thread d: digit d's count in the tiles so far
    uint64_t v[ITEMS], w[ITEMS];
    // element u of a thread's chunk share: pairs of neighbours moved with
    // 16-B loads when the CTA's range is 16-B aligned (chunks are TILE apart),
    // else single elements
    const bool vec = ((uintptr_t)(in + b) & 15) == 0;
    auto pos = [&](int64_t c0, int u) -> int64_t {
        return vec ? c0 + 2 * ((u >> 1) * THREADS + tid) + (u & 1) : c0 + u * THREADS + tid;
    };
    auto load = [&](uint64_t* x, int64_t c0) {
        if (vec && c0 + TILE <= e) {
#pragma unroll
            for (int u = 0; u < ITEMS; u += 2) {
                const ulonglong2 q = __ldcs(reinterpret_cast<const ulonglong2*>(in + pos(c0, u)));
                x[u] = q.x;
                x[u + 1] = q.y;
            }
        } else {
#pragma unroll
            for (int u = 0; u < ITEMS; ++u) {
                const int64_t i = pos(c0, u);
                x[u] = i < e ? ld_stream(in + i) : 0;
            }
        }
    };
    if (b < e) load(v, b);
    int k = 0, c = 0, q = 0;  // buffer, chunk within the tile, tile within the flush group
    int64_t ts[TPS];          // first element of each tile of the group
    // the histograms' shared address in a register (through the array ptxas
    // re-reads the CTA's shared window base, S2UR CgaCtaId, per atomic)
    uint32_t hbase;
    asm volatile("mov.u32 %0, %1;" : "=r"(hbase) : "r"(smem_addr(&h[0][0][0])));
    auto bump = [&](uint32_t row, uint32_t d) {
        asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(hbase + 4u * (row * MAX_BINS + d)) : "memory");
    };
    for (int64_t c0 = b; c0 < e; c0 += TILE) {
        if (c0 + TILE < e) load(w, c0 + TILE);  // next chunk in flight during this one
        const uint32_t row = (uint32_t)(k * TPS + (TPS == 1 ? 0 : q));
        if (c0 + TILE <= e) {  // a whole chunk: no per-item index guards
            uint64_t viol = 0;  // first pass: any key outside the domain (rare: then the exact index below)
#pragma unroll
            for (int u = 0; u < ITEMS; ++u) {
                if (d_bad) viol |= (uint64_t)(v[u] - dig.lower > span_m1);
                bump(row, TABLE ? dig.lookup(v[u]) : dig(v[u]));
            }
            if (viol) {
#pragma unroll
                for (int u = 0; u < ITEMS; ++u)
                    if (v[u] - dig.lower > span_m1) atomicMin(d_bad, (unsigned long long)pos(c0, u));
            }
        } else {
#pragma unroll
            for (int u = 0; u < ITEMS; ++u) {
                const int64_t i = pos(c0, u);
                if (i < e) {
                    if (d_bad && v[u] - dig.lower > span_m1) atomicMin(d_bad, (unsigned long long)i);
                    bump(row, TABLE ? dig.lookup(v[u]) : dig(v[u]));
                }
            }
        }
#pragma unroll
        for (int u = 0; u < ITEMS; ++u) v[u] = w[u];
        const bool last = c0 + TILE >= e;
        if (++c < CPT && !last) continue;
        ts[TPS == 1 ? 0 : q] = c0 - (c - 1) * TILE;  // this scatter tile's first element
        c = 0;
        if (++q < TPS && !last) continue;
        __syncthreads();  // h[k] complete; the next group counts into h[k ^ 1]
#pragma unroll
        for (int j = 0; j < TPS; ++j) {
            if (j < q) {
                if (tid < nbins)
                    toffs[(size_t)(MSEG ? tfirst + (ts[j] - b) / STILE : ts[j] / STILE) * MAX_BINS + tid] = run;
                run += h[k][j][tid];
                h[k][j][tid] = 0;
            }
        }
        k ^= 1;
        q = 0;
    }
    if (tid < nbins) counts[(size_t)blockIdx.x * nbins + tid] = run;
}

// ------------------------------------------------------------------- scan
// base[g][d] = sum_{g' < g} counts[g'][d] (segment-relative to digit d's
// start) and dtot[d] = digit d's total.  One CTA per 32 digits; thread
// (row group r, digit lane) sums its group of segments, the groups are
// scanned through shared memory.
constexpr int SCAN_GROUPS = 32;

__global__ void __launch_bounds__(32 * SCAN_GROUPS) k_scan(const uint32_t* __restrict__ counts, int G, int nbins,
                                                         int64_t* __restrict__ base, int64_t* __restrict__ dtot) {
    __shared__ int64_t part[SCAN_GROUPS][33];
    const int dl = threadIdx.x & 31, r = threadIdx.x >> 5;
    const int d = blockIdx.x * 32 + dl;
    const int rpg = (G + SCAN_GROUPS - 1) / SCAN_GROUPS;
    const int g0 = r * rpg, g1 = min(g0 + rpg, G);
    const bool mine = d < nbins;
    int64_t sum = 0;
#pragma unroll 8
    for (int g = g0; g < g1; ++g) sum += mine ? counts[(size_t)g * nbins + d] : 0;
    part[r][dl] = sum;
    __syncthreads();
    int64_t run = 0;
    for (int q = 0; q < r; ++q) run += part[q][dl];
    if (!mine) return;
    if (r == SCAN_GROUPS - 1) dtot[d] = run + sum;
#pragma unroll 8
    for (int g = g0; g < g1; ++g) {  // second read hits L2
        const uint32_t c = counts[(size_t)g * nbins + d];
        base[(size_t)g * nbins + d] = run;
        run += c;
    }
}

// multi-segment sorts: one CTA per sort segment s, thread d per digit.
// base[g][d] = off[s] + (digit d's start inside segment s) + sum over the
// segment's earlier count CTAs g' of counts[g'][d] -- the whole output offset
// of the first digit-d tuple of count CTA g (the scatter adds the tile's
// prefix and the in-tile rank)
__global__ void __launch_bounds__(MAX_BINS) k_scan_mseg(const uint32_t* __restrict__ counts, Segs sg, int nbins,
                                                        int64_t* __restrict__ base) {
    __shared__ int64_t wsum[MAX_BINS / 32];
    const int s = blockIdx.x, d = threadIdx.x, lane = d & 31, warp = d >> 5;
    const int64_t g0 = sg.gb[s], g1 = sg.gb[s + 1];
    const bool mine = d < nbins;
    int64_t tot = 0;
#pragma unroll 16
    for (int64_t g = g0; g < g1; ++g) tot += mine ? counts[(size_t)g * nbins + d] : 0;
    int64_t incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int64_t run = sg.off[s] + incl - tot;
    for (int w = 0; w < warp; ++w) run += wsum[w];
    if (!mine) return;
#pragma unroll 16
    for (int64_t g = g0; g < g1; ++g) {  // second read hits L2
        const uint32_t c = counts[(size_t)g * nbins + d];
        base[(size_t)g * nbins + d] = run;
        run += c;
    }
}

// multi-segment geometry of one pass (tile TL, tpc scatter tiles per count
// CTA): tb / gb from off (one CTA, nseg <= MAX_SEGS); count CTAs past gb[nseg]
// get empty ranges (Segs::cta)
constexpr int MAX_SEGS = 1024;
__global__ void __launch_bounds__(MAX_SEGS) k_seg_geom(const int64_t* __restrict__ off, int nseg, int64_t TL,
                                                       int64_t tpc, int64_t* __restrict__ tb,
                                                       int64_t* __restrict__ gb) {
    __shared__ int64_t s_nt[MAX_SEGS], s_ng[MAX_SEGS];
    const int s = threadIdx.x;
    int64_t nt = 0, ng = 0;
    if (s < nseg) {
        nt = (off[s + 1] - off[s] + TL - 1) / TL;
        ng = (nt + tpc - 1) / tpc;
    }
    s_nt[s] = nt;
    s_ng[s] = ng;
    __syncthreads();
    for (int o = 1; o < MAX_SEGS; o <<= 1) {  // inclusive scans
        const int64_t a = s >= o ? s_nt[s - o] : 0, b = s >= o ? s_ng[s - o] : 0;
        __syncthreads();
        s_nt[s] += a;
        s_ng[s] += b;
        __syncthreads();
    }
    if (s < nseg) {
        tb[s + 1] = s_nt[s];
        gb[s + 1] = s_ng[s];
    }
    if (s == 0) tb[0] = gb[0] = 0;
}

// ---------------------------------------------------------------- scatter
// Shared memory of one scatter CTA.  The digit histogram of a tile keeps one
// row per warp, two warps per 32-bit word (16-bit fields: a warp counts at
// most 32 * ITEMS = 256 tuples per digit, a tile offset is < TILE).
template <int LAYOUT>
struct Smem {
    static constexpr int NARR = (LAYOUT == PP) ? 1 : 2;
    static constexpr int TL = LCfg<LAYOUT>::TILE_L, NST = LCfg<LAYOUT>::NST;
    uint64_t buf[NST][NARR][TL + 2];     // tile buffers (+1 slot of alignment shift); staging in place
    uint32_t hist[WARPS / 2][MAX_BINS];  // [warp pair][digit]
    int64_t gdelta[MAX_BINS];            // output index - staging index, per digit
    uint32_t toffs[NST][MAX_BINS];       // per buffer: the tile's segment-local digit prefixes
    uint32_t wtot[WARPS];                // digit-scan carries
    int64_t tile[NST];                   // per buffer: tile index
    int64_t tstart[NST], tg[NST];        // per buffer: first element, count CTA (Segs::tile)
    int tcnt[NST], toffk[NST], toffp[NST];  // per buffer: tuples, alignment slots of the key / payload copies
    uint64_t bar[NST];                   // bulk-copy completion, per buffer
};
static_assert(THREADS == MAX_BINS, "the digit scan gives each thread one digit");
static_assert(ITEMS % 2 == 0, "count loads element pairs");
static_assert(WARPS % 2 == 0 && WARPS <= 32, "two warps per histogram word");

// lanes of the warp holding the same digit (fallback ranking: 9 ballots)
__device__ __forceinline__ unsigned ballot_peers(uint32_t d, unsigned vmask) {
    // lanes whose digit differs from mine in some bit; bits above a pass's
    // width are zero in every lane, so all MAX_BITS ballots run unconditionally
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
    return ~diff;
}

// element i of a tile of array g sits at s[off + i], off = (g / 8) & 1, so
// that global and shared addresses agree mod 16 and the 16-B aligned body
// moves with one bulk copy; an unaligned head/tail element is copied by the
// issuing thread itself.  Returns the bulk bytes.
__device__ __forceinline__ unsigned tile_plain(uint64_t* s, const uint64_t* g, int off, int cnt) {
    const int nb = (cnt - off) >> 1;
    if (off) s[1] = g[0];
    if (off + 2 * nb < cnt) s[off + cnt - 1] = g[cnt - 1];
    return 16u * nb;
}
__device__ __forceinline__ void tile_bulk(uint64_t* s, const uint64_t* g, int off, unsigned bytes, uint64_t* bar) {
    if (bytes) bulk_load(s + 2 * off, g + off, bytes, bar);
}

#ifdef MPSM_DBG_TIMING
__device__ long long g_seg_ts[1 << 22][8];
#define SEG_TS(i) \
    if (tid == 0) g_seg_ts[t & ((1 << 22) - 1)][i] = clock64();
#define WS_TS(who, tt, i) \
    if (tid == (who)) g_seg_ts[(tt) & ((1 << 22) - 1)][i] = clock64();
#else
#define SEG_TS(i)
#define WS_TS(who, tt, i)
#endif

// digit of a record whose key bits start at or above bit 32 (HI) -- one
// shift of the high word
template <bool HI>
__device__ __forceinline__ uint32_t rec_digit(uint64_t v, const Digit& d) {
    if (HI) return ((uint32_t)(v >> 32) >> (d.shift - 32)) & d.mask;
    return (uint32_t)(v >> d.shift) & d.mask;
}

// One persistent CTA per segment.  Per tile, five barriers:
//   S1 previous tile written out: thread 0 launches the bulk copy of the
//      next tile; all wait for this tile's copy, load items into
//      registers and rank them -- a stable rank within the warp's row
//   S2 histograms complete: thread d scans digit d over the warp rows and
//      the digits (block scan)
//   S3 carries of the digit scan published
//   S4 rows hold staging offsets: stage items in digit order in place
//   S5 staged: clear the histogram, stream the tile out in coalesced runs
// Ranking: lanes of a warp that add to one shared address in one atomicAdd
// instruction receive consecutive counts in lane order (sm_100; probed once
// per process by lane_ordered_atomics()), items of a warp go in program
// order and warps in row order, so one ATOMS per tuple gives a stable rank.
// Where the probe fails the peers come from ballots (ballot_peers).
// HI: the staged records' digit lies in the high word (PP/SP with pw >= 32).
template <int LAYOUT, bool HI, bool TABLE = false>
__global__ void __launch_bounds__(THREADS, LCfg<LAYOUT>::BLOCKS) k_scatter(
    const uint64_t* __restrict__ in_k, const uint64_t* __restrict__ in_p, uint64_t* __restrict__ out_k,
    uint64_t* __restrict__ out_p, Segs sg, Digit dig, Digit odig, int nbins, const int64_t* __restrict__ base,
    const uint32_t* __restrict__ toffs, const int64_t* __restrict__ dtot, unsigned int* __restrict__ ticket,
    uint64_t pk_lower, int pk_pw, unsigned int* __restrict__ overflow, bool lane_ordered) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem<LAYOUT>& sm = *reinterpret_cast<Smem<LAYOUT>*>(smem_raw);
    constexpr int NARR = Smem<LAYOUT>::NARR;
    constexpr int ROWS = WARPS / 2;
    constexpr int IT = LCfg<LAYOUT>::ITEMS_L, TL = LCfg<LAYOUT>::TILE_L, NST = LCfg<LAYOUT>::NST;
    static_assert(32 * IT < 65536 && TL < 65536, "16-bit histogram fields");
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned lt = lanemask_lt();
    const int64_t T = sg.ntiles(TL);
    if ((int64_t)blockIdx.x >= T) return;
    const bool mine = tid < nbins;  // the digit this thread scans
    uint32_t* hrow = sm.hist[warp >> 1];
    const uint32_t inc = (warp & 1) ? 0x10000u : 1u;
    const uint32_t half = (warp & 1) ? 0x4432u : 0x4410u;  // byte_perm: my 16-bit field
    for (int i = tid; i < ROWS * MAX_BINS / 4; i += THREADS)
        reinterpret_cast<uint4*>(&sm.hist[0][0])[i] = make_uint4(0, 0, 0, 0);
    // start of my digit's output region: exclusive scan of the digit totals
    // (multi-segment sorts: the scan kernel folded it into base)
    int64_t dstart = 0;
    if (sg.dbase) {
        dstart = mine ? sg.dbase[tid] : 0;
    } else if (sg.nseg == 0) {
        const int64_t v = mine ? dtot[tid] : 0;
        int64_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        if (lane == 31) sm.gdelta[warp] = incl;  // gdelta is free until the first tile
        __syncthreads();
        dstart = incl - v;
        for (int w = 0; w < warp; ++w) dstart += sm.gdelta[w];
    }

    // thread 0: one mbarrier phase brings tile t's tuples and its digit
    // prefixes into buffer bb
    SegCursor cur;  // the fetching thread's
    auto fetch = [&](int bb, int64_t t) {
        int64_t t0, g;
        int cnt;
        cur.tile(sg, t, TL, t0, cnt, g);
        const int offk = (int)(((uintptr_t)(in_k + t0) >> 3) & 1);
        const int offp = NARR == 2 ? (int)(((uintptr_t)(in_p + t0) >> 3) & 1) : 0;
        sm.tile[bb] = t;
        sm.tstart[bb] = t0;
        sm.tg[bb] = g;
        sm.tcnt[bb] = cnt;
        sm.toffk[bb] = offk;
        sm.toffp[bb] = offp;
        unsigned bk = tile_plain(sm.buf[bb][0], in_k + t0, offk, cnt), bp = 0;
        if (NARR == 2) bp = tile_plain(sm.buf[bb][NARR - 1], in_p + t0, offp, cnt);
        const unsigned bo = MAX_BINS * 4;
        mbar_arrive_expect_tx(&sm.bar[bb], bk + bp + bo);
        tile_bulk(sm.buf[bb][0], in_k + t0, offk, bk, &sm.bar[bb]);
        if (NARR == 2) tile_bulk(sm.buf[bb][NARR - 1], in_p + t0, offp, bp, &sm.bar[bb]);
        bulk_load(sm.toffs[bb], toffs + (size_t)t * MAX_BINS, bo, &sm.bar[bb]);
    };
    // tiles in global order: each CTA starts at tile blockIdx.x, later tiles
    // come from a dispenser in order, so the tiles in flight at any moment
    // are neighbours and their runs of one digit land next to each other in
    // the output (a CTA sweeping its own contiguous segment instead halves
    // the write bandwidth: tools/scatter_pattern_bench.cu)
    int64_t tnext = 0;  // thread 0: the next tile to fetch (ticket taken a tile earlier)
    if (tid == 0) {
        for (int q = 0; q < NST; ++q) mbar_init(&sm.bar[q], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fetch(0, blockIdx.x);
        for (int q = 1; q < NST - 1; ++q) {
            const int64_t tq = (int64_t)gridDim.x + atomicAdd(ticket, 1u);
            if (tq < T) fetch(q, tq);
            else sm.tile[q] = T;
        }
        tnext = (int64_t)gridDim.x + atomicAdd(ticket, 1u);
    }
    unsigned par = 0;
    int b = 0;
    for (;;) {
        __syncthreads();  // S1
        const int64_t t = sm.tile[b];  // set by thread 0 before S1
        if (t >= T) break;
        SEG_TS(0)
        if (NST > 1 && tid == 0) {
            const int nb = (b + NST - 1) % NST;  // the buffer of the previous tile
            if (tnext < T) {
                fence_proxy_async_smem();  // buf[nb] was staged through by generic stores
                fetch(nb, tnext);
                tnext = (int64_t)gridDim.x + atomicAdd(ticket, 1u);  // used one tile later
            } else {
                sm.tile[nb] = T;  // no more tiles
            }
        }
        // my digit's segment base (L2-resident, G x 512); consumed after the rank
        const int64_t sbase = mine ? base[(size_t)sm.tg[b] * nbins + tid] : 0;
        const int offk = sm.toffk[b], offp = sm.toffp[b];
        const int cnt = sm.tcnt[b];
        mbar_wait(&sm.bar[b], (par >> b) & 1u);
        par ^= 1u << b;
        SEG_TS(1)
        const int wb = warp * (32 * IT);
        const int lim = cnt - wb - lane;  // item k is valid iff 32 * k < lim

        // ---- items into registers (warp-striped) and rank
        uint64_t key[IT], pay[IT];
        uint32_t dg[IT], rk[IT];
#pragma unroll
        for (int k = 0; k < IT; ++k) {
            const int li = wb + 32 * k + lane;
            key[k] = sm.buf[b][0][offk + li];
            if (LAYOUT != PP) pay[k] = sm.buf[b][NARR - 1][offp + li];
            dg[k] = TABLE ? dig.lookup(key[k]) : (LAYOUT == PP ? rec_digit<HI>(key[k], dig) : dig(key[k]));
        }
        if (lane_ordered) {
            if (cnt == TL) {
#pragma unroll
                for (int k = 0; k < IT; ++k) rk[k] = __byte_perm(atomicAdd(&hrow[dg[k]], inc), 0, half);
            } else {
#pragma unroll
                for (int k = 0; k < IT; ++k)
                    if (32 * k < lim) rk[k] = __byte_perm(atomicAdd(&hrow[dg[k]], inc), 0, half);
            }
        } else {
#pragma unroll
            for (int k = 0; k < IT; ++k) {
                const bool valid = 32 * k < lim;
                const unsigned vmask = __ballot_sync(0xffffffffu, valid);
                const unsigned peers = ballot_peers(dg[k], vmask);
                const int leader = valid ? __ffs(peers) - 1 : lane;
                uint32_t old = 0;
                if (valid && leader == lane) old = atomicAdd(&hrow[dg[k]], inc * __popc(peers));
                old = __shfl_sync(0xffffffffu, old, leader);
                rk[k] = __byte_perm(old, 0, half) + __popc(peers & lt);
            }
        }
        __syncthreads();  // S2
        SEG_TS(2)

        // ---- digit scan: thread d sums its digit over the warp rows, then
        // a block-wide exclusive scan over the digits
        uint32_t col[ROWS];
        uint32_t sum = 0;
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
            col[r] = mine ? sm.hist[r][tid] : 0;
            sum += col[r];
        }
        const uint32_t tot = (sum & 0xffffu) + (sum >> 16);
        uint32_t incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) sm.wtot[warp] = incl;
        __syncthreads();  // S3
        const uint32_t toff = incl - tot + __reduce_add_sync(0xffffffffu, lane < warp ? sm.wtot[lane] : 0u);
        if (mine) {
            uint32_t run = toff;
#pragma unroll
            for (int r = 0; r < ROWS; ++r) {
                // fields (run, run + lo); hi + lo = high half of col + (col << 16)
                const uint32_t sh = col[r] << 16;
                sm.hist[r][tid] = run * 0x10001u + sh;
                run += (col[r] + sh) >> 16;
            }
            sm.gdelta[tid] = dstart + sbase + sm.toffs[b][tid] - (int64_t)toff;
        }
        if (LAYOUT == SP) {
            uint64_t ovf = 0;
            const uint64_t pmask = (1ull << pk_pw) - 1ull;
#pragma unroll
            for (int k = 0; k < IT; ++k) {
                if (32 * k < lim) ovf |= pay[k] >> pk_pw;
                // a wider payload is masked so the key bits stay exact; the
                // caller sees *overflow and redoes the join on pairs
                key[k] = ((key[k] - pk_lower) << pk_pw) | (pay[k] & pmask);
            }
            if (__any_sync(0xffffffffu, ovf != 0) && lane == 0) atomicOr(overflow, 1u);
        }
        __syncthreads();  // S4
        SEG_TS(3)

        // ---- stage in digit order
#pragma unroll
        for (int k = 0; k < IT; ++k) {
            if (cnt == TL || 32 * k < lim) {
                const uint32_t p = __byte_perm(hrow[dg[k]], 0, half) + rk[k];
                MPSM_CHECK(p < (uint32_t)cnt);
                sm.buf[b][0][p] = key[k];
                if (LAYOUT == SS) sm.buf[b][1][p] = pay[k];
            }
        }
        __syncthreads();  // S5
        SEG_TS(4)
        for (int i = tid; i < ROWS * MAX_BINS / 4; i += THREADS)
            reinterpret_cast<uint4*>(&sm.hist[0][0])[i] = make_uint4(0, 0, 0, 0);
#pragma unroll 4
        for (int i = tid; i < cnt; i += THREADS) {
            const uint64_t v = sm.buf[b][0][i];
            const uint32_t od = TABLE ? odig.lookup(v) : (LAYOUT == SS ? odig(v) : rec_digit<HI>(v, odig));
            const int64_t o = sm.gdelta[od] + i;
            // explicit digit starts (the arena scatter): inside the digit's
            // own region of the caller's output; else inside the n outputs
            MPSM_CHECK(o >= 0 && (sg.dbase ? (o >= sg.dbase[od] && o < sg.dbase[od] + dtot[od]) : o < sg.n));
            out_k[o] = v;
            if (LAYOUT == SS) out_p[o] = sm.buf[b][1][i];
        }
        SEG_TS(5)
        if (NST == 1) {  // one buffer: refill it once the tile is out (the
                         // other CTA on the SM covers the load latency)
            __syncthreads();
            if (tid == 0) {
                if (tnext < T) {
                    fence_proxy_async_smem();
                    fetch(0, tnext);
                    tnext = (int64_t)gridDim.x + atomicAdd(ticket, 1u);
                } else {
                    sm.tile[0] = T;
                }
            }
        }
        b = (b + 1) % NST;
    }
}

// ------------------------------------------------ warp-specialised scatter
// The record passes (SP, PP) with the write-out on its own warps: THREADS
// "rankers" load, rank, scan and stage tile i while WS_WRITERS "writers"
// stream tile i-1 out of its buffer and then refill that buffer with tile
// i+2.  k_scatter runs the phases back to back, so the SM's stores stop
// while it ranks and its ranking stops while it stores (tools/
// seg_phase_timing.py: the write is ~37 % of a tile); here they overlap.
// Three tile buffers (load / stage / write), one histogram.
#ifndef MPSM_SEG_WS  // 0: record passes on k_scatter
#define MPSM_SEG_WS 1
#endif
#ifndef MPSM_SEG_WS_WRITERS_SP  // writer threads (multiple of 32) of the SP / PP passes
#define MPSM_SEG_WS_WRITERS_SP 96
#endif
#ifndef MPSM_SEG_WS_WRITERS_PP
#define MPSM_SEG_WS_WRITERS_PP 128
#endif
template <int LAYOUT>
struct WsCfg {
    static constexpr int WRITERS = LAYOUT == PP ? MPSM_SEG_WS_WRITERS_PP : MPSM_SEG_WS_WRITERS_SP;
    static constexpr int THREADS_ALL = THREADS + WRITERS;
};
constexpr int WS_NB = 3;
// named barriers: 0 __syncthreads, 1 rankers, 2 writers, 3 + b buffer b staged
constexpr int BAR_RANK = 1, BAR_WRITE = 2, BAR_STAGED = 3;

template <int LAYOUT>
struct WsSmem {
    static constexpr int NARR = (LAYOUT == PP) ? 1 : 2;
    static constexpr int TL = LCfg<LAYOUT>::TILE_L;
    uint64_t buf[WS_NB][NARR][TL + 2];
    uint32_t hist[WARPS / 2][MAX_BINS];
    int64_t gdelta[WS_NB][MAX_BINS];  // per buffer: the writers read it while the next tile is ranked
    uint32_t toffs[WS_NB][MAX_BINS];
    uint32_t wtot[WARPS];
    int64_t tile[WS_NB];
    int64_t tg[WS_NB];                     // per buffer: count CTA of the tile (Segs::tile)
    int tcnt[WS_NB], toffk[WS_NB], toffp[WS_NB];  // per buffer: tuples, alignment slots
    uint64_t bar[WS_NB];
};

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int LAYOUT, bool HI, bool TABLE = false>
__global__ void __launch_bounds__(WsCfg<LAYOUT>::THREADS_ALL, 1) k_scatter_ws(
    const uint64_t* __restrict__ in_k, const uint64_t* __restrict__ in_p, uint64_t* __restrict__ out_k, Segs sg,
    Digit dig, Digit odig, int nbins, const int64_t* __restrict__ base, const uint32_t* __restrict__ toffs,
    const int64_t* __restrict__ dtot, unsigned int* __restrict__ ticket, uint64_t pk_lower, int pk_pw,
    unsigned int* __restrict__ overflow, bool lane_ordered, uint32_t* __restrict__ dense, int dshift) {
    static_assert(LAYOUT != SS, "record output only");
    constexpr int WS_WRITERS = WsCfg<LAYOUT>::WRITERS, WS_THREADS = WsCfg<LAYOUT>::THREADS_ALL;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WsSmem<LAYOUT>& sm = *reinterpret_cast<WsSmem<LAYOUT>*>(smem_raw);
    constexpr int NARR = WsSmem<LAYOUT>::NARR;
    constexpr int ROWS = WARPS / 2;
    constexpr int IT = LCfg<LAYOUT>::ITEMS_L, TL = LCfg<LAYOUT>::TILE_L;
    static_assert(32 * IT < 65536 && TL < 65536, "16-bit histogram fields");
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t T = sg.ntiles(TL);
    if ((int64_t)blockIdx.x >= T) return;
    const bool ranker = tid < THREADS;
    const bool mine = tid < nbins;

    SegCursor cur;  // the fetching thread's
    auto fetch = [&](int bb, int64_t t) {
        int64_t t0, g;
        int cnt;
        cur.tile(sg, t, TL, t0, cnt, g);
        const int offk = (int)(((uintptr_t)(in_k + t0) >> 3) & 1);
        const int offp = NARR == 2 ? (int)(((uintptr_t)(in_p + t0) >> 3) & 1) : 0;
        sm.tile[bb] = t;
        sm.tg[bb] = g;
        sm.tcnt[bb] = cnt;
        sm.toffk[bb] = offk;
        sm.toffp[bb] = offp;
        unsigned bk = tile_plain(sm.buf[bb][0], in_k + t0, offk, cnt), bp = 0;
        if (NARR == 2) bp = tile_plain(sm.buf[bb][NARR - 1], in_p + t0, offp, cnt);
        const unsigned bo = MAX_BINS * 4;
        mbar_arrive_expect_tx(&sm.bar[bb], bk + bp + bo);
        tile_bulk(sm.buf[bb][0], in_k + t0, offk, bk, &sm.bar[bb]);
        if (NARR == 2) tile_bulk(sm.buf[bb][NARR - 1], in_p + t0, offp, bp, &sm.bar[bb]);
        bulk_load(sm.toffs[bb], toffs + (size_t)t * MAX_BINS, bo, &sm.bar[bb]);
    };
    auto fetch_next = [&](int bb) {  // one writer thread: the next tile (global order) into buffer bb
        const int64_t t = (int64_t)gridDim.x + atomicAdd(ticket, 1u);
        if (t < T) {
            fetch(bb, t);
        } else {
            sm.tile[bb] = T;  // no more tiles: complete the phase without data
            mbar_arrive_expect_tx(&sm.bar[bb], 0);
        }
    };

    for (int i = tid; i < ROWS * MAX_BINS / 4; i += WS_THREADS)
        reinterpret_cast<uint4*>(&sm.hist[0][0])[i] = make_uint4(0, 0, 0, 0);
    int64_t dstart = 0;  // ranker d: start of digit d's output region (multi-segment: in base)
    {
        const int64_t v = (mine && sg.nseg == 0) ? dtot[tid] : 0;
        int64_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        if (ranker && lane == 31) sm.gdelta[0][warp] = incl;
        if (tid == THREADS) {
            for (int q = 0; q < WS_NB; ++q) mbar_init(&sm.bar[q], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if (ranker) {
            dstart = incl - v;
            for (int w = 0; w < warp; ++w) dstart += sm.gdelta[0][w];
        }
        __syncthreads();  // gdelta[0] is free again
        if (tid == THREADS) {
            fetch(0, blockIdx.x);
            for (int q = 1; q < WS_NB; ++q) fetch_next(q);
        }
    }

    if (!ranker) {  // ------------------------------------------ writers
        const int wt = tid - THREADS;
        // density probe (dense != null, the last pass of a sort): min / max
        // of key - output position over the records this writer stores
        uint32_t dmin = 0xffffffffu, dmax = 0;
        for (int b = 0;; b = (b == WS_NB - 1) ? 0 : b + 1) {
#ifdef MPSM_DBG_TIMING
            const long long w0 = clock64();
#endif
            named_sync(BAR_STAGED + b, WS_THREADS);
            const int64_t t = sm.tile[b];
            if (t >= T) break;
#ifdef MPSM_DBG_TIMING
            if (tid == THREADS) g_seg_ts[t & ((1 << 22) - 1)][3] = w0;
#endif
            WS_TS(THREADS, t, 4)
            const int cnt = sm.tcnt[b];
            const uint64_t* sb = sm.buf[b][0];
            const int64_t* gd = sm.gdelta[b];
            if (dense) {
#pragma unroll 4
                for (int i = wt; i < cnt; i += WS_WRITERS) {
                    const uint64_t v = sb[i];
                    const int64_t o = gd[TABLE ? odig.lookup(v) : rec_digit<HI>(v, odig)] + i;
                    MPSM_CHECK(o >= 0 && o < sg.n);
                    out_k[o] = v;
                    const uint32_t d = (uint32_t)(v >> dshift) - (uint32_t)o;
                    dmin = min(dmin, d);
                    dmax = max(dmax, d);
                }
            } else {
#pragma unroll 4
                for (int i = wt; i < cnt; i += WS_WRITERS) {
                    const uint64_t v = sb[i];
                    const int64_t o = gd[TABLE ? odig.lookup(v) : rec_digit<HI>(v, odig)] + i;
                    MPSM_CHECK(o >= 0 && o < sg.n);
                    out_k[o] = v;
                }
            }
            WS_TS(THREADS, t, 5)
            named_sync(BAR_WRITE, WS_WRITERS);  // buffer b read by every writer
            if (wt == 0) {
                fence_proxy_async_smem();  // generic accesses to buf[b] before the bulk copy
                fetch_next(b);
            }
        }
        if (dense) {
            dmin = __reduce_min_sync(0xffffffffu, dmin);
            dmax = __reduce_max_sync(0xffffffffu, dmax);
            if ((wt & 31) == 0) {
                atomicMin(&dense[0], dmin);
                atomicMax(&dense[1], dmax);
            }
        }
        return;
    }

    // ---------------------------------------------------------- rankers
    uint32_t* hrow = sm.hist[warp >> 1];
    const uint32_t inc = (warp & 1) ? 0x10000u : 1u;
    const uint32_t half = (warp & 1) ? 0x4432u : 0x4410u;
    const unsigned lt = lanemask_lt();
    unsigned par = 0;
    for (int b = 0;; b = (b == WS_NB - 1) ? 0 : b + 1) {
#ifdef MPSM_DBG_TIMING
        const long long r0 = clock64();
#endif
        mbar_wait(&sm.bar[b], (par >> b) & 1u);
        par ^= 1u << b;
        const int64_t t = sm.tile[b];
        if (t >= T) {
            named_arrive(BAR_STAGED + b, WS_THREADS);  // releases the writers
            break;
        }
#ifdef MPSM_DBG_TIMING
        if (tid == 0) g_seg_ts[t & ((1 << 22) - 1)][0] = r0;
#endif
        WS_TS(0, t, 1)
        const int64_t sbase = mine ? base[(size_t)sm.tg[b] * nbins + tid] : 0;
        const int cnt = sm.tcnt[b];
        const int offk = sm.toffk[b], offp = sm.toffp[b];
        const int wb = warp * (32 * IT);
        const int lim = cnt - wb - lane;
        uint64_t key[IT], pay[LAYOUT == SP ? IT : 1];
        uint32_t rk[IT];
#pragma unroll
        for (int k = 0; k < IT; ++k) {
            const int li = wb + 32 * k + lane;
            key[k] = sm.buf[b][0][offk + li];
            if (LAYOUT == SP) pay[k] = sm.buf[b][1][offp + li];
        }
        named_sync(BAR_RANK, THREADS);  // S1: the previous tile's histogram is cleared
#pragma unroll
        for (int k = 0; k < IT; ++k) {
            const uint32_t dg =
                TABLE ? dig.lookup(key[k]) : (LAYOUT == PP ? rec_digit<HI>(key[k], dig) : dig(key[k]));
            if (lane_ordered) {
                if (cnt == TL || 32 * k < lim) rk[k] = __byte_perm(atomicAdd(&hrow[dg], inc), 0, half);
            } else {
                const bool valid = 32 * k < lim;
                const unsigned vmask = __ballot_sync(0xffffffffu, valid);
                const unsigned peers = ballot_peers(dg, vmask);
                const int leader = valid ? __ffs(peers) - 1 : lane;
                uint32_t old = 0;
                if (valid && leader == lane) old = atomicAdd(&hrow[dg], inc * __popc(peers));
                old = __shfl_sync(0xffffffffu, old, leader);
                rk[k] = __byte_perm(old, 0, half) + __popc(peers & lt);
            }
        }
        named_sync(BAR_RANK, THREADS);  // S2
        WS_TS(0, t, 6)
        uint32_t col[ROWS];
        uint32_t sum = 0;
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
            col[r] = mine ? sm.hist[r][tid] : 0;
            sum += col[r];
        }
        const uint32_t tot = (sum & 0xffffu) + (sum >> 16);
        uint32_t incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) sm.wtot[warp] = incl;
        named_sync(BAR_RANK, THREADS);  // S3
        const uint32_t toff = incl - tot + __reduce_add_sync(0xffffffffu, lane < warp ? sm.wtot[lane] : 0u);
        if (mine) {
            uint32_t run = toff;
#pragma unroll
            for (int r = 0; r < ROWS; ++r) {
                const uint32_t sh = col[r] << 16;
                sm.hist[r][tid] = run * 0x10001u + sh;
                run += (col[r] + sh) >> 16;
            }
            sm.gdelta[b][tid] = dstart + sbase + sm.toffs[b][tid] - (int64_t)toff;
        }
        if (LAYOUT == SP) {
            uint64_t ovf = 0;
            const uint64_t pmask = (1ull << pk_pw) - 1ull;
#pragma unroll
            for (int k = 0; k < IT; ++k) {
                if (32 * k < lim) ovf |= pay[k] >> pk_pw;
                key[k] = ((key[k] - pk_lower) << pk_pw) | (pay[k] & pmask);
            }
            if (__any_sync(0xffffffffu, ovf != 0) && lane == 0) atomicOr(overflow, 1u);
        }
        named_sync(BAR_RANK, THREADS);  // S4
#pragma unroll
        for (int k = 0; k < IT; ++k) {
            if (cnt == TL || 32 * k < lim) {
                const uint32_t d = TABLE ? odig.lookup(key[k]) : rec_digit<HI>(key[k], odig);
                const uint32_t p = __byte_perm(hrow[d], 0, half) + rk[k];
                MPSM_CHECK(p < (uint32_t)cnt);
                sm.buf[b][0][p] = key[k];
            }
        }
        named_sync(BAR_RANK, THREADS);  // S5: staged, histogram free
        for (int i = tid; i < ROWS * MAX_BINS / 4; i += THREADS)
            reinterpret_cast<uint4*>(&sm.hist[0][0])[i] = make_uint4(0, 0, 0, 0);
        WS_TS(0, t, 2)
        named_arrive(BAR_STAGED + b, WS_THREADS);
    }
}

// ------------------------------------------------------------------- host
// start-up probe: do shared atomicAdds that collide within one warp
// instruction return their counts in lane order?  (true on sm_100; if a
// device ever says no, the stable passes fall back to ballot ranking)
// The probe mirrors k_scatter's use: two warps share a row of 32-bit words
// (16-bit field per warp, increment 1 or 1 << 16), concurrent warps add to
// the same rows, and the returned field must equal the lane's rank among
// the lanes of its warp instruction that hit the same word, plus the field's
// value before the instruction.
__global__ void k_probe_lane_order(int* bad) {
    __shared__ uint32_t hs[4][64];  // 8 warps, two per row, 64 words per row
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* h = hs[warp >> 1];
    const uint32_t inc = (warp & 1) ? 0x10000u : 1u;
    const int sh = (warp & 1) * 16;
    for (int i = threadIdx.x; i < 4 * 64; i += blockDim.x) (&hs[0][0])[i] = 0;
    __syncthreads();
    uint32_t x = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x;
    for (int it = 0; it < 96; ++it) {
        x ^= x << 13;
        x ^= x >> 17;
        x ^= x << 5;
        const uint32_t d = (x >> 7) % (1 + (it & 63));  // 1..64 distinct words: from all-equal to spread
        const uint32_t old = (atomicAdd(&h[d], inc) >> sh) & 0xffffu;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const uint32_t base = __shfl_sync(0xffffffffu, old, __ffs(peers) - 1);
        if (old != base + __popc(peers & ((1u << lane) - 1u))) atomicAdd(bad, 1);
        if ((it & 15) == 15) {  // keep the 16-bit fields far from overflow
            __syncthreads();
            for (int i = threadIdx.x; i < 4 * 64; i += blockDim.x) (&hs[0][0])[i] = 0;
            __syncthreads();
        }
    }
}

// probed once per device (the merge-join's Run order check catches a pass
// that came out unstable anyway: InternalConsistencyError, not a silent miss)
static bool lane_ordered_atomics() {
    constexpr int MAXDEV = 64;
    static std::atomic<int> state[MAXDEV];  // 0 unknown, 1 ordered, 2 not
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= MAXDEV) return false;
    int s = state[dev].load();
    if (s == 0) {
        int* d = nullptr;
        int bad = 1;
        if (cudaMalloc(&d, sizeof(int)) == cudaSuccess) {
            cudaMemset(d, 0, sizeof(int));
            k_probe_lane_order<<<num_sms(), 256>>>(d);
            cudaMemcpy(&bad, d, sizeof(int), cudaMemcpyDeviceToHost);
            cudaFree(d);
        }
        s = (bad == 0 && cudaGetLastError() == cudaSuccess) ? 1 : 2;
        // MPSM_SEG_BALLOT_RANK=1 forces the ballot ranking (tests of the fallback)
        const char* force = getenv("MPSM_SEG_BALLOT_RANK");
        if (force && force[0] == '1') s = 2;
        state[dev].store(s);
    }
    return s == 1;
}

extern "C" int mpsm_dbg_lane_ordered() { return lane_ordered_atomics() ? 1 : 0; }

struct Ws {
    uint32_t* counts;  // [G][MAX_BINS]
    int64_t* base;     // [G][MAX_BINS]
    uint32_t* toffs;   // [tiles][MAX_BINS]
    int64_t* dtot;     // [MAX_BINS]
    unsigned int* ticket;
    int64_t *off, *tb, *gb;  // multi-segment sorts: [nseg + 1] each
    int nseg;
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

// G segments of whole scatter tiles (tile: the layout's TILE_L)
static Segs make_segs(int64_t n, int G, int tile = TILE) {
    int64_t seg = (n + G - 1) / G;
    seg = (seg + tile - 1) / tile * tile;
    if (seg == 0) seg = tile;
    return Segs{n, seg};
}

static size_t ntiles(int64_t n) { return (size_t)((n + TILE - 1) / TILE); }

// multi-segment sorts: count CTAs (at most max_grid() + nseg) and scatter
// tiles (at most one partial tile per segment more)
static size_t ws_bytes(int64_t n, int nseg = 0) {
    const size_t G = (size_t)max_grid() + nseg;
    return align_up(sizeof(uint32_t) * G * MAX_BINS) + align_up(sizeof(int64_t) * G * MAX_BINS) +
           align_up(sizeof(uint32_t) * (ntiles(n) + nseg) * MAX_BINS) + align_up(sizeof(int64_t) * MAX_BINS) +
           align_up(sizeof(unsigned int)) + 3 * align_up(sizeof(int64_t) * (nseg + 1));
}

static bool carve(void* ws, size_t bytes, int64_t n, Ws* o, int nseg = 0) {
    Carve c{(char*)ws, bytes};
    const size_t G = (size_t)max_grid() + nseg;
    o->counts = c.take<uint32_t>(G * MAX_BINS);
    o->base = c.take<int64_t>(G * MAX_BINS);
    o->toffs = c.take<uint32_t>((ntiles(n) + nseg) * MAX_BINS);
    o->dtot = c.take<int64_t>(MAX_BINS);
    o->ticket = c.take<unsigned int>(1);
    o->off = c.take<int64_t>(nseg + 1);
    o->tb = c.take<int64_t>(nseg + 1);
    o->gb = c.take<int64_t>(nseg + 1);
    o->nseg = nseg;
    return c.ok;
}

// the host offsets of a multi-segment sort -> ws.off, through a pinned
// staging buffer (a pageable copy would wait for the stream)
static int upload_offsets(const int64_t* h_off, int nseg, const Ws& ws, cudaStream_t st) {
    static int64_t* stage = nullptr;
    static size_t cap = 0;
    static cudaEvent_t done = nullptr;
    if (!done) MPSM_TRY(cuda_status(cudaEventCreateWithFlags(&done, cudaEventDisableTiming), "event"));
    MPSM_TRY(cuda_status(cudaEventSynchronize(done), "event"));  // the previous copy has left the buffer
    if (cap < (size_t)nseg + 1) {
        if (stage) cudaFreeHost(stage);
        cap = std::max<size_t>(nseg + 1, 1025);
        MPSM_TRY(cuda_status(cudaMallocHost(&stage, sizeof(int64_t) * cap), "cudaMallocHost"));
    }
    std::copy(h_off, h_off + nseg + 1, stage);
    MPSM_TRY(cuda_status(cudaMemcpyAsync(ws.off, stage, sizeof(int64_t) * (nseg + 1), cudaMemcpyHostToDevice, st),
                         "h2d"));
    return cuda_status(cudaEventRecord(done, st), "event");
}

template <int LAYOUT, bool HI, bool TABLE = false>
static int set_attr() {
    static bool done = false;
    if (!done) {
        MPSM_TRY(cuda_status(cudaFuncSetAttribute(k_scatter<LAYOUT, HI, TABLE>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem<LAYOUT>)),
                             "smem attr"));
        done = true;
    }
    return MPSM_OK;
}

template <int LAYOUT, bool HI, bool TABLE>
static int set_attr_ws() {
    static bool done = false;
    if (!done) {
        MPSM_TRY(cuda_status(cudaFuncSetAttribute(k_scatter_ws<LAYOUT, HI, TABLE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)sizeof(WsSmem<LAYOUT>)),
                             "smem attr"));
        done = true;
    }
    return MPSM_OK;
}

// one digit pass: count, scan, scatter (TABLE: the digit is a partition id)
template <int LAYOUT, bool TABLE = false>
static int pass(const uint64_t* in_k, const uint64_t* in_p, uint64_t* out_k, uint64_t* out_p, int64_t n,
                Digit count_dig, Digit dig, int bits, const Ws& ws, uint64_t span_m1, unsigned long long* d_bad,
                uint64_t pk_lower, int pk_pw, unsigned int* overflow, cudaStream_t st,
                const int64_t* dbase = nullptr, uint32_t* dense = nullptr, int dshift = 0) {
    // segments (count CTAs) are independent of the scatter grid: the tile
    // prefixes make every tile self-contained
    constexpr int64_t TL = LCfg<LAYOUT>::TILE_L;
    const int G = std::min(grid_size<LAYOUT>(), max_grid());
    int GC = std::min(num_sms() * MPSM_SEG_COUNT_PER_SM, max_grid());
    Segs sg = make_segs(n, GC, (int)TL);
    sg.dbase = dbase;
    const int nbins = 1 << bits;
    if (ws.nseg > 0) {  // multi-segment: geometry of this pass's tiles on the device
        const int64_t tpc = std::max<int64_t>(1, ((n + TL - 1) / TL + ws.nseg + GC - 1) / GC);
        k_seg_geom<<<1, MAX_SEGS, 0, st>>>(ws.off, ws.nseg, TL, tpc, ws.tb, ws.gb);
        MPSM_TRY(check_launch("k_seg_geom"));
        sg.nseg = ws.nseg;
        sg.off = ws.off;
        sg.tb = ws.tb;
        sg.gb = ws.gb;
        sg.tpc = tpc;
        GC += ws.nseg;  // a bound: the surplus count CTAs exit at once
    }
    {
        ProfScope ps("seg_count", st);
        constexpr int CPT = LCfg<LAYOUT>::TILE_L / TILE;
        if (ws.nseg > 0)
            k_count<CPT, TABLE, true><<<GC, THREADS, 0, st>>>(in_k, sg, count_dig, nbins, ws.counts, ws.toffs,
                                                               ws.ticket, span_m1, d_bad);
        else
            k_count<CPT, TABLE, false><<<GC, THREADS, 0, st>>>(in_k, sg, count_dig, nbins, ws.counts, ws.toffs,
                                                                ws.ticket, span_m1, d_bad);
    }
    MPSM_TRY(check_launch("k_count"));
    if (ws.nseg > 0)
        k_scan_mseg<<<ws.nseg, MAX_BINS, 0, st>>>(ws.counts, sg, nbins, ws.base);
    else
        k_scan<<<(nbins + 31) / 32, 32 * SCAN_GROUPS, 0, st>>>(ws.counts, GC, nbins, ws.base, ws.dtot);
    MPSM_TRY(check_launch("k_scan"));
    // digit of a staged value: records staged by the SP pass carry the key
    // above the payload bits
    const Digit odig = (LAYOUT == SP) ? Digit{0, pk_pw + dig.shift, dig.mask, dig.table, dig.nbuckets} : dig;
    const bool hi = LAYOUT != SS && odig.shift >= 32;
    MPSM_TRY(hi ? (set_attr<LAYOUT, true, TABLE>()) : (set_attr<LAYOUT, false, TABLE>()));
    {
        ProfScope ps("seg_scatter", st);
        ProfScope ps2(LAYOUT == SS ? "seg_scatter_ss" : (LAYOUT == SP ? "seg_scatter_sp" : "seg_scatter_pp"), st);
        const bool lo = lane_ordered_atomics();
        if constexpr (MPSM_SEG_WS && LAYOUT != SS && !TABLE) {
            MPSM_TRY(hi ? (set_attr_ws<LAYOUT, true, TABLE>()) : (set_attr_ws<LAYOUT, false, TABLE>()));
            const int GW = num_sms();
            if (hi)
                k_scatter_ws<LAYOUT, true, TABLE><<<GW, WsCfg<LAYOUT>::THREADS_ALL, sizeof(WsSmem<LAYOUT>), st>>>(
                    in_k, in_p, out_k, sg, dig, odig, nbins, ws.base, ws.toffs, ws.dtot, ws.ticket, pk_lower, pk_pw,
                    overflow, lo, dense, dshift);
            else
                k_scatter_ws<LAYOUT, false, TABLE><<<GW, WsCfg<LAYOUT>::THREADS_ALL, sizeof(WsSmem<LAYOUT>), st>>>(
                    in_k, in_p, out_k, sg, dig, odig, nbins, ws.base, ws.toffs, ws.dtot, ws.ticket, pk_lower, pk_pw,
                    overflow, lo, dense, dshift);
            return check_launch("k_scatter_ws");
        }
        if (hi)
            k_scatter<LAYOUT, true, TABLE><<<G, THREADS, sizeof(Smem<LAYOUT>), st>>>(
                in_k, in_p, out_k, out_p, sg, dig, odig, nbins, ws.base, ws.toffs, ws.dtot, ws.ticket, pk_lower, pk_pw, overflow, lo);
        else
            k_scatter<LAYOUT, false, TABLE><<<G, THREADS, sizeof(Smem<LAYOUT>), st>>>(
                in_k, in_p, out_k, out_p, sg, dig, odig, nbins, ws.base, ws.toffs, ws.dtot, ws.ticket, pk_lower, pk_pw, overflow, lo);
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
    *bytes = seg::ws_bytes(n);
    return MPSM_OK;
}

namespace mpsm {
namespace seg {
// the workspace of a (multi-segment) sort, its segment offsets uploaded
static int prepare(void* workspace, size_t bytes, int64_t n, int nseg, const int64_t* h_off, Ws* ws,
                   cudaStream_t st) {
    if (nseg < 0 || nseg > MAX_SEGS || (nseg > 0 && !h_off)) {
        set_error("segment count must be 0 (one sort) or 1.." + std::to_string(MAX_SEGS));
        return MPSM_ERR_ARG;
    }
    if (nseg > 0) {
        if (h_off[0] != 0 || h_off[nseg] != n) {
            set_error("segment offsets must run from 0 to n");
            return MPSM_ERR_ARG;
        }
        for (int s = 0; s < nseg; ++s)
            if (h_off[s + 1] < h_off[s]) {
                set_error("segment offsets must not decrease");
                return MPSM_ERR_ARG;
            }
    }
    if (!carve(workspace, bytes, n, ws, nseg)) {
        set_error("sort workspace too small");
        return MPSM_ERR_ARG;
    }
    return nseg > 0 ? upload_offsets(h_off, nseg, *ws, st) : MPSM_OK;
}
}  // namespace seg
}  // namespace mpsm

static int sort_pairs_impl(const uint64_t* in_keys, const uint64_t* in_pays, int64_t n, int nseg, const int64_t* h_off,
                           uint64_t lower, uint64_t span_m1, int width_bits, uint64_t* out_keys, uint64_t* out_pays,
                           uint64_t* tmp_keys, uint64_t* tmp_pays, void* workspace, size_t ws_bytes,
                           unsigned long long* d_bad, void* stream) {
    using namespace seg;
    cudaStream_t st = (cudaStream_t)stream;
    if (n < 0 || width_bits < 0 || width_bits > 64) return MPSM_ERR_ARG;
    if (n == 0) return MPSM_OK;
    Ws ws;
    MPSM_TRY(prepare(workspace, ws_bytes, n, nseg, h_off, &ws, st));
    const Plan plan = make_plan(width_bits);
    if (plan.npasses == 0) {  // one-value domain: check it and copy
        const int G = max_grid();
        k_count<1><<<G, THREADS, 0, st>>>(in_keys, make_segs(n, G), Digit{lower, 0, 0}, 1, ws.counts, ws.toffs,
                                          nullptr, span_m1, d_bad);
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
        MPSM_TRY(pass<SS>(sk, sp, dk, dp, n, dg, dg, plan.bits[i], ws, i == 0 ? span_m1 : ~0ull, i == 0 ? d_bad : nullptr,
                          0, 0, nullptr, st));
        sk = dk;
        sp = dp;
    }
    return MPSM_OK;
}

// d_dense (optional): the density probe of the sorted output (see
// mpsm_sort_packed_dense); set to "unknown" (min > max) where it cannot run
static int dense_init(uint32_t* d_dense, bool probe, cudaStream_t st) {
    if (!d_dense) return MPSM_OK;
    const uint32_t init[2] = {probe ? 0xffffffffu : 0x01010101u, 0u};
    PutBatch pb;  // a kernel, not two memsets: see PutBatch
    MPSM_TRY(put_or_copy(pb, d_dense, init, sizeof(init), st));
    return put_flush(pb, st);
}

static int sort_packed_impl(const uint64_t* in_keys, const uint64_t* in_pays, int64_t n, int nseg,
                            const int64_t* h_off, uint64_t lower, uint64_t span_m1, int width_bits, uint64_t* out_rec,
                            uint64_t* tmp_rec, void* workspace, size_t ws_bytes, unsigned long long* d_bad,
                            unsigned int* d_overflow, void* stream, uint32_t* d_dense = nullptr) {
    using namespace seg;
    cudaStream_t st = (cudaStream_t)stream;
    if (n < 0 || width_bits < 1 || width_bits > 63 || !d_overflow) return MPSM_ERR_ARG;
    const bool probe = d_dense && nseg == 0 && width_bits <= 32 && n > 0 && n < ((int64_t)1 << 32);
    MPSM_TRY(dense_init(d_dense, probe, st));
    if (n == 0) return MPSM_OK;
    Ws ws;
    MPSM_TRY(prepare(workspace, ws_bytes, n, nseg, h_off, &ws, st));
    const Plan plan = make_plan(width_bits);
    const int pw = 64 - width_bits;
    const int P = plan.npasses;
    const uint64_t* src = nullptr;
    for (int i = 0; i < P; ++i) {
        uint64_t* dst = ((P - 1 - i) % 2 == 0) ? out_rec : tmp_rec;
        uint32_t* dense = (probe && i == P - 1) ? d_dense : nullptr;  // the last pass probes its output
        if (i == 0) {
            const Digit dg{lower, plan.shift[0], (1u << plan.bits[0]) - 1u};
            MPSM_TRY(pass<SP>(in_keys, in_pays, dst, nullptr, n, dg, dg, plan.bits[0], ws, span_m1, d_bad, lower, pw,
                              d_overflow, st, nullptr, dense, pw));
        } else {
            const Digit dg{0, pw + plan.shift[i], (1u << plan.bits[i]) - 1u};
            MPSM_TRY(pass<PP>(src, nullptr, dst, nullptr, n, dg, dg, plan.bits[i], ws, ~0ull, nullptr, 0, pw, nullptr,
                              st, nullptr, dense, pw));
        }
        src = dst;
    }
    return MPSM_OK;
}

static int sort_records_impl(const uint64_t* in_rec, int64_t n, int nseg, const int64_t* h_off, int width_bits,
                             uint64_t* out_rec, uint64_t* tmp_rec, void* workspace, size_t ws_bytes, void* stream,
                             uint32_t* d_dense = nullptr) {
    using namespace seg;
    cudaStream_t st = (cudaStream_t)stream;
    if (n < 0 || width_bits < 1 || width_bits > 63) return MPSM_ERR_ARG;
    const bool probe = d_dense && nseg == 0 && width_bits <= 32 && n > 0 && n < ((int64_t)1 << 32);
    MPSM_TRY(dense_init(d_dense, probe, st));
    if (n == 0) return MPSM_OK;
    const Plan plan = make_plan(width_bits);
    const int pw = 64 - width_bits;
    const int P = plan.npasses;
    // in place (in == out) with an even number of passes: the first pass
    // writes tmp, the last one lands back in the input buffer
    if (in_rec == tmp_rec || out_rec == tmp_rec || (in_rec == out_rec && P % 2 != 0)) {
        set_error("mpsm_sort_records: in, out and tmp must be distinct (in == out only for an even pass count)");
        return MPSM_ERR_ARG;
    }
    Ws ws;
    MPSM_TRY(prepare(workspace, ws_bytes, n, nseg, h_off, &ws, st));
    const uint64_t* src = in_rec;
    for (int i = 0; i < P; ++i) {
        uint64_t* dst = ((P - 1 - i) % 2 == 0) ? out_rec : tmp_rec;
        const Digit dg{0, pw + plan.shift[i], (1u << plan.bits[i]) - 1u};
        MPSM_TRY(pass<PP>(src, nullptr, dst, nullptr, n, dg, dg, plan.bits[i], ws, ~0ull, nullptr, 0, pw, nullptr, st,
                          nullptr, (probe && i == P - 1) ? d_dense : nullptr, pw));
        src = dst;
    }
    return MPSM_OK;
}

extern "C" int mpsm_sort_pairs(const uint64_t* in_keys, const uint64_t* in_pays, int64_t n, uint64_t lower,
                               uint64_t span_m1, int width_bits, uint64_t* out_keys, uint64_t* out_pays,
                               uint64_t* tmp_keys, uint64_t* tmp_pays, void* workspace, size_t ws_bytes,
                               unsigned long long* d_bad, void* stream) {
    return sort_pairs_impl(in_keys, in_pays, n, 0, nullptr, lower, span_m1, width_bits, out_keys, out_pays, tmp_keys,
                           tmp_pays, workspace, ws_bytes, d_bad, stream);
}

extern "C" int mpsm_sort_packed(const uint64_t* in_keys, const uint64_t* in_pays, int64_t n, uint64_t lower,
                                uint64_t span_m1, int width_bits, uint64_t* out_rec, uint64_t* tmp_rec, void* workspace,
                                size_t ws_bytes, unsigned long long* d_bad, unsigned int* d_overflow, void* stream) {
    return sort_packed_impl(in_keys, in_pays, n, 0, nullptr, lower, span_m1, width_bits, out_rec, tmp_rec, workspace,
                            ws_bytes, d_bad, d_overflow, stream);
}

extern "C" int mpsm_sort_records(const uint64_t* in_rec, int64_t n, int width_bits, uint64_t* out_rec,
                                 uint64_t* tmp_rec, void* workspace, size_t ws_bytes, void* stream) {
    return sort_records_impl(in_rec, n, 0, nullptr, width_bits, out_rec, tmp_rec, workspace, ws_bytes, stream);
}

extern "C" int mpsm_sort_packed_dense(const uint64_t* in_keys, const uint64_t* in_pays, int64_t n, uint64_t lower,
                                      uint64_t span_m1, int width_bits, uint64_t* out_rec, uint64_t* tmp_rec,
                                      void* workspace, size_t ws_bytes, unsigned long long* d_bad,
                                      unsigned int* d_overflow, uint32_t* d_dense, void* stream) {
    if (!d_dense) return MPSM_ERR_ARG;
    return sort_packed_impl(in_keys, in_pays, n, 0, nullptr, lower, span_m1, width_bits, out_rec, tmp_rec, workspace,
                            ws_bytes, d_bad, d_overflow, stream, d_dense);
}

extern "C" int mpsm_sort_records_dense(const uint64_t* in_rec, int64_t n, int width_bits, uint64_t* out_rec,
                                       uint64_t* tmp_rec, void* workspace, size_t ws_bytes, uint32_t* d_dense,
                                       void* stream) {
    if (!d_dense) return MPSM_ERR_ARG;
    return sort_records_impl(in_rec, n, 0, nullptr, width_bits, out_rec, tmp_rec, workspace, ws_bytes, stream,
                             d_dense);
}

extern "C" int mpsm_sort_segments_workspace_bytes(int64_t n, int nseg, int width_bits, size_t* bytes) {
    if (!bytes || n < 0 || nseg < 0 || nseg > seg::MAX_SEGS || width_bits < 0 || width_bits > 64) return MPSM_ERR_ARG;
    *bytes = seg::ws_bytes(n, nseg);
    return MPSM_OK;
}

extern "C" int mpsm_sort_pairs_segments(const uint64_t* in_keys, const uint64_t* in_pays, int64_t n, int nseg,
                                        const int64_t* h_offsets, uint64_t lower, uint64_t span_m1, int width_bits,
                                        uint64_t* out_keys, uint64_t* out_pays, uint64_t* tmp_keys, uint64_t* tmp_pays,
                                        void* workspace, size_t ws_bytes, unsigned long long* d_bad, void* stream) {
    if (nseg < 1 || in_keys == out_keys) return MPSM_ERR_ARG;
    return sort_pairs_impl(in_keys, in_pays, n, nseg, h_offsets, lower, span_m1, width_bits, out_keys, out_pays,
                           tmp_keys, tmp_pays, workspace, ws_bytes, d_bad, stream);
}

extern "C" int mpsm_sort_packed_segments(const uint64_t* in_keys, const uint64_t* in_pays, int64_t n, int nseg,
                                         const int64_t* h_offsets, uint64_t lower, uint64_t span_m1, int width_bits,
                                         uint64_t* out_rec, uint64_t* tmp_rec, void* workspace, size_t ws_bytes,
                                         unsigned long long* d_bad, unsigned int* d_overflow, void* stream) {
    if (nseg < 1) return MPSM_ERR_ARG;
    return sort_packed_impl(in_keys, in_pays, n, nseg, h_offsets, lower, span_m1, width_bits, out_rec, tmp_rec,
                            workspace, ws_bytes, d_bad, d_overflow, stream);
}

extern "C" int mpsm_sort_records_segments(const uint64_t* in_rec, int64_t n, int nseg, const int64_t* h_offsets,
                                          int width_bits, uint64_t* out_rec, uint64_t* tmp_rec, void* workspace,
                                          size_t ws_bytes, void* stream) {
    if (nseg < 1) return MPSM_ERR_ARG;
    return sort_records_impl(in_rec, n, nseg, h_offsets, width_bits, out_rec, tmp_rec, workspace, ws_bytes, stream);
}

namespace mpsm {
namespace seg {
__global__ void k_add_written(const int64_t* __restrict__ dtot, int npart, int64_t* __restrict__ written) {
    const int d = threadIdx.x;
    if (d < npart) written[d] += dtot[d];
}
}  // namespace seg
}  // namespace mpsm

// ------------------------------------------------------------ partition scatter
// The reference's scatter_chunk (_kernels.py:262-284) / partition.scatter
// (partition.py:233-276): one stable radix pass over (key, payload) pairs
// whose digit is the partition of the key's bucket (splitter table) and whose
// digit regions start at the worker's cursors -- the arena layout of the
// reference.  d_written += the tuples each partition received.
extern "C" int mpsm_scatter_workspace_bytes(int64_t n, int npart, size_t* bytes) {
    if (!bytes || n < 0 || npart < 1 || npart > seg::MAX_BINS) return MPSM_ERR_ARG;
    *bytes = seg::ws_bytes(n);
    return MPSM_OK;
}

extern "C" int mpsm_scatter_chunk(const uint64_t* keys, const uint64_t* pays, int64_t n, uint64_t lower, int shift,
                                  const int32_t* d_sp, int nbuckets, int npart, const int64_t* d_cursors,
                                  uint64_t* arena_keys, uint64_t* arena_pays, int64_t* d_written, void* workspace,
                                  size_t ws_bytes, void* stream) {
    using namespace seg;
    cudaStream_t st = (cudaStream_t)stream;
    if (n < 0 || npart < 1 || npart > MAX_BINS || nbuckets < 1 || shift < 0 || shift > 63 || !d_sp || !d_cursors) {
        set_error("scatter: bad arguments (1 <= npart <= 512)");
        return MPSM_ERR_ARG;
    }
    if (n == 0) return MPSM_OK;
    Ws ws;
    if (!carve(workspace, ws_bytes, n, &ws)) {
        set_error("scatter workspace too small");
        return MPSM_ERR_ARG;
    }
    int pbits = 0;
    while ((1 << pbits) < npart) ++pbits;
    const Digit dg{lower, shift, 0u, d_sp, nbuckets};
    {
        ProfScope ps("scatter", st);
        MPSM_TRY((pass<SS, true>(keys, pays, arena_keys, arena_pays, n, dg, dg, pbits, ws, ~0ull, nullptr, 0, 0,
                                 nullptr, st, d_cursors)));
    }
    if (d_written) {
        k_add_written<<<1, MAX_BINS, 0, st>>>(ws.dtot, npart, d_written);
        MPSM_TRY(check_launch("k_add_written"));
    }
    return MPSM_OK;
}

extern "C" int mpsm_partition_records(const uint64_t* keys, const uint64_t* pays, int64_t n, uint64_t lower,
                                      uint64_t span_m1, int width_bits, int shift, const int32_t* d_sp, int nbuckets,
                                      int npart, uint64_t* out_rec, void* workspace, size_t ws_bytes,
                                      unsigned long long* d_bad, unsigned int* d_overflow, void* stream) {
    using namespace seg;
    if (n < 0 || width_bits < 1 || width_bits > 63 || npart < 1 || npart > MAX_BINS || nbuckets < 1 || shift < 0 ||
        !d_sp || !d_overflow)
        return MPSM_ERR_ARG;
    if (n == 0) return MPSM_OK;
    Ws ws;
    if (!carve(workspace, ws_bytes, n, &ws)) {
        set_error("partition workspace too small");
        return MPSM_ERR_ARG;
    }
    int pbits = 0;
    while ((1 << pbits) < npart) ++pbits;
    const Digit dg{lower, shift, 0u, d_sp, nbuckets};
    return pass<SP, true>(keys, pays, out_rec, nullptr, n, dg, dg, pbits, ws, span_m1, d_bad, lower, 64 - width_bits,
                          d_overflow, (cudaStream_t)stream);
}
