// merge_join.cu -- merge-path merge-join of sorted private runs against sorted
// public runs with a fused COUNT / MAX(r+s) / checksum reduction (sm_100a).
//
// Replaces engine._join_private_run (/root/reference/pkg/src/mpsm/engine.py
// 228-276) for all workers at once: per (private run i, public run j) the
// interpolation search for the start (_kernels.interp_lower_bound,
// _kernels.py:287-337) and the merge with mark/rewind over duplicate key
// groups (_kernels.merge_join_run, _kernels.py:340-408).
//
// Pipeline (all stream-ordered, no host sync):
//   k_windows    one thread per pair: S window [lb(r_first), ub(r_last)) by
//                the reference's interpolation search (identical probe count)
//                plus a binary search; "examined" statistic; tiles per pair
//   k_tile_scan  exclusive scan of tiles over pairs
//   k_part_coarse / k_partition / k_split_fill
//                merge-path tile boundaries in two levels (every 32nd tile
//                by a full search, the rest inside their coarse bracket),
//                written as flat tile descriptors (direct pointers)
//   k_merge      persistent CTAs, two stages: thread 0 brings tile g+grid into
//                shared memory with TMA bulk copies (descriptor loaded a tile
//                earlier) while tile g merges.  MODE 0 (aggregates) runs two
//                phases per tile: each thread walks MJ_ITEMS merge steps from
//                its merge-path split and records, per S tuple, how many tile
//                R tuples have key <= its key (and whether any two R keys of
//                the tile are equal); then the S tuples are dealt
//                round-robin and each matches the equal-key R group ending
//                there (ties merge R first) -- the reference's cross product
//                of duplicate key groups, with the walk-back only in tiles
//                that have repeated R keys.  COUNT / MAX / checksum are
//                reduced per CTA and flushed with one atomic per pair.  The
//                materialize modes (count, then emit at scanned offsets) use
//                the one-phase walk.
//
// Runs come in two layouts: (keys, payloads) SoA, or packed 8-B records
// (key - lower) << pw | payload written by mpsm_sort_packed (PK = true).

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <type_traits>
#include <vector>

#include "common.cuh"

namespace mpsm {

// 256 threads x 23 = 5888-tuple tiles, 2 CTAs per SM: larger tiles amortise
// the per-tile work (partition searches, staging, table setup) -- A/B on B200
// (tools/merge_variants_run.py, merge + tile partition, FK 100M x 400M):
// 128 x 15 (round 1) 1.68 ms, 256 x 15 1.62, 256 x 19 1.61, 256 x 23 1.57,
// 256 x 27 (one CTA per SM) 1.97, 512 x 15 1.76, 64 x 15 1.99
#ifndef MPSM_MJ_THREADS
#define MPSM_MJ_THREADS 256
#endif
#ifndef MPSM_MJ_ITEMS
#define MPSM_MJ_ITEMS 23
#endif
#ifndef MPSM_MJ_BLOCKS
#define MPSM_MJ_BLOCKS 2
#endif
#ifndef MPSM_MJ_P2_UNROLL  // match-phase loop unroll (independent W tuples in flight)
#define MPSM_MJ_P2_UNROLL 2
#endif
#ifndef MPSM_MJ_ORDER_CHECK  // the Run order check in the walk (0: off, A/B timing only; 1: per array; 2: merged)
#define MPSM_MJ_ORDER_CHECK 2
#endif
#define MPSM_PRAGMA(x) _Pragma(#x)
#define MPSM_UNROLL(n) MPSM_PRAGMA(unroll n)
constexpr int MJ_THREADS = MPSM_MJ_THREADS;
constexpr int MJ_ITEMS = MPSM_MJ_ITEMS;  // odd: 64-bit smem accesses at stride ITEMS are conflict-free
constexpr int MJ_TILE = MJ_THREADS * MJ_ITEMS;
#ifndef MPSM_MJ_TABLE  // MODE 0 direct-address match path (0: always the merge walk)
#define MPSM_MJ_TABLE 1
#endif
constexpr int MJ_TBL = 2048;  // table slots (a tile's R keys must span fewer)
// a table entry (16 bits): tile tag << MJ_IDX_BITS | stage index + 1; the
// table is cleared when the tags run out
constexpr int MJ_IDX_BITS = (MJ_TILE + 3 < (1 << 11)) ? 11 : (MJ_TILE + 3 < (1 << 12)) ? 12 : 13;
static_assert(MJ_TILE + 3 < (1 << MJ_IDX_BITS), "stage index + 1 fits the index field of a table entry");
constexpr int MJ_TBL_TAGS = 1 << (16 - MJ_IDX_BITS);
constexpr uint32_t MJ_IDX_MASK = (1u << MJ_IDX_BITS) - 1;

// Masked accumulation on the FMA pipe (the merge is bound by the ALU pipe:
// LOP3 / SHF / IADD3 / SEL / ISETP share it, IMAD runs beside it).  m is 0
// or 1: acc += h * m as a 64-bit add with carry through two IMADs.
__device__ __forceinline__ uint64_t mad_mask64(uint64_t acc, uint64_t h, uint32_t m) {
    uint32_t alo = (uint32_t)acc, ahi = (uint32_t)(acc >> 32);
    asm("mad.lo.cc.u32 %0, %2, %4, %0;\n\tmadc.lo.u32 %1, %3, %4, %1;"
        : "+r"(alo), "+r"(ahi)
        : "r"((uint32_t)h), "r"((uint32_t)(h >> 32)), "r"(m));
    return ((uint64_t)ahi << 32) | alo;
}
// splitmix64(a ^ rotl64(b, 17)) for 32-bit a, b (the rotation is a shift),
// the input's halves built explicitly: lo = a ^ (b << 17), hi = b >> 15
__device__ __forceinline__ uint64_t pair_hash32(uint32_t a, uint32_t b) {
    const uint32_t lo = a ^ (b << 17), hi = b >> 15;
    return mix64(((uint64_t)hi << 32) | lo);
}
// best = max(best, v) with the compare on the ALU pipe and the moves
// predicated (IMAD.MOV on the FMA pipe instead of two SELs)
__device__ __forceinline__ void max_into(uint64_t& best, uint64_t v) {
    asm("{\n\t.reg .pred p;\n\tsetp.gt.u64 p, %1, %0;\n\t@p mov.b64 %0, %1;\n\t}" : "+l"(best) : "l"(v));
}
// MAX(r + s) of 32-bit payloads without 64-bit compares: the sums split by
// the carry of the 32-bit add into two 32-bit maxima (b1: sums >= 2^32, h1
// set once one occurred) -- an IADD3 with carry-out and predicated VIMNMX
__device__ __forceinline__ void max33(uint32_t r, uint32_t s, uint32_t& b0, uint32_t& b1, uint32_t& h1) {
    asm("{\n\t.reg .pred p;\n\t.reg .u32 t, c;\n\t"
        "add.cc.u32 t, %3, %4;\n\t"
        "addc.u32 c, 0, 0;\n\t"
        "setp.ne.u32 p, c, 0;\n\t"
        "@p max.u32 %1, %1, t;\n\t"
        "@!p max.u32 %0, %0, t;\n\t"
        "@p mov.u32 %2, 1;\n\t}"
        : "+r"(b0), "+r"(b1), "+r"(h1)
        : "r"(r), "r"(s));
}
// (a + b) * m, 64-bit, on the FMA pipe
__device__ __forceinline__ uint64_t add_mask64(uint64_t a, uint64_t b, uint32_t m) {
    uint32_t lo, hi;
    asm("mul.lo.u32 %0, %2, %6;\n\tmul.lo.u32 %1, %3, %6;\n\t"
        "mad.lo.cc.u32 %0, %4, %6, %0;\n\tmadc.lo.u32 %1, %5, %6, %1;"
        : "=r"(lo), "=r"(hi)
        : "r"((uint32_t)b), "r"((uint32_t)(b >> 32)), "r"((uint32_t)a), "r"((uint32_t)(a >> 32)), "r"(m));
    return ((uint64_t)hi << 32) | lo;
}

#ifndef MPSM_MJ_FMA_SHR  // splitmix's 64-bit right shifts as IMAD.HI / IMAD (FMA pipe) in the probe loop
#define MPSM_MJ_FMA_SHR 0
#endif
// z ^ (z >> k) with the shift on the FMA pipe: mul = 2^(32-k) (1 <= k <= 31)
// from a register ptxas cannot fold, hi >> k = umulhi(hi, mul) and
// (lo >> k) | (hi << (32-k)) = umulhi(lo, mul) + hi * mul
__device__ __forceinline__ uint64_t xorshr_fma(uint64_t z, uint32_t mul) {
    const uint32_t lo = (uint32_t)z, hi = (uint32_t)(z >> 32);
    const uint32_t hs = __umulhi(hi, mul);
    const uint32_t ls = __umulhi(lo, mul) + hi * mul;
    return ((uint64_t)(hi ^ hs) << 32) | (lo ^ ls);
}
__device__ __forceinline__ uint64_t pair_hash_fma(uint64_t r_pay, uint64_t s_pay, uint32_t m30, uint32_t m27,
                                                  uint32_t m31) {
    uint64_t z = (r_pay ^ rotl64(s_pay, 17)) + 0x9E3779B97F4A7C15ull;
    z = xorshr_fma(z, m30) * 0xBF58476D1CE4E5B9ull;
    z = xorshr_fma(z, m27) * 0x94D049BB133111EBull;
    return xorshr_fma(z, m31);
}

// splitmix64(a ^ rotl64(b, 17)) of 32-bit a, b with a chosen share of the
// work on the FMA pipe (the dense-run join is bound by the ALU pipe): FMA
// bit 0 the input's shifts as IMAD / IMAD.HI, bit 1 the add of the golden
// ratio as a mad chain, bits 2-4 the three xor-shifts as IMAD.HI (see
// xorshr_fma).  K holds 2^17, 2^2, 2^5, 2^1 and 1 where ptxas cannot fold
// them (read through volatile shared loads).
struct FmaK {
    uint32_t m17, m30, m27, m31, one;
};
__device__ __forceinline__ uint64_t xorshr_alu(uint64_t z, int k) { return z ^ (z >> k); }
template <int FMA>
__device__ __forceinline__ uint64_t pair_hash32_mix(uint32_t a, uint32_t b, const FmaK& K) {
    uint32_t lo, hi;
    if (FMA & 1) {
        lo = a ^ (b * K.m17);
        hi = __umulhi(b, K.m17);
    } else {
        lo = a ^ (b << 17);
        hi = b >> 15;
    }
    uint64_t z;
    if (FMA & 2) {
        uint32_t zl, zh;
        asm("mad.lo.cc.u32 %0, %2, %4, 0x7F4A7C15;\n\tmadc.lo.u32 %1, %3, %4, 0x9E3779B9;"
            : "=r"(zl), "=r"(zh)
            : "r"(lo), "r"(hi), "r"(K.one));
        z = ((uint64_t)zh << 32) | zl;
    } else {
        z = (((uint64_t)hi << 32) | lo) + 0x9E3779B97F4A7C15ull;
    }
    z = ((FMA & 4) ? xorshr_fma(z, K.m30) : xorshr_alu(z, 30)) * 0xBF58476D1CE4E5B9ull;
    z = ((FMA & 8) ? xorshr_fma(z, K.m27) : xorshr_alu(z, 27)) * 0x94D049BB133111EBull;
    return (FMA & 16) ? xorshr_fma(z, K.m31) : xorshr_alu(z, 31);
}

struct PackInfo {
    int pw;          // payload bits of a packed record (0: SoA runs)
    uint64_t lower;  // key domain lower bound (packed keys are key - lower)
    uint64_t pmask;  // (1 << pw) - 1
    uint32_t kmask;  // pw >= 32: payload bits in a record's high word, (1 << (pw - 32)) - 1
};

// original key of element i of a run
template <bool PK>
__device__ __forceinline__ uint64_t key_of(const uint64_t* __restrict__ k, int64_t i, const PackInfo& pi) {
    return PK ? (k[i] >> pi.pw) + pi.lower : k[i];
}

struct PairWin {
    int64_t start, end;  // S window in public run j
    int64_t tiles;       // merge tiles of this pair
    int64_t tile_base;   // first global tile id
};

// flat tile descriptor: R tile = R[i0, i0+nR), W tile = S[w0, w0+nW)
struct TileSplit {
    const uint64_t* rk;  // R keys (or records) of the pair's private run
    const uint64_t* rp;  // R payloads (SoA only)
    const uint64_t* wk;  // S keys (or records) of the public run
    const uint64_t* wp;  // S payloads (SoA only)
    int64_t i0, w0;
    int32_t nR, nW;
    int32_t pair, pad;
};

// reference probe rule, _kernels.py:287-337 (fp64 probe position, bisect
// after a step that fails to halve the window)
template <bool PK>
__device__ int64_t interp_lb(const uint64_t* __restrict__ keys, int64_t n, uint64_t target, int64_t* probes_out,
                             const PackInfo& pi) {
    int64_t lo = 0, hi = n, probes = 0;
    bool bisect_next = false;
    while (lo < hi) {
        const int64_t width = hi - lo;
        if (width == 1) {
            ++probes;
            if (key_of<PK>(keys, lo, pi) < target) ++lo;
            else hi = lo;
            break;
        }
        const uint64_t klo = key_of<PK>(keys, lo, pi), khi = key_of<PK>(keys, hi - 1, pi);
        probes += 2;
        if (klo >= target) {
            hi = lo;
            break;
        }
        if (khi < target) {
            lo = hi;
            break;
        }
        int64_t pos;
        bool interp;
        if (bisect_next || khi == klo) {
            pos = lo + width / 2;
            interp = false;
        } else {
            const double frac = __ddiv_rn(__ull2double_rn(target - klo), __ull2double_rn(khi - klo));
            pos = lo + (int64_t)__dmul_rn(frac, __ll2double_rn(width - 1));
            if (pos <= lo) pos = lo + 1;
            if (pos > hi - 1) pos = hi - 1;
            interp = true;
        }
        ++probes;
        if (key_of<PK>(keys, pos, pi) < target) lo = pos + 1;
        else hi = pos;
        bisect_next = interp && (2 * (hi - lo) > width);
    }
    if (probes_out) *probes_out = probes;
    return lo;
}

template <bool PK>
__device__ __forceinline__ int64_t upper_bound_key(const uint64_t* __restrict__ keys, int64_t lo, int64_t hi,
                                                   uint64_t target, const PackInfo& pi) {
    while (lo < hi) {
        const int64_t mid = lo + ((hi - lo) >> 1);
        if (key_of<PK>(keys, mid, pi) <= target) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void k_interp_batch(const uint64_t* __restrict__ keys, int64_t n, const uint64_t* __restrict__ targets,
                               int64_t nt, int64_t* __restrict__ idx, int64_t* __restrict__ probes) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nt) return;
    int64_t pr = 0;
    const int64_t r = interp_lb<false>(keys, n, targets[t], &pr, PackInfo{0, 0, 0, 0});
    idx[t] = r;
    if (probes) probes[t] = pr;
}

// nondense (optional): per private run, nonzero unless the dense-run path
// (k_dense_join) takes its pairs; those get no merge tiles
template <bool PK>
__global__ void k_windows(const mpsm_run_t* __restrict__ priv, int n_priv, const mpsm_run_t* __restrict__ pub,
                          int n_pub, PairWin* __restrict__ win, uint64_t* __restrict__ out, PackInfo pi,
                          const uint32_t* __restrict__ nondense) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n_priv * n_pub) return;
    const mpsm_run_t r = priv[p / n_pub];
    const mpsm_run_t s = pub[p % n_pub];
    uint64_t* o = out + (size_t)p * MPSM_PAIR_FIELDS;
    PairWin w{0, 0, 0, 0};
    int64_t probes = 0, examined = 0;
    if (r.n > 0 && s.n > 0) {
        w.start = interp_lb<PK>(s.keys, s.n, key_of<PK>(r.keys, 0, pi), &probes, pi);
        w.end = upper_bound_key<PK>(s.keys, w.start, s.n, key_of<PK>(r.keys, r.n - 1, pi), pi);
        // engine.py:253-260 / _kernels.py:405-407: distinct public positions
        // read = up to the first key past the private maximum (or the end)
        examined = (w.end < s.n - 1 ? w.end : s.n - 1) - w.start + 1;
        if (examined < 0) examined = 0;
        const int64_t len = r.n + (w.end - w.start);
        const bool merge = nondense == nullptr || nondense[p / n_pub] != 0;
        w.tiles = (merge && w.end > w.start) ? (len + MJ_TILE - 1) / MJ_TILE : 0;
    }
    win[p] = w;
    o[MPSM_PAIR_COUNT] = 0;
    o[MPSM_PAIR_BEST] = 0;
    o[MPSM_PAIR_CHECKSUM] = 0;
    o[MPSM_PAIR_START] = (uint64_t)w.start;
    o[MPSM_PAIR_PROBES] = (uint64_t)probes;
    o[MPSM_PAIR_END] = (uint64_t)w.end;
    o[MPSM_PAIR_EXAMINED] = (uint64_t)examined;
    o[MPSM_PAIR_EMITTED] = 0;
    o[MPSM_PAIR_FLAGS] = 0;
}

__global__ void __launch_bounds__(1024) k_tile_scan(PairWin* __restrict__ win, int npairs, int64_t* __restrict__ total) {
    __shared__ int64_t s[1024];
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < npairs; base += 1024) {
        const int p = base + threadIdx.x;
        const int64_t v = p < npairs ? win[p].tiles : 0;
        s[threadIdx.x] = v;
        __syncthreads();
        for (int off = 1; off < 1024; off <<= 1) {
            const int64_t a = threadIdx.x >= off ? s[threadIdx.x - off] : 0;
            __syncthreads();
            s[threadIdx.x] += a;
            __syncthreads();
        }
        if (p < npairs) win[p].tile_base = carry + s[threadIdx.x] - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry += s[1023];
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

// merge path: number of R elements among the first k of merge(R, W), ties R
// first, searched among R indices [lo, hi] (a coarse bracket)
template <bool PK>
__device__ __forceinline__ int64_t merge_path_in(const uint64_t* __restrict__ rk, int64_t nr,
                                                 const uint64_t* __restrict__ wk, int64_t nw, int64_t k, int64_t lo,
                                                 int64_t hi, const PackInfo& pi) {
    lo = max(lo, k > nw ? k - nw : (int64_t)0);
    hi = min(hi, k < nr ? k : nr);
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (key_of<PK>(rk, mid, pi) <= key_of<PK>(wk, k - 1 - mid, pi)) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// pair of global tile g: last p with tile_base <= g and tiles > 0
__device__ __forceinline__ int pair_of_tile(const PairWin* __restrict__ win, int npairs, int64_t g) {
    int lo = 0, hi = npairs - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (win[mid].tile_base <= g) lo = mid;
        else hi = mid - 1;
    }
    int p = lo;
    while (win[p].tiles == 0 || win[p].tile_base + win[p].tiles <= g) --p;
    return p;
}

// Tile boundaries in two levels: k_part_coarse places every PART_STRIDE-th
// tile start of a pair by a full merge-path search; k_partition places each
// tile start inside its coarse bracket (log2(PART_STRIDE * MJ_TILE) steps
// instead of log2(|R|)); k_split_fill closes each tile at its successor's
// start.  One search per boundary.
constexpr int PART_STRIDE = 32;

template <bool PK>
__global__ void k_part_coarse(const mpsm_run_t* __restrict__ priv, const mpsm_run_t* __restrict__ pub, int n_pub,
                              const PairWin* __restrict__ win, int npairs, const int64_t* __restrict__ total,
                              int64_t* __restrict__ coarse, PackInfo pi) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= *total) return;
    const int p = pair_of_tile(win, npairs, g);
    const PairWin w = win[p];
    const int64_t local = g - w.tile_base;
    if (local % PART_STRIDE) return;
    const mpsm_run_t r = priv[p / n_pub];
    const mpsm_run_t s = pub[p % n_pub];
    const int64_t nw = w.end - w.start;
    coarse[g] = merge_path_in<PK>(r.keys, r.n, s.keys + w.start, nw, local * MJ_TILE, 0, r.n, pi);
}

template <bool PK>
__global__ void k_partition(const mpsm_run_t* __restrict__ priv, const mpsm_run_t* __restrict__ pub, int n_pub,
                            const PairWin* __restrict__ win, int npairs, const int64_t* __restrict__ total,
                            const int64_t* __restrict__ coarse, TileSplit* __restrict__ splits, PackInfo pi) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= *total) return;
    const int p = pair_of_tile(win, npairs, g);
    const mpsm_run_t r = priv[p / n_pub];
    const mpsm_run_t s = pub[p % n_pub];
    const PairWin w = win[p];
    const int64_t nw = w.end - w.start;
    const int64_t local = g - w.tile_base;
    const int64_t c0 = local - local % PART_STRIDE, c1 = c0 + PART_STRIDE;
    const int64_t lo = coarse[w.tile_base + c0];
    const int64_t hi = c1 < w.tiles ? coarse[w.tile_base + c1] : r.n;
    const int64_t k0 = local * MJ_TILE;
    const int64_t i0 = (local == c0) ? lo : merge_path_in<PK>(r.keys, r.n, s.keys + w.start, nw, k0, lo, hi, pi);
    TileSplit t;
    t.rk = r.keys;
    t.rp = r.pays;
    t.wk = s.keys;
    t.wp = s.pays;
    t.i0 = i0;
    t.w0 = w.start + (k0 - i0);
    t.nR = 0;
    t.nW = 0;
    t.pair = p;
    t.pad = 0;
    splits[g] = t;
}

__global__ void k_split_fill(const mpsm_run_t* __restrict__ priv, int n_pub, const PairWin* __restrict__ win,
                             const int64_t* __restrict__ total, TileSplit* __restrict__ splits) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n = *total;
    if (g >= n) return;
    TileSplit& t = splits[g];
    const PairWin w = win[t.pair];
    const int64_t nr = priv[t.pair / n_pub].n;
    const int64_t L = nr + (w.end - w.start);
    const int64_t local = g - w.tile_base;
    const int64_t k0 = local * MJ_TILE;
    const int64_t k1 = min(k0 + MJ_TILE, L);
    const int64_t i1 = (local + 1 < w.tiles) ? splits[g + 1].i0 : nr;
    t.nR = (int32_t)(i1 - t.i0);
    t.nW = (int32_t)((k1 - i1) - (k0 - t.i0));
}

// Tile staging.  A stage holds the 16-B aligned superset of the tile's R
// range (with the prior tuples R[i0-2], R[i0-1] when they exist: the S tuples
// that open a tile usually match the R tuple that closed the previous one,
// and R[i0-2] tells whether that group reaches back further) followed by
// the aligned superset of its W range; each range arrives with one bulk copy
// (TMA).  Reading up to 8 B beyond a range stays inside its 16-B block, so
// inside the mapped allocation.
template <bool PK>
struct alignas(16) MergeStage {
    uint64_t k[MJ_TILE + 8];           // R span (<= 4 extra slots) + W span (<= 3 extra slots)
    uint64_t p[PK ? 2 : MJ_TILE + 8];  // payloads (SoA runs only)
    TileSplit t;                       // descriptor of the staged tile
    int r0, w0, rp0, wp0, hp, whp;     // where R tile element 0 / W element 0 sit in k[] (p[]); prior R / W tuples
};
template <bool PK>
struct MergeSmem {
    MergeStage<PK> st[2];
    union {
        uint16_t ub[MJ_TILE];   // MODE 0 walk: per W tuple of the tile, R tuples <= its key (tile-relative)
        uint16_t tbl[MJ_TBL];   // MODE 0 table: slot key - key(R[-hp]) -> tag << MJ_IDX_BITS | stage index + 1
    };
    int tdup[2];           // MODE 0, per tile parity: some R key of the tile repeats
    int wend[MJ_THREADS / 32], wlo[MJ_THREADS / 32];  // MODE 0: where each warp's walk ends / starts (R index)
    uint32_t kmask;        // PackInfo::kmask, read back with a volatile load (see k_merge)
    uint32_t shr_mul[3];   // 2^(32-30), 2^(32-27), 2^(32-31): the splitmix shifts as IMAD.HI (see mix64_fma)
    uint64_t bar[2];
    uint64_t red[3][MJ_THREADS / 32];
    int64_t warp_cnt[MJ_THREADS / 32];
};

// a range [first, first + n) of array a as an aligned bulk copy: element
// first sits at index off of the copy
struct Span {
    const uint64_t* src;
    int off;
    unsigned bytes;
};
__device__ __forceinline__ Span span_of(const uint64_t* a, int64_t first, int n) {
    if (n <= 0) return Span{a, 0, 0u};
    const uintptr_t lo = (uintptr_t)(a + first), hi = (uintptr_t)(a + first + n);
    const uintptr_t a0 = lo & ~(uintptr_t)15, a1 = (hi + 15) & ~(uintptr_t)15;
    return Span{(const uint64_t*)a0, (int)((lo - a0) >> 3), (unsigned)(a1 - a0)};
}

// where tile t's elements sit in a stage
struct TilePlace {
    Span rk, wk, rp, wp;
    int hp, whp;
};
template <bool PK>
__device__ __forceinline__ TilePlace place_of(const TileSplit& t) {
    TilePlace q;
    q.hp = t.i0 >= 2 ? 2 : (int)t.i0;  // up to two prior R tuples
    q.rk = span_of(t.rk, t.i0 - q.hp, t.nR + q.hp);
    // the W key before the tile comes along (the order check of the tile
    // boundary); its payload is never read
    q.whp = (t.w0 > 0 && t.nW > 0) ? 1 : 0;
    q.wk = span_of(t.wk, t.w0 - q.whp, t.nW + q.whp);
    if (!PK) {
        q.rp = span_of(t.rp, t.i0 - q.hp, t.nR + q.hp);
        q.wp = span_of(t.wp, t.w0, t.nW);
    }
    return q;
}

template <bool PK>
__device__ __forceinline__ void fetch_tile(MergeStage<PK>& st, uint64_t* bar, const TileSplit& t) {
    const TilePlace q = place_of<PK>(t);
    st.t = t;
    // the placement, computed once here for every thread of the CTA
    st.hp = q.hp;
    st.whp = q.whp;
    st.r0 = q.rk.off + q.hp;
    st.w0 = (int)(q.rk.bytes / 8) + q.wk.off + q.whp;
    if (!PK) {
        st.rp0 = q.rp.off + q.hp;
        st.wp0 = (int)(q.rp.bytes / 8) + q.wp.off;
    }
    MPSM_CHECK(q.rk.bytes / 8 + q.wk.bytes / 8 <= MJ_TILE + 8);
    unsigned tx = q.rk.bytes + q.wk.bytes;
    if (!PK) tx += q.rp.bytes + q.wp.bytes;
    mbar_arrive_expect_tx(bar, tx);
    if (q.rk.bytes) bulk_load(st.k, q.rk.src, q.rk.bytes, bar);
    if (q.wk.bytes) bulk_load(st.k + q.rk.bytes / 8, q.wk.src, q.wk.bytes, bar);
    if (!PK) {
        if (q.rp.bytes) bulk_load(st.p, q.rp.src, q.rp.bytes, bar);
        if (q.wp.bytes) bulk_load(st.p + q.rp.bytes / 8, q.wp.src, q.wp.bytes, bar);
    }
}

template <bool PK>
__device__ __forceinline__ void flush_pair(MergeSmem<PK>& sm, uint64_t* __restrict__ out, int pair, uint64_t count,
                                           uint64_t best, uint64_t csum) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    count = warp_sum(count);
    csum = warp_sum(csum);
    best = warp_max_u64(best);
    if (lane == 0) {
        sm.red[0][warp] = count;
        sm.red[1][warp] = best;
        sm.red[2][warp] = csum;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t c = 0, b = 0, s = 0;
        for (int w = 0; w < MJ_THREADS / 32; ++w) {
            c += sm.red[0][w];
            b = sm.red[1][w] > b ? sm.red[1][w] : b;
            s += sm.red[2][w];
        }
        if (c) {
            uint64_t* o = out + (size_t)pair * MPSM_PAIR_FIELDS;
            atomicAdd((unsigned long long*)(o + MPSM_PAIR_COUNT), (unsigned long long)c);
            atomicMax((unsigned long long*)(o + MPSM_PAIR_BEST), (unsigned long long)b);
            atomicAdd((unsigned long long*)(o + MPSM_PAIR_CHECKSUM), (unsigned long long)s);
        }
    }
    __syncthreads();
}

#ifdef MPSM_DBG_TIMING
__device__ long long g_mj_ts[1 << 20][6];
#define MJ_TS(i) \
    if (MODE == 0 && tid == 0 && g < (1 << 20)) g_mj_ts[g][i] = clock64();
#else
#define MJ_TS(i)
#endif

// MODE 0: aggregate into pair records; MODE 1: per-tile counts only;
// MODE 2: emit pairs at tile_out[g] + thread offset
// Persistent CTAs, two stages: thread 0 launches the bulk copies of tile
// g + grid (descriptor loaded a tile earlier) while tile g merges.  Each
// thread takes MJ_ITEMS steps of the merge from its merge-path split; for
// every S tuple the matching R tuples are the equal-key run that ends right
// before its merge position (ties merge R first) -- the reference's cross
// product of duplicate key groups.  Per-thread accumulators are reduced per
// CTA and flushed with one atomic per (pair, CTA).
template <int MODE, bool PK, bool K32 = false>
__global__ void __launch_bounds__(MJ_THREADS, PK ? MPSM_MJ_BLOCKS : 2) k_merge(const TileSplit* __restrict__ splits,
                                                                 const int64_t* __restrict__ total, int swap,
                                                                 uint64_t* __restrict__ out_pairs,
                                                                 int64_t* __restrict__ tile_cnt,
                                                                 uint64_t* __restrict__ emit_out, int64_t cap,
                                                                 PackInfo pi) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    MergeSmem<PK>& sm = *reinterpret_cast<MergeSmem<PK>*>(smem_raw);
    const int tid = threadIdx.x;
    const int64_t ntiles = *total;
    const int64_t G = gridDim.x;
    int64_t g = blockIdx.x;
    if (g >= ntiles) return;
    int cur_pair = -1;
    uint64_t count = 0, best = 0, csum = 0;
    int buf = 0;
    unsigned par = 0;
    TileSplit t_nxt{};  // thread 0: descriptor of tile g + grid
    if (tid == 0) {
        mbar_init(&sm.bar[0], 1);
        mbar_init(&sm.bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        sm.tdup[0] = sm.tdup[1] = 0;
        sm.kmask = pi.kmask;
        sm.shr_mul[0] = 1u << 2;
        sm.shr_mul[1] = 1u << 5;
        sm.shr_mul[2] = 1u << 1;
        fetch_tile<PK>(sm.st[0], &sm.bar[0], splits[g]);
        if (g + G < ntiles) t_nxt = splits[g + G];
    }
    using KT = typename std::conditional<K32, uint32_t, uint64_t>::type;
    int tgen = MJ_TBL_TAGS;  // MODE 0 table: tag of the next table tile (MJ_TBL_TAGS: clear first)
    for (; g < ntiles; g += G) {
        MJ_TS(0)
        __syncthreads();  // stage buf^1 free, stage buf's descriptor visible
        if (tid == 0 && g + G < ntiles) {
            fetch_tile<PK>(sm.st[buf ^ 1], &sm.bar[buf ^ 1], t_nxt);
            if (g + 2 * G < ntiles) t_nxt = splits[g + 2 * G];  // consumed one tile later
        }
        if (MODE == 0 && tid == 0) sm.tdup[buf ^ 1] = 0;  // last read before this tile's S1
        const TileSplit t = sm.st[buf].t;
        if (MODE == 0 && t.pair != cur_pair) {
            if (cur_pair >= 0) flush_pair<PK>(sm, out_pairs, cur_pair, count, best, csum);
            cur_pair = t.pair;
            count = best = csum = 0;
        }
        MJ_TS(1)
        mbar_wait(&sm.bar[buf], (par >> buf) & 1u);
        par ^= 1u << buf;
        MJ_TS(2)
        const int nR = t.nR, nW = t.nW, hp = sm.st[buf].hp;
        // R tile element i (i >= -hp) and W tile element j in the stage
        const uint64_t* RK = sm.st[buf].k + sm.st[buf].r0;
        const uint64_t* WK = sm.st[buf].k + sm.st[buf].w0;
        const uint64_t* RP = PK ? RK : sm.st[buf].p + sm.st[buf].rp0;
        const uint64_t* WP = PK ? WK : sm.st[buf].p + sm.st[buf].wp0;
        // normalized keys and payloads; K32: packed keys of a domain at most
        // 32 bits wide compare as their record's high word with the payload
        // bits in it set (same order and equality as the keys; no shift)
        // kept in a register: a value from a volatile shared load cannot be
        // re-read from the parameter bank (ptxas otherwise trades the
        // register for an LDC per key)
        uint32_t kmask;
        asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(kmask) : "r"(smem_addr(&sm.kmask)));
#if MPSM_MJ_FMA_SHR
        uint32_t m30, m27, m31;  // opaque to ptxas, so the products stay IMADs
        asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(m30) : "r"(smem_addr(&sm.shr_mul[0])));
        asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(m27) : "r"(smem_addr(&sm.shr_mul[1])));
        asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(m31) : "r"(smem_addr(&sm.shr_mul[2])));
        auto hash2 = [&](uint64_t a, uint64_t b) -> uint64_t { return pair_hash_fma(a, b, m30, m27, m31); };
#else
        auto hash2 = [&](uint64_t a, uint64_t b) -> uint64_t { return pair_hash(a, b); };
#endif
        auto nkey = [&](uint64_t v) -> KT {
            if (K32) return (KT)((uint32_t)(v >> 32) | kmask);
            return PK ? (KT)(v >> pi.pw) : (KT)v;
        };
        auto rkey = [&](int i) -> KT { return nkey(RK[i]); };
        auto wkey = [&](int j) -> KT { return nkey(WK[j]); };
        auto rpay = [&](int i) -> uint64_t { return PK ? (RP[i] & pi.pmask) : RP[i]; };
        auto wpay = [&](int j) -> uint64_t { return PK ? (WP[j] & pi.pmask) : WP[j]; };
        bool tile_done = false;
#if MPSM_MJ_TABLE
        // ---- MODE 0 direct-address match.  When the tile's R keys (with
        // the staged prior tuples) span fewer than MJ_TBL key values, every
        // R tuple is entered at slot key - key(R[-hp]) of a shared table and
        // every W tuple looks its key up: a hit is the R tuple with that key
        // (the last one written if the key repeats; the group is then walked
        // in both directions).  No merge-path split and no merge walk inside
        // the tile: per W tuple a load, a table probe, the compare and the
        // aggregate, two W tuples per lane and step without branches (two
        // independent hash chains for the scheduler).  Both passes deal
        // warp-contiguous runs of the tile to the lanes, so every adjacent R
        // and W pair of the tile (and the staged prior tuples) is compared
        // through a lane shuffle: the Run order check of core.py:153-154.
        // Tiles whose R keys spread wider (sparse R) take the merge walk.
        if (MODE == 0) {
            const int nRh = nR + hp;
            // K32 keys are key << ksh | kmask: slot = (k - kb) >> ksh; the
            // span limit keeps every in-tile key difference inside int32
            const int ksh = K32 ? pi.pw - 32 : 0;
            const uint64_t tlim64 = min((uint64_t)MJ_TBL << ksh, (uint64_t)0x7fffffff);
            const KT tlim = (KT)tlim64;
            const KT kb = nRh > 0 ? rkey(-hp) : (KT)0;
            const KT span = nRh > 0 ? (KT)(rkey(nR - 1) - kb) : (KT)0;
            // a span of exactly nRh - 1 keys is dense if the steps say so
            // (checked below): then no table is needed, so R-heavy dense
            // tiles (T > 1) of any span below 2^31 take this path too
            const bool span_dense = nRh > 0 && span == (KT)((uint64_t)(nRh - 1) << ksh) && span <= (KT)0x7fffffff;
            const bool table_ok = nRh > 0 && span < tlim;
            if (table_ok || span_dense) {
                tile_done = true;
                if (tgen >= MJ_TBL_TAGS) {  // tags used up (or the walk wrote ub over the table)
                    for (int q = tid; q < MJ_TBL / 8; q += MJ_THREADS)
                        reinterpret_cast<uint4*>(sm.tbl)[q] = make_uint4(0, 0, 0, 0);
                    __syncthreads();
                    tgen = 1;
                }
                const uint32_t tag = (uint32_t)tgen << MJ_IDX_BITS;
                const int lane = tid & 31, warp = tid >> 5;
                constexpr int NWARP = MJ_THREADS / 32;
                uint32_t bad = 0;
                // insert: stage indices e = 0 .. nRh-1 (R index e - hp); the
                // order check as the minimum of the in-tile key steps (int32:
                // keys inside the span), keys outside it are out of order
                // dense: every step is exactly one key (R keys consecutive, the
                // FK case: a W key's R tuple is at stage index (k - kb) >> ksh
                // without the table)
                int32_t mind = 1;
                uint32_t nondense = 0;
                const uint32_t step1 = 1u << ksh;
                const int cw_r = (nRh + NWARP - 1) / NWARP;
                const int beg_r = min(warp * cw_r, nRh), end_r = min(beg_r + cw_r, nRh);
                // a span of exactly nRh - 1 keys is dense if the steps say so:
                // then the pass only checks them (no table stores; R-heavy
                // tiles, e.g. T > 1, read each R tuple once more and that is all)
                auto store = [&](int e, KT d) {
                    bad |= (uint32_t)(d >= tlim);
                    if (d < tlim) {
                        MPSM_CHECK(((uint32_t)d >> ksh) < (uint32_t)MJ_TBL);
                        sm.tbl[(uint32_t)d >> ksh] = (uint16_t)(tag | (uint32_t)(e + 1));
                    }
                };
                {
                    uint32_t carry = beg_r > 0 ? (uint32_t)(rkey(beg_r - 1 - hp) - kb) : 0u;
                    for (int e0 = beg_r; e0 < end_r; e0 += 32) {
                        const int e = e0 + lane;
                        const bool valid = e < end_r;
                        const KT d = valid ? (KT)(rkey(e - hp) - kb) : (KT)0;
                        const uint32_t d32 = (uint32_t)d;
                        uint32_t prev = __shfl_up_sync(0xffffffffu, d32, 1);
                        if (lane == 0) prev = carry;
                        carry = __shfl_sync(0xffffffffu, d32, 31);
                        if (valid && e > 0) {
                            mind = min(mind, (int32_t)(d32 - prev));
                            nondense |= (d32 - prev) ^ step1;
                        }
                        if (valid && !span_dense) store(e, d);
                    }
                }
                bad |= (uint32_t)(mind < 0);
                // K32: does a record of the tile carry payload bits above bit
                // 31 (in its high word, under kmask)?  If none does, the probe
                // works on the low words (32-bit payloads: the hash input
                // r ^ (s << 17) and the sum need no 64-bit payload math)
                uint32_t wide = 0;
                if (K32) {
                    const uint32_t* hw = reinterpret_cast<const uint32_t*>(sm.st[buf].k);
                    const int n_all = (int)((sm.st[buf].w0 + nW + 1) & ~1);  // every staged record (R span, W span)
                    for (int q = tid; q < n_all; q += MJ_THREADS) wide |= hw[2 * q + 1];
                    wide &= kmask;
                }
                {
                    const uint32_t f = __reduce_or_sync(0xffffffffu, (mind == 0 ? 1u : 0u) | (nondense ? 4u : 0u) |
                                                                         (wide ? 8u : 0u));
                    if (lane == 0 && f) atomicOr(&sm.tdup[buf], (int)f);
                }
                __syncthreads();
                const int tflags = sm.tdup[buf];
                if (span_dense && (tflags & 4) && !table_ok) {
                    // not dense after all and too wide for the table: the walk
                    tile_done = false;
                    if (__any_sync(0xffffffffu, bad != 0) && lane == 0)
                        atomicOr((unsigned long long*)(out_pairs + (size_t)t.pair * MPSM_PAIR_FIELDS + MPSM_PAIR_FLAGS),
                                 (unsigned long long)MPSM_FLAG_UNSORTED);
                    tgen = MJ_TBL_TAGS;
                } else {
                if (span_dense && (tflags & 4)) {  // not dense after all: the table it is
                    for (int e = beg_r + lane; e < end_r; e += 32) store(e, (KT)(rkey(e - hp) - kb));
                    __syncthreads();
                }
                const bool tdup = tflags & 1;
                const bool dense = !(tflags & 5);
                const bool narrow = K32 && !(tflags & 8);
                // probe: W indices j = 0 .. nW-1
                uint64_t best_t = best, csum_t = 0;
                uint32_t cnt_t = 0;
                {
                    const int cw = (nW + NWARP - 1) / NWARP;
                    const int beg = min(warp * cw, nW), end = min(beg + cw, nW);
                    const int whp = sm.st[buf].whp;
                    KT carry = beg > 0 ? wkey(beg - 1) : (whp ? wkey(-1) : (KT)0);
                    const bool has_prev0 = beg > 0 || whp;
                    const uint64_t pmask = K32 ? (pi.pmask | 0xffffffffull) : pi.pmask;
                    // the R tuple of a W tuple: its stage index + 1, or 0
                    auto probe = [&](KT k, bool valid) -> int {
                        const KT d = k - kb;
                        if (!valid || d >= tlim) return 0;
                        const uint32_t ent = sm.tbl[(uint32_t)d >> ksh];
                        return (ent ^ tag) <= MJ_IDX_MASK ? (int)(ent & MJ_IDX_MASK) : 0;
                    };
                    auto rpay_of = [&](uint64_t rv, int i) -> uint64_t { return PK ? (rv & pmask) : RP[i]; };
                    auto wpay_of = [&](uint64_t wv, int j) -> uint64_t { return PK ? (wv & pmask) : WP[j]; };
                    // dense tiles: the R tuple of key k is at stage index
                    // (k - kb) >> ksh if that is below nRh
                    const KT dlim = (KT)((uint64_t)nRh << ksh);
                    auto dense_probe = [&](KT k, bool valid) -> int {
                        const KT d = k - kb;
                        return (valid && d < dlim) ? (int)((uint32_t)d >> ksh) + 1 : 0;
                    };
                    auto unique_probe = [&](auto SW, auto DENSE, auto NARROW) {
                        // unique R keys: two W tuples per lane and step, the
                        // aggregate masked (IMADs) instead of branched; the W
                        // loads past the end stay inside shared memory
                        for (int j0 = beg; j0 < end; j0 += 64) {
                            const int ja = j0 + lane, jb = ja + 32;
                            const bool va = ja < end, vb = jb < end;
                            const uint64_t wa = WK[ja], wb = WK[jb];
                            const KT ka = nkey(wa), kb2 = nkey(wb);
                            KT pa = __shfl_up_sync(0xffffffffu, ka, 1), pb = __shfl_up_sync(0xffffffffu, kb2, 1);
                            const KT la = __shfl_sync(0xffffffffu, ka, 31);
                            if (lane == 0) {
                                pa = carry;
                                pb = la;
                            }
                            carry = __shfl_sync(0xffffffffu, kb2, 31);
                            bad |= (uint32_t)(va && (ja > beg || has_prev0) && pa > ka);
                            bad |= (uint32_t)(vb && pb > kb2);
                            // hit flags (0/1) and R stage indices (a miss reads R[-hp])
                            uint32_t ma, mb;
                            int ia, ib;
                            if (decltype(DENSE)::value) {
                                const KT da = ka - kb, db = kb2 - kb;
                                ma = (va && da < dlim) ? 1u : 0u;
                                mb = (vb && db < dlim) ? 1u : 0u;
                                ia = (int)(ma * ((uint32_t)da >> ksh)) - hp;
                                ib = (int)(mb * ((uint32_t)db >> ksh)) - hp;
                            } else {
                                const int ea = probe(ka, va), eb = probe(kb2, vb);
                                ma = ea ? 1u : 0u;
                                mb = eb ? 1u : 0u;
                                ia = (ea ? ea : 1) - 1 - hp;
                                ib = (eb ? eb : 1) - 1 - hp;
                            }
                            MPSM_CHECK(ia >= -hp && ia < nR && ib >= -hp && ib < nR);
                            // the W loads past the end stay inside the CTA's shared memory
                            MPSM_CHECK((const char*)(WK + jb + 1) <= (const char*)&sm + sizeof(MergeSmem<PK>));
                            const uint64_t ra = RK[ia], rb = RK[ib];
                            uint64_t ha, hb, sa, sb;
                            if (decltype(NARROW)::value) {
                                // 32-bit payloads in the low words: rotl64(s, 17) is a shift
                                const uint32_t rpa = (uint32_t)ra, spa = (uint32_t)wa;
                                const uint32_t rpb = (uint32_t)rb, spb = (uint32_t)wb;
                                ha = decltype(SW)::value ? pair_hash32(spa, rpa) : pair_hash32(rpa, spa);
                                hb = decltype(SW)::value ? pair_hash32(spb, rpb) : pair_hash32(rpb, spb);
                                sa = add_mask64(rpa, spa, ma);
                                sb = add_mask64(rpb, spb, mb);
                            } else {
                                const uint64_t rpa = rpay_of(ra, ia), spa = PK ? (wa & pmask) : (va ? WP[ja] : 0);
                                const uint64_t rpb = rpay_of(rb, ib), spb = PK ? (wb & pmask) : (vb ? WP[jb] : 0);
                                ha = decltype(SW)::value ? hash2(spa, rpa) : hash2(rpa, spa);
                                hb = decltype(SW)::value ? hash2(spb, rpb) : hash2(rpb, spb);
                                sa = add_mask64(rpa, spa, ma);
                                sb = add_mask64(rpb, spb, mb);
                            }
                            max_into(best_t, sa);
                            max_into(best_t, sb);
                            csum_t = mad_mask64(mad_mask64(csum_t, ha, ma), hb, mb);
                            cnt_t += ma + mb;
                        }
                    };
                    using T_ = std::true_type;
                    using F_ = std::false_type;
                    if (dense && narrow) {
                        if (swap) unique_probe(T_{}, T_{}, std::integral_constant<bool, K32>{});
                        else unique_probe(F_{}, T_{}, std::integral_constant<bool, K32>{});
                    } else if (dense) {
                        if (swap) unique_probe(T_{}, T_{}, F_{});
                        else unique_probe(F_{}, T_{}, F_{});
                    } else if (!tdup) {
                        if (swap) unique_probe(T_{}, F_{}, F_{});
                        else unique_probe(F_{}, F_{}, F_{});
                    } else {
                        for (int j0 = beg; j0 < end; j0 += 32) {
                            const int j = j0 + lane;
                            const bool valid = j < end;
                            const uint64_t wv = valid ? WK[j] : 0;
                            const KT k = nkey(wv);
                            KT prev = __shfl_up_sync(0xffffffffu, k, 1);
                            if (lane == 0) prev = carry;
                            carry = __shfl_sync(0xffffffffu, k, 31);
                            bad |= (uint32_t)(valid && (j > beg || has_prev0) && prev > k);
                            const int ent = probe(k, valid);
                            if (!ent) continue;  // no R tuple with this key
                            int i = ent - 1 - hp;
                            const uint64_t sp = wpay_of(wv, j);
                            auto acc = [&](uint64_t rp) {
                                const uint64_t v = rp + sp;
                                best_t = v > best_t ? v : best_t;
                                csum_t += swap ? pair_hash(sp, rp) : pair_hash(rp, sp);
                                ++cnt_t;
                            };
                            // repeated R keys: the whole equal-key group
                            while (i + 1 < nR && rkey(i + 1) == k) ++i;
                            for (;;) {
                                acc(rpay_of(RK[i], i));
                                if (--i < -hp) {  // the group reaches back before the stage
                                    for (int64_t gi = t.i0 + i; gi >= 0; --gi) {
                                        const uint64_t gv = t.rk[gi];
                                        if (nkey(gv) != k) break;
                                        acc(PK ? (gv & pmask) : t.rp[gi]);
                                    }
                                    break;
                                }
                                if (rkey(i) != k) break;
                            }
                        }
                    }
                }
                count += cnt_t;
                best = best_t;
                csum += csum_t;
                if (__any_sync(0xffffffffu, bad != 0) && lane == 0)
                    atomicOr((unsigned long long*)(out_pairs + (size_t)t.pair * MPSM_PAIR_FIELDS + MPSM_PAIR_FLAGS),
                             (unsigned long long)MPSM_FLAG_UNSORTED);
                ++tgen;
                }  // dense or table
            } else {
                tgen = MJ_TBL_TAGS;  // the walk writes ub over the table
            }
        }
#endif
        if (!tile_done) {
        const int L = nR + nW;
        const int k0 = min(tid * MJ_ITEMS, L);
        const int k1 = min(k0 + MJ_ITEMS, L);
        // per-thread split inside the tile
        int lo = k0 > nW ? k0 - nW : 0, hi = k0 < nR ? k0 : nR;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (rkey(mid) <= wkey(k0 - 1 - mid)) lo = mid + 1;
            else hi = mid;
        }
        MJ_TS(3)
        int64_t my_pairs = 0;
        int64_t emit_base = 0;
#ifndef MPSM_MJ_ONE_PHASE
        if (MODE == 0) {
            // phase 1 -- the thread's merge steps, branch-light: record for
            // every W tuple the number of tile R tuples with key <= its key
            // ... and whether two neighbouring R keys of the tile (or of its
            // two prior tuples) are equal: then some S tuple matches an
            // equal-key group of several R tuples
            {
                // K32: also whether a record of the tile carries payload
                // bits above bit 31 (in its high word: hi & kmask); if none
                // does, the match phase works on the low words alone
                uint32_t wide = 0;
                auto hi_of = [&](uint64_t v) -> uint32_t { return (uint32_t)(v >> 32); };
                auto rk_w = [&](int i) -> KT {
                    if (K32) wide |= hi_of(RK[i]);
                    return rkey(i);
                };
                auto wk_w = [&](int j) -> KT {
                    if (K32) wide |= hi_of(WK[j]);
                    return wkey(j);
                };
                int ri = lo, wj = k0 - lo;
                KT rkc = ri < nR ? rk_w(ri) : 0;
                KT wkc = wj < nW ? wk_w(wj) : 0;
                // the reference's Run invariant (core.py:153-154), checked on
                // every adjacent pair the walk advances over: a run out of
                // order (e.g. an unstable radix pass) flags the pair record
                bool unsorted = false;
                bool dup = false;
                if (ri < nR && ri - 1 >= -hp) {
                    const KT pk = rkey(ri - 1);
                    dup = pk == rkc;
                    unsorted = pk > rkc;
                }
                // the W pair across the thread boundary (the one inside the
                // walk ranges of two threads)
                if (wj >= 1 && wj < nW) unsorted = unsorted || wkey(wj - 1) > wkc;
                if (tid == 0) {
                    if (hp == 2) {
                        const KT a = rk_w(-2), b = rk_w(-1);
                        dup = dup || a == b;
                        unsorted = unsorted || a > b;
                    } else if (hp == 1) {
                        rk_w(-1);
                    }
                    // the W element before the tile (staged with it)
                    if (sm.st[buf].whp) unsorted = unsorted || wkey(-1) > wkey(0);
                }
                KT dmin = dup ? (KT)0 : (KT)1;  // 0 iff two neighbouring R keys are equal (one min per step)
                // the keys the walk takes must not decrease: within a thread
                // that covers every adjacent R pair and W pair it steps over
                // (both arrays are taken in order); the pairs across thread
                // and tile boundaries are checked above, and the threads'
                // walks must meet (checked below), so every adjacent pair of
                // the tile is compared
                KT last = 0;
                uint32_t down = 0;
                // the shared address of ub[0] in a register: through the
                // array ptxas rebuilt the shared window base (S2R CgaCtaId,
                // LEA) at every store of the walk
                uint32_t ub_base;  // opaque to ptxas (a volatile mov): kept, not rematerialised
                asm volatile("mov.u32 %0, %1;" : "=r"(ub_base) : "r"(smem_addr(&sm.ub[0])));
                for (int st = k0; st < k1; ++st) {
                    const bool take_r = ri < nR && (wj >= nW || rkc <= wkc);
                    if (MPSM_MJ_ORDER_CHECK == 2) {
                        const KT m = take_r ? rkc : wkc;
                        down |= (uint32_t)(m < last);
                        last = m;
                    }
                    MPSM_CHECK(take_r || wj < nW);
                    if (!take_r) asm volatile("st.shared.u16 [%0], %1;" ::"r"(ub_base + 2u * (uint32_t)wj), "h"((unsigned short)ri) : "memory");
                    ri += take_r;
                    wj += !take_r;
                    if (take_r && ri < nR) {
                        const KT nk = rk_w(ri);
                        dmin = min(dmin, (KT)(nk ^ rkc));
                        if (MPSM_MJ_ORDER_CHECK == 1) unsorted = unsorted || nk < rkc;
                        rkc = nk;
                    }
                    if (!take_r && wj < nW) {
                        const KT nw = wk_w(wj);
                        if (MPSM_MJ_ORDER_CHECK == 1) unsorted = unsorted || nw < wkc;
                        wkc = nw;
                    }
                }
                unsorted = unsorted || down != 0;
                // the walks meet: my end is the next thread's merge-path split
                if (MPSM_MJ_ORDER_CHECK) {
                    const int nlo = __shfl_down_sync(0xffffffffu, lo, 1);
                    if ((tid & 31) != 31) unsorted = unsorted || nlo != ri;
                    else sm.wend[tid >> 5] = ri;
                    if ((tid & 31) == 0) sm.wlo[tid >> 5] = lo;
                }
                dup = dmin == 0;
                const int fl = (dup ? 1 : 0) | ((K32 && (wide & kmask)) ? 2 : 0);
                if (fl) atomicOr(&sm.tdup[buf], fl);
                if (__any_sync(0xffffffffu, unsorted) && (tid & 31) == 0)
                    atomicOr((unsigned long long*)(out_pairs + (size_t)t.pair * MPSM_PAIR_FIELDS + MPSM_PAIR_FLAGS),
                             (unsigned long long)MPSM_FLAG_UNSORTED);
            }
            __syncthreads();
            // the walks of consecutive warps meet
            if (MPSM_MJ_ORDER_CHECK && tid < MJ_THREADS / 32 - 1 && sm.wend[tid] != sm.wlo[tid + 1])
                atomicOr((unsigned long long*)(out_pairs + (size_t)t.pair * MPSM_PAIR_FIELDS + MPSM_PAIR_FLAGS),
                         (unsigned long long)MPSM_FLAG_UNSORTED);
            MJ_TS(4)
            // phase 2 -- W tuples dealt round-robin (balanced, no merge
            // control flow): each matches the equal-key R group ending at
            // tile index ub - 1 (walked back; usually one tuple)
            // K32: the payload field covers the whole low word, so the mask
            // touches the high word only
            const uint64_t pmask = K32 ? (pi.pmask | 0xffffffffull) : pi.pmask;
            auto acc = [&](uint64_t rp, uint64_t sp) {
                const uint64_t v = rp + sp;
                best = v > best ? v : best;
                ++count;
                csum += swap ? pair_hash(sp, rp) : pair_hash(rp, sp);
            };
            // unique R keys: at most one match per W tuple; the orientation
            // test is hoisted out of the loop (SW: checksum of (s, r))
            auto unique_pass = [&](auto SW) {
                MPSM_UNROLL(MPSM_MJ_P2_UNROLL)
                for (int j = tid; j < nW; j += MJ_THREADS) {
                    const int i = (int)sm.ub[j] - 1;
                    if (i < -hp) continue;  // no R tuple <= the key (tile at the run start)
                    const uint64_t wv = WK[j], rv = RK[i];
                    if (nkey(rv) != nkey(wv)) continue;
                    const uint64_t rp = PK ? (rv & pmask) : RP[i], sp = PK ? (wv & pmask) : WP[j];
                    const uint64_t v = rp + sp;
                    best = v > best ? v : best;
                    ++count;
                    csum += decltype(SW)::value ? pair_hash(sp, rp) : pair_hash(rp, sp);
                }
            };
            // K32 and every payload of the tile below 2^32: keys compare as
            // the high words outside the payload bits, payloads are the low
            // words, and rotl64(s, 17) of a 32-bit s is a plain shift
            // CHK: only a pair's first tile (no prior R tuple, hp == 0) can
            // hold a W tuple with no R tuple <= its key
            auto unique_pass32 = [&](auto SW, auto CHK) {
                MPSM_UNROLL(MPSM_MJ_P2_UNROLL)
                for (int j = tid; j < nW; j += MJ_THREADS) {
                    const int i = (int)sm.ub[j] - 1;
                    if (decltype(CHK)::value && i < -hp) continue;
                    const uint64_t wv = WK[j], rv = RK[i];
                    if (((uint32_t)(wv >> 32) ^ (uint32_t)(rv >> 32)) & ~pi.kmask) continue;  // a uniform-register operand
                    const uint32_t rp = (uint32_t)rv, sp = (uint32_t)wv;
                    const uint64_t v = (uint64_t)rp + sp;
                    best = v > best ? v : best;
                    ++count;
                    const uint32_t a = decltype(SW)::value ? sp : rp, b = decltype(SW)::value ? rp : sp;
                    csum += mix64((uint64_t)a ^ ((uint64_t)b << 17));
                }
            };
            const int tfl = sm.tdup[buf];
            if (K32 && tfl == 0) {
                if (hp == 0) {
                    if (swap) unique_pass32(std::true_type{}, std::true_type{});
                    else unique_pass32(std::false_type{}, std::true_type{});
                } else {
                    if (swap) unique_pass32(std::true_type{}, std::false_type{});
                    else unique_pass32(std::false_type{}, std::false_type{});
                }
            } else if (!(tfl & 1)) {
                if (swap) unique_pass(std::true_type{});
                else unique_pass(std::false_type{});
            } else
            for (int j = tid; j < nW; j += MJ_THREADS) {
                const uint64_t wv = WK[j];
                const KT wk = nkey(wv);
                int i = (int)sm.ub[j] - 1;
                if (i < -hp) continue;  // no R tuple <= the key (tile at the run start)
                uint64_t rv = RK[i];
                if (nkey(rv) != wk) continue;
                const uint64_t sp = PK ? (wv & pmask) : WP[j];
                for (;;) {  // the equal-key R group, backwards; usually one tuple
                    acc(PK ? (rv & pmask) : RP[i], sp);
                    if (--i < -hp) {  // the group reaches back before the tile
                        for (int64_t g = t.i0 + i; g >= 0; --g) {
                            const uint64_t gv = t.rk[g];
                            if (nkey(gv) != wk) break;
                            acc(PK ? (gv & pmask) : t.rp[g], sp);
                        }
                        break;
                    }
                    rv = RK[i];
                    if (nkey(rv) != wk) break;
                }
            }
        } else
#endif
        for (int pass = (MODE == 2 ? 0 : 1); pass < 2; ++pass) {
            // MODE 2 runs the thread's merge twice: count, then emit at its offset
            if (MODE == 2 && pass == 1) {
                const int64_t v = my_pairs;
                const int lane = tid & 31, warp = tid >> 5;
                int64_t incl = v;
                for (int o = 1; o < 32; o <<= 1) {
                    const int64_t u = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += u;
                }
                if (lane == 31) sm.warp_cnt[warp] = incl;
                __syncthreads();
                int64_t before = 0;
                for (int w = 0; w < warp; ++w) before += sm.warp_cnt[w];
                emit_base = tile_cnt[g] + before + incl - v;  // tile_cnt holds the tile's output offset here
            }
            int64_t e = 0;
            // R accessors by tile index i (i < -hp falls back to global memory)
            auto rkey_at = [&](int64_t i) -> KT {
                if (i >= -hp) return rkey((int)i);
                return nkey(t.rk[t.i0 + i]);
            };
            auto rpay_at = [&](int64_t i) -> uint64_t {
                if (i >= -hp) return rpay((int)i);
                return PK ? (t.rk[t.i0 + i] & pi.pmask) : t.rp[t.i0 + i];
            };
            auto emit = [&](uint64_t rp, uint64_t sp) {
                if (MODE == 0) {
                    const uint64_t v = rp + sp;
                    best = v > best ? v : best;
                    ++count;
                    csum += swap ? pair_hash(sp, rp) : pair_hash(rp, sp);
                } else if (MODE == 1 || pass == 0) {
                    ++e;
                } else {
                    // storage stops at capacity (the reference's merge_join_run,
                    // _kernels.py:382-390); PAIR_EMITTED says how many landed
                    const int64_t o = emit_base + e;
                    if (o < cap) {
                        emit_out[2 * o] = swap ? sp : rp;
                        emit_out[2 * o + 1] = swap ? rp : sp;
                    }
                    ++e;
                }
            };
            int ri = lo, wj = k0 - lo;
            // the equal-key R group ending at ri-1: key gk, first index gs,
            // payload of its last element lrp (register-carried; an S tuple
            // with key gk matches exactly R[gs, ri))
            bool gvalid = t.i0 + ri - 1 >= 0;
            KT gk = 0;
            uint64_t lrp = 0;
            int gs = ri - 1;
            if (gvalid) {
                gk = rkey_at(ri - 1);
                lrp = rpay_at(ri - 1);
                while (t.i0 + gs - 1 >= 0 && rkey_at(gs - 1) == gk) --gs;
            }
            KT rkc = ri < nR ? rkey(ri) : 0;  // next R key
            KT wkc = wj < nW ? wkey(wj) : 0;  // next S key
            auto step = [&]() {
                if (ri < nR && (wj >= nW || rkc <= wkc)) {
                    if (!gvalid || rkc != gk) {
                        gk = rkc;
                        gs = ri;
                        gvalid = true;
                    }
                    lrp = rpay(ri);
                    ++ri;
                    if (ri < nR) rkc = rkey(ri);
                    return;
                }
                if (gvalid && wkc == gk) {
                    const uint64_t sp = wpay(wj);
                    emit(lrp, sp);
                    for (int i = ri - 2; i >= gs; --i) emit(rpay_at(i), sp);  // duplicate R keys
                }
                ++wj;
                if (wj < nW) wkc = wkey(wj);
            };
            for (int st = k0; st < k1; ++st) step();
            my_pairs = e;
        }
        if (MODE != 0) MJ_TS(4)
        if (MODE == 1) {
            const int64_t c = warp_sum((unsigned long long)my_pairs);
            if ((tid & 31) == 0) sm.warp_cnt[tid >> 5] = c;
            __syncthreads();
            if (tid == 0) {
                int64_t sum = 0;
                for (int w = 0; w < MJ_THREADS / 32; ++w) sum += sm.warp_cnt[w];
                tile_cnt[g] = sum;
            }
        }
        }  // !tile_done
        MJ_TS(5)
        buf ^= 1;
    }
    if (MODE == 0 && cur_pair >= 0) flush_pair<PK>(sm, out_pairs, cur_pair, count, best, csum);
}

// per-pair emitted counts from per-tile counts; tile offsets (exclusive scan)
__global__ void __launch_bounds__(1024) k_emit_offsets(int64_t* __restrict__ tile_cnt, const TileSplit* __restrict__ splits,
                                                       const int64_t* __restrict__ total, uint64_t* __restrict__ out_pairs,
                                                       int64_t cap, int64_t* __restrict__ grand) {
    __shared__ int64_t s[1024];
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int64_t n = *total;
    for (int64_t base = 0; base < n; base += 1024) {
        const int64_t g = base + threadIdx.x;
        const int64_t v = g < n ? tile_cnt[g] : 0;
        s[threadIdx.x] = v;
        __syncthreads();
        for (int off = 1; off < 1024; off <<= 1) {
            const int64_t a = threadIdx.x >= off ? s[threadIdx.x - off] : 0;
            __syncthreads();
            s[threadIdx.x] += a;
            __syncthreads();
        }
        if (g < n) {
            const int64_t off = carry + s[threadIdx.x] - v;
            tile_cnt[g] = off;
            // pairs of this tile that land below the capacity
            const int64_t w = min(v, max(cap - off, (int64_t)0));
            if (w)
                atomicAdd((unsigned long long*)(out_pairs + (size_t)splits[g].pair * MPSM_PAIR_FIELDS +
                                                MPSM_PAIR_EMITTED),
                          (unsigned long long)w);
        }
        __syncthreads();
        if (threadIdx.x == 1023) carry += s[1023];
        __syncthreads();
    }
    if (threadIdx.x == 0) *grand = carry;
}

static int64_t max_tiles(const mpsm_run_t* priv, int n_priv, const mpsm_run_t* pub, int n_pub) {
    int64_t m = 0;
    for (int i = 0; i < n_priv; ++i)
        for (int j = 0; j < n_pub; ++j) {
            if (priv[i].n == 0 || pub[j].n == 0) continue;
            m += (priv[i].n + pub[j].n + MJ_TILE - 1) / MJ_TILE;
        }
    return std::max<int64_t>(m, 1);
}

struct JoinWs {
    mpsm_run_t* d_priv;
    mpsm_run_t* d_pub;
    PairWin* win;
    int64_t* total;
    int64_t* grand;
    TileSplit* splits;
    int64_t* tile_cnt;
};

static bool carve_join(Carve& c, int n_priv, int n_pub, int64_t mt, JoinWs* o) {
    o->d_priv = c.take<mpsm_run_t>(std::max(n_priv, 1));
    o->d_pub = c.take<mpsm_run_t>(std::max(n_pub, 1));
    o->win = c.take<PairWin>((size_t)std::max(n_priv * n_pub, 1));
    o->total = c.take<int64_t>(1);
    o->grand = c.take<int64_t>(1);
    o->splits = c.take<TileSplit>(mt);
    o->tile_cnt = c.take<int64_t>(mt);
    return c.ok;
}


template <int MODE, bool PK, bool K32 = false>
static int launch_merge(const JoinWs& w, int swap, uint64_t* d_pairs, uint64_t* emit_out, int64_t cap, int64_t mt,
                        const PackInfo& pi, cudaStream_t st) {
    static int per_sm = 0;
    if (per_sm == 0) {
        MPSM_TRY(cuda_status(cudaFuncSetAttribute(k_merge<MODE, PK, K32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)sizeof(MergeSmem<PK>)),
                             "smem attr"));
        MPSM_TRY(cuda_status(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_merge<MODE, PK, K32>, MJ_THREADS,
                                                                           sizeof(MergeSmem<PK>)),
                             "occupancy"));
        if (per_sm < 1) per_sm = 1;
    }
    // persistent grid: exactly the resident CTAs
    const int grid = (int)std::min<int64_t>((int64_t)num_sms() * per_sm, mt);
    ProfScope ps(MODE == 0 ? "merge" : (MODE == 1 ? "merge_count" : "merge_emit"), st);
    k_merge<MODE, PK, K32><<<grid, MJ_THREADS, sizeof(MergeSmem<PK>), st>>>(w.splits, w.total, swap, d_pairs, w.tile_cnt,
                                                                    emit_out, cap, pi);
    return check_launch("k_merge");
}

// ================================================================ dense private runs
// MODE 0 over packed records when a private run is dense: its keys step by
// exactly one (R[k+1] = R[k] + 1 -- the primary-key side of an FK join, or a
// range partition of one).  Merging a sorted S window against such a run
// needs no merge walk: the R tuple of public key k sits at index k - key(R[0]),
// and every S tuple of the window [lb(key(R[0])), ub(key(R[n-1]))) has one.
//   k_dense_check  one read of each private run: dense or not (a run out of
//                  order is never dense; it takes the merge walk, which
//                  flags it), and key(R[0])
//   k_blk_bounds   each dense run cut into blocks of K tuples; per block b
//                  and public run j the lower bound L(b, j) of the block's
//                  first key inside the pair's window (b = 0: the window
//                  start, b = nblk: its end)
//   k_blk_count / k_scan_i64 / k_blk_tiles
//                  tiles per block: ceil(S tuples of the block / DJ_TW)
//   k_dense_join   persistent CTAs, one producer warp: per tile the R block
//                  and the tile's share of the block's S pieces from ALL
//                  public runs arrive by TMA (two stages, full/empty
//                  mbarriers); 8 consumer warps take 64-tuple chunks: load,
//                  index, gather the R tuple from shared memory, aggregate.
// With T public runs the R block is staged once for all of them (the merge
// path reads every R tuple once per (i, j) pair, T times), and the work per
// tile is proportional to its S tuples.  The Run order check covers every
// adjacent S pair of the windows: lane shuffles inside a piece, the staged
// tuple before each piece, block bounds that must not decrease, and every S
// key inside its block's key range.  Per-pair COUNT / MAX / checksum are
// reduced per warp and piece into shared accumulators of the CTA's current
// private run, flushed with one atomic per pair when the run changes.
#ifndef MPSM_DJ_WARPS
#define MPSM_DJ_WARPS 8
#endif
#ifndef MPSM_DJ_CTAS  // resident CTAs per SM
#define MPSM_DJ_CTAS 2
#endif
constexpr int DJ_WARPS = MPSM_DJ_WARPS;  // consumer warps; DJ_NPROD more warps produce
#ifndef MPSM_DJ_PRODUCERS  // producer warps, each placing every NPROD-th tile of the CTA
#define MPSM_DJ_PRODUCERS 1
#endif
constexpr int DJ_NPROD = MPSM_DJ_PRODUCERS;
constexpr int DJ_THREADS = 32 * (DJ_WARPS + DJ_NPROD);
#ifndef MPSM_DJ_TW
#define MPSM_DJ_TW 4096
#endif
constexpr int DJ_TW = MPSM_DJ_TW;  // S tuples per tile (at most)
#ifndef MPSM_DJ_KMAX
#define MPSM_DJ_KMAX 2048
#endif
constexpr int DJ_KMAX = MPSM_DJ_KMAX;  // R tuples per block (at most)
#ifndef MPSM_DJ_STAGES
#define MPSM_DJ_STAGES 2
#endif
constexpr int DJ_STAGES = MPSM_DJ_STAGES;
constexpr int DJ_MAXRUNS = 64;     // runs per side on this path
#ifndef MPSM_DJ_CHUNK
#define MPSM_DJ_CHUNK 128
#endif
constexpr int DJ_CHUNK = MPSM_DJ_CHUNK;  // S tuples per warp step
constexpr int DJ_U = DJ_CHUNK / 32;       // per lane
#ifndef MPSM_DJ_CONSEC  // consumer lanes own 4 consecutive S tuples (16-B loads, in-lane order check)
#define MPSM_DJ_CONSEC 1
#endif
static_assert(!MPSM_DJ_CONSEC || DJ_U == 4, "the consecutive consumer layout moves 4 tuples per lane");
#ifndef MPSM_DJ_DYN  // consumer warps take a tile's chunks from a shared counter (else a static split)
#define MPSM_DJ_DYN 0
#endif
#ifndef MPSM_DJ_GRAB  // chunks per take
#define MPSM_DJ_GRAB 1
#endif
#ifndef MPSM_DJ_FMA  // pair_hash32_mix's FMA-pipe share (bit 5: the checksum adds as mad chains)
#define MPSM_DJ_FMA 5
#endif

struct DjTile {
    int32_t e;  // block entry
    int32_t q;  // which share of the entry's S tuples
};

struct alignas(16) DjStage {
    uint64_t r[DJ_KMAX + 4];                             // R block (aligned superset)
    uint64_t w[DJ_TW + 3 * DJ_MAXRUNS + 2 * DJ_CHUNK];  // pieces (aligned supersets + prior tuple) + over-read slack
    int poff[DJ_MAXRUNS], pn[DJ_MAXRUNS], pj[DJ_MAXRUNS], phas[DJ_MAXRUNS];
    int pcb[DJ_MAXRUNS + 1];  // exclusive chunk offsets of the pieces
    int npieces, i, r0, nb;
    int next;       // MPSM_DJ_DYN: the next chunk a consumer warp takes
    uint64_t kblk;  // normalized key of the block's first R tuple
};
struct DjSmem {
    DjStage st[DJ_STAGES];
    uint64_t full[DJ_STAGES], empty[DJ_STAGES];
    unsigned long long acc_cnt[DJ_MAXRUNS], acc_best[DJ_MAXRUNS], acc_csum[DJ_MAXRUNS];
    mpsm_run_t priv[DJ_MAXRUNS];
    int64_t blk_base[DJ_MAXRUNS + 1];
    uint64_t kb[DJ_MAXRUNS];
    uint32_t fmak[5];  // FmaK, read back through volatile loads
};

struct DjArgs {
    const mpsm_run_t* priv;
    const mpsm_run_t* pub;
    int n_priv, n_pub;
    int64_t K;                // R tuples per block
    int64_t nent;             // block entries (nblk + 1 per private run)
    uint32_t* nondense;       // per private run
    uint64_t* kb;             // per private run: normalized key of R[0]
    const int64_t* blk_base;  // per private run: its first entry (n_priv + 1)
    const PairWin* win;
    int64_t* L;       // [nent][n_pub] piece bounds
    int64_t* tb;      // [nent + 1] first tile of each entry
    int32_t* nsub;    // [nent] tiles of each entry
    int64_t* part;    // per 1024 entries: tiles (k_blk_count), then their offsets
    DjTile* tiles;
    int64_t* ntiles;
    uint64_t* out_pairs;
    PackInfo pi;
};

__device__ __forceinline__ int dj_run_of(const int64_t* __restrict__ blk_base, int n_priv, int64_t e) {
    int lo = 0, hi = n_priv - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (blk_base[mid] <= e) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// per private run: nondense[i] = 1 unless every key steps by one; kb[i] =
// normalized key of R[0].  Each warp checks 256 consecutive records per
// step: four 16-B loads in flight per lane (record pairs), neighbours across
// lanes by shuffles.  A run not 16-B aligned is checked from its second
// record on, the first against it separately.
// hint (optional): the density probe of the sorted array the private runs
// were cut from (mpsm_sort_*_dense: min / max of key - position over its hn
// records at hbase).  Equal, with key(last) - key(first) = hn - 1, the array
// is dense -- and so is every run cut from it: no run is read.
__global__ void __launch_bounds__(256) k_dense_check(const mpsm_run_t* __restrict__ priv, int pw,
                                                     uint32_t* __restrict__ nondense, uint64_t* __restrict__ kb,
                                                     const uint32_t* __restrict__ hint,
                                                     const uint64_t* __restrict__ hbase, int64_t hn) {
    const int i = blockIdx.y;
    const mpsm_run_t r = priv[i];
    const int lane = threadIdx.x & 31;
    if (r.n <= 0) {
        if (blockIdx.x == 0 && threadIdx.x == 0) nondense[i] = 1;
        return;
    }
    if (hint && hn > 0 && hint[0] == hint[1] && r.keys >= hbase && r.keys + r.n <= hbase + hn) {
        const uint64_t k0 = hbase[0] >> pw, k1 = hbase[hn - 1] >> pw;
        if (k1 >= k0 && k1 - k0 == (uint64_t)(hn - 1)) {
            if (blockIdx.x == 0 && threadIdx.x == 0) kb[i] = k0 + (uint64_t)(r.keys - hbase);
            return;  // nondense[i] stays 0
        }
    }
    const int64_t head = ((uintptr_t)r.keys & 15) ? 1 : 0;
    bool bad = false;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        kb[i] = r.keys[0] >> pw;
        if (head && r.n > 1) bad = ((r.keys[1] >> pw) - (r.keys[0] >> pw)) != 1;
    }
    const uint64_t* base = r.keys + head;
    const int64_t n = r.n - head;  // records from the aligned one on
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    int iter = 0;
    for (int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); c * 256 < n - 1; c += nw) {
        // a run found not dense: the rest need not be read (the skewed and
        // sparse runs of cfg4 stop after their first chunks); the flag other
        // warps raised is polled every 8th chunk
        if (__any_sync(0xffffffffu, bad)) {
            if (lane == 0) atomicOr(&nondense[i], 1u);
            break;
        }
        if ((++iter & 7) == 0 && *(volatile const uint32_t*)&nondense[i]) break;
        const int64_t k0 = c * 256;
        ulonglong2 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t k = k0 + 64 * u + 2 * lane;
            if (k + 1 < n) {
                v[u] = __ldcs(reinterpret_cast<const ulonglong2*>(base + k));
            } else {
                v[u].x = k < n ? base[k] : 0;
                v[u].y = 0;
            }
        }
        const int64_t kn = k0 + 256;
        const uint64_t tail = (lane == 31 && kn < n) ? base[kn] : 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t k = k0 + 64 * u + 2 * lane;
            uint64_t nx = __shfl_down_sync(0xffffffffu, v[u].x, 1);
            const uint64_t first_next = __shfl_sync(0xffffffffu, v[u < 3 ? u + 1 : 3].x, 0);
            if (lane == 31) nx = u < 3 ? first_next : tail;
            if (k + 1 < n) bad |= ((v[u].y >> pw) - (v[u].x >> pw)) != 1;
            if (k + 2 < n) bad |= ((nx >> pw) - (v[u].y >> pw)) != 1;
        }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&nondense[i], 1u);
}

// two levels (as the merge partition): COARSE places the bound of every
// DJ_COARSE-th block (and the run's end) by a search over the whole window,
// the fine pass each other bound inside its coarse bracket
constexpr int DJ_COARSE = 32;
template <bool COARSE>
__global__ void k_blk_bounds(DjArgs a) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= a.nent * a.n_pub) return;
    const int64_t e = t / a.n_pub;
    const int j = (int)(t - e * a.n_pub);
    const int i = dj_run_of(a.blk_base, a.n_priv, e);
    const int64_t b = e - a.blk_base[i];
    const int64_t nblk = a.blk_base[i + 1] - a.blk_base[i] - 1;
    const bool coarse_entry = b % DJ_COARSE == 0 || b >= nblk;
    if (COARSE != coarse_entry) return;
    int64_t v = 0;
    if (!a.nondense[i]) {
        const PairWin w = a.win[(int64_t)i * a.n_pub + j];
        if (b == 0) {
            v = w.start;
        } else if (b >= nblk) {
            v = w.end;
        } else if (!COARSE) {
            // inside the bracket of the coarse bounds around b
            const uint64_t key = a.kb[i] + (uint64_t)(b * a.K);
            const uint64_t* sk = a.pub[j].keys;
            const int pw = a.pi.pw;
            const int64_t b0 = b - b % DJ_COARSE, b1 = min(b0 + DJ_COARSE, nblk);
            int64_t lo = a.L[(a.blk_base[i] + b0) * a.n_pub + j], hi = a.L[(a.blk_base[i] + b1) * a.n_pub + j];
            hi = max(hi, lo);
            while (lo < hi) {
                const int64_t mid = lo + ((hi - lo) >> 1);
                if ((sk[mid] >> pw) < key) lo = mid + 1;
                else hi = mid;
            }
            v = lo;
        } else {
            const uint64_t key = a.kb[i] + (uint64_t)(b * a.K);
            const uint64_t* sk = a.pub[j].keys;
            const int pw = a.pi.pw;
            // lower bound of key in [start, end): interpolation steps
            // alternating with halvings (a few probes on spread keys, at
            // most twice the binary search's on any)
            int64_t lo = w.start, hi = w.end;
            bool interp = true;
            while (hi - lo > 16) {
                int64_t mid;
                if (interp) {
                    const uint64_t klo = sk[lo] >> pw, khi = sk[hi - 1] >> pw;
                    if (key <= klo) {
                        hi = lo;
                        break;
                    }
                    if (key > khi) {
                        lo = hi;
                        break;
                    }
                    const double f = (double)(key - klo) / (double)(khi - klo);
                    mid = lo + (int64_t)(f * (double)(hi - 1 - lo));
                    mid = min(max(mid, lo), hi - 1);
                } else {
                    mid = lo + ((hi - lo) >> 1);
                }
                const int64_t w0 = hi - lo;
                if ((sk[mid] >> pw) < key) lo = mid + 1;
                else hi = mid;
                // keep interpolating while it more than halves the window
                interp = !interp || 2 * (hi - lo) < w0;
            }
            while (lo < hi) {
                const int64_t mid = lo + ((hi - lo) >> 1);
                if ((sk[mid] >> pw) < key) lo = mid + 1;
                else hi = mid;
            }
            v = lo;
        }
    }
    a.L[t] = v;
}

// tiles per entry (local exclusive offsets per 1024 entries + their totals);
// decreasing bounds (a public run out of order) flag the pair
__global__ void __launch_bounds__(1024) k_blk_count(DjArgs a) {
    __shared__ int64_t s[1024];
    const int64_t e = (int64_t)blockIdx.x * 1024 + threadIdx.x;
    int64_t ns = 0;
    if (e < a.nent) {
        const int i = dj_run_of(a.blk_base, a.n_priv, e);
        const int64_t b = e - a.blk_base[i];
        const int64_t nblk = a.blk_base[i + 1] - a.blk_base[i] - 1;
        if (!a.nondense[i] && b < nblk) {
            const int64_t* L0 = a.L + e * a.n_pub;
            const int64_t* L1 = L0 + a.n_pub;
            int64_t c = 0;
            for (int j = 0; j < a.n_pub; ++j) {
                const int64_t d = L1[j] - L0[j];
                if (d < 0)
                    atomicOr((unsigned long long*)(a.out_pairs + ((size_t)i * a.n_pub + j) * MPSM_PAIR_FIELDS +
                                                   MPSM_PAIR_FLAGS),
                             (unsigned long long)MPSM_FLAG_UNSORTED);
                else c += d;
            }
            ns = (c + DJ_TW - 1) / DJ_TW;
        }
        a.nsub[e] = (int32_t)ns;
    }
    s[threadIdx.x] = ns;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
        const int64_t u = threadIdx.x >= off ? s[threadIdx.x - off] : 0;
        __syncthreads();
        s[threadIdx.x] += u;
        __syncthreads();
    }
    if (e < a.nent) a.tb[e] = s[threadIdx.x] - ns;
    if (threadIdx.x == 1023) a.part[blockIdx.x] = s[1023];
}

// in-place exclusive scan of v[0, n) (one CTA), *total = the sum
__global__ void __launch_bounds__(1024) k_scan_i64(int64_t* __restrict__ v, int64_t n, int64_t* __restrict__ total) {
    __shared__ int64_t s[1024];
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < n; base += 1024) {
        const int64_t p = base + threadIdx.x;
        const int64_t x = p < n ? v[p] : 0;
        s[threadIdx.x] = x;
        __syncthreads();
        for (int off = 1; off < 1024; off <<= 1) {
            const int64_t u = threadIdx.x >= off ? s[threadIdx.x - off] : 0;
            __syncthreads();
            s[threadIdx.x] += u;
            __syncthreads();
        }
        if (p < n) v[p] = carry + s[threadIdx.x] - x;
        __syncthreads();
        if (threadIdx.x == 1023) carry += s[1023];
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

__global__ void k_blk_tiles(DjArgs a) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= a.nent) return;
    const int64_t base = a.tb[e] + a.part[e / 1024];
    a.tb[e] = base;
    if (e == a.nent - 1) a.tb[a.nent] = *a.ntiles;
    const int32_t ns = a.nsub[e];
    for (int32_t q = 0; q < ns; ++q) a.tiles[base + q] = DjTile{(int32_t)e, q};
}

#ifdef MPSM_DBG_TIMING
__device__ long long g_dj_ts[1 << 20][8];
#define DJ_TS(who, gg, i) \
    if (lane == 0 && (who) && (gg) < (1 << 20)) g_dj_ts[gg][i] = clock64();
extern "C" int mpsm_dbg_dj_ts(long long* host, int ntiles) {
    return cuda_status(cudaMemcpyFromSymbol(host, g_dj_ts, sizeof(long long) * 8 * (size_t)ntiles), "dbg");
}
#else
#define DJ_TS(who, gg, i)
#endif
template <bool K32, bool SW>
__global__ void __launch_bounds__(DJ_THREADS, MPSM_DJ_CTAS) k_dense_join(DjArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    DjSmem& sm = *reinterpret_cast<DjSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t ntiles = *a.ntiles;
    const int64_t G = gridDim.x;
    if ((int64_t)blockIdx.x >= ntiles) return;
    const int n_pub = a.n_pub, n_priv = a.n_priv;
    if (tid == 0) {
        for (int q = 0; q < DJ_STAGES; ++q) {
            mbar_init(&sm.full[q], 1);
            mbar_init(&sm.empty[q], DJ_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int q = tid; q < DJ_MAXRUNS; q += DJ_THREADS) sm.acc_cnt[q] = sm.acc_best[q] = sm.acc_csum[q] = 0;
    for (int q = tid; q < n_priv; q += DJ_THREADS) {
        sm.priv[q] = a.priv[q];
        sm.kb[q] = a.kb[q];
    }
    for (int q = tid; q <= n_priv; q += DJ_THREADS) sm.blk_base[q] = a.blk_base[q];
    if (tid == 0) {
        sm.fmak[0] = 1u << 17;
        sm.fmak[1] = 1u << 2;
        sm.fmak[2] = 1u << 5;
        sm.fmak[3] = 1u << 1;
        sm.fmak[4] = 1u;
    }
    __syncthreads();
    const int pw = a.pi.pw;
    if (warp >= DJ_WARPS) {
        // ---- producer.  Software-pipelined: the descriptor of tile k + 2
        // and the bounds rows of tile k + 1 are in flight while tile k's
        // pieces are placed and its copies issued.
        const unsigned lt = lanemask_lt();
        struct Rows {
            DjTile t;
            int64_t tb0, tb1, l0[2], l1[2];
        };
        auto load_rows = [&](const DjTile& t) {
            Rows r;
            r.t = t;
            r.tb0 = a.tb[t.e];
            r.tb1 = a.tb[t.e + 1];
            const int64_t* L0 = a.L + (int64_t)t.e * n_pub;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j = lane + 32 * h;
                r.l0[h] = j < n_pub ? L0[j] : 0;
                r.l1[h] = j < n_pub ? L0[n_pub + j] : 0;
            }
            return r;
        };
        // producer pw places the CTA's tiles it = pw, pw + NPROD, ... (the
        // placement is a chain of shuffles and dependent loads; with one
        // producer it bounded the tile rate)
        const int pw = warp - DJ_WARPS;
        const int64_t GS = G * DJ_NPROD;
        const int64_t g0 = blockIdx.x + (int64_t)pw * G;
        if (g0 >= ntiles) return;
        Rows cur = load_rows(a.tiles[g0]);
        DjTile t_nxt = g0 + GS < ntiles ? a.tiles[g0 + GS] : DjTile{0, 0};
        int it = pw;
        for (int64_t g = g0; g < ntiles; g += GS, it += DJ_NPROD) {
            Rows nxt;
            const bool more = g + GS < ntiles;
            if (more) nxt = load_rows(t_nxt);
            if (g + 2 * GS < ntiles) t_nxt = a.tiles[g + 2 * GS];
            const int s = it % DJ_STAGES;
            DjStage& st = sm.st[s];
            const DjTile t = cur.t;
            const int i = dj_run_of(sm.blk_base, n_priv, t.e);
            const int64_t b = t.e - sm.blk_base[i];
            const mpsm_run_t R = sm.priv[i];
            const int64_t r_first = b * a.K;
            const int nb = (int)min(a.K, R.n - r_first);
            const int64_t nsub = cur.tb1 - cur.tb0;
            // public run j = lane + 32 h: its piece of the block, then this
            // tile's share [c0, c1) of the block's pieces in run order
            int64_t c[2], P[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                c[h] = max(cur.l1[h] - cur.l0[h], (int64_t)0);
                P[h] = c[h];
            }
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t u0 = __shfl_up_sync(0xffffffffu, P[0], o), u1 = __shfl_up_sync(0xffffffffu, P[1], o);
                if (lane >= o) {
                    P[0] += u0;
                    P[1] += u1;
                }
            }
            P[1] += __shfl_sync(0xffffffffu, P[0], 31);
            const int64_t total = __shfl_sync(0xffffffffu, P[1], 31);
            const int64_t c0 = t.q * total / nsub, c1 = (t.q + 1) * total / nsub;
            int n[2], hp[2], recs[2], chs[2];
            Span sp[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t excl = P[h] - c[h];
                const int64_t lo = max(excl, c0), hi = min(P[h], c1);
                n[h] = hi > lo ? (int)(hi - lo) : 0;
                const int64_t gs = cur.l0[h] + (lo - excl);
                hp[h] = (n[h] > 0 && gs > 0) ? 1 : 0;
                sp[h] = n[h] > 0 ? span_of(a.pub[lane + 32 * h].keys, gs - hp[h], n[h] + hp[h]) : Span{nullptr, 0, 0u};
                recs[h] = (int)(sp[h].bytes / 8);
                // CONSEC: a piece is consumed from the even stage slot at or
                // below its first tuple (lead = 1 puts the tuple before it,
                // prior or alignment slack, in front)
                const int lead = MPSM_DJ_CONSEC ? ((sp[h].off + hp[h]) & 1) : 0;
                chs[h] = n[h] > 0 ? (n[h] + lead + DJ_CHUNK - 1) / DJ_CHUNK : 0;
            }
            const unsigned m0 = __ballot_sync(0xffffffffu, n[0] > 0), m1 = __ballot_sync(0xffffffffu, n[1] > 0);
            const int slot0 = __popc(m0 & lt), slot1 = __popc(m0) + __popc(m1 & lt);
            const int np = __popc(m0) + __popc(m1);
            // stage positions and chunk offsets: exclusive scans in run order
            int rp[2] = {recs[0], recs[1]}, cp[2] = {chs[0], chs[1]};
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int a0 = __shfl_up_sync(0xffffffffu, rp[0], o), a1 = __shfl_up_sync(0xffffffffu, rp[1], o);
                const int b0 = __shfl_up_sync(0xffffffffu, cp[0], o), b1 = __shfl_up_sync(0xffffffffu, cp[1], o);
                if (lane >= o) {
                    rp[0] += a0;
                    rp[1] += a1;
                    cp[0] += b0;
                    cp[1] += b1;
                }
            }
            rp[1] += __shfl_sync(0xffffffffu, rp[0], 31);
            cp[1] += __shfl_sync(0xffffffffu, cp[0], 31);
            const int nchunks = __shfl_sync(0xffffffffu, cp[1], 31);
            const Span rs = span_of(R.keys, r_first, nb);
            unsigned tx = sp[0].bytes + sp[1].bytes;
            tx = warp_sum(tx) + rs.bytes;
            // the tile is placed; now wait for its stage
            DJ_TS(true, g, 0)
            if (it >= DJ_STAGES) mbar_wait(&sm.empty[s], ((it / DJ_STAGES) - 1) & 1);
            DJ_TS(true, g, 1)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (n[h] > 0) {
                    const int slot = h ? slot1 : slot0;
                    const int pos = rp[h] - recs[h];
                    MPSM_CHECK(slot < DJ_MAXRUNS && pos + recs[h] <= DJ_TW + 3 * DJ_MAXRUNS);
                    st.poff[slot] = pos + sp[h].off + hp[h];
                    st.pn[slot] = n[h];
                    st.pj[slot] = lane + 32 * h;
                    st.phas[slot] = hp[h];
                    st.pcb[slot] = cp[h] - chs[h];
                }
            }
            if (lane == 0) {
                st.pcb[np] = nchunks;
                st.npieces = np;
                st.next = 0;
                st.i = i;
                st.nb = nb;
                st.r0 = rs.off;
                st.kblk = sm.kb[i] + (uint64_t)r_first;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive_expect_tx(&sm.full[s], tx);
            __syncwarp();
            if (lane == 0 && rs.bytes) bulk_load(st.r, rs.src, rs.bytes, &sm.full[s]);
#pragma unroll
            for (int h = 0; h < 2; ++h)
                if (n[h] > 0) bulk_load(st.w + (rp[h] - recs[h]), sp[h].src, sp[h].bytes, &sm.full[s]);
            DJ_TS(true, g, 2)
            if (more) cur = nxt;
        }
        return;
    }
    // ---- consumers.  Per-lane COUNT / MAX / checksum of the warp's current
    // pair stay in registers across chunks and tiles; they are reduced into
    // the CTA's shared accumulators when the pair changes.
    using KT = typename std::conditional<K32, uint32_t, uint64_t>::type;
    const uint32_t kmask = a.pi.kmask;
    const uint64_t pmask = a.pi.pmask;
    const uint32_t pmask32 = (uint32_t)pmask;
    auto nk = [&](uint64_t v) -> KT {
        if (K32) return (KT)((uint32_t)(v >> 32) >> (pw - 32));
        return (KT)(v >> pw);
    };
    int cur_i = -1, acc_j = -1;
    uint64_t best = 0, csum = 0;
    int64_t cnt = 0;  // warp-uniform
    bool bad = false;
    uint32_t b0 = 0, b1 = 0, h1 = 0;  // max33 classes of the warp's current pair
    auto flush_regs = [&]() {
        if (acc_j < 0) return;
        {
            const uint64_t cb = h1 ? ((1ull << 32) | b1) : (uint64_t)b0;
            if (cb > best) best = cb;
            b0 = b1 = h1 = 0;
        }
        // warp reductions as REDUX: the 64-bit sum from four 16-bit slices,
        // the 64-bit max as the max high word, then the max low word under it
        const uint32_t lo = (uint32_t)csum, hi = (uint32_t)(csum >> 32);
        const uint64_t cs = (uint64_t)__reduce_add_sync(0xffffffffu, lo & 0xffffu) +
                            ((uint64_t)__reduce_add_sync(0xffffffffu, lo >> 16) << 16) +
                            ((uint64_t)__reduce_add_sync(0xffffffffu, hi & 0xffffu) << 32) +
                            ((uint64_t)__reduce_add_sync(0xffffffffu, hi >> 16) << 48);
        const uint32_t bh = __reduce_max_sync(0xffffffffu, (uint32_t)(best >> 32));
        const uint32_t bl = __reduce_max_sync(0xffffffffu, (uint32_t)(best >> 32) == bh ? (uint32_t)best : 0u);
        const uint64_t bs = ((uint64_t)bh << 32) | bl;
        const bool anybad = __any_sync(0xffffffffu, bad);
        if (lane == 0) {
            if (cnt) {
                atomicAdd(&sm.acc_cnt[acc_j], (unsigned long long)cnt);
                atomicMax(&sm.acc_best[acc_j], (unsigned long long)bs);
                atomicAdd(&sm.acc_csum[acc_j], (unsigned long long)cs);
            }
            if (anybad)
                atomicOr((unsigned long long*)(a.out_pairs + ((size_t)cur_i * n_pub + acc_j) * MPSM_PAIR_FIELDS +
                                               MPSM_PAIR_FLAGS),
                         (unsigned long long)MPSM_FLAG_UNSORTED);
        }
        best = csum = 0;
        cnt = 0;
        bad = false;
        acc_j = -1;
    };
    auto flush_runs = [&](int ci) {
        named_bar_sync(1, DJ_WARPS * 32);
        if (warp == 0) {
            for (int j = lane; j < n_pub; j += 32) {
                const unsigned long long cn = sm.acc_cnt[j];
                if (cn) {
                    uint64_t* o = a.out_pairs + ((size_t)ci * n_pub + j) * MPSM_PAIR_FIELDS;
                    atomicAdd((unsigned long long*)(o + MPSM_PAIR_COUNT), cn);
                    atomicMax((unsigned long long*)(o + MPSM_PAIR_BEST), sm.acc_best[j]);
                    atomicAdd((unsigned long long*)(o + MPSM_PAIR_CHECKSUM), sm.acc_csum[j]);
                }
                sm.acc_cnt[j] = sm.acc_best[j] = sm.acc_csum[j] = 0;
            }
        }
        named_bar_sync(1, DJ_WARPS * 32);
    };
    // hash + sum of one matched pair of low words / full payloads
    FmaK fk;
    {
        uint32_t* kp = &fk.m17;
        for (int q = 0; q < 5; ++q)
            asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(kp[q]) : "r"(smem_addr(&sm.fmak[q])));
    }
    auto agg32 = [&](uint32_t rp, uint32_t sp, uint64_t& h, uint64_t& sum) {
        h = SW ? pair_hash32_mix<MPSM_DJ_FMA>(sp, rp, fk) : pair_hash32_mix<MPSM_DJ_FMA>(rp, sp, fk);
        sum = (uint64_t)rp + sp;
    };
    auto agg64 = [&](uint64_t rp, uint64_t sp, uint64_t& h, uint64_t& sum) {
        h = SW ? pair_hash(sp, rp) : pair_hash(rp, sp);
        sum = rp + sp;
    };
    int it = 0;
    for (int64_t g = blockIdx.x; g < ntiles; g += G, ++it) {
        const int s = it % DJ_STAGES;
        DJ_TS(warp == 0, g, 3)
        mbar_wait(&sm.full[s], (it / DJ_STAGES) & 1);
        DJ_TS(warp == 0, g, 4)
        const DjStage& st = sm.st[s];
        const int i = st.i;
        if (i != cur_i) {
            flush_regs();
            if (cur_i >= 0) flush_runs(cur_i);
            cur_i = i;
        }
        const int C = st.pcb[st.npieces];
        const uint32_t rb_addr = smem_addr(st.r + st.r0);
        const uint64_t* W = st.w;
        const KT kblk = (KT)st.kblk;
        const KT nbk = (KT)st.nb, nbm1 = nbk - 1;
        int p = 0;
        // the warp's chunks [cb, ce): with MPSM_DJ_DYN taken MPSM_DJ_GRAB at a
        // time from the stage's counter until the tile is used up (the stage
        // is released when its slowest warp is done: a static split left
        // warps idle behind the slowest, tools/dj_timing.py), else one
        // static share
        for (int take = 0;; ++take) {
        int cb, ce;
        if (MPSM_DJ_DYN) {
            int q = 0;
            if (lane == 0) q = atomicAdd(&sm.st[s].next, MPSM_DJ_GRAB);
            q = __shfl_sync(0xffffffffu, q, 0);
            if (q >= C) break;
            cb = q;
            ce = min(q + MPSM_DJ_GRAB, C);
        } else {
            if (take > 0) break;
            cb = warp * C / DJ_WARPS;
            ce = (warp + 1) * C / DJ_WARPS;
        }
        int c = cb;
        if (c < ce)
            while (st.pcb[p + 1] <= c) ++p;
        while (c < ce) {
            // the warp's chunks of piece p
            const int off = st.poff[p], n = st.pn[p], pc = st.pcb[p], pe = min(st.pcb[p + 1], ce);
            const int j = st.pj[p];
            if (j != acc_j) {
                flush_regs();
                acc_j = j;
            }
            int k0 = (c - pc) * DJ_CHUNK;
            const bool has = st.phas[p] != 0;
#if MPSM_DJ_CONSEC
            // lane l owns the 4 consecutive stage slots base + k0 + 4l + u of
            // the piece seen from the even slot base <= off (lead = 1: slot
            // base is the tuple before the piece -- its prior, or with no
            // prior (the run's first tuple) alignment slack, never aggregated)
            const int lead = off & 1, base = off - lead, nv = n + lead;
            const int lo_ok = lead - (has ? 1 : 0);  // pairs (v - 1, v) with v - 1 >= lo_ok are run neighbours
            // key before the warp's first tuple here (0: nothing to check)
            KT carry = 0;
            if (k0 > 0) carry = nk(W[base + k0 - 1]);
            else if (lead == 0 && has) carry = nk(W[base - 1]);
            for (; c < pe; ++c, k0 += DJ_CHUNK) {
                const int rem = nv - k0;
                const uint64_t* wq = W + base + k0 + 4 * lane;
                const ulonglong2 q0 = *reinterpret_cast<const ulonglong2*>(wq);
                const ulonglong2 q1 = *reinterpret_cast<const ulonglong2*>(wq + 2);
                const uint64_t wv[4] = {q0.x, q0.y, q1.x, q1.y};
                uint64_t rv[4];
                KT kk[4], dd[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    kk[u] = nk(wv[u]);
                    dd[u] = kk[u] - kblk;
                }
                MPSM_CHECK(base + k0 + DJ_CHUNK <= DJ_TW + 3 * DJ_MAXRUNS + 2 * DJ_CHUNK);
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    asm("ld.shared.u64 %0, [%1];" : "=l"(rv[u]) : "r"(rb_addr + 8u * (uint32_t)min(dd[u], nbm1)));
                KT prv = __shfl_up_sync(0xffffffffu, kk[3], 1);
                if (lane == 0) prv = carry;
                carry = __shfl_sync(0xffffffffu, kk[3], 31);
                bool wide = false;
                if (K32 && kmask != 0) {
                    uint32_t hiw = 0;
#pragma unroll
                    for (int u = 0; u < 4; ++u) hiw |= (uint32_t)(wv[u] >> 32) | (uint32_t)(rv[u] >> 32);
                    wide = __any_sync(0xffffffffu, (hiw & kmask) != 0);
                }
                const bool full = rem >= DJ_CHUNK && (k0 > 0 || lead == 0);
                if (!wide) {
                    uint32_t r32[4], s32[4];
                    uint64_t hh[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        r32[u] = K32 ? (uint32_t)rv[u] : (uint32_t)rv[u] & pmask32;
                        s32[u] = K32 ? (uint32_t)wv[u] : (uint32_t)wv[u] & pmask32;
                        hh[u] = SW ? pair_hash32_mix<MPSM_DJ_FMA>(s32[u], r32[u], fk)
                                   : pair_hash32_mix<MPSM_DJ_FMA>(r32[u], s32[u], fk);
                    }
                    if (full) {
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            max33(r32[u], s32[u], b0, b1, h1);
                            if (MPSM_DJ_FMA & 32) csum = mad_mask64(csum, hh[u], fk.one);
                            else csum += hh[u];
                        }
                    } else {
                        const int v0 = k0 + 4 * lane;
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const uint32_t m = (v0 + u >= lead && v0 + u < nv) ? 1u : 0u;
                            max33(r32[u] * m, s32[u] * m, b0, b1, h1);
                            csum = mad_mask64(csum, hh[u], m);
                        }
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        uint64_t h, sm_;
                        agg64(rv[u] & pmask, wv[u] & pmask, h, sm_);
                        const int v = k0 + 4 * lane + u;
                        const uint32_t mu = (full || (v >= lead && v < nv)) ? 1u : 0u;
                        max_into(best, sm_ * mu);
                        csum = mad_mask64(csum, h, mu);
                    }
                }
                if (full) {
                    bad |= (prv > kk[0]) | (kk[0] > kk[1]) | (kk[1] > kk[2]) | (kk[2] > kk[3]);
                    // every gathered R tuple must carry the S key (a private
                    // run that is not dense after all: flagged, not miscounted)
                    bad |= (nk(rv[0]) != kk[0]) | (nk(rv[1]) != kk[1]) | (nk(rv[2]) != kk[2]) | (nk(rv[3]) != kk[3]);
                    cnt += DJ_CHUNK;
                } else {
                    const int v0 = k0 + 4 * lane;
                    KT pv = prv;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int v = v0 + u;
                        bad |= (v < nv && v - 1 >= lo_ok) && pv > kk[u];
                        bad |= (v >= lead && v < nv) && nk(rv[u]) != kk[u];
                        pv = kk[u];
                    }
                    cnt += max(0, min(nv, k0 + DJ_CHUNK) - max(k0, lead));
                }
            }
#else
            for (; c < pe; ++c, k0 += DJ_CHUNK) {
                // DJ_U tuples per lane: element u of lane l is k0 + 32 u + l
                const int rem = n - k0;
                uint64_t wv[DJ_U], rv[DJ_U];
                KT kk[DJ_U], dd[DJ_U], pk[DJ_U];
#pragma unroll
                for (int u = 0; u < DJ_U; ++u) {
                    wv[u] = W[off + k0 + 32 * u + lane];
                    kk[u] = nk(wv[u]);
                    dd[u] = kk[u] - kblk;
                    // the order check: each key against the one before it,
                    // read from the stage (the piece's first tuple has its
                    // staged prior, or none: W[off - 1] is then ignored)
                    pk[u] = nk(W[off + k0 + 32 * u + lane - 1]);
                }
                if (lane == 0 && k0 == 0 && !has) pk[0] = 0;
                MPSM_CHECK(off + k0 + DJ_CHUNK - 32 + lane < DJ_TW + 3 * DJ_MAXRUNS + 2 * DJ_CHUNK);
                // R gathers through a 32-bit shared address (one IMAD each)
#pragma unroll
                for (int u = 0; u < DJ_U; ++u)
                    asm("ld.shared.u64 %0, [%1];" : "=l"(rv[u]) : "r"(rb_addr + 8u * (uint32_t)min(dd[u], nbm1)));
                bool wide = false;
                if (K32 && kmask != 0) {
                    uint32_t hiw = 0;
#pragma unroll
                    for (int u = 0; u < DJ_U; ++u) hiw |= (uint32_t)(wv[u] >> 32) | (uint32_t)(rv[u] >> 32);
                    wide = __any_sync(0xffffffffu, (hiw & kmask) != 0);
                }
                uint64_t hh[DJ_U], ss[DJ_U];
                if (!wide) {
                    // K32 (pw >= 32): the low word is the whole payload
#pragma unroll
                    for (int u = 0; u < DJ_U; ++u)
                        agg32(K32 ? (uint32_t)rv[u] : (uint32_t)rv[u] & pmask32,
                              K32 ? (uint32_t)wv[u] : (uint32_t)wv[u] & pmask32, hh[u], ss[u]);
                } else {
#pragma unroll
                    for (int u = 0; u < DJ_U; ++u) agg64(rv[u] & pmask, wv[u] & pmask, hh[u], ss[u]);
                }
                if (rem >= DJ_CHUNK) {
                    // a full chunk: every tuple matches (a key outside the
                    // block or a step down is a run out of order: flagged)
#pragma unroll
                    for (int u = 0; u < DJ_U; ++u) {
                        bad |= (pk[u] > kk[u]) | (dd[u] > nbm1);
                        max_into(best, ss[u]);
                        if (MPSM_DJ_FMA & 32) csum = mad_mask64(csum, hh[u], fk.one);
                        else csum += hh[u];
                    }
                    cnt += DJ_CHUNK;
                } else {
#pragma unroll
                    for (int u = 0; u < DJ_U; ++u) {
                        const bool v = lane + 32 * u < rem;
                        bad |= v && (pk[u] > kk[u] || dd[u] > nbm1);
                        const uint32_t m = v ? 1u : 0u;
                        max_into(best, ss[u] * m);
                        csum = mad_mask64(csum, hh[u], m);
                    }
                    cnt += rem;
                }
            }
#endif
            if (c < ce) ++p;
        }
        }
        __syncwarp();
        DJ_TS(warp == 0, g, 5)
        DJ_TS(warp == DJ_WARPS - 1, g, 6)
        if (lane == 0) mbar_arrive(&sm.empty[s]);
    }
    flush_regs();
    if (cur_i >= 0) flush_runs(cur_i);
}

// ---------------------------------------------------------------------------
// Dense private runs against public runs, streamed (the FK join at any T):
// every (private run i, public run j) pair whose run i is dense contributes
// the 128-tuple steps of its S window; the steps of all pairs (private-run
// major) are dealt to warps in chunks of DF_CHUNK consecutive steps, chunk k
// to warp k mod W, so the warps sweep the step sequence together and run i's
// records stay in L2 while its T pairs are streamed.  In a step lane l owns
// the 4 consecutive S records 4l..4l+3 (two 16-B loads, the next step's in
// flight while this one is hashed) and gathers each tuple's R record from
// global memory at index key - key(R_i[0]) (S is sorted: a step's R records
// are a few consecutive lines).  No staging, tiles or barriers.  Run order
// check: every adjacent S pair of each window and the pair before it
// (in-lane, one shuffle across lanes, the step before through a carried key
// or one load at a chunk / pair start).  Per-warp COUNT / MAX / checksum go
// to the pair's record with atomics when the warp's pair changes.
//   k_df_plan    per pair: first step index (scan) and aligned window start
//   k_dense_flat the stream
constexpr int DF_THREADS = 256;
#ifndef MPSM_DF_MINB  // resident CTAs per SM the register budget is cut for
#define MPSM_DF_MINB 3
#endif
#ifndef MPSM_DF_CHUNK  // consecutive steps a warp takes at a time
#define MPSM_DF_CHUNK 64
#endif
constexpr int DF_MAXPAIRS = 4096;

struct DfArgs {
    const mpsm_run_t* priv;
    const mpsm_run_t* pub;
    const PairWin* win;
    const uint32_t* nondense;
    const uint64_t* kb;
    int n_priv, n_pub;
    int64_t* pstep;  // [npairs + 1] first step of each pair (exclusive scan)
    int64_t* pb0;    // [npairs] 16-B aligned index at or below the window start
    uint64_t* out_pairs;
    PackInfo pi;
};

__global__ void __launch_bounds__(1024) k_df_plan(DfArgs a) {
    __shared__ int64_t part[32];
    const int np = a.n_priv * a.n_pub;
    constexpr int PER = DF_MAXPAIRS / 1024;
    int64_t v[PER];
    int64_t tot = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int p = threadIdx.x * PER + q;
        int64_t st = 0;
        if (p < np) {
            const PairWin w = a.win[p];
            const int i = p / a.n_pub, j = p - i * a.n_pub;
            if (!a.nondense[i] && w.end > w.start) {
                const int al = (int)(((uintptr_t)a.pub[j].keys >> 3) & 1);
                const int64_t b0 = w.start - ((w.start + al) & 1);
                a.pb0[p] = b0;
                st = (w.end - b0 + 127) >> 7;
            } else {
                a.pb0[p] = 0;
            }
        }
        v[q] = st;
        tot += st;
    }
    // exclusive scan of the per-thread totals
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
    }
    if (lane == 31) part[wid] = incl;
    __syncthreads();
    int64_t run = incl - tot;
    for (int q = 0; q < wid; ++q) run += part[q];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int p = threadIdx.x * PER + q;
        if (p < np) a.pstep[p] = run;
        run += v[q];
    }
    if (threadIdx.x == 1023) a.pstep[np] = run;
}

template <bool K32, bool SW>
__global__ void __launch_bounds__(DF_THREADS, MPSM_DF_MINB) k_dense_flat(DfArgs a) {
    __shared__ uint32_t s_fmak[5];
    const int tid = threadIdx.x, lane = tid & 31;
    if (tid == 0) {
        s_fmak[0] = 1u << 17;
        s_fmak[1] = 1u << 2;
        s_fmak[2] = 1u << 5;
        s_fmak[3] = 1u << 1;
        s_fmak[4] = 1u;
    }
    __syncthreads();
    using KT = typename std::conditional<K32, uint32_t, uint64_t>::type;
    const int np = a.n_priv * a.n_pub;
    const int64_t total = a.pstep[np];
    const int pw = a.pi.pw;
    const uint32_t kmask = a.pi.kmask;
    const uint64_t pmask = a.pi.pmask;
    const uint32_t pmask32 = (uint32_t)pmask;
    auto nk = [&](uint64_t v) -> KT {
        if (K32) return (KT)((uint32_t)(v >> 32) >> (pw - 32));
        return (KT)(v >> pw);
    };
    FmaK fk;
    {
        uint32_t* kp = &fk.m17;
        for (int q = 0; q < 5; ++q)
            asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(kp[q]) : "r"(smem_addr(&s_fmak[q])));
    }
    const int64_t gw = ((int64_t)blockIdx.x * DF_THREADS + tid) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * DF_THREADS) >> 5;
    const int64_t nchunks = (total + MPSM_DF_CHUNK - 1) / MPSM_DF_CHUNK;

    // the warp's current pair and its parameters
    int p = -1;
    int64_t p_first = 0, p_end = 0;  // the pair's steps [p_first, p_end)
    const uint64_t* sk = nullptr;
    const uint64_t* rk = nullptr;
    int64_t sn = 0, b0 = 0, wstart = 0, wend = 0, lo_chk = 0;
    KT kb = 0, nrm1 = 0;
    // per-warp aggregates of pair p
    uint64_t best = 0, csum = 0;
    uint32_t b0m = 0, b1m = 0, h1 = 0;
    int64_t cnt = 0;  // warp-uniform
    bool bad = false;
    auto flush = [&]() {
        if (p < 0) return;
        const uint64_t cb = h1 ? ((1ull << 32) | b1m) : (uint64_t)b0m;
        if (cb > best) best = cb;
        const uint32_t lo = (uint32_t)csum, hi = (uint32_t)(csum >> 32);
        const uint64_t cs = (uint64_t)__reduce_add_sync(0xffffffffu, lo & 0xffffu) +
                            ((uint64_t)__reduce_add_sync(0xffffffffu, lo >> 16) << 16) +
                            ((uint64_t)__reduce_add_sync(0xffffffffu, hi & 0xffffu) << 32) +
                            ((uint64_t)__reduce_add_sync(0xffffffffu, hi >> 16) << 48);
        const uint32_t bh = __reduce_max_sync(0xffffffffu, (uint32_t)(best >> 32));
        const uint32_t bl = __reduce_max_sync(0xffffffffu, (uint32_t)(best >> 32) == bh ? (uint32_t)best : 0u);
        const bool anybad = __any_sync(0xffffffffu, bad);
        if (lane == 0) {
            uint64_t* o = a.out_pairs + (size_t)p * MPSM_PAIR_FIELDS;
            if (cnt) {
                atomicAdd((unsigned long long*)(o + MPSM_PAIR_COUNT), (unsigned long long)cnt);
                atomicMax((unsigned long long*)(o + MPSM_PAIR_BEST), (unsigned long long)(((uint64_t)bh << 32) | bl));
                atomicAdd((unsigned long long*)(o + MPSM_PAIR_CHECKSUM), (unsigned long long)cs);
            }
            if (anybad) atomicOr((unsigned long long*)(o + MPSM_PAIR_FLAGS), (unsigned long long)MPSM_FLAG_UNSORTED);
        }
        best = csum = 0;
        b0m = b1m = h1 = 0;
        cnt = 0;
        bad = false;
    };
    auto enter = [&](int q) {  // make pair q current
        flush();
        p = q;
        p_first = a.pstep[q];
        p_end = a.pstep[q + 1];
        const int i = q / a.n_pub, j = q - i * a.n_pub;
        const mpsm_run_t S = a.pub[j], R = a.priv[i];
        sk = S.keys;
        sn = S.n;
        rk = R.keys;
        nrm1 = (KT)(R.n - 1);
        kb = (KT)a.kb[i];
        b0 = a.pb0[q];
        const PairWin w = a.win[q];
        wstart = w.start;
        wend = w.end;
        lo_chk = wstart > 1 ? wstart : 1;
    };
    auto load4 = [&](int64_t e0, uint64_t* x) {
        if (e0 >= 0 && e0 + 3 < sn) {
            const ulonglong2 u0 = __ldcs(reinterpret_cast<const ulonglong2*>(sk + e0));
            const ulonglong2 u1 = __ldcs(reinterpret_cast<const ulonglong2*>(sk + e0 + 2));
            x[0] = u0.x;
            x[1] = u0.y;
            x[2] = u1.x;
            x[3] = u1.y;
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) x[u] = (e0 + u >= 0 && e0 + u < sn) ? sk[e0 + u] : 0;
        }
    };
    uint64_t nx[4] = {0, 0, 0, 0};
    int64_t pre_step = -1;  // the step whose S nx holds (prefetched across chunks), else -1
    for (int64_t ch = gw; ch < nchunks; ch += nw) {
        const int64_t c0 = ch * MPSM_DF_CHUNK, c1 = min(c0 + MPSM_DF_CHUNK, total);
        // the pair holding step c0 (pairs are visited in increasing order)
        if (p < 0 || c0 >= p_end) {
            int lo = p < 0 ? 0 : p, hi = np - 1;
            while (lo < hi) {  // last q with pstep[q] <= c0
                const int mid = (lo + hi + 1) >> 1;
                if (a.pstep[mid] <= c0) lo = mid;
                else hi = mid - 1;
            }
            while (a.pstep[lo + 1] <= c0) ++lo;  // skip pairs without steps
            if (lo != p) enter(lo);
        }
        int64_t st = c0;
        while (st < c1) {
            if (st >= p_end) {  // the chunk runs into the next pair(s)
                int q = p + 1;
                while (a.pstep[q + 1] <= st) ++q;
                enter(q);
            }
            const int64_t se = min(c1, p_end);  // this chunk's steps of pair p
            // key before the first step here (0: nothing to check)
            int64_t base = b0 + ((st - p_first) << 7);
            KT carry = (base - 1 >= 0) ? nk(sk[base - 1]) : (KT)0;
            if (st != pre_step) load4(base + 4 * lane, nx);  // not prefetched
            pre_step = -1;
            // a segment inside the window (all but a pair's first and last
            // few steps) runs lean: no bounds, masks or 64-bit index math
            const bool inside = base >= lo_chk && b0 + ((se - p_first) << 7) <= wend;
            auto segment = [&](auto lean_tag) {
                constexpr bool LEAN = decltype(lean_tag)::value;
                const uint64_t* sq = sk + base + 4 * lane;
                auto ld16 = [&](const uint64_t* q, uint64_t* x) {
                    const ulonglong2 a0 = __ldcs(reinterpret_cast<const ulonglong2*>(q));
                    const ulonglong2 a1 = __ldcs(reinterpret_cast<const ulonglong2*>(q + 2));
                    x[0] = a0.x;
                    x[1] = a0.y;
                    x[2] = a1.x;
                    x[3] = a1.y;
                };
                for (; st < se; ++st, base += 128) {
                    uint64_t wv[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) wv[u] = nx[u];
                    if (st + 1 < se) {
                        if (LEAN) {
                            sq += 128;
                            ld16(sq, nx);
                        } else {
                            load4(base + 128 + 4 * lane, nx);
                        }
                    } else if (st + 1 == c1) {
                        // the warp's next chunk, when it continues this pair:
                        // its first step's S in flight during this step
                        const int64_t nc = c0 + nw * MPSM_DF_CHUNK;
                        if (nc < p_end) {
                            load4(b0 + ((nc - p_first) << 7) + 4 * lane, nx);
                            pre_step = nc;
                        }
                    }
                    KT kk[4];
                    uint64_t rv[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        kk[u] = nk(wv[u]);
                        const KT d = kk[u] - kb;
#ifdef MPSM_DBG_DF_NO_GATHER
                        rv[u] = wv[u] ^ (uint64_t)d;
#else
                        rv[u] = __ldg(rk + (d < nrm1 ? d : nrm1));
#endif
                    }
                    KT prv = __shfl_up_sync(0xffffffffu, kk[3], 1);
                    if (lane == 0) prv = carry;
                    carry = __shfl_sync(0xffffffffu, kk[3], 31);
                    bool wide = false;
                    if (K32 && kmask != 0) {
                        uint32_t hiw = 0;
#pragma unroll
                        for (int u = 0; u < 4; ++u) hiw |= (uint32_t)(wv[u] >> 32) | (uint32_t)(rv[u] >> 32);
                        wide = __any_sync(0xffffffffu, (hiw & kmask) != 0);
                    }
                    const bool full = LEAN || (base >= lo_chk && base + 128 <= wend);
                    if (!wide) {
                        uint32_t r32[4], s32[4];
                        uint64_t hh[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            r32[u] = K32 ? (uint32_t)rv[u] : (uint32_t)rv[u] & pmask32;
                            s32[u] = K32 ? (uint32_t)wv[u] : (uint32_t)wv[u] & pmask32;
#ifdef MPSM_DBG_DF_NO_HASH
                            hh[u] = (uint64_t)r32[u] * s32[u];
#else
                            hh[u] = SW ? pair_hash32_mix<MPSM_DJ_FMA>(s32[u], r32[u], fk)
                                       : pair_hash32_mix<MPSM_DJ_FMA>(r32[u], s32[u], fk);
#endif
                        }
                        if (full) {
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                max33(r32[u], s32[u], b0m, b1m, h1);
                                if (MPSM_DJ_FMA & 32) csum = mad_mask64(csum, hh[u], fk.one);
                                else csum += hh[u];
                            }
                        } else {
                            const int64_t v0 = base + 4 * lane;
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const uint32_t m = (v0 + u >= wstart && v0 + u < wend) ? 1u : 0u;
                                max33(r32[u] * m, s32[u] * m, b0m, b1m, h1);
                                csum = mad_mask64(csum, hh[u], m);
                            }
                        }
                    } else {
                        const int64_t v0 = base + 4 * lane;
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const uint64_t rp = rv[u] & pmask, sp = wv[u] & pmask;
                            const uint64_t h = SW ? pair_hash(sp, rp) : pair_hash(rp, sp);
                            const uint32_t m = (full || (v0 + u >= wstart && v0 + u < wend)) ? 1u : 0u;
                            max_into(best, (rp + sp) * m);
                            csum = mad_mask64(csum, h, m);
                        }
                    }
                    if (full) {
                        bad |= (prv > kk[0]) | (kk[0] > kk[1]) | (kk[1] > kk[2]) | (kk[2] > kk[3]);
                    // every gathered R tuple must carry the S key (a private
                    // run that is not dense after all: flagged, not miscounted)
                    bad |= (nk(rv[0]) != kk[0]) | (nk(rv[1]) != kk[1]) | (nk(rv[2]) != kk[2]) | (nk(rv[3]) != kk[3]);
                        cnt += 128;
                    } else {
                        const int64_t v0 = base + 4 * lane;
                        KT pv = prv;
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int64_t v = v0 + u;
                            bad |= (v >= lo_chk && v < wend) && pv > kk[u];
                            bad |= (v >= wstart && v < wend) && nk(rv[u]) != kk[u];
                            pv = kk[u];
                        }
                        cnt += max((int64_t)0, min(wend, base + 128) - max(wstart, base));
                    }
                }
            };
            if (inside) segment(std::true_type{});
            else segment(std::false_type{});
        }
    }
    flush();
}

template <bool K32>
static int launch_dense_flat(const DfArgs& a, int swap, cudaStream_t st) {
    static int per_sm = 0;
    if (!per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dense_flat<K32, false>, DF_THREADS, 0);
        if (per_sm < 1) per_sm = 1;
    }
    const int grid = num_sms() * per_sm;
    ProfScope ps("dense_join", st);
    k_df_plan<<<1, 1024, 0, st>>>(a);
    MPSM_TRY(check_launch("k_df_plan"));
    if (swap) k_dense_flat<K32, true><<<grid, DF_THREADS, 0, st>>>(a);
    else k_dense_flat<K32, false><<<grid, DF_THREADS, 0, st>>>(a);
    return check_launch("k_dense_flat");
}

// One pair (T = 1): each warp streams one contiguous range of steps (no
// chunk dealing or pair lookup; S prefetched one step ahead in registers).
// Measured (FK 100M x 400M): 1.05 ms vs 1.12-1.15 for the dealt-chunk kernel
// on the same pair; S loads two steps ahead 1.08-1.10, a per-warp cp.async
// ring 1.21-1.33, the R gather issued one step ahead 1.20-1.60 (spills or
// fewer warps).  Bounds: the S stream alone 0.56 ms (5.7 TB/s), + the R
// gather 0.80, + the hash 0.90 (MPSM_DBG_DF_NO_GATHER / _NO_HASH in the
// dealt kernel).
template <bool K32, bool SW>
__global__ void __launch_bounds__(DF_THREADS, 4) k_dense_flat1(const mpsm_run_t* __restrict__ priv,
                                                           const mpsm_run_t* __restrict__ pub,
                                                           const PairWin* __restrict__ win,
                                                           const uint32_t* __restrict__ nondense,
                                                           const uint64_t* __restrict__ kbp, PackInfo pi,
                                                           uint64_t* __restrict__ out_pairs) {
    __shared__ unsigned long long s_cnt, s_best, s_csum;
    __shared__ unsigned s_bad;
    __shared__ uint32_t s_fmak[5];
    const int tid = threadIdx.x, lane = tid & 31;
    if (tid == 0) {
        s_cnt = s_best = s_csum = 0;
        s_bad = 0;
        s_fmak[0] = 1u << 17;
        s_fmak[1] = 1u << 2;
        s_fmak[2] = 1u << 5;
        s_fmak[3] = 1u << 1;
        s_fmak[4] = 1u;
    }
    __syncthreads();
    if (nondense[0]) return;
    const PairWin w = win[0];
    if (w.end <= w.start) return;
    using KT = typename std::conditional<K32, uint32_t, uint64_t>::type;
    const mpsm_run_t R = priv[0], S = pub[0];
    const uint64_t* __restrict__ sk = S.keys;
    const uint64_t* __restrict__ rk = R.keys;
    const int pw = pi.pw;
    const uint32_t kmask = pi.kmask;
    const uint64_t pmask = pi.pmask;
    const uint32_t pmask32 = (uint32_t)pmask;
    auto nk = [&](uint64_t v) -> KT {
        if (K32) return (KT)((uint32_t)(v >> 32) >> (pw - 32));
        return (KT)(v >> pw);
    };
    const KT kb = (KT)kbp[0];
    const KT nrm1 = (KT)(R.n - 1);
    FmaK fk;
    {
        uint32_t* kp = &fk.m17;
        for (int q = 0; q < 5; ++q)
            asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(kp[q]) : "r"(smem_addr(&s_fmak[q])));
    }
    // step grid from the 16-B aligned index at or below the window start
    const int64_t n = S.n;
    const int al = (int)(((uintptr_t)sk >> 3) & 1);
    const int64_t b0 = w.start - ((w.start + al) & 1);
    const int64_t nsteps = (w.end - b0 + 127) >> 7;
    const int64_t gw = ((int64_t)blockIdx.x * DF_THREADS + tid) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * DF_THREADS) >> 5;
    const int64_t s0 = nsteps * gw / nw, s1 = nsteps * (gw + 1) / nw;
    const int64_t lo_chk = w.start > 1 ? w.start : 1;  // pairs (v - 1, v) checked for v >= lo_chk
    auto load4 = [&](int64_t e0, uint64_t* x) {
        if (e0 >= 0 && e0 + 3 < n) {
            const ulonglong2 a = __ldcs(reinterpret_cast<const ulonglong2*>(sk + e0));
            const ulonglong2 b = __ldcs(reinterpret_cast<const ulonglong2*>(sk + e0 + 2));
            x[0] = a.x;
            x[1] = a.y;
            x[2] = b.x;
            x[3] = b.y;
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) x[u] = (e0 + u >= 0 && e0 + u < n) ? sk[e0 + u] : 0;
        }
    };
    uint64_t best = 0, csum = 0;
    uint32_t b0m = 0, b1m = 0, h1 = 0;
    int64_t cnt = 0;  // warp-uniform
    bool bad = false;
    KT carry = 0;
    if (s0 < s1) {
        const int64_t first = b0 + (s0 << 7);
        if (first - 1 >= 0) carry = nk(sk[first - 1]);
    }
    // a warp whose steps all lie inside the window (every warp but the
    // first and the last) runs the lean loop: no bounds or window masks, S
    // through a running pointer
    const bool interior = s0 < s1 && b0 + (s0 << 7) >= lo_chk && b0 + (s1 << 7) <= w.end;
    auto run = [&](auto lean_tag) {
        constexpr bool LEAN = decltype(lean_tag)::value;
        const uint64_t* sq = sk + b0 + (s0 << 7) + 4 * lane;  // LEAN: this lane's records of the current step
        uint64_t nx[4];
        auto ld16 = [&](const uint64_t* q, uint64_t* x) {
            const ulonglong2 a0 = __ldcs(reinterpret_cast<const ulonglong2*>(q));
            const ulonglong2 a1 = __ldcs(reinterpret_cast<const ulonglong2*>(q + 2));
            x[0] = a0.x;
            x[1] = a0.y;
            x[2] = a1.x;
            x[3] = a1.y;
        };
        if (s0 < s1) {
            if (LEAN) ld16(sq, nx);
            else load4(b0 + (s0 << 7) + 4 * lane, nx);
        }
        for (int64_t st = s0; st < s1; ++st) {
            const int64_t base = b0 + (st << 7);
            uint64_t wv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) wv[u] = nx[u];
            if (st + 1 < s1) {
                if (LEAN) {
                    sq += 128;
                    ld16(sq, nx);
                } else {
                    load4(base + 128 + 4 * lane, nx);
                }
            }
            KT kk[4];
            uint64_t rv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                kk[u] = nk(wv[u]);
                const KT d = kk[u] - kb;
                rv[u] = __ldg(rk + (d < nrm1 ? d : nrm1));
            }
            KT prv = __shfl_up_sync(0xffffffffu, kk[3], 1);
            if (lane == 0) prv = carry;
            carry = __shfl_sync(0xffffffffu, kk[3], 31);
            bool wide = false;
            if (K32 && kmask != 0) {
                uint32_t hiw = 0;
#pragma unroll
                for (int u = 0; u < 4; ++u) hiw |= (uint32_t)(wv[u] >> 32) | (uint32_t)(rv[u] >> 32);
                wide = __any_sync(0xffffffffu, (hiw & kmask) != 0);
            }
            const bool full = LEAN || (base >= lo_chk && base + 128 <= w.end);
            if (!wide) {
                uint32_t r32[4], s32[4];
                uint64_t hh[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    r32[u] = K32 ? (uint32_t)rv[u] : (uint32_t)rv[u] & pmask32;
                    s32[u] = K32 ? (uint32_t)wv[u] : (uint32_t)wv[u] & pmask32;
                    hh[u] = SW ? pair_hash32_mix<MPSM_DJ_FMA>(s32[u], r32[u], fk)
                               : pair_hash32_mix<MPSM_DJ_FMA>(r32[u], s32[u], fk);
                }
                if (full) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        max33(r32[u], s32[u], b0m, b1m, h1);
                        if (MPSM_DJ_FMA & 32) csum = mad_mask64(csum, hh[u], fk.one);
                        else csum += hh[u];
                    }
                } else {
                    const int64_t v0 = base + 4 * lane;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const uint32_t m = (v0 + u >= w.start && v0 + u < w.end) ? 1u : 0u;
                        max33(r32[u] * m, s32[u] * m, b0m, b1m, h1);
                        csum = mad_mask64(csum, hh[u], m);
                    }
                }
            } else {
                const int64_t v0 = base + 4 * lane;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint64_t rp = rv[u] & pmask, sp = wv[u] & pmask;
                    const uint64_t h = SW ? pair_hash(sp, rp) : pair_hash(rp, sp);
                    const uint32_t m = (full || (v0 + u >= w.start && v0 + u < w.end)) ? 1u : 0u;
                    max_into(best, (rp + sp) * m);
                    csum = mad_mask64(csum, h, m);
                }
            }
            if (full) {
                bad |= (prv > kk[0]) | (kk[0] > kk[1]) | (kk[1] > kk[2]) | (kk[2] > kk[3]);
                    // every gathered R tuple must carry the S key (a private
                    // run that is not dense after all: flagged, not miscounted)
                    bad |= (nk(rv[0]) != kk[0]) | (nk(rv[1]) != kk[1]) | (nk(rv[2]) != kk[2]) | (nk(rv[3]) != kk[3]);
                cnt += 128;
            } else {
                const int64_t v0 = base + 4 * lane;
                KT pv = prv;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int64_t v = v0 + u;
                    bad |= (v >= lo_chk && v < w.end) && pv > kk[u];
                    bad |= (v >= w.start && v < w.end) && nk(rv[u]) != kk[u];
                    pv = kk[u];
                }
                cnt += max((int64_t)0, min(w.end, base + 128) - max(w.start, base));
            }
        }
    };
    if (interior) run(std::true_type{});
    else run(std::false_type{});
    {
        const uint64_t cb = h1 ? ((1ull << 32) | b1m) : (uint64_t)b0m;
        if (cb > best) best = cb;
    }
    const uint32_t lo = (uint32_t)csum, hi = (uint32_t)(csum >> 32);
    const uint64_t cs = (uint64_t)__reduce_add_sync(0xffffffffu, lo & 0xffffu) +
                        ((uint64_t)__reduce_add_sync(0xffffffffu, lo >> 16) << 16) +
                        ((uint64_t)__reduce_add_sync(0xffffffffu, hi & 0xffffu) << 32) +
                        ((uint64_t)__reduce_add_sync(0xffffffffu, hi >> 16) << 48);
    const uint32_t bh = __reduce_max_sync(0xffffffffu, (uint32_t)(best >> 32));
    const uint32_t bl = __reduce_max_sync(0xffffffffu, (uint32_t)(best >> 32) == bh ? (uint32_t)best : 0u);
    const bool anybad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
        if (cnt) {
            atomicAdd(&s_cnt, (unsigned long long)cnt);
            atomicMax(&s_best, (unsigned long long)(((uint64_t)bh << 32) | bl));
            atomicAdd(&s_csum, (unsigned long long)cs);
        }
        if (anybad) atomicOr(&s_bad, 1u);
    }
    __syncthreads();
    if (tid == 0) {
        if (s_cnt) {
            atomicAdd((unsigned long long*)(out_pairs + MPSM_PAIR_COUNT), s_cnt);
            atomicMax((unsigned long long*)(out_pairs + MPSM_PAIR_BEST), s_best);
            atomicAdd((unsigned long long*)(out_pairs + MPSM_PAIR_CHECKSUM), s_csum);
        }
        if (s_bad) atomicOr((unsigned long long*)(out_pairs + MPSM_PAIR_FLAGS), (unsigned long long)MPSM_FLAG_UNSORTED);
    }
}

template <bool K32>
static int launch_dense_flat1(const mpsm_run_t* d_priv, const mpsm_run_t* d_pub, const PairWin* win,
                             const uint32_t* nondense, const uint64_t* kb, const PackInfo& pi, uint64_t* d_pairs,
                             int swap, cudaStream_t st) {
    static int per_sm = 0;
    if (!per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dense_flat1<K32, false>, DF_THREADS, 0);
        if (per_sm < 1) per_sm = 1;
    }
    const int grid = num_sms() * per_sm;
    ProfScope ps("dense_join", st);
    if (swap) k_dense_flat1<K32, true><<<grid, DF_THREADS, 0, st>>>(d_priv, d_pub, win, nondense, kb, pi, d_pairs);
    else k_dense_flat1<K32, false><<<grid, DF_THREADS, 0, st>>>(d_priv, d_pub, win, nondense, kb, pi, d_pairs);
    return check_launch("k_dense_flat1");
}

// MPSM_DENSE_FLAT=0 selects the staged k_dense_join instead (read per call:
// the tests run both paths in one process)
static bool df_enabled() {
    const char* e = getenv("MPSM_DENSE_FLAT");
    return !(e && e[0] == '0');
}

static bool dj_enabled() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("MPSM_DENSE_JOIN");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}

// host plan of the dense-run path: block size, entries, tile bound
struct DjPlan {
    bool on = false;
    int64_t K = 0, nent = 0, maxt = 0, nparts = 0;
    std::vector<int64_t> blk_base;
};
static DjPlan dj_plan(const mpsm_run_t* priv, int n_priv, const mpsm_run_t* pub, int n_pub) {
    DjPlan p;
    if (!dj_enabled() || n_priv < 1 || n_pub < 1 || n_priv > DJ_MAXRUNS || n_pub > DJ_MAXRUNS) return p;
    int64_t nr = 0, ns = 0;
    for (int i = 0; i < n_priv; ++i) nr += priv[i].n;
    for (int j = 0; j < n_pub; ++j) ns += pub[j].n;
    // the largest blocks: fewer bound searches, full tiles (a block's S
    // tuples split into tiles of DJ_TW), larger pieces per public run
    // (A/B, FK 100M x 400M: K = 819 / 1024 / 2048 -> join 1.57 / 1.63 / 1.46
    // ms at T = 1, 2.47 / 2.51 / 2.07 ms at T = 16)
    double k = DJ_KMAX;
    if (const char* ev = getenv("MPSM_DJ_K")) k = atof(ev);
    (void)nr;
    (void)ns;
    p.K = std::min<int64_t>(DJ_KMAX, std::max<int64_t>(64, (int64_t)std::min(k, (double)DJ_KMAX) & ~(int64_t)15));
    p.blk_base.resize(n_priv + 1);
    int64_t e = 0;
    for (int i = 0; i < n_priv; ++i) {
        p.blk_base[i] = e;
        e += (std::max<int64_t>(priv[i].n, 0) + p.K - 1) / p.K + 1;
    }
    p.blk_base[n_priv] = e;
    p.nent = e;
    p.nparts = (e + 1023) / 1024;
    // a tile per entry plus one per DJ_TW S tuples of the windows (each
    // private run's windows hold at most all of S)
    p.maxt = e + ((int64_t)n_priv * ns + DJ_TW - 1) / DJ_TW + 1;
    p.on = p.maxt < (int64_t)INT32_MAX && e < (int64_t)INT32_MAX;
    return p;
}

struct DjWs {
    uint32_t* nondense;
    uint64_t* kb;
    int64_t* blk_base;
    int64_t* L;
    int64_t* tb;
    int32_t* nsub;
    int64_t* part;
    DjTile* tiles;
    int64_t* ntiles;
    int64_t* pstep;  // streamed path: [npairs + 1]
    int64_t* pb0;    // streamed path: [npairs]
};
static bool carve_dj(Carve& c, int n_priv, int n_pub, const DjPlan& p, DjWs* o) {
    o->nondense = c.take<uint32_t>(n_priv);
    o->kb = c.take<uint64_t>(n_priv);
    o->blk_base = c.take<int64_t>(n_priv + 1);
    o->L = c.take<int64_t>((size_t)p.nent * n_pub);
    o->tb = c.take<int64_t>(p.nent + 1);
    o->nsub = c.take<int32_t>(p.nent);
    o->part = c.take<int64_t>(p.nparts + 1);
    o->tiles = c.take<DjTile>(p.maxt);
    o->ntiles = c.take<int64_t>(1);
    o->pstep = c.take<int64_t>((size_t)n_priv * n_pub + 1);
    o->pb0 = c.take<int64_t>((size_t)n_priv * n_pub);
    return c.ok;
}

static size_t join_ws_size(const mpsm_run_t* priv, int n_priv, const mpsm_run_t* pub, int n_pub) {
    const int64_t mt = max_tiles(priv, n_priv, pub, n_pub);
    Carve c{nullptr, (size_t)-1};
    JoinWs w;
    carve_join(c, n_priv, n_pub, mt, &w);
    const DjPlan dp = dj_plan(priv, n_priv, pub, n_pub);
    if (dp.on) {
        DjWs d;
        carve_dj(c, n_priv, n_pub, dp, &d);
    }
    return c.off;
}

template <bool K32>
static int launch_dense(const DjArgs& a, int swap, cudaStream_t st) {
    static int attr = 0;
    if (!attr) {
        MPSM_TRY(cuda_status(cudaFuncSetAttribute(k_dense_join<K32, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)sizeof(DjSmem)),
                             "smem attr"));
        MPSM_TRY(cuda_status(cudaFuncSetAttribute(k_dense_join<K32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)sizeof(DjSmem)),
                             "smem attr"));
        attr = 1;
    }
    const int grid = num_sms() * MPSM_DJ_CTAS;
    ProfScope ps("dense_join", st);
    if (swap) k_dense_join<K32, true><<<grid, DJ_THREADS, sizeof(DjSmem), st>>>(a);
    else k_dense_join<K32, false><<<grid, DJ_THREADS, sizeof(DjSmem), st>>>(a);
    return check_launch("k_dense_join");
}

template <bool PK>
static int join_pairs_impl(const mpsm_run_t* priv, int n_priv, const mpsm_run_t* pub, int n_pub, int swap, int mode,
                           uint64_t* d_out, int64_t cap, uint64_t* d_pairs, void* workspace, size_t ws_bytes,
                           const PackInfo& pi, cudaStream_t st, const uint32_t* hint = nullptr,
                           const uint64_t* hbase = nullptr, int64_t hn = 0) {
    if (n_priv < 1 || n_pub < 1 || !d_pairs) return MPSM_ERR_ARG;
    if (mode == MPSM_MODE_MATERIALIZE && d_out && cap < 0) return MPSM_ERR_ARG;
    if (mode < 0 || mode > 2) return MPSM_ERR_ARG;
    const int npairs = n_priv * n_pub;
    const int64_t mt = max_tiles(priv, n_priv, pub, n_pub);
    JoinWs w;
    Carve cv{(char*)workspace, ws_bytes};
    if (!carve_join(cv, n_priv, n_pub, mt, &w)) {
        set_error("join workspace too small");
        return MPSM_ERR_ARG;
    }
    // the dense-run path: aggregates over packed records (the materialize
    // modes walk the merge tiles of every pair)
    DjPlan dp = dj_plan(priv, n_priv, pub, n_pub);
    DjWs dw{};
    const bool dense = PK && dp.on && (mode != MPSM_MODE_MATERIALIZE || d_out == nullptr) &&
                       carve_dj(cv, n_priv, n_pub, dp, &dw);
    // the run descriptors (and the dense plan's block bases and flags) as
    // one small-put kernel when they fit its parameters
    PutBatch pb;
    MPSM_TRY(put_or_copy(pb, w.d_priv, priv, sizeof(mpsm_run_t) * n_priv, st));
    MPSM_TRY(put_or_copy(pb, w.d_pub, pub, sizeof(mpsm_run_t) * n_pub, st));
    DjArgs da{};
    if (dense) {
        MPSM_TRY(put_or_copy(pb, dw.blk_base, dp.blk_base.data(), sizeof(int64_t) * (n_priv + 1), st));
        MPSM_TRY(put_or_copy(pb, dw.nondense, nullptr, sizeof(uint32_t) * n_priv, st));
    }
    MPSM_TRY(put_flush(pb, st));
    if (dense) {
        da = DjArgs{w.d_priv, w.d_pub, n_priv,   n_pub,   dp.K,      dp.nent,   dw.nondense, dw.kb,     dw.blk_base,
                    w.win,    dw.L,    dw.tb,    dw.nsub, dw.part,   dw.tiles,  dw.ntiles,   d_pairs,   pi};
        ProfScope ps("dense_check", st);
        const dim3 grid((unsigned)std::max(1, num_sms() * 4 / n_priv), (unsigned)n_priv);
        k_dense_check<<<grid, 256, 0, st>>>(w.d_priv, pi.pw, dw.nondense, dw.kb, hint, hbase, hn);
        MPSM_TRY(check_launch("k_dense_check"));
    }
    k_windows<PK><<<(npairs + 127) / 128, 128, 0, st>>>(w.d_priv, n_priv, w.d_pub, n_pub, w.win, d_pairs, pi,
                                                        dense ? dw.nondense : nullptr);
    MPSM_TRY(check_launch("k_windows"));
    if (dense && df_enabled() && npairs <= DF_MAXPAIRS) {
        // the streamed path (no tile plan)
        const DfArgs fa{w.d_priv, w.d_pub, w.win, dw.nondense, dw.kb, n_priv, n_pub, dw.pstep, dw.pb0, d_pairs, pi};
        const bool k32f = (64 - pi.pw) <= 32;
        if (npairs == 1) {
            if (k32f) MPSM_TRY(launch_dense_flat1<true>(w.d_priv, w.d_pub, w.win, dw.nondense, dw.kb, pi, d_pairs, swap, st));
            else MPSM_TRY(launch_dense_flat1<false>(w.d_priv, w.d_pub, w.win, dw.nondense, dw.kb, pi, d_pairs, swap, st));
        } else if (k32f) {
            MPSM_TRY(launch_dense_flat<true>(fa, swap, st));
        } else {
            MPSM_TRY(launch_dense_flat<false>(fa, swap, st));
        }
    } else if (dense) {
        {
            ProfScope ps("dense_tiles", st);
            const int64_t nb = dp.nent * n_pub;
            {
                ProfScope ps1("dense_bounds", st);
                k_blk_bounds<true><<<(unsigned)((nb + 255) / 256), 256, 0, st>>>(da);
                MPSM_TRY(check_launch("k_blk_bounds"));
                k_blk_bounds<false><<<(unsigned)((nb + 255) / 256), 256, 0, st>>>(da);
                MPSM_TRY(check_launch("k_blk_bounds"));
            }
            {
                ProfScope ps2("dense_count", st);
                k_blk_count<<<(unsigned)dp.nparts, 1024, 0, st>>>(da);
                MPSM_TRY(check_launch("k_blk_count"));
            }
            k_scan_i64<<<1, 1024, 0, st>>>(dw.part, dp.nparts, dw.ntiles);
            MPSM_TRY(check_launch("k_scan_i64"));
            k_blk_tiles<<<(unsigned)((dp.nent + 255) / 256), 256, 0, st>>>(da);
            MPSM_TRY(check_launch("k_blk_tiles"));
        }
        const bool k32d = (64 - pi.pw) <= 32;
        if (k32d) MPSM_TRY(launch_dense<true>(da, swap, st));
        else MPSM_TRY(launch_dense<false>(da, swap, st));
    }
    k_tile_scan<<<1, 1024, 0, st>>>(w.win, npairs, w.total);
    MPSM_TRY(check_launch("k_tile_scan"));
    {
        ProfScope ps("merge_partition", st);
        const unsigned pg = (unsigned)((mt + 255) / 256);
        k_part_coarse<PK><<<pg, 256, 0, st>>>(w.d_priv, w.d_pub, n_pub, w.win, npairs, w.total, w.tile_cnt, pi);
        k_partition<PK><<<pg, 256, 0, st>>>(w.d_priv, w.d_pub, n_pub, w.win, npairs, w.total, w.tile_cnt, w.splits,
                                            pi);
        k_split_fill<<<pg, 256, 0, st>>>(w.d_priv, n_pub, w.win, w.total, w.splits);
    }
    MPSM_TRY(check_launch("k_partition"));
    const bool k32 = PK && (64 - pi.pw) <= 32;  // packed keys fit 32 bits
    if (k32) MPSM_TRY((launch_merge<0, PK, PK>(w, swap, d_pairs, nullptr, 0, mt, pi, st)));
    else MPSM_TRY((launch_merge<0, PK>(w, swap, d_pairs, nullptr, 0, mt, pi, st)));
    if (mode != MPSM_MODE_MATERIALIZE || d_out == nullptr) return MPSM_OK;
    // materialize: per-tile counts, offsets, emission
    MPSM_TRY((launch_merge<1, PK>(w, swap, d_pairs, nullptr, 0, mt, pi, st)));
    k_emit_offsets<<<1, 1024, 0, st>>>(w.tile_cnt, w.splits, w.total, d_pairs, cap, w.grand);
    MPSM_TRY(check_launch("k_emit_offsets"));
    return launch_merge<2, PK>(w, swap, d_pairs, d_out, cap, mt, pi, st);
}

}  // namespace mpsm

using namespace mpsm;

extern "C" int mpsm_interp_lower_bound(const uint64_t* keys, int64_t n, const uint64_t* d_targets, int64_t ntargets,
                                       int64_t* d_index, int64_t* d_probes, void* stream) {
    if (n < 0 || ntargets < 0) return MPSM_ERR_ARG;
    if (ntargets == 0) return MPSM_OK;
    k_interp_batch<<<(unsigned)((ntargets + 127) / 128), 128, 0, (cudaStream_t)stream>>>(keys, n, d_targets, ntargets,
                                                                                        d_index, d_probes);
    return check_launch("k_interp_batch");
}

#ifdef MPSM_DBG_TIMING
extern "C" int mpsm_dbg_mj_ts(long long* host, int ntiles) {
    return cuda_status(cudaMemcpyFromSymbol(host, g_mj_ts, sizeof(long long) * 6 * (size_t)ntiles), "dbg");
}
#endif

extern "C" int mpsm_join_workspace_bytes(const mpsm_run_t* priv, int n_priv, const mpsm_run_t* pub, int n_pub,
                                         size_t* bytes) {
    if (!bytes || n_priv < 0 || n_pub < 0) return MPSM_ERR_ARG;
    *bytes = join_ws_size(priv, n_priv, pub, n_pub);
    return MPSM_OK;
}

extern "C" int mpsm_join_pairs(const mpsm_run_t* priv, int n_priv, const mpsm_run_t* pub, int n_pub, int swap,
                               int mode, uint64_t* d_out, int64_t cap, uint64_t* d_pairs, void* workspace,
                               size_t ws_bytes, void* stream) {
    return join_pairs_impl<false>(priv, n_priv, pub, n_pub, swap, mode, d_out, cap, d_pairs, workspace, ws_bytes,
                                  PackInfo{0, 0, 0, 0}, (cudaStream_t)stream);
}

extern "C" int mpsm_join_pairs_packed(const mpsm_run_t* priv, int n_priv, const mpsm_run_t* pub, int n_pub,
                                      int width_bits, uint64_t lower, int swap, int mode, uint64_t* d_out, int64_t cap,
                                      uint64_t* d_pairs, void* workspace, size_t ws_bytes, void* stream) {
    if (width_bits < 1 || width_bits > 63) return MPSM_ERR_ARG;
    const int pw = 64 - width_bits;
    return join_pairs_impl<true>(priv, n_priv, pub, n_pub, swap, mode, d_out, cap, d_pairs, workspace, ws_bytes,
                                 PackInfo{pw, lower, (1ull << pw) - 1, pw >= 32 ? (1u << (pw - 32)) - 1u : 0u},
                                 (cudaStream_t)stream);
}

extern "C" int mpsm_join_pairs_packed_hint(const mpsm_run_t* priv, int n_priv, const mpsm_run_t* pub, int n_pub,
                                           int width_bits, uint64_t lower, int swap, int mode, uint64_t* d_out,
                                           int64_t cap, uint64_t* d_pairs, void* workspace, size_t ws_bytes,
                                           const uint32_t* d_dense, const uint64_t* priv_base, int64_t priv_n,
                                           void* stream) {
    if (width_bits < 1 || width_bits > 63 || priv_n < 0 || (d_dense && priv_n > 0 && !priv_base)) {
        set_error("mpsm_join_pairs_packed_hint: bad width, private length or missing base");
        return MPSM_ERR_ARG;
    }
    if (priv_n == 0) d_dense = nullptr;  // nothing to hint
    const int pw = 64 - width_bits;
    return join_pairs_impl<true>(priv, n_priv, pub, n_pub, swap, mode, d_out, cap, d_pairs, workspace, ws_bytes,
                                 PackInfo{pw, lower, (1ull << pw) - 1, pw >= 32 ? (1u << (pw - 32)) - 1u : 0u},
                                 (cudaStream_t)stream, d_dense, priv_base, priv_n);
}
