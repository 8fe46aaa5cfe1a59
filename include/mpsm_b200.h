/*
 * mpsm_b200.h -- C ABI of the B200-native MPSM join path.
 *
 * This is the drop-in boundary: plain pointers, sizes and status codes, no
 * torch or CUDA runtime types in the signatures (streams travel as void*,
 * they are cudaStream_t).  Every pointer argument named d_* or documented as
 * "device" is device memory owned by the caller; workspace is caller-
 * allocated after a *_workspace_bytes() query (two-phase, CUB style).
 * All compute calls are stream-ordered and asynchronous unless stated.
 *
 * Each entry point replaces one operator of the reference package
 * /root/reference/pkg/src/mpsm (cited per function).  The reference operator
 * layer is its numba kernel module (_kernels.py); its "FFI" is numba's
 * njit call boundary: 1-D contiguous uint64 arrays + scalar u64/int64 args,
 * results as ints/tuples and in-place mutation of output arrays
 * (SURVEY.md 8(b)).  INTEGRATION.md shows the ctypes binding
 * (paper_1207_0145_b200/_lib.py) a maintainer adds on the reference side.
 */
#ifndef MPSM_B200_H
#define MPSM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (map to the reference's exceptions, core.py:26-49) ---- */
#define MPSM_OK 0
#define MPSM_ERR_DOMAIN (-1)   /* DomainError                                   */
#define MPSM_ERR_INTERNAL (-2) /* InternalConsistencyError                      */
#define MPSM_ERR_CONFIG (-3)   /* ConfigurationError                            */
#define MPSM_ERR_CUDA (-4)     /* RuntimeError (CUDA / NCCL failure)            */
#define MPSM_ERR_CAP (-5)      /* MaterializeCapExceeded                        */
#define MPSM_ERR_ARG (-6)      /* ValueError (bad argument)                     */
#define MPSM_ERR_FORMAT (-7)   /* FormatError (malformed relation file)         */
#define MPSM_ERR_IO (-8)       /* OSError (file could not be opened / read)     */

/* query modes (core.py:23) */
#define MPSM_MODE_AGGREGATE_MAX 0
#define MPSM_MODE_COUNT 1
#define MPSM_MODE_MATERIALIZE 2

/* per (private run, public run) result record written by mpsm_join_pairs,
 * MPSM_PAIR_FIELDS uint64 words each */
#define MPSM_PAIR_COUNT 0    /* matched pairs                                  */
#define MPSM_PAIR_BEST 1     /* max(r_pay + s_pay) mod 2^64, valid iff count>0 */
#define MPSM_PAIR_CHECKSUM 2 /* sum splitmix64(r_pay ^ rotl(s_pay,17))         */
#define MPSM_PAIR_START 3    /* lower bound of the private run's first key     */
#define MPSM_PAIR_PROBES 4   /* interpolation-search positions read            */
#define MPSM_PAIR_END 5      /* upper bound of the private run's last key      */
#define MPSM_PAIR_EXAMINED 6 /* distinct public positions the merge scan reads */
#define MPSM_PAIR_EMITTED 7  /* pairs written (materialize, at most the cap)   */
#define MPSM_PAIR_FLAGS 8    /* MPSM_FLAG_* bits found by the merge            */
#define MPSM_PAIR_FIELDS 9

/* MPSM_PAIR_FLAGS bits */
#define MPSM_FLAG_UNSORTED 1 /* a run the merge walked is not sorted ascending
                                (the reference's Run invariant, core.py:153-154) */

/* a sorted run or a relation chunk in device memory */
typedef struct {
    const uint64_t* keys;
    const uint64_t* pays;
    int64_t n;
} mpsm_run_t;

/* ------------------------------------------------------------ library ---- */
int mpsm_version(void);
/* last error message of the calling thread ("" if none) */
const char* mpsm_last_error(void);
/* select the device and check it is sm_100 (B200); returns SM count or <0 */
int mpsm_device_init(int device);
/* number of kernels this library launched (process-wide counter) */
uint64_t mpsm_launch_count(void);
/* copy words_a uint64 from src_a then words_b from src_b (device memory) to
 * host_dst, which must be pinned host memory (cudaHostAlloc / torch
 * pin_memory), by a kernel on `stream` -- a join's pair records and flags
 * without a copy-engine hand-off (meant for small results: every word
 * crosses PCIe as a posted write).  Synchronise the stream before reading
 * host_dst. */
int mpsm_fetch_small(void* host_dst, const void* src_a, int64_t words_a, const void* src_b, int64_t words_b,
                     void* stream);
/* per-kernel CUDA-event timing: enable (and reset) / read the summed device
 * time and launch count of one kernel family ("seg_scatter", "seg_count",
 * "seg_scatter_sp", "seg_scatter_pp", "merge", "merge_partition", ...) */
int mpsm_profile_enable(int on);
int mpsm_profile_read(const char* name, double* total_ms, uint64_t* launches);

/* ---------------------------------------------------------- run sort ----
 * Replaces _kernels.three_phase_sort (_kernels.py:217-244) as called by
 * sorter.sort_run_with_stats (sorter.py:91-100): sort (key, payload) pairs
 * by key.  Reads in_*, leaves the sorted run in out_* (in may equal out);
 * tmp_* is a ping-pong buffer of n elements.  LSD radix over the width_bits
 * significant bits of (key - lower), digits of <= 9 bits; per digit a count
 * sweep (per-tile digit prefixes) and a scatter pass that takes tiles in
 * global order (segsort.cu).  Keys outside [lower, lower + span_m1] are
 * reported through *d_bad (atomicMin of the index; initialise to UINT64_MAX)
 * -- the reference returns -1 from the kernel and raises DomainError
 * (sorter.py:97-98).  The sort is stable (equal keys keep their input
 * order); callers must not rely on it -- the reference's order among equal
 * keys is unspecified.  The workspace grows with n (4 B per 512 digits per
 * 4096-tuple tile). */
int mpsm_sort_workspace_bytes(int64_t n, int width_bits, size_t* bytes);
/* number of scatter passes (digits) the sort uses for width_bits */
int mpsm_sort_pass_count(int width_bits);
int mpsm_sort_pairs(const uint64_t* in_keys, const uint64_t* in_pays, int64_t n, uint64_t lower,
                    uint64_t span_m1, int width_bits, uint64_t* out_keys, uint64_t* out_pays,
                    uint64_t* tmp_keys, uint64_t* tmp_pays, void* workspace, size_t ws_bytes,
                    unsigned long long* d_bad, void* stream);

/* packed-record variant of the run sort: the first pass reads (key, payload)
 * SoA and every pass moves one 8-B record (key - lower) << pw | payload with
 * pw = 64 - width_bits (1 <= width_bits <= 63).  Valid when every payload is
 * below 2^pw; otherwise *d_overflow is set to 1 and the caller must use
 * mpsm_sort_pairs.  The sorted run of records lands in out_rec; tmp_rec is a
 * ping-pong buffer.  Same workspace as mpsm_sort_pairs. */
int mpsm_sort_packed(const uint64_t* in_keys, const uint64_t* in_pays, int64_t n, uint64_t lower, uint64_t span_m1,
                     int width_bits, uint64_t* out_rec, uint64_t* tmp_rec, void* workspace, size_t ws_bytes,
                     unsigned long long* d_bad, unsigned int* d_overflow, void* stream);

/* the same with a density probe of the sorted output (the private side of
 * an FK join): the last pass reduces key(R[p]) - p over every output record
 * p into d_dense[0] (min) and d_dense[1] (max), uint32, written by the call.
 * Runs for width_bits <= 32 and n < 2^32; otherwise d_dense is set to
 * "unknown" (d_dense[0] > d_dense[1]).  The sorted run is dense (its keys
 * consecutive) iff d_dense[0] == d_dense[1] and key(R[n-1]) - key(R[0]) ==
 * n - 1; mpsm_join_pairs_packed_hint takes it instead of reading the run. */
int mpsm_sort_packed_dense(const uint64_t* in_keys, const uint64_t* in_pays, int64_t n, uint64_t lower,
                           uint64_t span_m1, int width_bits, uint64_t* out_rec, uint64_t* tmp_rec, void* workspace,
                           size_t ws_bytes, unsigned long long* d_bad, unsigned int* d_overflow, uint32_t* d_dense,
                           void* stream);

/* ------------------------------------------------- radix histogram ----
 * Replaces _kernels.radix_histogram (_kernels.py:247-259) / partition.
 * build_radix_histogram (partition.py:110-122): d_counts[(key-lower)>>shift]
 * += 1 for nbuckets buckets (d_counts int64, accumulated, not zeroed);
 * out-of-domain keys -> *d_bad (atomicMin of index). */
int mpsm_radix_histogram(const uint64_t* keys, int64_t n, uint64_t lower, uint64_t span_m1, int shift,
                         int nbuckets, int64_t* d_counts, unsigned long long* d_bad, void* stream);

/* ------------------------------------------------- boundary checks ----
 * Replaces core.validate_relation (core.py:248-260) as used by
 * engine._prepare (engine.py:181-190) to word its DomainError: d_report
 * (2 words, initialised by the call) receives [0] the number of keys outside
 * [lower, lower + span_m1] and [1] the index of the first one (UINT64_MAX if
 * none).  Only called once a sort or histogram pass has flagged a bad key. */
int mpsm_domain_report(const uint64_t* keys, int64_t n, uint64_t lower, uint64_t span_m1,
                       unsigned long long* d_report, void* stream);
/* Replaces the order check of core.Run (core.py:153-154) for device runs:
 * *d_flag |= 1 if some keys[i] > keys[i + 1]. */
int mpsm_check_sorted(const uint64_t* keys, int64_t n, unsigned int* d_flag, void* stream);

/* --------------------------------------------------- partition scatter ----
 * Replaces _kernels.scatter_chunk (_kernels.py:262-284) / partition.scatter
 * (partition.py:233-276): each tuple goes to partition d_sp[(key-lower)>>shift]
 * at the worker's cursor for that partition (d_cursors: int64[npart] absolute
 * arena offsets).  Order within each (worker, partition) region is the input
 * order, i.e. the exact arena layout of the reference.  d_written (int64
 * [npart], accumulated) receives how many tuples went to each partition so
 * the caller can check it against the histogram (InternalConsistencyError). */
int mpsm_scatter_workspace_bytes(int64_t n, int npart, size_t* bytes);
int mpsm_scatter_chunk(const uint64_t* keys, const uint64_t* pays, int64_t n, uint64_t lower, int shift,
                       const int32_t* d_sp, int nbuckets, int npart, const int64_t* d_cursors,
                       uint64_t* arena_keys, uint64_t* arena_pays, int64_t* d_written, void* workspace,
                       size_t ws_bytes, void* stream);

/* multi-GPU partition of a private shard straight into packed records:
 * every tuple goes to partition d_sp[min((key - lower) >> shift, nbuckets-1)]
 * and out_rec receives the records (key - lower) << (64 - width_bits) |
 * payload grouped by partition (stable), ready for the all-to-all -- one
 * radix-style pass (the packing pass of mpsm_sort_packed with the partition
 * id as its digit).  Same workspace as mpsm_sort_pairs; domain and payload-
 * width checks as mpsm_sort_packed. */
int mpsm_partition_records(const uint64_t* keys, const uint64_t* pays, int64_t n, uint64_t lower, uint64_t span_m1,
                           int width_bits, int shift, const int32_t* d_sp, int nbuckets, int npart,
                           uint64_t* out_rec, void* workspace, size_t ws_bytes, unsigned long long* d_bad,
                           unsigned int* d_overflow, void* stream);

/* -------------------------------------------- interpolation search ----
 * Replaces _kernels.interp_lower_bound (_kernels.py:287-337) used by
 * engine.interpolation_search (engine.py:124-128): for each target, the
 * first index with key >= target and the number of positions probed (the
 * same fp64 probe rule, so identical probe counts). */
int mpsm_interp_lower_bound(const uint64_t* keys, int64_t n, const uint64_t* d_targets, int64_t ntargets,
                            int64_t* d_index, int64_t* d_probes, void* stream);

/* ---------------------------------------------------------- merge join ----
 * Replaces engine._join_private_run (engine.py:228-276) over all workers,
 * i.e. _kernels.interp_lower_bound + _kernels.merge_join_run
 * (_kernels.py:340-408) for every (private run i, public run j) pair:
 * window search, merge-path tiling over all pairs, merge with duplicate
 * cross products, fused COUNT / MAX(r+s) / checksum reduction.
 * priv / pub are HOST arrays of run descriptors pointing to device memory.
 * d_pairs: uint64[n_priv * n_pub * MPSM_PAIR_FIELDS] (zeroed by the call).
 * swap != 0: the private side is the reference's S (role swap, engine.py
 * 69-78, 217-218), so pairs are oriented (public, private) for the checksum
 * and materialized output.
 * mode MPSM_MODE_MATERIALIZE additionally writes matched pairs as
 * (r_pay, s_pay) rows into d_out (uint64[2*cap], row-major); storage stops
 * at cap rows (pairs beyond it are counted, not written: the reference's
 * merge_join_run, _kernels.py:382-390) and each pair record's
 * MPSM_PAIR_EMITTED says how many of its pairs landed.  Call once with
 * d_out == NULL to obtain counts, then again with an output buffer.
 * Every adjacent pair of keys the merge walks (the whole private run and
 * the public window) is checked for order; a violation sets
 * MPSM_FLAG_UNSORTED in the pair's MPSM_PAIR_FLAGS (the caller raises
 * InternalConsistencyError; the reference's Run rejects unsorted runs,
 * core.py:153-154).  */
int mpsm_join_workspace_bytes(const mpsm_run_t* priv, int n_priv, const mpsm_run_t* pub, int n_pub,
                              size_t* bytes);
int mpsm_join_pairs(const mpsm_run_t* priv, int n_priv, const mpsm_run_t* pub, int n_pub, int swap, int mode,
                    uint64_t* d_out, int64_t cap, uint64_t* d_pairs, void* workspace, size_t ws_bytes,
                    void* stream);

/* the same over runs of packed records (mpsm_sort_packed): each run's keys
 * pointer points at its records, pays is ignored */
int mpsm_join_pairs_packed(const mpsm_run_t* priv, int n_priv, const mpsm_run_t* pub, int n_pub, int width_bits,
                           uint64_t lower, int swap, int mode, uint64_t* d_out, int64_t cap, uint64_t* d_pairs,
                           void* workspace, size_t ws_bytes, void* stream);
/* mpsm_join_pairs_packed with the density probe of the sorted array the
 * private runs were cut from (priv_n records at priv_base; d_dense from
 * mpsm_sort_packed_dense / mpsm_sort_records_dense): when it proves the
 * array dense, the dense-run path skips its own read of the private runs
 * (d_dense may be NULL: the same as mpsm_join_pairs_packed) */
int mpsm_join_pairs_packed_hint(const mpsm_run_t* priv, int n_priv, const mpsm_run_t* pub, int n_pub,
                                int width_bits, uint64_t lower, int swap, int mode, uint64_t* d_out, int64_t cap,
                                uint64_t* d_pairs, void* workspace, size_t ws_bytes, const uint32_t* d_dense,
                                const uint64_t* priv_base, int64_t priv_n, void* stream);

/* ------------------------------------------------ splitter search ----
 * Replaces skew._minmax_contiguous (skew.py:180-273) as used by
 * skew.compute_splitters (skew.py:287-315): split n buckets into t
 * contiguous ranges minimising the largest
 *   cost(a,b) = |R_ab| log2|R_ab| + t |R_ab| + (edge_cdf[b] - edge_cdf[a])
 * with the lexicographically smallest bounds.  Host function.
 * prefix: int64[n+1] bucket-count prefix sums; edge_cdf: double[n+1];
 * cand: the bound candidates computed by the caller with numpy exactly as
 * the reference does (sorted unique batch costs when n <= 256, else the n
 * single-bucket costs) so the floating-point values are bit-identical.
 * out_bounds: int64[t+1].  Returns MPSM_ERR_CONFIG if t > n. */
int mpsm_minmax_contiguous(int64_t n, int t, const int64_t* prefix, const double* edge_cdf,
                           const double* cand, int64_t ncand, int64_t* out_bounds);

/* ------------------------------------------------ multi-GPU helpers ----
 * CUDA IPC so a rank can merge against peer ranks' public runs with NVLink
 * peer loads (the paper's sequential remote-NUMA reads, engine.py:249-260).
 * handle buffers are 64 bytes.  get_handle names the cudaMalloc block that
 * holds d_ptr and returns d_ptr's byte offset in it; open_handle maps the
 * block into the calling thread's current device with lazy peer access
 * (open each block once per process; add the offset). */
int mpsm_ipc_get_handle(const void* d_ptr, void* handle64, int64_t* offset);
int mpsm_ipc_open_handle(const void* handle64, void** d_ptr);
int mpsm_ipc_close_handle(void* d_ptr);

/* ------------------------------------------------ relation files ----
 * The reference's relation file (bench.py:8-11, read_relation bench.py:84-102,
 * write_relation bench.py:73-81): magic "MPSMREL1", u64 n, then n
 * little-endian (key u64, payload u64) records.
 * mpsm_relfile_header checks magic and exact length like read_relation and
 * returns n; on MPSM_ERR_FORMAT *bad_offset is the byte offset the reference
 * reports (0 for bad magic, the file size for a truncated header,
 * min(size, 16 + 16 n) for a length mismatch).  Host functions. */
int mpsm_relfile_header(const char* path, uint64_t* n, int64_t* bad_offset);
/* reads the n records (16 n bytes, interleaved) into host memory dst (pinned
 * or pageable) with `threads` parallel readers (0: all cores) */
int mpsm_relfile_read(const char* path, uint64_t n, void* dst, int threads);
/* reads the n records straight into SoA host arrays keys / pays (the reading
 * threads split the records; read_relation's columns, bench.py:100-102) */
int mpsm_relfile_read_columns(const char* path, uint64_t n, uint64_t* keys, uint64_t* pays, int threads);
/* writes a relation file from SoA host arrays (parallel, all cores) */
int mpsm_relfile_write(const char* path, const uint64_t* keys, const uint64_t* pays, uint64_t n);
/* device: split n interleaved records into SoA keys / payloads */
int mpsm_deinterleave(const uint64_t* d_records, int64_t n, uint64_t* d_keys, uint64_t* d_pays, void* stream);

/* ------------------------------------------------- packed upload ----
 * Host (key, payload) SoA -> device packed records (key - lower) << (64 - w)
 * | payload, the layout mpsm_sort_records sorts.  Host worker threads pack
 * 128K-tuple chunks into pinned staging slots and each chunk is copied while
 * later ones are packed: half the PCIe bytes of copying the columns.  When
 * the columns are pinned, every gpu_pack_every-th chunk is instead packed by
 * the GPU reading the mapped columns (balances host memory bandwidth against
 * PCIe; 0: the host packs all, -1: default 0, MPSM_UPLOAD_RAW_EVERY).  Keys
 * outside [lower, lower + span_m1]: *bad_index = first such index (else -1;
 * the reference raises DomainError, sorter.py:97-98).  A payload >= 2^(64-w):
 * *overflow = 1 and the records are invalid (use the column path).  The
 * copies are ordered before later work on `stream`; returns once the host
 * buffers have been read.  The copies start after the work queued on
 * `stream` before `ready_event` (a cudaEvent_t recorded when d_rec was
 * allocated; NULL: after all work queued on `stream` so far), so work queued
 * later overlaps the upload.  threads <= 0: MPSM_UPLOAD_THREADS, else 3/4 of
 * the cores this process may run on, divided by LOCAL_WORLD_SIZE when a
 * launcher runs one process per GPU.  Not thread-safe (one uploader per
 * process). */
int mpsm_upload_records(const uint64_t* h_keys, const uint64_t* h_pays, int64_t n, uint64_t lower,
                        uint64_t span_m1, int width_bits, uint64_t* d_rec, int threads, int gpu_pack_every,
                        void* stream, void* ready_event, int64_t* bad_index, int* overflow);
/* device (key, payload) columns -> packed records (before an exchange: the
 * multi-GPU all-to-all moves 8 B per tuple).  Same domain / payload-width
 * checks as mpsm_upload_records, reported through device flags: *d_bad =
 * atomicMin of the first out-of-domain index, *d_overflow |= 1. */
int mpsm_pack_records(const uint64_t* d_keys, const uint64_t* d_pays, int64_t n, uint64_t lower, uint64_t span_m1,
                      int width_bits, uint64_t* d_rec, unsigned long long* d_bad, unsigned int* d_overflow,
                      void* stream);
/* host->device bytes moved by mpsm_upload_records since the last reset
 * (8 per host-packed tuple, 16 per tuple the GPU packs from mapped memory) */
uint64_t mpsm_upload_bytes(int reset);
/* sort packed records (key in the top width_bits bits) by key: every pass
 * moves 8 B (the mpsm_sort_packed passes after its packing pass).  tmp_rec
 * must differ from both; in_rec may equal out_rec (sort in place) when
 * mpsm_sort_pass_count(width_bits) is even.  Same workspace as
 * mpsm_sort_pairs. */
int mpsm_sort_records(const uint64_t* in_rec, int64_t n, int width_bits, uint64_t* out_rec, uint64_t* tmp_rec,
                      void* workspace, size_t ws_bytes, void* stream);
/* mpsm_sort_records with the density probe of mpsm_sort_packed_dense */
int mpsm_sort_records_dense(const uint64_t* in_rec, int64_t n, int width_bits, uint64_t* out_rec,
                            uint64_t* tmp_rec, void* workspace, size_t ws_bytes, uint32_t* d_dense, void* stream);

/* ------------------------------------------------ segmented run sort ----
 * nseg independent sorts in one launch sequence: elements [h_offsets[s],
 * h_offsets[s+1]) form segment s and are sorted among themselves, in place
 * of position (the T public chunks of a join -> T runs, engine.py:389-395;
 * B-MPSM's private chunks, engine.py:297-309).  h_offsets: HOST int64
 * [nseg + 1], 0 = h_offsets[0] <= ... <= h_offsets[nseg] = n, 1 <= nseg <=
 * 1024.  Scatter tiles never straddle a segment; every pass is one count, one
 * scan and one scatter launch for all segments.  Domain errors report the
 * index in the whole array.  Workspace from
 * mpsm_sort_segments_workspace_bytes; otherwise as the unsegmented calls
 * (mpsm_sort_pairs_segments needs in_keys != out_keys). */
int mpsm_sort_segments_workspace_bytes(int64_t n, int nseg, int width_bits, size_t* bytes);
int mpsm_sort_pairs_segments(const uint64_t* in_keys, const uint64_t* in_pays, int64_t n, int nseg,
                             const int64_t* h_offsets, uint64_t lower, uint64_t span_m1, int width_bits,
                             uint64_t* out_keys, uint64_t* out_pays, uint64_t* tmp_keys, uint64_t* tmp_pays,
                             void* workspace, size_t ws_bytes, unsigned long long* d_bad, void* stream);
int mpsm_sort_packed_segments(const uint64_t* in_keys, const uint64_t* in_pays, int64_t n, int nseg,
                              const int64_t* h_offsets, uint64_t lower, uint64_t span_m1, int width_bits,
                              uint64_t* out_rec, uint64_t* tmp_rec, void* workspace, size_t ws_bytes,
                              unsigned long long* d_bad, unsigned int* d_overflow, void* stream);
int mpsm_sort_records_segments(const uint64_t* in_rec, int64_t n, int nseg, const int64_t* h_offsets,
                               int width_bits, uint64_t* out_rec, uint64_t* tmp_rec, void* workspace,
                               size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MPSM_B200_H */
