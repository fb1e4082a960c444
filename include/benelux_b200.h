/*
 * benelux_b200.h -- C ABI of the B200-native Benelux-pair search (libbenelux_b200.so).
 *
 * Plain pointers and sizes only; no torch or CUDA types in the signatures (a stream is
 * passed as an opaque `void*` holding a cudaStream_t, 0 = the library's own stream).
 * Host pointers unless a name ends in `_dev`.  Every entry point returns a status code.
 *
 * Each entry point replaces one seam of the reference package `benelux_pairs`
 * (paths relative to /root/reference/pkg/src/benelux_pairs/):
 *
 *   bnx_primes_up_to            <- primes.py:24-35           primes_up_to(limit)
 *   bnx_sieve_radicals          <- radical.py:109-124 +      sieve_radicals(Interval, PrimeList,
 *                                  _kernels.py:22-84           ctz_fast_path) / sieve_segment
 *   bnx_radicals_trial_division <- _kernels.py:87-112        radicals_trial_division(start, length)
 *   bnx_search                  <- sort_search.py:37-91      find_pairs_sorted(limit, primes)
 *   bnx_search_domain           <- chunked.py:307-359        search_chunk(index, s, primes, n_limit)
 *                                  (+ chunked.py:362-412      run_full_chunked, one call per chunk)
 *   bnx_brute_force             <- bruteforce.py:16-42       brute_force_pairs(limit) (_kernels.py:235-263)
 *   bnx_table_*                 <- chunked.py:129-359 +      SignatureTable / build_table / probe_table /
 *                                  _kernels.py:130-232         search_chunk (the paper's Algorithm 3)
 *   bnx_slot_of                 <- _kernels.py:115-123 /     _slot_of / commutative_hash
 *                                  chunked.py:93-109
 *   status codes                <- _kernels.py:17-19         STATUS_OK / TABLE_FULL / BUFFER_FULL
 *
 * Error convention (mirrors _kernels.py:17-19 and the front-ends' exceptions):
 *   BNX_OK                   0  success
 *   BNX_TABLE_FULL           1  (reserved; TableFullError)
 *   BNX_BUFFER_FULL          2  `cap` too small: *found holds the required count; the
 *                               caller grows the buffer and calls again (chunked.py:268-270)
 *   BNX_ERR_PRIMES_UNCOVERED 3  supplied primes do not reach isqrt(endpoint) -> ValueError
 *                               (radical.py:119-120)
 *   BNX_ERR_INVALID          4  bad argument (limit < 3, empty interval, ...) -> ValueError
 *   BNX_ERR_CUDA             5  CUDA runtime failure / no device           -> RuntimeError
 *   BNX_ERR_RANGE            6  bound beyond this build's exact range (S > 2^48; S >= 2^42
 *                                with the byte-screen engine)
 *   bnx_last_error() gives a message for the most recent failure on the calling thread.
 */
#ifndef BENELUX_B200_H
#define BENELUX_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define BNX_API __attribute__((visibility("default")))
#else
#define BNX_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define BNX_OK 0
#define BNX_TABLE_FULL 1
#define BNX_BUFFER_FULL 2
#define BNX_ERR_PRIMES_UNCOVERED 3
#define BNX_ERR_INVALID 4
#define BNX_ERR_CUDA 5
#define BNX_ERR_RANGE 6

#define BNX_KIND_FIRST 1u  /* signatures.py:14-16 Kind.FIRST  */
#define BNX_KIND_SECOND 2u /* signatures.py:14-16 Kind.SECOND */
#define BNX_KIND_BOTH 3u

/* One result row: BeneluxPair (signatures.py:48-64) / CLI row kind,m,n,rad_m,rad_m1
 * (cli.py:111-125).  rad_m, rad_m1 are rad(m), rad(m+1) in natural order. */
typedef struct bnx_pair {
    uint64_t m;
    uint64_t n;
    uint64_t rad_m;
    uint64_t rad_m1;
    int32_t kind; /* 1 first, 2 second */
    int32_t reserved;
} bnx_pair_t;

/* Per-call counters of the last search (diagnostics and bench). */
typedef struct bnx_stats {
    uint64_t integers;       /* n values examined by the screen                      */
    uint64_t survivors;      /* n passing the on-chip log-surplus screen              */
    uint64_t candidates;     /* n with rad(n)*rad(n+1) <= 2n (exact)                  */
    uint64_t residue_checks; /* m values enumerated on the residue classes            */
    uint64_t matches;        /* (m, n) with equal signatures                          */
    uint64_t pairs;          /* rows emitted after the kind filter                    */
    uint64_t kernel_launches;/* this library's own kernels launched for the call (the   */
                             /* cub scan of the heavy generator is not counted)         */
    int32_t bucket_overflow; /* nonzero if a tile bucket overflowed (call failed)     */
    int32_t reserved;
    uint64_t max_residue_checks; /* most residue-class members of a single candidate     */
} bnx_stats_t;

typedef struct bnx_ctx bnx_ctx_t;

BNX_API int bnx_version(void);
BNX_API const char* bnx_last_error(void);
BNX_API int bnx_device_count(int* count);

/* Context: one GPU, one stream, cached prime tables and work buffers. */
BNX_API int bnx_ctx_create(int device, bnx_ctx_t** out);
BNX_API int bnx_ctx_destroy(bnx_ctx_t* ctx);
BNX_API int bnx_ctx_set_stream(bnx_ctx_t* ctx, void* stream);
BNX_API int bnx_ctx_stats(const bnx_ctx_t* ctx, bnx_stats_t* out);
/* Kernel timing with CUDA events on the context stream: with mode 1, each search records
 * events around the candidate generator (screen) and around the whole device pipeline; bnx_ctx_timing
 * returns the last search's milliseconds (valid after bnx_search_collect / bnx_search*).  Mode 2
 * launches the heavy engine's kernels directly (no graph, no programmatic overlap) with events
 * between them; bnx_ctx_kernel_timing returns up to 4 stage times in ms: [0] k_heavy_count + scan,
 * [1] k_heavy_screen (with k_heavy_sieve beside it above ~2^33), [2] k_heavy_exact, [3] the tail.
 * Mode 0 (default) records nothing. */
BNX_API int bnx_ctx_set_timing(bnx_ctx_t* ctx, int mode);
BNX_API int bnx_ctx_kernel_timing(const bnx_ctx_t* ctx, float* ms, int n);
/* Diagnostics (tests): prepare for bound max_x and copy out the heavy generator's surplus-class
 * table in its device order: b_out[i] = b, m_out[i] = m | r << 40 (either may be NULL).
 * *count receives the class count; BNX_BUFFER_FULL if it exceeds cap. */
BNX_API int bnx_ctx_class_table(bnx_ctx_t* ctx, uint64_t max_x, uint64_t* b_out, uint64_t* m_out, size_t cap,
                                size_t* count);
/* Candidate generator of the search (results are identical):
 * BNX_ENGINE_HEAVY (default) lists the heavy integers (2 s(x)^2 >= x, s = x / rad x) and tests
 * their neighbours; BNX_ENGINE_SCREEN sieves a log-surplus byte per integer.  The environment
 * variable BNX_ENGINE=screen selects the screen at context creation. */
#define BNX_ENGINE_HEAVY 0
#define BNX_ENGINE_SCREEN 1
BNX_API int bnx_ctx_set_engine(bnx_ctx_t* ctx, int engine);
BNX_API int bnx_ctx_engine(const bnx_ctx_t* ctx);
/* Multi-GPU: subsequent searches on this context compute only shard `shard` of `nshards`
 * (0 <= shard < nshards); the row sets of the shards of one search are disjoint and their
 * union is the full result.  The heavy generator splits its (surplus class, k) items and
 * sieve chunks evenly (balanced work: heavy integers thin out as n grows); the byte screen
 * splits the n-range into contiguous slabs.  Default 0 of 1. */
BNX_API int bnx_ctx_set_shard(bnx_ctx_t* ctx, uint32_t shard, uint32_t nshards);
BNX_API int bnx_ctx_timing(const bnx_ctx_t* ctx, float* screen_ms, float* pipeline_ms);

/* primes.py:24-35: all primes <= limit, ascending.  *count always receives the total;
 * BNX_BUFFER_FULL if it exceeds cap. */
BNX_API int bnx_primes_up_to(bnx_ctx_t* ctx, uint64_t limit, uint64_t* out, size_t cap, size_t* count);

/* radical.py:109-124: out[k] = rad(start + k), k < length.  `primes` (ascending, covering
 * `primes_limit` = PrimeList.limit) may be NULL to let the device build them.  Returns
 * BNX_ERR_PRIMES_UNCOVERED when primes_limit < isqrt(start + length - 1). */
BNX_API int bnx_sieve_radicals(bnx_ctx_t* ctx, uint64_t start, uint64_t length, const uint64_t* primes,
                       size_t nprimes, uint64_t primes_limit, int ctz_fast_path, uint64_t* out);
/* Same, writing into device memory `out_dev` (any 8-byte aligned pointer) on the context
 * stream, with the device prime table; no host copy of the radicals.  The call waits for
 * the stream once at the end to read the bucket-overflow flag. */
BNX_API int bnx_sieve_radicals_dev(bnx_ctx_t* ctx, uint64_t start, uint64_t length, int ctz_fast_path,
                           uint64_t* out_dev);

/* _kernels.py:87-112: out[k] = rad(start + k) by per-integer trial division on the GPU. */
BNX_API int bnx_radicals_trial_division(bnx_ctx_t* ctx, uint64_t start, uint64_t length, uint64_t* out);

/* bruteforce.py:16-42 + _kernels.py:235-263: the quadratic scan over trial-division radicals,
 * on the GPU (limit <= 2^22); rows sorted by (m, n).  An independent check of bnx_search. */
BNX_API int bnx_brute_force(bnx_ctx_t* ctx, uint64_t limit, bnx_pair_t* out, size_t cap, size_t* found);

/* sort_search.py:37-91: every pair m < n < limit of the kinds in kinds_mask.
 * Rows come back sorted by (m, n).  primes may be NULL (device-built). */
BNX_API int bnx_search(bnx_ctx_t* ctx, uint64_t limit, uint32_t kinds_mask, const uint64_t* primes,
               size_t nprimes, uint64_t primes_limit, bnx_pair_t* out, size_t cap, size_t* found);

/* chunked.py:307-359: every pair (m, n), m < n, with n_first <= n <= n_last (any m >= 1).
 * Rows sorted by (n, m) (chunked.py:358). */
/* The survey's multi-GPU entry point (one host thread drives ndev GPUs):
 * context i on devices[i] (a process-wide pool) computes shard i of ndev of the search below
 * `limit` (bnx_ctx_set_shard), all shards run concurrently, and the rows are merged and
 * sorted by (m, n) -- identical to bnx_search for any device list.  A device may appear
 * more than once (several shards on one GPU). */
BNX_API int bnx_search_multi(const int* devices, int ndev, uint64_t limit, uint32_t kinds_mask,
                             const uint64_t* primes, size_t nprimes, uint64_t primes_limit, bnx_pair_t* out,
                             size_t cap, size_t* found);
BNX_API int bnx_search_domain(bnx_ctx_t* ctx, uint64_t n_first, uint64_t n_last, uint32_t kinds_mask,
                      const uint64_t* primes, size_t nprimes, uint64_t primes_limit, bnx_pair_t* out,
                      size_t cap, size_t* found);

/* Split-phase form for timing: enqueue the whole search on the context stream without a
 * host sync (device-resident prime tables must already exist: call bnx_prepare first),
 * then collect.  bnx_prepare builds / uploads the tables for bound `max_x`.  A collect that
 * returns BNX_BUFFER_FULL keeps the rows: call it again with a buffer of *found rows. */
BNX_API int bnx_prepare(bnx_ctx_t* ctx, uint64_t max_x, const uint64_t* primes, size_t nprimes,
                uint64_t primes_limit);
BNX_API int bnx_search_enqueue(bnx_ctx_t* ctx, uint64_t n_first, uint64_t n_last, uint32_t kinds_mask);
BNX_API int bnx_search_collect(bnx_ctx_t* ctx, bnx_pair_t* out, size_t cap, size_t* found);

/* ---- Algorithm 3 of the paper (chunked.py:129-359, _kernels.py:130-232) on the GPU -------
 * An open-addressing signature table with the reference's slot word ((t+1) << 32 | home,
 * 0 = empty), hash and linear probing, built by all threads at once (64-bit CAS).  The pair
 * set equals the serial build's; slot placement may differ.  Rows sorted by (n, m).
 * BNX_TABLE_FULL when a walk wraps the table (TableFullError). */
typedef struct bnx_table bnx_table_t;
BNX_API int bnx_table_create(bnx_ctx_t* ctx, uint64_t table_size, bnx_table_t** out);
BNX_API int bnx_table_destroy(bnx_table_t* table);
/* chunked.py:243-272 insert_all: domain elements t < count, n = domain_start + t < n_limit. */
BNX_API int bnx_table_insert_all(bnx_table_t* table, uint64_t domain_start, const uint64_t* rad_of,
                                 const uint64_t* rad_next, size_t count, uint64_t n_limit, bnx_pair_t* out,
                                 size_t cap, size_t* found, uint64_t* inserted);
/* chunked.py:274-304 probe_all: read-only probe with the domain starting at probe_start. */
BNX_API int bnx_table_probe_all(bnx_table_t* table, uint64_t probe_start, const uint64_t* rad_of,
                                const uint64_t* rad_next, size_t count, bnx_pair_t* out, size_t cap, size_t* found);
/* copy of the slot words (table_size u64). */
BNX_API int bnx_table_slots(const bnx_table_t* table, uint64_t* out, size_t cap);
/* chunked.py:307-359 search_chunk with Algorithm 3 on the device: sieve chunk `index`, build
 * its table, re-sieve and probe every earlier chunk j in [j_lo, j_hi). */
BNX_API int bnx_table_search_chunk(bnx_ctx_t* ctx, uint64_t index, uint64_t chunk_size, uint64_t n_limit,
                                   uint64_t j_lo, uint64_t j_hi, bnx_pair_t* out, size_t cap, size_t* found);

/* _kernels.py:115-123: the reference's commutative slot hash (host, for API parity). */
BNX_API uint64_t bnx_slot_of(uint64_t lo, uint64_t hi, uint64_t mask, uint64_t phi, uint64_t mul1, uint64_t mul2);

#ifdef __cplusplus
}
#endif

#endif /* BENELUX_B200_H */
