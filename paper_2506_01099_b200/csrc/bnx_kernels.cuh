// bnx_kernels.cuh -- kernel argument blocks, tile geometry and launchers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/benelux_b200.h"
#include "bnx_math.cuh"

namespace bnx {

// Screen: per-tile progressions (q < tile) at most SCREEN_MAXS; geometry variants below.
constexpr int SCREEN_MAXS = 160;

// Exact radical sieve geometry: 8192 u64 slots per tile (64 KB), 64 tiles per segment.
constexpr int SIEVE_TILE = 8192;
constexpr int SIEVE_NT = 64;
constexpr int SIEVE_THREADS = 512;
constexpr int SIEVE_BCAP = 64;
constexpr int SIEVE_MAXS = 160;

// Counter block (device): [0] survivors [1] candidates [2] residue checks [3] matches [4] pairs
// [5] the tail's work queue head [6] most residue-class members of one candidate
// [7] heavy candidates queued for k_tail_heavy
// [8] heavy engine: candidates in the light list (k_tail); the rest went to the heavy queue
constexpr size_t IO_CTR = 0, IO_FLAGS = 8 * 16, IO_PAIRS = 8 * 16 + 4 * 4 + 16;  // search I/O block (bnx_capi.cu)
constexpr uint64_t PAIR_PREFIX = 64;   // pair rows read back with the counters (bnx_capi.cu read_back)
constexpr int CTR_SURV = 0, CTR_CAND = 1, CTR_CHECKS = 2, CTR_MATCH = 3, CTR_PAIRS = 4, CTR_NEXT = 5, CTR_MAXCHK = 6,
              CTR_HEAVY = 7, CTR_LIGHT = 8, CTR_RUNS = 9, CTR_N = 10;
static_assert(8 * CTR_N <= IO_FLAGS, "counters overlap the flags in the search I/O block");
// Candidates with more than this many residue-class members are handed to k_tail_heavy
// which spreads their members over many warps (one candidate below 2^32 has ~1,500).
constexpr uint64_t TAIL_HEAVY = 48;

struct ScreenArgs {
    uint64_t x_begin;  // multiple of the tile
    uint64_t ntiles;   // tiles covering [x_begin, n_last]
    uint64_t n_first, n_last;
    const BnxProg* small;
    int nsmall;
    const BnxProg* large;
    int nlarge;
    const uint32_t* items;  // work items over `small` (sorted by q), see build_items
    int nitems;
    uint64_t* surv;
    uint64_t surv_cap;
    unsigned long long* ctr;
    int* flags;  // [0] bucket overflow
    int skip;    // profiling only (BNX_SCREEN_SKIP): 1 items, 2 buckets, 4 scan, 8 init, 16 segment setup
};

struct TailArgs {
    const uint64_t* surv;  // screen engine: survivors n (the tail computes the radicals)
    uint64_t surv_cap;
    const BnxCand* cands;  // heavy engine: exact candidates (n, rad n, rad n+1); null for the screen
    uint64_t cand_cap;
    BnxCand* heavy;      // candidates with many residue-class members
    uint64_t heavy_cap;
    const BnxPDiv* pdiv;
    uint64_t npdiv;
    uint32_t kinds;
    bnx_pair_t* pairs;
    uint64_t pair_cap;
    unsigned long long* ctr;
    // heavy engine: the first host_prefix rows also go straight to mapped pinned host memory,
    // and any overflow raises host_flags[2] (capacity) / [3] (more rows than the prefix), so
    // the search needs no read-back copy; null for the byte screen
    bnx_pair_t* host_pairs;
    uint64_t host_prefix;
    int* host_flags;
};

// Heavy-side generator (bnx_heavy.cu).
constexpr int HEAVY_THREADS = 256;
constexpr int HEAVY_TILE = 256;          // classes per tile of k_heavy_count_local
constexpr int HEAVY_TILES_MAX = 1024;    // tile offsets staged in k_heavy_screen's shared memory (8 KB)
constexpr int HEAVY_NP2 = 1023;  // odd primes <= y_max^(1/4) staged in shared memory (10-bit task index)
constexpr int HEAVY_NP3 = 7000;  // odd primes <= cbrt(y_max) staged in shared memory (S <= 2^48)
// Classes with at least HEAVY_KMIN values of k in a domain are sieved over k (k_heavy_sieve)
// in chunks of up to kc values; the rest go through trial division (k_heavy_screen).  Item
// counts are packed: low 40 bits trial items, high 24 bits sieve chunks (one scan).
constexpr uint64_t HEAVY_KMIN_DEFAULT = 256;
constexpr uint64_t HEAVY_TRIAL_MASK = (1ull << 40) - 1;
constexpr int HEAVY_TASK_HITS = 16;  // marks per sieve task (host-built task list)
constexpr int HEAVY_HITS = 8;        // hit-list slots per (k, side) in k_heavy_sieve (more: trial division)
struct HeavyArgs {
    const BnxHeavyEnt* ent;
    uint64_t nent;
    uint64_t* cnt;    // per class: number of k in the domain
    uint64_t* incl;   // inclusive scan of cnt (ntiles > 0: within each tile of HEAVY_TILE classes)
    uint64_t* tile_tot;  // ntiles > 0: the tiles' totals (k_heavy_count_local)
    uint32_t ntiles;     // > 0: per-tile scan, the screen adds the tile offsets (no sieve classes)
    uint32_t* klo;    // per class: first k in the domain
    uint32_t* kcnt;   // per class: number of k in the domain
    const uint32_t* tasks;  // sieve marking tasks: j | side << 10 | r << 11 | R << 21
    int ntasks;
    int kc;                 // k values per sieve chunk
    uint64_t kmin;          // classes with >= kmin k in the domain are sieved
    const uint16_t* invtab; // per prime j <= P2: a^-1 mod p at invtab[invoff[j] + a]
    const uint32_t* invoff;
    const uint32_t* kinfo;  // per k: bits 0..30 = primes 2..127 dividing k, bit 31 = k not squarefree
    uint64_t nkinfo;
    uint64_t x_lo, x_hi;    // heavy x range: [n_first, n_last + 1]
    uint64_t n_first, n_last;
    const BnxPDiv* pdiv;    // odd primes ascending
    const uint4* pd32;      // the same primes (<= cbrt(y_max)): (p^-1 mod 2^32, floor((2^32-1)/p), p, 2^32 mod p)
    int np2;                // odd primes <= P2 = floor(y_max^(1/4))
    uint64_t np3;           // odd primes <= cbrt(y_max)
    uint64_t p1, p1sq, p1cube;  // P2 + 1 and its powers
    float inv_p1f;
    int cube_filter;        // P2 >= 7: cube residues mod 63 pre-filter the p^3 test
    BnxSurv* q1;            // stage-1 survivors (n | side << 63, rad x, cofactor, its radical part)
    uint64_t q1_cap;
    BnxCand* cand;          // exact candidates with <= TAIL_HEAVY residue-class members (k_tail)
    uint64_t cand_cap;
    BnxCand* heavy;         // the others (k_tail_heavy, concurrently on a second stream)
    uint64_t heavy_cap;
    uint32_t kinds;
    unsigned long long* ctr;
    int* flags;             // [1] k outside kinfo (internal error)
    uint32_t shard, nshards;  // this search covers items/chunks [shard, shard + 1) / nshards
    uint64_t tail_heavy;      // candidates with more residue-class members go to k_tail_heavy
    uint32_t run_mult;        // k_heavy_screen: fetched runs per CTA (from CTR_RUNS) after the first
    uint32_t run_first;       // k_heavy_screen: share of the items in the first (static) runs, /256
    int* host_flags;          // mapped pinned host flags: [1] k outside its table, [2] a buffer overflowed
    uint32_t sieve_ctas;      // k_heavy_sieve grid (0: the screen's)
    uint32_t sieve_threads;   // k_heavy_sieve CTA size (0: 256)
    int exact_warp;           // k_heavy_exact: one warp per survivor, cut prime ranges (else one thread each)
    int probe_walk;           // profiling only (BNX_PROBE_WALK=1): k_heavy_screen walks and queues, no y tests
};
size_t heavy_scan_temp_bytes(uint64_t nent);
void launch_pdiv32(const BnxPDiv* pdiv, uint64_t n, uint4* out, cudaStream_t st);
cudaError_t heavy_configure();
bool heavy_sieve_mask(int np2);  // k_heavy_sieve marks bit masks (else hit lists)
size_t heavy_sieve_smem(int np2, int kc, int ntasks);
void launch_heavy(const HeavyArgs& a, void* scan_temp, size_t scan_temp_bytes, int grid, cudaStream_t st,
                  cudaEvent_t ev_generated, cudaStream_t aux, cudaEvent_t ev_fork, cudaEvent_t ev_join,
                  const cudaEvent_t* kev = nullptr,  // kev[0..3]: per-kernel timing (count, screen, exact)
                  int stop_after = 0);  // profiling only: 1 = count + scan, 2 = + screen (0: all)

// The surplus-class table built on the device (bnx_classes.cu).
struct ClassPlan {
    uint64_t X, L, V;  // bound, isqrt(X) (factor table), icbrt(X) (the v of b = u^2 v^3)
    int D, bits, dpw, nwords;  // sort key: D codes of `bits` bits, dpw per 64-bit word
    bool ok;
};
ClassPlan class_plan(uint64_t X, uint64_t nprimes_root);
cudaError_t classes_preload(cudaStream_t st);
cudaError_t kernels_preload();
cudaError_t heavy_preload_cub(cudaStream_t st);
size_t class_scratch_bytes(const ClassPlan& pl, uint64_t total);
// tab: Ltab + 1 entries (Ltab >= pl.L; np_tab = primes <= Ltab in the list); cnt, offs: V + 2
cudaError_t class_count(const ClassPlan& pl, uint64_t Ltab, const uint32_t* primes, uint64_t np_tab, uint32_t* tab,
                        uint64_t* cnt, uint64_t* offs, void* scratch, size_t scratch_bytes, cudaStream_t st);
cudaError_t class_build(const ClassPlan& pl, uint64_t total, const uint32_t* primes, const uint32_t* tab,
                        const uint64_t* offs, BnxHeavyEnt* ent_tmp, BnxHeavyEnt* ent, uint64_t* keys,
                        uint64_t* key_tmp, uint32_t* perm, uint32_t* perm_tmp, void* scratch, size_t scratch_bytes,
                        uint32_t* kinfo, uint64_t K, cudaStream_t st);

struct SieveArgs {
    uint64_t start, length;
    const BnxProg* small;
    int nsmall;
    const BnxProg* large;
    uint64_t nlarge;
    const uint32_t* items;
    int nitems;
    int fast;
    uint64_t* out;
    int* flags;
    // the large progressions' hits, pre-sorted by segment (launch_sieve_buckets): entry
    // p << 32 | offset in the segment, gcnt[seg] of them at gbuck + seg * gcap; null: each
    // segment scans all large progressions itself
    const uint64_t* gbuck;
    const uint32_t* gcnt;
    uint32_t gcap;
    uint64_t nmedium;  // with gbuck: large[0, nmedium) (q < SIEVE_HUGE_Q) are scanned per segment,
                       // the rest come from the buckets
};
constexpr uint64_t SIEVE_HUGE_Q = 1ull << 24;  // above every segment length (at most one hit per segment, 64 per 2^30)
// The large progressions split in place order-free: q < SIEVE_HUGE_Q to the front, the rest
// to the back of `out` (n entries); *nmed = the front count.
void launch_split_large(const BnxProg* in, uint64_t n, BnxProg* out, unsigned long long* counts, cudaStream_t st);
// One pass over the large progressions of a window: every hit appended to its segment's
// global bucket (flags[3] on a full bucket).
void launch_sieve_buckets(const SieveArgs& a, uint64_t seg_len, uint64_t* gbuck, uint32_t* gcnt, cudaStream_t st);

// Compiled screen geometries (tile, tiles per segment, threads, bucket capacity); the
// context picks one at creation (BNX_SCREEN_VARIANT, default 0).
struct ScreenVariant {
    int tile, nt, threads, bcap;
    const void* fn;
    size_t smem;
    void (*launch)(const ScreenArgs&, int, cudaStream_t);
};
int screen_variant_count();
const ScreenVariant& screen_variant(int i);
// Algorithm 3 (signature table) arguments.
struct TableArgs {
    uint64_t domain_start;
    const uint64_t* rad_of;     // table chunk: rad(domain_start + t), t < count_n
    const uint64_t* rad_next;   // rad(domain_start + t + 1)
    uint64_t count_n;
    uint64_t n_limit;           // insert only n < n_limit
    uint64_t probe_start;
    const uint64_t* probe_of;   // probing chunk
    const uint64_t* probe_next;
    uint64_t count_m;
    uint64_t* slots;
    uint64_t mask;
    bnx_pair_t* out;
    uint64_t cap;
    unsigned long long* count;
    unsigned long long* inserted;
    int* status;
};
// lanes: 1 (a thread per element) or 4 (the paper's four-slot parallel probe, k_table_quad)
void launch_table_insert(const TableArgs& a, int grid, cudaStream_t st, int lanes);
void launch_table_probe(const TableArgs& a, int grid, cudaStream_t st, int lanes);
// Compiled exact-sieve geometries (tile, tiles per segment, threads, bucket capacity); the
// context picks one at creation (BNX_SIEVE_VARIANT, default 0).
struct SieveVariant {
    int tile, nt, threads, bcap;
    const void* fn;
    size_t smem;
    void (*launch)(const SieveArgs&, int, cudaStream_t);
};
int sieve_variant_count();
const SieveVariant& sieve_variant(int i);
int sieve_narrow_count();  // the same kernel with 32-bit slots (windows ending below 2^32)
const SieveVariant& sieve_narrow(int i);

void launch_tail(const TailArgs& a, int grid, cudaStream_t st);
void launch_tail_light(const TailArgs& a, int grid, cudaStream_t st, bool pdl = false);  // heavy engine: k_tail only
void launch_tail_heavy(const TailArgs& a, cudaStream_t st);            // heavy engine: k_tail_heavy only
void launch_base_primes(uint32_t ls, uint32_t* out, uint32_t* count, cudaStream_t st);
void launch_prime_seg(uint64_t lo, uint64_t hi, const uint32_t* base, uint32_t nbase, uint32_t* counts,
                      const uint64_t* offsets, uint32_t* out, uint64_t nblocks, cudaStream_t st);
void launch_scan_counts(const uint32_t* counts, uint64_t n, uint64_t base, uint64_t* offsets, cudaStream_t st);
void launch_narrow(const uint64_t* in, uint64_t n, uint32_t* out, cudaStream_t st);
void launch_widen(const uint32_t* in, uint64_t n, uint64_t* out, cudaStream_t st);
void launch_build_tables(const uint32_t* primes, uint64_t np, uint64_t max_x, int include_two, uint32_t tile,
                         BnxProg* small, uint32_t* nsmall, uint32_t small_cap, BnxProg* large,
                         unsigned long long* nlarge, uint64_t large_cap, BnxPDiv* pdiv, uint64_t* npdiv,
                         int* overflow, cudaStream_t st);
void launch_brute_force(const uint64_t* rads, uint64_t limit, bnx_pair_t* out, uint64_t cap,
                        unsigned long long* count, cudaStream_t st);
void launch_trial_division(uint64_t start, uint64_t length, const BnxPDiv* pd, uint64_t npd, uint64_t* out,
                           int grid, cudaStream_t st);

}  // namespace bnx
