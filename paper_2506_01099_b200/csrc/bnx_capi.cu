// bnx_capi.cu -- host runtime and C ABI (include/benelux_b200.h) of libbenelux_b200.so.
//
// One context = one GPU + one stream + cached device tables (primes, prime-power
// progressions, exact-division constants) + work buffers reused across calls.  All device
// work of a search is enqueued back to back on the context stream; the host synchronises
// once to read the counters and the (tiny) pair list.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/benelux_b200.h"
#include "bnx_kernels.cuh"

using namespace bnx;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CK(call)                                                                                  \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess) return fail(BNX_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define TRY(call)                   \
    do {                            \
        int r_ = (call);            \
        if (r_ != BNX_OK) return r_; \
    } while (0)

// Device buffers come from the device's stream-ordered memory pool (cudaMallocAsync on the
// active context's stream; the pool keeps freed memory, so a new context or a grown buffer
// does not map fresh pages or synchronise the device the way cudaMalloc / cudaFree do).
thread_local cudaStream_t g_alloc_stream = nullptr;

template <class T>
struct DBuf {
    T* p = nullptr;
    size_t cap = 0;
    int ensure(size_t n) {
        if (n <= cap && p) return BNX_OK;
        if (p) cudaFreeAsync(p, g_alloc_stream);
        p = nullptr;
        cap = 0;
        size_t want = std::max<size_t>(n, 1);
        cudaError_t e = cudaMallocAsync((void**)&p, want * sizeof(T), g_alloc_stream);
        if (e != cudaSuccess) return fail(BNX_ERR_CUDA, std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
        cap = want;
        return BNX_OK;
    }
    void release() {
        if (p) cudaFreeAsync(p, g_alloc_stream);
        p = nullptr;
        cap = 0;
    }
};

uint64_t isqrt_u64(uint64_t x) {
    uint64_t r = (uint64_t)std::sqrt((long double)x);
    while (r > 0 && (r > 0xFFFFFFFFull || r * r > x)) --r;
    while (r + 1 <= 0xFFFFFFFFull && (r + 1) * (r + 1) <= x) ++r;
    return r;
}

uint64_t icbrt_u64(uint64_t x) {
    uint64_t r = (uint64_t)std::cbrt((long double)x);
    auto cube_le = [&](uint64_t v) { return v <= 2642245ull && v * v * v <= x; };
    while (r > 0 && !cube_le(r)) --r;
    while (cube_le(r + 1)) ++r;
    return r;
}

struct Tables {
    uint64_t max_x = 0;
    int include_two = -1;
    uint32_t tile = 0;
    int nwarps = 0;
    uint64_t gen = ~0ull;
    DBuf<BnxProg> small, large;
    DBuf<BnxPDiv> pdiv;
    DBuf<uint4> pd32;  // the first primes of pdiv: (p^-1 mod 2^32, floor((2^32-1)/p), p, 2^32 mod p)
    DBuf<uint32_t> items;
    int nitems = 0;
    uint32_t nsmall = 0;
    uint64_t nlarge = 0, npdiv = 0;
    uint64_t nmedium = 0;  // large[0, nmedium): q < SIEVE_HUGE_Q, once `split` (exact sieve)
    bool split = false;
    void release() {
        small.release();
        large.release();
        pdiv.release();
        pd32.release();
        items.release();
        gen = ~0ull;
    }
};

// Heavy-side generator tables (bnx_heavy.cu): the surplus classes of every powerful number
// b <= max_x, the per-k bit table, and the per-search scratch (counts, scan).
struct HeavyTab {
    uint64_t max_x = 0;
    uint64_t gen = ~0ull;
    DBuf<BnxHeavyEnt> ent;
    uint64_t nent = 0;
    DBuf<uint32_t> kinfo;
    uint64_t nkinfo = 0;
    DBuf<uint64_t> cnt, incl, tile_tot;
    DBuf<uint32_t> klo, kcnt;
    DBuf<uint32_t> tasks;  // k_heavy_sieve marking tasks for (tasks_np2, tasks_kc)
    DBuf<uint16_t> invtab;  // inverses mod p of the primes <= P2 (k_heavy_sieve)
    DBuf<uint32_t> invoff;
    int ntasks = 0, tasks_np2 = -1, tasks_kc = 0;
    DBuf<unsigned char> scan_temp;
    size_t scan_bytes = 0;
    // device build of the class table (bnx_classes.cu): factor table, per-v counts and
    // offsets, unsorted classes, sort keys and permutations, cub scratch
    DBuf<uint32_t> ftab;
    DBuf<uint64_t> vcnt, voff, keys, key_tmp;
    DBuf<BnxHeavyEnt> ent_tmp;
    DBuf<uint32_t> perm, perm_tmp;
    DBuf<unsigned char> cls_scratch;
    void release_build() {
        ftab.release();
        vcnt.release();
        voff.release();
        keys.release();
        key_tmp.release();
        ent_tmp.release();
        perm.release();
        perm_tmp.release();
        cls_scratch.release();
    }
    void release() {
        release_build();
        ent.release();
        kinfo.release();
        cnt.release();
        incl.release();
        tile_tot.release();
        klo.release();
        kcnt.release();
        tasks.release();
        invtab.release();
        invoff.release();
        tasks_np2 = -1;
        scan_temp.release();
        gen = ~0ull;
        max_x = 0;
    }
};

}  // namespace

struct bnx_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    cudaStream_t aux = nullptr;  // second stream: k_tail_heavy beside k_tail (heavy engine)
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    // the heavy engine's search as a CUDA graph, re-captured whenever its parameters change
    bool use_graphs = true;
    // captured searches keyed by their parameters, least recently used evicted: alternating
    // searches (shards of one search run one after another, a streaming run's batch shapes)
    // replay their own graphs instead of re-capturing
    struct GraphEntry {
        std::vector<unsigned char> key;
        cudaGraph_t g = nullptr, g2 = nullptr;
        cudaGraphExec_t e = nullptr, e2 = nullptr;
        uint64_t used = 0;
        void destroy() {
            if (e) cudaGraphExecDestroy(e);
            if (e2) cudaGraphExecDestroy(e2);
            if (g) cudaGraphDestroy(g);
            if (g2) cudaGraphDestroy(g2);
            e = e2 = nullptr;
            g = g2 = nullptr;
        }
    };
    std::vector<GraphEntry> graphs;
    uint64_t graph_tick = 0;
    int num_sms = 148;
    int screen_blocks_per_sm = 1;
    int screen_v = 0;
    int screen_skip = 0;  // profiling only
    int sieve_blocks_per_sm = 1;
    int sieve_v = 0;
    int sieve_nv = 0;              // 32-bit-slot geometry for windows below 2^32 (BNX_SIEVE_NARROW; -1: off)
    int sieve_narrow_blocks_per_sm = 1;
    bool sieve_gbuckets = true;    // large progressions bucketed per window (BNX_SIEVE_GBUCKETS=0: per-segment scan)
    uint32_t sieve_gcap = 0;       // test only (BNX_SIEVE_GCAP): bucket capacity per segment; 0 = SEG / 128
    DBuf<uint64_t> sieve_gbuck;
    DBuf<uint32_t> sieve_gcnt;
    DBuf<unsigned long long> t_split;

    // prime table (device u32 + host mirror)
    DBuf<uint32_t> primes;
    std::vector<uint32_t> h_primes;
    std::vector<uint64_t> h_primes64;  // the last caller-supplied list (memcmp: unchanged?)
    uint64_t primes_limit = 0;  // PrimeList.limit the table covers
    uint64_t gen = 0;           // bumps whenever the table changes
    DBuf<uint64_t> stage64;

    Tables screen_tab, sieve_tab, td_tab;
    HeavyTab heavy_tab;
    int engine = 0;  // 0: heavy-side generator (default), 1: byte screen (BNX_ENGINE=screen)
    bool trace = false;         // BNX_TRACE=1 (see Trace)
    int stop_after = 0;         // profiling only (BNX_STOP_AFTER): run a prefix of the heavy pipeline
    int publish_env = 1;        // BNX_PUBLISH=0: heavy searches read back with a copy node
    int table_lanes = 1;        // Algorithm 3: lanes per element (BNX_TABLE_LANES: 1 or 4; 4 measured slower)
    bool skip_readback = false; // profiling only (BNX_SKIP_READBACK): no D2H copy (results invalid)
    bool host_classes = false;  // BNX_HOST_CLASSES=1: the class table by the host DFS (tests)
    uint64_t heavy_kmin = 0;  // tuning only (BNX_HEAVY_KMIN); 0 = default
    int heavy_grid = 0;       // tuning only (BNX_HEAVY_GRID, CTAs per SM); 0 = default
    int heavy_runs = -1;      // tuning only (BNX_HEAVY_RUNS, fetched screen runs per CTA); -1 = default
    int heavy_run_first = -1; // tuning only (BNX_HEAVY_RUN_FIRST, static share /256); -1 = default
    int heavy_kc = 0;         // tuning only (BNX_HEAVY_KC, k per sieve chunk, multiple of 8); 0 = default
    int sieve_grid = 0;       // tuning only (BNX_SIEVE_GRID, k_heavy_sieve CTAs per SM); 0 = default
    int sieve_threads = 0;    // tuning only (BNX_SIEVE_THREADS, k_heavy_sieve CTA size, 64..256); 0 = default
    int probe_walk = 0;       // profiling only (BNX_PROBE_WALK)
    int local_scan = 1;       // tuning only (BNX_LOCAL_SCAN=0: the cub scan at every bound)
    int exact_warp = -1;      // tuning only (BNX_EXACT_WARP: 1 warp / 0 thread per survivor); -1 = by bound
    uint64_t tail_heavy = 0;  // tuning only (BNX_TAIL_HEAVY); 0 = TAIL_HEAVY
    uint32_t shard = 0, nshards = 1;  // bnx_ctx_set_shard
    DBuf<BnxSurv> q1;
    DBuf<BnxCand> cand;

    DBuf<uint64_t> surv;
    DBuf<BnxCand> heavy;
    DBuf<int> flags;  // (radical sieve)
    int* h_flags = nullptr;  // (radical sieve)
    // The search's device I/O block: counters, flags and the pair rows in one allocation, so
    // one copy reads back the counters, flags and the first PAIR_PREFIX rows (h_io, pinned).
    DBuf<unsigned char> io;
    unsigned long long* ctr_p = nullptr;
    int* sflags_p = nullptr;
    bnx_pair_t* pairs_p = nullptr;
    size_t pairs_cap = 0;
    unsigned char* h_io = nullptr;
    unsigned char* d_h_io = nullptr;  // h_io as the device sees it (mapped pinned memory)
    bool publish = true;              // heavy engine: rows and flags written to h_io by the kernels
    bool q_publish = false;           // ... for the enqueued search
    bool stats_stale = false;         // counters not yet read back (bnx_ctx_stats fetches them)
    uint64_t q_pairs_hint = 0;
    uint64_t pair_prefix = PAIR_PREFIX;  // rows read back with the counters (BNX_PAIR_PREFIX: tests)
    unsigned long long* h_sctr = nullptr;
    int* h_sflags = nullptr;
    bnx_pair_t* h_pairs = nullptr;

    DBuf<uint32_t> t_nsmall;
    DBuf<unsigned long long> t_nlarge;
    DBuf<uint64_t> t_npdiv;
    DBuf<int> t_over;
    DBuf<uint64_t> sieve_out;

    // optional event timing of the pipeline
    int timing = 0;  // 1: generator / pipeline split (two graphs); 2: per-kernel events, direct launches
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
    cudaEvent_t kev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    float screen_ms = 0.f, pipeline_ms = 0.f;
    float kernel_ms[4] = {0.f, 0.f, 0.f, 0.f};  // count + scan, screen (+ sieve), exact, tail

    // rows of a collected search the caller's buffer could not take (bnx_search_collect
    // returns them again on the next call instead of losing them)
    bool rows_pending = false;
    std::vector<bnx_pair_t> pending;

    // the enqueued search
    bool q_valid = false;
    uint64_t q_first = 0, q_last = 0;
    uint32_t q_kinds = 0;
    bnx_stats_t stats{};
};

struct bnx_table {
    bnx_ctx* ctx = nullptr;
    uint64_t size = 0;
    DBuf<uint64_t> slots;
    DBuf<uint64_t> rad_of, rad_next, probe_of, probe_next;  // device copies of the domains
    uint64_t domain_start = 0, count = 0;
    DBuf<bnx_pair_t> rows;
    DBuf<unsigned long long> cnt;  // [0] pairs [1] inserted
    DBuf<int> status;
};

namespace {

// Once per device and process: load every search-path kernel (CUDA loads kernels lazily at
// their first launch, which would otherwise fall inside the first search of a context).
cudaError_t preload_device(int device, cudaStream_t st) {
    static std::mutex mu;
    static std::vector<bool> done;
    std::lock_guard<std::mutex> lock(mu);
    if ((int)done.size() <= device) done.resize(device + 1, false);
    if (done[device]) return cudaSuccess;
    cudaError_t e = heavy_configure();
    if (e == cudaSuccess) e = kernels_preload();
    if (e == cudaSuccess) e = classes_preload(st);
    if (e == cudaSuccess) e = heavy_preload_cub(st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) done[device] = true;
    return e;
}

// BNX_TRACE=1: host wall time of each setup phase (stream synchronised), to stderr.
struct Trace {
    bnx_ctx* c;
    std::chrono::steady_clock::time_point t;
    explicit Trace(bnx_ctx* ctx);
    void mark(const char* what);
};

int activate(bnx_ctx* c) {
    CK(cudaSetDevice(c->device));
    g_alloc_stream = c->stream;
    return BNX_OK;
}

Trace::Trace(bnx_ctx* ctx) : c(ctx) {
    if (c->trace) {
        cudaStreamSynchronize(c->stream);
        t = std::chrono::steady_clock::now();
    }
}

void Trace::mark(const char* what) {
    if (!c->trace) return;
    cudaStreamSynchronize(c->stream);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[bnx] %-28s %9.3f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
}

// Device Eratosthenes up to `limit` (< 2^32): base primes by one block, then a segmented
// pass (count, scan, write).  Replaces the table; host mirror refreshed.
int gen_primes(bnx_ctx* c, uint64_t limit) {
    if (limit >= (1ull << 32)) return fail(BNX_ERR_RANGE, "prime tables are limited to < 2^32");
    if (limit < 2) limit = 2;
    const uint32_t ls = (uint32_t)std::min<uint64_t>(limit, (uint64_t)std::max<uint64_t>(isqrt_u64(limit), 2));
    DBuf<uint32_t> base, cnt;
    TRY(base.ensure(ls / 2 + 16));
    TRY(cnt.ensure(1));
    launch_base_primes(ls, base.p, cnt.p, c->stream);
    CK(cudaGetLastError());
    uint32_t nbase = 0;
    CK(cudaMemcpyAsync(&nbase, cnt.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    uint64_t total = 0;
    if (limit <= ls) {
        TRY(c->primes.ensure(nbase));
        CK(cudaMemcpyAsync(c->primes.p, base.p, sizeof(uint32_t) * nbase, cudaMemcpyDeviceToDevice, c->stream));
        total = nbase;
    } else {
        const uint64_t nblocks = (limit + 1 + 32767) / 32768;
        DBuf<uint32_t> counts;
        DBuf<uint64_t> offs;
        TRY(counts.ensure(nblocks));
        TRY(offs.ensure(nblocks + 1));
        launch_prime_seg(0, limit, base.p, nbase, counts.p, nullptr, nullptr, nblocks, c->stream);
        launch_scan_counts(counts.p, nblocks, 0, offs.p, c->stream);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(&total, offs.p + nblocks, sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        TRY(c->primes.ensure(total));
        launch_prime_seg(0, limit, base.p, nbase, counts.p, offs.p, c->primes.p, nblocks, c->stream);
        CK(cudaGetLastError());
        counts.release();
        offs.release();
    }
    c->h_primes.resize(total);
    c->h_primes64.clear();
    CK(cudaMemcpyAsync(c->h_primes.data(), c->primes.p, sizeof(uint32_t) * total, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    base.release();
    cnt.release();
    c->primes_limit = limit;
    c->gen++;
    return BNX_OK;
}

// Caller-supplied PrimeList (host, ascending, uint64): checked for coverage, the primes up to
// `need` are copied to the device.
int upload_primes(bnx_ctx* c, const uint64_t* primes, size_t np, uint64_t primes_limit, uint64_t need) {
    if (primes_limit < need)
        return fail(BNX_ERR_PRIMES_UNCOVERED, "prime list covers " + std::to_string(primes_limit) +
                                                  " but interval endpoint needs " + std::to_string(need));
    size_t k = (size_t)(std::upper_bound(primes, primes + np, need) - primes);
    TRY(c->stage64.ensure(k));
    TRY(c->primes.ensure(k));
    // The list is compared with the host copy of the one the device tables were built from;
    // only a changed list is copied to the device (and the tables rebuilt).
    // (a list already on the device that extends this one serves too: a streaming run
    // prepares for its final bound once, then searches batches with smaller bounds)
    const bool same = c->gen > 0 && c->h_primes64.size() >= k && c->primes_limit >= need &&
                      (c->h_primes64.size() == k || c->h_primes64[k] > need) &&
                      (k == 0 || std::memcmp(c->h_primes64.data(), primes, sizeof(uint64_t) * k) == 0);
    if (k && !same) {
        CK(cudaMemcpyAsync(c->stage64.p, primes, sizeof(uint64_t) * k, cudaMemcpyHostToDevice, c->stream));
        launch_narrow(c->stage64.p, k, c->primes.p, c->stream);
        CK(cudaGetLastError());
    }
    if (!same) {
        c->h_primes.resize(k);
        for (size_t i = 0; i < k; ++i) c->h_primes[i] = (uint32_t)primes[i];
        c->h_primes64.assign(primes, primes + k);
        c->primes_limit = need;  // the device copy holds exactly the primes <= need
        c->gen++;
    }
    return BNX_OK;
}

int ensure_primes(bnx_ctx* c, const uint64_t* primes, size_t np, uint64_t primes_limit, uint64_t need) {
    if (primes) return upload_primes(c, primes, np, primes_limit, need);
    if (c->gen > 0 && c->primes_limit >= need) return BNX_OK;
    uint64_t lim = std::max<uint64_t>(need, 65536);
    if (lim >= (1ull << 32)) lim = (1ull << 32) - 1;
    return gen_primes(c, lim);
}

// Work items of the screen's per-tile progressions (q < tile, sorted by q): a progression
// with q < 2048 is split into R interleaved items of about ITEM_HITS hits per tile; the
// rest go 32 progressions per item (one per lane).  Encoding: j | r << 8 | R << 16 |
// packed << 31.  The items are dealt to the `nwarps` warps of a CTA by longest-processing-
// time-first on a cost model (SASS-measured: ~40 instructions of setup per item, ~4 per
// split-loop iteration, ~9 per lane-packed iteration), so the warps reach the tile barrier
// together.  Layout returned: [nwarps + 1 offsets][items grouped by warp].
std::vector<uint32_t> build_items(const std::vector<BnxProg>& small, uint32_t tile, int nwarps) {
    constexpr uint32_t ITEM_HITS = 32 * 12;
    constexpr uint32_t C_SETUP = 40, C_SPLIT = 4, C_PACKED = 9;
    std::vector<std::pair<uint32_t, uint32_t>> v;  // (cost, item)
    size_t j = 0;
    for (; j < small.size() && small[j].q < 2048; ++j) {
        const uint32_t hits = tile / (uint32_t)small[j].q;
        const uint32_t R = std::max(1u, (hits + ITEM_HITS / 2) / ITEM_HITS);
        const uint32_t iters = (hits / R + 31) / 32;
        for (uint32_t r = 0; r < R; ++r) v.push_back({C_SETUP + C_SPLIT * iters, (uint32_t)j | (r << 8) | (R << 16)});
    }
    for (; j < small.size(); j += 32)
        v.push_back({C_SETUP + C_PACKED * ((tile + (uint32_t)small[j].q - 1) / (uint32_t)small[j].q),
                     (uint32_t)j | (1u << 31)});
    std::stable_sort(v.begin(), v.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
    std::vector<std::vector<uint32_t>> per(nwarps);
    std::vector<uint64_t> load(nwarps, 0);
    for (auto& e : v) {
        const int w = (int)(std::min_element(load.begin(), load.end()) - load.begin());
        load[w] += e.first;
        per[w].push_back(e.second);
    }
    std::vector<uint32_t> out(nwarps + 1, 0);
    for (int w = 0; w < nwarps; ++w) {
        out[w + 1] = out[w] + (uint32_t)per[w].size();
    }
    for (int w = 0; w < nwarps; ++w) out.insert(out.end(), per[w].begin(), per[w].end());
    return out;
}

int build_tables(bnx_ctx* c, Tables& t, uint64_t max_x, int include_two, uint32_t tile, int nwarps) {
    // a table built for a larger bound serves a smaller one: progressions q > x never divide x
    if (t.gen == c->gen && t.max_x >= max_x && t.include_two == include_two && t.tile == tile && t.nwarps == nwarps)
        return BNX_OK;
    const uint64_t root = isqrt_u64(max_x);
    const uint64_t np = (uint64_t)(std::upper_bound(c->h_primes.begin(), c->h_primes.end(), (uint32_t)std::min<uint64_t>(root, 0xFFFFFFFFull)) - c->h_primes.begin());
    const uint64_t cb = icbrt_u64(max_x);
    const uint64_t npc = (uint64_t)(std::upper_bound(c->h_primes.begin(), c->h_primes.end(), (uint32_t)std::min<uint64_t>(cb, 0xFFFFFFFFull)) - c->h_primes.begin());
    const uint64_t large_cap = np + 63 * npc + 64;
    const uint32_t small_cap = (uint32_t)(tile == (uint32_t)SIEVE_TILE ? SIEVE_MAXS : SCREEN_MAXS);
    TRY(t.small.ensure(small_cap));
    TRY(t.large.ensure(large_cap));
    TRY(t.pdiv.ensure(np + 1));
    TRY(c->t_nsmall.ensure(1));
    TRY(c->t_nlarge.ensure(1));
    TRY(c->t_npdiv.ensure(1));
    TRY(c->t_over.ensure(1));
    CK(cudaMemsetAsync(c->t_nsmall.p, 0, sizeof(uint32_t), c->stream));
    CK(cudaMemsetAsync(c->t_nlarge.p, 0, sizeof(unsigned long long), c->stream));
    CK(cudaMemsetAsync(c->t_npdiv.p, 0, sizeof(uint64_t), c->stream));
    CK(cudaMemsetAsync(c->t_over.p, 0, sizeof(int), c->stream));
    if (np) {
        launch_build_tables(c->primes.p, np, max_x, include_two, tile, t.small.p, c->t_nsmall.p, small_cap, t.large.p,
                            c->t_nlarge.p, large_cap, t.pdiv.p, c->t_npdiv.p, c->t_over.p, c->stream);
        CK(cudaGetLastError());
    }
    uint32_t ns = 0;
    unsigned long long nl = 0;
    uint64_t npd = 0;
    int over = 0;
    CK(cudaMemcpyAsync(&ns, c->t_nsmall.p, sizeof(ns), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(&nl, c->t_nlarge.p, sizeof(nl), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(&npd, c->t_npdiv.p, sizeof(npd), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(&over, c->t_over.p, sizeof(over), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (over) return fail(BNX_ERR_CUDA, "progression table overflow");
    // per-tile progressions sorted by q, and the screen's work items (see k_screen)
    if (ns > small_cap) return fail(BNX_ERR_CUDA, "too many small progressions");
    std::vector<BnxProg> hs(ns);
    if (ns) {
        CK(cudaMemcpyAsync(hs.data(), t.small.p, sizeof(BnxProg) * ns, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        std::sort(hs.begin(), hs.end(), [](const BnxProg& x, const BnxProg& y) { return x.q < y.q; });
        CK(cudaMemcpyAsync(t.small.p, hs.data(), sizeof(BnxProg) * ns, cudaMemcpyHostToDevice, c->stream));
    }
    std::vector<uint32_t> items = build_items(hs, tile, nwarps);
    if (items.size() > 2 * (size_t)SCREEN_MAXS) return fail(BNX_ERR_CUDA, "too many screen work items");
    TRY(t.items.ensure(items.size() + 1));
    if (!items.empty())
        CK(cudaMemcpyAsync(t.items.p, items.data(), sizeof(uint32_t) * items.size(), cudaMemcpyHostToDevice,
                           c->stream));
    {  // 32-bit divisibility constants of the heavy path's trial primes (<= cbrt(S))
        const uint64_t n32 = std::min<uint64_t>(npd, HEAVY_NP3);
        TRY(t.pd32.ensure(n32 + 1));
        launch_pdiv32(t.pdiv.p, n32, t.pd32.p, c->stream);
        CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(c->stream));  // the host vectors above must outlive the copies
    t.nitems = (int)items.size();
    t.nsmall = ns;
    t.nlarge = nl;
    t.npdiv = npd;
    t.max_x = max_x;
    t.include_two = include_two;
    t.tile = tile;
    t.nwarps = nwarps;
    t.split = false;
    t.nmedium = 0;
    t.gen = c->gen;
    return BNX_OK;
}

// The surplus classes: every powerful b = prod p^(e+1) <= max_x (DFS over the primes up to
// sqrt(max_x)) with sigma = prod p^e = m r, r = prod p; and kinfo[k] for k <= sqrt(max_x / 2)
// (the largest k any class can use: k^2 <= 2m * max_x / (m r^2) <= max_x / 2 for r >= 2).
int build_heavy_host(bnx_ctx* c, uint64_t max_x);

// The surplus-class table on the device (bnx_classes.cu): one host sync, to size the table.
int build_heavy(bnx_ctx* c, uint64_t max_x) {
    HeavyTab& h = c->heavy_tab;
    // a table for a larger bound serves (its extra classes count zero items), unless it is so
    // much larger that the per-search class pass would dominate: then rebuild for this bound
    if (h.gen == c->gen && h.max_x >= max_x && h.max_x / 16 <= max_x) return BNX_OK;
    if (h.gen == c->gen && h.max_x && h.max_x < max_x) {
        // growing (a streaming run's batches come in with rising bounds): build for twice the
        // old bound at least, so a run to S rebuilds O(log S) times -- if the primes cover it
        const uint64_t grown = std::min<uint64_t>(std::max<uint64_t>(max_x, 2 * h.max_x), 1ull << 48);
        if (c->primes_limit >= isqrt_u64(grown) || (!c->h_primes.empty() && c->h_primes.back() >= isqrt_u64(grown)))
            max_x = grown;
    }
    if (c->host_classes) return build_heavy_host(c, max_x);
    const std::vector<uint32_t>& P = c->h_primes;
    const uint64_t root = isqrt_u64(max_x);
    if (c->primes_limit < root && (P.empty() || P.back() < root))
        return fail(BNX_ERR_PRIMES_UNCOVERED, "prime table does not cover sqrt(bound)");
    const uint64_t K = isqrt_u64(max_x / 2) + 3;  // kinfo entries (see build_heavy_host)
    const uint64_t Ltab = std::max<uint64_t>(root, K);
    auto upto = [&](uint64_t v) {
        return (uint64_t)(std::upper_bound(P.begin(), P.end(), (uint32_t)std::min<uint64_t>(v, 0xFFFFFFFFull)) - P.begin());
    };
    const ClassPlan pl = class_plan(max_x, upto(root));
    if (!pl.ok) return fail(BNX_ERR_RANGE, "class table key too long");
    Trace tr(c);
    TRY(h.ftab.ensure(Ltab + 1));
    TRY(h.vcnt.ensure(pl.V + 2));
    TRY(h.voff.ensure(pl.V + 2));
    size_t sb = class_scratch_bytes(pl, 0);
    TRY(h.cls_scratch.ensure(sb));
    CK(class_count(pl, Ltab, c->primes.p, upto(Ltab), h.ftab.p, h.vcnt.p, h.voff.p, h.cls_scratch.p, h.cls_scratch.cap,
                   c->stream));
    uint64_t total = 0;
    CK(cudaMemcpyAsync(&total, h.voff.p + pl.V + 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    tr.mark("classes: factor table + count");
    if (total == 0 || total > 0xFFFFFFFFull) return fail(BNX_ERR_CUDA, "class table size out of range");
    sb = class_scratch_bytes(pl, total);
    TRY(h.cls_scratch.ensure(sb));
    TRY(h.ent_tmp.ensure(total));
    TRY(h.ent.ensure(total));
    TRY(h.keys.ensure(total * pl.nwords));
    TRY(h.key_tmp.ensure(total));
    TRY(h.perm.ensure(total));
    TRY(h.perm_tmp.ensure(total));
    TRY(h.kinfo.ensure(K));
    tr.mark("classes: allocate");
    CK(class_build(pl, total, c->primes.p, h.ftab.p, h.voff.p, h.ent_tmp.p, h.ent.p, h.keys.p, h.key_tmp.p, h.perm.p,
                   h.perm_tmp.p, h.cls_scratch.p, h.cls_scratch.cap, h.kinfo.p, K, c->stream));
    tr.mark("classes: build + sort");
    h.release_build();  // (stream-ordered: the per-search buffers below reuse the memory)
    TRY(h.cnt.ensure(total));
    TRY(h.tile_tot.ensure((total + HEAVY_TILE - 1) / HEAVY_TILE));
    TRY(h.incl.ensure(total));
    TRY(h.klo.ensure(total));
    TRY(h.kcnt.ensure(total));
    h.scan_bytes = heavy_scan_temp_bytes(total);
    TRY(h.scan_temp.ensure(h.scan_bytes));
    tr.mark("classes: search buffers");
    h.nent = total;
    h.nkinfo = K;
    h.max_x = max_x;
    h.gen = c->gen;
    return BNX_OK;
}

// The same table by a depth-first search on the host (BNX_HOST_CLASSES=1; tests compare the
// two): every powerful b = prod p^(e+1) <= max_x (DFS over the primes up to sqrt(max_x)) with
// sigma = prod p^e = m r, r = prod p; and kinfo[k] for k <= sqrt(max_x / 2) (the largest k
// any class can use: k^2 <= 2m * max_x / (m r^2) <= max_x / 2 for r >= 2).
int build_heavy_host(bnx_ctx* c, uint64_t max_x) {
    HeavyTab& h = c->heavy_tab;
    const std::vector<uint32_t>& P = c->h_primes;
    const uint64_t root = isqrt_u64(max_x);
    if (root >= 2 && (P.empty() || (P.back() < root && c->primes_limit < root)))
        return fail(BNX_ERR_PRIMES_UNCOVERED, "prime table does not cover sqrt(bound)");
    std::vector<BnxHeavyEnt> ents;
    ents.reserve((size_t)(2.5 * std::sqrt((double)max_x)) + 64);
    struct Node { uint64_t b, sigma, r; uint32_t rmask, rbig, rbig_min; size_t next; };
    std::vector<Node> stack;
    stack.push_back(Node{1, 1, 1, 0, 1, 0, 0});
    while (!stack.empty()) {
        const Node f = stack.back();
        stack.pop_back();
        ents.push_back(BnxHeavyEnt{f.b, f.sigma / f.r, (uint32_t)f.r, f.rmask, f.rbig, f.rbig_min});
        for (size_t i = f.next; i < P.size(); ++i) {
            const uint64_t p = P[i];
            if (p > root || f.b > max_x / (p * p)) break;
            Node ch{f.b * p * p, f.sigma * p, f.r * p, f.rmask, f.rbig, f.rbig_min, i + 1};
            if (i < 31) ch.rmask |= 1u << i;
            else {
                ch.rbig = (uint32_t)(f.rbig * p);
                if (!ch.rbig_min) ch.rbig_min = (uint32_t)p;
            }
            for (;;) {
                stack.push_back(ch);
                if (ch.b > max_x / p) break;
                ch.b *= p;
                ch.sigma *= p;
            }
        }
    }
    // (kept in DFS order: classes of one prime structure stay together, which measured ~10%
    // faster at 2^32 than sorting by sigma, and the host sort cost 0.35 s at 2^40, 7 s at 2^48;
    // classes with no k in a domain simply count zero items)
    const uint64_t K = isqrt_u64(max_x / 2) + 3;
    std::vector<uint32_t> kinfo(K, 0);
    for (size_t i = 0; i < 31 && i < P.size(); ++i)
        for (uint64_t k = P[i]; k < K; k += P[i]) kinfo[k] |= 1u << i;
    for (size_t i = 0; i < P.size() && (uint64_t)P[i] * P[i] < K; ++i) {
        const uint64_t q = (uint64_t)P[i] * P[i];
        for (uint64_t k = q; k < K; k += q) kinfo[k] |= 0x80000000u;
    }
    kinfo[0] = 0x80000000u;
    TRY(h.ent.ensure(ents.size()));
    TRY(h.kinfo.ensure(K));
    TRY(h.cnt.ensure(ents.size()));
    TRY(h.tile_tot.ensure((ents.size() + HEAVY_TILE - 1) / HEAVY_TILE));
    TRY(h.incl.ensure(ents.size()));
    TRY(h.klo.ensure(ents.size()));
    TRY(h.kcnt.ensure(ents.size()));
    h.scan_bytes = heavy_scan_temp_bytes(ents.size());
    TRY(h.scan_temp.ensure(h.scan_bytes));
    CK(cudaMemcpyAsync(h.ent.p, ents.data(), sizeof(BnxHeavyEnt) * ents.size(), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(h.kinfo.p, kinfo.data(), sizeof(uint32_t) * K, cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));  // the host vectors must outlive the copies
    h.nent = ents.size();
    h.nkinfo = K;
    h.max_x = max_x;
    h.gen = c->gen;
    return BNX_OK;
}

// (Re)allocate the I/O block for `rows` pair rows (the counters are reset by every search).
int ensure_pairs(bnx_ctx* c, size_t rows) {
    rows = std::max<size_t>(rows, PAIR_PREFIX);
    TRY(c->io.ensure(IO_PAIRS + sizeof(bnx_pair_t) * rows));
    c->ctr_p = reinterpret_cast<unsigned long long*>(c->io.p + IO_CTR);
    c->sflags_p = reinterpret_cast<int*>(c->io.p + IO_FLAGS);
    c->pairs_p = reinterpret_cast<bnx_pair_t*>(c->io.p + IO_PAIRS);
    c->pairs_cap = (c->io.cap - IO_PAIRS) / sizeof(bnx_pair_t);
    return BNX_OK;
}

int ensure_work(bnx_ctx* c) {
    if (!c->surv.p) TRY(c->surv.ensure(1 << 20));
    if (!c->heavy.p) TRY(c->heavy.ensure(1 << 16));  // (k_tail_heavy's list: a few hundred below 1.4e12)
    if (!c->pairs_p) TRY(ensure_pairs(c, 1 << 14));
    return BNX_OK;
}

// The read-back at the end of every search, one copy: counters, flags and the first
// PAIR_PREFIX pair rows (every search up to 2^48 has fewer: 49 of both kinds), so collect()
// needs no second copy.
int read_back(bnx_ctx* c) {
    if (c->skip_readback) return BNX_OK;  // (profiling only)
    CK(cudaMemcpyAsync(c->h_io, c->io.p, IO_PAIRS + sizeof(bnx_pair_t) * c->pair_prefix, cudaMemcpyDeviceToHost,
                       c->stream));
    return BNX_OK;
}

int grid_for(bnx_ctx* c) { return c->num_sms * 4; }

uint64_t iroot4_u64(uint64_t x) {
    uint64_t r = isqrt_u64(isqrt_u64(x));
    while ((r + 1) * (r + 1) * (r + 1) * (r + 1) <= x) ++r;
    return r;
}

// Heavy engine: k_heavy_count, scan, k_heavy_screen, k_heavy_exact, then the tail on the
// exact candidates.
int enqueue_heavy(bnx_ctx* c, uint64_t n_first, uint64_t n_last, uint32_t kinds) {
    Trace tr(c);
    HeavyTab& h = c->heavy_tab;
    Tables& t = c->screen_tab;  // pdiv: odd primes <= sqrt(bound)
    TRY(ensure_work(c));
    {  // screen survivors grow like sqrt(bound) (88,139 below 2^32, 1.45M below 1.4e12): sized
        // up front so that a first search does not overflow, grow and run again
        const double est = 1.3 * 88139.0 * std::sqrt((double)(n_last + 1) / 4294967296.0) + 65536.0;
        TRY(c->q1.ensure(std::max<size_t>(c->q1.cap, (size_t)std::min(est, 1e9))));
    }
    if (!c->cand.p) TRY(c->cand.ensure(1 << 16));
    const uint64_t y_max = n_last + 2;
    const uint64_t p2 = iroot4_u64(y_max), p3 = icbrt_u64(y_max);
    auto odd_upto = [&](uint64_t v) -> uint64_t {  // odd primes <= v in the host table
        const uint64_t all = (uint64_t)(std::upper_bound(c->h_primes.begin(), c->h_primes.end(),
                                                         (uint32_t)std::min<uint64_t>(v, 0xFFFFFFFFull)) -
                                        c->h_primes.begin());
        return (all && c->h_primes[0] == 2) ? all - 1 : all;
    };
    const uint64_t np3 = std::min<uint64_t>(odd_upto(p3), t.npdiv);
    // stage-1 primes: the odd primes <= y_max^(1/4), rounded up to a multiple of 32 (the
    // screen tests 32 per unrolled block anyway, and every extra prime tightens U(c): the
    // bound only needs every prime factor of the cofactor to exceed the last prime tested)
    const uint64_t np2 = std::min<uint64_t>({(odd_upto(p2) + 31) & ~31ull, t.npdiv, (uint64_t)HEAVY_NP3});
    const uint64_t off2 = c->h_primes[0] == 2 ? 1 : 0;
    const uint64_t p_last = np2 ? c->h_primes[np2 - 1 + off2] : 2;
    const uint64_t p1 = np2 < t.npdiv ? c->h_primes[np2 + off2] : p_last + 1;  // smallest untested prime
    if (np2 > (uint64_t)HEAVY_NP2 || np3 > (uint64_t)HEAVY_NP3)
        return fail(BNX_ERR_RANGE, "bound too large for the heavy generator");
    // k_heavy_sieve: chunk length (masks of 32 primes per word, ~32 KB of shared memory) and
    // the marking tasks: prime j, side, sub-progression r of R, about HEAVY_TASK_HITS hits each
    const int W = (int)((np2 + 31) / 32);
    (void)W;
    // hit lists: 2 x kc x (8 slots x 2 B + 1 B) = 26 KB of shared memory at kc = 768 (measured
    // sweep, BNX_HEAVY_KC: 768 beats 1536 by 7% at 2^40 and 14% at 2^48 -- twice the CTAs per SM)
    const int kc = c->heavy_kc ? c->heavy_kc : 768;
    if (h.tasks_np2 != (int)np2 || h.tasks_kc != kc) {
        std::vector<uint32_t> tk, ioff;
        std::vector<uint16_t> itab;
        for (uint64_t j = 0; j < np2; ++j) {
            const uint32_t p = c->h_primes[j + (c->h_primes[0] == 2 ? 1 : 0)];
            ioff.push_back((uint32_t)itab.size());
            const size_t o = itab.size();
            itab.resize(o + p);
            itab[o] = 0;
            if (p > 1) itab[o + 1] = 1;
            for (uint32_t v = 2; v < p; ++v)  // v^-1 = -(p / v) (p mod v)^-1 (mod p)
                itab[o + v] = (uint16_t)((uint64_t)(p - p / v) * itab[o + p % v] % p);
            const uint32_t hits = (uint32_t)((kc + p - 1) / p);
            const uint32_t R = std::max<uint32_t>(1, (hits + HEAVY_TASK_HITS - 1) / HEAVY_TASK_HITS);
            for (uint32_t side = 0; side < 2; ++side)
                for (uint32_t r = 0; r < R; ++r) tk.push_back((uint32_t)j | side << 10 | r << 11 | R << 21);
        }
        TRY(h.tasks.ensure(tk.size()));
        TRY(h.invtab.ensure(itab.size()));
        TRY(h.invoff.ensure(ioff.size() + 1));
        CK(cudaMemcpyAsync(h.tasks.p, tk.data(), sizeof(uint32_t) * tk.size(), cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(h.invtab.p, itab.data(), sizeof(uint16_t) * itab.size(), cudaMemcpyHostToDevice, c->stream));
        if (!ioff.empty())
            CK(cudaMemcpyAsync(h.invoff.p, ioff.data(), sizeof(uint32_t) * ioff.size(), cudaMemcpyHostToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        h.ntasks = (int)tk.size();
        h.tasks_np2 = (int)np2;
        h.tasks_kc = kc;
    }
    tr.mark("enqueue: sieve tasks");
    HeavyArgs ha;
    std::memset(&ha, 0, sizeof(ha));  // (the graph key compares bytes, padding included)
    ha.kcnt = h.kcnt.p;
    ha.tasks = h.tasks.p;
    ha.ntasks = h.ntasks;
    ha.kc = kc;
    // measured (scripts/engine_compare.py, KMIN sweep): with <= 64 primes below P2 (bounds
    // up to ~2^33) trial division is as fast as the sieve; above, sieving classes with >= 256
    // k is best (measured sweep at 2^40)
    ha.kmin = c->heavy_kmin ? c->heavy_kmin : (np2 <= 64 ? ~0ull : HEAVY_KMIN_DEFAULT);
    ha.invtab = h.invtab.p;
    ha.invoff = h.invoff.p;
    ha.ent = h.ent.p;
    ha.nent = h.nent;
    ha.cnt = h.cnt.p;
    ha.incl = h.incl.p;
    ha.klo = h.klo.p;
    ha.kinfo = h.kinfo.p;
    ha.nkinfo = h.nkinfo;
    ha.x_lo = n_first;
    ha.x_hi = n_last + 1;
    ha.n_first = n_first;
    ha.n_last = n_last;
    ha.pdiv = t.pdiv.p;
    ha.pd32 = t.pd32.p;
    ha.np2 = (int)np2;
    ha.np3 = np3;
    ha.p1 = p1;
    ha.p1sq = ha.p1 * ha.p1;
    ha.p1cube = ha.p1sq * ha.p1;
    ha.inv_p1f = 1.0f / (float)ha.p1;
    ha.cube_filter = p_last >= 7;
    ha.q1 = c->q1.p;
    ha.q1_cap = c->q1.cap;
    ha.cand = c->cand.p;
    ha.cand_cap = c->cand.cap;
    ha.heavy = c->heavy.p;
    ha.heavy_cap = c->heavy.cap;
    ha.kinds = kinds;
    ha.ctr = c->ctr_p;
    ha.flags = c->sflags_p;
    ha.shard = c->shard;
    ha.nshards = c->nshards;
    ha.tail_heavy = c->tail_heavy ? c->tail_heavy : TAIL_HEAVY;
    // CTAs per SM (measured sweeps, scripts/engine_compare.py, scripts/sweep_time.sh): one
    // wave of k_heavy_screen below ~2^33 -- 7 CTAs per SM (8 fit at 32 registers, but the
    // eighth slot left free lets k_heavy_exact's CTAs start early: -1% at 2^32); more, smaller runs when the sieve
    // shares the GPU (40 per SM for domains of 2^38 or more: -2% at 2^40 and 2^44)
    const bool wide_sieve = ha.kmin != ~0ull && !heavy_sieve_mask((int)np2);
    const int grid_mult = c->heavy_grid ? c->heavy_grid
                                        : (!wide_sieve ? 7 : (n_last - n_first >= (1ull << 38) ? 40 : 20));
    const int grid = c->num_sms * grid_mult;
    // k_heavy_exact: a thread per survivor from P2 on (measured: 0.45 ms at 2^40 against
    // 1.17 ms for a warp per survivor trying only the deciding primes, whose per-survivor set-up
    // outweighs the primes it skips); the warp form serves domains with few survivors
    ha.exact_warp = c->exact_warp >= 0 ? c->exact_warp : 0;
    ha.probe_walk = c->probe_walk;
    {  // no sieve classes and few tiles: per-tile count scan, the tile offsets scanned by the
        // screen itself (no scan kernels between the count and the screen)
        const uint64_t nt = (h.nent + HEAVY_TILE - 1) / HEAVY_TILE;
        if (c->local_scan && ha.kmin == ~0ull && nt && nt <= (uint64_t)HEAVY_TILES_MAX) {
            ha.ntiles = (uint32_t)nt;
            ha.tile_tot = h.tile_tot.p;
        }
    }
    // (measured, scripts/sweep_sieve40.sh: 256-thread CTAs with kc = 768 beat 128 and 64 at
    // 2^40 and 1.4e12 by 6-28%)
    ha.sieve_threads = (uint32_t)c->sieve_threads;
    ha.sieve_ctas = c->sieve_grid ? (uint32_t)(c->num_sms * c->sieve_grid) : (wide_sieve ? 0u : (uint32_t)(c->num_sms * 4));
    // measured (scripts/sweep_env.sh BNX_HEAVY_RUNS / BNX_HEAVY_RUN_FIRST): in the one-wave
    // case, half the items in static runs and the rest in 2 fetched runs per CTA (-10% at
    // 2^32); with several waves (sieve bounds) the CTA scheduler already balances
    ha.run_mult = c->heavy_runs >= 0 ? (uint32_t)c->heavy_runs : (!wide_sieve ? 2u : 0u);
    ha.run_first = c->heavy_run_first >= 0 ? (uint32_t)c->heavy_run_first : 128u;
    TailArgs ta;
    std::memset(&ta, 0, sizeof(ta));
    ta.cands = c->cand.p;
    ta.cand_cap = c->cand.cap;
    ta.heavy = c->heavy.p;
    ta.heavy_cap = c->heavy.cap;
    ta.pdiv = t.pdiv.p;
    ta.npdiv = t.npdiv;
    ta.kinds = kinds;
    ta.pairs = c->pairs_p;
    ta.pair_cap = c->pairs_cap;
    ta.ctr = c->ctr_p;
    // the kernels publish the rows and overflow flags into the mapped host block themselves
    // (no read-back copy node at the end of the graph); the block is zeroed here first, so a
    // row with m = 0 marks the end of the list
    const bool publish = c->publish_env && !c->stop_after && !c->skip_readback;
    if (publish) {
        ta.host_pairs = reinterpret_cast<bnx_pair_t*>(c->d_h_io + IO_PAIRS);
        ta.host_prefix = c->pair_prefix;
        ta.host_flags = reinterpret_cast<int*>(c->d_h_io + IO_FLAGS);
        ha.host_flags = ta.host_flags;
        std::memset(c->h_io + IO_FLAGS, 0, IO_PAIRS - IO_FLAGS + sizeof(bnx_pair_t) * c->pair_prefix);
    }
    // two phases (generator; tail + read-back), so the timing events sit between them
    auto record_gen = [&]() -> int {
        if (!ha.nent) {  // (otherwise k_heavy_count zeroes the counters and flags)
            CK(cudaMemsetAsync(c->ctr_p, 0, sizeof(unsigned long long) * CTR_N, c->stream));
            CK(cudaMemsetAsync(c->sflags_p, 0, sizeof(int) * 4, c->stream));
        }
        launch_heavy(ha, h.scan_temp.p, h.scan_bytes, grid, c->stream, nullptr, c->aux, c->fork_ev, c->join_ev,
                     c->timing == 2 ? c->kev : nullptr, c->stop_after);
        CK(cudaGetLastError());
        return BNX_OK;
    };
    // without timing events the whole search is one graph, and k_tail a programmatic
    // dependent of k_heavy_exact
    const bool single = c->use_graphs && !c->timing;
    auto record_tail = [&]() -> int {
        if (c->stop_after) return read_back(c);  // (profiling: a prefix of the pipeline)
        // k_tail_heavy (the few candidates with many residue-class members) overlaps k_tail
        CK(cudaEventRecord(c->fork_ev, c->stream));
        CK(cudaStreamWaitEvent(c->aux, c->fork_ev, 0));
        launch_tail_heavy(ta, c->aux);
        CK(cudaEventRecord(c->join_ev, c->aux));
        launch_tail_light(ta, grid_for(c), c->stream, single);
        CK(cudaStreamWaitEvent(c->stream, c->join_ev, 0));
        CK(cudaGetLastError());
        return publish ? BNX_OK : read_back(c);
    };
    if (!c->use_graphs || c->timing == 2) {
        if (c->timing) CK(cudaEventRecord(c->ev[0], c->stream));
        TRY(record_gen());
        if (c->timing) CK(cudaEventRecord(c->ev[1], c->stream));
        TRY(record_tail());
        if (c->timing) CK(cudaEventRecord(c->ev[2], c->stream));
        if (c->timing == 2) CK(cudaEventRecord(c->kev[4], c->stream));
    } else {
        // two graph launches replay the whole search (about ten stream operations): the host
        // enqueue cost and the inter-kernel gaps go; re-captured when any parameter changes
        std::vector<unsigned char> key(sizeof(ha) + sizeof(ta) + 4 * sizeof(uint64_t));
        unsigned char* kp = key.data();
        std::memcpy(kp, &ha, sizeof(ha));
        std::memcpy(kp + sizeof(ha), &ta, sizeof(ta));
        const uint64_t extra[4] = {(uint64_t)(uintptr_t)c->stream, (uint64_t)grid,
                                   (uint64_t)(uintptr_t)h.scan_temp.p ^ (uint64_t)h.scan_bytes << 1, (uint64_t)single};
        std::memcpy(kp + sizeof(ha) + sizeof(ta), extra, sizeof(extra));
        bnx_ctx::GraphEntry* ge = nullptr;
        for (auto& g : c->graphs)
            if (g.key == key) ge = &g;
        if (!ge) {
            constexpr size_t MAX_GRAPHS = 8;
            if (c->graphs.size() >= MAX_GRAPHS) {
                auto lru = std::min_element(c->graphs.begin(), c->graphs.end(),
                                            [](const auto& x, const auto& y) { return x.used < y.used; });
                CK(cudaStreamSynchronize(c->stream));  // (no launch of the evicted graph may be pending)
                lru->destroy();
                c->graphs.erase(lru);
            }
            c->graphs.emplace_back();
            ge = &c->graphs.back();
            auto capture = [&](auto&& fn, cudaGraph_t* g, cudaGraphExec_t* ex) -> int {
                CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
                const int rc = fn();
                const cudaError_t ec = cudaStreamEndCapture(c->stream, g);
                if (rc != BNX_OK) return rc;
                if (ec != cudaSuccess) return fail(BNX_ERR_CUDA, std::string("stream capture: ") + cudaGetErrorString(ec));
                CK(cudaGraphInstantiate(ex, *g, 0));
                return BNX_OK;
            };
            int rc;
            if (single) {
                rc = capture([&]() -> int { TRY(record_gen()); return record_tail(); }, &ge->g, &ge->e);
            } else {
                rc = capture(record_gen, &ge->g, &ge->e);
                if (rc == BNX_OK) rc = capture(record_tail, &ge->g2, &ge->e2);
            }
            if (rc != BNX_OK) {
                ge->destroy();
                c->graphs.pop_back();
                return rc;
            }
            ge->key = key;
            tr.mark("enqueue: graph capture");
        }
        ge->used = ++c->graph_tick;
        if (single) {
            CK(cudaGraphLaunch(ge->e, c->stream));
        } else {
            CK(cudaEventRecord(c->ev[0], c->stream));
            CK(cudaGraphLaunch(ge->e, c->stream));
            CK(cudaEventRecord(c->ev[1], c->stream));
            CK(cudaGraphLaunch(ge->e2, c->stream));
            CK(cudaEventRecord(c->ev[2], c->stream));
        }
    }
    c->q_valid = true;
    c->q_publish = publish;
    c->q_first = n_first;
    c->q_last = n_last;
    c->q_kinds = kinds;
    c->stats = bnx_stats_t{};
    c->stats.integers = n_last - n_first + 1;
    // this library's kernels: count, screen, [sieve], exact, tail, tail_heavy (the two cub
    // scan kernels are library code and not counted)
    c->stats.kernel_launches = ha.nent ? (ha.kmin != ~0ull ? 6 : 5) : 3;
    return BNX_OK;
}

int empty_search(bnx_ctx* c, uint64_t n_first, uint64_t n_last, uint32_t kinds);
int enqueue_screen(bnx_ctx* c, uint64_t n_first, uint64_t n_last, uint32_t kinds);

int enqueue(bnx_ctx* c, uint64_t n_first, uint64_t n_last, uint32_t kinds) {
    if (c->engine == 0) return enqueue_heavy(c, n_first, n_last, kinds);
    if (c->nshards == 1) return enqueue_screen(c, n_first, n_last, kinds);
    // byte screen: the shard is a contiguous slab of n (the recorded domain stays the full
    // one, so a capacity retry re-shards it identically)
    const uint64_t total = n_last - n_first + 1;
    const uint64_t lo = n_first + total * c->shard / c->nshards;
    const uint64_t hi = n_first + total * (c->shard + 1) / c->nshards;  // exclusive
    TRY(lo < hi ? enqueue_screen(c, lo, hi - 1, kinds) : empty_search(c, n_first, n_last, kinds));
    c->q_first = n_first;
    c->q_last = n_last;
    return BNX_OK;
}

int enqueue_screen(bnx_ctx* c, uint64_t n_first, uint64_t n_last, uint32_t kinds) {
    Tables& t = c->screen_tab;
    TRY(ensure_work(c));
    const ScreenVariant& sv = screen_variant(c->screen_v);
    const uint64_t x_begin = n_first / sv.tile * sv.tile;
    const uint64_t ntiles = (n_last - x_begin) / sv.tile + 1;
    CK(cudaMemsetAsync(c->ctr_p, 0, sizeof(unsigned long long) * CTR_N, c->stream));
    CK(cudaMemsetAsync(c->sflags_p, 0, sizeof(int) * 4, c->stream));
    ScreenArgs sa{x_begin, ntiles, n_first, n_last, t.small.p, (int)t.nsmall, t.large.p, (int)t.nlarge,
                  t.items.p, t.nitems, c->surv.p, c->surv.cap, c->ctr_p, c->sflags_p, c->screen_skip};
    const int sgrid = (int)std::min<uint64_t>(ntiles, (uint64_t)c->num_sms * c->screen_blocks_per_sm);
    if (c->timing) CK(cudaEventRecord(c->ev[0], c->stream));
    sv.launch(sa, sgrid, c->stream);
    if (c->timing) CK(cudaEventRecord(c->ev[1], c->stream));
    TailArgs ta{c->surv.p, c->surv.cap, nullptr, 0, c->heavy.p, c->heavy.cap, t.pdiv.p, t.npdiv, kinds, c->pairs_p, c->pairs_cap,
                c->ctr_p};
    launch_tail(ta, grid_for(c), c->stream);
    CK(cudaGetLastError());
    if (c->timing) CK(cudaEventRecord(c->ev[2], c->stream));
    TRY(read_back(c));
    c->q_valid = true;
    c->q_publish = false;
    c->q_first = n_first;
    c->q_last = n_last;
    c->q_kinds = kinds;
    c->stats = bnx_stats_t{};
    c->stats.integers = n_last - n_first + 1;
    c->stats.kernel_launches = 3;
    return BNX_OK;
}

// A search with nothing to do (an empty shard): zeroed counters, no launches.
int empty_search(bnx_ctx* c, uint64_t n_first, uint64_t n_last, uint32_t kinds) {
    TRY(ensure_work(c));
    CK(cudaMemsetAsync(c->ctr_p, 0, sizeof(unsigned long long) * CTR_N, c->stream));
    CK(cudaMemsetAsync(c->sflags_p, 0, sizeof(int) * 4, c->stream));
    TRY(read_back(c));
    c->q_publish = false;
    if (c->timing) {
        CK(cudaEventRecord(c->ev[0], c->stream));
        CK(cudaEventRecord(c->ev[1], c->stream));
        CK(cudaEventRecord(c->ev[2], c->stream));
    }
    c->q_valid = true;
    c->q_first = n_first;
    c->q_last = n_last;
    c->q_kinds = kinds;
    c->stats = bnx_stats_t{};
    return BNX_OK;
}

int prepare(bnx_ctx* c, uint64_t max_x, const uint64_t* primes, size_t np, uint64_t plimit) {
    // heavy generator: 64-bit arithmetic with margin and its shared-memory prime tables up to
    // S = 2^48; the byte screen's 7-bit surplus weights up to S < 2^42
    if (c->engine == 0 && max_x > (1ull << 48)) return fail(BNX_ERR_RANGE, "search bound must be at most 2^48");
    if (c->engine != 0 && max_x >= (1ull << 42))
        return fail(BNX_ERR_RANGE, "search bound must be below 2^42 with the byte-screen engine");
    const uint64_t need = isqrt_u64(max_x);
    Trace tr(c);
    TRY(ensure_primes(c, primes, np, plimit, need));
    tr.mark("prepare: primes");
    TRY(build_tables(c, c->screen_tab, max_x, 0, (uint32_t)screen_variant(c->screen_v).tile,
                     screen_variant(c->screen_v).threads / 32));
    tr.mark("prepare: progression tables");
    if (c->screen_tab.nsmall > (uint32_t)SCREEN_MAXS) return fail(BNX_ERR_CUDA, "too many small progressions");
    if (c->engine == 0) TRY(build_heavy(c, max_x));
    tr.mark("prepare: class table");
    return BNX_OK;
}

// The search's counters into the host block (a published search has not copied them).
int read_counters(bnx_ctx* c) {
    CK(cudaMemcpyAsync(c->h_io + IO_CTR, c->io.p + IO_CTR, sizeof(unsigned long long) * CTR_N, cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return BNX_OK;
}

void fill_stats(bnx_ctx* c) {
    const unsigned long long* h = c->h_sctr;
    c->stats.survivors = h[CTR_SURV];
    c->stats.candidates = h[CTR_CAND];
    c->stats.residue_checks = h[CTR_CHECKS];
    c->stats.matches = h[CTR_MATCH];
    c->stats.max_residue_checks = h[CTR_MAXCHK];
    c->stats.pairs = h[CTR_PAIRS];
    c->stats_stale = false;
}

// Sync, grow-and-retry on any capacity overflow, copy the pair list out.  A published heavy
// search (q_publish) left its first rows and its overflow flags in the host block: without
// an overflow the rows are read from there and the counters only on request (stats).
int collect(bnx_ctx* c, std::vector<bnx_pair_t>& rows) {
    if (!c->q_valid) return fail(BNX_ERR_INVALID, "no search enqueued");
    for (int attempt = 0; attempt < 8; ++attempt) {
        CK(cudaStreamSynchronize(c->stream));
        if (c->h_sflags[0]) return fail(BNX_ERR_CUDA, "screen bucket overflow");
        if (c->h_sflags[1]) return fail(BNX_ERR_CUDA, "heavy generator: k outside its table");
        const bool published = c->q_publish;
        if (published && !c->h_sflags[2] && !c->h_sflags[3]) {  // the common case: no copy at all
            uint64_t np = 0;
            while (np < c->pair_prefix && c->h_pairs[np].m) ++np;
            rows.assign(c->h_pairs, c->h_pairs + np);
            c->stats_stale = true;
        } else {
            if (published) TRY(read_counters(c));
            const unsigned long long* h = c->h_sctr;
            bool again = false;
            if (c->engine == 0) {
                if (h[CTR_SURV] > c->q1.cap) { TRY(c->q1.ensure(h[CTR_SURV] * 2)); again = true; }
                if (h[CTR_LIGHT] > c->cand.cap) { TRY(c->cand.ensure(h[CTR_LIGHT] * 2)); again = true; }
            } else if (h[CTR_SURV] > c->surv.cap) { TRY(c->surv.ensure(h[CTR_SURV] * 2)); again = true; }
            if (h[CTR_HEAVY] > c->heavy.cap) { TRY(c->heavy.ensure(h[CTR_HEAVY] * 2)); again = true; }
            if (h[CTR_PAIRS] > c->pairs_cap) { TRY(ensure_pairs(c, h[CTR_PAIRS] * 2)); again = true; }
            if (again) {
                TRY(enqueue(c, c->q_first, c->q_last, c->q_kinds));
                continue;
            }
            const uint64_t np = h[CTR_PAIRS];
            rows.resize(np);
            if (np <= c->pair_prefix) {
                if (np) std::memcpy(rows.data(), c->h_pairs, sizeof(bnx_pair_t) * np);
            } else {
                CK(cudaMemcpyAsync(rows.data(), c->pairs_p, sizeof(bnx_pair_t) * np, cudaMemcpyDeviceToHost, c->stream));
                CK(cudaStreamSynchronize(c->stream));
            }
            fill_stats(c);
        }
        if (c->timing) {
            CK(cudaEventElapsedTime(&c->screen_ms, c->ev[0], c->ev[1]));
            CK(cudaEventElapsedTime(&c->pipeline_ms, c->ev[0], c->ev[2]));
        }
        if (c->timing == 2 && c->engine == 0)
            for (int i = 0; i < 4; ++i) CK(cudaEventElapsedTime(&c->kernel_ms[i], c->kev[i], c->kev[i + 1]));
        c->q_valid = false;
        return BNX_OK;
    }
    return fail(BNX_ERR_CUDA, "capacity retries exhausted");
}

int emit(const std::vector<bnx_pair_t>& rows, bnx_pair_t* out, size_t cap, size_t* found) {
    if (found) *found = rows.size();
    if (rows.size() > cap) return fail(BNX_BUFFER_FULL, "pair buffer too small");
    if (out && !rows.empty()) std::memcpy(out, rows.data(), rows.size() * sizeof(bnx_pair_t));
    return BNX_OK;
}

int search_rows(bnx_ctx* c, uint64_t n_first, uint64_t n_last, uint32_t kinds, const uint64_t* primes, size_t np,
                uint64_t plimit, std::vector<bnx_pair_t>& rows) {
    if (n_first < 1 || n_last < n_first) return fail(BNX_ERR_INVALID, "empty search domain");
    if ((kinds & 3u) == 0) return fail(BNX_ERR_INVALID, "kinds_mask selects no kind");
    TRY(activate(c));
    TRY(prepare(c, n_last + 1, primes, np, plimit));
    Trace tr(c);
    TRY(enqueue(c, n_first, n_last, kinds & 3u));
    tr.mark("search: enqueue (+ capture)");
    TRY(collect(c, rows));
    tr.mark("search: device + collect");
    return BNX_OK;
}

}  // namespace

extern "C" {

int bnx_version(void) { return 10000; }

const char* bnx_last_error(void) { return g_err.c_str(); }

int bnx_device_count(int* count) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) n = 0;
    if (count) *count = n;
    return n > 0 ? BNX_OK : fail(BNX_ERR_CUDA, "no CUDA device");
}

int bnx_ctx_create(int device, bnx_ctx_t** out) {
    if (!out) return fail(BNX_ERR_INVALID, "null out");
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return fail(BNX_ERR_CUDA, "no CUDA device");
    if (device < 0 || device >= n) return fail(BNX_ERR_INVALID, "bad device index");
    bnx_ctx* c = new bnx_ctx();
    c->device = device;
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
    g_alloc_stream = c->stream;
    {  // the pool keeps what contexts free (DBuf); load this library's kernels once per device
        cudaMemPool_t pool;
        CK(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t keep = ~0ull;
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
        CK(preload_device(device, c->stream));
        CK(cudaHostAlloc(&c->h_io, IO_PAIRS + sizeof(bnx_pair_t) * PAIR_PREFIX, cudaHostAllocMapped));
        CK(cudaHostGetDevicePointer((void**)&c->d_h_io, c->h_io, 0));
        c->h_sctr = reinterpret_cast<unsigned long long*>(c->h_io + IO_CTR);
        c->h_sflags = reinterpret_cast<int*>(c->h_io + IO_FLAGS);
        c->h_pairs = reinterpret_cast<bnx_pair_t*>(c->h_io + IO_PAIRS);
    }
    CK(cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->join_ev, cudaEventDisableTiming));
    if (const char* env = std::getenv("BNX_GRAPHS")) c->use_graphs = std::atoi(env) != 0;
    CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    if (const char* env = std::getenv("BNX_SCREEN_SKIP")) c->screen_skip = std::atoi(env);
    if (const char* env = std::getenv("BNX_ENGINE")) c->engine = std::strcmp(env, "screen") == 0 ? 1 : 0;
    if (const char* env = std::getenv("BNX_STOP_AFTER")) c->stop_after = std::atoi(env);
    if (const char* env = std::getenv("BNX_PUBLISH")) c->publish_env = std::atoi(env);
    if (const char* env = std::getenv("BNX_TABLE_LANES")) c->table_lanes = std::atoi(env) == 4 ? 4 : 1;
    if (const char* env = std::getenv("BNX_SKIP_READBACK")) c->skip_readback = std::atoi(env) != 0;
    if (const char* env = std::getenv("BNX_TRACE")) c->trace = std::atoi(env) != 0;
    if (const char* env = std::getenv("BNX_HOST_CLASSES")) c->host_classes = std::atoi(env) != 0;
    if (const char* env = std::getenv("BNX_HEAVY_KMIN")) c->heavy_kmin = std::strtoull(env, nullptr, 10);
    if (const char* env = std::getenv("BNX_HEAVY_GRID")) c->heavy_grid = std::max(0, std::atoi(env));
    if (const char* env = std::getenv("BNX_HEAVY_RUNS")) c->heavy_runs = std::max(0, std::atoi(env));
    if (const char* env = std::getenv("BNX_HEAVY_RUN_FIRST")) c->heavy_run_first = std::max(0, std::atoi(env));
    if (const char* env = std::getenv("BNX_HEAVY_KC")) c->heavy_kc = std::max(0, std::atoi(env)) & ~7;
    if (const char* env = std::getenv("BNX_SIEVE_GRID")) c->sieve_grid = std::max(0, std::atoi(env));
    if (const char* env = std::getenv("BNX_SIEVE_THREADS")) c->sieve_threads = std::min(256, std::max(0, std::atoi(env)) & ~31);
    if (const char* env = std::getenv("BNX_PROBE_WALK")) c->probe_walk = std::atoi(env) != 0;
    if (const char* env = std::getenv("BNX_LOCAL_SCAN")) c->local_scan = std::atoi(env) != 0;
    if (const char* env = std::getenv("BNX_EXACT_WARP")) c->exact_warp = std::atoi(env) != 0;
    if (const char* env = std::getenv("BNX_PAIR_PREFIX"))
        c->pair_prefix = std::min<uint64_t>(PAIR_PREFIX, (uint64_t)std::max(0, std::atoi(env)));
    if (const char* env = std::getenv("BNX_TAIL_HEAVY")) c->tail_heavy = std::strtoull(env, nullptr, 10);
    if (const char* env = std::getenv("BNX_SCREEN_VARIANT")) {
        const int v = std::atoi(env);
        if (v >= 0 && v < screen_variant_count()) c->screen_v = v;
    }
    {
        const ScreenVariant& sv = screen_variant(c->screen_v);
        CK(cudaFuncSetAttribute(sv.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sv.smem));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->screen_blocks_per_sm, sv.fn, sv.threads, sv.smem));
    }
    if (const char* env = std::getenv("BNX_SIEVE_VARIANT")) {
        const int v = std::atoi(env);
        if (v >= 0 && v < sieve_variant_count()) c->sieve_v = v;
    }
    {
        const SieveVariant& sv = sieve_variant(c->sieve_v);
        CK(cudaFuncSetAttribute(sv.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sv.smem));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->sieve_blocks_per_sm, sv.fn, sv.threads, sv.smem));
    }
    c->screen_blocks_per_sm = std::max(1, c->screen_blocks_per_sm);
    if (const char* env = std::getenv("BNX_SIEVE_NARROW")) {
        const int v = std::atoi(env);
        c->sieve_nv = (v >= 0 && v < sieve_narrow_count()) ? v : -1;
    }
    if (c->sieve_nv >= 0) {
        const SieveVariant& sv = sieve_narrow(c->sieve_nv);
        CK(cudaFuncSetAttribute(sv.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sv.smem));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->sieve_narrow_blocks_per_sm, sv.fn, sv.threads, sv.smem));
    }
    if (const char* env = std::getenv("BNX_SIEVE_GBUCKETS")) c->sieve_gbuckets = std::atoi(env) != 0;
    if (const char* env = std::getenv("BNX_SIEVE_GCAP")) c->sieve_gcap = (uint32_t)std::max(0, std::atoi(env));
    c->sieve_blocks_per_sm = std::max(1, c->sieve_blocks_per_sm);
    c->sieve_narrow_blocks_per_sm = std::max(1, c->sieve_narrow_blocks_per_sm);
    *out = c;
    return BNX_OK;
}

int bnx_ctx_destroy(bnx_ctx_t* c) {
    if (!c) return BNX_OK;
    cudaSetDevice(c->device);
    g_alloc_stream = c->stream;
    if (c->stream) cudaStreamSynchronize(c->stream);
    c->primes.release();
    c->stage64.release();
    c->screen_tab.release();
    c->sieve_tab.release();
    c->td_tab.release();
    c->heavy_tab.release();
    c->q1.release();
    c->cand.release();
    c->surv.release();
    c->heavy.release();
    c->io.release();
    c->flags.release();
    c->t_nsmall.release();
    c->t_nlarge.release();
    c->t_npdiv.release();
    c->t_over.release();
    c->t_split.release();
    c->sieve_out.release();
    c->sieve_gbuck.release();
    c->sieve_gcnt.release();
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : c->kev)
        if (e) cudaEventDestroy(e);
    if (c->stream) cudaStreamSynchronize(c->stream);  // (the stream-ordered frees above)
    if (c->h_flags) cudaFreeHost(c->h_flags);
    if (c->h_io) cudaFreeHost(c->h_io);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    g_alloc_stream = nullptr;
    for (auto& g : c->graphs) g.destroy();
    c->graphs.clear();
    if (c->aux) cudaStreamDestroy(c->aux);
    if (c->fork_ev) cudaEventDestroy(c->fork_ev);
    if (c->join_ev) cudaEventDestroy(c->join_ev);
    delete c;
    return BNX_OK;
}

int bnx_ctx_set_stream(bnx_ctx_t* c, void* stream) {
    if (!c) return fail(BNX_ERR_INVALID, "null context");
    TRY(activate(c));
    cudaStreamSynchronize(c->stream);  // (buffers allocated on it are freed on the new one later)
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    if (stream) {
        c->stream = (cudaStream_t)stream;
        c->own_stream = false;
    } else {
        CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
    }
    g_alloc_stream = c->stream;
    return BNX_OK;
}

int bnx_ctx_stats(const bnx_ctx_t* cc, bnx_stats_t* out) {
    if (!cc || !out) return fail(BNX_ERR_INVALID, "null argument");
    bnx_ctx* c = const_cast<bnx_ctx*>(cc);  // (the counters of a published search are read lazily)
    if (c->stats_stale) {
        TRY(activate(c));
        TRY(read_counters(c));
        fill_stats(c);
    }
    *out = c->stats;
    return BNX_OK;
}

int bnx_ctx_set_timing(bnx_ctx_t* c, int enabled) {
    if (!c) return fail(BNX_ERR_INVALID, "null context");
    TRY(activate(c));
    if (enabled < 0 || enabled > 2) return fail(BNX_ERR_INVALID, "timing mode must be 0, 1 or 2");
    if (enabled)
        for (auto& e : c->ev)
            if (!e) CK(cudaEventCreate(&e));
    if (enabled == 2)
        for (auto& e : c->kev)
            if (!e) CK(cudaEventCreate(&e));
    c->timing = enabled;
    return BNX_OK;
}

int bnx_ctx_class_table(bnx_ctx_t* c, uint64_t max_x, uint64_t* b_out, uint64_t* m_out, size_t cap, size_t* count) {
    if (!c || !count) return fail(BNX_ERR_INVALID, "null argument");
    if (c->engine != 0) return fail(BNX_ERR_INVALID, "the class table belongs to the heavy engine");
    TRY(activate(c));
    TRY(prepare(c, max_x, nullptr, 0, 0));
    const HeavyTab& h = c->heavy_tab;
    *count = h.nent;
    if (h.nent > cap) return fail(BNX_BUFFER_FULL, "class buffer too small");
    std::vector<BnxHeavyEnt> e(h.nent);
    CK(cudaMemcpyAsync(e.data(), h.ent.p, sizeof(BnxHeavyEnt) * h.nent, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (size_t i = 0; i < e.size(); ++i) {
        if (b_out) b_out[i] = e[i].b;
        if (m_out) m_out[i] = e[i].m | (uint64_t)e[i].r << 40;  // (m < 2^24 up to 2^48)
    }
    return BNX_OK;
}

int bnx_ctx_kernel_timing(const bnx_ctx_t* c, float* ms, int n) {
    if (!c || !ms) return fail(BNX_ERR_INVALID, "null argument");
    for (int i = 0; i < n && i < 4; ++i) ms[i] = c->kernel_ms[i];
    return BNX_OK;
}

int bnx_ctx_set_engine(bnx_ctx_t* c, int engine) {
    if (!c) return fail(BNX_ERR_INVALID, "null context");
    if (engine != BNX_ENGINE_HEAVY && engine != BNX_ENGINE_SCREEN) return fail(BNX_ERR_INVALID, "unknown engine");
    if (c->q_valid) return fail(BNX_ERR_INVALID, "a search is enqueued");
    c->engine = engine;
    return BNX_OK;
}

int bnx_ctx_engine(const bnx_ctx_t* c) { return c ? c->engine : -1; }

int bnx_ctx_set_shard(bnx_ctx_t* c, uint32_t shard, uint32_t nshards) {
    if (!c) return fail(BNX_ERR_INVALID, "null context");
    if (nshards < 1 || shard >= nshards || nshards > (1u << 20)) return fail(BNX_ERR_INVALID, "bad shard");
    if (c->q_valid) return fail(BNX_ERR_INVALID, "a search is enqueued");
    c->shard = shard;
    c->nshards = nshards;
    return BNX_OK;
}

int bnx_ctx_timing(const bnx_ctx_t* c, float* screen_ms, float* pipeline_ms) {
    if (!c) return fail(BNX_ERR_INVALID, "null context");
    if (screen_ms) *screen_ms = c->screen_ms;
    if (pipeline_ms) *pipeline_ms = c->pipeline_ms;
    return BNX_OK;
}

int bnx_primes_up_to(bnx_ctx_t* c, uint64_t limit, uint64_t* out, size_t cap, size_t* count) {
    if (!c) return fail(BNX_ERR_INVALID, "null context");
    if (count) *count = 0;
    if (limit < 2) return BNX_OK;
    TRY(activate(c));
    TRY(gen_primes(c, limit));
    const size_t n = c->h_primes.size();
    if (count) *count = n;
    if (n > cap) return fail(BNX_BUFFER_FULL, "prime buffer too small");
    for (size_t i = 0; i < n; ++i) out[i] = c->h_primes[i];
    return BNX_OK;
}

static int sieve_common(bnx_ctx* c, uint64_t start, uint64_t length, const uint64_t* primes, size_t np,
                        uint64_t plimit, int fast, uint64_t* out_host, uint64_t* out_dev) {
    if (start < 1) return fail(BNX_ERR_INVALID, "interval must start at 1 or above");
    if (length < 1) return fail(BNX_ERR_INVALID, "interval length must be >= 1");
    if (length - 1 > ~0ull - start) return fail(BNX_ERR_INVALID, "interval endpoint exceeds 64 bits");
    TRY(activate(c));
    const uint64_t end = start + (length - 1);
    const uint64_t need = isqrt_u64(end);
    TRY(ensure_primes(c, primes, np, plimit, need));
    // every slot value is at most the window's end: 32-bit slots below 2^32
    const bool narrow = c->sieve_nv >= 0 && end < (1ull << 32);
    const SieveVariant& sv = narrow ? sieve_narrow(c->sieve_nv) : sieve_variant(c->sieve_v);
    const int bps = narrow ? c->sieve_narrow_blocks_per_sm : c->sieve_blocks_per_sm;
    // global buckets for the huge progressions above 2^32 (below, at most ~6,500 large
    // progressions: the per-segment scan is cheaper than the extra pass)
    for (bool gbuckets = c->sieve_gbuckets && !narrow;; gbuckets = false) {
    TRY(build_tables(c, c->sieve_tab, end, fast ? 0 : 1, (uint32_t)sv.tile, sv.threads / 32));
    if (c->sieve_tab.nsmall > (uint32_t)SIEVE_MAXS) return fail(BNX_ERR_CUDA, "too many small progressions");
    TRY(c->flags.ensure(4));
    if (!c->h_flags) CK(cudaMallocHost(&c->h_flags, sizeof(int) * 4));
    CK(cudaMemsetAsync(c->flags.p, 0, sizeof(int) * 4, c->stream));
    const uint64_t piece = out_dev ? std::min<uint64_t>(length, 1ull << 32) : std::min<uint64_t>(length, 1ull << 27);
    if (!out_dev) TRY(c->sieve_out.ensure(piece));
    const uint64_t SEG = (uint64_t)sv.tile * sv.nt;
    // global buckets for the large progressions: SEG / 128 entries per segment, ~2.8x the
    // expected hits (the sum over q >= the tile of SEG / q is below SEG / 350); a full one
    // re-runs the call with the per-segment scan
    const uint32_t gcap = c->sieve_gcap ? c->sieve_gcap : (uint32_t)(SEG / 128);
    const uint64_t nseg_max = (piece + SEG - 1) / SEG;
    if (gbuckets) {
        TRY(c->sieve_gcnt.ensure(nseg_max));
        TRY(c->sieve_gbuck.ensure(nseg_max * gcap));
        Tables& t = c->sieve_tab;
        if (!t.split && t.nlarge) {  // medium progressions to the front, huge ones to the back (once per table)
            struct Scratch {  // (released on every path out)
                DBuf<BnxProg> b;
                ~Scratch() { b.release(); }
            } tmp;
            TRY(tmp.b.ensure(t.nlarge));
            TRY(c->t_split.ensure(2));
            CK(cudaMemsetAsync(c->t_split.p, 0, 2 * sizeof(unsigned long long), c->stream));
            launch_split_large(t.large.p, t.nlarge, tmp.b.p, c->t_split.p, c->stream);
            CK(cudaGetLastError());
            CK(cudaMemcpyAsync(t.large.p, tmp.b.p, sizeof(BnxProg) * t.nlarge, cudaMemcpyDeviceToDevice, c->stream));
            unsigned long long nm = 0;
            CK(cudaMemcpyAsync(&nm, c->t_split.p, sizeof(nm), cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
            t.nmedium = nm;
            t.split = true;
        } else if (!t.nlarge) {
            t.split = true;
        }
    }
    for (uint64_t off = 0; off < length; off += piece) {
        const uint64_t len = std::min<uint64_t>(piece, length - off);
        uint64_t* dst = out_dev ? out_dev + off : c->sieve_out.p;
        SieveArgs sa{start + off, len, c->sieve_tab.small.p, (int)c->sieve_tab.nsmall, c->sieve_tab.large.p,
                     c->sieve_tab.nlarge, c->sieve_tab.items.p, c->sieve_tab.nitems, fast, dst, c->flags.p,
                     nullptr, nullptr, 0, 0};
        const uint64_t nseg = (len + SEG - 1) / SEG;
        if (gbuckets && sa.nlarge) {
            CK(cudaMemsetAsync(c->sieve_gcnt.p, 0, sizeof(uint32_t) * nseg, c->stream));
            sa.gbuck = c->sieve_gbuck.p;
            sa.gcnt = c->sieve_gcnt.p;
            sa.gcap = gcap;
            sa.nmedium = c->sieve_tab.nmedium;
            launch_sieve_buckets(sa, SEG, c->sieve_gbuck.p, c->sieve_gcnt.p, c->stream);
        }
        const int grid = (int)std::min<uint64_t>(nseg, (uint64_t)c->num_sms * bps);
        sv.launch(sa, grid, c->stream);
        CK(cudaGetLastError());
        if (!out_dev) CK(cudaMemcpyAsync(out_host + off, dst, sizeof(uint64_t) * len, cudaMemcpyDeviceToHost, c->stream));
    }
    CK(cudaMemcpyAsync(c->h_flags, c->flags.p, sizeof(int) * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (c->h_flags[0]) return fail(BNX_ERR_CUDA, "sieve bucket overflow");
    if (gbuckets && c->h_flags[3]) {  // a full global bucket: again with the per-segment scan
        CK(cudaMemsetAsync(c->flags.p, 0, sizeof(int) * 4, c->stream));
        continue;
    }
    return BNX_OK;
    }
}

int bnx_sieve_radicals(bnx_ctx_t* c, uint64_t start, uint64_t length, const uint64_t* primes, size_t nprimes,
                       uint64_t primes_limit, int ctz_fast_path, uint64_t* out) {
    if (!c || !out) return fail(BNX_ERR_INVALID, "null argument");
    return sieve_common(c, start, length, primes, nprimes, primes_limit, ctz_fast_path, out, nullptr);
}

int bnx_sieve_radicals_dev(bnx_ctx_t* c, uint64_t start, uint64_t length, int ctz_fast_path, uint64_t* out_dev) {
    if (!c || !out_dev) return fail(BNX_ERR_INVALID, "null argument");
    if (((uintptr_t)out_dev) & 7) return fail(BNX_ERR_INVALID, "out_dev must be 8-byte aligned");
    return sieve_common(c, start, length, nullptr, 0, 0, ctz_fast_path, nullptr, out_dev);
}

int bnx_radicals_trial_division(bnx_ctx_t* c, uint64_t start, uint64_t length, uint64_t* out) {
    if (!c || !out) return fail(BNX_ERR_INVALID, "null argument");
    if (start < 1) return fail(BNX_ERR_INVALID, "interval must start at 1 or above");
    if (length < 1) return fail(BNX_ERR_INVALID, "interval length must be >= 1");
    if (length - 1 > ~0ull - start) return fail(BNX_ERR_INVALID, "interval endpoint exceeds 64 bits");
    TRY(activate(c));
    const uint64_t end = start + (length - 1);
    TRY(ensure_primes(c, nullptr, 0, 0, isqrt_u64(end)));
    TRY(build_tables(c, c->td_tab, end, 0, SIEVE_TILE, SIEVE_THREADS / 32));
    const uint64_t piece = std::min<uint64_t>(length, 1ull << 26);
    TRY(c->sieve_out.ensure(piece));
    for (uint64_t off = 0; off < length; off += piece) {
        const uint64_t len = std::min<uint64_t>(piece, length - off);
        launch_trial_division(start + off, len, c->td_tab.pdiv.p, c->td_tab.npdiv, c->sieve_out.p, c->num_sms * 8,
                              c->stream);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(out + off, c->sieve_out.p, sizeof(uint64_t) * len, cudaMemcpyDeviceToHost, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    return BNX_OK;
}

int bnx_brute_force(bnx_ctx_t* c, uint64_t limit, bnx_pair_t* out, size_t cap, size_t* found) {
    if (!c) return fail(BNX_ERR_INVALID, "null context");
    if (limit < 3) return fail(BNX_ERR_INVALID, "limit must be >= 3");
    if (limit > (1ull << 22)) return fail(BNX_ERR_RANGE, "brute force is limited to 2^22 (quadratic)");
    TRY(activate(c));
    TRY(ensure_primes(c, nullptr, 0, 0, isqrt_u64(limit)));
    TRY(build_tables(c, c->td_tab, limit, 0, SIEVE_TILE, SIEVE_THREADS / 32));
    DBuf<uint64_t> rads;
    DBuf<bnx_pair_t> rows;
    DBuf<unsigned long long> cnt;
    TRY(rads.ensure(limit));
    TRY(cnt.ensure(1));
    launch_trial_division(1, limit, c->td_tab.pdiv.p, c->td_tab.npdiv, rads.p, c->num_sms * 8, c->stream);
    uint64_t cap_dev = 4096;
    unsigned long long n = 0;
    for (;;) {
        TRY(rows.ensure(cap_dev));
        CK(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), c->stream));
        launch_brute_force(rads.p, limit, rows.p, cap_dev, cnt.p, c->stream);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(&n, cnt.p, sizeof(n), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (n <= cap_dev) break;
        cap_dev = n;
    }
    std::vector<bnx_pair_t> v(n);
    if (n) CK(cudaMemcpy(v.data(), rows.p, sizeof(bnx_pair_t) * n, cudaMemcpyDeviceToHost));
    rads.release();
    rows.release();
    cnt.release();
    std::sort(v.begin(), v.end(), [](const bnx_pair_t& a, const bnx_pair_t& b) {
        return a.m != b.m ? a.m < b.m : a.n < b.n;
    });
    return emit(v, out, cap, found);
}

int bnx_prepare(bnx_ctx_t* c, uint64_t max_x, const uint64_t* primes, size_t nprimes, uint64_t primes_limit) {
    if (!c) return fail(BNX_ERR_INVALID, "null context");
    TRY(activate(c));
    return prepare(c, max_x, primes, nprimes, primes_limit);
}

int bnx_search_enqueue(bnx_ctx_t* c, uint64_t n_first, uint64_t n_last, uint32_t kinds_mask) {
    if (!c) return fail(BNX_ERR_INVALID, "null context");
    if (n_first < 1 || n_last < n_first) return fail(BNX_ERR_INVALID, "empty search domain");
    c->rows_pending = false;  // a new search drops rows nobody collected
    c->pending.clear();
    if (c->q_valid) {  // an uncollected search may still write the host block the next one reuses
        TRY(activate(c));
        CK(cudaStreamSynchronize(c->stream));
    }
    if (c->screen_tab.gen != c->gen || c->screen_tab.max_x < n_last + 1)  // prepared for a large enough bound
        return fail(BNX_ERR_INVALID, "bnx_prepare must cover n_last + 1 first");
    TRY(activate(c));
    return enqueue(c, n_first, n_last, kinds_mask & 3u);
}

int bnx_search_collect(bnx_ctx_t* c, bnx_pair_t* out, size_t cap, size_t* found) {
    if (!c) return fail(BNX_ERR_INVALID, "null context");
    TRY(activate(c));
    if (c->rows_pending) {  // a retry after BNX_BUFFER_FULL
        const int r = emit(c->pending, out, cap, found);
        if (r == BNX_OK) {
            c->rows_pending = false;
            c->pending.clear();
        }
        return r;
    }
    std::vector<bnx_pair_t> rows;
    TRY(collect(c, rows));
    std::sort(rows.begin(), rows.end(), [](const bnx_pair_t& a, const bnx_pair_t& b) {
        return a.n != b.n ? a.n < b.n : a.m < b.m;
    });
    const int r = emit(rows, out, cap, found);
    if (r == BNX_BUFFER_FULL) {
        c->pending.swap(rows);
        c->rows_pending = true;
    }
    return r;
}

int bnx_search(bnx_ctx_t* c, uint64_t limit, uint32_t kinds_mask, const uint64_t* primes, size_t nprimes,
               uint64_t primes_limit, bnx_pair_t* out, size_t cap, size_t* found) {
    if (!c) return fail(BNX_ERR_INVALID, "null context");
    if (limit < 3) return fail(BNX_ERR_INVALID, "limit must be >= 3");
    std::vector<bnx_pair_t> rows;
    TRY(search_rows(c, 1, limit - 1, kinds_mask, primes, nprimes, primes_limit, rows));
    std::sort(rows.begin(), rows.end(), [](const bnx_pair_t& a, const bnx_pair_t& b) {
        return a.m != b.m ? a.m < b.m : a.n < b.n;
    });
    return emit(rows, out, cap, found);
}

// One host thread drives several GPUs: context i (device devices[i], a process-wide pool) runs
// shard i of ndev of the search; all shards are enqueued before any is collected.
static std::mutex g_multi_mu;
static std::vector<bnx_ctx*> g_multi;

int bnx_search_multi(const int* devices, int ndev, uint64_t limit, uint32_t kinds_mask, const uint64_t* primes,
                     size_t nprimes, uint64_t primes_limit, bnx_pair_t* out, size_t cap, size_t* found) {
    if (!devices || ndev < 1 || ndev > 1024) return fail(BNX_ERR_INVALID, "bad device list");
    if (limit < 3) return fail(BNX_ERR_INVALID, "limit must be >= 3");
    if ((kinds_mask & 3u) == 0) return fail(BNX_ERR_INVALID, "kinds_mask selects no kind");
    std::lock_guard<std::mutex> lock(g_multi_mu);
    if (g_multi.size() < (size_t)ndev) g_multi.resize(ndev, nullptr);
    for (int i = 0; i < ndev; ++i) {
        if (g_multi[i] && g_multi[i]->device != devices[i]) {
            bnx_ctx_destroy(g_multi[i]);
            g_multi[i] = nullptr;
        }
        if (!g_multi[i]) TRY(bnx_ctx_create(devices[i], &g_multi[i]));
        g_multi[i]->shard = (uint32_t)i;
        g_multi[i]->nshards = (uint32_t)ndev;
    }
    {  // the contexts' tables are built concurrently, one host thread per context
        std::vector<int> rc(ndev, BNX_OK);
        std::vector<std::string> err(ndev);
        std::vector<std::thread> th;
        for (int i = 0; i < ndev; ++i)
            th.emplace_back([&, i] {
                bnx_ctx* c = g_multi[i];
                rc[i] = activate(c);
                if (rc[i] == BNX_OK) rc[i] = prepare(c, limit, primes, nprimes, primes_limit);
                if (rc[i] != BNX_OK) err[i] = g_err;
            });
        for (auto& t : th) t.join();
        for (int i = 0; i < ndev; ++i)
            if (rc[i] != BNX_OK) return fail(rc[i], err[i]);
    }
    for (int i = 0; i < ndev; ++i) {
        TRY(activate(g_multi[i]));
        TRY(enqueue(g_multi[i], 1, limit - 1, kinds_mask & 3u));
    }
    std::vector<bnx_pair_t> rows;
    for (int i = 0; i < ndev; ++i) {
        std::vector<bnx_pair_t> part;
        TRY(activate(g_multi[i]));
        TRY(collect(g_multi[i], part));
        rows.insert(rows.end(), part.begin(), part.end());
    }
    std::sort(rows.begin(), rows.end(), [](const bnx_pair_t& a, const bnx_pair_t& b) {
        return a.m != b.m ? a.m < b.m : a.n < b.n;
    });
    return emit(rows, out, cap, found);
}

int bnx_search_domain(bnx_ctx_t* c, uint64_t n_first, uint64_t n_last, uint32_t kinds_mask, const uint64_t* primes,
                      size_t nprimes, uint64_t primes_limit, bnx_pair_t* out, size_t cap, size_t* found) {
    if (!c) return fail(BNX_ERR_INVALID, "null context");
    std::vector<bnx_pair_t> rows;
    TRY(search_rows(c, n_first, n_last, kinds_mask, primes, nprimes, primes_limit, rows));
    std::sort(rows.begin(), rows.end(), [](const bnx_pair_t& a, const bnx_pair_t& b) {
        return a.n != b.n ? a.n < b.n : a.m < b.m;
    });
    return emit(rows, out, cap, found);
}

// ---- Algorithm 3 ----------------------------------------------------------------------
static int table_run(bnx_table* tb, bool insert, uint64_t a0, uint64_t count, uint64_t n_limit,
                     std::vector<bnx_pair_t>& rows, uint64_t* inserted) {
    bnx_ctx* c = tb->ctx;
    uint64_t cap = std::max<uint64_t>(tb->rows.cap, 1024);
    for (;;) {
        TRY(tb->rows.ensure(cap));
        TRY(tb->cnt.ensure(2));
        TRY(tb->status.ensure(1));
        CK(cudaMemsetAsync(tb->cnt.p, 0, 2 * sizeof(unsigned long long), c->stream));
        CK(cudaMemsetAsync(tb->status.p, 0, sizeof(int), c->stream));
        if (insert) CK(cudaMemsetAsync(tb->slots.p, 0, sizeof(uint64_t) * tb->size, c->stream));
        TableArgs ta{};
        ta.domain_start = tb->domain_start;
        ta.rad_of = tb->rad_of.p;
        ta.rad_next = tb->rad_next.p;
        ta.count_n = insert ? count : tb->count;
        ta.n_limit = n_limit;
        ta.probe_start = a0;
        ta.probe_of = tb->probe_of.p;
        ta.probe_next = tb->probe_next.p;
        ta.count_m = insert ? 0 : count;
        ta.slots = tb->slots.p;
        ta.mask = tb->size - 1;
        ta.out = tb->rows.p;
        ta.cap = tb->rows.cap;
        ta.count = tb->cnt.p;
        ta.inserted = tb->cnt.p + 1;
        ta.status = tb->status.p;
        const int grid = c->num_sms * 8;
        if (insert) launch_table_insert(ta, grid, c->stream, c->table_lanes);
        else launch_table_probe(ta, grid, c->stream, c->table_lanes);
        CK(cudaGetLastError());
        unsigned long long h[2] = {0, 0};
        int st = 0;
        CK(cudaMemcpyAsync(h, tb->cnt.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(&st, tb->status.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (st == BNX_TABLE_FULL) return fail(BNX_TABLE_FULL, "no empty slot in a table of " + std::to_string(tb->size));
        if (h[0] > tb->rows.cap) { cap = h[0] * 2; continue; }
        const size_t base = rows.size();
        rows.resize(base + h[0]);
        if (h[0]) CK(cudaMemcpy(rows.data() + base, tb->rows.p, sizeof(bnx_pair_t) * h[0], cudaMemcpyDeviceToHost));
        if (inserted) *inserted = h[1];
        return BNX_OK;
    }
}

static void sort_nm(std::vector<bnx_pair_t>& rows) {
    std::sort(rows.begin(), rows.end(), [](const bnx_pair_t& a, const bnx_pair_t& b) {
        return a.n != b.n ? a.n < b.n : a.m < b.m;
    });
}

int bnx_table_create(bnx_ctx_t* c, uint64_t table_size, bnx_table_t** out) {
    if (!c || !out) return fail(BNX_ERR_INVALID, "null argument");
    if (table_size < 1 || (table_size & (table_size - 1))) return fail(BNX_ERR_INVALID, "table size must be a power of two");
    if (table_size > (1ull << 32)) return fail(BNX_ERR_INVALID, "table too large for 32-bit home slots");
    TRY(activate(c));
    bnx_table* tb = new bnx_table();
    tb->ctx = c;
    tb->size = table_size;
    int r = tb->slots.ensure(table_size);
    if (r != BNX_OK) { delete tb; return r; }
    CK(cudaMemsetAsync(tb->slots.p, 0, sizeof(uint64_t) * table_size, c->stream));
    *out = tb;
    return BNX_OK;
}

int bnx_table_destroy(bnx_table_t* tb) {
    if (!tb) return BNX_OK;
    cudaSetDevice(tb->ctx->device);
    g_alloc_stream = tb->ctx->stream;
    cudaStreamSynchronize(tb->ctx->stream);
    tb->slots.release(); tb->rad_of.release(); tb->rad_next.release();
    tb->probe_of.release(); tb->probe_next.release(); tb->rows.release(); tb->cnt.release(); tb->status.release();
    delete tb;
    return BNX_OK;
}

int bnx_table_insert_all(bnx_table_t* tb, uint64_t domain_start, const uint64_t* rad_of, const uint64_t* rad_next,
                         size_t count, uint64_t n_limit, bnx_pair_t* out, size_t cap, size_t* found, uint64_t* inserted) {
    if (!tb) return fail(BNX_ERR_INVALID, "null table");
    if (count > 0xFFFFFFFEull) return fail(BNX_ERR_INVALID, "domain too large for 32-bit slot offsets");
    TRY(activate(tb->ctx));
    TRY(tb->rad_of.ensure(count));
    TRY(tb->rad_next.ensure(count));
    if (count) {
        CK(cudaMemcpyAsync(tb->rad_of.p, rad_of, sizeof(uint64_t) * count, cudaMemcpyHostToDevice, tb->ctx->stream));
        CK(cudaMemcpyAsync(tb->rad_next.p, rad_next, sizeof(uint64_t) * count, cudaMemcpyHostToDevice, tb->ctx->stream));
    }
    tb->domain_start = domain_start;
    tb->count = count;
    std::vector<bnx_pair_t> rows;
    TRY(table_run(tb, true, 0, count, n_limit, rows, inserted));
    sort_nm(rows);
    return emit(rows, out, cap, found);
}

int bnx_table_probe_all(bnx_table_t* tb, uint64_t probe_start, const uint64_t* rad_of, const uint64_t* rad_next,
                        size_t count, bnx_pair_t* out, size_t cap, size_t* found) {
    if (!tb) return fail(BNX_ERR_INVALID, "null table");
    TRY(activate(tb->ctx));
    TRY(tb->probe_of.ensure(count));
    TRY(tb->probe_next.ensure(count));
    if (count) {
        CK(cudaMemcpyAsync(tb->probe_of.p, rad_of, sizeof(uint64_t) * count, cudaMemcpyHostToDevice, tb->ctx->stream));
        CK(cudaMemcpyAsync(tb->probe_next.p, rad_next, sizeof(uint64_t) * count, cudaMemcpyHostToDevice, tb->ctx->stream));
    }
    std::vector<bnx_pair_t> rows;
    TRY(table_run(tb, false, probe_start, count, 0, rows, nullptr));
    std::sort(rows.begin(), rows.end(), [](const bnx_pair_t& a, const bnx_pair_t& b) {
        return a.m != b.m ? a.m < b.m : a.n < b.n;
    });
    return emit(rows, out, cap, found);
}

int bnx_table_slots(const bnx_table_t* tb, uint64_t* out, size_t cap) {
    if (!tb || !out) return fail(BNX_ERR_INVALID, "null argument");
    if (cap < tb->size) return fail(BNX_BUFFER_FULL, "slot buffer too small");
    CK(cudaSetDevice(tb->ctx->device));
    CK(cudaStreamSynchronize(tb->ctx->stream));
    CK(cudaMemcpy(out, tb->slots.p, sizeof(uint64_t) * tb->size, cudaMemcpyDeviceToHost));
    return BNX_OK;
}

int bnx_table_search_chunk(bnx_ctx_t* c, uint64_t index, uint64_t chunk_size, uint64_t n_limit, uint64_t j_lo,
                           uint64_t j_hi, bnx_pair_t* out, size_t cap, size_t* found) {
    if (!c) return fail(BNX_ERR_INVALID, "null context");
    if (chunk_size < 3) return fail(BNX_ERR_INVALID, "chunk size must be >= 3");
    TRY(activate(c));
    const uint64_t s = chunk_size, count = s - 1;
    // the slot word keeps the home slot in 32 bits and the offset + 1 in the other 32
    // (chunked.py:136-138, :157-158): the reference refuses larger tables (ValueError)
    if (count > 0xFFFFFFFEull || count > (1ull << 30)) return fail(BNX_ERR_INVALID, "chunk too large for 32-bit slots");
    uint64_t v = 4 * count - 1, bits = 0;
    while (v) { ++bits; v >>= 1; }
    const uint64_t tsize = 1ull << bits;  // table_size_for (chunked.py:86-90)
    if (tsize > (1ull << 32)) return fail(BNX_ERR_INVALID, "table too large for 32-bit home slots");
    bnx_table tb;
    tb.ctx = c;
    tb.size = tsize;
    TRY(tb.slots.ensure(tsize));
    TRY(tb.rad_of.ensure(s));
    TRY(tb.probe_of.ensure(s));
    const uint64_t first = 1 + index * (s - 1);
    std::vector<bnx_pair_t> rows;
    TRY(sieve_common(c, first, s, nullptr, 0, 0, 1, nullptr, tb.rad_of.p));
    tb.rad_next.p = tb.rad_of.p + 1;  // views, as chunked.py:330-332
    tb.domain_start = first;
    tb.count = count;
    int r = table_run(&tb, true, 0, count, n_limit, rows, nullptr);
    for (uint64_t j = j_lo; r == BNX_OK && j < j_hi; ++j) {
        const uint64_t fj = 1 + j * (s - 1);
        r = sieve_common(c, fj, s, nullptr, 0, 0, 1, nullptr, tb.probe_of.p);
        if (r != BNX_OK) break;
        tb.probe_next.p = tb.probe_of.p + 1;
        r = table_run(&tb, false, fj, count, 0, rows, nullptr);
    }
    tb.rad_next.p = nullptr;
    tb.probe_next.p = nullptr;
    tb.slots.release(); tb.rad_of.release(); tb.probe_of.release(); tb.rows.release(); tb.cnt.release(); tb.status.release();
    TRY(r);
    sort_nm(rows);
    return emit(rows, out, cap, found);
}

uint64_t bnx_slot_of(uint64_t lo, uint64_t hi, uint64_t mask, uint64_t phi, uint64_t mul1, uint64_t mul2) {
    uint64_t x = lo ^ (hi * phi);
    x = (x ^ (x >> 30)) * mul1;
    x = (x ^ (x >> 27)) * mul2;
    x = x ^ (x >> 31);
    return x & mask;
}

}  // extern "C"
