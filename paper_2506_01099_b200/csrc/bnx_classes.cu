// bnx_classes.cu -- the heavy generator's surplus-class table, built on the device.
//
// The table lists every powerful number b <= X (b = prod p^(e_p), all e_p >= 2) with
// sigma = prod p^(e_p - 1) = m r, r = rad(b), plus per-k bits for k <=
// sqrt(X / 2).  The host used to build it by a depth-first search over the primes up to sqrt(X)
// (children of a node = the node times p^e for primes p above its largest prime, pushed in
// ascending (p, e) and popped last-first), and k_heavy_screen runs ~10% faster at 2^32 with
// the classes in that DFS order than sorted by b.  This file builds the same table in the same
// order with no host work:
//
//   k_cls_sieve    factor table for 0..L = isqrt(X): composite x -> index of its smallest
//                  prime factor (flag bit 31); segmented sieve in shared memory
//   k_cls_scatter  prime p -> its index in the device prime list
//   k_cls_count    per squarefree v <= cbrt(X): the number of u with u^2 v^3 <= X (every
//                  powerful b is u^2 v^3 with v squarefree, exactly once)
//   (cub scan)     item offsets per v
//   k_cls_build    per item (v, u): factor u and v through the table, merge to b's
//                  factorisation (p, 2 e_u + 3 e_v), write the class and its DFS sort key
//   (cub sort)     LSD radix passes over the key words -> the DFS permutation
//   k_cls_gather   the classes in DFS order
//   k_cls_kinfo    per k: which of the primes 2..127 divide k, and whether k is squarefree
//
// DFS order as a sort key: with the factorisation read as a sequence of codes c = idx(p) * 64
// + e in ascending p, the DFS visits a node before its descendants and its children in
// descending (p, e), so it is the lexicographic order of the sequences (CMAX - c_1, CMAX -
// c_2, ..., 0, 0, ...) (a prefix sorts first).  The sequence has at most D codes (D primes
// whose squares multiply to <= X); the codes are packed most significant first into 64-bit
// words and sorted least significant word first (cub's radix sort is stable).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "bnx_kernels.cuh"

namespace bnx {

namespace {

constexpr uint32_t CLS_COMPOSITE = 0x80000000u;
constexpr uint32_t CLS_UNLISTED = 0x7FFFFFFFu;  // a prime beyond the prime list (index >= 31)
constexpr int CLS_SEG = 16384;  // sieve segment (u32 entries, 64 KB of shared memory)
constexpr int CLS_MAXD = 12;    // codes per key (2^48 needs 8)
constexpr int CLS_MAXW = 6;     // key words

__global__ void __launch_bounds__(512) k_cls_sieve(uint32_t* __restrict__ tab, uint64_t L,
                                                   const uint32_t* __restrict__ primes, uint32_t np_sqrt) {
    extern __shared__ uint32_t s_min[];
    const uint64_t nseg = (L + 1 + CLS_SEG - 1) / CLS_SEG;
    for (uint64_t sg = blockIdx.x; sg < nseg; sg += gridDim.x) {
        const uint64_t lo = sg * CLS_SEG, hi = min(lo + CLS_SEG, L + 1);
        for (int i = threadIdx.x; i < CLS_SEG; i += blockDim.x) s_min[i] = 0xFFFFFFFFu;
        __syncthreads();
        for (uint32_t j = threadIdx.x; j < np_sqrt; j += blockDim.x) {
            const uint64_t p = primes[j];
            if (p * p >= hi) break;  // primes ascending: the rest start beyond the segment
            uint64_t x = max(p * p, (lo + p - 1) / p * p);
            for (; x < hi; x += p) atomicMin(&s_min[x - lo], j);
        }
        __syncthreads();
        for (uint64_t x = lo + threadIdx.x; x < hi; x += blockDim.x) {
            const uint32_t j = s_min[x - lo];
            tab[x] = j == 0xFFFFFFFFu ? CLS_UNLISTED : (j | CLS_COMPOSITE);  // primes: k_cls_scatter
        }
        __syncthreads();
    }
}

__global__ void k_cls_scatter(uint32_t* __restrict__ tab, const uint32_t* __restrict__ primes, uint64_t np) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < np; j += (uint64_t)gridDim.x * blockDim.x)
        tab[primes[j]] = (uint32_t)j;
}

// Distinct primes of x (1 <= x <= L) as (prime index, exponent), ascending; returns the count.
__device__ __forceinline__ int factor_tab(uint32_t x, const uint32_t* __restrict__ tab,
                                          const uint32_t* __restrict__ primes, uint32_t* idx, uint32_t* ex) {
    int n = 0;
    while (x > 1) {
        const uint32_t t = tab[x];
        BNX_CHECK(n < CLS_MAXD);
        if (!(t & CLS_COMPOSITE)) {  // x is prime
            idx[n] = t;
            ex[n] = 1;
            return n + 1;
        }
        const uint32_t j = t & ~CLS_COMPOSITE;
        const uint32_t p = primes[j];
        uint32_t e = 0;
        do {
            x /= p;
            ++e;
        } while (x % p == 0);
        idx[n] = j;
        ex[n] = e;
        ++n;
    }
    return n;
}

__device__ __forceinline__ uint64_t isqrt_dev(uint64_t x) {
    uint64_t r = (uint64_t)sqrt((double)x);
    while (r * r > x) --r;
    while ((r + 1) * (r + 1) <= x) ++r;
    return r;
}

__global__ void k_cls_count(uint64_t X, uint64_t V, const uint32_t* __restrict__ tab,
                            const uint32_t* __restrict__ primes, uint64_t* __restrict__ cnt) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v <= V; v += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t c = 0;
        if (v >= 1) {
            uint32_t idx[CLS_MAXD], ex[CLS_MAXD];
            const int n = factor_tab((uint32_t)v, tab, primes, idx, ex);
            bool sqf = true;
            for (int i = 0; i < n; ++i) sqf &= ex[i] == 1;
            if (sqf) c = isqrt_dev(X / (v * v * v));
        }
        cnt[v] = c;  // cnt[0] = 0
    }
}

struct ClsBuildArgs {
    uint64_t X, V, total;
    const uint64_t* offs;  // exclusive item offsets per v (V + 2 entries)
    const uint32_t* tab;
    const uint32_t* primes;
    BnxHeavyEnt* ent;      // unsorted classes
    uint64_t* keys;        // nwords arrays of `total` key words
    uint32_t* perm;        // identity permutation
    int nwords, dpw, bits;
};

__global__ void k_cls_build(ClsBuildArgs a) {
    const uint64_t cmax = (1ull << a.bits) - 1;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < a.total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t lo = 1, hi = a.V;  // v: the last v with offs[v] <= i
        while (lo < hi) {
            const uint64_t mid = (lo + hi + 1) >> 1;
            if (a.offs[mid] <= i) lo = mid; else hi = mid - 1;
        }
        const uint64_t v = lo, u = i - a.offs[v] + 1;
        uint32_t iu[CLS_MAXD], eu[CLS_MAXD], iv[CLS_MAXD], evv[CLS_MAXD];
        const int nu = factor_tab((uint32_t)u, a.tab, a.primes, iu, eu);
        const int nv = factor_tab((uint32_t)v, a.tab, a.primes, iv, evv);
        uint64_t r = 1;
        uint32_t rmask = 0, rbig = 1, rbig_min = 0;
        uint64_t words[CLS_MAXW] = {0, 0, 0, 0, 0, 0};
        int pu = 0, pv = 0, d = 0;
        while (pu < nu || pv < nv) {  // merge the two ascending factor lists
            uint32_t j, e;
            if (pv >= nv || (pu < nu && iu[pu] < iv[pv])) {
                j = iu[pu];
                e = 2 * eu[pu++];
            } else if (pu >= nu || iv[pv] < iu[pu]) {
                j = iv[pv];
                e = 3 * evv[pv++];
            } else {
                j = iu[pu];
                e = 2 * eu[pu++] + 3 * evv[pv++];
            }
            const uint32_t p = a.primes[j];
            r *= p;
            if (j < 31) {
                rmask |= 1u << j;
            } else {
                rbig *= p;
                if (!rbig_min) rbig_min = p;
            }
            const uint64_t code = cmax - ((uint64_t)j * 64 + e);
            const int w = d / a.dpw, pos = a.dpw - 1 - d % a.dpw;  // most significant first
            BNX_CHECK(w < a.nwords && w < CLS_MAXW && e < 64);
            words[w] |= code << (pos * a.bits);
            ++d;
        }
        const uint64_t b = u * u * v * v * v;
        a.ent[i] = BnxHeavyEnt{b, b / (r * r), (uint32_t)r, rmask, rbig, rbig_min};
        for (int w = 0; w < a.nwords; ++w) a.keys[(uint64_t)w * a.total + i] = words[w];
        a.perm[i] = (uint32_t)i;
    }
}

__global__ void k_cls_gather_key(const uint64_t* __restrict__ key, const uint32_t* __restrict__ perm, uint64_t n,
                                 uint64_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = key[perm[i]];
}

__global__ void k_cls_gather(const BnxHeavyEnt* __restrict__ in, const uint32_t* __restrict__ perm, uint64_t n,
                             BnxHeavyEnt* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = in[perm[i]];
}

__global__ void k_cls_kinfo(uint64_t K, const uint32_t* __restrict__ tab, const uint32_t* __restrict__ primes,
                            uint32_t* __restrict__ kinfo) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < K; k += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t bits = 0;
        if (k == 0) {
            bits = 0x80000000u;
        } else {
            uint32_t idx[CLS_MAXD], ex[CLS_MAXD];
            const int n = factor_tab((uint32_t)k, tab, primes, idx, ex);
            for (int i = 0; i < n; ++i) {
                if (idx[i] < 31) bits |= 1u << idx[i];
                if (ex[i] > 1) bits |= 0x80000000u;
            }
        }
        kinfo[k] = bits;
    }
}

unsigned grid_for(uint64_t n, unsigned threads, unsigned cap = 148 * 16) {
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + threads - 1) / threads, cap));
}

}  // namespace

ClassPlan class_plan(uint64_t X, uint64_t nprimes_root) {
    ClassPlan pl{};
    pl.X = X;
    uint64_t root = (uint64_t)sqrt((double)X);
    while (root * root > X) --root;
    while ((root + 1) * (root + 1) <= X) ++root;
    pl.L = root;
    uint64_t V = (uint64_t)cbrt((double)X);
    while (V > 0 && V * V * V > X) --V;
    while ((V + 1) * (V + 1) * (V + 1) <= X) ++V;
    pl.V = V;
    // D: the most distinct primes of a powerful b <= X (their squares' product <= X)
    static const uint32_t small[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    uint64_t prod = 1;
    int D = 0;
    while (D < CLS_MAXD && prod * small[D] <= root) prod *= small[D++];
    pl.D = std::max(D, 1);
    const uint64_t maxcode = std::max<uint64_t>(nprimes_root, 1) * 64 + 64;
    int bits = 1;
    while ((1ull << bits) <= maxcode + 1) ++bits;
    pl.bits = bits;
    pl.dpw = std::max(1, 64 / bits);
    pl.nwords = (pl.D + pl.dpw - 1) / pl.dpw;
    pl.ok = pl.nwords <= CLS_MAXW;
    return pl;
}

size_t class_scratch_bytes(const ClassPlan& pl, uint64_t total) {
    size_t b1 = 0, b2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, b1, (const uint64_t*)nullptr, (uint64_t*)nullptr, (int64_t)(pl.V + 2));
    cub::DeviceRadixSort::SortPairs(nullptr, b2, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                    (const uint32_t*)nullptr, (uint32_t*)nullptr, (int64_t)std::max<uint64_t>(total, 1));
    return std::max(b1, b2);
}

cudaError_t class_count(const ClassPlan& pl, uint64_t Ltab, const uint32_t* primes, uint64_t np_tab, uint32_t* tab,
                        uint64_t* cnt, uint64_t* offs, void* scratch, size_t scratch_bytes, cudaStream_t st) {
    // (k_cls_sieve marks with the primes whose square lies in the segment; it stops at the
    // first larger one, so passing every listed prime costs nothing)
    const uint64_t nseg = (Ltab + 1 + CLS_SEG - 1) / CLS_SEG;
    cudaFuncSetAttribute(k_cls_sieve, cudaFuncAttributeMaxDynamicSharedMemorySize, CLS_SEG * sizeof(uint32_t));
    k_cls_sieve<<<grid_for(nseg, 1, 148 * 4), 512, CLS_SEG * sizeof(uint32_t), st>>>(tab, Ltab, primes,
                                                                                    (uint32_t)np_tab);
    if (np_tab) k_cls_scatter<<<grid_for(np_tab, 256), 256, 0, st>>>(tab, primes, np_tab);
    k_cls_count<<<grid_for(pl.V + 1, 256), 256, 0, st>>>(pl.X, pl.V, tab, primes, cnt);
    cudaMemsetAsync(cnt + pl.V + 1, 0, sizeof(uint64_t), st);
    size_t bytes = scratch_bytes;
    cub::DeviceScan::ExclusiveSum(scratch, bytes, cnt, offs, (int64_t)(pl.V + 2), st);
    return cudaGetLastError();
}

cudaError_t class_build(const ClassPlan& pl, uint64_t total, const uint32_t* primes, const uint32_t* tab,
                        const uint64_t* offs, BnxHeavyEnt* ent_tmp, BnxHeavyEnt* ent, uint64_t* keys,
                        uint64_t* key_tmp, uint32_t* perm, uint32_t* perm_tmp, void* scratch, size_t scratch_bytes,
                        uint32_t* kinfo, uint64_t K, cudaStream_t st) {
    ClsBuildArgs a{pl.X, pl.V, total, offs, tab, primes, ent_tmp, keys, perm, pl.nwords, pl.dpw, pl.bits};
    k_cls_build<<<grid_for(total, 256), 256, 0, st>>>(a);
    k_cls_kinfo<<<grid_for(K, 256), 256, 0, st>>>(K, tab, primes, kinfo);
    // LSD: least significant word first; each pass sorts (word[perm], perm) stably.  The
    // sorted keys themselves are not needed: they go to whichever buffer is free
    uint32_t* pin = perm;
    uint32_t* pout = perm_tmp;
    const int wbits = pl.dpw * pl.bits;
    for (int w = pl.nwords - 1; w >= 0; --w) {
        uint64_t* kw = keys + (uint64_t)w * total;
        const uint64_t* kin = kw;
        uint64_t* kout = key_tmp;
        if (w != pl.nwords - 1) {  // the word in the current order, then sorted into its own slot
            k_cls_gather_key<<<grid_for(total, 256), 256, 0, st>>>(kw, pin, total, key_tmp);
            kin = key_tmp;
            kout = kw;
        }
        size_t bytes = scratch_bytes;
        cub::DeviceRadixSort::SortPairs(scratch, bytes, kin, kout, pin, pout, (int64_t)total, 0, wbits, st);
        std::swap(pin, pout);
    }
    k_cls_gather<<<grid_for(total, 256), 256, 0, st>>>(ent_tmp, pin, total, ent);
    return cudaGetLastError();
}

// Load this file's kernels and the cub scan / radix-sort kernels it uses (a warm call of each,
// large enough for the multi-pass sort path).
cudaError_t classes_preload(cudaStream_t st) {
    const void* fns[] = {(const void*)k_cls_sieve, (const void*)k_cls_scatter, (const void*)k_cls_count,
                         (const void*)k_cls_build, (const void*)k_cls_gather_key, (const void*)k_cls_gather,
                         (const void*)k_cls_kinfo};
    for (const void* f : fns) {
        cudaFuncAttributes at;
        const cudaError_t e = cudaFuncGetAttributes(&at, f);
        if (e != cudaSuccess) return e;
    }
    cudaError_t e = cudaFuncSetAttribute(k_cls_sieve, cudaFuncAttributeMaxDynamicSharedMemorySize, CLS_SEG * sizeof(uint32_t));
    if (e != cudaSuccess) return e;
    constexpr int64_t n = 1 << 17;
    size_t b1 = 0, b2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, b1, (const uint64_t*)nullptr, (uint64_t*)nullptr, n);
    cub::DeviceRadixSort::SortPairs(nullptr, b2, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                    (const uint32_t*)nullptr, (uint32_t*)nullptr, n);
    const size_t tb = std::max(b1, b2);
    unsigned char* buf = nullptr;
    e = cudaMallocAsync((void**)&buf, n * (2 * sizeof(uint64_t) + 2 * sizeof(uint32_t)) + tb, st);
    if (e != cudaSuccess) return e;
    uint64_t* k0 = reinterpret_cast<uint64_t*>(buf);
    uint64_t* k1 = k0 + n;
    uint32_t* v0 = reinterpret_cast<uint32_t*>(k1 + n);
    uint32_t* v1 = v0 + n;
    void* tmp = v1 + n;
    cudaMemsetAsync(buf, 0, n * (2 * sizeof(uint64_t) + 2 * sizeof(uint32_t)), st);
    size_t bytes = tb;
    cub::DeviceScan::ExclusiveSum(tmp, bytes, k0, k1, n, st);
    bytes = tb;
    cub::DeviceRadixSort::SortPairs(tmp, bytes, k0, k1, v0, v1, n, 0, 60, st);
    e = cudaGetLastError();
    cudaFreeAsync(buf, st);
    return e;
}

}  // namespace bnx
