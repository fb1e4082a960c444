// bnx_heavy.cu -- the candidate generator of the search: heavy-side enumeration.
//
// A candidate is an n with R = rad(n) rad(n+1) <= 2n (Lemma 1).  With the
// surplus s(x) = x / rad(x) that reads  s(n) s(n+1) >= (n+1)/2, so the larger surplus is at
// least sqrt((n+1)/2): one of x in {n, n+1} is HEAVY, 2 s(x)^2 >= x.  Heavy integers are
// rare (about 50 sqrt(N) below N) and can be listed without looking at the others:
//   x = k * sigma * rad(sigma),  sigma = s(x),  k = the squarefree part of x (coprime to
//   sigma),  and  x heavy  <=>  k * rad(sigma) <= 2 sigma.
// b = sigma * rad(sigma) runs over the powerful numbers (b = prod p^(e+1) <-> sigma =
// prod p^e), so the host lists the classes (b, sigma) once per bound (a DFS over primes) and
// the device walks every (class, k) of the domain:
//   k_heavy_count   per class: the k range that lands in the domain; classes with many k
//                   are counted in sieve chunks, the others in single items (one packed scan)
//   (cub scan)      flattened item / chunk offsets
//   k_heavy_screen  per item: canonical k (squarefree, coprime to sigma: bit tables), then
//                   for y = x - 1 and y = x + 1 a conservative test of s(x) s(y) >= (n+1)/2:
//                   y is trial-divided by the primes <= P2 = y_max^(1/4) only; the cofactor
//                   c then has at most three prime factors, all > P2, so s(c) is 1, p (c = p^2
//                   or p^2 q, p <= sqrt(c / (P2+1))) or p^2 (c = p^3) and is bounded exactly
//   k_heavy_sieve   the same test for the classes with many k, with the trial division
//                   replaced by sieving the progressions k = -+b^-1 (mod p) over a chunk of k
//   k_heavy_exact   per survivor: rad(y) exactly (trial division to cbrt, cofactor 1, p,
//                   p^2 or pq), the exact test R <= 2n, and de-duplication (a candidate with
//                   both sides heavy is kept only from x = n)
// The survivors of k_heavy_exact are exactly the candidates, with rad(n), rad(n+1) attached;
// k_tail / k_tail_heavy then walk their residue classes (bnx_kernels.cu).  Work: ~1.2M
// canonical heavy x below 2^32 (instead of 2^32 integers), each costing ~54 trial divisions
// per side.  Every kernel here can run one shard of a search (HeavyArgs::shard, multi-GPU).
#include <cub/device/device_scan.cuh>
#include <type_traits>

#include "bnx_kernels.cuh"
#include "bnx_rad.cuh"

namespace bnx {

namespace {

__device__ __forceinline__ uint32_t gcd32(uint32_t a, uint32_t b) {
    if (!a) return b;
    if (!b) return a;
    const int sh = __ffs(a | b) - 1;
    a >>= __ffs(a) - 1;
    do {
        b >>= __ffs(b) - 1;
        if (a > b) { const uint32_t t = a; a = b; b = t; }
        b -= a;
    } while (b);
    return a << sh;
}

// Exact integer square root test: q with q^2 = c, or 0.  A float root, rounded, is within
// 0.4 of the integer one for c < 2^45; above, a double root (exact to 2^52).
__device__ __forceinline__ uint64_t exact_sqrt(uint64_t c) {
    const uint64_t q = c < (1ull << 45) ? (uint64_t)rintf(sqrtf((float)c)) : (uint64_t)llrint(sqrt((double)c));
    return q * q == c ? q : 0;
}

// Upper bound of s(c) for an odd cofactor c > 0 whose prime factors all exceed P2 (p1 =
// P2 + 1, p1^4 > c): c is 1, p, pq, pqr (s = 1), p^2 (s = sqrt c), p^2 q (s = p <=
// sqrt(c / p1)) or p^3 (s = c^(2/3)).  Only an upper bound is needed (k_heavy_exact
// decides), so the p^2 q case uses a rounded-up float root; squares and cubes are detected
// exactly (rounded roots checked in integers, see exact_sqrt; the cube root of c < 2^50 is
// below 2^17, where cbrtf's error is < 0.02).
__device__ __forceinline__ float approx_rsqrt(float x);
__device__ __forceinline__ float approx_cbrt(float x);
__device__ __forceinline__ uint64_t surplus_bound(uint64_t c, const HeavyArgs& a) {
    if (c < a.p1sq) return 1;  // 1 or a prime
    uint64_t u = 1;
    const float cf = (float)c;
    if ((c & 7) == 1) {  // odd squares are 1 mod 8
        const uint64_t q = exact_sqrt(c);
        if (q) u = q;
    }
    if (c >= a.p1cube) {
        // >= sqrt(c / p1): the MUFU root's relative error (~1e-6) is inside the 1.0001 margin
        const float t = cf * a.inv_p1f;
        const uint64_t v = (uint64_t)(t * approx_rsqrt(t) * 1.0001f) + 1;
        if (v > u) u = v;
        // p^3 with p > P2 >= 7: p^3 = +-1 mod 7 and mod 9, i.e. c mod 63 in {1, 8, 55, 62};
        // c mod 63 from the 32-bit halves (2^32 = 4 mod 63; c < 2^53: hi < 2^21)
        const uint32_t lo = (uint32_t)c, hi = (uint32_t)(c >> 32);
        const uint32_t m63 = (4u * hi + lo % 63u) % 63u;
        if (!a.cube_filter || m63 == 1 || m63 == 8 || m63 == 55 || m63 == 62) {
            // a cube below 2^53 has its root below 2^18: the MUFU cube root lands within 0.3
            const uint64_t r = (uint64_t)rintf(c < (1ull << 45) ? approx_cbrt(cf) : cbrtf(cf));
            if (r * r * r == c && r * r > u) u = r * r;
        }
    }
    return u;
}

// The same for c < 2^32 in 32-bit arithmetic (narrow y: the 64-bit remainder and products
// are most of the bound's cost).
__device__ __forceinline__ float approx_rsqrt(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float approx_cbrt(float x) {  // x > 0: 2^(log2(x) / 3)
    float l, r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(x));
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(l * (1.0f / 3.0f)));
    return r;
}
// The roots here only have to land within 0.5 of the integer ones (c < 2^32: sqrt < 2^16,
// cbrt < 1626, relative errors of the MUFU approximations ~1e-6), or be an upper bound with
// the 1.0001 margin, so the hardware approximations replace the IEEE sqrtf / cbrtf.
__device__ __forceinline__ uint64_t surplus_bound32(uint32_t c, const HeavyArgs& a) {
    if (c < a.p1sq) return 1;
    uint32_t u = 1;
    const float cf = (float)c;
    if ((c & 7) == 1) {
        const uint32_t q = (uint32_t)rintf(cf * approx_rsqrt(cf));  // q < 2^16 (q = 2^16 wraps to 0 != c)
        if (q * q == c) u = q;
    }
    if (c >= a.p1cube) {
        const float t = cf * a.inv_p1f;
        const uint32_t v = (uint32_t)(t * approx_rsqrt(t) * 1.0001f) + 1;
        if (v > u) u = v;
        const uint32_t m63 = c % 63u;
        if (!a.cube_filter || m63 == 1 || m63 == 8 || m63 == 55 || m63 == 62) {
            const uint64_t r = (uint64_t)rintf(approx_cbrt(cf));
            if (r * r * r == c && r * r > u) u = (uint32_t)(r * r);
        }
    }
    return u;
}

// 2 * sigma * v >= rhs without overflow (sigma, v < 2^62).
__device__ __forceinline__ bool twice_prod_ge(uint64_t sigma, uint64_t v, uint64_t rhs) {
    const uint64_t s2 = 2 * sigma;
    return __umul64hi(s2, v) != 0 || s2 * v >= rhs;
}

// Trial classes list only the k that can be canonical as far as 2 and 3 go (gcd(k, sigma)
// = 1): wsel = rmask & 3 = [2 | sigma] + 2 [3 | sigma] selects every k, the odd k, the k
// not divisible by 3, or k = +-1 (mod 6).  wheel_rank(K) = listed k in [0, K]; wheel_k(rho)
// = the listed k of rank rho (0-based, k = 0 listed only for wsel = 0).
__device__ __forceinline__ uint64_t wheel_rank(uint64_t K, uint32_t wsel) {
    switch (wsel) {
        case 0: return K + 1;
        case 1: return (K + 1) / 2;
        case 2: return K - K / 3;
        default: return 2 * (K / 6) + (K % 6 >= 1) + (K % 6 >= 5);
    }
}
__device__ __forceinline__ uint64_t wheel_k(uint64_t rho, uint32_t wsel) {
    switch (wsel) {
        case 0: return rho;
        case 1: return 2 * rho + 1;
        case 2: return 3 * (rho >> 1) + 1 + (rho & 1);
        default: return 6 * (rho >> 1) + 1 + 4 * (rho & 1);
    }
}

// The packed item count of class i (trial items in the low 40 bits, sieve chunks above): the
// k range [ceil(x_lo / b), min(2m, floor(x_hi / b))] of the domain; also the class's first
// listed k / item rank (klo) and, for a sieve class, its number of listed k (kcnt).
__device__ __forceinline__ uint64_t class_count(const HeavyArgs& a, uint64_t i) {
    const BnxHeavyEnt e = a.ent[i];
    uint64_t kh = 2 * e.m;
    uint64_t kl = 1;
    if (e.b > a.x_hi) {
        kh = 0;
    } else {
        // floor(x_hi / b) and ceil(x_lo / b): a double estimate, corrected in integers
        const double rb = 1.0 / (double)e.b;
        uint64_t top = (uint64_t)((double)a.x_hi * rb);
        while (top * e.b > a.x_hi) --top;
        while ((top + 1) * e.b <= a.x_hi) ++top;
        if (top < kh) kh = top;
        if (a.x_lo > e.b) {  // (else ceil(x_lo / b) = 1: every search from n = 1)
            uint64_t lo = (uint64_t)((double)a.x_lo * rb);
            while (lo > 0 && lo * e.b >= a.x_lo) --lo;
            while (lo * e.b < a.x_lo) ++lo;  // smallest lo with lo * b >= x_lo
            if (lo > kl) kl = lo;
        }
    }
    const uint64_t c = kh >= kl ? kh - kl + 1 : 0;
    if (c >= a.kmin) {  // sieve chunks over every k (every odd k when sigma is even)
        const uint64_t st = (e.rmask & 1u) ? 2 : 1;
        const uint64_t ks = st == 2 ? (kl | 1u) : kl;
        const uint64_t cs = kh >= ks ? (kh - ks) / st + 1 : 0;
        a.klo[i] = (uint32_t)ks;
        a.kcnt[i] = (uint32_t)cs;  // listed k (index space)
        return ((cs + a.kc - 1) / a.kc) << 40;
    }
    // trial items: the k coprime to 2 and 3 where sigma has them (wheel_k)
    const uint32_t wsel = e.rmask & 3u;
    const uint64_t r0 = wheel_rank(kl - 1, wsel);
    a.klo[i] = (uint32_t)r0;  // rank of the class's first item
    a.kcnt[i] = 0;            // (sieve classes only)
    return c ? wheel_rank(kh, wsel) - r0 : 0;
}

__global__ void k_heavy_count(HeavyArgs a) {
    // the search's counters and flags start here (no memset launches; every later kernel
    // runs after this one)
    if (blockIdx.x == 0 && threadIdx.x < CTR_N) a.ctr[threadIdx.x] = 0;
    if (blockIdx.x == 0 && threadIdx.x < 4) a.flags[threadIdx.x] = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < a.nent;
         i += (uint64_t)gridDim.x * blockDim.x)
        a.cnt[i] = class_count(a, i);
}

// Inclusive scan of the values of one block of 256 threads (every thread gets its own).
__device__ __forceinline__ uint64_t block_scan256(uint64_t v, uint64_t* s_w, uint64_t& total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint64_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint64_t y = __shfl_up_sync(0xFFFFFFFFu, x, d);
        if (lane >= d) x += y;
    }
    if (lane == 31) s_w[wid] = x;
    __syncthreads();
    uint64_t pre = 0;
    total = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        const uint64_t t = s_w[w];
        pre += w < wid ? t : 0;
        total += t;
    }
    return pre + x;
}

// Few classes and no sieve classes (bounds below ~2^33): the counts scanned per tile of
// HEAVY_TILE classes only -- incl holds the prefix within the tile, tile_tot the tile totals,
// which k_heavy_screen scans for itself in its prologue (no scan kernels between the count
// and the screen).
__global__ void __launch_bounds__(HEAVY_TILE) k_heavy_count_local(HeavyArgs a) {
    if (blockIdx.x == 0 && threadIdx.x < CTR_N) a.ctr[threadIdx.x] = 0;
    if (blockIdx.x == 0 && threadIdx.x < 4) a.flags[threadIdx.x] = 0;
    __shared__ uint64_t s_w[8];
    const uint64_t i = (uint64_t)blockIdx.x * HEAVY_TILE + threadIdx.x;
    uint64_t total;
    const uint64_t x = block_scan256(i < a.nent ? class_count(a, i) : 0, s_w, total);
    if (i < a.nent) a.incl[i] = x;
    if (threadIdx.x == 0) a.tile_tot[blockIdx.x] = total;
}

// Class of item w: smallest i >= lo with incl[i] > w (galloping, then binary search).
template <class Incl>
__device__ __forceinline__ uint64_t first_class_above(const Incl& incl, uint64_t lo, uint64_t n, uint64_t w) {
    uint64_t step = 1, hi = lo;
    while (hi < n - 1 && (incl(hi) & HEAVY_TRIAL_MASK) <= w) {
        lo = hi + 1;
        hi = min(n - 1, hi + step);
        step <<= 1;
    }
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if ((incl(mid) & HEAVY_TRIAL_MASK) > w) hi = mid; else lo = mid + 1;
    }
    return lo;
}

// The same search by a whole warp: 32 probes per round narrow [lo, hi] 32-fold, so a run's
// first class costs ~4 dependent L2 loads instead of ~2 log2(nent) (requires w < incl[n-1]).
// CHUNKS: search the sieve-chunk prefix (incl >> 40) instead of the trial-item prefix.
template <bool CHUNKS = false, class Incl>
__device__ __forceinline__ uint64_t first_class_above_warp(const Incl& incl, uint64_t n, uint64_t w, int lane) {
    uint64_t lo = 0, hi = n - 1;  // the answer lies in [lo, hi]
    while (lo < hi) {
        const uint64_t span = hi - lo;
        const uint64_t v = incl(lo + span * (lane + 1) / 32);
        const bool above = (CHUNKS ? v >> 40 : v & HEAVY_TRIAL_MASK) > w;
        const int j = __ffs(__ballot_sync(0xFFFFFFFFu, above)) - 1;  // lane 31 probes hi: j >= 0
        const uint64_t nlo = j ? lo + span * j / 32 + 1 : lo;
        hi = lo + span * (j + 1) / 32;
        lo = nlo;
    }
    return lo;
}

struct HeavyItem {
    uint64_t x, sigma, radx;
};

// The y tests of one heavy x (both sides), see the file comment.  Shared tables per odd
// prime <= P2: (p^-1 mod 2^64, floor((2^64-1)/p)), the same mod 2^32, p, and 2^32 mod p.
// NARROW: both y below 2^32 -- every test, division and bound in 32-bit arithmetic (the
// kernel is bound by its ALU/IMAD instruction count).  SIEVED: the divisibility masks come
// from k_heavy_sieve's progression marks (word w of the item at sm[w * stride]) instead of
// the per-prime tests.
template <bool NARROW, bool SIEVED = false>
__device__ __forceinline__ void y_tests_impl(const HeavyArgs& a, const HeavyItem& it, const ulonglong2* s_il,
                                             const uint32_t* s_p, const uint2* s_pd32, const uint32_t* s_c32,
                                             const uint32_t* sm = nullptr, int stride = 0,
                                             const uint32_t* s_e32 = nullptr) {
    using W = typename std::conditional<NARROW, uint32_t, uint64_t>::type;
    const uint64_t x = it.x;
    const bool vL = x >= 2 && x - 1 >= a.n_first && x - 1 <= a.n_last;
    const bool vU = x >= a.n_first && x <= a.n_last;
    const uint64_t yL = vL ? x - 1 : 1, yU = x + 1;
    const int tL = __ffsll((long long)yL) - 1, tU = __ffsll((long long)yU) - 1;
    W cL = (W)(yL >> tL), cU = (W)(yU >> tU);
    W sL = tL ? (W)1 << (tL - 1) : (W)1, sU = tU ? (W)1 << (tU - 1) : (W)1;
    W rL = tL ? (W)2 : (W)1, rU = tU ? (W)2 : (W)1;  // radicals of the divided-off parts
    const uint32_t x32 = (uint32_t)x, xh = (uint32_t)(x >> 32);
    // x >= 2^32: W = x_lo + x_hi (2^32 mod p) = x (mod p) stays below 2^32 - 1 for every
    // stage-1 prime (all below p1) unless x_lo is within x_hi p1 of 2^32 (rare)
    const bool nowrap = s_e32 && xh < 65536u && x32 < 0xFFFFFFFFu - xh * (uint32_t)a.p1;
    // Divisibility by 32 primes at a time into a bit mask, branch-free (the lanes of a warp
    // stay converged): one bit per prime for both sides (an odd p divides at most one of
    // x - 1, x + 1), the side is found in the post-pass.  The table is padded to a multiple
    // of 32 (the padding bits are masked off) so that the loop unrolls with constant bit
    // positions.  Then the hits (about 1.5 per y) are divided out with their powers.
    for (int j0 = 0; j0 < a.np2; j0 += 32) {
        const int jn = min(32, a.np2 - j0);
        uint32_t m = 0;
        if constexpr (SIEVED) {
            m = sm[(j0 >> 5) * stride];
        } else if constexpr (NARROW) {
            // one multiply per prime for both sides: (x -+ 1) p^-1 = x p^-1 -+ p^-1 (mod 2^32)
#pragma unroll
            for (int u = 0; u < 32; ++u) {
                const uint2 d = s_pd32[j0 + u];
                const uint32_t t = x32 * d.x;
                m |= (uint32_t)(min(t - d.x, t + d.x) <= d.y) << u;
            }
        } else if (nowrap) {
            // (W -+ 1) p^-1 = (x_lo -+ 1) p^-1 + x_hi e (mod 2^32), e = (2^32 mod p) p^-1: three
            // multiply-adds per prime for both sides, exact since 0 <= W - 1, W + 1 < 2^32
            const uint32_t xm = x32 - 1u, xp = x32 + 1u;
#pragma unroll
            for (int u = 0; u < 32; ++u) {
                const uint2 d = s_pd32[j0 + u];
                const uint32_t h = xh * s_e32[j0 + u];
                m |= (uint32_t)(min(xm * d.x + h, xp * d.x + h) <= d.y) << u;
            }
        } else {
            // x >= 2^32 (x < 2^53): w = x_lo + x_hi (2^32 mod p) is x mod p shifted into 32
            // bits (a carry out of the add is 2^32 = 2^32 mod p); then the same test on w -+ 1.
            // w - 1 and w + 1 can wrap at 0 and 2^32 - 1: such rare false bits are rejected by
            // the exact division check below.
#pragma unroll
            for (int u = 0; u < 32; ++u) {
                const uint2 d = s_pd32[j0 + u];
                const uint32_t cp = s_c32[j0 + u];
                uint32_t w = x32 + xh * cp;
                if (w < x32) w += cp;
                const uint32_t t = w * d.x;
                m |= (uint32_t)(min(t - d.x, t + d.x) <= d.y) << u;
            }
        }
        if (jn < 32) m &= (1u << jn) - 1;
        while (m) {  // exact division of the side the prime divides (with its powers)
            const int u = __ffs(m) - 1;
            m &= m - 1;
            W inv, lim;
            if constexpr (NARROW) {
                const uint2 d = s_pd32[j0 + u];
                inv = d.x;
                lim = d.y;
            } else {
                const ulonglong2 d = s_il[j0 + u];
                inv = d.x;
                lim = d.y;
            }
            const W pp = s_p[j0 + u];
            W t = cL * inv;
            if (vL && t <= lim) {  // p | cL exactly (rejects a wrapped false bit)
                cL = t;
                rL *= pp;
                for (t = cL * inv; t <= lim; t = cL * inv) { cL = t; sL *= pp; }
            } else if ((t = cU * inv) <= lim) {
                cU = t;
                rU *= pp;
                for (t = cU * inv; t <= lim; t = cU * inv) { cU = t; sU *= pp; }
            }
        }
    }
    uint64_t uL, uU;
    if constexpr (NARROW) {
        uL = surplus_bound32(cL, a);
        uU = surplus_bound32(cU, a);
    } else {
        uL = surplus_bound(cL, a);
        uU = surplus_bound(cU, a);
    }
    const bool pL = vL && twice_prod_ge(it.sigma, (uint64_t)sL * uL, x);
    const bool pU = vU && twice_prod_ge(it.sigma, (uint64_t)sU * uU, x + 1);
    if (pL || pU) {
        const unsigned long long slot = atomicAdd(&a.ctr[CTR_SURV], (unsigned long long)(pL + pU));
        if (pL && slot < a.q1_cap) a.q1[slot] = BnxSurv{(x - 1) | (1ull << 63), it.radx, (uint64_t)cL, (uint64_t)rL};
        const unsigned long long s2 = slot + pL;
        if (pU && s2 < a.q1_cap) a.q1[s2] = BnxSurv{x, it.radx, (uint64_t)cU, (uint64_t)rU};
        if (a.host_flags && slot + pL + pU > a.q1_cap) a.host_flags[2] = 1;
    }
}

__device__ __forceinline__ void y_tests(const HeavyArgs& a, const HeavyItem& it, const ulonglong2* s_il,
                                        const uint32_t* s_p, const uint2* s_pd32, const uint32_t* s_c32,
                                        const uint32_t* s_e32) {
    if (it.x + 1 < (1ull << 32))
        y_tests_impl<true>(a, it, s_il, s_p, s_pd32, s_c32);
    else
        y_tests_impl<false>(a, it, s_il, s_p, s_pd32, s_c32, nullptr, 0, s_e32);
}

// Each CTA owns a contiguous run of items and walks it in windows of HEAVY_THREADS (thread t
// takes item base + t: neighbouring k of one class, or neighbouring classes).  Canonical
// items go to a shared-memory queue; whenever it holds a full CTA's worth, every thread
// takes one and runs the y tests, so the expensive part always runs with full warps.
// LOCAL: the class prefix counts come per tile (k_heavy_count_local); the tile offsets are
// scanned here into shared memory and added on every read.
template <bool LOCAL>
__global__ void __launch_bounds__(HEAVY_THREADS, 8) k_heavy_screen(HeavyArgs a) {
    constexpr int T = HEAVY_THREADS;
    // np2p (inv32, lim32) first -- the hot table at a fixed shared address, so the unrolled
    // mask loop addresses it by immediates -- then np2 (inv, lim), np2 p, np2p 2^32 mod p,
    // np2p (2^32 mod p) p^-1 mod 2^32 (np2p: np2 padded to 32)
    extern __shared__ uint2 s_pd32[];
    const int np2p = (a.np2 + 31) & ~31;
    ulonglong2* s_il = reinterpret_cast<ulonglong2*>(s_pd32 + np2p);  // (np2p * 8 B: 16-byte aligned)
    uint32_t* s_p = reinterpret_cast<uint32_t*>(s_il + a.np2);
    uint32_t* s_c32 = s_p + a.np2;
    uint32_t* s_e32 = s_c32 + np2p;
    // LOCAL: ntiles tile offsets (8-byte aligned: the tables above end 4 bytes short of it when
    // np2 is odd)
    uint64_t* s_pre = reinterpret_cast<uint64_t*>(s_e32 + np2p + (a.np2 & 1));
    __shared__ HeavyItem s_q[2 * T];
    __shared__ uint64_t s_end[T];  // class ends of a multi-class window
    __shared__ int s_cnt;
    __shared__ unsigned long long s_cls;
    const int tid = threadIdx.x;
    for (int j = tid; j < a.np2; j += T) {
        s_il[j] = make_ulonglong2(a.pdiv[j].inv, a.pdiv[j].lim);
        const uint4 q = a.pd32[j];
        s_pd32[j] = make_uint2(q.x, q.y);
        s_p[j] = q.z;
        s_c32[j] = q.w;
        s_e32[j] = q.w * q.x;
    }
    for (int j = a.np2 + tid; j < np2p; j += T) {  // padding (its bits are masked off)
        s_pd32[j] = make_uint2(1u, 0u);
        s_c32[j] = 0u;
        s_e32[j] = 0u;
    }
    if (tid == 0) s_cnt = 0;
    if constexpr (LOCAL) {  // exclusive scan of the tile totals (each thread a run of tiles)
        static_assert(T == 256, "block_scan256");
        const int nt = (int)a.ntiles, per = (nt + T - 1) / T;
        uint64_t loc = 0;
        for (int j = 0; j < per; ++j) {
            const int t = tid * per + j;
            if (t < nt) {
                const uint64_t v = a.tile_tot[t];
                s_pre[t] = v;
                loc += v;
            }
        }
        __shared__ uint64_t s_w[8];
        uint64_t total;
        uint64_t run = block_scan256(loc, s_w, total) - loc;
        for (int j = 0; j < per; ++j) {
            const int t = tid * per + j;
            if (t < nt) {
                const uint64_t v = s_pre[t];
                s_pre[t] = run;
                run += v;
            }
        }
        __syncthreads();
    }
    // the global inclusive prefix of class i
    auto incl = [&](uint64_t i) -> uint64_t {
        if constexpr (LOCAL) return a.incl[i] + s_pre[i / HEAVY_TILE];
        else return a.incl[i];
    };
    // k_heavy_exact may be scheduled now (programmatic dependent launch): its CTAs take the
    // SMs our CTAs leave and stage their prime tables before they wait for our completion
    asm volatile("griddepcontrol.launch_dependents;");
    if (a.nent == 0) return;
    // The trial items in gridDim * run_mult * nshards equal runs; run r of shard s is run
    // r * nshards + s, so every shard samples the whole class range (the classes differ in
    // canonical density).  CTA g starts with run g and then fetches runs from a counter, so
    // CTAs that drew sparse runs take more of them (the SMs finish together).
    const uint64_t Wt = incl(a.nent - 1) & HEAVY_TRIAL_MASK;
    const uint64_t WA = a.run_mult ? Wt * min(a.run_first, 256u) / 256 : Wt;  // items of the static runs
    const uint64_t nr = (uint64_t)gridDim.x * (1 + a.run_mult);
    __shared__ unsigned long long s_run;
    uint64_t run = blockIdx.x, b1 = 0, base = 0;
    bool more = true;
    // `cnt` is every thread's copy of s_cnt, read only between the two barriers of a fill
    // step (after all appends, before the next) so that the loop conditions agree.
    int cnt = 0;
    for (;;) {
        // fill the queue up to at least T entries (or until the runs are exhausted)
        while (cnt < T && more) {
            if (base >= b1) {  // next run
                if (run == ~0ull) {
                    if (tid == 0) s_run = gridDim.x + atomicAdd(&a.ctr[CTR_RUNS], 1ull);
                    __syncthreads();
                    run = s_run;
                }
                if (run >= nr) {
                    more = false;
                    break;
                }
                if (run < gridDim.x) {  // static run
                    const uint64_t blk = run * a.nshards + a.shard, nb = (uint64_t)gridDim.x * a.nshards;
                    base = WA * blk / nb;
                    b1 = WA * (blk + 1) / nb;
                } else {
                    const uint64_t blk = (run - gridDim.x) * a.nshards + a.shard, nb = (nr - gridDim.x) * a.nshards;
                    base = WA + (Wt - WA) * blk / nb;
                    b1 = WA + (Wt - WA) * (blk + 1) / nb;
                }
                run = ~0ull;
                if (tid < 32 && base < b1) {
                    const uint64_t c0 = first_class_above_warp(incl, a.nent, base, tid);
                    if (tid == 0) s_cls = c0;
                }
                __syncthreads();
                continue;
            }
            const uint64_t w = base + tid;
            const uint64_t cls0 = s_cls;
            // class of each item: the whole window in class cls0 (most windows), else the
            // ends of the next T classes staged in shared memory and searched there
            const uint64_t wend = min(base + T, b1);  // the window's end
            const bool one = (incl(cls0) & HEAVY_TRIAL_MASK) >= wend;  // CTA-uniform
            int kwin = T - 1;  // every item of the window lies in staged classes [0, kwin] (or beyond T - 1)
            if (!one) {
                const uint64_t j = cls0 + tid;
                const uint64_t end = j < a.nent ? (incl(j) & HEAVY_TRIAL_MASK) : ~0ull;
                s_end[tid] = end;
                // the ends are ascending: the classes ending at or after the window's end are
                // the last `count` staged ones, so the first of them closes the search range
                kwin = min(T - 1, T - __syncthreads_count(end >= wend));
            }
            uint64_t i = cls0;
            if (w < b1) {
                if (!one) {
                    if (w < s_end[T - 1]) {
                        int lo = 0, hi = kwin;  // first staged class ending above w
                        while (lo < hi) {
                            const int mid = (lo + hi) >> 1;
                            if (s_end[mid] > w) hi = mid; else lo = mid + 1;
                        }
                        i = cls0 + lo;
                    } else {
                        i = first_class_above(incl, cls0 + T - 1, a.nent, w);
                    }
                }
                BNX_CHECK(i < a.nent);
                const BnxHeavyEnt e = a.ent[i];
                // item -> k: the class's listed k (see wheel_k)
                const uint64_t k = wheel_k(a.klo[i] + (w - (i ? incl(i - 1) & HEAVY_TRIAL_MASK : 0)), e.rmask & 3u);
                if (k < a.nkinfo) {
                    bool canon = (a.kinfo[k] & (e.rmask | 0x80000000u)) == 0;
                    if (canon && e.rbig > 1 && k >= e.rbig_min) canon = gcd32((uint32_t)k, e.rbig) == 1;
                    if (canon) {
                        const int slot = atomicAdd(&s_cnt, 1);
                        BNX_CHECK(slot < 2 * T);
                        s_q[slot] = HeavyItem{k * e.b, e.m * e.r, k * e.r};
                    }
                } else {
                    a.flags[1] = 1;
                    if (a.host_flags) a.host_flags[1] = 1;
                }
            }
            __syncthreads();
            cnt = s_cnt;
            if (w == min(base + T, b1) - 1) s_cls = i;  // class of the window's last item
            base += T;
            __syncthreads();
        }
        if (cnt == 0) break;
        const int take = min(cnt, T);
        if (tid < take && !a.probe_walk) y_tests(a, s_q[cnt - 1 - tid], s_il, s_p, s_pd32, s_c32, s_e32);
        cnt -= take;
        __syncthreads();
        if (tid == 0) s_cnt = cnt;
        __syncthreads();
    }
}

// Classes with many k: y = k b -+ 1 runs through an arithmetic progression in k, so for an
// odd prime p not dividing b, p | k b + 1 <=> k = -b^-1 and p | k b - 1 <=> k = +b^-1 (mod p).
// A class with sigma even lists only its odd k (index i -> k = k0 + 2i; the progression
// offsets are multiplied by 2^-1 mod p).  Each CTA owns runs of chunks (up to kc listed k
// of one class each):
//   1. per prime <= P2, on entering a class: b mod p (Barrett with the table's
//      floor((2^64-1)/p)), b^-1 mod p (host table), the first index of each side's
//      progression in the chunk; for the next chunk of the same class the indices just
//      move by kc mod p;
//   2. marks: host-built tasks of ~16 hits each append the prime's index to the (k, side)
//      hit list in shared memory (a packed byte counter per list, HEAVY_HITS slots; a list
//      that overflows is redone by trial division in step 4);
//   3. canonical k of the chunk are compacted into a shared list;
//   4. per canonical k: the listed primes are divided out of both y exactly (with their
//      powers) and the same stage-1 test as k_heavy_screen decides.
// So the per-k work is ~3 marks and ~3 exact divisions instead of 2 pi(P2) trial divisions,
// and it does not grow with pi(P2).
__device__ __forceinline__ uint64_t mod_by_lim(uint64_t v, uint64_t p, uint64_t lim) {
    uint64_t r = v - __umul64hi(v, lim) * p;  // lim = floor((2^64-1)/p): quotient off by <= 1
    while (r >= p) r -= p;
    return r;
}

// MASK (at most 64 primes <= P2, bounds up to ~2^33): the marks set one bit per prime in two
// mask words per k (an odd prime divides at most one of x - 1, x + 1), and step 4 is the
// screen's own post-pass (y_tests_impl<., true>) on those words, in 32-bit arithmetic when
// the chunk's y are below 2^32.  Otherwise (up to 1023 primes): hit lists of prime indices
// per (k, side), 64-bit.
template <bool MASK>
__global__ void __launch_bounds__(256) k_heavy_sieve(HeavyArgs a) {
    extern __shared__ __align__(16) unsigned char sm_raw[];
    const int np2 = a.np2, kc = a.kc, np2p = (np2 + 31) & ~31;
    ulonglong2* s_il = reinterpret_cast<ulonglong2*>(sm_raw);                  // np2
    uint2* s_pd32 = reinterpret_cast<uint2*>(s_il + np2);                      // MASK: np2p
    uint32_t* s_p = reinterpret_cast<uint32_t*>(s_pd32 + (MASK ? np2p : 0));   // np2
    uint32_t* s_c32 = s_p + np2;                                               // MASK: np2p
    int32_t* s_off = reinterpret_cast<int32_t*>(s_c32 + (MASK ? np2p : 0));    // 2 np2
    uint32_t* s_kcm = reinterpret_cast<uint32_t*>(s_off + 2 * np2);            // np2: kc mod p
    uint32_t* s_task = s_kcm + np2;                                            // ntasks
    uint32_t* s_list = s_task + a.ntasks;                                      // kc
    // MASK: mask word w of index kk at s_marks[w * kc + kk] (2 kc words); else packed byte
    // counters [2][kc / 4] then the hit lists [2][kc][HEAVY_HITS]
    uint32_t* s_marks = s_list + kc;
    uint32_t* hcnt = s_marks;
    uint16_t* hits = reinterpret_cast<uint16_t*>(s_marks + kc / 2);
    __shared__ BnxHeavyEnt s_e;
    __shared__ uint64_t s_k0, s_kend, s_cls_end, s_cls, s_kfirst;
    __shared__ int s_nl, s_fresh;
    const int tid = threadIdx.x;
    for (int j = tid; j < np2; j += blockDim.x) {
        s_il[j] = make_ulonglong2(a.pdiv[j].inv, a.pdiv[j].lim);
        s_p[j] = (uint32_t)a.pdiv[j].p;
        s_kcm[j] = (uint32_t)kc % (uint32_t)a.pdiv[j].p;
        if constexpr (MASK) {
            const uint4 q = a.pd32[j];
            s_pd32[j] = make_uint2(q.x, q.y);
            s_c32[j] = q.w;
        }
    }
    if constexpr (MASK) {
        for (int j = np2 + tid; j < np2p; j += blockDim.x) {  // padding (its bits are masked off)
            s_pd32[j] = make_uint2(1u, 0u);
            s_c32[j] = 0u;
        }
    }
    for (int t = tid; t < a.ntasks; t += blockDim.x) s_task[t] = a.tasks[t];
    if (a.nent == 0) return;
    const uint64_t Ct = a.incl[a.nent - 1] >> 40;  // runs of chunks interleaved over the shards (as above)
    const uint64_t nb = (uint64_t)gridDim.x * a.nshards, blk = (uint64_t)blockIdx.x * a.nshards + a.shard;
    const uint64_t c_begin = Ct * blk / nb, c_end = Ct * (blk + 1) / nb;
    for (uint64_t ch = c_begin; ch < c_end; ++ch) {
        __syncthreads();
        if (tid < 32) {  // warp 0 finds the chunk's class
            const bool enter = ch == c_begin || ch >= s_cls_end;
            if (enter) {
                // the class: first with chunk prefix > ch (a 32-way search: the sieved classes
                // can be sparse among the trial classes, so no linear probe from the last one)
                const uint64_t cls = first_class_above_warp<true>([&](uint64_t j) { return a.incl[j]; }, a.nent, ch, tid);
                if (tid == 0) {
                    BNX_CHECK(cls < a.nent);
                    const uint64_t first = cls ? a.incl[cls - 1] >> 40 : 0;
                    s_e = a.ent[cls];
                    s_k0 = (ch - first) * (uint64_t)kc;  // index of the chunk's first listed k
                    s_kend = a.kcnt[cls];                 // listed k of the class
                    s_kfirst = a.klo[cls];
                    s_cls_end = a.incl[cls] >> 40;
                    s_cls = cls;
                    s_fresh = 1;
                }
            } else if (tid == 0) {
                s_k0 += (uint64_t)kc;
                s_fresh = 0;
            }
            if (tid == 0) s_nl = 0;
        }
        __syncthreads();
        const BnxHeavyEnt e = s_e;
        const uint32_t st = (e.rmask & 1u) ? 2 : 1;  // listed k: every k, or every odd k
        const int kn = (int)min((uint64_t)kc, s_kend - s_k0);
        const uint64_t k0 = s_kfirst + st * s_k0;  // the k of index 0 of this chunk
        const bool fresh = s_fresh;
        // 1. progressions (full set-up on entering a class, else shifted by kc)
        for (int j = tid; j < np2; j += blockDim.x) {
            const uint32_t p = s_p[j];
            if (fresh) {
                const uint64_t lim = s_il[j].y;
                const uint32_t bm = (uint32_t)mod_by_lim(e.b, p, lim);
                if (bm == 0) {
                    s_off[2 * j] = s_off[2 * j + 1] = -1;
                } else {
                    const uint32_t inv = a.invtab[a.invoff[j] + bm];
                    const uint32_t k0m = (uint32_t)mod_by_lim(k0, p, lim);
                    // index i of k0 + st i: (root - k0) st^-1 mod p (st^-1 = (p+1)/2 for st = 2)
                    const uint32_t ist = st == 2 ? (p + 1) / 2 : 1;
                    s_off[2 * j] = (int32_t)((2 * p - inv - k0m) % p * ist % p);  // k = -b^-1: p | k b + 1
                    s_off[2 * j + 1] = (int32_t)((inv + p - k0m) % p * ist % p);  // k = +b^-1: p | k b - 1
                }
            } else if (s_off[2 * j] >= 0) {
                const uint32_t d = p - s_kcm[j];
                s_off[2 * j] = (int32_t)(((uint32_t)s_off[2 * j] + d) % p);
                s_off[2 * j + 1] = (int32_t)(((uint32_t)s_off[2 * j + 1] + d) % p);
            }
        }
        for (int w = tid; w < (MASK ? 2 * kc : kc / 2); w += blockDim.x) s_marks[w] = 0;
        __syncthreads();
        // 2. marks: append j to the hit list of (k, side)
        for (int t = tid; t < a.ntasks; t += blockDim.x) {
            const uint32_t tk = s_task[t];
            const int j = tk & 0x3FF, side = (tk >> 10) & 1;
            BNX_CHECK(j < np2);
            const uint32_t r = (tk >> 11) & 0x3FF, R = tk >> 21;
            const int32_t off = s_off[2 * j + side];
            if (off < 0) continue;
            const uint32_t p = s_p[j];
            for (uint32_t kk = (uint32_t)off + r * p; kk < (uint32_t)kn; kk += R * p) {
                if constexpr (MASK) {
                    atomicOr(&s_marks[(j >> 5) * kc + kk], 1u << (j & 31));
                } else {
                    const uint32_t li = (uint32_t)side * kc + kk;
                    const uint32_t sh = 8 * (li & 3);
                    const uint32_t slot = (atomicAdd(&hcnt[li >> 2], 1u << sh) >> sh) & 0xFF;
                    if (slot < HEAVY_HITS) hits[li * HEAVY_HITS + slot] = (uint16_t)j;
                }
            }
        }
        // 3. canonical k of the chunk
        for (int kk = tid; kk < kn; kk += blockDim.x) {
            const uint64_t k = k0 + (uint64_t)st * kk;
            if (k >= a.nkinfo) {
                a.flags[1] = 1;
                if (a.host_flags) a.host_flags[1] = 1;
                continue;
            }
            bool canon = (a.kinfo[k] & (e.rmask | 0x80000000u)) == 0;
            if (canon && e.rbig > 1 && k >= e.rbig_min) canon = gcd32((uint32_t)k, e.rbig) == 1;
            if (canon) {
                const int li = atomicAdd(&s_nl, 1);
                BNX_CHECK(li < kc);
                s_list[li] = (uint32_t)kk;
            }
        }
        __syncthreads();
        // 4. exact small factors of both sides, then the stage-1 test
        const int nl = s_nl;
        const uint64_t sigma = e.m * e.r;
        if constexpr (MASK) {
            const bool narrow = (k0 + (uint64_t)st * (uint64_t)(kn - 1)) * e.b + 1 < (1ull << 32);  // CTA-uniform
            for (int li = tid; li < nl; li += blockDim.x) {
                const uint32_t kk = s_list[li];
                const uint64_t k = k0 + (uint64_t)st * kk;
                const HeavyItem it{k * e.b, sigma, k * e.r};
                if (narrow)
                    y_tests_impl<true, true>(a, it, s_il, s_p, s_pd32, s_c32, s_marks + kk, kc);
                else
                    y_tests_impl<false, true>(a, it, s_il, s_p, s_pd32, s_c32, s_marks + kk, kc);
            }
        } else {
        for (int li = tid; li < nl; li += blockDim.x) {
            const uint32_t kk = s_list[li];
            const uint64_t k = k0 + (uint64_t)st * kk;
            const uint64_t x = k * e.b;
            const bool vL = x >= 2 && x - 1 >= a.n_first && x - 1 <= a.n_last;
            const bool vU = x >= a.n_first && x <= a.n_last;
            bool pL = false, pU = false;
            uint64_t cs[2] = {1, 1}, rs[2] = {1, 1};  // cofactor and radical of the divided-off part
#pragma unroll
            for (int side = 0; side < 2; ++side) {
                const bool valid = side ? vL : vU;
                if (!valid) continue;
                const uint64_t y = side ? x - 1 : x + 1;
                const int tz = __ffsll((long long)y) - 1;
                uint64_t c = y >> tz, sy = tz ? 1ull << (tz - 1) : 1ull, ry = tz ? 2 : 1;
                const uint32_t hl = (uint32_t)side * kc + kk;
                const uint32_t nh = (hcnt[hl >> 2] >> (8 * (hl & 3))) & 0xFF;
                if (nh <= (uint32_t)HEAVY_HITS) {
                    for (uint32_t h = 0; h < nh; ++h) {
                        const int j = hits[hl * HEAVY_HITS + h];
                        const ulonglong2 d = s_il[j];
                        c *= d.x;
                        ry *= s_p[j];
                        while (c * d.x <= d.y) { c *= d.x; sy *= s_p[j]; }
                    }
                } else {  // more distinct small primes than slots (rare): trial division
                    for (int j = 0; j < np2; ++j) {
                        const ulonglong2 d = s_il[j];
                        if (c * d.x <= d.y) {
                            c *= d.x;
                            ry *= s_p[j];
                            while (c * d.x <= d.y) { c *= d.x; sy *= s_p[j]; }
                        }
                    }
                }
                const bool pass = twice_prod_ge(sigma, sy * surplus_bound(c, a), side ? x : x + 1);
                if (side) pL = pass; else pU = pass;
                cs[side] = c;
                rs[side] = ry;
            }
            if (pL || pU) {
                const uint64_t radx = k * e.r;
                const unsigned long long slot = atomicAdd(&a.ctr[CTR_SURV], (unsigned long long)(pL + pU));
                if (pL && slot < a.q1_cap) a.q1[slot] = BnxSurv{(x - 1) | (1ull << 63), radx, cs[1], rs[1]};
                const unsigned long long s2 = slot + pL;
                if (pU && s2 < a.q1_cap) a.q1[s2] = BnxSurv{x, radx, cs[0], rs[0]};
                if (a.host_flags && slot + pL + pU > a.q1_cap) a.host_flags[2] = 1;
            }
        }
        }
    }
}

// A candidate goes to k_tail's list, or (more than TAIL_HEAVY residue-class members) to the
// queue of k_tail_heavy, which runs concurrently on a second stream; the residue-class
// counters are kept here (the member count as in k_tail).
__device__ __forceinline__ void emit_candidate(const HeavyArgs& a, const BnxCand c) {
    const uint64_t R = c.r0 * c.r1;
    const uint64_t t1 = (a.kinds & 1u) ? (c.n - 1) / R : 0;
    const uint64_t t0 = (c.n + 1) / R + 1, t2 = (2 * c.n) / R;
    const uint64_t total = t1 + (((a.kinds & 2u) && t2 >= t0) ? t2 - t0 + 1 : 0);
    atomicAdd(&a.ctr[CTR_CAND], 1ull);
    if (total) atomicAdd(&a.ctr[CTR_CHECKS], (unsigned long long)total);
    atomicMax(&a.ctr[CTR_MAXCHK], (unsigned long long)total);
    if (total > a.tail_heavy) {
        const unsigned long long h = atomicAdd(&a.ctr[CTR_HEAVY], 1ull);
        if (h < a.heavy_cap) a.heavy[h] = c;
        else if (a.host_flags) a.host_flags[2] = 1;
    } else {
        const unsigned long long slot = atomicAdd(&a.ctr[CTR_LIGHT], 1ull);
        if (slot < a.cand_cap) a.cand[slot] = c;
        else if (a.host_flags) a.host_flags[2] = 1;
    }
}

// Exact radical of the other side.  The survivor record carries y's cofactor c after the
// odd primes <= P2 (every prime factor of c exceeds P2, so c has at most three) and the
// radical `base` of the part divided off, so rad y = base * rad(c) and only the primes in
// (P2, cbrt c] can still matter.
//
// rad(c) of such a c by one thread: trial division by the odd primes from P2 up to
// cbrt(y_max) (32 at a time into a bit mask, unrolled with constant bit positions over the
// table padded to a multiple of 32), then at most two primes remain (p, p^2 or pq).
// NARROW: c < 2^32, everything in 32-bit arithmetic.
template <bool NARROW>
__device__ __forceinline__ uint64_t rad_cofactor_thread(uint64_t o, int j_first, int np3, const ulonglong2* s_il3,
                                                        const uint2* s_pd3, const uint32_t* s_p3, const uint32_t* s_e3,
                                                        bool nowrap = false, uint32_t top = 0xFFFFFFFFu) {
    using W = typename std::conditional<NARROW, uint32_t, uint64_t>::type;
    W c = (W)o, rad = 1;
    const uint32_t ol = (uint32_t)o, oh = (uint32_t)(o >> 32);
    // blocks up to the first prime above `top` (>= cbrt of every cofactor of the warp: beyond
    // it at most two prime factors remain, settled by the square test below)
    for (int j0 = j_first; j0 < np3 && s_p3[j0] <= top; j0 += 32) {
        const int jn = min(32, np3 - j0);
        uint32_t m = 0;
        if constexpr (NARROW) {
#pragma unroll
            for (int u = 0; u < 32; ++u) {
                const uint2 d = s_pd3[j0 + u];
                m |= (uint32_t)(ol * d.x <= d.y) << u;
            }
        } else if (nowrap) {  // W = ol + oh (2^32 mod p) < 2^32: W p^-1 = ol p^-1 + oh e (mod 2^32)
#pragma unroll
            for (int u = 0; u < 32; ++u) {
                const uint2 d = s_pd3[j0 + u];
                m |= (uint32_t)(ol * d.x + oh * s_e3[j0 + u] <= d.y) << u;
            }
        } else {  // o = oh 2^32 + ol: w = ol + oh (2^32 mod p) = o (mod p) in 32 bits (p, oh < 2^16)
#pragma unroll
            for (int u = 0; u < 32; ++u) {
                const uint2 d = s_pd3[j0 + u];
                const uint32_t cp = s_e3[j0 + u] * s_p3[j0 + u];  // (e p = 2^32 mod p)
                uint32_t w = ol + oh * cp;
                if (w < ol) w += cp;
                m |= (uint32_t)(w * d.x <= d.y) << u;
            }
        }
        if (jn < 32) m &= (1u << jn) - 1;
        while (m) {
            const int u = __ffs(m) - 1;
            m &= m - 1;
            W inv, lim;
            if constexpr (NARROW) {
                inv = s_pd3[j0 + u].x;
                lim = s_pd3[j0 + u].y;
            } else {
                inv = s_il3[j0 + u].x;
                lim = s_il3[j0 + u].y;
            }
            rad *= (W)s_p3[j0 + u];
            c *= inv;
            while (c * inv <= lim) c *= inv;
        }
    }
    uint64_t r = rad;
    if (c > 1) {  // at most two primes > cbrt(y) remain: c = p, p^2 or pq
        const uint64_t q = exact_sqrt(c);
        r *= q ? q : (uint64_t)c;
    }
    return r;
}

// First index i in [0, n) with sp[i] >= v (n if none), by the whole warp (warp-uniform v): 32
// probes per round narrow [lo, hi] 32-fold.
__device__ __forceinline__ int lower_bound_warp(const uint32_t* sp, int n, uint64_t v, int lane) {
    int lo = 0, hi = n;  // the answer lies in [lo, hi]
    while (hi - lo > 31) {
        const int span = hi - lo;
        const int q = lo + (int)((int64_t)span * (lane + 1) / 32);  // lane 31 probes hi
        const unsigned bal = __ballot_sync(0xFFFFFFFFu, q >= n || sp[q] >= v);
        const int j = __ffs(bal) - 1;
        const int nlo = j ? lo + (int)((int64_t)span * j / 32) + 1 : lo;
        hi = lo + (int)((int64_t)span * (j + 1) / 32);
        lo = nlo;
    }
    const int q = lo + lane;
    const unsigned bal = __ballot_sync(0xFFFFFFFFu, q >= hi || sp[q] >= v);
    return lo + __ffs(bal) - 1;
}

// Index of a prime in [i0, i1) dividing c (the first such block of 32, lowest lane), or -1:
// the warp tests 32 primes per step.
__device__ __forceinline__ int divisor_in_warp(uint64_t c, int i0, int i1, const ulonglong2* s_il3, const uint2* s_pd3,
                                               int lane) {
    const bool narrow = c < (1ull << 32);
    for (int b = i0; b < i1; b += 32) {
        const int j = b + lane;
        bool hit = false;
        if (j < i1) {
            if (narrow) {
                const uint2 d = s_pd3[j];
                hit = (uint32_t)c * d.x <= d.y;
            } else {
                const ulonglong2 d = s_il3[j];
                hit = c * d.x <= d.y;
            }
        }
        const unsigned bal = __ballot_sync(0xFFFFFFFFu, hit);
        if (bal) return b + __ffs(bal) - 1;
    }
    return -1;
}

// rad(c) from one prime divisor d = p_j of c (c has at most three prime factors, none of
// them a repeated d unless d^2 | c): d^2 | c -> c = d^2 q, rad = d q; else c / d is p^2
// (rad = d p) or squarefree (rad = c).
__device__ __forceinline__ uint64_t rad_from_divisor(uint64_t c, int j, const ulonglong2* s_il3, const uint32_t* s_p3) {
    const ulonglong2 dv = s_il3[j];
    const uint64_t d = s_p3[j], c1 = c * dv.x;
    if (c1 * dv.x <= dv.y) return d * (c1 * dv.x);
    const uint64_t q = exact_sqrt(c1);
    return q > 1 ? d * q : c;
}

// rad(c) by one warp, deciding only what the survivor needs (warp-uniform inputs):
// rad x * base * rad(c) <= 2n requires s(c) = c / rad(c) >= tau = c rad x base / (2n).  c is
// 1, p, pq, pqr (s = 1), p^2 (s = p), p^3 (s = p^2) or p^2 q (s = p), all primes > P2.
// Squares and cubes are found exactly; for tau > 1, p^2 q needs p >= t' = max(tau, p1), so
// either p < q, p in [t', cbrt c], or q < p, q in [p1, c / t'^2] -- the only primes tried
// (the tau bound is taken 1e-9 low, which only widens the ranges).  A c for which no prime
// in those ranges divides gets rad = c: squarefree, or p^2 q with p < tau -- rejected either
// way by the exact R <= 2n test that follows.  tau <= 1: every prime up to cbrt c.
__device__ uint64_t rad_cofactor_warp(uint64_t c, uint64_t radx, uint64_t base, uint64_t n, const HeavyArgs& a,
                                      int np2, int np3, const ulonglong2* s_il3, const uint2* s_pd3,
                                      const uint32_t* s_p3, int lane) {
    if (c == 1 || c < a.p1sq) return c;  // 1 or a prime
    if (const uint64_t q = exact_sqrt(c)) return q;
    const double cd = (double)c;
    if (c >= a.p1cube) {
        const uint64_t r = (uint64_t)llrint(cbrt(cd));
        if (r * r * r == c) return r;
    } else {
        return c;  // pq (a square was handled above)
    }
    const double tau = cd * (double)radx * (double)base / (2.0 * (double)n);
    const uint64_t top = (uint64_t)cbrt(cd) + 1;  // p < cbrt c (p < q) or q < cbrt c (q < p)
    const int i_top = lower_bound_warp(s_p3, np3, top + 1, lane);
    int j;
    if (tau <= 1.0 + 1e-6) {
        j = divisor_in_warp(c, np2, i_top, s_il3, s_pd3, lane);
    } else {
        const double tp = fmax(tau * (1.0 - 1e-9), (double)a.p1);
        if (tp * tp * (double)a.p1 > cd * (1.0 + 1e-9)) return c;  // no p >= t' with q = c / p^2 >= p1
        const double hb = cd / (tp * tp) * (1.0 + 1e-9) + 1.0;
        const uint64_t hiB = hb >= (double)top ? top : (uint64_t)hb;
        const int iB1 = lower_bound_warp(s_p3, np3, hiB + 1, lane);
        const int iA0 = tp >= (double)top ? i_top : lower_bound_warp(s_p3, np3, (uint64_t)tp, lane);
        if (iA0 <= iB1) {
            j = divisor_in_warp(c, np2, i_top, s_il3, s_pd3, lane);
        } else {
            j = divisor_in_warp(c, np2, iB1, s_il3, s_pd3, lane);
            if (j < 0) j = divisor_in_warp(c, iA0, i_top, s_il3, s_pd3, lane);
        }
    }
    return j < 0 ? c : rad_from_divisor(c, j, s_il3, s_p3);
}

__device__ __forceinline__ void exact_emit(const HeavyArgs& a, bool sideL, uint64_t n, uint64_t radx, uint64_t rady) {
    if (__umul64hi(radx, rady) != 0 || radx * rady > 2 * n) return;
    if (sideL) {  // keep from x = n + 1 only if n itself is not heavy
        const uint64_t y = n, sy = y / rady;
        if (__umul64hi(2 * sy, sy) != 0 || 2 * sy * sy >= y) return;
    }
    emit_candidate(a, sideL ? BnxCand{n, rady, radx} : BnxCand{n, radx, rady});
}

__global__ void __launch_bounds__(256) k_heavy_exact(HeavyArgs a) {
    // np3p (inv32, lim32) first (a fixed shared address: immediate offsets in the unrolled
    // loops), np3 (inv, lim), np3 p, np3p e = (2^32 mod p) p^-1 mod 2^32 (np3p: np3 padded to 32)
    extern __shared__ uint2 s_pd3[];
    const int np3 = (int)a.np3, np3p = (np3 + 31) & ~31;
    ulonglong2* s_il3 = reinterpret_cast<ulonglong2*>(s_pd3 + np3p);
    uint32_t* s_p3 = reinterpret_cast<uint32_t*>(s_il3 + np3);
    uint32_t* s_c3 = s_p3 + np3;
    for (int j = threadIdx.x; j < np3; j += blockDim.x) {
        s_il3[j] = make_ulonglong2(a.pdiv[j].inv, a.pdiv[j].lim);
        const uint4 q = a.pd32[j];
        s_pd3[j] = make_uint2(q.x, q.y);
        s_p3[j] = q.z;
        s_c3[j] = q.w * q.x;
    }
    for (int j = np3 + threadIdx.x; j < np3p; j += blockDim.x) {  // padding (its bits are masked off)
        s_pd3[j] = make_uint2(1u, 0u);
        s_c3[j] = 0u;
    }
    __syncthreads();
    const uint64_t pmax = np3 ? s_p3[np3 - 1] : 1;
    // launched as a programmatic dependent of k_heavy_screen: the tables above overlap its
    // last CTAs; the survivors are read only after it has completed (and flushed).  k_tail
    // (one-graph searches) may in turn be scheduled from here.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    const uint64_t nq = min((uint64_t)a.ctr[CTR_SURV], a.q1_cap);
    const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
    const int np2 = min(a.np2, np3);  // the cofactors hold no prime of index < np2
    if (a.exact_warp || nq * 32 <= nthreads) {
        // one warp per survivor, only the primes that can decide it (bounds above ~2^33, or
        // few survivors)
        const int lane = threadIdx.x & 31;
        for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < nq; i += nthreads >> 5) {
            const BnxSurv rec = a.q1[i];
            const bool sideL = rec.nside >> 63;
            const uint64_t n = rec.nside & ~(1ull << 63);
            const uint64_t radc = rad_cofactor_warp(rec.c, rec.radx, rec.base, n, a, np2, np3, s_il3, s_pd3, s_p3, lane);
            if (lane == 0) exact_emit(a, sideL, n, rec.radx, rec.base * radc);
        }
        return;
    }
    const int j_first = np2 & ~31;  // (a block boundary: the primes below np2 no longer divide)
    // Each CTA takes 256 survivors at a time and sorts them by the last prime they need (bins by powers of two, a
    // counting sort in shared memory), so that a warp's cofactors are alike: the 32-bit form
    // for whole warps below 2^32, and the trial division stops at the warp's largest cube root.
    __shared__ uint32_t s_srt[256];  // survivor indices (the records are re-read: L1/L2 hits)
    constexpr int NBIN = 18;  // by the bit length of the last prime needed (below 2^17)
    __shared__ int s_bcnt[NBIN], s_boff[NBIN];
    for (uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x; i0 < nq; i0 += nthreads) {
        const uint64_t i = i0 + threadIdx.x;
        const bool live = i < nq;
        BnxSurv rec = live ? a.q1[i] : BnxSurv{0, 1, 1, 1};
        uint32_t top = 0xFFFFFFFFu;
        // The last prime the trial division needs: cbrt(c) (beyond it at most two prime
        // factors remain); or, when the survivor can only pass through a p^2 q factor with
        // p >= tau' = max(tau, p1) > cbrt(c) (tau = c rad x base / 2n, as in
        // rad_cofactor_warp), only q <= c / tau'^2 -- a q found is divided off, a c left
        // unfactored is taken squarefree, which then fails the exact test as it must (cubes,
        // whose s = p^2 may pass, keep the full range).
        auto need_of = [&](const BnxSurv& r) -> uint32_t {
            const float cf = (float)r.c;
            const uint32_t t3 = (uint32_t)approx_cbrt(cf) + 2u;
            const uint64_t n = r.nside & ~(1ull << 63);
            const float tau = cf * (float)r.radx * (float)r.base / (2.0f * (float)n) * 0.9999f;
            const float tp = fmaxf(tau, (float)a.p1);
            if (tp <= (float)t3) return t3;
            const uint64_t cr = (uint64_t)rintf(approx_cbrt(cf));
            if (cr * cr * cr == r.c) return t3;
            const float hb = cf / (tp * tp) * 1.0001f + 2.0f;
            return hb < (float)t3 ? (uint32_t)hb : t3;
        };
        if (np3 > 128) {  // (short prime tables gain nothing from it)
            const uint32_t nd = need_of(rec);
            const int bin = min(NBIN - 1, 32 - __clz(nd));
            if (threadIdx.x < NBIN) s_bcnt[threadIdx.x] = 0;
            __syncthreads();
            const int pos = live ? atomicAdd(&s_bcnt[bin], 1) : 0;
            __syncthreads();
            if (threadIdx.x == 0) {
                int o = 0;
                for (int b = 0; b < NBIN; ++b) {
                    s_boff[b] = o;
                    o += s_bcnt[b];
                }
            }
            __syncthreads();
            if (live) s_srt[s_boff[bin] + pos] = (uint32_t)threadIdx.x;
            __syncthreads();
            rec = live ? a.q1[i0 + s_srt[threadIdx.x]] : BnxSurv{0, 1, 1, 1};  // (the live ones fill the front)
            top = __reduce_max_sync(0xFFFFFFFFu, need_of(rec));
            __syncthreads();  // (s_srt is refilled next round)
        }
        // 32-bit arithmetic when every cofactor of the warp fits (mixed warps would run both);
        // above, the one-step reduction when no cofactor of the warp can wrap
        const uint64_t radc =
            __all_sync(0xFFFFFFFFu, rec.c < (1ull << 32))
                ? rad_cofactor_thread<true>(rec.c, j_first, np3, s_il3, s_pd3, s_p3, s_c3, false, top)
                : rad_cofactor_thread<false>(rec.c, j_first, np3, s_il3, s_pd3, s_p3, s_c3,
                                             __all_sync(0xFFFFFFFFu, (rec.c & 0xFFFFFFFFull) + (rec.c >> 32) * pmax < (1ull << 32)),
                                             top);
        if (live) exact_emit(a, rec.nside >> 63, rec.nside & ~(1ull << 63), rec.radx, rec.base * radc);
    }
}

}  // namespace

__global__ void k_pdiv32(const BnxPDiv* __restrict__ pdiv, uint64_t n, uint4* __restrict__ out) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t p = (uint32_t)pdiv[j].p;
        out[j] = make_uint4((uint32_t)pdiv[j].inv, 0xFFFFFFFFu / p, p, (uint32_t)((1ull << 32) % p));
    }
}

bool heavy_sieve_mask(int np2) { return np2 <= 64; }

size_t heavy_sieve_smem(int np2, int kc, int ntasks) {
    const size_t common = (sizeof(ulonglong2) + 2 * sizeof(uint32_t) + 2 * sizeof(int32_t)) * np2 +
                          sizeof(uint32_t) * ((size_t)ntasks + kc);
    if (heavy_sieve_mask(np2))  // + (inv32, lim32) and 2^32 mod p over np2p, 2 mask words per k
        return common + (sizeof(uint2) + sizeof(uint32_t)) * (size_t)((np2 + 31) & ~31) + sizeof(uint32_t) * 2 * kc;
    return common + sizeof(uint16_t) * (size_t)2 * kc * HEAVY_HITS + (size_t)2 * kc;
}

// Dynamic shared memory limits of the heavy kernels, set once per device (outside any
// stream capture): the sieve's hit lists and the exact stage's prime table exceed 48 KB.
cudaError_t heavy_configure() {
    cudaError_t e = cudaFuncSetAttribute(k_heavy_sieve<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_heavy_sieve<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e == cudaSuccess) {  // (227 KB per block in all, its static shared memory included)
        cudaFuncAttributes fa;
        e = cudaFuncGetAttributes(&fa, k_heavy_exact);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(k_heavy_exact, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     227 * 1024 - (int)fa.sharedSizeBytes);
    }
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_heavy_screen<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_heavy_screen<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);

    cudaFuncAttributes at;  // (the attribute calls above load those three; see kernels_preload)
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&at, k_heavy_count);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&at, k_heavy_count_local);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&at, k_pdiv32);
    return e;
}

// The cub scan this file launches, run once on two elements (loads its kernels).
cudaError_t heavy_preload_cub(cudaStream_t st) {
    uint64_t* d = nullptr;
    void* tmp = nullptr;
    size_t bytes = 0;
    cub::DeviceScan::InclusiveSum(nullptr, bytes, d, d, (int64_t)2);
    cudaError_t e = cudaMallocAsync((void**)&d, 4 * sizeof(uint64_t) + bytes + 256, st);
    if (e != cudaSuccess) return e;
    tmp = (void*)(d + 4);
    cudaMemsetAsync(d, 0, 2 * sizeof(uint64_t), st);
    cub::DeviceScan::InclusiveSum(tmp, bytes, d, d + 2, (int64_t)2, st);
    e = cudaGetLastError();
    cudaFreeAsync(d, st);
    return e;
}

void launch_pdiv32(const BnxPDiv* pdiv, uint64_t n, uint4* out, cudaStream_t st) {
    if (n) k_pdiv32<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 1024), 256, 0, st>>>(pdiv, n, out);
}

size_t heavy_scan_temp_bytes(uint64_t nent) {
    size_t bytes = 0;
    cub::DeviceScan::InclusiveSum(nullptr, bytes, (const uint64_t*)nullptr, (uint64_t*)nullptr, (int64_t)nent);
    return bytes;
}

void launch_heavy(const HeavyArgs& a, void* scan_temp, size_t scan_temp_bytes, int grid, cudaStream_t st,
                  cudaEvent_t ev_generated, cudaStream_t aux, cudaEvent_t ev_fork, cudaEvent_t ev_join,
                  const cudaEvent_t* kev, int stop_after) {
    bool pdl = false;
    if (kev) cudaEventRecord(kev[0], st);
    if (a.nent) {
        if (a.ntiles) {
            k_heavy_count_local<<<a.ntiles, HEAVY_TILE, 0, st>>>(a);
        } else {
            const unsigned cb = (unsigned)std::min<uint64_t>((a.nent + 255) / 256, 4096);
            k_heavy_count<<<cb, 256, 0, st>>>(a);
            size_t bytes = scan_temp_bytes;
            cub::DeviceScan::InclusiveSum(scan_temp, bytes, a.cnt, a.incl, (int64_t)a.nent, st);
        }
        const bool sieve = a.kmin != ~0ull;
        if (sieve) {  // the sieve (shared-memory atomics) runs beside the trial screen (IMAD pipe)
            cudaEventRecord(ev_fork, st);
            cudaStreamWaitEvent(aux, ev_fork, 0);
            const size_t smemS = heavy_sieve_smem(a.np2, a.kc, a.ntasks);
            const int sgrid = a.sieve_ctas ? (int)a.sieve_ctas : grid;
            const int sthreads = a.sieve_threads ? (int)a.sieve_threads : 256;
            if (heavy_sieve_mask(a.np2))
                k_heavy_sieve<true><<<sgrid, sthreads, smemS, aux>>>(a);
            else
                k_heavy_sieve<false><<<sgrid, sthreads, smemS, aux>>>(a);
            cudaEventRecord(ev_join, aux);
        }
        const size_t np2p = (size_t)(a.np2 + 31) & ~(size_t)31;  // (see k_heavy_screen)
        const size_t smem2 = (size_t)a.np2 * (sizeof(ulonglong2) + sizeof(uint32_t)) +
                             np2p * (sizeof(uint2) + 2 * sizeof(uint32_t));
        if (kev) cudaEventRecord(kev[1], st);
        if (stop_after == 1) {
            if (kev) for (int i = 2; i < 4; ++i) cudaEventRecord(kev[i], st);
            return;
        }
        if (a.ntiles)
            k_heavy_screen<true><<<grid, HEAVY_THREADS, smem2 + sizeof(uint64_t) * (a.ntiles + 1), st>>>(a);
        else
            k_heavy_screen<false><<<grid, HEAVY_THREADS, smem2, st>>>(a);
        if (sieve) cudaStreamWaitEvent(st, ev_join, 0);
        pdl = !sieve && !kev;
    } else if (kev) {
        cudaEventRecord(kev[1], st);
    }
    if (kev) cudaEventRecord(kev[2], st);
    if (stop_after == 2) {
        if (kev) cudaEventRecord(kev[3], st);
        return;
    }
    const size_t np3p = (size_t)(a.np3 + 31) & ~(size_t)31;  // (see k_heavy_exact)
    const size_t smem3 = (size_t)a.np3 * (sizeof(ulonglong2) + sizeof(uint32_t)) + np3p * (sizeof(uint2) + sizeof(uint32_t));
    {  // a programmatic dependent launch right after k_heavy_screen (see k_heavy_exact)
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)grid);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = smem3;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = pdl ? 1 : 0;
        cudaLaunchKernelEx(&cfg, k_heavy_exact, a);
    }
    if (kev) cudaEventRecord(kev[3], st);
    if (ev_generated) cudaEventRecord(ev_generated, st);
}

}  // namespace bnx
