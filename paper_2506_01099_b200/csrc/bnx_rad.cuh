// bnx_rad.cuh -- exact radicals by warp-cooperative trial division (shared by the tail of
// bnx_kernels.cu and the heavy-side generator of bnx_heavy.cu).
#pragma once
#include "bnx_math.cuh"

namespace bnx {

// ------------------------------------------------------------------------------------
// Exact rad(x) (x < 2^42) by warp-cooperative trial division over the odd-prime table up to
// cbrt(x) only: afterwards the cofactor c has at most two prime factors, all > cbrt(x), so
// c is 1, p, p^2 or p*q and rad(c) = isqrt(c) if c is a square, else c.  Each lane owns
// primes j = lane (mod 32), four loads in flight; the partial products of the primes and of
// the prime powers dividing x are multiplied across the warp.  Warp-collective.
__device__ __forceinline__ uint64_t rad_warp(uint64_t x, const BnxPDiv* __restrict__ pd, uint64_t npd) {
    const int lane = threadIdx.x & 31;
    const int tz = bnx_ctz64(x);
    const uint64_t y = x >> tz;
    uint64_t pr = 1, pp = 1;
    bool go = true;
    for (uint64_t j = lane; go && j < npd; j += 128) {
        BnxPDiv d[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint64_t jj = j + 32u * u;
            d[u] = jj < npd ? pd[jj] : BnxPDiv{1ull << 21, 0, 0};  // sentinel: p^3 = 2^63 > y
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (d[u].p * d[u].p * d[u].p > y) { go = false; break; }  // p <= 2^21: no overflow
            uint64_t t = y * d[u].inv;
            if (t <= d[u].lim) {
                pr *= d[u].p;
                pp *= d[u].p;
                while (t * d[u].inv <= d[u].lim) { t *= d[u].inv; pp *= d[u].p; }
            }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        pr *= __shfl_xor_sync(0xffffffffu, pr, o);
        pp *= __shfl_xor_sync(0xffffffffu, pp, o);
    }
    const uint64_t c = y * bnx_inv64(pp);  // exact: pp | y, both odd
    uint64_t rc = c;
    if (c > 1) {
        uint64_t s = (uint64_t)sqrt((double)c);
        while (s * s > c) --s;
        while ((s + 1) * (s + 1) <= c) ++s;
        if (s * s == c) rc = s;
    }
    return (tz ? 2ull : 1ull) * pr * rc;
}

// rad(x) and rad(x+1) in one warp-cooperative pass (same method as rad_warp): each lane
// tests its primes against both odd parts, so the two chains overlap.
__device__ __forceinline__ void rad2_warp(uint64_t x, const BnxPDiv* __restrict__ pd, uint64_t npd, uint64_t& rx, uint64_t& rx1) {
    const int lane = threadIdx.x & 31;
    const int tz0 = bnx_ctz64(x), tz1 = bnx_ctz64(x + 1);
    const uint64_t y0 = x >> tz0, y1 = (x + 1) >> tz1;
    const uint64_t ymax = y0 > y1 ? y0 : y1;
    uint64_t pr0 = 1, pp0 = 1, pr1 = 1, pp1 = 1;
    bool go = true;
    for (uint64_t j = lane; go && j < npd; j += 128) {
        BnxPDiv d[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint64_t jj = j + 32u * u;
            d[u] = jj < npd ? pd[jj] : BnxPDiv{1ull << 21, 0, 0};  // sentinel: p^3 = 2^63 > y
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (d[u].p * d[u].p * d[u].p > ymax) { go = false; break; }
            uint64_t t = y0 * d[u].inv;
            if (t <= d[u].lim) {
                pr0 *= d[u].p;
                pp0 *= d[u].p;
                while (t * d[u].inv <= d[u].lim) { t *= d[u].inv; pp0 *= d[u].p; }
            }
            t = y1 * d[u].inv;
            if (t <= d[u].lim) {
                pr1 *= d[u].p;
                pp1 *= d[u].p;
                while (t * d[u].inv <= d[u].lim) { t *= d[u].inv; pp1 *= d[u].p; }
            }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        pr0 *= __shfl_xor_sync(0xffffffffu, pr0, o);
        pp0 *= __shfl_xor_sync(0xffffffffu, pp0, o);
        pr1 *= __shfl_xor_sync(0xffffffffu, pr1, o);
        pp1 *= __shfl_xor_sync(0xffffffffu, pp1, o);
    }
    auto finish = [](uint64_t y, uint64_t pr, uint64_t pp, int tz) {
        const uint64_t c = y * bnx_inv64(pp);
        uint64_t rc = c;
        if (c > 1) {
            uint64_t sq = (uint64_t)sqrt((double)c);
            while (sq * sq > c) --sq;
            while ((sq + 1) * (sq + 1) <= c) ++sq;
            if (sq * sq == c) rc = sq;
        }
        return (tz ? 2ull : 1ull) * pr * rc;
    };
    rx = finish(y0, pr0, pp0, tz0);
    rx1 = finish(y1, pr1, pp1, tz1);
}

}  // namespace bnx
