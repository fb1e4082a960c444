// bnx_math.cuh -- 64-bit integer helpers shared by the Benelux-pair kernels (sm_100a).
//
// No hardware u64 divide exists on the GPU, so the hot loops never divide:
//  * exact division by an odd prime p is a multiply by p^-1 mod 2^64 (Newton inverse);
//  * "p | x" for odd p is  x * p^-1 (mod 2^64) <= floor((2^64-1)/p);
//  * a residue a mod q uses a precomputed reciprocal floor((2^64-1)/q) and __umul64hi.
#pragma once
#include <stdint.h>

#define BNX_HD __host__ __device__ __forceinline__
#define BNX_D __device__ __forceinline__

// Device bounds checks of the checked build (make EXTRA=-DBNX_CHECKED; compute-sanitizer is
// not available on the GPU pool): a failed check prints its site and traps the kernel.
#ifdef BNX_CHECKED
#include <cstdio>
#define BNX_CHECK(c)                                                                           \
    do {                                                                                       \
        if (!(c)) {                                                                            \
            printf("BNX_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, \
                   (int)blockIdx.x, (int)threadIdx.x);                                         \
            __trap();                                                                          \
        }                                                                                      \
    } while (0)
#else
#define BNX_CHECK(c) \
    do {             \
    } while (0)
#endif

// Inverse of odd a modulo 2^64 (Newton: 3 -> 6 -> 12 -> 24 -> 48 -> 96 correct bits).
BNX_HD uint64_t bnx_inv64(uint64_t a) {
    uint64_t x = a;
    for (int i = 0; i < 5; ++i) x *= 2 - a * x;
    return x;
}

BNX_D int bnx_ctz64(uint64_t x) { return __ffsll((long long)x) - 1; }

// a mod q given recip = floor((2^64-1)/q); at most two corrections.
BNX_D uint64_t bnx_mod(uint64_t a, uint64_t q, uint64_t recip) {
    uint64_t t = __umul64hi(a, recip);
    uint64_t r = a - t * q;
    while (r >= q) r -= q;
    return r;
}

// Smallest o >= 0 with (base + o) % q == 0.
BNX_D uint64_t bnx_first_offset(uint64_t base, uint64_t q, uint64_t recip) {
    uint64_t r = bnx_mod(base, q, recip);
    return r ? q - r : 0;
}

BNX_D uint64_t bnx_gcd64(uint64_t a, uint64_t b) {
    if (a == 0) return b;
    if (b == 0) return a;
    int sh = bnx_ctz64(a | b);
    a >>= bnx_ctz64(a);
    do {
        b >>= bnx_ctz64(b);
        if (a > b) { uint64_t t = a; a = b; b = t; }
        b -= a;
    } while (b);
    return a << sh;
}

// u | r^inf, i.e. every prime of u divides r (rad(u) | r).  1 <= u < 2^63, r >= 1.
// Branch-free (the lanes of a warp stay converged): the twos first, then for the odd part
// u | r^64 (every odd prime exponent of u is below 64) by six Montgomery squarings mod u.
// Montgomery products carry a factor 2^-64, a unit mod odd u, so the result is 0 exactly
// when r^64 is; no conversion into or out of the Montgomery domain is needed.
BNX_D uint64_t bnx_redc(uint64_t hi, uint64_t lo, uint64_t u, uint64_t nu) {  // (hi:lo) 2^-64 mod u
    const uint64_t m = lo * nu;                                                 // nu = -u^-1 mod 2^64
    uint64_t t = hi + __umul64hi(m, u) + (lo != 0);                             // < 2u (hi:lo < u 2^64)
    return t >= u ? t - u : t;
}

BNX_D bool bnx_supported_by(uint64_t u, uint64_t r) {
    const int tz = __ffsll((long long)u) - 1;
    const bool twos_ok = tz == 0 || (r & 1) == 0;
    u >>= tz;
    const uint64_t nu = 0 - bnx_inv64(u);
    uint64_t x = bnx_redc(0, r, u, nu);  // r 2^-64 mod u (r < 2^64 <= u 2^64)
#pragma unroll
    for (int i = 0; i < 6; ++i) x = bnx_redc(__umul64hi(x, x), x * x, u, nu);
    return twos_ok && (u == 1 || x == 0);
}

// The same below 2^32 (u, r < 2^32): 32-bit Montgomery products, a quarter of the multiplies.
BNX_D uint32_t bnx_redc32(uint32_t hi, uint32_t lo, uint32_t u, uint32_t nu) {  // (hi:lo) 2^-32 mod u
    const uint32_t m = lo * nu;                                                 // nu = -u^-1 mod 2^32
    const uint64_t t = (uint64_t)hi + __umulhi(m, u) + (lo != 0);               // < 2u
    return (uint32_t)(t >= u ? t - u : t);
}

BNX_D bool bnx_supported_by32(uint32_t u, uint32_t r) {
    const int tz = __ffs(u) - 1;
    const bool twos_ok = tz == 0 || (r & 1) == 0;
    u >>= tz;
    uint32_t v = u;  // u^-1 mod 2^32 (3 correct bits, doubled by each step)
#pragma unroll
    for (int i = 0; i < 4; ++i) v *= 2u - u * v;
    const uint32_t nu = 0u - v;
    uint32_t x = bnx_redc32(0, r, u, nu);  // r 2^-32 mod u
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        const uint64_t s = (uint64_t)x * x;
        x = bnx_redc32((uint32_t)(s >> 32), (uint32_t)s, u, nu);
    }
    return twos_ok && (u == 1 || x == 0);
}

// floor(4 * log2(v)) for v >= 1, exact: 4e + #{k in 1..3 : mantissa >= 2^(k/4)}.
// The constants are ceil(2^(63 + k/4)), computed with integer roots.
BNX_D int bnx_floor4log2(uint64_t v) {
    int lz = __clzll((long long)v);
    uint64_t m = v << lz;
    int e = 63 - lz;
    return 4 * e + (m >= 0x9837f0518db8a970ull) + (m >= 0xb504f333f9de6485ull) + (m >= 0xd744fccad69d6af5ull);
}

// floor(2 * log2(v)) for v >= 1, exact (constant = ceil(2^63.5)).
BNX_D int bnx_floor2log2(uint64_t v) {
    int lz = __clzll((long long)v);
    uint64_t m = v << lz;
    return 2 * (63 - lz) + (m >= 0xb504f333f9de6485ull);
}

// A prime power progression q = p^e (e >= 2) of the sieve, with its reciprocal and the
// screen weight w = ceil(2 log2 p) (half-bits of log2 p, rounded up).
struct BnxProg {
    uint64_t q;
    uint64_t recip;
    uint32_t p;
    uint32_t w;
};

// An odd prime with its exact-division constants (trial division / verification).
struct BnxPDiv {
    uint64_t p;
    uint64_t inv;
    uint64_t lim;  // floor((2^64-1)/p)
};

// Candidate n with rad(n) * rad(n+1) <= 2n, and a signature match (m, n).
struct BnxCand {
    uint64_t n, r0, r1;
};
// A stage-1 survivor of the heavy generator: n with the side bit (63: y = n, else y = n + 1),
// rad x of the heavy side, and y's odd cofactor after the primes <= P2 with the radical of
// the part divided off (times 2 if y is even): rad y = base * rad(c).
struct BnxSurv {
    uint64_t nside, radx, c, base;
};
// One "surplus class" of the heavy-side generator (see bnx_heavy.cu): sigma = m * r with
// r = rad(sigma), b = sigma * r = m * r^2 (a powerful number); the heavy integers of the class
// are x = k * b with k squarefree, gcd(k, r) = 1 and k <= 2m.  rmask: which of the first 31
// primes (2..127) divide r; rbig: product of r's primes >= 131 (1 if none), rbig_min the least.
struct BnxHeavyEnt {
    uint64_t b, m;
    uint32_t r, rmask, rbig, rbig_min;
};
struct BnxMatch {
    uint64_t m, n;
    uint32_t kind, pad;
};
