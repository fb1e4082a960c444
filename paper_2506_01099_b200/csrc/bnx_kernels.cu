// bnx_kernels.cu -- sm_100a kernels of the B200-native Benelux-pair search.
//
// Hot path:
//   k_screen        on-chip segmented sieve of the half-bit log of the "surplus"
//                   s(x) = x / rad(x) over shared-memory tiles; flags every n whose
//                   signature could collide:  rad(n) * rad(n+1) <= 2n   (Lemma).
//                   Nothing per integer touches HBM.
//   k_verify        exact rad(n), rad(n+1) of each flagged n by warp-cooperative trial
//                   division; keeps n with rad(n) rad(n+1) <= 2n  (the "key" test).
//   k_enumerate     collision pass: every partner m of n lies on the residue class
//                   m = n - tR (first kind) or m = tR - n - 1 (second kind), R = rad(n)rad(n+1);
//                   each is checked exactly with gcds (rad(m) == r  <=>  r | m and m/r | r^inf).
//   k_finalize      exact verification of each match by full radical comparison and the
//                   reference's classification (signatures.py:67-81).
// Also: k_sieve_exact (rad(x) materialised, radical.py:109-124), k_trial_division
// (_kernels.py:87-112) and the prime-table kernels (primes.py:24-35).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <type_traits>

#include "bnx_kernels.cuh"
#include "bnx_math.cuh"
#include "bnx_rad.cuh"

namespace bnx {

// ------------------------------------------------------------------------------------
// Block-wide exclusive scan of one uint32 per thread (blockDim.x multiple of 32, <= 1024).
__device__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp, uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < nw ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        s_warp[lane] = w;
    }
    __syncthreads();
    uint32_t base = warp ? s_warp[warp - 1] : 0;
    *total = s_warp[nw - 1];
    __syncthreads();
    return base + x - v;
}

// ------------------------------------------------------------------------------------
// Prime tables (primes.py:24-35).  Base primes <= ls (ls <= 65536) by one block.
__global__ void k_base_primes(uint32_t ls, uint32_t* out, uint32_t* count) {
    extern __shared__ uint8_t comp[];
    __shared__ uint32_t s_warp[32];
    for (uint32_t i = threadIdx.x; i <= ls; i += blockDim.x) comp[i] = (i < 2);
    __syncthreads();
    for (uint32_t d = 2; d * d <= ls; ++d) {
        if (!comp[d])
            for (uint32_t k = d * d + threadIdx.x * d; k <= ls; k += blockDim.x * d) comp[k] = 1;
        __syncthreads();
    }
    uint32_t per = (ls + 1 + blockDim.x - 1) / blockDim.x;
    uint32_t b = threadIdx.x * per, e = min(b + per, ls + 1);
    uint32_t c = 0;
    for (uint32_t i = b; i < e; ++i) c += !comp[i];
    uint32_t total;
    uint32_t off = block_excl_scan(c, s_warp, &total);
    for (uint32_t i = b; i < e; ++i)
        if (!comp[i]) out[off++] = i;
    if (threadIdx.x == 0) *count = total;
}

// Segmented Eratosthenes over [lo, hi] in blocks of SEGP numbers, sieving with base
// primes (ascending, covering isqrt(hi)).  Pass 1 (offsets == nullptr) writes per-block
// counts; pass 2 writes the primes at the scanned offsets.
constexpr uint32_t SEGP = 32768;
__global__ void __launch_bounds__(1024) k_prime_seg(uint64_t lo, uint64_t hi, const uint32_t* base, uint32_t nbase,
                                                    uint32_t* counts, const uint64_t* offsets, uint32_t* out) {
    __shared__ uint8_t flag[SEGP];
    __shared__ uint32_t s_warp[32];
    const uint64_t s0 = lo + (uint64_t)blockIdx.x * SEGP;
    const uint32_t len = (uint32_t)min((uint64_t)SEGP, hi - s0 + 1);
    for (uint32_t i = threadIdx.x; i < SEGP; i += blockDim.x) flag[i] = (i < len) && (s0 + i >= 2);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint64_t last = s0 + len - 1;
    for (uint32_t j = warp; j < nbase; j += nw) {
        uint64_t p = base[j];
        if (p * p > last) break;
        uint64_t first = p * p;
        if (first < s0) first = (s0 + p - 1) / p * p;
        for (uint64_t k = first - s0 + lane * p; k < len; k += 32 * p) flag[k] = 0;
    }
    __syncthreads();
    const uint32_t per = SEGP / blockDim.x;
    const uint32_t b = threadIdx.x * per;
    uint32_t c = 0;
    for (uint32_t i = 0; i < per; ++i) c += flag[b + i];
    uint32_t total;
    uint32_t off = block_excl_scan(c, s_warp, &total);
    if (offsets == nullptr) {
        if (threadIdx.x == 0) counts[blockIdx.x] = total;
    } else {
        uint64_t o = offsets[blockIdx.x] + off;
        for (uint32_t i = 0; i < per; ++i)
            if (flag[b + i]) out[o++] = (uint32_t)(s0 + b + i);
    }
}

// Exclusive scan of n uint32 counts into uint64 offsets (+ total at offsets[n]); one block.
__global__ void k_scan_counts(const uint32_t* counts, uint64_t n, uint64_t base, uint64_t* offsets) {
    __shared__ uint32_t s_warp[32];
    __shared__ uint64_t carry;
    if (threadIdx.x == 0) carry = base;
    __syncthreads();
    for (uint64_t s = 0; s < n; s += blockDim.x) {
        uint64_t i = s + threadIdx.x;
        uint32_t v = i < n ? counts[i] : 0;
        uint32_t total;
        uint32_t ex = block_excl_scan(v, s_warp, &total);
        uint64_t c = carry;
        if (i < n) offsets[i] = c + ex;
        __syncthreads();
        if (threadIdx.x == 0) carry = c + total;
        __syncthreads();
    }
    if (threadIdx.x == 0) offsets[n] = carry;
}

// u64 host primes -> u32 device primes (values < 2^32 by construction).
__global__ void k_narrow_primes(const uint64_t* in, uint64_t n, uint32_t* out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = (uint32_t)in[i];
}
__global__ void k_widen_primes(const uint32_t* in, uint64_t n, uint64_t* out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = in[i];
}

// ------------------------------------------------------------------------------------
// Progression tables: every q = p^e <= max_x, e >= 2 (odd p; p = 2 too when include_two),
// split at `tile` into the per-tile list (q < tile) and the bucketed list.  Order inside a
// list is irrelevant: hits commute.  Also the odd-prime exact-division table.
// Screen weight of an odd prime: half-bits of log2 p rounded up (an over-estimate is safe:
// the screen only needs A(x) >= 2 log2 s(x)).
__device__ uint32_t prime_weight(uint32_t p) {
    if (p == 2) return 2;
    return (uint32_t)ceil(2.0 * log2((double)p) + 1e-7);
}

__global__ void k_build_tables(const uint32_t* primes, uint64_t np, uint64_t max_x, int include_two, uint32_t tile,
                               BnxProg* small, uint32_t* nsmall, uint32_t small_cap, BnxProg* large,
                               unsigned long long* nlarge, uint64_t large_cap, BnxPDiv* pdiv, uint64_t* npdiv,
                               int* overflow) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < np; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t p = primes[i];
        if (p * p > max_x) continue;
        if (p != 2) {
            // pdiv is indexed like the odd primes, so it stays ascending.
            uint64_t slot = (primes[0] == 2) ? i - 1 : i;
            pdiv[slot] = BnxPDiv{p, bnx_inv64(p), ~0ull / p};
            atomicMax((unsigned long long*)npdiv, (unsigned long long)(slot + 1));
        }
        if (p == 2 && !include_two) continue;
        const uint32_t w = prime_weight((uint32_t)p);
        uint64_t q = p * p;
        for (;;) {
            BnxProg e{q, ~0ull / q, (uint32_t)p, w};
            if (q < tile) {
                uint32_t k = atomicAdd(nsmall, 1u);
                if (k < small_cap) small[k] = e; else *overflow = 1;
            } else {
                unsigned long long k = atomicAdd(nlarge, 1ull);
                if (k < large_cap) large[k] = e; else *overflow = 1;
            }
            if (q > max_x / p) break;
            q *= p;
        }
    }
}

// ------------------------------------------------------------------------------------
// THE SCREEN.  One CTA owns a segment of NT tiles of TILE integers.  Per tile it builds,
// in shared memory, one byte per integer:
//     A(x) = sum over prime powers p^e | x (e >= 2) of w_p,   w_p = ceil(2 log2 p) >= 2 log2 p
// (half-bits of log2 s(x), s(x) = x / rad(x), rounded up; p = 2 is exact).  The bytes start
// from the 2-adic part (written by the tile initialisation) and odd prime powers add in
// with 32-bit shared atomics:
//   * q = p^e < 2048: "work items" of up to ITEM_HITS hits each (a progression with many
//     hits per tile is split into R interleaved items), dealt to the warps in decreasing
//     size so every warp carries the same load into the barrier.  A lane's stride 32*R*q is
//     a multiple of 4, so its byte lane (and the shifted weight) never changes: the inner
//     loop is one add, one shared atomic, one compare.
//   * 2048 <= q < TILE: one lane per progression (items of 32 progressions, sorted by q).
//   * q >= TILE: at most one hit per tile: enumerated once per segment into per-tile
//     shared-memory buckets and applied block-wide.
// Since rad(n)rad(n+1) <= 2n  <=>  s(n)s(n+1) >= (n+1)/2, every pair candidate satisfies
//     A(n) + A(n+1) >= 2 log2(n+1) - 2 >= floor(2 log2(n+1)) - 2,
// tested four integers per 32-bit word (SWAR; A(x) <= 108 < 128 so byte sums never carry),
// after a one-AND pre-test on the high bits of the pair sums of 16 integers.
template <int TILE, int NT, int THREADS, int BCAP, int MAXS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) k_screen(ScreenArgs a) {
    constexpr int NW = THREADS / 32;
    constexpr int WORDS = TILE / 4;
    constexpr int GROUPS = WORDS / 4;  // 16 integers each
    constexpr int GPT = GROUPS / THREADS;
    static_assert(GROUPS % THREADS == 0, "scan: whole groups per thread");
    static_assert((WORDS & (WORDS - 1)) == 0, "geometry");
    extern __shared__ __align__(16) uint32_t smem[];
    uint32_t* acc = smem;                    // WORDS + 4 (the tile, then the next tile's first word group)
    uint32_t* bcnt = acc + WORDS + 4;        // NT
    uint32_t* bent = bcnt + NT;              // NT * BCAP: (loc | w << 17)
    uint32_t* s_q = bent + NT * BCAP;        // MAXS, ascending q
    uint32_t* s_w = s_q + MAXS;
    uint32_t* s_tm = s_w + MAXS;
    uint32_t* s_off = s_tm + MAXS;
    uint32_t* s_item = s_off + MAXS;         // 2*MAXS items: j | r << 8 | R << 16 | lanepacked << 31
    uint64_t* s_rc = (uint64_t*)(s_item + 2 * MAXS);  // MAXS reciprocals

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nsmall = a.nsmall;
    // per-tile progressions (sorted by q on the host) and their work items (build_tables)
    for (int j = tid; j < nsmall; j += THREADS) {
        const BnxProg pr = a.small[j];
        s_q[j] = (uint32_t)pr.q;
        s_w[j] = pr.w;
        s_rc[j] = pr.recip;
        s_tm[j] = (uint32_t)TILE % (uint32_t)pr.q;
    }
    for (int j = tid; j < a.nitems; j += THREADS) s_item[j] = a.items[j];
    __syncthreads();
    // 2-adic half-bits 2(v2(x) - 1) of x = tile0 + 4j for the first word of each of this
    // thread's groups (j = 4i, i = tid + k*THREADS): tile0 is a multiple of TILE > 4j, so
    // v2(x) = 2 + v2(j) and the value is 2*ffs(j), the same for every k unless tid == 0.
    const uint32_t c_grp = 2u * (uint32_t)__ffs(4 * (tid ? tid : THREADS));

    // Each CTA owns an equal contiguous run of tiles (to within one), processed in segments of
    // up to NT tiles: the grid finishes together whatever the bound.
    const uint64_t t_begin = a.ntiles * blockIdx.x / gridDim.x, t_end = a.ntiles * (blockIdx.x + 1) / gridDim.x;
    for (uint64_t st = t_begin; st < t_end; st += NT) {
        const int nt = (int)min((uint64_t)NT, t_end - st);
        const uint32_t seg_len = (uint32_t)nt * TILE;
        const uint64_t seg0 = a.x_begin + st * TILE;
        __syncthreads();
        for (int j = tid; j < NT; j += THREADS) bcnt[j] = 0;
        for (int j = tid; j < nsmall; j += THREADS) {
            uint64_t o = bnx_first_offset(seg0, s_q[j], s_rc[j]);
            if (seg0 == 0 && o == 0) o = s_q[j];  // never sieve x = 0
            s_off[j] = (uint32_t)o;
        }
        __syncthreads();
        for (int j = (a.skip & 16) ? a.nlarge : tid; j < a.nlarge; j += THREADS) {
            const BnxProg pr = a.large[j];
            uint64_t o = bnx_first_offset(seg0, pr.q, pr.recip);
            if (seg0 == 0 && o == 0) o = pr.q;
            for (; o < seg_len + 4; o += pr.q) {
                const uint32_t t = (uint32_t)(o / TILE), loc = (uint32_t)(o % TILE);
                const uint32_t ent = pr.w << 17;  // loc needs 17 bits: TILE + 4 > 2^16
                if (t < (uint32_t)nt) {
                    uint32_t k = atomicAdd(&bcnt[t], 1u);
                    if (k < BCAP) bent[t * BCAP + k] = loc | ent; else a.flags[0] = 1;
                }
                if (loc < 4 && t > 0) {
                    uint32_t k = atomicAdd(&bcnt[t - 1], 1u);
                    if (k < BCAP) bent[(t - 1) * BCAP + k] = (loc + TILE) | ent; else a.flags[0] = 1;
                }
            }
        }
        __syncthreads();

        for (int t = 0; t < nt; ++t) {
            const uint64_t tile0 = seg0 + (uint64_t)t * TILE;
            if (tile0 > a.n_last) break;
            // ---- init with the 2-adic part
            uint4* acc4 = reinterpret_cast<uint4*>(acc);
            if (!(a.skip & 8)) {
#pragma unroll
            for (int k = 0; k < GPT; ++k) acc4[tid + k * THREADS] = make_uint4(c_grp, 2u, 4u, 2u);
            }
            if (tid == 0) {
#pragma unroll
                for (int k = 0; k < GPT; ++k)
                    acc4[k * THREADS].x = k ? 2u * (uint32_t)__ffs(4 * k * THREADS)
                                            : (tile0 ? 2u * (uint32_t)(bnx_ctz64(tile0) - 1) : 0u);
                acc4[GROUPS] = make_uint4(2u * (uint32_t)(bnx_ctz64(tile0 + TILE) - 1), 2u, 4u, 2u);
            }
            __syncthreads();
            // ---- progressions q < TILE: balanced work items
            const int it_end = (a.skip & 1) ? 0 : (int)s_item[warp + 1];
            for (int it = (int)s_item[warp]; it < it_end; ++it) {  // this warp's items (host LPT deal)
                const uint32_t e = s_item[NW + 1 + it];
                const int j = (int)(e & 0xFFu);
                if (e >> 31) {  // lane-packed: one progression per lane
                    const int jj = j + lane;
                    if (jj < nsmall) {
                        const uint32_t q = s_q[jj], w = s_w[jj];
                        for (uint32_t o = s_off[jj]; o < TILE + 4; o += q) atomicAdd(&acc[o >> 2], w << ((o & 3) << 3));
                    }
                } else {
                    const uint32_t r = (e >> 8) & 0xFFu, R = (e >> 16) & 0x7FFFu;
                    const uint32_t q = s_q[j];
                    const uint32_t o = s_off[j] + (r * 32u + (uint32_t)lane) * q;
                    if (o < TILE + 4) {
                        const uint32_t wsh = s_w[j] << ((o & 3) << 3);     // invariant: stride % 4 == 0
                        const uint32_t step = (32u * R * q) >> 2;            // words
                        const uint32_t lim = (TILE + 4 - (o & 3) + 3) >> 2;  // word bound for this byte lane
                        uint32_t wd = o >> 2;
                        for (; wd + step < lim; wd += 2 * step) {
                            atomicAdd(&acc[wd], wsh);
                            atomicAdd(&acc[wd + step], wsh);
                        }
                        if (wd < lim) atomicAdd(&acc[wd], wsh);
                    }
                }
            }
            // ---- q >= TILE: this tile's bucket
            {
                const uint32_t nb = (a.skip & 2) ? 0u : min(bcnt[t], (uint32_t)BCAP);
                for (uint32_t i = tid; i < nb; i += THREADS) {
                    const uint32_t e = bent[t * BCAP + i];
                    const uint32_t loc = e & 0x1FFFFu;
                    atomicAdd(&acc[loc >> 2], (e >> 17) << ((loc & 3) << 3));
                }
            }
            __syncthreads();
            for (int j = tid; j < nsmall; j += THREADS) {
                int no = (int)s_off[j] - (int)s_tm[j];
                if (no < 0) no += (int)s_q[j];
                s_off[j] = (uint32_t)no;
            }
            // ---- scan: pair sums of 16 integers, exact SWAR byte compare against the tile
            // threshold (A(x) <= 108, so no byte carries); a divergent branch only on a hit
            const bool low = tile0 < (1u << 20);
            const uint32_t tt = (uint32_t)max(0, bnx_floor2log2(tile0 + 1) - 2);
#pragma unroll
            for (int k = 0; k < ((a.skip & 4) ? 0 : GPT); ++k) {
                const int i = tid + k * THREADS;
                const uint4 v = reinterpret_cast<const uint4*>(acc)[i];
                uint32_t nx = __shfl_down_sync(0xffffffffu, v.x, 1);  // next group's first word
                if (lane == 31) nx = acc[4 * i + 4];
                const uint64_t g0 = tile0 + 16u * (uint32_t)i;
                const uint32_t tw = low ? (uint32_t)max(0, bnx_floor2log2(g0 + 1) - 2) : tt;
                const uint32_t T4 = tw * 0x01010101u;
                uint32_t sv[4];
                sv[0] = v.x + __funnelshift_r(v.x, v.y, 8);  // A(x) + A(x+1), 4 bytes
                sv[1] = v.y + __funnelshift_r(v.y, v.z, 8);
                sv[2] = v.z + __funnelshift_r(v.z, v.w, 8);
                sv[3] = v.w + __funnelshift_r(v.w, nx, 8);
                // byte b passes iff bit 7 of ((s | 0x80) - T) | s is set; OR the four words
                // first and mask once (the other bits are don't-care)
                uint32_t any = 0;
#pragma unroll
                for (int w = 0; w < 4; ++w) any |= ((sv[w] | 0x80808080u) - T4) | sv[w];
                if (any & 0x80808080u) {
#pragma unroll
                    for (int w = 0; w < 4; ++w) {
                        uint32_t m = (((sv[w] | 0x80808080u) - T4) | sv[w]) & 0x80808080u;
                        while (m) {
                            const int b = (__ffs(m) - 1) >> 3;
                            m &= m - 1;
                            const uint64_t n = g0 + 4u * w + b;
                            if (n >= a.n_first && n <= a.n_last) {
                                unsigned long long slot = atomicAdd(&a.ctr[0], 1ull);
                                if (slot < a.surv_cap) a.surv[slot] = n;
                            }
                        }
                    }
                }
            }
            __syncthreads();
        }
    }
}

// The tail of the search, one warp per screen survivor n:
//  1. key:  exact r0 = rad(n), r1 = rad(n+1); n is a candidate iff R = r0 r1 <= 2n.
//  2. collision pass on the residue classes.  For a pair m < n with S_m = S_n,
//       first kind:  rad(n), rad(n+1) both divide n - m      ->  m = n - tR      (t >= 1)
//       second kind: rad(n), rad(n+1) both divide n + m + 1  ->  m = tR - n - 1
//     so the lanes walk those t; m is kept iff rad(m), rad(m+1) equal the required
//     radicals, tested exactly: rad(m) == r  <=>  r | m  and  m / r | r^inf (gcds).
//  3. every kept m is classified as the reference does (signatures.py:67-81) and emitted:
//     the two tests fix rad(m) and rad(m+1) exactly, so no radical is recomputed.
// One candidate n (R = r0 r1 <= 2n) and a range [k_begin, k_end) of its residue-class members:
// k < t1 -> first kind m = n - (k+1) R; else second kind m = (t0 + k - t1) R - n - 1.  With
// s0 = n / r0 and s1 = (n+1) / r1 the cofactors are linear in t, so no division is needed:
//   first kind   m / r0 = s0 - t r1,   (m+1) / r1 = s1 - t r0
//   second kind  m / r1 = t r0 - s1,   (m+1) / r0 = t r1 - s0
// and m is kept iff both cofactors are supported by their radical (u | r^inf), which makes
// rad(m) and rad(m+1) the required radicals exactly (signatures.py:67-81 classifies).
// Warp-collective.
struct TailCand {
    uint64_t n, r0, r1, R, s0, s1, t0, t1;
};

// n < 2^32 (n + 1 <= 2^32): every cofactor is below 2^32 (the products t r1, t r0 of the
// second kind too: t r0 = m / r1 + s1 < 2 (n + 1) / r1 <= 2^32 with r1 >= 2), so they are
// formed mod 2^32 and tested with 32-bit Montgomery products; m itself (t R can pass 2^32) in
// 64 bits.  The quotients of n + 1 (which may be 2^32) come from those of n: r1 | n + 1
// gives (n + 1) / r1 = n / r1 + 1, and (n + 1) / R = q + [r + 1 = R] for n = q R + r.
__device__ __forceinline__ TailCand tail_cand(uint64_t n, uint64_t r0, uint64_t r1, unsigned kinds) {
    TailCand c;
    c.n = n; c.r0 = r0; c.r1 = r1; c.R = r0 * r1;
    if (n < (1ull << 32)) {
        const uint32_t n32 = (uint32_t)n;
        c.s0 = n32 / (uint32_t)r0;
        c.s1 = n32 / (uint32_t)r1 + 1u;
        if (c.R >> 32) {  // R >= 2^32 >= n + 1
            c.t1 = 0;
            c.t0 = (n + 1 == c.R) + 1;
        } else {
            const uint32_t R32 = (uint32_t)c.R, q = n32 / R32, r = n32 - q * R32;
            c.t1 = (kinds & 1u) ? (n32 - 1u) / R32 : 0;
            c.t0 = (uint64_t)q + (r + 1u == R32) + 1;
        }
    } else {
        c.s0 = n / r0; c.s1 = (n + 1) / r1;
        c.t1 = (kinds & 1u) ? (n - 1) / c.R : 0;          // m = n - tR >= 1
        c.t0 = (n + 1) / c.R + 1;                          // n + 2 <= tR <= 2n
    }
    return c;
}
__device__ __forceinline__ uint64_t tail_total(const TailCand& c, unsigned kinds) {
    // second kind: t0 <= t <= floor(2n / R)
    uint64_t t2;
    const bool narrow = c.n < (1ull << 32);
    if (narrow && (c.R >> 32)) {  // R > n: the quotient is 0 or 1
        t2 = 2 * c.n >= c.R;
    } else if (narrow) {  // floor(2n / R) = 2q + [2 (n mod R) >= R], q = n / R
        const uint32_t n32 = (uint32_t)c.n, R32 = (uint32_t)c.R, q = n32 / R32;
        t2 = 2ull * q + (2ull * (n32 - q * R32) >= R32);
    } else {
        t2 = (2 * c.n) / c.R;
    }
    return c.t1 + (((kinds & 2u) && t2 >= c.t0) ? t2 - c.t0 + 1 : 0);
}

__device__ void tail_members(const TailArgs& a, const TailCand& c, uint64_t k_begin, uint64_t k_end) {
    const int lane = threadIdx.x & 31;
    const bool narrow = c.n < (1ull << 32);
    for (uint64_t base = k_begin; base < k_end; base += 32) {
        const uint64_t k = base + lane;
        uint64_t m = 0;
        bool ok = false;
        if (k < k_end && narrow) {
            const uint32_t r0 = (uint32_t)c.r0, r1 = (uint32_t)c.r1, s0 = (uint32_t)c.s0, s1 = (uint32_t)c.s1;
            if (k < c.t1) {
                const uint32_t t = (uint32_t)k + 1u;
                m = c.n - (uint64_t)t * c.R;
                ok = bnx_supported_by32(s0 - t * r1, r0) && bnx_supported_by32(s1 - t * r0, r1);
            } else {
                const uint32_t t = (uint32_t)(c.t0 + (k - c.t1));
                m = (uint64_t)t * c.R - c.n - 1;
                ok = bnx_supported_by32(t * r0 - s1, r1) && bnx_supported_by32(t * r1 - s0, r0);
            }
        } else if (k < k_end) {
            if (k < c.t1) {
                const uint64_t t = k + 1;
                m = c.n - t * c.R;
                ok = bnx_supported_by(c.s0 - t * c.r1, c.r0) && bnx_supported_by(c.s1 - t * c.r0, c.r1);
            } else {
                const uint64_t t = c.t0 + (k - c.t1);
                m = t * c.R - c.n - 1;
                ok = bnx_supported_by(t * c.r0 - c.s1, c.r1) && bnx_supported_by(t * c.r1 - c.s0, c.r0);
            }
        }
        // A kept m has its radicals exactly: r0 | m (m = n - tR) and m / r0 | r0^inf give
        // rad(m) = r0 (r0 squarefree), and likewise for m + 1 and for the second kind.
        if (ok) {
            const int kind = k < c.t1 ? 1 : 2;
            atomicAdd(&a.ctr[CTR_MATCH], 1ull);
            if ((a.kinds & (1u << (kind - 1))) && m >= 1 && m < c.n) {
                const unsigned long long s = atomicAdd(&a.ctr[CTR_PAIRS], 1ull);
                const bnx_pair_t row =
                    kind == 1 ? bnx_pair_t{m, c.n, c.r0, c.r1, 1, 0} : bnx_pair_t{m, c.n, c.r1, c.r0, 2, 0};
                if (s < a.pair_cap) a.pairs[s] = row;
                if (a.host_pairs) {
                    if (s < a.host_prefix) a.host_pairs[s] = row;
                    else a.host_flags[3] = 1;
                    if (s >= a.pair_cap) a.host_flags[2] = 1;
                }
            }
        }
    }
}

__global__ void __launch_bounds__(256) k_tail(TailArgs a) {
    // (a programmatic dependent launch: wait for the producer grid's completion and flush;
    // a no-op for an ordinary launch)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int lane = threadIdx.x & 31;
    const uint64_t cnt = a.cands ? min((uint64_t)a.ctr[CTR_LIGHT], a.cand_cap)
                                 : min((uint64_t)a.ctr[CTR_SURV], a.surv_cap);
    // the first round is static (warp w takes item w: no contended atomic when the grid has a
    // warp per item), later items come one at a time from a shared counter
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    uint64_t first = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    for (;;) {
        unsigned long long i = first;
        if (first == ~0ull) {
            if (nwarps >= cnt) break;  // the static round covered every item
            if (lane == 0) i = nwarps + atomicAdd(&a.ctr[CTR_NEXT], 1ull);
            i = __shfl_sync(0xffffffffu, i, 0);
        }
        first = ~0ull;
        if (i >= cnt) break;
        uint64_t n, r0, r1;
        if (a.cands) {  // heavy engine: radicals known exactly, R <= 2n already checked
            const BnxCand cc = a.cands[i];
            n = cc.n; r0 = cc.r0; r1 = cc.r1;
        } else {
            n = a.surv[i];
            rad2_warp(n, a.pdiv, a.npdiv, r0, r1);
            if (__umul64hi(r0, r1) != 0 || r0 * r1 > 2 * n) continue;  // warp-uniform
        }
        const TailCand c = tail_cand(n, r0, r1, a.kinds);
        const uint64_t total = tail_total(c, a.kinds);
        if (lane == 0 && !a.cands) {  // (heavy engine: counted and routed by k_heavy_exact)
            atomicAdd(&a.ctr[CTR_CAND], 1ull);
            if (total) atomicAdd(&a.ctr[CTR_CHECKS], (unsigned long long)total);
            atomicMax(&a.ctr[CTR_MAXCHK], (unsigned long long)total);
        }
        if (total > TAIL_HEAVY && !a.cands) {
            bool queued = false;
            if (lane == 0) {
                const unsigned long long h = atomicAdd(&a.ctr[CTR_HEAVY], 1ull);
                if (h < a.heavy_cap) {
                    a.heavy[h] = BnxCand{n, r0, r1};
                    queued = true;
                }
            }
            if (__shfl_sync(0xffffffffu, (int)queued, 0)) continue;
        }
        tail_members(a, c, 0, total);
    }
}

// Heavy candidates: blockIdx.y picks the candidate (strided over the list), the warps of the
// x-blocks split its members into chunks of 32.
__global__ void __launch_bounds__(256) k_tail_heavy(TailArgs a) {
    const uint64_t nh = min((uint64_t)a.ctr[CTR_HEAVY], a.heavy_cap);
    for (uint64_t y = blockIdx.y; y < nh; y += gridDim.y) {
        const BnxCand h = a.heavy[y];
        const TailCand c = tail_cand(h.n, h.r0, h.r1, a.kinds);
        const uint64_t total = tail_total(c, a.kinds);
        const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x >> 5);
        for (uint64_t chunk = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); chunk * 32 < total;
             chunk += nwarps)
            tail_members(a, c, chunk * 32, min(total, chunk * 32 + 32));
    }
}

// ------------------------------------------------------------------------------------
// rad(x) materialised (radical.py:109-124 / _kernels.py:48-84): u64 tiles in shared memory,
// start value x (or x with surplus twos stripped, _kernels.py:33-45), each hit of p^e
// divides the slot by p exactly (multiply by p^-1 mod 2^64; shift for p = 2) through a
// 64-bit shared CAS so concurrent progressions on one slot compose.
// (V = unsigned int: windows below 2^32, where every slot value fits 32 bits and p^-1 mod
// 2^32 is the low half of p^-1 mod 2^64.)
template <typename V>
__device__ __forceinline__ void div_slot(V* s, uint64_t inv, bool two) {
    V old = *s, assumed;
    do {
        assumed = old;
        const V nv = two ? (V)(assumed >> 1) : (V)(assumed * (V)inv);
        old = atomicCAS(s, assumed, nv);
    } while (old != assumed);
}

// ASYNC: two tile buffers; a finished tile leaves through one bulk asynchronous copy
// (cp.async.bulk shared -> global, issued by one thread, streaming L2 policy) while the
// threads initialise the other buffer and run its progressions, so the HBM write stream
// overlaps the next tile's compute and the warps issue no store instructions.
__device__ __forceinline__ void bulk_store_tile(uint64_t* dst, const unsigned long long* src, uint32_t bytes) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(src);
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
                 :: "l"(dst), "r"(s), "r"(bytes), "l"(pol) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {  // the issuing thread's groups but the newest N have read smem
    asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// NARROW (windows ending below 2^32): 32-bit slots -- half the shared memory per tile, so
// more CTAs per SM, and 32-bit CAS; the write-out widens each pair to the u64 output.
template <int TILE, int NT, int THREADS, int BCAP, int MAXS, int MINB, bool ASYNC, bool NARROW = false>
__global__ void __launch_bounds__(THREADS, MINB) k_sieve_exact(SieveArgs a) {
    static_assert(!(ASYNC && NARROW), "the bulk write-out copies u64 slots");
    using V = typename std::conditional<NARROW, unsigned int, unsigned long long>::type;
    constexpr int NW = THREADS / 32;
    constexpr uint64_t SEG = (uint64_t)TILE * NT;
    constexpr int NBUF = ASYNC ? 2 : 1;
    extern __shared__ __align__(16) unsigned long long sm64[];
    V* r0 = reinterpret_cast<V*>(sm64);                  // NBUF * TILE slots
    unsigned long long* bent = sm64 + NBUF * TILE * sizeof(V) / 8;  // NT * BCAP : (p << 16 | loc)
    unsigned long long* s_inv = bent + NT * BCAP;        // MAXS
    uint32_t* bcnt = (uint32_t*)(s_inv + MAXS);          // NT
    uint32_t* s_q = bcnt + NT;                           // MAXS (sorted by q on the host)
    uint32_t* s_tm = s_q + MAXS;
    uint32_t* s_off = s_tm + MAXS;
    uint32_t* s_item = s_off + MAXS;                     // 2 * MAXS work items

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nsmall = a.nsmall, nitems = a.nitems;
    for (int j = tid; j < nsmall; j += THREADS) {
        const uint32_t q = (uint32_t)a.small[j].q, p = a.small[j].p;
        s_q[j] = q;
        s_tm[j] = (uint32_t)TILE % q;
        s_inv[j] = (p == 2) ? 0ull : bnx_inv64(p);  // 0 marks p = 2: a right shift
    }
    for (int j = tid; j < nitems; j += THREADS) s_item[j] = a.items[j];
    const uint64_t nseg = (a.length + SEG - 1) / SEG;
    int cur = 0;  // the buffer of the tile being sieved (ASYNC)
    for (uint64_t seg = blockIdx.x; seg < nseg; seg += gridDim.x) {
        const uint64_t seg_off = seg * SEG;
        const uint64_t seg0 = a.start + seg_off;
        if (ASYNC && tid == 0) bulk_wait_read<0>();  // (no store may still read the buffers)
        __syncthreads();
        for (int j = tid; j < NT; j += THREADS) bcnt[j] = 0;
        for (int j = tid; j < nsmall; j += THREADS) s_off[j] = (uint32_t)bnx_first_offset(seg0, s_q[j], a.small[j].recip);
        __syncthreads();
        // (windows below 2^32 -- NARROW -- always scan: the host buckets only above)
        if (!NARROW && a.gbuck) {  // the medium progressions here, the huge ones' hits from the window's buckets
            for (uint64_t j = tid; j < a.nmedium; j += THREADS) {
                const BnxProg pr = a.large[j];
                for (uint64_t o = bnx_first_offset(seg0, pr.q, pr.recip); o < SEG; o += pr.q) {
                    const uint32_t t = (uint32_t)(o / TILE), loc = (uint32_t)(o % TILE);
                    uint32_t k = atomicAdd(&bcnt[t], 1u);
                    if (k < BCAP) bent[t * BCAP + k] = ((uint64_t)pr.p << 16) | loc; else a.flags[0] = 1;
                }
            }
            const uint32_t nh = min(a.gcnt[seg], a.gcap);
            const uint64_t* gb = a.gbuck + seg * (uint64_t)a.gcap;
            for (uint32_t i = tid; i < nh; i += THREADS) {
                const uint64_t e = gb[i];
                const uint32_t o = (uint32_t)e, t = o / TILE, loc = o % TILE;
                BNX_CHECK(o < SEG);
                uint32_t k = atomicAdd(&bcnt[t], 1u);
                if (k < BCAP) bent[t * BCAP + k] = ((e >> 32) << 16) | loc; else a.flags[0] = 1;
            }
        } else {
            for (uint64_t j = tid; j < a.nlarge; j += THREADS) {
                const BnxProg pr = a.large[j];
                uint64_t o = bnx_first_offset(seg0, pr.q, pr.recip);
                while (o < SEG) {
                    const uint32_t t = (uint32_t)(o / TILE), loc = (uint32_t)(o % TILE);
                    uint32_t k = atomicAdd(&bcnt[t], 1u);
                    if (k < BCAP) bent[t * BCAP + k] = ((uint64_t)pr.p << 16) | loc; else a.flags[0] = 1;
                    if (pr.q >= SEG) break;
                    o += pr.q;
                }
            }
        }
        __syncthreads();
        // init: x, or x with all but one factor two removed (_kernels.py:33-45); two integers
        // per thread and 16-byte stores: exactly one of them is even, and only that one can
        // need the shift.  Thread g always owns slots 2g, 2g+1 (init, write-out), so the
        // write-out of tile t and the init of tile t+1 share one pass with no barrier.
        auto init_pair = [&](V* buf, uint64_t tile0, int g) {
            if constexpr (NARROW) {  // 32-bit and branch-free: the even one is x0 + (x0 odd), and
                // xe >> (ctz(xe) - 1) leaves xe = 2 (mod 4) unchanged (xe = 0 only past the window's end)
                const uint32_t x0 = (uint32_t)tile0 + 2u * (uint32_t)g;
                uint32_t v0 = x0, v1 = x0 + 1u;
                if (a.fast) {
                    const uint32_t odd0 = x0 & 1u;
                    const uint32_t xe = x0 + odd0;
                    const uint32_t ve = xe ? xe >> (__ffs(xe) - 2) : 0u;
                    v0 = odd0 ? v0 : ve;
                    v1 = odd0 ? ve : v1;
                }
                reinterpret_cast<uint2*>(buf)[g] = make_uint2(v0, v1);
                return;
            }
            const uint64_t x0 = tile0 + 2u * (uint32_t)g;
            uint64_t v0 = x0, v1 = x0 + 1;
            if (a.fast) {
                const bool odd0 = x0 & 1;
                const uint64_t xe = odd0 ? v1 : v0;
                if ((xe & 3) == 0 && xe) {
                    const uint32_t lo = (uint32_t)xe;
                    const int tz = lo ? __ffs(lo) - 1 : 31 + __ffs((uint32_t)(xe >> 32));
                    const uint64_t ve = xe >> (tz - 1);
                    if (odd0) v1 = ve; else v0 = ve;
                }
            }
            reinterpret_cast<ulonglong2*>(buf)[g] = make_ulonglong2(v0, v1);
        };
        for (int g = tid; g < TILE / 2; g += THREADS) init_pair(r0 + cur * TILE, a.start + seg_off, g);
        for (int t = 0; t < NT; ++t) {
            const uint64_t toff = seg_off + (uint64_t)t * TILE;
            if (toff >= a.length) break;
            V* r = r0 + cur * TILE;
            __syncthreads();
            // per-tile progressions: balanced work items (see k_screen), exact division per hit
            const int it_end = (int)s_item[warp + 1];
            for (int it = (int)s_item[warp]; it < it_end; ++it) {
                BNX_CHECK(NW + 1 + it < 2 * MAXS);
                const uint32_t e = s_item[NW + 1 + it];
                const int j = (int)(e & 0xFFu);
                BNX_CHECK(j < nsmall || (e >> 31));
                if (e >> 31) {
                    const int jj = j + lane;
                    if (jj < nsmall) {
                        const uint32_t q = s_q[jj];
                        const uint64_t inv = s_inv[jj];
                        for (uint32_t o = s_off[jj]; o < TILE; o += q) div_slot(&r[o], inv, inv == 0);
                    }
                } else {
                    const uint32_t rr = (e >> 8) & 0xFFu, R = (e >> 16) & 0x7FFFu;
                    const uint32_t q = s_q[j];
                    const uint64_t inv = s_inv[j];
                    const uint32_t step = 32u * R * q;
                    for (uint32_t o = s_off[j] + (rr * 32u + (uint32_t)lane) * q; o < TILE; o += step)
                        div_slot(&r[o], inv, inv == 0);
                }
            }
            {
                const uint32_t nb = min(bcnt[t], (uint32_t)BCAP);
                for (uint32_t i = tid; i < nb; i += THREADS) {
                    const unsigned long long e = bent[t * BCAP + i];
                    const uint32_t p = (uint32_t)(e >> 16);
                    div_slot(&r[e & 0xFFFFu], p == 2 ? 0ull : bnx_inv64(p), p == 2);
                }
            }
            __syncthreads();
            for (int j = tid; j < nsmall; j += THREADS) {
                int no = (int)s_off[j] - (int)s_tm[j];
                if (no < 0) no += (int)s_q[j];
                s_off[j] = (uint32_t)no;
            }
            const uint64_t rem = a.length - toff;
            const int lim = rem < (uint64_t)TILE ? (int)rem : TILE;
            uint64_t* dst = a.out + toff;
            const bool next = t + 1 < NT && toff + TILE < a.length;
            const bool whole = lim == TILE && ((((uintptr_t)dst) & 15) == 0);
            if constexpr (ASYNC) {
                unsigned long long* rn = r0 + (cur ^ 1) * TILE;
                if (whole) {
                    if (tid == 0) {
                        bulk_store_tile(dst, r, TILE * 8u);
                        bulk_wait_read<1>();  // the other buffer's store (one tile ago) has read it
                    }
                    __syncthreads();
                    if (next)
                        for (int g = tid; g < TILE / 2; g += THREADS) init_pair(rn, a.start + toff + TILE, g);
                } else {  // ragged last tile or an output only 8-byte aligned: plain stores
                    if (tid == 0) bulk_wait_read<0>();
                    __syncthreads();
                    for (int g = tid; g < TILE / 2; g += THREADS) {
                        if (2 * g < lim) dst[2 * g] = r[2 * g];
                        if (2 * g + 1 < lim) dst[2 * g + 1] = r[2 * g + 1];
                        if (next) init_pair(rn, a.start + toff + TILE, g);
                    }
                }
                cur ^= 1;
            } else if (whole) {
                // write out (16-byte streaming stores; the values are not re-read on the device)
                // fused with the next tile's init
                for (int g = tid; g < TILE / 2; g += THREADS) {
                    if constexpr (NARROW) {
                        const uint2 v = reinterpret_cast<const uint2*>(r)[g];
                        __stcs(reinterpret_cast<ulonglong2*>(dst) + g, make_ulonglong2(v.x, v.y));
                    } else {
                        __stcs(reinterpret_cast<ulonglong2*>(dst) + g, reinterpret_cast<const ulonglong2*>(r)[g]);
                    }
                    if (next) init_pair(r, a.start + toff + TILE, g);
                }
            } else {  // ragged last tile or an output only 8-byte aligned: same slot ownership
                for (int g = tid; g < TILE / 2; g += THREADS) {
                    if (2 * g < lim) dst[2 * g] = r[2 * g];
                    if (2 * g + 1 < lim) dst[2 * g + 1] = r[2 * g + 1];
                    if (next) init_pair(r, a.start + toff + TILE, g);
                }
            }
        }
    }
    if (ASYNC && tid == 0) bulk_wait_all();  // (the last stores complete before the kernel retires)
}

// ---- k_sieve_pipe: the same sieve as a barrier-free software pipeline --------------------
// k_sieve_exact synchronises the whole CTA twice per tile, and a third of its stall samples
// wait at the barrier behind the slowest warp's progressions.  Here the tiles of a CTA run
// through three shared-memory buffers with mbarriers instead of CTA barriers:
//   compute warps (NWC)  wait ready[b] -> progressions + buckets of tile k -> arrive full[b]
//                        -> wait freed (tile k-1's buffer) -> initialise their slice of tile
//                        k+2 (values and progression offsets) -> arrive ready
//   store warp (1)       wait full[b] -> one bulk asynchronous copy of the tile to HBM
//                        (cp.async.bulk, streaming L2 policy) -> wait for its shared-memory
//                        read -> arrive freed[b]
// so a warp can run up to a tile ahead of the slowest one and the HBM stream never waits for
// a barrier.  Large-progression buckets are double-buffered per segment: the compute warps
// fill segment i+1's set while they start segment i.
namespace pipe {
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void init(uint64_t* bar, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(sa(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(sa(bar)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(sa(bar)), "r"(parity) : "memory");
}
}  // namespace pipe

template <int TILE, int NT, int NWC, int BCAP, int MAXS>
__global__ void __launch_bounds__(NWC * 32 + 32, 1) k_sieve_pipe(SieveArgs a) {
    constexpr int TC = NWC * 32;  // compute threads
    constexpr uint64_t SEG = (uint64_t)TILE * NT;
    constexpr int PAIRS_W = TILE / 2 / NWC;  // init pairs per compute warp
    static_assert(TILE / 2 % NWC == 0, "the compute warps must split the tile's pairs evenly");
    extern __shared__ __align__(16) unsigned long long sm64[];
    unsigned long long* buf = sm64;                                    // 3 * TILE
    unsigned long long* bent = buf + 3 * TILE;                         // 2 * NT * BCAP
    unsigned long long* s_inv = bent + 2 * NT * BCAP;                  // MAXS
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_inv + MAXS);        // ready[3] full[3] freed[3] bready[2] bfree[2]
    uint32_t* bcnt = reinterpret_cast<uint32_t*>(bars + 16);           // 2 * NT
    uint32_t* s_q = bcnt + 2 * NT;                                     // MAXS
    uint32_t* s_tm = s_q + MAXS;                                       // MAXS
    uint32_t* s_base = s_tm + MAXS;                                    // 2 * MAXS (segment start offsets)
    uint32_t* s_off = s_base + 2 * MAXS;                               // 3 * MAXS (per buffer)
    uint32_t* s_item = s_off + 3 * MAXS;                               // 2 * MAXS work items
    uint64_t* ready = bars;
    uint64_t* full = bars + 3;
    uint64_t* freed = bars + 6;
    uint64_t* bready = bars + 9;
    uint64_t* bfree = bars + 11;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nsmall = a.nsmall, nitems = a.nitems;
    for (int j = tid; j < nsmall; j += blockDim.x) {
        const uint32_t q = (uint32_t)a.small[j].q, p = a.small[j].p;
        s_q[j] = q;
        s_tm[j] = (uint32_t)TILE % q;
        s_inv[j] = (p == 2) ? 0ull : bnx_inv64(p);
    }
    for (int j = tid; j < nitems; j += blockDim.x) s_item[j] = a.items[j];
    for (int j = tid; j < 2 * NT; j += blockDim.x) bcnt[j] = 0;
    if (tid == 0) {
        for (int b = 0; b < 3; ++b) {
            pipe::init(ready + b, NWC);
            pipe::init(full + b, NWC);
            pipe::init(freed + b, 1);
        }
        for (int s = 0; s < 2; ++s) {
            pipe::init(bready + s, NWC);
            pipe::init(bfree + s, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // this CTA's tiles: segments blockIdx.x + i * gridDim.x, each up to NT tiles of the input
    const uint64_t nseg_all = (a.length + SEG - 1) / SEG;
    const uint64_t nseg = blockIdx.x < nseg_all ? (nseg_all - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    auto seg_off_of = [&](uint64_t i) { return (blockIdx.x + i * gridDim.x) * SEG; };
    auto tiles_of = [&](uint64_t i) {
        const uint64_t rem = a.length - seg_off_of(i);
        return (int)min((uint64_t)NT, (rem + TILE - 1) / TILE);
    };
    if (nseg == 0) return;
    // tile k (CTA order) -> (segment, tile in segment): every segment but the last has NT tiles
    const uint64_t ktotal = (nseg - 1) * NT + (uint64_t)tiles_of(nseg - 1);
    auto seg_of = [&](uint64_t k) { return k / NT; };
    auto jt_of = [&](uint64_t k) { return (int)(k % NT); };

    if (warp == NWC) {  // ---------------------------------------------- store warp
        for (uint64_t k = 0; k < ktotal; ++k) {
            const int b = (int)(k % 3);
            pipe::wait(full + b, (uint32_t)((k / 3) & 1));
            const uint64_t i = seg_of(k);
            const int jt = jt_of(k);
            const uint64_t toff = seg_off_of(i) + (uint64_t)jt * TILE;
            const uint64_t rem = a.length - toff;
            const int lim = rem < (uint64_t)TILE ? (int)rem : TILE;
            uint64_t* dst = a.out + toff;
            const unsigned long long* r = buf + b * TILE;
            if (lim == TILE && ((((uintptr_t)dst) & 15) == 0)) {
                if (lane == 0) {
                    bulk_store_tile(dst, r, TILE * 8u);
                    bulk_wait_read<0>();
                }
            } else {
                for (int g = lane; g < lim; g += 32) dst[g] = r[g];
            }
            __syncwarp();
            if (lane == 0) {
                bcnt[(i & 1) * NT + jt] = 0;  // this tile's bucket slot, ready for segment i + 2
                pipe::arrive(freed + b);
                if (jt == tiles_of(i) - 1) pipe::arrive(bfree + (i & 1));
            }
        }
        if (lane == 0) bulk_wait_all();
        return;
    }

    // ------------------------------------------------------------------ compute warps
    // bucket fill (large progressions) and segment start offsets (small ones) for segment i,
    // shared by all compute threads; set i & 1 must be free (segment i - 2 consumed)
    auto fill = [&](uint64_t i) {
        const int set = (int)(i & 1);
        if (i >= 2) pipe::wait(bfree + set, (uint32_t)(((i - 2) >> 1) & 1));
        const uint64_t seg0 = a.start + seg_off_of(i);
        for (uint64_t j = tid; j < a.nlarge; j += TC) {
            const BnxProg pr = a.large[j];
            uint64_t o = bnx_first_offset(seg0, pr.q, pr.recip);
            while (o < SEG) {
                const uint32_t t = (uint32_t)(o / TILE), loc = (uint32_t)(o % TILE);
                const uint32_t kk = atomicAdd(&bcnt[set * NT + t], 1u);
                if (kk < BCAP) bent[(set * NT + t) * BCAP + kk] = ((uint64_t)pr.p << 16) | loc; else a.flags[0] = 1;
                if (pr.q >= SEG) break;
                o += pr.q;
            }
        }
        for (int j = tid; j < nsmall; j += TC) s_base[set * MAXS + j] = (uint32_t)bnx_first_offset(seg0, s_q[j], a.small[j].recip);
        __syncwarp();
        if (lane == 0) pipe::arrive(bready + set);
    };
    // this warp's slice of tile k: values (or the ctz-stripped values) and a share of the
    // progression offsets; the buffer must have been read out by the store of tile k - 3
    auto prepare = [&](uint64_t k) {
        const int b = (int)(k % 3);
        if (k >= 3) pipe::wait(freed + b, (uint32_t)(((k - 3) / 3) & 1));
        const uint64_t i = seg_of(k);
        const int jt = jt_of(k);
        const uint64_t tile0 = a.start + seg_off_of(i) + (uint64_t)jt * TILE;
        unsigned long long* r = buf + b * TILE;
        for (int g = warp * PAIRS_W + lane; g < (warp + 1) * PAIRS_W; g += 32) {
            const uint64_t x0 = tile0 + 2u * (uint32_t)g;
            uint64_t v0 = x0, v1 = x0 + 1;
            if (a.fast) {
                const bool odd0 = x0 & 1;
                const uint64_t xe = odd0 ? v1 : v0;
                if ((xe & 3) == 0 && xe) {
                    const uint32_t lo = (uint32_t)xe;
                    const int tz = lo ? __ffs(lo) - 1 : 31 + __ffs((uint32_t)(xe >> 32));
                    const uint64_t ve = xe >> (tz - 1);
                    if (odd0) v1 = ve; else v0 = ve;
                }
            }
            reinterpret_cast<ulonglong2*>(r)[g] = make_ulonglong2(v0, v1);
        }
        pipe::wait(bready + (i & 1), (uint32_t)((i >> 1) & 1));  // (segment i's start offsets)
        for (int j = warp * 32 + lane; j < nsmall; j += TC) {
            const uint32_t q = s_q[j];
            const uint32_t back = (uint32_t)(((uint64_t)jt * s_tm[j]) % q);
            uint32_t o = s_base[(i & 1) * MAXS + j] + q - back;
            if (o >= q) o -= q;
            s_off[b * MAXS + j] = o;
        }
        __syncwarp();
        if (lane == 0) pipe::arrive(ready + b);
    };

    fill(0);
    prepare(0);
    if (ktotal > 1) prepare(1);
    for (uint64_t k = 0; k < ktotal; ++k) {
        const int b = (int)(k % 3);
        const uint64_t i = seg_of(k);
        const int jt = jt_of(k);
        // (segment i+1's set is free once segment i-1 has been stored: a few tiles into i)
        if (i + 1 < nseg && jt == min(2, tiles_of(i) - 1)) fill(i + 1);
        pipe::wait(ready + b, (uint32_t)((k / 3) & 1));
        unsigned long long* r = buf + b * TILE;
        const uint32_t* off = s_off + b * MAXS;
        const int it_end = (int)s_item[warp + 1];
        for (int it = (int)s_item[warp]; it < it_end; ++it) {
            const uint32_t e = s_item[NWC + 1 + it];
            const int j = (int)(e & 0xFFu);
            if (e >> 31) {
                const int jj = j + lane;
                if (jj < nsmall) {
                    const uint32_t q = s_q[jj];
                    const uint64_t inv = s_inv[jj];
                    for (uint32_t o = off[jj]; o < TILE; o += q) div_slot(&r[o], inv, inv == 0);
                }
            } else {
                const uint32_t rr = (e >> 8) & 0xFFu, R = (e >> 16) & 0x7FFFu;
                const uint32_t q = s_q[j];
                const uint64_t inv = s_inv[j];
                const uint32_t step = 32u * R * q;
                for (uint32_t o = off[j] + (rr * 32u + (uint32_t)lane) * q; o < TILE; o += step)
                    div_slot(&r[o], inv, inv == 0);
            }
        }
        {
            const int set = (int)(i & 1);
            const uint32_t nb = min(bcnt[set * NT + jt], (uint32_t)BCAP);
            for (uint32_t t = tid; t < nb; t += TC) {
                const unsigned long long e = bent[(set * NT + jt) * BCAP + t];
                const uint32_t p = (uint32_t)(e >> 16);
                div_slot(&r[e & 0xFFFFu], p == 2 ? 0ull : bnx_inv64(p), p == 2);
            }
        }
        __syncwarp();
        if (lane == 0) pipe::arrive(full + b);
        if (k + 2 < ktotal) prepare(k + 2);
    }
}

template <int TILE, int NT, int NWC, int BCAP>
constexpr size_t sieve_pipe_smem() {
    return sizeof(unsigned long long) * ((size_t)3 * TILE + (size_t)2 * NT * BCAP + SIEVE_MAXS) + 16 * 8 +
           sizeof(uint32_t) * ((size_t)2 * NT + 9 * SIEVE_MAXS);
}

// _kernels.py:87-112 on the GPU: one thread per integer, trial division by the odd primes.
__global__ void k_trial_division(uint64_t start, uint64_t length, const BnxPDiv* pd, uint64_t npd, uint64_t* out) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < length; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t x = start + k;
        const int tz = bnx_ctz64(x);
        uint64_t y = x >> tz;
        uint64_t r = tz ? 2 : 1;
        for (uint64_t j = 0; j < npd; ++j) {
            const BnxPDiv d = pd[j];
            if (d.p * d.p > y) break;
            uint64_t t = y * d.inv;
            if (t <= d.lim) {
                r *= d.p;
                do { y = t; t = y * d.inv; } while (t <= d.lim);
            }
        }
        if (y > 1) r *= y;
        out[k] = r;
    }
}

// ------------------------------------------------------------------------------------
// bruteforce.py:16-42 / _kernels.py:235-263 on the GPU: the quadratic reference scan, an
// independent check of the search (no sieve, no screen, no residue classes).  rads[t] =
// rad(t+1) for t < limit (from k_trial_division); a block owns 256 consecutive m and streams
// all n > m through shared-memory tiles.
__global__ void __launch_bounds__(256) k_brute_force(const uint64_t* __restrict__ rads, uint64_t limit,
                                                     bnx_pair_t* out, uint64_t cap, unsigned long long* count) {
    __shared__ uint64_t tile[2049];
    const uint64_t m0 = 1 + (uint64_t)blockIdx.x * blockDim.x;
    const uint64_t m = m0 + threadIdx.x;
    const bool live = m + 1 < limit;
    const uint64_t rm = live ? rads[m - 1] : 0, rm1 = live ? rads[m] : 0;
    for (uint64_t n0 = m0 + 1; n0 < limit; n0 += 2048) {
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < 2049; i += blockDim.x) {  // rads of n0-1 .. n0+2047
            const uint64_t t = n0 - 1 + i;
            tile[i] = t < limit ? rads[t] : 0;
        }
        __syncthreads();
        if (!live) continue;
        const uint64_t nend = min(limit, n0 + 2048);
        for (uint64_t n = max(n0, m + 1); n < nend; ++n) {
            const uint64_t rn = tile[n - n0], rn1 = tile[n - n0 + 1];
            int kind = 0;
            if (rn == rm && rn1 == rm1) kind = 1;
            else if (rn == rm1 && rn1 == rm) kind = 2;
            if (kind) {
                unsigned long long k = atomicAdd(count, 1ull);
                if (k < cap) out[k] = bnx_pair_t{m, n, rm, rm1, kind, 0};
            }
        }
    }
}

// ------------------------------------------------------------------------------------
// Algorithm 3 of the paper on the GPU (chunked.py:129-304, _kernels.py:115-232): the
// open-addressing signature table with the reference's slot word ((t+1) << 32 | home, 0 =
// empty), hash (_slot_of) and linear probing, built by all threads at once with 64-bit
// CAS.  Two elements with equal signatures share a home slot, and whichever claims its
// slot later walks past the earlier one, so every equal pair is reported exactly once (as
// (smaller, larger) domain index, classified like _kernels.py:172).  Slot placement can
// differ from the serial build; the pair set cannot.
__device__ __forceinline__ uint64_t table_slot_of(uint64_t lo, uint64_t hi, uint64_t mask) {
    uint64_t x = lo ^ (hi * 0x9E3779B97F4A7C15ull);
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return (x ^ (x >> 31)) & mask;
}

__device__ __forceinline__ void table_emit(TableArgs& a, int kind, uint64_t m, uint64_t n, uint64_t rm, uint64_t rm1) {
    unsigned long long k = atomicAdd(a.count, 1ull);
    if (k < a.cap) a.out[k] = bnx_pair_t{m, n, rm, rm1, kind, 0};
}

__global__ void k_table_insert(TableArgs a) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < a.count_n; t += (uint64_t)gridDim.x * blockDim.x) {
        if (a.domain_start + t >= a.n_limit) continue;
        const uint64_t x = a.rad_of[t], y = a.rad_next[t];
        const uint64_t lo = x < y ? x : y, hi = x < y ? y : x;
        const uint64_t home = table_slot_of(lo, hi, a.mask);
        const unsigned long long mine = ((unsigned long long)(t + 1) << 32) | home;
        uint64_t idx = home, steps = 0;
        for (;;) {
            unsigned long long stored = a.slots[idx];
            if (stored == 0) {
                stored = atomicCAS(reinterpret_cast<unsigned long long*>(a.slots) + idx, 0ull, mine);
                if (stored == 0) { atomicAdd(a.inserted, 1ull); break; }
            }
            if ((stored & 0xFFFFFFFFull) == home) {
                const uint64_t tp = (stored >> 32) - 1;
                const uint64_t x2 = a.rad_of[tp], y2 = a.rad_next[tp];
                if ((x2 < y2 ? x2 : y2) == lo && (x2 < y2 ? y2 : x2) == hi) {
                    const uint64_t tm = tp < t ? tp : t, tn = tp < t ? t : tp;
                    const uint64_t rm = a.rad_of[tm], rm1 = a.rad_next[tm];
                    table_emit(a, rm == a.rad_of[tn] ? 1 : 2, a.domain_start + tm, a.domain_start + tn, rm, rm1);
                }
            }
            idx = (idx + 1) & a.mask;
            if (++steps > a.mask) { *a.status = BNX_TABLE_FULL; break; }
        }
    }
}

__global__ void k_table_probe(TableArgs a) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < a.count_m; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t x = a.probe_of[t], y = a.probe_next[t];
        const uint64_t lo = x < y ? x : y, hi = x < y ? y : x;
        const uint64_t home = table_slot_of(lo, hi, a.mask);
        uint64_t idx = home, steps = 0;
        for (;;) {
            const uint64_t stored = a.slots[idx];
            if (stored == 0) break;
            if ((stored & 0xFFFFFFFFull) == home) {
                const uint64_t tp = (stored >> 32) - 1;
                const uint64_t x2 = a.rad_of[tp], y2 = a.rad_next[tp];
                if ((x2 < y2 ? x2 : y2) == lo && (x2 < y2 ? y2 : x2) == hi)
                    table_emit(a, x == x2 ? 1 : 2, a.probe_start + t, a.domain_start + tp, x, y);
            }
            idx = (idx + 1) & a.mask;
            if (++steps > a.mask) { *a.status = BNX_TABLE_FULL; break; }
        }
    }
}

// The paper's parallel probe ("examine the slot at the initial address, the
// next one, and so on ... the best performance was achieved by examining 4 addresses in
// parallel"): four lanes per element read four consecutive slots at once; every slot before
// the first empty one is checked for an equal signature, and insert claims that empty slot
// by CAS (a lost race re-reads from it: its new occupant may match).  Same pairs, same
// slot words and probe sequences as the one-lane kernels above.
template <bool INSERT>
__global__ void __launch_bounds__(256) k_table_quad(TableArgs a) {
    const int lane = threadIdx.x & 31, q = lane & 3;
    const unsigned qmask = 0xFu << (lane & ~3);
    const uint64_t nq = ((uint64_t)gridDim.x * blockDim.x) >> 2;
    const uint64_t count = INSERT ? a.count_n : a.count_m;
    const uint64_t* of = INSERT ? a.rad_of : a.probe_of;
    const uint64_t* nx = INSERT ? a.rad_next : a.probe_next;
    for (uint64_t t = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 2; t < count; t += nq) {
        if (INSERT && a.domain_start + t >= a.n_limit) continue;  // (quad-uniform)
        const uint64_t x = of[t], y = nx[t];
        const uint64_t lo = x < y ? x : y, hi = x < y ? y : x;
        const uint64_t home = table_slot_of(lo, hi, a.mask);
        const unsigned long long mine = ((unsigned long long)(t + 1) << 32) | home;
        uint64_t idx = home, steps = 0;
        for (;;) {
            const uint64_t slot = (idx + q) & a.mask;
            const unsigned long long stored = a.slots[slot];
            const unsigned emp = (__ballot_sync(qmask, stored == 0) >> (lane & ~3)) & 0xFu;
            const int fe = emp ? __ffs(emp) - 1 : 4;  // first empty slot of the window
            if (q < fe && (stored & 0xFFFFFFFFull) == home) {
                const uint64_t tp = (stored >> 32) - 1;
                const uint64_t x2 = a.rad_of[tp], y2 = a.rad_next[tp];
                if ((x2 < y2 ? x2 : y2) == lo && (x2 < y2 ? y2 : x2) == hi) {
                    if (INSERT) {
                        const uint64_t tm = tp < t ? tp : t, tn = tp < t ? t : tp;
                        const uint64_t rm = a.rad_of[tm], rm1 = a.rad_next[tm];
                        table_emit(a, rm == a.rad_of[tn] ? 1 : 2, a.domain_start + tm, a.domain_start + tn, rm, rm1);
                    } else {
                        table_emit(a, x == x2 ? 1 : 2, a.probe_start + t, a.domain_start + tp, x, y);
                    }
                }
            }
            if (fe < 4) {
                if (!INSERT) break;
                unsigned long long won = 1;
                if (q == fe) {
                    won = atomicCAS(reinterpret_cast<unsigned long long*>(a.slots) + slot, 0ull, mine) == 0ull;
                    if (won) atomicAdd(a.inserted, 1ull);
                }
                if (__shfl_sync(qmask, won, (lane & ~3) + fe)) break;
                idx += fe;  // lost the slot: look at its new occupant and on from there
                steps += fe;
            } else {
                idx += 4;
                steps += 4;
            }
            if (steps > a.mask) {
                if (q == 0) *a.status = BNX_TABLE_FULL;
                break;
            }
        }
    }
}

// Global buckets of the huge progressions (q >= SIEVE_HUGE_Q, above every segment length): a
// thread per progression walks its few hits in the window once and appends each to the
// bucket of its segment, so a segment reads its hits instead of testing every progression
// (the per-segment scan costs O(segments x pi(sqrt end)): 0.8 s for 2^30 integers at 2^62).
__global__ void k_sieve_buckets(SieveArgs a, uint64_t seg_len, uint64_t* gbuck, uint32_t* gcnt, uint32_t gcap) {
    for (uint64_t j = a.nmedium + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < a.nlarge;
         j += (uint64_t)gridDim.x * blockDim.x) {
        const BnxProg pr = a.large[j];
        for (uint64_t o = bnx_first_offset(a.start, pr.q, pr.recip); o < a.length; o += pr.q) {
            const uint64_t seg = o / seg_len;
            BNX_CHECK(seg < (a.length + seg_len - 1) / seg_len);
            const uint32_t k = atomicAdd(&gcnt[seg], 1u);
            if (k < gcap) gbuck[seg * gcap + k] = ((uint64_t)pr.p << 32) | (o - seg * seg_len);
            else a.flags[3] = 1;
            if (pr.q > a.length) break;
        }
    }
}
void launch_sieve_buckets(const SieveArgs& a, uint64_t seg_len, uint64_t* gbuck, uint32_t* gcnt, cudaStream_t st) {
    if (a.nlarge <= a.nmedium) return;
    const unsigned grid = (unsigned)std::min<uint64_t>((a.nlarge - a.nmedium + 255) / 256, 148 * 16);
    k_sieve_buckets<<<grid, 256, 0, st>>>(a, seg_len, gbuck, gcnt, a.gcap);
}
// Order-free split of the large progressions: q < SIEVE_HUGE_Q to the front of `out`, the
// rest to the back (counts[0], counts[1]).
__global__ void k_split_large(const BnxProg* in, uint64_t n, BnxProg* out, unsigned long long* counts) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
        const BnxProg pr = in[j];
        if (pr.q < SIEVE_HUGE_Q) out[atomicAdd(&counts[0], 1ull)] = pr;
        else out[n - 1 - atomicAdd(&counts[1], 1ull)] = pr;
    }
}
void launch_split_large(const BnxProg* in, uint64_t n, BnxProg* out, unsigned long long* counts, cudaStream_t st) {
    if (n) k_split_large<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(in, n, out, counts);
}

// ------------------------------------------------------------------------------------
// Launch helpers (instantiations and dynamic shared memory sizes).
template <int TILE, int NT, int BCAP, bool ASYNC = false, bool NARROW = false>
constexpr size_t sieve_smem() {
    return (NARROW ? sizeof(uint32_t) : sizeof(unsigned long long)) * (size_t)TILE * (ASYNC ? 2 : 1) +
           sizeof(unsigned long long) * ((size_t)NT * BCAP + SIEVE_MAXS) + sizeof(uint32_t) * ((size_t)NT + 5 * SIEVE_MAXS);
}
template <int TILE, int NT, int THREADS, int BCAP, int MINB, bool ASYNC, bool NARROW = false>
void launch_sieve_v(const SieveArgs& a, int grid, cudaStream_t st) {
    k_sieve_exact<TILE, NT, THREADS, BCAP, SIEVE_MAXS, MINB, ASYNC, NARROW>
        <<<grid, THREADS, sieve_smem<TILE, NT, BCAP, ASYNC, NARROW>(), st>>>(a);
}
template <int TILE, int NT, int NWC, int BCAP>
void launch_sieve_pipe(const SieveArgs& a, int grid, cudaStream_t st) {
    k_sieve_pipe<TILE, NT, NWC, BCAP, SIEVE_MAXS><<<grid, NWC * 32 + 32, sieve_pipe_smem<TILE, NT, NWC, BCAP>(), st>>>(a);
}
#define BNX_SIEVE_VARIANT(T, N, H, B, M, A)                                                                    \
    SieveVariant{T, N, H, B, (const void*)k_sieve_exact<T, N, H, B, SIEVE_MAXS, M, A>, sieve_smem<T, N, B, A>(), \
                 launch_sieve_v<T, N, H, B, M, A>}
static const SieveVariant kSieveVariants[] = {
    // u64 slots (windows reaching 2^32; below, kSieveNarrow).  Default: 6144-slot tiles (48 KB),
    // 384 threads, three CTAs per SM -- 2^30 integers at 2^40 in 2.03 ms against 2.19 ms for
    // the round-1 geometry (index 1: 8192 slots, 512 threads, two CTAs per SM), 2.08-2.63 ms for
    // the other tile sizes and CTA shapes tried (profiles/r02_sieve_windows.jsonl); identical
    // output hashes
    BNX_SIEVE_VARIANT(6144, 32, 384, 64, 3, false),
    BNX_SIEVE_VARIANT(SIEVE_TILE, SIEVE_NT, SIEVE_THREADS, SIEVE_BCAP, 2, false),
    BNX_SIEVE_VARIANT(8192, 64, 768, 64, 2, false),
    BNX_SIEVE_VARIANT(8192, 64, 256, 64, 4, false),
    BNX_SIEVE_VARIANT(4096, 64, 512, 48, 3, false),
    // bulk asynchronous write-out from a second tile buffer (see bulk_store_tile): one CTA
    // per SM fits two 64 KB tiles, and the lost second CTA costs more than the stores save
    // (3.41 / 3.35 ms on [1, 2^30]; 4096-slot tiles with two CTAs: 3.28 ms async, 3.84 ms not)
    BNX_SIEVE_VARIANT(8192, 64, 1024, 64, 1, true),
    BNX_SIEVE_VARIANT(8192, 64, 512, 64, 1, true),
    // the barrier-free pipeline (k_sieve_pipe): 16 compute warps + a store warp, one CTA per
    // SM (three 64 KB tiles): no barrier stalls, but too few warps to hide the shared-memory
    // CAS latency (3.84 ms on [1, 2^30] against 2.17 ms for the round-1 default)
    SieveVariant{8192, 24, 512, 64, (const void*)k_sieve_pipe<8192, 24, 16, 64, SIEVE_MAXS>,
                 sieve_pipe_smem<8192, 24, 16, 64>(), launch_sieve_pipe<8192, 24, 16, 64>},
    BNX_SIEVE_VARIANT(6144, 32, 320, 64, 3, false),
    BNX_SIEVE_VARIANT(6144, 16, 384, 64, 3, false),
};
int sieve_variant_count() { return (int)(sizeof(kSieveVariants) / sizeof(kSieveVariants[0])); }
const SieveVariant& sieve_variant(int i) { return kSieveVariants[i]; }
// 32-bit-slot geometries for windows ending below 2^32 (BNX_SIEVE_NARROW, default 0; -1: off).
// Measured on [1, 2^30] (scripts/sieve_variants.py, profiles/r02_sieve_narrow.jsonl): 1.40 ms
// for the default against 2.17 ms for the u64 kernel; 1.43, 1.54, 1.63 ms for the others.
// Half-size slots fit four CTAs per SM, and CTAs of 12 warps wait less at the per-tile
// barriers than CTAs of 16 (512 threads: 1.54 ms) or 32 (1024: 2.30 ms).
#define BNX_SIEVE_NARROW_VARIANT(T, N, H, B, M)                                                                        \
    SieveVariant{T, N, H, B, (const void*)k_sieve_exact<T, N, H, B, SIEVE_MAXS, M, false, true>,                    \
                 sieve_smem<T, N, B, false, true>(), launch_sieve_v<T, N, H, B, M, false, true>}
static const SieveVariant kSieveNarrow[] = {
    BNX_SIEVE_NARROW_VARIANT(8192, 32, 384, 64, 4),
    BNX_SIEVE_NARROW_VARIANT(8192, 16, 256, 64, 5),
    BNX_SIEVE_NARROW_VARIANT(8192, 32, 512, 64, 4),
    BNX_SIEVE_NARROW_VARIANT(8192, 64, 512, 64, 3),
};
int sieve_narrow_count() { return (int)(sizeof(kSieveNarrow) / sizeof(kSieveNarrow[0])); }
const SieveVariant& sieve_narrow(int i) { return kSieveNarrow[i]; }

template <int TILE, int NT, int THREADS, int BCAP>
constexpr size_t screen_smem() {
    return sizeof(uint32_t) * ((size_t)(TILE / 4 + 4) + NT + (size_t)NT * BCAP + 6 * SCREEN_MAXS) +
           sizeof(uint64_t) * SCREEN_MAXS;
}
template <int TILE, int NT, int THREADS, int BCAP, int MINB>
void launch_screen_v(const ScreenArgs& a, int grid, cudaStream_t st) {
    k_screen<TILE, NT, THREADS, BCAP, SCREEN_MAXS, MINB>
        <<<grid, THREADS, screen_smem<TILE, NT, THREADS, BCAP>(), st>>>(a);
}
#define BNX_SCREEN_VARIANT(T, N, H, B, M)                                                               \
    ScreenVariant{T, N, H, B, (const void*)k_screen<T, N, H, B, SCREEN_MAXS, M>, screen_smem<T, N, H, B>(), \
                  launch_screen_v<T, N, H, B, M>}
static const ScreenVariant kScreenVariants[] = {
    BNX_SCREEN_VARIANT(65536, 64, 512, 128, 2),  // default: fastest measured (profiles/)
    BNX_SCREEN_VARIANT(65536, 32, 512, 224, 2),
    BNX_SCREEN_VARIANT(32768, 64, 512, 96, 3),
    BNX_SCREEN_VARIANT(32768, 32, 512, 128, 4),
};
int screen_variant_count() { return (int)(sizeof(kScreenVariants) / sizeof(kScreenVariants[0])); }
const ScreenVariant& screen_variant(int i) { return kScreenVariants[i]; }
constexpr unsigned TAIL_HEAVY_Y = 256;  // k_tail_heavy grid rows (candidates strided over them)
void launch_tail(const TailArgs& a, int grid, cudaStream_t st) {
    k_tail<<<grid, 256, 0, st>>>(a);
    k_tail_heavy<<<dim3(8, (unsigned)std::min<uint64_t>(a.heavy_cap, TAIL_HEAVY_Y)), 256, 0, st>>>(a);
}
void launch_tail_light(const TailArgs& a, int grid, cudaStream_t st, bool pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;  // a programmatic dependent of k_heavy_exact (see k_tail)
    cudaLaunchKernelEx(&cfg, k_tail, a);
}
void launch_tail_heavy(const TailArgs& a, cudaStream_t st) {
    k_tail_heavy<<<dim3(8, (unsigned)std::min<uint64_t>(a.heavy_cap, TAIL_HEAVY_Y)), 256, 0, st>>>(a);
}

void launch_base_primes(uint32_t ls, uint32_t* out, uint32_t* count, cudaStream_t st) {
    if (ls + 1 > 48 * 1024) cudaFuncSetAttribute(k_base_primes, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(ls + 1));
    k_base_primes<<<1, 1024, ls + 1, st>>>(ls, out, count);
}
void launch_prime_seg(uint64_t lo, uint64_t hi, const uint32_t* base, uint32_t nbase, uint32_t* counts,
                      const uint64_t* offsets, uint32_t* out, uint64_t nblocks, cudaStream_t st) {
    k_prime_seg<<<(unsigned)nblocks, 1024, 0, st>>>(lo, hi, base, nbase, counts, offsets, out);
}
void launch_scan_counts(const uint32_t* counts, uint64_t n, uint64_t base, uint64_t* offsets, cudaStream_t st) {
    k_scan_counts<<<1, 1024, 0, st>>>(counts, n, base, offsets);
}
void launch_narrow(const uint64_t* in, uint64_t n, uint32_t* out, cudaStream_t st) {
    k_narrow_primes<<<256, 256, 0, st>>>(in, n, out);
}
void launch_widen(const uint32_t* in, uint64_t n, uint64_t* out, cudaStream_t st) {
    k_widen_primes<<<256, 256, 0, st>>>(in, n, out);
}
void launch_build_tables(const uint32_t* primes, uint64_t np, uint64_t max_x, int include_two, uint32_t tile,
                         BnxProg* small, uint32_t* nsmall, uint32_t small_cap, BnxProg* large,
                         unsigned long long* nlarge, uint64_t large_cap, BnxPDiv* pdiv, uint64_t* npdiv,
                         int* overflow, cudaStream_t st) {
    k_build_tables<<<256, 256, 0, st>>>(primes, np, max_x, include_two, tile, small, nsmall, small_cap, large, nlarge,
                                        large_cap, pdiv, npdiv, overflow);
}
void launch_brute_force(const uint64_t* rads, uint64_t limit, bnx_pair_t* out, uint64_t cap,
                        unsigned long long* count, cudaStream_t st) {
    const uint64_t blocks = (limit + 255) / 256;
    k_brute_force<<<(unsigned)blocks, 256, 0, st>>>(rads, limit, out, cap, count);
}
void launch_table_insert(const TableArgs& a, int grid, cudaStream_t st, int lanes) {
    if (lanes == 4) k_table_quad<true><<<grid, 256, 0, st>>>(a);
    else k_table_insert<<<grid, 256, 0, st>>>(a);
}
void launch_table_probe(const TableArgs& a, int grid, cudaStream_t st, int lanes) {
    if (lanes == 4) k_table_quad<false><<<grid, 256, 0, st>>>(a);
    else k_table_probe<<<grid, 256, 0, st>>>(a);
}
void launch_trial_division(uint64_t start, uint64_t length, const BnxPDiv* pd, uint64_t npd, uint64_t* out,
                           int grid, cudaStream_t st) {
    k_trial_division<<<grid, 256, 0, st>>>(start, length, pd, npd, out);
}

// Load the search-path kernels of this file now (CUDA loads a kernel lazily at its first
// launch, which would otherwise land inside a caller's first search).
cudaError_t kernels_preload() {
    const void* fns[] = {(const void*)k_base_primes, (const void*)k_prime_seg, (const void*)k_scan_counts,
                         (const void*)k_narrow_primes, (const void*)k_build_tables, (const void*)k_tail,
                         (const void*)k_tail_heavy, kSieveVariants[0].fn, kSieveNarrow[0].fn, kScreenVariants[0].fn};
    for (const void* f : fns) {
        cudaFuncAttributes at;
        const cudaError_t e = cudaFuncGetAttributes(&at, f);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace bnx
