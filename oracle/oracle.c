/*
 * oracle/oracle.c -- CPU restatement of the reference's Benelux-pair search path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links, loads or calls
 * this file; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg do, and only as the checker / the timed CPU reference.
 *
 * Parity pinned: tests/test_oracle_golden.py checks every function below against
 * golden vectors produced by importing the reference package itself
 * (tests/golden/make_golden.py, fixtures under tests/golden/) and against the
 * known-answer tests the reference's own suite holds.
 *
 * Every function cites the reference file:line it restates; paths are relative
 * to the reference's pkg/src/benelux_pairs/ directory.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define ORC_STATUS_OK 0          /* _kernels.py:17 */
#define ORC_STATUS_TABLE_FULL 1  /* _kernels.py:18 */
#define ORC_STATUS_BUFFER_FULL 2 /* _kernels.py:19 */
#define ORC_STATUS_NOMEM 3

typedef struct {
    int8_t* kind;
    uint64_t* m;
    uint64_t* n;
    uint64_t* rm;
    uint64_t* rm1;
    size_t cap;
    size_t found;
} orc_pairs_t;

static int push_pair(orc_pairs_t* out, int kind, uint64_t m, uint64_t n, uint64_t rm, uint64_t rm1) {
    if (out->found >= out->cap) { out->found++; return ORC_STATUS_BUFFER_FULL; }
    out->kind[out->found] = (int8_t)kind;
    out->m[out->found] = m;
    out->n[out->found] = n;
    out->rm[out->found] = rm;
    out->rm1[out->found] = rm1;
    out->found++;
    return ORC_STATUS_OK;
}

static uint64_t isqrt_u64(uint64_t x) {
    uint64_t r = 0;
    for (int b = 31; b >= 0; --b) {
        uint64_t t = r | (1ull << b);
        if (t * t <= x && t <= 0xFFFFFFFFull) r = t;
    }
    return r;
}

uint64_t orc_isqrt(uint64_t x) { return isqrt_u64(x); }

/* primes.py:24-35 -- flat-array Eratosthenes up to `limit`; returns the count. */
int64_t orc_primes_up_to(uint64_t limit, uint64_t* out, size_t cap) {
    if (limit < 2) return 0;
    uint8_t* composite = (uint8_t*)calloc(limit + 1, 1);
    if (!composite) return -1;
    composite[0] = composite[1] = 1;
    uint64_t r = isqrt_u64(limit);
    for (uint64_t p = 2; p <= r; ++p)
        if (!composite[p])
            for (uint64_t q = p * p; q <= limit; q += p) composite[q] = 1;
    int64_t count = 0;
    for (uint64_t p = 2; p <= limit; ++p)
        if (!composite[p]) {
            if ((size_t)count < cap) out[count] = p;
            count++;
        }
    free(composite);
    return count;
}

/* _kernels.py:22-30 */
void orc_identity_fill(uint64_t start, size_t length, uint64_t* vals) {
    for (size_t k = 0; k < length; ++k) vals[k] = start + k;
}

/* _kernels.py:33-45 -- multiples of four lose all but one factor two. */
void orc_strip_twos(uint64_t* vals, size_t length, uint64_t start) {
    size_t offset = (size_t)((4 - start % 4) % 4);
    for (size_t idx = offset; idx < length; idx += 4) {
        uint64_t v = vals[idx];
        uint64_t low = v & (~v + 1);
        vals[idx] = v / (low >> 1);
    }
}

/* _kernels.py:48-84 -- Algorithm 1: divide each progression of p^e (e >= 2) by p once. */
void orc_sieve_segment(uint64_t start, size_t length, const uint64_t* primes, size_t nprimes,
                       int fast_two, uint64_t* vals) {
    orc_identity_fill(start, length, vals);
    uint64_t endpoint = start + (uint64_t)(length - 1);
    uint64_t length_u = (uint64_t)length;
    if (fast_two) orc_strip_twos(vals, length, start);
    for (size_t j = 0; j < nprimes; ++j) {
        uint64_t p = primes[j];
        if (p > endpoint / p) break;          /* :64-65 */
        if (fast_two && p == 2) continue;     /* :66-67 */
        uint64_t power = p * p;
        for (;;) {
            uint64_t residue = start % power; /* :70-73 */
            if (residue == 0) residue = power;
            uint64_t shift = power - residue;
            if (shift > length_u) break;      /* :75-76 */
            for (uint64_t idx = shift; idx < length_u; idx += power) vals[idx] /= p;
            if (power > endpoint / p) break;  /* :81-82 */
            power *= p;
        }
    }
}

/* _kernels.py:87-112 -- per-integer trial division, shares nothing with the sieve. */
void orc_radicals_trial_division(uint64_t start, size_t length, uint64_t* out) {
    for (size_t k = 0; k < length; ++k) {
        uint64_t n = start + (uint64_t)k;
        uint64_t r = 1;
        if ((n & 1) == 0) {
            r = 2;
            while ((n & 1) == 0) n >>= 1;
        }
        for (uint64_t d = 3; d * d <= n; d += 2) {
            if (n % d == 0) {
                r *= d;
                while (n % d == 0) n /= d;
            }
        }
        if (n > 1) r *= n;
        out[k] = r;
    }
}

/* _kernels.py:115-123 (twin chunked.py:104-109) */
uint64_t orc_slot_of(uint64_t lo, uint64_t hi, uint64_t mask, uint64_t phi, uint64_t mul1, uint64_t mul2) {
    uint64_t x = lo ^ (hi * phi);
    x = (x ^ (x >> 30)) * mul1;
    x = (x ^ (x >> 27)) * mul2;
    x = x ^ (x >> 31);
    return x & mask;
}

/* _kernels.py:130-183 -- serial linear-probe insert, reporting every equal signature passed. */
int orc_build_table(uint64_t domain_start, const uint64_t* rad_of, const uint64_t* rad_next, size_t count,
                    uint64_t n_limit, uint64_t* slots, uint64_t mask, uint64_t phi, uint64_t mul1,
                    uint64_t mul2, orc_pairs_t* out, size_t* inserted_out) {
    size_t inserted = 0;
    uint64_t n = domain_start;
    for (size_t t = 0; t < count; ++t) {
        if (n >= n_limit) break;
        uint64_t a = rad_of[t], b = rad_next[t];
        uint64_t lo = a < b ? a : b, hi = a < b ? b : a;
        uint64_t home = orc_slot_of(lo, hi, mask, phi, mul1, mul2);
        uint64_t idx = home, steps = 0;
        for (;;) {
            uint64_t stored = slots[idx];
            if (stored == 0) {
                slots[idx] = ((uint64_t)(t + 1) << 32) | home;
                inserted++;
                break;
            }
            if ((stored & 0xFFFFFFFFull) == home) {
                size_t tp = (size_t)(stored >> 32) - 1;
                uint64_t a2 = rad_of[tp], b2 = rad_next[tp];
                uint64_t lo2 = a2 < b2 ? a2 : b2, hi2 = a2 < b2 ? b2 : a2;
                if (lo2 == lo && hi2 == hi) {
                    if (push_pair(out, a2 == a ? 1 : 2, domain_start + tp, n, a2, b2) != ORC_STATUS_OK) {
                        *inserted_out = inserted;
                        return ORC_STATUS_BUFFER_FULL;
                    }
                }
            }
            idx = (idx + 1) & mask;
            if (++steps > mask) { *inserted_out = inserted; return ORC_STATUS_TABLE_FULL; }
        }
        n++;
    }
    *inserted_out = inserted;
    return ORC_STATUS_OK;
}

/* _kernels.py:186-232 -- read-only probe with an earlier domain. */
int orc_probe_table(uint64_t probe_start, const uint64_t* rad_of, const uint64_t* rad_next, size_t count,
                    uint64_t domain_start, const uint64_t* cur_rad_of, const uint64_t* cur_rad_next,
                    const uint64_t* slots, uint64_t mask, uint64_t phi, uint64_t mul1, uint64_t mul2,
                    orc_pairs_t* out) {
    uint64_t m = probe_start;
    for (size_t t = 0; t < count; ++t) {
        uint64_t a = rad_of[t], b = rad_next[t];
        uint64_t lo = a < b ? a : b, hi = a < b ? b : a;
        uint64_t home = orc_slot_of(lo, hi, mask, phi, mul1, mul2);
        uint64_t idx = home, steps = 0;
        for (;;) {
            uint64_t stored = slots[idx];
            if (stored == 0) break;
            if ((stored & 0xFFFFFFFFull) == home) {
                size_t tp = (size_t)(stored >> 32) - 1;
                uint64_t a2 = cur_rad_of[tp], b2 = cur_rad_next[tp];
                uint64_t lo2 = a2 < b2 ? a2 : b2, hi2 = a2 < b2 ? b2 : a2;
                if (lo2 == lo && hi2 == hi) {
                    if (push_pair(out, a == a2 ? 1 : 2, m, domain_start + tp, a, b) != ORC_STATUS_OK)
                        return ORC_STATUS_BUFFER_FULL;
                }
            }
            idx = (idx + 1) & mask;
            if (++steps > mask) return ORC_STATUS_TABLE_FULL;
        }
        m++;
    }
    return ORC_STATUS_OK;
}

/* _kernels.py:235-263 -- O(S^2) ground-truth double loop; rads[t] = rad(t+1), t < limit. */
int orc_brute_force_scan(const uint64_t* rads, size_t limit, orc_pairs_t* out) {
    for (size_t m = 1; m + 1 < limit; ++m) {
        uint64_t rm = rads[m - 1], rm1 = rads[m];
        for (size_t n = m + 1; n < limit; ++n) {
            uint64_t rn = rads[n - 1], rn1 = rads[n];
            int kind;
            if (rn == rm && rn1 == rm1) kind = 1;
            else if (rn == rm1 && rn1 == rm) kind = 2;
            else continue;
            if (push_pair(out, kind, m, n, rm, rm1) != ORC_STATUS_OK) return ORC_STATUS_BUFFER_FULL;
        }
    }
    return ORC_STATUS_OK;
}

/* ---------------------------------------------------------------------------------------
 * sort_search.py:37-91 -- Algorithm 2: sieve [1, limit], stable sort the canonical
 * signatures of n = 1..limit-1 by (lo, hi) (ties ascending in n, as np.lexsort is stable),
 * emit every pair inside each maximal equal run, classify (signatures.py:67-81).
 * The caller sorts the result by (m, n) (sort_search.py:90).
 */
typedef struct { uint64_t lo, hi, x; } sig_rec_t;

static int cmp_sig(const void* pa, const void* pb) {
    const sig_rec_t* a = (const sig_rec_t*)pa;
    const sig_rec_t* b = (const sig_rec_t*)pb;
    if (a->lo != b->lo) return a->lo < b->lo ? -1 : 1;
    if (a->hi != b->hi) return a->hi < b->hi ? -1 : 1;
    if (a->x != b->x) return a->x < b->x ? -1 : 1; /* stability of lexsort */
    return 0;
}

int orc_find_pairs_sorted(uint64_t limit, const uint64_t* primes, size_t nprimes, orc_pairs_t* out) {
    uint64_t* values = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)limit);
    sig_rec_t* recs = (sig_rec_t*)malloc(sizeof(sig_rec_t) * (size_t)(limit - 1));
    if (!values || !recs) { free(values); free(recs); return ORC_STATUS_NOMEM; }
    orc_sieve_segment(1, (size_t)limit, primes, nprimes, 1, values);
    for (uint64_t x = 1; x < limit; ++x) {
        uint64_t a = values[x - 1], b = values[x];
        recs[x - 1].lo = a < b ? a : b;
        recs[x - 1].hi = a < b ? b : a;
        recs[x - 1].x = x;
    }
    qsort(recs, (size_t)(limit - 1), sizeof(sig_rec_t), cmp_sig);
    int status = ORC_STATUS_OK;
    size_t i = 0, count = (size_t)(limit - 1);
    while (i < count) {
        size_t j = i + 1;
        while (j < count && recs[j].lo == recs[i].lo && recs[j].hi == recs[i].hi) j++;
        for (size_t u = i; u + 1 < j; ++u)
            for (size_t v = u + 1; v < j; ++v) {
                uint64_t m = recs[u].x, n = recs[v].x;
                uint64_t rm = values[m - 1], rm1 = values[m], rn = values[n - 1], rn1 = values[n];
                int kind = (rm == rn && rm1 == rn1) ? 1 : 2;
                if (push_pair(out, kind, m, n, rm, rm1) != ORC_STATUS_OK) status = ORC_STATUS_BUFFER_FULL;
            }
        i = j;
    }
    free(values);
    free(recs);
    return status;
}

/* ---------------------------------------------------------------------------------------
 * chunked.py:70-90, 307-412 -- Algorithm 3: per chunk, sieve, build the signature table
 * (intra-chunk pairs), then re-sieve every earlier chunk and probe (threads split the
 * earlier chunks, chunked.py:344-356).  Pairs of one chunk are left in discovery order;
 * the Python wrapper sorts each chunk by (n, m) (chunked.py:358).
 */
static const uint64_t HASH_PHI = 0x9E3779B97F4A7C15ull;  /* chunked.py:27 */
static const uint64_t HASH_MUL1 = 0xBF58476D1CE4E5B9ull;
static const uint64_t HASH_MUL2 = 0x94D049BB133111EBull;

uint64_t orc_num_chunks(uint64_t limit, uint64_t chunk_size) { return (limit - 2) / (chunk_size - 1) + 1; }

uint64_t orc_table_size_for(uint64_t domain_count) { /* chunked.py:86-90 */
    uint64_t v = 4 * domain_count - 1;
    int bits = 0;
    while (v) { bits++; v >>= 1; }
    return 1ull << bits;
}

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

typedef struct {
    uint64_t chunk_size;
    const uint64_t* primes;
    size_t nprimes;
    uint64_t domain_start;
    const uint64_t* cur_vals; /* sieve of the table's chunk */
    const uint64_t* slots;
    uint64_t mask;
    uint64_t j_begin, j_end, j_step; /* earlier chunks this worker probes */
    uint64_t sub_len;                /* >0: probe only the first sub_len values of each */
    orc_pairs_t out;
    int status;
} probe_job_t;

static void* probe_worker(void* arg) {
    probe_job_t* job = (probe_job_t*)arg;
    uint64_t s = job->chunk_size;
    uint64_t* vals = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)s);
    if (!vals) { job->status = ORC_STATUS_NOMEM; return NULL; }
    uint64_t len = job->sub_len ? job->sub_len + 1 : s;
    for (uint64_t j = job->j_begin; j < job->j_end; j += job->j_step) {
        uint64_t first = 1 + j * (s - 1);
        orc_sieve_segment(first, (size_t)len, job->primes, job->nprimes, 1, vals);
        int st = orc_probe_table(first, vals, vals + 1, (size_t)(len - 1), job->domain_start, job->cur_vals,
                                 job->cur_vals + 1, job->slots, job->mask, HASH_PHI, HASH_MUL1, HASH_MUL2,
                                 &job->out);
        if (st != ORC_STATUS_OK && job->status == ORC_STATUS_OK) job->status = st;
    }
    free(vals);
    return NULL;
}

/* chunked.py:326-333 -- sieve chunk `index` into vals and build its table (intra-chunk
 * pairs appended to out).  Returns the build status; *t_build gets the wall seconds. */
int orc_build_chunk(uint64_t index, uint64_t chunk_size, const uint64_t* primes, size_t nprimes,
                    uint64_t n_limit, uint64_t* slots, uint64_t table_size, uint64_t* vals, orc_pairs_t* out,
                    double* t_build) {
    uint64_t s = chunk_size;
    uint64_t first = 1 + index * (s - 1);
    double t0 = now_s();
    orc_sieve_segment(first, (size_t)s, primes, nprimes, 1, vals);
    memset(slots, 0, sizeof(uint64_t) * (size_t)table_size);
    size_t inserted = 0;
    int status = orc_build_table(first, vals, vals + 1, (size_t)(s - 1), n_limit, slots, table_size - 1,
                                 HASH_PHI, HASH_MUL1, HASH_MUL2, out, &inserted);
    if (t_build) *t_build = now_s() - t0;
    return status;
}

/* chunked.py:335-356 -- re-sieve the earlier chunks j in [j_lo, j_hi) and probe the table of
 * chunk `index` (built by orc_build_chunk) with them, on `threads` pthreads. */
int orc_probe_chunks(uint64_t index, uint64_t chunk_size, const uint64_t* primes, size_t nprimes, int threads,
                     uint64_t j_lo, uint64_t j_hi, const uint64_t* slots, uint64_t table_size,
                     const uint64_t* vals, uint64_t sub_len, orc_pairs_t* out, double* t_probe) {
    uint64_t s = chunk_size;
    uint64_t first = 1 + index * (s - 1);
    double t1 = now_s();
    int status = ORC_STATUS_OK;
    if (j_hi > j_lo) {
        if (threads < 1) threads = 1;
        uint64_t njobs = j_hi - j_lo;
        if ((uint64_t)threads > njobs) threads = (int)njobs;
        probe_job_t* jobs = (probe_job_t*)calloc((size_t)threads, sizeof(probe_job_t));
        pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
        size_t per_cap = out->cap > out->found ? out->cap - out->found : 0;
        for (int w = 0; w < threads; ++w) {
            probe_job_t* jb = &jobs[w];
            jb->chunk_size = s; jb->primes = primes; jb->nprimes = nprimes;
            jb->domain_start = first; jb->cur_vals = vals; jb->slots = slots; jb->mask = table_size - 1;
            jb->j_begin = j_lo + (uint64_t)w; jb->j_end = j_hi; jb->j_step = (uint64_t)threads;
            jb->sub_len = sub_len < s - 1 ? sub_len : 0;
            jb->out.cap = per_cap;
            jb->out.kind = (int8_t*)malloc(per_cap + 1);
            jb->out.m = (uint64_t*)malloc(8 * (per_cap + 1));
            jb->out.n = (uint64_t*)malloc(8 * (per_cap + 1));
            jb->out.rm = (uint64_t*)malloc(8 * (per_cap + 1));
            jb->out.rm1 = (uint64_t*)malloc(8 * (per_cap + 1));
            pthread_create(&tids[w], NULL, probe_worker, jb);
        }
        for (int w = 0; w < threads; ++w) pthread_join(tids[w], NULL);
        for (int w = 0; w < threads; ++w) {
            probe_job_t* jb = &jobs[w];
            if (jb->status != ORC_STATUS_OK && status == ORC_STATUS_OK) status = jb->status;
            size_t k = jb->out.found < jb->out.cap ? jb->out.found : jb->out.cap;
            for (size_t t = 0; t < k; ++t)
                if (push_pair(out, jb->out.kind[t], jb->out.m[t], jb->out.n[t], jb->out.rm[t], jb->out.rm1[t]))
                    status = ORC_STATUS_BUFFER_FULL;
            if (jb->out.found > jb->out.cap) status = ORC_STATUS_BUFFER_FULL;
            free(jb->out.kind); free(jb->out.m); free(jb->out.n); free(jb->out.rm); free(jb->out.rm1);
        }
        free(jobs);
        free(tids);
    }
    if (t_probe) *t_probe = now_s() - t1;
    return status;
}

/* chunked.py:307-359 -- all pairs whose n lies in chunk `index`'s domain, probing the
 * earlier chunks j in [j_lo, j_hi) (the full search uses j_lo=0, j_hi=index). */
int orc_search_chunk(uint64_t index, uint64_t chunk_size, const uint64_t* primes, size_t nprimes,
                     uint64_t n_limit, int threads, uint64_t j_lo, uint64_t j_hi, uint64_t* slots,
                     uint64_t table_size, uint64_t* vals, orc_pairs_t* out, double* t_build, double* t_probe) {
    int status = orc_build_chunk(index, chunk_size, primes, nprimes, n_limit, slots, table_size, vals, out, t_build);
    if (status == ORC_STATUS_TABLE_FULL) return status;
    int st2 = orc_probe_chunks(index, chunk_size, primes, nprimes, threads, j_lo, j_hi, slots, table_size, vals,
                               0, out, t_probe);
    return status != ORC_STATUS_OK ? status : st2;
}

/* chunked.py:362-412 -- every chunk from resume_from on; pairs appended chunk by chunk. */
int orc_run_full_chunked(uint64_t limit, uint64_t chunk_size, const uint64_t* primes, size_t nprimes,
                         uint64_t resume_from, int threads, orc_pairs_t* out, uint64_t* chunk_ends) {
    uint64_t total = orc_num_chunks(limit, chunk_size);
    uint64_t table_size = orc_table_size_for(chunk_size - 1);
    uint64_t* slots = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)table_size);
    uint64_t* vals = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)chunk_size);
    if (!slots || !vals) { free(slots); free(vals); return ORC_STATUS_NOMEM; }
    int status = ORC_STATUS_OK;
    for (uint64_t index = resume_from; index < total; ++index) {
        int st = orc_search_chunk(index, chunk_size, primes, nprimes, limit, threads, 0, index, slots,
                                  table_size, vals, out, NULL, NULL);
        if (chunk_ends) chunk_ends[index - resume_from] = out->found;
        if (st == ORC_STATUS_TABLE_FULL || st == ORC_STATUS_NOMEM) { status = st; break; }
        if (st != ORC_STATUS_OK) status = st;
    }
    free(slots);
    free(vals);
    return status;
}
