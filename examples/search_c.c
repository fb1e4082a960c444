/* The C ABI from plain C: every pair below a bound, printed as
 * the reference CLI's CSV rows (cli.py: kind,m,n,rad_m,rad_m1), sorted by (m, n).
 *   gcc -O2 -I include examples/search_c.c -L paper_2506_01099_b200 -lbenelux_b200 \
 *       -Wl,-rpath,paper_2506_01099_b200 -o search_c && ./search_c 4294967296 */
#include <stdio.h>
#include <stdlib.h>

#include "benelux_b200.h"

int main(int argc, char** argv) {
    const unsigned long long limit = argc > 1 ? strtoull(argv[1], NULL, 0) : (1ull << 32);
    const unsigned kinds = argc > 2 ? (unsigned)atoi(argv[2]) : BNX_KIND_BOTH;
    bnx_ctx_t* ctx = NULL;
    if (bnx_ctx_create(0, &ctx) != BNX_OK) {
        fprintf(stderr, "bnx_ctx_create: %s\n", bnx_last_error());
        return 1;
    }
    size_t cap = 8, found = 0;
    bnx_pair_t* rows = malloc(cap * sizeof(bnx_pair_t));
    int st = bnx_search(ctx, limit, kinds, NULL, 0, 0, rows, cap, &found);
    if (st == BNX_BUFFER_FULL) { /* the reference's grow-and-retry protocol */
        cap = found;
        rows = realloc(rows, cap * sizeof(bnx_pair_t));
        st = bnx_search(ctx, limit, kinds, NULL, 0, 0, rows, cap, &found);
    }
    if (st != BNX_OK) {
        fprintf(stderr, "bnx_search: %s (status %d)\n", bnx_last_error(), st);
        return 2;
    }
    printf("kind,m,n,rad_m,rad_m1\n");
    for (size_t i = 0; i < found; ++i)
        printf("%d,%llu,%llu,%llu,%llu\n", rows[i].kind, (unsigned long long)rows[i].m, (unsigned long long)rows[i].n,
               (unsigned long long)rows[i].rad_m, (unsigned long long)rows[i].rad_m1);
    free(rows);
    bnx_ctx_destroy(ctx);
    return 0;
}
