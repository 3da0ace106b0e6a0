/* abi_consumer.c — TEST PROGRAM: a plain C99 translation unit compiled with
 * -Wall -Wextra -Werror -pedantic against include/pag_gpu.h and linked to
 * libpag_gpu.so. Pins the struct layouts the bindings rely on and exercises
 * the host-only entry points (no GPU needed): default parameters, the default
 * subspace count (projection.cpp:151-166), the reference family
 * (projection.cpp:40-74), index inspection (builder.cpp:434-492) and the
 * error path (status code + thread-local message).
 * usage: abi_consumer <index.pagidx>   (prints one line "ok ..." on success) */
#include <stddef.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "pag_gpu.h"

_Static_assert(sizeof(pag_search_stats) == 40, "pag_search_stats: five u64");
_Static_assert(offsetof(pag_search_stats, edges_scanned) == 32, "edges_scanned offset");
_Static_assert(sizeof(pag_search_params) == 16, "pag_search_params: three u32 + four u8");
_Static_assert(offsetof(pag_search_params, use_prt) == 12, "use_prt offset");
_Static_assert(offsetof(pag_search_params, exact_dist) == 14, "exact_dist offset");
_Static_assert(sizeof(pag_index_arrays) == 112, "pag_index_arrays: u64, 8 x u32, u64, 4 x u8, u32, 7 pointers");
_Static_assert(offsetof(pag_index_arrays, seed) == 40, "seed offset");
_Static_assert(offsetof(pag_index_arrays, n_entries) == 52, "n_entries offset");
_Static_assert(offsetof(pag_index_arrays, entry_nodes) == 56, "entry_nodes offset");
_Static_assert(offsetof(pag_index_arrays, norms) == 104, "norms offset");

#define CHECK(c)                                                       \
    do {                                                               \
        if (!(c)) {                                                    \
            fprintf(stderr, "check failed: %s (line %d)\n", #c, __LINE__); \
            return 1;                                                  \
        }                                                              \
    } while (0)

int main(int argc, char** argv) {
    pag_search_params p;
    uint64_t info[12];
    float* refs;
    size_t i, nz = 0;
    int rc;
    CHECK(argc == 2);
    pag_gpu_default_params(&p);
    CHECK(p.K == 10 && p.efS == 100 && p.b_override == 0 && p.use_prt == 1 && p.use_tfb == 1 && p.exact_dist == 1);
    CHECK(pag_gpu_default_subspace_count(128) == 16 && pag_gpu_default_subspace_count(768) == 32);
    /* reference family: L = 16 subspaces of 8, m = 16 references */
    refs = (float*)malloc(sizeof(float) * 16 * 16 * 8);
    CHECK(refs != NULL);
    CHECK(pag_gpu_reference_family(128, 16, 16, 42, refs, 16 * 16 * 8) == PAG_GPU_OK);
    for (i = 0; i < 16 * 16 * 8; ++i) nz += refs[i] != 0.0f;
    CHECK(nz > 0);
    rc = pag_gpu_reference_family(128, 16, 16, 42, refs, 10); /* buffer too small */
    CHECK(rc == PAG_GPU_EINVAL && strstr(pag_gpu_last_error(), "too small") != NULL);
    rc = pag_gpu_reference_family(130, 16, 16, 42, refs, 16 * 16 * 8); /* 130 % 16 != 0 */
    CHECK(rc == PAG_GPU_EINVAL && strcmp(pag_gpu_last_error(), "padded_dim not divisible by L") == 0);
    free(refs);
    /* index inspection (host only) and the load errors' texts */
    CHECK(pag_gpu_inspect(argv[1], info, 12) == PAG_GPU_OK);
    CHECK(info[0] > 0 && info[1] > 0 && info[2] >= info[1] && info[9] > 0);
    rc = pag_gpu_inspect("/nonexistent/pag.bin", info, 12);
    CHECK(rc == PAG_GPU_ERUNTIME && strcmp(pag_gpu_last_error(), "cannot open index: /nonexistent/pag.bin") == 0);
    {   /* the in-memory source: argument errors are raised before any GPU work */
        pag_index_arrays a;
        pag_gpu_index* h = NULL;
        memset(&a, 0, sizeof a);
        CHECK(pag_gpu_open_from_arrays(NULL, NULL, 0, &h) == PAG_GPU_EINVAL && h == NULL);
        a.n = 4; /* n > 0 with no arrays */
        CHECK(pag_gpu_open_from_arrays(&a, NULL, 0, &h) == PAG_GPU_EINVAL && h == NULL);
        CHECK(strcmp(pag_gpu_last_error(), "null argument") == 0);
        CHECK(pag_gpu_refresh_from_arrays(NULL, &a, NULL) == PAG_GPU_EINVAL);
    }
    CHECK(strstr(pag_gpu_version(), "sm_100a") != NULL);
    printf("ok n=%llu dim=%llu padded=%llu edges=%llu\n", (unsigned long long)info[0], (unsigned long long)info[1],
           (unsigned long long)info[2], (unsigned long long)info[9]);
    return 0;
}
