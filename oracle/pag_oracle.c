/*
 * pag_oracle.c — CPU ORACLE (test infrastructure only; see pag_oracle.h).
 *
 * Plain-C restatement of the reference PAG query path. Every function cites
 * the reference file:line it follows (paths relative to /root/reference).
 * Compile with -ffp-contract=off and no -march flags: the reference is built
 * the same way so fp32 results are bit-identical.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker.
 */
#include "pag_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

const char* pago_last_error(void) { return g_err; }

/* ------------------------------------------------------------------------ */
/* L0 distances: proj/src/vecstore.cpp:77-108                                */
/* ------------------------------------------------------------------------ */

/* vecstore.cpp:77-95 — four strided fp32 accumulators, square then add, tail
 * into acc0, combined as (a0+a1)+(a2+a3). */
float pago_sq_dist(const float* a, const float* b, size_t padded_dim) {
    float acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    size_t k = 0;
    for (; k + 4 <= padded_dim; k += 4) {
        float d0 = a[k] - b[k];
        float d1 = a[k + 1] - b[k + 1];
        float d2 = a[k + 2] - b[k + 2];
        float d3 = a[k + 3] - b[k + 3];
        acc0 += d0 * d0;
        acc1 += d1 * d1;
        acc2 += d2 * d2;
        acc3 += d3 * d3;
    }
    for (; k < padded_dim; ++k) {
        float d = a[k] - b[k];
        acc0 += d * d;
    }
    return ((acc0 + acc1) + (acc2 + acc3));
}

/* vecstore.cpp:97-108 */
float pago_vec_norm(const float* a, size_t padded_dim) {
    float acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    size_t k = 0;
    for (; k + 4 <= padded_dim; k += 4) {
        acc0 += a[k] * a[k];
        acc1 += a[k + 1] * a[k + 1];
        acc2 += a[k + 2] * a[k + 2];
        acc3 += a[k + 3] * a[k + 3];
    }
    for (; k < padded_dim; ++k) acc0 += a[k] * a[k];
    return sqrtf((acc0 + acc1) + (acc2 + acc3));
}

/* ------------------------------------------------------------------------ */
/* libstdc++ RNG restatement (used by projection.cpp:14,56)                  */
/* std::mt19937_64 and std::normal_distribution<double> (Marsaglia polar,    */
/* generate_canonical<double,53> over one 64-bit draw), GCC 13 libstdc++.    */
/* ------------------------------------------------------------------------ */

typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    if (g->idx >= 312) {
        int k;
        for (k = 0; k < 312 - 156; ++k) {
            uint64_t y = (g->mt[k] & UM) | (g->mt[k + 1] & LM);
            g->mt[k] = g->mt[k + 156] ^ (y >> 1) ^ ((y & 1) ? 0xB5026F5AA96619E9ULL : 0);
        }
        for (; k < 311; ++k) {
            uint64_t y = (g->mt[k] & UM) | (g->mt[k + 1] & LM);
            g->mt[k] = g->mt[k + (156 - 312)] ^ (y >> 1) ^ ((y & 1) ? 0xB5026F5AA96619E9ULL : 0);
        }
        uint64_t y = (g->mt[311] & UM) | (g->mt[0] & LM);
        g->mt[311] = g->mt[155] ^ (y >> 1) ^ ((y & 1) ? 0xB5026F5AA96619E9ULL : 0);
        g->idx = 0;
    }
    uint64_t z = g->mt[g->idx++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= (z >> 43);
    return z;
}

/* generate_canonical<double, 53>: one draw, sum / 2^64, clamp below 1 */
static double canonical53(mt64* g) {
    double sum = (double)mt64_next(g);
    double r = sum / 18446744073709551616.0;
    if (r >= 1.0) r = nextafter(1.0, 0.0);
    return r;
}

typedef struct {
    int saved_available;
    double saved;
} normal_dist;

static double normal_next(normal_dist* nd, mt64* g) {
    double ret;
    if (nd->saved_available) {
        nd->saved_available = 0;
        ret = nd->saved;
    } else {
        double x, y, r2;
        do {
            x = 2.0 * canonical53(g) - 1.0;
            y = 2.0 * canonical53(g) - 1.0;
            r2 = x * x + y * y;
        } while (r2 > 1.0 || r2 == 0.0);
        double mult = sqrt(-2 * log(r2) / r2);
        nd->saved = x * mult;
        nd->saved_available = 1;
        ret = y * mult;
    }
    return ret * 1.0 + 0.0; /* stddev 1, mean 0 */
}

void pago_mt64_stream(uint64_t seed, uint64_t* out, size_t n) {
    mt64 g;
    mt64_seed(&g, seed);
    for (size_t i = 0; i < n; ++i) out[i] = mt64_next(&g);
}

void pago_normal_stream(uint64_t seed, double* out, size_t n) {
    mt64 g;
    normal_dist nd = {0, 0.0};
    mt64_seed(&g, seed);
    for (size_t i = 0; i < n; ++i) out[i] = normal_next(&nd, &g);
}

/* ------------------------------------------------------------------------ */
/* L1 projection: proj/src/projection.cpp                                    */
/* ------------------------------------------------------------------------ */

/* projection.cpp:13-38 — Haar rotation by modified Gram-Schmidt in double;
 * a fresh normal_distribution per call (its cached spare is discarded). */
static void random_rotation(uint32_t k, mt64* rng, float* q) {
    normal_dist gauss = {0, 0.0};
    double* qd = (double*)calloc((size_t)k * k, sizeof(double));
    double* col = (double*)malloc(sizeof(double) * k);
    for (uint32_t c = 0; c < k; ++c) {
        for (;;) {
            for (uint32_t r = 0; r < k; ++r) col[r] = normal_next(&gauss, rng);
            for (uint32_t p = 0; p < c; ++p) {
                double dot = 0;
                for (uint32_t r = 0; r < k; ++r) dot += col[r] * qd[(size_t)p * k + r];
                for (uint32_t r = 0; r < k; ++r) col[r] -= dot * qd[(size_t)p * k + r];
            }
            double nrm = 0;
            for (uint32_t r = 0; r < k; ++r) nrm += col[r] * col[r];
            nrm = sqrt(nrm);
            if (nrm > 1e-9) {
                for (uint32_t r = 0; r < k; ++r) qd[(size_t)c * k + r] = col[r] / nrm;
                break;
            }
        }
    }
    for (size_t i = 0; i < (size_t)k * k; ++i) q[i] = (float)qd[i];
    free(col);
    free(qd);
}

/* projection.cpp:40-74 */
int pago_build_reference_set(uint32_t padded_dim, uint32_t L, uint32_t m, uint64_t seed,
                             float* out) {
    if (L == 0 || padded_dim % L != 0)
        return fail(PAGO_EINVAL, "padded_dim not divisible by L");
    uint32_t sub_dim = padded_dim / L;
    if (sub_dim < 2) return fail(PAGO_EINVAL, "sub_dim < 2: cross-polytope degenerate");
    if (m == 0 || m > 16) return fail(PAGO_EINVAL, "m must be in [1, 16] (4-bit codes)");
    memset(out, 0, sizeof(float) * (size_t)L * m * sub_dim);
    const float scale = 1.0f / sqrtf((float)L);
    const uint32_t polytopes = (m + 2 * sub_dim - 1) / (2 * sub_dim);
    mt64 rng;
    mt64_seed(&rng, seed);
    float* rot = (float*)malloc(sizeof(float) * (size_t)sub_dim * sub_dim);
    for (uint32_t l = 0; l < L; ++l) {
        uint32_t j = 0;
        for (uint32_t p = 0; p < polytopes && j < m; ++p) {
            random_rotation(sub_dim, &rng, rot);
            for (uint32_t sgn = 0; sgn < 2 && j < m; ++sgn) {
                for (uint32_t c = 0; c < sub_dim && j < m; ++c, ++j) {
                    float* dst = out + ((size_t)l * m + j) * sub_dim;
                    float s = (sgn == 0) ? scale : -scale;
                    for (uint32_t r = 0; r < sub_dim; ++r)
                        dst[r] = s * rot[(size_t)c * sub_dim + r];
                }
            }
        }
    }
    free(rot);
    return PAGO_OK;
}

/* projection.hpp:25-33 */
uint32_t pago_code_at(const uint8_t* codes, uint32_t l) {
    return (codes[l >> 1] >> ((l & 1u) * 4)) & 0xFu;
}

void pago_set_code(uint8_t* codes, uint32_t l, uint32_t j) {
    uint8_t* b = &codes[l >> 1];
    uint32_t shift = (l & 1u) * 4;
    *b = (uint8_t)((*b & ~(0xFu << shift)) | ((j & 0xFu) << shift));
}

/* projection.cpp:123-137 — serial fp32 dot per (l, j) */
void pago_build_projection_table(const float* x, const float* refs, uint32_t L, uint32_t m,
                                 uint32_t k, float* out) {
    for (uint32_t l = 0; l < L; ++l) {
        const float* xl = x + (size_t)l * k;
        for (uint32_t j = 0; j < m; ++j) {
            const float* r = refs + ((size_t)l * m + j) * k;
            float dot = 0;
            for (uint32_t c = 0; c < k; ++c) dot += xl[c] * r[c];
            out[(size_t)l * m + j] = dot;
        }
    }
}

/* projection.cpp:145-149 — serial in l */
float pago_table_code_sum(const float* table, uint32_t L, uint32_t m, const uint8_t* codes) {
    float sum = 0;
    for (uint32_t l = 0; l < L; ++l) sum += table[(size_t)l * m + pago_code_at(codes, l)];
    return sum;
}

/* projection.cpp:151-166 */
uint32_t pago_default_subspace_count(uint32_t dim) {
    uint32_t p = 1;
    double root = sqrt((double)dim);
    while (p * 2 <= root * sqrt(2.0) && p * 2 <= dim) p *= 2;
    uint32_t hi = 1;
    while (hi * 2 <= dim / 8) hi *= 2;
    uint32_t lo = 8;
    if (hi < lo) {
        lo = hi = (hi > 1u ? hi : 1u);
        while (lo * 2 <= dim / 4) lo = hi = lo * 2;
    }
    if (p < lo) p = lo;
    if (p > hi) p = hi;
    return p;
}

/* routing.hpp:40-51 */
float pago_prt_threshold(float edge_norm, float dist_uv, float dist_zmax_v) {
    return (edge_norm * edge_norm + dist_uv * dist_uv - dist_zmax_v * dist_zmax_v) /
           (2.0f * dist_uv * edge_norm);
}

int pago_prt_test(float cos_theta, float cos_beta, float tau) {
    if (tau >= 1.0f + 1e-6f) return 0;
    if (tau <= -1.0f) return 1;
    return cos_theta / cos_beta - tau >= 0.0f;
}

/* ------------------------------------------------------------------------ */
/* L3 index file: proj/src/builder.cpp:389-492 (PAGIDX01 v1)                 */
/* ------------------------------------------------------------------------ */

struct pago_index {
    uint64_t n;
    uint32_t dim, padded, L, m, M, efC, b_build, pes_flush;
    uint64_t seed;
    uint8_t metric, enable_pes;
    uint32_t n_entries;
    uint32_t* entries;
    uint32_t maxdeg, cb, sub_dim;
    uint32_t* degree;    /* n */
    uint32_t* targets;   /* n * maxdeg */
    float* scalars;      /* n * maxdeg * 3 {cos_beta, edge_norm, base_offset} */
    uint8_t* codes;      /* n * maxdeg * cb */
    float* rows;         /* n * padded */
    float* norms;        /* n */
    float* refs;         /* L * m * sub_dim */
    uint64_t total_edges;
    int dist_mode;       /* 0: reference order (vecstore.cpp:77-95); 1: the B200 warp-tree order */
};

/* The B200 library's second distance mode (exact_dist = 0): FMA partials per
 * lane over the float4s it loads, then a fixed xor-butterfly reduction
 * (paper_2603_06660_b200/csrc/pag_search.cu, dist_fast_pairs / dist_fast).
 * Restated here so that the GPU's warp-tree mode can be checked bit for bit
 * too: the traversal logic is shared, so any difference between the two
 * modes' results is attributable to the summation order alone. The GPU row
 * stride is round_up(padded, 4); elements past padded are zero on both
 * sides and contribute exact zeros. */
static float warp_tree_sq_dist(const float* a, const float* q, uint32_t padded) {
    const uint32_t ds = (padded + 3u) & ~3u;
    const uint32_t nch = ds / 128u;
    if (padded == ds && ds % 128u == 0 && (nch == 1 || nch == 4 || nch == 6 || nch == 8)) {
        /* dist_fast_pairs<NCH>: 16 lanes, lane h owns float4 i at 64 i + 4 h */
        float s[16];
        for (uint32_t h = 0; h < 16; ++h) {
            float ax = 0.0f, ay = 0.0f;
            for (uint32_t i = 0; i < 2 * nch; ++i) {
                const uint32_t k = 64u * i + 4u * h;
                const float d0 = a[k] - q[k], d1 = a[k + 1] - q[k + 1], d2 = a[k + 2] - q[k + 2],
                            d3 = a[k + 3] - q[k + 3];
                ax = fmaf(d0, d0, ax);
                ay = fmaf(d1, d1, ay);
                ax = fmaf(d2, d2, ax);
                ay = fmaf(d3, d3, ay);
            }
            s[h] = ax + ay;
        }
        for (uint32_t m = 8; m; m >>= 1)
            for (uint32_t h = 0; h < m; ++h) s[h] = s[h] + s[h + m];
        return s[0];
    }
    /* dist_fast<0>: 32 lanes, lane l owns float4 l of every 128-float chunk */
    float p[32];
    for (uint32_t l = 0; l < 32; ++l) {
        float px = 0.0f, py = 0.0f;
        for (uint32_t base = 0; base + 4u * l < ds; base += 128u) {
            const uint32_t k = base + 4u * l;
            float d[4];
            for (uint32_t c = 0; c < 4; ++c) d[c] = k + c < padded ? a[k + c] - q[k + c] : 0.0f;
            px = fmaf(d[0], d[0], px);
            py = fmaf(d[1], d[1], py);
            px = fmaf(d[2], d[2], px);
            py = fmaf(d[3], d[3], py);
        }
        p[l] = px + py;
    }
    for (uint32_t m = 16; m; m >>= 1)
        for (uint32_t l = 0; l < m; ++l) p[l] = p[l] + p[l + m];
    return p[0];
}

static float row_dist(const struct pago_index* ix, uint32_t id, const float* q) {
    const float* row = ix->rows + (size_t)id * ix->padded;
    return ix->dist_mode ? warp_tree_sq_dist(row, q, ix->padded) : pago_sq_dist(row, q, ix->padded);
}

void pago_set_distance_mode(struct pago_index* ix, int mode) { ix->dist_mode = mode ? 1 : 0; }

static int rd(FILE* f, void* p, size_t n) { return fread(p, 1, n, f) == n; }

void pago_free(pago_index* ix) {
    if (!ix) return;
    free(ix->entries);
    free(ix->degree);
    free(ix->targets);
    free(ix->scalars);
    free(ix->codes);
    free(ix->rows);
    free(ix->norms);
    free(ix->refs);
    free(ix);
}

/* builder.cpp:434-492 plus the PagIndex constructor (builder.cpp:40-46):
 * L==0 resolves to the dimension default, the set is repadded to a multiple
 * of L and must reproduce the stored padded_dim, references are regenerated
 * from (padded_dim, L, m, seed). Targets are additionally range-checked
 * (the reference trusts them). */
int pago_load(const char* path, pago_index** out) {
    *out = NULL;
    FILE* f = fopen(path, "rb");
    if (!f) return fail(PAGO_ERUNTIME, "cannot open index: %s", path);
    pago_index* ix = (pago_index*)calloc(1, sizeof *ix);
    int rc = PAGO_OK;
    uint64_t magic = 0;
    uint32_t version = 0;
#define RD(p, n)                                                  \
    do {                                                          \
        if (!rd(f, (p), (n))) {                                   \
            rc = fail(PAGO_ERUNTIME, "index read failed");        \
            goto done;                                            \
        }                                                         \
    } while (0)
    RD(&magic, 8);
    if (magic != 0x5041474944583031ULL) {
        rc = fail(PAGO_ERUNTIME, "bad index magic");
        goto done;
    }
    RD(&version, 4);
    if (version != 1) {
        rc = fail(PAGO_ERUNTIME, "unsupported index version");
        goto done;
    }
    RD(&ix->n, 8);
    RD(&ix->dim, 4);
    RD(&ix->padded, 4);
    RD(&ix->L, 4);
    RD(&ix->m, 4);
    RD(&ix->M, 4);
    RD(&ix->efC, 4);
    RD(&ix->b_build, 4);
    RD(&ix->pes_flush, 4);
    RD(&ix->seed, 8);
    RD(&ix->metric, 1);
    RD(&ix->enable_pes, 1);
    RD(&ix->n_entries, 4);
    ix->entries = (uint32_t*)malloc(sizeof(uint32_t) * (ix->n_entries ? ix->n_entries : 1));
    RD(ix->entries, (size_t)ix->n_entries * 4);
    if (ix->padded < ix->dim) {
        rc = fail(PAGO_EINVAL, "padded_dim < dim");
        goto done;
    }
    if (ix->L == 0) ix->L = pago_default_subspace_count(ix->dim);
    {
        uint64_t want = ((uint64_t)(ix->dim + ix->L - 1) / ix->L) * ix->L;
        if (want != ix->padded) {
            rc = fail(PAGO_ERUNTIME, "padded_dim mismatch on load");
            goto done;
        }
    }
    ix->sub_dim = ix->padded / ix->L;
    ix->refs = (float*)malloc(sizeof(float) * (size_t)ix->L * (ix->m ? ix->m : 1) * ix->sub_dim);
    rc = pago_build_reference_set(ix->padded, ix->L, ix->m, ix->seed, ix->refs);
    if (rc) goto done;
    ix->maxdeg = 2 * ix->M;
    ix->cb = (ix->L + 1) / 2;
    {
        const uint64_t n = ix->n;
        const size_t slots = (size_t)n * ix->maxdeg;
        ix->degree = (uint32_t*)calloc(n ? n : 1, 4);
        ix->targets = (uint32_t*)calloc(slots ? slots : 1, 4);
        ix->scalars = (float*)calloc(slots ? slots * 3 : 1, 4);
        ix->codes = (uint8_t*)calloc(slots ? slots * ix->cb : 1, 1);
        if (!ix->degree || !ix->targets || !ix->scalars || !ix->codes) {
            rc = fail(PAGO_ENOMEM, "out of host memory");
            goto done;
        }
        for (uint64_t u = 0; u < n; ++u) {
            uint32_t deg;
            RD(&deg, 4);
            if (deg > ix->maxdeg) {
                rc = fail(PAGO_ERUNTIME, "degree over cap in file");
                goto done;
            }
            ix->degree[u] = deg;
            ix->total_edges += deg;
            for (uint32_t j = 0; j < deg; ++j) {
                size_t s = (size_t)u * ix->maxdeg + j;
                RD(&ix->targets[s], 4);
                RD(ix->codes + s * ix->cb, ix->cb);
                RD(&ix->scalars[s * 3 + 0], 4);
                RD(&ix->scalars[s * 3 + 1], 4);
                RD(&ix->scalars[s * 3 + 2], 4);
                if (ix->targets[s] >= n) {
                    rc = fail(PAGO_ERUNTIME, "edge target out of range in file");
                    goto done;
                }
            }
        }
        ix->rows = (float*)malloc(sizeof(float) * (n ? n : 1) * ix->padded);
        ix->norms = (float*)malloc(sizeof(float) * (n ? n : 1));
        if (!ix->rows || !ix->norms) {
            rc = fail(PAGO_ENOMEM, "out of host memory");
            goto done;
        }
        RD(ix->rows, sizeof(float) * n * ix->padded);
        RD(ix->norms, sizeof(float) * n);
    }
#undef RD
done:
    fclose(f);
    if (rc) {
        pago_free(ix);
        return rc;
    }
    *out = ix;
    return PAGO_OK;
}

void pago_info(const pago_index* ix, uint64_t* info) {
    info[0] = ix->n;
    info[1] = ix->dim;
    info[2] = ix->padded;
    info[3] = ix->L;
    info[4] = ix->m;
    info[5] = ix->M;
    info[6] = ix->metric;
    info[7] = ix->n_entries;
    info[8] = ix->seed;
    info[9] = ix->total_edges;
}
const float* pago_refs(const pago_index* ix) { return ix->refs; }
const uint32_t* pago_entry_nodes(const pago_index* ix) { return ix->entries; }
uint32_t pago_degree(const pago_index* ix, uint32_t u) { return ix->degree[u]; }
const uint32_t* pago_targets(const pago_index* ix, uint32_t u) {
    return ix->targets + (size_t)u * ix->maxdeg;
}
const float* pago_scalars(const pago_index* ix, uint32_t u) {
    return ix->scalars + (size_t)u * ix->maxdeg * 3;
}
const uint8_t* pago_codes(const pago_index* ix, uint32_t u) {
    return ix->codes + (size_t)u * ix->maxdeg * ix->cb;
}
const float* pago_row(const pago_index* ix, uint32_t i) { return ix->rows + (size_t)i * ix->padded; }

/* ------------------------------------------------------------------------ */
/* L2 TfbState: proj/include/pag/routing.hpp:62-161, proj/src/routing.cpp    */
/* ------------------------------------------------------------------------ */

typedef struct {
    uint32_t id;
    float sq;
} cand;

static int cand_less(cand a, cand b) { /* builder.hpp:23-25 */
    return a.sq < b.sq || (a.sq == b.sq && a.id < b.id);
}

static int cand_cmp(const void* pa, const void* pb) {
    cand a = *(const cand*)pa, b = *(const cand*)pb;
    return cand_less(a, b) ? -1 : (cand_less(b, a) ? 1 : 0);
}

typedef struct {
    uint32_t id;
    float sq;
    int visited;
} went;

typedef struct { /* routing.hpp:72-96: FIFO, overwrite-oldest */
    uint32_t cap;
    cand* buf;
    size_t head, size;
} ring;

static void ring_reset(ring* r, uint32_t cap) {
    free(r->buf);
    r->cap = cap;
    r->buf = (cand*)calloc(cap ? cap : 1, sizeof(cand));
    r->head = r->size = 0;
}
static void ring_push(ring* r, cand c) {
    r->buf[(r->head + r->size) % r->cap] = c;
    if (r->size < r->cap)
        ++r->size;
    else
        r->head = (r->head + 1) % r->cap;
}
static cand ring_at(const ring* r, size_t i) { return r->buf[(r->head + i) % r->cap]; }

struct pago_tfb {
    uint32_t b, capR, round;
    went* W;
    size_t wsize;
    ring rf, rt;
    cand* R;
    size_t rsize;
    float zmax_sq, zmax_dist;
    size_t zmax_idx;
    uint32_t* marks;
    size_t n_marks;
    uint32_t epoch;
    cand* merge;
    float* table;
};

/* routing.cpp:12-30 */
static void tfb_reset(struct pago_tfb* st, size_t n_nodes, uint32_t b, uint32_t cap_R) {
    st->b = b;
    st->capR = cap_R;
    st->round = 0;
    free(st->W);
    st->W = (went*)calloc(b ? b : 1, sizeof(went));
    st->wsize = 0;
    ring_reset(&st->rf, b);
    ring_reset(&st->rt, b);
    free(st->R);
    st->R = (cand*)calloc(cap_R ? cap_R : 1, sizeof(cand));
    st->rsize = 0;
    free(st->merge);
    st->merge = (cand*)calloc(2 * (size_t)b + 1, sizeof(cand));
    st->zmax_sq = st->zmax_dist = 0;
    st->zmax_idx = 0;
    if (st->n_marks < n_nodes) {
        st->marks = (uint32_t*)realloc(st->marks, n_nodes * sizeof(uint32_t));
        memset(st->marks + st->n_marks, 0, (n_nodes - st->n_marks) * sizeof(uint32_t));
        st->n_marks = n_nodes;
    }
    if (st->epoch == 0xFFFFFFFFu) {
        memset(st->marks, 0, st->n_marks * sizeof(uint32_t));
        st->epoch = 0;
    }
    ++st->epoch;
}

static int tfb_marked(const struct pago_tfb* st, uint32_t id) { return st->marks[id] == st->epoch; }
static void tfb_mark(struct pago_tfb* st, uint32_t id) { st->marks[id] = st->epoch; }

static float tfb_admission_sq(const struct pago_tfb* st) { /* routing.hpp:116-118 */
    return st->wsize < st->b ? INFINITY : st->zmax_sq;
}
static float tfb_admission_dist(const struct pago_tfb* st) { /* routing.hpp:119-121 */
    return st->wsize < st->b ? INFINITY : st->zmax_dist;
}

/* routing.cpp:32-44 — first max wins (strict >) */
static void tfb_recompute_zmax(struct pago_tfb* st) {
    if (st->wsize == 0) {
        st->zmax_sq = st->zmax_dist = 0;
        st->zmax_idx = 0;
        return;
    }
    size_t best = 0;
    for (size_t i = 1; i < st->wsize; ++i)
        if (st->W[i].sq > st->W[best].sq) best = i;
    st->zmax_idx = best;
    st->zmax_sq = st->W[best].sq;
    st->zmax_dist = sqrtf(st->zmax_sq);
}

/* routing.cpp:46-53 */
static void tfb_seed(struct pago_tfb* st, uint32_t id, float sq) {
    st->W[st->wsize++] = (went){id, sq, 0};
    if (sq > st->zmax_sq || st->wsize == 1) {
        st->zmax_idx = st->wsize - 1;
        st->zmax_sq = sq;
        st->zmax_dist = sqrtf(sq);
    }
}

/* routing.cpp:55-69 */
static void tfb_admit(struct pago_tfb* st, uint32_t id, float sq) {
    if (st->wsize < st->b) {
        st->W[st->wsize++] = (went){id, sq, 0};
        if (sq > st->zmax_sq || st->wsize == 1) {
            st->zmax_idx = st->wsize - 1;
            st->zmax_sq = sq;
            st->zmax_dist = sqrtf(sq);
        }
        return;
    }
    went* slot = &st->W[st->zmax_idx];
    ring_push(&st->rt, (cand){slot->id, slot->sq});
    *slot = (went){id, sq, 0};
    tfb_recompute_zmax(st);
}

/* routing.cpp:71-80 — argmin over unvisited by (sq, id) */
static int64_t tfb_next_unvisited(const struct pago_tfb* st) {
    int64_t best = -1;
    for (size_t i = 0; i < st->wsize; ++i) {
        if (st->W[i].visited) continue;
        if (best < 0 || st->W[i].sq < st->W[best].sq ||
            (st->W[i].sq == st->W[best].sq && st->W[i].id < st->W[best].id))
            best = (int64_t)i;
    }
    return best;
}

/* routing.cpp:82-90 — bounded sorted insert, capacity cap_R */
static void tfb_push_result(struct pago_tfb* st, cand c) {
    size_t lo = 0, hi = st->rsize; /* lower_bound */
    while (lo < hi) {
        size_t mid = (lo + hi) / 2;
        if (cand_less(st->R[mid], c))
            lo = mid + 1;
        else
            hi = mid;
    }
    size_t pos = lo;
    if (st->rsize >= st->capR) {
        if (pos == st->rsize) return;
        --st->rsize; /* pop_back; pos is unchanged by a re-search */
    }
    memmove(st->R + pos + 1, st->R + pos, (st->rsize - pos) * sizeof(cand));
    st->R[pos] = c;
    ++st->rsize;
}

/* routing.cpp:92-114 */
static int tfb_end_round(struct pago_tfb* st) {
    for (size_t i = 0; i < st->wsize; ++i) tfb_push_result(st, (cand){st->W[i].id, st->W[i].sq});
    st->wsize = 0;
    size_t nm = 0;
    for (size_t i = 0; i < st->rf.size; ++i) st->merge[nm++] = ring_at(&st->rf, i);
    for (size_t i = 0; i < st->rt.size; ++i) st->merge[nm++] = ring_at(&st->rt, i);
    st->rf.head = st->rf.size = 0;
    st->rt.head = st->rt.size = 0;
    qsort(st->merge, nm, sizeof(cand), cand_cmp);
    ++st->round;
    if (nm == 0) {
        st->zmax_sq = st->zmax_dist = 0;
        return 0;
    }
    size_t refill = nm < st->b ? nm : st->b;
    for (size_t i = 0; i < refill; ++i) st->W[st->wsize++] = (went){st->merge[i].id, st->merge[i].sq, 0};
    for (size_t i = refill; i < nm; ++i) ring_push(&st->rt, st->merge[i]);
    tfb_recompute_zmax(st);
    return 1;
}

typedef struct {
    uint64_t exact, test, pass, visited, edges;
} stats5;

/* routing.cpp:139-204. With collect_pes (the construction search,
   builder.cpp:218-224) the PES margin of every edge is tracked
   (routing.cpp:150,190-199) and the return value is out.pes_rejected. */
static int expand_node(size_t work_idx, struct pago_tfb* st, const pago_index* ix, const float* q,
                       int use_prt, int collect_pes, stats5* stats) {
    went* entry = &st->W[work_idx];
    entry->visited = 1;
    ++stats->visited;
    const uint32_t u = entry->id;
    const float dist_uq = sqrtf(entry->sq);
    const int exact_mode = (dist_uq == 0.0f) || !use_prt;
    const int track_pes = collect_pes && dist_uq > 0.0f;
    float pes_max = -INFINITY;
    const uint32_t deg = ix->degree[u];
    const uint32_t* tg = ix->targets + (size_t)u * ix->maxdeg;
    const float* sc = ix->scalars + (size_t)u * ix->maxdeg * 3;
    stats->edges += deg;
    for (uint32_t j = 0; j < deg; ++j) {
        const uint32_t w = tg[j];
        const float cos_beta = sc[3 * j + 0], edge_norm = sc[3 * j + 1], base_off = sc[3 * j + 2];
        const uint8_t* codes = ix->codes + ((size_t)u * ix->maxdeg + j) * ix->cb;
        float quot = 0.0f;
        int have_quot = 0;
        if (!tfb_marked(st, w)) {
            ++stats->test;
            int pass;
            if (exact_mode) {
                pass = 1;
            } else {
                float tau = pago_prt_threshold(edge_norm, dist_uq, tfb_admission_dist(st));
                if (tau >= 1.0f + 1e-6f) {
                    pass = 0;
                } else if (tau <= -1.0f) {
                    pass = 1;
                } else {
                    /* projection.hpp:71-74 */
                    quot = ((pago_table_code_sum(st->table, ix->L, ix->m, codes) - base_off) /
                            dist_uq) /
                           cos_beta;
                    have_quot = 1;
                    pass = quot >= tau;
                }
            }
            if (pass) {
                ++stats->pass;
                float sq = row_dist(ix, w, q);
                ++stats->exact;
                tfb_mark(st, w);
                if (sq < tfb_admission_sq(st))
                    tfb_admit(st, w, sq);
                else
                    ring_push(&st->rf, (cand){w, sq});
            }
        }
        if (track_pes) { /* routing.cpp:190-199, std::max(pes_max, quot - delta) */
            if (!have_quot)
                quot = ((pago_table_code_sum(st->table, ix->L, ix->m, codes) - base_off) /
                        dist_uq) /
                       cos_beta;
            const float delta = edge_norm / (2.0f * dist_uq);
            const float x = quot - delta;
            if (pes_max < x) pes_max = x;
        }
    }
    return track_pes && pes_max < 0.0f;
}

/* routing.cpp:206-247 */
static int search_padded(const pago_index* ix, const float* q, uint32_t K, uint32_t efS,
                         uint32_t b_override, int use_prt, int use_tfb, int collect_pes,
                         struct pago_tfb* st, uint32_t* ids, float* sq, uint32_t* n_out,
                         stats5* stats, uint32_t* pes, uint32_t pes_cap, uint32_t* pes_n) {
    uint32_t npes = 0;
    const uint32_t n = (uint32_t)ix->n;
    const uint32_t bdef = b_override ? b_override : (K > 10u ? K : 10u);
    const uint32_t b = use_tfb ? bdef : (efS > bdef ? efS : bdef);
    const uint32_t r_max = use_tfb ? (efS + b - 1) / b : 1;
    tfb_reset(st, n, b, efS);
    pago_build_projection_table(q, ix->refs, ix->L, ix->m, ix->sub_dim, st->table);

    for (uint32_t e = 0; e < ix->n_entries; ++e) {
        uint32_t id = ix->entries[e];
        if (st->wsize >= b) break;
        if (id >= n || tfb_marked(st, id)) continue;
        float s = row_dist(ix, id, q);
        ++stats->exact;
        tfb_mark(st, id);
        tfb_seed(st, id, s);
    }
    for (uint32_t r = 0; r < r_max; ++r) {
        int64_t i;
        while ((i = tfb_next_unvisited(st)) >= 0) {
            const uint32_t u = st->W[i].id;
            if (expand_node((size_t)i, st, ix, q, use_prt, collect_pes, stats)) { /* :235 */
                if (npes < pes_cap) pes[npes] = u;
                ++npes;
            }
        }
        if (r + 1 == r_max || !tfb_end_round(st)) break;
    }
    for (size_t i = 0; i < st->wsize; ++i) tfb_push_result(st, (cand){st->W[i].id, st->W[i].sq});
    size_t k = K < st->rsize ? K : st->rsize;
    for (size_t i = 0; i < k; ++i) {
        ids[i] = st->R[i].id;
        sq[i] = st->R[i].sq;
    }
    *n_out = (uint32_t)k;
    if (pes_n) *pes_n = npes;
    return PAGO_OK;
}

/* routing.cpp:249-261: pad, cosine-normalise by division */
static int prep_query(const pago_index* ix, const float* qraw, float* qbuf) {
    memset(qbuf, 0, sizeof(float) * ix->padded);
    memcpy(qbuf, qraw, sizeof(float) * ix->dim);
    if (ix->metric == 1) {
        float nrm = pago_vec_norm(qbuf, ix->padded);
        if (nrm == 0.0f) return fail(PAGO_EINVAL, "zero query under cosine metric");
        for (uint32_t k = 0; k < ix->padded; ++k) qbuf[k] /= nrm;
    }
    return PAGO_OK;
}

int pago_search(const pago_index* ix, const float* q, uint64_t nq, uint32_t K, uint32_t efS,
                uint32_t b_override, int use_prt, int use_tfb, uint32_t* ids, float* sq,
                uint32_t* n_out, uint64_t* stats) {
    if (ix->n == 0) return fail(PAGO_ERUNTIME, "search on empty index");
    if (K > efS) return fail(PAGO_EINVAL, "K > efS");
    struct pago_tfb st;
    memset(&st, 0, sizeof st);
    st.table = (float*)malloc(sizeof(float) * (size_t)ix->L * (ix->m ? ix->m : 1));
    float* qbuf = (float*)malloc(sizeof(float) * ix->padded);
    int rc = PAGO_OK;
    for (uint64_t i = 0; i < nq; ++i) {
        rc = prep_query(ix, q + i * ix->dim, qbuf);
        if (rc) break;
        stats5 s = {0, 0, 0, 0, 0};
        search_padded(ix, qbuf, K, efS, b_override, use_prt, use_tfb, 0, &st, ids + i * K,
                      sq + i * K, n_out + i, &s, NULL, 0, NULL);
        if (stats) {
            stats[i * 5 + 0] = s.exact;
            stats[i * 5 + 1] = s.test;
            stats[i * 5 + 2] = s.pass;
            stats[i * 5 + 3] = s.visited;
            stats[i * 5 + 4] = s.edges;
        }
    }
    free(qbuf);
    free(st.table);
    free(st.W);
    free(st.rf.buf);
    free(st.rt.buf);
    free(st.R);
    free(st.merge);
    free(st.marks);
    return rc;
}

/* insert_with_state's search (builder.cpp:218-227): the query is the node's
   own stored (padded, already normalised) row, passed to search_padded
   directly; SearchResult.pes_rejected (routing.hpp:176) per node, at most
   pes_cap ids kept, pes_n = the full count. */
int pago_construction_search(const pago_index* ix, const uint32_t* nodes, uint64_t nn, uint32_t K,
                             uint32_t efS, uint32_t b_override, int collect_pes, uint32_t* ids,
                             float* sq, uint32_t* n_out, uint64_t* stats, uint32_t* pes,
                             uint32_t pes_cap, uint32_t* pes_n) {
    if (ix->n == 0) return fail(PAGO_ERUNTIME, "search on empty index");
    if (K > efS) return fail(PAGO_EINVAL, "K > efS");
    for (uint64_t i = 0; i < nn; ++i)
        if (nodes[i] >= ix->n) return fail(PAGO_EINVAL, "node id out of range");
    struct pago_tfb st;
    memset(&st, 0, sizeof st);
    st.table = (float*)malloc(sizeof(float) * (size_t)ix->L * (ix->m ? ix->m : 1));
    for (uint64_t i = 0; i < nn; ++i) {
        stats5 s = {0, 0, 0, 0, 0};
        search_padded(ix, ix->rows + (size_t)nodes[i] * ix->padded, K, efS, b_override, 1, 1,
                      collect_pes, &st, ids + i * K, sq + i * K, n_out + i, &s,
                      pes + i * pes_cap, pes_cap, pes_n + i);
        if (stats) {
            stats[i * 5 + 0] = s.exact;
            stats[i * 5 + 1] = s.test;
            stats[i * 5 + 2] = s.pass;
            stats[i * 5 + 3] = s.visited;
            stats[i * 5 + 4] = s.edges;
        }
    }
    free(st.table);
    free(st.W);
    free(st.rf.buf);
    free(st.rt.buf);
    free(st.R);
    free(st.merge);
    free(st.marks);
    return PAGO_OK;
}

void pago_build_params(const pago_index* ix, uint32_t* out) {
    out[0] = ix->efC;
    out[1] = ix->b_build;
    out[2] = ix->enable_pes;
    out[3] = ix->pes_flush;
}

int pago_query_table(const pago_index* ix, const float* q, float* out) {
    float* qbuf = (float*)malloc(sizeof(float) * ix->padded);
    int rc = prep_query(ix, q, qbuf);
    if (!rc) pago_build_projection_table(qbuf, ix->refs, ix->L, ix->m, ix->sub_dim, out);
    free(qbuf);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* L4 ground truth + recall: proj/src/bench.cpp:18-71                        */
/* ------------------------------------------------------------------------ */

static void heap_sift_down(cand* h, size_t n, size_t i) { /* max-heap by cand_less */
    for (;;) {
        size_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < n && cand_less(h[m], h[l])) m = l;
        if (r < n && cand_less(h[m], h[r])) m = r;
        if (m == i) return;
        cand t = h[i];
        h[i] = h[m];
        h[m] = t;
        i = m;
    }
}

/* bench.cpp:18-53: exact top-k by (sq, id); k = min(k_star, n). The strict
 * total order makes the kept set identical to partial_sort's. */
int pago_ground_truth(const float* base, uint64_t n, const float* queries, uint64_t nq,
                      uint32_t padded_dim, uint32_t k_star, uint32_t* ids, float* sq) {
    uint64_t k = k_star < n ? k_star : n;
    cand* h = (cand*)malloc(sizeof(cand) * (k ? k : 1));
    for (uint64_t qi = 0; qi < nq; ++qi) {
        const float* q = queries + qi * padded_dim;
        size_t hs = 0;
        for (uint64_t i = 0; i < n && k; ++i) {
            cand c = {(uint32_t)i, pago_sq_dist(base + i * padded_dim, q, padded_dim)};
            if (hs < k) {
                h[hs++] = c;
                if (hs == k)
                    for (size_t j = k / 2 + 1; j-- > 0;) heap_sift_down(h, hs, j);
            } else if (cand_less(c, h[0])) {
                h[0] = c;
                heap_sift_down(h, hs, 0);
            }
        }
        qsort(h, hs, sizeof(cand), cand_cmp);
        for (size_t j = 0; j < hs; ++j) {
            ids[qi * k_star + j] = h[j].id;
            sq[qi * k_star + j] = h[j].sq;
        }
    }
    free(h);
    return PAGO_OK;
}

/* bench.cpp:55-71: distance-tied ids count as hits */
double pago_recall_at_k(const uint32_t* result_ids, size_t n_result, const uint32_t* truth_ids,
                        const float* truth_sq, size_t truth_len, uint32_t K) {
    size_t k = K < truth_len ? K : truth_len;
    if (k == 0) return 0.0;
    const float tie_sq = truth_sq[k - 1];
    size_t hits = 0;
    size_t limit = K < n_result ? K : n_result;
    for (size_t i = 0; i < limit; ++i) {
        for (size_t t = 0; t < truth_len; ++t) {
            if (truth_ids[t] == result_ids[i]) { /* first occurrence, as unordered_map::emplace */
                if (truth_sq[t] <= tie_sq) ++hits;
                break;
            }
        }
    }
    return (double)hits / K;
}

/* ------------------------------------------------------------------------ */
/* KAT hooks                                                                 */
/* ------------------------------------------------------------------------ */

pago_tfb* pago_tfb_new(size_t n_nodes, uint32_t b, uint32_t cap_R) {
    pago_tfb* st = (pago_tfb*)calloc(1, sizeof *st);
    tfb_reset(st, n_nodes, b, cap_R);
    return st;
}
void pago_tfb_free(pago_tfb* st) {
    if (!st) return;
    free(st->W);
    free(st->rf.buf);
    free(st->rt.buf);
    free(st->R);
    free(st->merge);
    free(st->marks);
    free(st->table);
    free(st);
}
void pago_tfb_seed(pago_tfb* st, uint32_t id, float sq) { tfb_seed(st, id, sq); }
void pago_tfb_admit(pago_tfb* st, uint32_t id, float sq) { tfb_admit(st, id, sq); }
void pago_tfb_push_fp(pago_tfb* st, uint32_t id, float sq) { ring_push(&st->rf, (cand){id, sq}); }
void pago_tfb_push_result(pago_tfb* st, uint32_t id, float sq) { tfb_push_result(st, (cand){id, sq}); }
int pago_tfb_end_round(pago_tfb* st) { return tfb_end_round(st); }
int64_t pago_tfb_next_unvisited(const pago_tfb* st) { return tfb_next_unvisited(st); }
void pago_tfb_set_visited(pago_tfb* st, size_t i, int v) { st->W[i].visited = v; }
float pago_tfb_admission_sq(const pago_tfb* st) { return tfb_admission_sq(st); }
float pago_tfb_admission_dist(const pago_tfb* st) { return tfb_admission_dist(st); }

size_t pago_tfb_dump(const pago_tfb* st, int which, uint32_t* ids, float* sq, uint8_t* visited,
                     size_t cap) {
    size_t n = 0;
    if (which == 0) {
        for (; n < st->wsize && n < cap; ++n) {
            ids[n] = st->W[n].id;
            sq[n] = st->W[n].sq;
            if (visited) visited[n] = (uint8_t)st->W[n].visited;
        }
    } else if (which == 1 || which == 2) {
        const ring* r = which == 1 ? &st->rf : &st->rt;
        for (; n < r->size && n < cap; ++n) {
            cand c = ring_at(r, n);
            ids[n] = c.id;
            sq[n] = c.sq;
        }
    } else {
        for (; n < st->rsize && n < cap; ++n) {
            ids[n] = st->R[n].id;
            sq[n] = st->R[n].sq;
        }
    }
    return n;
}

/* routing.cpp:116-137 */
int pago_tfb_validate(const pago_tfb* st) {
    if (st->rf.cap != st->b || st->rt.cap != st->b)
        return fail(PAGO_ELOGIC, "TFB: ring capacity != b");
    if (st->wsize > st->b) return fail(PAGO_ELOGIC, "TFB: working set over capacity");
    if (st->rsize > st->capR) return fail(PAGO_ELOGIC, "TFB: result list over capacity");
    if (st->wsize) {
        float mx = st->W[0].sq;
        for (size_t i = 0; i < st->wsize; ++i) mx = st->W[i].sq > mx ? st->W[i].sq : mx;
        if (mx != st->zmax_sq) return fail(PAGO_ELOGIC, "TFB: stale z_max");
    }
    size_t total = st->wsize + st->rf.size + st->rt.size + st->rsize, n = 0;
    uint32_t* all = (uint32_t*)malloc(sizeof(uint32_t) * (total ? total : 1));
    for (size_t i = 0; i < st->wsize; ++i) all[n++] = st->W[i].id;
    for (size_t i = 0; i < st->rf.size; ++i) all[n++] = ring_at(&st->rf, i).id;
    for (size_t i = 0; i < st->rt.size; ++i) all[n++] = ring_at(&st->rt, i).id;
    for (size_t i = 0; i < st->rsize; ++i) all[n++] = st->R[i].id;
    int dup = 0;
    for (size_t i = 0; i < n && !dup; ++i)
        for (size_t j = i + 1; j < n; ++j)
            if (all[i] == all[j]) {
                dup = 1;
                break;
            }
    free(all);
    if (dup) return fail(PAGO_ELOGIC, "TFB: duplicate node residence");
    for (size_t i = 1; i < st->rsize; ++i)
        if (cand_less(st->R[i], st->R[i - 1])) return fail(PAGO_ELOGIC, "TFB: result list out of order");
    return PAGO_OK;
}

size_t pago_ring_kat(uint32_t cap, const uint32_t* ids, const float* sq, size_t n,
                     uint32_t* out_ids) {
    ring r = {0, NULL, 0, 0};
    ring_reset(&r, cap);
    for (size_t i = 0; i < n; ++i) ring_push(&r, (cand){ids[i], sq[i]});
    for (size_t i = 0; i < r.size; ++i) out_ids[i] = ring_at(&r, i).id;
    size_t s = r.size;
    free(r.buf);
    return s;
}
