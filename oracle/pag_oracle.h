/*
 * pag_oracle.h — CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the reference PAG query path
 * (/root/reference/proj/src/{routing,projection,vecstore,builder,bench}.cpp),
 * used ONLY by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
 * as the checker. It is never linked into, called by, or shipped with the
 * product library (paper_2603_06660_b200/csrc).
 *
 * Parity is pinned two ways (see tests/test_oracle.py):
 *   - bit-exact against the reference itself, compiled from its own sources
 *     into oracle/_ref/pag_ref by oracle/Makefile (ids, squared distances,
 *     counters, projection tables, reference family);
 *   - the reference's recorded golden recall / gamma values on the acceptance
 *     fixture (proj/test_output.txt:8,12) and its unit-test KATs
 *     (proj/tests/test_routing.cpp, test_projection.cpp, test_bench.cpp).
 */
#ifndef PAG_ORACLE_H
#define PAG_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pago_index pago_index;
typedef struct pago_tfb pago_tfb;

/* status codes (shared meaning with include/pag_gpu.h) */
#define PAGO_OK 0
#define PAGO_EINVAL 1   /* std::invalid_argument in the reference */
#define PAGO_ERUNTIME 2 /* std::runtime_error */
#define PAGO_ELOGIC 3   /* std::logic_error */
#define PAGO_ENOMEM 4

const char* pago_last_error(void);

/* ---- L0: distances (vecstore.cpp:77-108) ---- */
float pago_sq_dist(const float* a, const float* b, size_t padded_dim);
float pago_vec_norm(const float* a, size_t padded_dim);

/* ---- L1: reference family, table, estimator (projection.cpp) ---- */
uint32_t pago_default_subspace_count(uint32_t dim);
/* out: L*m*(padded_dim/L) floats */
int pago_build_reference_set(uint32_t padded_dim, uint32_t L, uint32_t m, uint64_t seed,
                             float* out);
void pago_build_projection_table(const float* x, const float* refs, uint32_t L, uint32_t m,
                                 uint32_t sub_dim, float* out);
float pago_table_code_sum(const float* table, uint32_t L, uint32_t m, const uint8_t* codes);
uint32_t pago_code_at(const uint8_t* codes, uint32_t l);
void pago_set_code(uint8_t* codes, uint32_t l, uint32_t j);
int pago_prt_test(float cos_theta, float cos_beta, float tau);
float pago_prt_threshold(float edge_norm, float dist_uv, float dist_zmax_v);

/* libstdc++ RNG restatement (mt19937_64 + normal_distribution<double>) */
void pago_mt64_stream(uint64_t seed, uint64_t* out, size_t n);
void pago_normal_stream(uint64_t seed, double* out, size_t n);

/* ---- L3: PAGIDX01 v1 file (builder.cpp:389-492) ---- */
int pago_load(const char* path, pago_index** out);
void pago_free(pago_index* ix);
/* info[0..9] = n, dim, padded, L, m, M, metric, n_entries, seed, total_edges */
void pago_info(const pago_index* ix, uint64_t* info);
const float* pago_refs(const pago_index* ix);
const uint32_t* pago_entry_nodes(const pago_index* ix);
uint32_t pago_degree(const pago_index* ix, uint32_t u);
const uint32_t* pago_targets(const pago_index* ix, uint32_t u);
/* scalars as {cos_beta, edge_norm, base_offset} triples */
const float* pago_scalars(const pago_index* ix, uint32_t u);
const uint8_t* pago_codes(const pago_index* ix, uint32_t u);
const float* pago_row(const pago_index* ix, uint32_t i);

/* ---- L2: search (routing.cpp:139-261) ----
 * q: nq x dim raw query rows. ids/sq: nq x K. n_out: nq.
 * stats: nq x 5 {exact_dist_count, test_count, pass_count, visited_count,
 *               edges_scanned}. edges_scanned (sum of deg over expansions) is
 * an extra counter for the algorithmic-bytes model; it does not alter the
 * algorithm. */
/* 0: reference-order sq_dist (vecstore.cpp:77-95, default); 1: the B200
 * library's warp-tree order (its exact_dist = 0 mode), for checking that mode
 * bit for bit. Applies to the search and the construction search. */
void pago_set_distance_mode(pago_index* ix, int mode);
int pago_search(const pago_index* ix, const float* q, uint64_t nq, uint32_t K, uint32_t efS,
                uint32_t b_override, int use_prt, int use_tfb, uint32_t* ids, float* sq,
                uint32_t* n_out, uint64_t* stats);
/* Construction search (builder.cpp:218-227 insert_with_state): query = the
 * stored row of nodes[i]; PES margins tracked when collect_pes
 * (routing.cpp:150,190-199). pes: nn x pes_cap expanded node ids whose PES
 * max was negative, in expansion order (routing.cpp:235); pes_n: full count
 * per node (entries beyond pes_cap are counted, not stored). */
int pago_construction_search(const pago_index* ix, const uint32_t* nodes, uint64_t nn, uint32_t K,
                             uint32_t efS, uint32_t b_override, int collect_pes, uint32_t* ids,
                             float* sq, uint32_t* n_out, uint64_t* stats, uint32_t* pes,
                             uint32_t pes_cap, uint32_t* pes_n);
/* out[0..3] = efC, b_build, enable_pes, pes_flush_interval from the header */
void pago_build_params(const pago_index* ix, uint32_t* out);
/* projection table of one raw query (after the same pad/normalise as search) */
int pago_query_table(const pago_index* ix, const float* q, float* out);

/* ---- L4: ground truth + recall (bench.cpp:18-71) ---- */
int pago_ground_truth(const float* base, uint64_t n, const float* queries, uint64_t nq,
                      uint32_t padded_dim, uint32_t k_star, uint32_t* ids, float* sq);
double pago_recall_at_k(const uint32_t* result_ids, size_t n_result, const uint32_t* truth_ids,
                        const float* truth_sq, size_t truth_len, uint32_t K);

/* ---- TfbState hooks for the reference's KATs (routing.hpp:62-161) ---- */
pago_tfb* pago_tfb_new(size_t n_nodes, uint32_t b, uint32_t cap_R);
void pago_tfb_free(pago_tfb* st);
void pago_tfb_seed(pago_tfb* st, uint32_t id, float sq);
void pago_tfb_admit(pago_tfb* st, uint32_t id, float sq);
void pago_tfb_push_fp(pago_tfb* st, uint32_t id, float sq);
void pago_tfb_push_result(pago_tfb* st, uint32_t id, float sq);
int pago_tfb_end_round(pago_tfb* st);
int64_t pago_tfb_next_unvisited(const pago_tfb* st);
void pago_tfb_set_visited(pago_tfb* st, size_t i, int v);
float pago_tfb_admission_sq(const pago_tfb* st);
float pago_tfb_admission_dist(const pago_tfb* st);
/* which: 0 = working (id, sq, visited), 1 = ring_f, 2 = ring_t, 3 = result.
 * Writes up to cap entries; returns the count. */
size_t pago_tfb_dump(const pago_tfb* st, int which, uint32_t* ids, float* sq, uint8_t* visited,
                     size_t cap);
int pago_tfb_validate(const pago_tfb* st);

/* standalone ring (routing.hpp:72-96) for the overwrite KAT */
size_t pago_ring_kat(uint32_t cap, const uint32_t* ids, const float* sq, size_t n,
                     uint32_t* out_ids);

#ifdef __cplusplus
}
#endif
#endif
