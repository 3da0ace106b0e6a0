/*
 * pag_gpu.h — C ABI of the B200-native PAG query path (libpag_gpu.so).
 *
 * Drop-in boundary for the reference's C++ search API. Each entry point
 * names the reference interface it replaces (paths relative to the
 * reference repo root). Plain pointers and sizes only; every call returns a
 * status code and, on failure, leaves a thread-local message readable with
 * pag_gpu_last_error(). Message texts are the reference's exception texts.
 *
 * Status codes map the reference's exception classes:
 *   PAG_GPU_EINVAL   <- std::invalid_argument  (e.g. "K > efS",
 *                       "query dimension mismatch",
 *                       "zero query under cosine metric")
 *   PAG_GPU_ERUNTIME <- std::runtime_error     (e.g. "search on empty index",
 *                       "cannot open index: <path>", "bad index magic",
 *                       "unsupported index version", "degree over cap in file",
 *                       "index read failed")
 *   PAG_GPU_ECUDA       a CUDA runtime failure (no reference counterpart)
 */
#ifndef PAG_GPU_H
#define PAG_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PAG_GPU_OK 0
#define PAG_GPU_EINVAL 1
#define PAG_GPU_ERUNTIME 2
#define PAG_GPU_ELOGIC 3
#define PAG_GPU_ENOMEM 4
#define PAG_GPU_ECUDA 5

typedef struct pag_gpu_index pag_gpu_index;

/* Per-query counters: proj/include/pag/routing.hpp:24-34 (SearchStats)
 * plus edges_scanned = sum of deg(u) over expansions (algorithmic-bytes
 * model). */
typedef struct pag_search_stats {
    uint64_t exact_dist_count;
    uint64_t test_count;
    uint64_t pass_count;
    uint64_t visited_count;
    uint64_t edges_scanned;
} pag_search_stats;

/* Search knobs: proj/include/pag/routing.hpp:13-22 (SearchParams).
 * collect_pes (build-only) is an argument of pag_gpu_construction_search. */
typedef struct pag_search_params {
    uint32_t K;          /* default 10 */
    uint32_t efS;        /* default 100 */
    uint32_t b_override; /* 0 = max(10, K) */
    uint8_t use_prt;     /* ablation: 0 degenerates to exact expansion */
    uint8_t use_tfb;     /* ablation: 0 = one round with b = max(efS, b) */
    uint8_t exact_dist;  /* 1 (default): reference-order fp32 sq_dist, bit-identical
                            results (the first such search builds a second,
                            chain-interleaved copy of the rows in HBM);
                            0: warp-tree FMA distances (within 1e-5 rel) */
    uint8_t reserved;
} pag_search_params;

/* Fills the reference defaults (K=10, efS=100, use_prt=use_tfb=1, exact_dist=1). */
void pag_gpu_default_params(pag_search_params* p);

/* Replaces: PagIndex load_index(const std::string&)
 *           proj/include/pag/builder.hpp:157, proj/src/builder.cpp:434-492.
 * Loads a PAGIDX01 v1 file, regenerates the reference family from
 * (padded_dim, L, m, seed) (proj/src/projection.cpp:40-74) and makes the
 * graph, per-edge codes/scalars, references and base vectors resident in
 * HBM on every GPU of device_mask (bit i = CUDA device i; 0 = device 0).
 * Batches are split across those GPUs (query sharding, no collective). */
int pag_gpu_open(const char* index_path, uint32_t device_mask, pag_gpu_index** out);

/* pag_gpu_open with an explicit replica list: one full replica of the index
 * per entry of devices[0..n_devices) (CUDA device ordinals). An ordinal may
 * repeat: several replicas then share one GPU, each with its own copy,
 * stream, scratch and host worker (the multi-replica path exercised on a
 * single GPU). The file streams once over the host link into the first
 * replica; the others are filled device to device. n_devices = 0 = {0}. */
int pag_gpu_open_devices(const char* index_path, const int* devices, uint32_t n_devices, pag_gpu_index** out);

/* The reference's in-memory PagIndex (proj/include/pag/builder.hpp:62-132),
 * borrowed for the duration of a call: the source of pag_gpu_open_from_arrays
 * and pag_gpu_refresh_from_arrays, so an index the reference has just built
 * or extended (build / insert_online) reaches the GPU without a file.
 *   header        BuildParams (builder.hpp:27-36) + VectorSet dim / padded_dim / metric
 *   degrees       n x u32, a snapshot of PagIndex::degree(u) (:74-76; atomics there)
 *   targets       n x 2M u32, PagIndex::targets(0) (:77-79, fixed stride 2M)
 *   scalars       n x 2M x {cos_beta, edge_norm, base_offset} f32, scalars(0) (:38-42,80-82)
 *   codes         n x 2M x ceil(L/2) bytes, edge_codes(0, 0) (:83-85)
 *   rows          n x padded_dim f32, vectors().row(0) (vecstore.hpp:38)
 *   norms         n cached norms (vecstore.hpp:39) or NULL (computed from the rows)
 * L is the resolved subspace count (refs().L), or 0 for the dimension default. */
typedef struct pag_index_arrays {
    uint64_t n;
    uint32_t dim, padded_dim, L, m, M, efC, b_build, pes_flush_interval;
    uint64_t seed;
    uint8_t metric;      /* 0 euclidean, 1 cosine */
    uint8_t enable_pes;
    uint8_t reserved[2];
    uint32_t n_entries;
    const uint32_t* entry_nodes;
    const uint32_t* degrees;
    const uint32_t* targets;
    const float* scalars;
    const uint8_t* codes;
    const float* rows;
    const float* norms;
} pag_index_arrays;

/* pag_gpu_open_devices with the in-memory arrays as the source (same
 * validation and errors as the file path; nothing of `a` is kept). */
int pag_gpu_open_from_arrays(const pag_index_arrays* a, const int* devices, uint32_t n_devices,
                             pag_gpu_index** out);

/* pag_gpu_refresh with the in-memory arrays as the newer state (after
 * insert_online batches on the PagIndex the GPU index was opened from). */
int pag_gpu_refresh_from_arrays(pag_gpu_index* ix, const pag_index_arrays* a, uint64_t* stats);

/* Releases every device replica (the PagIndex destructor). */
int pag_gpu_close(pag_gpu_index* ix);

/* info[0..11] = n, dim, padded_dim, L, m, M, metric (0 euclidean, 1 cosine),
 * n_entries, seed, total_edges, n_devices, device_bytes_per_replica (grows
 * by one more copy of the rows at the first reference-order search);
 * info[12] = tensor-core ground-truth queries re-run exactly so far;
 * info[13..15] = the header's efC, b_build, enable_pes;
 * info[16] = nodes that repeat a target inside one 32-edge group (0 lets
 * the search skip its in-group duplicate resolution).
 * Replaces the PagIndex/VectorSet accessors (builder.hpp:71-91). */
int pag_gpu_info(const pag_gpu_index* ix, uint64_t* info, size_t n_info);

/* Replaces: SearchResult search(const PagIndex&, std::span<const float> q,
 *                                const SearchParams&, TfbState&)
 *           proj/include/pag/routing.hpp:181-184, proj/src/routing.cpp:249-261,
 * batched over nq queries. q: nq x dim raw host rows (padding and cosine
 * normalisation happen exactly as routing.cpp:253-259). Outputs (host):
 * ids/sq nq x K (the first n_out[i] entries valid, (sq, id) ascending,
 * squared distances), n_out nq, stats nq (may be NULL). Same validation and
 * messages as the reference; a zero query under cosine fails the call. */
int pag_gpu_search(pag_gpu_index* ix, const float* q, uint64_t nq,
                   const pag_search_params* params, uint32_t* ids, float* sq,
                   uint32_t* n_out, pag_search_stats* stats);

/* Same engine with every buffer already on device 0 of the handle
 * (q_dev: nq x dim fp32, ids/sq: nq x K, n_out: nq, stats_dev: nq x 8 u32
 * raw counters {exact,test,pass,visited,edges,status,marks,0}), launched on
 * `stream` (a cudaStream_t; NULL = the legacy default stream) without host
 * synchronisation. For resident-input throughput measurement and for
 * callers that keep queries on the GPU. Consecutive launches on one stream
 * overlap (programmatic dependent launch); a launch on a different stream
 * than the handle's previous one first waits for that stream's work (an
 * event recorded there at the switch), so a caller stream must stay valid
 * until the handle's next launch on another stream or its close. */
int pag_gpu_search_device(pag_gpu_index* ix, const float* q_dev, uint64_t nq,
                          const pag_search_params* params, uint32_t* ids_dev, float* sq_dev,
                          uint32_t* n_out_dev, uint32_t* stats_dev, void* stream);

/* Asynchronous pag_gpu_search: enqueues the batch and returns a ticket; the
 * results land in the caller's ids / sq / n_out / stats when
 * pag_gpu_search_wait(ticket) returns (host buffers must stay valid until
 * then). Queries in pinned host memory are read by the kernel in place;
 * pageable ones are copied at submit. Up to 4 batches are in flight per GPU
 * (a 5th submit first completes the oldest); consecutive batches overlap on
 * the GPU like back-to-back pag_gpu_search_device calls. Errors of a batch
 * (e.g. "zero query under cosine metric") are reported by that batch's own
 * wait, also when a later submit completed it to free its ring slot. A
 * submit that fails launches nothing that outlives it. Calls on one handle
 * serialise; a handle with several replicas splits each batch into one
 * contiguous shard per replica. */
int pag_gpu_search_submit(pag_gpu_index* ix, const float* q, uint64_t nq, const pag_search_params* params,
                          uint32_t* ids, float* sq, uint32_t* n_out, pag_search_stats* stats, uint64_t* ticket);
int pag_gpu_search_wait(pag_gpu_index* ix, uint64_t ticket);

/* Construction search. Replaces the search step of
 *   insert_with_state(PagIndex&, uint32_t v, PesSet&, TfbState&)
 *   proj/src/builder.cpp:218-227 — search_padded(index, vectors().row(v), sp)
 *   with sp.K = sp.efS = efC, sp.b_override = b_build, sp.collect_pes =
 *   enable_pes (proj/include/pag/routing.hpp:186-187, proj/src/routing.cpp:206-247)
 * — batched over nodes already in the resident index: the query of node
 * nodes[i] is its stored row (no padding or normalisation). params NULL =
 * the header's efC / b_build; collect_pes < 0 = the header's enable_pes.
 * SearchResult.pes_rejected (routing.hpp:176, routing.cpp:190-199,235): up
 * to pes_cap expanded ids per node in pes[i * pes_cap ...], in expansion
 * order; pes_n[i] = the full count (> pes_cap means truncated). Results are
 * bit-identical to the reference (reference-order distances) unless
 * params->exact_dist = 0. Errors: "node id out of range" (EINVAL), plus
 * those of pag_gpu_search. */
int pag_gpu_construction_search(pag_gpu_index* ix, const uint32_t* nodes, uint64_t nn,
                                const pag_search_params* params, int collect_pes, uint32_t* ids, float* sq,
                                uint32_t* n_out, pag_search_stats* stats, uint32_t* pes, uint32_t pes_cap,
                                uint32_t* pes_n);

/* pag_gpu_construction_search with every buffer on device 0 of the handle
 * (node ids must be < n; not checked here), launched on `stream` without
 * host synchronisation; stats_dev: nn x 8 u32 raw counters as
 * pag_gpu_search_device (the same stream rule). */
int pag_gpu_construction_search_device(pag_gpu_index* ix, const uint32_t* nodes_dev, uint64_t nn,
                                       const pag_search_params* params, int collect_pes, uint32_t* ids_dev,
                                       float* sq_dev, uint32_t* n_out_dev, uint32_t* stats_dev,
                                       uint32_t* pes_dev, uint32_t pes_cap, uint32_t* pes_n_dev, void* stream);

/* Asynchronous pag_gpu_construction_search: same arguments (params NULL =
 * the header's efC / b_build, collect_pes < 0 = enable_pes), returns a ticket
 * completed by pag_gpu_search_wait (the same ring of up to 4 batches per GPU
 * as pag_gpu_search_submit); the caller's arrays are filled at wait. */
int pag_gpu_construction_submit(pag_gpu_index* ix, const uint32_t* nodes, uint64_t nn,
                                const pag_search_params* params, int collect_pes, uint32_t* ids, float* sq,
                                uint32_t* n_out, pag_search_stats* stats, uint32_t* pes, uint32_t pes_cap,
                                uint32_t* pes_n, uint64_t* ticket);

/* Replaces: GroundTruth ground_truth(const VectorSet& base,
 *                                    const VectorSet& queries, uint32_t k_star)
 *           proj/include/pag/bench.hpp:19, proj/src/bench.cpp:18-53,
 * over the handle's resident base vectors: exact reference-order fp32
 * squared distances, top-min(k, n) by (sq, id). queries: nq x dim raw host
 * rows, zero-padded to padded_dim (no normalisation, as ground_truth reads
 * the stored rows). ids/sq: nq x k host. */
int pag_gpu_ground_truth(pag_gpu_index* ix, const float* queries, uint64_t nq, uint32_t k,
                         uint32_t* ids, float* sq);

/* Online-insert refresh: re-synchronise the
 * resident index with a newer PAGIDX01 file the reference saved after
 * appending nodes (insert_online, proj/src/builder.cpp:354-363; adjacency
 * rewiring :92-139, PES flush :250-279). The file must extend the loaded one
 * (same header parameters and entry nodes, n_new >= n). Only new rows/norms
 * and node blocks whose contents changed are uploaded. stats (may be NULL):
 * {new nodes, changed node blocks, bytes uploaded, microseconds}. */
int pag_gpu_refresh(pag_gpu_index* ix, const char* index_path, uint64_t* stats);

/* Host-only: parse and validate a PAGIDX01 file exactly as pag_gpu_open
 * does (same errors), without touching a GPU; fills info[0..9] as
 * pag_gpu_info (n_devices and device bytes are 0). */
int pag_gpu_inspect(const char* index_path, uint64_t* info, size_t n_info);

/* Host-only: the regenerated reference family the loader uploads.
 * Replaces: ReferenceSet build_reference_set(uint32_t padded_dim, uint32_t L,
 *           uint32_t m, uint64_t seed), proj/include/pag/projection.hpp:35,
 *           proj/src/projection.cpp:40-74 (same validation messages).
 * out: L*m*(padded_dim/L) floats, refs[(l*m + j)*sub_dim + c]. */
int pag_gpu_reference_family(uint32_t padded_dim, uint32_t L, uint32_t m, uint64_t seed,
                             float* out, size_t n_out);

/* Replaces: uint32_t default_subspace_count(uint32_t dim),
 *           proj/include/pag/projection.hpp:83, proj/src/projection.cpp:151-166. */
uint32_t pag_gpu_default_subspace_count(uint32_t dim);

/* Thread-local message of the last failing call on this thread. */
const char* pag_gpu_last_error(void);

/* Library version string. */
const char* pag_gpu_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PAG_GPU_H */
