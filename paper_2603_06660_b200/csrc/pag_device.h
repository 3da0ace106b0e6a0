// pag_device.h — device-side data layout and kernel launch interface shared
// by the host library (pag_host.cpp) and the kernels (pag_search.cu,
// pag_gt.cu). No torch types; plain pointers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace pagdev {

// Per-query status bits written next to the counters.
enum : uint32_t {
    kStatusZeroCosineQuery = 1u << 0,  // routing.cpp:257 "zero query under cosine metric"
    // PAG_VALIDATE debug builds only: the device counterpart of
    // TfbState::validate (routing.cpp:116-137) found a violated invariant
    kStatusTfbCapacity = 1u << 4,      // "TFB: working set over capacity" / ring size over b
    kStatusTfbZmax = 1u << 5,          // "TFB: stale z_max"
    kStatusTfbDuplicate = 1u << 6,     // "TFB: duplicate node residence"
    kStatusTfbOrder = 1u << 7,         // "TFB: result list out of order"
};

// Per-query counters (routing.hpp:24-34 plus edges_scanned and status).
enum : uint32_t {
    kStatExact = 0,
    kStatTest = 1,
    kStatPass = 2,
    kStatVisited = 3,
    kStatEdges = 4,
    kStatStatus = 5,
    kStatWords = 8,
};

// Index resident in HBM (one replica per GPU). Layout:
//  rows   : n x dstride fp32, dstride = round_up(padded_dim, 4), zero padded
//  deg    : n x u32
//  adj    : n node blocks of block_bytes, slot stride S = round_up(2M, 32):
//           targets u32[S] | edge_norm f32[S] | cos_beta f32[S] |
//           base_offset f32[S] | codes u32[S][cwp]   (edge-major codes)
//  refsT  : L x sub_dim x m fp32 (reference family, transposed so one
//           subspace's m references are contiguous per component)
//  rowsX  : n x xstride fp32, the chain-interleaved copy of rows read by the
//           reference-order distances (built on the device at the first
//           search that needs it, see chain_positions / launch_interleave_rows)
struct IndexView {
    const float* rows;
    const float* rowsX;
    const uint32_t* deg;
    const uint8_t* adj;
    const float* refsT;
    const uint32_t* entries;
    uint64_t n;
    uint32_t dim, padded, dstride;
    uint32_t xstride;  // floats per rowsX row (multiple of 32)
    uint32_t L, m, sub_dim;
    uint32_t slot_stride, cwp, block_bytes;
    uint32_t n_entries;
    uint32_t cosine;
    // no node repeats a target inside a 32-edge group (checked on the device
    // after load and refresh): the search skips its duplicate resolution
    uint32_t dup_free;
};

// One batched search launch.
struct SearchLaunch {
    IndexView ix;
    const float* queries;  // nq x dim raw rows (device)
    uint32_t nq;
    uint32_t K, efS, b, r_max;
    uint32_t use_prt;
    uint32_t exact_dist;  // 1: reference-order (bit-exact) sq_dist; 0: warp-tree
    // outputs (device)
    uint32_t* out_ids;    // nq x K
    float* out_sq;        // nq x K
    uint32_t* out_n;      // nq
    uint32_t* out_stats;  // nq x kStatWords
    // construction search (builder.cpp:218-227): query i is the stored row of
    // node qnodes[i] (queries unused); with collect_pes the expanded nodes
    // whose PES max is negative (routing.cpp:190-199,235) go to
    // out_pes[i * pes_cap ...], the full count to out_pes_n[i]
    const uint32_t* qnodes;
    uint32_t collect_pes, pes_cap;
    uint32_t* out_pes;
    uint32_t* out_pes_n;
    // scheduling + scratch
    // query claim counter of this launch's parity. Counters are never reset:
    // every warp of a launch claims until it draws an index >= nq, so a
    // launch advances its counter by exactly nq + (warps in the grid), and
    // the host passes the value at launch as qbase (query = claim - qbase,
    // mod 2^32). Consecutive launches alternate between two counters and two
    // scratch sets (programmatic dependent launch: launch N+1 may start while
    // N drains; N+2, same parity as N, starts only after N has completed).
    uint32_t* qcounter;
    uint32_t qbase;
    uint32_t pdl;  // launch with programmatic stream serialisation (0 after a stream switch)
    // asynchronous host API (pag_gpu_search_submit): when host_flag is set,
    // the last warp to exit writes flag_value to this pinned host word after
    // a system-scope fence (all outputs, written to pinned host memory, are
    // then visible); done_ctr counts exited warps (n_warps in the grid)
    uint32_t* done_ctr;
    uint32_t* host_flag;
    uint32_t flag_value, n_warps;
    uint32_t* gbm;          // per slot: visited bitmap of gbm_words (all zero between queries)
    uint32_t gbm_words;     // multiple of 4 (>= n / 32)
    uint8_t* gscratch;      // per slot: gscratch_stride bytes
    uint64_t gscratch_stride;
    // layout: per-warp smem and per-slot global regions (byte offsets);
    // a region lives in smem when its *_in_smem flag is set
    uint32_t warp_smem_bytes;
    uint32_t off_q, off_T, off_hash, hash_log2, off_sqbuf;
    uint32_t hash_limit;  // marks the smem table takes before spilling to the bitmap
    uint32_t off_W, W_in_smem;
    uint32_t off_rf, off_rt, rings_in_smem;
    uint32_t off_rl, rl_in_smem, rl_cap;  // R_L append buffer (+ sort scratch)
    uint32_t off_merge, merge_in_smem;
    uint32_t off_dbg;  // PAG_VALIDATE builds: per-slot HBM scratch for the resident-id check
    uint32_t warps_per_block;
};

size_t search_kernel_smem(const SearchLaunch& L);
// kernels bounded for 6 resident blocks per SM (large efS) instead of 4
bool search_high_occupancy(const SearchLaunch& L);
// b <= 32: working set and rings in registers (no smem for them)
bool search_uses_registers(const SearchLaunch& L);
cudaError_t launch_search(const SearchLaunch& L, int grid, cudaStream_t stream);
cudaError_t search_occupancy(const SearchLaunch& L, int* blocks_per_sm);
// PAG_PHASE_TIMING builds only: summed per-warp cycles per phase
void search_phase_cycles(unsigned long long* out8, bool reset);

// Exact brute-force ground truth (bench.cpp:18-53): reference-order fp32
// distances, top-k by (sq, id).
struct GtLaunch {
    const float* base;     // n x dstride
    uint64_t n;
    uint32_t padded, dstride;
    const float* queries;  // nq x dstride (already padded)
    uint32_t nq;
    uint32_t k;
    uint32_t* out_ids;     // nq x k
    float* out_sq;         // nq x k
    float* scratch_sq;     // tiles
    uint32_t* scratch_id;
};
cudaError_t launch_ground_truth(const GtLaunch& g, cudaStream_t stream);

// Tensor-core ground truth (pag_gt_tc.cu): TF32 tcgen05 candidate GEMM with a
// fused per-split top-C epilogue, exact reference-order re-rank, certificate.
struct GtTcLaunch {
    const void* tmA;  // CUtensorMap over queries (nq x padded, row pitch dstride*4)
    const void* tmB;  // CUtensorMap over base rows (n x padded)
    const float* base;
    uint64_t n;
    uint32_t padded, dstride;
    const float* queries;  // nq x dstride, zero padded
    uint32_t nq, k, nsplit, C;
    uint64_t rows_per_split;  // multiple of gt_tc_block_n()
    float* qnorm;             // nq scratch (squared norms)
    const float* bnorm;       // n squared norms of the base rows
    float max_bnorm;          // max squared base norm
    float* cand_d;            // nq x nsplit x C
    uint32_t* cand_id;        // nq x nsplit x C
    float* cand_thr;          // nq x nsplit
    uint32_t* out_ids;        // nq x k
    float* out_sq;            // nq x k
    uint32_t* uncertified;    // nq flags: 1 = re-run exactly
};
cudaError_t launch_gt_tc(const GtTcLaunch& g, cudaStream_t stream);

// Tensor-core ground truth for 32 < k <= 1000 (pag_gt_tc.cu): per-query
// distance bound from k search-result rows, TF32 tcgen05 GEMM whose epilogue
// appends the rows under the bound to the query's pool, exact re-rank of the
// pool. Queries whose pool overflowed are flagged for the exact re-run.
struct GtTcPoolLaunch {
    const void* tmA;  // CUtensorMap over queries (nq x padded, row pitch dstride*4)
    const void* tmB;  // CUtensorMap over base rows (n x padded)
    const float* base;
    uint64_t n;
    uint32_t padded, dstride;
    const float* queries;       // nq x dstride, zero padded
    uint32_t nq, k, nsplit;
    uint64_t rows_per_split;    // multiple of gt_tc_block_n()
    float* qnorm;               // nq scratch
    const float* bnorm;         // n squared base norms
    float max_bnorm;
    const uint32_t* search_ids; // nq x k: rows of a graph search of each query (any k distinct rows)
    const uint32_t* search_n;   // nq: valid entries (< k: the query is re-run exactly)
    float* thrx;                // nq scratch: filter bound
    uint32_t* pool_cnt;         // nq
    uint32_t* pool_id;          // nq x pool_cap
    uint32_t pool_cap;          // <= 8192
    uint32_t* out_ids;          // nq x k
    float* out_sq;              // nq x k
    uint32_t* uncertified;      // nq flags: 1 = re-run exactly
};
cudaError_t launch_gt_tc_pool(const GtTcPoolLaunch& g, cudaStream_t stream);

// Chain-interleaved row layout (reference-order distances, vecstore.cpp:77-95).
// sq_dist runs four accumulator chains: chain c takes elements c, c + 4, ...
// of the first D4 = padded & ~3 elements, and chain 0 then takes the tail
// elements D4 .. padded-1. Call "position" p the p-th step of the chains:
// p < D4/4 holds elements 4p .. 4p+3 (one per chain), position D4/4 + t holds
// tail element D4 + t for chain 0 and zeros for chains 1-3 (a zero difference
// adds +0 to a chain: no change). Positions are padded with zeros to a
// multiple of 8, and every 8 positions are stored as one 128-B line
//   chain 0: 8 floats | chain 1: 8 floats | chain 2: 8 floats | chain 3: 8 floats
// so that the lane running chain c of a row reads its next 8 elements with
// one 32-B load, and the 4 lanes of a row read whole lines.
__host__ __device__ inline uint32_t chain_positions(uint32_t padded) { return (padded >> 2) + (padded & 3u); }
__host__ __device__ inline uint32_t chain_xstride(uint32_t padded) { return ((chain_positions(padded) + 7u) >> 3) << 5; }
// rows (n x dstride) -> rowsX (n x chain_xstride(padded)), rows [first, n)
cudaError_t launch_interleave_rows(const float* rows, float* rowsX, uint64_t first, uint64_t n, uint32_t padded,
                                   uint32_t dstride, cudaStream_t stream);

// pag_util.cu: staged node blocks -> their slots in the adjacency array
cudaError_t scatter_blocks(const void* staging, const uint32_t* ids, uint32_t count, void* adj,
                           uint32_t block_bytes, cudaStream_t stream);
// nodes with a target repeated inside one 32-edge group -> *count_dev
cudaError_t count_dup_groups(const void* adj, const uint32_t* deg, uint64_t n, uint32_t block_bytes,
                             uint32_t* count_dev, cudaStream_t stream);
size_t gt_tc_smem_bytes();
uint32_t gt_tc_cmax();
uint32_t gt_tc_block_n();
uint32_t gt_tc_block_k();
uint32_t gt_tc_block_m();
size_t gt_scratch_elems(uint64_t n, uint32_t nq, uint32_t k);

}  // namespace pagdev
