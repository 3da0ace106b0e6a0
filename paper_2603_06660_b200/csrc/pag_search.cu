// pag_search.cu — batched PAG search (PRT + TFB, Algorithm 2) for sm_100a.
//
// One warp per query, persistent grid, queries claimed from an atomic
// counter. Replaces the reference's per-query host loop
//   search / search_padded      proj/src/routing.cpp:206-261
//   expand_node                 proj/src/routing.cpp:139-204
//   TfbState                    proj/include/pag/routing.hpp:62-161,
//                               proj/src/routing.cpp:12-114
//   build_projection_table      proj/src/projection.cpp:123-137
//   table_code_sum              proj/src/projection.cpp:145-149
//   sq_dist / vec_norm          proj/src/vecstore.cpp:77-108
//
// Semantics are the reference's, bit for bit: every fp32 operation uses the
// _rn intrinsics (no FMA contraction) in the reference's evaluation order,
// and the data-dependent TFB state machine is replayed in edge order.
// Parallelism inside an expansion (SURVEY.md §7 "Semantic details"):
//   (i)   lane j owns out-edge j: visited lookup, PRT at the radius in effect
//         when the 32-edge group starts (the radius only shrinks inside an
//         expansion and the test is monotone in it, so this set is a
//         superset of the reference's passes);
//   (ii)  __ballot_sync compaction of the survivors;
//   (iii) their exact distances (rows prefetched to L2 by bulk copy; warp-tree
//         mode: two rows per pass, all loads of a row pair in flight;
//         reference order: chain-interleaved row copy, 8 rows per batch);
//   (iv)  an in-order replay re-evaluating the PRT with the live radius
//         before marking and admitting / pushing to R_F.
//
// Two state layouts share the code (template parameter TFB):
//   TfbReg  (b <= 32, K <= 32): the working set W and both FIFO rings live in
//           registers, slot i on lane i; argmin/argmax are __reduce_*_sync.
//   TfbMem  (b > 32): W and rings as arrays in smem or the warp's HBM slot.
// R_L (capacity efS) is an array in smem, or HBM when it does not fit.
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdlib.h>
#include <stdint.h>

#include "pag_device.h"

// Build flavours of this file (csrc/Makefile compiles it four times):
//   PAG_PES   0/1  query kernels / construction kernels with PES tracking
//   PAG_OCC   4/6  resident blocks of 4 warps per SM the kernels are
//                  register-bounded for: 4 (128 regs) for the usual
//                  operating points, 6 (80 regs) for large efS, where the
//                  visited set lives mostly in the HBM bitmap and latency
//                  hiding (more warps) pays more than registers
// The (PES 0, OCC 4) object holds the public entry points and dispatches.
#ifndef PAG_PES
#define PAG_PES 0
#endif
#ifndef PAG_OCC
#define PAG_OCC 4
#endif

namespace pagdev {
namespace {

#ifdef PAG_PHASE_TIMING
// per-warp cycle accounting of the expansion phases (diagnostic build only)
__device__ unsigned long long g_phase[8];
#define PT(k) do { long long t_ = clock64(); c.pt_acc[k] += t_ - c.pt_t0; c.pt_t0 = t_; } while (0)
#else
#define PT(k) do { } while (0)
#endif

constexpr uint32_t FULL = 0xffffffffu;
constexpr uint32_t EMPTY = 0xffffffffu;
constexpr uint32_t VISITED = 0x80000000u;
// A single-round search (r_max == 1) never reads its rings: end_round is not
// reached (routing.cpp:238-242 breaks before it after the last round) and
// ring contents never reach the results, so ring pushes are skipped there
// (kept in PAG_VALIDATE builds, whose validate_state inspects the rings).
// Evaluated from the kernel parameter where used (no register held).
__device__ __forceinline__ bool rings_are_read(const SearchLaunch& P) {
#ifdef PAG_VALIDATE
    (void)P;
    return true;
#else
    return P.r_max > 1;
#endif
}

__device__ __forceinline__ bool cless(float sa, uint32_t ia, float sb, uint32_t ib) {
    return sa < sb || (sa == sb && ia < ib);  // candidate_less, builder.hpp:23-25
}

// order-preserving key of a non-negative float (-0 folds onto +0)
__device__ __forceinline__ uint32_t fkey(float x) { return __float_as_uint(__fadd_rn(x, 0.0f)); }

// routing.hpp:40-43 — ((e*e + d*d) - z*z) / ((2*d)*e), no contraction
__device__ __forceinline__ float prt_threshold(float en, float duq, float dz) {
    float num = __fsub_rn(__fadd_rn(__fmul_rn(en, en), __fmul_rn(duq, duq)), __fmul_rn(dz, dz));
    float den = __fmul_rn(__fmul_rn(2.0f, duq), en);
    return __fdiv_rn(num, den);
}


__device__ __forceinline__ uint32_t hslot(uint32_t id, uint32_t log2) {
    return (id * 2654435761u) >> (32 - log2);
}

__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Row data is streamed (a row is mostly read once per query): row loads and
// row prefetches carry an L2 evict-first policy, which keeps adjacency
// blocks, visited bitmaps and spilled working sets resident (+1.1-1.2% on
// cfg-2 / cfg-3)
__device__ __forceinline__ uint64_t row_policy() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ float4 ldg_f4(const float* p) {
    float4 v;
    asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p), "l"(row_policy()));
    return v;
}
__device__ __forceinline__ void prefetch_row(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(p), "r"(bytes),
                 "l"(row_policy())
                 : "memory");
}

struct Arr {  // SoA entries {id, sq, aux}; generic pointers (smem or HBM)
    uint32_t* id;
    float* sq;
    uint32_t* aux;
};

__device__ __forceinline__ Arr make_arr(uint8_t* base, uint32_t cap) {
    Arr a;
    a.id = reinterpret_cast<uint32_t*>(base);
    a.sq = reinterpret_cast<float*>(base + 4ull * cap);
    a.aux = reinterpret_cast<uint32_t*>(base + 8ull * cap);
    return a;
}

// ---------------------------------------------------------------------------
// Per-warp state shared by both TFB layouts: query, projection table, visited
// set, result list, counters.
// ---------------------------------------------------------------------------
struct Common {
    float* q;
    float* T;
    float* sqbuf;
    __device__ uint32_t* degbuf() const { return reinterpret_cast<uint32_t*>(sqbuf + 32); }
    // visited marks (routing.hpp:104-105): smem open addressing; once the
    // smem table is half full further marks go to this warp's n-bit HBM
    // bitmap (one load per lookup, no probe chains), cleared after the query
    uint32_t* hs;
    uint32_t hs_log2, hs_count, hs_limit;  // marks held on chip before the bitmap takes over
    uint32_t* gbm;
    uint32_t gbm_words, gt_count;
    bool gt_used;
    // R_L (routing.hpp:150, capacity efS) is never read during the search:
    // flushed W entries are appended here and the cap-limited sorted list is
    // formed once at the end (the bounded insert keeps the efS smallest, an
    // order-independent result). rl_tmp is the final sort's scratch.
    // (bases only: the three-array views are formed where used, so they do
    // not occupy registers through the search loop)
    uint8_t* rl_base;
    uint8_t* mo_base;
    uint32_t rl_cap, mo_cap;
    uint32_t rl_size, cap_r;
    __device__ Arr rl() const { return make_arr(rl_base, rl_cap); }
    __device__ Arr rl_tmp() const { return make_arr(rl_base + 12ull * rl_cap, rl_cap); }
    __device__ Arr mo() const { return make_arr(mo_base, mo_cap); }
    // counters (routing.hpp:24-34 + edges_scanned)
    uint32_t n_exact, n_test, n_pass, n_visited, n_edges, n_pes;
#ifdef PAG_VALIDATE
    uint32_t invalid;  // kStatusTfb* bits found by validate_state
#endif
#ifdef PAG_PHASE_TIMING
    long long pt_t0, pt_acc[8];
#endif

};

// visited-bitmap words: evict-first in L2 (a query touches its whole n-bit
// bitmap once; keeping it would push out the working sets; cfg-4 +1.1%)
__device__ __forceinline__ uint64_t bm_policy() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint32_t bm_load(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.cg.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(bm_policy()) : "memory");
    return v;
}
__device__ __forceinline__ void bm_or(uint32_t* p, uint32_t bits) {
    asm volatile("red.global.or.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(bits), "l"(bm_policy()) : "memory");
}

// off-chip working-set words (the warp's HBM scratch, WOFF): L2 evict-last,
// so a warp's W stays resident while rows and bitmaps stream through
__device__ __forceinline__ uint32_t ld_keep(const uint32_t* p) {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    uint32_t v;
    asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol) : "memory");
    return v;
}
__device__ __forceinline__ float ld_keep(const float* p) { return __uint_as_float(ld_keep(reinterpret_cast<const uint32_t*>(p))); }

// The smem visited table is bucketed: 4-slot buckets (one 16-B load), an id
// hashes to a bucket, inserts take the bucket's first empty slot (atomicCAS
// in slot order) or move on to the next bucket. Slots fill in order and are
// never freed, so a bucket with an empty slot ends the probe.
__device__ __forceinline__ bool hash_has(const Common& c, uint32_t id) {
    const uint32_t bmask = (1u << (c.hs_log2 - 2)) - 1;
    uint32_t bk = hslot(id, c.hs_log2 - 2);
    while (true) {
        const uint4 v = reinterpret_cast<const uint4*>(c.hs)[bk];
        if (v.x == id || v.y == id || v.z == id || v.w == id) return true;
        if (v.w == EMPTY) return false;  // (slots fill in order: w empty <=> some empty)
        bk = (bk + 1) & bmask;
    }
}

__device__ __forceinline__ bool marked(const Common& c, uint32_t id) {
    if (hash_has(c, id)) return true;
    if (!c.gt_used) return false;
    return (c.gbm[id >> 5] >> (id & 31u)) & 1u;
}

// one id into the table (the caller keeps the load at most half)
__device__ __forceinline__ void hash_insert(const Common& c, uint32_t id) {
    const uint32_t bmask = (1u << (c.hs_log2 - 2)) - 1;
    uint32_t bk = hslot(id, c.hs_log2 - 2);
    while (true) {
        uint32_t* b4 = c.hs + 4 * bk;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (atomicCAS(b4 + k, EMPTY, id) == EMPTY) return;
        bk = (bk + 1) & bmask;
    }
}

// warp-uniform call; lane 0 writes
__device__ __forceinline__ void mark(Common& c, uint32_t id, int lane) {
    if (c.hs_count < c.hs_limit) {
        if (lane == 0) hash_insert(c, id);
        ++c.hs_count;
    } else {
        if (lane == 0) bm_or(&c.gbm[id >> 5], 1u << (id & 31u));
        c.gt_used = true;
        ++c.gt_count;
    }
    __syncwarp();
}

// marks the targets of the lanes in `lanes` (distinct ids), in parallel:
// atomicCAS probing while everything fits the smem half-load budget, else
// the HBM bitmap.
__device__ __forceinline__ void mark_many(Common& c, uint32_t lanes, uint32_t w, int lane) {
    const uint32_t np = __popc(lanes);
    const bool mine = (lanes >> lane) & 1u;
    if (c.hs_count + np <= c.hs_limit) {
        if (mine) hash_insert(c, w);
        c.hs_count += np;
    } else {
        if (mine) bm_or(&c.gbm[w >> 5], 1u << (w & 31u));
        c.gt_used = true;
        c.gt_count += np;
    }
    __syncwarp();
}

// zero this warp's bitmap after a query that used it
__device__ __forceinline__ void clear_bitmap(Common& c, int lane) {
    if (!c.gt_used) return;
    uint4* p = reinterpret_cast<uint4*>(c.gbm);
    const uint4 z = make_uint4(0u, 0u, 0u, 0u);
    for (uint32_t i = lane; i < c.gbm_words / 4; i += 32) p[i] = z;
    c.gt_used = false;
    __syncwarp();
}

// routing.cpp:82-90: R_L receives flushed W entries (distinct ids); they are
// appended and the capacity-limited sorted list is formed at the end.
__device__ __forceinline__ void rl_append(Common& c, uint32_t id, float sq, bool valid, uint32_t offset) {
    if (valid) {
        const Arr rl = c.rl();
        rl.id[c.rl_size + offset] = id;
        rl.sq[c.rl_size + offset] = sq;
    }
}

// warp bitonic sort of 32 (sq, id, aux) tuples, one per lane, ascending
__device__ __forceinline__ void bitonic32(float& s, uint32_t& id, uint32_t& ax, int lane) {
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const float ps = __shfl_xor_sync(FULL, s, j);
            const uint32_t pid = __shfl_xor_sync(FULL, id, j);
            const uint32_t pax = __shfl_xor_sync(FULL, ax, j);
            const bool up = (lane & k) == 0, lower = (lane & j) == 0;
            const bool pless = cless(ps, pid, s, id);
            if (lower == up ? pless : !pless) {
                s = ps;
                id = pid;
                ax = pax;
            }
        }
    }
}

// number of entries of sorted a[0..n) strictly less than (v, id)
__device__ __forceinline__ uint32_t count_less(const Arr& a, uint32_t n, float v, uint32_t id) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (cless(a.sq[mid], a.id[mid], v, id))
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// merge path: how many of the first d outputs of merge(A[0..la), B[0..lb))
// come from A (distinct (sq, id) keys, so the split is unique)
__device__ __forceinline__ uint32_t merge_split(const Arr& A, uint32_t la, const Arr& B, uint32_t lb, uint32_t d) {
    uint32_t lo = d > lb ? d - lb : 0u, hi = min(d, la);
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        const uint32_t bj = d - mid - 1;
        if (cless(A.sq[mid], A.id[mid], B.sq[bj], B.id[bj]))
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// Sort n entries of `a` ascending by (sq, id) (distinct ids): 32-element
// bitonic runs in registers, then merge passes: for runs of <= 64 every
// element binary-searches its slot in the partner run; longer passes cut the
// output of every run pair into 32-entry tiles; the lanes find the tiles' merge-path
// splits in parallel (one binary search per 32 outputs), then each tile is
// loaded as A-part ascending + B-part descending (a bitonic sequence) and
// finished by a 5-step bitonic merge in registers. `t` is scratch of the
// same capacity; returns whichever of a / t holds the result.
__device__ __noinline__ Arr warp_sort(Arr a, Arr t, uint32_t n, int lane) {
    for (uint32_t base = 0; base < n; base += 32) {
        const uint32_t i = base + lane;
        const bool v = i < n;
        float s = v ? a.sq[i] : CUDART_INF_F;
        uint32_t id = v ? a.id[i] : EMPTY, ax = v ? a.aux[i] : 0u;
        bitonic32(s, id, ax, lane);
        if (v) {
            a.sq[i] = s;
            a.id[i] = id;
            a.aux[i] = ax;
        }
    }
    __syncwarp();
    Arr src = a, dst = t;
    const uint32_t ntiles = (n + 31) / 32;
    for (uint32_t w = 32; w < n; w <<= 1) {
        if (w <= 64) {  // short runs: every element binary-searches its partner run (<= 6 steps)
            for (uint32_t i = lane; i < n; i += 32) {
                const uint32_t start = i & ~(w - 1), pstart = start ^ w;
                const float s = src.sq[i];
                const uint32_t id = src.id[i], ax = src.aux[i];
                uint32_t out = i;
                if (pstart < n) {
                    Arr p;
                    p.id = src.id + pstart;
                    p.sq = src.sq + pstart;
                    p.aux = src.aux + pstart;
                    out = min(start, pstart) + (i - start) + count_less(p, min(w, n - pstart), s, id);
                }
                dst.id[out] = id;
                dst.sq[out] = s;
                dst.aux[out] = ax;
            }
            __syncwarp();
            const Arr tmp = src;
            src = dst;
            dst = tmp;
            continue;
        }
        for (uint32_t tb = 0; tb < ntiles; tb += 32) {
            // this lane's tile: its run pair and merge-path splits
            const uint32_t tt = tb + lane;
            uint32_t ps = 0, la = 0, lb = 0, d0 = 0, d1 = 0, i0 = 0, i1 = 0;
            if (tt < ntiles) {
                const uint32_t o = tt * 32;
                ps = o & ~(2 * w - 1);
                la = min(w, n - ps);
                lb = ps + w < n ? min(w, n - ps - w) : 0u;
                d0 = o - ps;
                d1 = min(d0 + 32, la + lb);
                Arr A, B;
                A.id = src.id + ps;
                A.sq = src.sq + ps;
                A.aux = src.aux + ps;
                B.id = src.id + ps + w;
                B.sq = src.sq + ps + w;
                B.aux = src.aux + ps + w;
                i0 = lb ? merge_split(A, la, B, lb, d0) : d0;
                i1 = lb ? merge_split(A, la, B, lb, d1) : d1;
            }
            const uint32_t nt = min(32u, ntiles - tb);
            for (uint32_t k = 0; k < nt; ++k) {
                const uint32_t kps = __shfl_sync(FULL, ps, k), kd0 = __shfl_sync(FULL, d0, k);
                const uint32_t kd1 = __shfl_sync(FULL, d1, k), ki0 = __shfl_sync(FULL, i0, k);
                const uint32_t ki1 = __shfl_sync(FULL, i1, k);
                const uint32_t na = ki1 - ki0, nb = (kd1 - kd0) - na, j0 = kd0 - ki0;
                const uint32_t L = static_cast<uint32_t>(lane);
                float s = CUDART_INF_F;
                uint32_t id = EMPTY, ax = 0u;
                uint32_t src_i = EMPTY;
                if (L < na) src_i = kps + ki0 + L;                            // A ascending
                else if (L >= 32u - nb) src_i = kps + w + j0 + (31u - L);     // B descending
                if (src_i != EMPTY) {
                    s = src.sq[src_i];
                    id = src.id[src_i];
                    ax = src.aux[src_i];
                }
#pragma unroll
                for (int j = 16; j > 0; j >>= 1) {  // bitonic merge, ascending
                    const float ps2 = __shfl_xor_sync(FULL, s, j);
                    const uint32_t pid = __shfl_xor_sync(FULL, id, j);
                    const uint32_t pax = __shfl_xor_sync(FULL, ax, j);
                    const bool lower = (lane & j) == 0;
                    const bool pless = cless(ps2, pid, s, id);
                    if (lower ? pless : !pless) {
                        s = ps2;
                        id = pid;
                        ax = pax;
                    }
                }
                if (L < kd1 - kd0) {
                    const uint32_t o = kps + kd0 + L;
                    dst.id[o] = id;
                    dst.sq[o] = s;
                    dst.aux[o] = ax;
                }
            }
        }
        __syncwarp();
        const Arr tmp = src;
        src = dst;
        dst = tmp;
    }
    return src;
}

// ---------------------------------------------------------------------------
// TfbReg: b <= 32. Lane i holds W slot i, ring_f physical slot i and ring_t
// physical slot i (routing.hpp:62-161 with the reference's slot placement).
// ---------------------------------------------------------------------------
struct TfbReg {
    uint32_t b;
    uint32_t w_id, w_deg;
    float w_sq;
    bool w_vis;
    uint8_t* rf_base;  // ring R_F: 32 slots {id | sq | aux} in smem (bulk pushes scatter into it)
    __device__ Arr rf() const { return make_arr(rf_base, 32); }
    uint32_t t_id, t_deg;
    float t_sq;
    uint32_t wsize, rf_head, rf_size, rt_head, rt_size;
    float zmax_sq, zmax_dist;
    uint32_t zmax_idx;

    __device__ void init(uint32_t b_, uint8_t* sw, uint8_t* gw, const SearchLaunch& P) {
        b = b_;
        rf_base = (P.rings_in_smem ? sw : gw) + P.off_rf;
    }
    __device__ void reset() {
        wsize = rf_head = rf_size = rt_head = rt_size = 0;
        zmax_sq = zmax_dist = 0.0f;
        zmax_idx = 0;
        w_vis = false;
    }
    __device__ float admission_sq() const { return wsize < b ? CUDART_INF_F : zmax_sq; }
    __device__ float admission_dist() const { return wsize < b ? CUDART_INF_F : zmax_dist; }

    // routing.cpp:32-44: argmax, first slot on ties
    __device__ void recompute_zmax(int lane) {
        if (wsize == 0) {
            zmax_sq = zmax_dist = 0.0f;
            zmax_idx = 0;
            return;
        }
        const bool v = static_cast<uint32_t>(lane) < wsize;
        const uint32_t k = v ? fkey(w_sq) : 0u;
        const uint32_t m = __reduce_max_sync(FULL, k);
        zmax_sq = __uint_as_float(m);  // the key is the value (sq >= 0: x + 0 == x)
        zmax_dist = __fsqrt_rn(zmax_sq);
        zmax_idx = __ffs(__ballot_sync(FULL, v && k == m)) - 1;
    }
    // routing.cpp:71-80: argmin over unvisited by (sq, id); `skip` excluded
    __device__ uint32_t next_unvisited(int lane, uint32_t skip = EMPTY) const {
        const bool v = static_cast<uint32_t>(lane) < wsize && !w_vis && static_cast<uint32_t>(lane) != skip;
        if (!__ballot_sync(FULL, v)) return EMPTY;
        const uint32_t k = v ? fkey(w_sq) : 0xffffffffu;
        const uint32_t m1 = __reduce_min_sync(FULL, k);
        const bool c1 = v && k == m1;
        const uint32_t m2 = __reduce_min_sync(FULL, c1 ? w_id : 0xffffffffu);
        return __ffs(__ballot_sync(FULL, c1 && w_id == m2)) - 1;
    }
    __device__ void entry(uint32_t slot, uint32_t& id, float& sq, uint32_t& deg) const {
        id = __shfl_sync(FULL, w_id, slot);
        sq = __shfl_sync(FULL, w_sq, slot);
        deg = __shfl_sync(FULL, w_deg, slot);
    }
    __device__ uint32_t entry_id(uint32_t slot) const { return __shfl_sync(FULL, w_id, slot); }
    __device__ void set_visited(uint32_t slot, int lane) {
        if (static_cast<uint32_t>(lane) == slot) w_vis = true;
    }
    // routing.cpp:46-53 / :57-63
    __device__ void append(uint32_t id, float sq, uint32_t deg, int lane) {
        if (static_cast<uint32_t>(lane) == wsize) {
            w_id = id;
            w_sq = sq;
            w_deg = deg;
            w_vis = false;
        }
        ++wsize;
        if (sq > zmax_sq || wsize == 1) {
            zmax_idx = wsize - 1;
            zmax_sq = sq;
            zmax_dist = __fsqrt_rn(sq);
        }
    }
    __device__ void push_rt(uint32_t id, float sq, uint32_t deg, int lane) {
        uint32_t pos = rt_head + rt_size;
        if (pos >= b) pos -= b;
        if (static_cast<uint32_t>(lane) == pos) {
            t_id = id;
            t_sq = sq;
            t_deg = deg;
        }
        if (rt_size < b) ++rt_size;
        else rt_head = (rt_head + 1 == b) ? 0 : rt_head + 1;
    }
    __device__ void push_fp(uint32_t id, float sq, uint32_t deg, int lane) {  // routing.hpp:128
        uint32_t pos = rf_head + rf_size;
        if (pos >= b) pos -= b;
        if (lane == 0) {
            rf().id[pos] = id;
            rf().sq[pos] = sq;
            rf().aux[pos] = deg;
        }
        if (rf_size < b) ++rf_size;
        else rf_head = (rf_head + 1 == b) ? 0 : rf_head + 1;
        __syncwarp();
    }
    // push_fp of the lanes in pm, in lane order (lane l supplies its entry):
    // element i lands in slot (head + size + i) mod b; when a call wraps the
    // ring, only the last element aimed at a slot writes it (the sequential
    // overwrite-oldest pushes keep that one)
    __device__ void push_fp_many(uint32_t pm, uint32_t id, float sq, uint32_t deg, int lane) {
        const uint32_t np = __popc(pm);
        if ((pm >> lane) & 1u) {
            const uint32_t r = __popc(pm & ((1u << lane) - 1u));
            if (r + b >= np) {
                uint32_t pos = rf_head + rf_size + r;
                while (pos >= b) pos -= b;
                rf().id[pos] = id;
                rf().sq[pos] = sq;
                rf().aux[pos] = deg;
            }
        }
        const uint32_t tot = rf_size + np;
        if (tot <= b) {
            rf_size = tot;
        } else {
            uint32_t h = rf_head + (tot - b);
            while (h >= b) h -= b;
            rf_head = h;
            rf_size = b;
        }
        __syncwarp();
    }
    // routing.cpp:55-69 (rings_live: see rings_are_read)
    __device__ void admit(uint32_t id, float sq, uint32_t deg, int lane, bool rings_live) {
        if (wsize < b) {
            append(id, sq, deg, lane);
            return;
        }
        const uint32_t z = zmax_idx;
        if (rings_live) {
            const uint32_t oid = __shfl_sync(FULL, w_id, z);
            const float osq = __shfl_sync(FULL, w_sq, z);
            const uint32_t odeg = __shfl_sync(FULL, w_deg, z);
            push_rt(oid, osq, odeg, lane);
        }
        if (static_cast<uint32_t>(lane) == z) {
            w_id = id;
            w_sq = sq;
            w_deg = deg;
            w_vis = false;
        }
        recompute_zmax(lane);
    }
    // W -> R_L (routing.cpp:93 and :242)
    __device__ void flush(Common& c, int lane) {
        rl_append(c, w_id, w_sq, static_cast<uint32_t>(lane) < wsize, lane);
        c.rl_size += wsize;
        __syncwarp();
    }
#ifdef PAG_VALIDATE
    // debug: max sq of W, and the resident ids of W, R_F, R_T -> dst
    __device__ float w_max(int lane) const {
        const uint32_t k = static_cast<uint32_t>(lane) < wsize ? fkey(w_sq) : 0u;
        return __uint_as_float(__reduce_max_sync(FULL, k));
    }
    __device__ uint32_t dump_ids(uint32_t* dst, int lane) const {
        const uint32_t L = static_cast<uint32_t>(lane);
        if (L < wsize) dst[L] = w_id;
        for (uint32_t i = L; i < rf_size; i += 32) {
            uint32_t p = rf_head + i;
            if (p >= b) p -= b;
            dst[wsize + i] = rf().id[p];
        }
        if (L < b && ((L + b - rt_head) % b) < rt_size) dst[wsize + rf_size + (L + b - rt_head) % b] = t_id;
        return wsize + rf_size + rt_size;
    }
#endif
    // routing.cpp:92-114
    __device__ bool end_round(Common& c, int lane) {
        flush(c, lane);
        wsize = 0;
        const uint32_t L = static_cast<uint32_t>(lane);
        const bool fv = L < b && ((L + b - rf_head) % b) < rf_size;
        uint32_t f_id = 0, f_deg = 0;
        float f_sq = 0.0f;
        if (L < b) {
            f_id = rf().id[L];
            f_sq = rf().sq[L];
            f_deg = rf().aux[L];
        }
        const bool tv = L < b && ((L + b - rt_head) % b) < rt_size;
        const uint32_t nm = rf_size + rt_size;
        rf_head = rf_size = rt_head = rt_size = 0;
        if (nm == 0) {
            zmax_sq = zmax_dist = 0.0f;
            return false;
        }
        uint32_t fr = 0, tr = 0;
        for (uint32_t j = 0; j < b; ++j) {
            const bool fvj = __shfl_sync(FULL, fv, j);
            const bool tvj = __shfl_sync(FULL, tv, j);
            const float fs = __shfl_sync(FULL, f_sq, j), ts = __shfl_sync(FULL, t_sq, j);
            const uint32_t fi = __shfl_sync(FULL, f_id, j), ti = __shfl_sync(FULL, t_id, j);
            if (fvj) {
                fr += cless(fs, fi, f_sq, f_id) ? 1u : 0u;
                tr += cless(fs, fi, t_sq, t_id) ? 1u : 0u;
            }
            if (tvj) {
                fr += cless(ts, ti, f_sq, f_id) ? 1u : 0u;
                tr += cless(ts, ti, t_sq, t_id) ? 1u : 0u;
            }
        }
        __syncwarp();
        const Arr mo = c.mo();
        if (fv) {
            mo.id[fr] = f_id;
            mo.sq[fr] = f_sq;
            mo.aux[fr] = f_deg;
        }
        if (tv) {
            mo.id[tr] = t_id;
            mo.sq[tr] = t_sq;
            mo.aux[tr] = t_deg;
        }
        __syncwarp();
        const uint32_t refill = min(nm, b);
        if (L < refill) {
            w_id = mo.id[L];
            w_sq = mo.sq[L];
            w_deg = mo.aux[L];
            w_vis = false;
        }
        if (L < nm - refill) {  // ring_t was cleared; the rest (<= b) in ascending order
            t_id = mo.id[refill + L];
            t_sq = mo.sq[refill + L];
            t_deg = mo.aux[refill + L];
        }
        wsize = refill;
        rt_size = nm - refill;
        __syncwarp();
        recompute_zmax(lane);
        return true;
    }
};

// ---------------------------------------------------------------------------
// TfbMem: b > 32. Arrays in smem or the warp's HBM slot.
// ---------------------------------------------------------------------------
// b > 32: W and the rings as arrays (smem, or the warp's HBM slot). Lane o
// owns the contiguous W slots [o*S, o*S+S), S = ceil(b/32), and caches in
// registers the best unvisited (sq, id) and the largest sq (lowest slot on
// ties) of its slots. argmin / argmax are then one warp reduction over the
// caches; a change to a slot re-scans only its owner's S slots, all lanes
// reading consecutive slots (conflict-free). Same selections as the full
// scans of routing.cpp:32-44,71-80.
//
// WOFF (W in the warp's HBM scratch, L2 latency per access): the caches also
// carry the winners' aux / id, so the expanded entry and the evicted z_max
// come from registers; set_visited writes the flag without reading and its
// owner re-scan is issued at once but folded in only before the next argmin
// (the loads overlap the expansion); an admission or append touching that
// owner first folds or supersedes it.
template <bool WOFF>
struct TfbMemT {
    Arr W, rf, rt, mi;
    uint32_t b, S;
    uint32_t wsize, rf_head, rf_size, rt_head, rt_size;
    float zmax_sq, zmax_dist;
    uint32_t zmax_idx;
    // this lane's caches over its slots
    uint32_t mn_key, mn_id, mn_slot;  // best unvisited by (sq, id); mn_slot EMPTY if none
    uint32_t mx_key, mx_slot;         // largest sq, lowest slot; mx_slot EMPTY if none
    // WOFF only
    uint32_t mn_aux, mx_id, mx_aux;   // aux of the best unvisited, id/aux of the largest
    uint32_t nx_slot, nx_id, nx_aux;  // warp-uniform: the entry next_unvisited returned
    float nx_sq;
    uint32_t zmax_id, zmax_aux;       // warp-uniform
    uint32_t pend_o;                  // owner whose re-scan is in flight (EMPTY: none)
    uint32_t pk, pid, pax;            // its slot o*S + lane as loaded

    __device__ void init(uint32_t b_, uint8_t* sw, uint8_t* gw, const SearchLaunch& P) {
        b = b_;
        S = (b + 31) / 32;
        W = make_arr((P.W_in_smem ? sw : gw) + P.off_W, b);
        rf = make_arr((P.rings_in_smem ? sw : gw) + P.off_rf, b);
        rt = make_arr((P.rings_in_smem ? sw : gw) + P.off_rt, b);
        mi = make_arr((P.merge_in_smem ? sw : gw) + P.off_merge, 2 * b);
    }
    __device__ void clear_caches() {
        mn_key = mn_id = 0xffffffffu;
        mn_slot = mx_slot = EMPTY;
        mx_key = 0;
        if (WOFF) {
            mn_aux = mx_id = mx_aux = 0;
            nx_slot = EMPTY;
            pend_o = EMPTY;
        }
    }
    __device__ void reset() {
        wsize = rf_head = rf_size = rt_head = rt_size = 0;
        zmax_sq = zmax_dist = 0.0f;
        zmax_idx = 0;
        clear_caches();
    }
    __device__ float admission_sq() const { return wsize < b ? CUDART_INF_F : zmax_sq; }
    __device__ float admission_dist() const { return wsize < b ? CUDART_INF_F : zmax_dist; }

    // owner o's caches from per-lane candidates (one set of warp reductions);
    // W ids are distinct, so (key, id) names one slot, whose lane supplies
    // slot and aux; the max is the lowest slot among equal keys
    __device__ void fold(uint32_t o, uint32_t nk, uint32_t ni, uint32_t ns, uint32_t na, uint32_t xk, uint32_t xs,
                         uint32_t xi, uint32_t xa, int lane) {
        const uint32_t m1 = __reduce_min_sync(FULL, ns == EMPTY ? 0xffffffffu : nk);
        const bool c1 = ns != EMPTY && nk == m1;
        const uint32_t m2 = __reduce_min_sync(FULL, c1 ? ni : 0xffffffffu);
        const uint32_t x1 = __reduce_max_sync(FULL, xs == EMPTY ? 0u : xk);
        const uint32_t xs1 = __reduce_min_sync(FULL, (xs != EMPTY && xk == x1) ? xs : EMPTY);
        uint32_t s1, a1 = 0, xi1 = 0, xa1 = 0;
        if (WOFF) {
            const uint32_t wm = __ballot_sync(FULL, c1 && ni == m2);
            const int lm = wm ? __ffs(wm) - 1 : 0;
            s1 = wm ? __shfl_sync(FULL, ns, lm) : EMPTY;
            a1 = __shfl_sync(FULL, na, lm);
            const uint32_t wx = __ballot_sync(FULL, xs != EMPTY && xs == xs1);
            const int lx = wx ? __ffs(wx) - 1 : 0;
            xi1 = __shfl_sync(FULL, xi, lx);
            xa1 = __shfl_sync(FULL, xa, lx);
        } else {
            s1 = __reduce_min_sync(FULL, (c1 && ni == m2) ? ns : EMPTY);
        }
        if (static_cast<uint32_t>(lane) == o) {
            mn_key = m1;
            mn_id = m2;
            mn_slot = s1;
            mx_key = x1;
            mx_slot = xs1;
            if (WOFF) {
                mn_aux = a1;
                mx_id = xi1;
                mx_aux = xa1;
            }
        }
    }
    // re-derive owner o's caches from its slots (warp-cooperative)
    __device__ void rescan(uint32_t o, int lane) {
        if (WOFF && pend_o == o) pend_o = EMPTY;  // superseded
        uint32_t nk = 0xffffffffu, ni = 0xffffffffu, ns = EMPTY, na = 0, xk = 0, xs = EMPTY, xi = 0, xa = 0;
        for (uint32_t j = lane; j < S; j += 32) {
            const uint32_t i = o * S + j;
            if (i >= wsize) break;
            const uint32_t k = fkey(WOFF ? ld_keep(W.sq + i) : W.sq[i]);
            const uint32_t a = WOFF ? ld_keep(W.aux + i) : W.aux[i];
            const uint32_t id = WOFF ? ld_keep(W.id + i) : 0u;
            if (xs == EMPTY || k > xk) {
                xk = k;
                xs = i;
                xi = id;
                xa = a;
            }
            if (!(a & VISITED)) {
                const uint32_t idn = WOFF ? id : W.id[i];
                if (ns == EMPTY || k < nk || (k == nk && idn < ni)) {
                    nk = k;
                    ni = idn;
                    ns = i;
                    na = a;
                }
            }
        }
        fold(o, nk, ni, ns, na, xk, xs, xi, xa, lane);
    }
    // WOFF: fold the in-flight re-scan of pend_o (S <= 32: one slot per lane)
    __device__ void fold_pending(int lane) {
        if (!WOFF || pend_o == EMPTY) return;
        const uint32_t o = pend_o;
        pend_o = EMPTY;
        uint32_t nk = 0xffffffffu, ni = 0xffffffffu, ns = EMPTY, na = 0, xk = 0, xs = EMPTY, xi = 0, xa = 0;
        const uint32_t i = o * S + static_cast<uint32_t>(lane);
        if (static_cast<uint32_t>(lane) < S && i < wsize) {
            xk = pk;
            xs = i;
            xi = pid;
            xa = pax;
            if (!(pax & VISITED)) {
                nk = pk;
                ni = pid;
                ns = i;
                na = pax;
            }
        }
        fold(o, nk, ni, ns, na, xk, xs, xi, xa, lane);
    }
    // routing.cpp:32-44 from the caches: argmax, first slot on ties
    __device__ void zmax_from_caches() {
        const uint32_t m = __reduce_max_sync(FULL, mx_slot == EMPTY ? 0u : mx_key);
        zmax_sq = __uint_as_float(m);  // the key is the value (sq >= 0: x + 0 == x)
        zmax_dist = __fsqrt_rn(zmax_sq);
        zmax_idx = __reduce_min_sync(FULL, (mx_slot != EMPTY && mx_key == m) ? mx_slot : EMPTY);
        if (WOFF) {
            const uint32_t wz = __ballot_sync(FULL, mx_slot != EMPTY && mx_slot == zmax_idx);
            const int lz = wz ? __ffs(wz) - 1 : 0;
            zmax_id = __shfl_sync(FULL, mx_id, lz);
            zmax_aux = __shfl_sync(FULL, mx_aux, lz);
        }
    }
    __device__ void recompute_zmax(int lane) {  // after a wholesale refill of W
        clear_caches();
        if (wsize == 0) {
            zmax_sq = zmax_dist = 0.0f;
            zmax_idx = 0;
            return;
        }
        const uint32_t owners = (wsize + S - 1) / S;
        for (uint32_t o = 0; o < owners; ++o) rescan(o, lane);
        zmax_from_caches();
    }
    // routing.cpp:71-80: argmin over unvisited by (sq, id)
    __device__ uint32_t next_unvisited(int lane) {
        fold_pending(lane);
        if (!__ballot_sync(FULL, mn_slot != EMPTY)) return EMPTY;
        const uint32_t m1 = __reduce_min_sync(FULL, mn_slot == EMPTY ? 0xffffffffu : mn_key);
        const bool c1 = mn_slot != EMPTY && mn_key == m1;
        const uint32_t m2 = __reduce_min_sync(FULL, c1 ? mn_id : 0xffffffffu);
        if (!WOFF) return __reduce_min_sync(FULL, (c1 && mn_id == m2) ? mn_slot : EMPTY);
        const int l = __ffs(__ballot_sync(FULL, c1 && mn_id == m2)) - 1;  // distinct ids: one owner
        nx_slot = __shfl_sync(FULL, mn_slot, l);
        nx_aux = __shfl_sync(FULL, mn_aux, l);
        nx_id = m2;
        nx_sq = __uint_as_float(m1);  // the key is the value (sq >= 0)
        return nx_slot;
    }
    __device__ void entry(uint32_t slot, uint32_t& id, float& sq, uint32_t& deg) const {
        if (WOFF && slot == nx_slot) {
            id = nx_id;
            sq = nx_sq;
            deg = nx_aux & ~VISITED;
            return;
        }
        id = W.id[slot];
        sq = W.sq[slot];
        deg = W.aux[slot] & ~VISITED;
    }
    __device__ uint32_t entry_id(uint32_t slot) const { return W.id[slot]; }
    __device__ void set_visited(uint32_t slot, int lane) {
        if (WOFF && slot == nx_slot && S <= 32) {
            // no read: the flag is stored, the owner's slots are requested now
            // and folded in before the next argmin (fold_pending)
            const uint32_t o = slot / S;
            if (lane == 0) W.aux[slot] = nx_aux | VISITED;
            nx_slot = EMPTY;
            const uint32_t i = o * S + static_cast<uint32_t>(lane);
            if (static_cast<uint32_t>(lane) < S && i < wsize) {
                pk = fkey(ld_keep(W.sq + i));
                pid = ld_keep(W.id + i);
                pax = (i == slot) ? (nx_aux | VISITED) : ld_keep(W.aux + i);
            }
            pend_o = o;
            __syncwarp();
            return;
        }
        const uint32_t a = W.aux[slot];
        __syncwarp();
        if (lane == 0) W.aux[slot] = a | VISITED;
        __syncwarp();
        rescan(slot / S, lane);
    }
    __device__ void append(uint32_t id, float sq, uint32_t deg, int lane) {
        const uint32_t slot = wsize;
        if (WOFF && pend_o == slot / S) fold_pending(lane);
        if (lane == 0) {
            W.id[slot] = id;
            W.sq[slot] = sq;
            W.aux[slot] = deg;
        }
        if (static_cast<uint32_t>(lane) == slot / S) {  // the owner folds the new slot in
            const uint32_t k = fkey(sq);
            if (mn_slot == EMPTY || k < mn_key || (k == mn_key && id < mn_id)) {
                mn_key = k;
                mn_id = id;
                mn_slot = slot;
                if (WOFF) mn_aux = deg;
            }
            if (mx_slot == EMPTY || k > mx_key) {
                mx_key = k;
                mx_slot = slot;
                if (WOFF) {
                    mx_id = id;
                    mx_aux = deg;
                }
            }
        }
        ++wsize;
        if (sq > zmax_sq || wsize == 1) {
            zmax_idx = wsize - 1;
            zmax_sq = sq;
            zmax_dist = __fsqrt_rn(sq);
            if (WOFF) {
                zmax_id = id;
                zmax_aux = deg;
            }
        }
        __syncwarp();
    }
    __device__ static void ring_push(const Arr& r, uint32_t cap, uint32_t& head, uint32_t& size,
                                     uint32_t id, float sq, uint32_t aux, int lane) {
        uint32_t pos = head + size;
        if (pos >= cap) pos -= cap;
        if (lane == 0) {
            r.id[pos] = id;
            r.sq[pos] = sq;
            r.aux[pos] = aux;
        }
        if (size < cap) ++size;
        else head = (head + 1 == cap) ? 0 : head + 1;
    }
    __device__ void push_fp(uint32_t id, float sq, uint32_t deg, int lane) {
        ring_push(rf, b, rf_head, rf_size, id, sq, deg, lane);
        __syncwarp();
    }
    // push_fp of the lanes in pm in lane order; b > 32 >= popc(pm), so no two
    // pushes of one call share a slot
    __device__ void push_fp_many(uint32_t pm, uint32_t id, float sq, uint32_t deg, int lane) {
        if ((pm >> lane) & 1u) {
            uint32_t pos = rf_head + rf_size + __popc(pm & ((1u << lane) - 1u));
            while (pos >= b) pos -= b;
            rf.id[pos] = id;
            rf.sq[pos] = sq;
            rf.aux[pos] = deg;
        }
        const uint32_t tot = rf_size + __popc(pm);
        if (tot <= b) {
            rf_size = tot;
        } else {
            uint32_t h = rf_head + (tot - b);
            while (h >= b) h -= b;
            rf_head = h;
            rf_size = b;
        }
        __syncwarp();
    }
    __device__ void admit(uint32_t id, float sq, uint32_t deg, int lane, bool rings_live) {
        if (wsize < b) {
            append(id, sq, deg, lane);
            return;
        }
        const uint32_t z = zmax_idx;
        if (!rings_live) {
            // single round: R_T is never read
        } else if (WOFF) {
            ring_push(rt, b, rt_head, rt_size, zmax_id, zmax_sq, zmax_aux & ~VISITED, lane);
        } else {
            const uint32_t oid = W.id[z];
            const float osq = W.sq[z];
            const uint32_t oaux = W.aux[z] & ~VISITED;
            __syncwarp();
            ring_push(rt, b, rt_head, rt_size, oid, osq, oaux, lane);
        }
        if (lane == 0) {
            W.id[z] = id;
            W.sq[z] = sq;
            W.aux[z] = deg;
        }
        __syncwarp();
        rescan(z / S, lane);
        zmax_from_caches();
    }
#ifdef PAG_VALIDATE
    __device__ float w_max(int lane) const {
        uint32_t k = 0;
        for (uint32_t i = lane; i < wsize; i += 32) k = max(k, fkey(W.sq[i]));
        return __uint_as_float(__reduce_max_sync(FULL, k));
    }
    __device__ uint32_t dump_ids(uint32_t* dst, int lane) const {
        for (uint32_t i = lane; i < wsize; i += 32) dst[i] = W.id[i];
        for (uint32_t i = lane; i < rf_size; i += 32) dst[wsize + i] = rf.id[(rf_head + i) % b];
        for (uint32_t i = lane; i < rt_size; i += 32) dst[wsize + rf_size + i] = rt.id[(rt_head + i) % b];
        return wsize + rf_size + rt_size;
    }
#endif
    __device__ void flush(Common& c, int lane) {
        for (uint32_t i = lane; i < wsize; i += 32) rl_append(c, W.id[i], W.sq[i], true, i);
        c.rl_size += wsize;
        __syncwarp();
    }
    __device__ bool end_round(Common& c, int lane) {
        flush(c, lane);
        wsize = 0;
        for (uint32_t i = lane; i < rf_size; i += 32) {
            uint32_t p = rf_head + i;
            if (p >= b) p -= b;
            mi.id[i] = rf.id[p];
            mi.sq[i] = rf.sq[p];
            mi.aux[i] = rf.aux[p];
        }
        const uint32_t nf = rf_size;
        for (uint32_t i = lane; i < rt_size; i += 32) {
            uint32_t p = rt_head + i;
            if (p >= b) p -= b;
            mi.id[nf + i] = rt.id[p];
            mi.sq[nf + i] = rt.sq[p];
            mi.aux[nf + i] = rt.aux[p];
        }
        const uint32_t nm = nf + rt_size;
        rf_head = rf_size = rt_head = rt_size = 0;
        __syncwarp();
        if (nm == 0) {
            zmax_sq = zmax_dist = 0.0f;
            clear_caches();
            return false;
        }
        const Arr srt = warp_sort(mi, c.mo(), nm, lane);
        const uint32_t refill = min(nm, b);
        for (uint32_t i = lane; i < nm; i += 32) {
            if (i < refill) {
                W.id[i] = srt.id[i];
                W.sq[i] = srt.sq[i];
                W.aux[i] = srt.aux[i];
            } else {
                const uint32_t p = i - refill;
                rt.id[p] = srt.id[i];
                rt.sq[p] = srt.sq[i];
                rt.aux[p] = srt.aux[i];
            }
        }
        wsize = refill;
        rt_size = nm - refill;
        __syncwarp();
        recompute_zmax(lane);
        return true;
    }
};

// ---------------------------------------------------------------------------
// Exact squared distances for the rows named by lanes in `items` (lane j:
// row id w). Results land in c.sqbuf[j], deg[w] in c.degbuf()[j].
// EXACT: the reference order (vecstore.cpp:77-95), from the chain-interleaved
//   row copy: 4 lanes per row run the four strided accumulator chains
//   serially, 8 rows per batch (dist_exact_x).
// !EXACT: lane-parallel packed-FMA partials + xor tree (within 1e-5 rel).
// NCH > 0: padded_dim == dstride == 128 * NCH (compile-time chunk count);
// NCH == 0: any padded_dim.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float2 sq2n(float2 v, float2 nq) {  // (v + nq)^2 per component, no contraction
    const float2 d = __fadd2_rn(v, nq);
    return __fmul2_rn(d, d);
}

__device__ __forceinline__ int take_batch(uint32_t& rest, int (&jr)[4]) {
    int nb = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        jr[r] = 0;
        if (rest) {
            jr[r] = __ffs(rest) - 1;
            rest &= rest - 1;
            nb = r + 1;
        }
    }
    return nb;
}

// Reference-order distances (vecstore.cpp:77-95) from the chain-interleaved
// row copy (pag_device.h chain_positions): lane 4r + c runs accumulator chain
// c of the batch's r-th row, up to 8 rows per batch. A 128-B line of rowsX
// holds 8 consecutive elements of each of the four chains, so the lane's
// next 8 chain elements are one 32-B load (the four lanes of a row read whole
// lines) and no transposition is needed: packed differences and squares, then
// the 8 serial adds of the chain. The tail elements of a padded_dim that is
// not a multiple of 4 are extra chain-0 positions in the layout (zeros for
// the other chains), and the layout's zero padding adds +0 to every chain,
// so any shape runs the same loop. The query is laid out the same way in
// smem, negated (interleave_query): x - q is computed as x + (-q), the same
// value bit for bit. NLN: lines per row, 0 = run-time count.
struct F8 {
    float4 lo, hi;
};
__device__ __forceinline__ F8 ldg_f8(const float* p) {
    F8 v;
    asm volatile("ld.global.nc.L2::cache_hint.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8], %9;"
                 : "=f"(v.lo.x), "=f"(v.lo.y), "=f"(v.lo.z), "=f"(v.lo.w), "=f"(v.hi.x), "=f"(v.hi.y),
                   "=f"(v.hi.z), "=f"(v.hi.w)
                 : "l"(p), "l"(row_policy()));
    return v;
}

template <int NLN>
__device__ void dist_exact_x(const SearchLaunch& P, Common& c, uint32_t items, uint32_t w, int lane) {
    // lines in flight per lane (register budget; cfg-2: 4 / 6 / 8 / 12 -> 2.30 / 2.23 / 2.33 / 2.35 ms)
    constexpr int LA = NLN ? (PAG_OCC >= 6 ? 3 : 6) : 2;
    const IndexView& ix = P.ix;
    const uint32_t XS = NLN ? 32u * NLN : ix.xstride;
    const uint32_t nln = NLN ? NLN : XS / 32u;
    const int cr = lane >> 2, cc = lane & 3;
    uint32_t rest = items;
    while (rest) {
        // this lane's row: the cr-th remaining survivor (none: idle lane)
        int jm = -1;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            if (rest) {
                if (r == cr) jm = __ffs(rest) - 1;
                rest &= rest - 1;
            }
        }
        const uint32_t wr = __shfl_sync(FULL, w, jm < 0 ? 0 : jm);
        float acc = 0.0f;
        if (jm >= 0) {
            const float* rp = ix.rowsX + static_cast<uint64_t>(wr) * XS + 8u * cc;
            const float* qp = c.q + 8u * cc;
            F8 buf[LA];
#pragma unroll
            for (int i = 0; i < LA; ++i)
                if (NLN ? (i < NLN) : (static_cast<uint32_t>(i) < nln)) buf[i] = ldg_f8(rp + 32 * i);
            // the construction kernels (PES) are the largest (143 KB of SASS, 23% of
            // their stall samples wait for instructions): there the line loop stays
            // rolled, 6 lines per iteration (7.32 vs 7.64 ms per 10k nodes); the query
            // kernels run it fully unrolled (cfg-2: 2.26 vs 2.37 ms rolled)
#if PAG_PES
#pragma unroll 1
#else
#pragma unroll(NLN ? (NLN + LA - 1) / LA : 1)
#endif
            for (uint32_t l0 = 0; l0 < nln; l0 += LA) {
#pragma unroll
                for (int i = 0; i < LA; ++i) {
                    const uint32_t l = l0 + i;
                    if (l < nln) {
                        const F8 v = buf[i];
                        if (l + LA < nln) buf[i] = ldg_f8(rp + 32u * (l + LA));
                        const float4 q0 = *reinterpret_cast<const float4*>(qp + 32u * l);
                        const float4 q1 = *reinterpret_cast<const float4*>(qp + 32u * l + 4);
                        const float2 e0 = sq2n(make_float2(v.lo.x, v.lo.y), make_float2(q0.x, q0.y));
                        const float2 e1 = sq2n(make_float2(v.lo.z, v.lo.w), make_float2(q0.z, q0.w));
                        const float2 e2 = sq2n(make_float2(v.hi.x, v.hi.y), make_float2(q1.x, q1.y));
                        const float2 e3 = sq2n(make_float2(v.hi.z, v.hi.w), make_float2(q1.z, q1.w));
                        acc = __fadd_rn(acc, e0.x);
                        acc = __fadd_rn(acc, e0.y);
                        acc = __fadd_rn(acc, e1.x);
                        acc = __fadd_rn(acc, e1.y);
                        acc = __fadd_rn(acc, e2.x);
                        acc = __fadd_rn(acc, e2.y);
                        acc = __fadd_rn(acc, e3.x);
                        acc = __fadd_rn(acc, e3.y);
                    }
                }
            }
        }
        const float a1 = __shfl_down_sync(FULL, acc, 1);
        const float a2 = __shfl_down_sync(FULL, acc, 2);
        const float a3 = __shfl_down_sync(FULL, acc, 3);
        if (cc == 0 && jm >= 0) c.sqbuf[jm] = __fadd_rn(__fadd_rn(acc, a1), __fadd_rn(a2, a3));
    }
}

// the padded query in smem, negated and re-laid chain-interleaved in place
// (after the projection table and the cosine norm have read it as it was):
// elements below D4 = padded & ~3 move inside their own 32-float block, the
// <= 3 tail elements become extra chain-0 positions
__device__ void interleave_query(float* q, uint32_t padded, uint32_t xstride, int lane) {
    const uint32_t D4 = padded & ~3u, P = D4 >> 2;
    const bool tail = lane < 3 && D4 + lane < padded;
    const float tv = tail ? q[D4 + lane] : 0.0f;
    __syncwarp();
    const uint32_t dst = 8u * (lane & 3) + (lane >> 2);
    for (uint32_t b0 = 0; b0 < xstride; b0 += 32) {
        const uint32_t k = b0 + lane;
        const float v = k < D4 ? -q[k] : 0.0f;
        __syncwarp();
        q[b0 + dst] = v;
    }
    __syncwarp();
    if (tail) {
        const uint32_t p = P + lane;
        q[((p >> 3) << 5) + (p & 7u)] = -tv;
    }
    __syncwarp();
}

// Warp-tree distances, two rows at a time: each half-warp owns one row and
// every lane issues all of its 2*NCH float4 loads back to back (one memory
// latency per row pair instead of one per 128-float chunk), then a 16-lane
// xor tree. For NCH <= 6 (padded_dim <= 768).
template <int NCH>
__device__ void dist_fast_pairs(const SearchLaunch& P, Common& c, uint32_t items, uint32_t w, int lane) {
    constexpr int NL = 2 * NCH;  // float4 loads per lane per row
    const IndexView& ix = P.ix;
    const uint32_t DS = 128u * NCH;
    const int half = lane >> 4, hl = lane & 15;
    uint32_t rest = items;
    while (rest) {
        const int j0 = __ffs(rest) - 1;
        rest &= rest - 1;
        int j1 = j0;
        bool two = false;
        if (rest) {
            j1 = __ffs(rest) - 1;
            rest &= rest - 1;
            two = true;
        }
        const int jm = half ? j1 : j0;
        const uint32_t wr = __shfl_sync(FULL, w, jm);
        const float* rp = ix.rows + static_cast<uint64_t>(wr) * DS + 4u * hl;
        float4 v[NL];
#pragma unroll
        for (int i = 0; i < NL; ++i) v[i] = ldg_f4(rp + 64 * i);
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int i = 0; i < NL; ++i) {
            const float4 qv = *reinterpret_cast<const float4*>(c.q + 64 * i + 4 * hl);
            const float2 dlo = __fadd2_rn(make_float2(v[i].x, v[i].y), make_float2(-qv.x, -qv.y));
            const float2 dhi = __fadd2_rn(make_float2(v[i].z, v[i].w), make_float2(-qv.z, -qv.w));
            acc = __ffma2_rn(dlo, dlo, acc);
            acc = __ffma2_rn(dhi, dhi, acc);
        }
        float s = acc.x + acc.y;
        s += __shfl_xor_sync(FULL, s, 8);
        s += __shfl_xor_sync(FULL, s, 4);
        s += __shfl_xor_sync(FULL, s, 2);
        s += __shfl_xor_sync(FULL, s, 1);
        if (hl == 0 && (half == 0 || two)) c.sqbuf[jm] = s;
    }
}

template <int NCH>
__device__ void dist_fast(const SearchLaunch& P, Common& c, uint32_t items, uint32_t w, int lane) {
    const IndexView& ix = P.ix;
    const uint32_t DS = NCH ? 128u * NCH : ix.dstride;
    const uint32_t nch = NCH ? NCH : (DS + 127u) / 128u;
    uint32_t rest = items;
    while (rest) {
        int jr[4];
        const int nb = take_batch(rest, jr);
        const float* rp[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const uint32_t wr = __shfl_sync(FULL, w, r < nb ? jr[r] : jr[0]);
            rp[r] = ix.rows + static_cast<uint64_t>(wr) * DS + 4u * lane;
        }
        float2 part[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) part[r] = make_float2(0.f, 0.f);
        // one chunk of look-ahead (rows past nb alias row 0: no load predicates)
        float4 cur[4], nxt[4];
        const bool in0 = NCH || 4u * lane < DS;
#pragma unroll
        for (int r = 0; r < 4; ++r) cur[r] = in0 ? ldg_f4(rp[r]) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll(NCH ? NCH : 1)
        for (uint32_t ch = 0; ch < nch; ++ch) {
            const uint32_t base = 128u * ch;
            const bool inn = NCH ? (ch + 1 < nch) : (base + 128u + 4u * lane < DS);
#pragma unroll
            for (int r = 0; r < 4; ++r)
                nxt[r] = inn ? ldg_f4(rp[r] + base + 128u) : make_float4(0.f, 0.f, 0.f, 0.f);
            if (NCH || base + 4u * lane < DS) {
                const float4 qv = *reinterpret_cast<const float4*>(c.q + base + 4u * lane);
                const float2 nqlo = make_float2(-qv.x, -qv.y), nqhi = make_float2(-qv.z, -qv.w);
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    if (r < nb) {
                        const float2 dlo = __fadd2_rn(make_float2(cur[r].x, cur[r].y), nqlo);
                        const float2 dhi = __fadd2_rn(make_float2(cur[r].z, cur[r].w), nqhi);
                        part[r] = __ffma2_rn(dlo, dlo, part[r]);
                        part[r] = __ffma2_rn(dhi, dhi, part[r]);
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) cur[r] = nxt[r];
        }
        // transpose-reduce the 4 row partials in 6 shuffles: after the xor-16
        // and xor-8 exchanges lane group 8r..8r+7 holds row r, then a 3-step tree
        const bool h16 = lane & 16, h8 = lane & 8;
        const float p0 = part[0].x + part[0].y, p1 = part[1].x + part[1].y;
        const float p2 = part[2].x + part[2].y, p3 = part[3].x + part[3].y;
        float k0 = h16 ? p2 : p0, k1 = h16 ? p3 : p1;
        k0 += __shfl_xor_sync(FULL, h16 ? p0 : p2, 16);
        k1 += __shfl_xor_sync(FULL, h16 ? p1 : p3, 16);
        float v = h8 ? k1 : k0;
        v += __shfl_xor_sync(FULL, h8 ? k0 : k1, 8);
        v += __shfl_xor_sync(FULL, v, 4);
        v += __shfl_xor_sync(FULL, v, 2);
        v += __shfl_xor_sync(FULL, v, 1);
        const int row = lane >> 3;
        int jrow = jr[0];
#pragma unroll
        for (int r = 1; r < 4; ++r)
            if (r == row) jrow = jr[r];
        if ((lane & 7) == 0 && row < nb) c.sqbuf[jrow] = v;
    }
}

template <bool EXACT, int NCH>
__device__ __forceinline__ void distances(const SearchLaunch& P, Common& c, uint32_t items, uint32_t w,
                                          int lane) {
    const IndexView& ix = P.ix;
    const bool mine = (items >> lane) & 1u;
    uint32_t deg = 0;
    if (mine) {
        if (EXACT)
            prefetch_row(ix.rowsX + static_cast<uint64_t>(w) * ix.xstride, ix.xstride * 4u);
        else
            prefetch_row(ix.rows + static_cast<uint64_t>(w) * ix.dstride, ix.dstride * 4u);
        deg = __ldg(ix.deg + w);  // consumed after the rows: its latency overlaps theirs
    }
    if (EXACT) {
        // padded_dim == 128 NCH: the interleaved row has 4 NCH lines
        dist_exact_x<4 * NCH>(P, c, items, w, lane);
    } else {
        if constexpr (NCH > 0 && NCH <= 8) {
            dist_fast_pairs<NCH>(P, c, items, w, lane);
        } else {
            dist_fast<NCH>(P, c, items, w, lane);
        }
    }
    if (mine) c.degbuf()[lane] = deg;
    __syncwarp();
}

// vecstore.cpp:97-108 on the padded query in smem (4 lanes, serial chains)
__device__ float query_norm(const float* q, uint32_t D, int lane) {
    const uint32_t D4 = D & ~3u;
    float acc = 0.0f;
    if (lane < 4) {
        for (uint32_t k = lane; k < D4; k += 4) acc = __fadd_rn(acc, __fmul_rn(q[k], q[k]));
        if (lane == 0)
            for (uint32_t k = D4; k < D; ++k) acc = __fadd_rn(acc, __fmul_rn(q[k], q[k]));
    }
    const float a1 = __shfl_sync(FULL, acc, 1), a2 = __shfl_sync(FULL, acc, 2),
                a3 = __shfl_sync(FULL, acc, 3), a0 = __shfl_sync(FULL, acc, 0);
    return __fsqrt_rn(__fadd_rn(__fadd_rn(a0, a1), __fadd_rn(a2, a3)));
}

// table sum of one edge's codes (projection.cpp:145-149), serial in l.
// T is stored with a row stride of 16 (m <= 16), so l*16 + code needs no
// multiply; fully unrolled for the default subspace counts.
template <int L0, int LL>
struct CodeSumStep {  // subspace L0 of LL, compile-time unrolled (immediate row offset)
    __device__ __forceinline__ static void run(float& sum, uint32_t tb, const uint32_t (&cw)[4]) {
        const uint32_t w = cw[L0 >> 3];
        constexpr int sh = 4 * (L0 & 7) - 2;
        const uint32_t off = ((sh >= 0) ? (w >> (sh >= 0 ? sh : 0)) : (w << 2)) & 0x3Cu;
        float v;
        asm("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(off | tb), "n"(L0 * 64));
        sum = __fadd_rn(sum, v);
        CodeSumStep<L0 + 1, LL>::run(sum, tb, cw);
    }
};
template <int LL>
struct CodeSumStep<LL, LL> {
    __device__ __forceinline__ static void run(float&, uint32_t, const uint32_t (&)[4]) {}
};

template <int LL>
__device__ __forceinline__ float code_sum_fixed(const float* T, const uint32_t (&cw)[4]) {
    // T is 64-B aligned in smem, so (4 * code) | base is the entry of row 0 and
    // the row offset l * 64 folds into the load's immediate: shift, and-or,
    // load, add per subspace
    const uint32_t tb = static_cast<uint32_t>(__cvta_generic_to_shared(T));
    float sum = 0.0f;
    CodeSumStep<0, LL>::run(sum, tb, cw);
    return sum;
}

__device__ __forceinline__ float code_sum(const float* T, uint32_t L, const uint32_t* cw_global,
                                          uint32_t cwp, const uint32_t (&cw)[4]) {
    if (L == 32) return code_sum_fixed<32>(T, cw);
    if (L == 16) return code_sum_fixed<16>(T, cw);
    if (L == 8) return code_sum_fixed<8>(T, cw);
    (void)cwp;
    float sum = 0.0f;
    for (uint32_t l = 0; l < L; ++l) {
        const uint32_t word = __ldg(cw_global + (l >> 3));
        sum = __fadd_rn(sum, T[l * 16 + ((word >> (4 * (l & 7))) & 15u)]);
    }
    return sum;
}

// routing.cpp:139-204 for W slot `slot`; returns out.pes_rejected
// (always false unless PES: the construction search with collect_pes)
template <class TFB, bool EXACT, int NCH, bool PES>
__device__ bool expand(const SearchLaunch& P, Common& c, TFB& s, uint32_t slot, int lane) {
    const IndexView& ix = P.ix;
    const float TAU_HI = 1.0f + 1e-6f;
    uint32_t u, deg;
    float usq;
    s.entry(slot, u, usq, deg);
    s.set_visited(slot, lane);
    ++c.n_visited;
    c.n_edges += deg;
    const float duq = __fsqrt_rn(usq);
    const bool exact_mode = (duq == 0.0f) || !P.use_prt;
    // PES margin (routing.cpp:150,190-199): rejected iff no edge reaches a
    // margin >= 0 (pes_max starts at -inf; NaN margins never raise it)
    const bool track_pes = PES && duq > 0.0f;
    bool pes_ok = false;
    const uint8_t* blk = ix.adj + static_cast<uint64_t>(u) * ix.block_bytes;
    const uint32_t S = ix.slot_stride;
    const uint32_t* tg = reinterpret_cast<const uint32_t*>(blk);
    const float* en_a = reinterpret_cast<const float*>(blk + 4u * S);
    const float* cb_a = reinterpret_cast<const float*>(blk + 8u * S);
    const float* bo_a = reinterpret_cast<const float*>(blk + 12u * S);
    const uint32_t* cw_a = reinterpret_cast<const uint32_t*>(blk + 16u * S);
    const unsigned lt = (1u << lane) - 1u;

    for (uint32_t g0 = 0; g0 < deg; g0 += 32) {
        const uint32_t j = g0 + lane;
        const bool active = j < deg;
        uint32_t w = 0;
        float en = 0.f, cbeta = 1.f, bo = 0.f;
        uint32_t cw[4] = {0, 0, 0, 0};
        if (active) {
            w = __ldg(tg + j);
            en = __ldg(en_a + j);
            cbeta = __ldg(cb_a + j);
            bo = __ldg(bo_a + j);
            const uint32_t* cp = cw_a + static_cast<uint64_t>(j) * ix.cwp;
            if (ix.cwp == 4) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(cp));
                cw[0] = v.x; cw[1] = v.y; cw[2] = v.z; cw[3] = v.w;
            } else if (ix.cwp == 2) {
                const uint2 v = __ldg(reinterpret_cast<const uint2*>(cp));
                cw[0] = v.x; cw[1] = v.y;
            } else if (ix.cwp == 1) {
                cw[0] = __ldg(cp);
            }
        }
        PT(2);
        // visited (routing.hpp:104-105): the HBM bitmap word is requested
        // before the smem probe and the PRT so that its latency overlaps them
        uint32_t bmw = 0;
        if (active && c.gt_used) bmw = bm_load(c.gbm + (w >> 5));
        const bool in_hs = active && hash_has(c, w);
        // (i) speculative PRT at the group-start radius (evaluated for every
        // active lane; only unmarked ones count)
        const float adist0 = s.admission_dist();
        float quot = 0.0f, tau0 = 0.0f;
        bool pass0 = false, have_quot = false;
        if (active) {
            if (exact_mode) {
                pass0 = true;
            } else {
                const float tau = prt_threshold(en, duq, adist0);
                tau0 = tau;
                if (tau < TAU_HI) {
                    const uint32_t* cp = cw_a + static_cast<uint64_t>(j) * ix.cwp;
                    const float sum = code_sum(c.T, ix.L, cp, ix.cwp, cw);
                    quot = __fdiv_rn(__fdiv_rn(__fsub_rn(sum, bo), duq), cbeta);
                    have_quot = true;
                    pass0 = (tau <= -1.0f) || (quot >= tau);
                }
            }
        }
        const bool cand = active && !in_hs && !((bmw >> (w & 31u)) & 1u);
        PT(3);
        const uint32_t cand_mask = __ballot_sync(FULL, cand);
        // duplicate targets inside the group (reference order: a later copy
        // is skipped when an earlier copy passed and marked it)
        // (none in an index whose groups are all duplicate-free: ix.dup_free)
        uint32_t same = cand ? 1u << lane : 0u;
        bool any_dup = false;
        if (!ix.dup_free) {
            const unsigned long long key =
                cand ? static_cast<unsigned long long>(w) : ((1ull << 32) | static_cast<unsigned>(lane));
            same = __match_any_sync(FULL, key) & cand_mask;
            any_dup = __any_sync(FULL, __popc(same) > 1);
        }

        const bool spec = cand && pass0;
        if (track_pes) {  // every edge, marked or not; quot does not depend on the radius
            float x = -CUDART_INF_F;
            if (active) {
                if (!have_quot) {
                    const uint32_t* cp = cw_a + static_cast<uint64_t>(j) * ix.cwp;
                    quot = __fdiv_rn(__fdiv_rn(__fsub_rn(code_sum(c.T, ix.L, cp, ix.cwp, cw), bo), duq), cbeta);
                }
                x = __fsub_rn(quot, __fdiv_rn(en, __fmul_rn(2.0f, duq)));
            }
            pes_ok |= __any_sync(FULL, x >= 0.0f);
        }
        // (ii) compaction, (iii) exact distances of survivors
        const uint32_t surv = __ballot_sync(FULL, spec);
#ifdef PAG_PHASE_TIMING
        c.gt_count += __popc(surv) << 16;  // diagnostic: speculative survivors (high half of stat 7)
#endif
        PT(4);
        if (surv) distances<EXACT, NCH>(P, c, surv, w, lane);
        PT(5);

        // (iv) in-order replay with the live radius, one step per admission:
        // every remaining survivor is re-tested in parallel at the current
        // radius; the passes before the first admissible one go to R_F in
        // order (the radius cannot change before it), that one is admitted
        // (the radius shrinks) and the rest are re-tested
        uint32_t passed = 0;
        if (!any_dup) {
            const float sqv = spec ? c.sqbuf[lane] : 0.0f;
            const uint32_t dgv = spec ? c.degbuf()[lane] : 0u;
            uint32_t rem = surv;
            while (rem) {
                const float adist = s.admission_dist(), asq = s.admission_sq();
                bool pl = false;
                if ((rem >> lane) & 1u) {
                    if (exact_mode) {
                        pl = true;
                    } else {
                        const float tau = adist == adist0 ? tau0 : prt_threshold(en, duq, adist);
                        pl = tau < TAU_HI && (tau <= -1.0f || quot >= tau);
                    }
                }
                const uint32_t pm = __ballot_sync(FULL, pl);
                // the radius only shrinks and the test is monotone in it: a
                // survivor failing now fails at its own (later) turn too
                rem &= pm;
                const uint32_t am = __ballot_sync(FULL, pl && sqv < asq);
                const uint32_t fp = pm & (am ? (am & (0u - am)) - 1u : 0xffffffffu);
                if (fp && rings_are_read(P)) s.push_fp_many(fp, w, sqv, dgv, lane);
                passed |= fp;
                if (!am) break;
                const int k = __ffs(am) - 1;
                // b <= 32: an admitted node is usually expanded soon, so its
                // adjacency block goes to L2 now (cfg2 +1.2%; with b = 100
                // many admissions are evicted unexpanded: cfg3 -1.8%)
                if (P.b <= 32 && lane == k)
                    prefetch_l2_bulk(ix.adj + static_cast<uint64_t>(w) * ix.block_bytes, ix.block_bytes);
                s.admit(__shfl_sync(FULL, w, k), __shfl_sync(FULL, sqv, k), __shfl_sync(FULL, dgv, k), lane,
                        rings_are_read(P));
                passed |= 1u << k;
                rem &= ~((2u << k) - 1u);
            }
            c.n_pass += __popc(passed);
            c.n_exact += __popc(passed);
        }
        uint32_t rem = any_dup ? surv : 0u;  // sequential replay (in-group duplicates)
        while (rem) {
            const int jl = __ffs(rem) - 1;
            rem &= rem - 1;
            if (any_dup) {  // rare: a target repeated inside this group
                const uint32_t same_j = __shfl_sync(FULL, same, jl);
                if (same_j & ((1u << jl) - 1u) & passed) continue;  // marked earlier in this group
            }
            const float en_j = __shfl_sync(FULL, en, jl);
            const float quot_j = __shfl_sync(FULL, quot, jl);
            const float tau0_j = __shfl_sync(FULL, tau0, jl);
            const uint32_t w_j = __shfl_sync(FULL, w, jl);
            bool pass = true;
            if (!exact_mode) {
                // the radius is unchanged since the speculative test: reuse its tau
                const float adist = s.admission_dist();
                const float tau = adist == adist0 ? tau0_j : prt_threshold(en_j, duq, adist);
                if (tau >= TAU_HI)
                    pass = false;
                else if (tau <= -1.0f)
                    pass = true;
                else
                    pass = quot_j >= tau;
            }
            if (!pass) continue;
            passed |= 1u << jl;
            ++c.n_pass;
            ++c.n_exact;
            const float sq_j = c.sqbuf[jl];
            const uint32_t deg_j = c.degbuf()[jl];
            if (sq_j < s.admission_sq()) {
                s.admit(w_j, sq_j, deg_j, lane, rings_are_read(P));
            } else {
                if (rings_are_read(P)) s.push_fp(w_j, sq_j, deg_j, lane);
            }
        }
        // marks of this group's passes (routing.cpp:183). Later lookups come
        // from the next group/expansion only (in-group duplicates are resolved
        // by `same`), so the inserts are deferred and done in parallel.
        PT(6);
        if (passed) mark_many(c, passed, w, lane);
        // a copy skipped after an earlier copy in the group passed is no test
        c.n_test += __popc(cand_mask);
        if (any_dup) c.n_test -= __popc(__ballot_sync(FULL, cand && ((same & lt & passed) != 0u)));
        PT(1);
        __syncwarp();
    }
    return track_pes && !pes_ok;
}

#ifdef PAG_VALIDATE
// Debug builds: the device counterpart of TfbState::validate
// (routing.cpp:116-137), run after every expansion and end_round. Checks
// capacities (W, both rings <= b), that z_max is the largest sq in W, and
// that no node resides twice across W, R_F, R_T and the flushed R_L entries
// (the reference's bounded sorted R_L is formed here only at the end; its
// order is checked there). Violations set kStatusTfb* bits in the query's
// status; the host raises the reference's logic_error texts.
template <class TFB>
__device__ void validate_state(const SearchLaunch& P, Common& c, TFB& s, uint8_t* gw, int lane) {
    uint32_t bad = 0;
    if (s.wsize > P.b || s.rf_size > P.b || s.rt_size > P.b) bad |= kStatusTfbCapacity;
    const float mx = s.w_max(lane);
    if (s.wsize && fkey(mx) != fkey(s.zmax_sq)) bad |= kStatusTfbZmax;
    uint32_t* dbg = reinterpret_cast<uint32_t*>(gw + P.off_dbg);
    uint32_t n = s.dump_ids(dbg, lane);
    const Arr rl = c.rl();
    for (uint32_t i = lane; i < c.rl_size; i += 32) dbg[n + i] = rl.id[i];
    n += c.rl_size;
    __syncwarp();
    bool dup = false;
    for (uint32_t i = 0; i < n; ++i) {
        const uint32_t x = dbg[i];
        for (uint32_t j = i + 1 + lane; j < n; j += 32) dup |= dbg[j] == x;
    }
    if (__any_sync(FULL, dup)) bad |= kStatusTfbDuplicate;
    __syncwarp();
    c.invalid |= bad;
}
#define PAG_VALIDATE_STATE() validate_state(P, c, s, gw, lane)
#else
#define PAG_VALIDATE_STATE() do { } while (0)
#endif

template <class TFB, bool EXACT, int NCH, bool PES>
#ifndef PAG_MIN_BLOCKS
#define PAG_MIN_BLOCKS PAG_OCC
#endif
__global__ void __launch_bounds__(128, PAG_MIN_BLOCKS) pag_search_kernel(const __grid_constant__ SearchLaunch P) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const uint32_t slot = blockIdx.x * P.warps_per_block + wib;
    uint8_t* sw = smem + static_cast<size_t>(wib) * P.warp_smem_bytes;
    uint8_t* gw = P.gscratch + static_cast<uint64_t>(slot) * P.gscratch_stride;
    const IndexView& ix = P.ix;

    Common c;
#ifdef PAG_PHASE_TIMING
    c.pt_t0 = clock64();
    for (int k = 0; k < 8; ++k) c.pt_acc[k] = 0;
#endif
    c.q = reinterpret_cast<float*>(sw + P.off_q);
    c.T = reinterpret_cast<float*>(sw + P.off_T);
    c.sqbuf = reinterpret_cast<float*>(sw + P.off_sqbuf);
    {
        uint8_t* rl = (P.rl_in_smem ? sw : gw) + P.off_rl;
        const uint32_t cap = P.rl_cap;  // >= all W flushes of a query (r_max * b + b)
        c.rl_base = rl;
        c.rl_cap = cap;
        uint8_t* mg = (P.merge_in_smem ? sw : gw) + P.off_merge;
        c.mo_base = mg + 24ull * P.b;
        c.mo_cap = 2 * P.b;
    }
    c.cap_r = P.efS;
    c.hs = reinterpret_cast<uint32_t*>(sw + P.off_hash);
    c.hs_log2 = P.hash_log2;
    c.hs_limit = P.hash_limit;
    c.gbm = P.gbm + static_cast<uint64_t>(slot) * P.gbm_words;  // zero between queries
    c.gbm_words = P.gbm_words;
    TFB s;
    s.init(P.b, sw, gw, P);
    // Programmatic dependent launch (pag_host.cpp launch_t): this grid may
    // start while the previous search launch on the stream drains its last
    // queries. Everything before a warp's first output write only reads the
    // index and this launch's own counter/scratch set; before that write the
    // warp waits for the predecessor to complete and lets the next launch be
    // scheduled (whose counter and scratch set are the predecessor's).
    bool released = false;
    auto release = [&]() {
        if (released) return;
        released = true;
        asm volatile("griddepcontrol.wait;" ::: "memory");
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    };

    while (true) {
        uint32_t qi = 0;
        if (lane == 0) qi = atomicAdd(P.qcounter, 1u) - P.qbase;  // (mod 2^32, see SearchLaunch::qbase)
        qi = __shfl_sync(FULL, qi, 0);
        if (qi >= P.nq) {  // each warp draws exactly one index >= nq
            release();
            break;
        }
        const uint32_t qid = qi;

        // ---- reset (routing.cpp:12-30)
        c.rl_size = 0;
        c.hs_count = 0;
        c.gt_count = 0;
        c.gt_used = false;
        c.n_exact = c.n_test = c.n_pass = c.n_visited = c.n_edges = c.n_pes = 0;
#ifdef PAG_VALIDATE
        c.invalid = 0;
#endif
        s.reset();
        for (uint32_t i = lane; i < (1u << c.hs_log2) / 4; i += 32)
            reinterpret_cast<uint4*>(c.hs)[i] = make_uint4(EMPTY, EMPTY, EMPTY, EMPTY);

        // ---- query prep (routing.cpp:253-259): pad, cosine-normalise
        uint32_t status = 0;
        if (P.qnodes) {  // construction: the node's stored (padded, normalised) row as is
            const float* row = ix.rows + static_cast<uint64_t>(P.qnodes[qid]) * ix.dstride;
            for (uint32_t k = lane; k < ix.dstride; k += 32) c.q[k] = (k < ix.padded) ? __ldg(row + k) : 0.0f;
            __syncwarp();
        } else {
            const float* qraw = P.queries + static_cast<uint64_t>(qid) * ix.dim;
            if (ix.dim == ix.dstride && (reinterpret_cast<uintptr_t>(qraw) & 15u) == 0) {  // 16-B rows
                for (uint32_t k = lane; k < ix.dim / 4; k += 32)
                    reinterpret_cast<float4*>(c.q)[k] = __ldg(reinterpret_cast<const float4*>(qraw) + k);
            } else {
                for (uint32_t k = lane; k < ix.dstride; k += 32) c.q[k] = (k < ix.dim) ? __ldg(qraw + k) : 0.0f;
            }
            __syncwarp();
        }
        if (ix.cosine && !P.qnodes) {
            const float nrm = query_norm(c.q, ix.padded, lane);
            if (nrm == 0.0f) {
                status |= kStatusZeroCosineQuery;
            } else {
                __syncwarp();
                for (uint32_t k = lane; k < ix.padded; k += 32) c.q[k] = __fdiv_rn(c.q[k], nrm);
            }
            __syncwarp();
        }
        if (status) {
            release();
            if (lane == 0) {
                P.out_n[qid] = 0;
                uint32_t* st = P.out_stats + static_cast<uint64_t>(qid) * kStatWords;
                for (int i = 0; i < kStatWords; ++i) st[i] = 0;
                st[kStatStatus] = status;
            }
            continue;
        }

        // ---- seeds (routing.cpp:219-227): first <= b unmarked valid entries.
        // Their rows are requested before the table is built so the two overlap.
        uint32_t seed_sel[2] = {0, 0}, seed_id[2] = {0, 0};
        {
            uint32_t room = P.b;
            for (uint32_t e0 = 0, g = 0; e0 < ix.n_entries && room && g < 2; e0 += 32, ++g) {
                for (uint32_t t = 0; t < 32 && e0 + t < ix.n_entries && room; ++t) {
                    const uint32_t id = __ldg(ix.entries + e0 + t);
                    if (static_cast<uint64_t>(id) >= ix.n) continue;
                    if (marked(c, id)) continue;
                    mark(c, id, lane);
                    if (lane == static_cast<int>(t)) seed_id[g] = id;
                    seed_sel[g] |= 1u << t;
                    --room;
                }
            }
            if ((seed_sel[0] >> lane) & 1u) {
                if (EXACT)
                    prefetch_l2_bulk(ix.rowsX + static_cast<uint64_t>(seed_id[0]) * ix.xstride, ix.xstride * 4u);
                else
                    prefetch_l2_bulk(ix.rows + static_cast<uint64_t>(seed_id[0]) * ix.dstride, ix.dstride * 4u);
            }
        }

        // ---- projection table (projection.cpp:123-137), serial dot per entry
        {
            // four entries per lane at a time: four independent serial chains
            // interleave instead of one chain's latency per entry
            const uint32_t Lm = ix.L * ix.m, sub = ix.sub_dim, m = ix.m;
            for (uint32_t e0 = 0; e0 < Lm; e0 += 128) {
                const float* xl[4];
                const float* rT[4];
                uint32_t to[4];
                float dot[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t e = min(e0 + lane + 32u * k, Lm - 1u);  // clamped lanes recompute a valid entry
                    const uint32_t l = e / m, jj = e - l * m;
                    xl[k] = c.q + l * sub;
                    rT[k] = ix.refsT + static_cast<uint64_t>(l) * sub * m + jj;
                    to[k] = l * 16 + jj;  // row stride 16 (m <= 16)
                    dot[k] = 0.0f;
                }
                uint32_t cc = 0;
                for (; cc + 4 <= sub; cc += 4) {
                    float rv[4][4];
#pragma unroll
                    for (int k = 0; k < 4; ++k)
#pragma unroll
                        for (int i = 0; i < 4; ++i) rv[k][i] = __ldg(rT[k] + (cc + i) * m);
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int k = 0; k < 4; ++k) dot[k] = __fadd_rn(dot[k], __fmul_rn(xl[k][cc + i], rv[k][i]));
                }
                for (; cc < sub; ++cc)
#pragma unroll
                    for (int k = 0; k < 4; ++k) dot[k] = __fadd_rn(dot[k], __fmul_rn(xl[k][cc], __ldg(rT[k] + cc * m)));
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (e0 + lane + 32u * k < Lm) c.T[to[k]] = dot[k];
            }
        }
        __syncwarp();
        if (EXACT) interleave_query(c.q, ix.padded, ix.xstride, lane);

        for (int g = 0; g < 2; ++g) {
            if (!seed_sel[g]) continue;
            distances<EXACT, NCH>(P, c, seed_sel[g], seed_id[g], lane);
            uint32_t rem = seed_sel[g];
            while (rem) {
                const int t = __ffs(rem) - 1;
                rem &= rem - 1;
                const uint32_t id = __shfl_sync(FULL, seed_id[g], t);
                ++c.n_exact;
                s.append(id, c.sqbuf[t], c.degbuf()[t], lane);
            }
            __syncwarp();
        }
        // entry lists longer than 64 (b > 64 and n_entries > 64): remaining seeds
        for (uint32_t e0 = 64; e0 < ix.n_entries && s.wsize < P.b; e0 += 32) {
            uint32_t sel = 0, myid = 0, room = P.b - s.wsize;
            for (uint32_t t = 0; t < 32 && e0 + t < ix.n_entries && room; ++t) {
                const uint32_t id = __ldg(ix.entries + e0 + t);
                if (static_cast<uint64_t>(id) >= ix.n) continue;
                if (marked(c, id)) continue;
                mark(c, id, lane);
                if (lane == static_cast<int>(t)) myid = id;
                sel |= 1u << t;
                --room;
            }
            distances<EXACT, NCH>(P, c, sel, myid, lane);
            uint32_t rem = sel;
            while (rem) {
                const int t = __ffs(rem) - 1;
                rem &= rem - 1;
                ++c.n_exact;
                s.append(__shfl_sync(FULL, myid, t), c.sqbuf[t], c.degbuf()[t], lane);
            }
            __syncwarp();
        }

        PT(0);
        PAG_VALIDATE_STATE();
        // ---- rounds (routing.cpp:229-240)
        for (uint32_t r = 0; r < P.r_max; ++r) {
            while (true) {
                const uint32_t i = s.next_unvisited(lane);
                if (i == EMPTY) break;
                const uint32_t u = PES ? s.entry_id(i) : 0u;
                if (expand<TFB, EXACT, NCH, PES>(P, c, s, i, lane)) {  // routing.cpp:235
                    release();
                    if (lane == 0 && c.n_pes < P.pes_cap)
                        P.out_pes[static_cast<uint64_t>(qid) * P.pes_cap + c.n_pes] = u;
                    ++c.n_pes;
                }
                PAG_VALIDATE_STATE();
            }
            PT(2);
            if (r + 1 == P.r_max || !s.end_round(c, lane)) break;
            PAG_VALIDATE_STATE();
            PT(7);
        }
        // final flush (routing.cpp:242) and truncation to K (:244-246)
        PT(2);
        s.flush(c, lane);
        // R_L = the min(efS, flushed) smallest, output its first K
        // (routing.cpp:244-246): the K smallest of all flushed entries
        const uint32_t k_out = min(P.K, min(c.cap_r, c.rl_size));
        for (uint32_t i = lane; i < c.rl_size; i += 32) c.rl().aux[i] = 0u;
        __syncwarp();
        const Arr res = warp_sort(c.rl(), c.rl_tmp(), c.rl_size, lane);
#ifdef PAG_VALIDATE
        {  // routing.cpp:132-134: result list order (the sorted list R_L is cut from)
            bool bad_order = false;
            for (uint32_t i = lane + 1; i < c.rl_size; i += 32)
                bad_order |= cless(res.sq[i], res.id[i], res.sq[i - 1], res.id[i - 1]);
            if (__any_sync(FULL, bad_order)) c.invalid |= kStatusTfbOrder;
        }
#endif
        release();
        for (uint32_t i = lane; i < k_out; i += 32) {
            P.out_ids[static_cast<uint64_t>(qid) * P.K + i] = res.id[i];
            P.out_sq[static_cast<uint64_t>(qid) * P.K + i] = res.sq[i];
        }
        PT(7);
        if (lane == 0) {
            P.out_n[qid] = k_out;
            uint32_t* st = P.out_stats + static_cast<uint64_t>(qid) * kStatWords;
            st[kStatExact] = c.n_exact;
            st[kStatTest] = c.n_test;
            st[kStatPass] = c.n_pass;
            st[kStatVisited] = c.n_visited;
            st[kStatEdges] = c.n_edges;
#ifdef PAG_VALIDATE
            st[kStatStatus] = c.invalid;
#else
            st[kStatStatus] = 0u;
#endif
            st[6] = c.hs_count + c.gt_count;  // marks held
            st[7] = c.gt_count;               // of which in the HBM bitmap
            if (P.out_pes_n) P.out_pes_n[qid] = c.n_pes;
        }
        clear_bitmap(c, lane);
        __syncwarp();
    }
#ifdef PAG_PHASE_TIMING
    if (lane == 0)
        for (int k = 0; k < 8; ++k) atomicAdd(&g_phase[k], static_cast<unsigned long long>(c.pt_acc[k]));
#endif
    if (P.host_flag) {  // grid-completion flag for the asynchronous host API
        __threadfence_system();  // every lane's output writes (pinned host memory)
        __syncwarp();
        if (lane == 0 && atomicAdd(P.done_ctr, 1u) + 1u == P.n_warps) {
            *P.done_ctr = 0u;  // ready for the slot's next launch
            __threadfence_system();
            *reinterpret_cast<volatile uint32_t*>(P.host_flag) = P.flag_value;
        }
    }
}

template <class TFB, bool EXACT, int NCH>
cudaError_t launch_t(const SearchLaunch& L, int grid, size_t smem, cudaStream_t stream, int* bps) {
    auto k = pag_search_kernel<TFB, EXACT, NCH, PAG_PES != 0>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    if (bps) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, k, L.warps_per_block * 32, smem);
    // programmatic stream serialisation: the grid may be scheduled once the
    // previous search grid on the stream has triggered (see release())
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(L.warps_per_block * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    static const int pdl = std::getenv("PAG_GPU_NO_PDL") ? 0 : 1;
    attr[0].val.programmaticStreamSerializationAllowed = pdl && L.pdl;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, L);
}

template <class TFB, bool EXACT>
cudaError_t dispatch_nch(const SearchLaunch& L, int grid, size_t smem, cudaStream_t stream, int* bps) {
    const uint32_t ds = L.ix.dstride;
    const bool full = L.ix.padded == ds && ds % 128 == 0;
    switch (full ? ds / 128 : 0) {
        case 1: return launch_t<TFB, EXACT, 1>(L, grid, smem, stream, bps);
        case 4: return launch_t<TFB, EXACT, 4>(L, grid, smem, stream, bps);
        case 6: return launch_t<TFB, EXACT, 6>(L, grid, smem, stream, bps);
        case 8: return launch_t<TFB, EXACT, 8>(L, grid, smem, stream, bps);
        default: return launch_t<TFB, EXACT, 0>(L, grid, smem, stream, bps);
    }
}

cudaError_t dispatch_tfb(const SearchLaunch& L, int grid, cudaStream_t stream, int* bps) {
    const size_t smem = static_cast<size_t>(L.warp_smem_bytes) * L.warps_per_block;
    if (L.b <= 32)
        return L.exact_dist ? dispatch_nch<TfbReg, true>(L, grid, smem, stream, bps)
                            : dispatch_nch<TfbReg, false>(L, grid, smem, stream, bps);
    if (!L.W_in_smem)
        return L.exact_dist ? dispatch_nch<TfbMemT<true>, true>(L, grid, smem, stream, bps)
                            : dispatch_nch<TfbMemT<true>, false>(L, grid, smem, stream, bps);
    return L.exact_dist ? dispatch_nch<TfbMemT<false>, true>(L, grid, smem, stream, bps)
                        : dispatch_nch<TfbMemT<false>, false>(L, grid, smem, stream, bps);
}

}  // namespace

#define PAG_CAT2(a, b, c) dispatch_p##a##_o##b##c
#define PAG_CAT(a, b) PAG_CAT2(a, b, )
cudaError_t dispatch_p0_o4(const SearchLaunch& L, int grid, cudaStream_t stream, int* bps);
cudaError_t dispatch_p1_o4(const SearchLaunch& L, int grid, cudaStream_t stream, int* bps);
cudaError_t dispatch_p0_o6(const SearchLaunch& L, int grid, cudaStream_t stream, int* bps);
cudaError_t dispatch_p1_o6(const SearchLaunch& L, int grid, cudaStream_t stream, int* bps);

cudaError_t PAG_CAT(PAG_PES, PAG_OCC)(const SearchLaunch& L, int grid, cudaStream_t stream, int* bps) {
    return dispatch_tfb(L, grid, stream, bps);
}

#if PAG_PES == 0 && PAG_OCC == 4
namespace {
cudaError_t dispatch(const SearchLaunch& L, int grid, cudaStream_t stream, int* bps) {
    const bool occ6 = search_high_occupancy(L);
    if (L.collect_pes) return occ6 ? dispatch_p1_o6(L, grid, stream, bps) : dispatch_p1_o4(L, grid, stream, bps);
    return occ6 ? dispatch_p0_o6(L, grid, stream, bps) : dispatch_p0_o4(L, grid, stream, bps);
}
}  // namespace

// efS > 200 with a large working set (b > 128, K = 1000): the marks outgrow
// the on-chip visited table (up to 20k marks per query),
// W is off-chip, and latency hiding by more warps pays more than registers
// (cfg-4: 209 vs 233 ms). With b <= 128 the 128-register flavour stays faster
// at every efS (cfg-2 efS 300: 8.2 vs 9.0 ms; cfg-3 efS 800: 23.0 vs 24.4 ms).
bool search_high_occupancy(const SearchLaunch& L) {
    static const bool force_occ4 = std::getenv("PAG_GPU_OCC4") != nullptr;  // experiments
    return L.efS > 200 && L.b > 128 && !force_occ4;
}

size_t search_kernel_smem(const SearchLaunch& L) {
    return static_cast<size_t>(L.warp_smem_bytes) * L.warps_per_block;
}

bool search_uses_registers(const SearchLaunch& L) { return L.b <= 32; }

void search_phase_cycles(unsigned long long* out8, bool reset) {
#ifdef PAG_PHASE_TIMING
    cudaMemcpyFromSymbol(out8, g_phase, sizeof(unsigned long long) * 8);
    if (reset) {
        unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(g_phase, z, sizeof(z));
    }
#else
    for (int k = 0; k < 8; ++k) out8[k] = 0;
    (void)reset;
#endif
}

cudaError_t search_occupancy(const SearchLaunch& L, int* blocks_per_sm) { return dispatch(L, 0, nullptr, blocks_per_sm); }

cudaError_t launch_search(const SearchLaunch& L, int grid, cudaStream_t stream) {
    return dispatch(L, grid, stream, nullptr);
}
#endif

}  // namespace pagdev
