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
//   (iii) their exact distances, batched 8 rows per warp;
//   (iv)  an in-order replay re-evaluating the PRT with the live radius
//         before marking and admitting / pushing to R_F.
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "pag_device.h"

namespace pagdev {
namespace {

constexpr uint32_t FULL = 0xffffffffu;
constexpr uint32_t EMPTY = 0xffffffffu;
constexpr uint32_t VISITED = 0x80000000u;
constexpr int STAGE_STRIDE = 132;  // floats per staged row chunk (bank-conflict-free)
constexpr int MAX_STAGE_ROWS = 8;

__device__ __forceinline__ bool cless(float sa, uint32_t ia, float sb, uint32_t ib) {
    return sa < sb || (sa == sb && ia < ib);  // candidate_less, builder.hpp:23-25
}

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

__device__ __forceinline__ float4 ldg_f4(const float* p) {
    return __ldg(reinterpret_cast<const float4*>(p));
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

// Per-warp search state. Scalars are warp-uniform registers; arrays are
// generic pointers into this warp's smem region or its HBM slot.
struct Tfb {
    Arr W;                 // working set, cap b (aux = deg | VISITED)
    Arr rf, rt;            // FIFO rings, cap b (aux = deg)
    Arr rlA, rlB;          // result list double buffer, cap efS (aux unused)
    Arr mi, mo;            // merge scratch, cap 2b
    uint32_t b, cap_r;
    uint32_t wsize;
    float zmax_sq, zmax_dist;
    uint32_t zmax_idx;
    uint32_t rf_head, rf_size, rt_head, rt_size;
    uint32_t rl_cur, rl_size;
    // visited set
    uint32_t* hs;
    uint32_t hs_log2, hs_count;
    uint64_t* gt;
    uint32_t gt_log2, gt_count, epoch;
    bool gt_used, overflow;
    // counters
    uint32_t n_exact, n_test, n_pass, n_visited, n_edges;

    __device__ Arr rl_cur_arr() const { return rl_cur ? rlB : rlA; }
    __device__ Arr rl_next_arr() const { return rl_cur ? rlA : rlB; }
    __device__ float admission_sq() const { return wsize < b ? CUDART_INF_F : zmax_sq; }
    __device__ float admission_dist() const { return wsize < b ? CUDART_INF_F : zmax_dist; }
};

// ---- visited marks (routing.hpp:104-105): smem open addressing, spilling
// to an epoch-stamped per-slot HBM table once the smem table is half full.
__device__ __forceinline__ bool marked(const Tfb& s, uint32_t id) {
    const uint32_t mask = (1u << s.hs_log2) - 1;
    uint32_t h = hslot(id, s.hs_log2);
    while (true) {
        uint32_t v = s.hs[h];
        if (v == id) return true;
        if (v == EMPTY) break;
        h = (h + 1) & mask;
    }
    if (!s.gt_used) return false;
    const uint32_t gm = (1u << s.gt_log2) - 1;
    h = hslot(id, s.gt_log2);
    while (true) {
        uint64_t e = s.gt[h];
        if (static_cast<uint32_t>(e >> 32) != s.epoch) return false;
        if (static_cast<uint32_t>(e) == id) return true;
        h = (h + 1) & gm;
    }
}

// warp-uniform call; one lane writes
__device__ __forceinline__ void mark(Tfb& s, uint32_t id, int lane) {
    if (s.hs_count < (1u << s.hs_log2) / 2) {
        if (lane == 0) {
            const uint32_t mask = (1u << s.hs_log2) - 1;
            uint32_t h = hslot(id, s.hs_log2);
            while (s.hs[h] != EMPTY) h = (h + 1) & mask;
            s.hs[h] = id;
        }
        ++s.hs_count;
    } else {
        const uint32_t cap = 1u << s.gt_log2;
        if (s.gt_count + 1 >= cap - cap / 4) {
            s.overflow = true;  // host re-runs this query with a larger table
            return;
        }
        if (lane == 0) {
            const uint32_t gm = cap - 1;
            uint32_t h = hslot(id, s.gt_log2);
            while (static_cast<uint32_t>(s.gt[h] >> 32) == s.epoch) h = (h + 1) & gm;
            s.gt[h] = (static_cast<uint64_t>(s.epoch) << 32) | id;
        }
        s.gt_used = true;
        ++s.gt_count;
    }
    __syncwarp();
}

// ---- routing.cpp:32-44: argmax sq over W, first slot on ties
__device__ void recompute_zmax(Tfb& s, int lane) {
    if (s.wsize == 0) {
        s.zmax_sq = s.zmax_dist = 0.0f;
        s.zmax_idx = 0;
        return;
    }
    float bs = -CUDART_INF_F;
    uint32_t bi = EMPTY;
    for (uint32_t i = lane; i < s.wsize; i += 32) {
        float v = s.W.sq[i];
        if (bi == EMPTY || v > bs) {
            bs = v;
            bi = i;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        float v2 = __shfl_xor_sync(FULL, bs, o);
        uint32_t i2 = __shfl_xor_sync(FULL, bi, o);
        if (i2 != EMPTY && (bi == EMPTY || v2 > bs || (v2 == bs && i2 < bi))) {
            bs = v2;
            bi = i2;
        }
    }
    s.zmax_idx = bi;
    s.zmax_sq = bs;
    s.zmax_dist = __fsqrt_rn(bs);
}

// ---- routing.cpp:71-80: argmin over unvisited W by (sq, id); EMPTY if none
__device__ uint32_t next_unvisited(const Tfb& s, int lane) {
    float bs = CUDART_INF_F;
    uint32_t bid = EMPTY, bslot = EMPTY;
    for (uint32_t i = lane; i < s.wsize; i += 32) {
        if (s.W.aux[i] & VISITED) continue;
        float v = s.W.sq[i];
        uint32_t id = s.W.id[i];
        if (bslot == EMPTY || cless(v, id, bs, bid)) {
            bs = v;
            bid = id;
            bslot = i;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        float v2 = __shfl_xor_sync(FULL, bs, o);
        uint32_t id2 = __shfl_xor_sync(FULL, bid, o);
        uint32_t sl2 = __shfl_xor_sync(FULL, bslot, o);
        if (sl2 != EMPTY && (bslot == EMPTY || cless(v2, id2, bs, bid))) {
            bs = v2;
            bid = id2;
            bslot = sl2;
        }
    }
    return bslot;
}

// ---- ring push (routing.hpp:79-86), one lane writes
__device__ __forceinline__ void ring_push(const Arr& r, uint32_t cap, uint32_t& head,
                                          uint32_t& size, uint32_t id, float sq, uint32_t aux,
                                          int lane) {
    uint32_t pos = head + size;
    if (pos >= cap) pos -= cap;
    if (lane == 0) {
        r.id[pos] = id;
        r.sq[pos] = sq;
        r.aux[pos] = aux;
    }
    if (size < cap) {
        ++size;
    } else {
        head = (head + 1 == cap) ? 0 : head + 1;
    }
}

// ---- routing.cpp:46-53 (seed) and :55-69 (admit)
__device__ __forceinline__ void w_append(Tfb& s, uint32_t id, float sq, uint32_t deg, int lane) {
    if (lane == 0) {
        s.W.id[s.wsize] = id;
        s.W.sq[s.wsize] = sq;
        s.W.aux[s.wsize] = deg;
    }
    ++s.wsize;
    if (sq > s.zmax_sq || s.wsize == 1) {
        s.zmax_idx = s.wsize - 1;
        s.zmax_sq = sq;
        s.zmax_dist = __fsqrt_rn(sq);
    }
}

__device__ void admit(Tfb& s, uint32_t id, float sq, uint32_t deg, int lane) {
    if (s.wsize < s.b) {
        w_append(s, id, sq, deg, lane);
        __syncwarp();
        return;
    }
    const uint32_t z = s.zmax_idx;
    uint32_t oid = s.W.id[z];
    float osq = s.W.sq[z];
    uint32_t oaux = s.W.aux[z] & ~VISITED;
    __syncwarp();
    ring_push(s.rt, s.b, s.rt_head, s.rt_size, oid, osq, oaux, lane);
    if (lane == 0) {
        s.W.id[z] = id;
        s.W.sq[z] = sq;
        s.W.aux[z] = deg;
    }
    __syncwarp();
    recompute_zmax(s, lane);
}

// rank sort of n entries (distinct ids => strict total order)
__device__ void rank_sort(const Arr& in, const Arr& out, uint32_t n, int lane) {
    for (uint32_t i = lane; i < n; i += 32) {
        float v = in.sq[i];
        uint32_t id = in.id[i];
        uint32_t r = 0;
        for (uint32_t j = 0; j < n; ++j) r += cless(in.sq[j], in.id[j], v, id) ? 1u : 0u;
        out.id[r] = id;
        out.sq[r] = v;
        out.aux[r] = in.aux[i];
    }
    __syncwarp();
}

// number of entries of sorted a[0..n) strictly less than (v, id)
__device__ __forceinline__ uint32_t count_less(const Arr& a, uint32_t n, float v, uint32_t id) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (cless(a.sq[mid], a.id[mid], v, id))
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// routing.cpp:82-90 applied to a whole batch: R_L keeps the cap_r smallest
// (the bounded sorted insert is order-independent for distinct ids).
// `batch` must be sorted.
__device__ void rl_merge(Tfb& s, const Arr& batch, uint32_t nb, int lane) {
    if (nb == 0) return;
    const Arr cur = s.rl_cur_arr(), nxt = s.rl_next_arr();
    const uint32_t cap = s.cap_r;
    for (uint32_t i = lane; i < s.rl_size; i += 32) {
        float v = cur.sq[i];
        uint32_t id = cur.id[i];
        uint32_t pos = i + count_less(batch, nb, v, id);
        if (pos < cap) {
            nxt.id[pos] = id;
            nxt.sq[pos] = v;
        }
    }
    for (uint32_t j = lane; j < nb; j += 32) {
        float v = batch.sq[j];
        uint32_t id = batch.id[j];
        uint32_t pos = j + count_less(cur, s.rl_size, v, id);
        if (pos < cap) {
            nxt.id[pos] = id;
            nxt.sq[pos] = v;
        }
    }
    __syncwarp();
    s.rl_size = min(cap, s.rl_size + nb);
    s.rl_cur ^= 1;
}

// flush W into R_L (routing.cpp:93, :242)
__device__ void flush_working(Tfb& s, int lane) {
    rank_sort(s.W, s.mo, s.wsize, lane);
    rl_merge(s, s.mo, s.wsize, lane);
}

// routing.cpp:92-114
__device__ bool end_round(Tfb& s, int lane) {
    flush_working(s, lane);
    s.wsize = 0;
    uint32_t nm = 0;
    for (uint32_t i = lane; i < s.rf_size; i += 32) {
        uint32_t p = s.rf_head + i;
        if (p >= s.b) p -= s.b;
        s.mi.id[i] = s.rf.id[p];
        s.mi.sq[i] = s.rf.sq[p];
        s.mi.aux[i] = s.rf.aux[p];
    }
    nm = s.rf_size;
    for (uint32_t i = lane; i < s.rt_size; i += 32) {
        uint32_t p = s.rt_head + i;
        if (p >= s.b) p -= s.b;
        s.mi.id[nm + i] = s.rt.id[p];
        s.mi.sq[nm + i] = s.rt.sq[p];
        s.mi.aux[nm + i] = s.rt.aux[p];
    }
    nm += s.rt_size;
    s.rf_head = s.rf_size = 0;
    s.rt_head = s.rt_size = 0;
    __syncwarp();
    if (nm == 0) {
        s.zmax_sq = s.zmax_dist = 0.0f;
        return false;
    }
    rank_sort(s.mi, s.mo, nm, lane);
    const uint32_t refill = min(nm, s.b);
    for (uint32_t i = lane; i < nm; i += 32) {
        if (i < refill) {
            s.W.id[i] = s.mo.id[i];
            s.W.sq[i] = s.mo.sq[i];
            s.W.aux[i] = s.mo.aux[i];
        } else {
            uint32_t p = i - refill;  // ring_t was cleared and rest <= b
            s.rt.id[p] = s.mo.id[i];
            s.rt.sq[p] = s.mo.sq[i];
            s.rt.aux[p] = s.mo.aux[i];
        }
    }
    s.wsize = refill;
    s.rt_size = nm - refill;
    __syncwarp();
    recompute_zmax(s, lane);
    return true;
}

// ---- exact squared distances for the rows named by lanes in `items`
// (lane j: row id w). Results land in sqbuf[j] (and deg[w] in degbuf[j]).
// exact=1: the reference order (vecstore.cpp:77-95) — rows are streamed
// coalesced in 128-float chunks, squared differences staged in smem, and
// 4 lanes per row run the four strided accumulator chains serially.
// exact=0: lane-parallel FMA partials + xor-tree (ablation / fast mode).
__device__ void distances(const SearchLaunch& P, uint32_t items, uint32_t w, const float* q,
                          float* stage, float* sqbuf, uint32_t* degbuf, int lane) {
    const IndexView& ix = P.ix;
    const uint32_t DS = ix.dstride, D = ix.padded, D4 = D & ~3u;
    const int R = static_cast<int>(P.stage_rows);
    if ((items >> lane) & 1u) {
        const float* row = ix.rows + static_cast<uint64_t>(w) * DS;
        prefetch_l2_bulk(row, DS * 4u);
        degbuf[lane] = __ldg(ix.deg + w);
    }
    uint32_t rest = items;
    while (rest) {
        int jr[MAX_STAGE_ROWS];
        const float* rp[MAX_STAGE_ROWS];
        int nb = 0;
#pragma unroll
        for (int r = 0; r < MAX_STAGE_ROWS; ++r) {
            jr[r] = 0;
            if (r < R && rest) {
                jr[r] = __ffs(rest) - 1;
                rest &= rest - 1;
                nb = r + 1;
            }
            uint32_t wr = __shfl_sync(FULL, w, jr[r]);
            rp[r] = ix.rows + static_cast<uint64_t>(wr) * DS;
        }
        if (P.exact_dist) {
            const int cr = lane >> 2, cc = lane & 3;
            float acc = 0.0f;
            for (uint32_t base = 0; base < DS; base += 128) {
                const uint32_t k = base + 4u * lane;
                float4 qv = make_float4(0.f, 0.f, 0.f, 0.f);
                if (k < DS) qv = *reinterpret_cast<const float4*>(q + k);
#pragma unroll
                for (int r = 0; r < MAX_STAGE_ROWS; ++r) {
                    if (r < nb) {
                        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                        if (k < DS) v = ldg_f4(rp[r] + k);
                        float d0 = __fsub_rn(v.x, qv.x), d1 = __fsub_rn(v.y, qv.y);
                        float d2 = __fsub_rn(v.z, qv.z), d3 = __fsub_rn(v.w, qv.w);
                        float4 p = make_float4(__fmul_rn(d0, d0), __fmul_rn(d1, d1),
                                               __fmul_rn(d2, d2), __fmul_rn(d3, d3));
                        *reinterpret_cast<float4*>(stage + r * STAGE_STRIDE + 4 * lane) = p;
                    }
                }
                __syncwarp();
                if (cr < nb) {
                    const float* sp = stage + cr * STAGE_STRIDE + cc;
                    if (base + 128 <= D4) {
#pragma unroll 8
                        for (int t = 0; t < 32; ++t) acc = __fadd_rn(acc, sp[4 * t]);
                    } else {
                        for (int t = 0; t < 32; ++t) {
                            uint32_t kk = base + 4u * t + cc;
                            if (kk < D4) {
                                acc = __fadd_rn(acc, sp[4 * t]);
                            } else if (cc == 0 && kk < D) {
                                // tail elements all go to acc0, in order
                                acc = __fadd_rn(acc, sp[4 * t]);
                                if (kk + 1 < D) acc = __fadd_rn(acc, sp[4 * t + 1]);
                                if (kk + 2 < D) acc = __fadd_rn(acc, sp[4 * t + 2]);
                            }
                        }
                    }
                }
                __syncwarp();
            }
            float a1 = __shfl_down_sync(FULL, acc, 1);
            float a2 = __shfl_down_sync(FULL, acc, 2);
            float a3 = __shfl_down_sync(FULL, acc, 3);
            int jmine = 0;
#pragma unroll
            for (int r = 0; r < MAX_STAGE_ROWS; ++r)
                if (r == cr) jmine = jr[r];
            if (cc == 0 && cr < nb) sqbuf[jmine] = __fadd_rn(__fadd_rn(acc, a1), __fadd_rn(a2, a3));
        } else {
            float part[MAX_STAGE_ROWS];
#pragma unroll
            for (int r = 0; r < MAX_STAGE_ROWS; ++r) part[r] = 0.0f;
            for (uint32_t base = 0; base < DS; base += 128) {
                const uint32_t k = base + 4u * lane;
                if (k < DS) {
                    float4 qv = *reinterpret_cast<const float4*>(q + k);
#pragma unroll
                    for (int r = 0; r < MAX_STAGE_ROWS; ++r) {
                        if (r < nb) {
                            float4 v = ldg_f4(rp[r] + k);
                            float d0 = v.x - qv.x, d1 = v.y - qv.y, d2 = v.z - qv.z, d3 = v.w - qv.w;
                            part[r] = fmaf(d0, d0, part[r]);
                            part[r] = fmaf(d1, d1, part[r]);
                            part[r] = fmaf(d2, d2, part[r]);
                            part[r] = fmaf(d3, d3, part[r]);
                        }
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < MAX_STAGE_ROWS; ++r) {
                if (r < nb) {
                    float v = part[r];
#pragma unroll
                    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
                    if (lane == 0) sqbuf[jr[r]] = v;
                }
            }
        }
    }
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
    float a1 = __shfl_sync(FULL, acc, 1), a2 = __shfl_sync(FULL, acc, 2),
          a3 = __shfl_sync(FULL, acc, 3), a0 = __shfl_sync(FULL, acc, 0);
    return __fsqrt_rn(__fadd_rn(__fadd_rn(a0, a1), __fadd_rn(a2, a3)));
}

// table sum of one edge's codes (projection.cpp:145-149), serial in l
__device__ __forceinline__ float code_sum(const float* T, uint32_t L, uint32_t m,
                                          const uint32_t* cw_global, uint32_t cwp,
                                          const uint32_t (&cw)[4]) {
    float sum = 0.0f;
    if (cwp <= 4) {
#pragma unroll
        for (int wi = 0; wi < 4; ++wi) {
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const uint32_t l = wi * 8 + t;
                if (l < L) sum = __fadd_rn(sum, T[l * m + ((cw[wi] >> (4 * t)) & 15u)]);
            }
        }
    } else {
        for (uint32_t l = 0; l < L; ++l) {
            uint32_t word = __ldg(cw_global + (l >> 3));
            sum = __fadd_rn(sum, T[l * m + ((word >> (4 * (l & 7))) & 15u)]);
        }
    }
    return sum;
}

// routing.cpp:139-204 for W slot `slot`
__device__ void expand(const SearchLaunch& P, Tfb& s, uint32_t slot, const float* q,
                       const float* T, float* stage, float* sqbuf, uint32_t* degbuf, int lane) {
    const IndexView& ix = P.ix;
    const float TAU_HI = 1.0f + 1e-6f;
    const uint32_t u = s.W.id[slot];
    const float usq = s.W.sq[slot];
    const uint32_t deg = s.W.aux[slot] & ~VISITED;
    __syncwarp();
    if (lane == 0) s.W.aux[slot] = deg | VISITED;
    __syncwarp();
    ++s.n_visited;
    s.n_edges += deg;
    const float duq = __fsqrt_rn(usq);
    const bool exact_mode = (duq == 0.0f) || !P.use_prt;
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
                uint4 v = __ldg(reinterpret_cast<const uint4*>(cp));
                cw[0] = v.x; cw[1] = v.y; cw[2] = v.z; cw[3] = v.w;
            } else if (ix.cwp == 2) {
                uint2 v = __ldg(reinterpret_cast<const uint2*>(cp));
                cw[0] = v.x; cw[1] = v.y;
            } else if (ix.cwp == 1) {
                cw[0] = __ldg(cp);
            }
        }
        const bool cand = active && !marked(s, w);
        const uint32_t cand_mask = __ballot_sync(FULL, cand);
        // duplicate targets inside the group (reference order: a later copy
        // is skipped when an earlier copy passed and marked it)
        unsigned long long key =
            cand ? static_cast<unsigned long long>(w) : ((1ull << 32) | static_cast<unsigned>(lane));
        const uint32_t same = __match_any_sync(FULL, key) & cand_mask;

        // (i) speculative PRT at the group-start radius
        const float adist0 = s.admission_dist();
        float quot = 0.0f;
        bool spec = false;
        if (cand) {
            if (exact_mode) {
                spec = true;
            } else {
                float tau = prt_threshold(en, duq, adist0);
                if (tau < TAU_HI) {
                    const uint32_t* cp = cw_a + static_cast<uint64_t>(j) * ix.cwp;
                    float sum = code_sum(T, ix.L, ix.m, cp, ix.cwp, cw);
                    quot = __fdiv_rn(__fdiv_rn(__fsub_rn(sum, bo), duq), cbeta);
                    spec = (tau <= -1.0f) || (quot >= tau);
                }
            }
        }
        // (ii) compaction, (iii) exact distances of survivors
        const uint32_t surv = __ballot_sync(FULL, spec);
        if (surv) distances(P, surv, w, q, stage, sqbuf, degbuf, lane);

        // (iv) in-order replay with the live radius
        uint32_t passed = 0;
        uint32_t rem = surv;
        while (rem) {
            const int jl = __ffs(rem) - 1;
            rem &= rem - 1;
            const uint32_t same_j = __shfl_sync(FULL, same, jl);
            if (same_j & ((1u << jl) - 1u) & passed) continue;  // marked earlier in this group
            const float en_j = __shfl_sync(FULL, en, jl);
            const float quot_j = __shfl_sync(FULL, quot, jl);
            const uint32_t w_j = __shfl_sync(FULL, w, jl);
            bool pass = true;
            if (!exact_mode) {
                float tau = prt_threshold(en_j, duq, s.admission_dist());
                if (tau >= TAU_HI)
                    pass = false;
                else if (tau <= -1.0f)
                    pass = true;
                else
                    pass = quot_j >= tau;
            }
            if (!pass) continue;
            passed |= 1u << jl;
            ++s.n_pass;
            ++s.n_exact;
            const float sq_j = sqbuf[jl];
            const uint32_t deg_j = degbuf[jl];
            __syncwarp();
            mark(s, w_j, lane);
            if (sq_j < s.admission_sq()) {
                admit(s, w_j, sq_j, deg_j, lane);
            } else {
                ring_push(s.rf, s.b, s.rf_head, s.rf_size, w_j, sq_j, deg_j, lane);
                __syncwarp();
            }
        }
        const bool not_test = cand && ((same & lt & passed) != 0u);
        s.n_test += __popc(cand_mask) - __popc(__ballot_sync(FULL, not_test));
        __syncwarp();
    }
}

__global__ void __launch_bounds__(128) pag_search_kernel(const __grid_constant__ SearchLaunch P) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const uint32_t slot = blockIdx.x * P.warps_per_block + wib;
    uint8_t* sw = smem + static_cast<size_t>(wib) * P.warp_smem_bytes;
    uint8_t* gw = P.gscratch + static_cast<uint64_t>(slot) * P.gscratch_stride;
    const IndexView& ix = P.ix;

    float* q = reinterpret_cast<float*>(sw + P.off_q);
    float* T = reinterpret_cast<float*>(sw + P.off_T);
    float* sqbuf = reinterpret_cast<float*>(sw + P.off_sqbuf);
    uint32_t* degbuf = reinterpret_cast<uint32_t*>(sw + P.off_sqbuf + 128);
    float* stage = reinterpret_cast<float*>(sw + P.off_stage);

    Tfb s;
    s.b = P.b;
    s.cap_r = P.efS;
    s.W = make_arr((P.W_in_smem ? sw : gw) + P.off_W, P.b);
    s.rf = make_arr((P.rings_in_smem ? sw : gw) + P.off_rf, P.b);
    s.rt = make_arr((P.rings_in_smem ? sw : gw) + P.off_rt, P.b);
    {
        uint8_t* rl = (P.rl_in_smem ? sw : gw) + P.off_rl;
        const uint32_t cap = P.efS ? P.efS : 1;
        s.rlA = make_arr(rl, cap);
        s.rlB = make_arr(rl + 12ull * cap, cap);
        uint8_t* mg = (P.merge_in_smem ? sw : gw) + P.off_merge;
        s.mi = make_arr(mg, 2 * P.b);
        s.mo = make_arr(mg + 24ull * P.b, 2 * P.b);
    }
    s.hs = reinterpret_cast<uint32_t*>(sw + P.off_hash);
    s.hs_log2 = P.hash_log2;
    s.gt = P.gtab + (static_cast<uint64_t>(slot) << P.gtab_log2);
    s.gt_log2 = P.gtab_log2;
    uint32_t epoch = P.slot_epoch[slot];

    while (true) {
        uint32_t qi = 0;
        if (lane == 0) qi = atomicAdd(P.qcounter, 1u);
        qi = __shfl_sync(FULL, qi, 0);
        if (qi >= P.nq) break;
        const uint32_t qid = P.qlist ? P.qlist[qi] : qi;

        // ---- reset (routing.cpp:12-30)
        if (++epoch == 0) {  // epoch wrap: clear this slot's table
            for (uint32_t i = lane; i < (1u << s.gt_log2); i += 32) s.gt[i] = 0;
            epoch = 1;
        }
        s.epoch = epoch;
        s.wsize = 0;
        s.zmax_sq = s.zmax_dist = 0.0f;
        s.zmax_idx = 0;
        s.rf_head = s.rf_size = s.rt_head = s.rt_size = 0;
        s.rl_cur = 0;
        s.rl_size = 0;
        s.hs_count = 0;
        s.gt_count = 0;
        s.gt_used = false;
        s.overflow = false;
        s.n_exact = s.n_test = s.n_pass = s.n_visited = s.n_edges = 0;
        for (uint32_t i = lane; i < (1u << s.hs_log2); i += 32) s.hs[i] = EMPTY;

        // ---- query prep (routing.cpp:253-259): pad, cosine-normalise
        const float* qraw = P.queries + static_cast<uint64_t>(qid) * ix.dim;
        for (uint32_t k = lane; k < ix.dstride; k += 32) q[k] = (k < ix.dim) ? __ldg(qraw + k) : 0.0f;
        __syncwarp();
        uint32_t status = 0;
        if (ix.cosine) {
            const float nrm = query_norm(q, ix.padded, lane);
            if (nrm == 0.0f) {
                status |= kStatusZeroCosineQuery;
            } else {
                __syncwarp();
                for (uint32_t k = lane; k < ix.padded; k += 32) q[k] = __fdiv_rn(q[k], nrm);
            }
            __syncwarp();
        }
        if (status) {
            if (lane == 0) {
                P.out_n[qid] = 0;
                uint32_t* st = P.out_stats + static_cast<uint64_t>(qid) * kStatWords;
                for (int i = 0; i < kStatWords; ++i) st[i] = 0;
                st[kStatStatus] = status;
            }
            continue;
        }

        // ---- projection table (projection.cpp:123-137), serial dot per entry
        {
            const uint32_t Lm = ix.L * ix.m, sub = ix.sub_dim, m = ix.m;
            for (uint32_t e = lane; e < Lm; e += 32) {
                const uint32_t l = e / m, jj = e - l * m;
                const float* xl = q + l * sub;
                const float* rT = ix.refsT + static_cast<uint64_t>(l) * sub * m + jj;
                float dot = 0.0f;
                for (uint32_t c = 0; c < sub; ++c) dot = __fadd_rn(dot, __fmul_rn(xl[c], __ldg(rT + c * m)));
                T[e] = dot;
            }
        }
        __syncwarp();

        // ---- seeds (routing.cpp:219-227): first <= b unmarked valid entries
        for (uint32_t e0 = 0; e0 < ix.n_entries && s.wsize < s.b; e0 += 32) {
            // sequential selection (duplicates / out-of-range skipped)
            uint32_t sel = 0, myid = 0;
            uint32_t room = s.b - s.wsize;
            for (uint32_t t = 0; t < 32 && e0 + t < ix.n_entries && room; ++t) {
                const uint32_t id = __ldg(ix.entries + e0 + t);
                if (static_cast<uint64_t>(id) >= ix.n) continue;
                if (marked(s, id)) continue;
                mark(s, id, lane);
                if (lane == static_cast<int>(t)) myid = id;
                sel |= 1u << t;
                --room;
            }
            if (s.overflow) break;
            distances(P, sel, myid, q, stage, sqbuf, degbuf, lane);
            uint32_t rem = sel;
            while (rem) {
                const int t = __ffs(rem) - 1;
                rem &= rem - 1;
                const uint32_t id = __shfl_sync(FULL, myid, t);
                ++s.n_exact;
                w_append(s, id, sqbuf[t], degbuf[t], lane);
                __syncwarp();
            }
            __syncwarp();
        }

        // ---- rounds (routing.cpp:229-240)
        for (uint32_t r = 0; r < P.r_max && !s.overflow; ++r) {
            while (!s.overflow) {
                const uint32_t i = next_unvisited(s, lane);
                if (i == EMPTY) break;
                expand(P, s, i, q, T, stage, sqbuf, degbuf, lane);
            }
            if (r + 1 == P.r_max || !end_round(s, lane)) break;
        }
        // final flush (routing.cpp:242) and truncation to K (:244-246)
        flush_working(s, lane);
        const uint32_t k_out = min(P.K, s.rl_size);
        const Arr res = s.rl_cur_arr();
        for (uint32_t i = lane; i < k_out; i += 32) {
            P.out_ids[static_cast<uint64_t>(qid) * P.K + i] = res.id[i];
            P.out_sq[static_cast<uint64_t>(qid) * P.K + i] = res.sq[i];
        }
        if (lane == 0) {
            P.out_n[qid] = k_out;
            uint32_t* st = P.out_stats + static_cast<uint64_t>(qid) * kStatWords;
            st[kStatExact] = s.n_exact;
            st[kStatTest] = s.n_test;
            st[kStatPass] = s.n_pass;
            st[kStatVisited] = s.n_visited;
            st[kStatEdges] = s.n_edges;
            st[kStatStatus] = s.overflow ? kStatusVisitedOverflow : 0u;
            st[6] = s.hs_count + s.gt_count;  // marks held
            st[7] = 0;
        }
        __syncwarp();
    }
    if (lane == 0) P.slot_epoch[slot] = epoch;
}

}  // namespace

size_t search_kernel_smem(const SearchLaunch& L) {
    return static_cast<size_t>(L.warp_smem_bytes) * L.warps_per_block;
}

cudaError_t search_occupancy(int warps_per_block, size_t smem_bytes, int* blocks_per_sm) {
    cudaError_t e = cudaFuncSetAttribute(pag_search_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem_bytes));
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, pag_search_kernel,
                                                         warps_per_block * 32, smem_bytes);
}

cudaError_t launch_search(const SearchLaunch& L, int grid, cudaStream_t stream) {
    const size_t smem = search_kernel_smem(L);
    cudaError_t e = cudaFuncSetAttribute(pag_search_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    pag_search_kernel<<<grid, L.warps_per_block * 32, smem, stream>>>(L);
    return cudaGetLastError();
}

}  // namespace pagdev
