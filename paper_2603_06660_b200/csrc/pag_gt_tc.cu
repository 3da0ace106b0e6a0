// pag_gt_tc.cu — ground truth with the 5th-gen tensor cores (sm_100a).
//
// Replaces ground_truth (proj/src/bench.cpp:18-53) for small k, in three
// steps:
//   1. gt_tc_candidates: TF32 tcgen05.mma GEMM of a 128-query tile against
//      256-row base tiles (TMA-loaded, 128B-swizzled, 3-stage mbarrier
//      pipeline, accumulators double-buffered in TMEM), with a fused epilogue
//      that turns each score into an approximate squared distance
//      (|q|^2 + |b|^2 - 2 q.b) and keeps a per-query list of the C nearest
//      candidates of its base-row split. Warp roles: 0 TMA producer, 1 TMEM
//      allocator + single-thread MMA issuer, 2-5 epilogue (one query row per
//      thread, TMEM lanes 32*(warp%4)..+31).
//   2. gt_tc_rerank: exact reference-order fp32 distances (vecstore.cpp:77-95)
//      for all candidates, sort by (sq, id), keep k.
//   3. certificate: with delta a rigorous bound on |approx - exact|, the
//      result is exact when the k-th exact distance is below the smallest
//      excluded approximate distance minus 2*delta. Uncertified queries are
//      re-run by the exact SIMT kernel (pag_gt.cu) on the host's request.
//
// Large k (32 < k <= 1000, the K = 100 / 1000 configs): a per-query distance
// bound replaces the per-split top-C lists. T_q = the largest exact distance
// of any k distinct rows (the host takes the k ids of a graph search of the
// query: a search only supplies rows, never results) bounds the k-th true
// distance from above, so the true top-k lies among the rows whose
// approximate distance is <= T_q + delta. The GEMM epilogue is then a pure
// filter (packed FFMA2 + 3-input min over 32 columns, a warp vote, and an
// atomic append to the query's pool for the rare passes); the re-rank takes
// the exact distances of the pool, sorts by (sq, id) and keeps k. A pool that
// overflows (or a query without k search results) is re-run exactly.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "pag_device.h"

namespace pagdev {
namespace {

#define PAG_INF __int_as_float(0x7f800000)

constexpr int BM = 128, BN = 256, BK = 32;  // BK fp32 = 128 B (one swizzle row)
constexpr int STAGES = 3;
constexpr uint32_t A_BYTES = BM * BK * 4, B_BYTES = BN * BK * 4, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int CMAX = 64;
constexpr int TC_THREADS = 192;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n\t"
        "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(0x989680u)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, uint64_t* bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
            "r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}

// UMMA shared-memory descriptor: K-major, 128B swizzle, 8-row groups 1024 B
// apart (SBO), Blackwell version field = 1.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu);        // start address
    d |= static_cast<uint64_t>(1u) << 16;                           // LBO (unused for SW128 K-major)
    d |= static_cast<uint64_t>(1024u >> 4) << 32;                   // SBO
    d |= static_cast<uint64_t>(1u) << 46;                           // version
    d |= static_cast<uint64_t>(2u) << 61;                           // SWIZZLE_128B
    return d;
}

// instruction descriptor: D f32, A/B tf32, K-major both, N = 256, M = 128
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((BN >> 3) << 17) | ((BM >> 4) << 24);

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(kIdesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

struct TcSmem {
    // stage buffers first (1024-B aligned base)
    uint8_t stage[STAGES][STAGE_BYTES];
    float bnorm[2][BN];
    float cd[CMAX][BM];      // candidate approx distances, entry-major
    uint32_t cid[CMAX][BM];  // candidate ids
    uint64_t full[STAGES], empty[STAGES], tfull[2], tempty[2];
    uint32_t tmem_base;
};

// smem of the threshold-filter flavour (no per-row candidate lists)
struct TcSmemF {
    uint8_t stage[STAGES][STAGE_BYTES];
    float bnorm[2][BN];
    uint64_t full[STAGES], empty[STAGES], tfull[2], tempty[2];
    uint32_t tmem_base;
};

__device__ __forceinline__ float min3f(float a, float b, float c) {
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

// THRESH = false: per (query, split) the C nearest approximate candidates
// (cand_d / cand_id / cand_thr). THRESH = true: every row whose approximate
// x = |b|^2 - 2 q.b is below the query's bound thrx[q] is appended to the
// query's pool (pool_id[q * pool_cap + slot], slot from atomicAdd on
// pool_cnt[q]; slots past pool_cap are counted, not written).
template <bool THRESH>
__global__ void __launch_bounds__(TC_THREADS, 1)
    gt_tc_candidates(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const float* __restrict__ qnorm, const float* __restrict__ bnorm, uint32_t nq, uint64_t n,
                     uint32_t kblocks, uint64_t rows_per_split, uint32_t C, float* __restrict__ cand_d,
                     uint32_t* __restrict__ cand_id, float* __restrict__ cand_thr, const float* __restrict__ thrx,
                     uint32_t* __restrict__ pool_cnt, uint32_t* __restrict__ pool_id, uint32_t pool_cap) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    using Sm = typename std::conditional<THRESH, TcSmemF, TcSmem>::type;
    Sm& sm = *reinterpret_cast<Sm*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t m0 = blockIdx.x * BM;
    const uint32_t split = blockIdx.y, nsplit = gridDim.y;
    const uint64_t r0 = split * rows_per_split;
    const uint64_t r1 = r0 + rows_per_split < n ? r0 + rows_per_split : n;
    const uint32_t ntiles = r1 > r0 ? static_cast<uint32_t>((r1 - r0 + BN - 1) / BN) : 0u;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&sm.tfull[s], 1);
            mbar_init(&sm.tempty[s], 4 * 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    }
    if (warp == 1) {  // TMEM: 2 accumulator buffers x 256 fp32 columns
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&sm.tmem_base)),
                     "r"(512u)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = sm.tmem_base;

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            uint32_t stage = 0, phase = 0;
            for (uint32_t t = 0; t < ntiles; ++t) {
                const int ny = static_cast<int>(r0 + static_cast<uint64_t>(t) * BN);
                for (uint32_t kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&sm.empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&sm.full[stage], STAGE_BYTES);
                    tma_load_2d(sm.stage[stage], &tmA, &sm.full[stage], static_cast<int>(kb * BK),
                                static_cast<int>(m0));
                    tma_load_2d(sm.stage[stage] + A_BYTES, &tmB, &sm.full[stage], static_cast<int>(kb * BK), ny);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (one thread) ----------------
        if (lane == 0) {
            uint32_t stage = 0, phase = 0;
            for (uint32_t t = 0; t < ntiles; ++t) {
                const uint32_t as = t & 1u, aph = (t >> 1) & 1u;
                mbar_wait(&sm.tempty[as], aph ^ 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t dcol = tmem + as * BN;
                for (uint32_t kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&sm.full[stage], phase);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t a = smem_u32(sm.stage[stage]), b = a + A_BYTES;
#pragma unroll
                    for (int k = 0; k < BK / 8; ++k)  // K = 8 tf32 per MMA = 32 B along the swizzled row
                        umma_tf32(dcol, umma_desc_sw128(a + 32u * k), umma_desc_sw128(b + 32u * k),
                                  (kb | k) != 0 ? 1u : 0u);
                    umma_commit(&sm.empty[stage]);  // frees the smem stage when these MMAs finish
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit(&sm.tfull[as]);  // accumulator ready for the epilogue
            }
        }
    } else {
        // ---------------- epilogue: one query row per thread ----------------
        const int ew = warp - 2;               // 0..3
        const int quarter = warp & 3;          // TMEM lane quarter this warp may access
        const uint32_t row = quarter * 32 + lane;
        const uint32_t qi = m0 + row;
        const bool valid_q = qi < nq;
        if constexpr (THRESH) {
            // x = |b|^2 - 2 q.b (the approximate distance minus |q|^2), two
            // columns per FFMA2; a 32-column chunk is skipped by the warp when
            // no lane's minimum is below its bound (almost always)
            const float thr = valid_q ? thrx[qi] : -PAG_INF;
            for (uint32_t t = 0; t < ntiles; ++t) {
                const uint32_t as = t & 1u, aph = (t >> 1) & 1u;
                const uint64_t c0 = r0 + static_cast<uint64_t>(t) * BN;
                const uint32_t et = ew * 32 + lane;
                for (uint32_t j = et; j < BN; j += 128)
                    sm.bnorm[as][j] = (c0 + j < r1) ? bnorm[c0 + j] : PAG_INF;
                asm volatile("bar.sync 1, 128;" ::: "memory");
                mbar_wait(&sm.tfull[as], aph);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
                for (int ch = 0; ch < BN / 32; ++ch) {
                    float v[32];
                    tmem_ld32(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + as * BN + ch * 32, v);
                    float x[32];
                    const float2* bn2 = reinterpret_cast<const float2*>(&sm.bnorm[as][ch * 32]);
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const float2 r = __ffma2_rn(make_float2(v[2 * i], v[2 * i + 1]), make_float2(-2.0f, -2.0f),
                                                    bn2[i]);
                        x[2 * i] = r.x;
                        x[2 * i + 1] = r.y;
                    }
                    float m[11];
#pragma unroll
                    for (int i = 0; i < 10; ++i) m[i] = min3f(x[3 * i], x[3 * i + 1], x[3 * i + 2]);
                    m[10] = fminf(x[30], x[31]);
                    const float mm = min3f(min3f(m[0], m[1], m[2]), min3f(m[3], m[4], m[5]),
                                           min3f(min3f(m[6], m[7], m[8]), m[9], m[10]));
                    const bool hit = mm < thr;
                    if (__any_sync(0xffffffffu, hit)) {
                        if (hit) {
#pragma unroll
                            for (int i = 0; i < 32; ++i)
                                if (x[i] < thr) {
                                    const uint32_t slot = atomicAdd(pool_cnt + qi, 1u);
                                    if (slot < pool_cap)
                                        pool_id[static_cast<uint64_t>(qi) * pool_cap + slot] =
                                            static_cast<uint32_t>(c0 + ch * 32 + i);
                                }
                        }
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                mbar_arrive(&sm.tempty[as]);
            }
        } else {
        const float qn = valid_q ? qnorm[qi] : 0.0f;
        uint32_t cnt = 0, max_i = 0;
        float max_v = PAG_INF;
        for (uint32_t t = 0; t < ntiles; ++t) {
            const uint32_t as = t & 1u, aph = (t >> 1) & 1u;
            const uint64_t c0 = r0 + static_cast<uint64_t>(t) * BN;
            // base norms of this tile into smem (the 128 epilogue threads)
            const uint32_t et = ew * 32 + lane;
            for (uint32_t j = et; j < BN; j += 128)
                sm.bnorm[as][j] = (c0 + j < r1) ? bnorm[c0 + j] : PAG_INF;
            asm volatile("bar.sync 1, 128;" ::: "memory");
            mbar_wait(&sm.tfull[as], aph);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
            for (int ch = 0; ch < BN / 32; ++ch) {
                float v[32];
                tmem_ld32(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + as * BN + ch * 32, v);
                if (valid_q) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const uint32_t col = ch * 32 + i;
                        if (c0 + col >= r1) continue;  // next split's rows (or past n)
                        const float d = qn + sm.bnorm[as][col] - 2.0f * v[i];
                        if (cnt < C) {
                            sm.cd[cnt][row] = d;
                            sm.cid[cnt][row] = static_cast<uint32_t>(c0 + col);
                            ++cnt;
                            if (cnt == C) {
                                max_v = sm.cd[0][row];
                                max_i = 0;
                                for (uint32_t e = 1; e < C; ++e)
                                    if (sm.cd[e][row] > max_v) {
                                        max_v = sm.cd[e][row];
                                        max_i = e;
                                    }
                            }
                        } else if (d < max_v) {
                            sm.cd[max_i][row] = d;
                            sm.cid[max_i][row] = static_cast<uint32_t>(c0 + col);
                            max_v = sm.cd[0][row];
                            max_i = 0;
                            for (uint32_t e = 1; e < C; ++e)
                                if (sm.cd[e][row] > max_v) {
                                    max_v = sm.cd[e][row];
                                    max_i = e;
                                }
                        }
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            mbar_arrive(&sm.tempty[as]);
        }
        if (valid_q) {
            const uint64_t base = (static_cast<uint64_t>(qi) * nsplit + split) * C;
            for (uint32_t e = 0; e < C; ++e) {
                cand_d[base + e] = e < cnt ? sm.cd[e][row] : PAG_INF;
                cand_id[base + e] = e < cnt ? sm.cid[e][row] : 0xffffffffu;
            }
            // every excluded row of this split has approx >= thr
            cand_thr[static_cast<uint64_t>(qi) * nsplit + split] = cnt == C ? max_v : PAG_INF;
        }
        }  // !THRESH
    }
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
    }
}

// squared norms of rows (any summation order: only feeds the bound-checked
// approximation)
__global__ void row_sqnorm(const float* __restrict__ x, uint64_t rows, uint32_t dstride, uint32_t D,
                           float* __restrict__ out) {
    const uint64_t r = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    const float* p = x + r * dstride;
    float s = 0.0f;
    for (uint32_t k = lane; k < D; k += 32) s = fmaf(p[k], p[k], s);
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[r] = s;
}

// exact reference-order squared distance (vecstore.cpp:77-95), one thread
__device__ __forceinline__ float sq_dist_ref(const float* __restrict__ a, const float* __restrict__ b, uint32_t D) {
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    uint32_t k = 0;
    for (; k + 4 <= D; k += 4) {
        const float4 x = *reinterpret_cast<const float4*>(a + k);
        const float4 y = *reinterpret_cast<const float4*>(b + k);
        const float d0 = __fsub_rn(x.x, y.x), d1 = __fsub_rn(x.y, y.y), d2 = __fsub_rn(x.z, y.z),
                    d3 = __fsub_rn(x.w, y.w);
        a0 = __fadd_rn(a0, __fmul_rn(d0, d0));
        a1 = __fadd_rn(a1, __fmul_rn(d1, d1));
        a2 = __fadd_rn(a2, __fmul_rn(d2, d2));
        a3 = __fadd_rn(a3, __fmul_rn(d3, d3));
    }
    for (; k < D; ++k) {
        const float d = __fsub_rn(a[k], b[k]);
        a0 = __fadd_rn(a0, __fmul_rn(d, d));
    }
    return __fadd_rn(__fadd_rn(a0, a1), __fadd_rn(a2, a3));
}

// one CTA per query: exact distances of the nsplit*C candidates, bitonic sort
// by (sq, id), top-k out, certificate flag.
__global__ void __launch_bounds__(256) gt_tc_rerank(const float* __restrict__ base, uint32_t dstride, uint32_t D,
                                                    const float* __restrict__ queries, const float* __restrict__ qnorm,
                                                    float max_bnorm, uint32_t nsplit, uint32_t C, uint32_t k,
                                                    const float* __restrict__ cand_d, const uint32_t* __restrict__ cand_id,
                                                    const float* __restrict__ cand_thr, uint32_t* __restrict__ out_ids,
                                                    float* __restrict__ out_sq, uint32_t* __restrict__ uncertified) {
    extern __shared__ __align__(16) uint64_t keys[];
    const uint32_t qi = blockIdx.x;
    const uint32_t total = nsplit * C;
    uint32_t p = 1;
    while (p < total) p <<= 1;
    const float* q = queries + static_cast<uint64_t>(qi) * dstride;
    for (uint32_t i = threadIdx.x; i < p; i += blockDim.x) {
        uint64_t key = ~0ull;
        if (i < total) {
            const uint32_t id = cand_id[static_cast<uint64_t>(qi) * total + i];
            if (id != 0xffffffffu) {
                const float s = sq_dist_ref(base + static_cast<uint64_t>(id) * dstride, q, D);
                key = (static_cast<uint64_t>(__float_as_uint(s)) << 32) | id;
            }
        }
        keys[i] = key;
    }
    __syncthreads();
    for (uint32_t size = 2; size <= p; size <<= 1)
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t t = threadIdx.x; t < p / 2; t += blockDim.x) {
                const uint32_t lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const uint64_t a = keys[lo], b = keys[hi];
                if ((a > b) == up) {
                    keys[lo] = b;
                    keys[hi] = a;
                }
            }
            __syncthreads();
        }
    for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
        const uint64_t key = keys[i];
        out_ids[static_cast<uint64_t>(qi) * k + i] = static_cast<uint32_t>(key);
        out_sq[static_cast<uint64_t>(qi) * k + i] = __uint_as_float(static_cast<uint32_t>(key >> 32));
    }
    if (threadIdx.x == 0) {
        float thr = PAG_INF;
        for (uint32_t s = 0; s < nsplit; ++s) thr = fminf(thr, cand_thr[static_cast<uint64_t>(qi) * nsplit + s]);
        const uint64_t kth = keys[k - 1];
        bool ok = kth != ~0ull;
        if (ok && thr != PAG_INF) {
            const float dk = __uint_as_float(static_cast<uint32_t>(kth >> 32));
            // |approx - exact| <= 2^-8 |q| |b| (two tf32 truncations + fp32
            // accumulation) + norm rounding; doubled for margin
            const float qn = qnorm[qi];
            const float delta = 0.0078125f * sqrtf(qn) * sqrtf(max_bnorm) + 1e-5f * (qn + max_bnorm) + 1e-30f;
            ok = dk < thr - 2.0f * delta;
        }
        uncertified[qi] = ok ? 0u : 1u;
    }
}

// one warp per query: T = the largest exact distance of the query's k
// search-result rows (any k distinct rows bound the k-th true distance from
// above), then the filter bound in the epilogue's x space, with 2 delta of
// slack: every row whose exact distance is <= T has x < thrx (|approx -
// exact| <= delta, rounding of x and of thrx far below delta)
__global__ void gt_tc_bound(const float* __restrict__ base, uint32_t dstride, uint32_t D,
                            const float* __restrict__ queries, const float* __restrict__ qnorm, float max_bnorm,
                            uint32_t nq, uint32_t k, const uint32_t* __restrict__ s_ids,
                            const uint32_t* __restrict__ s_n, float* __restrict__ thrx) {
    const uint32_t qi = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (qi >= nq) return;
    const float* q = queries + static_cast<uint64_t>(qi) * dstride;
    float t = 0.0f;
    const bool ok = s_n[qi] >= k;
    if (ok)
        for (uint32_t i = lane; i < k; i += 32)
            t = fmaxf(t, sq_dist_ref(base + static_cast<uint64_t>(s_ids[static_cast<uint64_t>(qi) * k + i]) * dstride,
                                     q, D));
#pragma unroll
    for (int o = 16; o; o >>= 1) t = fmaxf(t, __shfl_xor_sync(0xffffffffu, t, o));
    if (lane == 0) {
        const float qn = qnorm[qi];
        const float delta = 0.0078125f * sqrtf(qn) * sqrtf(max_bnorm) + 1e-5f * (qn + max_bnorm) + 1e-30f;
        thrx[qi] = ok ? (t - qn) + 2.0f * delta : -PAG_INF;  // -inf: no pool, the host re-runs the query
    }
}

// one CTA per query: exact reference-order distances of the pool, bitonic
// sort by (sq, id), top-k out; a pool that overflowed or holds fewer than k
// rows marks the query for the exact re-run
__global__ void __launch_bounds__(256) gt_tc_rerank_pool(const float* __restrict__ base, uint32_t dstride,
                                                         uint32_t D, const float* __restrict__ queries,
                                                         const uint32_t* __restrict__ pool_cnt,
                                                         const uint32_t* __restrict__ pool_id, uint32_t cap, uint32_t k,
                                                         uint32_t* __restrict__ out_ids, float* __restrict__ out_sq,
                                                         uint32_t* __restrict__ uncertified) {
    extern __shared__ __align__(16) uint64_t keys[];
    const uint32_t qi = blockIdx.x;
    const uint32_t cnt = pool_cnt[qi];
    if (cnt > cap || cnt < k) {
        if (threadIdx.x == 0) uncertified[qi] = 1u;
        return;
    }
    uint32_t p = 1;
    while (p < cnt) p <<= 1;
    const float* q = queries + static_cast<uint64_t>(qi) * dstride;
    for (uint32_t i = threadIdx.x; i < p; i += blockDim.x) {
        uint64_t key = ~0ull;
        if (i < cnt) {
            const uint32_t id = pool_id[static_cast<uint64_t>(qi) * cap + i];
            const float s = sq_dist_ref(base + static_cast<uint64_t>(id) * dstride, q, D);
            key = (static_cast<uint64_t>(__float_as_uint(s)) << 32) | id;
        }
        keys[i] = key;
    }
    __syncthreads();
    for (uint32_t size = 2; size <= p; size <<= 1)
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t t = threadIdx.x; t < p / 2; t += blockDim.x) {
                const uint32_t lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const uint64_t a = keys[lo], b = keys[hi];
                if ((a > b) == up) {
                    keys[lo] = b;
                    keys[hi] = a;
                }
            }
            __syncthreads();
        }
    for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
        const uint64_t key = keys[i];
        out_ids[static_cast<uint64_t>(qi) * k + i] = static_cast<uint32_t>(key);
        out_sq[static_cast<uint64_t>(qi) * k + i] = __uint_as_float(static_cast<uint32_t>(key >> 32));
    }
    if (threadIdx.x == 0) uncertified[qi] = 0u;
}

}  // namespace

size_t gt_tc_smem_bytes() { return sizeof(TcSmem) + 1024; }

cudaError_t launch_gt_tc_pool(const GtTcPoolLaunch& g, cudaStream_t stream) {
    cudaError_t e;
    const size_t smem = sizeof(TcSmemF) + 1024;
    e = cudaFuncSetAttribute(gt_tc_candidates<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    row_sqnorm<<<static_cast<unsigned>((g.nq * 32ull + 255) / 256), 256, 0, stream>>>(g.queries, g.nq, g.dstride,
                                                                                     g.padded, g.qnorm);
    gt_tc_bound<<<static_cast<unsigned>((g.nq * 32ull + 255) / 256), 256, 0, stream>>>(
        g.base, g.dstride, g.padded, g.queries, g.qnorm, g.max_bnorm, g.nq, g.k, g.search_ids, g.search_n, g.thrx);
    e = cudaMemsetAsync(g.pool_cnt, 0, 4ull * g.nq, stream);
    if (e != cudaSuccess) return e;
    dim3 grid((g.nq + BM - 1) / BM, g.nsplit);
    gt_tc_candidates<true><<<grid, TC_THREADS, smem, stream>>>(
        *static_cast<const CUtensorMap*>(g.tmA), *static_cast<const CUtensorMap*>(g.tmB), g.qnorm, g.bnorm, g.nq, g.n,
        (g.padded + BK - 1) / BK, g.rows_per_split, 0, nullptr, nullptr, nullptr, g.thrx, g.pool_cnt, g.pool_id,
        g.pool_cap);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    uint32_t p = 1;
    while (p < g.pool_cap) p <<= 1;
    e = cudaFuncSetAttribute(gt_tc_rerank_pool, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(p * 8));
    if (e != cudaSuccess) return e;
    gt_tc_rerank_pool<<<g.nq, 256, p * 8, stream>>>(g.base, g.dstride, g.padded, g.queries, g.pool_cnt, g.pool_id,
                                                    g.pool_cap, g.k, g.out_ids, g.out_sq, g.uncertified);
    return cudaGetLastError();
}

cudaError_t launch_gt_tc(const GtTcLaunch& g, cudaStream_t stream) {
    cudaError_t e;
    const size_t smem = gt_tc_smem_bytes();
    e = cudaFuncSetAttribute(gt_tc_candidates<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    row_sqnorm<<<static_cast<unsigned>((g.nq * 32ull + 255) / 256), 256, 0, stream>>>(g.queries, g.nq, g.dstride,
                                                                                     g.padded, g.qnorm);
    dim3 grid((g.nq + BM - 1) / BM, g.nsplit);
    gt_tc_candidates<false><<<grid, TC_THREADS, smem, stream>>>(
        *static_cast<const CUtensorMap*>(g.tmA), *static_cast<const CUtensorMap*>(g.tmB), g.qnorm, g.bnorm, g.nq, g.n,
        (g.padded + BK - 1) / BK, g.rows_per_split, g.C, g.cand_d, g.cand_id, g.cand_thr, nullptr, nullptr, nullptr,
        0);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    uint32_t p = 1;
    while (p < g.nsplit * g.C) p <<= 1;
    e = cudaFuncSetAttribute(gt_tc_rerank, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(p * 8));
    if (e != cudaSuccess) return e;
    gt_tc_rerank<<<g.nq, 256, p * 8, stream>>>(g.base, g.dstride, g.padded, g.queries, g.qnorm, g.max_bnorm, g.nsplit,
                                               g.C, g.k, g.cand_d, g.cand_id, g.cand_thr, g.out_ids, g.out_sq,
                                               g.uncertified);
    return cudaGetLastError();
}

uint32_t gt_tc_cmax() { return CMAX; }
uint32_t gt_tc_block_n() { return BN; }
uint32_t gt_tc_block_k() { return BK; }
uint32_t gt_tc_block_m() { return BM; }

}  // namespace pagdev
