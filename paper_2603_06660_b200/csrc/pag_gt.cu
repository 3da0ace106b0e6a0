// pag_gt.cu — exact brute-force ground truth on the GPU (replaces
// ground_truth, proj/src/bench.cpp:18-53): per query the top-min(k, n) base
// rows by (sq, id), with sq computed in the reference's own fp32 order
// (vecstore.cpp:77-95: four strided accumulators, no FMA, (a0+a1)+(a2+a3)),
// so ids AND distances are bit-identical to the reference.
//
// Two kernels per (query group x base chunk):
//   gt_dist_kernel   : 64x64 register-tiled distance tiles; every pair keeps
//                      its four accumulator chains in k order.
//   gt_select_kernel : one CTA per query merges the chunk into a running
//                      sorted top-k list of 64-bit keys (sq_bits << 32 | id),
//                      filtering by the current k-th key and sorting only the
//                      survivors (adaptive window, bitonic sort in smem).
#include <cuda_runtime.h>
#include <stdint.h>

#include "pag_device.h"

namespace pagdev {
namespace {

constexpr int TQ = 64, TB = 64, KC = 32;
constexpr uint32_t kGroupQ = 2048;     // queries per group
constexpr uint32_t kChunkN = 1u << 16; // base rows per chunk
constexpr int kSelThreads = 1024;
constexpr uint32_t kSelBuf = 8192;     // smem keys per select CTA (64 KB)

__global__ void __launch_bounds__(256) gt_dist_kernel(const float* __restrict__ base, uint32_t dstride,
                                                      uint32_t D4, uint32_t D,
                                                      const float* __restrict__ queries, uint32_t nqg,
                                                      uint64_t col0, uint32_t ncols,
                                                      float* __restrict__ out, uint32_t ld) {
    __shared__ __align__(16) float sQ[KC][TQ];
    __shared__ __align__(16) float sB[KC][TB];
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    const uint32_t q0 = blockIdx.y * TQ;
    const uint32_t b0 = blockIdx.x * TB;
    float acc[4][4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0f;

    for (uint32_t kc = 0; kc < D4; kc += KC) {
#pragma unroll
        for (int it = 0; it < 2; ++it) {
            const int idx = tid + 256 * it;
            const int r = idx >> 3, c4 = idx & 7;
            const uint32_t k = kc + 4 * c4;
            float4 vq = make_float4(0.f, 0.f, 0.f, 0.f), vb = make_float4(0.f, 0.f, 0.f, 0.f);
            if (q0 + r < nqg && k < D4)
                vq = *reinterpret_cast<const float4*>(queries + static_cast<uint64_t>(q0 + r) * dstride + k);
            if (b0 + r < ncols && k < D4)
                vb = __ldg(reinterpret_cast<const float4*>(base + (col0 + b0 + r) * dstride + k));
            sQ[4 * c4 + 0][r] = vq.x;
            sQ[4 * c4 + 1][r] = vq.y;
            sQ[4 * c4 + 2][r] = vq.z;
            sQ[4 * c4 + 3][r] = vq.w;
            sB[4 * c4 + 0][r] = vb.x;
            sB[4 * c4 + 1][r] = vb.y;
            sB[4 * c4 + 2][r] = vb.z;
            sB[4 * c4 + 3][r] = vb.w;
        }
        __syncthreads();
#pragma unroll 2
        for (int kk = 0; kk < KC; kk += 4) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float4 qa = *reinterpret_cast<const float4*>(&sQ[kk + e][ty * 4]);
                const float4 ba = *reinterpret_cast<const float4*>(&sB[kk + e][tx * 4]);
                const float qv[4] = {qa.x, qa.y, qa.z, qa.w};
                const float bv[4] = {ba.x, ba.y, ba.z, ba.w};
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const float d = __fsub_rn(bv[j], qv[i]);  // a = base row, b = query
                        acc[i][j][e] = __fadd_rn(acc[i][j][e], __fmul_rn(d, d));
                    }
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t qi = q0 + ty * 4 + i;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t bj = b0 + tx * 4 + j;
            if (qi < nqg && bj < ncols) {
                float a0 = acc[i][j][0];
                for (uint32_t k = D4; k < D; ++k) {  // tail into acc0 (vecstore.cpp:90-93)
                    const float d = __fsub_rn(base[(col0 + bj) * dstride + k],
                                              queries[static_cast<uint64_t>(qi) * dstride + k]);
                    a0 = __fadd_rn(a0, __fmul_rn(d, d));
                }
                out[static_cast<uint64_t>(qi) * ld + bj] =
                    __fadd_rn(__fadd_rn(a0, acc[i][j][1]), __fadd_rn(acc[i][j][2], acc[i][j][3]));
            }
        }
    }
}

__device__ __forceinline__ uint64_t make_key(float sq, uint32_t id) {
    return (static_cast<uint64_t>(__float_as_uint(sq)) << 32) | id;
}

// block-wide bitonic sort of keys[0..n), padded to a power of two with ~0
__device__ void block_sort(uint64_t* keys, uint32_t n) {
    uint32_t p = 1;
    while (p < n) p <<= 1;
    for (uint32_t i = n + threadIdx.x; i < p; i += blockDim.x) keys[i] = ~0ull;
    __syncthreads();
    for (uint32_t size = 2; size <= p; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t t = threadIdx.x; t < p / 2; t += blockDim.x) {
                const uint32_t lo = 2 * t - (t & (stride - 1));
                const uint32_t hi = lo + stride;
                const bool up = ((lo & size) == 0);
                const uint64_t a = keys[lo], b = keys[hi];
                if ((a > b) == up) {
                    keys[lo] = b;
                    keys[hi] = a;
                }
            }
            __syncthreads();
        }
    }
}

__device__ uint32_t block_count(uint32_t v, uint32_t* red) {
    v = __reduce_add_sync(0xffffffffu, v);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) red[w] = v;
    __syncthreads();
    uint32_t tot = 0;
    if (threadIdx.x < 32) {
        uint32_t x = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0u;
        tot = __reduce_add_sync(0xffffffffu, x);
        if (threadIdx.x == 0) red[32] = tot;
    }
    __syncthreads();
    tot = red[32];
    __syncthreads();
    return tot;
}

__global__ void __launch_bounds__(kSelThreads) gt_select_kernel(const float* __restrict__ dist, uint32_t ld,
                                                                uint32_t ncols, uint64_t col0, uint32_t k,
                                                                uint64_t* __restrict__ lists,
                                                                uint32_t* __restrict__ list_size) {
    extern __shared__ __align__(16) uint64_t keys[];
    __shared__ uint32_t red[33];
    __shared__ uint32_t fill;
    const uint32_t qi = blockIdx.x;
    const float* row = dist + static_cast<uint64_t>(qi) * ld;
    uint64_t* list = lists + static_cast<uint64_t>(qi) * k;
    uint32_t size = list_size[qi];
    for (uint32_t i = threadIdx.x; i < size; i += blockDim.x) keys[i] = list[i];
    __syncthreads();
    uint64_t tau = size == k ? keys[k - 1] : ~0ull;
    uint32_t pos = 0;
    uint32_t win = kSelBuf - k;
    while (pos < ncols) {
        const uint32_t w = min(win, ncols - pos);
        uint32_t c = 0;
        for (uint32_t i = threadIdx.x; i < w; i += blockDim.x) {
            const uint64_t key = make_key(row[pos + i], static_cast<uint32_t>(col0 + pos + i));
            c += key < tau ? 1u : 0u;
        }
        const uint32_t cnt = block_count(c, red);
        if (size + cnt > kSelBuf) {
            win = max(1u, w / 2);
            continue;
        }
        if (cnt) {
            if (threadIdx.x == 0) fill = size;
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < w; i += blockDim.x) {
                const uint64_t key = make_key(row[pos + i], static_cast<uint32_t>(col0 + pos + i));
                if (key < tau) keys[atomicAdd(&fill, 1u)] = key;
            }
            __syncthreads();
            block_sort(keys, size + cnt);
            size = min(k, size + cnt);
            tau = size == k ? keys[k - 1] : ~0ull;
        }
        pos += w;
        win = min(kSelBuf - k, win * 2);
        __syncthreads();
    }
    for (uint32_t i = threadIdx.x; i < size; i += blockDim.x) list[i] = keys[i];
    if (threadIdx.x == 0) list_size[qi] = size;
}

__global__ void gt_unpack_kernel(const uint64_t* __restrict__ lists, uint32_t nqg, uint32_t k,
                                 uint32_t* __restrict__ ids, float* __restrict__ sq) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= static_cast<uint64_t>(nqg) * k) return;
    const uint64_t key = lists[i];
    ids[i] = static_cast<uint32_t>(key);
    sq[i] = __uint_as_float(static_cast<uint32_t>(key >> 32));
}

}  // namespace

size_t gt_scratch_elems(uint64_t n, uint32_t nq, uint32_t k) {
    const uint64_t g = nq < kGroupQ ? nq : kGroupQ;
    const uint64_t c = n < kChunkN ? n : kChunkN;
    // distance tile + lists (2 words per key) + sizes
    return g * c + 2ull * g * k + g + 64;
}

cudaError_t launch_ground_truth(const GtLaunch& g, cudaStream_t stream) {
    if (g.k > kSelBuf / 2) return cudaErrorInvalidValue;
    const uint32_t D = g.padded, D4 = D & ~3u;
    const uint32_t chunk = static_cast<uint32_t>(g.n < kChunkN ? g.n : kChunkN);
    float* dist = g.scratch_sq;
    const uint64_t G = g.nq < kGroupQ ? g.nq : kGroupQ;
    uint64_t* lists = reinterpret_cast<uint64_t*>(g.scratch_sq + G * chunk + (G * chunk & 1));
    uint32_t* sizes = reinterpret_cast<uint32_t*>(lists + G * g.k);
    cudaError_t e = cudaFuncSetAttribute(gt_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kSelBuf * 8));
    if (e != cudaSuccess) return e;
    for (uint32_t q0 = 0; q0 < g.nq; q0 += kGroupQ) {
        const uint32_t nqg = min(kGroupQ, g.nq - q0);
        const float* qg = g.queries + static_cast<uint64_t>(q0) * g.dstride;
        e = cudaMemsetAsync(sizes, 0, 4ull * nqg, stream);
        if (e != cudaSuccess) return e;
        for (uint64_t c0 = 0; c0 < g.n; c0 += chunk) {
            const uint32_t nc = static_cast<uint32_t>((g.n - c0) < chunk ? (g.n - c0) : chunk);
            dim3 grid((nc + TB - 1) / TB, (nqg + TQ - 1) / TQ);
            gt_dist_kernel<<<grid, 256, 0, stream>>>(g.base, g.dstride, D4, D, qg, nqg, c0, nc, dist, chunk);
            gt_select_kernel<<<nqg, kSelThreads, kSelBuf * 8, stream>>>(dist, chunk, nc, c0, g.k, lists, sizes);
        }
        const uint64_t tot = static_cast<uint64_t>(nqg) * g.k;
        gt_unpack_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, stream>>>(
            lists, nqg, g.k, g.out_ids + static_cast<uint64_t>(q0) * g.k,
            g.out_sq + static_cast<uint64_t>(q0) * g.k);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace pagdev
