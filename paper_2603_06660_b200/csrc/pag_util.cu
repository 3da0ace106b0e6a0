// pag_util.cu — small device helpers for index maintenance (online-insert
// refresh).
#include <cuda_runtime.h>
#include <stdint.h>

#include "pag_device.h"

namespace pagdev {
namespace {

// block i of `staging` (block_bytes, 16-B multiple) -> adj[ids[i]]
__global__ void scatter_blocks_kernel(const uint4* __restrict__ staging, const uint32_t* __restrict__ ids,
                                      uint32_t count, uint4* __restrict__ adj, uint32_t words) {
    for (uint32_t b = blockIdx.x; b < count; b += gridDim.x) {
        const uint4* src = staging + static_cast<uint64_t>(b) * words;
        uint4* dst = adj + static_cast<uint64_t>(ids[b]) * words;
        for (uint32_t w = threadIdx.x; w < words; w += blockDim.x) dst[w] = src[w];
    }
}

// nodes whose adjacency repeats a target inside one 32-edge group (one warp
// per node; lane j holds edge g0 + j, as the search kernel does)
__global__ void dup_groups_kernel(const uint8_t* __restrict__ adj, const uint32_t* __restrict__ deg, uint64_t n,
                                  uint32_t block_bytes, uint32_t* __restrict__ count) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t u = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; u < n; u += warps) {
        const uint32_t d = deg[u];
        const uint32_t* tg = reinterpret_cast<const uint32_t*>(adj + u * block_bytes);
        bool dup = false;
        for (uint32_t g0 = 0; g0 < d; g0 += 32) {
            const bool act = g0 + lane < d;
            const unsigned long long key = act ? static_cast<unsigned long long>(tg[g0 + lane])
                                               : ((1ull << 32) | lane);
            const uint32_t same = __match_any_sync(0xffffffffu, key);  // all lanes (no short-circuit)
            dup |= act && __popc(same) > 1;
        }
        if (__any_sync(0xffffffffu, dup) && lane == 0) atomicAdd(count, 1u);
    }
}

// rows -> the chain-interleaved copy (pag_device.h chain_positions): one
// thread per output float; a row's reads stay inside its own lines
__global__ void interleave_rows_kernel(const float* __restrict__ rows, float* __restrict__ rowsX, uint64_t first,
                                       uint64_t n, uint32_t padded, uint32_t dstride, uint32_t xstride) {
    const uint32_t D4 = padded & ~3u, P = D4 >> 2;
    const uint64_t total = (n - first) * xstride;
    for (uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
         t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t row = first + t / xstride;
        const uint32_t xi = static_cast<uint32_t>(t % xstride);
        const uint32_t c = (xi >> 3) & 3u, p = ((xi >> 5) << 3) + (xi & 7u);
        float v = 0.0f;
        if (p < P)
            v = rows[row * dstride + 4u * p + c];
        else if (c == 0 && D4 + (p - P) < padded)
            v = rows[row * dstride + D4 + (p - P)];
        rowsX[row * xstride + xi] = v;
    }
}

}  // namespace

cudaError_t launch_interleave_rows(const float* rows, float* rowsX, uint64_t first, uint64_t n, uint32_t padded,
                                   uint32_t dstride, cudaStream_t stream) {
    if (n <= first) return cudaSuccess;
    interleave_rows_kernel<<<148 * 16, 256, 0, stream>>>(rows, rowsX, first, n, padded, dstride,
                                                          chain_xstride(padded));
    return cudaGetLastError();
}

cudaError_t count_dup_groups(const void* adj, const uint32_t* deg, uint64_t n, uint32_t block_bytes,
                             uint32_t* count_dev, cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(count_dev, 0, 4, stream);
    if (e != cudaSuccess || n == 0) return e;
    dup_groups_kernel<<<148 * 8, 256, 0, stream>>>(static_cast<const uint8_t*>(adj), deg, n, block_bytes, count_dev);
    return cudaGetLastError();
}

cudaError_t scatter_blocks(const void* staging, const uint32_t* ids, uint32_t count, void* adj,
                           uint32_t block_bytes, cudaStream_t stream) {
    if (count == 0) return cudaSuccess;
    const uint32_t words = block_bytes / 16;
    const unsigned grid = count < 4096u ? count : 4096u;
    scatter_blocks_kernel<<<grid, 64, 0, stream>>>(static_cast<const uint4*>(staging), ids, count,
                                                    static_cast<uint4*>(adj), words);
    return cudaGetLastError();
}

}  // namespace pagdev
