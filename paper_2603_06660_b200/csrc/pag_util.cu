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

}  // namespace

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
