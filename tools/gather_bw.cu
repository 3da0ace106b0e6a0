// Random-row gather bandwidth on this GPU: the practical ceiling for the
// search kernel's access pattern (rows of `row_bytes` at random ids from a
// multi-GB array, whole rows read with 16-B loads). Each warp reads `rpw`
// rows at a time (independent, all loads in flight), sums them and writes one
// float per warp. Prints GB/s for several row sizes / rows in flight.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bw gather_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

template <int RPW>
__global__ void gather(const float4* __restrict__ base, uint64_t nrows, uint32_t row_f4, uint32_t iters,
                       float* out) {
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    float acc = 0.f;
    for (uint32_t it = 0; it < iters; ++it) {
        const float4* rp[RPW];
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
            const uint32_t id = hash32(warp * 7919u + it * 104729u + r * 31u) % nrows;
            rp[r] = base + static_cast<uint64_t>(id) * row_f4;
        }
        for (uint32_t k = lane; k < row_f4; k += 32) {
            float4 v[RPW];
#pragma unroll
            for (int r = 0; r < RPW; ++r) v[r] = __ldg(rp[r] + k);
#pragma unroll
            for (int r = 0; r < RPW; ++r) acc += v[r].x + v[r].y + v[r].z + v[r].w;
        }
    }
    if (acc == 12345.f) out[warp] = acc;
}

template <int RPW>
void run(const float4* base, uint64_t bytes, uint32_t row_bytes, int blocks, int threads, float* out) {
    const uint32_t row_f4 = row_bytes / 16;
    const uint64_t nrows = bytes / row_bytes;
    const uint32_t iters = 64;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    gather<RPW><<<blocks, threads>>>(base, nrows, row_f4, iters, out);
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) gather<RPW><<<blocks, threads>>>(base, nrows, row_f4, iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double total = 5.0 * blocks * (threads / 32) * iters * RPW * (double)row_bytes;
    printf("row %5u B  rows/warp in flight %d  warps/SM %3d : %7.1f GB/s\n", row_bytes, RPW,
           blocks / 148 * threads / 32, total / (ms / 1e3) / 1e9);
}

int main() {
    const uint64_t bytes = 3ull << 30;
    float4* base;
    float* out;
    cudaMalloc(&base, bytes);
    cudaMalloc(&out, 1 << 24);
    cudaMemset(base, 0, bytes);
    for (uint32_t rb : {512u, 1024u, 2048u, 3072u, 4096u}) {
        run<1>(base, bytes, rb, 148 * 4, 128, out);
        run<2>(base, bytes, rb, 148 * 4, 128, out);
        run<4>(base, bytes, rb, 148 * 4, 128, out);
        run<2>(base, bytes, rb, 148 * 8, 256, out);
        run<4>(base, bytes, rb, 148 * 8, 256, out);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
