// Probe: does reading only the 32-B sectors a C2 gather needs (x,v = bytes
// 0..44 of each 88-B default record) cut DRAM traffic vs whole records?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_sector probe_sector.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kWordsRec = 11;  // 88 B

__global__ void k_full(const uint64_t* __restrict__ rec, uint64_t n, uint64_t* out) {
    uint64_t acc = 0;
    const uint64_t words = n * kWordsRec;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < words; i += uint64_t(gridDim.x) * blockDim.x)
        acc ^= __ldcs(rec + i);
    if (acc == 0x123456789ull) out[0] = acc;
}

__global__ void k_sectors(const uint64_t* __restrict__ rec, uint64_t n, uint64_t* out) {
    // five 8-B words per record at byte offsets 0,8,16,32,40
    const int off[5] = {0, 1, 2, 4, 5};
    uint64_t acc = 0;
    const uint64_t words = n * 5;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < words; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t r = i / 5;
        acc ^= __ldcs(rec + r * kWordsRec + off[i % 5]);
    }
    if (acc == 0x123456789ull) out[0] = acc;
}

int main() {
    const uint64_t n = 1ull << 24;
    uint64_t *rec, *out;
    cudaMalloc(&rec, n * 88);
    cudaMalloc(&out, 8);
    cudaMemset(rec, 1, n * 88);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int grid = 148 * 8, block = 512;
    for (int which = 0; which < 2; ++which) {
        for (int w = 0; w < 3; ++w) which ? k_sectors<<<grid, block>>>(rec, n, out) : k_full<<<grid, block>>>(rec, n, out);
        cudaEventRecord(a);
        const int it = 20;
        for (int w = 0; w < it; ++w) which ? k_sectors<<<grid, block>>>(rec, n, out) : k_full<<<grid, block>>>(rec, n, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= it;
        printf("%s: %.4f ms  (%.1f GB/s of whole records)\n", which ? "sectors" : "full", ms, n * 88 / ms / 1e6);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
