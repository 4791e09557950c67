#include <cstdio>
typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__global__ void k1(float* out, int iters) {
    float a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
    const float b = 1.0001f, c = 0.5f;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], b, c);
    float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k2(float* out, int iters) {
    u64 a[8]; for (int i = 0; i < 8; ++i) { float2 f = make_float2(threadIdx.x + i, i); a[i] = *reinterpret_cast<u64*>(&f); }
    float2 bf = make_float2(1.0001f, 1.0001f), cf = make_float2(0.5f, 0.5f);
    u64 b = *reinterpret_cast<u64*>(&bf), c = *reinterpret_cast<u64*>(&cf);
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma2(a[i], b, c);
    float s = 0; for (int i = 0; i < 8; ++i) { float2 f = *reinterpret_cast<float2*>(&a[i]); s += f.x + f.y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    float* d; cudaMalloc(&d, 148 * 8 * 1024 * 4 * 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int iters = 4096;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0); k1<<<148 * 8, 1024>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 8 * iters * 148.0 * 8 * 1024;
        printf("FFMA : %.3f ms  %.1f TFLOP/s\n", ms, flops / ms / 1e9);
        cudaEventRecord(e0); k2<<<148 * 8, 1024>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("FFMA2: %.3f ms  %.1f TFLOP/s\n", ms, 2 * flops / ms / 1e9);
    }
}
