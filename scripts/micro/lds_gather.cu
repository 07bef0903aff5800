// Microbenchmark (not product code): random shared-memory gathers (the sweep's panel lookups) with
// a concurrent HBM stream, vs the size of the shared-memory allocation and the index range.
// Question: why are gathers from a 225 KB panel slower than from a 75 KB one?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(1024, 1) kern(const float4* __restrict__ R, const uint2* __restrict__ I,
                                                long long n4, int range, float* out) {
    extern __shared__ float sm[];
    const int smem_floats = range;
    for (int i = threadIdx.x; i < smem_floats; i += blockDim.x) sm[i] = 1.0f + i * 1e-6f;
    __syncthreads();
    float acc = 0.f;
    long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i + stride < n4; i += 2 * stride) {
        float4 r0 = __ldcs(R + i), r1 = __ldcs(R + i + stride);
        uint2 x0 = __ldcs(I + i), x1 = __ldcs(I + i + stride);
        unsigned k[8] = {x0.x & 0xffff, x0.x >> 16, x0.y & 0xffff, x0.y >> 16, x1.x & 0xffff, x1.x >> 16, x1.y & 0xffff, x1.y >> 16};
        float rv[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
        for (int c = 0; c < 8; ++c) acc = fmaf(rv[c], sm[k[c] % range], acc);
    }
    if (acc == 123.f) out[0] = acc;
}
int main() {
    long long n4 = 64LL << 20;  // 1 GB of R + 0.5 GB of idx
    float4* R; uint2* I; cudaMalloc(&R, n4 * 16); cudaMalloc(&I, n4 * 8);
    cudaMemset(R, 0, n4 * 16);
    // random 16-bit indices
    unsigned* h = new unsigned[n4 * 2];
    unsigned s = 12345;
    for (long long i = 0; i < n4 * 2; ++i) { s = s * 1664525u + 1013904223u; h[i] = s; }
    cudaMemcpy(I, h, n4 * 8, cudaMemcpyHostToDevice);
    float* out; cudaMalloc(&out, 4);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    for (int alloc_kb : {72, 112, 150, 190, 225}) for (int range : {16384, 18000, 28000, 37000, 47000, 56000}) {
        if (range * 4 > alloc_kb * 1024) continue;
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        kern<<<148, 1024, alloc_kb * 1024>>>(R, I, n4, range, out);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) kern<<<148, 1024, alloc_kb * 1024>>>(R, I, n4, range, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("smem alloc %3d KB  index range %6d floats : %6.1f us/pass  %7.1f GB/s  %s\n", alloc_kb, range, ms * 200,
               5.0 * n4 * 24 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
