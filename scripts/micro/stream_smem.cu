// Microbenchmark (not product code): HBM streaming-read bandwidth of a persistent 1024-thread
// kernel vs the dynamic shared memory the CTA reserves (which shrinks L1) and the load flavour.
// Question: do in-flight global loads need L1 capacity (so a 225 KB smem panel starves them)?
#include <cstdio>
#include <cuda_runtime.h>
template <int F>
__device__ __forceinline__ float4 ld(const float4* p) {
    float4 v;
    if (F == 0) v = __ldcs(p);
    else if (F == 1) v = __ldcg(p);
    else if (F == 2)
        asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    else v = *p;
    return v;
}
template <int U, int F>
__global__ void __launch_bounds__(1024, 1) stream_read(const float4* __restrict__ p, long long n4, float* out) {
    extern __shared__ float sm[];
    float acc = 0.f;
    long long stride = (long long)gridDim.x * blockDim.x;
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n4; i += U * stride) {
        float4 v[U];
#pragma unroll
        for (int q = 0; q < U; ++q) v[q] = ld<F>(p + i + q * stride);
#pragma unroll
        for (int q = 0; q < U; ++q) acc += v[q].x + v[q].y + v[q].z + v[q].w;
    }
    if (acc == 123.f) out[0] = acc + sm[threadIdx.x];
}
template <int U, int F>
void run(const float4* p, long long n4, float* out, int smem_kb) {
    auto k = stream_read<U, F>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    const int smem = smem_kb * 1024;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    k<<<148, 1024, smem>>>(p, n4, out);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k<<<148, 1024, smem>>>(p, n4, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const char* fl[] = {"ld.cs", "ld.cg", "ld.nc.L1::no_allocate", "ld"};
    printf("smem %3d KB  U %d  %-22s : %7.1f GB/s  %s\n", smem_kb, U, fl[F], 5.0 * n4 * 16 / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
}
int main() {
    long long bytes = 2LL << 30;
    float4* p; cudaMalloc(&p, bytes); cudaMemset(p, 0, bytes);
    float* out; cudaMalloc(&out, 4);
    long long n4 = bytes / 16;
    for (int kb : {0, 40, 72, 100, 132, 164, 196, 225}) {
        run<2, 0>(p, n4, out, kb); run<4, 0>(p, n4, out, kb); run<8, 0>(p, n4, out, kb);
        run<4, 1>(p, n4, out, kb); run<4, 2>(p, n4, out, kb); run<4, 3>(p, n4, out, kb);
        run<8, 2>(p, n4, out, kb);
    }
    return 0;
}
