// Microbenchmark (not product code): HBM read bandwidth of a persistent streaming kernel vs
// threads per CTA / CTAs per SM / independent 16-byte loads in flight per thread.
#include <cstdio>
#include <cuda_runtime.h>
template <int U>
__global__ void stream_read(const float4* __restrict__ p, long long n4, float* out) {
    float acc = 0.f;
    long long stride = (long long)gridDim.x * blockDim.x;
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n4; i += U * stride) {
        float4 v[U];
#pragma unroll
        for (int q = 0; q < U; ++q) v[q] = __ldcs(p + i + q * stride);
#pragma unroll
        for (int q = 0; q < U; ++q) acc += v[q].x + v[q].y + v[q].z + v[q].w;
    }
    if (acc == 123.f) out[0] = acc;
}
template <int U>
void run(const float4* p, long long n4, float* out, int threads, int ctas) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    stream_read<U><<<ctas, threads>>>(p, n4, out);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) stream_read<U><<<ctas, threads>>>(p, n4, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double gbs = 5.0 * n4 * 16 / (ms * 1e-3) / 1e9;
    printf("threads %4d ctas/SM %d U %2d inflight/SM %6.1f KB : %7.1f GB/s\n", threads, ctas / 148, U,
           threads * (ctas / 148) * U * 16 / 1024.0, gbs);
}
int main() {
    long long bytes = 2LL << 30;
    float4* p; cudaMalloc(&p, bytes); cudaMemset(p, 0, bytes);
    float* out; cudaMalloc(&out, 4);
    long long n4 = bytes / 16;
    for (int cps : {1, 2, 4}) for (int th : {256, 512, 1024}) {
        if (th * cps > 2048) continue;
        run<1>(p, n4, out, th, 148 * cps); run<2>(p, n4, out, th, 148 * cps); run<4>(p, n4, out, th, 148 * cps);
        run<8>(p, n4, out, th, 148 * cps); run<16>(p, n4, out, th, 148 * cps);
    }
    return 0;
}
