// cudaMalloc cost for the context's large buffers (3 x 411 MB per layout side) vs one allocation and
// vs a stream-ordered pool.  nvcc -O3 -o malloc_cost malloc_cost.cu
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
    cudaFree(nullptr);
    const size_t sz = 411u << 20;
    for (int rep = 0; rep < 3; ++rep) {
        void* p[6];
        double t0 = now();
        for (int i = 0; i < 6; ++i) cudaMalloc(&p[i], sz);
        double t1 = now();
        for (int i = 0; i < 6; ++i) cudaFree(p[i]);
        double t2 = now();
        void* q;
        cudaMalloc(&q, 6 * sz);
        double t3 = now();
        cudaFree(q);
        double t4 = now();
        std::printf("6 x 411 MB cudaMalloc %.1f ms, free %.1f ms; one 2.4 GB cudaMalloc %.1f ms, free %.1f ms\n",
                    1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2), 1e3 * (t4 - t3));
    }
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaMemPool_t pool;
    cudaDeviceGetDefaultMemPool(&pool, 0);
    unsigned long long thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    for (int rep = 0; rep < 3; ++rep) {
        void* p[6];
        double t0 = now();
        for (int i = 0; i < 6; ++i) cudaMallocAsync(&p[i], sz, s);
        cudaStreamSynchronize(s);
        double t1 = now();
        for (int i = 0; i < 6; ++i) cudaFreeAsync(p[i], s);
        cudaStreamSynchronize(s);
        double t2 = now();
        std::printf("pool: 6 x 411 MB %.1f ms, free %.1f ms\n", 1e3 * (t1 - t0), 1e3 * (t2 - t1));
    }
    return 0;
}
