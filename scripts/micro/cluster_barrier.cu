// Cost of barrier.cluster (arrive.release + wait.acquire) for one cluster of C CTAs x 1024 threads, with
// and without a DSMEM store per thread before each barrier (the small-matrix CCD++ kernel's phase
// structure).  nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o cb cluster_barrier.cu && ./cb
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__global__ void bar_kernel(int iters, int dsmem, int cl, float* out) {
    __shared__ float buf[1024];
    buf[threadIdx.x] = 0.f;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    for (int i = 0; i < iters; ++i) {
        if (dsmem) {
            uint32_t a;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                         : "=r"(a)
                         : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(&buf[threadIdx.x]))), "r"((rank + 1) % cl));
            asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(a), "f"(static_cast<float>(i)) : "memory");
        }
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    if (threadIdx.x == 0 && buf[5] == -1.f) out[0] = 1.f;
}

int main() {
    float* out;
    cudaMalloc(&out, 4);
    cudaFuncSetAttribute(bar_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int cl : {2, 8, 16})
        for (int ds : {0, 1}) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(cl);
            cfg.blockDim = dim3(1024);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cl;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            const int iters = 10000;
            cudaLaunchKernelEx(&cfg, bar_kernel, iters, ds, cl, out);
            cudaEventRecord(e0);
            cudaLaunchKernelEx(&cfg, bar_kernel, iters, ds, cl, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            std::printf("cluster %2d dsmem %d: %.3f us per barrier %s\n", cl, ds, ms * 1e3 / iters,
                        cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
