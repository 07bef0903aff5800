// L2 persistence for the CCD++ sweep pattern: two 600 MB streams read alternately (the CSR residual of the
// u-sweeps and the CSC residual of the v-sweeps).  Without persistence every read comes from HBM (the
// other stream evicts L2); with an access-policy window per stream part of each stays in L2.  Prints the
// limits and the per-read time / effective bandwidth for several windows.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o l2_persist l2_persist.cu && ./l2_persist
#include <cuda_runtime.h>

#include <cstdio>

__global__ void read_sum(const float4* __restrict__ p, size_t n4, float* out) {
    float s = 0.f;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        const float4 v = p[i];
        s += v.x + v.y + v.z + v.w;
    }
    if (s == 12345.f) out[0] = s;
}

int main() {
    int maxPersist = 0, maxWin = 0, l2 = 0, sms = 0;
    cudaDeviceGetAttribute(&maxPersist, cudaDevAttrMaxPersistingL2CacheSize, 0);
    cudaDeviceGetAttribute(&maxWin, cudaDevAttrMaxAccessPolicyWindowSize, 0);
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    std::printf("L2 %d MB, max persisting %d MB, max window %d MB\n", l2 >> 20, maxPersist >> 20, maxWin >> 20);
    const size_t bytes = 600ull << 20;
    char *A, *B;
    float* out;
    cudaMalloc(&A, bytes);
    cudaMalloc(&B, bytes);
    cudaMalloc(&out, 4);
    cudaMemset(A, 0, bytes);
    cudaMemset(B, 0, bytes);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, size_t win, float ratio, size_t carve) {
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve);
        cudaCtxResetPersistingL2Cache();
        float tot = 0.f;
        const int reps = 20;
        for (int r = 0; r < reps + 2; ++r) {
            for (int w = 0; w < 2; ++w) {
                char* p = w ? B : A;
                cudaStreamAttrValue v{};
                if (win > 0) {
                    v.accessPolicyWindow.base_ptr = p;
                    v.accessPolicyWindow.num_bytes = win;
                    v.accessPolicyWindow.hitRatio = ratio;
                    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
                    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
                }
                cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v);
                cudaEventRecord(e0, s);
                read_sum<<<sms * 2, 1024, 0, s>>>(reinterpret_cast<const float4*>(p), bytes / 16, out);
                cudaEventRecord(e1, s);
                cudaEventSynchronize(e1);
                float ms = 0.f;
                cudaEventElapsedTime(&ms, e0, e1);
                if (r >= 2) tot += ms;
            }
        }
        const float ms = tot / (2 * 20);
        std::printf("%-40s %7.1f us per 600 MB read  %7.0f GB/s effective  %s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9,
                    cudaGetErrorString(cudaGetLastError()));
    };
    run("no window", 0, 0.f, 0);
    for (size_t w : {32ull << 20, 48ull << 20, 64ull << 20, 96ull << 20})
        for (float ratio : {1.0f, 0.6f}) {
            char name[96];
            std::snprintf(name, sizeof name, "window %zu MB each, hitRatio %.1f", w >> 20, ratio);
            size_t win = w < (size_t)maxWin ? w : (size_t)maxWin;
            run(name, win, ratio, (size_t)maxPersist);
        }
    return 0;
}
