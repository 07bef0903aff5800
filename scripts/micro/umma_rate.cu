// Issue-rate micro-benchmark for single-CTA tcgen05.mma (M = 128) from a K-major SWIZZLE_128B shared-memory
// tile: cycles per instruction for kind::tf32 and kind::f16 at several N, with one commit per `per_commit`
// instructions and a wait on the last commit.  One CTA per SM on all SMs (the ALS gram kernel's shape).
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o umma_rate umma_rate.cu && ./umma_rate
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    return static_cast<uint64_t>((saddr >> 4) & 0x3fff) | (static_cast<uint64_t>(1) << 16) |
           (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(2) << 61);
}

template <int KIND>  // 0 = tf32, 1 = f16 (bf16 operands)
__global__ void __launch_bounds__(128, 1) umma_rate(int n, int iters, int per_commit, long long* out, int m, int nacc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t bar, bar2;
    for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.001f * (i % 7);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar2)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = s_tmem;
    const uint32_t idesc = (1u << 4) | (KIND == 0 ? (2u << 7) | (2u << 10) : (1u << 7) | (1u << 10)) |
                           (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
    long long t = 0;
    if (threadIdx.x == 0) {
        const uint32_t base = sa(smem);
        uint32_t phase = 0;
        const long long t0 = clock64();
        const uint64_t desc0 = sw128_desc(base);
        for (int i = 0; i < iters; i += 8) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint64_t desc = desc0 + ((j & 3) * 32 >> 4);  // start address += 32 B per K step
                const uint32_t d = tmem + (j % 8) * (512 / 8) * (nacc > 1 ? 1 : 0);
                if (KIND == 0)
                    asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n" ::"r"(d), "l"(desc), "l"(desc),
                                 "r"(idesc));
                else
                    asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n" ::"r"(d), "l"(desc), "l"(desc),
                                 "r"(idesc));
                if (per_commit == 4 && (j & 3) == 3)
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar2))
                                 : "memory");
                if (per_commit == 5 && (j & 3) == 3)
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)) : "memory");
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                         sa(&bar)), "r"(phase) : "memory");
        t = clock64() - t0;
        if (blockIdx.x == 0) out[0] = t;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int smem = 32768 + 1024;
    cudaFuncSetAttribute(umma_rate<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(umma_rate<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 4096;
    for (int nacc : {1})
    for (int m : {128})
    for (int kind = 0; kind < 1; ++kind)
        for (int pc : {4096, 4, 5})
            for (int n : {48}) {
                if (kind == 0) umma_rate<0><<<sms, 128, smem>>>(n, iters, pc, d, m, nacc);
                else umma_rate<1><<<sms, 128, smem>>>(n, iters, pc, d, m, nacc);
                cudaError_t e = cudaDeviceSynchronize();
                long long t = 0;
                cudaMemcpy(&t, d, 8, cudaMemcpyDeviceToHost);
                const double macs = double(m) * n * (kind == 0 ? 8 : 16);
                std::printf("pc %d acc %d M=%3d %s N=%3d: %7.1f cycles/mma  %6.0f MAC/cycle/SM %s\n", pc, nacc, m, kind == 0 ? "tf32" : "f16 ", n,
                            double(t) / iters, macs * iters / double(t), e == cudaSuccess ? "" : cudaGetErrorString(e));
            }
    return 0;
}
