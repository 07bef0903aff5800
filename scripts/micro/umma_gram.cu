// Groundwork for a tcgen05 ALS gram ("Next"): G = X^T X for one 32-entry chunk of
// gathered rows X (entries x 64 features, feature 40 = the rating column) with tcgen05.mma.kind::tf32
// (M = 64, N = 48, K = 8 per instruction), accumulator in TMEM, read back with tcgen05.ld.32x32b.
// Verified on the B200 with both operands K-major, no swizzle (core matrices of 8 features x 16 B;
// UG_FLAG=4): max relative error 5.6e-2 on near-zero entries, absolute 4e-3 (TF32 operands), and the
// M = 64 accumulator layout row m -> TMEM lane (m % 16) + 32 (m / 16).  The MN-major SWIZZLE_128B
// variant (UG_FLAG=0, the layout TMA gather4 would write directly) reads zero operands, with LBO / SBO
// either way round (UG_FLAG=8), and so does MN-major without swizzle (UG_FLAG=16): with these
// instruction-descriptor bits (a/b major = 1, bits 15/16) MN-major TF32 operands come back as zeros,
// so the product path will transpose the gathered rows into K-major core matrices.  UG_FLAG bits:
// 1 = seed D with 7 and accumulate (shows what the MMA added), 2 = print the smem / TMEM bases,
// 4 = K-major layout, 8 = swapped LBO / SBO, 16 = MN-major no swizzle.  UG_DUMP=1 prints rows.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o umma_gram umma_gram.cu && UG_FLAG=4 ./umma_gram
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int K = 32;  // entries (UMMA K = 8 per instruction for tf32 -> 4 MMAs)
constexpr int F = 64;  // features (M)
constexpr int N = 48;  // B columns (features 0..47)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// byte offset of element (entry e, feature f) in the MN-major SW128 layout:
// MN atoms of 32 features (128 B) x 8 entries, atoms stacked along K every SBO = 1 KB, the two MN
// atoms LBO = 4 KB apart; 16-byte chunk index XOR (entry % 8) inside an atom.
__host__ __device__ inline uint32_t sw128_offset(int e, int f) {
    const int atom_mn = f / 32, atom_k = e / 8, r = e % 8, c = (f % 32) / 4;
    return atom_mn * 4096 + atom_k * 1024 + r * 128 + ((c ^ r) * 16) + (f % 4) * 4;
}

// K-major, no swizzle: core matrices of 8 rows (features) x 16 B (4 entries), LBO = next 4 entries
// (128 B), SBO = next 8 features (K / 4 core matrices = 1 KB)
__host__ __device__ inline uint32_t kmajor_offset(int e, int f) {
    return (f % 8) * 16 + (f / 8) * 1024 + (e % 4) * 4 + (e / 4) * 128;
}

// MN-major, no swizzle: core matrices of 4 features (16 B) x 8 entries (128 B contiguous), the next
// 4 features SBO = 128 B on, the next 8 entries LBO = 2 KB on
__host__ __device__ inline uint32_t mn_inter_offset(int e, int f) {
    return (f % 4) * 4 + (e % 8) * 16 + (f / 4) * 128 + (e / 8) * 2048;
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3fff);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3fff) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3fff) << 32;
    d |= static_cast<uint64_t>(1) << 46;  // version (sm100)
    d |= static_cast<uint64_t>(layout) << 61;  // 2 = SWIZZLE_128B, 0 = none
    return d;
}

__global__ void __launch_bounds__(128, 1) umma_gram(const float* __restrict__ X, float* __restrict__ G,
                                                      uint32_t idesc, int lbo, int sbo, int getenv_flag) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t s_bar;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // stage X (K x F, row-major in global) into the swizzled MN-major layout
    for (int i = tid; i < K * F; i += blockDim.x) {
        const int e = i / F, f = i % F;
        *reinterpret_cast<float*>(smem + ((getenv_flag & 4)    ? kmajor_offset(e, f)
                                          : (getenv_flag & 16) ? mn_inter_offset(e, f)
                                                               : sw128_offset(e, f))) = X[i];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = s_tmem;
    if (getenv_flag & 1) {  // debug: seed the accumulator with 7 and accumulate onto it
        const uint32_t seven = __float_as_uint(7.f);
        const uint32_t ta = tmem + (static_cast<uint32_t>(32 * warp) << 16);
#pragma unroll
        for (int c = 0; c < 3; ++c)
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                    ta + 16 * c),
                "r"(seven));
        asm volatile("tcgen05.wait::st.sync.aligned;");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
    }
    if (tid == 0 && (getenv_flag & 2)) printf("smem base %u (mod 1024 = %u), tmem 0x%08x\n", smem_u32(smem), smem_u32(smem) & 1023u, tmem);
    if (tid == 0) {
        const uint32_t base = smem_u32(smem);
        for (int s = 0; s < K / 8; ++s) {
            const bool km = getenv_flag & 4;
            const bool swap = getenv_flag & 8;  // MN-major: try LBO / SBO the other way round
            const uint64_t ad = km                  ? make_desc(base + s * 256, 128, 1024, 0)
                                : (getenv_flag & 16) ? make_desc(base + s * 2048, 2048, 128, 0)
                                : swap ? make_desc(base + s * sbo, sbo, lbo, 2)
                                       : make_desc(base + s * sbo, lbo, sbo, 2);
            const uint64_t bd = ad;
            const uint32_t acc = (s > 0 || (getenv_flag & 1)) ? 1u : 0u;
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&s_bar)));
    }
    // wait for the MMAs
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(
            smem_u32(&s_bar))
        : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    // M = 64: row m lives in TMEM lane (m % 16) + 32 * (m / 16); warp w reads its 32-lane quadrant
    uint32_t v[48];
    const uint32_t taddr = tmem + (static_cast<uint32_t>(32 * warp) << 16);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[16 * c + 0]), "=r"(v[16 * c + 1]), "=r"(v[16 * c + 2]), "=r"(v[16 * c + 3]),
              "=r"(v[16 * c + 4]), "=r"(v[16 * c + 5]), "=r"(v[16 * c + 6]), "=r"(v[16 * c + 7]),
              "=r"(v[16 * c + 8]), "=r"(v[16 * c + 9]), "=r"(v[16 * c + 10]), "=r"(v[16 * c + 11]),
              "=r"(v[16 * c + 12]), "=r"(v[16 * c + 13]), "=r"(v[16 * c + 14]), "=r"(v[16 * c + 15])
            : "r"(taddr + 16 * c));
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (lane < 16) {
        const int m = 16 * warp + lane;
        for (int n = 0; n < N; ++n) G[m * N + n] = __uint_as_float(v[n]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

int main() {
    std::vector<float> X(K * F, 0.f);
    srand(7);
    for (int e = 0; e < K; ++e) {
        for (int f = 0; f < 40; ++f) X[e * F + f] = (rand() / float(RAND_MAX) - 0.5f) * 0.6f;
        X[e * F + 40] = 1.f + rand() % 5;  // rating column
    }
    std::vector<double> ref(F * N, 0.0);
    for (int m = 0; m < F; ++m)
        for (int n = 0; n < N; ++n)
            for (int e = 0; e < K; ++e) ref[m * N + n] += double(X[e * F + m]) * X[e * F + n];
    float *dX, *dG;
    cudaMalloc(&dX, X.size() * 4);
    cudaMalloc(&dG, F * N * 4);
    cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dG, 0xff, F * N * 4);
    // instruction descriptor: D f32, A/B tf32, both MN-major, N = 48, M = 64
    const int flag0 = getenv("UG_FLAG") ? atoi(getenv("UG_FLAG")) : 0;
    const uint32_t major = (flag0 & 4) ? 0u : 1u;  // K-major test layout / MN-major
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (major << 15) | (major << 16) | ((N >> 3) << 17) |
                           ((F >> 4) << 24);
    const int smem = 8192 + 1024;
    cudaFuncSetAttribute(umma_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int flag = getenv("UG_FLAG") ? atoi(getenv("UG_FLAG")) : 0;
    umma_gram<<<1, 128, smem>>>(dX, dG, idesc, 4096, 1024, flag);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) {
        std::printf("kernel error: %s\n", cudaGetErrorString(err));
        return 1;
    }
    std::vector<float> G(F * N);
    cudaMemcpy(G.data(), dG, G.size() * 4, cudaMemcpyDeviceToHost);
    if (getenv("UG_DUMP")) {
        for (int m = 0; m < F; ++m)
            std::printf("row %2d: G %9.4f %9.4f %9.4f | ref %9.4f %9.4f %9.4f | G[.,40] %9.4f ref %9.4f\n", m,
                        G[m * N], G[m * N + 1], G[m * N + 2], ref[m * N], ref[m * N + 1], ref[m * N + 2],
                        G[m * N + 40], ref[m * N + 40]);
        // where does ref[0][0] appear?
        for (int x = 0; x < F * N; ++x)
            if (std::fabs(G[x] - ref[0]) < 1e-3 * std::fabs(ref[0])) std::printf("ref[0][0] found at G[%d][%d]\n", x / N, x % N);
    }
    double max_rel = 0, max_abs = 0;
    int bad = 0;
    for (int m = 0; m < F; ++m)
        for (int n = 0; n < N; ++n) {
            const double r = ref[m * N + n], g = G[m * N + n];
            const double d = std::fabs(g - r);
            max_abs = std::max(max_abs, d);
            if (std::fabs(r) > 1e-3) max_rel = std::max(max_rel, d / std::fabs(r));
            if (d > 2e-3 * std::max(1.0, std::fabs(r))) {
                if (bad < 8) std::printf("mismatch G[%d][%d] = %g, ref %g\n", m, n, g, r);
                ++bad;
            }
        }
    std::printf("umma tf32 gram 64x48 from MN-major SW128: max abs err %.3g, max rel err %.3g, %d bad -> %s\n",
                max_abs, max_rel, bad, bad ? "FAIL" : "ok");
    return bad ? 1 : 0;
}
