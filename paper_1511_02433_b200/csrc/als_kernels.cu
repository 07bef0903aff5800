// als_kernels.cu -- ALS row solves for sm_100a (als.hpp:47-68, dense.hpp:35-124).
//
// One warp per work unit (a chunk of <= chunk entries of one output row / column).  The warp
// stages up to 32 gathered opposing factor rows in shared memory, then every lane accumulates a
// BR x BC register block of the k x k Gram matrix G = sum h_j h_j^T (lanes form an 8 x 4 grid over
// the matrix) plus its share of the right-hand side b = sum A_ij h_j, in FP32.  Units that are the
// only chunk of their output go straight on to G + lambda I, an in-warp Cholesky factorisation
// (left-looking by column, the order of dense.hpp:74-96) and forward/back substitution; chunks of
// long columns write (G, b) partials that a second kernel sums in chunk order before solving.
// A non-positive pivot sets the status word to PMF_NOT_POSITIVE_DEFINITE (dense.hpp:82-84).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "device.hpp"

namespace pmfgpu {

namespace {

constexpr int kAlsThreads = 256;
constexpr int kAlsWarps = kAlsThreads / 32;

template <int KMAX>
struct Tile {
    static constexpr int BR = (KMAX + 7) / 8;   // rows per lane block
    static constexpr int BC = (KMAX + 3) / 4;   // cols per lane block
    static constexpr int KS0 = KMAX > 8 * BR ? KMAX : 8 * BR;
    static constexpr int KS = KS0 > 4 * BC ? KS0 : 4 * BC;   // staged row stride
    static constexpr int GS = KMAX + 1;                      // gram row stride in smem
    static constexpr int STAGE = 32 * KS;
    static constexpr int GRAM = KMAX * GS + 2 * KMAX;
    static constexpr int WARP_FLOATS = (STAGE > GRAM ? STAGE : GRAM) + 64;
};

// In-warp Cholesky of G (k x k in smem, stride GS, full symmetric) and solve of G x = b.
// b lives in registers: lane owns t = lane and lane + 32.  Returns false on a bad pivot.
template <int KMAX>
__device__ bool warp_cholesky_solve(float* G, int k, float& b0, float& b1) {
    constexpr int GS = Tile<KMAX>::GS;
    const int lane = threadIdx.x & 31;
    bool ok = true;
    for (int j = 0; j < k; ++j) {
        // d = a_jj - sum_{t<j} l_jt^2
        float part = 0.f;
        for (int t = lane; t < j; t += 32) {
            const float l = G[j * GS + t];
            part = fmaf(l, l, part);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
        const float d = G[j * GS + j] - part;
        if (!(d > 0.f)) {
            ok = false;
            break;
        }
        const float ljj = sqrtf(d);
        __syncwarp();
        for (int i = j + 1 + lane; i < k; i += 32) {
            float s = G[i * GS + j];
            for (int t = 0; t < j; ++t) s = fmaf(-G[i * GS + t], G[j * GS + t], s);
            G[i * GS + j] = s / ljj;
        }
        if (lane == 0) G[j * GS + j] = ljj;
        __syncwarp();
    }
    if (!ok) return false;
    // forward: L y = b (column-oriented)
    for (int i = 0; i < k; ++i) {
        const float bi = __shfl_sync(0xffffffffu, i < 32 ? b0 : b1, i & 31);
        const float yi = bi / G[i * GS + i];
        if (lane == (i & 31)) {
            if (i < 32) b0 = yi;
            else b1 = yi;
        }
        if (lane > i && lane < k) b0 = fmaf(-G[lane * GS + i], yi, b0);
        if (lane + 32 > i && lane + 32 < k) b1 = fmaf(-G[(lane + 32) * GS + i], yi, b1);
    }
    // backward: L^T x = y
    for (int i = k - 1; i >= 0; --i) {
        const float yi = __shfl_sync(0xffffffffu, i < 32 ? b0 : b1, i & 31);
        const float xi = yi / G[i * GS + i];
        if (lane == (i & 31)) {
            if (i < 32) b0 = xi;
            else b1 = xi;
        }
        if (lane < i) b0 = fmaf(-G[i * GS + lane], xi, b0);
        if (lane + 32 < i) b1 = fmaf(-G[i * GS + lane + 32], xi, b1);
    }
    return true;
}

template <int KMAX>
__global__ void __launch_bounds__(kAlsThreads)
als_gram_kernel(const Unit* __restrict__ units, int32_t n_units, const int32_t* __restrict__ idx,
                const float* __restrict__ val, const float* __restrict__ opp, float* __restrict__ out,
                int32_t out_off, int k, float lambda, int weighted, float* __restrict__ partial,
                int* __restrict__ counter, int* __restrict__ status) {
    using T = Tile<KMAX>;
    constexpr int BR = T::BR, BC = T::BC, KS = T::KS, GS = T::GS;
    extern __shared__ float smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    float* X = smem + warp * T::WARP_FLOATS;
    float* G = X;  // reused after accumulation
    int* sidx = reinterpret_cast<int*>(X + T::WARP_FLOATS - 64);
    float* sval = X + T::WARP_FLOATS - 32;
    const int rb = lane >> 2, cb = lane & 3;
    const int r0 = rb * BR, c0 = cb * BC;

    for (;;) {
        int u = 0;
        if (lane == 0) u = atomicAdd(counter, 1);
        u = __shfl_sync(0xffffffffu, u, 0);
        if (u >= n_units) break;
        const Unit U = units[u];
        float acc[BR][BC];
#pragma unroll
        for (int i = 0; i < BR; ++i)
#pragma unroll
            for (int j = 0; j < BC; ++j) acc[i][j] = 0.f;
        float rhs0 = 0.f, rhs1 = 0.f;
        for (int base = 0; base < U.len; base += 32) {
            const int cnt = min(32, U.len - base);
            __syncwarp();
            if (lane < cnt) {
                sidx[lane] = idx[U.e0 + base + lane];
                sval[lane] = val[U.e0 + base + lane];
            }
            __syncwarp();
            for (int x = lane; x < cnt * KS; x += 32) {
                const int s = x / KS, c = x - s * KS;
                X[x] = c < k ? __ldg(opp + static_cast<int64_t>(sidx[s]) * k + c) : 0.f;
            }
            __syncwarp();
            for (int s = 0; s < cnt; ++s) {
                const float* xs = X + s * KS;
                float a[BR], b[BC];
#pragma unroll
                for (int i = 0; i < BR; ++i) a[i] = xs[r0 + i];
#pragma unroll
                for (int j = 0; j < BC; ++j) b[j] = xs[c0 + j];
#pragma unroll
                for (int i = 0; i < BR; ++i)
#pragma unroll
                    for (int j = 0; j < BC; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
                const float av = sval[s];
                rhs0 = fmaf(av, xs[lane], rhs0);
                if (KMAX > 32) rhs1 = fmaf(av, xs[lane + 32], rhs1);
            }
        }
        __syncwarp();
        if (U.slot >= 0) {
            float* P = partial + static_cast<int64_t>(U.slot) * (k * k + k + 1);
#pragma unroll
            for (int i = 0; i < BR; ++i)
#pragma unroll
                for (int j = 0; j < BC; ++j)
                    if (r0 + i < k && c0 + j < k) P[(r0 + i) * k + c0 + j] = acc[i][j];
            if (lane < k) P[k * k + lane] = rhs0;
            if (lane + 32 < k) P[k * k + lane + 32] = rhs1;
            if (lane == 0) P[k * k + k] = static_cast<float>(U.len);
            continue;
        }
        // single-chunk output: G + lambda I, Cholesky, solve (als.hpp:64-67)
        const float ridge = weighted ? lambda * static_cast<float>(U.len) : lambda;
#pragma unroll
        for (int i = 0; i < BR; ++i)
#pragma unroll
            for (int j = 0; j < BC; ++j)
                if (r0 + i < k && c0 + j < k)
                    G[(r0 + i) * GS + c0 + j] = acc[i][j] + ((r0 + i == c0 + j) ? ridge : 0.f);
        __syncwarp();
        const bool ok = warp_cholesky_solve<KMAX>(G, k, rhs0, rhs1);
        if (!ok) {
            if (lane == 0) atomicExch(status, 4);
            rhs0 = rhs1 = 0.f;
        }
        float* dst = out + static_cast<int64_t>(out_off + U.o) * k;
        if (lane < k) dst[lane] = rhs0;
        if (lane + 32 < k) dst[lane + 32] = rhs1;
        __syncwarp();
    }
}

template <int KMAX>
__global__ void __launch_bounds__(kAlsThreads)
als_reduce_solve_kernel(const int32_t* __restrict__ mo_out, const int32_t* __restrict__ mo_start,
                        int32_t n_mo, const float* __restrict__ partial, float* __restrict__ out,
                        int32_t out_off, int k, float lambda, int weighted, int* __restrict__ status) {
    using T = Tile<KMAX>;
    constexpr int GS = T::GS;
    extern __shared__ float smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    float* G = smem + warp * T::WARP_FLOATS;
    const int64_t wid = static_cast<int64_t>(blockIdx.x) * kAlsWarps + warp;
    const int64_t nw = static_cast<int64_t>(gridDim.x) * kAlsWarps;
    const int stride = k * k + k + 1;
    for (int64_t q = wid; q < n_mo; q += nw) {
        const int s0 = mo_start[q], s1 = mo_start[q + 1];
        float cntf = 0.f;
        for (int s = s0; s < s1; ++s) cntf += partial[static_cast<int64_t>(s) * stride + k * k + k];
        for (int e = lane; e < k * k; e += 32) {
            float a = 0.f;
            for (int s = s0; s < s1; ++s) a += partial[static_cast<int64_t>(s) * stride + e];
            const int r = e / k, c = e - r * k;
            G[r * GS + c] = a;
        }
        float b0 = 0.f, b1 = 0.f;
        for (int s = s0; s < s1; ++s) {
            const float* P = partial + static_cast<int64_t>(s) * stride + k * k;
            if (lane < k) b0 += P[lane];
            if (lane + 32 < k) b1 += P[lane + 32];
        }
        __syncwarp();
        const float ridge = weighted ? lambda * cntf : lambda;
        for (int d = lane; d < k; d += 32) G[d * GS + d] += ridge;
        __syncwarp();
        const bool ok = warp_cholesky_solve<KMAX>(G, k, b0, b1);
        if (!ok) {
            if (lane == 0) atomicExch(status, 4);
            b0 = b1 = 0.f;
        }
        float* dst = out + static_cast<int64_t>(out_off + mo_out[q]) * k;
        if (lane < k) dst[lane] = b0;
        if (lane + 32 < k) dst[lane + 32] = b1;
        __syncwarp();
    }
}

__global__ void zero_rows_kernel(const int32_t* __restrict__ rows, int32_t n, float* __restrict__ out,
                                 int32_t out_off, int k) {
    for (int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; x < static_cast<int64_t>(n) * k;
         x += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = x / k;
        out[static_cast<int64_t>(out_off + rows[r]) * k + (x - r * k)] = 0.f;
    }
}

// Batched Cholesky (KAT entry point): one warp per system, a overwritten with L.
template <int KMAX>
__global__ void __launch_bounds__(kAlsThreads)
chol_batched_kernel(float* __restrict__ a, float* __restrict__ x, int batch, int k, int* __restrict__ status) {
    using T = Tile<KMAX>;
    constexpr int GS = T::GS;
    extern __shared__ float smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    float* G = smem + warp * T::WARP_FLOATS;
    const int64_t wid = static_cast<int64_t>(blockIdx.x) * kAlsWarps + warp;
    const int64_t nw = static_cast<int64_t>(gridDim.x) * kAlsWarps;
    for (int64_t q = wid; q < batch; q += nw) {
        float* A = a + q * k * k;
        for (int e = lane; e < k * k; e += 32) G[(e / k) * GS + e % k] = A[e];
        float b0 = lane < k ? x[q * k + lane] : 0.f;
        float b1 = lane + 32 < k ? x[q * k + lane + 32] : 0.f;
        __syncwarp();
        const bool ok = warp_cholesky_solve<KMAX>(G, k, b0, b1);
        if (!ok && lane == 0) atomicExch(status, 4);
        __syncwarp();
        for (int e = lane; e < k * k; e += 32) {
            const int r = e / k, c = e % k;
            A[e] = c <= r ? G[r * GS + c] : 0.f;
        }
        if (lane < k) x[q * k + lane] = b0;
        if (lane + 32 < k) x[q * k + lane + 32] = b1;
        __syncwarp();
    }
}

template <int KMAX>
size_t smem_for() {
    return static_cast<size_t>(kAlsWarps) * Tile<KMAX>::WARP_FLOATS * sizeof(float);
}

template <int KMAX>
int launch_k(const DevAls& L, const float* opp, float* out, int32_t out_off, int k, float lambda, bool weighted,
             int* d_counter, int* d_status, int sm_count, cudaStream_t s) {
    int launched = 0;
    const size_t sm = smem_for<KMAX>();
    if (L.n_units > 0) {
        cudaMemsetAsync(d_counter, 0, sizeof(int), s);
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, als_gram_kernel<KMAX>, kAlsThreads, sm);
        const int blocks = std::max(1, std::min<int>(per_sm * sm_count, (L.n_units + kAlsWarps - 1) / kAlsWarps));
        als_gram_kernel<KMAX><<<blocks, kAlsThreads, sm, s>>>(L.units, L.n_units, L.idx, L.val, opp, out, out_off,
                                                               k, lambda, weighted ? 1 : 0, L.partial, d_counter,
                                                               d_status);
        ++launched;
    }
    if (L.n_mo > 0) {
        const int blocks = std::max(1, std::min(4 * sm_count, (L.n_mo + kAlsWarps - 1) / kAlsWarps));
        als_reduce_solve_kernel<KMAX><<<blocks, kAlsThreads, sm, s>>>(L.mo_out, L.mo_start, L.n_mo, L.partial, out,
                                                                       out_off, k, lambda, weighted ? 1 : 0, d_status);
        ++launched;
    }
    if (L.n_empty > 0) {
        zero_rows_kernel<<<std::min(1024, (L.n_empty * k + 255) / 256), 256, 0, s>>>(L.empty_out, L.n_empty, out,
                                                                                      out_off, k);
        ++launched;
    }
    return launched;
}

template <int KMAX>
void set_attr_k() {
    cudaFuncSetAttribute(als_gram_kernel<KMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem_for<KMAX>()));
    cudaFuncSetAttribute(als_reduce_solve_kernel<KMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem_for<KMAX>()));
    cudaFuncSetAttribute(chol_batched_kernel<KMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem_for<KMAX>()));
}

}  // namespace

void als_set_attributes() {
    set_attr_k<8>();
    set_attr_k<16>();
    set_attr_k<32>();
    set_attr_k<40>();
    set_attr_k<64>();
}

int launch_als_half(const DevAls& L, const float* opp, float* out, int32_t out_off, int k, float lambda,
                    bool weighted, int* d_counter, int* d_status, int sm_count, cudaStream_t stream) {
    if (k <= 8) return launch_k<8>(L, opp, out, out_off, k, lambda, weighted, d_counter, d_status, sm_count, stream);
    if (k <= 16) return launch_k<16>(L, opp, out, out_off, k, lambda, weighted, d_counter, d_status, sm_count, stream);
    if (k <= 32) return launch_k<32>(L, opp, out, out_off, k, lambda, weighted, d_counter, d_status, sm_count, stream);
    if (k <= 40) return launch_k<40>(L, opp, out, out_off, k, lambda, weighted, d_counter, d_status, sm_count, stream);
    return launch_k<64>(L, opp, out, out_off, k, lambda, weighted, d_counter, d_status, sm_count, stream);
}

void launch_cholesky_batched(float* a, float* x, int batch, int k, int* d_status, cudaStream_t s) {
    const int blocks = std::max(1, std::min(4096, (batch + kAlsWarps - 1) / kAlsWarps));
    if (k <= 8) chol_batched_kernel<8><<<blocks, kAlsThreads, smem_for<8>(), s>>>(a, x, batch, k, d_status);
    else if (k <= 16) chol_batched_kernel<16><<<blocks, kAlsThreads, smem_for<16>(), s>>>(a, x, batch, k, d_status);
    else if (k <= 32) chol_batched_kernel<32><<<blocks, kAlsThreads, smem_for<32>(), s>>>(a, x, batch, k, d_status);
    else if (k <= 40) chol_batched_kernel<40><<<blocks, kAlsThreads, smem_for<40>(), s>>>(a, x, batch, k, d_status);
    else chol_batched_kernel<64><<<blocks, kAlsThreads, smem_for<64>(), s>>>(a, x, batch, k, d_status);
}

}  // namespace pmfgpu
