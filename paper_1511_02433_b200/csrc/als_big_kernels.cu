// als_big_kernels.cu -- ALS row solves for k > 64 (als.hpp:47-68 solve_row, dense.hpp:35-124): one CTA per
// work unit instead of one warp, the k x k system in shared memory (global scratch past ~216).
//
// The reference places no bound on k (als.hpp:26-40).  Here the order of operations follows it:
//   gram    G[a][b] += h_a h_b over the unit's entries in ascending j, a thread per (a <= b) pair, each
//           product rounded before the add (dense.hpp:35-42, the reference's Release build has no FMA);
//           rhs b[t] += A_ij h_t likewise (als.hpp:61-62);
//   finish  G[r][r] += ridge, upper mirrored into lower (dense.hpp:46-53);
//   factor  left-looking column by column (dense.hpp:74-96): for column j every thread i >= j forms
//           s_i = a_ij - sum_{t<j} l_it l_jt in ascending t (s_j = d), then l_jj = sqrt(d), l_ij = s_i / l_jj;
//           a pivot d <= 0 flags not_positive_definite;
//   solves  forward substitution as a column sweep (row i subtracts l_it x_t in ascending t, as
//           dense.hpp:114-117), backward as a column sweep in descending t (the reference's ascending
//           inner order differs in rounding only).
// So a single-unit output reproduces the reference's float gram, factor and forward solve exactly.
// Outputs longer than one unit (ALS chunk) write (upper gram, rhs, count) partials and are summed
// in slot order by als_big_reduce_kernel before the same finish + solve.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "device.hpp"

namespace pmfgpu {

namespace {

constexpr int kBigThreads = 256;
constexpr int kBigTile = 32;                   // opposing rows staged per step
constexpr size_t kBigSmemMax = 200 * 1024;     // the k x k system stays in shared memory up to here

size_t big_floats_extra(int k) { return static_cast<size_t>(kBigTile) * k + kBigTile + 4 * static_cast<size_t>(k) + 8; }
bool big_g_in_smem(int k) {
    return (static_cast<size_t>(k) * k + big_floats_extra(k)) * sizeof(float) <= kBigSmemMax;
}
size_t big_smem_bytes(int k) {
    return ((big_g_in_smem(k) ? static_cast<size_t>(k) * k : 0) + big_floats_extra(k)) * sizeof(float);
}

struct BigWs {
    float *G, *X, *v, *b, *s, *x, *tmp;
    int* flag;
};

__device__ __forceinline__ BigWs big_ws(float* smem, float* gscratch, int k) {
    BigWs w;
    float* p = smem;
    if (gscratch) {
        w.G = gscratch + static_cast<int64_t>(blockIdx.x) * k * k;
    } else {
        w.G = p;
        p += k * k;
    }
    w.X = p;
    p += kBigTile * k;
    w.v = p;
    p += kBigTile;
    w.b = p;
    p += k;
    w.s = p;
    p += k;
    w.x = p;
    p += k;
    w.tmp = p;
    p += k;
    w.flag = reinterpret_cast<int*>(p);
    return w;
}

// G (k x k, upper triangle + rhs valid) -> x = (G + ridge I)^-1 b; false on a non-positive pivot.
// `finish`: add the ridge and mirror the upper triangle first (gram_finish); the batched Cholesky
// entry point passes a full SPD matrix.
__device__ bool cta_cholesky_solve(const BigWs& w, int k, float ridge, bool finish) {
    const int tid = threadIdx.x;
    if (finish) {
        for (int f = tid; f < k * k; f += kBigThreads) {
            const int a = f / k, c = f - a * k;
            if (c == a) w.G[f] = __fadd_rn(w.G[f], ridge);
            else if (c < a) w.G[f] = w.G[c * k + a];  // lower <- upper (distinct entries)
        }
    }
    if (tid == 0) *w.flag = 0;
    __syncthreads();
    for (int j = 0; j < k; ++j) {
        const float* Lj = w.G + static_cast<int64_t>(j) * k;
        for (int i = j + tid; i < k; i += kBigThreads) {
            const float* Li = w.G + static_cast<int64_t>(i) * k;
            float s = Li[j];
            for (int t = 0; t < j; ++t) s = __fsub_rn(s, __fmul_rn(Li[t], Lj[t]));
            w.tmp[i] = s;
        }
        __syncthreads();
        const float d = w.tmp[j];
        if (!(d > 0.f)) {  // dense.hpp:82-84
            if (tid == 0) *w.flag = 1;
            __syncthreads();
            return false;
        }
        const float ljj = __fsqrt_rn(d);
        for (int i = j + tid; i < k; i += kBigThreads)
            w.G[static_cast<int64_t>(i) * k + j] = i == j ? ljj : __fdiv_rn(w.tmp[i], ljj);
        __syncthreads();
    }
    // forward: L y = b (row i: s -= l_it y_t in ascending t)
    for (int i = tid; i < k; i += kBigThreads) w.s[i] = w.b[i];
    __syncthreads();
    for (int t = 0; t < k; ++t) {
        if (tid == 0) w.x[t] = __fdiv_rn(w.s[t], w.G[static_cast<int64_t>(t) * k + t]);
        __syncthreads();
        const float xt = w.x[t];
        for (int i = t + 1 + tid; i < k; i += kBigThreads)
            w.s[i] = __fsub_rn(w.s[i], __fmul_rn(w.G[static_cast<int64_t>(i) * k + t], xt));
        __syncthreads();
    }
    // backward: L^T x = y (column sweep, descending t)
    for (int i = tid; i < k; i += kBigThreads) w.s[i] = w.x[i];
    __syncthreads();
    for (int t = k - 1; t >= 0; --t) {
        if (tid == 0) w.x[t] = __fdiv_rn(w.s[t], w.G[static_cast<int64_t>(t) * k + t]);
        __syncthreads();
        const float xt = w.x[t];
        const float* Lt = w.G + static_cast<int64_t>(t) * k;
        for (int i = tid; i < t; i += kBigThreads) w.s[i] = __fsub_rn(w.s[i], __fmul_rn(Lt[i], xt));
        __syncthreads();
    }
    return true;
}

__global__ void __launch_bounds__(kBigThreads)
als_big_unit_kernel(const Unit* __restrict__ units, int32_t n_units, const int32_t* __restrict__ idx,
                    const float* __restrict__ val, const float* __restrict__ opp, float* __restrict__ out,
                    int32_t out_off, int k, float lambda, int weighted, float* __restrict__ partial,
                    int* __restrict__ counter, int* __restrict__ status, float* __restrict__ gscratch) {
    extern __shared__ __align__(16) float smem[];
    __shared__ int s_u;
    const BigWs w = big_ws(smem, gscratch, k);
    const int tid = threadIdx.x;
    for (;;) {
        if (tid == 0) s_u = atomicAdd(counter, 1);
        __syncthreads();
        const int u = s_u;
        if (u >= n_units) break;
        const Unit U = units[u];
        for (int f = tid; f < k * k; f += kBigThreads) w.G[f] = 0.f;
        for (int t = tid; t < k; t += kBigThreads) w.b[t] = 0.f;
        for (int e0 = 0; e0 < U.len; e0 += kBigTile) {
            const int cnt = min(kBigTile, U.len - e0);
            __syncthreads();  // previous tile consumed (and G / b zeroed)
            for (int f = tid; f < cnt * k; f += kBigThreads) {
                const int r = f / k, t = f - r * k;
                w.X[f] = opp[static_cast<int64_t>(idx[U.e0 + e0 + r]) * k + t];
            }
            if (tid < cnt) w.v[tid] = val[U.e0 + e0 + tid];
            __syncthreads();
            for (int f = tid; f < k * k; f += kBigThreads) {
                const int a = f / k, c = f - a * k;
                if (c < a) continue;
                float acc = w.G[f];
                for (int r = 0; r < cnt; ++r) acc = __fadd_rn(acc, __fmul_rn(w.X[r * k + a], w.X[r * k + c]));
                w.G[f] = acc;
            }
            for (int t = tid; t < k; t += kBigThreads) {
                float acc = w.b[t];
                for (int r = 0; r < cnt; ++r) acc = __fadd_rn(acc, __fmul_rn(w.v[r], w.X[r * k + t]));
                w.b[t] = acc;
            }
        }
        __syncthreads();
        if (U.slot >= 0) {  // one chunk of a long output: partial (upper gram, rhs, count)
            const int64_t stride = static_cast<int64_t>(k) * k + k + 1;
            float* P = partial + static_cast<int64_t>(U.slot) * stride;
            for (int f = tid; f < k * k; f += kBigThreads) P[f] = w.G[f];
            for (int t = tid; t < k; t += kBigThreads) P[k * k + t] = w.b[t];
            if (tid == 0) P[k * k + k] = static_cast<float>(U.len);
            continue;  // the loop head's barrier orders these reads before the next unit's writes
        }
        const float ridge = weighted ? lambda * static_cast<float>(U.len) : lambda;
        const bool ok = cta_cholesky_solve(w, k, ridge, true);
        float* dst = out + static_cast<int64_t>(out_off + U.o) * k;
        for (int t = tid; t < k; t += kBigThreads) dst[t] = ok ? w.x[t] : 0.f;
        if (!ok && tid == 0) atomicExch(status, 4);
    }
}

__global__ void __launch_bounds__(kBigThreads)
als_big_reduce_kernel(const int32_t* __restrict__ mo_out, const int32_t* __restrict__ mo_start, int32_t n_mo,
                      const float* __restrict__ partial, float* __restrict__ out, int32_t out_off, int k, float lambda,
                      int weighted, int* __restrict__ status, float* __restrict__ gscratch) {
    extern __shared__ __align__(16) float smem[];
    const BigWs w = big_ws(smem, gscratch, k);
    const int tid = threadIdx.x;
    const int64_t stride = static_cast<int64_t>(k) * k + k + 1;
    for (int q = blockIdx.x; q < n_mo; q += gridDim.x) {
        const int s0 = mo_start[q], s1 = mo_start[q + 1];
        __syncthreads();
        for (int f = tid; f < k * k; f += kBigThreads) {
            const int a = f / k, c = f - a * k;
            if (c < a) continue;
            float acc = 0.f;
            for (int s = s0; s < s1; ++s) acc = __fadd_rn(acc, partial[s * stride + f]);
            w.G[f] = acc;
        }
        for (int t = tid; t < k; t += kBigThreads) {
            float acc = 0.f;
            for (int s = s0; s < s1; ++s) acc = __fadd_rn(acc, partial[s * stride + k * k + t]);
            w.b[t] = acc;
        }
        float cnt = 0.f;
        for (int s = s0; s < s1; ++s) cnt += partial[s * stride + k * k + k];
        __syncthreads();
        const bool ok = cta_cholesky_solve(w, k, weighted ? lambda * cnt : lambda, true);
        float* dst = out + static_cast<int64_t>(out_off + mo_out[q]) * k;
        for (int t = tid; t < k; t += kBigThreads) dst[t] = ok ? w.x[t] : 0.f;
        if (!ok && tid == 0) atomicExch(status, 4);
    }
}

// pmf_cholesky_solve_batched for k > 64: a CTA per system; a <- L (strict upper zeroed, as
// cholesky_factor_inplace leaves it), x <- the solution.
__global__ void __launch_bounds__(kBigThreads)
chol_big_kernel(float* __restrict__ a, float* __restrict__ x, int batch, int k, int* __restrict__ status,
                float* __restrict__ gscratch) {
    extern __shared__ __align__(16) float smem[];
    const BigWs w = big_ws(smem, gscratch, k);
    const int tid = threadIdx.x;
    for (int q = blockIdx.x; q < batch; q += gridDim.x) {
        float* A = a + static_cast<int64_t>(q) * k * k;
        __syncthreads();
        for (int f = tid; f < k * k; f += kBigThreads) w.G[f] = A[f];
        for (int t = tid; t < k; t += kBigThreads) w.b[t] = x[static_cast<int64_t>(q) * k + t];
        __syncthreads();
        const bool ok = cta_cholesky_solve(w, k, 0.f, false);
        if (!ok && tid == 0) atomicExch(status, 4);
        for (int f = tid; f < k * k; f += kBigThreads) {
            const int r = f / k, c = f - r * k;
            A[f] = c <= r ? w.G[f] : 0.f;
        }
        for (int t = tid; t < k; t += kBigThreads) x[static_cast<int64_t>(q) * k + t] = ok ? w.x[t] : w.b[t];
    }
}

int big_blocks(const void* fn, int k, int sm_count) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kBigThreads, big_smem_bytes(k));
    return std::max(1, std::min(per_sm, 4)) * sm_count;
}

void set_big_attr(const void* fn, int k) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(big_smem_bytes(k)));
}

}  // namespace

int64_t als_big_scratch_floats(int k, int sm_count) {
    return big_g_in_smem(k) ? 0 : static_cast<int64_t>(4) * sm_count * k * k;
}

int launch_als_big(const DevAls& L, const float* opp, float* out, int32_t out_off, int k, float lambda, bool weighted,
                   int* d_counter, int* d_status, int sm_count, float* gscratch, cudaStream_t s) {
    float* gs = big_g_in_smem(k) ? nullptr : gscratch;
    const size_t sm = big_smem_bytes(k);
    int launched = 0;
    if (L.n_units > 0) {
        set_big_attr(reinterpret_cast<const void*>(als_big_unit_kernel), k);
        const int blocks = std::min(big_blocks(reinterpret_cast<const void*>(als_big_unit_kernel), k, sm_count),
                                    std::max(1, L.n_units));
        cudaMemsetAsync(d_counter, 0, sizeof(int), s);
        als_big_unit_kernel<<<blocks, kBigThreads, sm, s>>>(L.units, L.n_units, L.idx, L.val, opp, out, out_off, k,
                                                            lambda, weighted ? 1 : 0, L.partial, d_counter, d_status, gs);
        ++launched;
    }
    if (L.n_mo > 0) {
        set_big_attr(reinterpret_cast<const void*>(als_big_reduce_kernel), k);
        const int blocks = std::min(big_blocks(reinterpret_cast<const void*>(als_big_reduce_kernel), k, sm_count),
                                    L.n_mo);
        als_big_reduce_kernel<<<blocks, kBigThreads, sm, s>>>(L.mo_out, L.mo_start, L.n_mo, L.partial, out, out_off, k,
                                                              lambda, weighted ? 1 : 0, d_status, gs);
        ++launched;
    }
    return launched;
}

void launch_cholesky_big(float* a, float* x, int batch, int k, int* d_status, int sm_count, float* gscratch,
                         cudaStream_t s) {
    set_big_attr(reinterpret_cast<const void*>(chol_big_kernel), k);
    const int blocks = std::min(big_blocks(reinterpret_cast<const void*>(chol_big_kernel), k, sm_count), batch);
    chol_big_kernel<<<blocks, kBigThreads, big_smem_bytes(k), s>>>(a, x, batch, k, d_status,
                                                                  big_g_in_smem(k) ? nullptr : gscratch);
}

}  // namespace pmfgpu
