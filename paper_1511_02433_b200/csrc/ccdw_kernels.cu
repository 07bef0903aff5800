// ccdw_kernels.cu -- item/user-wise CCD (ccd.hpp:52-125, ccd_train :310-344) on the GPU, residual form.
//
// The default path.  PMF_CCD_GRAM=1 (k <= 64) runs the equivalent gram form instead (als_kernels.cu
// warp_gauss_seidel: one Gauss-Seidel sweep per row on its normal equations, gram + right-hand side on
// the tensor cores, no residual): 10x faster, but without the reference's float-residual rounding its
// trajectory drifts from the reference's (objective 1.9e-4 apart after 5 Netflix epochs vs 3e-6 here).
//
// One CCD epoch updates every coordinate w_it (rows in order, t = 0..k-1 within a row) with the
// closed-form 1-D minimiser z* = sum_j (R_ij + w_it h_jt) h_jt / (lambda + sum_j h_jt^2), shifting the
// row's residual by (z* - w_it) h_jt, then mirrors the same for every h_jt over the columns.  Rows
// only touch their own residual entries and W row while H is fixed, so the W sweep is exact with a
// warp per row (the reference runs it on one worker only because it loops rows sequentially); the
// same holds for columns in the H sweep, with a CTA per column (columns reach m entries).  Within a
// row / column the t loop stays sequential.  The residual lives in CSR order for the W sweep and in
// CSC order for the H sweep; between the sweeps one layout is copied into the other through the
// position maps, so both stay bitwise equal (the reference's set_from_row / set_from_col mirror,
// sparse.hpp:241-250).  Per-entry arithmetic rounds like the reference (products before adds); the
// sums over a row / column are warp / CTA trees (reduction order differs, as everywhere on the GPU).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "device.hpp"

namespace pmfgpu {

namespace {

constexpr int kRowCache = 8;      // residual entries per lane kept in registers (rows <= 256)
constexpr int kColThreads = 256;

// position maps between the two layouts: csr2csc[p] = q and csc2csr[q] = p
__global__ void ccd_xlink_kernel(const int64_t* __restrict__ row_start, const int32_t* __restrict__ col_of,
                                 const int64_t* __restrict__ col_start, const int32_t* __restrict__ row_of,
                                 int32_t m, int32_t* __restrict__ csr2csc, int32_t* __restrict__ csc2csr) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < m;
         i += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
        for (int64_t p = row_start[i] + lane; p < row_start[i + 1]; p += 32) {
            const int32_t j = col_of[p];
            int64_t lo = col_start[j], hi = col_start[j + 1];
            while (lo < hi) {  // first position of column j whose row is >= i
                const int64_t mid = (lo + hi) >> 1;
                if (row_of[mid] < i) lo = mid + 1;
                else hi = mid;
            }
            csr2csc[p] = static_cast<int32_t>(lo);
            csc2csr[lo] = static_cast<int32_t>(p);
        }
    }
}

__global__ void ccd_gather_kernel(float* __restrict__ dst, const float* __restrict__ src,
                                  const int32_t* __restrict__ map, int64_t n) {
    for (int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; x < n;
         x += static_cast<int64_t>(gridDim.x) * blockDim.x)
        dst[x] = src[map[x]];
}

__device__ __forceinline__ void warp_sum2(float& a, float& b) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, off);
        b += __shfl_xor_sync(0xffffffffu, b, off);
    }
}

// W sweep (ccd.hpp:113-116): a warp per row; for each t the z* of ccd_z_star (:56-68) and the
// residual shift of ccd_apply_z (:73-80).  Rows <= 256 entries keep their residual in registers and
// take the gathered h of kRowChunk coordinates at once: one 4 kRowChunk-byte read of the row-major H
// row per entry (a 32-byte sector serves kRowChunk coordinates instead of one), parked in the warp's
// shared-memory slice (each lane only touches its own entries' values), and the row's w of the chunk
// by one load; longer rows stream R and gather per coordinate.
#ifndef PMF_CCDW_ROW_CHUNK
#define PMF_CCDW_ROW_CHUNK 8
#endif
constexpr int kRowChunk = PMF_CCDW_ROW_CHUNK;
constexpr int kRowThreads = 256;
constexpr int kRowSmemFloats = (kRowThreads / 32) * kRowChunk * kRowCache * 32;
__global__ void __launch_bounds__(kRowThreads, 3)
ccd_rows_kernel(const int64_t* __restrict__ row_start, const int32_t* __restrict__ col_of,
                float* __restrict__ R, float* __restrict__ W, const float* __restrict__ H,
                int32_t m, int k, float lambda) {
    extern __shared__ __align__(16) float rsm[];
    const int lane = threadIdx.x & 31;
    float* hs = rsm + (threadIdx.x >> 5) * (kRowChunk * kRowCache * 32);  // [q][c][lane]
    const bool vec = (k & 3) == 0 && (kRowChunk & 3) == 0;
    for (int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < m;
         i += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
        const int64_t b = row_start[i], e = row_start[i + 1];
        if (e - b <= 32 * kRowCache) {
            float r[kRowCache];
            int32_t jj[kRowCache];
#pragma unroll
            for (int c = 0; c < kRowCache; ++c) {
                const int64_t p = b + lane + 32 * c;
                r[c] = p < e ? R[p] : 0.f;
                jj[c] = p < e ? col_of[p] : -1;
            }
            for (int t0 = 0; t0 < k; t0 += kRowChunk) {
                const int cc = min(kRowChunk, k - t0);
#pragma unroll
                for (int c = 0; c < kRowCache; ++c) {
                    if (jj[c] < 0) continue;
                    const float* src = H + static_cast<int64_t>(jj[c]) * k + t0;
                    if (vec && cc == kRowChunk) {
#pragma unroll
                        for (int q = 0; q < kRowChunk; q += 4) {
                            const float4 v = *reinterpret_cast<const float4*>(src + q);
                            hs[((q + 0) * kRowCache + c) * 32 + lane] = v.x;
                            hs[((q + 1) * kRowCache + c) * 32 + lane] = v.y;
                            hs[((q + 2) * kRowCache + c) * 32 + lane] = v.z;
                            hs[((q + 3) * kRowCache + c) * 32 + lane] = v.w;
                        }
                    } else {
                        for (int q = 0; q < cc; ++q) hs[(q * kRowCache + c) * 32 + lane] = src[q];
                    }
                }
                const float wl = lane < cc ? W[i * k + t0 + lane] : 0.f;
                float zl = 0.f;
                for (int tt = 0; tt < cc; ++tt) {
                    const float wit = __shfl_sync(0xffffffffu, wl, tt);
                    float num = 0.f, den = 0.f;
                    float hc[kRowCache];
#pragma unroll
                    for (int c = 0; c < kRowCache; ++c) {
                        hc[c] = jj[c] >= 0 ? hs[(tt * kRowCache + c) * 32 + lane] : 0.f;
                        if (jj[c] >= 0) {
                            num = __fadd_rn(num, __fmul_rn(__fadd_rn(r[c], __fmul_rn(wit, hc[c])), hc[c]));
                            den = __fadd_rn(den, __fmul_rn(hc[c], hc[c]));
                        }
                    }
                    warp_sum2(num, den);
                    const float dt = __fadd_rn(lambda, den);
                    const float z = dt == 0.f ? 0.f : __fdiv_rn(num, dt);
                    const float delta = __fsub_rn(z, wit);
#pragma unroll
                    for (int c = 0; c < kRowCache; ++c) r[c] = __fsub_rn(r[c], __fmul_rn(delta, hc[c]));
                    if (lane == tt) zl = z;
                }
                if (lane < cc) W[i * k + t0 + lane] = zl;
            }
#pragma unroll
            for (int c = 0; c < kRowCache; ++c) {
                const int64_t p = b + lane + 32 * c;
                if (p < e) R[p] = r[c];
            }
            continue;
        }
        for (int t = 0; t < k; ++t) {
            const float wit = W[i * k + t];
            float num = 0.f, den = 0.f;
            for (int64_t p = b + lane; p < e; p += 32) {
                const float h = H[static_cast<int64_t>(col_of[p]) * k + t];
                num = __fadd_rn(num, __fmul_rn(__fadd_rn(R[p], __fmul_rn(wit, h)), h));
                den = __fadd_rn(den, __fmul_rn(h, h));
            }
            warp_sum2(num, den);
            const float dt = __fadd_rn(lambda, den);
            const float z = dt == 0.f ? 0.f : __fdiv_rn(num, dt);
            const float delta = __fsub_rn(z, wit);
            for (int64_t p = b + lane; p < e; p += 32)
                R[p] = __fsub_rn(R[p], __fmul_rn(delta, H[static_cast<int64_t>(col_of[p]) * k + t]));
            if (lane == 0) W[i * k + t] = z;
        }
    }
}

// H sweep (ccd.hpp:117-119): a CTA per column, ccd_s_star (:84-96) / ccd_apply_s (:99-106).
__global__ void __launch_bounds__(kColThreads)
ccd_cols_kernel(const int64_t* __restrict__ col_start, const int32_t* __restrict__ row_of, float* __restrict__ R,
                const float* __restrict__ W, float* __restrict__ H, int32_t n, int k, float lambda) {
    __shared__ float s_num[kColThreads / 32], s_den[kColThreads / 32];
    __shared__ float s_z;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t j = blockIdx.x; j < n; j += gridDim.x) {
        const int64_t b = col_start[j], e = col_start[j + 1];
        for (int t = 0; t < k; ++t) {
            const float hjt = H[j * k + t];
            float num = 0.f, den = 0.f;
            for (int64_t q = b + threadIdx.x; q < e; q += kColThreads) {
                const float w = W[static_cast<int64_t>(row_of[q]) * k + t];
                num = __fadd_rn(num, __fmul_rn(__fadd_rn(R[q], __fmul_rn(w, hjt)), w));
                den = __fadd_rn(den, __fmul_rn(w, w));
            }
            warp_sum2(num, den);
            if (lane == 0) {
                s_num[warp] = num;
                s_den[warp] = den;
            }
            __syncthreads();
            if (warp == 0) {
                num = lane < kColThreads / 32 ? s_num[lane] : 0.f;
                den = lane < kColThreads / 32 ? s_den[lane] : 0.f;
                warp_sum2(num, den);
                if (lane == 0) {
                    const float dt = __fadd_rn(lambda, den);
                    s_z = dt == 0.f ? 0.f : __fdiv_rn(num, dt);
                }
            }
            __syncthreads();
            const float z = s_z;
            const float delta = __fsub_rn(z, hjt);
            for (int64_t q = b + threadIdx.x; q < e; q += kColThreads)
                R[q] = __fsub_rn(R[q], __fmul_rn(delta, W[static_cast<int64_t>(row_of[q]) * k + t]));
            if (threadIdx.x == 0) H[j * k + t] = z;
            __syncthreads();  // H[j,t] and s_z settled before the next t
        }
    }
}

// H sweep, longest columns first: CTAs of kColThreadsL threads claim columns from a counter over col_order (LPT;
// the popular columns hold up to ~5 % of the entries each), and gather w_it from the column-major copy
// WT (k x m), so that the dense row ranges of long columns read coalesced.  One pass per coordinate t:
// the pass of t applies the residual shift of t - 1 (R -= (z - h_j,t-1) w_i,t-1, the reference's
// ccd_apply_s arithmetic, deferred) and accumulates the sums of t; a last pass applies the shift of k - 1.
// threads per column CTA (2 CTAs per SM): Netflix k = 40 epoch 37.3 ms with 512, 39.0 with 256, 40.1 with 1024
#ifndef PMF_CCDW_COL_THREADS
#define PMF_CCDW_COL_THREADS 512
#endif
constexpr int kColThreadsL = PMF_CCDW_COL_THREADS;
#ifndef PMF_CCDW_COL_CACHE
#define PMF_CCDW_COL_CACHE 16
#endif
// residual entries per thread of a cached column (columns <= 8K entries: ~46 % of Netflix's ratings) and
// coordinates gathered per chunk: Netflix k = 40 epoch 25.4 ms with 16 / 4, 26.6 with 8 / 4, 28.7 with 16 / 2,
// 32.0 without the cached path (scripts/ccdw_run.py)
constexpr int kColCache = PMF_CCDW_COL_CACHE;
#ifndef PMF_CCDW_COL_CHUNK
#define PMF_CCDW_COL_CHUNK 4
#endif
constexpr int kColChunk = PMF_CCDW_COL_CHUNK;
constexpr int kColSmemFloats = kColChunk * kColCache * kColThreadsL;
__global__ void __launch_bounds__(kColThreadsL)
ccd_cols_lpt_kernel(const int64_t* __restrict__ col_start, const int32_t* __restrict__ row_of, float* __restrict__ R,
                    const float* __restrict__ W, const float* __restrict__ WT, float* __restrict__ H, int32_t n,
                    int32_t m, int k, float lambda, const int32_t* __restrict__ col_order, int* __restrict__ counter) {
    __shared__ float s_num[kColThreadsL / 32], s_den[kColThreadsL / 32];
    __shared__ float s_z;
    __shared__ int s_j;
    extern __shared__ __align__(16) float csm[];  // cached columns: [q][c][thread] gathered w of a chunk
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tid = threadIdx.x;
    const bool vec = (k & 3) == 0 && (kColChunk & 3) == 0;
    for (;;) {
        if (threadIdx.x == 0) s_j = atomicAdd(counter, 1);
        __syncthreads();
        const int jj = s_j;
        __syncthreads();
        if (jj >= n) break;
        const int32_t j = col_order[jj];
        const int64_t b = col_start[j], e = col_start[j + 1];
        if (e - b <= static_cast<int64_t>(kColThreadsL) * kColCache) {
            // the column's residual in registers (kColCache per thread); the w of kColChunk coordinates
            // gathered at once from the row-major W (one sector per entry and chunk)
            float r[kColCache];
            int32_t ii[kColCache];
#pragma unroll
            for (int c = 0; c < kColCache; ++c) {
                const int64_t p = b + tid + static_cast<int64_t>(kColThreadsL) * c;
                r[c] = p < e ? R[p] : 0.f;
                ii[c] = p < e ? row_of[p] : -1;
            }
            for (int t0 = 0; t0 < k; t0 += kColChunk) {
                const int cc = min(kColChunk, k - t0);
#pragma unroll
                for (int c = 0; c < kColCache; ++c) {
                    if (ii[c] < 0) continue;
                    const float* src = W + static_cast<int64_t>(ii[c]) * k + t0;
                    if (vec && cc == kColChunk) {
#pragma unroll
                        for (int q = 0; q < kColChunk; q += 4) {
                            const float4 v = *reinterpret_cast<const float4*>(src + q);
                            csm[((q + 0) * kColCache + c) * kColThreadsL + tid] = v.x;
                            csm[((q + 1) * kColCache + c) * kColThreadsL + tid] = v.y;
                            csm[((q + 2) * kColCache + c) * kColThreadsL + tid] = v.z;
                            csm[((q + 3) * kColCache + c) * kColThreadsL + tid] = v.w;
                        }
                    } else {
                        for (int q = 0; q < cc; ++q) csm[(q * kColCache + c) * kColThreadsL + tid] = src[q];
                    }
                }
                for (int tt = 0; tt < cc; ++tt) {
                    const float hjt = H[static_cast<int64_t>(j) * k + t0 + tt];
                    float num = 0.f, den = 0.f;
                    float wc[kColCache];
#pragma unroll
                    for (int c = 0; c < kColCache; ++c) {
                        wc[c] = ii[c] >= 0 ? csm[(tt * kColCache + c) * kColThreadsL + tid] : 0.f;
                        if (ii[c] >= 0) {
                            num = __fadd_rn(num, __fmul_rn(__fadd_rn(r[c], __fmul_rn(wc[c], hjt)), wc[c]));
                            den = __fadd_rn(den, __fmul_rn(wc[c], wc[c]));
                        }
                    }
                    warp_sum2(num, den);
                    if (lane == 0) {
                        s_num[warp] = num;
                        s_den[warp] = den;
                    }
                    __syncthreads();
                    if (warp == 0) {
                        num = lane < kColThreadsL / 32 ? s_num[lane] : 0.f;
                        den = lane < kColThreadsL / 32 ? s_den[lane] : 0.f;
                        warp_sum2(num, den);
                        if (lane == 0) {
                            const float dt = __fadd_rn(lambda, den);
                            s_z = dt == 0.f ? 0.f : __fdiv_rn(num, dt);
                            H[static_cast<int64_t>(j) * k + t0 + tt] = s_z;
                        }
                    }
                    __syncthreads();
                    const float delta = __fsub_rn(s_z, hjt);
#pragma unroll
                    for (int c = 0; c < kColCache; ++c) r[c] = __fsub_rn(r[c], __fmul_rn(delta, wc[c]));
                }
            }
#pragma unroll
            for (int c = 0; c < kColCache; ++c) {
                const int64_t p = b + tid + static_cast<int64_t>(kColThreadsL) * c;
                if (p < e) R[p] = r[c];
            }
            continue;
        }
        float dprev = 0.f;
        for (int t = 0; t <= k; ++t) {
            const bool last = t == k;
            const float hjt = last ? 0.f : H[static_cast<int64_t>(j) * k + t];
            const float* wt = WT + static_cast<int64_t>(t) * m;
            const float* wp = WT + static_cast<int64_t>(t - 1) * m;
            float num = 0.f, den = 0.f;
            // four entries per thread per step, all loads issued before their use (long columns stream
            // through one CTA: the dependent row -> w gathers need several in flight per thread)
            constexpr int U = 4;
            for (int64_t q0 = b + threadIdx.x; q0 < e; q0 += U * kColThreadsL) {
                int32_t iu[U];
                float ru[U], pu[U], wu[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int64_t q = q0 + static_cast<int64_t>(u) * kColThreadsL;
                    iu[u] = q < e ? row_of[q] : 0;
                    ru[u] = q < e ? R[q] : 0.f;
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    pu[u] = t > 0 ? wp[iu[u]] : 0.f;
                    wu[u] = last ? 0.f : wt[iu[u]];
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int64_t q = q0 + static_cast<int64_t>(u) * kColThreadsL;
                    if (q >= e) continue;
                    float r = ru[u];
                    if (t > 0) {
                        r = __fsub_rn(r, __fmul_rn(dprev, pu[u]));
                        R[q] = r;
                    }
                    if (!last) {
                        num = __fadd_rn(num, __fmul_rn(__fadd_rn(r, __fmul_rn(wu[u], hjt)), wu[u]));
                        den = __fadd_rn(den, __fmul_rn(wu[u], wu[u]));
                    }
                }
            }
            if (last) break;
            warp_sum2(num, den);
            if (lane == 0) {
                s_num[warp] = num;
                s_den[warp] = den;
            }
            __syncthreads();
            if (warp == 0) {
                num = lane < kColThreadsL / 32 ? s_num[lane] : 0.f;
                den = lane < kColThreadsL / 32 ? s_den[lane] : 0.f;
                warp_sum2(num, den);
                if (lane == 0) {
                    const float dt = __fadd_rn(lambda, den);
                    s_z = dt == 0.f ? 0.f : __fdiv_rn(num, dt);
                }
            }
            __syncthreads();
            const float z = s_z;
            dprev = __fsub_rn(z, hjt);
            if (threadIdx.x == 0) H[static_cast<int64_t>(j) * k + t] = z;
            __syncthreads();  // s_z read by every thread before the next t overwrites it
        }
    }
}

// WT (k x m, column-major) <- W (m x k, row-major): 32 x 32 tiles through shared memory
__global__ void ccd_transpose_kernel(const float* __restrict__ W, float* __restrict__ WT, int32_t m, int k) {
    __shared__ float tile[32][33];
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * 32;
    const int t0 = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t i = i0 + r;
        const int t = t0 + threadIdx.x;
        tile[r][threadIdx.x] = (i < m && t < k) ? W[i * k + t] : 0.f;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int t = t0 + r;
        const int64_t i = i0 + threadIdx.x;
        if (t < k && i < m) WT[static_cast<int64_t>(t) * m + i] = tile[threadIdx.x][r];
    }
}

// R = A - W H^T from scratch (a warp per row; t ascending, each product rounded before the subtract):
// the residual of a model installed with set_model (residual_from + the writebacks' arithmetic).
__global__ void ccd_residual_kernel(const int64_t* __restrict__ row_start, const int32_t* __restrict__ col_of,
                                    const float* __restrict__ A, const float* __restrict__ W,
                                    const float* __restrict__ H, int32_t m, int k, float* __restrict__ R) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < m;
         i += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
        const float* w = W + i * k;
        for (int64_t p = row_start[i] + lane; p < row_start[i + 1]; p += 32) {
            const float* h = H + static_cast<int64_t>(col_of[p]) * k;
            float r = A[p];
            for (int t = 0; t < k; ++t) r = __fsub_rn(r, __fmul_rn(w[t], h[t]));
            R[p] = r;
        }
    }
}

}  // namespace

void launch_ccd_residual(const CcdWs& ws, const float* A_row, const float* W, const float* H, int k, cudaStream_t s) {
    if (ws.m > 0) ccd_residual_kernel<<<148 * 8, 256, 0, s>>>(ws.row_start, ws.col_of, A_row, W, H, ws.m, k, ws.R_row);
    if (ws.nnz > 0) ccd_gather_kernel<<<148 * 16, 256, 0, s>>>(ws.R_col, ws.R_row, ws.csc2csr, ws.nnz);
}

void launch_ccd_xlinks(const int64_t* row_start, const int32_t* col_of, const int64_t* col_start,
                       const int32_t* row_of, int32_t m, int32_t* csr2csc, int32_t* csc2csr, cudaStream_t s) {
    if (m <= 0) return;
    ccd_xlink_kernel<<<148 * 8, 256, 0, s>>>(row_start, col_of, col_start, row_of, m, csr2csc, csc2csr);
}

int launch_ccd_epoch(const CcdWs& ws, float* W, float* H, int k, float lambda, cudaStream_t s) {
    int launched = 0;
    if (ws.m > 0) {
        static const int per_sm = [] {
            const int bytes = kRowSmemFloats * static_cast<int>(sizeof(float));
            cudaFuncSetAttribute(ccd_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
            int n = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, ccd_rows_kernel, kRowThreads, bytes);
            return std::max(n, 1);
        }();
        ccd_rows_kernel<<<148 * per_sm, kRowThreads, kRowSmemFloats * sizeof(float), s>>>(ws.row_start, ws.col_of,
                                                                                          ws.R_row, W, H, ws.m, k,
                                                                                          lambda);
        ++launched;
    }
    if (ws.nnz > 0) {
        ccd_gather_kernel<<<148 * 16, 256, 0, s>>>(ws.R_col, ws.R_row, ws.csc2csr, ws.nnz);  // set_from_row
        ++launched;
    }
    if (ws.n > 0 && ws.WT) {
        ccd_transpose_kernel<<<dim3((ws.m + 31) / 32, (k + 31) / 32), dim3(32, 8), 0, s>>>(W, ws.WT, ws.m, k);
        cudaMemsetAsync(ws.counter, 0, sizeof(int), s);
        static const int col_per_sm = [] {
            const int bytes = kColSmemFloats * static_cast<int>(sizeof(float));
            cudaFuncSetAttribute(ccd_cols_lpt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
            int nb = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, ccd_cols_lpt_kernel, kColThreadsL, bytes);
            return std::max(1, std::min(nb, 1024 / kColThreadsL));
        }();
        ccd_cols_lpt_kernel<<<148 * col_per_sm, kColThreadsL, kColSmemFloats * sizeof(float), s>>>(
            ws.col_start, ws.row_of, ws.R_col, W, ws.WT, H, ws.n, ws.m, k, lambda, ws.col_order, ws.counter);
        launched += 2;
    } else if (ws.n > 0) {
        ccd_cols_kernel<<<148 * 8, kColThreads, 0, s>>>(ws.col_start, ws.row_of, ws.R_col, W, H, ws.n, k, lambda);
        ++launched;
    }
    if (ws.nnz > 0) {
        ccd_gather_kernel<<<148 * 16, 256, 0, s>>>(ws.R_row, ws.R_col, ws.csr2csc, ws.nnz);  // set_from_col
        ++launched;
    }
    return launched;
}

}  // namespace pmfgpu
