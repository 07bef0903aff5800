// layout_device.cu -- the per-entry passes of the sweep-layout build on the device, for contexts built
// straight from triplets (pmf_ctx_create_from_triplets): the CSR / CSC stay in HBM after the device
// ingest (ingest.cu), the host builds the layout's structure (panels, units, slots, CTA partition --
// layout.cpp, build_sweep_layout with a SegCounter) from per-(panel, output) segment lengths counted
// here, and the residual / index streams are filled here.  The result is bitwise the host builder's
// layout (tests/test_gpu_ctx_triplets.py compares training runs on both).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "device.hpp"

namespace pmfgpu {

namespace {

// first position in [lo, hi) of a sorted index array whose value is >= key
__device__ __forceinline__ int64_t lower_bound_idx(const int32_t* __restrict__ a, int64_t lo, int64_t hi, int64_t key) {
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// seg_len[p * n_out + o] = entries of output o whose gather index lies in panel p (outputs' indices
// ascend: two binary searches per (p, o))
__global__ void seg_count_kernel(const int64_t* __restrict__ start, const int32_t* __restrict__ idx, int32_t n_out,
                                 int32_t pg, int32_t np, int32_t* __restrict__ seg_len) {
    const int64_t total = static_cast<int64_t>(n_out) * np;
    for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < total;
         s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t p = static_cast<int32_t>(s / n_out), o = static_cast<int32_t>(s % n_out);
        const int64_t b = start[o], e = start[o + 1];
        const int64_t lo = p == 0 ? b : lower_bound_idx(idx, b, e, static_cast<int64_t>(p) * pg);
        const int64_t hi = p == np - 1 ? e : lower_bound_idx(idx, lo, e, static_cast<int64_t>(p + 1) * pg);
        seg_len[s] = static_cast<int32_t>(hi - lo);
    }
}

// padding everywhere first (sentinel index, zero value), the real entries are scattered over it
template <typename I>
__global__ void pad_fill_kernel(I* __restrict__ out_idx, float* __restrict__ out_val, int64_t n, I sentinel) {
    for (int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; x < n;
         x += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        out_idx[x] = sentinel;
        out_val[x] = 0.f;
    }
}

// Entry e of output o with gather index g goes to e + delta[p * n_out + o], p = g / pg, as panel-local
// index g - p pg.  A CTA takes a tile of kTile consecutive entries; its outputs are found by binary
// search over start between the tile's first and last entry's outputs.
constexpr int kFillThreads = 256;
constexpr int kTile = 2048;
template <typename I>
__global__ void __launch_bounds__(kFillThreads)
scatter_fill_kernel(const int64_t* __restrict__ start, const int32_t* __restrict__ idx, const float* __restrict__ val,
                    int32_t n_out, int64_t nnz, int32_t pg, int32_t np, const int64_t* __restrict__ delta,
                    I* __restrict__ out_idx, float* __restrict__ out_val) {
    __shared__ int32_t s_o[2];
    for (int64_t t0 = static_cast<int64_t>(blockIdx.x) * kTile; t0 < nnz; t0 += static_cast<int64_t>(gridDim.x) * kTile) {
        const int64_t t1 = min(nnz, t0 + kTile);
        __syncthreads();
        if (threadIdx.x < 2) {  // output containing entry t0 / t1 - 1: last o with start[o] <= e
            const int64_t e = threadIdx.x == 0 ? t0 : t1 - 1;
            int32_t lo = 0, hi = n_out;  // start[lo] <= e < start[hi]
            while (hi - lo > 1) {
                const int32_t mid = (lo + hi) >> 1;
                if (start[mid] <= e) lo = mid;
                else hi = mid;
            }
            s_o[threadIdx.x] = lo;
        }
        __syncthreads();
        const int32_t ob = s_o[0], oe = s_o[1];
        for (int64_t e = t0 + threadIdx.x; e < t1; e += kFillThreads) {
            int32_t lo = ob, hi = oe + 1;
            while (hi - lo > 1) {
                const int32_t mid = (lo + hi) >> 1;
                if (start[mid] <= e) lo = mid;
                else hi = mid;
            }
            const int32_t g = idx[e];
            const int32_t p = np > 1 ? g / pg : 0;
            const int64_t w = e + delta[static_cast<int64_t>(p) * n_out + lo];
            out_idx[w] = static_cast<I>(g - p * pg);
            out_val[w] = val[e];
        }
    }
}

// usplit[u * (S + 1) + q]: entries of unit u (ascending panel-local indices) below q * sub_width
__global__ void usplit_kernel(const Unit* __restrict__ units, const int32_t* __restrict__ real, int64_t nu,
                              const uint16_t* __restrict__ idx, int S, int32_t sub_width, uint16_t* __restrict__ out) {
    for (int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u < nu;
         u += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t e0 = units[u].e0;
        const int32_t n = real[u];
        uint16_t* sp = out + u * (S + 1);
        sp[0] = 0;
        int32_t x = 0;
        for (int q = 1; q < S; ++q) {
            const int32_t bound = q * sub_width;
            int32_t lo = x, hi = n;
            while (lo < hi) {
                const int32_t mid = (lo + hi) >> 1;
                if (static_cast<int32_t>(idx[e0 + mid]) < bound) lo = mid + 1;
                else hi = mid;
            }
            x = lo;
            sp[q] = static_cast<uint16_t>(x);
        }
        sp[S] = static_cast<uint16_t>(n);
    }
}

int grid_for(int64_t n, int threads) {
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, 148 * 16)));
}

}  // namespace

void seg_count_device(const int64_t* start, const int32_t* idx, int32_t n_out, int32_t pg, int32_t np,
                      int32_t* seg_len, cudaStream_t s) {
    const int64_t total = static_cast<int64_t>(n_out) * np;
    if (total > 0) seg_count_kernel<<<grid_for(total, 256), 256, 0, s>>>(start, idx, n_out, pg, np, seg_len);
}

void layout_fill_device(const int64_t* start, const int32_t* idx, const float* val, int32_t n_out, int64_t nnz,
                        int32_t pg, int32_t np, const int64_t* delta, bool idx16, int32_t sentinel, int64_t n_entries,
                        void* out_idx, float* out_val, cudaStream_t s) {
    const int tiles = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((nnz + kTile - 1) / kTile, 148 * 32)));
    if (idx16) {
        auto* oi = static_cast<uint16_t*>(out_idx);
        pad_fill_kernel<<<grid_for(n_entries, 256), 256, 0, s>>>(oi, out_val, n_entries, static_cast<uint16_t>(sentinel));
        if (nnz > 0)
            scatter_fill_kernel<<<tiles, kFillThreads, 0, s>>>(start, idx, val, n_out, nnz, pg, np, delta, oi, out_val);
    } else {
        auto* oi = static_cast<int32_t*>(out_idx);
        pad_fill_kernel<<<grid_for(n_entries, 256), 256, 0, s>>>(oi, out_val, n_entries, sentinel);
        if (nnz > 0)
            scatter_fill_kernel<<<tiles, kFillThreads, 0, s>>>(start, idx, val, n_out, nnz, pg, np, delta, oi, out_val);
    }
}

void usplit_device(const Unit* units, const int32_t* real, int64_t nu, const uint16_t* idx, int S, int32_t sub_width,
                   uint16_t* out, cudaStream_t s) {
    if (nu > 0) usplit_kernel<<<grid_for(nu, 256), 256, 0, s>>>(units, real, nu, idx, S, sub_width, out);
}

}  // namespace pmfgpu
