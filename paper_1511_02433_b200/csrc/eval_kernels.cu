// eval_kernels.cu -- objective / train RMSE / probe RMSE (model.hpp:103-167) on the device.
//
// The reference accumulates in double in a fixed sequential order.  Here every per-entry term is
// formed exactly as the reference forms it (objective: dot in double, products rounded before the
// add; predict: FP32 sequential over t, products rounded before the add) and the sums use
// fixed-shape reductions, so results are deterministic and agree with the reference to double
// rounding of the summation order.
#include <cuda_runtime.h>

#include <algorithm>

#include <cstdint>

#include "device.hpp"

namespace pmfgpu {

namespace {

constexpr int kRedThreads = 1024;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// block-wide fixed-shape sum; result valid in thread 0
__device__ double block_sum(double v, double* sm) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) sm[warp] = v;
    __syncthreads();
    const int nw = blockDim.x >> 5;
    double r = 0.0;
    if (warp == 0) {
        r = lane < nw ? sm[lane] : 0.0;
        r = warp_sum(r);
    }
    __syncthreads();
    return r;
}

// row-major factor rows with k % 4 == 0 are read as float4 (the products and their order are the
// same either way: t ascending, each product rounded before the add)
template <bool VEC>
__device__ __forceinline__ double dot_double(FactorView W, int64_t i, FactorView H, int64_t j, int k) {
    double pred = 0.0;
    if (VEC) {
        const float4* wr = reinterpret_cast<const float4*>(W.p + i * W.si);
        const float4* hr = reinterpret_cast<const float4*>(H.p + j * H.si);
        for (int t4 = 0; t4 < (k >> 2); ++t4) {
            const float4 w = wr[t4], h = hr[t4];
            pred = __dadd_rn(pred, __dmul_rn(static_cast<double>(w.x), static_cast<double>(h.x)));
            pred = __dadd_rn(pred, __dmul_rn(static_cast<double>(w.y), static_cast<double>(h.y)));
            pred = __dadd_rn(pred, __dmul_rn(static_cast<double>(w.z), static_cast<double>(h.z)));
            pred = __dadd_rn(pred, __dmul_rn(static_cast<double>(w.w), static_cast<double>(h.w)));
        }
    } else {
        for (int t = 0; t < k; ++t)
            pred = __dadd_rn(pred, __dmul_rn(static_cast<double>(W.p[i * W.si + t * W.st]),
                                             static_cast<double>(H.p[j * H.si + t * H.st])));
    }
    return pred;
}

template <bool IDX16, bool VEC>
__global__ void unit_loss_kernel(const Unit* __restrict__ units, const int32_t* __restrict__ unit_panel,
                                 const int32_t* __restrict__ panel_base, const void* __restrict__ idx,
                                 const float* __restrict__ A, int32_t n_units, int32_t sentinel,
                                 int32_t row_off, FactorView W, FactorView H, int k,
                                 double* __restrict__ unit_loss) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t u = wid; u < n_units; u += nw) {
        const Unit U = units[u];
        const int32_t gb = panel_base[unit_panel[u]];
        const int64_t i = row_off + U.o;
        double acc = 0.0;
        for (int64_t e = U.e0 + lane; e < static_cast<int64_t>(U.e0) + U.len; e += 32) {
            const int g = IDX16 ? static_cast<const uint16_t*>(idx)[e] : static_cast<const int32_t*>(idx)[e];
            if (g == sentinel) continue;
            const double err = static_cast<double>(A[e]) - dot_double<VEC>(W, i, H, gb + g, k);
            acc += err * err;
        }
        acc = warp_sum(acc);
        if (lane == 0) unit_loss[u] = acc;
    }
}

__global__ void sum_stage1(const double* __restrict__ x, int64_t n, double* __restrict__ part) {
    __shared__ double sm[32];
    double v = 0.0;
    for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < n;
         q += static_cast<int64_t>(gridDim.x) * blockDim.x)
        v += x[q];
    v = block_sum(v, sm);
    if (threadIdx.x == 0) part[blockIdx.x] = v;
}

__global__ void sumsq_stage1(const float* __restrict__ x, int64_t n, double* __restrict__ part) {
    __shared__ double sm[32];
    double v = 0.0;
    for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < n;
         q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double d = static_cast<double>(x[q]);
        v += d * d;
    }
    v = block_sum(v, sm);
    if (threadIdx.x == 0) part[blockIdx.x] = v;
}

__global__ void sum_stage2(const double* __restrict__ part, int n, double* __restrict__ out) {
    __shared__ double sm[32];
    double v = 0.0;
    for (int q = threadIdx.x; q < n; q += blockDim.x) v += part[q];
    v = block_sum(v, sm);
    if (threadIdx.x == 0) *out = v;
}

__global__ void probe_sse_kernel(const DevTriplet* __restrict__ probe, int64_t n, FactorView W,
                                 FactorView H, int k, double* __restrict__ part) {
    __shared__ double sm[32];
    double v = 0.0;
    for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < n;
         q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const DevTriplet t = probe[q];
        float s = 0.f;
        for (int f = 0; f < k; ++f)
            s = __fadd_rn(s, __fmul_rn(W.p[static_cast<int64_t>(t.user) * W.si + f * W.st],
                                       H.p[static_cast<int64_t>(t.item) * H.si + f * H.st]));
        const double e = static_cast<double>(t.rating) - static_cast<double>(s);
        v += e * e;
    }
    v = block_sum(v, sm);
    if (threadIdx.x == 0) part[blockIdx.x] = v;
}

constexpr int kStage1Blocks = 1024;

}  // namespace

void launch_unit_loss(const DevSweep& L, const float* A, int32_t row_off, FactorView W, FactorView H,
                      int k, double* unit_loss, cudaStream_t stream) {
    if (L.n_units == 0) return;
    const int threads = 256;
    const int blocks =
        static_cast<int>(std::min<int64_t>((static_cast<int64_t>(L.n_units) * 32 + threads - 1) / threads, 8192));
    const bool vec = W.st == 1 && H.st == 1 && k % 4 == 0 && W.si == k && H.si == k &&
                     (reinterpret_cast<uintptr_t>(W.p) & 15) == 0 && (reinterpret_cast<uintptr_t>(H.p) & 15) == 0;
#define PMF_LOSS(I16, V)                                                                                        \
    unit_loss_kernel<I16, V><<<blocks, threads, 0, stream>>>(L.units, L.unit_panel, L.panel_base, L.idx, A, \
                                                             L.n_units, L.sentinel, row_off, W, H, k, unit_loss)
    if (L.idx16) {
        if (vec) PMF_LOSS(true, true);
        else PMF_LOSS(true, false);
    } else {
        if (vec) PMF_LOSS(false, true);
        else PMF_LOSS(false, false);
    }
#undef PMF_LOSS
}

void launch_sum(const double* x, int64_t n, double* scratch, double* out, cudaStream_t stream) {
    sum_stage1<<<kStage1Blocks, kRedThreads, 0, stream>>>(x, n, scratch);
    sum_stage2<<<1, kRedThreads, 0, stream>>>(scratch, kStage1Blocks, out);
}

void launch_sumsq(const float* x, int64_t n, double* scratch, double* out, cudaStream_t stream) {
    sumsq_stage1<<<kStage1Blocks, kRedThreads, 0, stream>>>(x, n, scratch);
    sum_stage2<<<1, kRedThreads, 0, stream>>>(scratch, kStage1Blocks, out);
}

void launch_probe_sse(const DevTriplet* probe, int64_t n, FactorView W, FactorView H, int k, double* scratch,
                      double* out, cudaStream_t stream) {
    probe_sse_kernel<<<kStage1Blocks, 256, 0, stream>>>(probe, n, W, H, k, scratch);
    sum_stage2<<<1, kRedThreads, 0, stream>>>(scratch, kStage1Blocks, out);
}

// 32 x 32 tiles through shared memory: reads of src rows (fixed t) and writes of dst rows coalesced.
__global__ void transpose_kernel(const float* __restrict__ src, int64_t ld, int k, int32_t count,
                                 float* __restrict__ dst) {
    __shared__ float tile[32][33];
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * 32;
    const int t0 = blockIdx.y * 32;
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int t = t0 + y;
        const int64_t i = i0 + threadIdx.x;
        if (t < k && i < count) tile[y][threadIdx.x] = src[static_cast<int64_t>(t) * ld + i];
    }
    __syncthreads();
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int64_t i = i0 + y;
        const int t = t0 + threadIdx.x;
        if (t < k && i < count) dst[i * k + t] = tile[threadIdx.x][y];
    }
}

void launch_transpose(const float* src, int64_t ld, int k, int32_t count, float* dst, cudaStream_t stream) {
    if (count <= 0 || k <= 0) return;
    const dim3 grid(static_cast<unsigned>((count + 31) / 32), static_cast<unsigned>((k + 31) / 32));
    transpose_kernel<<<grid, dim3(32, 8), 0, stream>>>(src, ld, k, count, dst);
}

}  // namespace pmfgpu
