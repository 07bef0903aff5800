// small_kernels.cu -- a whole CCD++ outer iteration (ccd.hpp:370-398) in ONE kernel for small matrices
// (BASELINE configs[0], the MovieLens-100K shape: 943 x 1682, 90K ratings).
//
// At that size a sweep is a few microseconds of work and the CUDA-graph schedule of the large shapes
// (2 T k sweeps = 300 kernels per iteration at k = 10) is bound by the launches.  Here one thread-block
// cluster (16 CTAs x 1024 threads) runs every rank-one step: the fused promote (deferred writeback of the
// previous step + build-rhat, ccd.hpp:133-151 / :199-218) in the first u / v sweep of the step, the T
// inner (u, v) sweeps, and the column writeback W[t] = u, H[t] = v, with a hardware cluster barrier
// (barrier.cluster, release / acquire) between dependent sweeps.  It reads the same sweep layouts as the
// graph path -- one gather panel per side, 16-bit indices, one unit per output -- and applies the same
// per-entry arithmetic (products rounded before the subtract / add, no FMA in the residual update, FMA
// sums), a warp per unit; the gathered vectors are read through L1 / L2 instead of shared-memory panels
// (the barrier's release / acquire orders them after the other CTAs' writes; L2-only loads measured
// 2.89 vs 1.55 ms per iteration: the sweep reuses each gathered value many times).
// Both residual copies are therefore updated identically (bitwise equal, as on the graph path); the
// num / den sums use a different (fixed) order, so u, v agree with the graph path to FP32 rounding.
#include <cuda_runtime.h>

#include <cstdint>

#include "device.hpp"

namespace pmfgpu {

namespace {

constexpr int kSmallThreads = 1024;

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

struct SmallSide {
    const Unit* units;
    const uint16_t* idx;
    float* R;
    int32_t n_units, sent;  // sentinel index of padding entries (= the panel width)
};

// One sweep over a side's units, a warp per unit (4-entry vectors per lane).  PROMOTE: the first sweep of
// a step, R <- (R - oa_o ga_g) then + w h if w != 0 (CSR: w = ob_o, h = gb_g; CSC: w = gb_g, h = ob_o).
template <bool PROMOTE, bool CSR>
__device__ __forceinline__ void small_sweep(const SmallSide& S, const float* __restrict__ ga, const float* __restrict__ gb,
                                            const float* __restrict__ gn, const float* __restrict__ oa,
                                            const float* __restrict__ ob, float* __restrict__ out, float lambda) {
    // a warp per unit (a half-warp per unit measured no faster: 1.61 vs 1.55 ms per ML-100K iteration)
    constexpr int G = 32;
    const int lane = threadIdx.x & (G - 1);
    const int gw = (blockIdx.x * kSmallThreads + threadIdx.x) / G;
    const int nw = gridDim.x * kSmallThreads / G;
    const int ng = (S.n_units + nw - 1) / nw;  // uniform trip count per warp (shuffles below are warp-wide)
    for (int it = 0; it < ng; ++it) {
        const int u = gw + it * nw;
        const bool live = u < S.n_units;
        const Unit U = live ? S.units[u] : Unit{0u, 0, 0, -1};
        const float a_o = PROMOTE ? oa[U.o] : 0.f;
        const float b_o = PROMOTE ? ob[U.o] : 0.f;
        float num = 0.f, den = 0.f;
        for (int v = lane; 4 * v < U.len; v += G) {
            const int64_t e = static_cast<int64_t>(U.e0) + 4 * v;
            float4 r4 = *reinterpret_cast<const float4*>(S.R + e);
            const uint2 ix = *reinterpret_cast<const uint2*>(S.idx + e);
            float rv[4] = {r4.x, r4.y, r4.z, r4.w};
            const int gi[4] = {static_cast<int>(ix.x & 0xffffu), static_cast<int>(ix.x >> 16),
                               static_cast<int>(ix.y & 0xffffu), static_cast<int>(ix.y >> 16)};
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const bool pad = gi[c] == S.sent;
                float r = rv[c];
                if (PROMOTE) {
                    const float a = pad ? 0.f : ga[gi[c]];
                    const float b = pad ? 0.f : gb[gi[c]];
                    r = __fsub_rn(r, __fmul_rn(a_o, a));
                    const float w = CSR ? b_o : b;
                    const float h = CSR ? b : b_o;
                    if (w != 0.f) r = __fadd_rn(r, __fmul_rn(w, h));
                    rv[c] = r;
                }
                const float g = pad ? 0.f : gn[gi[c]];
                num = fmaf(r, g, num);
                den = fmaf(g, g, den);
            }
            if (PROMOTE) *reinterpret_cast<float4*>(S.R + e) = make_float4(rv[0], rv[1], rv[2], rv[3]);
        }
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) {
            num += __shfl_xor_sync(0xffffffffu, num, off);
            den += __shfl_xor_sync(0xffffffffu, den, off);
        }
        if (lane == 0 && live) {
            const float dt = __fadd_rn(lambda, den);
            out[U.o] = dt == 0.f ? 0.f : __fdiv_rn(num, dt);
        }
    }
}

// W, H column-major (k x ldm / k x ldn); u, v the step's working vectors.
__global__ void __launch_bounds__(kSmallThreads, 1)
small_ccdpp_kernel(SmallSide csr, SmallSide csc, float* __restrict__ W, float* __restrict__ H, float* __restrict__ ub,
                   float* __restrict__ vb, int64_t ldm, int64_t ldn, int32_t m, int32_t n, int k, int inner,
                   float lambda) {
    for (int t = 0; t < k; ++t) {
        const int tp = (t + k - 1) % k;
        float* Wt = W + static_cast<int64_t>(t) * ldm;
        float* Ht = H + static_cast<int64_t>(t) * ldn;
        const float* Wp = W + static_cast<int64_t>(tp) * ldm;
        const float* Hp = H + static_cast<int64_t>(tp) * ldn;
        for (int s = 0; s < inner; ++s) {
            // u-sweep over CSR (gathered: v' = H[tp], h = H[t], v; per output: u' = W[tp], w = W[t])
            if (s == 0) small_sweep<true, true>(csr, Hp, Ht, Ht, Wp, Wt, ub, lambda);
            else small_sweep<false, true>(csr, nullptr, nullptr, vb, nullptr, nullptr, ub, lambda);
            cluster_sync_all();
            // v-sweep over CSC (gathered: u' = W[tp], w = W[t], u; per output: v' = H[tp], h = H[t])
            if (s == 0) small_sweep<true, false>(csc, Wp, Wt, ub, Hp, Ht, vb, lambda);
            else small_sweep<false, false>(csc, nullptr, nullptr, ub, nullptr, nullptr, vb, lambda);
            cluster_sync_all();
        }
        // writeback of the column pair (ccd.hpp:209, :226); the residual part is deferred to the next step
        const int64_t tid = static_cast<int64_t>(blockIdx.x) * kSmallThreads + threadIdx.x;
        const int64_t nt = static_cast<int64_t>(gridDim.x) * kSmallThreads;
        for (int64_t i = tid; i < m; i += nt) Wt[i] = ub[i];
        for (int64_t j = tid; j < n; j += nt) Ht[j] = vb[j];
        cluster_sync_all();
    }
}

}  // namespace

bool small_ccdpp_eligible(const DevSweep& csr, const DevSweep& csc, int64_t nnz) {
    auto ok = [](const DevSweep& L) {
        return L.smem && L.idx16 && !L.flat && L.n_panels == 1 && L.n_mo == 0 && L.n_slots == 0;
    };
    return nnz <= (int64_t(1) << 18) && ok(csr) && ok(csc);
}

cudaError_t launch_small_ccdpp(const DevSweep& csr, const DevSweep& csc, float* W, float* H, float* ub, float* vb,
                               int64_t ldm, int64_t ldn, int32_t m, int32_t n, int k, int inner, float lambda,
                               cudaStream_t s) {
    static const bool attr = [] {
        return cudaFuncSetAttribute(small_ccdpp_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
               cudaSuccess;
    }();
    SmallSide a{csr.units, static_cast<const uint16_t*>(csr.idx), csr.R, csr.n_units, csr.sentinel};
    SmallSide b{csc.units, static_cast<const uint16_t*>(csc.idx), csc.R, csc.n_units, csc.sentinel};
    cudaError_t err = cudaErrorUnknown;
    for (int cl : {16, 8}) {
        if (cl > 8 && !attr) continue;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(cl);
        cfg.blockDim = dim3(kSmallThreads);
        cfg.dynamicSmemBytes = 0;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cl;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        err = cudaLaunchKernelEx(&cfg, small_ccdpp_kernel, a, b, W, H, ub, vb, ldm, ldn, m, n, k, inner, lambda);
        if (err == cudaSuccess) break;
        (void)cudaGetLastError();
    }
    return err;
}

}  // namespace pmfgpu
