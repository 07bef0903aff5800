// small_kernels.cu -- a whole CCD++ outer iteration (ccd.hpp:370-398) in ONE kernel for small matrices
// (BASELINE configs[0], the MovieLens-100K shape: 943 x 1682, 90K ratings).
//
// At that size a sweep is a few microseconds of work and the CUDA-graph schedule of the large shapes
// (2 T k sweeps = 300 kernels per iteration at k = 10) is bound by the launches.  Here one thread-block
// cluster (16 CTAs x 1024 threads) runs every rank-one step: the fused promote (deferred writeback of the
// previous step + build-rhat, ccd.hpp:133-151 / :199-218) in the first u / v sweep of the step, the T
// inner (u, v) sweeps, and the column writeback W[t] = u, H[t] = v, with a hardware cluster barrier
// (barrier.cluster, release / acquire) between dependent sweeps.
//
// Everything a sweep touches is in shared memory: each CTA owns a contiguous run of units on each side
// (the layout's own CTA pieces, grouped) and keeps their residual and 16-bit indices resident for the
// whole iteration; every CTA holds full copies of u, v and the step's factor columns W[t], W[t-1],
// H[t], H[t-1].  A unit's result is stored into all 16 CTAs' copy of u (or v) over distributed shared
// memory (st.shared::cluster, one lane per CTA), so after the barrier every gather is a local
// shared-memory read.  Per entry the arithmetic is the graph path's (products rounded before the
// subtract / add, no FMA in the residual update, FMA sums; 8 lanes per unit, 4-entry vectors per lane,
// xor-shuffle sums), so both residual copies stay bitwise equal; u, v agree with the graph path to
// FP32 rounding (the graph path sums a unit's entries in a different fixed order).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "device.hpp"

namespace pmfgpu {

namespace {

constexpr int kSmallThreads = 1024;
constexpr int kSmallCtas = 16;
constexpr int kSmallSmemMax = 200 * 1024;
// lanes per unit (4 units per warp at once): ML-100K 0.83 ms per iteration with 8, 1.11 with 4, 1.01 with
// 16, 1.51 with 32 (scripts/small_timing.py; the sweeps are issue-bound, shorter reductions win)
#ifndef PMF_SMALL_G
#define PMF_SMALL_G 8
#endif
constexpr int kSmallG = PMF_SMALL_G;

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void dsmem_st(const float* local, uint32_t rank, float v) {
    uint32_t a;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(local))), "r"(rank));
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}

// One side's share of CTA c: units [u0[c], u0[c + 1]), their entries inside [e0[c], e0[c] + elen[c]).
struct SmallSide {
    const Unit* units;
    const uint16_t* idx;
    float* R;
    int32_t sent;  // sentinel index of padding entries (= the panel width)
    int32_t u0[kSmallCtas + 1];
    int64_t e0[kSmallCtas];
    int32_t elen[kSmallCtas];
};

// One sweep over the CTA's units of a side, G lanes per unit (4-entry vectors per lane); Rs / Is: the
// CTA's resident residual / indices (entry e at e - ebase).  PROMOTE: the first sweep of a step,
// R <- (R - oa_o ga_g) then + w h if w != 0 (CSR: w = ob_o, h = gb_g; CSC: w = gb_g, h = ob_o).
// The result of output o goes to out[o] in every CTA of the cluster.
template <bool PROMOTE, bool CSR, int G>
__device__ __forceinline__ void small_sweep(const SmallSide& S, int c, const Unit* Us, float* Rs, const uint16_t* Is,
                                            const float* ga, const float* gb, const float* gn, const float* oa,
                                            const float* ob, float* out, float lambda) {
    constexpr int PER_WARP = 32 / G;  // units a warp works on together (a group of G lanes each)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int l = lane % G, grp = lane / G;
    const int nu = S.u0[c + 1] - S.u0[c];
    const int64_t ebase = S.e0[c];
    for (int u0 = warp * PER_WARP; u0 < nu; u0 += 32 * PER_WARP) {  // warp-uniform trip count
        const int u = u0 + grp;
        const bool live = u < nu;
        const Unit U = live ? Us[u] : Unit{0u, 0, 0, -1};
        const float a_o = PROMOTE && live ? oa[U.o] : 0.f;
        const float b_o = PROMOTE && live ? ob[U.o] : 0.f;
        float num = 0.f, den = 0.f;
        for (int v = l; 4 * v < U.len; v += G) {
            const int64_t e = static_cast<int64_t>(U.e0) + 4 * v - ebase;
            float4 r4 = *reinterpret_cast<const float4*>(Rs + e);
            const uint2 ix = *reinterpret_cast<const uint2*>(Is + e);
            float rv[4] = {r4.x, r4.y, r4.z, r4.w};
            const int gi[4] = {static_cast<int>(ix.x & 0xffffu), static_cast<int>(ix.x >> 16),
                               static_cast<int>(ix.y & 0xffffu), static_cast<int>(ix.y >> 16)};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const bool pad = gi[q] == S.sent;
                float r = rv[q];
                if (PROMOTE) {
                    const float a = pad ? 0.f : ga[gi[q]];
                    const float b = pad ? 0.f : gb[gi[q]];
                    r = __fsub_rn(r, __fmul_rn(a_o, a));
                    const float w = CSR ? b_o : b;
                    const float h = CSR ? b : b_o;
                    if (w != 0.f) r = __fadd_rn(r, __fmul_rn(w, h));
                    rv[q] = r;
                }
                const float g = pad ? 0.f : gn[gi[q]];
                num = fmaf(r, g, num);
                den = fmaf(g, g, den);
            }
            if (PROMOTE) *reinterpret_cast<float4*>(Rs + e) = make_float4(rv[0], rv[1], rv[2], rv[3]);
        }
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) {
            num += __shfl_xor_sync(0xffffffffu, num, off);
            den += __shfl_xor_sync(0xffffffffu, den, off);
        }
        if (live) {
            const float dt = __fadd_rn(lambda, den);
            const float z = dt == 0.f ? 0.f : __fdiv_rn(num, dt);
            for (int r = l; r < kSmallCtas; r += G) dsmem_st(out + U.o, r, z);
        }
    }
}

// resident residual / indices of a side: global <-> shared (16-byte vectors; ranges start on 4 entries)
__device__ __forceinline__ void side_load(const SmallSide& S, int c, float* Rs, uint16_t* Is) {
    const int64_t b = S.e0[c];
    const int n4 = S.elen[c] / 4;
    for (int v = threadIdx.x; v < n4; v += kSmallThreads) {
        reinterpret_cast<float4*>(Rs)[v] = reinterpret_cast<const float4*>(S.R + b)[v];
        reinterpret_cast<uint2*>(Is)[v] = reinterpret_cast<const uint2*>(S.idx + b)[v];
    }
}
__device__ __forceinline__ void side_store(const SmallSide& S, int c, const float* Rs) {
    const int64_t b = S.e0[c];
    const int n4 = S.elen[c] / 4;
    for (int v = threadIdx.x; v < n4; v += kSmallThreads)
        reinterpret_cast<float4*>(S.R + b)[v] = reinterpret_cast<const float4*>(Rs)[v];
}

// W, H column-major (k x ldm / k x ldn); ub, vb: the working vectors' global copies.  Shared memory:
// u[m+1], v[n+1], W[t], W[t-1] (m+1 each), H[t], H[t-1] (n+1 each), the two sides' resident residual
// runs, their unit descriptors, and their index runs.
__global__ void __launch_bounds__(kSmallThreads, 1)
small_ccdpp_kernel(const __grid_constant__ SmallSide csr, const __grid_constant__ SmallSide csc, float* __restrict__ W,
                   float* __restrict__ H, float* __restrict__ ub, float* __restrict__ vb, int64_t ldm, int64_t ldn,
                   int32_t m, int32_t n, int k, int inner, float lambda, int32_t rlen_csr, int32_t ulen_csr) {
    extern __shared__ __align__(16) float sm[];
    const int c = static_cast<int>(cluster_rank());
    const int mp = (m + 1 + 3) & ~3, np = (n + 1 + 3) & ~3;
    float* su = sm;
    float* sv = su + mp;
    float* swt = sv + np;
    float* swp = swt + mp;
    float* sht = swp + mp;
    float* shp = sht + np;
    float* Rr = shp + np;                 // CSR run
    float* Rc = Rr + rlen_csr;            // CSC run
    const int32_t rlen_csc = (csc.elen[c] + 3) & ~3;
    Unit* Ur = reinterpret_cast<Unit*>(Rc + rlen_csc);  // the CTA's unit descriptors (16-byte aligned)
    Unit* Uc = Ur + ulen_csr;
    uint16_t* Ir = reinterpret_cast<uint16_t*>(Uc + (csc.u0[c + 1] - csc.u0[c]));
    uint16_t* Ic = Ir + rlen_csr;
    side_load(csr, c, Rr, Ir);
    side_load(csc, c, Rc, Ic);
    for (int u = threadIdx.x; u < csr.u0[c + 1] - csr.u0[c]; u += kSmallThreads) Ur[u] = csr.units[csr.u0[c] + u];
    for (int u = threadIdx.x; u < csc.u0[c + 1] - csc.u0[c]; u += kSmallThreads) Uc[u] = csc.units[csc.u0[c] + u];
    const int tid = threadIdx.x;
    const int64_t ms = (static_cast<int64_t>(m) + kSmallCtas - 1) / kSmallCtas, ns = (static_cast<int64_t>(n) + kSmallCtas - 1) / kSmallCtas;
    for (int t = 0; t < k; ++t) {
        const int tp = (t + k - 1) % k;
        const float* Wt = W + static_cast<int64_t>(t) * ldm;
        const float* Ht = H + static_cast<int64_t>(t) * ldn;
        const float* Wp = W + static_cast<int64_t>(tp) * ldm;
        const float* Hp = H + static_cast<int64_t>(tp) * ldn;
        for (int i = tid; i < m; i += kSmallThreads) {
            swt[i] = Wt[i];
            swp[i] = Wp[i];
        }
        for (int j = tid; j < n; j += kSmallThreads) {
            sht[j] = Ht[j];
            shp[j] = Hp[j];
        }
        __syncthreads();
        for (int s = 0; s < inner; ++s) {
            // u-sweep over CSR (gathered: v' = H[tp], h = H[t], v; per output: u' = W[tp], w = W[t])
            if (s == 0) small_sweep<true, true, kSmallG>(csr, c, Ur, Rr, Ir, shp, sht, sht, swp, swt, su, lambda);
            else small_sweep<false, true, kSmallG>(csr, c, Ur, Rr, Ir, nullptr, nullptr, sv, nullptr, nullptr, su, lambda);
            cluster_sync_all();
            // v-sweep over CSC (gathered: u' = W[tp], w = W[t], u; per output: v' = H[tp], h = H[t])
            if (s == 0) small_sweep<true, false, kSmallG>(csc, c, Uc, Rc, Ic, swp, swt, su, shp, sht, sv, lambda);
            else small_sweep<false, false, kSmallG>(csc, c, Uc, Rc, Ic, nullptr, nullptr, su, nullptr, nullptr, sv, lambda);
            cluster_sync_all();
        }
        // writeback of the column pair (ccd.hpp:209, :226), a slice per CTA; the residual part is deferred
        // to the next step's promote
        for (int64_t i = c * ms + tid; i < min(static_cast<int64_t>(m), (c + 1) * ms); i += kSmallThreads) {
            W[static_cast<int64_t>(t) * ldm + i] = su[i];
            ub[i] = su[i];
        }
        for (int64_t j = c * ns + tid; j < min(static_cast<int64_t>(n), (c + 1) * ns); j += kSmallThreads) {
            H[static_cast<int64_t>(t) * ldn + j] = sv[j];
            vb[j] = sv[j];
        }
        cluster_sync_all();  // the next step's staging reads these columns
    }
    side_store(csr, c, Rr);
    side_store(csc, c, Rc);
}

bool small_shape_ok(const DevSweep& L) {
    return L.smem && L.idx16 && !L.flat && L.n_panels == 1 && L.n_mo == 0 && L.n_slots == 0;
}

// CTA c of the cluster takes the layout's CTAs [c * ctas / 16, (c + 1) * ctas / 16): their pieces are a
// contiguous unit range whose entries are a contiguous run of the side's streams.
bool small_partition(const DevSweep& D, const SweepLayout& L, SmallSide* S) {
    S->units = D.units;
    S->idx = static_cast<const uint16_t*>(D.idx);
    S->R = D.R;
    S->sent = D.sentinel;
    const int ctas = static_cast<int>(L.piece_start.size()) - 1;
    for (int c = 0; c <= kSmallCtas; ++c) {
        const int lc = static_cast<int>(static_cast<int64_t>(c) * ctas / kSmallCtas);
        const int p = L.piece_start[lc];
        S->u0[c] = p < static_cast<int>(L.pieces.size()) ? L.pieces[p].ub : static_cast<int32_t>(L.units.size());
    }
    S->u0[kSmallCtas] = static_cast<int32_t>(L.units.size());
    for (int c = 0; c < kSmallCtas; ++c) {
        int64_t lo = INT64_MAX, hi = 0;
        for (int u = S->u0[c]; u < S->u0[c + 1]; ++u) {
            lo = std::min<int64_t>(lo, L.units[u].e0);
            hi = std::max<int64_t>(hi, static_cast<int64_t>(L.units[u].e0) + L.units[u].len);
        }
        if (lo > hi) lo = hi = 0;
        if ((lo & 3) || (hi & 3)) return false;
        S->e0[c] = lo;
        S->elen[c] = static_cast<int32_t>(hi - lo);
    }
    return true;
}

size_t small_smem_bytes(int32_t m, int32_t n, int32_t rlen_csr, int32_t rlen_csc, int32_t ulen_csr, int32_t ulen_csc) {
    const int64_t mp = (m + 1 + 3) & ~3, np = (n + 1 + 3) & ~3;
    return sizeof(float) * static_cast<size_t>(3 * mp + 3 * np + rlen_csr + rlen_csc) +
           sizeof(Unit) * static_cast<size_t>(ulen_csr + ulen_csc) + sizeof(uint16_t) * static_cast<size_t>(rlen_csr + rlen_csc);
}

struct SmallPlan {
    SmallSide a, b;
    int32_t rlen_csr = 0, rlen_csc = 0, ulen_csr = 0, ulen_csc = 0;
    size_t smem = 0;
    bool ok = false;
};

SmallPlan small_plan(const DevSweep& csr, const DevSweep& csc, const SweepLayout& hcsr, const SweepLayout& hcsc,
                     int32_t m, int32_t n) {
    SmallPlan P;
    if (!small_shape_ok(csr) || !small_shape_ok(csc)) return P;
    if (!small_partition(csr, hcsr, &P.a) || !small_partition(csc, hcsc, &P.b)) return P;
    int32_t la = 0, lb = 0;
    for (int c = 0; c < kSmallCtas; ++c) {
        la = std::max(la, P.a.elen[c]);
        lb = std::max(lb, P.b.elen[c]);
        P.ulen_csr = std::max(P.ulen_csr, P.a.u0[c + 1] - P.a.u0[c]);
        P.ulen_csc = std::max(P.ulen_csc, P.b.u0[c + 1] - P.b.u0[c]);
    }
    // every CTA carves the same CSR run size (the CSC run follows it); runs are multiples of 4 entries
    P.rlen_csr = (la + 3) & ~3;
    P.rlen_csc = (lb + 3) & ~3;
    P.smem = small_smem_bytes(m, n, P.rlen_csr, P.rlen_csc, P.ulen_csr, P.ulen_csc);
    P.ok = P.smem <= static_cast<size_t>(kSmallSmemMax);
    return P;
}

bool small_attr_ok() {
    static const bool ok = cudaFuncSetAttribute(small_ccdpp_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed,
                                                1) == cudaSuccess &&
                           cudaFuncSetAttribute(small_ccdpp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                kSmallSmemMax) == cudaSuccess;
    if (!ok) (void)cudaGetLastError();
    return ok;
}

}  // namespace

bool small_ccdpp_eligible(const DevSweep& csr, const DevSweep& csc, const SweepLayout& hcsr, const SweepLayout& hcsc,
                          int32_t m, int32_t n) {
    return small_attr_ok() && small_plan(csr, csc, hcsr, hcsc, m, n).ok;
}

cudaError_t launch_small_ccdpp(const DevSweep& csr, const DevSweep& csc, const SweepLayout& hcsr,
                               const SweepLayout& hcsc, float* W, float* H, float* ub, float* vb, int64_t ldm,
                               int64_t ldn, int32_t m, int32_t n, int k, int inner, float lambda, cudaStream_t s) {
    const SmallPlan P = small_plan(csr, csc, hcsr, hcsc, m, n);
    if (!P.ok) return cudaErrorInvalidValue;
    if (!small_attr_ok()) return cudaErrorNotSupported;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(kSmallCtas);
    cfg.blockDim = dim3(kSmallThreads);
    cfg.dynamicSmemBytes = P.smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kSmallCtas;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, small_ccdpp_kernel, P.a, P.b, W, H, ub, vb, ldm, ldn, m, n, k, inner, lambda,
                              P.rlen_csr, P.ulen_csr);
}

}  // namespace pmfgpu
