// ccd_kernels.cu -- CCD++ rank-one sweeps for sm_100a.
//
// One persistent CTA per SM walks its pieces (contiguous unit runs inside one gather panel,
// layout.cpp).  Per piece it stages the panel's slice of the gather vectors (v, or u, plus the
// promote/demote factors) into shared memory, then its warps pull work units from a shared
// counter.  A warp streams its unit with 128-bit loads (4 residual values + 4 panel-local indices
// per lane per step), gathers the factor values from shared memory and accumulates
// num = sum R*g and den = sum g*g (ccd.hpp:165-171 / :188-194) in FP32, then reduces with a
// fixed xor-shuffle tree.  On the first inner sweep of a rank-one step (kPromote) the residual is
// rewritten in the same pass:  R <- (R - u'_i v'_j) [deferred writeback of the previous step,
// ccd.hpp:213-214] then, if w_i != 0, R <- R + w_i h_j [build-rhat, ccd.hpp:142-147], each product
// rounded before the add exactly like the reference (no FMA contraction), so the CSR and CSC
// copies stay bitwise equal without the reference's cross-link mirror (sparse.hpp:241-250).
#include <cuda_runtime.h>

#include <algorithm>

#include <cstdint>

#include "device.hpp"

namespace pmfgpu {

namespace {

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;

template <bool IDX16>
struct IdxVec;
template <>
struct IdxVec<true> {
    __device__ __forceinline__ static void load(const void* base, int64_t e, int (&g)[4]) {
        const uint2 raw = __ldcs(reinterpret_cast<const uint2*>(static_cast<const uint16_t*>(base) + e));
        g[0] = raw.x & 0xffffu;
        g[1] = raw.x >> 16;
        g[2] = raw.y & 0xffffu;
        g[3] = raw.y >> 16;
    }
};
template <>
struct IdxVec<false> {
    __device__ __forceinline__ static void load(const void* base, int64_t e, int (&g)[4]) {
        const int4 raw = __ldcs(reinterpret_cast<const int4*>(static_cast<const int32_t*>(base) + e));
        g[0] = raw.x;
        g[1] = raw.y;
        g[2] = raw.z;
        g[3] = raw.w;
    }
};

template <int MODE, bool CSR, bool SMEM>
struct Gather {
    // number of staged arrays
    static constexpr int kArrays = MODE == kPlain ? 1 : MODE == kDemote ? 1 : (CSR ? 2 : 3);
};

template <int MODE, bool CSR, bool IDX16, bool SMEM>
__global__ void __launch_bounds__(kThreads, 1)
sweep_kernel(const Unit* __restrict__ units, const Piece* __restrict__ pieces,
             const int32_t* __restrict__ piece_start, const int32_t* __restrict__ panel_base,
             const void* __restrict__ idx, float* __restrict__ R, float2* __restrict__ partial,
             SweepOperands op, int32_t panel_size) {
    extern __shared__ float smem[];
    __shared__ int s_next;
    constexpr int A = Gather<MODE, CSR, SMEM>::kArrays;
    const int stride = panel_size + 1;
    // staged array roles: plain: s0 = gn;  promote CSR: s0 = ga, s1 = gb (gn == gb);
    // promote CSC: s0 = ga, s1 = gb, s2 = gn;  demote: s0 = ga.
    float* s0 = smem;
    float* s1 = smem + stride;
    float* s2 = smem + 2 * stride;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;

    const int pb = piece_start[blockIdx.x], pe = piece_start[blockIdx.x + 1];
    for (int pc = pb; pc < pe; ++pc) {
        const Piece pz = pieces[pc];
        int32_t gbase = 0;
        __syncthreads();
        if (SMEM) {
            gbase = panel_base[pz.panel];
            const int len = panel_base[pz.panel + 1] - gbase;
            const float* src0 = MODE == kPlain ? op.gn : op.ga;
            for (int x = threadIdx.x; x < len; x += kThreads) {
                s0[x] = __ldg(src0 + gbase + x);
                if (A >= 2) s1[x] = __ldg(op.gb + gbase + x);
                if (A >= 3) s2[x] = __ldg(op.gn + gbase + x);
            }
            if (threadIdx.x == 0) {
                s0[panel_size] = 0.f;
                if (A >= 2) s1[panel_size] = 0.f;
                if (A >= 3) s2[panel_size] = 0.f;
            }
        }
        if (threadIdx.x == 0) s_next = pz.ub;
        __syncthreads();
        const float* g0 = SMEM ? s0 : (MODE == kPlain ? op.gn : op.ga);
        const float* g1 = SMEM ? s1 : op.gb;
        const float* g2 = SMEM ? s2 : op.gn;
        for (;;) {
            int u = 0;
            if (lane == 0) u = atomicAdd(&s_next, 1);
            u = __shfl_sync(0xffffffffu, u, 0);
            if (u >= pz.ue) break;
            const Unit U = units[u];
            const int32_t oidx = op.out_off + U.o;
            float oa = 0.f, ob = 0.f;
            if (MODE != kPlain) oa = __ldg(op.oa + oidx);
            if (MODE == kPromote) ob = __ldg(op.ob + oidx);
            float num = 0.f, den = 0.f;
            const int64_t end = static_cast<int64_t>(U.e0) + U.len;
            for (int64_t e = static_cast<int64_t>(U.e0) + 4 * lane; e < end; e += 256) {
                const bool two = e + 128 < end;
                float4 ra, rb;
                int ia[4], ib[4];
                ra = __ldcs(reinterpret_cast<const float4*>(R + e));
                IdxVec<IDX16>::load(idx, e, ia);
                if (two) {
                    rb = __ldcs(reinterpret_cast<const float4*>(R + e + 128));
                    IdxVec<IDX16>::load(idx, e + 128, ib);
                }
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    if (half == 1 && !two) break;
                    float4& r4 = half == 0 ? ra : rb;
                    const int(&gi)[4] = half == 0 ? ia : ib;
                    float rv[4] = {r4.x, r4.y, r4.z, r4.w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int g = gi[q];
                        float r = rv[q];
                        if (MODE == kPlain) {
                            const float gv = g0[g];
                            num = fmaf(r, gv, num);
                            den = fmaf(gv, gv, den);
                        } else if (MODE == kDemote) {
                            r = __fsub_rn(r, __fmul_rn(oa, g0[g]));
                        } else {
                            const float a = g0[g];
                            const float b = g1[g];
                            // deferred writeback of the previous step: R - u'_i v'_j
                            r = __fsub_rn(r, __fmul_rn(oa, a));
                            // build-rhat: skip when w_i == 0 (ccd.hpp:142)
                            const float w = CSR ? ob : b;
                            const float h = CSR ? b : ob;
                            if (w != 0.f) r = __fadd_rn(r, __fmul_rn(w, h));
                            const float gv = CSR ? b : g2[g];
                            num = fmaf(r, gv, num);
                            den = fmaf(gv, gv, den);
                        }
                        rv[q] = r;
                    }
                    if (MODE != kPlain) {
                        float4 w4 = make_float4(rv[0], rv[1], rv[2], rv[3]);
                        __stcs(reinterpret_cast<float4*>(R + e + 128 * half), w4);
                    }
                }
            }
            if (MODE == kDemote) continue;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                num += __shfl_xor_sync(0xffffffffu, num, off);
                den += __shfl_xor_sync(0xffffffffu, den, off);
            }
            if (lane == 0) {
                if (U.slot < 0) {
                    const float dt = __fadd_rn(op.lambda, den);
                    op.out[oidx] = dt == 0.f ? 0.f : __fdiv_rn(num, dt);
                } else {
                    partial[U.slot] = make_float2(num, den);
                }
            }
        }
    }
}

// Fixed-order combination of the partial sums of outputs with several (or zero) units.
__global__ void finalize_kernel(const int32_t* __restrict__ mo_out, const int32_t* __restrict__ mo_start,
                                int32_t n_mo, const float2* __restrict__ partial, float* __restrict__ out,
                                int32_t out_off, float lambda) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t q = wid; q < n_mo; q += nw) {
        const int s0 = mo_start[q], s1 = mo_start[q + 1];
        float num = 0.f, den = 0.f;
        for (int s = s0 + lane; s < s1; s += 32) {
            const float2 p = partial[s];
            num += p.x;
            den += p.y;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            num += __shfl_xor_sync(0xffffffffu, num, off);
            den += __shfl_xor_sync(0xffffffffu, den, off);
        }
        if (lane == 0) {
            const float dt = __fadd_rn(lambda, den);
            out[out_off + mo_out[q]] = dt == 0.f ? 0.f : __fdiv_rn(num, dt);
        }
    }
}

template <int MODE, bool CSR, bool IDX16, bool SMEM>
void launch_one(const DevSweep& L, const SweepOperands& op, size_t smem, cudaStream_t s) {
    sweep_kernel<MODE, CSR, IDX16, SMEM><<<L.ctas, kThreads, smem, s>>>(
        L.units, L.pieces, L.piece_start, L.panel_base, L.idx, L.R, L.partial, op, L.panel_size);
}

template <int MODE, bool CSR>
void dispatch_idx(const DevSweep& L, const SweepOperands& op, size_t smem, cudaStream_t s) {
    if (L.idx16) {
        if (L.smem) launch_one<MODE, CSR, true, true>(L, op, smem, s);
        else launch_one<MODE, CSR, true, false>(L, op, smem, s);
    } else {
        if (L.smem) launch_one<MODE, CSR, false, true>(L, op, smem, s);
        else launch_one<MODE, CSR, false, false>(L, op, smem, s);
    }
}

template <int MODE, bool CSR, bool IDX16, bool SMEM>
void set_attr(size_t max_smem) {
    cudaFuncSetAttribute(sweep_kernel<MODE, CSR, IDX16, SMEM>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(max_smem));
}

template <int MODE, bool CSR>
void set_attr_all(size_t max_smem) {
    set_attr<MODE, CSR, true, true>(max_smem);
    set_attr<MODE, CSR, true, false>(max_smem);
    set_attr<MODE, CSR, false, true>(max_smem);
    set_attr<MODE, CSR, false, false>(max_smem);
}

}  // namespace

size_t sweep_smem_bytes(const DevSweep& L, SweepMode mode, bool csr_side) {
    if (!L.smem) return 0;
    const int arrays = mode == kPromote ? (csr_side ? 2 : 3) : 1;
    return static_cast<size_t>(arrays) * (L.panel_size + 1) * sizeof(float);
}

void sweep_set_attributes(size_t max_smem) {
    set_attr_all<kPlain, true>(max_smem);
    set_attr_all<kPlain, false>(max_smem);
    set_attr_all<kPromote, true>(max_smem);
    set_attr_all<kPromote, false>(max_smem);
    set_attr_all<kDemote, true>(max_smem);
    set_attr_all<kDemote, false>(max_smem);
}

int launch_sweep(const DevSweep& L, SweepMode mode, bool csr_side, const SweepOperands& op,
                 cudaStream_t stream) {
    const size_t smem = sweep_smem_bytes(L, mode, csr_side);
    int launched = 0;
    if (L.n_units > 0) {
        if (mode == kPlain) {
            if (csr_side) dispatch_idx<kPlain, true>(L, op, smem, stream);
            else dispatch_idx<kPlain, false>(L, op, smem, stream);
        } else if (mode == kPromote) {
            if (csr_side) dispatch_idx<kPromote, true>(L, op, smem, stream);
            else dispatch_idx<kPromote, false>(L, op, smem, stream);
        } else {
            if (csr_side) dispatch_idx<kDemote, true>(L, op, smem, stream);
            else dispatch_idx<kDemote, false>(L, op, smem, stream);
        }
        ++launched;
    }
    if (mode != kDemote && L.n_mo > 0) {
        const int threads = 256;
        const int64_t warps = L.n_mo;
        const int blocks = static_cast<int>(std::min<int64_t>((warps * 32 + threads - 1) / threads, 4096));
        finalize_kernel<<<blocks, threads, 0, stream>>>(L.mo_out, L.mo_start, L.n_mo, L.partial, op.out,
                                                        op.out_off, op.lambda);
        ++launched;
    }
    return launched;
}

}  // namespace pmfgpu
