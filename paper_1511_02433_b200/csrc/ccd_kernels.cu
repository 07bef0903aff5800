// ccd_kernels.cu -- CCD++ rank-one sweeps for sm_100a.
//
// One persistent CTA per SM walks its pieces (contiguous unit runs inside one gather panel,
// layout.cpp).  Per piece, one thread stages the panel's slice of the gather vectors (v, or u, plus
// the promote/demote factors) into shared memory with TMA bulk copies (cp.async.bulk completing on
// an mbarrier).  Warps then pull batches of 32/G work units from a shared counter; each group of G
// lanes owns one unit, so a warp works on 32/G units at once, converged.  Every lane keeps U
// independent 128-bit loads in flight (4 residual values + 4 panel-local indices each), gathers the
// factor values from shared memory and accumulates num = sum R*g and den = sum g*g
// (ccd.hpp:165-171 / :188-194) in FP32, then the group reduces with a fixed xor-shuffle tree.  The
// next batch's descriptors are fetched before the current batch is processed.
//
// On the first inner sweep of a rank-one step (kPromote) the residual is rewritten in the same pass:
// R <- (R - u'_i v'_j) [deferred writeback of the previous step, ccd.hpp:213-214] then, if w_i != 0,
// R <- R + w_i h_j [build-rhat, ccd.hpp:142-147]; each product is rounded before the add exactly like
// the reference (no FMA contraction), so the CSR and CSC copies stay bitwise equal without the
// reference's cross-link mirror (sparse.hpp:241-250).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "device.hpp"

namespace pmfgpu {

namespace {

constexpr int kDefaultPlainVariantCsr = 1;  // u-sweep: 1024 threads, unroll 4/2/2
constexpr int kDefaultPlainVariantCsc = 2;  // v-sweep: 1024 threads, unroll 2/2/2
#ifndef PMF_PROMOTE_VARIANT_CSR
#define PMF_PROMOTE_VARIANT_CSR 0
#endif
#ifndef PMF_PROMOTE_VARIANT_CSC
#define PMF_PROMOTE_VARIANT_CSC 0
#endif
constexpr int kDefaultPromoteVariantCsr = PMF_PROMOTE_VARIANT_CSR;  // 512 threads, unroll 8/4/4
constexpr int kDefaultPromoteVariantCsc = PMF_PROMOTE_VARIANT_CSC;

// Launch variants (threads per CTA, unroll of the long / medium / short length classes).  More
// resident warps keep more loads in flight (scripts/micro/stream_bw.cu: 8 warps/SM cap at ~4 TB/s,
// 16 at ~6.5, 32 at ~6.9); larger unrolls need more registers.  Round 1 also measured 768-thread
// CTAs, a software-pipelined plain sweep and larger short-class unrolls: all slower, removed.
template <int V>
struct Var;
template <>
struct Var<0> {
    static constexpr int NT = 512, UA = 8, UB = 4, UC = 4;
};
template <>
struct Var<1> {
    static constexpr int NT = 1024, UA = 4, UB = 2, UC = 2;
};
template <>
struct Var<2> {
    static constexpr int NT = 1024, UA = 2, UB = 2, UC = 2;
};
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(phase)
        : "memory");
}

// TMA bulk copy global -> shared, completion counted on `bar` (bytes multiple of 16, 16B aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

// Streaming loads of read-only data (indices always; the residual in plain sweeps): ld.global.cs.
// (ld.global.nc.L1::no_allocate measured slower in round 1: wide-panel v-sweep 188 -> 208 us.)
__device__ __forceinline__ float4 ld_stream(const float4* p) { return __ldcs(p); }
__device__ __forceinline__ uint2 ld_stream(const uint2* p) { return __ldcs(p); }
__device__ __forceinline__ int4 ld_stream(const int4* p) { return __ldcs(p); }

template <bool IDX16>
struct IdxVec;
template <>
struct IdxVec<true> {
    using raw_t = uint2;
    __device__ __forceinline__ static raw_t load(const void* base, int64_t e) {
        return ld_stream(reinterpret_cast<const uint2*>(static_cast<const uint16_t*>(base) + e));
    }
    __device__ __forceinline__ static int get(const raw_t& r, int q) {
        const uint32_t w = q < 2 ? r.x : r.y;
        return (q & 1) ? static_cast<int>(w >> 16) : static_cast<int>(w & 0xffffu);
    }
};
template <>
struct IdxVec<false> {
    using raw_t = int4;
    __device__ __forceinline__ static raw_t load(const void* base, int64_t e) {
        return ld_stream(reinterpret_cast<const int4*>(static_cast<const int32_t*>(base) + e));
    }
    __device__ __forceinline__ static int get(const raw_t& r, int q) {
        return q == 0 ? r.x : q == 1 ? r.y : q == 2 ? r.z : r.w;
    }
};

template <int MODE, bool CSR>
struct Roles {
    // staged arrays: plain: s0 = gn;  promote CSR: s0 = ga, s1 = gb (gn == gb);
    // promote CSC: s0 = gb, s1 = gn, and the demote's ga read through L1 (kGaL1): three staged vectors
    // (225 KB at Netflix panel widths) leave ~28 KB of L1 and put the sweep on the L1 cliff
    // (DESIGN.md 4); with two, the ~75 KB ga slice of a panel stays L1-resident;  demote: s0 = ga.
    static constexpr bool kGaL1 = MODE == kPromote && !CSR;
    static constexpr int kArrays = MODE == kPromote ? 2 : MODE == kRmw ? 2 : 1;
};

__host__ __device__ __forceinline__ int stage_stride(int panel_size) { return ((panel_size + 1) + 3) & ~3; }

// A thief restages its shared-memory panel only for a piece with at least this much work left
// (entries, estimated from the remaining long / medium / short units).
constexpr int kStealRestageMin = 16384;

// Processes units [ub, ue) of the current piece in warp batches of 32/G units, one unit per group
// of G lanes.  `counter` is the piece's shared counter for this length class.
template <int MODE, bool CSR, bool IDX16, int G, int kUnroll, bool GA_GLOBAL = false>
__device__ __noinline__ void run_class(int* counter, int32_t ub, int32_t ue, const Unit* __restrict__ units,
                                          const void* __restrict__ idx, float* __restrict__ R,
                                          float2* __restrict__ partial, const SweepOperands& op,
                                          const float* g0, const float* g1, const float* g2) {
    using IV = IdxVec<IDX16>;
    constexpr int B = 32 / G;  // units per warp batch
    const int lane = threadIdx.x & 31;
    const int g = lane / G;   // group within the warp
    const int gl = lane % G;  // lane within the group
    if (ub >= ue) return;
    // Batches are claimed two ahead: the claim for batch b+2 is issued while batch b starts and
    // consumed (shuffle + descriptor load) one batch later, so the counter's latency (a global
    // atomic when pieces are shared for stealing) never stalls the in-order warp.
    int a = 0, a1 = 0;
    if (lane == 0) a = atomicAdd(counter, B);
    int nb = __shfl_sync(0xffffffffu, a, 0);
    Unit Un = (nb + g < ue) ? units[nb + g] : Unit{0u, 0, 0, -2};
    if (lane == 0) a1 = atomicAdd(counter, B);
    while (nb < ue) {
        const Unit U = Un;
        int a2 = 0;
        if (lane == 0) a2 = atomicAdd(counter, B);
        // descriptors of the next batch (claimed one batch ago) while this one streams
        nb = __shfl_sync(0xffffffffu, a1, 0);
        a1 = a2;
        Un = (nb + g < ue) ? units[nb + g] : Unit{0u, 0, 0, -2};

        const int32_t oidx = op.out_off + U.o;
        float oa = 0.f, ob = 0.f;
        if (MODE != kPlain && U.len > 0) oa = __ldg(op.oa + oidx);
        if ((MODE == kPromote || MODE == kRmw) && U.len > 0) ob = __ldg(op.ob + oidx);
        const int64_t end = static_cast<int64_t>(U.e0) + U.len;
        const int my_steps = (U.len + 4 * G * kUnroll - 1) / (4 * G * kUnroll);
        const int steps = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(my_steps)));
        float num = 0.f, den = 0.f;
        for (int s = 0; s < steps; ++s) {
            float4 r4[kUnroll];
            typename IV::raw_t ix[kUnroll];
            const int64_t base = static_cast<int64_t>(U.e0) + 4 * (gl + G * kUnroll * s);
            // one base pointer per stream + immediate offsets; predicate on the remaining length
            const int rem = static_cast<int>(end - base);
            float4* rp = reinterpret_cast<float4*>(R + base);
            const typename IV::raw_t* ip = reinterpret_cast<const typename IV::raw_t*>(
                static_cast<const char*>(idx) + base * (IDX16 ? 2 : 4));
#pragma unroll
            for (int q = 0; q < kUnroll; ++q) {
                if (4 * G * q < rem) {
                    r4[q] = MODE == kPlain ? ld_stream(rp + G * q) : __ldcs(rp + G * q);
                    ix[q] = ld_stream(ip + G * q);
                }
            }
#pragma unroll
            for (int q = 0; q < kUnroll; ++q) {
                if (4 * G * q < rem) {
                    float rv[4] = {r4[q].x, r4[q].y, r4[q].z, r4[q].w};
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const int gi = IV::get(ix[q], c);
                        float r = rv[c];
                        if (MODE == kPlain) {
                            const float gv = g0[gi];
                            num = fmaf(r, gv, num);
                            den = fmaf(gv, gv, den);
                        } else if (MODE == kDemote) {
                            r = __fsub_rn(r, __fmul_rn(oa, g0[gi]));
                        } else if (MODE == kRmw) {
                            const float a = g0[gi];
                            const float b = g1[gi];
                            r = __fsub_rn(r, __fmul_rn(oa, a));
                            const float w = CSR ? ob : b;
                            const float h = CSR ? b : ob;
                            if (w != 0.f) r = __fadd_rn(r, __fmul_rn(w, h));
                        } else {
                            // CSC: g0 is global memory (the panel's ga slice, read through L1) and the
                            // padding entries' sentinel index must read 0 as the staged sentinel slot does
                            const float a = Roles<MODE, CSR>::kGaL1 && GA_GLOBAL ? (gi < op.psz ? __ldg(g0 + gi) : 0.f)
                                                                                  : g0[gi];
                            const float b = g1[gi];
                            // deferred writeback of the previous step: R - u'_i v'_j
                            r = __fsub_rn(r, __fmul_rn(oa, a));
                            // build-rhat, skipped when w_i == 0 (ccd.hpp:142)
                            const float w = CSR ? ob : b;
                            const float h = CSR ? b : ob;
                            if (w != 0.f) r = __fadd_rn(r, __fmul_rn(w, h));
                            const float gv = CSR ? b : g2[gi];
                            num = fmaf(r, gv, num);
                            den = fmaf(gv, gv, den);
                        }
                        rv[c] = r;
                    }
                    if (MODE != kPlain) __stcs(rp + G * q, make_float4(rv[0], rv[1], rv[2], rv[3]));
                }
            }
        }
        if (MODE == kDemote || MODE == kRmw) continue;
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) {
            num += __shfl_xor_sync(0xffffffffu, num, off);
            den += __shfl_xor_sync(0xffffffffu, den, off);
        }
        if (gl == 0 && U.len > 0) {
            if (U.slot < 0) {
                const float dt = __fadd_rn(op.lambda, den);
                op.out[oidx] = dt == 0.f ? 0.f : __fdiv_rn(num, dt);
            } else {
                partial[U.slot] = make_float2(num, den);
            }
        }
    }
}

// Residual pass of a split promote over one sub-panel q of the piece's panel: the unit's entries
// whose gather index falls in sub-panel q are [lo, hi) (usplit, ascending indices), processed as
// 128-bit vectors from lo & ~3 with a per-entry range predicate.  A vector straddling two
// sub-panels is rewritten in both sub-passes; they run one after the other in this CTA (the piece
// is this CTA's), so the second sees the first's stores.  Same arithmetic as the fused promote.
template <bool CSR, bool IDX16, int G, int kUnroll>
__device__ __noinline__ void run_rmw_sub(int* counter, int32_t ub, int32_t ue, const Unit* __restrict__ units,
                                         const uint16_t* __restrict__ usplit, int S, int q, int32_t gofs,
                                         const void* __restrict__ idx, float* __restrict__ R,
                                         const SweepOperands& op, const float* ga, const float* gb) {
    using IV = IdxVec<IDX16>;
    constexpr int B = 32 / G;
    const int lane = threadIdx.x & 31;
    const int g = lane / G;
    const int gl = lane % G;
    if (ub >= ue) return;
    for (;;) {
        int nb = 0;
        if (lane == 0) nb = atomicAdd(counter, B);
        nb = __shfl_sync(0xffffffffu, nb, 0);
        if (nb >= ue) break;
        const int32_t u = nb + g;
        int lo = 0, hi = 0;
        int64_t e0 = 0;
        float oa = 0.f, ob = 0.f;
        if (u < ue) {
            const Unit U = units[u];
            const uint16_t* sp = usplit + static_cast<int64_t>(u) * (S + 1) + q;
            lo = sp[0];
            hi = sp[1];
            e0 = U.e0;
            if (hi > lo) {
                oa = __ldg(op.oa + op.out_off + U.o);
                ob = __ldg(op.ob + op.out_off + U.o);
            }
        }
        const int v0 = lo & ~3;
        const int nvec = hi > lo ? (hi - v0 + 3) >> 2 : 0;
        const int my_steps = (nvec + G * kUnroll - 1) / (G * kUnroll);
        const int steps = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(my_steps)));
        float4* rp = reinterpret_cast<float4*>(R + e0 + v0);
        const typename IV::raw_t* ip = reinterpret_cast<const typename IV::raw_t*>(
            static_cast<const char*>(idx) + (e0 + v0) * (IDX16 ? 2 : 4));
        for (int s = 0; s < steps; ++s) {
            float4 r4[kUnroll];
            typename IV::raw_t ix[kUnroll];
#pragma unroll
            for (int x = 0; x < kUnroll; ++x) {
                const int vi = gl + G * (kUnroll * s + x);
                if (vi < nvec) {
                    r4[x] = __ldcs(rp + vi);
                    ix[x] = ld_stream(ip + vi);
                }
            }
#pragma unroll
            for (int x = 0; x < kUnroll; ++x) {
                const int vi = gl + G * (kUnroll * s + x);
                if (vi < nvec) {
                    float rv[4] = {r4[x].x, r4[x].y, r4[x].z, r4[x].w};
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const int pos = v0 + 4 * vi + c;
                        if (pos >= lo && pos < hi) {
                            const int gi = IV::get(ix[x], c) - gofs;
                            const float a = ga[gi];
                            const float b = gb[gi];
                            float r = __fsub_rn(rv[c], __fmul_rn(oa, a));
                            const float w = CSR ? ob : b;
                            const float h = CSR ? b : ob;
                            if (w != 0.f) r = __fadd_rn(r, __fmul_rn(w, h));
                            rv[c] = r;
                        }
                    }
                    __stcs(rp + vi, make_float4(rv[0], rv[1], rv[2], rv[3]));
                }
            }
        }
    }
}


template <int MODE, bool CSR, bool IDX16, bool SMEM, int V>
__global__ void __launch_bounds__(Var<V>::NT, 1)
sweep_kernel(const Unit* __restrict__ units, const Piece* __restrict__ pieces,
             const int32_t* __restrict__ piece_start, const int32_t* __restrict__ panel_base,
             const void* __restrict__ idx, float* __restrict__ R, float2* __restrict__ partial,
             SweepOperands op, int32_t panel_size, const uint16_t* __restrict__ usplit, int32_t rmw_sub,
             int* __restrict__ gcnt, int32_t n_pieces) {
    extern __shared__ __align__(16) float smem[];
    __shared__ int s_next[3];
    __shared__ __align__(8) uint64_t s_bar;
    constexpr int A = Roles<MODE, CSR>::kArrays;
    const int stride = stage_stride(panel_size);
    float* s0 = smem;
    float* s1 = smem + stride;
    float* s2 = smem + 2 * stride;

    if (op.cta_clock && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        op.cta_clock[2 * blockIdx.x] = t;
    }
    if (SMEM && threadIdx.x == 0) mbar_init(&s_bar, 1);
    uint32_t phase = 0;

    const int pb = piece_start[blockIdx.x], pe = piece_start[blockIdx.x + 1];
    // split-promote residual pass: the panel is staged in rmw_sub sub-panels of width panel_size
    const int nsub = MODE == kRmw ? rmw_sub : 1;
    // Work stealing (single-pass sweeps): the unit counters of every piece live in global memory
    // (gcnt[4 * piece + class], absolute unit indices), so a CTA that has finished its own pieces
    // scans all pieces and joins the one with the most remaining work; the last CTA to finish
    // resets the counters for the next launch.
    const bool steal = gcnt != nullptr && nsub == 1;
    __shared__ int s_victim;
    int cur_panel = -1;
    int own = pb;
    for (;;) {
        int pc;
        if (own < pe) {
            pc = own++;
        } else {
            if (!steal) break;
            __syncthreads();  // the previous piece is fully consumed
            if (threadIdx.x < 32) {
                // remaining work per piece (entries, roughly: long / medium / short units)
                int best = -1, bestw = 0;
                for (int p = threadIdx.x; p < n_pieces; p += 32) {
                    const Piece z = pieces[p];
                    const volatile int* g = gcnt + 4 * p;
                    const int r0 = max(0, z.um - g[0]), r1 = max(0, z.us - g[1]), r2 = max(0, z.ue - g[2]);
                    int w = r0 * 512 + r1 * 96 + r2 * 32;
                    if (z.panel != cur_panel && w < kStealRestageMin) w = 0;  // not worth a restage
                    if (w > bestw) {
                        bestw = w;
                        best = p;
                    }
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    const int ow = __shfl_xor_sync(0xffffffffu, bestw, off);
                    const int ob = __shfl_xor_sync(0xffffffffu, best, off);
                    if (ow > bestw || (ow == bestw && ob > best)) {
                        bestw = ow;
                        best = ob;
                    }
                }
                if (threadIdx.x == 0) s_victim = best;
            }
            __syncthreads();
            pc = s_victim;
            if (pc < 0) break;
        }
        const Piece pz = pieces[pc];
        int* c0 = steal ? gcnt + 4 * pc : &s_next[0];
        int* c1 = steal ? gcnt + 4 * pc + 1 : &s_next[1];
        int* c2 = steal ? gcnt + 4 * pc + 2 : &s_next[2];
        for (int q = 0; q < nsub; ++q) {
            const int32_t gbase = panel_base[pz.panel] + q * panel_size;
            const int len = nsub > 1 ? min(panel_size, panel_base[pz.panel + 1] - gbase)
                                     : panel_base[pz.panel + 1] - gbase;
            if (nsub > 1 && len <= 0) break;  // uniform: no index of this panel lies beyond
            const bool stage = nsub > 1 || pz.panel != cur_panel;
            __syncthreads();  // previous piece / sub-pass fully consumed (and barrier initialised)
            if (threadIdx.x == 0) {
                s_next[0] = pz.ub;
                s_next[1] = pz.um;
                s_next[2] = pz.us;
                if (SMEM && stage) {
                    const uint32_t bytes = static_cast<uint32_t>(((len + 3) & ~3) * sizeof(float));
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_expect_tx(&s_bar, bytes * A);
                    if (Roles<MODE, CSR>::kGaL1) {
                        bulk_g2s(s0, op.gb + gbase, bytes, &s_bar);
                        bulk_g2s(s1, op.gn + gbase, bytes, &s_bar);
                    } else {
                        bulk_g2s(s0, (MODE == kPlain ? op.gn : op.ga) + gbase, bytes, &s_bar);
                        if (A >= 2) bulk_g2s(s1, op.gb + gbase, bytes, &s_bar);
                        if (A >= 3) bulk_g2s(s2, op.gn + gbase, bytes, &s_bar);
                    }
                }
            }
            if (SMEM && stage) {
                mbar_wait(&s_bar, phase);
                phase ^= 1;
                if (threadIdx.x == 0) {
                    s0[panel_size] = 0.f;  // sentinel slot of padding entries
                    if (A >= 2) s1[panel_size] = 0.f;
                    if (A >= 3) s2[panel_size] = 0.f;
                }
            }
            cur_panel = nsub > 1 ? -1 : pz.panel;
            __syncthreads();
            const float* g0 = SMEM ? s0 : (MODE == kPlain ? op.gn : op.ga);
            const float* g1 = SMEM ? s1 : op.gb;
            const float* g2 = SMEM ? s2 : op.gn;
            if (Roles<MODE, CSR>::kGaL1 && SMEM) {
                g0 = op.ga + panel_base[pz.panel];
                g1 = s0;
                g2 = s1;
            }
            if constexpr (MODE == kRmw && SMEM) {
                if (nsub > 1) {
                    const int32_t gofs = q * panel_size;
                    run_rmw_sub<CSR, IDX16, 8, Var<V>::UA>(&s_next[0], pz.ub, pz.um, units, usplit, nsub, q, gofs, idx, R, op, g0, g1);
                    run_rmw_sub<CSR, IDX16, 4, Var<V>::UB>(&s_next[1], pz.um, pz.us, units, usplit, nsub, q, gofs, idx, R, op, g0, g1);
                    run_rmw_sub<CSR, IDX16, 2, Var<V>::UC>(&s_next[2], pz.us, pz.ue, units, usplit, nsub, q, gofs, idx, R, op, g0, g1);
                    continue;
                }
            }
            constexpr bool kGG = Roles<MODE, CSR>::kGaL1 && SMEM;
            run_class<MODE, CSR, IDX16, 8, Var<V>::UA, kGG>(c0, pz.ub, pz.um, units, idx, R, partial, op, g0, g1, g2);
            run_class<MODE, CSR, IDX16, 4, Var<V>::UB, kGG>(c1, pz.um, pz.us, units, idx, R, partial, op, g0, g1, g2);
            run_class<MODE, CSR, IDX16, 2, Var<V>::UC, kGG>(c2, pz.us, pz.ue, units, idx, R, partial, op, g0, g1, g2);
        }
    }
    if (steal) {
        // the last CTA out resets every piece's counters to its class starts for the next launch
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            s_victim = atomicAdd(gcnt + 4 * n_pieces, 1) == static_cast<int>(gridDim.x) - 1;
        }
        __syncthreads();
        if (s_victim) {
            for (int p = threadIdx.x; p < n_pieces; p += blockDim.x) {
                const Piece z = pieces[p];
                gcnt[4 * p] = z.ub;
                gcnt[4 * p + 1] = z.um;
                gcnt[4 * p + 2] = z.us;
            }
            if (threadIdx.x == 0) gcnt[4 * n_pieces] = 0;
        }
    }
    if (op.cta_clock) {
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            op.cta_clock[2 * blockIdx.x + 1] = t;
        }
    }
}

// Fixed-order combination of the partial sums of outputs with several (or zero) units: the dense
// slots p * n_out + o over the panels in order, then the output's overflow slots.  Outputs
// [0, n_big) have many slots: a warp each (lane-strided, xor tree); the rest 1 lane each, or 4 lanes
// each with >= 24 panels (every 4th slot per lane, then a 2-level xor tree); the dense slots of
// adjacent outputs are adjacent.
constexpr int kFinalizeThreads = 256;
__global__ void finalize_kernel(const int32_t* __restrict__ mo_out, const int32_t* __restrict__ mo_start,
                                int32_t n_mo, int32_t n_big, int32_t big_blocks, const float2* __restrict__ partial,
                                int32_t n_panels, int32_t n_out, int64_t n_dense, float* __restrict__ out,
                                int32_t out_off, float lambda, int lpo) {
    const float2* ovf = partial + n_dense;
    if (static_cast<int32_t>(blockIdx.x) < big_blocks) {
        const int lane = threadIdx.x & 31;
        const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
        const int64_t nw = (static_cast<int64_t>(big_blocks) * blockDim.x) >> 5;
        for (int64_t q = wid; q < n_big; q += nw) {
            const int o = mo_out[q];
            const int s0 = mo_start[q], s1 = mo_start[q + 1];
            float num = 0.f, den = 0.f;
            for (int p = lane; p < n_panels; p += 32) {
                const float2 v = partial[static_cast<int64_t>(p) * n_out + o];
                num += v.x;
                den += v.y;
            }
            for (int s = s0 + lane; s < s1; s += 32) {
                const float2 v = ovf[s];
                num += v.x;
                den += v.y;
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                num += __shfl_xor_sync(0xffffffffu, num, off);
                den += __shfl_xor_sync(0xffffffffu, den, off);
            }
            if (lane == 0) {
                const float dt = __fadd_rn(lambda, den);
                out[out_off + o] = dt == 0.f ? 0.f : __fdiv_rn(num, dt);
            }
        }
        return;
    }
    // the rest: lpo (1 or 4) lanes per output, each summing every lpo-th slot in order, then a fixed
    // 2-level tree (with many panels: a few dependent loads per lane instead of one long chain)
    const int64_t q =
        n_big + (static_cast<int64_t>(blockIdx.x - big_blocks) * blockDim.x + threadIdx.x) / lpo;
    const int sub = lpo == 4 ? (threadIdx.x & 3) : 0;
    const bool valid = q < n_mo;
    float num = 0.f, den = 0.f;
    int o = 0;
    if (valid) {
        o = mo_out[q];
        const int s0 = mo_start[q], s1 = mo_start[q + 1];
#pragma unroll 4
        for (int p = sub; p < n_panels; p += lpo) {
            const float2 v = partial[static_cast<int64_t>(p) * n_out + o];
            num += v.x;
            den += v.y;
        }
        for (int s = s0 + sub; s < s1; s += lpo) {
            const float2 v = ovf[s];
            num += v.x;
            den += v.y;
        }
    }
    if (lpo == 4) {
        num += __shfl_xor_sync(0xffffffffu, num, 1);
        den += __shfl_xor_sync(0xffffffffu, den, 1);
        num += __shfl_xor_sync(0xffffffffu, num, 2);
        den += __shfl_xor_sync(0xffffffffu, den, 2);
    }
    if (valid && sub == 0) {
        const float dt = __fadd_rn(lambda, den);
        out[out_off + o] = dt == 0.f ? 0.f : __fdiv_rn(num, dt);
    }
}

// Work stealing is on for layouts of short segments, whose per-CTA cost the static partition
// predicts poorly (Yahoo-Music shape: max/avg CTA time 1.4 -> 1.01); on long-segment layouts the
// static partition is already within a few % and the shared counters cost more than they recover.
// PMF_STEAL=0 / 1 forces it off / on.
bool steal_enabled(const DevSweep& L) {
    static const int force = [] {
        const char* e = std::getenv("PMF_STEAL");
        return e ? std::atoi(e) : -1;
    }();
    return force >= 0 ? force != 0 : L.avg_segment < 64.0;
}

template <int MODE, bool CSR, bool IDX16, bool SMEM, int V>
void launch_one(const DevSweep& L, const SweepOperands& op, size_t smem, cudaStream_t s) {
    const bool sub = MODE == kRmw && L.rmw_sub > 1;
    SweepOperands o = op;
    o.psz = sub ? L.sub_width : L.panel_size;
    sweep_kernel<MODE, CSR, IDX16, SMEM, V><<<L.ctas, Var<V>::NT, smem, s>>>(
        L.units, L.pieces, L.piece_start, L.panel_base, L.idx, L.R, L.partial, o,
        sub ? L.sub_width : L.panel_size, L.usplit, sub ? L.rmw_sub : 1, steal_enabled(L) ? L.gcnt : nullptr,
        L.n_pieces);
}

// plain sweeps: 1024 threads (u-sweep unroll 4/2/2, v-sweep 2/2/2); promote: 512 threads, 8/4/4;
// split-promote residual pass: 1024 threads, 2/2/2
int variant_for(int mode, bool csr) {
    if (mode == kRmw) return 2;
    if (mode == kPlain) return csr ? kDefaultPlainVariantCsr : kDefaultPlainVariantCsc;
    return csr ? kDefaultPromoteVariantCsr : kDefaultPromoteVariantCsc;
}

template <int MODE, bool CSR>
void dispatch_idx(const DevSweep& L, const SweepOperands& op, size_t smem, cudaStream_t s) {
    if (L.idx16 && L.smem) {
        switch (variant_for(MODE, CSR)) {
            case 1: launch_one<MODE, CSR, true, true, 1>(L, op, smem, s); return;
            case 2: launch_one<MODE, CSR, true, true, 2>(L, op, smem, s); return;
            default: break;
        }
        launch_one<MODE, CSR, true, true, 0>(L, op, smem, s);
        return;
    }
    if (L.idx16) launch_one<MODE, CSR, true, false, 0>(L, op, smem, s);
    else if (L.smem) launch_one<MODE, CSR, false, true, 0>(L, op, smem, s);
    else launch_one<MODE, CSR, false, false, 0>(L, op, smem, s);
}

template <int MODE, bool CSR, bool IDX16, bool SMEM, int V>
void set_attr(size_t max_smem) {
    cudaFuncSetAttribute(sweep_kernel<MODE, CSR, IDX16, SMEM, V>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(max_smem));
}

template <int MODE, bool CSR>
void set_attr_all(size_t max_smem) {
    set_attr<MODE, CSR, true, true, 0>(max_smem);
    set_attr<MODE, CSR, true, true, 1>(max_smem);
    set_attr<MODE, CSR, true, true, 2>(max_smem);
    set_attr<MODE, CSR, true, false, 0>(max_smem);
    set_attr<MODE, CSR, false, true, 0>(max_smem);
    set_attr<MODE, CSR, false, false, 0>(max_smem);
}

}  // namespace

size_t sweep_smem_bytes(const DevSweep& L, SweepMode mode, bool csr_side) {
    if (!L.smem) return 0;
    const int arrays = mode == kPromote ? 2 : mode == kRmw ? 2 : 1;  // CSC promote: ga through L1
    const int width = mode == kRmw && L.rmw_sub > 1 ? L.sub_width : L.panel_size;
    return static_cast<size_t>(arrays) * stage_stride(width) * sizeof(float);
}

void sweep_set_attributes(size_t max_smem) {
    set_attr_all<kPlain, true>(max_smem);
    set_attr_all<kPlain, false>(max_smem);
    set_attr_all<kPromote, true>(max_smem);
    set_attr_all<kPromote, false>(max_smem);
    set_attr_all<kDemote, true>(max_smem);
    set_attr_all<kDemote, false>(max_smem);
    set_attr_all<kRmw, true>(max_smem);
    set_attr_all<kRmw, false>(max_smem);
}

int launch_finalize(const DevSweep& L, const SweepOperands& op, cudaStream_t stream) {
    if (L.n_mo <= 0) return 0;
    const int big_blocks = static_cast<int>(std::min<int64_t>(
        (static_cast<int64_t>(L.n_mo_big) * 32 + kFinalizeThreads - 1) / kFinalizeThreads, 1184));
    const int lpo = L.n_dense && L.n_panels >= 24 ? 4 : 1;  // lanes per output (Netflix CSC: 26 panels)
    const int small_blocks = static_cast<int>((lpo * static_cast<int64_t>(L.n_mo - L.n_mo_big) + kFinalizeThreads - 1) /
                                              kFinalizeThreads);
    finalize_kernel<<<big_blocks + small_blocks, kFinalizeThreads, 0, stream>>>(
        L.mo_out, L.mo_start, L.n_mo, L.n_mo_big, big_blocks, L.partial, L.n_dense ? L.n_panels : 0, L.n_out,
        L.n_dense, op.out, op.out_off, op.lambda, lpo);
    return 1;
}

int launch_sweep(const DevSweep& L, SweepMode mode, bool csr_side, const SweepOperands& op,
                 cudaStream_t stream) {
    if (L.flat) return launch_flat(L, mode, csr_side, op, stream);
    if (mode == kPromote && L.smem && !L.promote_fused) {
        // the promote's staged vectors do not fit beside each other at this panel width: residual
        // pass over sub-panels, then a plain sweep (bitwise the same residual and result)
        return launch_sweep(L, kRmw, csr_side, op, stream) + launch_sweep(L, kPlain, csr_side, op, stream);
    }
    const size_t smem = sweep_smem_bytes(L, mode, csr_side);
    int launched = 0;
    if (L.n_units > 0) {
        if (mode == kPlain) {
            if (csr_side) dispatch_idx<kPlain, true>(L, op, smem, stream);
            else dispatch_idx<kPlain, false>(L, op, smem, stream);
        } else if (mode == kPromote) {
            if (csr_side) dispatch_idx<kPromote, true>(L, op, smem, stream);
            else dispatch_idx<kPromote, false>(L, op, smem, stream);
        } else if (mode == kRmw) {
            if (csr_side) dispatch_idx<kRmw, true>(L, op, smem, stream);
            else dispatch_idx<kRmw, false>(L, op, smem, stream);
        } else {
            if (csr_side) dispatch_idx<kDemote, true>(L, op, smem, stream);
            else dispatch_idx<kDemote, false>(L, op, smem, stream);
        }
        ++launched;
    }
    if (mode != kDemote && mode != kRmw) launched += launch_finalize(L, op, stream);
    return launched;
}

}  // namespace pmfgpu
