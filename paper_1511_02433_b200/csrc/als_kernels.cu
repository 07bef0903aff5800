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
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "als_solve.cuh"
#include "device.hpp"

namespace pmfgpu {

namespace {

constexpr int kAlsThreads = 256;
constexpr int kAlsWarps = kAlsThreads / 32;
// tensor-core gram kernel: 4-warp CTAs, 5 per SM (20 warps, <= 96 registers; the gram aliases the
// stage so the shared-memory footprint allows it)
#ifndef PMF_TC_THREADS
#define PMF_TC_THREADS 128
#endif
#ifndef PMF_TC_LDL
#define PMF_TC_LDL 1
#endif
#ifndef PMF_TC_KMAX
#define PMF_TC_KMAX 64  // largest k of the mma.sync tensor-core gram (Netflix k = 44 / 48 / 56 / 64: 21 / 21 / 32 / 60 ms
                        // against 64 / 66 / ~70 / 74 ms for the FP32 SIMT gram it replaces)
#endif
#ifndef PMF_TC_MINB
#define PMF_TC_MINB (PMF_TC_LDL ? 4 : 5)
#endif
constexpr int kTcThreads = PMF_TC_THREADS;
constexpr int kTcWarps = kTcThreads / 32;

// Stages the gathered opposing rows of one 32-entry chunk into X[s][0..KS): lanes own features
// (coalesced 4k-byte row reads), 8 rows' loads are issued before they are stored (bank-conflict
// free stores); columns [k, KS) and rows [cnt, rows_pad) are zero.
template <int KMAX, int KS, bool AUG = false>
__device__ __forceinline__ void stage_rows(float* X, const float* __restrict__ opp, const int* sidx, int cnt,
                                           int rows_pad, int k, const float* sval = nullptr) {
    const int lane = threadIdx.x & 31;
    constexpr int CW = (KS + 31) / 32;  // columns per lane
    for (int s0 = 0; s0 < rows_pad; s0 += 8) {
        float v[8][CW];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int srow = s0 + r;
            const bool live = srow < cnt;
            const int64_t base = live ? static_cast<int64_t>(sidx[srow]) * k : 0;
#pragma unroll
            for (int w = 0; w < CW; ++w) {
                const int c = lane + 32 * w;
                v[r][w] = (live && c < k) ? __ldg(opp + base + c) : 0.f;
                if (AUG && live && c == k) v[r][w] = sval[srow];  // rating column: G[:, k] = X^T a
            }
        }
#pragma unroll
        for (int r = 0; r < 8; ++r)
            if (s0 + r < rows_pad)
#pragma unroll
                for (int w = 0; w < CW; ++w)
                    if (lane + 32 * w < KS) X[(s0 + r) * KS + lane + 32 * w] = v[r][w];
    }
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
            stage_rows<KMAX, KS>(X, opp, sidx, cnt, cnt, k);
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

// ---- tensor-core gram (3xTF32) -----------------------------------------------------------------
// G = X^T X over the unit's gathered rows X (entries x features) with mma.sync m16n8k8 TF32: the
// feature axis is tiled 16 (M) x 8 (N), the entry axis is the MMA K.  Only tiles touching the upper
// triangle are computed (9 of 15 at k = 40).  Each operand is split x = hi + lo (split_tf32) and G
// accumulates hi*hi + hi*lo + lo*hi in FP32, which keeps ~FP32 accuracy
// (the north_star's 3xTF32 condition; parity is checked against the reference in the tests).
template <int NT, int MT>
struct TcGeo {
    static constexpr int KMAX = 8 * NT;                       // padded k (Cholesky order bound)
    static constexpr int KS = (NT % 2) ? 8 * NT : 8 * NT + 8;  // staged row stride (bank-conflict free)
    static constexpr int JN = NT > 2 * MT ? NT : 2 * MT;      // feature slots per lane: g + 8j
    static constexpr int STAGE = 32 * KS;
    // gram row stride: a multiple of 4 (16-byte rows for 128-bit loads) that is an odd multiple of 4
    // modulo 32, so the rows of 8 consecutive lanes fall in distinct 4-bank groups (conflict-free
    // LDS.128 of the lanes' own rows in the Cholesky)
    static constexpr int GS0 = (KMAX + 1 + 3) & ~3;
    static constexpr int GS = (GS0 % 8 == 0) ? GS0 + 4 : GS0;
    static constexpr int GRAM = KMAX * GS + 2 * KMAX;
    // the gram aliases the stage (it is formed after the unit's last chunk is consumed): a warp's
    // footprint is max(stage, gram) + 64 floats, 128-byte aligned for the TMA destinations
    static constexpr int WARP_FLOATS = ((STAGE > GRAM ? STAGE : GRAM) + 64 + 31) & ~31;
    static constexpr int count_tiles() {
        int c = 0;
        for (int mi = 0; mi < MT; ++mi)
            for (int ni = 0; ni < NT; ++ni)
                if (8 * ni + 7 >= 16 * mi) ++c;
        return c;
    }
    static constexpr int NTILES = count_tiles();
};

// x = hi + lo for the 3xTF32 products: hi = x rounded to nearest (ties away) at the TF32 mantissa
// width by integer add + mask (2 instructions; sm_100's cvt.rna.tf32 is a 4-instruction sequence
// with an inf/NaN guard that finite factors do not need), lo = x - hi exactly in FP32, then
// truncated to TF32 (the MMA reads only the top 19 bits).
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
    hi = (__float_as_uint(x) + 0x1000u) & 0xffffe000u;
    lo = __float_as_uint(x - __uint_as_float(hi)) & 0xffffe000u;
}

__device__ __forceinline__ void mma_tf32(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm(  // not volatile: the compiler may interleave independent accumulators
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// G4: the gather4 staging only (tma == 2, the B200 default; the other stagings stay behind the runtime
// `tma` of G4 = false).  GSW: the item/user-wise CCD Gauss-Seidel epilogue instead of the ALS solve.  Both
// are compile-time so the hot kernel carries one staging and one epilogue (smaller code: the W side
// stalled on instruction fetch with all of them in one body).
template <int NT, int MT, bool G4, bool GSW>
__global__ void __launch_bounds__(kTcThreads, PMF_TC_MINB)
als_gram_tc_kernel(const Unit* __restrict__ units, int32_t n_units, const int32_t* __restrict__ idx,
                   const float* __restrict__ val, const float* __restrict__ opp, float* __restrict__ out,
                   int32_t out_off, int k, float lambda, int weighted, float* __restrict__ partial,
                   int* __restrict__ counter, int* __restrict__ status, int tma, int gs,
                   const __grid_constant__ CUtensorMap rows_map) {
    using T = TcGeo<NT, MT>;
    constexpr int KS = T::KS, JN = T::JN, NTILES = T::NTILES, KMAX = T::KMAX;
    constexpr int GS = T::GS;
    extern __shared__ __align__(128) float smem[];
    __shared__ __align__(8) uint64_t s_bar[kTcWarps];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int g = lane >> 2, tig = lane & 3;
    float* X = smem + warp * T::WARP_FLOATS;
    float* G = X;  // aliases the stage
    int* sidx = reinterpret_cast<int*>(X + T::WARP_FLOATS - 64);
    float* sval = X + T::WARP_FLOATS - 32;
    uint64_t* bar = &s_bar[warp];
    uint32_t phase = 0;
    if (G4) tma = 2;
    else if (tma == 2) tma = 1;
    if (tma) {
        // TMA rows (4k bytes each) leave columns [k, KS) untouched: zero them here (and per unit after
        // the aliased gram has overwritten them)
        for (int e = lane; e < T::STAGE; e += 32) X[e] = 0.f;
        if (lane == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
                static_cast<uint32_t>(__cvta_generic_to_shared(bar))));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
    }

    for (;;) {
        int u = 0;
        if (lane == 0) u = atomicAdd(counter, 1);
        u = __shfl_sync(0xffffffffu, u, 0);
        if (u >= n_units) break;
        const Unit U = units[u];
        float acc[NTILES][4];
#pragma unroll
        for (int t = 0; t < NTILES; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.f;
        float accr[MT][4];
#pragma unroll
        for (int t = 0; t < MT; ++t) accr[t][0] = accr[t][1] = accr[t][2] = accr[t][3] = 0.f;
        float rhs0 = 0.f, rhs1 = 0.f;
        if (!G4 && tma == 1 && KS != k) {
            // per-row bulk copies write k columns: re-zero the padding columns the previous unit's
            // gram (aliasing the stage) overwrote
            __syncwarp();
            for (int e = lane; e < 32 * (KS - k); e += 32) X[(e / (KS - k)) * KS + k + e % (KS - k)] = 0.f;
        }
        for (int base = 0; base < U.len; base += 32) {
            const int cnt = min(32, U.len - base);
            const int cnt8 = (cnt + 7) & ~7;
            __syncwarp();
            if (G4) {
                // TMA gather4: one elected lane issues cnt8 / 4 tensor copies of 4 rows each (rows past
                // cnt use an out-of-bounds row coordinate and arrive zero-filled); X's row stride is k
                const int row = lane < cnt ? idx[U.e0 + base + lane] : 0x7fffffff;
                if (lane < cnt) sval[lane] = val[U.e0 + base + lane];
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
                if (lane == 0)
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b),
                                 "r"(static_cast<uint32_t>(cnt8 * k * 4))
                                 : "memory");
                for (int q = 0; q < cnt8; q += 4) {
                    const int r0 = __shfl_sync(0xffffffffu, row, q), r1 = __shfl_sync(0xffffffffu, row, q + 1);
                    const int r2 = __shfl_sync(0xffffffffu, row, q + 2), r3 = __shfl_sync(0xffffffffu, row, q + 3);
                    if (lane == 0)
                        asm volatile(
                            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
                                static_cast<uint32_t>(__cvta_generic_to_shared(X + q * KS))),
                            "l"(reinterpret_cast<uint64_t>(&rows_map)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
                            "r"(b)
                            : "memory");
                }
                asm volatile(
                    "{\n"
                    ".reg .pred p;\n"
                    "ALSG_%=:\n"
                    "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                    "@!p bra ALSG_%=;\n"
                    "}\n" ::"r"(b),
                    "r"(phase)
                    : "memory");
                phase ^= 1;
            } else if (tma) {
                // one bulk copy per gathered row, issued by the row's lane, completing on the warp's
                // mbarrier; the rows past cnt up to the MMA's multiple of 8 are zeroed
                const int row = lane < cnt ? idx[U.e0 + base + lane] : 0;
                if (lane < cnt) sval[lane] = val[U.e0 + base + lane];
                for (int r = cnt; r < cnt8; ++r)
                    for (int c = lane; c < KS; c += 32) X[r * KS + c] = 0.f;
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
                if (lane == 0)
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b),
                                 "r"(static_cast<uint32_t>(cnt * k * 4))
                                 : "memory");
                __syncwarp();
                if (lane < cnt)
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            static_cast<uint32_t>(__cvta_generic_to_shared(X + lane * KS))),
                        "l"(opp + static_cast<int64_t>(row) * k), "r"(static_cast<uint32_t>(k * 4)), "r"(b)
                        : "memory");
                asm volatile(
                    "{\n"
                    ".reg .pred p;\n"
                    "ALSW_%=:\n"
                    "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                    "@!p bra ALSW_%=;\n"
                    "}\n" ::"r"(b),
                    "r"(phase)
                    : "memory");
                phase ^= 1;
            } else {
                if (lane < cnt) {
                    sidx[lane] = idx[U.e0 + base + lane];
                    sval[lane] = val[U.e0 + base + lane];
                }
                __syncwarp();
                stage_rows<KMAX, KS>(X, opp, sidx, cnt, cnt8, k);
            }
            __syncwarp();
            for (int e0 = 0; e0 < cnt8; e0 += 8) {
                uint32_t hi[JN][2], lo[JN][2];
#pragma unroll
                for (int j = 0; j < JN; ++j)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const float x = j < NT ? X[(e0 + tig + 4 * h) * KS + 8 * j + g] : 0.f;
                        split_tf32(x, hi[j][h], lo[j][h]);
                    }
                // the ratings as one more B column block (column 8 NT, lanes g == 0): X^T a rides the
                // same MMAs as the gram instead of a per-entry FMA loop
                uint32_t ahi[2], alo[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int e = e0 + tig + 4 * h;
                    const float av = (g == 0 && e < cnt) ? sval[e] : 0.f;
                    split_tf32(av, ahi[h], alo[h]);
                }
                // three passes (hi*hi, hi*lo, lo*hi) over all tiles: consecutive MMAs are independent
#pragma unroll
                for (int pass = 0; pass < 3; ++pass) {
                    int t = 0;
#pragma unroll
                    for (int mi = 0; mi < MT; ++mi) {
                        const uint32_t(&A)[JN][2] = pass == 2 ? lo : hi;
#pragma unroll
                        for (int ni = 0; ni < NT; ++ni) {
                            if (8 * ni + 7 < 16 * mi) continue;
                            const uint32_t(&B)[JN][2] = pass == 1 ? lo : hi;
                            mma_tf32(acc[t], A[2 * mi][0], A[2 * mi + 1][0], A[2 * mi][1], A[2 * mi + 1][1],
                                     B[ni][0], B[ni][1]);
                            ++t;
                        }
                        mma_tf32(accr[mi], A[2 * mi][0], A[2 * mi + 1][0], A[2 * mi][1], A[2 * mi + 1][1],
                                 pass == 1 ? alo[0] : ahi[0], pass == 1 ? alo[1] : ahi[1]);
                    }
                }
            }
        }
        // X^T a: lanes tig == 0 hold features 16 mi + g (+ 8) in accumulator elements 0 and 2
        {
            float* Bv = G + KMAX * GS + KMAX;  // past Rinv
#pragma unroll
            for (int mi = 0; mi < MT; ++mi)
                if (tig == 0) {
                    if (16 * mi + g < KMAX) Bv[16 * mi + g] = accr[mi][0];
                    if (16 * mi + g + 8 < KMAX) Bv[16 * mi + g + 8] = accr[mi][2];
                }
            __syncwarp();
            rhs0 = lane < k ? Bv[lane] : 0.f;
            rhs1 = lane + 32 < k ? Bv[lane + 32] : 0.f;
        }
        __syncwarp();
        // scatter the upper-triangle tiles (and their mirror) into the gram / partial
        float* P = U.slot >= 0 ? partial + static_cast<int64_t>(U.slot) * (k * k + k + 1) : nullptr;
        const float ridge = weighted ? lambda * static_cast<float>(U.len) : lambda;
        int t = 0;
#pragma unroll
        for (int mi = 0; mi < MT; ++mi)
#pragma unroll
            for (int ni = 0; ni < NT; ++ni) {
                if (8 * ni + 7 < 16 * mi) continue;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int m = 16 * mi + g + 8 * (c >> 1);
                    const int n = 8 * ni + 2 * tig + (c & 1);
                    const float v = acc[t][c];
                    if (m <= n && n < k) {
                        if (P) {
                            P[m * k + n] = v;
                            P[n * k + m] = v;
                        } else {
                            G[m * GS + n] = m == n ? v + ridge : v;
                            G[n * GS + m] = m == n ? v + ridge : v;
                        }
                    }
                }
                ++t;
            }
        if (P) {
            if (lane < k) P[k * k + lane] = rhs0;
            if (lane + 32 < k) P[k * k + lane + 32] = rhs1;
            if (lane == 0) P[k * k + k] = static_cast<float>(U.len);
            __syncwarp();
            continue;
        }
        __syncwarp();
        float* dst = out + static_cast<int64_t>(out_off + U.o) * k;
        if (GSW) {  // item/user-wise CCD: one coordinate sweep from the current row
            float x0 = lane < k ? dst[lane] : 0.f, x1 = lane + 32 < k ? dst[lane + 32] : 0.f;
            warp_gauss_seidel<KMAX, GS>(G, k, rhs0, rhs1, x0, x1);
            if (lane < k) dst[lane] = x0;
            if (lane + 32 < k) dst[lane + 32] = x1;
            __syncwarp();
            continue;
        }
#if PMF_TC_LDL
        const bool ok = warp_ldl_solve<KMAX>(G, GS, G + KMAX * GS + KMAX, k, G + KMAX * GS, rhs0, rhs1);
#else
        const bool ok = warp_cholesky_solve_v4<KMAX, GS>(G, k, rhs0, rhs1);
#endif
        if (!ok) {
            if (lane == 0) atomicExch(status, 4);
            rhs0 = rhs1 = 0.f;
        }
        if (lane < k) dst[lane] = rhs0;
        if (lane + 32 < k) dst[lane + 32] = rhs1;
        __syncwarp();
    }
}

template <int KMAX>
__global__ void __launch_bounds__(kAlsThreads)
als_reduce_solve_kernel(const int32_t* __restrict__ mo_out, const int32_t* __restrict__ mo_start,
                        int32_t n_mo, const float* __restrict__ partial, float* __restrict__ out,
                        int32_t out_off, int k, float lambda, int weighted, int* __restrict__ status, int gs) {
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
        float* dst = out + static_cast<int64_t>(out_off + mo_out[q]) * k;
        if (gs) {
            float x0 = lane < k ? dst[lane] : 0.f, x1 = lane + 32 < k ? dst[lane + 32] : 0.f;
            warp_gauss_seidel<KMAX, GS>(G, k, b0, b1, x0, x1);
            b0 = x0;
            b1 = x1;
        } else if (!warp_cholesky_solve<KMAX>(G, k, b0, b1)) {
            if (lane == 0) atomicExch(status, 4);
            b0 = b1 = 0.f;
        }
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

template <int NT, int MT>
size_t smem_for_tc() {
    return static_cast<size_t>(kTcWarps) * TcGeo<NT, MT>::WARP_FLOATS * sizeof(float);
}

bool use_tensor_cores() {
    static const bool tc = std::getenv("PMF_ALS_SIMT") == nullptr;
    return tc;
}

// PMF_ALS_UMMA=1: the tcgen05 / TMEM gram kernel (als_umma_kernels.cu, k <= 48) instead of the mma.sync
// one.  Parity-green, but slower at the BASELINE shapes: with N <= 48 columns per row gram every
// operand tile is re-read from shared memory per MMA, and the transpose into K-major tiles plus the
// gathers put ~580 shared-memory wavefronts on each 32-entry chunk, where mma.sync keeps its operands
// in registers (profiles/r02_ncu_als_umma.txt).
bool use_umma() {
    static const bool on = std::getenv("PMF_ALS_UMMA") != nullptr;
    return on;
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
    static const EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

// 2-D tensor map over the opposing factor (n_opp rows of k floats) with a 1-row box of k floats:
// the gather4 staging's descriptor (rows outside [0, n_opp) arrive zero-filled).
bool make_rows_map(CUtensorMap* map, const float* opp, int64_t n_opp, int k) {
    const EncodeTiledFn fn = encode_tiled();
    if (!fn || n_opp <= 0) return false;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(n_opp)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(k) * sizeof(float)};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(k), 1u};
    const cuuint32_t estr[2] = {1u, 1u};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(opp), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// PMF_ALS_TMA: unset = gather4 where the staged row stride equals k (else per-row bulk copies),
// 1 = per-row bulk copies, 0 = LSU staging.
int als_tma_mode() {
    static const int m = std::getenv("PMF_ALS_TMA") ? std::atoi(std::getenv("PMF_ALS_TMA")) : 2;
    return m;
}

template <int NT, int MT>
void launch_tc(const DevAls& L, const float* opp, int64_t n_opp, float* out, int32_t out_off, int k, float lambda,
               bool weighted, int* d_counter, int* d_status, int sm_count, cudaStream_t s, bool gs) {
    const size_t sm = smem_for_tc<NT, MT>();
    int per_sm = 0;
    // TMA row staging needs 16-byte rows (k % 4 == 0; the factor base is cudaMalloc-aligned)
    const int mode = als_tma_mode();
    int tma = mode != 0 && k % 4 == 0 && (reinterpret_cast<uintptr_t>(opp) & 15) == 0 ? 1 : 0;
    alignas(64) CUtensorMap map{};
    if (tma && mode == 2 && k == TcGeo<NT, MT>::KS && make_rows_map(&map, opp, n_opp, k)) tma = 2;
    auto go = [&](auto kern) {
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTcThreads, sm);
        const int blocks = std::max(1, std::min<int>(per_sm * sm_count, (L.n_units + kTcWarps - 1) / kTcWarps));
        kern<<<blocks, kTcThreads, sm, s>>>(L.units, L.n_units, L.idx, L.val, opp, out, out_off, k, lambda,
                                            weighted ? 1 : 0, L.partial, d_counter, d_status, tma, gs ? 1 : 0, map);
    };
    if (tma == 2) {
        if (gs) go(als_gram_tc_kernel<NT, MT, true, true>);
        else go(als_gram_tc_kernel<NT, MT, true, false>);
    } else {
        if (gs) go(als_gram_tc_kernel<NT, MT, false, true>);
        else go(als_gram_tc_kernel<NT, MT, false, false>);
    }
}

template <int KMAX>
int launch_k(const DevAls& L, const float* opp, int64_t n_opp, float* out, int32_t out_off, int k, float lambda, bool weighted,
             int* d_counter, int* d_status, int sm_count, cudaStream_t s, bool gs) {
    int launched = 0;
    const size_t sm = smem_for<KMAX>();
    if (L.n_units > 0) {
        cudaMemsetAsync(d_counter, 0, sizeof(int), s);
        if (use_tensor_cores() && als_umma_supported(k) && use_umma()) {
            launch_als_umma(L, opp, n_opp, out, out_off, k, lambda, weighted, d_counter, d_status, sm_count, s, gs);
        } else if (use_tensor_cores() && k <= PMF_TC_KMAX) {
            // N tiles (8 features) and M tiles (16 features) covering the k features
            const int nt = (k + 7) / 8, mt = (k + 15) / 16;
#define PMF_TC(NT_, MT_) \
    if (nt == NT_ && mt == MT_) launch_tc<NT_, MT_>(L, opp, n_opp, out, out_off, k, lambda, weighted, d_counter, d_status, sm_count, s, gs)
            PMF_TC(1, 1); else PMF_TC(2, 1); else PMF_TC(3, 1); else PMF_TC(3, 2); else PMF_TC(4, 2);
            else PMF_TC(5, 2); else PMF_TC(5, 3); else PMF_TC(6, 3); else PMF_TC(7, 4); else PMF_TC(8, 4);
#undef PMF_TC
        } else {
            int per_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, als_gram_kernel<KMAX>, kAlsThreads, sm);
            const int blocks = std::max(1, std::min<int>(per_sm * sm_count, (L.n_units + kAlsWarps - 1) / kAlsWarps));
            als_gram_kernel<KMAX><<<blocks, kAlsThreads, sm, s>>>(L.units, L.n_units, L.idx, L.val, opp, out, out_off,
                                                                   k, lambda, weighted ? 1 : 0, L.partial, d_counter,
                                                                   d_status);
        }
        ++launched;
    }
    if (L.n_mo > 0) {
        const int blocks = std::max(1, std::min(4 * sm_count, (L.n_mo + kAlsWarps - 1) / kAlsWarps));
        als_reduce_solve_kernel<KMAX><<<blocks, kAlsThreads, sm, s>>>(L.mo_out, L.mo_start, L.n_mo, L.partial, out,
                                                                       out_off, k, lambda, weighted ? 1 : 0, d_status,
                                                                       gs ? 1 : 0);
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

template <int NT, int MT>
void set_attr_tc() {
    const int bytes = static_cast<int>(smem_for_tc<NT, MT>());
    cudaFuncSetAttribute(als_gram_tc_kernel<NT, MT, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(als_gram_tc_kernel<NT, MT, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(als_gram_tc_kernel<NT, MT, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(als_gram_tc_kernel<NT, MT, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

void als_set_attributes() {
    als_umma_set_attributes();
    set_attr_tc<1, 1>();
    set_attr_tc<2, 1>();
    set_attr_tc<3, 1>();
    set_attr_tc<3, 2>();
    set_attr_tc<4, 2>();
    set_attr_tc<5, 2>();
    set_attr_tc<5, 3>();
    set_attr_tc<6, 3>();
    set_attr_tc<7, 4>();
    set_attr_tc<8, 4>();
    set_attr_k<8>();
    set_attr_k<16>();
    set_attr_k<32>();
    set_attr_k<40>();
    set_attr_k<64>();
}

bool als_gram_gs_supported(int k) { return use_tensor_cores() && k >= 1 && k <= (use_umma() ? 48 : PMF_TC_KMAX); }

int launch_als_half(const DevAls& L, const float* opp, int64_t n_opp, float* out, int32_t out_off, int k,
                    float lambda, bool weighted, int* d_counter, int* d_status, int sm_count, cudaStream_t stream,
                    bool gs) {
    if (gs && !als_gram_gs_supported(k)) return -1;  // the Gauss-Seidel solve lives in the tensor-core path
    if (k > 64) {
        int launched = launch_als_big(L, opp, out, out_off, k, lambda, weighted, d_counter, d_status, sm_count,
                                      L.big_scratch, stream);
        if (L.n_empty > 0) {
            zero_rows_kernel<<<std::min(1024, (L.n_empty * k + 255) / 256), 256, 0, stream>>>(L.empty_out, L.n_empty,
                                                                                           out, out_off, k);
            ++launched;
        }
        return launched;
    }
#define PMF_HALF(K) \
    return launch_k<K>(L, opp, n_opp, out, out_off, k, lambda, weighted, d_counter, d_status, sm_count, stream, gs)
    if (k <= 8) PMF_HALF(8);
    if (k <= 16) PMF_HALF(16);
    if (k <= 32) PMF_HALF(32);
    if (k <= 40) PMF_HALF(40);
    PMF_HALF(64);
#undef PMF_HALF
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
