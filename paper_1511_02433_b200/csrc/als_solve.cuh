// als_solve.cuh -- in-warp k x k solves shared by the ALS gram kernels (als_kernels.cu, als_umma_kernels.cu):
// Cholesky factor + forward / back substitution (dense.hpp:74-124) and the item/user-wise CCD
// Gauss-Seidel sweep (ccd.hpp:56-80).  The gram G lives in shared memory (full symmetric, row stride GS).
#pragma once

#include <cuda_runtime.h>

namespace pmfgpu {

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
__device__ inline bool warp_cholesky_solve(float* G, int k, float& b0, float& b1) {
    constexpr int GS = Tile<KMAX>::GS;
    const int lane = threadIdx.x & 31;
    bool ok = true;
    for (int j = 0; j < k; ++j) {
        // every lane forms the pivot d = a_jj - sum_{t<j} l_jt^2 itself (broadcast reads of row j, no
        // shuffle reduction) fused with its rows' dot products sum_{t<j} l_it l_jt
        const int i0 = j + 1 + lane, i1 = i0 + 32;
        const bool h0 = i0 < k, h1 = i1 < k;
        float d0 = G[j * GS + j], d1 = 0.f, d2 = 0.f, d3 = 0.f;
        float s0 = h0 ? G[i0 * GS + j] : 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
        float r0 = h1 ? G[i1 * GS + j] : 0.f, r1 = 0.f;
        int t = 0;
        for (; t + 4 <= j; t += 4) {
            const float g0 = G[j * GS + t], g1 = G[j * GS + t + 1], g2 = G[j * GS + t + 2], g3 = G[j * GS + t + 3];
            d0 = fmaf(-g0, g0, d0);
            d1 = fmaf(-g1, g1, d1);
            d2 = fmaf(-g2, g2, d2);
            d3 = fmaf(-g3, g3, d3);
            if (h0) {
                s0 = fmaf(-G[i0 * GS + t], g0, s0);
                s1 = fmaf(-G[i0 * GS + t + 1], g1, s1);
                s2 = fmaf(-G[i0 * GS + t + 2], g2, s2);
                s3 = fmaf(-G[i0 * GS + t + 3], g3, s3);
            }
            if (h1) {
                r0 = fmaf(-G[i1 * GS + t], g0, r0);
                r1 = fmaf(-G[i1 * GS + t + 1], g1, r1);
                r0 = fmaf(-G[i1 * GS + t + 2], g2, r0);
                r1 = fmaf(-G[i1 * GS + t + 3], g3, r1);
            }
        }
        for (; t < j; ++t) {
            const float g0 = G[j * GS + t];
            d0 = fmaf(-g0, g0, d0);
            if (h0) s0 = fmaf(-G[i0 * GS + t], g0, s0);
            if (h1) r0 = fmaf(-G[i1 * GS + t], g0, r0);
        }
        const float d = (d0 + d1) + (d2 + d3);
        if (!(d > 0.f)) {
            ok = false;
            break;
        }
        const float ljj = sqrtf(d);
        const float rl = 1.0f / ljj;
        __syncwarp();
        if (h0) G[i0 * GS + j] = ((s0 + s1) + (s2 + s3)) * rl;
        if (h1) G[i1 * GS + j] = (r0 + r1) * rl;
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

// warp_cholesky_solve for the tensor-core kernels' gram (row stride GS: 16-byte rows, GS / 4 odd):
// the lane's row and the pivot row are read 4 columns at a time with 128-bit loads (the pivot row is a
// broadcast, the lanes' rows are conflict-free), the second row set of a lane (i0 + 32) is only
// visited while it exists (j < k - 33, warp-uniform), and each pivot comes from a running sum of its
// row's squared L entries carried down the lanes instead of a dot product every lane repeats.
template <int KMAX, int GS>
__device__ inline bool warp_cholesky_solve_v4(float* G, int k, float& b0, float& b1) {
    static_assert(GS % 4 == 0 && (GS / 4) % 2 == 1, "row stride must be an odd multiple of 4 floats");
    const int lane = threadIdx.x & 31;
    float* Rinv = G + KMAX * GS;  // 1 / L_jj (the solves multiply instead of dividing)
    bool ok = true;
    // running sum of squares of each row's finished L entries, carried by the lane that owns the
    // row: the pivot is G_jj minus that sum (no per-lane recomputation of row j's squared norm);
    // rows move down one lane per step, so the sums shift with them
    float n0 = 0.f, n1 = 0.f;
    for (int j = 0; j < k; ++j) {
        const int i0 = j + 1 + lane, i1 = i0 + 32;
        const bool h0 = i0 < k;
        const float* Gj = G + j * GS;
        const float* G0 = G + (h0 ? i0 : j) * GS;
        const float nj = __shfl_sync(0xffffffffu, n0, 0);  // row j was lane 0's row at step j - 1
        {
            const float up0 = __shfl_down_sync(0xffffffffu, n0, 1);
            const float wrap = __shfl_sync(0xffffffffu, n1, 0);
            const float up1 = __shfl_down_sync(0xffffffffu, n1, 1);
            n0 = j == 0 ? 0.f : (lane == 31 ? wrap : up0);
            n1 = j == 0 ? 0.f : (lane == 31 ? 0.f : up1);
        }
        const float d = Gj[j] - nj;
        float s0 = h0 ? G0[j] : 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
        int t = 0;
        if (KMAX > 32 && j < k - 33) {  // some lanes own a second row i1
            const bool h1 = i1 < k;
            const float* G1 = G + (h1 ? i1 : j) * GS;
            float r0 = h1 ? G1[j] : 0.f, r1 = 0.f;
            for (; t + 4 <= j; t += 4) {
                const float4 g = *reinterpret_cast<const float4*>(Gj + t);
                const float4 a = *reinterpret_cast<const float4*>(G0 + t);
                const float4 c = *reinterpret_cast<const float4*>(G1 + t);
                s0 = fmaf(-a.x, g.x, s0);
                s1 = fmaf(-a.y, g.y, s1);
                s2 = fmaf(-a.z, g.z, s2);
                s3 = fmaf(-a.w, g.w, s3);
                r0 = fmaf(-c.x, g.x, r0);
                r1 = fmaf(-c.y, g.y, r1);
                r0 = fmaf(-c.z, g.z, r0);
                r1 = fmaf(-c.w, g.w, r1);
            }
            for (; t < j; ++t) {
                const float g0 = Gj[t];
                s0 = fmaf(-G0[t], g0, s0);
                r0 = fmaf(-G1[t], g0, r0);
            }
            if (!(d > 0.f)) {
                ok = false;
                break;
            }
            const float ljj = sqrtf(d);
            const float rl = 1.0f / ljj;
            const float l0 = ((s0 + s1) + (s2 + s3)) * rl, l1 = (r0 + r1) * rl;
            n0 = fmaf(l0, l0, n0);
            n1 = fmaf(l1, l1, n1);
            __syncwarp();
            if (h0) G[i0 * GS + j] = G[j * GS + i0] = l0;
            if (h1) G[i1 * GS + j] = G[j * GS + i1] = l1;
            if (lane == 0) {
                G[j * GS + j] = ljj;
                Rinv[j] = rl;
            }
            __syncwarp();
            continue;
        }
        for (; t + 4 <= j; t += 4) {
            const float4 g = *reinterpret_cast<const float4*>(Gj + t);
            const float4 a = *reinterpret_cast<const float4*>(G0 + t);
            s0 = fmaf(-a.x, g.x, s0);
            s1 = fmaf(-a.y, g.y, s1);
            s2 = fmaf(-a.z, g.z, s2);
            s3 = fmaf(-a.w, g.w, s3);
        }
        for (; t < j; ++t) s0 = fmaf(-G0[t], Gj[t], s0);
        if (!(d > 0.f)) {
            ok = false;
            break;
        }
        const float ljj = sqrtf(d);
        const float rl = 1.0f / ljj;
        const float l0 = ((s0 + s1) + (s2 + s3)) * rl;
        n0 = fmaf(l0, l0, n0);
        __syncwarp();
        if (h0) G[i0 * GS + j] = G[j * GS + i0] = l0;
        if (lane == 0) {
            G[j * GS + j] = ljj;
            Rinv[j] = rl;
        }
        __syncwarp();
    }
    if (!ok) return false;
    // forward: L y = b (column-oriented; L^T mirrored in the upper triangle: row reads, no conflicts)
    for (int i = 0; i < k; ++i) {
        const float bi = __shfl_sync(0xffffffffu, i < 32 ? b0 : b1, i & 31);
        const float yi = bi * Rinv[i];
        if (lane == (i & 31)) {
            if (i < 32) b0 = yi;
            else b1 = yi;
        }
        if (lane > i && lane < k) b0 = fmaf(-G[i * GS + lane], yi, b0);
        if (KMAX > 32 && lane + 32 > i && lane + 32 < k) b1 = fmaf(-G[i * GS + lane + 32], yi, b1);
    }
    // backward: L^T x = y
    for (int i = k - 1; i >= 0; --i) {
        const float yi = __shfl_sync(0xffffffffu, i < 32 ? b0 : b1, i & 31);
        const float xi = yi * Rinv[i];
        if (lane == (i & 31)) {
            if (i < 32) b0 = xi;
            else b1 = xi;
        }
        if (lane < i) b0 = fmaf(-G[i * GS + lane], xi, b0);
        if (KMAX > 32 && lane + 32 < i) b1 = fmaf(-G[i * GS + lane + 32], xi, b1);
    }
    return true;
}

// One Gauss-Seidel sweep over t = 0..k-1 on (G + lambda I) x = b from the current x: the item/user-wise
// CCD coordinate update (ccd.hpp:56-80).  With R_ij = a_ij - sum_t' x_t' h_jt', the reference's
// z* = sum_j (R_ij + x_t h_jt) h_jt / (lambda + sum_j h_jt^2) equals (b_t - sum_{t' != t} G_tt' x_t') /
// (lambda + G_tt), so the epoch needs the per-row gram (the ALS gram, on the tensor cores) and no
// residual.  G rows are read along the lanes (conflict-free); den == 0 -> 0 as in the reference.
template <int KMAX, int GS>
__device__ __forceinline__ void warp_gauss_seidel(const float* G, int k, float b0, float b1, float& x0, float& x1) {
    const int lane = threadIdx.x & 31;
    for (int t = 0; t < k; ++t) {
        const float* Gt = G + t * GS;
        float p = (lane < k && lane != t) ? Gt[lane] * x0 : 0.f;
        if (KMAX > 32 && lane + 32 < k && lane + 32 != t) p = fmaf(Gt[lane + 32], x1, p);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) p += __shfl_xor_sync(0xffffffffu, p, off);
        const float bt = __shfl_sync(0xffffffffu, t < 32 ? b0 : b1, t & 31);
        const float den = Gt[t];
        const float z = den == 0.f ? 0.f : __fdiv_rn(bt - p, den);
        if (t < 32) x0 = lane == t ? z : x0;
        else x1 = lane + 32 == t ? z : x1;
    }
}


// Register-resident LDL^T solve of the symmetric positive definite k x k system (k <= KMAX) held in shared
// memory G (row stride gs, entries (m, n) with m, n < k; columns [k, KMAX) of those rows zero) with
// right-hand side rb[0..k).  Lane c holds column c of the system in registers (and column c + 32 when
// KMAX > 32); columns past k are identity, so the padded system has x = 0 there.  Right-looking
// elimination: at step j the pivot column j is broadcast from its lane entry by entry and every lane
// applies the rank-one Schur update to its own column, A_ic -= A_ij A_jc / d_j, which keeps the
// trailing matrix symmetric -- so afterwards lane c holds row c of L D (registers < c) and column c of
// L D (registers > c), and both substitutions run without any transpose.  inv (KMAX floats of shared
// memory) keeps 1/d_j.  Returns false if a pivot is not positive (dense.hpp:82-84).
template <int KMAX>
__device__ __forceinline__ bool warp_ldl_solve(const float* G, int gs, const float* rb, int k, float* inv, float& x0,
                                               float& x1) {
    constexpr bool TWO = KMAX > 32;
    constexpr int KB = TWO ? KMAX : 1;
    const int lane = threadIdx.x & 31;
    const int c0 = lane, c1 = lane + 32;
    float a[KMAX], b[KB];
#pragma unroll
    for (int i = 0; i < KMAX; i += 4) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (c0 < k) v = *reinterpret_cast<const float4*>(G + c0 * gs + i);
        a[i] = c0 < k ? v.x : (i == c0 ? 1.f : 0.f);
        a[i + 1] = c0 < k ? v.y : (i + 1 == c0 ? 1.f : 0.f);
        a[i + 2] = c0 < k ? v.z : (i + 2 == c0 ? 1.f : 0.f);
        a[i + 3] = c0 < k ? v.w : (i + 3 == c0 ? 1.f : 0.f);
        if (TWO) {
            float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
            if (c1 < k) w = *reinterpret_cast<const float4*>(G + c1 * gs + i);
            b[i] = c1 < k ? w.x : (i == c1 ? 1.f : 0.f);
            b[i + 1] = c1 < k ? w.y : (i + 1 == c1 ? 1.f : 0.f);
            b[i + 2] = c1 < k ? w.z : (i + 2 == c1 ? 1.f : 0.f);
            b[i + 3] = c1 < k ? w.w : (i + 3 == c1 ? 1.f : 0.f);
        }
    }
    bool ok = true;
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
        const int o = j & 31;
        const float d = __shfl_sync(0xffffffffu, j < 32 ? a[j] : b[j], o);
        ok = ok && d > 0.f;
        const float r = 1.0f / d;
        if (lane == 0) inv[j] = r;
        const float fa = a[j] * r;
        const float fb = TWO ? b[j] * r : 0.f;
        const bool ua = c0 > j, ub = c1 > j;
#pragma unroll
        for (int i = 1; i < KMAX; ++i) {
            if (i <= j) continue;  // compile-time once both loops are unrolled
            const float li = __shfl_sync(0xffffffffu, j < 32 ? a[i] : b[i], o);
            if (ua) a[i] = fmaf(-li, fa, a[i]);
            if (TWO && ub) b[i] = fmaf(-li, fb, b[i]);
        }
    }
    __syncwarp();
    // forward: z_i -= (l_ic d_c) y_c, y_c = z_c / d_c (lane i's register c, c < i, holds l_ic d_c)
    float z0 = c0 < k ? rb[c0] : 0.f, z1 = (TWO && c1 < k) ? rb[c1] : 0.f;
#pragma unroll
    for (int c = 0; c < KMAX; ++c) {
        const float yc = __shfl_sync(0xffffffffu, c < 32 ? z0 : z1, c & 31) * inv[c];
        if (c0 > c) z0 = fmaf(-a[c], yc, z0);
        if (TWO && c1 > c) z1 = fmaf(-b[c], yc, z1);
        if (c < 32 && c0 == c) z0 = yc;
        if (TWO && c >= 32 && c1 == c) z1 = yc;
    }
    // backward: x_c = y_c - (1 / d_c) sum_{i > c} (l_ic d_c) x_i (lane c's register i, i > c)
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int i = KMAX - 1; i >= 0; --i) {
        if (i < 32 && c0 == i) z0 = fmaf(-s0, inv[i], z0);
        if (TWO && i >= 32 && c1 == i) z1 = fmaf(-s1, inv[i], z1);
        const float xi = __shfl_sync(0xffffffffu, i < 32 ? z0 : z1, i & 31);
        if (c0 < i) s0 = fmaf(a[i], xi, s0);
        if (TWO && c1 < i) s1 = fmaf(b[i], xi, s1);
    }
    x0 = z0;
    x1 = z1;
    return ok;
}

}  // namespace pmfgpu
