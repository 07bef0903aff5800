// topn_kernels.cu -- top_n (model.hpp:172-209) for a batch of users on the GPU.
//
// top_n(model, i, count, rated_sorted) scores every unrated item j with predict(model, i, j) -- a Real
// (FP32) sum over t of w_it * h_jt in ascending t, each product rounded before the add
// (model.hpp:103-114; no FMA at the reference's Release flags) -- and keeps the `count` best,
// ordered by score descending, ties by ascending item index.  Scores here are formed with exactly
// those roundings (__fmul_rn / __fadd_rn), so rankings and scores are bitwise the reference's.
//
// A CTA takes 64 users (8 per warp) and walks the items in tiles of 256: the tile of H is staged
// transposed in shared memory, each lane computes 8 users x 8 items (items lane + 32 q), unrated-item
// exclusion comes from a per-tile bitmap built from each user's sorted rated list, and each user's
// running top-`count` list lives in shared memory.  A candidate enters the list only if it beats the
// current last entry; insertions are warp-cooperative (position by ballot, then shift).
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "device.hpp"

namespace pmfgpu {

namespace {

constexpr int kTnThreads = 256;
constexpr int kTnUsers = 64;  // per CTA, 8 per warp
constexpr int kTnTile = 256;  // items per tile, 8 per lane

struct TnEntry {
    float s;
    int j;
};

// a beats b: higher score, or equal score and lower item (model.hpp:192-195)
__device__ __forceinline__ bool beats(float sa, int ja, float sb, int jb) {
    return sa > sb || (sa == sb && ja < jb);
}

__global__ void __launch_bounds__(kTnThreads)
topn_kernel(const float* __restrict__ W, const float* __restrict__ H, int32_t n, int k,
            const int32_t* __restrict__ users, int32_t n_users, const int64_t* __restrict__ ex_start,
            const int32_t* __restrict__ ex_items, int count, int32_t* __restrict__ out_items,
            float* __restrict__ out_scores, int32_t* __restrict__ out_count) {
    extern __shared__ __align__(16) float sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int u0 = blockIdx.x * kTnUsers;
    const int nu = min(kTnUsers, n_users - u0);
    constexpr int HS = kTnTile + 4;  // transposed tile row stride
    float* Ht = sm;                                      // [k][HS]
    float* Wb = Ht + k * HS;                             // [k][kTnUsers]
    uint32_t* bm = reinterpret_cast<uint32_t*>(Wb + k * kTnUsers);  // [kTnUsers][kTnTile / 32]
    TnEntry* lists = reinterpret_cast<TnEntry*>(bm + kTnUsers * (kTnTile / 32));  // [kTnUsers][count]
    __shared__ int s_filled[kTnUsers];
    __shared__ int s_ex[kTnUsers];  // exclusion cursor (position in the user's rated list)

    // the CTA's user factors, transposed
    for (int e = threadIdx.x; e < k * kTnUsers; e += kTnThreads) {
        const int u = e % kTnUsers, t = e / kTnUsers;
        Wb[t * kTnUsers + u] = u < nu ? W[static_cast<int64_t>(users[u0 + u]) * k + t] : 0.f;
    }
    if (threadIdx.x < kTnUsers) {
        s_filled[threadIdx.x] = 0;
        s_ex[threadIdx.x] = threadIdx.x < nu ? static_cast<int>(0) : 0;
    }
    const int ub = warp * 8;  // this warp's users ub .. ub + 7

    for (int j0 = 0; j0 < n; j0 += kTnTile) {
        __syncthreads();  // previous tile consumed
        const int tn = min(kTnTile, n - j0);
        for (int e = threadIdx.x; e < tn * k; e += kTnThreads) {
            const int jj = e / k, t = e - jj * k;
            Ht[t * HS + jj] = H[static_cast<int64_t>(j0 + jj) * k + t];
        }
        for (int e = threadIdx.x; e < kTnUsers * (kTnTile / 32); e += kTnThreads) bm[e] = 0u;
        __syncthreads();
        // exclusion bitmap: each warp marks its users' rated items inside [j0, j0 + tn)
        for (int uu = 0; uu < 8; ++uu) {
            const int u = ub + uu;
            if (u >= nu) break;
            const int64_t base = ex_start[u0 + u], end = ex_start[u0 + u + 1];
            int cur = s_ex[u];
            for (;;) {
                const int64_t p = base + cur + lane;
                const int jx = p < end ? ex_items[p] : INT32_MAX;
                const bool in = jx < j0 + tn;
                if (in && jx >= j0) atomicOr(&bm[u * (kTnTile / 32) + ((jx - j0) >> 5)], 1u << ((jx - j0) & 31));
                const uint32_t bal = __ballot_sync(0xffffffffu, in);
                cur += __popc(bal);
                if (bal != 0xffffffffu) break;
            }
            __syncwarp();
            if (lane == 0) s_ex[u] = cur;
        }
        __syncwarp();
        // scores of 8 users x 8 items per lane, exactly predict()'s roundings
        float acc[8][8];
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[a][q] = 0.f;
        for (int t = 0; t < k; ++t) {
            const float4 wa = *reinterpret_cast<const float4*>(Wb + t * kTnUsers + ub);
            const float4 wb = *reinterpret_cast<const float4*>(Wb + t * kTnUsers + ub + 4);
            const float w[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
            float h[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) h[q] = Ht[t * HS + lane + 32 * q];
#pragma unroll
            for (int a = 0; a < 8; ++a)
#pragma unroll
                for (int q = 0; q < 8; ++q) acc[a][q] = __fadd_rn(acc[a][q], __fmul_rn(w[a], h[q]));
        }
        // selection, one user at a time
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            const int u = ub + a;
            if (u >= nu) break;
            TnEntry* L = lists + u * count;
            uint32_t pend = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int jj = lane + 32 * q;
                const bool ok = jj < tn && !((bm[u * (kTnTile / 32) + q] >> lane) & 1u);
                pend |= ok ? (1u << q) : 0u;
            }
            int filled = s_filled[u];
            for (;;) {
                // drop candidates that cannot enter a full list
                if (filled == count) {
                    const TnEntry last = L[count - 1];
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        if (((pend >> q) & 1u) && !beats(acc[a][q], j0 + lane + 32 * q, last.s, last.j))
                            pend &= ~(1u << q);
                }
                const uint32_t bal = __ballot_sync(0xffffffffu, pend != 0u);
                if (!bal) break;
                // the first pending lane's lowest pending item enters
                const int src = __ffs(bal) - 1;
                int qsel = __ffs(pend) - 1;
                float cs = 0.f;
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (q == qsel) cs = acc[a][q];
                const float s = __shfl_sync(0xffffffffu, cs, src);
                qsel = __shfl_sync(0xffffffffu, qsel, src);
                const int j = j0 + src + 32 * qsel;
                if (lane == src) pend &= ~(1u << qsel);
                // position = entries that beat the candidate
                int pos = 0;
                for (int b = 0; b < filled; b += 32) {
                    const int e = b + lane;
                    const bool bt = e < filled && beats(L[e].s, L[e].j, s, j);
                    pos += __popc(__ballot_sync(0xffffffffu, bt));
                }
                const int nf = min(filled + 1, count);
                // shift [pos, nf - 1) down by one, back to front in 32-entry steps
                for (int b = nf - 1; b > pos; b -= 32) {
                    const int e = b - lane;
                    TnEntry v{0.f, 0};
                    const bool mv = e > pos;
                    if (mv) v = L[e - 1];
                    __syncwarp();
                    if (mv) L[e] = v;
                    __syncwarp();
                }
                if (lane == 0 && pos < count) L[pos] = TnEntry{s, j};
                __syncwarp();
                filled = nf;
            }
            if (lane == 0) s_filled[u] = filled;
            __syncwarp();
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nu * count; e += kTnThreads) {
        const int u = e / count, r = e - u * count;
        const int64_t o = static_cast<int64_t>(u0 + u) * count + r;
        if (r < s_filled[u]) {
            out_items[o] = lists[u * count + r].j;
            out_scores[o] = lists[u * count + r].s;
        } else {
            out_items[o] = -1;
            out_scores[o] = 0.f;
        }
    }
    if (threadIdx.x < nu) out_count[u0 + threadIdx.x] = s_filled[threadIdx.x];
}

}  // namespace

size_t topn_smem_bytes(int k, int count) {
    return static_cast<size_t>(k) * (kTnTile + 4) * sizeof(float) + static_cast<size_t>(k) * kTnUsers * sizeof(float) +
           kTnUsers * (kTnTile / 32) * sizeof(uint32_t) + static_cast<size_t>(kTnUsers) * count * sizeof(TnEntry);
}

void topn_set_attributes(size_t max_smem) {
    cudaFuncSetAttribute(topn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(max_smem));
}

void launch_topn(const float* W, const float* H, int32_t n, int k, const int32_t* users, int32_t n_users,
                 const int64_t* ex_start, const int32_t* ex_items, int count, int32_t* out_items, float* out_scores,
                 int32_t* out_count, cudaStream_t s) {
    if (n_users <= 0) return;
    const int blocks = (n_users + kTnUsers - 1) / kTnUsers;
    topn_kernel<<<blocks, kTnThreads, topn_smem_bytes(k, count), s>>>(W, H, n, k, users, n_users, ex_start, ex_items,
                                                                      count, out_items, out_scores, out_count);
}

}  // namespace pmfgpu
