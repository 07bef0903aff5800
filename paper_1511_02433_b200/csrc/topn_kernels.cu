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

#include <cub/device/device_segmented_radix_sort.cuh>

#include <algorithm>
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

// ---- wide path: any count / any k (model.hpp:172-209 accepts both) -------------------------------
// A batch of users at a time: every item scored with predict()'s roundings, rated items' sort keys
// forced below every score, then one stable segmented radix sort (descending) per user over
// order-preserving keys -- -0 is keyed as +0, so equal scores keep ascending item order exactly as
// the reference's comparator (a.second != b.second ? a.second > b.second : a.first < b.first).

__device__ __forceinline__ uint32_t score_key(float s) {
    const uint32_t b = s == 0.f ? 0u : __float_as_uint(s);  // -0 == +0
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__global__ void topn_score_kernel(const float* __restrict__ W, const float* __restrict__ H, int32_t n, int k,
                                  const int32_t* __restrict__ users, float* __restrict__ scores,
                                  uint32_t* __restrict__ keys, int32_t* __restrict__ items) {
    const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const int b = blockIdx.y;
    const float* w = W + static_cast<int64_t>(users[b]) * k;
    const float* h = H + static_cast<int64_t>(j) * k;
    float acc = 0.f;
    for (int t = 0; t < k; ++t) acc = __fadd_rn(acc, __fmul_rn(w[t], h[t]));
    const int64_t o = static_cast<int64_t>(b) * n + j;
    scores[o] = acc;
    keys[o] = score_key(acc);
    items[o] = j;
}

__global__ void topn_exclude_kernel(const int64_t* __restrict__ ex_start, const int32_t* __restrict__ ex_items,
                                    int32_t n, uint32_t* __restrict__ keys, int32_t* __restrict__ excluded,
                                    int32_t* __restrict__ seg) {
    const int b = blockIdx.x;
    __shared__ int cnt;
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    int mine = 0;
    for (int64_t p = ex_start[b] + threadIdx.x; p < ex_start[b + 1]; p += blockDim.x) {
        const int32_t j = ex_items[p];
        if (j >= 0 && j < n) {
            keys[static_cast<int64_t>(b) * n + j] = 0u;  // below every score key
            ++mine;
        }
    }
    atomicAdd(&cnt, mine);
    __syncthreads();
    if (threadIdx.x == 0) {
        excluded[b] = cnt;
        seg[b] = b * n;
        if (b == gridDim.x - 1) seg[b + 1] = (b + 1) * n;
    }
}

__global__ void topn_emit_kernel(const float* __restrict__ scores, const int32_t* __restrict__ sorted_items,
                                 const int32_t* __restrict__ excluded, int32_t n, int count,
                                 int32_t* __restrict__ out_items, float* __restrict__ out_scores,
                                 int32_t* __restrict__ out_count) {
    const int b = blockIdx.x;
    const int keep = min(count, n - excluded[b]);
    for (int r = threadIdx.x; r < count; r += blockDim.x) {
        const int64_t o = static_cast<int64_t>(b) * count + r;
        if (r < keep) {
            const int32_t j = sorted_items[static_cast<int64_t>(b) * n + r];
            out_items[o] = j;
            out_scores[o] = scores[static_cast<int64_t>(b) * n + j];
        } else {
            out_items[o] = -1;
            out_scores[o] = 0.f;
        }
    }
    if (threadIdx.x == 0) out_count[b] = keep;
}

struct WideScratch {
    float* scores;
    uint32_t *keys, *keys_out;
    int32_t *items, *items_out, *excluded, *seg;
    void* temp;
    size_t temp_bytes;
};

WideScratch carve(void* base, int32_t n, int batch, size_t temp_bytes) {
    auto* p = static_cast<char*>(base);
    const size_t e = static_cast<size_t>(batch) * n;
    auto take = [&](size_t bytes) {
        char* q = p;
        p += (bytes + 255) & ~size_t(255);
        return q;
    };
    WideScratch w;
    w.scores = reinterpret_cast<float*>(take(e * 4));
    w.keys = reinterpret_cast<uint32_t*>(take(e * 4));
    w.keys_out = reinterpret_cast<uint32_t*>(take(e * 4));
    w.items = reinterpret_cast<int32_t*>(take(e * 4));
    w.items_out = reinterpret_cast<int32_t*>(take(e * 4));
    w.excluded = reinterpret_cast<int32_t*>(take(static_cast<size_t>(batch) * 4));
    w.seg = reinterpret_cast<int32_t*>(take((static_cast<size_t>(batch) + 1) * 4));
    w.temp = take(temp_bytes);
    w.temp_bytes = temp_bytes;
    return w;
}

size_t sort_temp_bytes(int32_t n, int batch) {
    size_t bytes = 0;
    cub::DeviceSegmentedRadixSort::SortPairsDescending(nullptr, bytes, static_cast<const uint32_t*>(nullptr),
                                                       static_cast<uint32_t*>(nullptr),
                                                       static_cast<const int32_t*>(nullptr),
                                                       static_cast<int32_t*>(nullptr), batch * n, batch,
                                                       static_cast<const int32_t*>(nullptr),
                                                       static_cast<const int32_t*>(nullptr));
    return bytes;
}

}  // namespace

int topn_wide_batch(int32_t n) {
    const int64_t per_user = std::max<int64_t>(1, 24 * static_cast<int64_t>(n));
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(4096, (int64_t(768) << 20) / per_user)));
}

size_t topn_wide_scratch_bytes(int32_t n, int batch) {
    const size_t e = static_cast<size_t>(batch) * std::max(n, 1);
    return 5 * ((e * 4 + 255) & ~size_t(255)) + 2 * 256 + static_cast<size_t>(batch + 1) * 8 +
           sort_temp_bytes(std::max(n, 1), batch) + 256;
}

cudaError_t launch_topn_wide(const float* W, const float* H, int32_t n, int k, const int32_t* users, int32_t n_users,
                             const int64_t* ex_start, const int32_t* ex_items, int count, int32_t* out_items,
                             float* out_scores, int32_t* out_count, void* scratch, int batch, cudaStream_t s) {
    if (n_users <= 0) return cudaSuccess;
    if (n <= 0) {  // nothing to rank: every list is empty
        cudaMemsetAsync(out_count, 0, sizeof(int32_t) * n_users, s);
        cudaMemsetAsync(out_scores, 0, sizeof(float) * static_cast<size_t>(n_users) * count, s);
        return cudaMemsetAsync(out_items, 0xff, sizeof(int32_t) * static_cast<size_t>(n_users) * count, s);
    }
    const size_t tb = sort_temp_bytes(n, batch);
    WideScratch w = carve(scratch, n, batch, tb);
    for (int32_t u0 = 0; u0 < n_users; u0 += batch) {
        const int B = std::min<int32_t>(batch, n_users - u0);
        topn_score_kernel<<<dim3((n + 255) / 256, B), 256, 0, s>>>(W, H, n, k, users + u0, w.scores, w.keys, w.items);
        topn_exclude_kernel<<<B, 256, 0, s>>>(ex_start + u0, ex_items, n, w.keys, w.excluded, w.seg);
        size_t bytes = w.temp_bytes;
        const cudaError_t e = cub::DeviceSegmentedRadixSort::SortPairsDescending(
            w.temp, bytes, w.keys, w.keys_out, w.items, w.items_out, B * n, B, w.seg, w.seg + 1, 0, 32, s);
        if (e != cudaSuccess) return e;
        topn_emit_kernel<<<B, 256, 0, s>>>(w.scores, w.items_out, w.excluded, n, count,
                                           out_items + static_cast<int64_t>(u0) * count,
                                           out_scores + static_cast<int64_t>(u0) * count, out_count + u0);
    }
    return cudaGetLastError();
}

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
