// flat_kernels.cu -- segmented-stream CCD++ sweeps for short-segment layouts (Yahoo-Music shape).
//
// The unit kernel (ccd_kernels.cu) gives every segment (one output's entries inside one gather
// panel) to a group of lanes; with segments of ~20 entries its per-unit overhead (claim, descriptor,
// group reduction, partial store) dominates and the loads in flight per lane are few.  Here a warp
// streams a chunk of consecutive 4-entry vectors -- one vector per lane per 32-vector block, fully
// coalesced, independent of where segments start -- and reduces each lane's partial (num, den)
// (ccd.hpp:165-171 / :188-194) with a segmented inclusive scan over the lanes.  Segment ends come from
// a bit per vector (tailbits); a segment that continues past a block is carried in registers to the
// next block.  The lane holding a segment's last vector writes its result (direct, or a partial slot
// combined by the fixed-order finalize).  The order of every sum is fixed by the layout, so results
// are deterministic.
//
// Residual passes stream the same way: kDemote  R <- R - u'_i v'_j           (ccd.hpp:213-214)
//                                        kBuild   R <- R + w_i h_j if w != 0  (ccd.hpp:142-147)
// and kBuildSweep fuses the build into the first u-sweep of a step on the CSR side, where the build's
// gathered vector h is also the sweep's v.  Each staged panel holds one vector, so panels are as wide
// as shared memory allows.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "device.hpp"

namespace pmfgpu {

namespace {

enum FlatMode { kFPlain = 0, kFDemote = 1, kFBuild = 2, kFBuildSweep = 3 };

// 1024 threads per CTA, one CTA per SM.  Round 1 measured 512 / 768-thread CTAs, more 32-vector
// blocks in flight per warp and a software-pipelined (chunk, block) sequence: all slower, removed.
constexpr int kFlatThreads = 1024;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void fbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "FW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra FW_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ void fstage(float* dst, const float* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ int idx16_get(const uint2& r, int c) {
    const uint32_t w = c < 2 ? r.x : r.y;
    return (c & 1) ? static_cast<int>(w >> 16) : static_cast<int>(w & 0xffffu);
}

// 256-bit streaming loads / stores (sm_100: LDG.E.EF.ENL2.256): a lane moves 8 residual values or
// 16 panel-local indices per instruction, the warp 1 KB, fully coalesced.
__device__ __forceinline__ void ld8(const float* p, float* r) {
    asm volatile("ld.global.cs.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
                 : "l"(p));
}
__device__ __forceinline__ void ld8u(const uint16_t* p, uint32_t* w) {
    asm volatile("ld.global.cs.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                 : "l"(p));
}
__device__ __forceinline__ void st8(float* p, const float* r) {
    asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r[0]), "f"(r[1]), "f"(r[2]),
                 "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7])
                 : "memory");
}

// One warp streams chunk [v0, v1) = units [ua, ub) (<= 32 units, <= 256 vectors).  Lane l takes 4
// consecutive vectors (16 entries) of each 128-vector block, folds them sequentially (restarting at
// every unit end), and a segmented scan over the lanes' open sums connects units that span lanes;
// the open sum at the block end is carried to the next block.  Unit descriptors (packed slot or
// output; for residual passes the output's factor) sit one per lane and are fetched by shuffles.
// A chunk's per-lane prologue: its unit descriptors (one per lane) and tail words.  The raw loaded
// fields are kept as they are and only combined where they are used (in flat_block), so a warp does
// not stall on the descriptor loads of the chunk after next while it streams the current one.
struct ChunkInfo {
    int infoA, oA;  // unit ua + lane: partial slot, or -(output + 1) for a direct write; output
    int infoB, oB;  // unit ua + 32 + lane
    float facA, facB;  // residual passes: the units' output factors
    uint32_t tw;    // tail word w0 + lane
};

// Unit descriptors of a flat layout as separate 4-byte streams (uinfo: slot or -(output + 1); uout:
// output, read by the residual passes only): the plain sweeps read 4 bytes per unit instead of the
// 16-byte Unit (12M units per Yahoo-Music sweep).
template <int FM>
__device__ __forceinline__ ChunkInfo chunk_info(const FlatChunk& ch, const int32_t* __restrict__ uinfo,
                                                const int32_t* __restrict__ uout, const uint32_t* __restrict__ tb,
                                                const SweepOperands& op) {
    constexpr bool kWrite = FM != kFPlain;
    const int lane = threadIdx.x & 31;
    ChunkInfo ci{0, 0, 0, 0, 0.f, 0.f, 0u};
    const int last = max(ch.ub - 1, 0);
    const int ua = min(ch.ua + lane, last), ub = min(ch.ua + 32 + lane, last);  // clamped: no branch
    ci.infoA = uinfo[ua];
    ci.infoB = uinfo[ub];
    if (kWrite) {
        ci.oA = uout[ua];
        ci.oB = uout[ub];
        const float* f = FM == kFDemote ? op.oa : op.ob;
        ci.facA = f[op.out_off + ci.oA];
        ci.facB = f[op.out_off + ci.oB];
    }
    const int w0 = ch.v0 >> 5;
    ci.tw = __ldg(tb + w0 + min(lane, kFlatChunkVectors / 32 + 1));
    return ci;
}

// One 128-vector block of a chunk, its residual / index vectors already loaded into r / ix.
// cn, cd: the open unit's sum carried across blocks; ucur: unit (relative to the chunk's first)
// of the block's first valid vector.
template <int FM, bool CSR>
__device__ __forceinline__ void flat_block(float (&r)[16], const uint32_t (&ix)[8], const FlatChunk& ch,
                                           const ChunkInfo& ci, int vb, float& cn, float& cd, int& ucur,
                                           float* __restrict__ R, float2* __restrict__ partial,
                                           const SweepOperands& op, const float* g0, int sent) {
    constexpr bool kReduce = FM == kFPlain || FM == kFBuildSweep;
    constexpr bool kWrite = FM != kFPlain;
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    const int v0 = ch.v0, v1 = ch.v1;
    const int infoA = ci.infoA, infoB = ci.infoB;  // slot, or -(output + 1): direct write
    const int w0 = v0 >> 5;
    const uint32_t tw = ci.tw;
    const int lv = vb + 4 * lane;
    const bool any = lv + 3 >= v0 && lv < v1;
    uint32_t vmask = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) vmask |= (lv + j >= v0 && lv + j < v1) ? (1u << j) : 0u;
    const uint32_t word = __shfl_sync(0xffffffffu, tw, ((lv >> 5) - w0) & 31);
    const uint32_t nib = (word >> (lv & 31)) & 0xfu & vmask;
    const uint32_t b0 = __ballot_sync(0xffffffffu, nib & 1u), b1 = __ballot_sync(0xffffffffu, nib & 2u);
    const uint32_t b2 = __ballot_sync(0xffffffffu, nib & 4u), b3 = __ballot_sync(0xffffffffu, nib & 8u);
    int uj = ucur + __popc(b0 & lt) + __popc(b1 & lt) + __popc(b2 & lt) + __popc(b3 & lt);
    const int ul = uj;
    // branch-free over the lane's 4 vectors: entries of vectors outside the chunk read the zero
    // sentinel slot with a zero residual (they add exactly 0 and are never stored)
    float pn[4], pd[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        pn[j] = pd[j] = 0.f;
        const bool vj = (vmask >> j) & 1u;
        float fj = 0.f;
        if (kWrite) {
            const float fa = __shfl_sync(0xffffffffu, ci.facA, uj & 31), fb = __shfl_sync(0xffffffffu, ci.facB, uj & 31);
            fj = uj < 32 ? fa : fb;
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int e = 4 * j + c;
            const uint32_t w = ix[e >> 1];
            const int gi = vj ? ((e & 1) ? static_cast<int>(w >> 16) : static_cast<int>(w & 0xffffu)) : sent;
            const float g = g0[gi];
            float rr = vj ? r[e] : 0.f;
            if (FM == kFDemote) {
                rr = __fsub_rn(rr, __fmul_rn(fj, g));
            } else if (FM == kFBuild || FM == kFBuildSweep) {
                // CSR: w = output factor, h = gathered; CSC: w = gathered, h = output factor
                const float wv = CSR ? fj : g;
                const float hv = CSR ? g : fj;
                if (wv != 0.f) rr = __fadd_rn(rr, __fmul_rn(wv, hv));
            }
            if (kReduce) {
                pn[j] = fmaf(rr, g, pn[j]);
                pd[j] = fmaf(g, g, pd[j]);
            }
            r[e] = rr;
        }
        uj += (nib >> j) & 1u;
    }
    if (kWrite && any) {
        if (vmask == 0xfu) {
            st8(R + 4 * static_cast<int64_t>(lv), r);
            st8(R + 4 * static_cast<int64_t>(lv) + 8, r + 8);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if ((vmask >> j) & 1u)
                    __stcs(reinterpret_cast<float4*>(R) + lv + j,
                           make_float4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]));
        }
    }
    if (kReduce) {
        // lane's open sum after its last unit end (all of it if none), and the segmented scan
        // of those sums: a lane with a unit end starts a new run
        float vn = 0.f, vd = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if ((nib >> j) & 1u) {
                vn = 0.f;
                vd = 0.f;
            } else {
                vn += pn[j];
                vd += pd[j];
            }
        }
        // (the sum restarts after each end: vn holds the part after the last end)
        const uint32_t fm = __ballot_sync(0xffffffffu, nib != 0u);
        const uint32_t le = fm & (lt | (1u << lane));
        const int start = le ? 31 - __clz(le) : 0;
        float in = vn, id = vd;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const float n2 = __shfl_up_sync(0xffffffffu, in, off);
            const float d2 = __shfl_up_sync(0xffffffffu, id, off);
            if (lane - off >= start) {
                in += n2;
                id += d2;
            }
        }
        if (!le) {
            in += cn;
            id += cd;
        }
        float en = __shfl_up_sync(0xffffffffu, in, 1), ed = __shfl_up_sync(0xffffffffu, id, 1);
        if (lane == 0) {
            en = cn;
            ed = cd;
        }
        // walk the lane's vectors from the open sum before it, emitting at every unit end
        int u = ul;
        const uint32_t bj[4] = {b0, b1, b2, b3};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            en += pn[j];
            ed += pd[j];
            if (!bj[j]) continue;  // warp-uniform: no unit ends at this vector slot
            const int ia = __shfl_sync(0xffffffffu, infoA, u & 31), ib = __shfl_sync(0xffffffffu, infoB, u & 31);
            const int inf = u < 32 ? ia : ib;
            if ((nib >> j) & 1u) {
                if (inf >= 0) {
                    partial[inf] = make_float2(en, ed);
                } else {
                    const float dt = __fadd_rn(op.lambda, ed);
                    op.out[op.out_off - inf - 1] = dt == 0.f ? 0.f : __fdiv_rn(en, dt);
                }
                en = 0.f;
                ed = 0.f;
                ++u;
            }
        }
        cn = __shfl_sync(0xffffffffu, in, 31);
        cd = __shfl_sync(0xffffffffu, id, 31);
    }
    ucur += __popc(b0) + __popc(b1) + __popc(b2) + __popc(b3);
}

__device__ __forceinline__ void load_block(float (&r)[16], uint32_t (&ix)[8], const FlatChunk& ch, int vb,
                                           const uint16_t* __restrict__ idx, const float* __restrict__ R) {
    const int lv = vb + 4 * (threadIdx.x & 31);
    if (lv + 3 >= ch.v0 && lv < ch.v1) {
        ld8(R + 4 * static_cast<int64_t>(lv), r);
        ld8(R + 4 * static_cast<int64_t>(lv) + 8, r + 8);
        ld8u(idx + 4 * static_cast<int64_t>(lv), ix);
    }
}

// Non-pipelined: one block's loads, then its processing.
template <int FM, bool CSR>
__device__ __forceinline__ void flat_chunk(const FlatChunk& ch, const ChunkInfo& ci,
                                           const uint16_t* __restrict__ idx, float* __restrict__ R,
                                           float2* __restrict__ partial, const SweepOperands& op, const float* g0,
                                           int sent) {
    float cn = 0.f, cd = 0.f;
    int ucur = 0;
    for (int vb = ch.v0 & ~3; vb < ch.v1; vb += 128) {
        float r[16];
        uint32_t ix[8];
        load_block(r, ix, ch, vb, idx, R);
        flat_block<FM, CSR>(r, ix, ch, ci, vb, cn, cd, ucur, R, partial, op, g0, sent);
    }
}

// Chunk claims from a piece's counter, two chunks per atomic; the next pair's atomic is issued when
// the current pair is first used, so its latency overlaps the streaming of two chunks.
struct FlatClaim {
    int* counter;
    int a;       // outstanding atomic result (lane 0)
    int second;  // second chunk of the current pair, or -1
    __device__ __forceinline__ void issue() {
        if ((threadIdx.x & 31) == 0) a = atomicAdd(counter, 2);
    }
    __device__ __forceinline__ int next() {
        if (second >= 0) {
            const int c = second;
            second = -1;
            return c;
        }
        const int b = __shfl_sync(0xffffffffu, a, 0);
        issue();
        second = b + 1;
        return b;
    }
};

template <int FM, bool CSR>
__global__ void __launch_bounds__(kFlatThreads, 1)
flat_kernel(const int32_t* __restrict__ uinfo, const int32_t* __restrict__ uout, const Piece* __restrict__ pieces, const int32_t* __restrict__ piece_start,
            const int32_t* __restrict__ panel_base, const FlatChunk* __restrict__ chunks,
            const uint32_t* __restrict__ tb, const uint16_t* __restrict__ idx, float* __restrict__ R,
            float2* __restrict__ partial, SweepOperands op, const float* __restrict__ gsrc, int32_t panel_size,
            int* __restrict__ gcnt, int32_t n_pieces, int32_t restage_min) {
    extern __shared__ __align__(16) float smem[];
    __shared__ __align__(8) uint64_t s_bar;
    __shared__ int s_victim;
    if (op.cta_clock && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        op.cta_clock[2 * blockIdx.x] = t;
    }
    if (threadIdx.x == 0) fbar_init(&s_bar);
    uint32_t phase = 0;
    const int lane = threadIdx.x & 31;
    const bool steal = gcnt != nullptr;
    const int pb = piece_start[blockIdx.x], pe = piece_start[blockIdx.x + 1];
    int cur_panel = -1, own = pb;
    for (;;) {
        int pc;
        if (own < pe) {
            pc = own++;
        } else {
            if (!steal) break;
            __syncthreads();
            if (threadIdx.x < 32) {  // join the piece with the most chunks left
                int best = -1, bestw = 0;
                for (int p = lane; p < n_pieces; p += 32) {
                    const Piece z = pieces[p];
                    int w = max(0, z.pad[1] - *(volatile int*)(gcnt + 4 * p));
                    if (z.panel != cur_panel && w < restage_min) w = 0;  // not worth restaging the panel
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
                if (lane == 0) s_victim = best;
            }
            __syncthreads();
            pc = s_victim;
            if (pc < 0) break;
        }
        const Piece pz = pieces[pc];
        __syncthreads();  // previous piece consumed
        if (pz.panel != cur_panel) {
            if (threadIdx.x == 0) {
                const int32_t gbase = panel_base[pz.panel];
                const int len = panel_base[pz.panel + 1] - gbase;
                fstage(smem, gsrc + gbase, static_cast<uint32_t>(((len + 3) & ~3) * sizeof(float)), &s_bar);
            }
            fbar_wait(&s_bar, phase);
            phase ^= 1;
            if (threadIdx.x == 0) smem[panel_size] = 0.f;  // sentinel slot of padding entries
            cur_panel = pz.panel;
            __syncthreads();
        }
        int* counter = steal ? gcnt + 4 * pc : nullptr;
        __shared__ int s_next;
        if (!steal) {
            if (threadIdx.x == 0) s_next = pz.pad[0];
            __syncthreads();
            counter = &s_next;
        }
        // Warps claim chunks from the piece's counter, pipelined three deep so that no memory
        // round trip of a chunk's prologue is exposed: while chunk i streams, chunk i+1's unit
        // descriptors / tail words, chunk i+2's descriptor and the claim of chunk i+3 are in flight.
        const int cend = pz.pad[1];
        const FlatChunk none{0, 0, 0, 0};
        // chunks are claimed in pairs (one atomic per two chunks), a pair ahead of use
        FlatClaim cl{counter, 0, -1};
        cl.issue();
        int c1 = cl.next(), c2 = cl.next();
        FlatChunk ch1 = c1 < cend ? chunks[c1] : none;
        FlatChunk ch2 = c2 < cend ? chunks[c2] : none;
        ChunkInfo ci1 = chunk_info<FM>(ch1, uinfo, uout, tb, op);
        while (c1 < cend) {
            const ChunkInfo ci2 = chunk_info<FM>(ch2, uinfo, uout, tb, op);
            const int c3 = cl.next();
            const FlatChunk ch3 = c3 < cend ? chunks[c3] : none;
            flat_chunk<FM, CSR>(ch1, ci1, idx, R, partial, op, smem, panel_size);
            c1 = c2;
            ch1 = ch2;
            ci1 = ci2;
            c2 = c3;
            ch2 = ch3;
        }
    }
    if (steal) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            s_victim = atomicAdd(gcnt + 4 * n_pieces, 1) == static_cast<int>(gridDim.x) - 1;
        }
        __syncthreads();
        if (s_victim) {
            for (int p = threadIdx.x; p < n_pieces; p += blockDim.x) gcnt[4 * p] = pieces[p].pad[0];
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

// A thief restages its panel only for a piece with at least this many chunks left (a restage is a
// 225 KB TMA copy with the whole CTA waiting; a chunk is ~1.5 us of one warp).
int flat_restage_min() {
    static const int v = [] {
        const char* e = std::getenv("PMF_STEAL_MIN");
        return e ? std::atoi(e) : 128;
    }();
    return v;
}

template <int FM, bool CSR>
void launch_flat_mode(const DevSweep& L, const SweepOperands& op, const float* gsrc, bool steal,
                      cudaStream_t s) {
    const size_t smem = static_cast<size_t>(((L.panel_size + 1) + 3) & ~3) * sizeof(float);
    flat_kernel<FM, CSR><<<L.ctas, kFlatThreads, smem, s>>>(
        L.uinfo, L.uout, L.pieces, L.piece_start, L.panel_base, L.chunks, L.tailbits, static_cast<const uint16_t*>(L.idx),
        L.R, L.partial, op, gsrc, L.panel_size, steal ? L.gcnt : nullptr, L.n_pieces, flat_restage_min());
}

template <int FM>
void set_flat_attr(size_t max_smem) {
    cudaFuncSetAttribute(flat_kernel<FM, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(max_smem));
    cudaFuncSetAttribute(flat_kernel<FM, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(max_smem));
}

bool flat_steal() {
    static const int v = [] {
        const char* e = std::getenv("PMF_STEAL");
        return e ? std::atoi(e) : 1;
    }();
    return v != 0;
}

}  // namespace

void flat_set_attributes(size_t max_smem) {
    set_flat_attr<kFPlain>(max_smem);
    set_flat_attr<kFDemote>(max_smem);
    set_flat_attr<kFBuild>(max_smem);
    set_flat_attr<kFBuildSweep>(max_smem);
}

// Flat-layout counterpart of launch_sweep: plain sweep, demote, or the promote as
// demote + (build fused into the sweep on the CSR side | build + sweep on the CSC side).
int launch_flat(const DevSweep& L, SweepMode mode, bool csr, const SweepOperands& op, cudaStream_t s) {
    if (L.n_units == 0) return 0;
    const bool st = flat_steal();
    int launched = 0;
    auto go = [&](int fm, const float* gsrc) {
        if (csr) {
            switch (fm) {
                case kFPlain: launch_flat_mode<kFPlain, true>(L, op, gsrc, st, s); break;
                case kFDemote: launch_flat_mode<kFDemote, true>(L, op, gsrc, st, s); break;
                case kFBuild: launch_flat_mode<kFBuild, true>(L, op, gsrc, st, s); break;
                default: launch_flat_mode<kFBuildSweep, true>(L, op, gsrc, st, s); break;
            }
        } else {
            switch (fm) {
                case kFPlain: launch_flat_mode<kFPlain, false>(L, op, gsrc, st, s); break;
                case kFDemote: launch_flat_mode<kFDemote, false>(L, op, gsrc, st, s); break;
                case kFBuild: launch_flat_mode<kFBuild, false>(L, op, gsrc, st, s); break;
                default: launch_flat_mode<kFBuildSweep, false>(L, op, gsrc, st, s); break;
            }
        }
        ++launched;
    };
    bool sweep = false;
    if (mode == kPlain) {
        go(kFPlain, op.gn);
        sweep = true;
    } else if (mode == kDemote) {
        go(kFDemote, op.ga);
    } else if (mode == kRmw) {
        go(kFDemote, op.ga);
        go(kFBuild, op.gb);
    } else {  // kPromote
        go(kFDemote, op.ga);
        if (csr) {
            go(kFBuildSweep, op.gb);  // h is both the build's gathered vector and the sweep's v
        } else {
            go(kFBuild, op.gb);
            go(kFPlain, op.gn);
        }
        sweep = true;
    }
    if (sweep) launched += launch_finalize(L, op, s);
    return launched;
}

}  // namespace pmfgpu
