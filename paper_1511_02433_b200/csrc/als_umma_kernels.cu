// als_umma_kernels.cu -- the ALS row solves (als.hpp:47-68, dense.hpp:35-124) with the per-row gram on the
// 5th-generation tensor cores: tcgen05.mma.kind::tf32 into TMEM accumulators.
//
// Opt-in (PMF_ALS_UMMA=1): the default ALS gram is the mma.sync kernel of als_kernels.cu, which this one
// does not beat at the BASELINE shapes -- see the note at the end of this comment.
//
// Per output row o with gathered opposing rows X (entries x k features) and ratings a, the reference
// forms G = X^T X + lambda I and b = X^T a in the working precision (FP32 here) and solves G x = b by
// Cholesky.  On sm_100a one persistent CTA per SM (16 warps) runs a warp-specialised pipeline over
// 32-entry chunks:
//
//   warp 0       producer: claims units (chunks of <= `chunk` entries of one output, LPT order) from a
//                global counter in batches and streams every chunk's indices and ratings into a ring of
//                kPF slots by cp.async (a slot's mbarrier completes when they land);
//   warps 1..4   workers: chunk c belongs to worker c % 4, which gathers its 32 opposing rows into its
//                own X stage by 16-byte cp.async (4-byte when k % 4 != 0; rows past the chunk and the
//                feature padding zero-filled), up to 3 chunks ahead, then transposes the stage into its
//                own K-major, 128B-swizzled operand tile of 128 rows x 32 entries: rows [0, kp) =
//                hi(X^T), row kp = hi(a), row kp+1 = lo(a), rows [64, 64+kp) = lo(X^T), everything else
//                zero (kp = k rounded up to 4; hi(x) = x rounded to TF32, lo(x) = x - hi(x), exact in
//                FP32) -- 4 x 4 blocks per lane, register transpose, conflict-free swizzled stores;
//   warp 5       MMA issuer: one tcgen05.mma (M = 128, N = round16(kp+2), K = 8) per 8 entries with
//                A = the whole tile and B = its first N rows, so the TMEM accumulator (lanes = tile
//                rows) holds hi^T hi (rows < 64), lo^T hi (rows >= 64) and, in columns kp / kp+1, the
//                right-hand-side terms -- the 3xTF32 products (hi*hi + hi*lo + lo*hi) come out of ONE
//                MMA per K step, hi^T lo = (lo^T hi)^T being taken in the epilogue;
//   warps 6, 7   idle (16 warps x 128 registers is the register file);
//   warps 8..15  two epilogue groups of 4 warps (one per TMEM lane quadrant): tcgen05.ld the
//                accumulator, G = D_hi + D_lo + D_lo^T (+ lambda on the diagonal) and b likewise into a
//                shared-memory system; a group dumps 4 units, then its 4 warps solve one each with the
//                register LDL^T solver (als_solve.cuh), or write the (G, b) partial of a chunk of a long
//                output for the fixed-order reduce kernel.
//
// Every ring slot, X stage and operand tile is owned by one worker, so no mbarrier is waited on by two
// warps a phase apart; every wait has a 10 s watchdog that traps.  TMEM holds 8 accumulators of 64
// columns (512 columns, one CTA per SM), so the MMA runs up to 8 units ahead of the solves.
//
// Why it is not the default (measured on the B200, profiles/r02_ncu_als_umma.txt): the tensor pipe is ~9 %
// active.  Each 32-entry chunk costs ~580 shared-memory wavefronts (cp.async gather 134, transform /
// epilogue stores 128 and loads 151, tensor-core operand reads 166 -- A is re-read by every MMA and
// N <= 48 amortises nothing; an MMA costs >= 45 cycles whatever N <= 64, profiles/
// r02_microbench_umma_rate.txt), so the kernel is bound by shared-memory traffic and hand-off latency,
// while the mma.sync kernel loads each gathered operand into registers once.  Netflix k = 40: 20.6 vs
// 15.8 ms per ALS iteration.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "als_solve.cuh"
#include "device.hpp"

namespace pmfgpu {

namespace {

constexpr int kUThreads = 512;
constexpr int kCh = 32;             // entries per chunk (4 MMA K-steps)
constexpr int kPF = 16;             // chunks of indices / ratings prefetched ahead (cp.async)
constexpr int kNTW = 4;             // gather + transform workers (warps 1..4)
constexpr int kMmaWarp = 5;
constexpr int kEpiWarp0 = 8;        // epilogue groups: warps 8..11 and 12..15 (one warp per TMEM lane quadrant)
constexpr int kSlots = 8;           // TMEM accumulators of kSlotCols columns
constexpr int kSlotCols = 64;
constexpr int kOpBytes = 128 * kCh * 4;  // 16 KB operand tile
constexpr int kLoRow = 64;          // first lo row of the tile

template <int KMAX>
struct UGeo {
    static_assert(KMAX % 8 == 0 && KMAX + 2 <= kLoRow, "hi rows + the two rating rows must fit below row 64");
    static constexpr int GS0 = (KMAX + 1 + 3) & ~3;
    static constexpr int GS = (GS0 % 8 == 0) ? GS0 + 4 : GS0;  // row stride of a system: 16-byte rows
    static constexpr int BUF = KMAX * GS + 2 * KMAX;            // gram + 1/d_j + rhs
    static constexpr int ES = KMAX + 1;                         // odd: conflict-free rows and columns
    static constexpr int NMAX = (KMAX + 2 + 15) & ~15;          // accumulator columns loaded
    static constexpr int RSMAX = KMAX + 4;                      // X stage row stride bound
    // gathered-row stages in flight: enough to cover the gather latency (~1 us at ~12 chunks / us / SM)
    // within 227 KB of shared memory
    static constexpr int NX = KMAX <= 40 ? 12 : 8;
    static constexpr int NO = kNTW;                             // operand tiles: one per worker
    static constexpr size_t OFF_X = static_cast<size_t>(NO) * kOpBytes;
    static constexpr size_t X_BYTES = static_cast<size_t>(kCh) * RSMAX * 4;
    static constexpr size_t OFF_XV = OFF_X + NX * X_BYTES;
    static constexpr size_t OFF_PI = OFF_XV + NX * kCh * 4;      // prefetch ring: indices
    static constexpr size_t OFF_PV = OFF_PI + kPF * kCh * 4;     //                ratings
    static constexpr size_t OFF_E = OFF_PV + kPF * kCh * 4;
    static constexpr size_t OFF_G = (OFF_E + 2ull * KMAX * ES * 4 + 15) & ~size_t(15);
    static constexpr size_t END = OFF_G + 8ull * BUF * 4;
    static constexpr size_t SMEM = END + 1024;  // + alignment slack for the 1 KB-aligned base
    static_assert(SMEM <= 227 * 1024, "shared memory budget");
    // every ring slot, X stage and operand tile belongs to exactly one worker (chunk c -> worker c % kNTW),
    // so no mbarrier is ever waited on by two warps a phase apart (parity waits cannot alias)
    static_assert(NX % kNTW == 0 && kPF % kNTW == 0 && NO % kNTW == 0 && kPF >= NX, "slot ownership");
};

struct ChunkMeta {
    int cnt8;   // entries rounded up to the MMA K step of 8 (-1: end of stream)
    int cnt;
    int flags;  // 1: first chunk of its unit, 2: last chunk
    int slot;   // TMEM accumulator
};
struct UnitMeta {
    int o, pslot, len, pad;  // o < 0: end of stream
};
struct PfMeta {  // a chunk of the stream (cnt -1 / -2: end of stream, first / further markers)
    int cnt, flags, slot, pad;
};

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(count));
}
// non-blocking: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t parity) {
    uint32_t r;
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(r)
        : "r"(sa(b)), "r"(parity)
        : "memory");
    return r != 0;
}
__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// Wait for the phase with this parity: test, then sleep with exponential backoff (32 ns .. max_ns; 0 = spin)
// so that waiting warps leave the issue slots to the working ones.  Watchdog: a wait longer than 10 s is a
// pipeline bug -- trap (the launch fails with an error) instead of hanging the device.
__device__ __noinline__ void mbar_wait_slow(uint64_t* b, uint32_t parity, uint32_t max_ns) {
    const uint64_t t0 = gtimer();
    uint32_t ns = 32;
    while (!mbar_test(b, parity)) {
        if (max_ns) {
            __nanosleep(ns);
            ns = min(2 * ns, max_ns);
        }
        if (gtimer() - t0 > 10000000000ull) __trap();
    }
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity, uint32_t max_ns = 0) {
    if (!mbar_test(b, parity)) mbar_wait_slow(b, parity, max_ns);
}
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, uint32_t parity, uint32_t max_ns = 1024) {
    if (!mbar_test(b, parity)) mbar_wait_slow(b, parity, max_ns);
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
// asynchronous global -> shared copies; src_bytes = 0 writes zeros
__device__ __forceinline__ void cp_async4(void* dst, const void* src, int src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(sa(dst)), "l"(src), "r"(src_bytes) : "memory");
}
// predicated, no memory clobber: completion is tracked by an mbarrier (cp_async_mbar_arrive), so the
// compiler need not reload anything around the issue
__device__ __forceinline__ void cp_async16_if(uint32_t dst, const void* src, int src_bytes, bool pred) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %3, 0;\n@p cp.async.cg.shared.global [%0], [%1], 16, %2;\n}\n" ::"r"(dst),
        "l"(src), "r"(src_bytes), "r"(static_cast<int>(pred)));
}
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
// the barrier's current phase also waits for this thread's cp.async copies issued so far
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* b) {
    asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major, 128-byte-swizzled shared-memory matrix descriptor (sm_100 format: start >> 4, LBO = 1 (unused
// for swizzled K-major), SBO = 1024 B between 8-row groups, version 1 at bit 46, layout 2 = SWIZZLE_128B
// at bit 61).  A K step of 8 TF32 entries advances the start address by 32 B inside the 1 KB atom.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    return static_cast<uint64_t>((saddr >> 4) & 0x3fff) | (static_cast<uint64_t>(1) << 16) |
           (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) |
           (static_cast<uint64_t>(2) << 61);
}

__device__ __forceinline__ float hi_tf32(float x) {
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
}

// byte offset of (row r, entries 4q..4q+3) in a 128B-swizzled K-major tile: 8-row atoms of 1 KB, rows of
// 128 B (32 entries), 16-byte chunk q stored at chunk q ^ (r % 8)
__device__ __forceinline__ uint32_t tile_off(int r, int q) {
    return (r >> 3) * 1024 + (r & 7) * 128 + ((q ^ (r & 7)) << 4);
}

// PMF_UMMA_PROFILE=1 (experiment builds only): per-warp clock64 cycles spent in each wait site / the
// solves, printed by CTA 0 at exit
#ifndef PMF_UMMA_PROFILE
#define PMF_UMMA_PROFILE 0
#endif
#if PMF_UMMA_PROFILE
#define PT(site, ...)                          \
    do {                                       \
        const long long t_ = clock64();        \
        __VA_ARGS__;                           \
        pt[site] += clock64() - t_;            \
    } while (0)
#else
#define PT(site, ...) \
    do {              \
        __VA_ARGS__;  \
    } while (0)
#endif

template <int KMAX, bool W16>
__global__ void __launch_bounds__(kUThreads, 1)
als_umma_kernel(const Unit* __restrict__ units, int32_t n_units, const int32_t* __restrict__ idx,
                const float* __restrict__ val, const float* __restrict__ opp, float* __restrict__ out,
                int32_t out_off, int k, float lambda, int weighted, float* __restrict__ partial,
                int* __restrict__ counter, int* __restrict__ status, int gs, int gb) {
    using Geo = UGeo<KMAX>;
    constexpr int GS = Geo::GS, ES = Geo::ES, NMAX = Geo::NMAX;
    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t bar_rfull[kPF], bar_rempty[kPF], bar_xfull[Geo::NX];
    __shared__ __align__(8) uint64_t bar_opfull[Geo::NO], bar_opempty[Geo::NO];
    __shared__ __align__(8) uint64_t bar_accfull[kSlots], bar_accempty[kSlots];
    __shared__ ChunkMeta xmeta[Geo::NX], opmeta[Geo::NO];
    __shared__ UnitMeta umeta[kSlots];
    __shared__ PfMeta pmeta[kPF];
    __shared__ uint32_t s_tmem;

    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int kp = (k + 3) & ~3;                           // features padded to 16 bytes
    const int rs = ((kp >> 2) & 1) ? kp : kp + 4;          // X row stride: an odd number of 16-byte pieces
    auto opbuf = [&](int t) { return smem + static_cast<size_t>(t) * kOpBytes; };
    auto xbuf = [&](int t) { return reinterpret_cast<float*>(smem + Geo::OFF_X + t * Geo::X_BYTES); };
    auto xval = [&](int t) { return reinterpret_cast<float*>(smem + Geo::OFF_XV) + t * kCh; };
    int32_t* ring_idx = reinterpret_cast<int32_t*>(smem + Geo::OFF_PI);
    float* ring_val = reinterpret_cast<float*>(smem + Geo::OFF_PV);

    // operand tiles start (and their never-written rows stay) zero
    for (int i = threadIdx.x; i < Geo::NO * kOpBytes / 16; i += kUThreads)
        reinterpret_cast<float4*>(smem)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        for (int i = 0; i < kPF; ++i) {
            mbar_init(&bar_rfull[i], 1);
            mbar_init(&bar_rempty[i], 1);
        }
        for (int i = 0; i < Geo::NX; ++i) mbar_init(&bar_xfull[i], 1);
        for (int i = 0; i < Geo::NO; ++i) {
            mbar_init(&bar_opfull[i], 1);
            mbar_init(&bar_opempty[i], 1);
        }
        for (int i = 0; i < kSlots; ++i) {
            mbar_init(&bar_accfull[i], 1);
            mbar_init(&bar_accempty[i], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;
#if PMF_UMMA_PROFILE
    long long pt[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    const long long t_start = clock64();
#endif

    if (warp == 0) {
        // ---- producer: the chunk stream ----
        // Unit claims: batches of gb consecutive (LPT-ordered) units from the global counter; lane j holds
        // the descriptor of unit u0 + j.  The next batch's descriptors and the claim after it are in
        // flight while the current batch is walked.  Chunk c's indices and ratings stream into ring slot
        // c % kPF by cp.async; the slot's mbarrier completes when they have landed.
        auto load_unit = [&](int u) {
            int4 d = make_int4(0, 0, -1, -1);
            if (u < n_units) d = *reinterpret_cast<const int4*>(units + u);
            return d;
        };
        int claim = 0, u0a = 0, u0b = 0;
        if (lane == 0) {
            u0a = atomicAdd(counter, gb);
            u0b = atomicAdd(counter, gb);
            claim = atomicAdd(counter, gb);
        }
        int cur_u0 = __shfl_sync(0xffffffffu, u0a, 0), nxt_u0 = __shfl_sync(0xffffffffu, u0b, 0);
        int4 cur_d = load_unit(lane < gb ? cur_u0 + lane : n_units);
        int4 nxt_d = load_unit(lane < gb ? nxt_u0 + lane : n_units);
        int bj = 0;  // next unit of the current batch
        bool p_active = false;
        int p_e0 = 0, p_len = 0, p_o = 0, p_ps = 0, p_base = 0, p_slot = 0;
        uint32_t pf = 0, s = 0;
        for (int ends = 0; ends < kNTW;) {
            if (!p_active && ends == 0) {
                if (bj == gb) {  // next batch
                    cur_u0 = nxt_u0;
                    cur_d = nxt_d;
                    nxt_u0 = __shfl_sync(0xffffffffu, claim, 0);
                    nxt_d = load_unit(lane < gb ? nxt_u0 + lane : n_units);
                    if (lane == 0) claim = atomicAdd(counter, gb);
                    bj = 0;
                }
                if (cur_u0 + bj < n_units) {
                    p_e0 = __shfl_sync(0xffffffffu, cur_d.x, bj);
                    p_len = __shfl_sync(0xffffffffu, cur_d.y, bj);
                    p_o = __shfl_sync(0xffffffffu, cur_d.z, bj);
                    p_ps = __shfl_sync(0xffffffffu, cur_d.w, bj);
                    p_base = 0;
                    p_active = true;
                    ++bj;
                    // a TMEM accumulator for the unit: free once the epilogue has read its previous unit
                    p_slot = s & (kSlots - 1);
                    PT(0, mbar_wait_sleep(&bar_accempty[p_slot], ((s / kSlots) & 1) ^ 1));
                    if (lane == 0) umeta[p_slot] = UnitMeta{p_o, p_ps, p_len, 0};
                    ++s;
                }
            }
            const int rsl = pf % kPF;
            PT(1, mbar_wait_sleep(&bar_rempty[rsl], ((pf / kPF) & 1) ^ 1, 256));
            if (!p_active) {
                // end of stream: one marker per worker (the first also ends the MMA's stream)
                if (lane == 0) {
                    pmeta[rsl].cnt = ends == 0 ? -1 : -2;
                    mbar_arrive(&bar_rfull[rsl]);
                }
                ++ends;
            } else {
                const int cnt = min(kCh, p_len - p_base);
                const int64_t e = static_cast<int64_t>(static_cast<uint32_t>(p_e0)) + p_base + lane;
                const bool live = lane < cnt;
                cp_async4(ring_idx + rsl * kCh + lane, live ? idx + e : idx, live ? 4 : 0);
                cp_async4(ring_val + rsl * kCh + lane, live ? val + e : val, live ? 4 : 0);
                if (lane == 0)
                    pmeta[rsl] = PfMeta{cnt, (p_base == 0 ? 1 : 0) | (p_base + kCh >= p_len ? 2 : 0), p_slot, 0};
                cp_async_mbar_arrive(&bar_rfull[rsl]);
                __syncwarp();
                if (lane == 0) mbar_arrive(&bar_rfull[rsl]);
                p_base += kCh;
                if (p_base >= p_len) p_active = false;
            }
            ++pf;
        }
        // end of stream for the epilogue groups: a terminal marker in every accumulator slot
        for (int j = 0; j < kSlots; ++j, ++s) {
            const int slot = s & (kSlots - 1);
            PT(0, mbar_wait_sleep(&bar_accempty[slot], ((s / kSlots) & 1) ^ 1));
            if (lane == 0) {
                umeta[slot] = UnitMeta{-1, -1, 0, 0};
                mbar_arrive(&bar_accfull[slot]);
            }
        }
        cp_async_wait<0>();
    } else if (warp <= kNTW) {
        // ---- workers: worker w owns chunks c = w (mod kNTW) and X stages st = w (mod kNTW) ----
        // gather: the chunk's rows into X stage c % NX by cp.async (16-byte pieces, 4-byte when k % 4 != 0;
        // rows past the chunk and feature padding zero-filled), up to NX / kNTW chunks ahead;
        // transform: X stage -> K-major hi / lo operand tile c % NO.  Item (fg, q) = features
        // 4fg..4fg+3 x entries 4q..4q+3; lanes (q & 3) + 4 (fg % 4) + 16 (q >> 2), so each 8-lane phase of
        // a 16-byte access touches 2 feature groups x 4 entry groups: conflict-free swizzled stores,
        // 2-way loads.  Group fg = kp / 4 is the ratings: rows kp (hi) and kp + 1 (lo).
        const int w = warp - 1;
        const int FG = kp >> 2;
        const int nblk = (FG + 1 + 3) >> 2;
        constexpr int MAXB = (KMAX / 4 + 1 + 3) / 4;
        const int lq = (lane & 3) | ((lane >> 4) << 2), lf = (lane >> 2) & 3;
        int xoff[MAXB];
        uint32_t toff[MAXB];
#pragma unroll
        for (int bb = 0; bb < MAXB; ++bb) {
            const int fg = 4 * bb + lf;
            xoff[bb] = 4 * lq * rs + 4 * fg;
            toff[bb] = fg < FG ? tile_off(4 * fg, lq) : tile_off(kp, lq);
        }
        // this lane's 16-byte gather pieces: piece p = 32 t + lane is row p / PR, piece p % PR
        constexpr int NT16 = (KMAX + 3) / 4;
        const int PR = kp >> 2;
        int p_row[W16 ? NT16 : 1], p_off[W16 ? NT16 : 1], p_src[W16 ? NT16 : 1];
        const char* obase = reinterpret_cast<const char*>(opp);
        const uint64_t rowbytes = static_cast<uint64_t>(k) * 4;
        if (W16) {
#pragma unroll
            for (int t = 0; t < NT16; ++t) {
                const int p = 32 * t + lane, r = p / PR, c = p - r * PR;
                p_row[t] = t < PR ? r : 32;
                p_off[t] = 4 * (r * rs + 4 * c);  // bytes
                p_src[t] = 16 * c;
            }
        }
        uint32_t ci = w, cp = w, end_c = 0xffffffffu;
        int end_kind = 0;
        for (;;) {
            while (end_c == 0xffffffffu && ci < cp + Geo::NX) {
                const int rsl = ci % kPF;
                // with gathered chunks still to transform, never block on the stream: the producer may be
                // waiting for an accumulator that those chunks complete
                if (ci != cp && !mbar_test(&bar_rfull[rsl], (ci / kPF) & 1)) break;
                PT(2, mbar_wait_sleep(&bar_rfull[rsl], (ci / kPF) & 1, 256));
                const PfMeta M = pmeta[rsl];
                if (M.cnt < 0) {
                    end_c = ci;
                    end_kind = M.cnt;
                    break;
                }
                const int st = ci % Geo::NX;
                const int cnt = M.cnt, cnt8 = (cnt + 7) & ~7;
                const int row = ring_idx[rsl * kCh + lane];
                xval(st)[lane] = ring_val[rsl * kCh + lane];
                if (lane == 0) xmeta[st] = ChunkMeta{cnt8, cnt, M.flags, M.slot};
                __syncwarp();
                if (lane == 0) mbar_arrive(&bar_rempty[rsl]);
                float* X = xbuf(st);
                if (W16) {
                    const uint32_t xs_base = sa(X);
#pragma unroll
                    for (int t = 0; t < NT16; ++t) {
                        const int r = p_row[t];
                        const int src = __shfl_sync(0xffffffffu, row, r & 31);
                        const bool live = r < cnt;
                        const char* gp = obase + static_cast<uint64_t>(static_cast<uint32_t>(live ? src : 0)) * rowbytes +
                                         p_src[t];
                        cp_async16_if(xs_base + p_off[t], gp, live ? 16 : 0, r < cnt8);
                    }
                } else {
                    // element e = 32 t + lane of the cnt8 x kp block; r = e / kp by a 20-bit reciprocal
                    const int tot = cnt8 * kp;
                    const int inv = ((1 << 20) + kp - 1) / kp;
                    for (int e0 = 0; e0 < tot; e0 += 32) {
                        const int e = e0 + lane;
                        const int r = (e * inv) >> 20, c = e - r * kp;
                        const int src = __shfl_sync(0xffffffffu, row, r & 31);
                        if (e < tot) {
                            const bool live = r < cnt && c < k;
                            cp_async4(X + r * rs + c, live ? opp + static_cast<int64_t>(src) * k + c : opp,
                                      live ? 4 : 0);
                        }
                    }
                }
                cp_async_mbar_arrive(&bar_xfull[st]);
                __syncwarp();
                if (lane == 0) mbar_arrive(&bar_xfull[st]);
                ci += kNTW;
            }
            if (cp >= end_c) {
                if (cp == end_c && end_kind == -1) {  // the stream's first end marker: end the MMA's too
                    const int ot = cp % Geo::NO;
                    PT(4, mbar_wait(&bar_opempty[ot], ((cp / Geo::NO) & 1) ^ 1));
                    if (lane == 0) {
                        opmeta[ot] = ChunkMeta{-1, -1, 0, 0};
                        mbar_arrive(&bar_opfull[ot]);
                    }
                }
                break;
            }
            const int st = cp % Geo::NX, ot = cp % Geo::NO;
            PT(3, mbar_wait_sleep(&bar_xfull[st], (cp / Geo::NX) & 1, 256));
            const ChunkMeta mt = xmeta[st];
            PT(4, mbar_wait_sleep(&bar_opempty[ot], ((cp / Geo::NO) & 1) ^ 1, 256));
            const float* X = xbuf(st);
            const float* XV = xval(st);
            uint8_t* op = opbuf(ot);
            const int Q = mt.cnt8 >> 2;
            if (lq < Q) {
#pragma unroll
                for (int bb = 0; bb < MAXB; ++bb) {
                    const int fg = 4 * bb + lf;
                    if (bb >= nblk || fg > FG) continue;
                    if (fg < FG) {
                        const float* p = X + xoff[bb];
                        const float4 v0 = *reinterpret_cast<const float4*>(p);
                        const float4 v1 = *reinterpret_cast<const float4*>(p + rs);
                        const float4 v2 = *reinterpret_cast<const float4*>(p + 2 * rs);
                        const float4 v3 = *reinterpret_cast<const float4*>(p + 3 * rs);
                        const float4 rows[4] = {make_float4(v0.x, v1.x, v2.x, v3.x), make_float4(v0.y, v1.y, v2.y, v3.y),
                                                make_float4(v0.z, v1.z, v2.z, v3.z), make_float4(v0.w, v1.w, v2.w, v3.w)};
                        // rows 4fg + j share the 1 KB atom (4fg is a multiple of 4): row offset + 128 j,
                        // chunk q ^ (row % 8)
                        const uint32_t rbase = toff[bb] & ~uint32_t(1023);
                        const int r7 = (4 * fg) & 7;
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const float4 x = rows[j];
                            const float4 h = make_float4(hi_tf32(x.x), hi_tf32(x.y), hi_tf32(x.z), hi_tf32(x.w));
                            const float4 l = make_float4(x.x - h.x, x.y - h.y, x.z - h.z, x.w - h.w);
                            const uint32_t o = rbase + (r7 + j) * 128 + ((lq ^ (r7 + j)) << 4);
                            *reinterpret_cast<float4*>(op + o) = h;
                            *reinterpret_cast<float4*>(op + o + 8 * 1024) = l;
                        }
                    } else {
                        const float4 x = *reinterpret_cast<const float4*>(XV + 4 * lq);
                        const float4 h = make_float4(hi_tf32(x.x), hi_tf32(x.y), hi_tf32(x.z), hi_tf32(x.w));
                        const float4 l = make_float4(x.x - h.x, x.y - h.y, x.z - h.z, x.w - h.w);
                        *reinterpret_cast<float4*>(op + toff[bb]) = h;
                        *reinterpret_cast<float4*>(op + tile_off(kp + 1, lq)) = l;
                    }
                }
            }
            if (lane == 0) opmeta[ot] = mt;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_opfull[ot]);
            cp += kNTW;
        }
    } else if (warp > kMmaWarp && warp < kEpiWarp0) {
        // warps 6, 7: no role (the register file sizes 16 warps of 128 registers; a fifth worker would
        // share slots with another and a third epilogue group would not fit in TMEM)
    } else if (warp == kMmaWarp) {
        // ---- MMA issuer: D[slot] (+)= tile (128 x 8) . tile[0:N]^T per K step ----
        // descriptors precomputed (a K step adds 32 B >> 4 = 2 to the start-address field), up to four
        // MMAs per chunk issued back to back by one elected lane: ~45 cycles each at N <= 64 (measured,
        // scripts/micro/umma_rate.cu)
        const int N = (kp + 2 + 15) & ~15;
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
                               (static_cast<uint32_t>(128 >> 4) << 24);
        const uint64_t desc0 = sw128_desc(sa(opbuf(0)));
        uint32_t os = 0, s = 0;
        for (;;) {
            const int ot = os % Geo::NO;
            PT(5, mbar_wait(&bar_opfull[ot], (os / Geo::NO) & 1));
            const ChunkMeta mt = opmeta[ot];
            if (mt.cnt8 < 0) break;
            const bool first = mt.flags & 1;
            if (first) PT(6, mbar_wait_sleep(&bar_accempty[mt.slot], ((s / kSlots) & 1) ^ 1, 256));
            tc_fence_after();
            if (lane == 0) {
                // one asm block: the operands go to uniform registers once per chunk
                const uint64_t desc = desc0 + static_cast<uint64_t>(ot * (kOpBytes >> 4));
                const uint32_t d = tmem + static_cast<uint32_t>(mt.slot * kSlotCols);
                asm volatile(
                    "{\n.reg .pred p0, p1, p2, p3, p4;\n"
                    "setp.eq.b32 p0, %4, 0;\n"
                    "setp.gt.s32 p1, %5, 8;\n"
                    "setp.gt.s32 p2, %5, 16;\n"
                    "setp.gt.s32 p3, %5, 24;\n"
                    "setp.ne.b32 p4, %9, 0;\n"
                    "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %1, %3, p0;\n"
                    "@p1 tcgen05.mma.cta_group::1.kind::tf32 [%0], %2, %2, %3, 1;\n"
                    "@p2 tcgen05.mma.cta_group::1.kind::tf32 [%0], %6, %6, %3, 1;\n"
                    "@p3 tcgen05.mma.cta_group::1.kind::tf32 [%0], %7, %7, %3, 1;\n"
                    "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%8];\n"
                    "@p4 tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%10];\n"
                    "}\n" ::"r"(d),
                    "l"(desc), "l"(desc + 2), "r"(idesc), "r"(first ? 1 : 0), "r"(mt.cnt8), "l"(desc + 4), "l"(desc + 6),
                    "r"(sa(&bar_opempty[ot])), "r"(mt.flags & 2), "r"(sa(&bar_accfull[mt.slot]))
                    : "memory");
            }
            __syncwarp();
            if (first) ++s;
            ++os;
        }
    } else {
        // ---- epilogue groups: accumulator -> (G + lambda I, b) -> solve ----
        const int g = (warp - kEpiWarp0) >> 2, qd = warp & 3;
        float* E = reinterpret_cast<float*>(smem + Geo::OFF_E) + g * KMAX * ES;
        auto gbuf = [&](int j) { return reinterpret_cast<float*>(smem + Geo::OFF_G) + (4 * g + j) * Geo::BUF; };
        const int m = 32 * (qd & 1) + lane;  // hi row (qd < 2) or lo row (qd >= 2) of this lane
        const int nchunks = (kp + 2 + 15) >> 4;
        const int stride = k * k + k + 1;
        for (int b = 0;; ++b) {
            int n_in = 0, my_o = -1, my_len = 0;
            bool done = false, my_solve = false;
            for (int j = 0; j < 4; ++j) {
                const int slot = 4 * g + j;
                PT(7, mbar_wait_sleep(&bar_accfull[slot], b & 1));
                const UnitMeta um = umeta[slot];
                if (um.o < 0) {
                    done = true;
                    break;
                }
                tc_fence_after();
                uint32_t v[NMAX];
                const uint32_t ta = tmem + (static_cast<uint32_t>(32 * qd) << 16) + slot * kSlotCols;
#pragma unroll
                for (int c = 0; c < NMAX / 16; ++c)
                    if (c < nchunks)
                        asm volatile(
                            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
                            "%15}, [%16];"
                            : "=r"(v[16 * c + 0]), "=r"(v[16 * c + 1]), "=r"(v[16 * c + 2]), "=r"(v[16 * c + 3]),
                              "=r"(v[16 * c + 4]), "=r"(v[16 * c + 5]), "=r"(v[16 * c + 6]), "=r"(v[16 * c + 7]),
                              "=r"(v[16 * c + 8]), "=r"(v[16 * c + 9]), "=r"(v[16 * c + 10]), "=r"(v[16 * c + 11]),
                              "=r"(v[16 * c + 12]), "=r"(v[16 * c + 13]), "=r"(v[16 * c + 14]), "=r"(v[16 * c + 15])
                            : "r"(ta + 16 * c));
                    else
#pragma unroll
                        for (int x = 0; x < 16; ++x) v[16 * c + x] = 0u;
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                // lo rows: E[m][n] = (lo^T hi)[m][n], n < k, and E[m][k] = (lo^T hi(a))[m] (column kp)
                if (qd >= 2 && m < k) {
#pragma unroll
                    for (int n = 0; n < NMAX; ++n) {
                        if (n < k) E[m * ES + n] = __uint_as_float(v[n]);
                        if (n == kp) E[m * ES + k] = __uint_as_float(v[n]);
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bar_accempty[slot]);
                named_sync(1 + g, 128);
                if (qd < 2 && m < k) {
                    // G[m][n] = hi^T hi + lo^T hi + (lo^T hi)^T; b[m] = hi^T hi(a) + hi^T lo(a) + lo^T hi(a)
                    float rhs = E[m * ES + k];
#pragma unroll
                    for (int n = 0; n < NMAX; ++n)
                        if (n == kp || n == kp + 1) rhs += __uint_as_float(v[n]);
                    if (um.pslot >= 0) {
                        float* P = partial + static_cast<int64_t>(um.pslot) * stride;
#pragma unroll
                        for (int n = 0; n < KMAX; ++n)
                            if (n < k) P[m * k + n] = __uint_as_float(v[n]) + E[m * ES + n] + E[n * ES + m];
                        P[k * k + m] = rhs;
                        if (m == 0) P[k * k + k] = static_cast<float>(um.len);
                    } else {
                        float* G = gbuf(j);
                        const float ridge = weighted ? lambda * static_cast<float>(um.len) : lambda;
#pragma unroll
                        for (int n = 0; n < KMAX; n += 4) {
                            float4 w;
                            float* wp = reinterpret_cast<float*>(&w);
#pragma unroll
                            for (int x = 0; x < 4; ++x) {
                                const int nn = n + x;
                                const float gv = __uint_as_float(v[nn]) + E[m * ES + nn] + E[nn * ES + m];
                                wp[x] = nn < k ? (nn == m ? gv + ridge : gv) : 0.f;
                            }
                            *reinterpret_cast<float4*>(G + m * GS + n) = w;
                        }
                        G[KMAX * GS + KMAX + m] = rhs;
                    }
                }
                if (j == qd) {
                    my_o = um.o;
                    my_len = um.len;
                    my_solve = um.pslot < 0;
                }
                n_in = j + 1;
                named_sync(1 + g, 128);  // E free for the next unit; the systems complete
            }
            (void)my_len;
#if PMF_UMMA_PROFILE
            const long long ts_ = clock64();
#endif
            if (qd < n_in && my_solve) {
                float* G = gbuf(qd);
                float* dst = out + static_cast<int64_t>(out_off + my_o) * k;
                float b0 = lane < k ? G[KMAX * GS + KMAX + lane] : 0.f;
                float b1 = lane + 32 < k ? G[KMAX * GS + KMAX + lane + 32] : 0.f;
                if (gs) {
                    float x0 = lane < k ? dst[lane] : 0.f, x1 = lane + 32 < k ? dst[lane + 32] : 0.f;
                    warp_gauss_seidel<KMAX, GS>(G, k, b0, b1, x0, x1);
                    b0 = x0;
                    b1 = x1;
                } else if (!warp_ldl_solve<KMAX>(G, GS, G + KMAX * GS + KMAX, k, G + KMAX * GS, b0, b1)) {
                    if (lane == 0) atomicExch(status, 4);
                    b0 = b1 = 0.f;
                }
                if (lane < k) dst[lane] = b0;
                if (lane + 32 < k) dst[lane + 32] = b1;
            }
#if PMF_UMMA_PROFILE
            pt[8] += clock64() - ts_;
#endif
            PT(9, named_sync(1 + g, 128));  // systems free for the next batch
            if (done) break;
        }
    }
#if PMF_UMMA_PROFILE
    if (blockIdx.x == 0 && lane == 0)
        printf("umma-prof warp %2d total %lld | p_acc %lld p_rempty %lld w_rfull %lld w_xfull %lld w_opempty %lld "
               "m_opfull %lld m_acc %lld e_accfull %lld e_solve %lld e_bar %lld\n",
               warp, clock64() - t_start, pt[0], pt[1], pt[2], pt[3], pt[4], pt[5], pt[6], pt[7], pt[8], pt[9]);
#endif
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int KMAX>
void launch_umma_k(const DevAls& L, const float* opp, float* out, int32_t out_off, int k, float lambda, bool weighted,
                   int* d_counter, int* d_status, int sm_count, cudaStream_t s, bool gs) {
    const int blocks = std::max(1, std::min(sm_count, L.n_units));
    // claim batch: ~64 claims per CTA at least (units are LPT-ordered, so a batch is units of similar
    // length), at most one unit per lane
    const int gb = std::max(1, std::min(32, L.n_units / (64 * std::max(1, blocks))));
    // 16-byte row pieces need 16-byte aligned rows
    if (k % 4 == 0 && (reinterpret_cast<uintptr_t>(opp) & 15) == 0)
        als_umma_kernel<KMAX, true><<<blocks, kUThreads, UGeo<KMAX>::SMEM, s>>>(
            L.units, L.n_units, L.idx, L.val, opp, out, out_off, k, lambda, weighted ? 1 : 0, L.partial, d_counter,
            d_status, gs ? 1 : 0, gb);
    else
        als_umma_kernel<KMAX, false><<<blocks, kUThreads, UGeo<KMAX>::SMEM, s>>>(
            L.units, L.n_units, L.idx, L.val, opp, out, out_off, k, lambda, weighted ? 1 : 0, L.partial, d_counter,
            d_status, gs ? 1 : 0, gb);
}

template <int KMAX>
void set_attr_umma() {
    cudaFuncSetAttribute(als_umma_kernel<KMAX, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(UGeo<KMAX>::SMEM));
    cudaFuncSetAttribute(als_umma_kernel<KMAX, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(UGeo<KMAX>::SMEM));
}

}  // namespace

bool als_umma_supported(int k) { return k >= 1 && k <= 48; }

void als_umma_set_attributes() {
    set_attr_umma<16>();
    set_attr_umma<32>();
    set_attr_umma<40>();
    set_attr_umma<48>();
}

// The gram kernel of one ALS half (the caller resets *d_counter); returns false when k is out of range.
bool launch_als_umma(const DevAls& L, const float* opp, int64_t n_opp, float* out, int32_t out_off, int k,
                     float lambda, bool weighted, int* d_counter, int* d_status, int sm_count, cudaStream_t s,
                     bool gs) {
    (void)n_opp;
    if (k <= 16) launch_umma_k<16>(L, opp, out, out_off, k, lambda, weighted, d_counter, d_status, sm_count, s, gs);
    else if (k <= 32) launch_umma_k<32>(L, opp, out, out_off, k, lambda, weighted, d_counter, d_status, sm_count, s, gs);
    else if (k <= 40) launch_umma_k<40>(L, opp, out, out_off, k, lambda, weighted, d_counter, d_status, sm_count, s, gs);
    else if (k <= 48) launch_umma_k<48>(L, opp, out, out_off, k, lambda, weighted, d_counter, d_status, sm_count, s, gs);
    else return false;
    return true;
}

}  // namespace pmfgpu
