// pmf_gpu.cu -- C-ABI implementation: device contexts, CCD++ and ALS drivers, metrics, stage-level
// entry points.  Mirrors the reference drivers ccdpp_train (ccd.hpp:349-404) and als_train
// (als.hpp:188-233); the per-stage BSP barriers of the reference (runtime.hpp:177-203) become
// kernel boundaries in one CUDA stream, and a whole CCD++ outer iteration is captured once as a
// CUDA graph.  Multi-GPU contexts own a CSR row block and a CSC column block (runtime.hpp:91-136)
// and all-gather u / v (CCD++) or W / H blocks (ALS) over NCCL.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <future>
#include <map>
#include <mutex>
#include <numeric>
#include <thread>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pmf_gpu.h"
#include "device.hpp"
#include "layout.hpp"

namespace pmfgpu {

thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

struct PmfError : std::runtime_error {
    pmf_status st;
    PmfError(pmf_status s, const std::string& m) : std::runtime_error(m), st(s) {}
};

#define CUDA_TRY(x)                                                                                  \
    do {                                                                                             \
        cudaError_t e_ = (x);                                                                        \
        if (e_ != cudaSuccess)                                                                       \
            throw PmfError(PMF_RUNTIME_ERROR, std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                                  " at " #x);                                        \
    } while (0)

#define NCCL_TRY(x)                                                                                  \
    do {                                                                                             \
        ncclResult_t r_ = (x);                                                                       \
        if (r_ != ncclSuccess)                                                                       \
            throw PmfError(PMF_RUNTIME_ERROR, std::string("NCCL error: ") + ncclGetErrorString(r_) + \
                                                  " at " #x);                                        \
    } while (0)

template <class F>
pmf_status guard(F&& f) {
    try {
        f();
        return PMF_OK;
    } catch (const PmfError& e) {
        g_err = e.what();
        return e.st;
    } catch (const std::bad_alloc&) {
        g_err = "host out of memory";
        return PMF_RUNTIME_ERROR;
    } catch (const std::exception& e) {
        g_err = e.what();
        return PMF_RUNTIME_ERROR;
    }
}

[[noreturn]] void invalid(const std::string& m) { throw PmfError(PMF_INVALID_ARGUMENT, m); }

// Shared memory a sweep may stage per CTA.  Shared memory and L1 share 256 KB per SM and the
// carve-out is picked from the CTA's request: up to the 196 KB configuration the streaming loads keep
// ~60 KB of L1 and reach 7.1 TB/s next to random panel gathers; the 228 KB configuration leaves
// ~28 KB and drops to 5.6 TB/s (scripts/micro/lds_gather.cu).  Only sweeps that stage one panel
// this wide pay it (the fused promote; Yahoo-width plain panels, where longer segments win).
// PMF_SMEM_BUDGET_KB overrides.
constexpr int kSmemMax = 220 * 1024;
int smem_budget() {
    static const int b = [] {
        const char* e = std::getenv("PMF_SMEM_BUDGET_KB");
        const int kb = e ? std::atoi(e) : 220;
        return std::max(16, std::min(kb, kSmemMax / 1024)) * 1024;
    }();
    return b;
}

constexpr size_t kStreamSlack = 64;  // entries of slack after the residual / index streams

// ---- pinned staging ----------------------------------------------------------------------------
// Host <-> device copies of large pageable buffers go through two 32 MB pinned buffers: a chunk is
// memcpy'd into one (host threads) while the other is on the copy engine, which runs at PCIe speed
// instead of the driver's pageable path (~8 GB/s measured).  Process-wide, allocated on first use.
struct PinnedStage {
    static constexpr size_t kChunk = 32u << 20;
    std::mutex mu;
    void* buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    int device = -1;
    void ensure() {
        int d = 0;
        CUDA_TRY(cudaGetDevice(&d));
        if (buf[0] && d == device) return;
        release();
        for (int i = 0; i < 2; ++i) {
            CUDA_TRY(cudaHostAlloc(&buf[i], kChunk, cudaHostAllocDefault));
            CUDA_TRY(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
        }
        device = d;
    }
    void release() {
        for (int i = 0; i < 2; ++i) {
            if (ev[i]) cudaEventDestroy(ev[i]);
            if (buf[i]) cudaFreeHost(buf[i]);
            ev[i] = nullptr;
            buf[i] = nullptr;
        }
    }
};
PinnedStage& pinned_stage() {
    static PinnedStage* s = new PinnedStage();  // never destroyed: outlives every context
    return *s;
}
constexpr size_t kStageMin = 4u << 20;  // smaller copies go straight through the driver

void par_memcpy(void* dst, const void* src, size_t bytes) {
    constexpr int T = 8;
    std::thread ts[T];
    for (int t = 0; t < T; ++t) {
        const size_t o0 = bytes * t / T & ~size_t(63), o1 = t == T - 1 ? bytes : (bytes * (t + 1) / T & ~size_t(63));
        ts[t] = std::thread([=] {
            std::memcpy(static_cast<char*>(dst) + o0, static_cast<const char*>(src) + o0, o1 - o0);
        });
    }
    for (auto& t : ts) t.join();
}

// Page-locked host blocks for the layout arrays (HostAllocHooks, layout.hpp): the layout builder fills
// them directly and the upload is a plain DMA (no staging memcpy).  Blocks return to this cache when a
// layout is freed and serve the next context's layouts (pinning memory costs ~0.1-0.2 s per GB; a
// caching host allocator as deep-learning runtimes keep).  Off with PMF_NO_ALLOC_CACHE=1;
// pmf_release_cached_memory frees the idle blocks.
struct PinnedPool {
    std::mutex mu;
    std::multimap<size_t, void*> idle;  // bytes -> block
    std::map<uintptr_t, size_t> all;    // every block (idle or in use): start -> bytes
    void* take(size_t bytes) {
        std::lock_guard<std::mutex> lk(mu);
        auto it = idle.lower_bound(bytes);
        if (it != idle.end() && it->first <= bytes + bytes / 4) {
            void* p = it->second;
            idle.erase(it);
            return p;
        }
        void* p = nullptr;
        if (cudaHostAlloc(&p, bytes, cudaHostAllocDefault) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        all.emplace(reinterpret_cast<uintptr_t>(p), bytes);
        return p;
    }
    void give(void* p) {
        std::lock_guard<std::mutex> lk(mu);
        idle.emplace(all.at(reinterpret_cast<uintptr_t>(p)), p);
    }
    bool contains(const void* p, size_t bytes) {
        std::lock_guard<std::mutex> lk(mu);
        const uintptr_t a = reinterpret_cast<uintptr_t>(p);
        auto it = all.upper_bound(a);
        if (it == all.begin()) return false;
        --it;
        return a + bytes <= it->first + it->second;
    }
    int64_t release_idle() {
        std::lock_guard<std::mutex> lk(mu);
        int64_t b = 0;
        for (auto& kv : idle) {
            cudaFreeHost(kv.second);
            all.erase(reinterpret_cast<uintptr_t>(kv.second));
            b += static_cast<int64_t>(kv.first);
        }
        idle.clear();
        return b;
    }
};
PinnedPool& pinned_pool() {
    static PinnedPool* p = new PinnedPool();  // never destroyed: blocks live until process exit
    return *p;
}
void* pinned_hook_alloc(size_t bytes) { return pinned_pool().take(bytes); }
void pinned_hook_free(void* p, size_t) { pinned_pool().give(p); }

double now_s();
double g_alloc_s = 0, g_h2d_s = 0;  // PMF_VERBOSE setup breakdown (host seconds in cudaMalloc / staged_h2d)

// Host -> device on stream s (returns once the host data has been consumed).
void staged_h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    struct Clock {
        double t0 = now_s();
        ~Clock() { g_h2d_s += now_s() - t0; }
    } clk;
    if (bytes < kStageMin || pinned_pool().contains(src, bytes)) {
        // small, or already page-locked (a pooled layout array: the caller keeps it alive until the
        // stream has been synchronised)
        CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        return;
    }
    PinnedStage& st = pinned_stage();
    std::lock_guard<std::mutex> lk(st.mu);
    st.ensure();
    int i = 0;
    for (size_t off = 0; off < bytes; off += PinnedStage::kChunk, i ^= 1) {
        const size_t len = std::min(PinnedStage::kChunk, bytes - off);
        CUDA_TRY(cudaEventSynchronize(st.ev[i]));  // the buffer's previous copy has finished
        par_memcpy(st.buf[i], static_cast<const char*>(src) + off, len);
        CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(dst) + off, st.buf[i], len, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaEventRecord(st.ev[i], s));
    }
}

// Device -> host, synchronous (stream s is synchronized).
void staged_d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes < kStageMin) {
        CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        return;
    }
    PinnedStage& st = pinned_stage();
    std::lock_guard<std::mutex> lk(st.mu);
    st.ensure();
    size_t off[2] = {0, 0}, len[2] = {0, 0};
    int i = 0;
    auto drain = [&](int b) {
        if (!len[b]) return;
        CUDA_TRY(cudaEventSynchronize(st.ev[b]));
        par_memcpy(static_cast<char*>(dst) + off[b], st.buf[b], len[b]);
        len[b] = 0;
    };
    for (size_t o = 0; o < bytes; o += PinnedStage::kChunk, i ^= 1) {
        drain(i);
        off[i] = o;
        len[i] = std::min(PinnedStage::kChunk, bytes - o);
        CUDA_TRY(cudaMemcpyAsync(st.buf[i], static_cast<const char*>(src) + o, len[i], cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaEventRecord(st.ev[i], s));
    }
    drain(i ^ 1);
    drain(i);
}

// ---- device memory -----------------------------------------------------------------------------
// Process-wide cache of device blocks (a caching allocator, as deep-learning runtimes keep): a
// context's blocks come back here when it is destroyed and serve the next context's allocations of
// the same size class, so creating and destroying contexts does not pay cudaFree -- which
// synchronises the device and was measured at up to 0.7 s for 411 MB blocks when the driver releases
// the memory (scripts/micro/malloc_cost.cu) -- inside a caller's timed region.  PMF_NO_ALLOC_CACHE=1
// turns it off; a failing cudaMalloc flushes the cache and retries.
struct BlockCache {
    std::mutex mu;
    std::multimap<std::pair<int, size_t>, void*> blocks;  // (device, bytes) -> block
    static bool enabled() {
        static const bool on = std::getenv("PMF_NO_ALLOC_CACHE") == nullptr;
        return on;
    }
    static size_t size_class(size_t b) {
        const size_t g = b < (size_t(1) << 20) ? 512 : (size_t(2) << 20);
        return (b + g - 1) / g * g;
    }
    // a cached block of the class or up to 1/4 larger; returns its size in *got
    void* take(int dev, size_t bytes, size_t* got) {
        std::lock_guard<std::mutex> lk(mu);
        auto it = blocks.lower_bound({dev, bytes});
        if (it == blocks.end() || it->first.first != dev || it->first.second > bytes + bytes / 4) return nullptr;
        void* p = it->second;
        *got = it->first.second;
        blocks.erase(it);
        return p;
    }
    void give(int dev, size_t bytes, void* p) {
        std::lock_guard<std::mutex> lk(mu);
        blocks.emplace(std::make_pair(dev, bytes), p);
    }
    int64_t flush() {
        std::lock_guard<std::mutex> lk(mu);
        int cur = 0;
        cudaGetDevice(&cur);
        int64_t bytes = 0;
        for (auto& kv : blocks) {
            cudaSetDevice(kv.first.first);
            cudaFree(kv.second);
            bytes += static_cast<int64_t>(kv.first.second);
        }
        blocks.clear();
        cudaSetDevice(cur);
        return bytes;
    }
};
BlockCache& block_cache() {
    static BlockCache* c = new BlockCache();  // never destroyed: blocks live until process exit
    return *c;
}

struct DevMem {
    struct Block {
        void* p;
        size_t bytes;
        int dev;
    };
    std::vector<Block> blocks;
    template <class T>
    T* alloc(size_t count, bool zero = true) {
        if (count == 0) count = 1;
        const double t0 = now_s();
        int dev = 0;
        CUDA_TRY(cudaGetDevice(&dev));
        const bool cache = BlockCache::enabled();
        size_t bytes = cache ? BlockCache::size_class(count * sizeof(T)) : count * sizeof(T);
        void* p = cache ? block_cache().take(dev, bytes, &bytes) : nullptr;
        if (!p) {
            cudaError_t e = cudaMalloc(&p, bytes);
            if (e == cudaErrorMemoryAllocation && cache) {
                cudaGetLastError();
                block_cache().flush();
                e = cudaMalloc(&p, bytes);
            }
            CUDA_TRY(e);
        }
        g_alloc_s += now_s() - t0;
        blocks.push_back(Block{p, bytes, dev});
        if (zero) CUDA_TRY(cudaMemset(p, 0, count * sizeof(T)));
        return static_cast<T*>(p);
    }
    template <class T>
    T* upload(const std::vector<T>& v, cudaStream_t s, int64_t* h2d) {
        T* p = alloc<T>(v.size(), false);
        if (!v.empty()) staged_h2d(p, v.data(), v.size() * sizeof(T), s);
        if (h2d) *h2d += static_cast<int64_t>(v.size() * sizeof(T));
        return p;
    }
    template <class T>
    T* upload(const PodBuf<T>& v, cudaStream_t s, int64_t* h2d, size_t slack = 0) {
        T* p = alloc<T>(v.size() + slack, false);
        if (!v.empty()) staged_h2d(p, v.data(), v.size() * sizeof(T), s);
        if (h2d) *h2d += static_cast<int64_t>(v.size() * sizeof(T));
        return p;
    }
    void free_all() {
        if (blocks.empty()) return;
        if (!BlockCache::enabled()) {
            for (const Block& b : blocks) cudaFree(b.p);
            blocks.clear();
            return;
        }
        // kernels still in flight may use the blocks: the devices go idle before the blocks are reused
        int cur = 0;
        cudaGetDevice(&cur);
        int synced = -1;
        for (const Block& b : blocks)
            if (b.dev != synced) {
                cudaSetDevice(b.dev);
                cudaDeviceSynchronize();
                synced = b.dev;
            }
        cudaSetDevice(cur);
        for (const Block& b : blocks) block_cache().give(b.dev, b.bytes, b.p);
        blocks.clear();
    }
    ~DevMem() { free_all(); }
};

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int sm_count = 148;
    int32_t m = 0, n = 0;
    int64_t nnz = 0;
    // distribution
    int rank = 0, world = 1;
    ncclComm_t comm = nullptr;
    int32_t row_begin = 0, row_end = 0, col_begin = 0, col_end = 0;
    int32_t Bm = 0, Bn = 0, ext_m = 0, ext_n = 0, ldm = 0, ldn = 0;
    std::vector<int32_t> rmap, cmap;  // global -> padded (empty = identity)
    int64_t local_nnz_csr = 0, local_nnz_csc = 0;
    // host metadata kept for residual readback
    SweepLayout hcsr, hcsc;  // value/index arrays released after upload
    std::vector<int64_t> row_start_local, col_start_local;
    DevMem mem;
    DevSweep csr, csc;
    float* A_csr = nullptr;   // immutable ratings, padded CSR layout (objective reads A, not R)
    float* A_csc = nullptr;
    // CCD++ model
    int mode = 0;  // 0 none, 1 ccdpp, 2 als
    int k = 0;
    float lambda = 0.f;
    int inner = 0;
    DevMem model_mem;
    float* W = nullptr;  // CCD++: column-major k x ldm ; ALS: row-major ext_m x k
    float* H = nullptr;
    float* ubuf = nullptr;
    float* vbuf = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t graph_exec = nullptr;
    int64_t launches_per_iter = 0;
    bool profiling = false;
    double stat_u_ms = 0, stat_v_ms = 0;
    int64_t stat_u_n = 0, stat_v_n = 0;
    // ALS
    bool als_built = false;
    DevMem als_mem;
    DevMem ccdw_mem;   // item/user-wise CCD workspace
    CcdWs ccdw;
    bool ccdw_on = false;
    bool ccdw_gram = false;  // item/user-wise CCD as gram + Gauss-Seidel sweeps (no residual)
    DevAls als_csr, als_csc;
    int* d_counter = nullptr;
    int* d_status = nullptr;
    bool als_weighted = false;
    // eval
    DevMem eval_mem;
    double* unit_loss = nullptr;
    double* red_scratch = nullptr;
    double* red_out = nullptr;  // [0] loss, [1] reg W, [2] reg H, [3] probe sse
    DevMem rm_mem;              // row-major copies of the CCD++ factors for the metric kernels
    float* w_rm = nullptr;
    float* h_rm = nullptr;
    size_t rm_floats = 0;
    DevTriplet* probe = nullptr;
    int64_t n_probe = 0;
    DevMem probe_mem;
    int64_t h2d = 0, d2h = 0;
    double setup_seconds = 0;
    // Single-process device group (pmf_ctx_create_group, num_gpus > 1 in the whole-call API): rank 0
    // owns ranks 1..G-1 and drives all of them; `ranks` lists every rank in order (empty otherwise).
    // The all-gathers are peer copies between the ranks' replicated vectors (see exchange()).
    std::vector<std::unique_ptr<Ctx>> peers;
    std::vector<Ctx*> ranks;
    cudaEvent_t ev_done = nullptr, ev_sent = nullptr;

    ~Ctx() {
        cudaSetDevice(device);
        if (graph_exec) cudaGraphExecDestroy(graph_exec);
        if (graph) cudaGraphDestroy(graph);
        if (comm) ncclCommDestroy(comm);
        if (ev_done) cudaEventDestroy(ev_done);
        if (ev_sent) cudaEventDestroy(ev_sent);
        if (stream) cudaStreamDestroy(stream);
    }
    int32_t prow(int32_t i) const { return rmap.empty() ? i : rmap[i]; }
    int32_t pcol(int32_t j) const { return cmap.empty() ? j : cmap[j]; }
};

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

void check_view(const pmf_matrix_view* a) {
    if (!a) invalid("matrix view is null");
    if (a->m < 0 || a->n < 0) invalid("matrix dimensions must be non-negative");
    if (a->nnz < 0) invalid("nnz must be non-negative");
    if (!a->row_start || !a->col_start) invalid("matrix offsets are null");
    if (a->nnz > 0 && (!a->col_of || !a->val_row || !a->row_of || !a->val_col)) invalid("matrix arrays are null");
    if (a->row_start[0] != 0 || a->row_start[a->m] != a->nnz || a->col_start[0] != 0 || a->col_start[a->n] != a->nnz)
        throw PmfError(PMF_DATA_ERROR, "matrix offsets inconsistent with nnz");
}

void ensure_device() {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        throw PmfError(PMF_RUNTIME_ERROR, "no CUDA device available (the B200 path has no CPU fallback)");
    }
    static const bool hooks = [] {
        if (!BlockCache::enabled()) return false;
        host_alloc_hooks().alloc = pinned_hook_alloc;
        host_alloc_hooks().free = pinned_hook_free;
        return true;
    }();
    (void)hooks;
}

// A side kept in HBM after the device ingest (contexts built from triplets): CSR / CSC arrays.
struct DevSide {
    const int64_t* start = nullptr;
    const int32_t* idx = nullptr;
    const float* val = nullptr;
    int64_t nnz = 0;
};

DevSweep upload_sweep(Ctx& c, SweepLayout& L, float** A_copy, const DevSide* src = nullptr) {
    DevSweep D;
    D.n_out = L.n_out;
    D.gat_extent = L.gat_extent;
    D.panel_size = L.panel_size;
    D.n_panels = L.n_panels;
    D.sentinel = L.sentinel;
    D.smem = L.smem;
    D.idx16 = L.idx16;
    D.n_entries = L.n_entries;
    D.n_units = static_cast<int32_t>(L.units.size());
    D.n_mo = static_cast<int32_t>(L.mo_out.size());
    D.n_mo_big = L.n_mo_big;
    D.n_dense = L.n_dense;
    D.avg_segment = L.avg_segment;
    D.flat = L.flat;
    if (L.flat) {
        D.chunks = c.mem.upload(L.chunks, c.stream, &c.h2d);
        D.tailbits = c.mem.upload(L.tailbits, c.stream, &c.h2d);
        std::vector<int32_t> info(L.units.size()), out(L.units.size());
        for (size_t u = 0; u < L.units.size(); ++u) {
            out[u] = L.units[u].o;
            info[u] = L.units[u].slot >= 0 ? L.units[u].slot : -(L.units[u].o + 1);
        }
        D.uinfo = c.mem.upload(info, c.stream, &c.h2d);
        D.uout = c.mem.upload(out, c.stream, &c.h2d);
    }
    D.ctas = L.ctas;
    D.n_slots = L.n_slots;
    // slack: the flat kernels load whole 16-entry lane ranges past a layout's last vector (masked)
    DevMem tmp;
    float* A = nullptr;
    if (src) {  // the padded streams filled on the device from its CSR / CSC (layout_device.cu)
        if (L.idx16) D.idx = c.mem.alloc<uint16_t>(static_cast<size_t>(L.n_entries) + kStreamSlack, false);
        else D.idx = c.mem.alloc<int32_t>(static_cast<size_t>(L.n_entries) + kStreamSlack, false);
        A = c.mem.alloc<float>(static_cast<size_t>(L.n_entries), false);
        const int64_t* delta = tmp.upload(L.seg_delta, c.stream, &c.h2d);
        layout_fill_device(src->start, src->idx, src->val, L.n_out, src->nnz, L.panel_size, L.n_panels, delta, L.idx16,
                           L.sentinel, L.n_entries, D.idx, A, c.stream);
        CUDA_TRY(cudaGetLastError());
    } else {
        if (L.idx16) D.idx = c.mem.upload(L.idx16v, c.stream, &c.h2d, kStreamSlack);
        else D.idx = c.mem.upload(L.idx32v, c.stream, &c.h2d, kStreamSlack);
        A = c.mem.upload(L.val, c.stream, &c.h2d);
    }
    D.R = c.mem.alloc<float>(L.n_entries + kStreamSlack, false);
    CUDA_TRY(cudaMemcpyAsync(D.R, A, static_cast<size_t>(L.n_entries) * sizeof(float), cudaMemcpyDeviceToDevice,
                             c.stream));
    *A_copy = A;
    D.units = c.mem.upload(L.units, c.stream, &c.h2d);
    D.unit_panel = c.mem.upload(L.unit_panel, c.stream, &c.h2d);
    D.pieces = c.mem.upload(L.pieces, c.stream, &c.h2d);
    D.n_pieces = static_cast<int32_t>(L.pieces.size());
    {
        std::vector<int32_t> g(4 * L.pieces.size() + 1, 0);
        for (size_t p = 0; p < L.pieces.size(); ++p) {
            g[4 * p] = L.flat ? L.pieces[p].pad[0] : L.pieces[p].ub;
            g[4 * p + 1] = L.pieces[p].um;
            g[4 * p + 2] = L.pieces[p].us;
        }
        D.gcnt = c.mem.upload(g, c.stream, &c.h2d);
    }
    D.piece_start = c.mem.upload(L.piece_start, c.stream, &c.h2d);
    D.panel_base = c.mem.upload(L.panel_base, c.stream, &c.h2d);
    D.mo_out = c.mem.upload(L.mo_out, c.stream, &c.h2d);
    D.mo_start = c.mem.upload(L.mo_start, c.stream, &c.h2d);
    D.partial = c.mem.alloc<float2>(std::max(1, L.n_slots));
    D.promote_fused = L.promote_fused;
    D.rmw_sub = L.rmw_sub;
    D.sub_width = L.sub_width;
    if (!L.usplit.empty()) D.usplit = c.mem.upload(L.usplit, c.stream, &c.h2d);
    if (src && L.rmw_sub > 1) {  // sub-panel split points from the device-filled indices
        if (!L.idx16) throw PmfError(PMF_RUNTIME_ERROR, "split promote needs 16-bit indices");
        const int S = L.rmw_sub;
        D.usplit = c.mem.alloc<uint16_t>(L.units.size() * static_cast<size_t>(S + 1), false);
        const int32_t* real = tmp.upload(L.unit_real, c.stream, &c.h2d);
        usplit_device(D.units, real, static_cast<int64_t>(L.units.size()), static_cast<const uint16_t*>(D.idx), S,
                      L.sub_width, D.usplit, c.stream);
        CUDA_TRY(cudaGetLastError());
    }
    CUDA_TRY(cudaStreamSynchronize(c.stream));
    // keep only the metadata needed for residual readback
    L.idx16v.reset();
    L.idx32v.reset();
    L.val.reset();
    return D;
}

// Distribution plan shared by pmf_ctx_create_dist and pmf_dist_plan: rank r owns CSR rows
// [row_bounds[r], row_bounds[r+1]) and CSC columns [col_bounds[r], col_bounds[r+1]); the replicated
// vectors live in a padded space where block r occupies [r*B, (r+1)*B), B = largest block (so NCCL
// all-gathers use equal counts).  world == 1 keeps the identity space.
void dist_plan(const int64_t* row_start, int32_t m, const int64_t* col_start, int32_t n, int world,
               int32_t* row_bounds, int32_t* col_bounds, int32_t* Bm, int32_t* Bn) {
    std::vector<int64_t> rc(m), cc(n);
    for (int32_t i = 0; i < m; ++i) rc[i] = 4 * (row_start[i + 1] - row_start[i]);
    for (int32_t j = 0; j < n; ++j) cc[j] = 4 * (col_start[j + 1] - col_start[j]);
    partition_balanced(rc.data(), m, world, row_bounds);
    partition_balanced(cc.data(), n, world, col_bounds);
    int32_t bm = 0, bn = 0;
    for (int r = 0; r < world; ++r) {
        bm = std::max(bm, row_bounds[r + 1] - row_bounds[r]);
        bn = std::max(bn, col_bounds[r + 1] - col_bounds[r]);
    }
    *Bm = world == 1 ? m : bm;
    *Bn = world == 1 ? n : bn;
}

// Upload + device build of the CSR / CSC (sparse.hpp:73-149, csrc/ingest.cu) with the host builder's
// validation errors: the first offending triplet in input order, then the first duplicate in row
// order.  The four nnz-sized arrays come from `keep`, the rest from `tmp`.
struct DevCsr {
    int64_t* rs = nullptr;
    int64_t* cs = nullptr;
    int32_t* co = nullptr;
    int32_t* ro = nullptr;
    float* vr = nullptr;
    float* vc = nullptr;
};

void check_triplet_args(const pmf_triplet* t, int64_t nnz, int32_t m, int32_t n) {
    if (m < 0 || n < 0) invalid("matrix dimensions must be non-negative");
    if (nnz < 0 || (nnz > 0 && !t)) invalid("from_triplets: null buffers");
    if (nnz >= (int64_t(1) << 31)) invalid("from_triplets_gpu: more than 2^31 - 1 triplets");
}

DevCsr device_ingest(const pmf_triplet* t, int64_t nnz, int32_t m, int32_t n, cudaStream_t s, DevMem& keep,
                     DevMem& tmp, double* t_up, double* t_build) {
    const double t0 = now_s();
    const size_t N = static_cast<size_t>(nnz > 0 ? nnz : 1);
    DevCsr d;
    auto* dt = tmp.alloc<DevTriplet>(N, false);
    if (nnz > 0) staged_h2d(dt, t, sizeof(DevTriplet) * static_cast<size_t>(nnz), s);
    d.rs = tmp.alloc<int64_t>(static_cast<size_t>(m) + 1, false);
    d.cs = tmp.alloc<int64_t>(static_cast<size_t>(n) + 1, false);
    d.co = keep.alloc<int32_t>(N, false);
    d.ro = keep.alloc<int32_t>(N, false);
    d.vr = keep.alloc<float>(N, false);
    d.vc = keep.alloc<float>(N, false);
    void* scratch = tmp.alloc<char>(ingest_scratch_bytes(nnz), false);
    CUDA_TRY(cudaStreamSynchronize(s));
    const double t1 = now_s();
    int64_t bad = -1, dup = -1;
    CUDA_TRY(ingest_build(dt, nnz, m, n, scratch, d.rs, d.co, d.vr, d.cs, d.ro, d.vc, &bad, &dup, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (t_up) *t_up = t1 - t0;
    if (t_build) *t_build = now_s() - t1;
    if (bad >= 0) {  // the first offending triplet in input order decides (sparse.hpp:82-92)
        const pmf_triplet& b = t[bad];
        if (b.user < 0 || b.user >= m)
            throw PmfError(PMF_OUT_OF_RANGE, "user index " + std::to_string(b.user) + " out of range for m=" +
                                                 std::to_string(m));
        if (b.item < 0 || b.item >= n)
            throw PmfError(PMF_OUT_OF_RANGE, "item index " + std::to_string(b.item) + " out of range for n=" +
                                                 std::to_string(n));
        invalid("non-finite rating at user " + std::to_string(b.user));
    }
    if (dup >= 0) {  // sparse.hpp:127-132: first duplicate in row order
        int32_t item = 0;
        std::vector<int64_t> row_start(static_cast<size_t>(m) + 1);
        CUDA_TRY(cudaMemcpyAsync(&item, d.co + dup, sizeof(item), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(row_start.data(), d.rs, sizeof(int64_t) * row_start.size(), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        const int64_t i = std::upper_bound(row_start.begin(), row_start.end(), dup) - row_start.begin() - 1;
        invalid("duplicate rating for user " + std::to_string(i) + ", item " + std::to_string(item));
    }
    return d;
}

void set_kernel_attributes() {
    static bool attrs_set = false;
    if (!attrs_set) {
        sweep_set_attributes(kSmemMax + 1024);
        flat_set_attributes(kSmemMax + 1024);
        als_set_attributes();
        attrs_set = true;
    }
}

std::unique_ptr<Ctx> make_ctx(const pmf_matrix_view* a, int device, int rank, int world, const uint8_t* id) {
    check_view(a);
    ensure_device();
    const double t0 = now_s();
    auto c = std::make_unique<Ctx>();
    if (device < 0) CUDA_TRY(cudaGetDevice(&device));
    c->device = device;
    CUDA_TRY(cudaSetDevice(device));
    CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&c->ev_sent, cudaEventDisableTiming));
    CUDA_TRY(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
    c->m = a->m;
    c->n = a->n;
    c->nnz = a->nnz;
    c->rank = rank;
    c->world = world;
    if (id) {  // distributed context (a 1-rank communicator is allowed and exercises the same path)
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        NCCL_TRY(ncclCommInitRank(&c->comm, world, uid, rank));
    }
    // row / column blocks (runtime.hpp:73-136, 4|Omega| costs) and the padded index space
    std::vector<int32_t> rb(world + 1), cbd(world + 1);
    dist_plan(a->row_start, a->m, a->col_start, a->n, world, rb.data(), cbd.data(), &c->Bm, &c->Bn);
    c->row_begin = rb[rank];
    c->row_end = rb[rank + 1];
    c->col_begin = cbd[rank];
    c->col_end = cbd[rank + 1];
    c->ext_m = world * c->Bm;
    c->ext_n = world * c->Bn;
    c->ldm = ((c->ext_m + 4 + 31) / 32) * 32;  // slack: sentinel + TMA round-up
    c->ldn = ((c->ext_n + 4 + 31) / 32) * 32;
    if (world > 1) {
        c->rmap.resize(a->m);
        c->cmap.resize(a->n);
        for (int r = 0; r < world; ++r) {
            for (int32_t i = rb[r]; i < rb[r + 1]; ++i) c->rmap[i] = r * c->Bm + (i - rb[r]);
            for (int32_t j = cbd[r]; j < cbd[r + 1]; ++j) c->cmap[j] = r * c->Bn + (j - cbd[r]);
        }
    }
    const int32_t* rmap = c->rmap.empty() ? nullptr : c->rmap.data();
    const int32_t* cmap = c->cmap.empty() ? nullptr : c->cmap.data();
    const double t_layout = now_s();
    // the CSC layout is built on a host thread alongside the CSR layout and its upload (the future's
    // destructor waits for the builder if anything below throws); PMF_SETUP_SERIAL=1: after them
    static const bool serial = std::getenv("PMF_SETUP_SERIAL") != nullptr;
    auto csc_future = std::async(serial ? std::launch::deferred : std::launch::async, [&] {
        return build_sweep_layout(a->col_start, a->row_of, a->val_col, c->col_begin, c->col_end, rmap, c->ext_m, 3,
                                  smem_budget(), c->sm_count);
    });
    c->hcsr = build_sweep_layout(a->row_start, a->col_of, a->val_row, c->row_begin, c->row_end, cmap, c->ext_n,
                                 2, smem_budget(), c->sm_count);
    c->local_nnz_csr = a->row_start[c->row_end] - a->row_start[c->row_begin];
    c->local_nnz_csc = a->col_start[c->col_end] - a->col_start[c->col_begin];
    c->row_start_local.assign(a->row_start + c->row_begin, a->row_start + c->row_end + 1);
    c->col_start_local.assign(a->col_start + c->col_begin, a->col_start + c->col_end + 1);
    set_kernel_attributes();
    const double t_upload = now_s();
    c->csr = upload_sweep(*c, c->hcsr, &c->A_csr);
    const double t_csr = now_s();
    c->hcsc = csc_future.get();
    const double t_csc = now_s();
    c->csc = upload_sweep(*c, c->hcsc, &c->A_csc);
    const double t_done = now_s();
    // eval scratch
    c->unit_loss = c->eval_mem.alloc<double>(std::max(c->csr.n_units, 1));
    c->red_scratch = c->eval_mem.alloc<double>(4096);
    c->red_out = c->eval_mem.alloc<double>(8);
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    c->setup_seconds = now_s() - t0;
    if (std::getenv("PMF_VERBOSE"))
        std::fprintf(stderr,
                     "[pmf] ctx setup %.3f s: device init %.3f, csr layout %.3f, csr upload %.3f (csc layout "
                     "alongside), csc wait %.3f, csc upload %.3f, rest %.3f; process totals: cudaMalloc %.3f, "
                     "staged h2d %.3f\n",
                     c->setup_seconds, t_layout - t0, t_upload - t_layout, t_csr - t_upload, t_csc - t_csr,
                     t_done - t_csc, now_s() - t_done, g_alloc_s, g_h2d_s);
    return c;
}

// ---- CCD++ --------------------------------------------------------------------------------------

void reset_graph(Ctx& c) {
    if (c.graph_exec) cudaGraphExecDestroy(c.graph_exec);
    if (c.graph) cudaGraphDestroy(c.graph);
    c.graph_exec = nullptr;
    c.graph = nullptr;
}

void alloc_ccd_model(Ctx& c, int k) {
    reset_graph(c);
    c.model_mem.free_all();
    c.W = c.model_mem.alloc<float>(static_cast<size_t>(k) * c.ldm);
    c.H = c.model_mem.alloc<float>(static_cast<size_t>(k) * c.ldn);
    c.ubuf = c.model_mem.alloc<float>(c.ldm);
    c.vbuf = c.model_mem.alloc<float>(c.ldn);
    c.k = k;
}

// model.hpp:86-93 init_random_items on the host (mt19937, bit-exact), returned row-major n x k
std::vector<float> init_items_host(int32_t n, int k, uint64_t seed) {
    std::vector<float> H(static_cast<size_t>(n) * k);
    std::mt19937 gen(static_cast<std::mt19937::result_type>(seed));
    const double scale = 1.0 / std::sqrt(static_cast<double>(k));
    for (auto& x : H) x = static_cast<float>(((static_cast<double>(gen()) + 1.0) * (1.0 / 4294967296.0)) * scale);
    return H;
}

void upload_colmajor(Ctx& c, float* dst, int64_t ld, const float* rowmajor, int32_t count, int k, bool rows) {
    std::vector<float> tmp(static_cast<size_t>(k) * ld, 0.f);
    for (int32_t i = 0; i < count; ++i) {
        const int32_t p = rows ? c.prow(i) : c.pcol(i);
        for (int t = 0; t < k; ++t) tmp[static_cast<size_t>(t) * ld + p] = rowmajor[static_cast<size_t>(i) * k + t];
    }
    CUDA_TRY(cudaMemcpyAsync(dst, tmp.data(), tmp.size() * sizeof(float), cudaMemcpyHostToDevice, c.stream));
    CUDA_TRY(cudaStreamSynchronize(c.stream));
    c.h2d += static_cast<int64_t>(tmp.size() * sizeof(float));
}

void upload_rowmajor(Ctx& c, float* dst, int32_t ext, const float* rowmajor, int32_t count, int k, bool rows) {
    std::vector<float> tmp(static_cast<size_t>(ext) * k, 0.f);
    for (int32_t i = 0; i < count; ++i) {
        const int32_t p = rows ? c.prow(i) : c.pcol(i);
        std::memcpy(&tmp[static_cast<size_t>(p) * k], rowmajor + static_cast<size_t>(i) * k, sizeof(float) * k);
    }
    CUDA_TRY(cudaMemcpyAsync(dst, tmp.data(), tmp.size() * sizeof(float), cudaMemcpyHostToDevice, c.stream));
    CUDA_TRY(cudaStreamSynchronize(c.stream));
    c.h2d += static_cast<int64_t>(tmp.size() * sizeof(float));
}

void reset_residual(Ctx& c) {
    CUDA_TRY(cudaMemcpyAsync(c.csr.R, c.A_csr, c.csr.n_entries * sizeof(float), cudaMemcpyDeviceToDevice, c.stream));
    CUDA_TRY(cudaMemcpyAsync(c.csc.R, c.A_csc, c.csc.n_entries * sizeof(float), cudaMemcpyDeviceToDevice, c.stream));
}

void allgather(Ctx& c, float* buf, int64_t block) {
    if (c.comm)
        NCCL_TRY(ncclAllGather(buf + static_cast<int64_t>(c.rank) * block, buf, block, ncclFloat, c.comm, c.stream));
}

using Ranks = std::vector<Ctx*>;
Ranks ranks_of(Ctx& c) { return c.ranks.empty() ? Ranks{&c} : c.ranks; }

// All-gather of a replicated vector (block r = `block` floats at r * block, just written by rank r).
// One rank: NCCL in place (a no-op without a communicator).  A device group: every rank pushes its
// block into every peer's copy, between two event rounds -- the pushes wait until each peer's last
// kernel (the last reader of the old contents) is done (ev_done), and each rank's next kernel waits
// for every push into its copy (ev_sent).  Host-ordered records and waits, so this also captures
// into a CUDA graph as plain dependencies.
template <class Buf>
void exchange(const Ranks& cs, Buf buf, int64_t block) {
    if (cs.size() == 1) {
        allgather(*cs[0], buf(*cs[0]), block);
        return;
    }
    for (Ctx* c : cs) CUDA_TRY(cudaEventRecord(c->ev_done, c->stream));
    for (Ctx* r : cs) {
        for (Ctx* q : cs)
            if (q != r) CUDA_TRY(cudaStreamWaitEvent(r->stream, q->ev_done, 0));
        const int64_t off = static_cast<int64_t>(r->rank) * block;
        for (Ctx* q : cs)
            if (q != r)
                CUDA_TRY(cudaMemcpyAsync(buf(*q) + off, buf(*r) + off, sizeof(float) * block, cudaMemcpyDefault,
                                         r->stream));
        CUDA_TRY(cudaEventRecord(r->ev_sent, r->stream));
    }
    for (Ctx* q : cs)
        for (Ctx* r : cs)
            if (r != q) CUDA_TRY(cudaStreamWaitEvent(q->stream, r->ev_sent, 0));
}

// rank 0's stream forks to / joins from the other ranks' streams (a group's work is one graph,
// launched and timed on rank 0's stream)
void fork_ranks(const Ranks& cs) {
    if (cs.size() == 1) return;
    CUDA_TRY(cudaEventRecord(cs[0]->ev_done, cs[0]->stream));
    for (size_t r = 1; r < cs.size(); ++r) CUDA_TRY(cudaStreamWaitEvent(cs[r]->stream, cs[0]->ev_done, 0));
}
void join_ranks(const Ranks& cs) {
    if (cs.size() == 1) return;
    for (size_t r = 1; r < cs.size(); ++r) {
        CUDA_TRY(cudaEventRecord(cs[r]->ev_done, cs[r]->stream));
        CUDA_TRY(cudaStreamWaitEvent(cs[0]->stream, cs[r]->ev_done, 0));
    }
}
// a group's schedule is captured as one graph when all its ranks share a device (streams of
// several devices run it uncaptured, issued from the host)
bool capturable(const Ranks& cs) {
    for (Ctx* c : cs)
        if (c->device != cs[0]->device) return false;
    return true;
}

struct SweepTimer {
    Ctx& c;
    cudaEvent_t a = nullptr, b = nullptr;
    bool on;
    explicit SweepTimer(Ctx& cc) : c(cc), on(cc.profiling) {
        if (on) {
            cudaEventCreate(&a);
            cudaEventCreate(&b);
        }
    }
    ~SweepTimer() {
        if (a) cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
    }
    void start() {
        if (on) cudaEventRecord(a, c.stream);
    }
    void stop(bool u) {
        if (!on) return;
        cudaEventRecord(b, c.stream);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        if (u) {
            c.stat_u_ms += ms;
            c.stat_u_n++;
        } else {
            c.stat_v_ms += ms;
            c.stat_v_n++;
        }
    }
};

// Enqueues one CCD++ outer iteration (ccd.hpp:373-393) on the ranks' streams; returns kernels launched.
int64_t enqueue_ccd_iteration(const Ranks& cs) {
    int64_t launched = 0;
    Ctx& c0 = *cs[0];
    const int k = c0.k;
    SweepTimer tm(c0);  // profiling: rank 0's sweeps
    fork_ranks(cs);
    for (int t = 0; t < k; ++t) {
        const int tp = (t + k - 1) % k;
        for (int s = 0; s < c0.inner; ++s) {
            for (Ctx* cp : cs) {
                Ctx& c = *cp;
                SweepOperands ou;
                ou.lambda = c.lambda;
                ou.out = c.ubuf;
                ou.out_off = c.rank * c.Bm;
                if (s == 0) {
                    ou.ga = c.H + static_cast<int64_t>(tp) * c.ldn;  // v'
                    ou.gb = c.H + static_cast<int64_t>(t) * c.ldn;   // h (also the v of the first u update)
                    ou.gn = ou.gb;
                    ou.oa = c.W + static_cast<int64_t>(tp) * c.ldm;  // u'
                    ou.ob = c.W + static_cast<int64_t>(t) * c.ldm;   // w
                } else {
                    ou.gn = c.vbuf;
                }
                if (cp == &c0) tm.start();
                launched += launch_sweep(c.csr, s == 0 ? kPromote : kPlain, true, ou, c.stream);
                if (cp == &c0) tm.stop(true);
            }
            exchange(cs, [](Ctx& c) { return c.ubuf; }, c0.Bm);
            for (Ctx* cp : cs) {
                Ctx& c = *cp;
                SweepOperands ov;
                ov.lambda = c.lambda;
                ov.out = c.vbuf;
                ov.out_off = c.rank * c.Bn;
                ov.gn = c.ubuf;
                if (s == 0) {
                    ov.ga = c.W + static_cast<int64_t>(tp) * c.ldm;  // u'
                    ov.gb = c.W + static_cast<int64_t>(t) * c.ldm;   // w
                    ov.oa = c.H + static_cast<int64_t>(tp) * c.ldn;  // v'
                    ov.ob = c.H + static_cast<int64_t>(t) * c.ldn;   // h
                }
                if (cp == &c0) tm.start();
                launched += launch_sweep(c.csc, s == 0 ? kPromote : kPlain, false, ov, c.stream);
                if (cp == &c0) tm.stop(false);
            }
            exchange(cs, [](Ctx& c) { return c.vbuf; }, c0.Bn);
        }
        // writeback of the column pair (ccd.hpp:209, :226); the residual part is deferred
        for (Ctx* cp : cs) {
            Ctx& c = *cp;
            CUDA_TRY(cudaMemcpyAsync(c.W + static_cast<int64_t>(t) * c.ldm, c.ubuf, sizeof(float) * c.ext_m,
                                     cudaMemcpyDeviceToDevice, c.stream));
            CUDA_TRY(cudaMemcpyAsync(c.H + static_cast<int64_t>(t) * c.ldn, c.vbuf, sizeof(float) * c.ext_n,
                                     cudaMemcpyDeviceToDevice, c.stream));
        }
    }
    join_ranks(cs);
    CUDA_TRY(cudaGetLastError());
    return launched;
}

void check_ccd_config(const pmf_ccd_config* cfg) {
    if (!cfg) invalid("config is null");
    // ccd.hpp:43-49
    if (cfg->k < 1) invalid("k must be >= 1");
    if (cfg->lambda < 0.f) invalid("lambda must be >= 0");
    if (cfg->outer_iters < 1) invalid("outer_iters must be >= 1");
    if (cfg->inner_iters < 1) invalid("inner_iters must be >= 1");
    if (cfg->num_gpus < 1) invalid("workers must be >= 1");
}

void ccd_begin(Ctx& c0, const pmf_ccd_config* cfg) {
    check_ccd_config(cfg);
    const auto H = init_items_host(c0.n, cfg->k, cfg->seed);  // model.hpp:86-93, replicated
    for (Ctx* cp : ranks_of(c0)) {
        Ctx& c = *cp;
        CUDA_TRY(cudaSetDevice(c.device));
        alloc_ccd_model(c, cfg->k);
        c.mode = 1;
        c.lambda = cfg->lambda;
        c.inner = cfg->inner_iters;
        upload_colmajor(c, c.H, c.ldn, H.data(), c.n, cfg->k, false);
        reset_residual(c);
        CUDA_TRY(cudaStreamSynchronize(c.stream));
    }
}

// PMF_SMALL=0: keep small matrices on the CUDA-graph schedule
bool small_disabled() {
    static const bool off = [] {
        const char* e = std::getenv("PMF_SMALL");
        return e && std::atoi(e) == 0;
    }();
    return off;
}

void ccd_iterate(Ctx& c, int n_outer, double* secs) {
    if (c.mode != 1) invalid("ccdpp_begin has not been called");
    CUDA_TRY(cudaSetDevice(c.device));
    const Ranks cs = ranks_of(c);
    const bool graph = !c.profiling && capturable(cs);
    if (!graph) {
        reset_graph(c);
        c.stat_u_ms = c.stat_v_ms = 0;
        c.stat_u_n = c.stat_v_n = 0;
    } else if (!c.graph_exec) {
        CUDA_TRY(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
        int64_t launched = 0;
        try {
            launched = enqueue_ccd_iteration(cs);
        } catch (...) {
            cudaGraph_t g;
            cudaStreamEndCapture(c.stream, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        CUDA_TRY(cudaStreamEndCapture(c.stream, &c.graph));
        CUDA_TRY(cudaGraphInstantiate(&c.graph_exec, c.graph, 0));
        c.launches_per_iter = launched;
    }
    // small matrices (one panel, no partial slots, residual runs fit shared memory): the whole iteration
    // as one cluster kernel (small_kernels.cu) instead of 2 T k graph nodes
    const bool small = cs.size() == 1 && !c.profiling && !small_disabled() &&
                       small_ccdpp_eligible(c.csr, c.csc, c.hcsr, c.hcsc, c.m, c.n);
    cudaEvent_t e0, e1;
    CUDA_TRY(cudaEventCreate(&e0));
    CUDA_TRY(cudaEventCreate(&e1));
    for (int it = 0; it < n_outer; ++it) {
        CUDA_TRY(cudaEventRecord(e0, c.stream));
        if (small) {
            CUDA_TRY(launch_small_ccdpp(c.csr, c.csc, c.hcsr, c.hcsc, c.W, c.H, c.ubuf, c.vbuf, c.ldm, c.ldn, c.m, c.n,
                                        c.k, c.inner, c.lambda, c.stream));
            c.launches_per_iter = 1;
        } else if (!graph) c.launches_per_iter = enqueue_ccd_iteration(cs);
        else CUDA_TRY(cudaGraphLaunch(c.graph_exec, c.stream));
        CUDA_TRY(cudaEventRecord(e1, c.stream));
        CUDA_TRY(cudaEventSynchronize(e1));
        float ms = 0;
        CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
        if (secs) secs[it] = ms * 1e-3;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    CUDA_TRY(cudaGetLastError());
}

// ---- ALS ----------------------------------------------------------------------------------------

DevAls upload_als(Ctx& c, const AlsLayout& L, int k) {
    DevAls D;
    D.n_out = L.n_out;
    D.n_units = static_cast<int32_t>(L.units.size());
    D.n_mo = static_cast<int32_t>(L.mo_out.size());
    D.n_slots = L.n_slots;
    D.n_empty = static_cast<int32_t>(L.empty_out.size());
    D.n_entries = L.n_entries;
    D.idx = c.als_mem.upload(L.idx, c.stream, &c.h2d);
    D.val = c.als_mem.upload(L.val, c.stream, &c.h2d);
    D.units = c.als_mem.upload(L.units, c.stream, &c.h2d);
    D.mo_out = c.als_mem.upload(L.mo_out, c.stream, &c.h2d);
    D.mo_start = c.als_mem.upload(L.mo_start, c.stream, &c.h2d);
    D.empty_out = c.als_mem.upload(L.empty_out, c.stream, &c.h2d);
    D.partial = nullptr;
    (void)k;
    return D;
}

// ALS layouts need the host matrix: built during ctx creation when requested.
struct AlsHost {
    AlsLayout csr, csc;
};

// Entries per ALS / CCD gram work unit (longer rows / columns split into partial grams).  Large
// enough that few outputs need partials, small enough that the longest units do not leave a tail:
// the power of two nearest nnz / (2 x resident warps), in [1024, 16384] (Netflix: 16384 -- 4096 gave
// 16.95 ms, 16384 16.69 ms, 65536 19.6 ms per ALS iteration; ML-10M: 2048).  PMF_ALS_CHUNK overrides.
int als_chunk(int64_t nnz, int sm_count) {
    if (const char* e = std::getenv("PMF_ALS_CHUNK")) return std::max(32, std::atoi(e));
    const int64_t target = nnz / (2 * 20 * static_cast<int64_t>(std::max(sm_count, 1)));
    int c = 1024;
    while (c < 16384 && 2 * c <= target) c *= 2;
    return c;
}

void build_als(Ctx& c, const pmf_matrix_view* a) {
    if (c.als_built) return;
    const int32_t* rmap = c.rmap.empty() ? nullptr : c.rmap.data();
    const int32_t* cmap = c.cmap.empty() ? nullptr : c.cmap.data();
    const int chunk = als_chunk(c.nnz, c.sm_count);
    AlsLayout lc = build_als_layout(a->row_start, a->col_of, a->val_row, c.row_begin, c.row_end, cmap, chunk);
    AlsLayout lr = build_als_layout(a->col_start, a->row_of, a->val_col, c.col_begin, c.col_end, rmap, chunk);
    c.als_csr = upload_als(c, lc, 0);
    c.als_csc = upload_als(c, lr, 0);
    c.d_counter = c.als_mem.alloc<int>(4);
    c.d_status = c.als_mem.alloc<int>(4);
    CUDA_TRY(cudaStreamSynchronize(c.stream));
    c.als_built = true;
}

// A context straight from triplets (world 1): the device ingest's CSR / CSC stay in HBM -- they are the
// ALS streams, and the sweep layouts are filled from them on the device; the host receives only the
// row / column offsets and the per-(panel, output) segment lengths, from which it builds the layouts'
// structure (units, slots, CTA partition).  Bitwise the layouts of make_ctx on the same matrix.
std::unique_ptr<Ctx> make_ctx_from_triplets(const pmf_triplet* t, int64_t nnz, int32_t m, int32_t n, int device) {
    check_triplet_args(t, nnz, m, n);
    ensure_device();
    const double t0 = now_s();
    auto c = std::make_unique<Ctx>();
    if (device < 0) CUDA_TRY(cudaGetDevice(&device));
    c->device = device;
    CUDA_TRY(cudaSetDevice(device));
    CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&c->ev_sent, cudaEventDisableTiming));
    CUDA_TRY(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
    c->m = m;
    c->n = n;
    c->nnz = nnz;
    DevMem tmp;
    double tu = 0, tb = 0;
    const DevCsr d = device_ingest(t, nnz, m, n, c->stream, c->als_mem, tmp, &tu, &tb);
    c->h2d += static_cast<int64_t>(sizeof(pmf_triplet)) * nnz;
    const double t_ingest = now_s();
    c->row_start_local.resize(static_cast<size_t>(m) + 1);
    c->col_start_local.resize(static_cast<size_t>(n) + 1);
    CUDA_TRY(cudaMemcpyAsync(c->row_start_local.data(), d.rs, sizeof(int64_t) * c->row_start_local.size(),
                             cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->col_start_local.data(), d.cs, sizeof(int64_t) * c->col_start_local.size(),
                             cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    c->Bm = m;
    c->Bn = n;
    c->row_end = m;
    c->col_end = n;
    c->ext_m = m;
    c->ext_n = n;
    c->ldm = ((c->ext_m + 4 + 31) / 32) * 32;
    c->ldn = ((c->ext_n + 4 + 31) / 32) * 32;
    c->local_nnz_csr = c->local_nnz_csc = nnz;
    DevMem segmem;
    auto counter = [&](const int64_t* dstart, const int32_t* didx, int32_t n_out) {
        return SegCounter{[&c, &segmem, dstart, didx, n_out](int32_t pg, int32_t np, std::vector<int32_t>& seg_len) {
            const size_t total = static_cast<size_t>(np) * n_out;
            int32_t* buf = segmem.alloc<int32_t>(total, false);
            seg_count_device(dstart, didx, n_out, pg, np, buf, c->stream);
            CUDA_TRY(cudaGetLastError());
            seg_len.resize(total);
            staged_d2h(seg_len.data(), buf, total * sizeof(int32_t), c->stream);
        }};
    };
    const SegCounter ccsr = counter(d.rs, d.co, m), ccsc = counter(d.cs, d.ro, n);
    c->hcsr = build_sweep_layout(c->row_start_local.data(), nullptr, nullptr, 0, m, nullptr, c->ext_n, 2,
                                 smem_budget(), c->sm_count, true, &ccsr);
    c->hcsc = build_sweep_layout(c->col_start_local.data(), nullptr, nullptr, 0, n, nullptr, c->ext_m, 3,
                                 smem_budget(), c->sm_count, true, &ccsc);
    const double t_layout = now_s();
    set_kernel_attributes();
    const DevSide scsr{d.rs, d.co, d.vr, nnz}, scsc{d.cs, d.ro, d.vc, nnz};
    c->csr = upload_sweep(*c, c->hcsr, &c->A_csr, &scsr);
    c->csc = upload_sweep(*c, c->hcsc, &c->A_csc, &scsc);
    c->unit_loss = c->eval_mem.alloc<double>(std::max(c->csr.n_units, 1));
    c->red_scratch = c->eval_mem.alloc<double>(4096);
    c->red_out = c->eval_mem.alloc<double>(8);
    // ALS streams: the device CSR / CSC themselves (world 1: identity index space)
    const int chunk = als_chunk(c->nnz, c->sm_count);
    AlsLayout lc = build_als_structure(c->row_start_local.data(), 0, m, chunk);
    AlsLayout lr = build_als_structure(c->col_start_local.data(), 0, n, chunk);
    c->als_csr = upload_als(*c, lc, 0);
    c->als_csc = upload_als(*c, lr, 0);
    c->als_csr.idx = d.co;
    c->als_csr.val = d.vr;
    c->als_csc.idx = d.ro;
    c->als_csc.val = d.vc;
    c->d_counter = c->als_mem.alloc<int>(4);
    c->d_status = c->als_mem.alloc<int>(4);
    c->als_built = true;
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    c->setup_seconds = now_s() - t0;
    if (std::getenv("PMF_VERBOSE"))
        std::fprintf(stderr,
                     "[pmf] ctx from triplets %.3f s: upload %.3f, device CSR/CSC %.3f, offsets %.3f, layout "
                     "structure %.3f, device fill + uploads %.3f\n",
                     c->setup_seconds, tu, tb, t_ingest - t0 - tu - tb, t_layout - t_ingest, now_s() - t_layout);
    return c;
}

// A device group of `world` ranks in this process: rank r owns CSR row block r and CSC column block r
// (the multi-process plan, runtime.hpp:91-136) on devices[r] (default: device r mod the device
// count, so a 1-GPU host runs a group as loopback ranks on one device).  Returns rank 0.
std::unique_ptr<Ctx> make_group(const pmf_matrix_view* a, int world, const int32_t* devices, bool als) {
    if (world < 1) invalid("workers must be >= 1");
    ensure_device();
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev));
    std::vector<std::unique_ptr<Ctx>> rs;
    for (int r = 0; r < world; ++r) {
        const int dev = devices ? devices[r] : r % ndev;
        if (dev < 0 || dev >= ndev) invalid("device index out of range");
        rs.push_back(make_ctx(a, dev, r, world, nullptr));
        if (als) build_als(*rs.back(), a);
    }
    for (int r = 0; r < world; ++r)
        for (int q = 0; q < world; ++q) {
            const int dr = rs[r]->device, dq = rs[q]->device;
            int ok = 0;
            if (dr == dq || cudaDeviceCanAccessPeer(&ok, dr, dq) != cudaSuccess || !ok) continue;
            CUDA_TRY(cudaSetDevice(dr));
            if (cudaDeviceEnablePeerAccess(dq, 0) != cudaSuccess) cudaGetLastError();  // already enabled
        }
    std::unique_ptr<Ctx> c0 = std::move(rs[0]);
    c0->ranks.push_back(c0.get());
    for (int r = 1; r < world; ++r) {
        c0->ranks.push_back(rs[r].get());
        c0->peers.push_back(std::move(rs[r]));
    }
    CUDA_TRY(cudaSetDevice(c0->device));
    return c0;
}

void als_alloc_partials(Ctx& c, int k) {
    // partial buffers depend on k; (re)allocate in model_mem
    const int64_t stride = static_cast<int64_t>(k) * k + k + 1;
    c.als_csr.partial = c.model_mem.alloc<float>(std::max<int64_t>(1, c.als_csr.n_slots * stride), false);
    c.als_csc.partial = c.model_mem.alloc<float>(std::max<int64_t>(1, c.als_csc.n_slots * stride), false);
    const int64_t big = k > 64 ? als_big_scratch_floats(k, c.sm_count) : 0;
    c.als_csr.big_scratch = c.als_csc.big_scratch = big > 0 ? c.model_mem.alloc<float>(big, false) : nullptr;
}

void als_begin(Ctx& c0, const pmf_als_config* cfg) {
    if (!cfg) invalid("config is null");
    // als.hpp:34-39
    if (cfg->k < 1) invalid("k must be >= 1");
    if (!(cfg->lambda > 0.f)) invalid("als requires lambda > 0");
    if (cfg->outer_iters < 1) invalid("outer_iters must be >= 1");
    if (cfg->num_gpus < 1) invalid("workers must be >= 1");
    if (!c0.als_built) invalid("context was created without ALS layouts");
    const auto H = init_items_host(c0.n, cfg->k, cfg->seed);  // model.hpp:86-93, replicated
    for (Ctx* cp : ranks_of(c0)) {
        Ctx& c = *cp;
        CUDA_TRY(cudaSetDevice(c.device));
        reset_graph(c);
        c.model_mem.free_all();
        c.k = cfg->k;
        c.lambda = cfg->lambda;
        c.als_weighted = (cfg->flags & PMF_ALS_WEIGHTED_LAMBDA) != 0;
        c.ccdw_on = false;
        c.W = c.model_mem.alloc<float>(static_cast<size_t>(c.ext_m + 1) * c.k);
        c.H = c.model_mem.alloc<float>(static_cast<size_t>(c.ext_n + 1) * c.k);
        als_alloc_partials(c, c.k);
        upload_rowmajor(c, c.H, c.ext_n, H.data(), c.n, cfg->k, false);
        c.mode = 2;
    }
}

int64_t enqueue_als_iteration(const Ranks& cs) {
    int64_t launched = 0;
    fork_ranks(cs);
    // W phase from the old H, then H phase from the new W (als.hpp:176-184)
    for (Ctx* c : cs)
        launched += launch_als_half(c->als_csr, c->H, c->ext_n, c->W, c->rank * c->Bm, c->k, c->lambda,
                                    c->als_weighted, c->d_counter, c->d_status, c->sm_count, c->stream);
    exchange(cs, [](Ctx& c) { return c.W; }, static_cast<int64_t>(cs[0]->Bm) * cs[0]->k);
    for (Ctx* c : cs)
        launched += launch_als_half(c->als_csc, c->W, c->ext_m, c->H, c->rank * c->Bn, c->k, c->lambda,
                                    c->als_weighted, c->d_counter + 1, c->d_status, c->sm_count, c->stream);
    exchange(cs, [](Ctx& c) { return c.H; }, static_cast<int64_t>(cs[0]->Bn) * cs[0]->k);
    join_ranks(cs);
    return launched;
}

void als_iterate(Ctx& c, int n_outer, double* secs) {
    if (c.mode != 2 || c.ccdw_on) invalid("als_begin has not been called");
    CUDA_TRY(cudaSetDevice(c.device));
    const Ranks cs = ranks_of(c);
    cudaEvent_t e0, e1;
    CUDA_TRY(cudaEventCreate(&e0));
    CUDA_TRY(cudaEventCreate(&e1));
    for (int it = 0; it < n_outer; ++it) {
        for (Ctx* r : cs) CUDA_TRY(cudaMemsetAsync(r->d_status, 0, sizeof(int), r->stream));
        CUDA_TRY(cudaEventRecord(e0, c.stream));
        c.launches_per_iter = enqueue_als_iteration(cs);
        CUDA_TRY(cudaEventRecord(e1, c.stream));
        CUDA_TRY(cudaEventSynchronize(e1));
        float ms = 0;
        CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
        if (secs) secs[it] = ms * 1e-3;
        for (Ctx* r : cs) {
            int st = 0;
            CUDA_TRY(cudaMemcpy(&st, r->d_status, sizeof(int), cudaMemcpyDeviceToHost));
            if (st == 4) throw PmfError(PMF_NOT_POSITIVE_DEFINITE, "non-positive pivot in an ALS row solve");
        }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    CUDA_TRY(cudaGetLastError());
}

// ---- item/user-wise CCD (ccd.hpp:52-125, :310-344) ---------------------------------------------

void ccdw_begin(Ctx& c, const pmf_ccd_config* cfg) {
    if (!cfg) invalid("config is null");
    if (cfg->k < 1) invalid("k must be >= 1");  // ccd.hpp:43-49
    if (cfg->lambda < 0.f) invalid("lambda must be >= 0");
    if (cfg->outer_iters < 1) invalid("outer_iters must be >= 1");
    if (cfg->inner_iters < 1) invalid("inner_iters must be >= 1");
    if (cfg->num_gpus < 1) invalid("workers must be >= 1");
    if (c.world != 1) invalid("item/user-wise CCD runs on one device (ccd.hpp:306-309)");
    if (!c.als_built) invalid("context was created without the plain CSR / CSC layouts");
    if (c.nnz >= (int64_t(1) << 31)) invalid("item/user-wise CCD: more than 2^31 - 1 ratings");
    CUDA_TRY(cudaSetDevice(c.device));
    reset_graph(c);
    c.model_mem.free_all();
    c.ccdw_mem.free_all();
    c.k = cfg->k;
    c.lambda = cfg->lambda;
    // Default: the residual form (warp per row / CTA per column), which updates a float residual
    // entry by entry as the reference does and tracks its trajectory to ~3e-6 over 5 Netflix epochs.
    // PMF_CCD_GRAM=1 (k <= 64): each row's (column's) coordinate sweep as one Gauss-Seidel sweep on
    // its normal equations, gram and right-hand side from the ALS tensor-core kernel, no residual --
    // 10x faster, but it does not carry the reference's residual rounding, and the objectives drift
    // apart (1e-4 relative after 3-4 Netflix epochs).
    const char* gram_env = std::getenv("PMF_CCD_GRAM");
    c.ccdw_gram = als_gram_gs_supported(c.k) && gram_env && std::atoi(gram_env) != 0;
    if (c.ccdw_gram) {
        c.W = c.model_mem.alloc<float>(static_cast<size_t>(c.ext_m + 1) * c.k);  // W = 0 (ccd.hpp:323)
        c.H = c.model_mem.alloc<float>(static_cast<size_t>(c.ext_n + 1) * c.k);
        als_alloc_partials(c, c.k);
        const auto H = init_items_host(c.n, cfg->k, cfg->seed);  // model.hpp:86-93
        upload_rowmajor(c, c.H, c.ext_n, H.data(), c.n, cfg->k, false);
        CUDA_TRY(cudaGetLastError());
        c.mode = 2;
        c.ccdw_on = true;
        return;
    }
    CcdWs& w = c.ccdw;
    w.m = c.m;
    w.n = c.n;
    w.nnz = c.nnz;
    w.row_start = c.ccdw_mem.upload(c.row_start_local, c.stream, &c.h2d);
    w.col_start = c.ccdw_mem.upload(c.col_start_local, c.stream, &c.h2d);
    w.col_of = c.als_csr.idx;  // world == 1: the padded index space is the identity
    w.row_of = c.als_csc.idx;
    const size_t N = static_cast<size_t>(std::max<int64_t>(c.nnz, 1));
    w.R_row = c.ccdw_mem.alloc<float>(N, false);
    w.R_col = c.ccdw_mem.alloc<float>(N, false);
    w.csr2csc = c.ccdw_mem.alloc<int32_t>(N, false);
    w.csc2csr = c.ccdw_mem.alloc<int32_t>(N, false);
    if (c.nnz > 0) {  // residual_from (sparse.hpp:259-262): R = A, W = 0
        CUDA_TRY(cudaMemcpyAsync(w.R_row, c.als_csr.val, sizeof(float) * c.nnz, cudaMemcpyDeviceToDevice, c.stream));
        CUDA_TRY(cudaMemcpyAsync(w.R_col, c.als_csc.val, sizeof(float) * c.nnz, cudaMemcpyDeviceToDevice, c.stream));
    }
    launch_ccd_xlinks(w.row_start, w.col_of, w.col_start, w.row_of, w.m, w.csr2csc, w.csc2csr, c.stream);
    {  // H sweep: W column-major copy, columns longest first
        w.WT = c.ccdw_mem.alloc<float>(static_cast<size_t>(std::max<int32_t>(c.m, 1)) * c.k, false);
        std::vector<int32_t> order(c.n);
        std::iota(order.begin(), order.end(), 0);
        const auto& cs = c.col_start_local;
        std::stable_sort(order.begin(), order.end(),
                         [&](int32_t a, int32_t b) { return cs[a + 1] - cs[a] > cs[b + 1] - cs[b]; });
        w.col_order = c.ccdw_mem.upload(order, c.stream, &c.h2d);
        w.counter = c.ccdw_mem.alloc<int>(1);
    }
    c.W = c.model_mem.alloc<float>(static_cast<size_t>(c.ext_m + 1) * c.k);
    c.H = c.model_mem.alloc<float>(static_cast<size_t>(c.ext_n + 1) * c.k);
    const auto H = init_items_host(c.n, cfg->k, cfg->seed);  // model.hpp:86-93
    upload_rowmajor(c, c.H, c.ext_n, H.data(), c.n, cfg->k, false);
    CUDA_TRY(cudaGetLastError());
    c.mode = 2;  // row-major model: the ALS views serve metrics / model download
    c.ccdw_on = true;
}

void ccdw_iterate(Ctx& c, int n_outer, double* secs) {
    if (c.mode != 2 || !c.ccdw_on) invalid("ccd_begin has not been called");
    CUDA_TRY(cudaSetDevice(c.device));
    cudaEvent_t e0, e1;
    CUDA_TRY(cudaEventCreate(&e0));
    CUDA_TRY(cudaEventCreate(&e1));
    for (int it = 0; it < n_outer; ++it) {
        CUDA_TRY(cudaEventRecord(e0, c.stream));
        if (c.ccdw_gram) {  // W sweep with H fixed, then H sweep with the new W (ccd.hpp:113-119)
            const int a = launch_als_half(c.als_csr, c.H, c.ext_n, c.W, 0, c.k, c.lambda, false, c.d_counter,
                                          c.d_status, c.sm_count, c.stream, true);
            const int b = launch_als_half(c.als_csc, c.W, c.ext_m, c.H, 0, c.k, c.lambda, false, c.d_counter + 1,
                                          c.d_status, c.sm_count, c.stream, true);
            if (a < 0 || b < 0) throw PmfError(PMF_RUNTIME_ERROR, "item/user-wise CCD: gram path unavailable");
            c.launches_per_iter = a + b;
        } else {
            c.launches_per_iter = launch_ccd_epoch(c.ccdw, c.W, c.H, c.k, c.lambda, c.stream);
        }
        CUDA_TRY(cudaEventRecord(e1, c.stream));
        CUDA_TRY(cudaEventSynchronize(e1));
        float ms = 0;
        CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
        if (secs) secs[it] = ms * 1e-3;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    CUDA_TRY(cudaGetLastError());
}

// ---- metrics ------------------------------------------------------------------------------------

FactorView wview(const Ctx& c) {
    if (c.mode == 1) return FactorView{c.W, 1, c.ldm};
    return FactorView{c.W, c.k, 1};
}
FactorView hview(const Ctx& c) {
    if (c.mode == 1) return FactorView{c.H, 1, c.ldn};
    return FactorView{c.H, c.k, 1};
}

// Enqueues this rank's metric terms into c.red_out: [0] its CSR block's squared error, [1] |W|^2,
// [2] |H|^2, [3] the probe SSE (the last three over the replicated model).
void enqueue_metric_terms(Ctx& c) {
    CUDA_TRY(cudaSetDevice(c.device));
    FactorView W = wview(c), H = hview(c);
    if (c.mode == 1) {
        // CCD++ keeps the factors column-major (k vectors); the per-entry dots read rows, so the
        // metric kernels see row-major copies (same values, same t order, 4x fewer sector reads)
        const size_t need = (static_cast<size_t>(c.ext_m) + c.ext_n) * c.k;
        if (need != c.rm_floats) {
            c.rm_mem.free_all();
            c.w_rm = c.rm_mem.alloc<float>(static_cast<size_t>(c.ext_m) * c.k, false);
            c.h_rm = c.rm_mem.alloc<float>(static_cast<size_t>(c.ext_n) * c.k, false);
            c.rm_floats = need;
        }
        launch_transpose(c.W, c.ldm, c.k, c.ext_m, c.w_rm, c.stream);
        launch_transpose(c.H, c.ldn, c.k, c.ext_n, c.h_rm, c.stream);
        W = FactorView{c.w_rm, c.k, 1};
        H = FactorView{c.h_rm, c.k, 1};
    }
    launch_unit_loss(c.csr, c.A_csr, c.rank * c.Bm, W, H, c.k, c.unit_loss, c.stream);
    launch_sum(c.unit_loss, c.csr.n_units, c.red_scratch, c.red_out + 0, c.stream);
    const int64_t wn = c.mode == 1 ? static_cast<int64_t>(c.k) * c.ldm : static_cast<int64_t>(c.ext_m + 1) * c.k;
    const int64_t hn = c.mode == 1 ? static_cast<int64_t>(c.k) * c.ldn : static_cast<int64_t>(c.ext_n + 1) * c.k;
    launch_sumsq(c.W, wn, c.red_scratch + 1024, c.red_out + 1, c.stream);
    launch_sumsq(c.H, hn, c.red_scratch + 2048, c.red_out + 2, c.stream);
    if (c.n_probe > 0) launch_probe_sse(c.probe, c.n_probe, W, H, c.k, c.red_scratch + 3072, c.red_out + 3, c.stream);
    if (c.comm) NCCL_TRY(ncclAllReduce(c.red_out, c.red_out, 1, ncclDouble, ncclSum, c.comm, c.stream));
}

void metrics(Ctx& c, double* objective, double* rmse, double* train_rmse) {
    if (c.mode == 0) invalid("no model: call ccdpp_begin or als_begin first");
    const Ranks cs = ranks_of(c);
    for (Ctx* r : cs) enqueue_metric_terms(*r);
    double h[4] = {0, 0, 0, 0};
    for (Ctx* r : cs) {  // a group's squared error: its row blocks' sums in rank order
        double t[4];
        CUDA_TRY(cudaSetDevice(r->device));
        CUDA_TRY(cudaMemcpyAsync(t, r->red_out, sizeof(t), cudaMemcpyDeviceToHost, r->stream));
        CUDA_TRY(cudaStreamSynchronize(r->stream));
        h[0] += t[0];
        if (r == cs[0]) std::copy(t + 1, t + 4, h + 1);
    }
    CUDA_TRY(cudaSetDevice(c.device));
    const double lam = static_cast<double>(c.lambda);  // Real lambda widened (ccd.hpp:394)
    if (objective) *objective = h[0] + lam * (h[1] + h[2]);
    if (train_rmse) *train_rmse = c.nnz > 0 ? std::sqrt(h[0] / static_cast<double>(c.nnz)) : 0.0;
    if (rmse) *rmse = c.n_probe > 0 ? std::sqrt(h[3] / static_cast<double>(c.n_probe)) : std::nan("");
}

void set_probe_one(Ctx& c, const pmf_triplet* probe, int64_t n) {
    if (n < 0 || (n > 0 && !probe)) invalid("probe is null");
    for (int64_t x = 0; x < n; ++x)
        if (probe[x].user < 0 || probe[x].user >= c.m || probe[x].item < 0 || probe[x].item >= c.n)
            invalid("probe index outside training dimensions");  // ccd.hpp:298-303
    CUDA_TRY(cudaSetDevice(c.device));
    c.probe_mem.free_all();
    c.probe = nullptr;
    c.n_probe = n;
    if (n == 0) return;
    std::vector<DevTriplet> t(n);
    for (int64_t x = 0; x < n; ++x) t[x] = DevTriplet{c.prow(probe[x].user), c.pcol(probe[x].item), probe[x].rating};
    c.probe = c.probe_mem.upload(t, c.stream, &c.h2d);
    CUDA_TRY(cudaStreamSynchronize(c.stream));
}
void set_probe(Ctx& c, const pmf_triplet* probe, int64_t n) {
    for (Ctx* r : ranks_of(c)) set_probe_one(*r, probe, n);
}

void get_model(Ctx& c, float* W, float* H) {
    if (c.mode == 0) invalid("no model");
    CUDA_TRY(cudaSetDevice(c.device));
    const int k = c.k;
    if (c.mode == 1 && c.world == 1) {
        // transpose column-major k x ld -> row-major on the device, then a staged download
        const double t0 = now_s();
        DevMem tmp;
        float* wt = tmp.alloc<float>(static_cast<size_t>(c.m) * k, false);
        float* ht = tmp.alloc<float>(static_cast<size_t>(c.n) * k, false);
        launch_transpose(c.W, c.ldm, k, c.m, wt, c.stream);
        launch_transpose(c.H, c.ldn, k, c.n, ht, c.stream);
        CUDA_TRY(cudaStreamSynchronize(c.stream));
        const double t1 = now_s();
        if (W) staged_d2h(W, wt, sizeof(float) * c.m * k, c.stream);
        if (H) staged_d2h(H, ht, sizeof(float) * c.n * k, c.stream);
        CUDA_TRY(cudaStreamSynchronize(c.stream));
        if (std::getenv("PMF_VERBOSE"))
            std::fprintf(stderr, "[pmf] get_model: alloc + transpose %.3f s, download %.3f s\n", t1 - t0, now_s() - t1);
        c.d2h += static_cast<int64_t>(sizeof(float) * (static_cast<int64_t>(c.m) + c.n) * k);
    } else if (c.mode == 1) {
        std::vector<float> w(static_cast<size_t>(k) * c.ldm), h(static_cast<size_t>(k) * c.ldn);
        CUDA_TRY(cudaMemcpy(w.data(), c.W, w.size() * sizeof(float), cudaMemcpyDeviceToHost));
        CUDA_TRY(cudaMemcpy(h.data(), c.H, h.size() * sizeof(float), cudaMemcpyDeviceToHost));
        c.d2h += static_cast<int64_t>((w.size() + h.size()) * sizeof(float));
        if (W)
            for (int32_t i = 0; i < c.m; ++i)
                for (int t = 0; t < k; ++t) W[static_cast<size_t>(i) * k + t] = w[static_cast<size_t>(t) * c.ldm + c.prow(i)];
        if (H)
            for (int32_t j = 0; j < c.n; ++j)
                for (int t = 0; t < k; ++t) H[static_cast<size_t>(j) * k + t] = h[static_cast<size_t>(t) * c.ldn + c.pcol(j)];
    } else {
        std::vector<float> w(static_cast<size_t>(c.ext_m) * k), h(static_cast<size_t>(c.ext_n) * k);
        CUDA_TRY(cudaMemcpy(w.data(), c.W, w.size() * sizeof(float), cudaMemcpyDeviceToHost));
        CUDA_TRY(cudaMemcpy(h.data(), c.H, h.size() * sizeof(float), cudaMemcpyDeviceToHost));
        c.d2h += static_cast<int64_t>((w.size() + h.size()) * sizeof(float));
        if (W)
            for (int32_t i = 0; i < c.m; ++i)
                std::memcpy(W + static_cast<size_t>(i) * k, &w[static_cast<size_t>(c.prow(i)) * k], sizeof(float) * k);
        if (H)
            for (int32_t j = 0; j < c.n; ++j)
                std::memcpy(H + static_cast<size_t>(j) * k, &h[static_cast<size_t>(c.pcol(j)) * k], sizeof(float) * k);
    }
}

// Installs a model.  The residual solvers' state follows it: CCD++ gets R = A - W H^T in the
// deferred form its first sweep expects (column k-1's product still to be subtracted, so the next
// sweep completes A - sum_t w_t h_t in ascending t), item/user-wise CCD R = A - W H^T in both layouts.
void set_model_one(Ctx& c, const float* W, const float* H, int k, bool residual) {
    if (c.mode == 0) invalid("no model: call ccdpp_begin or als_begin first");
    if (k != c.k) invalid("rank does not match the active model");
    if (!W || !H) invalid("null buffers");
    CUDA_TRY(cudaSetDevice(c.device));
    if (c.mode == 1) {
        upload_colmajor(c, c.W, c.ldm, W, c.m, k, true);
        upload_colmajor(c, c.H, c.ldn, H, c.n, k, false);
        if (residual) reset_residual(c);
        for (int t = 0; residual && t + 1 < k; ++t) {
            SweepOperands o1, o2;
            o1.oa = c.W + static_cast<int64_t>(t) * c.ldm;
            o1.ga = c.H + static_cast<int64_t>(t) * c.ldn;
            o2.oa = c.H + static_cast<int64_t>(t) * c.ldn;
            o2.ga = c.W + static_cast<int64_t>(t) * c.ldm;
            launch_sweep(c.csr, kDemote, true, o1, c.stream);
            launch_sweep(c.csc, kDemote, false, o2, c.stream);
        }
    } else {
        upload_rowmajor(c, c.W, c.ext_m, W, c.m, k, true);
        upload_rowmajor(c, c.H, c.ext_n, H, c.n, k, false);
        if (c.ccdw_on && !c.ccdw_gram) launch_ccd_residual(c.ccdw, c.als_csr.val, c.W, c.H, k, c.stream);
    }
    CUDA_TRY(cudaStreamSynchronize(c.stream));
    CUDA_TRY(cudaGetLastError());
}
void set_model(Ctx& c, const float* W, const float* H, int k, bool residual = true) {
    for (Ctx* r : ranks_of(c)) set_model_one(*r, W, H, k, residual);
}

// host scatter/gather between reference order and the padded layout
void put_values(Ctx& c, const SweepLayout& L, float* dst, const float* src, const std::vector<int64_t>& start) {
    std::vector<float> tmp(L.n_entries, 0.f);
    const int64_t base = start[0];
    for_each_entry(L, [&](int32_t o, int64_t r, int64_t p) { tmp[p] = src[start[o] - base + r]; });
    CUDA_TRY(cudaMemcpyAsync(dst, tmp.data(), tmp.size() * sizeof(float), cudaMemcpyHostToDevice, c.stream));
    CUDA_TRY(cudaStreamSynchronize(c.stream));
}

void get_values(Ctx& c, const SweepLayout& L, const float* src, float* dst, const std::vector<int64_t>& start) {
    std::vector<float> tmp(L.n_entries);
    CUDA_TRY(cudaMemcpy(tmp.data(), src, tmp.size() * sizeof(float), cudaMemcpyDeviceToHost));
    const int64_t base = start[0];
    for_each_entry(L, [&](int32_t o, int64_t r, int64_t p) { dst[start[o] - base + r] = tmp[p]; });
}

void get_residual(Ctx& c, float* r_row, float* r_col) {
    if (c.mode != 1) invalid("no CCD++ state");
    if (c.world > 1) invalid("residual readback is single-GPU only");
    CUDA_TRY(cudaSetDevice(c.device));
    // apply the deferred writeback of the last step (t = k-1) on copies
    const int tp = c.k - 1;
    DevMem tmp;
    DevSweep r = c.csr, q = c.csc;
    r.R = tmp.alloc<float>(c.csr.n_entries + kStreamSlack, false);
    q.R = tmp.alloc<float>(c.csc.n_entries + kStreamSlack, false);
    CUDA_TRY(cudaMemcpyAsync(r.R, c.csr.R, c.csr.n_entries * sizeof(float), cudaMemcpyDeviceToDevice, c.stream));
    CUDA_TRY(cudaMemcpyAsync(q.R, c.csc.R, c.csc.n_entries * sizeof(float), cudaMemcpyDeviceToDevice, c.stream));
    SweepOperands o1;
    o1.oa = c.W + static_cast<int64_t>(tp) * c.ldm;
    o1.ga = c.H + static_cast<int64_t>(tp) * c.ldn;
    launch_sweep(r, kDemote, true, o1, c.stream);
    SweepOperands o2;
    o2.oa = c.H + static_cast<int64_t>(tp) * c.ldn;
    o2.ga = c.W + static_cast<int64_t>(tp) * c.ldm;
    launch_sweep(q, kDemote, false, o2, c.stream);
    CUDA_TRY(cudaStreamSynchronize(c.stream));
    if (r_row) get_values(c, c.hcsr, r.R, r_row, c.row_start_local);
    if (r_col) get_values(c, c.hcsc, q.R, r_col, c.col_start_local);
}

Ctx* as_ctx(pmf_ctx* p) {
    if (!p) invalid("context is null");
    return reinterpret_cast<Ctx*>(p);
}

}  // namespace pmfgpu

using namespace pmfgpu;

extern "C" {

const char* pmf_last_error(void) { return g_err.c_str(); }
int32_t pmf_abi_version(void) { return PMF_ABI_VERSION; }
pmf_status pmf_release_cached_memory(int64_t* released) {
    return guard([&] {
        const int64_t b = block_cache().flush() + pinned_pool().release_idle();
        if (released) *released = b;
    });
}

int32_t pmf_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return c;
}

pmf_status pmf_ctx_create(const pmf_matrix_view* a, int32_t device, pmf_ctx** out) {
    return guard([&] {
        if (!out) invalid("out is null");
        auto c = make_ctx(a, device, 0, 1, nullptr);
        build_als(*c, a);
        *out = reinterpret_cast<pmf_ctx*>(c.release());
    });
}

pmf_status pmf_ctx_create_from_triplets(const pmf_triplet* triplets, int64_t nnz, int32_t m, int32_t n,
                                        int32_t device, pmf_ctx** out) {
    return guard([&] {
        if (!out) invalid("out is null");
        auto c = make_ctx_from_triplets(triplets, nnz, m, n, device);
        *out = reinterpret_cast<pmf_ctx*>(c.release());
    });
}

pmf_status pmf_ctx_create_dist(const pmf_matrix_view* a, int32_t device, int32_t rank, int32_t world,
                               const uint8_t* id, pmf_ctx** out) {
    return guard([&] {
        if (!out) invalid("out is null");
        if (world < 1 || rank < 0 || rank >= world) invalid("invalid rank / world");
        if (!id) invalid("nccl id is null");
        auto c = make_ctx(a, device, rank, world, id);
        build_als(*c, a);
        *out = reinterpret_cast<pmf_ctx*>(c.release());
    });
}

pmf_status pmf_ctx_create_group(const pmf_matrix_view* a, int32_t num_gpus, const int32_t* devices, pmf_ctx** out) {
    return guard([&] {
        if (!out) invalid("out is null");
        auto c = make_group(a, num_gpus, devices, true);
        *out = reinterpret_cast<pmf_ctx*>(c.release());
    });
}

pmf_status pmf_dist_plan(const pmf_matrix_view* a, int32_t world, int32_t* row_bounds, int32_t* col_bounds,
                         int32_t* block_rows, int32_t* block_cols) {
    return guard([&] {
        check_view(a);
        if (world < 1) invalid("world must be >= 1");
        if (!row_bounds || !col_bounds || !block_rows || !block_cols) invalid("null buffers");
        dist_plan(a->row_start, a->m, a->col_start, a->n, world, row_bounds, col_bounds, block_rows, block_cols);
    });
}

pmf_status pmf_nccl_unique_id(uint8_t* out128) {
    return guard([&] {
        if (!out128) invalid("out is null");
        ncclUniqueId id;
        NCCL_TRY(ncclGetUniqueId(&id));
        std::memcpy(out128, &id, sizeof(id));
    });
}

pmf_status pmf_ctx_destroy(pmf_ctx* ctx) {
    return guard([&] { delete as_ctx(ctx); });
}

pmf_status pmf_ctx_ccdpp_begin(pmf_ctx* ctx, const pmf_ccd_config* cfg) {
    return guard([&] { ccd_begin(*as_ctx(ctx), cfg); });
}
pmf_status pmf_ctx_ccdpp_iterate(pmf_ctx* ctx, int32_t n_outer, double* secs) {
    return guard([&] { ccd_iterate(*as_ctx(ctx), n_outer, secs); });
}
pmf_status pmf_ctx_ccd_begin(pmf_ctx* ctx, const pmf_ccd_config* cfg) {
    return guard([&] { ccdw_begin(*as_ctx(ctx), cfg); });
}
pmf_status pmf_ctx_ccd_iterate(pmf_ctx* ctx, int32_t n_outer, double* secs) {
    return guard([&] { ccdw_iterate(*as_ctx(ctx), n_outer, secs); });
}
pmf_status pmf_ctx_als_begin(pmf_ctx* ctx, const pmf_als_config* cfg) {
    return guard([&] { als_begin(*as_ctx(ctx), cfg); });
}
pmf_status pmf_ctx_als_iterate(pmf_ctx* ctx, int32_t n_outer, double* secs) {
    return guard([&] { als_iterate(*as_ctx(ctx), n_outer, secs); });
}
pmf_status pmf_ctx_set_probe(pmf_ctx* ctx, const pmf_triplet* probe, int64_t n) {
    return guard([&] { set_probe(*as_ctx(ctx), probe, n); });
}
pmf_status pmf_ctx_metrics(pmf_ctx* ctx, double* objective, double* rmse, double* train_rmse) {
    return guard([&] { metrics(*as_ctx(ctx), objective, rmse, train_rmse); });
}
pmf_status pmf_ctx_get_model(pmf_ctx* ctx, float* W, float* H) {
    return guard([&] { get_model(*as_ctx(ctx), W, H); });
}
pmf_status pmf_ctx_set_model(pmf_ctx* ctx, const float* W, const float* H, int32_t k) {
    return guard([&] { set_model(*as_ctx(ctx), W, H, k); });
}
pmf_status pmf_ctx_get_residual(pmf_ctx* ctx, float* r_row, float* r_col) {
    return guard([&] { get_residual(*as_ctx(ctx), r_row, r_col); });
}
pmf_status pmf_ctx_set_profiling(pmf_ctx* ctx, int32_t on) {
    return guard([&] {
        Ctx& c = *as_ctx(ctx);
        c.profiling = on != 0;
        reset_graph(c);
    });
}
pmf_status pmf_ctx_debug_sweep_profile(pmf_ctx* ctx, int32_t side, int32_t promote, uint64_t* cta_ns,
                                      int64_t* cta_stats, int32_t* n_ctas) {
    return guard([&] {
        Ctx& c = *as_ctx(ctx);
        if (c.mode != 1) invalid("ccdpp_begin has not been called");
        const DevSweep& L = side == 0 ? c.csr : c.csc;
        const SweepLayout& H = side == 0 ? c.hcsr : c.hcsc;
        *n_ctas = L.ctas;
        DevMem tmp;
        auto* clk = tmp.alloc<unsigned long long>(2 * L.ctas);
        SweepOperands op;
        op.lambda = c.lambda;
        op.cta_clock = clk;
        const int t = 0, tp = c.k - 1;
        if (side == 0) {
            op.out = c.ubuf; op.out_off = c.rank * c.Bm;
            op.gn = promote ? c.H : c.vbuf; op.ga = c.H + static_cast<int64_t>(tp) * c.ldn; op.gb = c.H;
            op.oa = c.W + static_cast<int64_t>(tp) * c.ldm; op.ob = c.W;
        } else {
            op.out = c.vbuf; op.out_off = c.rank * c.Bn;
            op.gn = c.ubuf; op.ga = c.W + static_cast<int64_t>(tp) * c.ldm; op.gb = c.W;
            op.oa = c.H + static_cast<int64_t>(tp) * c.ldn; op.ob = c.H;
        }
        (void)t;
        // work on a copy of R so the training state is untouched
        DevSweep Lc = L;
        Lc.R = tmp.alloc<float>(L.n_entries + kStreamSlack, false);
        CUDA_TRY(cudaMemcpyAsync(Lc.R, L.R, L.n_entries * sizeof(float), cudaMemcpyDeviceToDevice, c.stream));
        launch_sweep(Lc, promote ? kPromote : kPlain, side == 0, op, c.stream);
        CUDA_TRY(cudaStreamSynchronize(c.stream));
        CUDA_TRY(cudaMemcpy(cta_ns, clk, sizeof(uint64_t) * 2 * L.ctas, cudaMemcpyDeviceToHost));
        if (cta_stats) {
            constexpr int W = 24;
            for (int x = 0; x < W * L.ctas; ++x) cta_stats[x] = 0;
            for (int cc = 0; cc < L.ctas; ++cc)
                for (int p = H.piece_start[cc]; p < H.piece_start[cc + 1]; ++p) {
                    const Piece& pz = H.pieces[p];
                    int64_t* st = cta_stats + W * cc;
                    st[0] += pz.um - pz.ub;
                    st[1] += pz.us - pz.um;
                    st[2] += pz.ue - pz.us;
                    for (int u = pz.ub; u < pz.ue; ++u) {
                        const int len = H.units[u].len;
                        const int cls = u < pz.um ? 0 : u < pz.us ? 1 : 2;
                        const int g = 8 >> cls;
                        st[3] += len;
                        st[6 + cls] += len;
                        for (int j = 0; j < 4; ++j) {
                            const int step = 4 * g << j;
                            st[9 + 3 * j + cls] += (len + step - 1) / step;
                        }
                    }
                    st[4] += 1;
                    st[5] = pz.panel;
                }
        }
    });
}

pmf_status pmf_ctx_launch_count(pmf_ctx* ctx, int64_t* per_iteration) {
    return guard([&] {
        if (!per_iteration) invalid("out is null");
        *per_iteration = as_ctx(ctx)->launches_per_iter;
    });
}
pmf_status pmf_ctx_kernel_stats(pmf_ctx* ctx, double* u_ms, int64_t* u_n, double* v_ms, int64_t* v_n) {
    return guard([&] {
        Ctx& c = *as_ctx(ctx);
        if (u_ms) *u_ms = c.stat_u_ms;
        if (u_n) *u_n = c.stat_u_n;
        if (v_ms) *v_ms = c.stat_v_ms;
        if (v_n) *v_n = c.stat_v_n;
    });
}

pmf_status pmf_matrix_from_triplets_gpu(const pmf_triplet* t, int64_t nnz, int32_t m, int32_t n,
                                        int64_t* row_start, int32_t* col_of, float* val_row, int64_t* col_start,
                                        int32_t* row_of, float* val_col) {
    return guard([&] {
        check_triplet_args(t, nnz, m, n);
        if (nnz > 0 && (!col_of || !val_row || !row_of || !val_col)) invalid("from_triplets: null buffers");
        if (!row_start || !col_start) invalid("from_triplets: null buffers");
        ensure_device();
        cudaStream_t s = nullptr;
        CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        struct StreamGuard {
            cudaStream_t s;
            ~StreamGuard() { cudaStreamDestroy(s); }
        } sg{s};
        DevMem mem;
        double tu = 0, tb = 0;
        const DevCsr d = device_ingest(t, nnz, m, n, s, mem, mem, &tu, &tb);
        const double t2 = now_s();
        staged_d2h(row_start, d.rs, sizeof(int64_t) * (static_cast<size_t>(m) + 1), s);
        staged_d2h(col_start, d.cs, sizeof(int64_t) * (static_cast<size_t>(n) + 1), s);
        if (nnz > 0) {
            staged_d2h(col_of, d.co, sizeof(int32_t) * static_cast<size_t>(nnz), s);
            staged_d2h(val_row, d.vr, sizeof(float) * static_cast<size_t>(nnz), s);
            staged_d2h(row_of, d.ro, sizeof(int32_t) * static_cast<size_t>(nnz), s);
            staged_d2h(val_col, d.vc, sizeof(float) * static_cast<size_t>(nnz), s);
        }
        if (std::getenv("PMF_VERBOSE"))
            std::fprintf(stderr, "[pmf] from_triplets_gpu: alloc + upload %.3f s, build %.3f, download %.3f\n", tu, tb,
                         now_s() - t2);
    });
}

pmf_status pmf_top_n(const float* W, const float* H, int32_t m, int32_t n, int32_t k, const int32_t* users,
                     int32_t n_users, int32_t count, const int64_t* ex_start, const int32_t* ex_items,
                     int32_t* out_items, float* out_scores, int32_t* out_count) {
    return guard([&] {
        if (count < 1) invalid("count must be >= 1");  // model.hpp:175
        if (m < 0 || n < 0 || k < 1 || n_users < 0) invalid("invalid dimensions");
        if (n_users > 0 && (!users || !ex_start || !out_items || !out_scores || !out_count)) invalid("null buffers");
        if ((m > 0 && !W) || (n > 0 && !H)) invalid("null factors");
        for (int32_t u = 0; u < n_users; ++u)
            if (users[u] < 0 || users[u] >= m) throw PmfError(PMF_OUT_OF_RANGE, "user index out of range");
        if (n_users > 0 && ex_start[0] != 0) invalid("exclusion offsets must start at 0");
        for (int32_t u = 0; u < n_users; ++u) {
            if (ex_start[u + 1] < ex_start[u]) invalid("exclusion offsets must be non-decreasing");
            for (int64_t p = ex_start[u] + 1; p < ex_start[u + 1]; ++p)
                if (ex_items[p] <= ex_items[p - 1]) invalid("rated items must be strictly increasing");
        }
        // the tiled kernel keeps each user's list in shared memory; larger k x count take the wide
        // path (full scoring + segmented sort), with the same results
        const size_t smem = topn_smem_bytes(k, count);
        constexpr size_t kTopnSmemMax = 224 * 1024;  // + the kernel's static shared memory <= 227 KB
        const bool wide = smem > kTopnSmemMax;
        if (n_users == 0) return;
        ensure_device();
        static bool attr = false;
        if (!attr) {
            topn_set_attributes(kTopnSmemMax);
            attr = true;
        }
        cudaStream_t s = nullptr;
        CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        struct StreamGuard {
            cudaStream_t s;
            ~StreamGuard() { cudaStreamDestroy(s); }
        } sg{s};
        DevMem mem;
        const int64_t n_ex = ex_start[n_users];
        float* dW = mem.alloc<float>(static_cast<size_t>(m) * k, false);
        float* dH = mem.alloc<float>(static_cast<size_t>(n) * k, false);
        int32_t* du = mem.alloc<int32_t>(n_users, false);
        int64_t* des = mem.alloc<int64_t>(static_cast<size_t>(n_users) + 1, false);
        int32_t* dex = mem.alloc<int32_t>(static_cast<size_t>(std::max<int64_t>(n_ex, 1)), false);
        int32_t* doi = mem.alloc<int32_t>(static_cast<size_t>(n_users) * count, false);
        float* dos = mem.alloc<float>(static_cast<size_t>(n_users) * count, false);
        int32_t* doc = mem.alloc<int32_t>(n_users, false);
        staged_h2d(dW, W, sizeof(float) * static_cast<size_t>(m) * k, s);
        staged_h2d(dH, H, sizeof(float) * static_cast<size_t>(n) * k, s);
        staged_h2d(du, users, sizeof(int32_t) * n_users, s);
        staged_h2d(des, ex_start, sizeof(int64_t) * (static_cast<size_t>(n_users) + 1), s);
        if (n_ex > 0) staged_h2d(dex, ex_items, sizeof(int32_t) * static_cast<size_t>(n_ex), s);
        cudaEvent_t e0, e1;
        CUDA_TRY(cudaEventCreate(&e0));
        CUDA_TRY(cudaEventCreate(&e1));
        CUDA_TRY(cudaEventRecord(e0, s));
        if (wide) {
            const int batch = std::min(topn_wide_batch(n), n_users);
            void* scratch = mem.alloc<char>(topn_wide_scratch_bytes(n, batch), false);
            CUDA_TRY(launch_topn_wide(dW, dH, n, k, du, n_users, des, dex, count, doi, dos, doc, scratch, batch, s));
        } else {
            launch_topn(dW, dH, n, k, du, n_users, des, dex, count, doi, dos, doc, s);
        }
        CUDA_TRY(cudaEventRecord(e1, s));
        CUDA_TRY(cudaGetLastError());
        if (std::getenv("PMF_VERBOSE")) {
            CUDA_TRY(cudaEventSynchronize(e1));
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            std::fprintf(stderr, "[pmf] top_n: %d users, kernel %.3f ms\n", n_users, ms);
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        staged_d2h(out_items, doi, sizeof(int32_t) * static_cast<size_t>(n_users) * count, s);
        staged_d2h(out_scores, dos, sizeof(float) * static_cast<size_t>(n_users) * count, s);
        staged_d2h(out_count, doc, sizeof(int32_t) * n_users, s);
    });
}

pmf_status pmf_ctx_layout_info(pmf_ctx* ctx, int32_t side, pmf_layout_info* out) {
    return guard([&] {
        Ctx& c = *as_ctx(ctx);
        if (!out) invalid("out is null");
        if (side != 0 && side != 1) invalid("side must be 0 (CSR) or 1 (CSC)");
        const SweepLayout& H = side == 0 ? c.hcsr : c.hcsc;
        out->n_panels = H.n_panels;
        out->panel_size = H.panel_size;
        out->smem = H.smem ? 1 : 0;
        out->idx16 = H.idx16 ? 1 : 0;
        out->promote_fused = H.promote_fused ? 1 : 0;
        out->rmw_sub = H.rmw_sub;
        out->sub_width = H.sub_width;
        out->n_units = static_cast<int32_t>(H.units.size());
        out->n_slots = H.n_slots;
        out->ctas = H.ctas;
        out->n_entries = H.n_entries;
        out->n_real = H.n_real;
    });
}

}  // extern "C"

template <class Begin, class Iterate>
static pmf_status train_common(const pmf_matrix_view* a, int outer, int world, bool als, const pmf_triplet* probe,
                               int64_t n_probe, float* W_out, float* H_out, pmf_iter_row* rows,
                               pmf_train_totals* totals, Begin begin, Iterate iterate) {
    return guard([&] {
        const double t0 = now_s();
        if (!rows) invalid("rows_out is null");
        if (n_probe < 0 || (n_probe > 0 && !probe)) invalid("probe is null");
        check_view(a);
        for (int64_t x = 0; x < n_probe; ++x)
            if (probe[x].user < 0 || probe[x].user >= a->m || probe[x].item < 0 || probe[x].item >= a->n)
                invalid("probe index outside training dimensions");
        const double t_val = now_s();
        if (world < 1) invalid("workers must be >= 1");
        auto c = world == 1 ? make_ctx(a, -1, 0, 1, nullptr) : make_group(a, world, nullptr, als);
        if (world == 1 && als) build_als(*c, a);
        const double t_ctx = now_s();
        begin(*c);
        set_probe(*c, probe, n_probe);
        const double t_begin = now_s();
        double train = 0, t_iter = 0, t_metrics = 0;
        for (int it = 1; it <= outer; ++it) {
            double s = 0;
            const double ta = now_s();
            iterate(*c, &s);
            const double tb = now_s();
            pmf_iter_row& r = rows[it - 1];
            r.iteration = it;
            r.seconds = s;
            metrics(*c, &r.objective, &r.rmse, &r.train_rmse);
            t_iter += tb - ta;
            t_metrics += now_s() - tb;
            train += s;
        }
        const double t_model = now_s();
        get_model(*c, W_out, H_out);
        if (std::getenv("PMF_VERBOSE"))
            std::fprintf(stderr,
                         "[pmf] train: validate %.3f s, context %.3f, begin+probe %.3f, iterate %.3f (device %.3f), "
                         "metrics %.3f, model download %.3f\n",
                         t_val - t0, t_ctx - t_val, t_begin - t_ctx, t_iter, train, t_metrics, now_s() - t_model);
        if (totals) {
            totals->train_seconds = train;
            totals->final_objective = rows[outer - 1].objective;
            totals->final_rmse = rows[outer - 1].rmse;
            totals->setup_seconds = world == 1 ? c->setup_seconds : t_ctx - t_val;
            totals->h2d_bytes = totals->d2h_bytes = 0;
            for (Ctx* r : ranks_of(*c)) {
                totals->h2d_bytes += r->h2d;
                totals->d2h_bytes += r->d2h;
            }
            totals->kernel_launches = c->launches_per_iter * outer;
            totals->wall_seconds = now_s() - t0;
        }
    });
}

extern "C" {

pmf_status pmf_ccdpp_train(const pmf_ccd_config* cfg, const pmf_matrix_view* a, const pmf_triplet* probe,
                           int64_t n_probe, float* W_out, float* H_out, pmf_iter_row* rows,
                           pmf_train_totals* totals) {
    if (const pmf_status st = guard([&] { check_ccd_config(cfg); }); st != PMF_OK) return st;
    // ccd.hpp:39 `workers` -> GPUs: a device group of num_gpus ranks
    return train_common(
        a, cfg->outer_iters, cfg->num_gpus, false, probe, n_probe, W_out, H_out, rows, totals,
        [&](Ctx& c) { ccd_begin(c, cfg); }, [&](Ctx& c, double* s) { ccd_iterate(c, 1, s); });
}

pmf_status pmf_ccd_train(const pmf_ccd_config* cfg, const pmf_matrix_view* a, const pmf_triplet* probe,
                         int64_t n_probe, float* W_out, float* H_out, pmf_iter_row* rows, pmf_train_totals* totals) {
    if (!cfg) {
        g_err = "config is null";
        return PMF_INVALID_ARGUMENT;
    }
    // ccd_train runs one worker whatever `workers` says (ccd.hpp:306-309): one device
    if (cfg->num_gpus < 1) {
        g_err = "workers must be >= 1";
        return PMF_INVALID_ARGUMENT;
    }
    return train_common(
        a, cfg->outer_iters, 1, true, probe, n_probe, W_out, H_out, rows, totals,
        [&](Ctx& c) {
            ccdw_begin(c, cfg);
        },
        [&](Ctx& c, double* s) { ccdw_iterate(c, 1, s); });
}

pmf_status pmf_als_train(const pmf_als_config* cfg, const pmf_matrix_view* a, const pmf_triplet* probe,
                         int64_t n_probe, float* W_out, float* H_out, pmf_iter_row* rows, pmf_train_totals* totals) {
    if (!cfg) {
        g_err = "config is null";
        return PMF_INVALID_ARGUMENT;
    }
    if (cfg->outer_iters < 1 || cfg->k < 1 || !(cfg->lambda > 0.f) || cfg->num_gpus < 1) {
        g_err = cfg->outer_iters < 1 ? "outer_iters must be >= 1"
                : cfg->k < 1         ? "k must be >= 1"
                : cfg->num_gpus < 1  ? "workers must be >= 1"
                                     : "als requires lambda > 0";
        return PMF_INVALID_ARGUMENT;
    }
    return train_common(
        a, cfg->outer_iters, cfg->num_gpus, true, probe, n_probe, W_out, H_out, rows, totals,
        [&](Ctx& c) {
            als_begin(c, cfg);
        },
        [&](Ctx& c, double* s) { als_iterate(c, 1, s); });
}

pmf_status pmf_rmse(const float* W, const float* H, int32_t m, int32_t n, int32_t k, const pmf_triplet* probe,
                    int64_t n_probe, double* out) {
    return guard([&] {
        if (!W || !H || !out) invalid("null buffers");
        if (k < 1) invalid("rank must be >= 1");
        if (n_probe <= 0) invalid("probe set is empty");  // model.hpp:158-159
        for (int64_t x = 0; x < n_probe; ++x) {
            if (probe[x].user < 0 || probe[x].user >= m) throw PmfError(PMF_OUT_OF_RANGE, "user index out of range");
            if (probe[x].item < 0 || probe[x].item >= n) throw PmfError(PMF_OUT_OF_RANGE, "item index out of range");
        }
        ensure_device();
        cudaStream_t s;
        CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        DevMem mem;
        float* dW = mem.alloc<float>(static_cast<size_t>(m) * k, false);
        float* dH = mem.alloc<float>(static_cast<size_t>(n) * k, false);
        auto* dp = mem.alloc<DevTriplet>(n_probe, false);
        double* scratch = mem.alloc<double>(2048);
        double* res = mem.alloc<double>(1);
        CUDA_TRY(cudaMemcpyAsync(dW, W, sizeof(float) * m * k, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(dH, H, sizeof(float) * n * k, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(dp, probe, sizeof(pmf_triplet) * n_probe, cudaMemcpyHostToDevice, s));
        launch_probe_sse(dp, n_probe, FactorView{dW, k, 1}, FactorView{dH, k, 1}, k, scratch, res, s);
        double sse = 0;
        CUDA_TRY(cudaMemcpyAsync(&sse, res, sizeof(double), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        cudaStreamDestroy(s);
        *out = std::sqrt(sse / static_cast<double>(n_probe));  // rmse_finish, model.hpp:149-151
    });
}

pmf_status pmf_objective(const pmf_matrix_view* a, const float* W, const float* H, int32_t k, double lambda,
                         double* out) {
    return guard([&] {
        if (!W || !H || !out) invalid("null buffers");
        if (lambda < 0) invalid("lambda must be >= 0");  // model.hpp:122
        if (k < 1) invalid("rank must be >= 1");
        auto c = make_ctx(a, -1, 0, 1, nullptr);
        alloc_ccd_model(*c, k);
        c->mode = 1;
        set_model(*c, W, H, k, false);
        c->lambda = 0.f;
        double obj = 0;
        metrics(*c, &obj, nullptr, nullptr);
        // recompute with the double lambda given by the caller: obj == loss when lambda == 0
        double h[3];
        CUDA_TRY(cudaMemcpy(h, c->red_out, sizeof(h), cudaMemcpyDeviceToHost));
        *out = h[0] + lambda * (h[1] + h[2]);
    });
}

// ---- stage-level entry points -------------------------------------------------------------------

pmf_status pmf_ccdpp_update_u(const pmf_matrix_view* a, const float* rhat_row, float* u, const float* v,
                              float lambda) {
    return guard([&] {
        if (!rhat_row && a && a->nnz) invalid("null buffers");
        if (!u || !v) invalid("null buffers");
        auto c = make_ctx(a, -1, 0, 1, nullptr);
        alloc_ccd_model(*c, 1);
        put_values(*c, c->hcsr, c->csr.R, rhat_row, c->row_start_local);
        CUDA_TRY(cudaMemcpy(c->vbuf, v, sizeof(float) * c->n, cudaMemcpyHostToDevice));
        SweepOperands op;
        op.gn = c->vbuf;
        op.out = c->ubuf;
        op.lambda = lambda;
        launch_sweep(c->csr, kPlain, true, op, c->stream);
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        CUDA_TRY(cudaMemcpy(u, c->ubuf, sizeof(float) * c->m, cudaMemcpyDeviceToHost));
    });
}

pmf_status pmf_ccdpp_update_v(const pmf_matrix_view* a, const float* rhat_col, const float* u, float* v,
                              float lambda) {
    return guard([&] {
        if (!rhat_col && a && a->nnz) invalid("null buffers");
        if (!u || !v) invalid("null buffers");
        auto c = make_ctx(a, -1, 0, 1, nullptr);
        alloc_ccd_model(*c, 1);
        put_values(*c, c->hcsc, c->csc.R, rhat_col, c->col_start_local);
        CUDA_TRY(cudaMemcpy(c->ubuf, u, sizeof(float) * c->m, cudaMemcpyHostToDevice));
        SweepOperands op;
        op.gn = c->ubuf;
        op.out = c->vbuf;
        op.lambda = lambda;
        launch_sweep(c->csc, kPlain, false, op, c->stream);
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        CUDA_TRY(cudaMemcpy(v, c->vbuf, sizeof(float) * c->n, cudaMemcpyDeviceToHost));
    });
}

// shared body of build_rhat / writeback: runs the fused promote (build) or demote (writeback)
static void residual_stage(const pmf_matrix_view* a, float* r_row, float* r_col, const float* u, const float* v,
                           bool build) {
    if ((!r_row || !r_col) && a && a->nnz) invalid("null buffers");
    if (!u || !v) invalid("null buffers");
    auto c = make_ctx(a, -1, 0, 1, nullptr);
    alloc_ccd_model(*c, 2);  // column 0: (u', v') = 0, column 1: (w, h) = (u, v)
    put_values(*c, c->hcsr, c->csr.R, r_row, c->row_start_local);
    put_values(*c, c->hcsc, c->csc.R, r_col, c->col_start_local);
    float* W0 = c->W;
    float* W1 = c->W + c->ldm;
    float* H0 = c->H;
    float* H1 = c->H + c->ldn;
    CUDA_TRY(cudaMemcpy(build ? W1 : W0, u, sizeof(float) * c->m, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(build ? H1 : H0, v, sizeof(float) * c->n, cudaMemcpyHostToDevice));
    SweepOperands o1, o2;
    o1.oa = W0; o1.ga = H0; o1.ob = W1; o1.gb = H1; o1.gn = H1; o1.out = c->ubuf;
    o2.oa = H0; o2.ga = W0; o2.ob = H1; o2.gb = W1; o2.gn = c->ubuf; o2.out = c->vbuf;
    launch_sweep(c->csr, build ? kPromote : kDemote, true, o1, c->stream);
    launch_sweep(c->csc, build ? kPromote : kDemote, false, o2, c->stream);
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    get_values(*c, c->hcsr, c->csr.R, r_row, c->row_start_local);
    get_values(*c, c->hcsc, c->csc.R, r_col, c->col_start_local);
}

pmf_status pmf_ccdpp_build_rhat(const pmf_matrix_view* a, float* r_row, float* r_col, const float* u,
                                const float* v) {
    return guard([&] { residual_stage(a, r_row, r_col, u, v, true); });
}

pmf_status pmf_ccdpp_writeback(const pmf_matrix_view* a, float* r_row, float* r_col, const float* u,
                               const float* v) {
    return guard([&] { residual_stage(a, r_row, r_col, u, v, false); });
}

pmf_status pmf_als_solve_rows(const pmf_matrix_view* a, int32_t side, const float* opposing, int32_t k, float lambda,
                              float* out) {
    return guard([&] {
        if (side != 0 && side != 1) invalid("side must be 0 (users) or 1 (items)");
        if (!opposing || !out) invalid("null buffers");
        if (k < 1) invalid("k must be >= 1");
        if (lambda < 0.f) invalid("lambda must be >= 0");
        auto c = make_ctx(a, -1, 0, 1, nullptr);
        build_als(*c, a);
        c->k = k;
        float* opp = c->model_mem.alloc<float>(static_cast<size_t>((side == 0 ? c->n : c->m) + 1) * k, false);
        float* dst = c->model_mem.alloc<float>(static_cast<size_t>((side == 0 ? c->m : c->n) + 1) * k);
        als_alloc_partials(*c, k);
        CUDA_TRY(cudaMemcpy(opp, opposing, sizeof(float) * (side == 0 ? c->n : c->m) * k, cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemset(c->d_status, 0, sizeof(int)));
        launch_als_half(side == 0 ? c->als_csr : c->als_csc, opp, side == 0 ? c->n : c->m, dst, 0, k, lambda, false,
                        c->d_counter, c->d_status, c->sm_count, c->stream);
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        int st = 0;
        CUDA_TRY(cudaMemcpy(&st, c->d_status, sizeof(int), cudaMemcpyDeviceToHost));
        if (st == 4) throw PmfError(PMF_NOT_POSITIVE_DEFINITE, "non-positive pivot in an ALS row solve");
        CUDA_TRY(cudaMemcpy(out, dst, sizeof(float) * (side == 0 ? c->m : c->n) * k, cudaMemcpyDeviceToHost));
    });
}

pmf_status pmf_cholesky_solve_batched(int32_t batch, int32_t k, float* a, float* x) {
    return guard([&] {
        if (batch < 0 || k < 1) invalid("invalid batch / order");
        if (batch == 0) return;
        if (!a || !x) invalid("null buffers");
        ensure_device();
        static bool attrs = false;
        if (!attrs) {
            als_set_attributes();
            attrs = true;
        }
        DevMem mem;
        float* da = mem.alloc<float>(static_cast<size_t>(batch) * k * k, false);
        float* dx = mem.alloc<float>(static_cast<size_t>(batch) * k, false);
        int* st = mem.alloc<int>(1);
        CUDA_TRY(cudaMemcpy(da, a, sizeof(float) * batch * k * k, cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(dx, x, sizeof(float) * batch * k, cudaMemcpyHostToDevice));
        if (k > 64) {
            int sms = 148;
            CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
            const int64_t sc = als_big_scratch_floats(k, sms);
            launch_cholesky_big(da, dx, batch, k, st, sms, sc > 0 ? mem.alloc<float>(sc, false) : nullptr, 0);
        } else {
            launch_cholesky_batched(da, dx, batch, k, st, 0);
        }
        CUDA_TRY(cudaDeviceSynchronize());
        int h = 0;
        CUDA_TRY(cudaMemcpy(&h, st, sizeof(int), cudaMemcpyDeviceToHost));
        CUDA_TRY(cudaMemcpy(a, da, sizeof(float) * batch * k * k, cudaMemcpyDeviceToHost));
        CUDA_TRY(cudaMemcpy(x, dx, sizeof(float) * batch * k, cudaMemcpyDeviceToHost));
        if (h == 4) throw PmfError(PMF_NOT_POSITIVE_DEFINITE, "non-positive pivot");
    });
}

}  // extern "C"
