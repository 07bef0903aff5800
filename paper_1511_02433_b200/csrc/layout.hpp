// layout.hpp -- host-side construction of the device data layouts (C++17, no CUDA).
//
// The reference keeps one CSR + one CSC of the ratings plus cross-links (sparse.hpp:64-216) and
// walks them with per-row loops (ccd.hpp:153-197).  On the B200 each side of the matrix becomes a
// "sweep layout": the entries of every output row (CSR side: users; CSC side: items) are grouped
// by *gather panel* (a contiguous range of the opposing index whose factor values fit in shared
// memory), each (panel, output) segment is padded to a multiple of 4 entries so a lane issues
// 128-bit loads, and indices are stored panel-local (16-bit when the panel is <= 65535 wide).
// Segments are cut into warp work units of at most kUnitMax entries; units of one output that
// land in several panels / chunks produce partial (num, den) sums that a fixed-order finalize
// combines, so every result is deterministic run to run.
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <string>
#include <utility>
#include <vector>

namespace pmfgpu {

constexpr int kUnitMax = 1024;      // entries per warp work unit (multiple of 128)
// Cost model of the CTA partition, in picoseconds of CTA time, fitted by regression on per-CTA sweep
// timings under several partitions (scripts/cta_fit.py over pmf_ctx_debug_sweep_profile, Netflix
// shape).  One layout serves the 14 plain sweeps and the promote sweep of a rank-one step, so the
// model is 14 x plain + 1 x promote.  Per length class (long / medium / short): a cost per group-step
// of each kernel (a warp batch pays for its steps whatever their fill; plain steps 64/32/16 entries,
// promote 256/64/32), per entry and per unit; plus a cost per piece (panel staging and the barrier
// that drains the CTA before the next panel).
struct UnitCost {
    int64_t step_a[3] = {64, 32, 16};
    int64_t per_step_a[3] = {34552, 54236, 0};
    int64_t step_b[3] = {256, 64, 32};
    int64_t per_step_b[3] = {11776, 11471, 0};
    int64_t per_entry[3] = {1235, 203, 2878};
    int64_t per_unit[3] = {63621, 5735, 5628};
    int64_t per_piece = 109820213;
};
UnitCost unit_cost_model();

// Optional allocator for large host buffers, installed by the device library: page-locked blocks
// from a cache, so a layout is filled straight into DMA-able memory and uploaded without a staging
// copy.  alloc returns nullptr to decline (the buffer then comes from operator new).
struct HostAllocHooks {
    void* (*alloc)(size_t bytes) = nullptr;
    void (*free)(void* p, size_t bytes) = nullptr;
    size_t min_bytes = size_t(16) << 20;
};
HostAllocHooks& host_alloc_hooks();

// Uninitialised POD buffer (large layout arrays are filled in parallel; std::vector would first
// value-initialise them serially).
template <class T>
struct PodBuf {
    T* p = nullptr;
    size_t n = 0;
    size_t bytes = 0;
    bool hooked = false;
    PodBuf() = default;
    PodBuf(const PodBuf&) = delete;
    PodBuf& operator=(const PodBuf&) = delete;
    PodBuf(PodBuf&& o) noexcept { swap(o); }
    PodBuf& operator=(PodBuf&& o) noexcept {
        if (this != &o) {
            reset();
            swap(o);
        }
        return *this;
    }
    ~PodBuf() { reset(); }
    void swap(PodBuf& o) noexcept {
        std::swap(p, o.p);
        std::swap(n, o.n);
        std::swap(bytes, o.bytes);
        std::swap(hooked, o.hooked);
    }
    void alloc(size_t count) {
        reset();
        bytes = (count ? count : 1) * sizeof(T);
        const HostAllocHooks& h = host_alloc_hooks();
        if (h.alloc && bytes >= h.min_bytes) p = static_cast<T*>(h.alloc(bytes));
        hooked = p != nullptr;
        if (!p) p = static_cast<T*>(::operator new(bytes));
        n = count;
    }
    void reset() {
        if (p) {
            if (hooked) host_alloc_hooks().free(p, bytes);
            else ::operator delete(p);
        }
        p = nullptr;
        n = bytes = 0;
        hooked = false;
    }
    T* data() { return p; }
    const T* data() const { return p; }
    size_t size() const { return n; }
    bool empty() const { return n == 0; }
    T& operator[](size_t i) { return p[i]; }
    const T& operator[](size_t i) const { return p[i]; }
};

// 16-byte work unit, read with one 128-bit load.
struct Unit {
    uint32_t e0;   // first entry (multiple of 4 for sweep layouts)
    int32_t len;   // entries (padded length for sweep layouts)
    int32_t o;     // local output index
    int32_t slot;  // -1: the only unit of its output (finalizes directly); else partial slot
};

// A CTA's contiguous run of units inside one gather panel.  Units are sorted by length
// (descending); [ub, um) are long units (> kMidLen entries, 8-lane groups), [um, us) medium
// (4-lane groups), [us, ue) short (<= kShortLen, 2-lane groups), so short segments get more units
// in flight per warp.
constexpr int kMidLen = 128;
constexpr int kFinalizeWarpSlots = 32;  // outputs with more partial slots are finalized by a warp
constexpr int kShortLen = 64;
struct Piece {
    int32_t panel;
    int32_t ub, um, us, ue;
    int32_t pad[3];
};

// A warp's work item in a flat layout: units [ua, ub) = vectors [v0, v1) (4 entries each).
struct FlatChunk {
    int32_t ua, v0, v1, ub;
};
constexpr int kFlatChunkVectors = 512;
constexpr int kFlatChunkUnits = 64;  // a warp holds a chunk's unit descriptors in two registers per lane

struct SweepLayout {
    int32_t n_out = 0;        // outputs on this side (local)
    int32_t gat_extent = 0;   // size of the gather index space (padded global space)
    bool smem = true;         // gather vectors staged in shared memory per panel
    bool idx16 = true;        // 16-bit panel-local indices
    int32_t panel_size = 0;   // Pg; smem sentinel local index == Pg
    int32_t n_panels = 0;
    int32_t sentinel = 0;     // index value of padding entries
    std::vector<int32_t> panel_base;  // n_panels + 1
    int64_t n_entries = 0;            // padded entry count (multiple of 4)
    int64_t n_real = 0;
    PodBuf<uint16_t> idx16v;
    PodBuf<int32_t> idx32v;
    PodBuf<float> val;                // padded values (A), padding = 0
    std::vector<Unit> units;
    std::vector<int32_t> unit_panel;
    std::vector<int32_t> unit_real;   // real (unpadded) entries of each unit
    std::vector<Piece> pieces;
    std::vector<int32_t> piece_start; // ctas + 1
    std::vector<int32_t> mo_out;      // outputs whose unit count != 1 (incl. empty outputs)
    std::vector<int32_t> mo_start;    // size mo_out.size()+1, overflow slot ranges (after n_dense)
    int64_t n_dense = 0;              // dense partial slots n_panels * n_out (0: no partials)
    int32_t n_mo_big = 0;             // mo_out[0, n_mo_big): > kFinalizeWarpSlots slots
    int32_t n_slots = 0;
    int32_t ctas = 0;
    double avg_segment = 0.0;
    // Promote (first sweep of a rank-one step): fused into one sweep when its 2 (CSR) / 3 (CSC)
    // staged vectors fit shared memory at this panel width; otherwise a residual pass over
    // rmw_sub sub-panels of width sub_width (2 staged vectors each) followed by a plain sweep.
    bool promote_fused = true;
    int32_t rmw_sub = 1;
    int32_t sub_width = 0;
    std::vector<uint16_t> usplit;     // rmw_sub > 1: per unit rmw_sub+1 entry offsets (0 .. real)
    // Flat (segmented-stream) layout for short segments (flat_kernels.cu): units in memory order
    // and contiguous (segments padded to 4 entries, no alignment gaps); warps stream chunks of
    // whole units; tailbits marks the last 4-entry vector of every unit.
    bool flat = false;
    std::vector<FlatChunk> chunks;    // pieces' chunks: Piece::pad[0..1] = chunk range
    std::vector<uint32_t> tailbits;   // (n_entries / 4) bits + 24 words of slack
    std::vector<int64_t> seg_delta;   // device-built sides: per segment p * n_out + o (see build_sweep_layout)
};

// Shared-memory floats one staged vector of `width` occupies (sentinel slot, 16-byte rounded).
inline int64_t stage_stride_floats(int64_t width) { return ((width + 1) + 3) & ~int64_t(3); }

// Builds one side.  start/idx/val: the reference's CSR (or CSC) arrays restricted to outputs
// [out_begin, out_end) (global offsets into idx/val).  gmap maps a global gather index to the
// padded gather space (nullptr = identity); gat_extent is that space's size.  stage_arrays is the
// number of gather vectors the fused promote sweep stages (2 on the CSR side, 3 on the CSC side);
// panels are as wide as ONE staged vector allows (the 14 plain sweeps of a step stage one), and the
// promote is split when its vectors do not fit (PMF_PANEL_ARRAYS=n sizes panels for n vectors).
//
// Device-resident sides (pmf_ctx_create_from_triplets): with `dev` set, idx / val are not read (they
// may be null) -- the per-(panel, output) segment lengths come from dev->count (computed on the device
// from its CSR / CSC), steps that touch entries are skipped (idx16v / idx32v / val stay empty, usplit
// is left to the device), and seg_delta keeps, per segment (p, o), padded position - source position
// of its entries, for the device fill (layout_fill_device).
struct SegCounter {
    std::function<void(int32_t pg, int32_t np, std::vector<int32_t>& seg_len)> count;
};
SweepLayout build_sweep_layout(const int64_t* start, const int32_t* idx, const float* val,
                               int32_t out_begin, int32_t out_end, const int32_t* gmap,
                               int32_t gat_extent, int stage_arrays, int smem_budget_bytes,
                               int ctas, bool allow_idx16 = true, const SegCounter* dev = nullptr);

// Positions of the original entries of output o (in reference order) inside the padded layout:
// calls fn(o, real_pos_in_output, padded_pos) for every real entry.
void for_each_entry(const SweepLayout& L, const std::function<void(int32_t, int64_t, int64_t)>& fn);

// ALS side: per-output chunks of at most `chunk` entries, unpadded, global (padded-space)
// indices; balanced over `ctas` CTAs like the sweep layouts (no panels).
struct AlsLayout {
    int32_t n_out = 0;
    int64_t n_entries = 0;
    std::vector<int32_t> idx;
    std::vector<float> val;
    std::vector<Unit> units;         // slot -1: single-chunk output (solved in place)
    std::vector<int32_t> mo_out, mo_start;
    int32_t n_slots = 0;
    std::vector<int32_t> empty_out;  // outputs with no entries (solve to 0, als.hpp:51-54)
};

AlsLayout build_als_layout(const int64_t* start, const int32_t* idx, const float* val,
                           int32_t out_begin, int32_t out_end, const int32_t* gmap, int chunk);
// The same without idx / val (they stay empty): units, slots and empty outputs from `start` alone.
AlsLayout build_als_structure(const int64_t* start, int32_t out_begin, int32_t out_end, int chunk);

// runtime.hpp:91-136 partition_balanced (bounds p+1); returns false on invalid input.
bool partition_balanced(const int64_t* costs, int32_t count, int p, int32_t* bounds);

// Simple fork-join helper over [0, n) split into contiguous chunks.
void parallel_for(int64_t n, const std::function<void(int64_t, int64_t)>& fn, int threads = 0);

}  // namespace pmfgpu
