// layout.cpp -- host construction of the device layouts (see layout.hpp).
#include "layout.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>

namespace pmfgpu {

HostAllocHooks& host_alloc_hooks() {
    static HostAllocHooks h;
    return h;
}


void parallel_for(int64_t n, const std::function<void(int64_t, int64_t)>& fn, int threads) {
    if (n <= 0) return;
    if (threads <= 0) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    threads = static_cast<int>(std::min<int64_t>(threads, std::max<int64_t>(1, n / 4096)));
    if (threads <= 1) {
        fn(0, n);
        return;
    }
    std::vector<std::thread> ts;
    ts.reserve(threads);
    for (int t = 0; t < threads; ++t) {
        const int64_t b = n * t / threads, e = n * (t + 1) / threads;
        ts.emplace_back([&fn, b, e] { fn(b, e); });
    }
    for (auto& t : ts) t.join();
}

UnitCost unit_cost_model() {
    UnitCost m;
    // PMF_UNIT_COST = 19 integers in UnitCost field order (experiments only)
    if (const char* e = std::getenv("PMF_UNIT_COST")) {
        int64_t v[19];
        int n = 0;
        for (const char* p = e; n < 19 && *p;) {
            char* q;
            const int64_t x = std::strtoll(p, &q, 10);
            if (q == p) break;
            v[n++] = x;
            p = *q == ',' ? q + 1 : q;
        }
        if (n == 19)
            for (int c = 0; c < 3; ++c) {
                m.step_a[c] = std::max<int64_t>(1, v[c]);
                m.per_step_a[c] = v[3 + c];
                m.step_b[c] = std::max<int64_t>(1, v[6 + c]);
                m.per_step_b[c] = v[9 + c];
                m.per_entry[c] = v[12 + c];
                m.per_unit[c] = v[15 + c];
                m.per_piece = v[18];
            }
    }
    return m;
}

bool partition_balanced(const int64_t* costs, int32_t count, int p, int32_t* bounds) {
    // runtime.hpp:91-136: binary search on the bottleneck, then a greedy packing sweep
    if (p < 1) return false;
    int64_t lo = 0, total = 0;
    for (int32_t i = 0; i < count; ++i) {
        if (costs[i] < 0) return false;
        lo = std::max(lo, costs[i]);
        total += costs[i];
    }
    auto blocks_needed = [&](int64_t budget) {
        int blocks = 1;
        int64_t cur = 0;
        for (int32_t i = 0; i < count; ++i) {
            if (cur + costs[i] > budget) {
                ++blocks;
                cur = costs[i];
            } else {
                cur += costs[i];
            }
        }
        return blocks;
    };
    int64_t hi = total;
    while (lo < hi) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (blocks_needed(mid) <= p) hi = mid;
        else lo = mid + 1;
    }
    int nb = 0;
    bounds[nb++] = 0;
    int64_t cur = 0;
    for (int32_t i = 0; i < count; ++i) {
        if (cur + costs[i] > lo && nb <= p - 1) {
            bounds[nb++] = i;
            cur = costs[i];
        } else {
            cur += costs[i];
        }
    }
    while (nb < p + 1) bounds[nb++] = count;
    return true;
}

// Segment alignment in entries (a multiple of 4).  Segments of at least kLongSeg real entries start
// (and are padded) on a multiple of PMF_SEG_ALIGN (default 16), so both the residual (4 B) and the
// 16-bit index streams of their units start on a 32-byte sector; shorter segments are padded to 4
// only (a 9-entry segment padded to 16 would stream 78 % padding).  The gap a long segment's
// alignment leaves after its predecessor belongs to no unit and is never read.
static int seg_align() {
    static const int a = [] {
        const char* e = std::getenv("PMF_SEG_ALIGN");
        const int v = e ? std::atoi(e) : 16;
        return v >= 4 && (v & (v - 1)) == 0 ? v : 4;
    }();
    return a;
}
constexpr int64_t kLongSeg = 48;
static inline int64_t seg_alignment(int64_t real) { return real >= kLongSeg ? seg_align() : 4; }
static inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) & ~(a - 1); }

// parallel_for over outputs [0, n_out) with chunks of equal entry counts (start = offsets)
static void parallel_for_outputs(const int64_t* start, int32_t out_begin, int32_t n_out,
                                 const std::function<void(int64_t, int64_t)>& fn) {
    const int T = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    const int64_t total = start[out_begin + n_out] - start[out_begin];
    if (T <= 1 || n_out < 2 * T || total < (int64_t(1) << 16)) {
        fn(0, n_out);
        return;
    }
    const int chunks = 4 * T;
    std::vector<int64_t> cut(chunks + 1, 0);
    for (int c = 1; c < chunks; ++c) {
        const int64_t target = start[out_begin] + total * c / chunks;
        cut[c] = std::lower_bound(start + out_begin, start + out_begin + n_out, target) - (start + out_begin);
        cut[c] = std::max(cut[c], cut[c - 1]);
    }
    cut[chunks] = n_out;
    std::atomic<int> next{0};
    std::vector<std::thread> ts;
    for (int t = 0; t < T; ++t)
        ts.emplace_back([&] {
            for (int c; (c = next++) < chunks;)
                if (cut[c] < cut[c + 1]) fn(cut[c], cut[c + 1]);
        });
    for (auto& t : ts) t.join();
}

SweepLayout build_sweep_layout(const int64_t* start, const int32_t* idx, const float* val,
                               int32_t out_begin, int32_t out_end, const int32_t* gmap,
                               int32_t gat_extent, int stage_arrays, int smem_budget_bytes,
                               int ctas, bool allow_idx16, const SegCounter* dev) {
    static const bool verbose = std::getenv("PMF_VERBOSE") != nullptr;
    auto clk = [] { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
    double tp[8] = {clk()};

    SweepLayout L;
    const int32_t n_out = out_end - out_begin;
    L.n_out = n_out;
    L.gat_extent = gat_extent;
    L.ctas = ctas;
    auto gidx = [&](int64_t e) -> int32_t { return gmap ? gmap[idx[e]] : idx[e]; };

    // ---- 1. gather panels ------------------------------------------------------------------
    // Panel width: a multiple of 4 floats so every panel base is 16-byte aligned for the TMA copy.
    // Preferred: panels narrow enough for the fused promote's `stage_arrays` vectors (one sweep per
    // step reads and rewrites the residual).  When that cuts segments short (a wide gather space:
    // Yahoo-Music), panels as wide as one vector allows, with the promote split into a residual pass
    // + a plain sweep.  When even those segments are a few entries long, gathers from global memory.
    static const int forced_arrays = [] {
        const char* e = std::getenv("PMF_PANEL_ARRAYS");
        return e ? std::max(1, std::min(3, std::atoi(e))) : 0;
    }();
    static const double min_avg = [] {  // wide panels pay off down to short segments
        const char* e = std::getenv("PMF_PANEL_MIN_AVG");
        return e ? std::atof(e) : 8.0;
    }();
    constexpr double kFusedMinAvg = 64.0;
    auto width_cap = [&](int arrays) {
        int64_t w = (smem_budget_bytes / (4 * arrays) - 4) & ~int64_t(3);
        if (allow_idx16) w = std::min<int64_t>(w, 65532);
        return w;
    };
    const int64_t nnz_side = start[out_end] - start[out_begin];
    L.n_real = nnz_side;
    // panel of gather index g, tracked incrementally along an output's ascending indices
    auto count_segments = [&](int32_t pg, int32_t np, std::vector<int32_t>& seg_len) {
        if (dev && np > 1) {
            dev->count(pg, np, seg_len);
            return;
        }
        seg_len.assign(static_cast<size_t>(np) * n_out, 0);
        if (np == 1) {  // one panel: the segments are the outputs
            for (int32_t o = 0; o < n_out; ++o)
                seg_len[o] = static_cast<int32_t>(start[out_begin + o + 1] - start[out_begin + o]);
            return;
        }
        parallel_for_outputs(start, out_begin, n_out, [&](int64_t ob, int64_t oe) {
            for (int64_t o = ob; o < oe; ++o) {
                int32_t p = 0;
                int64_t bound = pg;  // first gather index of panel p+1
                for (int64_t e = start[out_begin + o]; e < start[out_begin + o + 1]; ++e) {
                    const int32_t g = gidx(e);
                    while (g >= bound) {
                        ++p;
                        bound += pg;
                    }
                    seg_len[static_cast<size_t>(p) * n_out + o]++;
                }
            }
        });
    };
    // panels of width pg: segment lengths into seg_len, returns the mean non-empty segment length
    auto try_width = [&](int64_t pg, std::vector<int32_t>& seg_len) {
        const int32_t np = static_cast<int32_t>((static_cast<int64_t>(gat_extent) + pg - 1) / pg);
        count_segments(static_cast<int32_t>(pg), np, seg_len);
        int64_t segs = 0;
        for (auto x : seg_len) segs += x > 0;
        return segs ? static_cast<double>(nnz_side) / segs : 0.0;
    };
    auto use_panels = [&](int64_t pg) {
        L.smem = true;
        L.panel_size = static_cast<int32_t>(pg);
        L.n_panels = static_cast<int32_t>((static_cast<int64_t>(gat_extent) + pg - 1) / pg);
        L.idx16 = allow_idx16;
    };
    std::vector<int32_t> seg_len;
    const int64_t fused_w = width_cap(forced_arrays ? forced_arrays : stage_arrays);
    const int64_t wide_w = width_cap(forced_arrays ? forced_arrays : 1);
    if (gat_extent <= fused_w) {
        L.smem = true;
        L.panel_size = std::max(gat_extent, 1);
        L.n_panels = 1;
        L.idx16 = allow_idx16 && gat_extent <= 65535;
        count_segments(L.panel_size, 1, seg_len);
    } else if (try_width(fused_w, seg_len) >= kFusedMinAvg || fused_w == wide_w) {
        use_panels(fused_w);
    } else if (gat_extent <= wide_w || try_width(wide_w, seg_len) >= min_avg) {
        if (gat_extent <= wide_w) {
            L.smem = true;
            L.panel_size = std::max(gat_extent, 1);
            L.n_panels = 1;
            L.idx16 = allow_idx16 && gat_extent <= 65535;
            count_segments(L.panel_size, 1, seg_len);
        } else {
            use_panels(wide_w);
        }
    } else {  // segments too short for panels: gather from global memory, 32-bit indices
        L.smem = false;
        L.panel_size = gat_extent;
        L.n_panels = 1;
        L.idx16 = false;
        count_segments(std::max(gat_extent, 1), 1, seg_len);
    }
    L.sentinel = L.smem ? L.panel_size : gat_extent;
    L.panel_base.resize(L.n_panels + 1);
    for (int32_t p = 0; p < L.n_panels; ++p)
        L.panel_base[p] = static_cast<int32_t>(static_cast<int64_t>(p) * L.panel_size);
    L.panel_base[L.n_panels] = gat_extent;
    const int32_t pg = L.panel_size;
    const int32_t np = L.n_panels;
    // promote: fused if its vectors fit next to each other, else rmw_sub sub-panel residual passes
    if (L.smem) {
        L.promote_fused = stage_arrays * stage_stride_floats(pg) * 4 <= smem_budget_bytes;
        if (!L.promote_fused) {
            int32_t S = 1;
            for (;; ++S) {
                const int64_t w = round_up((pg + S - 1) / S, 4);
                if (2 * stage_stride_floats(w) * 4 <= smem_budget_bytes + 1024) break;  // + launch slack
            }
            L.rmw_sub = S;
            L.sub_width = static_cast<int32_t>(round_up((pg + S - 1) / S, 4));
        }
    }
    // wide panels (split promote) have short segments: segmented-stream sweeps (PMF_FLAT=0: off)
    static const int flat_env = [] {
        const char* e = std::getenv("PMF_FLAT");
        return e ? std::atoi(e) : -1;
    }();
    L.flat = L.smem && L.idx16 && (flat_env >= 0 ? flat_env != 0 : !L.promote_fused);

    tp[1] = clk();
    // ---- 2. segment offsets (panel-major) ----------------------------------------------------
    std::vector<int64_t> seg_off(seg_len.size() + 1, 0);  // start of segment s; seg_off[S] = end
    std::vector<int64_t> seg_end(seg_len.size(), 0);
    int64_t nonempty = 0;
    {
        int64_t cur = 0;
        for (size_t s = 0; s < seg_len.size(); ++s) {
            const int64_t real = seg_len[s];
            const int64_t a = real > 0 ? (L.flat ? 4 : seg_alignment(real)) : 1;
            seg_off[s] = round_up(cur, a);
            seg_end[s] = seg_off[s] + round_up(real, a);
            cur = seg_end[s];
            nonempty += real > 0;
        }
        seg_off[seg_len.size()] = cur;
    }
    L.n_entries = seg_off.back();
    L.avg_segment = nonempty ? static_cast<double>(nnz_side) / nonempty : 0.0;
    if (L.n_entries >= (int64_t(1) << 32)) throw std::length_error("too many entries for 32-bit units");

    tp[2] = clk();
    if (dev) {  // the device fills the entries: per segment, padded position - source position
        L.seg_delta.assign(seg_len.size(), 0);
        parallel_for_outputs(start, out_begin, n_out, [&](int64_t ob, int64_t oe) {
            for (int64_t o = ob; o < oe; ++o) {
                int64_t src = start[out_begin + o];
                for (int32_t p = 0; p < np; ++p) {
                    const size_t s = static_cast<size_t>(p) * n_out + o;
                    L.seg_delta[s] = seg_off[s] - src;
                    src += seg_len[s];
                }
            }
        });
    }
    // ---- 3. fill entries (padding of each segment written by its owner thread) -----------------
    if (!dev) {
    if (L.idx16) L.idx16v.alloc(L.n_entries);
    else L.idx32v.alloc(L.n_entries);
    L.val.alloc(L.n_entries);
    auto pad = [&](int64_t w, int64_t end) {
        for (; w < end; ++w) {
            if (L.idx16) L.idx16v[w] = static_cast<uint16_t>(L.sentinel);
            else L.idx32v[w] = L.sentinel;
            L.val[w] = 0.0f;
        }
    };
    // alignment gaps between segments
    parallel_for(static_cast<int64_t>(seg_len.size()), [&](int64_t b, int64_t e) {
        for (int64_t s = b; s < e; ++s) pad(s == 0 ? 0 : seg_end[s - 1], seg_off[s]);
    });
    parallel_for_outputs(start, out_begin, n_out, [&](int64_t ob, int64_t oe) {
        for (int64_t o = ob; o < oe; ++o) {
            int32_t cur_p = -1;
            int64_t w = 0, wend = 0;
            int32_t p = 0;
            int64_t bound = pg;
            for (int64_t e = start[out_begin + o]; e < start[out_begin + o + 1]; ++e) {
                const int32_t g = gidx(e);
                while (np > 1 && g >= bound) {
                    ++p;
                    bound += pg;
                }
                if (p != cur_p) {
                    if (cur_p >= 0) pad(w, wend);
                    cur_p = p;
                    const size_t sidx = static_cast<size_t>(p) * n_out + o;
                    w = seg_off[sidx];
                    wend = seg_end[sidx];
                }
                const int32_t local = g - L.panel_base[p];
                if (L.idx16) L.idx16v[w] = static_cast<uint16_t>(local);
                else L.idx32v[w] = local;
                L.val[w] = val[e];
                ++w;
            }
            if (cur_p >= 0) pad(w, wend);
        }
    });
    }  // !dev

    tp[3] = clk();
    // ---- 4. units ----------------------------------------------------------------------------
    std::vector<int32_t> cnt(n_out, 0), ovf(n_out, 0);
    std::vector<uint8_t> chunk0;  // unit is the first chunk of its segment
    {
        size_t n_units = 0;
        for (size_t s = 0; s < seg_len.size(); ++s)
            if (seg_len[s]) n_units += static_cast<size_t>((seg_end[s] - seg_off[s] + kUnitMax - 1) / kUnitMax);
        L.units.reserve(n_units);
        L.unit_panel.reserve(n_units);
        L.unit_real.reserve(n_units);
        chunk0.reserve(n_units);
    }
    for (int32_t p = 0; p < np; ++p)
        for (int32_t o = 0; o < n_out; ++o) {
            const size_t s = static_cast<size_t>(p) * n_out + o;
            const int64_t real = seg_len[s];
            if (real == 0) continue;
            const int64_t padded = seg_end[s] - seg_off[s];
            for (int64_t c = 0; c < padded; c += kUnitMax) {
                const int64_t clen = std::min<int64_t>(kUnitMax, padded - c);
                const int64_t creal = std::max<int64_t>(0, std::min<int64_t>(kUnitMax, real - c));
                L.units.push_back(Unit{static_cast<uint32_t>(seg_off[s] + c),
                                       static_cast<int32_t>(clen), o, -1});
                L.unit_panel.push_back(p);
                L.unit_real.push_back(static_cast<int32_t>(creal));
                chunk0.push_back(c == 0);
                cnt[o]++;
                if (c > 0) ovf[o]++;
            }
        }
    // Partial slots of outputs with several units (or none).  The first chunk of segment (p, o)
    // writes the dense slot p * n_out + o: the units of a warp batch are adjacent outputs of one
    // panel, so their 8-byte partials land in the same sectors (scattered 8-byte stores cost a
    // 32-byte ECC read-modify-write each), and the finalize reads slot p of adjacent outputs
    // coalesced.  Slots of (p, o) without a segment stay 0 (zeroed once).  Further chunks of a
    // long segment go to an overflow region after the dense one, contiguous per output.
    // Finalize order: outputs with many slots first (a warp each), then the rest (a thread each).
    bool any_mo = false;
    for (int32_t o = 0; o < n_out && !any_mo; ++o) any_mo = cnt[o] != 1;
    L.n_dense = any_mo ? static_cast<int64_t>(np) * n_out : 0;
    std::vector<int32_t> ovf_base(n_out, -1);
    L.mo_start.push_back(0);
    for (int pass = 0; pass < 2; ++pass)
        for (int32_t o = 0; o < n_out; ++o) {
            if (cnt[o] == 1 || (cnt[o] > kFinalizeWarpSlots) != (pass == 0)) continue;
            ovf_base[o] = L.mo_start.back();
            L.mo_out.push_back(o);
            L.mo_start.push_back(L.mo_start.back() + ovf[o]);
            if (pass == 0) L.n_mo_big++;
        }
    if (L.n_dense + L.mo_start.back() >= (int64_t(1) << 31)) throw std::length_error("too many partial slots");
    L.n_slots = static_cast<int32_t>(L.n_dense + L.mo_start.back());
    {
        std::vector<int32_t> run(n_out, 0);
        for (size_t x = 0; x < L.units.size(); ++x) {
            Unit& u = L.units[x];
            if (ovf_base[u.o] < 0) continue;
            u.slot = chunk0[x] ? static_cast<int32_t>(static_cast<int64_t>(L.unit_panel[x]) * n_out + u.o)
                               : static_cast<int32_t>(L.n_dense + ovf_base[u.o] + run[u.o]++);
        }
    }

    tp[4] = clk();
    // ---- 5. per-CTA pieces: contiguous unit ranges of equal cost, split at panel changes -----
    const int64_t nu = static_cast<int64_t>(L.units.size());
    const UnitCost cm = unit_cost_model();
    std::vector<int64_t> pre(nu + 1, 0);
    for (int64_t u = 0; u < nu; ++u) {
        const int64_t len = L.units[u].len;
        const int c = len > kMidLen ? 0 : len > kShortLen ? 1 : 2;
        if (L.flat) {  // flat sweeps: per-CTA time ~ 0.82 ns per vector + 1.45 ns per unit (fitted,
                       // scripts/flat_fit.py, Yahoo-Music shape, both sides)
            pre[u + 1] = pre[u] + len / 4 * 820 + 1450;
            continue;
        }
        pre[u + 1] = pre[u] + (len + cm.step_a[c] - 1) / cm.step_a[c] * cm.per_step_a[c] +
                     (len + cm.step_b[c] - 1) / cm.step_b[c] * cm.per_step_b[c] + len * cm.per_entry[c] +
                     cm.per_unit[c] + (u > 0 && L.unit_panel[u] != L.unit_panel[u - 1] ? cm.per_piece : 0);
    }
    L.piece_start.assign(ctas + 1, 0);
    std::vector<int64_t> cta_ub(ctas + 1, 0);
    for (int c = 0; c < ctas; ++c) {
        const int64_t target = pre[nu] * (c + 1) / ctas;
        int64_t ue = std::lower_bound(pre.begin(), pre.end(), target) - pre.begin();
        ue = std::max(cta_ub[c], std::min(ue, nu));
        if (c == ctas - 1) ue = nu;
        cta_ub[c + 1] = ue;
    }
    // the CTAs' unit ranges are disjoint: their pieces are formed on parallel threads (chunk indices
    // are per CTA here and rebased when the lists are joined)
    std::vector<std::vector<Piece>> cta_pieces(ctas);
    std::vector<std::vector<FlatChunk>> cta_chunks(ctas);
    auto form = [&](int c) {
        std::vector<Piece>& lpieces = cta_pieces[c];
        std::vector<FlatChunk>& lchunks = cta_chunks[c];
        const int64_t ub = cta_ub[c], ue = cta_ub[c + 1];
        for (int64_t u = ub; u < ue;) {
            int64_t v = u;
            while (v < ue && L.unit_panel[v] == L.unit_panel[u]) ++v;
            // Long units: longest first inside a piece (the 32/G units a warp takes together then have
            // similar lengths, and the long ones start early: LPT balance).  Medium and short units
            // keep their memory order inside their class, so the units of a warp batch are adjacent
            // and its loads cover one contiguous stretch (length-sorted short units scatter a batch
            // over the whole piece: sector-sized reads with no DRAM locality).  PMF_UNIT_ORDER=len
            // sorts every class by length.
            static const bool sort_all = [] {
                const char* e = std::getenv("PMF_UNIT_ORDER");
                return e && std::string(e) == "len";
            }();
            auto cls = [](int32_t len) { return len > kMidLen ? 0 : len > kShortLen ? 1 : 2; };
            std::vector<int64_t> ord(v - u);
            std::iota(ord.begin(), ord.end(), u);
            std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) {
                const int32_t la = L.units[a].len, lb = L.units[b].len;
                const int ca = cls(la), cb = cls(lb);
                if (L.flat) return false;  // flat layouts stream units in memory order
                if (ca != cb) return ca < cb;
                return (sort_all || ca == 0) ? la > lb : false;
            });
            std::vector<Unit> tu(v - u);
            std::vector<int32_t> tr(v - u);
            for (int64_t x = 0; x < v - u; ++x) {
                tu[x] = L.units[ord[x]];
                tr[x] = L.unit_real[ord[x]];
            }
            std::copy(tu.begin(), tu.end(), L.units.begin() + u);
            std::copy(tr.begin(), tr.end(), L.unit_real.begin() + u);
            int64_t um = u, us = u;
            if (!L.flat) {
                while (um < v && L.units[um].len > kMidLen) ++um;
                us = um;
                while (us < v && L.units[us].len > kShortLen) ++us;
            }
            Piece pz{L.unit_panel[u], static_cast<int32_t>(u), static_cast<int32_t>(um),
                     static_cast<int32_t>(us), static_cast<int32_t>(v), {0, 0, 0}};
            if (L.flat) {  // chunks of whole units: <= kFlatChunkVectors vectors (one unit if longer), <= kFlatChunkUnits units
                pz.pad[0] = static_cast<int32_t>(lchunks.size());
                for (int64_t x = u; x < v;) {
                    const int32_t v0 = static_cast<int32_t>(L.units[x].e0 / 4);
                    int64_t y = x;
                    int32_t v1 = v0;
                    while (y < v && (y == x || ((static_cast<int64_t>(L.units[y].e0) + L.units[y].len) / 4 - v0 <=
                                                        kFlatChunkVectors &&
                                                    y - x < kFlatChunkUnits))) {
                        v1 = static_cast<int32_t>((static_cast<int64_t>(L.units[y].e0) + L.units[y].len) / 4);
                        ++y;
                    }
                    lchunks.push_back(FlatChunk{static_cast<int32_t>(x), v0, v1, static_cast<int32_t>(y)});
                    x = y;
                }
                pz.pad[1] = static_cast<int32_t>(lchunks.size());
            }
            lpieces.push_back(pz);
            u = v;
        }
    };
    {
        const int T = std::max(1, std::min<int>(ctas, static_cast<int>(std::thread::hardware_concurrency())));
        std::vector<std::thread> ts;
        for (int t = 0; t < T; ++t)
            ts.emplace_back([&, t] {
                for (int c = t; c < ctas; c += T) form(c);
            });
        for (auto& t : ts) t.join();
    }
    for (int c = 0; c < ctas; ++c) {
        const int32_t base = static_cast<int32_t>(L.chunks.size());
        for (Piece pz : cta_pieces[c]) {
            if (L.flat) {
                pz.pad[0] += base;
                pz.pad[1] += base;
            }
            L.pieces.push_back(pz);
        }
        L.chunks.insert(L.chunks.end(), cta_chunks[c].begin(), cta_chunks[c].end());
        L.piece_start[c + 1] = static_cast<int32_t>(L.pieces.size());
    }

    if (L.flat) {
        if (L.n_entries / 4 >= (int64_t(1) << 31)) throw std::length_error("too many vectors for a flat layout");
        L.tailbits.assign(static_cast<size_t>(L.n_entries / 4 / 32 + 24), 0u);  // slack: chunk prologues load 18 words
        for (const Unit& u : L.units) {
            const int64_t last = (static_cast<int64_t>(u.e0) + u.len) / 4 - 1;
            L.tailbits[last >> 5] |= 1u << (last & 31);
        }
    }

    tp[5] = clk();
    // ---- 6. sub-panel split points of the residual pass (entries are ascending within a unit) ---
    if (L.rmw_sub > 1 && !dev) {
        const int S = L.rmw_sub;
        L.usplit.assign(static_cast<size_t>(nu) * (S + 1), 0);
        parallel_for(nu, [&](int64_t b, int64_t e) {
            for (int64_t u = b; u < e; ++u) {
                const int64_t e0 = L.units[u].e0;
                const int32_t real = L.unit_real[u];
                uint16_t* sp = &L.usplit[static_cast<size_t>(u) * (S + 1)];
                int32_t x = 0;
                for (int q = 1; q < S; ++q) {
                    const int64_t bound = static_cast<int64_t>(q) * L.sub_width;
                    while (x < real && (L.idx16 ? L.idx16v[e0 + x] : L.idx32v[e0 + x]) < bound) ++x;
                    sp[q] = static_cast<uint16_t>(x);
                }
                sp[S] = static_cast<uint16_t>(real);
            }
        });
    }
    if (verbose)
        std::fprintf(stderr,
                     "[pmf] layout (%d outputs, %lld entries): panels %.3f, offsets %.3f, fill %.3f, units %.3f, "
                     "pieces %.3f, rest %.3f s\n",
                     static_cast<int>(L.n_out), static_cast<long long>(L.n_entries), tp[1] - tp[0], tp[2] - tp[1],
                     tp[3] - tp[2], tp[4] - tp[3], tp[5] - tp[4], clk() - tp[5]);
    return L;
}

void for_each_entry(const SweepLayout& L, const std::function<void(int32_t, int64_t, int64_t)>& fn) {
    // an output's entries, in reference order, are its units sorted by entry offset (panels are
    // laid out in ascending order, chunks of a segment are consecutive)
    std::vector<int64_t> ord(L.units.size());
    std::iota(ord.begin(), ord.end(), 0);
    std::sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) {
        return L.units[a].o != L.units[b].o ? L.units[a].o < L.units[b].o : L.units[a].e0 < L.units[b].e0;
    });
    std::vector<int64_t> run(L.n_out, 0);
    for (int64_t u : ord) {
        const Unit& U = L.units[u];
        for (int32_t x = 0; x < L.unit_real[u]; ++x)
            fn(U.o, run[U.o] + x, static_cast<int64_t>(U.e0) + x);
        run[U.o] += L.unit_real[u];
    }
}

AlsLayout build_als_layout(const int64_t* start, const int32_t* idx, const float* val,
                           int32_t out_begin, int32_t out_end, const int32_t* gmap, int chunk) {
    AlsLayout L = build_als_structure(start, out_begin, out_end, chunk);
    const int64_t base = start[out_begin];
    L.idx.resize(L.n_entries);
    L.val.resize(L.n_entries);
    parallel_for(L.n_entries, [&](int64_t b, int64_t e) {
        for (int64_t x = b; x < e; ++x) {
            L.idx[x] = gmap ? gmap[idx[base + x]] : idx[base + x];
            L.val[x] = val[base + x];
        }
    });
    return L;
}

AlsLayout build_als_structure(const int64_t* start, int32_t out_begin, int32_t out_end, int chunk) {
    AlsLayout L;
    const int32_t n_out = out_end - out_begin;
    L.n_out = n_out;
    const int64_t base = start[out_begin];
    L.n_entries = start[out_end] - base;
    std::vector<int32_t> cnt(n_out, 0);
    for (int32_t o = 0; o < n_out; ++o) {
        const int64_t b = start[out_begin + o] - base, e = start[out_begin + o + 1] - base;
        if (b == e) {
            L.empty_out.push_back(o);
            continue;
        }
        for (int64_t c = b; c < e; c += chunk) {
            L.units.push_back(Unit{static_cast<uint32_t>(c),
                                   static_cast<int32_t>(std::min<int64_t>(chunk, e - c)), o, -1});
            cnt[o]++;
        }
    }
    std::vector<int32_t> slot_base(n_out, -1);
    L.mo_start.push_back(0);
    for (int32_t o = 0; o < n_out; ++o) {
        if (cnt[o] <= 1) continue;
        slot_base[o] = L.mo_start.back();
        L.mo_out.push_back(o);
        L.mo_start.push_back(L.mo_start.back() + cnt[o]);
    }
    L.n_slots = L.mo_start.back();
    std::vector<int32_t> run(n_out, 0);
    for (auto& u : L.units)
        if (slot_base[u.o] >= 0) u.slot = slot_base[u.o] + run[u.o]++;
    // longest units first: warps pull units from a global counter in this order (LPT balance)
    std::stable_sort(L.units.begin(), L.units.end(),
                     [](const Unit& a, const Unit& b) { return a.len > b.len; });
    return L;
}

}  // namespace pmfgpu
