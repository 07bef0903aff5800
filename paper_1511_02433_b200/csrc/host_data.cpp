// host_data.cpp -- host-side data entry points of the C-ABI (no CUDA):
//   pmf_matrix_from_triplets  (sparse.hpp:73-149 RatingsMatrix::from_triplets, multithreaded)
//   pmf_partition_balanced    (runtime.hpp:91-136)
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <random>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/pmf_gpu.h"
#include "layout.hpp"

namespace pmfgpu {
void set_error(const std::string& msg);
}

using pmfgpu::parallel_for;

namespace {

int hw_threads() { return static_cast<int>(std::max(1u, std::thread::hardware_concurrency())); }

}  // namespace

extern "C" {

pmf_status pmf_partition_balanced(const int64_t* costs, int32_t count, int32_t p, int32_t* bounds) {
    if (p < 1 || count < 0 || (count > 0 && !costs) || !bounds) {
        pmfgpu::set_error("partition_balanced: worker count must be >= 1 and costs non-null");
        return PMF_INVALID_ARGUMENT;
    }
    if (!pmfgpu::partition_balanced(costs, count, p, bounds)) {
        pmfgpu::set_error("partition_balanced: costs must be non-negative");
        return PMF_INVALID_ARGUMENT;
    }
    return PMF_OK;
}

pmf_status pmf_matrix_from_triplets(const pmf_triplet* t, int64_t nnz, int32_t m, int32_t n,
                                    int64_t* row_start, int32_t* col_of, float* val_row,
                                    int64_t* col_start, int32_t* row_of, float* val_col) {
    if (m < 0 || n < 0) {
        pmfgpu::set_error("matrix dimensions must be non-negative");
        return PMF_INVALID_ARGUMENT;
    }
    if (nnz < 0 || (nnz > 0 && !t) || !row_start || !col_start) {
        pmfgpu::set_error("from_triplets: null buffers");
        return PMF_INVALID_ARGUMENT;
    }
    // validation in input order (sparse.hpp:82-92): first offending triplet decides the error
    std::atomic<int64_t> first_bad{std::numeric_limits<int64_t>::max()};
    parallel_for(nnz, [&](int64_t b, int64_t e) {
        for (int64_t x = b; x < e; ++x) {
            const bool bad = t[x].user < 0 || t[x].user >= m || t[x].item < 0 || t[x].item >= n ||
                             !std::isfinite(static_cast<double>(t[x].rating));
            if (bad) {
                int64_t cur = first_bad.load();
                while (x < cur && !first_bad.compare_exchange_weak(cur, x)) {
                }
                break;
            }
        }
    });
    if (first_bad.load() != std::numeric_limits<int64_t>::max()) {
        const pmf_triplet& b = t[first_bad.load()];
        if (b.user < 0 || b.user >= m) {
            pmfgpu::set_error("user index " + std::to_string(b.user) + " out of range for m=" + std::to_string(m));
            return PMF_OUT_OF_RANGE;
        }
        if (b.item < 0 || b.item >= n) {
            pmfgpu::set_error("item index " + std::to_string(b.item) + " out of range for n=" + std::to_string(n));
            return PMF_OUT_OF_RANGE;
        }
        pmfgpu::set_error("non-finite rating at user " + std::to_string(b.user));
        return PMF_INVALID_ARGUMENT;
    }
    const int T = static_cast<int>(std::min<int64_t>(hw_threads(), std::max<int64_t>(1, nnz / 65536)));
    // CSR: per-thread row histograms, stable scatter, then sort each row by column
    std::vector<std::vector<int64_t>> rh(T, std::vector<int64_t>(static_cast<size_t>(m), 0));
    auto chunk = [&](int th, int64_t& b, int64_t& e) {
        b = nnz * th / T;
        e = nnz * (th + 1) / T;
    };
    {
        std::vector<std::thread> ts;
        for (int th = 0; th < T; ++th)
            ts.emplace_back([&, th] {
                int64_t b, e;
                chunk(th, b, e);
                for (int64_t x = b; x < e; ++x) rh[th][t[x].user]++;
            });
        for (auto& x : ts) x.join();
    }
    row_start[0] = 0;
    for (int32_t i = 0; i < m; ++i) {
        int64_t c = 0;
        for (int th = 0; th < T; ++th) {
            const int64_t v = rh[th][i];
            rh[th][i] = row_start[i] + c;  // per-thread fill pointer
            c += v;
        }
        row_start[i + 1] = row_start[i] + c;
    }
    {
        std::vector<std::thread> ts;
        for (int th = 0; th < T; ++th)
            ts.emplace_back([&, th] {
                int64_t b, e;
                chunk(th, b, e);
                for (int64_t x = b; x < e; ++x) {
                    const int64_t p = rh[th][t[x].user]++;
                    col_of[p] = t[x].item;
                    val_row[p] = t[x].rating;
                }
            });
        for (auto& x : ts) x.join();
    }
    rh.clear();
    std::atomic<int64_t> dup_row{-1};
    parallel_for(m, [&](int64_t b, int64_t e) {
        std::vector<std::pair<int32_t, float>> tmp;
        for (int64_t i = b; i < e; ++i) {
            const int64_t s = row_start[i], f = row_start[i + 1];
            bool sorted = true;
            for (int64_t p = s + 1; p < f; ++p)
                if (col_of[p - 1] >= col_of[p]) {
                    sorted = false;
                    break;
                }
            if (!sorted) {
                tmp.clear();
                for (int64_t p = s; p < f; ++p) tmp.emplace_back(col_of[p], val_row[p]);
                std::stable_sort(tmp.begin(), tmp.end(),
                                 [](const auto& a, const auto& c) { return a.first < c.first; });
                for (int64_t p = s; p < f; ++p) {
                    col_of[p] = tmp[p - s].first;
                    val_row[p] = tmp[p - s].second;
                }
            }
            for (int64_t p = s + 1; p < f; ++p)
                if (col_of[p - 1] == col_of[p]) {  // first duplicate in row order (sparse.hpp:127-132)
                    int64_t cur = dup_row.load();
                    while ((cur < 0 || p < cur) && !dup_row.compare_exchange_weak(cur, p)) {
                    }
                    break;
                }
        }
    });
    if (dup_row.load() >= 0) {
        const int64_t p = dup_row.load();
        const int64_t i = std::upper_bound(row_start, row_start + m + 1, p) - row_start - 1;
        pmfgpu::set_error("duplicate rating for user " + std::to_string(i) + ", item " + std::to_string(col_of[p]));
        return PMF_INVALID_ARGUMENT;
    }
    // CSC mirrored from CSR in ascending row order (sparse.hpp:134-147), per-thread row blocks
    const int TR = static_cast<int>(std::min<int64_t>(hw_threads(), std::max<int64_t>(1, m / 1024)));
    std::vector<std::vector<int64_t>> ch(TR, std::vector<int64_t>(static_cast<size_t>(n), 0));
    auto rchunk = [&](int th) { return std::pair<int64_t, int64_t>(int64_t(m) * th / TR, int64_t(m) * (th + 1) / TR); };
    {
        std::vector<std::thread> ts;
        for (int th = 0; th < TR; ++th)
            ts.emplace_back([&, th] {
                auto [b, e] = rchunk(th);
                for (int64_t p = row_start[b]; p < row_start[e]; ++p) ch[th][col_of[p]]++;
            });
        for (auto& x : ts) x.join();
    }
    col_start[0] = 0;
    for (int32_t j = 0; j < n; ++j) {
        int64_t c = 0;
        for (int th = 0; th < TR; ++th) {
            const int64_t v = ch[th][j];
            ch[th][j] = col_start[j] + c;
            c += v;
        }
        col_start[j + 1] = col_start[j] + c;
    }
    {
        std::vector<std::thread> ts;
        for (int th = 0; th < TR; ++th)
            ts.emplace_back([&, th] {
                auto [b, e] = rchunk(th);
                for (int64_t i = b; i < e; ++i)
                    for (int64_t p = row_start[i]; p < row_start[i + 1]; ++p) {
                        const int64_t q = ch[th][col_of[p]]++;
                        row_of[q] = static_cast<int32_t>(i);
                        val_col[q] = val_row[p];
                    }
            });
        for (auto& x : ts) x.join();
    }
    return PMF_OK;
}

}  // extern "C"

// ---- model.hpp:211-295 PMFB model files (single precision) --------------------------------------
// "PMFB", u32 version 1, u32 scalar size, i64 m, i64 n, i64 k, W (m*k), H (n*k), little-endian raw.
pmf_status pmf_save_model(const char* path, const float* W, const float* H, int64_t m, int64_t n, int64_t k) {
    if (!path || m < 0 || n < 0 || k < 1 || (m * k > 0 && !W) || (n * k > 0 && !H)) {
        pmfgpu::set_error("save_model: invalid arguments");
        return PMF_INVALID_ARGUMENT;
    }
    FILE* f = std::fopen(path, "wb");
    if (!f) {
        pmfgpu::set_error(std::string("cannot open ") + path + " for writing");
        return PMF_DATA_ERROR;
    }
    const uint32_t version = 1, scalar = sizeof(float);
    bool ok = std::fwrite("PMFB", 1, 4, f) == 4 && std::fwrite(&version, 4, 1, f) == 1 &&
              std::fwrite(&scalar, 4, 1, f) == 1 && std::fwrite(&m, 8, 1, f) == 1 && std::fwrite(&n, 8, 1, f) == 1 &&
              std::fwrite(&k, 8, 1, f) == 1;
    ok = ok && (m * k == 0 || std::fwrite(W, sizeof(float), static_cast<size_t>(m * k), f) == static_cast<size_t>(m * k));
    ok = ok && (n * k == 0 || std::fwrite(H, sizeof(float), static_cast<size_t>(n * k), f) == static_cast<size_t>(n * k));
    ok = std::fclose(f) == 0 && ok;
    if (!ok) {
        pmfgpu::set_error(std::string("short write to ") + path);
        return PMF_DATA_ERROR;
    }
    return PMF_OK;
}

// Reads the header (W, H == nullptr) or the whole model into caller buffers of the header's size.
pmf_status pmf_load_model(const char* path, int64_t* m, int64_t* n, int64_t* k, float* W, float* H) {
    if (!path || !m || !n || !k) {
        pmfgpu::set_error("load_model: invalid arguments");
        return PMF_INVALID_ARGUMENT;
    }
    FILE* f = std::fopen(path, "rb");
    if (!f) {
        pmfgpu::set_error(std::string("cannot open model file ") + path);
        return PMF_DATA_ERROR;
    }
    auto fail = [&](const std::string& msg) {
        std::fclose(f);
        pmfgpu::set_error(msg);
        return PMF_DATA_ERROR;
    };
    char magic[4];
    uint32_t version = 0, scalar = 0;
    if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "PMFB", 4) != 0)
        return fail(std::string(path) + " is not a model file");
    if (std::fread(&version, 4, 1, f) != 1 || std::fread(&scalar, 4, 1, f) != 1 || version != 1)
        return fail("unsupported model format version");
    if (scalar != sizeof(float)) return fail("model precision does not match requested precision");
    if (std::fread(m, 8, 1, f) != 1 || std::fread(n, 8, 1, f) != 1 || std::fread(k, 8, 1, f) != 1)
        return fail("model file truncated: " + std::string(path));
    if (*m < 0 || *n < 0 || *k < 1) return fail("corrupt model header");
    if (W || H) {
        const size_t wn = static_cast<size_t>(*m * *k), hn = static_cast<size_t>(*n * *k);
        if ((wn && std::fread(W, sizeof(float), wn, f) != wn) || (hn && std::fread(H, sizeof(float), hn, f) != hn))
            return fail("model file truncated: " + std::string(path));
    }
    std::fclose(f);
    return PMF_OK;
}

// ---- io.hpp:240-285 split_dataset (the probe mask; deterministic per seed) ------------------------
// Users with a single rating stay in train, no user loses their last training rating; `ratio` is the
// probe fraction of the eligible entries, drawn by a Fisher-Yates shuffle with std::mt19937(seed)
// and gen() % i exactly as the reference.
pmf_status pmf_split_mask(const int64_t* users, int64_t n, double ratio, uint64_t seed, uint8_t* to_probe,
                          int64_t* n_probe) {
    if (!(ratio > 0.0 && ratio < 1.0)) {
        pmfgpu::set_error("split ratio must be in (0, 1)");
        return PMF_INVALID_ARGUMENT;
    }
    if (n < 0 || (n > 0 && (!users || !to_probe)) || !n_probe || n >= (int64_t(1) << 32)) {
        pmfgpu::set_error("split: invalid arguments");
        return PMF_INVALID_ARGUMENT;
    }
    std::unordered_map<int64_t, int64_t> per_user;
    for (int64_t e = 0; e < n; ++e) per_user[users[e]]++;
    std::vector<uint32_t> eligible;
    eligible.reserve(static_cast<size_t>(n));
    for (uint32_t e = 0; e < static_cast<uint32_t>(n); ++e)
        if (per_user[users[e]] >= 2) eligible.push_back(e);
    std::mt19937 gen(static_cast<std::mt19937::result_type>(seed));
    for (uint32_t i = static_cast<uint32_t>(eligible.size()); i > 1; --i)
        std::swap(eligible[i - 1], eligible[gen() % i]);
    const auto target = static_cast<size_t>(std::llround(ratio * static_cast<double>(eligible.size())));
    std::memset(to_probe, 0, static_cast<size_t>(n));
    std::unordered_map<int64_t, int64_t> left = per_user;
    size_t taken = 0;
    for (const auto e : eligible) {
        if (taken >= target) break;
        auto& remaining = left[users[e]];
        if (remaining <= 1) continue;
        --remaining;
        to_probe[e] = 1;
        ++taken;
    }
    *n_probe = static_cast<int64_t>(taken);
    return PMF_OK;
}
