// host_data.cpp -- host-side data entry points of the C-ABI (no CUDA):
//   pmf_matrix_from_triplets  (sparse.hpp:73-149 RatingsMatrix::from_triplets, multithreaded)
//   pmf_synth_ratings         (tests/testutil.hpp:91-132 recipe, parallel per-user streams)
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

// splitmix64: per-user counter-based stream (independent of thread scheduling)
struct SplitMix {
    uint64_t s;
    explicit SplitMix(uint64_t seed) : s(seed) {}
    uint64_t next() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    double unit() { return (static_cast<double>(next() >> 32) + 1.0) * (1.0 / 4294967296.0); }  // (0,1]
    double gaussian() {
        const double u1 = unit(), u2 = unit();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
    }
};

double mt_unit(std::mt19937& g) { return (static_cast<double>(g()) + 1.0) * (1.0 / 4294967296.0); }
double mt_gauss(std::mt19937& g) {
    const double u1 = mt_unit(g), u2 = mt_unit(g);
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
}

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

pmf_status pmf_synth_ratings(int32_t m, int32_t n, int32_t true_rank, int64_t n_train, int64_t n_probe,
                             uint32_t seed, pmf_triplet* out_train, pmf_triplet* out_probe,
                             int64_t* got_train, int64_t* got_probe) {
    if (m < 1 || n < 1 || true_rank < 1 || n_train < 0 || n_probe < 0 || (n_train && !out_train) ||
        (n_probe && !out_probe)) {
        pmfgpu::set_error("synth_ratings: invalid arguments");
        return PMF_INVALID_ARGUMENT;
    }
    const int64_t total = n_train + n_probe;
    if (total > static_cast<int64_t>(m) * n) {
        pmfgpu::set_error("synth_ratings: more ratings than matrix cells");
        return PMF_INVALID_ARGUMENT;
    }
    // planted factors and biases, drawn in the order of testutil.hpp:103-111
    std::mt19937 gen(seed);
    const int r = true_rank;
    const double fscale = 0.45 / std::sqrt(static_cast<double>(r));
    std::vector<double> w(static_cast<size_t>(m) * r), h(static_cast<size_t>(n) * r), bu(m), bi(n);
    for (auto& x : w) x = mt_gauss(gen) * fscale;
    for (auto& x : h) x = mt_gauss(gen) * fscale;
    for (auto& x : bu) x = mt_gauss(gen) * 0.35;
    for (auto& x : bi) x = mt_gauss(gen) * 0.35;
    std::vector<double> cdf(n);
    double acc = 0.0;
    for (int32_t j = 0; j < n; ++j) {
        acc += 1.0 / std::pow(static_cast<double>(j) + 1.0, 0.8);
        cdf[j] = acc;
    }
    for (auto& x : cdf) x /= acc;
    // per-user counts ~ N(mean, mean) (the reference's uniform-user draw), fixed up to `total`
    const double mean = static_cast<double>(total) / m;
    std::vector<int64_t> cnt(m);
    parallel_for(m, [&](int64_t b, int64_t e) {
        for (int64_t i = b; i < e; ++i) {
            SplitMix sm(static_cast<uint64_t>(seed) * 0x100000001B3ull ^ (static_cast<uint64_t>(i) << 20) ^ 0xC0FFEEull);
            const double c = std::round(mean + std::sqrt(std::max(mean, 1e-9)) * sm.gaussian());
            cnt[i] = std::min<int64_t>(n, std::max<int64_t>(0, static_cast<int64_t>(c)));
        }
    });
    int64_t sum = 0;
    for (auto c : cnt) sum += c;
    for (int64_t pass = 0; sum != total && pass < 64; ++pass) {
        const int64_t diff = total - sum;
        const int64_t step = std::max<int64_t>(1, m / std::max<int64_t>(1, std::llabs(diff)));
        for (int64_t i = (pass * 7919) % m, done = 0; done < m && sum != total; ++done, i = (i + step) % m) {
            if (diff > 0 && cnt[i] < n) {
                cnt[i]++;
                sum++;
            } else if (diff < 0 && cnt[i] > 0) {
                cnt[i]--;
                sum--;
            }
        }
    }
    // deterministic per-user probe allocation proportional to the counts
    std::vector<int64_t> pcnt(m), tr_off(m + 1, 0), pr_off(m + 1, 0);
    {
        int64_t cum = 0;
        for (int32_t i = 0; i < m; ++i) {
            const int64_t a = total ? static_cast<int64_t>((static_cast<__int128>(n_probe) * cum) / total) : 0;
            cum += cnt[i];
            const int64_t b = total ? static_cast<int64_t>((static_cast<__int128>(n_probe) * cum) / total) : 0;
            pcnt[i] = std::min(b - a, cnt[i]);
            tr_off[i + 1] = tr_off[i] + cnt[i] - pcnt[i];
            pr_off[i + 1] = pr_off[i] + pcnt[i];
        }
    }
    parallel_for(m, [&](int64_t b, int64_t e) {
        std::vector<uint8_t> used(static_cast<size_t>(n), 0);
        std::vector<int32_t> items;
        std::vector<uint8_t> is_probe;
        for (int64_t i = b; i < e; ++i) {
            SplitMix sm(static_cast<uint64_t>(seed) * 0x9E3779B97F4A7C15ull + static_cast<uint64_t>(i) * 0xD1B54A32D192ED03ull + 1);
            items.clear();
            while (static_cast<int64_t>(items.size()) < cnt[i]) {
                const double u = sm.unit();
                const int32_t j = static_cast<int32_t>(std::lower_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
                const int32_t jj = std::min(j, n - 1);
                if (used[jj]) continue;
                used[jj] = 1;
                items.push_back(jj);
            }
            for (auto j : items) used[j] = 0;
            std::sort(items.begin(), items.end());
            // choose pcnt[i] probe positions (partial Fisher-Yates over positions)
            const int64_t c = static_cast<int64_t>(items.size());
            is_probe.assign(c, 0);
            std::vector<int32_t> pos(c);
            for (int64_t x = 0; x < c; ++x) pos[x] = static_cast<int32_t>(x);
            for (int64_t x = 0; x < pcnt[i]; ++x) {
                const int64_t y = x + static_cast<int64_t>(sm.next() % static_cast<uint64_t>(c - x));
                std::swap(pos[x], pos[y]);
                is_probe[pos[x]] = 1;
            }
            int64_t wt = tr_off[i], wp = pr_off[i];
            for (int64_t x = 0; x < c; ++x) {
                const int32_t j = items[x];
                double score = 3.6 + bu[i] + bi[j] + sm.gaussian() * 0.35;
                for (int t = 0; t < r; ++t)
                    score += w[static_cast<size_t>(i) * r + t] * h[static_cast<size_t>(j) * r + t] / (fscale * fscale) * 0.12;
                score = std::min(5.0, std::max(1.0, std::round(score)));
                pmf_triplet tr{static_cast<int32_t>(i), j, static_cast<float>(score)};
                if (is_probe[x]) out_probe[wp++] = tr;
                else out_train[wt++] = tr;
            }
        }
    });
    if (got_train) *got_train = tr_off[m];
    if (got_probe) *got_probe = pr_off[m];
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
