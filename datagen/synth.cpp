// synth.cpp -- synthetic rating corpora for the benchmarks and the large-shape parity tests
// (libpmf_synth.so; host C++, no CUDA).  Shared by both bench arms: the B200 arm and the reference
// arm (which must not load the product library) read the same bytes.
//
// The recipe follows tests/testutil.hpp:91-132 (synth_ratings): true rank r planted factors
// ~N(0,1) * 0.45/sqrt(r), user / item biases ~N(0, 0.35^2), items from a Zipf(0.8) CDF,
// score = 3.6 + b_u + b_i + N(0, 0.35^2) + 0.12 * w.h / fscale^2 rounded and clamped to 1..5,
// (user, item) pairs distinct.  Unlike the reference's sequential generator (one mt19937 stream and
// an unordered_set of keys: 252 s for 99M ratings) every user draws from its own splitmix64 stream
// on a thread pool (~5 s for 253M), the per-user counts are drawn up front (~N(mean, mean) as the
// reference's uniform user draws give, or a power law with user_skew > 0), and the probe is carved
// per user in proportion to its count (the reference's carve_probe, testutil.hpp:136-144, shuffles
// globally).  So the bytes differ from testutil's; both arms of every comparison read these bytes.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_err;

struct Triplet {  // parmf::Triplet<float> (sparse.hpp:20-25), 12 bytes
    int32_t user;
    int32_t item;
    float rating;
};

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

template <class F>
void parallel_for(int64_t n, F&& fn) {
    const int T = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    if (T <= 1 || n < 2 * T) {
        fn(int64_t(0), n);
        return;
    }
    std::vector<std::thread> ts;
    for (int t = 0; t < T; ++t) {
        const int64_t b = n * t / T, e = n * (t + 1) / T;
        ts.emplace_back([=, &fn] { fn(b, e); });
    }
    for (auto& x : ts) x.join();
}

}  // namespace

extern "C" {

const char* dg_last_error() { return g_err.c_str(); }

int dg_synth_ratings(int32_t m, int32_t n, int32_t true_rank, int64_t n_train, int64_t n_probe, uint32_t seed,
                     double user_skew, Triplet* out_train, Triplet* out_probe, int64_t* got_train,
                     int64_t* got_probe) {
    if (m < 1 || n < 1 || true_rank < 1 || n_train < 0 || n_probe < 0 || (n_train && !out_train) ||
        (n_probe && !out_probe)) {
        g_err = "synth_ratings: invalid arguments";
        return 1;
    }
    const int64_t total = n_train + n_probe;
    if (total > static_cast<int64_t>(m) * n) {
        g_err = "synth_ratings: more ratings than matrix cells";
        return 1;
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
    // per-user counts ~ N(mean, mean) (the reference's uniform-user draw), fixed up to `total`; with
    // user_skew > 0 a power law over a seeded permutation of the users instead: the user of activity
    // rank r gets ~ C (r + 1)^-user_skew ratings, capped at n (real rating data is power-law on users
    // as well -- a few rows as long as the item count, a long tail of short ones)
    const double mean = static_cast<double>(total) / m;
    std::vector<int64_t> cnt(m);
    if (user_skew > 0.0) {
        std::vector<int32_t> perm(m);
        for (int32_t i = 0; i < m; ++i) perm[i] = i;
        std::mt19937 pg(seed ^ 0x5eedu);
        for (int32_t i = m - 1; i > 0; --i) std::swap(perm[i], perm[static_cast<int32_t>(pg() % static_cast<uint32_t>(i + 1))]);
        double norm = 0.0;
        for (int32_t r = 0; r < m; ++r) norm += std::pow(r + 1.0, -user_skew);
        for (int32_t r = 0; r < m; ++r)
            cnt[perm[r]] = std::min<int64_t>(n, static_cast<int64_t>(std::llround(total * std::pow(r + 1.0, -user_skew) / norm)));
    } else {
        parallel_for(m, [&](int64_t b, int64_t e) {
            for (int64_t i = b; i < e; ++i) {
                SplitMix sm(static_cast<uint64_t>(seed) * 0x100000001B3ull ^ (static_cast<uint64_t>(i) << 20) ^ 0xC0FFEEull);
                const double c = std::round(mean + std::sqrt(std::max(mean, 1e-9)) * sm.gaussian());
                cnt[i] = std::min<int64_t>(n, std::max<int64_t>(0, static_cast<int64_t>(c)));
            }
        });
    }
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
            if (user_skew > 0.0 && 2 * cnt[i] > n) {
                // dense rows (skewed users): drop n - cnt items uniformly instead of rejection-sampling
                // the Zipf tail
                std::vector<int32_t> all(n);
                for (int32_t j = 0; j < n; ++j) all[j] = j;
                for (int64_t x = 0; x < n - cnt[i]; ++x) {
                    const int64_t y = x + static_cast<int64_t>(sm.next() % static_cast<uint64_t>(n - x));
                    std::swap(all[x], all[y]);
                }
                items.assign(all.begin() + (n - cnt[i]), all.end());
            } else {
                while (static_cast<int64_t>(items.size()) < cnt[i]) {
                    const double u = sm.unit();
                    const int32_t j = static_cast<int32_t>(std::lower_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
                    const int32_t jj = std::min(j, n - 1);
                    if (used[jj]) continue;
                    used[jj] = 1;
                    items.push_back(jj);
                }
                for (auto j : items) used[j] = 0;
            }
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
                Triplet tr{static_cast<int32_t>(i), j, static_cast<float>(score)};
                if (is_probe[x]) out_probe[wp++] = tr;
                else out_train[wt++] = tr;
            }
        }
    });
    if (got_train) *got_train = tr_off[m];
    if (got_probe) *got_probe = pr_off[m];
    return 0;
}

}  // extern "C"
